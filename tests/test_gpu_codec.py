"""GPU parity of the sm_100a codec kernels (through the C-ABI) against the CPU oracle:
quantize (A2/A7), dequantize (A5/A6) and the level reduce (A9/A10), bit-exact on
codes, scales, bf16/fp16 outputs and fp32 sums (same order, no FMA), at sizes that
span many warp steps and a ragged tail, at every block size, with the edge-case
blocks of paper_2501_04266_b200.synth, at GPT-layer sizes on sampled blocks, and
past 2^31 elements (64-bit indexing)."""

import ml_dtypes
import numpy as np
import pytest

from oracle import collectives as col
from oracle import quant
from paper_2501_04266_b200 import synth
from tests.gpu_util import assert_bitwise, to_dev, to_host

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def hz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_04266_b200 import hz as mod
    return mod


DT = {"bf16": ml_dtypes.bfloat16, "f16": np.float16, "f32": np.float32}


def _input(n, seed, block, dt):
    x = synth.gradient_like(n, seed, block=block) * np.float32(40.0)   # spans fp16 range too
    return x.astype(DT[dt])


@pytest.mark.parametrize("dt", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("block", [32, 64, 128, 256, 512, 2048])
def test_quantize_parity(hz, dt, bits, block):
    nblocks = 37 * max(1, 256 // block) * 9 + 5          # many warp steps + ragged tail
    n = nblocks * block
    x = _input(n, 10 + bits + block, block, dt)
    codes, scales = hz.quantize(to_dev(x), bits=bits, block=block)
    oc, os_ = quant.quantize(x, bits, block)
    assert_bitwise(to_host(codes), quant.wire_codes(oc, bits), f"codes {dt} int{bits} B={block}")
    assert_bitwise(to_host(scales), os_, f"scales {dt} int{bits} B={block}")


@pytest.mark.parametrize("out", ["bf16", "f16", "f32"])
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("block", [32, 256, 1024])
def test_dequantize_parity(hz, out, bits, block):
    n = (129 * max(1, 256 // block) + 3) * block
    x = _input(n, 20 + bits, block, "f32") / np.float32(40.0)
    oc, os_ = quant.quantize(x, bits, block)
    tdt = {"bf16": torch.bfloat16, "f16": torch.float16, "f32": torch.float32}[out]
    y = hz.dequantize(to_dev(quant.wire_codes(oc, bits)), to_dev(os_), n, bits=bits, block=block,
                      out_dtype=tdt)
    assert_bitwise(to_host(y), quant.dequantize(oc, os_, block, out=out), f"dequant {out} int{bits}")


@pytest.mark.parametrize("g", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("bits_in,bits_out", [(4, 0), (8, 0), (4, 4), (4, 8), (8, 8), (8, 4)])
@pytest.mark.parametrize("block", [64, 256, 512])
def test_reduce_parity(hz, g, bits_in, bits_out, block):
    n = (61 * max(1, 256 // block) + 1) * block
    coded = []
    dev_c, dev_s = [], []
    for p in range(g):
        x = synth.gradient_like(n, 30 + p, block=block)
        c, s = quant.quantize(x, bits_in, block)
        coded.append((c, s))
        dev_c.append(to_dev(quant.wire_codes(c, bits_in)))
        dev_s.append(to_dev(s))
    if bits_out:
        oc, os_ = hz.reduce_chunks(dev_c, dev_s, n, bits_in=bits_in, block=block, bits_out=bits_out)
        wc, ws = col.reduce_coded(coded, block, bits_out=bits_out)
        assert_bitwise(to_host(oc), quant.wire_codes(wc, bits_out), "requant codes")
        assert_bitwise(to_host(os_), ws, "requant scales")
    else:
        out = hz.reduce_chunks(dev_c, dev_s, n, bits_in=bits_in, block=block)
        assert_bitwise(to_host(out), col.reduce_coded(coded, block), "fp32 sum")
        acc0 = synth.gradient_like(n, 99, block=block, specials=False)
        acc = to_dev(acc0.copy())
        hz.reduce_chunks(dev_c, dev_s, n, bits_in=bits_in, block=block, out_f32=acc, accumulate=True)
        assert_bitwise(to_host(acc), col.reduce_coded(coded, block, accum=acc0), "fp32 accumulate")


def test_empty_and_single_block(hz):
    x = torch.zeros(0, dtype=torch.bfloat16, device="cuda")
    c, s = hz.quantize(x, bits=8, block=256)
    assert c.numel() == 0 and s.numel() == 0
    for block in (32, 256, 2048):
        xs = _input(block, 5, block, "bf16")
        c, s = hz.quantize(to_dev(xs), bits=4, block=block)
        oc, os_ = quant.quantize(xs, 4, block)
        assert_bitwise(to_host(c), quant.pack_int4(oc), "single block codes")
        assert_bitwise(to_host(s), os_, "single block scale")


def test_special_blocks_exact(hz):
    """Zero, constant, exact .5 ties (int8 and int4), subnormal-only, tiny-normal,
    just-above-2^-100 and outlier blocks, in bf16 and fp32."""
    sp = np.concatenate(synth.special_blocks(256))
    for dt in ("bf16", "f32"):
        x = sp.astype(DT[dt])
        for bits in (8, 4):
            c, s = hz.quantize(to_dev(x), bits=bits, block=256)
            oc, os_ = quant.quantize(x, bits, 256)
            assert_bitwise(to_host(c), quant.wire_codes(oc, bits), f"special {dt} int{bits}")
            assert_bitwise(to_host(s), os_, f"special scales {dt} int{bits}")
    # the tie blocks really are ties, and RNE picked the even neighbour
    ties = synth.special_blocks(256)[2]
    oc, os_ = quant.quantize(ties, 8, 256)
    prod = ties[1:] * np.float32(8.0)
    assert np.all(prod - np.floor(prod) == 0.5)
    assert np.all(oc[1:] % 2 == 0)


@pytest.mark.parametrize("model", ["gpt1.3b", "neox20b"])
def test_layer_size_sampled(hz, model):
    """Full GPT layer (psi = 12h^2 + 13h, padded) quantized / reduced on the GPU in the
    launch configuration the bench uses; the oracle checks sampled blocks (every 997th
    block plus edge blocks of the 8-way chunk boundaries) - blocks are independent, so
    the check is exact on the sample."""
    hidden = synth.GPT_CONFIGS[model]["hidden"]
    n = synth.layer_numel(hidden)
    B = 256
    unit = 8 * 4 * B
    Np = -(-n // unit) * unit
    gen_seed = 1234
    x = synth.torch_normal(Np, gen_seed, 1e-3, torch.bfloat16, "cuda")
    x[n:] = 0
    codes, scales = hz.quantize(x, bits=4, block=B)
    nb = Np // B
    idx = synth.sample_blocks(nb, [nb * k // 8 for k in range(1, 8)])
    xs = x.view(nb, B)[torch.from_numpy(idx).cuda()].contiguous()
    xs_h = to_host(xs.view(-1))
    oc, os_ = quant.quantize(xs_h, 4, B)
    got_c = to_host(codes.view(nb, B // 2)[torch.from_numpy(idx).cuda()].contiguous().view(-1))
    got_s = to_host(scales[torch.from_numpy(idx).cuda()])
    assert_bitwise(got_c, quant.pack_int4(oc), f"{model} layer codes (sampled)")
    assert_bitwise(got_s, os_, f"{model} layer scales (sampled)")
    # reduce of 2 inputs at full size, sampled
    y = synth.torch_normal(Np, gen_seed + 1, 1e-3, torch.bfloat16, "cuda")
    c2, s2 = hz.quantize(y, bits=4, block=B)
    out = hz.reduce_chunks([codes, c2], [scales, s2], Np, bits_in=4, block=B)
    ys_h = to_host(y.view(nb, B)[torch.from_numpy(idx).cuda()].contiguous().view(-1))
    want = col.reduce_coded([quant.quantize(xs_h, 4, B), quant.quantize(ys_h, 4, B)], B)
    got = to_host(out.view(nb, B)[torch.from_numpy(idx).cuda()].contiguous().view(-1))
    assert_bitwise(got, want, f"{model} layer reduce (sampled)")
    del x, y, codes, c2, out
    torch.cuda.empty_cache()


def test_beyond_int32_indexing(hz):
    """n > 2^31 elements: codes / scales at the far end are still right."""
    B = 256
    n = (1 << 31) + 64 * B
    x = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    tail = synth.gradient_like(128 * B, 77, block=B).astype(ml_dtypes.bfloat16)
    x[n - 128 * B:] = to_dev(tail)
    codes, scales = hz.quantize(x, bits=8, block=B)
    oc, os_ = quant.quantize(tail, 8, B)
    assert_bitwise(to_host(codes[n - 128 * B:]), quant.wire_codes(oc, 8), "codes past 2^31")
    assert_bitwise(to_host(scales[-128:]), os_, "scales past 2^31")
    y = hz.dequantize(codes, scales, n, bits=8, block=B, out_dtype=torch.bfloat16)
    assert_bitwise(to_host(y[n - 128 * B:]), quant.dequantize(oc, os_, B, out="bf16"), "dequant past 2^31")
    assert int(torch.count_nonzero(y[: n - 128 * B])) == 0
    del x, y, codes, scales
    torch.cuda.empty_cache()
