"""Out-of-bounds and input-integrity checks for the codec kernels (the GPU pool has
no compute-sanitizer): every output lives inside sentinel bands (tests.gpu_util.Guarded)
that must survive the call, every input must be bit-identical afterwards, and the
outputs must still match the oracle.  Sizes are ragged in the grid-stride sense (one
block, a partial warp step, a partial CTA step, several CTA waves plus a tail) and the
views sit at 16-byte (not 4 KB) offsets, the weakest alignment the ABI accepts."""

import ml_dtypes
import numpy as np
import pytest

from oracle import collectives as col
from oracle import quant
from paper_2501_04266_b200 import synth
from tests.gpu_util import Guarded, assert_bitwise, assert_unchanged, to_dev, to_host

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

NBLOCKS = [1, 3, 33, 257, 148 * 8 * 8 + 13]


@pytest.fixture(scope="module")
def hz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_04266_b200 import hz as mod
    return mod


def _guarded_input(x, dtype, guard=16):
    g = Guarded(x.size, dtype, guard_bytes=guard)
    g.t.copy_(to_dev(x))
    return g


@pytest.mark.parametrize("nb", NBLOCKS)
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("block", [32, 256, 2048])
def test_quantize_bounds(hz, nb, bits, block):
    n = nb * block
    x = synth.gradient_like(n, 5 + nb, block=block).astype(ml_dtypes.bfloat16)
    gx = _guarded_input(x, torch.bfloat16)
    gc = Guarded(n * bits // 8, torch.uint8, guard_bytes=16)
    gs = Guarded(n // block, torch.float32, guard_bytes=16)
    hz.quantize(gx.t, bits, block, gc.t, gs.t)
    torch.cuda.synchronize()
    oc, os_ = quant.quantize(x, bits, block)
    assert_bitwise(to_host(gc.t), quant.wire_codes(oc, bits), "codes")
    assert_bitwise(to_host(gs.t), os_, "scales")
    gc.check("codes")
    gs.check("scales")
    gx.check("input")
    assert_unchanged(gx.t, x, "x")


@pytest.mark.parametrize("nb", NBLOCKS)
@pytest.mark.parametrize("bits", [8, 4])
@pytest.mark.parametrize("block", [32, 256, 2048])
@pytest.mark.parametrize("out", ["bf16", "f32"])
def test_dequantize_bounds(hz, nb, bits, block, out):
    n = nb * block
    x = synth.params_like(n, 9 + nb, block=block)
    oc, os_ = quant.quantize(x, bits, block)
    wc = quant.wire_codes(oc, bits)
    gc = _guarded_input(wc, torch.uint8)
    gs = _guarded_input(os_, torch.float32)
    tdt = {"bf16": torch.bfloat16, "f32": torch.float32}[out]
    gy = Guarded(n, tdt, guard_bytes=16)
    hz.dequantize(gc.t, gs.t, n, bits, block, out=gy.t)
    torch.cuda.synchronize()
    assert_bitwise(to_host(gy.t), quant.dequantize(oc, os_, block, out=out), "dequantized")
    gy.check("output")
    assert_unchanged(gc.t, wc, "codes")
    assert_unchanged(gs.t, os_, "scales")


@pytest.mark.parametrize("nb", NBLOCKS)
@pytest.mark.parametrize("g", [1, 2, 4])
@pytest.mark.parametrize("bits_out", [0, 4, 8])
def test_reduce_bounds(hz, nb, g, bits_out):
    block, bits_in = 256, 4
    n = nb * block
    coded, dc, ds = [], [], []
    for p in range(g):
        c, s = quant.quantize(synth.gradient_like(n, 40 + p, block=block), bits_in, block)
        coded.append((c, s))
        dc.append(_guarded_input(quant.wire_codes(c, bits_in), torch.uint8))
        ds.append(_guarded_input(s, torch.float32))
    if bits_out:
        goc = Guarded(n * bits_out // 8, torch.uint8, guard_bytes=16)
        gos = Guarded(n // block, torch.float32, guard_bytes=16)
        hz.reduce_chunks([d.t for d in dc], [d.t for d in ds], n, bits_in, block, bits_out=bits_out,
                         out_codes=goc.t, out_scales=gos.t)
        torch.cuda.synchronize()
        wc, ws = col.reduce_coded(coded, block, bits_out=bits_out)
        assert_bitwise(to_host(goc.t), quant.wire_codes(wc, bits_out), "requant codes")
        assert_bitwise(to_host(gos.t), ws, "requant scales")
        goc.check("out codes")
        gos.check("out scales")
    else:
        gy = Guarded(n, torch.float32, guard_bytes=16)
        hz.reduce_chunks([d.t for d in dc], [d.t for d in ds], n, bits_in, block, out_f32=gy.t)
        torch.cuda.synchronize()
        assert_bitwise(to_host(gy.t), col.reduce_coded(coded, block), "fp32 sum")
        gy.check("out f32")
    for p in range(g):
        assert_unchanged(dc[p].t, quant.wire_codes(coded[p][0], bits_in), f"codes[{p}]")
        assert_unchanged(ds[p].t, coded[p][1], f"scales[{p}]")


def test_misaligned_pointer_rejected(hz):
    x = torch.zeros(256 + 8, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(hz.HZError):
        hz.quantize(x[1:257], 8, 256)
