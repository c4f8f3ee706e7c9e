"""Virtual-rank harness (test infrastructure, not a product backend): every rank of a
hierarchy is simulated on ONE GPU with its own device buffers; the exchange is a
device copy (torch.cat of the members' slices), and every arithmetic step runs in
the library kernels through the C-ABI (hz_quantize / hz_reduce_chunks /
hz_dequantize), in exactly the order the NCCL engine uses.  The whole 2x2x2
qgZ chain and the qwZ/hpZ gather chain must equal the oracle bit for bit."""

import ml_dtypes
import numpy as np
import pytest

from oracle import collectives as col
from oracle import partition as pm
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


@pytest.mark.parametrize("g", [(2, 2, 2), (2, 4), (4, 2), (8,), (2,), (1,), (3, 2)])
@pytest.mark.parametrize("bits", [4, 8])
def test_virtual_reduce_scatter_chain(hz, g, bits):
    B = 256
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(300_000, g, B)
    grads = {r: synth.gradient_like(Np, 500 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(W)}
    bpl = {l: bits if l == 1 else 4 for l in range(1, L + 1)}
    want = col.reduce_scatter(grads, g, Np, B, 1, L, bpl)

    # level 1 send buffers: each rank quantizes its whole gradient
    send = {r: hz.quantize(to_dev(grads[r]), bits=bpl[1], block=B) for r in range(W)}
    for level in range(1, L + 1):
        b = bpl[level]
        nxt = {}
        for r in range(W):
            d = pm.digits(r, g)[level - 1]
            _, cl = pm.range_at(r, g, Np, level)
            cb = cl * b // 8
            cs_ = cl // B
            members = pm.exchange_group(r, g, level)
            codes = [send[m][0][d * cb:(d + 1) * cb].clone() for m in members]   # "receive"
            scales = [send[m][1][d * cs_:(d + 1) * cs_].clone() for m in members]
            if level < L:
                nxt[r] = hz.reduce_chunks(codes, scales, cl, bits_in=b, block=B, bits_out=bpl[level + 1])
            else:
                nxt[r] = hz.reduce_chunks(codes, scales, cl, bits_in=b, block=B)
        send = nxt
    for r in range(W):
        assert_bitwise(to_host(send[r]), want[r], f"rank {r} shard")


@pytest.mark.parametrize("g,w,s", [((2, 2, 2), 1, 1), ((2, 2, 2), 3, 2), ((2, 2, 2), 1, 3), ((2, 4), 2, 1)])
def test_virtual_allgather_chain(hz, g, w, s):
    B = 256
    W = pm.world_of(g)
    Np = pm.padded_numel(200_000, g, B)
    full = synth.params_like(Np, 3, block=B).astype(ml_dtypes.bfloat16)
    prim = {}
    for r in range(W):
        off, ln = pm.range_at(r, g, Np, w)
        prim[r] = full[off:off + ln]
    want, want_sec = col.allgather_forward(prim, g, Np, B, w, s, bits=8)
    held = {r: hz.quantize(to_dev(prim[r]), bits=8, block=B) for r in range(W)}
    for level in range(w, 0, -1):
        held = {r: (torch.cat([held[m][0] for m in pm.exchange_group(r, g, level)]),
                    torch.cat([held[m][1] for m in pm.exchange_group(r, g, level)])) for r in range(W)}
    for r in range(W):
        out = hz.dequantize(held[r][0], held[r][1], Np, bits=8, block=B, out_dtype=torch.bfloat16)
        assert_bitwise(to_host(out), want[r], f"rank {r} gathered layer")
        off, ln = pm.range_at(r, g, Np, s)
        assert_bitwise(to_host(held[r][0][off:off + ln]), quant.wire_codes(want_sec[r][0], 8), "secondary codes")
