"""Pins for oracle/collectives.py (O7-O9): pass-through mode reduces to the plain
collectives exactly; the quantized gather equals the blockwise codec applied to
the flat tensor whatever the hierarchy; backward == forward; the reduce-scatter
matches an independently written recursive tree sum, stays within the fp32
bound of the fp64 sum, and within the summed quantization bounds; SPEC S:294 and
S:321 worked examples; allreduce+select == reduce-scatter."""

import ml_dtypes
import numpy as np
import pytest

from oracle import collectives as col
from oracle import partition as pm
from oracle import quant
from paper_2501_04266_b200 import synth

CASES = [  # (g, w, s)
    ((2,), 1, 1), ((1,), 1, 1), ((2, 2), 1, 1), ((2, 2), 1, 2), ((2, 2), 2, 1),
    ((2, 2, 2), 1, 1), ((2, 2, 2), 1, 2), ((2, 2, 2), 3, 2), ((2, 2, 2), 3, 0),
    ((2, 4), 1, 1), ((2, 4), 2, 1), ((4, 2), 2, 2), ((2, 2, 2), 0, 0),
]


def _full(Np, seed, block):
    x = synth.params_like(Np, seed, block=block)
    return x.astype(ml_dtypes.bfloat16)


def _primaries(full, g, Np, w):
    out = {}
    for r in range(pm.world_of(g)):
        off, ln = pm.range_at(r, g, Np, w)
        out[r] = full[off:off + ln]
    return out


@pytest.mark.parametrize("g,w,s", CASES)
def test_allgather_passthrough_is_identity(g, w, s):
    B = 4
    Np = pm.padded_numel(1000, g, B)
    full = _full(Np, 1, B)
    outs, sec = col.allgather_forward(_primaries(full, g, Np, w), g, Np, B, w, s, bits=None, out="bf16")
    for r in outs:
        assert np.array_equal(outs[r].view(np.uint16), full.view(np.uint16))
    bwd = col.allgather_backward(sec, g, Np, B, s, bits=None, out="bf16")
    for r in bwd:
        assert np.array_equal(bwd[r].view(np.uint16), full.view(np.uint16))


@pytest.mark.parametrize("g,w,s", CASES)
@pytest.mark.parametrize("bits", [8, 4])
def test_allgather_equals_flat_codec_and_backward(g, w, s, bits):
    B = 16
    Np = pm.padded_numel(3000, g, B)
    full = _full(Np, 2, B)
    ref = quant.dequantize(*quant.quantize(full, bits, B), B, out="bf16").view(np.uint16)
    outs, sec = col.allgather_forward(_primaries(full, g, Np, w), g, Np, B, w, s, bits=bits)
    bwd = col.allgather_backward(sec, g, Np, B, s, bits=bits)
    fc, fs = quant.quantize(full, bits, B)
    for r in range(pm.world_of(g)):
        assert np.array_equal(outs[r].view(np.uint16), ref)        # hierarchy-independent
        assert np.array_equal(bwd[r].view(np.uint16), ref)         # backward == forward
        off, ln = pm.range_at(r, g, Np, s)                         # secondary = range_s slice
        assert np.array_equal(sec[r][0], fc[off:off + ln])
        assert np.array_equal(sec[r][1], fs[off // B:(off + ln) // B])


def _tree_sum(xs, g, level, r):
    """Independent recursive definition: S_0(q) = x_q; S_l(q) = left fold over the level-l
    exchange group of S_{l-1}, ascending digit, fp32 adds."""
    if level == 0:
        return xs[r].astype(np.float32)
    acc = None
    for m in pm.exchange_group(r, g, level):
        v = _tree_sum(xs, g, level - 1, m)
        acc = v.copy() if acc is None else (acc + v).astype(np.float32)
    return acc


@pytest.mark.parametrize("g", [(2,), (2, 2), (2, 2, 2), (2, 4), (4, 2), (3, 2), (1,)])
def test_reduce_scatter_passthrough_tree_sum(g):
    B = 8
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(2000, g, B)
    xs = {r: synth.gradient_like(Np, 100 + r, block=B) for r in range(W)}
    out = col.reduce_scatter(xs, g, Np, B, 1, L, {l: None for l in range(1, L + 1)})
    exact = np.sum(np.stack([xs[r].astype(np.float64) for r in range(W)]), axis=0)
    absum = np.sum(np.stack([np.abs(xs[r].astype(np.float64)) for r in range(W)]), axis=0)
    for r in range(W):
        off, ln = pm.range_at(r, g, Np, L)
        want = _tree_sum(xs, g, L, r)[off:off + ln]
        assert np.array_equal(out[r], want)
        err = np.abs(out[r].astype(np.float64) - exact[off:off + ln])
        assert (err <= (W - 1) * 2.0 ** -24 * absum[off:off + ln] + 1e-45).all()


def test_spec_s294_and_s321():
    g = (2,)
    xs = {0: np.array([1, 2], np.float32), 1: np.array([3, 4], np.float32)}
    out = col.reduce_scatter(xs, g, 2, 1, 1, 1, {1: None})
    assert out[0].tolist() == [4.0] and out[1].tolist() == [6.0]
    xs = {0: np.array([2, 4], np.float32), 1: np.array([6, 8], np.float32)}
    out = col.reduce_scatter(xs, g, 2, 1, 1, 1, {1: 4})
    # member0 ~ 8, member1 ~ 12 within the summed block bounds (scale/2 each)
    assert abs(out[0][0] - 8) <= (2 / 7 + 6 / 7) / 2
    assert abs(out[1][0] - 12) <= (4 / 7 + 8 / 7) / 2


def _bound(trace, g, Np, B, level, q, i):
    """Sum over every quantization event feeding element i of rank q's level-`level`
    partial of (that event's block scale)/2."""
    if level == 0:
        return 0.0
    off, _ = pm.range_at(q, g, Np, level)
    blk = (i - off) // B
    tot = sum(float(sc[blk]) / 2 for sc in trace[(level, q)])
    for m in pm.exchange_group(q, g, level):
        tot += _bound(trace, g, Np, B, level - 1, m, i)
    return tot


@pytest.mark.parametrize("g,bits", [((2, 2, 2), 4), ((2, 2, 2), 8), ((2, 4), 4), ((4,), 4), ((1,), 4)])
def test_reduce_scatter_quantized_error_bound(g, bits):
    B = 32
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(4000, g, B)
    xs = {r: synth.gradient_like(Np, 200 + r, block=B) for r in range(W)}
    trace = {}
    out = col.reduce_scatter(xs, g, Np, B, 1, L, {l: bits for l in range(1, L + 1)}, trace=trace)
    exact = np.sum(np.stack([xs[r].astype(np.float64) for r in range(W)]), axis=0)
    absum = np.sum(np.stack([np.abs(xs[r].astype(np.float64)) for r in range(W)]), axis=0)
    worst = 0.0
    for r in range(W):
        off, ln = pm.range_at(r, g, Np, L)
        for j in range(0, ln, 7):
            i = off + j
            b = _bound(trace, g, Np, B, L, r, i) * (1 + 2.0 ** -20) + W * 2.0 ** -23 * (absum[i] + 2 * _bound(trace, g, Np, B, L, r, i)) + W * L * 2.0 ** -100
            e = abs(float(out[r][j]) - exact[i])
            assert e <= b, (r, i, e, b)
            if b > 0:
                worst = max(worst, e / b)
    assert worst > 0.05          # the bound is not vacuous


def test_world1_reduce_scatter_is_roundtrip():
    B = 256
    Np = pm.padded_numel(5000, (1,), B)
    x = synth.gradient_like(Np, 3, block=B).astype(ml_dtypes.bfloat16)
    out = col.reduce_scatter({0: x}, (1,), Np, B, 1, 1, {1: 4})
    want = quant.dequantize(*quant.quantize(x, 4, B), B)
    assert np.array_equal(out[0], want)


def test_accumulate_and_two_phase():
    """Setting T: levels 1..gl per micro-batch with A <- A + P, then levels gl+1..L once
    per step; with pass-through both phases equal the single-call reduce-scatter exactly
    when the accumulator starts at +0 and GA = 1."""
    g = (2, 2, 2)
    B = 8
    W = 8
    Np = pm.padded_numel(1500, g, B)
    xs = {r: synth.gradient_like(Np, 300 + r, block=B) for r in range(W)}
    nob = {1: None, 2: None, 3: None}
    one = col.reduce_scatter(xs, g, Np, B, 1, 3, nob)
    zero = {r: np.zeros(pm.range_at(r, g, Np, 2)[1], np.float32) for r in range(W)}
    A = col.reduce_scatter(xs, g, Np, B, 1, 2, nob, accum=zero)
    two = col.reduce_scatter(A, g, Np, B, 3, 3, nob)
    for r in range(W):
        assert np.array_equal(one[r], two[r])
    # accumulate really adds
    A2 = col.reduce_scatter(xs, g, Np, B, 1, 2, nob, accum=A)
    for r in range(W):
        assert np.array_equal(A2[r], (A[r] + A[r]).astype(np.float32))


@pytest.mark.parametrize("g,frm", [((2, 2, 2), 3), ((2, 2, 2), 2), ((2, 4), 2), ((2, 2), 1)])
def test_allreduce_select_equals_reduce_scatter(g, frm):
    """P:361 'call Allreduce ... select gradients matching the on-device optimizer states'
    gives the same range_L values as the reduce-scatter over the same levels."""
    B = 8
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(1200, g, B)
    shards = {}
    for r in range(W):
        off, ln = pm.range_at(r, g, Np, frm - 1)
        shards[r] = synth.gradient_like(ln, 400 + r, block=B, specials=False)
    rs = col.reduce_scatter(shards, g, Np, B, frm, L, {l: None for l in range(1, L + 1)})
    ar = col.allreduce_select(shards, g, Np, frm, L)
    for r in range(W):
        assert np.array_equal(rs[r], ar[r])
