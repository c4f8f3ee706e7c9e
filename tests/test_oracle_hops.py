"""Pins for oracle.collectives.reduce_scatter_hops (the qgZ hop grouping, "1-hop
all-to-all based Reduce-scatter", reading R15) and for the summation order of the
quantized branch of reduce_coded (R10, g >= 3).

Each pin ties the function to something other than itself:
  * one hop per level is the per-level reduce_scatter (pinned in
    test_oracle_collectives.py) bit for bit;
  * one hop over every level is the single-level hierarchy (W,) reduce-scatter, re-indexed
    by global position (a different ownership map, the same sum per element);
  * pass-through hops equal an fp32 sum over the hop groups written here from the
    definition (nested ascending-rank sums), bit for bit;
  * quantized hops stay within the summed per-event quantization bounds, which shrink
    with fewer hops (one quantization per hop and contributor);
  * hand-computed order examples: the fp32 sum of 2^24, 1, 1 (and -2^24) depends on the
    order of the adds, and only ascending member order gives the stated values.
"""

import ml_dtypes
import numpy as np
import pytest

from oracle import collectives as col
from oracle import partition as pm
from oracle import quant
from paper_2501_04266_b200 import synth

GROUPINGS = [  # (g, hops)
    ((2, 2, 2), [(1, 2), (3, 3)]), ((2, 2, 2), [(1, 1), (2, 3)]), ((2, 2, 2), [(1, 3)]),
    ((2, 4), [(1, 2)]), ((4, 2), [(1, 2)]), ((2, 2), [(1, 2)]), ((2, 1, 2), [(1, 2), (3, 3)]),
]


def _grads(g, Np, B, seed, dtype=ml_dtypes.bfloat16):
    return {r: synth.gradient_like(Np, seed + r, block=B).astype(dtype) for r in range(pm.world_of(g))}


def _flat(out, g, Np, level):
    f = np.full(Np, np.nan, np.float32)
    for r, v in out.items():
        off, ln = pm.range_at(r, g, Np, level)
        f[off:off + ln] = v
    return f


@pytest.mark.parametrize("g", [(2, 2, 2), (2, 4), (4, 2), (2,)])
@pytest.mark.parametrize("bits", [4, 8, None])
def test_one_hop_per_level_is_reduce_scatter(g, bits):
    B = 32
    L = len(g)
    Np = pm.padded_numel(5000, g, B)
    xs = _grads(g, Np, B, 100)
    a = col.reduce_scatter(xs, g, Np, B, 1, L, {l: bits for l in range(1, L + 1)})
    b = col.reduce_scatter_hops(xs, g, Np, B, [(l, l) for l in range(1, L + 1)], bits)
    for r in a:
        assert np.array_equal(a[r].view(np.uint32), b[r].view(np.uint32))


@pytest.mark.parametrize("g", [(2, 2, 2), (2, 4), (4, 2), (2, 2)])
@pytest.mark.parametrize("bits", [4, 8])
def test_single_hop_is_flat_hierarchy(g, bits):
    """All levels in one hop = the 1-hop all-to-all of a one-level hierarchy of the
    same world: identical per-element sums (every rank, ascending rank order), only the
    owner of each chunk differs (digit-reversed vs rank order)."""
    B = 32
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(6000, g, B)
    xs = _grads(g, Np, B, 200)
    a = _flat(col.reduce_scatter_hops(xs, g, Np, B, [(1, L)], bits), g, Np, L)
    b = _flat(col.reduce_scatter(xs, (W,), Np, B, 1, 1, {1: bits}), (W,), Np, 1)
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def _nested_sum(xs, g, hops, i):
    """fp32 value at global element i of the pass-through hop reduce-scatter, from the
    definition: the hop-k partial of rank r at i is the ascending-rank fp32 sum of the
    hop-(k-1) partials of the members of r's hop-k group."""
    W = pm.world_of(g)

    def partial(k, r):
        if k < 0:
            return np.float32(xs[r][i])
        a, b = hops[k]
        acc = None
        for m in range(W):
            if all(pm.digits(m, g)[j] == pm.digits(r, g)[j] for j in range(len(g)) if not a - 1 <= j <= b - 1):
                v = partial(k - 1, m)
                acc = v if acc is None else np.float32(acc + v)
        return acc

    owner = next(r for r in range(W)
                 if pm.range_at(r, g, len(xs[0]), len(g))[0] <= i < sum(pm.range_at(r, g, len(xs[0]), len(g))))
    return partial(len(hops) - 1, owner)


@pytest.mark.parametrize("g,hops", GROUPINGS)
def test_passthrough_equals_nested_sums(g, hops):
    B = 8
    L = len(g)
    Np = pm.padded_numel(700, g, B)
    xs = {r: synth.gradient_like(Np, 300 + r, block=B, specials=False) for r in range(pm.world_of(g))}
    out = _flat(col.reduce_scatter_hops(xs, g, Np, B, hops, None), g, Np, L)
    for i in range(0, Np, 13):
        assert out[i].view(np.uint32) == np.float32(_nested_sum(xs, g, hops, i)).view(np.uint32), i


def _bound_hops(trace, g, Np, B, hops, k, q, i):
    if k < 0:
        return 0.0
    a, b = hops[k]
    off, _ = pm.range_at(q, g, Np, b)
    blk = (i - off) // B
    tot = sum(float(sc[blk]) / 2 for sc in trace[(b, q)])
    for m in pm.hop_group(q, g, a, b):
        tot += _bound_hops(trace, g, Np, B, hops, k - 1, m, i)
    return tot


@pytest.mark.parametrize("g,hops", GROUPINGS)
def test_quantized_hops_error_bound(g, hops):
    B = 32
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(3000, g, B)
    xs = {r: synth.gradient_like(Np, 500 + r, block=B) for r in range(W)}
    trace = {}
    out = _flat(col.reduce_scatter_hops(xs, g, Np, B, hops, 4, trace=trace), g, Np, L)
    exact = np.sum(np.stack([xs[r].astype(np.float64) for r in range(W)]), axis=0)
    absum = np.sum(np.stack([np.abs(xs[r].astype(np.float64)) for r in range(W)]), axis=0)
    worst = 0.0
    for i in range(0, Np, 5):
        owner = next(r for r in range(W) if pm.range_at(r, g, Np, L)[0] <= i < sum(pm.range_at(r, g, Np, L)))
        qb = _bound_hops(trace, g, Np, B, hops, len(hops) - 1, owner, i)
        b = qb * (1 + 2.0 ** -20) + W * 2.0 ** -23 * (absum[i] + 2 * qb) + W * L * 2.0 ** -100
        e = abs(float(out[i]) - exact[i])
        assert e <= b, (i, e, b)
        if b > 0:
            worst = max(worst, e / b)
    assert worst > 0.05


def test_fewer_hops_fewer_quantizations():
    """requantizing at every hop accumulates error; merging levels 1..2 into one
    hop removes one requantization, merging all three removes two.  Mean |error| against
    the exact fp64 sum on 2x2x2, int4: 3 hops > 2 hops > 1 hop."""
    g = (2, 2, 2)
    B = 256
    W = 8
    Np = pm.padded_numel(1 << 16, g, B)
    xs = {r: synth.gradient_like(Np, 700 + r, block=B) for r in range(W)}
    exact = np.sum(np.stack([xs[r].astype(np.float64) for r in range(W)]), axis=0)
    err = []
    for hops in ([(1, 1), (2, 2), (3, 3)], [(1, 2), (3, 3)], [(1, 3)]):
        out = _flat(col.reduce_scatter_hops(xs, g, Np, B, hops, 4), g, Np, 3)
        err.append(float(np.mean(np.abs(out - exact))))
    assert err[0] > err[1] > err[2], err


# ----------------------------------------------------- reduce_coded summation order
def _coded(vals, bits, B=32):
    """One block per member: element 0 = code k * scale s (exact power-of-two scales),
    the other elements code 0."""
    out = []
    for code, scale in vals:
        c = np.zeros(B, np.int8)
        c[0] = code
        out.append((c, np.array([scale], np.float32)))
    return out


@pytest.mark.parametrize("bits,big", [(8, (64, 2.0 ** 18)), (4, (4, 2.0 ** 22))])
def test_reduce_coded_order_g3(bits, big):
    """x_hat = [2^24, 1, 1] (exact products).  Ascending order: fl(fl(2^24 + 1) + 1) =
    2^24 (each +1 is a tie that rounds to even); any order that adds the two ones first
    gives 2^24 + 2.  Hand-computed: 16777216."""
    coded = _coded([big, (1, 1.0), (1, 1.0)], bits)
    out = col.reduce_coded(coded, 32)
    assert out[0] == np.float32(16777216.0)
    assert np.all(out[1:] == 0)
    # the other orders really differ (the example is sensitive to the order)
    assert np.float32(np.float32(1 + 1) + np.float32(2 ** 24)) == np.float32(16777218.0)


@pytest.mark.parametrize("bits,big", [(8, (64, 2.0 ** 18)), (4, (4, 2.0 ** 22))])
def test_reduce_coded_order_g4_and_requant(bits, big):
    """x_hat = [2^24, 1, 1, -2^24]: ascending order gives ((2^24 + 1) + 1) - 2^24 = 0;
    reversed order gives ((-2^24 + 1) + 1) + 2^24 = 2, as does (m0 + m3) + m1 + m2.
    The requantized branch then sees a zero block: scale 0, codes 0 (R3)."""
    neg = (-big[0], big[1])
    coded = _coded([big, (1, 1.0), (1, 1.0), neg], bits)
    out = col.reduce_coded(coded, 32)
    assert out[0] == np.float32(0.0)
    rev = col.reduce_coded(coded[::-1], 32)
    assert rev[0] == np.float32(2.0)
    codes, scales = col.reduce_coded(coded, 32, bits_out=bits)
    assert scales[0] == 0.0 and np.all(np.asarray(codes) == 0)
