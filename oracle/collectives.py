"""O7-O9: the hierarchical qwZ/hpZ all-gather and qgZ reduce-scatter, all ranks
simulated in one process (sequential program, logical concurrency).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper passages followed step by step:
  * forward: "the training orchestration conducts gathering on parameters
    across primary weight shards before each forward pass and across secondary
    partitions before the backward pass"; weights quantized to INT8
    before the all-gather, "reducing the volume from M to 0.5M";
    a quantized secondary copy is kept after the forward gather (P:120, P:275,
    Table V).
  * gradients: "quantizes the FP16 gradients to INT4 ... All-to-All-based
    Reduce-scatter", "1-hop all-to-all based Reduce-scatter" inside the
    node, then "Allreduce on local gradients stored among nodes" and
    "select gradients matching the on-device optimizer states".
  * at each level a rank moves only the shard it owns (north_star).

Readings: R9 every rank, the owner included, dequantizes from
the codes; R10 reduction order ascending in the level digit, level 1 first,
fp32, one rounding per add (no FMA); R11 a rank also quantizes its own chunk;
R12 the cross-level step is a reduce-scatter by default, allreduce+select is
kept as an equivalence check (``allreduce_select``).

``bits=None`` selects an unquantized pass-through exchange (test mode used by
the pins: it must reduce to the plain collective exactly).
"""

import ml_dtypes
import numpy as np

from . import quant
from .partition import world_of, digits, range_at, exchange_group, hop_group


class Ledger:
    """Per-rank received bytes, keyed (phase, level): [payload, metadata]."""

    def __init__(self):
        self.rows = {}

    def add(self, rank, phase, level, payload, meta):
        key = (rank, phase, level)
        p, m = self.rows.get(key, (0, 0))
        self.rows[key] = (p + payload, m + meta)

    def per_rank(self, rank, phase):
        p = sum(v[0] for k, v in self.rows.items() if k[0] == rank and k[1] == phase)
        m = sum(v[1] for k, v in self.rows.items() if k[0] == rank and k[1] == phase)
        return p, m

    def level(self, rank, phase, level):
        return self.rows.get((rank, phase, level), (0, 0))


def _quantize_or_pass(x, bits, block):
    if bits is None:
        return (quant.to_f32(x), None)
    return quant.quantize(x, bits, block)


def _concat(parts, bits):
    codes = np.concatenate([p[0] for p in parts])
    scales = None if bits is None else np.concatenate([p[1] for p in parts])
    return (codes, scales)


def _materialise(held, bits, block, out):
    codes, scales = held
    if bits is None:
        return codes.astype(np.float32) if out == "f32" else codes.astype(ml_dtypes.bfloat16)
    return quant.dequantize(codes, scales, block, out=out)


def _gather_levels(held, g, Np, block, bits, top, bottom, phase, ledger, keep_at=None):
    """For level = top..bottom (descending): concatenate, within each level-l exchange
    group, the members' held codes/scales in ascending d_l (O7).  ``keep_at`` = s:
    snapshot the buffer that covers range_s (hpZ secondary)."""
    W = world_of(g)
    kept = None
    for level in range(top, bottom - 1, -1):
        new = {}
        for r in range(W):
            members = exchange_group(r, g, level)
            new[r] = _concat([held[m] for m in members], bits)
            if ledger is not None:
                _, ln = range_at(r, g, Np, level)
                k = len(members) - 1
                payload = k * ln * (4 if bits is None else bits) // (1 if bits is None else 8)
                meta = 0 if bits is None else k * (ln // block) * 4
                ledger.add(r, phase, level, payload, meta)
        held = new
        if keep_at is not None and level - 1 == keep_at:
            kept = dict(held)
    return held, kept


def allgather_forward(primaries, g, Np, block, w, s, bits=8, out="bf16", ledger=None):
    """O7: forward qwZ all-gather with hpZ secondary retention.

    primaries[r]: rank r's primary shard (bf16/fp32), covering range_w(r).
    Returns (full[r] over [0, Np), secondary[r] = (codes, scales) over range_s(r)).
    """
    W = world_of(g)
    held = {}
    for r in range(W):
        _, ln = range_at(r, g, Np, w)
        if len(primaries[r]) != ln:
            raise ValueError("primary shard length != len_w")
        held[r] = _quantize_or_pass(primaries[r], bits, block)          # A2
    secondary = None
    if s >= w:                                                          # A4, s >= w
        secondary = {}
        for r in range(W):
            offw, _ = range_at(r, g, Np, w)
            offs, lns = range_at(r, g, Np, s)
            a = offs - offw
            c = held[r][0][a:a + lns]
            sc = None if bits is None else held[r][1][a // block:(a + lns) // block]
            secondary[r] = (c.copy(), None if sc is None else sc.copy())
    held, kept = _gather_levels(held, g, Np, block, bits, w, 1, "forward_ag", ledger,
                                keep_at=s if s < w else None)           # A3
    if s < w:                                                           # A4, s < w
        secondary = kept
    full = {r: _materialise(held[r], bits, block, out) for r in range(W)}   # A5
    return full, secondary


def allgather_backward(secondary, g, Np, block, s, bits=8, out="bf16", ledger=None):
    """O8: backward all-gather from the hpZ secondary over levels s..1, no requantization (A6)."""
    W = world_of(g)
    held = {r: secondary[r] for r in range(W)}
    held, _ = _gather_levels(held, g, Np, block, bits, s, 1, "backward_ag", ledger)
    return {r: _materialise(held[r], bits, block, out) for r in range(W)}


def reduce_coded(coded, block, bits_out=None, accum=None):
    """A9, one level step for one rank: dequantize the received chunks (list over the
    sending members in ascending level digit of (codes, scales)) and sum them in that
    order in fp32, one rounding per add (R10).  Then either requantize the sum for the
    next level (bits_out 4/8, returns (codes, scales)), or return the fp32 sum,
    added to ``accum`` when given (A10: A = fl(A + P))."""
    acc = None
    for codes, scales in coded:
        xh = quant.dequantize(codes, scales, block, out="f32")
        acc = xh.copy() if acc is None else (acc + xh).astype(np.float32)
    if bits_out:
        return quant.quantize(acc, bits_out, block)
    if accum is not None:
        return (np.asarray(accum, np.float32) + acc).astype(np.float32)
    return acc


def reduce_scatter(inputs, g, Np, block, from_level, to_level, bits_per_level,
                   accum=None, ledger=None, trace=None):
    """O9: hierarchical quantized all-to-all reduce-scatter (qgZ).

    inputs[r]: rank r's gradient over range_{from_level-1}(r) (bf16/fp32).
    bits_per_level: {level: 4 | 8 | None}.
    accum[r] (optional): fp32 shard over range_{to_level}(r); result = fl(accum + P).
    trace (optional dict): trace[(level, r)] = list over sending members of the
    scales they used for the chunk destined to r (for the error-bound pins).
    Returns {r: fp32 array over range_{to_level}(r)}.
    """
    W = world_of(g)
    P = {r: quant.to_f32(inputs[r]) for r in range(W)}                 # P_r^(0)
    for level in range(from_level, to_level + 1):
        bits = bits_per_level[level]
        new = {}
        for r in range(W):
            members = exchange_group(r, g, level)
            d = digits(r, g)[level - 1]
            _, ln = range_at(r, g, Np, level)
            chunks = [P[m][d * ln:(d + 1) * ln] for m in members]       # member m's chunk for r
            if bits is None:
                acc = None
                for xh in chunks:                                        # ascending d_l (R10)
                    acc = xh.copy() if acc is None else (acc + xh).astype(np.float32)
                scales_used = []
            else:
                coded = [quant.quantize(ch, bits, block) for ch in chunks]   # A7 / requant (R11)
                acc = reduce_coded(coded, block)                          # A9
                scales_used = [sc for _, sc in coded]
            new[r] = acc
            if trace is not None:
                trace[(level, r)] = scales_used
            if ledger is not None:
                k = len(members) - 1
                payload = k * ln * 4 if bits is None else k * ln * bits // 8
                meta = 0 if bits is None else k * (ln // block) * 4
                ledger.add(r, "grad_rs", level, payload, meta)
        P = new
    if accum is not None:                                                # A10
        return {r: (accum[r].astype(np.float32) + P[r]).astype(np.float32) for r in range(W)}
    return P


def reduce_scatter_hops(inputs, g, Np, block, hops, bits, accum=None, trace=None):
    """O9 with the hop grouping as a parameter ("the hop grouping is a
    parameter"; the "1-hop all-to-all based Reduce-scatter" inside the node).

    hops: consecutive level ranges [(a, b), ...] covering the levels to reduce, e.g.
    [(1, 2), (3, 3)] on 2x2x2 = one all-to-all over the 4 ranks of a node-level group,
    then one over level 3.  For a hop a..b, each member m of r's hop group (ranks that
    share every digit outside a..b, ascending rank) quantizes (``bits``; None = pass
    through) the piece of its P_m^(a-1) that r owns after the hop — range_b(r), which
    lies at off_b(r) - off_{a-1} in the common range_{a-1} — and r sums the members'
    dequantized pieces in ascending rank, fp32, one rounding per add (R10, R11).
    One quantization per hop and contributor: the requantizations between levels of
    one hop disappear.  With one hop per level this is ``reduce_scatter``.
    inputs[r] covers range_{a_0 - 1}(r); returns {r: fp32 over range_{b_last}(r)},
    added to accum[r] when given (A10).  trace[(b, r)] = scales used (error pins)."""
    W = world_of(g)
    P = {r: quant.to_f32(inputs[r]) for r in range(W)}
    for a, b in hops:
        new = {}
        for r in range(W):
            base, _ = range_at(r, g, Np, a - 1)
            off, ln = range_at(r, g, Np, b)
            chunks = [P[m][off - base:off - base + ln] for m in hop_group(r, g, a, b)]
            if bits is None:
                acc = None
                for xh in chunks:
                    acc = xh.copy() if acc is None else (acc + xh).astype(np.float32)
                used = []
            else:
                coded = [quant.quantize(ch, bits, block) for ch in chunks]
                acc = reduce_coded(coded, block)
                used = [sc for _, sc in coded]
            new[r] = acc
            if trace is not None:
                trace[(b, r)] = used
        P = new
    if accum is not None:
        return {r: (np.asarray(accum[r], np.float32) + P[r]).astype(np.float32) for r in range(W)}
    return P


def allreduce_select(inputs, g, Np, from_level, to_level):
    """Paper-literal cross-node step: allreduce the shard over the group of
    levels from..to (tree order: level by level, ascending digit), then keep only the
    slice matching the rank's optimizer range_{to_level}.  Unquantized."""
    W = world_of(g)
    S = {r: quant.to_f32(inputs[r]) for r in range(W)}
    for level in range(from_level, to_level + 1):
        new = {}
        for r in range(W):
            acc = None
            for m in exchange_group(r, g, level):
                acc = S[m].copy() if acc is None else (acc + S[m]).astype(np.float32)
            new[r] = acc
        S = new
    out = {}
    for r in range(W):
        base, _ = range_at(r, g, Np, from_level - 1)
        off, ln = range_at(r, g, Np, to_level)
        out[r] = S[r][off - base: off - base + ln]
    return out
