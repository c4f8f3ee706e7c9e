"""O10: closed-form communication volumes and on-device memory from the paper.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Unit reading (DESIGN.md §3 R13): the paper's "psi x (d-1)/d" for ZeRO-3 is the
fp16 model of M = 2*psi bytes; qwZ halves it ("each parameter can
be represented using only 1 byte (INT8) instead of 2 bytes (FP16)"), qgZ
quarters it ("reduce communication volume by 4x").  Volumes are
per-device received payload bytes; fp32 scale metadata is counted apart
(SPEC S:165).
"""

import math


def zero3_allgather_bytes(Np, d):
    """Table VII row ZeRO-3: fp16 weights, M (d-1)/d with M = 2 Np bytes."""
    return 2 * Np * (d - 1) / d


def qwz_allgather_bytes(Np, d, bits=8):
    """Table VII rows ZeRO++/Ours: quantized weights, (M/2)(d-1)/d for INT8."""
    return Np * bits / 8 * (d - 1) / d


def qgz_reduce_scatter_bytes(Np, d, bits=4):
    """Table VIII rows ZeRO++/Ours: INT4 gradients, (M/4)(d-1)/d."""
    return Np * bits / 8 * (d - 1) / d


def zero3_reduce_scatter_bytes(Np, d):
    """Table VIII row ZeRO-3."""
    return 2 * Np * (d - 1) / d


def scale_meta_bytes(Np, d, block):
    """fp32 scale metadata that rides along a quantized collective over d devices."""
    return Np / block * 4 * (d - 1) / d


def hierarchical_level_bytes(Np, g, level, bits):
    """Per-rank received payload at one level of the hierarchy: (g_l - 1) * len_l * bits/8."""
    len_l = Np // math.prod(g[:level])
    return (g[level - 1] - 1) * len_l * bits // 8


def telescoped_fraction(g, top, bottom=1):
    """sum_{l=bottom}^{top} (g_l - 1)/g_l / prod_{k<l} g_k  ==  (D-1)/D, D = prod_{l<=top} g_l
    when bottom == 1.  Returned as the left-hand sum."""
    total = 0.0
    for level in range(bottom, top + 1):
        total += (g[level - 1] - 1) / g[level - 1] / math.prod(g[:level - 1])
    return total


def internode_volume_zero3_vs_zeropp(M):
    """ZeRO-3 moves 3M inter-node per step (fwd AG M, bwd AG M, RS M);
    ZeRO++ moves 0.75M (fwd AG 0.5M, bwd AG 0 via hpZ, RS 0.25M)."""
    zero3 = M + M + M
    zeropp = 0.5 * M + 0.0 + 0.25 * M
    return zero3, zeropp


def weight_memory_bytes(psi, scheme, sec_degree=2, Nw=1, Pw=1, P=8):
    """Table V: per-device weight memory in bytes."""
    if scheme == "zero3":
        return 2 * psi / (Nw * Pw)
    if scheme == "zero++":
        return 2 * psi / (Nw * Pw) + 2 * psi / P
    if scheme == "ours":
        return 2 * psi / 2 + psi / sec_degree
    raise ValueError(scheme)


def gradient_memory_bytes(psi, scheme, Ng=1, Pg=8, P=8):
    """Table VI: per-device fp16 gradient memory in bytes."""
    if scheme in ("zero3", "zero++"):
        return 2 * psi / (Ng * Pg)
    if scheme == "ours":
        return 2 * psi / P
    raise ValueError(scheme)
