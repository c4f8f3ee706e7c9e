"""O1-O3: rank digits, padding and the digit-reversed ownership map.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper: weights are sharded over 2 GCDs, gradients over the GCDs of a node,
optimizer states over all N x P GCDs (Table IV), subject to the
dependency rule N >= N_os >= N_g >= N_w, P >= P_os >= P_g >= P_w: "each worker
stores only the gradients and optimizer states related to its local
parameters".

Hierarchy g = (g_1, ..., g_L), innermost first; W = prod(g).
  O1  r = sum_l d_l(r) * prod_{k<l} g_k   (node-major rank numbering)
  O2  Np = ceil(n / (W*4*B)) * W*4*B, zero padded                  (reading R7)
  O3  off_0 = 0, len_0 = Np; len_l = len_{l-1} / g_l;
      off_l = off_{l-1} + d_l(r) * len_l                           (reading R8)
      role ranges: primary = range_w, secondary = range_s,
      gradient = range_gl, optimizer = range_L.
Nesting range_L c range_gl c range_w is the paper's dependency rule.
"""

import math


def world_of(g):
    return math.prod(g)


def digits(r, g):
    """O1: d_l(r) for l = 1..L (returned as a list indexed 0..L-1)."""
    out = []
    stride = 1
    for gl in g:
        out.append((r // stride) % gl)
        stride *= gl
    return out


def rank_of(ds, g):
    """Inverse of O1."""
    r, stride = 0, 1
    for d, gl in zip(ds, g):
        r += d * stride
        stride *= gl
    return r


def padded_numel(n, g, block):
    """O2."""
    unit = world_of(g) * 4 * block
    return -(-n // unit) * unit if n > 0 else 0


def ranges(r, g, Np):
    """O3: lists off[0..L], length[0..L] for rank r."""
    ds = digits(r, g)
    off = [0]
    ln = [Np]
    for level, gl in enumerate(g, start=1):
        if ln[-1] % gl:
            raise ValueError("Np not divisible by the hierarchy")
        ln.append(ln[-1] // gl)
        off.append(off[-1] + ds[level - 1] * ln[-1])
    return off, ln


def range_at(r, g, Np, level):
    off, ln = ranges(r, g, Np)
    return off[level], ln[level]


def exchange_group(r, g, level):
    """Ranks that differ from r only in digit ``level`` (1-based), ordered by that digit."""
    ds = digits(r, g)
    members = []
    for j in range(g[level - 1]):
        e = list(ds)
        e[level - 1] = j
        members.append(rank_of(e, g))
    return members


def hop_group(r, g, a, b):
    """Ranks sharing every digit outside levels a..b with r, in ascending rank order
    (= ascending merged digit, d_a least significant): the members of one merged-level
    qgZ all-to-all ("1-hop"; reading R15)."""
    ds = digits(r, g)
    W = world_of(g)
    keep = [k for k in range(len(g)) if not a - 1 <= k <= b - 1]
    return [q for q in range(W) if all(digits(q, g)[k] == ds[k] for k in keep)]


def cumulative_group(r, g, level):
    """Ranks sharing every digit above ``level`` with r (size prod_{k<=level} g_k)."""
    ds = digits(r, g)
    W = world_of(g)
    return [q for q in range(W) if digits(q, g)[level:] == ds[level:]]


def role_ranges(r, g, Np, w, s, gl):
    """O3 role ranges for one rank: dict name -> (off, len)."""
    L = len(g)
    for name, v in (("w", w), ("s", s), ("gl", gl)):
        if not 0 <= v <= L:
            raise ValueError(f"role level {name}={v} outside [0, {L}]")
    off, ln = ranges(r, g, Np)
    return {
        "primary": (off[w], ln[w]),
        "secondary": (off[s], ln[s]),
        "gradient": (off[gl], ln[gl]),
        "optimizer": (off[L], ln[L]),
    }
