"""Pins for oracle/partition.py (O1-O3): brute force over all ranks for tiny Np
(exact cover, nesting = the paper's dependency rule, contiguity of every level's
gather output), the 2x2x2 digit-reversal worked out by hand, and the paper's
Table V / VI per-device memory."""

import json
import os
import itertools

import pytest

from oracle import partition as pm
from oracle import volume

HIERS = [(2,), (2, 2), (2, 4), (4, 2), (2, 2, 2), (1,), (3, 2), (2, 2, 2, 2)]
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_digits_roundtrip_node_major():
    g = (2, 2, 2)
    # node-major numbering: pair = {2k, 2k+1}, level-2 groups = {4n..4n+3}
    assert [pm.digits(r, g) for r in range(8)] == [list(t[::-1]) for t in itertools.product(range(2), repeat=3)]
    for gg in HIERS:
        for r in range(pm.world_of(gg)):
            assert pm.rank_of(pm.digits(r, gg), gg) == r
    assert pm.exchange_group(5, g, 1) == [4, 5]
    assert pm.exchange_group(5, g, 2) == [5, 7]
    assert pm.exchange_group(5, g, 3) == [1, 5]
    assert pm.cumulative_group(5, g, 2) == [4, 5, 6, 7]


def test_bit_reverse_2x2x2():
    """Optimizer chunk index of rank r on 2x2x2 is the 3-bit reverse of r (worked by hand)."""
    g = (2, 2, 2)
    Np = 8 * 1024
    chunks = [pm.range_at(r, g, Np, 3)[0] // (Np // 8) for r in range(8)]
    assert chunks == [0, 4, 2, 6, 1, 5, 3, 7]


@pytest.mark.parametrize("g", HIERS)
def test_padding(g):
    W = pm.world_of(g)
    for B in (1, 4, 256):
        for n in (1, 5, W * 4 * B - 1, W * 4 * B, W * 4 * B + 1, 12345):
            Np = pm.padded_numel(n, g, B)
            assert Np >= n and Np % (W * 4 * B) == 0 and Np - n < W * 4 * B
    assert pm.padded_numel(0, g, 256) == 0


@pytest.mark.parametrize("g", HIERS)
def test_exact_cover_and_contiguity(g):
    W = pm.world_of(g)
    Np = W * 4 * 3
    L = len(g)
    for level in range(L + 1):
        # distinct digit prefixes (d_1..d_level) partition [0, Np)
        seen = {}
        for r in range(W):
            off, ln = pm.range_at(r, g, Np, level)
            key = tuple(pm.digits(r, g)[:level])
            if key in seen:
                assert seen[key] == (off, ln)
            seen[key] = (off, ln)
        cover = [0] * Np
        for off, ln in seen.values():
            for i in range(off, off + ln):
                cover[i] += 1
        assert cover == [1] * Np
    # contiguity: level-l exchange group's ranges in ascending d_l concatenate to range_{l-1}
    for r in range(W):
        for level in range(1, L + 1):
            members = pm.exchange_group(r, g, level)
            pos = pm.range_at(r, g, Np, level - 1)[0]
            for m in members:
                off, ln = pm.range_at(m, g, Np, level)
                assert off == pos
                pos += ln
            assert pos == sum(pm.range_at(r, g, Np, level - 1))


@pytest.mark.parametrize("g", HIERS)
def test_nesting_is_the_dependency_rule(g):
    """range_L c range_gl c range_w whenever w <= gl <= L."""
    W = pm.world_of(g)
    Np = W * 4 * 2
    L = len(g)
    for r in range(W):
        for w in range(L + 1):
            for gl in range(w, L + 1):
                rr = pm.role_ranges(r, g, Np, w, w, gl)
                po, pl = rr["primary"]
                go, gln = rr["gradient"]
                oo, ol = rr["optimizer"]
                assert po <= go and go + gln <= po + pl
                assert go <= oo and oo + ol <= go + gln
    with pytest.raises(ValueError):
        pm.role_ranges(0, g, Np, L + 1, 0, 0)


def test_table_v_vi_memory():
    """Role-range sizes reproduce the paper's per-device memory (Tables V, VI)."""
    paper = json.load(open(os.path.join(GOLDEN, "paper_numbers.json")))
    g = (2, 4)                      # pair, then the rest of an 8-GPU "node"
    Np = 8 * 4 * 256 * 10
    psi = Np
    for r in range(8):
        rr = pm.role_ranges(r, g, Np, w=1, s=1, gl=2)
        primary_bytes = 2 * rr["primary"][1]           # bf16
        sec2 = rr["secondary"][1] * 1                   # int8 codes
        assert primary_bytes == 2 * psi / paper["primary_degree"]["value"]
        assert (primary_bytes + sec2) / psi == paper["weight_bytes_per_psi_sec2"]["value"]
        assert primary_bytes + sec2 == volume.weight_memory_bytes(psi, "ours", sec_degree=2)
        rr8 = pm.role_ranges(r, g, Np, w=1, s=2, gl=2)
        assert (primary_bytes + rr8["secondary"][1]) / psi == paper["weight_bytes_per_psi_sec8"]["value"]
        grad_fp16 = 2 * rr["gradient"][1]
        assert grad_fp16 / psi == paper["grad_bytes_per_psi_fp16"]["value"]
        assert grad_fp16 == volume.gradient_memory_bytes(psi, "ours", P=8)
