"""Pins for oracle/volume.py and the oracle ledgers (O10): the simulated per-level byte
ledger equals the per-level closed form, the levels telescope to the paper's 1-hop
formulas with d = D (Tables VII, VIII), and the paper's ratios 0.5 / 0.25 and
3M -> 0.75M come out."""

import json
import os

import numpy as np
import pytest

from oracle import collectives as col
from oracle import partition as pm
from oracle import volume
from paper_2501_04266_b200 import synth

PAPER = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


@pytest.mark.parametrize("g", [(2, 2, 2), (2, 4), (2, 2), (4, 2)])
def test_telescoping(g):
    D = pm.world_of(g)
    assert abs(volume.telescoped_fraction(g, len(g)) - (D - 1) / D) < 1e-15


@pytest.mark.parametrize("g", [(2, 2, 2), (2, 4), (2, 2), (4, 2)])
def test_ledgers_match_closed_forms(g):
    B = 8
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(3000, g, B)
    full = synth.params_like(Np, 1, block=B)
    prim = {}
    for r in range(W):
        off, ln = pm.range_at(r, g, Np, L)
        prim[r] = full[off:off + ln]
    led = col.Ledger()
    _, sec = col.allgather_forward(prim, g, Np, B, L, L, bits=8, ledger=led)
    col.allgather_backward(sec, g, Np, B, L, bits=8, ledger=led)
    xs = {r: synth.gradient_like(Np, 10 + r, block=B) for r in range(W)}
    col.reduce_scatter(xs, g, Np, B, 1, L, {l: 4 for l in range(1, L + 1)}, ledger=led)
    for r in range(W):
        for level in range(1, L + 1):
            p, m = led.level(r, "forward_ag", level)
            assert p == volume.hierarchical_level_bytes(Np, g, level, 8)
            p, m = led.level(r, "grad_rs", level)
            assert p == volume.hierarchical_level_bytes(Np, g, level, 4)
        p, m = led.per_rank(r, "forward_ag")
        assert p == volume.qwz_allgather_bytes(Np, W, 8)
        assert m == volume.scale_meta_bytes(Np, W, B)
        assert led.per_rank(r, "backward_ag") == led.per_rank(r, "forward_ag")
        p, m = led.per_rank(r, "grad_rs")
        assert p == volume.qgz_reduce_scatter_bytes(Np, W, 4)
        # the paper's ratios against fp16 ZeRO-3 (Table VII / VIII)
        assert p / volume.zero3_reduce_scatter_bytes(Np, W) == PAPER["reduce_scatter_int4_ratio"]["value"]
        pf, _ = led.per_rank(r, "forward_ag")
        assert pf / volume.zero3_allgather_bytes(Np, W) == PAPER["allgather_int8_ratio"]["value"]


def test_setting_t_secondary_keeps_backward_in_the_pair():
    """Table VII 'Ours: Sec-Degree=2': backward d = 2, independent of the total D."""
    g = (2, 2, 2)
    B = 8
    Np = pm.padded_numel(1000, g, B)
    full = synth.params_like(Np, 2, block=B)
    prim = {r: full[slice(*(lambda o, l: (o, o + l))(*pm.range_at(r, g, Np, 1)))] for r in range(8)}
    led = col.Ledger()
    _, sec = col.allgather_forward(prim, g, Np, B, 1, 1, bits=8, ledger=led)
    col.allgather_backward(sec, g, Np, B, 1, bits=8, ledger=led)
    for r in range(8):
        assert led.per_rank(r, "backward_ag")[0] == volume.qwz_allgather_bytes(Np, 2, 8)
        assert led.level(r, "backward_ag", 2) == (0, 0) and led.level(r, "backward_ag", 3) == (0, 0)


def test_internode_3M_to_075M():
    z3, zpp = volume.internode_volume_zero3_vs_zeropp(1.0)
    assert z3 == PAPER["internode_zero3_M"]["value"]
    assert zpp == PAPER["internode_zeropp_M"]["value"]
