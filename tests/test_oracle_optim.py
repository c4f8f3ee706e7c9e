"""Pins for oracle/optim.py: AdamW against an independent fp64
textbook AdamW (Loshchilov & Hutter, decoupled weight decay, bias-corrected
moments) over several steps, the first-step closed form (update = lr * sign(g)),
the zero-gradient case (pure decay), and the post-update all-gather reassembling
the flat tensor from the optimizer shards for every hierarchy."""

import numpy as np
import pytest

from oracle import optim
from oracle import partition as pm


def _textbook(theta, g_seq, lr, b1, b2, eps, wd):
    th = theta.astype(np.float64)
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    for t, g in enumerate(g_seq, start=1):
        g = g.astype(np.float64)
        th = th - lr * wd * th
        m = b1 * m + (1 - b1) * g
        v = b2 * v + (1 - b2) * g * g
        mh = m / (1 - b1 ** t)
        vh = v / (1 - b2 ** t)
        th = th - lr * mh / (np.sqrt(vh) + eps)
    return th


def test_matches_fp64_textbook_over_steps():
    rng = np.random.default_rng(0)
    n = 4096
    theta = (rng.standard_normal(n) * 0.02).astype(np.float32)
    gs = [(rng.standard_normal(n) * 1e-3).astype(np.float32) for _ in range(5)]
    lr, b1, b2, eps, wd = 1e-3, 0.9, 0.95, 1e-8, 0.1
    th, m, v = theta, np.zeros(n, np.float32), np.zeros(n, np.float32)
    for t, g in enumerate(gs, start=1):
        th, m, v = optim.adamw(th, m, v, g, optim.adamw_scalars(lr, b1, b2, eps, wd, t))
    ref = _textbook(theta, gs, lr, b1, b2, eps, wd)
    # 5 steps of fp32 roundings on values ~0.02 with updates ~1e-3
    assert np.max(np.abs(th.astype(np.float64) - ref)) <= 5 * 2 ** -24 * 0.1 + 1e-9


def test_first_step_is_lr_sign_g():
    rng = np.random.default_rng(1)
    n = 1024
    theta = rng.standard_normal(n).astype(np.float32)
    g = (rng.standard_normal(n) * 1e-2).astype(np.float32)
    lr = 1e-3
    th, m, v = optim.adamw(theta, np.zeros(n, np.float32), np.zeros(n, np.float32), g,
                           optim.adamw_scalars(lr, 0.9, 0.999, 1e-12, 0.0, 1))
    assert np.allclose(m, 0.1 * g.astype(np.float64), rtol=1e-6)
    assert np.allclose(th.astype(np.float64), theta - lr * np.sign(g), rtol=0, atol=lr * 1e-5 + 1e-6)


def test_zero_gradient_is_pure_decay():
    theta = np.linspace(-1, 1, 512, dtype=np.float32)
    z = np.zeros(512, np.float32)
    s = optim.adamw_scalars(1e-2, 0.9, 0.999, 1e-8, 0.5, 3)
    th, m, v = optim.adamw(theta, z, z, z, s)
    assert not m.any() and not v.any()
    assert np.array_equal(th, (theta - (np.float32(1e-2 * 0.5) * theta).astype(np.float32)).astype(np.float32))


@pytest.mark.parametrize("g,w", [((2, 2, 2), 1), ((2, 2, 2), 0), ((2, 4), 1), ((4, 2), 1), ((2,), 1), ((1,), 1),
                                 ((2, 2, 2), 2)])
def test_post_update_allgather_reassembles(g, w):
    W = pm.world_of(g)
    L = len(g)
    Np = pm.padded_numel(3000, g, 32)
    flat = np.arange(Np, dtype=np.float32)
    shards = {r: flat[slice(*(lambda o, n: (o, o + n))(*pm.range_at(r, g, Np, L)))] for r in range(W)}
    out = optim.post_update_allgather(shards, g, Np, w)
    for r in range(W):
        off, ln = pm.range_at(r, g, Np, w)
        assert np.array_equal(out[r], flat[off:off + ln])
