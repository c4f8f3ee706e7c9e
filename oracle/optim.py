"""Step tail: AdamW on the optimizer shard and the post-update
all-gather of the updated weights.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Paper: optimizer states (fp32 master copy, momentum, variance of AdamW) are
sharded over all N x P ranks; gradients are reduced before
the update; "Following completion of model parameter updates, we conduct
an Allgather within the optimizer shards to gather the updated weights".

The paper does not write AdamW out; reading R19 is PyTorch's
decoupled-weight-decay AdamW with bias correction, in fp32, one rounding per
operation, the host-computed scalars passed in as fp32 values:

    m'    = fl(fl(b1 * m) + fl(omb1 * g))                 omb1 = 1 - b1
    v'    = fl(fl(b2 * v) + fl(fl(omb2 * g) * g))          omb2 = 1 - b2
    th1   = fl(th - fl(lr_wd * th))                        lr_wd = lr * wd
    denom = fl(fl(sqrt(v') / sqrt_bc2) + eps)              sqrt_bc2 = sqrt(1 - b2^t)
    th'   = fl(th1 - fl(step * fl(m' / denom)))            step = lr / (1 - b1^t)

The post-update all-gather (R20) concatenates the updated range_L shards of the
ranks that share every digit up to w, giving each rank its primary range_w
(the narrow form of P:399's exchange allowed by the nested map).
"""

import numpy as np

from . import partition as pm

F = np.float32


def adamw_scalars(lr, b1, b2, eps, wd, t):
    """Host-side constants of step t (t >= 1), rounded once to fp32."""
    return {
        "b1": F(b1), "omb1": F(1.0 - b1), "b2": F(b2), "omb2": F(1.0 - b2),
        "lr_wd": F(lr * wd), "sqrt_bc2": F(np.sqrt(1.0 - b2 ** t)), "eps": F(eps),
        "step": F(lr / (1.0 - b1 ** t)),
    }


def adamw(theta, m, v, g, s):
    """One AdamW update of fp32 arrays (R19).  Returns (theta', m', v')."""
    th, m, v, g = (np.asarray(a, np.float32) for a in (theta, m, v, g))
    m1 = (s["b1"] * m + s["omb1"] * g).astype(F)
    v1 = (s["b2"] * v + ((s["omb2"] * g).astype(F) * g).astype(F)).astype(F)
    th1 = (th - (s["lr_wd"] * th).astype(F)).astype(F)
    denom = ((np.sqrt(v1) / s["sqrt_bc2"]).astype(F) + s["eps"]).astype(F)
    th2 = (th1 - (s["step"] * (m1 / denom).astype(F)).astype(F)).astype(F)
    return th2, m1, v1


def post_update_allgather(shards, g, Np, w):
    """R20: shards[r] = rank r's updated values over range_L(r); returns out[r] over
    range_w(r) (concatenation in offset order of the members' shards)."""
    W = pm.world_of(g)
    L = len(g)
    out = {}
    for r in range(W):
        off_w, len_w = pm.range_at(r, g, Np, w)
        buf = np.empty(len_w, dtype=np.asarray(shards[r]).dtype)
        for q in range(W):
            off, ln = pm.range_at(q, g, Np, L)
            if off_w <= off < off_w + len_w:
                buf[off - off_w:off - off_w + ln] = shards[q]
        out[r] = buf
    return out
