"""Multi-rank parity worker for the NCCL path (launched by tests/test_gpu_collectives.py
under torchrun, one process per GPU; also callable in-process at world 1).

Each rank runs the product path (hz.Context -> libhz.so -> NCCL per-level
communicators) on seeded inputs, then runs the CPU oracle's all-ranks simulation
on the same inputs and compares its own rank's results bit for bit: the forward
and backward gathered layers, the hpZ secondary, and the qgZ fp32 shard (one-call
GA=1 and the setting-T two-phase GA=2 with accumulation)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import ml_dtypes  # noqa: E402
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import collectives as col  # noqa: E402
from oracle import partition as pm  # noqa: E402
from oracle import quant  # noqa: E402
from paper_2501_04266_b200 import synth  # noqa: E402
from tests.gpu_util import Guarded, assert_bitwise, assert_unchanged, to_dev, to_host  # noqa: E402

HIERARCHIES = {
    1: [(1,)],
    2: [(2,), (1, 2)],
    4: [(2, 2), (4,), (2, 1, 2)],
    8: [(2, 2, 2), (2, 4), (4, 2), (8,)],
}


def role_cases(L):
    cases = {(1, 1), (L, max(L - 1, 0)), (1, min(2, L)), (L, L), (0, 0)}
    return sorted(c for c in cases if 0 <= c[0] <= L and 0 <= c[1] <= L)


def check_hierarchy(hz, rank, world, g, uid, device, numel=150_001, B=256, p2p=False, vctx=None):
    """vctx: a virtual-world context (tests/vworld.py; P2P, one GPU, one thread per
    rank) instead of a context made here — then the CUDA-graph and flat-NCCL parts,
    which a virtual world does not support, are skipped."""
    errors = []
    virtual = vctx is not None
    if virtual:
        ctx, p2p = vctx, True
    else:
        ctx = hz.Context(rank, world, uid, g, device)
    L = len(g)
    tag = "vworld" if virtual else ("p2p" if p2p else "nccl")
    if p2p and not virtual:
        ctx.enable_p2p(64 << 20)

    def sec_buffers(n_codes, n_scales):
        if p2p:
            return (ctx.sym_alloc(n_codes, torch.uint8), ctx.sym_alloc(n_scales, torch.float32))
        return (torch.empty(n_codes, dtype=torch.uint8, device="cuda"),
                torch.empty(n_scales, dtype=torch.float32, device="cuda"))

    def guarded_sec(n_codes, n_scales):
        alloc = ctx.sym_alloc if p2p else None
        return Guarded(n_codes, torch.uint8, alloc), Guarded(n_scales, torch.float32, alloc)
    try:
        Np = pm.padded_numel(numel, g, B)
        full = np.zeros(Np, np.float32)
        full[:numel] = synth.params_like(numel, 7, block=B)
        full = full.astype(ml_dtypes.bfloat16)
        for w, s in role_cases(L):
            p = ctx.partition(numel, B, w, s, L)
            assert p.padded_numel == Np
            off, ln = p.range(w)
            prim = {r: full[pm.range_at(r, g, Np, w)[0]:sum(pm.range_at(r, g, Np, w))] for r in range(world)}
            want, want_sec = col.allgather_forward(prim, g, Np, B, w, s, bits=8)
            so, sl = p.range(s)
            gc, gs = guarded_sec(sl, sl // B)
            sec_c, sec_s = gc.t, gs.t
            go = Guarded(Np, torch.bfloat16)
            out = go.t
            prim_in = to_dev(full[off:off + ln])
            ctx.allgather_params(p, prim_in, sec_c, sec_s, out, bits=8)
            torch.cuda.synchronize()
            try:
                what = f"[{tag}] g={g} w={w} s={s} forward"
                go.check(what + " layer")
                gc.check(what + " secondary codes")
                gs.check(what + " secondary scales")
                assert_unchanged(prim_in, full[off:off + ln], what + " primary")
                assert_bitwise(to_host(out), want[rank], f"[{tag}] g={g} w={w} s={s} forward layer")
                assert_bitwise(to_host(sec_c), quant.wire_codes(want_sec[rank][0], 8), f"[{tag}] g={g} w={w} s={s} secondary codes")
                assert_bitwise(to_host(sec_s), want_sec[rank][1], f"[{tag}] g={g} w={w} s={s} secondary scales")
                go2 = Guarded(Np, torch.bfloat16)
                out2 = go2.t
                ctx.allgather_params(p, None, sec_c, sec_s, out2, bits=8, backward=True)
                torch.cuda.synchronize()
                assert_bitwise(to_host(out2), want[rank], f"[{tag}] g={g} w={w} s={s} backward layer")
                go2.check(f"[{tag}] g={g} w={w} s={s} backward layer")
                gc.check(f"[{tag}] g={g} w={w} s={s} backward: secondary codes")
            except AssertionError as e:
                errors.append(str(e))

        # qgZ: one call over all levels (GA = 1)
        grads = {r: synth.gradient_like(Np, 900 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(world)}
        for bits1 in (4, 8):
            bpl = [bits1] + [4] * (L - 1)
            p = ctx.partition(numel, B, 1, 1, L)
            want = col.reduce_scatter(grads, g, Np, B, 1, L, {l: bpl[l - 1] for l in range(1, L + 1)})
            gsh = Guarded(p.range(L)[1], torch.float32)
            shard = gsh.t
            grad_in = to_dev(grads[rank])
            ctx.reduce_scatter_grads(p, grad_in, shard, bpl)
            torch.cuda.synchronize()
            try:
                assert_bitwise(to_host(shard), want[rank], f"[{tag}] g={g} qgZ bits={bpl}")
                gsh.check(f"[{tag}] g={g} qgZ bits={bpl} shard")
                assert_unchanged(grad_in, grads[rank], f"[{tag}] g={g} qgZ bits={bpl} gradient")
            except AssertionError as e:
                errors.append(str(e))
            # accumulate into the shard (A = fl(A + P)): second micro-batch
            ctx.reduce_scatter_grads(p, to_dev(grads[rank]), shard, bpl, accumulate=True)
            torch.cuda.synchronize()
            try:
                assert_bitwise(to_host(shard), (want[rank] + want[rank]).astype(np.float32),
                               f"[{tag}] g={g} qgZ accumulate bits={bpl}")
            except AssertionError as e:
                errors.append(str(e))

        # setting T, GA = 2: levels 1..gl per micro-batch with accumulate, then gl+1..L once
        if L >= 2:
            gl = L - 1
            p = ctx.partition(numel, B, 1, 1, gl)
            grads2 = {r: synth.gradient_like(Np, 950 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(world)}
            bmap = {l: 4 for l in range(1, L + 1)}
            A = col.reduce_scatter(grads, g, Np, B, 1, gl, bmap)
            A = col.reduce_scatter(grads2, g, Np, B, 1, gl, bmap, accum=A)
            want = col.reduce_scatter(A, g, Np, B, gl + 1, L, bmap)
            acc = torch.empty(p.range(gl)[1], dtype=torch.float32, device="cuda")
            ctx.reduce_scatter_grads(p, to_dev(grads[rank]), acc, [4] * L, 1, gl, accumulate=False)
            ctx.reduce_scatter_grads(p, to_dev(grads2[rank]), acc, [4] * L, 1, gl, accumulate=True)
            shard = torch.empty(p.range(L)[1], dtype=torch.float32, device="cuda")
            ctx.reduce_scatter_grads(p, acc, shard, [4] * L, gl + 1, L)
            torch.cuda.synchronize()
            try:
                assert_bitwise(to_host(acc), A[rank], f"[{tag}] g={g} two-phase accumulated shard")
                assert_bitwise(to_host(shard), want[rank], f"[{tag}] g={g} two-phase final shard")
            except AssertionError as e:
                errors.append(str(e))

        # A10 paper-literal option: fp32 allreduce over levels frm..L, then select
        # range_L — bitwise equal to the oracle's allreduce_select
        for frm in sorted({1, L}):
            p = ctx.partition(numel, B, 1, 1, L)
            shards = {}
            for q in range(world):
                o, n_ = pm.range_at(q, g, Np, frm - 1)
                shards[q] = synth.gradient_like(n_, 300 + q, block=B, specials=False)
            want = col.allreduce_select(shards, g, Np, frm, L)
            gin = to_dev(shards[rank])
            gout = Guarded(p.range(L)[1], torch.float32)
            ctx.allreduce_select(p, gin, gout.t, frm, L)
            torch.cuda.synchronize()
            try:
                what = f"[{tag}] g={g} allreduce+select from level {frm}"
                assert_bitwise(to_host(gout.t), want[rank], what)
                gout.check(what)
                assert_unchanged(gin, shards[rank], what)
            except AssertionError as e:
                errors.append(str(e))

        # step tail (N2): AdamW on range_L, post-update all-gather into range_w
        from oracle import optim
        for w in sorted({1, L, 0} & set(range(L + 1))):
            p = ctx.partition(numel, B, w, w, L)
            oL, nL = p.range(L)
            ow, nw = p.range(w)
            rs = np.random.default_rng(77 + rank)
            th0 = {}
            upd = {}
            for q in range(world):
                rq = np.random.default_rng(500 + q)
                o, n_ = pm.range_at(q, g, Np, L)
                th_q = (rq.standard_normal(n_) * 0.02).astype(np.float32)
                m_q = (rq.standard_normal(n_) * 1e-3).astype(np.float32)
                v_q = (rq.random(n_) * 1e-6).astype(np.float32)
                g_q = (rq.standard_normal(n_) * 1e-3).astype(np.float32)
                th0[q] = (th_q, m_q, v_q, g_q)
                s = optim.adamw_scalars(1e-3, 0.9, 0.95, 1e-8, 0.1, 3)
                upd[q] = optim.adamw(th_q, m_q, v_q, g_q, s)
            want_prim = optim.post_update_allgather({q: upd[q][0].astype(ml_dtypes.bfloat16) for q in range(world)},
                                                    g, Np, w)
            th_d, m_d, v_d, g_d = (to_dev(a.copy()) for a in th0[rank])
            gpr = Guarded(nw, torch.bfloat16)
            prim = gpr.t
            ctx.adamw_step(p, g_d, th_d, m_d, v_d, hz.adamw_params(1e-3, 0.9, 0.95, 1e-8, 0.1, 3), prim)
            torch.cuda.synchronize()
            try:
                gpr.check(f"[{tag}] g={g} w={w} post-update primary")
                assert_unchanged(g_d, th0[rank][3], f"[{tag}] g={g} w={w} adamw gradient")
                assert_bitwise(to_host(th_d), upd[rank][0], f"[{tag}] g={g} w={w} adamw master")
                assert_bitwise(to_host(m_d), upd[rank][1], f"[{tag}] g={g} w={w} adamw m")
                assert_bitwise(to_host(v_d), upd[rank][2], f"[{tag}] g={g} w={w} adamw v")
                assert_bitwise(to_host(prim), want_prim[rank], f"[{tag}] g={g} w={w} post-update all-gather")
            except AssertionError as e:
                errors.append(str(e))

        if virtual:
            errors += check_step_host(ctx, hz, rank, world, g, sec_buffers, tag, B)
            errors += check_pipelined(ctx, hz, rank, world, g, sec_buffers, tag, B, p2p)
            errors += check_hops(ctx, hz, rank, world, g, sec_buffers, tag, B)
            return errors

        # CUDA graph: one captured step (forward gather, backward gather, qgZ) replayed
        # three times with fresh inputs copied into the captured buffers
        p = ctx.partition(numel, B, 1, 1, L)
        off, ln = p.range(1)
        _, sl = p.range(1)
        sec_c, sec_s = sec_buffers(sl, sl // B)
        prim_d = torch.empty(ln, dtype=torch.bfloat16, device="cuda")
        grad_d = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        fwd = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        bwd = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        shard = torch.empty(p.range(L)[1], dtype=torch.float32, device="cuda")

        def one_step(st):
            ctx.allgather_params(p, prim_d, sec_c, sec_s, fwd, bits=8, stream=st)
            ctx.allgather_params(p, None, sec_c, sec_s, bwd, bits=8, backward=True, stream=st)
            ctx.reduce_scatter_grads(p, grad_d, shard, [4] * L, stream=st)

        prim_d.copy_(to_dev(full[off:off + ln]))
        grad_d.copy_(to_dev(grads[rank]))
        one_step(torch.cuda.current_stream())          # eager warm-up (workspaces)
        torch.cuda.synchronize()
        cs = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cs):
            if p2p:
                ctx.p2p_capture_begin()
            one_step(cs)
            if p2p:
                ctx.p2p_capture_end(cs)
        for it in range(3):
            fr = np.zeros(Np, np.float32)
            fr[:numel] = synth.params_like(numel, 70 + it, block=B)
            fr = fr.astype(ml_dtypes.bfloat16)
            gr = {r: synth.gradient_like(Np, 700 + 10 * it + r, block=B).astype(ml_dtypes.bfloat16) for r in range(world)}
            prim_d.copy_(to_dev(fr[off:off + ln]))
            grad_d.copy_(to_dev(gr[rank]))
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            if p2p:
                ctx.p2p_replayed(1)
            prim = {r: fr[pm.range_at(r, g, Np, 1)[0]:sum(pm.range_at(r, g, Np, 1))] for r in range(world)}
            want_f, _ = col.allgather_forward(prim, g, Np, B, 1, 1, bits=8)
            want_r = col.reduce_scatter(gr, g, Np, B, 1, L, {l: 4 for l in range(1, L + 1)})
            try:
                assert_bitwise(to_host(fwd), want_f[rank], f"[{tag}] g={g} graph replay {it} forward")
                assert_bitwise(to_host(bwd), want_f[rank], f"[{tag}] g={g} graph replay {it} backward")
                assert_bitwise(to_host(shard), want_r[rank], f"[{tag}] g={g} graph replay {it} qgZ")
            except AssertionError as e:
                errors.append(str(e))
        # an eager call after the replays continues the phase numbering
        one_step(torch.cuda.current_stream())
        torch.cuda.synchronize()
        try:
            assert_bitwise(to_host(shard), col.reduce_scatter(gr, g, Np, B, 1, L, {l: 4 for l in range(1, L + 1)})[rank],
                           f"[{tag}] g={g} eager after graph")
        except AssertionError as e:
            errors.append(str(e))
        del graph

        errors += check_step_host(ctx, hz, rank, world, g, sec_buffers, tag, B)
        errors += check_pipelined(ctx, hz, rank, world, g, sec_buffers, tag, B, p2p)
        errors += check_hops(ctx, hz, rank, world, g, sec_buffers, tag, B)

        # flat ZeRO-3 baseline collectives (plain NCCL)
        n = world * 4096
        x = torch.arange(n, dtype=torch.float32, device="cuda") + rank
        chunk = x[rank * 4096:(rank + 1) * 4096].contiguous()
        outf = torch.empty(n, dtype=torch.float32, device="cuda")
        ctx.flat_allgather(chunk, outf)
        rs = torch.empty(4096, dtype=torch.float32, device="cuda")
        ctx.flat_reduce_scatter(x, rs)
        torch.cuda.synchronize()
        want_ag = np.concatenate([np.arange(q * 4096, (q + 1) * 4096, dtype=np.float32) + q for q in range(world)])
        want_rs = (np.arange(rank * 4096, (rank + 1) * 4096, dtype=np.float64) * world + sum(range(world)))
        try:
            assert_bitwise(to_host(outf), want_ag, "flat all-gather")
            assert np.allclose(to_host(rs), want_rs, rtol=1e-6), "flat reduce-scatter"
        except AssertionError as e:
            errors.append(str(e))
    finally:
        if not virtual:
            ctx.close()
    return errors


def hop_groupings(L):
    """Every qgZ hop grouping of L levels other than one hop per level (R15)."""
    out = []
    for mask in range(1 << (L - 1)):
        hl = [l for l in range(1, L) if (mask >> (l - 1)) & 1] + [L]
        if len(hl) < L:
            out.append(tuple(hl))
    return out


def check_hops(ctx, hz, rank, world, g, sec_buffers, tag, B, numel=150_001):
    """Merged-level qgZ (hz_partition_set_hops): every hop grouping of the hierarchy,
    one call over all levels, bitwise against the oracle's reduce_scatter_hops; then the
    paper-literal ZeRO-topo step: a 1-hop all-to-all over levels
    1..L-1 per micro-batch (GA = 2, accumulated), then the fp32 allreduce + select over
    level L (hz_allreduce_select)."""
    errors = []
    L = len(g)
    if L < 2:
        return errors
    Np = pm.padded_numel(numel, g, B)
    grads = {r: synth.gradient_like(Np, 4200 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(world)}
    for hl in hop_groupings(L):
        for bits in (4, 8):
            p = ctx.partition(numel, B, 1, 1, L, hops=hl)
            want = col.reduce_scatter_hops(grads, g, Np, B, hops_from_last(hl), bits)
            sh = torch.full((p.range(L)[1],), float("nan"), dtype=torch.float32, device="cuda")
            ctx.reduce_scatter_grads(p, to_dev(grads[rank]), sh, [bits] * L)
            torch.cuda.synchronize()
            try:
                assert_bitwise(to_host(sh), want[rank], f"[{tag}] g={g} hops={hl} bits={bits} qgZ")
            except AssertionError as e:
                errors.append(str(e))
    # ZeRO-topo: hops (1..L-1), (L); GA = 2 on levels 1..L-1 then allreduce + select at L
    hl = (L - 1, L)
    p = ctx.partition(numel, B, 1, 1, L - 1, hops=hl)
    grads2 = {r: synth.gradient_like(Np, 4300 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(world)}
    hops = hops_from_last(hl)
    A = col.reduce_scatter_hops(grads, g, Np, B, hops[:1], 4)
    A = col.reduce_scatter_hops(grads2, g, Np, B, hops[:1], 4, accum=A)
    want = col.allreduce_select(A, g, Np, L, L)
    acc = torch.empty(p.range(L - 1)[1], dtype=torch.float32, device="cuda")
    ctx.reduce_scatter_grads(p, to_dev(grads[rank]), acc, [4] * L, 1, L - 1)
    ctx.reduce_scatter_grads(p, to_dev(grads2[rank]), acc, [4] * L, 1, L - 1, accumulate=True)
    out = torch.empty(p.range(L)[1], dtype=torch.float32, device="cuda")
    ctx.allreduce_select(p, acc, out, L, L)
    torch.cuda.synchronize()
    try:
        assert_bitwise(to_host(acc), A[rank], f"[{tag}] g={g} ZeRO-topo 1-hop accumulated shard")
        assert_bitwise(to_host(out), want[rank], f"[{tag}] g={g} ZeRO-topo allreduce+select")
    except AssertionError as e:
        errors.append(str(e))
    return errors


def hops_from_last(hop_last):
    out, a = [], 1
    for b in hop_last:
        out.append((a, b))
        a = b + 1
    return out


def check_pipelined(ctx, hz, rank, world, g, sec_buffers, tag, B, p2p, sizes=(150_001, 70_000, 4097, 9000)):
    """hz_allgather_params_next / hz_backward_step (adjacent layers paired; on the P2P
    transport with B = 256 one dual kernel per pair): two back-to-back steps over four
    tensors (setting T, plus one tensor with s != w, which is not fusable and takes
    the two-call path), every gathered layer, secondary and shard bitwise against the
    oracle; with P2P and B = 256 the trace must show the dual kernels."""
    errors = []
    L = len(g)
    roles = [(1, 1), (1, 1), (L, max(L - 1, 0)), (1, 1)]
    parts = [ctx.partition(n, B, w, s, L) for n, (w, s) in zip(sizes, roles)]
    T = []
    for k, (n, p) in enumerate(zip(sizes, parts)):
        Np = p.padded_numel
        sl = p.range(p.s)[1]
        sc, ss = sec_buffers(sl, sl // B)
        T.append({"p": p, "n": n, "primary": torch.empty(p.range(p.w)[1], dtype=torch.bfloat16, device="cuda"),
                  "grad": torch.empty(Np, dtype=torch.bfloat16, device="cuda"), "sec_c": sc, "sec_s": ss,
                  "fwd": torch.empty(Np, dtype=torch.bfloat16, device="cuda"),
                  "bwd": torch.empty(Np, dtype=torch.bfloat16, device="cuda"),
                  "shard": torch.empty(p.range(L)[1], dtype=torch.float32, device="cuda")})
    if p2p:
        hz.trace_begin(capacity=4096, events=False, stamps=True)
    for step in range(2):
        want = []
        for k, t in enumerate(T):
            p, n, Np = t["p"], t["n"], t["p"].padded_numel
            fr = np.zeros(Np, np.float32)
            fr[:n] = synth.params_like(n, 500 + 10 * step + k, block=B)
            fr = fr.astype(ml_dtypes.bfloat16)
            gr = {}
            for r in range(world):
                x = np.zeros(Np, np.float32)
                x[:n] = synth.gradient_like(n, 1500 + 100 * step + 10 * k + r, block=B)
                gr[r] = x.astype(ml_dtypes.bfloat16)
            off, ln = p.range(p.w)
            t["primary"].copy_(to_dev(fr[off:off + ln]))
            t["grad"].copy_(to_dev(gr[rank]))
            prim = {r: fr[pm.range_at(r, g, Np, p.w)[0]:sum(pm.range_at(r, g, Np, p.w))] for r in range(world)}
            f, sec = col.allgather_forward(prim, g, Np, B, p.w, p.s, bits=8)
            want.append((f[rank], sec[rank], col.reduce_scatter(gr, g, Np, B, 1, L, {l: 4 for l in range(1, L + 1)})[rank]))
        torch.cuda.synchronize()
        n = len(T)
        for k, t in enumerate(T):
            nx = T[k + 1] if k + 1 < n else None
            ctx.allgather_params_next(t["p"], t["primary"], t["sec_c"], t["sec_s"], t["fwd"], bits=8,
                                      p_next=nx["p"] if nx else None, next_primary=nx["primary"] if nx else None,
                                      next_sec_codes=nx["sec_c"] if nx else None,
                                      next_sec_scales=nx["sec_s"] if nx else None)
        ctx.allgather_params(T[-1]["p"], None, T[-1]["sec_c"], T[-1]["sec_s"], T[-1]["bwd"], bits=8, backward=True)
        for k in range(n - 1, -1, -1):
            t, pv = T[k], (T[k - 1] if k > 0 else None)
            ctx.backward_step(t["p"], t["grad"], t["shard"], [4] * L, p_prev=pv["p"] if pv else None,
                              prev_sec_codes=pv["sec_c"] if pv else None, prev_sec_scales=pv["sec_s"] if pv else None,
                              prev_full_out=pv["bwd"] if pv else None, prev_bits=8)
        torch.cuda.synchronize()
        try:
            for k, t in enumerate(T):
                what = f"[{tag}] g={g} pipelined step {step} tensor {k} (w,s)={roles[k]}"
                assert_bitwise(to_host(t["fwd"]), want[k][0], what + " forward layer")
                assert_bitwise(to_host(t["bwd"]), want[k][0], what + " backward layer")
                assert_bitwise(to_host(t["sec_c"]), quant.wire_codes(want[k][1][0], 8), what + " secondary codes")
                assert_bitwise(to_host(t["sec_s"]), want[k][1][1], what + " secondary scales")
                assert_bitwise(to_host(t["shard"]), want[k][2], what + " qgZ shard")
        except AssertionError as e:
            errors.append(str(e))
    # an abandoned prefetch: the next layer's quantize is prefetched, then another
    # collective runs first (the library completes the orphan phase); the next
    # layer's own call quantizes again — no hang, same results
    ctx.allgather_params_next(T[0]["p"], T[0]["primary"], T[0]["sec_c"], T[0]["sec_s"], T[0]["fwd"], bits=8,
                              p_next=T[1]["p"], next_primary=T[1]["primary"], next_sec_codes=T[1]["sec_c"],
                              next_sec_scales=T[1]["sec_s"])
    ctx.reduce_scatter_grads(T[0]["p"], T[0]["grad"], T[0]["shard"], [4] * L)
    ctx.allgather_params(T[1]["p"], T[1]["primary"], T[1]["sec_c"], T[1]["sec_s"], T[1]["fwd"], bits=8)
    torch.cuda.synchronize()
    try:
        assert_bitwise(to_host(T[0]["fwd"]), want[0][0], f"[{tag}] g={g} abandoned prefetch: forward layer 0")
        assert_bitwise(to_host(T[1]["fwd"]), want[1][0], f"[{tag}] g={g} abandoned prefetch: forward layer 1")
        assert_bitwise(to_host(T[0]["shard"]), want[0][2], f"[{tag}] g={g} abandoned prefetch: qgZ shard 0")
    except AssertionError as e:
        errors.append(str(e))
    if p2p:
        hz.trace_end()
        kinds = [r["kind"] for r in hz.trace_read()]
        # per step: forward pairs (0,1) fused; (1,2) not (tensor 2 has s != w); backward pairs
        # (3,2), (2,1), (1,0): the gather side is any layout -> all three fused
        # backward calls (2,1) and (1,0) also carry the previous call's deferred last qgZ
        # hop (fp32 shard) when that hop's group has 2 or 4 members: the triple kernel
        paired = kinds.count("gather_quantize") + kinds.count("gather_quantize_reduce")
        if B == 256 and not os.environ.get("HZ_TUNE") and paired != 2 * 4 + 1:
            errors.append(f"[{tag}] g={g} pipelined: expected 9 paired launches, trace {kinds}")
        triples = 2 * 2 if g[-1] in (2, 4) else 0
        if B == 256 and not os.environ.get("HZ_TUNE") and kinds.count("gather_quantize_reduce") != triples:
            errors.append(f"[{tag}] g={g} pipelined: expected {triples} backward triple launches, trace {kinds}")
    return errors


def check_step_host(ctx, hz, rank, world, g, sec_buffers, tag, B, sizes=(150_001, 70_000, 4097)):
    """hz_step_host (host-staged executor): three tensors of different sizes, two
    back-to-back calls with different host inputs and host shard buffers, no sync
    in between (the second call's uploads overlap the first call's downloads).
    Every host shard must equal the oracle's qgZ shard of its own call's inputs, and
    the gathered buffers the oracle's forward gather of the last two tensors."""
    errors = []
    L = len(g)
    parts = [ctx.partition(n, B, 1, 1, L) for n in sizes]
    Nmax = max(p.padded_numel for p in parts)
    full = [torch.empty(Nmax, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    dev = []
    for p in parts:
        sl = p.range(1)[1]
        sc, ss = sec_buffers(sl, sl // B)
        dev.append({"p": p, "d_primary": torch.empty(p.range(1)[1], dtype=torch.bfloat16, device="cuda"),
                    "d_grad": torch.empty(p.padded_numel, dtype=torch.bfloat16, device="cuda"),
                    "sec_codes": sc, "sec_scales": ss,
                    "d_shard": torch.empty(p.range(L)[1], dtype=torch.float32, device="cuda")})
    calls = []
    for c in range(2):
        io, want = [], []
        for k, (n, p, d) in enumerate(zip(sizes, parts, dev)):
            Np = p.padded_numel
            fr = np.zeros(Np, np.float32)
            fr[:n] = synth.params_like(n, 300 + 10 * c + k, block=B)
            fr = fr.astype(ml_dtypes.bfloat16)
            gr = {}
            for r in range(world):
                x = np.zeros(Np, np.float32)
                x[:n] = synth.gradient_like(n, 900 + 100 * c + 10 * k + r, block=B)
                gr[r] = x.astype(ml_dtypes.bfloat16)
            off, ln = p.range(1)
            prim = {r: fr[pm.range_at(r, g, Np, 1)[0]:sum(pm.range_at(r, g, Np, 1))] for r in range(world)}
            h_primary = torch.from_numpy(fr[off:off + ln].view(np.uint16).copy()).view(torch.bfloat16).pin_memory()
            h_grad = torch.from_numpy(gr[rank].view(np.uint16).copy()).view(torch.bfloat16).pin_memory()
            h_shard = torch.full((p.range(L)[1],), float("nan"), dtype=torch.float32).pin_memory()
            io.append(dict(d, h_primary=h_primary, h_grad=h_grad, h_shard=h_shard))
            want.append((col.allgather_forward(prim, g, Np, B, 1, 1, bits=8)[0][rank],
                         col.reduce_scatter(gr, g, Np, B, 1, L, {l: 4 for l in range(1, L + 1)})[rank]))
        calls.append((ctx.step_host_args(io, [4] * L), io, want))
    st = torch.cuda.current_stream()
    for args, _, _ in calls:
        ctx.step_host(args, full, qwz_bits=8, stream=st)
    torch.cuda.synchronize()
    try:
        for c, (_, io, want) in enumerate(calls):
            for k, t in enumerate(io):
                assert_bitwise(t["h_shard"].numpy(), want[k][1], f"[{tag}] g={g} step_host call {c} tensor {k} shard")
        last = calls[-1][2]
        for k in (0, 1):   # full_out[k % 2] last written by tensor k's backward gather (tensors run n-1..0)
            Np = parts[k].padded_numel
            assert_bitwise(to_host(full[k][:Np]), last[k][0], f"[{tag}] g={g} step_host gathered tensor {k}")
    except AssertionError as e:
        errors.append(str(e))
    return errors


def check_full_size(hz, rank, world, g, uid, device, numel, p2p, B=256, vctx=None):
    """The bench configuration (GPT layer size, setting T w=s=1, gl=L, int8 qwZ, int4
    qgZ) checked on sampled blocks: every output block depends only on the same global
    block of the inputs, and the qgZ reduction tree does not depend on the block's
    position, so the oracle runs on a small layer made of the sampled blocks only.
    vctx: a virtual-world context (P2P; its pool must hold 2.5*Np + 64 MiB: the
    secondary and one qgZ send buffer per level)."""
    errors = []
    virtual = vctx is not None
    tag = "vworld" if virtual else ("p2p" if p2p else "nccl")
    ctx = vctx if virtual else hz.Context(rank, world, uid, g, device)
    p2p = p2p or virtual
    L = len(g)
    try:
        p = ctx.partition(numel, B, 1, 1, L)
        Np = p.padded_numel
        if p2p and not virtual:
            ctx.enable_p2p(3 * Np + (64 << 20))
        off, ln = p.range(1)
        nb = Np // B
        bounds = sorted({pm.range_at(r, g, Np, l)[0] // B for r in range(world) for l in range(L + 1)})
        idx = synth.sample_blocks(nb, bounds, every=499)
        it = torch.from_numpy(idx).cuda()
        pick = lambda t: to_host(t.view(nb, B)[it].contiguous().view(-1))   # noqa: E731
        full = synth.torch_normal(Np, 7000, 0.02, torch.bfloat16, "cuda", outlier_every=0)
        full[numel:] = 0
        picked = {}
        grad = None
        for q in range(world):                       # every rank can regenerate every gradient
            gq = synth.torch_normal(Np, 900 + q, 1e-3, torch.bfloat16, "cuda")
            gq[numel:] = 0
            picked[q] = pick(gq)
            if q == rank:
                grad = gq
            else:
                del gq
        if p2p:
            sec_c, sec_s = ctx.sym_alloc(ln, torch.uint8), ctx.sym_alloc(ln // B, torch.float32)
        else:
            sec_c = torch.empty(ln, dtype=torch.uint8, device="cuda")
            sec_s = torch.empty(ln // B, dtype=torch.float32, device="cuda")
        fwd = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        bwd = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        shard = torch.empty(p.range(L)[1], dtype=torch.float32, device="cuda")
        ctx.allgather_params(p, full[off:off + ln].contiguous(), sec_c, sec_s, fwd, bits=8)
        ctx.allgather_params(p, None, sec_c, sec_s, bwd, bits=8, backward=True)
        ctx.reduce_scatter_grads(p, grad, shard, [4] * L)
        torch.cuda.synchronize()

        xs = pick(full)
        want = quant.dequantize(*quant.quantize(xs, 8, B), B, out="bf16")
        for name, t in (("forward", fwd), ("backward", bwd)):
            try:
                assert_bitwise(pick(t), want, f"[{tag}] g={g} full-size {name} layer ({len(idx)} sampled blocks)")
            except AssertionError as e:
                errors.append(str(e))
        del fwd, bwd, full, grad
        # qgZ: a small layer made of the sampled blocks, same hierarchy and bits
        ns = len(idx)
        tnp = pm.padded_numel(ns * B, g, B)
        tiny = {}
        for q in range(world):
            a = np.zeros(tnp, np.float32).astype(ml_dtypes.bfloat16)
            a[:ns * B] = picked[q]
            tiny[q] = a
        tout = col.reduce_scatter(tiny, g, tnp, B, 1, L, {l: 4 for l in range(1, L + 1)})
        tflat = np.zeros(tnp, np.float32)
        for q in range(world):
            o, n_ = pm.range_at(q, g, tnp, L)
            tflat[o:o + n_] = tout[q]
        my_off, my_len = p.range(L)
        sh = to_host(shard)
        checked = 0
        for i, b in enumerate(idx):
            e0 = int(b) * B
            if my_off <= e0 < my_off + my_len:
                got = sh[e0 - my_off:e0 - my_off + B]
                ref = tflat[i * B:(i + 1) * B]
                if not np.array_equal(got.view(np.uint32), ref.view(np.uint32)):
                    errors.append(f"[{tag}] g={g} full-size qgZ block {b}: mismatch")
                    break
                checked += 1
        assert checked > 0 or world > 8
    finally:
        if not virtual:
            ctx.close()
    return errors


def check_full_size_paired(hz, rank, world, g, numel, vctx, B=256, layers=3):
    """The bench's PAIRED call sequence at full layer size (P2P): three layers of `numel`
    through hz_allgather_params_next (dual kernels), the first backward gather, and
    hz_backward_step with the previous layer (dual kernel, then the backward triple
    kernel carrying the deferred last hop, then the final flush) — every layer's forward
    and backward gathered layer and qgZ shard checked on sampled blocks against the
    oracle (block locality, as check_full_size)."""
    errors = []
    ctx = vctx
    L = len(g)
    p = ctx.partition(numel, B, 1, 1, L)
    Np = p.padded_numel
    off, ln = p.range(1)
    nb = Np // B
    bounds = sorted({pm.range_at(r, g, Np, l)[0] // B for r in range(world) for l in range(L + 1)})
    idx = synth.sample_blocks(nb, bounds, every=997)
    it = torch.from_numpy(idx).cuda()
    pick = lambda t: to_host(t.view(nb, B)[it].contiguous().view(-1))   # noqa: E731
    T = []
    for k in range(layers):
        full = synth.torch_normal(Np, 7100 + k, 0.02, torch.bfloat16, "cuda", outlier_every=0)
        full[numel:] = 0
        picked = {}
        grad = None
        for q in range(world):
            gq = synth.torch_normal(Np, 1900 + 10 * k + q, 1e-3, torch.bfloat16, "cuda")
            gq[numel:] = 0
            picked[q] = pick(gq)
            if q == rank:
                grad = gq
            else:
                del gq
        T.append({"prim": full[off:off + ln].contiguous(), "want_w": pick(full), "picked": picked, "grad": grad,
                  "sec_c": ctx.sym_alloc(ln, torch.uint8), "sec_s": ctx.sym_alloc(ln // B, torch.float32),
                  "fwd": torch.empty(Np, dtype=torch.bfloat16, device="cuda"),
                  "bwd": torch.empty(Np, dtype=torch.bfloat16, device="cuda"),
                  "shard": torch.empty(p.range(L)[1], dtype=torch.float32, device="cuda")})
        del full
    for k, t in enumerate(T):
        nx = T[k + 1] if k + 1 < layers else None
        ctx.allgather_params_next(p, t["prim"], t["sec_c"], t["sec_s"], t["fwd"], bits=8,
                                  p_next=p if nx else None, next_primary=nx["prim"] if nx else None,
                                  next_sec_codes=nx["sec_c"] if nx else None,
                                  next_sec_scales=nx["sec_s"] if nx else None)
    ctx.allgather_params(p, None, T[-1]["sec_c"], T[-1]["sec_s"], T[-1]["bwd"], bits=8, backward=True)
    for k in range(layers - 1, -1, -1):
        t, pv = T[k], (T[k - 1] if k > 0 else None)
        ctx.backward_step(p, t["grad"], t["shard"], [4] * L, p_prev=p if pv else None,
                          prev_sec_codes=pv["sec_c"] if pv else None, prev_sec_scales=pv["sec_s"] if pv else None,
                          prev_full_out=pv["bwd"] if pv else None, prev_bits=8)
    torch.cuda.current_stream().synchronize()
    ns = len(idx)
    tnp = pm.padded_numel(ns * B, g, B)
    my_off, my_len = p.range(L)
    for k, t in enumerate(T):
        want = quant.dequantize(*quant.quantize(t["want_w"], 8, B), B, out="bf16")
        for name in ("fwd", "bwd"):
            try:
                assert_bitwise(pick(t[name]), want, f"[vworld] g={g} paired full-size layer {k} {name}")
            except AssertionError as e:
                errors.append(str(e))
        tiny = {}
        for q in range(world):
            a = np.zeros(tnp, np.float32).astype(ml_dtypes.bfloat16)
            a[:ns * B] = t["picked"][q]
            tiny[q] = a
        tout = col.reduce_scatter(tiny, g, tnp, B, 1, L, {l: 4 for l in range(1, L + 1)})
        tflat = np.zeros(tnp, np.float32)
        for q in range(world):
            o, n_ = pm.range_at(q, g, tnp, L)
            tflat[o:o + n_] = tout[q]
        sh = to_host(t["shard"])
        for i, b in enumerate(idx):
            e0 = int(b) * B
            if my_off <= e0 < my_off + my_len:
                if not np.array_equal(sh[e0 - my_off:e0 - my_off + B].view(np.uint32),
                                      tflat[i * B:(i + 1) * B].view(np.uint32)):
                    errors.append(f"[vworld] g={g} paired full-size layer {k} qgZ block {b}: mismatch")
                    break
    return errors


def run(rank, world, local, bcast=None):
    from paper_2501_04266_b200 import hz
    torch.cuda.set_device(local)
    errors = []
    for g in HIERARCHIES[world]:
        for p2p in (False, True):
            uid = hz.get_uid() if rank == 0 else None
            if bcast is not None:
                uid = bcast(uid)
            errors += check_hierarchy(hz, rank, world, g, uid, local, p2p=p2p)
    # other block sizes through the fused P2P gather (its tile-scale fast path differs for B != 256)
    for B in (64, 1024):
        uid = hz.get_uid() if rank == 0 else None
        if bcast is not None:
            uid = bcast(uid)
        errors += check_hierarchy(hz, rank, world, HIERARCHIES[world][0], uid, local, numel=90_001, B=B, p2p=True)
    # bench configuration at GPT-1.3B layer size, first hierarchy of this world size
    numel = synth.layer_numel(synth.GPT_CONFIGS["gpt1.3b"]["hidden"])
    for p2p in (False, True):
        uid = hz.get_uid() if rank == 0 else None
        if bcast is not None:
            uid = bcast(uid)
        errors += check_full_size(hz, rank, world, HIERARCHIES[world][0], uid, local, numel, p2p)
    return errors


def main():
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")

    def bcast(obj):
        box = [obj]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    errors = run(rank, world, local, bcast)
    for e in errors:
        print(f"[rank {rank}] {e}", flush=True)
    n = torch.tensor([len(errors)])
    dist.all_reduce(n)
    dist.destroy_process_group()
    if rank == 0:
        print(f"mp_parity world={world}: {int(n)} failures", flush=True)
    sys.exit(1 if int(n) else 0)


if __name__ == "__main__":
    main()
