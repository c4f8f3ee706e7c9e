"""The multi-rank P2P path on ONE GPU: virtual worlds of 2..8 ranks (hz_init_virtual,
tests/vworld.py), every rank driving its own context from its own thread, through
the product's exchange kernels and phase protocol, checked bit for bit against the
oracle's all-ranks simulation — the same checks tests/mp_parity.py runs per process
under torchrun on W GPUs (forward/backward hpZ gathers over multi-piece groups, qgZ
over every hierarchy and hop grouping, two-phase setting T, allreduce+select, AdamW +
post-update gather, the host-staged step, the paired dual kernels), plus the
level-local synchronisation and the abort path."""

import os
import threading
import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

HIERARCHIES = [(2,), (2, 2), (4,), (2, 2, 2), (2, 4), (4, 2), (8,)]


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("g", HIERARCHIES, ids=lambda g: "x".join(map(str, g)))
def test_vworld_hierarchy(g):
    _need_gpu()
    from paper_2501_04266_b200 import hz
    from tests import mp_parity, vworld
    errors = vworld.run_ranks(hz, g, lambda r, w, ctx: mp_parity.check_hierarchy(hz, r, w, g, None, 0, vctx=ctx))
    assert not errors, "\n".join(errors[:20])


@pytest.mark.multigpu
@pytest.mark.parametrize("g", [(2,), (2, 2), (2, 2, 2), (2, 4)], ids=lambda g: "x".join(map(str, g)))
def test_vworld_multi_device(g):
    """hz_init_virtual_ex: rank r on GPU r % ngpu, so pair partners sit on different
    GPUs and every gather / qgZ piece of a partner crosses NVLink (peer access, one
    process); the same bitwise checks as on one GPU."""
    _need_gpu()
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip("needs >= 2 GPUs")
    from paper_2501_04266_b200 import hz
    from tests import mp_parity, vworld
    devices = [r % n for r in range(int(np.prod(g)))]
    errors = vworld.run_ranks(hz, g, lambda r, w, ctx: mp_parity.check_hierarchy(hz, r, w, g, None, 0, vctx=ctx),
                              devices=devices)
    assert not errors, "\n".join(errors[:20])


@pytest.mark.parametrize("B", [64, 1024])
def test_vworld_block_sizes(B):
    _need_gpu()
    from paper_2501_04266_b200 import hz
    from tests import mp_parity, vworld
    g = (2, 2, 2)
    errors = vworld.run_ranks(hz, g, lambda r, w, ctx: mp_parity.check_hierarchy(hz, r, w, g, None, 0, numel=90_001,
                                                                                 B=B, vctx=ctx))
    assert not errors, "\n".join(errors[:20])


@pytest.mark.parametrize("model,g", [("gpt1.3b", (2, 4)), ("gpt1.3b", (2, 2, 2)), ("gpt6.7b", (2, 2, 2)),
                                     ("neox20b", (2, 2, 2))])
def test_vworld_full_size(model, g):
    """BASELINE configs 2-4 at their layer size on the 8-rank hierarchies, sampled-block
    parity (every 499th block and both edge blocks of every chunk boundary)."""
    _need_gpu()
    from paper_2501_04266_b200 import hz, synth
    from tests import mp_parity, vworld
    numel = synth.layer_numel(synth.GPT_CONFIGS[model]["hidden"])
    Np = numel + 8192
    errors = vworld.run_ranks(hz, g, lambda r, w, ctx: mp_parity.check_full_size(hz, r, w, g, None, 0, numel, True,
                                                                                  vctx=ctx),
                              pool_bytes=7 * Np // 2 + (64 << 20))
    torch.cuda.empty_cache()
    assert not errors, "\n".join(errors[:20])


@pytest.mark.parametrize("model,g", [("gpt1.3b", (2, 4)), ("gpt6.7b", (2, 2, 2))])
def test_vworld_full_size_paired(model, g):
    """The bench's paired sequence (dual kernels forward, dual + backward triple kernels
    backward, the deferred last hop) at BASELINE layer size on 8 ranks, sampled-block
    parity for every layer."""
    _need_gpu()
    from paper_2501_04266_b200 import hz, synth
    from tests import mp_parity, vworld
    numel = synth.layer_numel(synth.GPT_CONFIGS[model]["hidden"])
    Np = numel + 8192
    errors = vworld.run_ranks(hz, g, lambda r, w, ctx: mp_parity.check_full_size_paired(hz, r, w, g, numel, ctx),
                              pool_bytes=4 * Np + (64 << 20))
    torch.cuda.empty_cache()
    assert not errors, "\n".join(errors[:20])


def test_vworld_trace_shows_multi_rank_kernels():
    """At W = 8 the pipelined step launches the dual gather+quantize kernels and the
    gathers read remote pieces (remote_bytes > 0) on every rank."""
    _need_gpu()
    from paper_2501_04266_b200 import hz
    from tests import mp_parity, vworld
    g = (2, 2, 2)
    seen = {}

    def fn(r, w, ctx):
        def sec(nc, ns):
            return ctx.sym_alloc(nc, torch.uint8), ctx.sym_alloc(ns, torch.float32)
        errs = mp_parity.check_pipelined(ctx, hz, r, w, g, sec, "vworld", 256, True)
        hz.trace_begin(capacity=256, events=False, stamps=True)
        errs += mp_parity.check_pipelined(ctx, hz, r, w, g, sec, "vworld", 256, False)
        hz.trace_end()
        seen[r] = hz.trace_read()
        return errs

    errors = vworld.run_ranks(hz, g, fn)
    assert not errors, "\n".join(errors[:20])
    for r in range(8):
        kinds = [x["kind"] for x in seen[r]]
        assert "gather_quantize" in kinds, kinds
        assert any(x["kind"] in ("gather_dequantize", "gather_quantize") and x["remote_bytes"] > 0 for x in seen[r])
        assert any(x["kind"].startswith("reduce") and x["remote_bytes"] > 0 for x in seen[r])


def test_vworld_pair_completes_while_nonmember_stalled():
    """Level-local synchronisation: on (2,2), ranks 0 and 1 (a level-1 pair) run
    forward + backward gathers of a pair-sharded layer and the level-1 qgZ while ranks 2
    and 3 have not issued anything; the pair finishes (bitwise vs the oracle) before the
    others start, then 2 and 3 run the same calls."""
    _need_gpu()
    import ml_dtypes
    from oracle import collectives as col
    from oracle import partition as pm
    from paper_2501_04266_b200 import hz, synth
    from tests import vworld
    from tests.gpu_util import assert_bitwise, to_dev, to_host
    g = (2, 2)
    numel, B = 70_001, 256
    Np = pm.padded_numel(numel, g, B)
    full = np.zeros(Np, np.float32)
    full[:numel] = synth.params_like(numel, 11, block=B)
    full = full.astype(ml_dtypes.bfloat16)
    prim = {r: full[pm.range_at(r, g, Np, 1)[0]:sum(pm.range_at(r, g, Np, 1))] for r in range(4)}
    want_f, _ = col.allgather_forward(prim, g, Np, B, 1, 1, bits=8)
    grads = {r: synth.gradient_like(Np, 60 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(4)}
    want_rs = col.reduce_scatter(grads, g, Np, B, 1, 1, {1: 4})
    ctxs = hz.virtual_world(g, pool_bytes=32 << 20)
    for c in ctxs:
        c.set_wait_timeout(60)
    done_at = {}

    def fn(r, w, ctx):
        p = ctx.partition(numel, B, 1, 1, 1)
        sc, ss = ctx.sym_alloc(p.range(1)[1], torch.uint8), ctx.sym_alloc(p.range(1)[1] // B, torch.float32)
        out = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        bwd = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        sh = torch.empty(p.range(1)[1], dtype=torch.float32, device="cuda")
        ctx.allgather_params(p, to_dev(prim[r]), sc, ss, out, bits=8)
        ctx.allgather_params(p, None, sc, ss, bwd, bits=8, backward=True)
        ctx.reduce_scatter_grads(p, to_dev(grads[r]), sh, [4, 4], 1, 1)
        torch.cuda.current_stream().synchronize()
        done_at[r] = time.monotonic()
        errs = []
        try:
            assert_bitwise(to_host(out), want_f[r], f"rank {r} forward")
            assert_bitwise(to_host(bwd), want_f[r], f"rank {r} backward")
            assert_bitwise(to_host(sh), want_rs[r], f"rank {r} level-1 qgZ")
        except AssertionError as e:
            errs.append(str(e))
        return errs

    try:
        errors = vworld.run_ranks(hz, g, fn, ranks=[0, 1], ctxs=ctxs)   # 2 and 3 idle
        assert not errors, "\n".join(errors)
        assert set(done_at) == {0, 1}
        errors = vworld.run_ranks(hz, g, fn, ranks=[2, 3], ctxs=ctxs)
        assert not errors, "\n".join(errors)
    finally:
        torch.cuda.synchronize()
        for c in ctxs:
            c.close()


def test_vworld_timeout_aborts_instead_of_hanging():
    """A rank whose peer never arrives: the wait times out after the configured timeout,
    the context reports HZ_ERR_ABORTED on its next call (no hang, no trap, no sticky CUDA
    error: the device stays usable)."""
    _need_gpu()
    from paper_2501_04266_b200 import hz
    ctxs = hz.virtual_world((2,), pool_bytes=8 << 20)
    try:
        ctxs[0].set_wait_timeout(0.5)
        p = ctxs[0].partition(4096 * 8, 256, 1, 1, 1)
        n = p.range(1)[1]
        sc, ss = ctxs[0].sym_alloc(n, torch.uint8), ctxs[0].sym_alloc(n // 256, torch.float32)
        prim = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
        out = torch.empty(p.padded_numel, dtype=torch.bfloat16, device="cuda")
        t0 = time.monotonic()
        with pytest.raises(hz.HZError) as ei:
            ctxs[0].allgather_params(p, prim, sc, ss, out)    # rank 1 never calls
        assert ei.value.status == hz.ERR_ABORTED
        assert time.monotonic() - t0 < 30
        with pytest.raises(hz.HZError) as ei:
            ctxs[0].check()
        assert ei.value.status == hz.ERR_ABORTED
        torch.cuda.synchronize()                           # the GPU is fine
        assert float(torch.ones(4, device="cuda").sum()) == 4.0
    finally:
        for c in ctxs:
            c.close()


def test_device_wait_timeout_and_abort():
    """The device-side wait (without the virtual world's host ordering, HZ_TUNE vworder=0):
    a kernel spinning for a peer that never signals returns after the timeout and the
    context is aborted; hz_abort from another thread releases a spinning kernel at once."""
    _need_gpu()
    import subprocess
    import sys
    code = r'''
import time, torch, sys
sys.path.insert(0, ".")
from paper_2501_04266_b200 import hz
for mode in ("timeout", "abort"):
    ctxs = hz.virtual_world((2,), pool_bytes=8 << 20)
    c = ctxs[0]
    c.set_wait_timeout(1.0 if mode == "timeout" else 600.0)
    p = c.partition(4096 * 8, 256, 1, 1, 1)
    n = p.range(1)[1]
    sc, ss = c.sym_alloc(n, torch.uint8), c.sym_alloc(n // 256, torch.float32)
    prim = torch.zeros(n, dtype=torch.bfloat16, device="cuda")
    out = torch.empty(p.padded_numel, dtype=torch.bfloat16, device="cuda")
    t0 = time.monotonic()
    c.allgather_params(p, prim, sc, ss, out)      # enqueued; the gather spins on rank 1
    if mode == "abort":
        time.sleep(0.5)
        c.abort()
    torch.cuda.synchronize()
    dt = time.monotonic() - t0
    try:
        c.check()
        print("NOT ABORTED", mode); sys.exit(1)
    except hz.HZError as e:
        assert e.status == hz.ERR_ABORTED, e
    assert dt < 30, dt
    print(mode, "ok", round(dt, 2))
    for x in ctxs:
        x.close()
assert float(torch.ones(4, device="cuda").sum()) == 4.0
print("DONE")
'''
    env = dict(os.environ, HZ_TUNE="vworder=0")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, env=env,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert p.returncode == 0 and "DONE" in p.stdout, p.stdout[-3000:] + p.stderr[-3000:]


def test_step_host_rejects_non_pool_secondaries():
    """P2P transport: hz_step_host validates, before enqueuing anything, that every
    tensor's hpZ secondary is symmetric-pool memory (peers read it in place) — a plain
    device allocation is HZ_ERR_INVALID naming the tensor and field."""
    _need_gpu()
    from paper_2501_04266_b200 import hz
    ctxs = hz.virtual_world((2,), pool_bytes=8 << 20)
    try:
        c = ctxs[0]
        p = c.partition(8192, 256, 1, 1, 1)
        n = p.range(1)[1]
        d = lambda k, dt: torch.empty(k, dtype=dt, device="cuda")
        t = {"p": p, "h_primary": torch.empty(n, dtype=torch.bfloat16).pin_memory(), "d_primary": d(n, torch.bfloat16),
             "h_grad": torch.empty(p.padded_numel, dtype=torch.bfloat16).pin_memory(),
             "d_grad": d(p.padded_numel, torch.bfloat16), "sec_codes": d(n, torch.uint8),
             "sec_scales": d(n // 256, torch.float32), "d_shard": d(n, torch.float32),
             "h_shard": torch.empty(n, dtype=torch.float32).pin_memory()}
        full = [d(p.padded_numel, torch.bfloat16) for _ in range(2)]
        with pytest.raises(hz.HZError) as ei:
            c.step_host([t], full)
        assert ei.value.status == hz.ERR_INVALID and "t[0].sec_codes" in str(ei.value), str(ei.value)
        c.check()                                   # nothing enqueued, context healthy
    finally:
        torch.cuda.synchronize()
        for x in ctxs:
            x.close()


def test_deferred_last_hop_completes_on_flush():
    """hz_backward_step with a previous layer defers the last qgZ hop (P2P, B = 256): the
    shard is not written by that call; hz_flush (or any later call) launches it, and the
    result is bitwise hz_reduce_scatter_grads'.  Checked on (2,) with the trace: no reduce
    launch before the flush, one after."""
    _need_gpu()
    import ml_dtypes
    from oracle import collectives as col
    from oracle import partition as pm
    from paper_2501_04266_b200 import hz, synth
    from tests import vworld
    from tests.gpu_util import assert_bitwise, to_dev, to_host
    g = (2,)
    numel, B = 60_001, 256
    Np = pm.padded_numel(numel, g, B)
    grads = {r: synth.gradient_like(Np, 900 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(2)}
    want = col.reduce_scatter(grads, g, Np, B, 1, 1, {1: 4})
    full = np.zeros(Np, np.float32)
    full[:numel] = synth.params_like(numel, 77, block=B)
    full = full.astype(ml_dtypes.bfloat16)
    got = {}

    def fn(r, w, ctx):
        p = ctx.partition(numel, B, 1, 1, 1)
        n1 = p.range(1)[1]
        sc, ss = ctx.sym_alloc(n1, torch.uint8), ctx.sym_alloc(n1 // B, torch.float32)
        prim = to_dev(full[pm.range_at(r, g, Np, 1)[0]:sum(pm.range_at(r, g, Np, 1))])
        out = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
        ctx.allgather_params(p, prim, sc, ss, out, bits=8)             # the previous layer's secondary
        shard = torch.full((n1,), float("nan"), dtype=torch.float32, device="cuda")
        hz.trace_begin(capacity=64, events=False, stamps=True)
        ctx.backward_step(p, to_dev(grads[r]), shard, [4], p_prev=p, prev_sec_codes=sc, prev_sec_scales=ss,
                          prev_full_out=out, prev_bits=8)
        torch.cuda.current_stream().synchronize()
        hz.trace_end()
        before = [x["kind"] for x in hz.trace_read()]
        pending = bool(torch.isnan(shard).all())
        hz.trace_begin(capacity=64, events=False, stamps=True)
        ctx.flush()
        torch.cuda.current_stream().synchronize()
        hz.trace_end()
        after = [x["kind"] for x in hz.trace_read()]
        got[r] = (before, pending, after, to_host(shard))
        return []

    errors = vworld.run_ranks(hz, g, fn)
    assert not errors, "\n".join(errors)
    for r in range(2):
        before, pending, after, shard = got[r]
        assert "reduce" not in before and pending, (before, pending)
        assert after.count("reduce") == 1, after
        assert_bitwise(shard, want[r], f"rank {r} deferred qgZ shard")
