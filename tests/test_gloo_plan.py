"""Multi-process CPU tests of the N>1 host logic (gloo, world size 2, 4 and 8).

Each process is one rank.  It asks libhz for its partition (hz_partition_ex) and
its communication plans (hz_plan_allgather / hz_plan_reduce_scatter — the plans
the NCCL engine issues its calls from), executes those plans with gloo
transport (all_gather on per-level subgroups, isend/irecv pairs) and the
oracle's codec arithmetic, and checks that
  * every step's offsets / sizes agree with the peers' steps (send_off of the
    sender == recv_off of the receiver, all-gather pieces tile range_{l-1}),
  * the executed result equals the oracle's single-process simulation bit for
    bit (forward / backward gathered layer, secondary, qgZ shard),
  * the bytes the plan moves equal the paper's per-level volumes (O10).
No GPU is involved."""

import os
import socket

import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _t(a):
    import numpy as np
    a = np.ascontiguousarray(a)
    if a.dtype == np.int8:
        return torch.from_numpy(a.copy())
    return torch.from_numpy(a.astype(np.float32))


def _worker(rank, world, port, hierarchies, errq):
    import ml_dtypes
    import numpy as np

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import collectives as col
        from oracle import partition as pm
        from oracle import quant, volume
        from paper_2501_04266_b200 import hz, synth

        for g in hierarchies:
            L = len(g)
            # one subgroup per exchange group per level, created in the same order everywhere
            groups = {}
            for level in range(1, L + 1):
                seen = set()
                for r in range(world):
                    mem = tuple(pm.exchange_group(r, g, level))
                    if mem not in seen:
                        seen.add(mem)
                        groups[(level, mem)] = dist.new_group(list(mem)) if len(mem) > 1 else None
            B, numel = 32, 4099
            for w, s in sorted({(1, 1), (L, max(L - 1, 0)), (1, L), (0, 0)}):
                p = hz.partition_ex(rank, g, numel, B, w, s, L)
                Np = p.padded_numel
                full = np.zeros(Np, np.float32)
                full[:numel] = synth.params_like(numel, 11, block=B)
                full = full.astype(ml_dtypes.bfloat16)
                prim = {r: full[pm.range_at(r, g, Np, w)[0]:sum(pm.range_at(r, g, Np, w))] for r in range(world)}
                want, want_sec = col.allgather_forward(prim, g, Np, B, w, s, bits=8)
                for backward in (False, True):
                    plan = hz.plan_allgather(p, backward, 8)
                    top = s if backward else w
                    off, ln = p.range(top)
                    if backward:
                        codes, scales = want_sec[rank]          # start from the secondary
                    else:
                        codes, scales = quant.quantize(full[off:off + ln], 8, B)
                    cur_off = off
                    sent = 0
                    for st in plan:
                        assert st["op"] == hz.PLAN_ALLGATHER
                        assert st["send_off"] == cur_off and st["elems"] == len(codes)
                        mem = tuple(pm.exchange_group(rank, g, st["level"]))
                        assert st["group"] == len(mem)
                        grp = groups[(st["level"], mem)]
                        meta = [torch.zeros(2, dtype=torch.int64) for _ in mem]
                        dist.all_gather(meta, torch.tensor([st["send_off"], st["elems"]]), group=grp)
                        for k, m in enumerate(meta):               # pieces tile range_{l-1} in digit order
                            assert int(m[0]) == st["recv_off"] + k * st["elems"] and int(m[1]) == st["elems"]
                        cs = [torch.zeros(len(codes), dtype=torch.int8) for _ in mem]
                        ss = [torch.zeros(len(scales), dtype=torch.float32) for _ in mem]
                        dist.all_gather(cs, _t(codes), group=grp)
                        dist.all_gather(ss, _t(scales), group=grp)
                        codes = np.concatenate([c.numpy() for c in cs])
                        scales = np.concatenate([x.numpy() for x in ss])
                        cur_off = st["recv_off"]
                        sent += (st["group"] - 1) * st["code_bytes"]       # received per rank
                    assert cur_off == 0 and len(codes) == Np
                    out = quant.dequantize(codes, scales, B, out="bf16")
                    if not np.array_equal(out.view(np.uint16), want[rank].view(np.uint16)):
                        raise AssertionError(f"g={g} w={w} s={s} bwd={backward}: gathered layer differs")
                    D = pm.world_of(g[:top])
                    assert sent == volume.qwz_allgather_bytes(Np, D, 8)     # Table VII with d = D

            # qgZ through the reduce-scatter plan
            Np = pm.padded_numel(numel, g, B)
            grads = {r: synth.gradient_like(Np, 60 + r, block=B).astype(ml_dtypes.bfloat16) for r in range(world)}
            for bits in ([4] * L, [8] + [4] * (L - 1)):
                p = hz.partition_ex(rank, g, numel, B, 1, 1, L)
                plan = hz.plan_reduce_scatter(p, bits)
                want = col.reduce_scatter(grads, g, Np, B, 1, L, {l: bits[l - 1] for l in range(1, L + 1)})
                codes, scales = quant.quantize(grads[rank], bits[0], B)
                base = 0
                sent = 0
                for level in range(1, L + 1):
                    d = p.digit[level - 1]
                    ln = p.len[level]
                    steps = [st for st in plan if st["level"] == level]
                    assert len(steps) == g[level - 1] - 1
                    contrib = {d: (codes[d * ln:(d + 1) * ln], scales[d * ln // B:(d + 1) * ln // B])}
                    reqs, bufs = [], {}
                    for st in steps:
                        rel = st["send_off"] - base
                        assert rel == st["peer"] * ln and st["recv_off"] == p.off[level]
                        mine = torch.tensor([st["send_off"], st["elems"], st["bits"]])
                        theirs = torch.zeros(3, dtype=torch.int64)
                        bc = torch.zeros(ln, dtype=torch.int8)
                        bs = torch.zeros(ln // B, dtype=torch.float32)
                        reqs += [dist.isend(mine, st["peer_rank"]), dist.irecv(theirs, st["peer_rank"]),
                                 dist.isend(_t(codes[rel:rel + ln]), st["peer_rank"]), dist.irecv(bc, st["peer_rank"]),
                                 dist.isend(_t(scales[rel // B:(rel + ln) // B]), st["peer_rank"]),
                                 dist.irecv(bs, st["peer_rank"])]
                        bufs[st["peer"]] = (theirs, bc, bs)
                        sent += st["code_bytes"]
                        assert st["code_bytes"] == ln * bits[level - 1] // 8
                    for rq in reqs:
                        rq.wait()
                    for j, (theirs, bc, bs) in bufs.items():
                        assert int(theirs[0]) == p.off[level] and int(theirs[1]) == ln   # matching send
                        contrib[j] = (bc.numpy(), bs.numpy())
                    coded = [contrib[j] for j in range(g[level - 1])]
                    if level < L:
                        codes, scales = col.reduce_coded(coded, B, bits_out=bits[level])
                    else:
                        shard = col.reduce_coded(coded, B)
                    base = p.off[level]
                if not np.array_equal(shard.view(np.uint32), want[rank].view(np.uint32)):
                    raise AssertionError(f"g={g} bits={bits}: qgZ shard differs")
                exp = sum(volume.hierarchical_level_bytes(Np, g, l, bits[l - 1]) for l in range(1, L + 1))
                assert sent == exp
        dist.barrier()
    except Exception as e:  # report to the parent
        import traceback
        errq.put(f"rank {rank}: {e}\n{traceback.format_exc()}")
    finally:
        dist.destroy_process_group()


def _run(world, hierarchies):
    from paper_2501_04266_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    errq = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, hierarchies, errq)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=600)
    errors = []
    while not errq.empty():
        errors.append(errq.get())
    assert not errors, "\n".join(errors)
    assert all(pr.exitcode == 0 for pr in procs)


def test_gloo_world2():
    _run(2, [(2,), (1, 2)])


def test_gloo_world4():
    _run(4, [(2, 2), (4,), (2, 1, 2)])


def test_gloo_world8():
    """The bench's eight-GPU hierarchies ((2,4) for GPT-1.3B, (2,2,2) for 6.7B / 20B)."""
    _run(8, [(2, 4), (2, 2, 2)])
