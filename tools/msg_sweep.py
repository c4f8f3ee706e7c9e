#!/usr/bin/env python
"""Message-size sweep (BASELINE.json config 5): the hierarchical
qwZ/hpZ all-gather (forward and backward) and qgZ reduce-scatter of one tensor of
1 MB .. 2 GB logical bf16 bytes (powers of two), next to the flat ZeRO-3 baseline
(NCCL bf16 all-gather / reduce-scatter on the world communicator, same logical bytes).

Timing discipline (§8(d)): 5 warm-up iterations, then ``--iters`` (>= 20) timed, each
preceded by a device synchronize + world barrier and bracketed by CUDA events on the
issuing stream; per-iteration times are max-reduced over ranks, then the median and
p10/p90 are reported; ``ms_loop`` is the per-call time of ``--iters`` calls issued
back to back after one barrier (the steady state of a stream of collectives).
Wire bytes per rank come from one stamps-only traced call
(the library's ``remote_bytes``, peer bytes read per rank); flat NCCL wire bytes are
(W-1)/W of the message.

    python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 \\
        tools/msg_sweep.py [--min-mb 1] [--max-mb 2048] [--iters 20] [--transport p2p]
Rank 0 prints one JSON line per (size, op).
"""

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

HIER = {2: (2,), 4: (2, 2), 8: (2, 2, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-mb", type=int, default=1)
    ap.add_argument("--max-mb", type=int, default=2048)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--block", type=int, default=256)
    ap.add_argument("--qgz-bits", type=int, default=4)
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p")
    ap.add_argument("--hierarchy", default="", help="e.g. 2,4 (default: 2 / 2,2 / 2,2,2)")
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from paper_2501_04266_b200 import hz

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world < 2:
        raise SystemExit("run under torchrun with >= 2 ranks")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("gloo")
    group = tuple(int(g) for g in args.hierarchy.split(",")) if args.hierarchy else HIER[world]
    assert math.prod(group) == world
    B, L = args.block, len(group)

    uid = hz.get_uid() if rank == 0 else None
    box = [uid]
    dist.broadcast_object_list(box, src=0)
    ctx = hz.Context(rank, world, box[0], group, local)

    sizes = []
    mb = args.min_mb
    while mb <= args.max_mb:
        sizes.append(mb << 20)
        mb *= 2
    pmax = ctx.partition(sizes[-1] // 2, B, 1, 1, L)
    Npm = pmax.padded_numel
    _, len_wm = pmax.range(1)
    _, len_lm = pmax.range(L)
    p2p = args.transport == "p2p"
    if p2p:
        ctx.enable_p2p(len_wm + len_wm // B * 4 + 2 * (L + 1) * (Npm + Npm // B * 4 + 512) + (64 << 20))
    sec_c = ctx.sym_alloc(len_wm, torch.uint8) if p2p else torch.empty(len_wm, dtype=torch.uint8, device=dev)
    sec_s = (ctx.sym_alloc(len_wm // B, torch.float32) if p2p
             else torch.empty(len_wm // B, dtype=torch.float32, device=dev))
    full = torch.empty(Npm, dtype=torch.bfloat16, device=dev)
    grad = torch.empty(Npm, dtype=torch.bfloat16, device=dev).normal_(0, 1e-3)
    prim = torch.empty(len_wm, dtype=torch.bfloat16, device=dev).normal_(0, 0.02)
    shard = torch.empty(len_lm, dtype=torch.float32, device=dev)
    fchunk = torch.empty(Npm // world, dtype=torch.bfloat16, device=dev).normal_(0, 0.02)
    frs = torch.empty(Npm // world, dtype=torch.bfloat16, device=dev)
    stream = torch.cuda.current_stream()
    bits = [args.qgz_bits] * L

    def ops_for(S):
        n = S // 2
        p = ctx.partition(n, B, 1, 1, L)
        Np = p.padded_numel
        _, len_w = p.range(1)
        fn = Np // world
        return {
            "hz_allgather_fwd": lambda: ctx.allgather_params(p, prim[:len_w], sec_c, sec_s, full[:Np], bits=8,
                                                             stream=stream),
            "hz_allgather_bwd": lambda: ctx.allgather_params(p, None, sec_c, sec_s, full[:Np], bits=8,
                                                             backward=True, stream=stream),
            "hz_reduce_scatter": lambda: ctx.reduce_scatter_grads(p, grad[:Np], shard, bits, stream=stream),
            "flat_allgather": lambda: ctx.flat_allgather(fchunk[:fn], full[:Np], stream=stream),
            "flat_reduce_scatter": lambda: ctx.flat_reduce_scatter(grad[:Np], frs[:fn], stream=stream),
        }

    lines = []
    for S in sizes:
        ops = ops_for(S)
        if "hz_allgather_fwd" in ops:      # the backward gather reads the forward's secondary
            ops["hz_allgather_fwd"]()
        for name, fn in ops.items():
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            wire = None
            if name.startswith("hz"):
                dist.barrier()
                hz.trace_begin(256, events=False, stamps=True)
                fn()
                torch.cuda.synchronize()
                hz.trace_end()
                recs = hz.trace_read()
                wire = sum(r["remote_bytes"] for r in recs)
            else:
                wire = S * (world - 1) // world
            times = []
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            for _ in range(args.iters):
                torch.cuda.synchronize()
                dist.barrier()
                e0.record(stream)
                fn()
                e1.record(stream)
                e1.synchronize()
                times.append(e0.elapsed_time(e1))
            # steady state: --iters calls back to back (no barrier between them), one
            # event pair; the per-call time of a stream of collectives
            torch.cuda.synchronize()
            dist.barrier()
            e0.record(stream)
            for _ in range(args.iters):
                fn()
            e1.record(stream)
            e1.synchronize()
            loop = torch.tensor([e0.elapsed_time(e1) / args.iters], dtype=torch.float64)
            dist.all_reduce(loop, op=dist.ReduceOp.MAX)
            loop_ms = float(loop.item())
            t = torch.tensor(times, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t = sorted(t.tolist())
            med = t[len(t) // 2]
            p10 = t[int(0.1 * (len(t) - 1))]
            p90 = t[int(math.ceil(0.9 * (len(t) - 1)))]
            line = {"bytes": S, "op": name, "n_gpus": world, "hierarchy": list(group),
                    "transport": args.transport if name.startswith("hz") else "nccl",
                    "ms_median": round(med, 4), "ms_p10": round(p10, 4), "ms_p90": round(p90, 4),
                    "ms_loop": round(loop_ms, 4),
                    "algbw_GBps": round(S / (med * 1e-3) / 1e9, 1),
                    "wire_bytes_per_rank": int(wire),
                    "wire_GBps_per_rank": round(wire / (med * 1e-3) / 1e9, 1)}
            lines.append(line)
            if rank == 0:
                print(json.dumps(line), flush=True)
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            for line in lines:
                f.write(json.dumps(line) + "\n")
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
