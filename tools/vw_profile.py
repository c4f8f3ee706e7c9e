#!/usr/bin/env python
"""One-process multi-GPU driver of the P2P exchange kernels, for ncu (tool, not product).

A virtual world (hz_init_virtual_ex) with rank r on GPU r % ngpu: the same contexts,
pools, flags and kernels as a W-process run, but every kernel starts only after the
kernels it waits for have completed (host-ordered launches, csrc/vworld.cpp).  A
profiler that serialises and replays launches (ncu) therefore never sees a kernel spin
on a peer that cannot run — which is why ncu may not wrap the multi-process bench.
Each rank issues bench.py's pipelined step (Model.step: the paired gather || quantize
kernels forward, gather || qgZ backward) over ``--layers`` GPT layers.  The gathers read
the partner's codes over NVLink; since the partner is idle while a kernel runs, the
link carries one direction at a time (ncu's per-kernel view; the concurrent bidirectional
case is the bench's).

    python tools/vw_profile.py --gpus 2 [--config gpt1.3b] [--layers 3] [--steps 2] [--time]
    HZ_TUNE=vwserial=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\\
        nvlrx__bytes.sum,nvltx__bytes.sum -k regex:k_ python tools/vw_profile.py --gpus 2

Under ncu set HZ_TUNE=vwserial=1: every synchronised launch then runs alone (ncu restores a
GPU's memory between replay passes of one of its kernels; a peer kernel running meanwhile
would have its flag writes into that memory reverted).
"""

import argparse
import json
import math
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--hierarchy", default="")
    ap.add_argument("--config", default="gpt1.3b")
    ap.add_argument("--layers", type=int, default=3)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--block", type=int, default=256)
    ap.add_argument("--qwz-bits", type=int, default=8)
    ap.add_argument("--qgz-bits", type=int, default=4)
    ap.add_argument("--roles", default="1,1")
    ap.add_argument("--no-pipelined", dest="pipelined", action="store_false")
    ap.add_argument("--time", action="store_true", help="print per-rank wall time per step (host-ordered: not a bench)")
    args = ap.parse_args()
    import torch

    import bench
    from paper_2501_04266_b200 import hz, synth
    from tests import vworld

    g = tuple(int(x) for x in args.hierarchy.split(",")) if args.hierarchy else (
        (2,) if args.gpus == 2 else (2, 2) if args.gpus == 4 else (2, 2, 2) if args.gpus == 8 else (args.gpus,))
    W = math.prod(g)
    ndev = torch.cuda.device_count()
    if ndev < args.gpus:
        raise SystemExit(f"needs {args.gpus} GPUs, have {ndev}")
    devices = [r % args.gpus for r in range(W)]
    w, s = (int(x) for x in args.roles.split(","))
    margs = types.SimpleNamespace(block=args.block, w=w, s=s, qwz_bits=args.qwz_bits, qgz_bits=args.qgz_bits,
                                  pipelined=args.pipelined, layers=args.layers)
    tensors = synth.model_tensors(args.config)[:args.layers]
    pool = bench.p2p_pool_bytes(types.SimpleNamespace(config=args.config, block=args.block, w=w, s=s,
                                                      qwz_bits=args.qwz_bits), g)
    out = {}

    def fn(r, world, ctx):
        model = bench.Model(hz, ctx, torch, args.config, r, world, margs, f"cuda:{ctx.device}")
        st = torch.cuda.current_stream()
        times = []
        for _ in range(args.steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            model.step(st)
            e1.record(st)
            st.synchronize()
            times.append(e0.elapsed_time(e1))
        out[r] = times
        return []

    errors = vworld.run_ranks(hz, g, fn, pool_bytes=pool, devices=devices, timeout_s=600.0)
    if errors:
        print("\n".join(errors[:20]), file=sys.stderr)
        raise SystemExit(1)
    rec = {"tool": "vw_profile", "hierarchy": list(g), "devices": devices, "config": args.config,
           "layers": len(tensors), "steps": args.steps, "ok": True}
    if args.time:
        rec["ms_per_step_by_rank"] = {r: [round(x, 3) for x in v] for r, v in sorted(out.items())}
    print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
