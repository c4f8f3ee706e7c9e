#!/usr/bin/env python
"""Overlap study: a synthetic ZeRO-topo training step of a GPT
model on B200s — the B200 analog of the paper's TFLOPS/GPU comparison (Fig. 7,
P:46).

Per micro-batch of T tokens and per transformer layer (hidden h), the compute is the
four weight GEMMs of the layer (QKV h->3h, projection h->h, MLP h->4h and 4h->h):
forward 2*T*12h^2 FLOPs, backward twice that (dX and dW), bf16 cuBLAS via torch
(library GEMMs, not the hot path).  Attention itself is left out (it does not touch
the sharded parameters).  The weights each GEMM uses are the layer's gathered
buffer; the dW GEMMs write the layer's gradient buffer that the reduce-scatter
consumes.

Modes (same GEMMs in every mode):
  compute   weights resident, no communication (upper bound)
  hz        this library: qwZ/hpZ gather of layer i+1 prefetched on a communication
            stream while layer i computes; backward gathers from the secondaries
            prefetched, qgZ reduce-scatter of layer i overlapped with the backward of
            layer i-1 (setting T, P2P transport unless --transport nccl)
  flat      ZeRO-3 baseline: NCCL bf16 all-gather / reduce-scatter on the world
            communicator, same overlap schedule

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/train_step.py --mode hz --steps 5
Rank 0 prints one JSON line: ms/step (device time, max over ranks), model TFLOPS
per GPU, and the ratio to the compute-only bound measured in the same run.
"""

import argparse
import json
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="gpt1.3b")
    ap.add_argument("--tokens", type=int, default=8192, help="tokens per micro-batch per GPU")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--modes", default="compute,hz,flat")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p")
    ap.add_argument("--pair", action=argparse.BooleanOptionalAction, default=True,
                    help="forward gathers through hz_allgather_params_next (next layer's quantize in the same launch)")
    ap.add_argument("--hierarchy", default="", help="override, e.g. 4 = ZeRO++-style one level over all ranks")
    ap.add_argument("--green", type=int, default=0,
                    help="run the communication stream in a CUDA green context of this many SMs "
                         "(libhz grids sized to it: hz_set_sm_budget)")
    ap.add_argument("--budget", type=int, default=0,
                    help="hz_set_sm_budget for the libhz grids (SMs x resident CTAs; e.g. 37 = 148 CTAs, one "
                         "per SM, leaving each SM room for a GEMM CTA)")
    ap.add_argument("--prio", action="store_true",
                    help="compute stream at high priority, communication stream at the lowest")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from paper_2501_04266_b200 import hz, synth
    import bench

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo")
    group = bench.hierarchy_of(args, world)
    cfg = synth.GPT_CONFIGS[args.config]
    h = cfg["hidden"]
    nl = args.layers or cfg["layers"]
    T = args.tokens
    B = 256

    uid = hz.get_uid() if rank == 0 else None
    if world > 1:
        box = [uid]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    ctx = hz.Context(rank, world, uid, group, local)
    if args.green:
        from tools.green_probe import green_stream
        comm_green, green_sms = green_stream(args.green)
        hz.set_sm_budget(green_sms)
    if args.budget:
        hz.set_sm_budget(args.budget)
    L = len(group)
    numel = synth.layer_numel(h)
    p = ctx.partition(numel, B, 1, 1, L)
    Np = p.padded_numel
    use_p2p = world > 1 and args.transport == "p2p"
    if use_p2p:
        ctx.enable_p2p(nl * (Np // group[0] + Np // group[0] // B * 4 + 512) + 4 * Np + (64 << 20))
    off_w, len_w = p.range(1)
    _, len_l = p.range(L)

    # per-layer sharded state
    layers = []
    for i in range(nl):
        full = synth.torch_normal(Np, 7000 + i, 0.02, torch.bfloat16, dev, outlier_every=0)
        full[numel:] = 0
        sec_c = ctx.sym_alloc(len_w, torch.uint8) if use_p2p else torch.empty(len_w, dtype=torch.uint8, device=dev)
        sec_s = (ctx.sym_alloc(len_w // B, torch.float32) if use_p2p
                 else torch.empty(len_w // B, dtype=torch.float32, device=dev))
        layers.append({"primary": full[off_w:off_w + len_w].clone(), "resident": full,
                       "flat_chunk": full[rank * (Np // world):(rank + 1) * (Np // world)].clone(),
                       "sec_c": sec_c, "sec_s": sec_s,
                       "shard": torch.empty(len_l, dtype=torch.float32, device=dev),
                       "flat_shard": torch.empty(Np // world, dtype=torch.bfloat16, device=dev)})
    gathered = [torch.empty(Np, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    grads = [torch.empty(Np, dtype=torch.bfloat16, device=dev) for _ in range(2)]
    x = torch.randn(T, h, device=dev, dtype=torch.bfloat16)
    acts = {"qkv": torch.empty(T, 3 * h, device=dev, dtype=torch.bfloat16),
            "proj": torch.empty(T, h, device=dev, dtype=torch.bfloat16),
            "up": torch.empty(T, 4 * h, device=dev, dtype=torch.bfloat16),
            "down": torch.empty(T, h, device=dev, dtype=torch.bfloat16)}
    gx = torch.randn(T, h, device=dev, dtype=torch.bfloat16)
    dacts = {"up": torch.empty(T, 4 * h, device=dev, dtype=torch.bfloat16),
             "h": torch.empty(T, h, device=dev, dtype=torch.bfloat16)}

    def views(buf):
        o = 0
        out = {}
        for name, shape in (("qkv", (3 * h, h)), ("proj", (h, h)), ("up", (4 * h, h)), ("down", (h, 4 * h))):
            n = shape[0] * shape[1]
            out[name] = buf[o:o + n].view(*shape)
            o += n
        return out

    def fwd(buf):
        W = views(buf)
        torch.matmul(x, W["qkv"].t(), out=acts["qkv"])
        torch.matmul(x, W["proj"].t(), out=acts["proj"])
        torch.matmul(acts["proj"], W["up"].t(), out=acts["up"])
        torch.matmul(acts["up"], W["down"].t(), out=acts["down"])

    def bwd(buf, gbuf):
        W = views(buf)
        G = views(gbuf)
        # dX and dW of the four GEMMs (dW written into the layer's gradient buffer)
        torch.matmul(gx, W["down"], out=dacts["up"])
        torch.matmul(gx.t(), acts["up"], out=G["down"])
        torch.matmul(dacts["up"], W["up"], out=dacts["h"])
        torch.matmul(dacts["up"].t(), acts["proj"], out=G["up"])
        torch.matmul(gx, W["proj"], out=dacts["h"])
        torch.matmul(gx.t(), x, out=G["proj"])
        torch.matmul(acts["qkv"], W["qkv"], out=dacts["h"])
        torch.matmul(acts["qkv"].t(), x, out=G["qkv"])

    flops = nl * 3 * 2 * T * 12 * h * h
    if args.prio:
        comp = torch.cuda.Stream(priority=-2)
        torch.cuda.set_stream(comp)
        comm = torch.cuda.Stream(priority=0)
    else:
        comp = torch.cuda.current_stream()
        comm = torch.cuda.Stream()
    if args.green:
        comm = comm_green

    def step(mode):
        if mode == "compute":
            for i in range(nl):
                fwd(layers[i]["resident"])
            for i in reversed(range(nl)):
                bwd(layers[i]["resident"], grads[i & 1])
            return
        ag_done = [torch.cuda.Event() for _ in range(nl)]
        used = [torch.cuda.Event() for _ in range(nl)]

        def ag(i, backward):
            t = layers[i]
            if mode == "hz" and not backward and args.pair:
                # forward: gather layer i and prefetch the quantize of layer i+1 in one launch
                nx = layers[i + 1] if i + 1 < nl else None
                ctx.allgather_params_next(p, t["primary"], t["sec_c"], t["sec_s"], gathered[i & 1], bits=8,
                                          p_next=p if nx else None, next_primary=nx["primary"] if nx else None,
                                          next_sec_codes=nx["sec_c"] if nx else None,
                                          next_sec_scales=nx["sec_s"] if nx else None, stream=comm)
            elif mode == "hz":
                ctx.allgather_params(p, None if backward else t["primary"], t["sec_c"], t["sec_s"], gathered[i & 1],
                                     bits=8, backward=backward, stream=comm)
            else:
                ctx.flat_allgather(t["flat_chunk"], gathered[i & 1], stream=comm)

        def rs(i):
            t = layers[i]
            if mode == "hz":
                ctx.reduce_scatter_grads(p, grads[i & 1], t["shard"], [4] * L, stream=comm)
            else:
                ctx.flat_reduce_scatter(grads[i & 1], t["flat_shard"], stream=comm)

        # forward: gather i+1 while layer i computes
        comm.wait_stream(comp)
        with torch.cuda.stream(comm):
            ag(0, False)
            ag_done[0].record(comm)
        for i in range(nl):
            if i + 1 < nl:
                if i >= 1:
                    comm.wait_event(used[i - 1])        # buffer (i+1)&1 is free
                ag(i + 1, False)
                ag_done[i + 1].record(comm)
            comp.wait_event(ag_done[i])
            fwd(gathered[i & 1])
            used[i].record(comp)
        # backward: gather i-1 from the secondaries while layer i computes; qgZ of i after
        bag = [torch.cuda.Event() for _ in range(nl)]
        bused = [torch.cuda.Event() for _ in range(nl)]
        gdone = [torch.cuda.Event() for _ in range(nl)]
        comm.wait_event(used[nl - 1])
        ag(nl - 1, True)
        bag[nl - 1].record(comm)
        for i in reversed(range(nl)):
            if i - 1 >= 0:
                if i + 1 < nl:
                    comm.wait_event(bused[i + 1])      # gathered buffer (i-1)&1 free
                ag(i - 1, True)
                bag[i - 1].record(comm)
            comp.wait_event(bag[i])
            if i + 2 < nl:
                comp.wait_event(gdone[i + 2])           # gradient buffer i&1 consumed by qgZ
            bwd(gathered[i & 1], grads[i & 1])
            bused[i].record(comp)
            comm.wait_event(bused[i])
            rs(i)
            gdone[i].record(comm)
        comp.wait_stream(comm)

    results = {}
    for mode in args.modes.split(","):
        for _ in range(args.warmup):
            step(mode)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(comp)
        for _ in range(args.steps):
            step(mode)
        e1.record(comp)
        torch.cuda.synchronize()
        ms = bench.max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
        results[mode] = {"ms_per_step": ms, "tflops_per_gpu": flops / (ms * 1e-3) / 1e12}
    if "compute" in results:
        for m in results:
            results[m]["fraction_of_compute_bound"] = results["compute"]["ms_per_step"] / results[m]["ms_per_step"]
    if "hz" in results and "flat" in results:
        results["hz_over_flat"] = results["flat"]["ms_per_step"] / results["hz"]["ms_per_step"]
    line = {"what": "synthetic ZeRO-topo training step (layer GEMMs + sharded collectives, overlapped)",
            "config": args.config, "layers": nl, "tokens_per_gpu": T, "n_gpus": world, "hierarchy": list(group),
            "transport": "p2p" if use_p2p else ("nccl" if world > 1 else "local"),
            "green_sms": green_sms if args.green else 0, "sm_budget": args.budget, "prio": args.prio, "pair": args.pair, "hz_tune": os.environ.get("HZ_TUNE", ""),
            "results": results}
    ctx.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
