#!/usr/bin/env python
"""Green-context probe (tool, not product): can the communication kernels run on a
fixed SM partition while GEMMs use the rest?  One GPU, world-1 context (the codec
round trips are HBM-bound like the P2P kernels' local half).

For K in --sms: a green context with K SMs (cuDevSmResourceSplitByCount), a stream
in it, and the libhz SM budget set to K; then, with CUDA events,
  comm alone      one GPT-1.3B layer's forward gather + backward gather + qgZ on the
                  green stream
  gemm alone      the layer GEMMs of tools/train_step.py (T tokens) on the primary
                  context's stream
  both            the two loops launched together, each on its stream
Prints one JSON line per K.
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def check(r):
    err = r[0] if isinstance(r, tuple) else r
    if int(err) != 0:
        raise RuntimeError(f"CUDA driver error {err}")
    return r[1:] if isinstance(r, tuple) and len(r) > 2 else (r[1] if isinstance(r, tuple) else None)


def green_stream(k):
    """A CUDA stream in a green context of (at least) k SMs of the current device,
    as a torch ExternalStream; returns (stream, SMs granted)."""
    import torch
    import cuda.bindings.driver as drv
    torch.zeros(1, device="cuda")
    dev = check(drv.cuCtxGetDevice())
    res = check(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    r = drv.cuDevSmResourceSplitByCount(1, res, 0, k)
    if int(r[0]) != 0:
        raise RuntimeError(f"cuDevSmResourceSplitByCount: {r[0]}")
    grp = r[1][0]
    desc = check(drv.cuDevResourceGenerateDesc([grp], 1))
    gctx = check(drv.cuGreenCtxCreate(desc, dev, drv.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
    gs = check(drv.cuGreenCtxStreamCreate(gctx, drv.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
    green_stream.keep.append(gctx)     # keep the context alive with the stream
    return torch.cuda.ExternalStream(int(gs)), grp.sm.smCount


green_stream.keep = []


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sms", default="16,24,32,48,148")
    ap.add_argument("--tokens", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=10)
    args = ap.parse_args()

    import torch
    import cuda.bindings.driver as drv
    from paper_2501_04266_b200 import hz, synth

    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")
    dev = check(drv.cuCtxGetDevice())
    res = check(drv.cuDeviceGetDevResource(dev, drv.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    total_sms = res.sm.smCount

    ctx = hz.Context(0, 1, hz.get_uid(), (1,), 0)
    numel = synth.layer_numel(2048)
    p = ctx.partition(numel, 256, 1, 1, 1)
    Np = p.padded_numel
    prim = synth.torch_normal(Np, 1, 0.02, torch.bfloat16, "cuda", outlier_every=0)
    grad = synth.torch_normal(Np, 2, 1e-3, torch.bfloat16, "cuda")
    sec_c = torch.empty(Np, dtype=torch.uint8, device="cuda")
    sec_s = torch.empty(Np // 256, dtype=torch.float32, device="cuda")
    out = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
    shard = torch.empty(Np, dtype=torch.float32, device="cuda")

    h, T = 2048, args.tokens
    x = torch.randn(T, h, device="cuda", dtype=torch.bfloat16)
    w = torch.randn(4 * h, h, device="cuda", dtype=torch.bfloat16)
    y = torch.empty(T, 4 * h, device="cuda", dtype=torch.bfloat16)

    def comm(stream):
        for _ in range(4):
            ctx.allgather_params(p, prim, sec_c, sec_s, out, stream=stream)
            ctx.allgather_params(p, None, sec_c, sec_s, out, backward=True, stream=stream)
            ctx.reduce_scatter_grads(p, grad, shard, [4], stream=stream)

    def gemm():
        for _ in range(24):
            torch.matmul(x, w.t(), out=y)

    def timed(fn_list):
        # fn_list: [(callable, torch stream)] launched back to back, timed per stream
        evs = []
        torch.cuda.synchronize()
        for fn, st in fn_list:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            with torch.cuda.stream(st):
                for _ in range(args.iters):
                    fn(st)
            e1.record(st)
            evs.append((e0, e1))
        torch.cuda.synchronize()
        return [a.elapsed_time(b) / args.iters for a, b in evs]

    main_stream = torch.cuda.current_stream()
    for k in [int(v) for v in args.sms.split(",")]:
        k = min(k, total_sms)
        if k < total_sms:
            cstream, k_eff = green_stream(k)
        else:
            k_eff = total_sms
            cstream = torch.cuda.Stream()
        hz.set_sm_budget(k_eff if k_eff < total_sms else 0)
        comm_fn = lambda st: comm(st)           # noqa: E731
        gemm_fn = lambda st: gemm()             # noqa: E731
        timed([(comm_fn, cstream)])             # warm-up
        (t_comm,) = timed([(comm_fn, cstream)])
        (t_gemm,) = timed([(gemm_fn, main_stream)])
        t_both = timed([(comm_fn, cstream), (gemm_fn, main_stream)])
        print(json.dumps({"sms": k_eff, "comm_alone_ms": round(t_comm, 3), "gemm_alone_ms": round(t_gemm, 3),
                          "both_comm_ms": round(t_both[0], 3), "both_gemm_ms": round(t_both[1], 3),
                          "serial_ms": round(t_comm + t_gemm, 3)}), flush=True)
    hz.set_sm_budget(0)
    ctx.close()


if __name__ == "__main__":
    main()
