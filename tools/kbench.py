#!/usr/bin/env python
"""Kernel microbenchmark: each libhz codec kernel alone at GPT-layer size, timed
with CUDA events on the launching stream, rotating over enough buffer sets that
the working set exceeds L2 (126 MB).  Prints one JSON line per kernel with the
algorithmic HBM bytes per launch and GB/s (and the fraction of the measured copy
peak).  ``--once`` runs each kernel once (for ncu captures).

    python tools/kbench.py [--numel N] [--iters K] [--once]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--numel", type=int, default=50_364_416)   # GPT-1.3B layer, padded
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--block", type=int, default=256)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--step1", action="store_true",
                    help="one world-1 step of one tensor through the collective API (fused round trips)")
    ap.add_argument("--pair", action="store_true",
                    help="world-1 P2P context: the adjacent-layer dual kernel (k_gather_quantize) forward and backward")
    args = ap.parse_args()
    if args.pair:
        return pair(args)
    if args.step1:
        return step1(args)

    import torch
    from paper_2501_04266_b200 import hz
    sys.path.insert(0, ROOT)
    import bench
    peak, _ = bench.measured_peaks()

    n, B = args.numel, args.block
    dev = "cuda"
    nsets = 4
    x = [torch.randn(n, device=dev).mul_(1e-3).to(torch.bfloat16) for _ in range(nsets)]
    c8 = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(nsets)]
    c4 = [torch.empty(n // 2, dtype=torch.uint8, device=dev) for _ in range(nsets)]
    c4b = [torch.empty(n // 2, dtype=torch.uint8, device=dev) for _ in range(nsets)]
    s = [torch.empty(n // B, dtype=torch.float32, device=dev) for _ in range(nsets)]
    s2 = [torch.empty(n // B, dtype=torch.float32, device=dev) for _ in range(nsets)]
    yb = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(nsets)]
    yf = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(nsets)]
    for i in range(nsets):
        hz.quantize(x[i], 8, B, c8[i], s[i])
        hz.quantize(x[i], 4, B, c4[i], s2[i])
        hz.quantize(x[(i + 1) % nsets], 4, B, c4b[i], s2[(i + 1) % nsets])
    torch.cuda.synchronize()

    sb = 4 * n // B
    cases = {
        "quantize_bf16_int8": (lambda i: hz.quantize(x[i], 8, B, c8[i], s[i]), 2 * n + n + sb),
        "quantize_bf16_int4": (lambda i: hz.quantize(x[i], 4, B, c4[i], s2[i]), 2 * n + n // 2 + sb),
        "dequantize_int8_bf16": (lambda i: hz.dequantize(c8[i], s[i], n, 8, B, out=yb[i]), n + sb + 2 * n),
        "reduce_g1_int4_f32": (lambda i: hz.reduce_chunks([c4[i]], [s2[i]], n, 4, B, out_f32=yf[i]),
                               n // 2 + sb + 4 * n),
        "reduce_g2_int4_f32": (lambda i: hz.reduce_chunks([c4[i], c4b[i]], [s2[i], s2[(i + 1) % nsets]], n // 2, 4, B,
                                                          out_f32=yf[i]), 2 * (n // 4 + sb // 2) + 2 * n),
        "reduce_g2_int4_acc": (lambda i: hz.reduce_chunks([c4[i], c4b[i]], [s2[i], s2[(i + 1) % nsets]], n // 2, 4, B,
                                                          out_f32=yf[i], accumulate=True), 2 * (n // 4 + sb // 2) + 4 * n),
        "reduce_g2_int4_requant4": (lambda i: hz.reduce_chunks([c4[i], c4b[i]], [s2[i], s2[(i + 1) % nsets]], n // 2, 4,
                                                               B, bits_out=4, out_codes=c8[i], out_scales=s[i]),
                                    2 * (n // 4 + sb // 2) + n // 4 + sb // 2),
    }
    stream = torch.cuda.current_stream()
    for name, (fn, byts) in cases.items():
        if args.only and args.only not in name:
            continue
        if args.once:
            fn(0)
            torch.cuda.synchronize()
            continue
        for i in range(3):
            fn(i % nsets)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.iters):
            fn(i % nsets)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
        gbs = byts / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": name, "numel": n, "us": round(ms * 1e3, 2), "bytes": byts,
                          "GBps": round(gbs, 1), "frac_of_copy_peak": round(gbs / peak, 3)}), flush=True)


def step1(args):
    """World-1 context, one GPT-1.3B layer: forward gather (fused quantize+dequantize,
    bf16), backward gather (dequantize), qgZ (fused quantize+dequantize, fp32 shard).
    --once: each kernel once (ncu); else timed with CUDA events per call."""
    import torch
    from paper_2501_04266_b200 import hz, synth
    sys.path.insert(0, ROOT)
    import bench
    peak, _ = bench.measured_peaks()
    ctx = hz.Context(0, 1, hz.get_uid(), (1,), 0)
    numel = synth.layer_numel(2048)
    p = ctx.partition(numel, 256, 1, 1, 1)
    Np = p.padded_numel
    nsets = 4
    prim = [synth.torch_normal(Np, 1 + i, 0.02, torch.bfloat16, "cuda", outlier_every=0) for i in range(nsets)]
    grad = [synth.torch_normal(Np, 11 + i, 1e-3, torch.bfloat16, "cuda") for i in range(nsets)]
    sec_c = [torch.empty(Np, dtype=torch.uint8, device="cuda") for _ in range(nsets)]
    sec_s = [torch.empty(Np // 256, dtype=torch.float32, device="cuda") for _ in range(nsets)]
    out = [torch.empty(Np, dtype=torch.bfloat16, device="cuda") for _ in range(nsets)]
    shard = [torch.empty(Np, dtype=torch.float32, device="cuda") for _ in range(nsets)]
    cases = {
        "fwd_quantize_dequantize_bf16": (lambda i: ctx.allgather_params(p, prim[i], sec_c[i], sec_s[i], out[i]),
                                         Np * (2 + 1 + 2) + Np // 64),
        "bwd_dequantize": (lambda i: ctx.allgather_params(p, None, sec_c[i], sec_s[i], out[i], backward=True),
                           Np * (1 + 2) + Np // 64),
        "qgz_quantize_dequantize_f32": (lambda i: ctx.reduce_scatter_grads(p, grad[i], shard[i], [4]), Np * (2 + 4)),
    }
    # calibration: torch copies with the same read:write mixes (bf16 -> bf16 is the
    # 1:1 copy of MEASURED_PEAKS; bf16 -> fp32 is the 1:2 mix of the fp32 shard)
    xf = [torch.empty(Np, dtype=torch.float32, device="cuda") for _ in range(nsets)]
    cases["torch_copy_bf16_bf16"] = (lambda i: out[i].copy_(prim[i]), Np * 4)
    cases["torch_copy_bf16_f32"] = (lambda i: xf[i].copy_(grad[i]), Np * 6)
    for i in range(nsets):
        for name, (fn, _) in cases.items():
            fn(i)
    torch.cuda.synchronize()
    for name, (fn, byts) in cases.items():
        if args.once:
            fn(0)
            torch.cuda.synchronize()
            continue
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.iters):
            fn(i % nsets)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.iters
        gbs = byts / (ms * 1e-3) / 1e9
        print(json.dumps({"kernel": name, "numel": Np, "us": round(ms * 1e3, 2), "bytes": byts,
                          "GBps": round(gbs, 1), "frac_of_copy_peak": round(gbs / peak, 3)}), flush=True)
    ctx.close()


def pair(args):
    """World-1 context with the P2P transport on, one GPT-1.3B layer pair: the dual
    kernel of hz_allgather_params_next (gather layer a || quantize layer b's primary,
    int8) and of hz_backward_step (gather layer a || quantize the gradient, int4, then
    the fp32 reduce).  The gather reads local codes here (no peers), so this is the
    kernel's HBM side; --once for ncu."""
    import torch
    from paper_2501_04266_b200 import hz, synth
    ctx = hz.Context(0, 1, hz.get_uid(), (1,), 0)
    numel = synth.layer_numel(2048)
    p = ctx.partition(numel, 256, 1, 1, 1)
    Np = p.padded_numel
    ctx.enable_p2p(4 * Np + (64 << 20))
    prim = [synth.torch_normal(Np, 1 + i, 0.02, torch.bfloat16, "cuda", outlier_every=0) for i in range(2)]
    grad = synth.torch_normal(Np, 11, 1e-3, torch.bfloat16, "cuda")
    sec_c = [ctx.sym_alloc(Np, torch.uint8) for _ in range(2)]
    sec_s = [ctx.sym_alloc(Np // 256, torch.float32) for _ in range(2)]
    out = torch.empty(Np, dtype=torch.bfloat16, device="cuda")
    shard = torch.empty(Np, dtype=torch.float32, device="cuda")
    ctx.allgather_params(p, prim[0], sec_c[0], sec_s[0], out)
    fwd = lambda: ctx.allgather_params_next(p, prim[0], sec_c[0], sec_s[0], out, p_next=p, next_primary=prim[1],
                                            next_sec_codes=sec_c[1], next_sec_scales=sec_s[1])
    bwd = lambda: ctx.backward_step(p, grad, shard, [4], p_prev=p, prev_sec_codes=sec_c[0], prev_sec_scales=sec_s[0],
                                    prev_full_out=out)
    for name, fn in (("pair_fwd", fwd), ("pair_bwd", bwd)):
        fn()
        torch.cuda.synchronize()
        if args.once:
            continue
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"call": name, "numel": Np, "us": round(e0.elapsed_time(e1) / args.iters * 1e3, 2)}),
              flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
