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
    args = ap.parse_args()

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


if __name__ == "__main__":
    main()
