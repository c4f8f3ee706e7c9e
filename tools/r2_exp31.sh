#!/bin/bash
# N=1: world-1 backward pairing (pair1) with the round-2 kernels
mkdir -p gpurun_out
for t in "" "pair1=1" "" "pair1=1"; do
  HZ_TUNE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e31.log 2>&1; echo "[$t] rc=$?"
  echo "[$t] $(grep '^{' gpurun_out/e31.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["roofline"]["frac"],4), d["gpu_launches"], {k:round(v["avg_ms"]*1e3,2) for k,v in d["stages"].items()})')"
done
