#!/bin/bash
# N = 1: world-1 carveout value (HZ_TUNE carve1) under the final store modes
mkdir -p gpurun_out
b1() {
  HZ_TUNE=$1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e45_b1.log 2>&1
  echo "N1 [$1] $(grep '^{' gpurun_out/e45_b1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})')"
}
for r in 1 2; do for t in "" "carve1=90" "carve1=75" "carve1=60"; do b1 "$t"; done; done
