#!/bin/bash
# shared-memory carveout as a per-call launch attribute: 100 for world-1 contexts (HZ_TUNE carve1)
mkdir -p gpurun_out
b1() {
  HZ_TUNE=$1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e36_b1.log 2>&1
  echo "N1 [$1] $(grep '^{' gpurun_out/e36_b1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})')"
}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e36_pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/e36_pt.log
for r in 1 2 3; do b1 ""; b1 "carve1=-1"; done
