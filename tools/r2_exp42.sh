#!/bin/bash
# N = 1 knobs re-checked under the world-1 carveout and the new store modes
mkdir -p gpurun_out
b1() {
  HZ_TUNE=$1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e42_b1.log 2>&1
  echo "N1 [$1] $(grep '^{' gpurun_out/e42_b1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})')"
}
for r in 1 2; do for t in "" "pdl=1" "deq_u=2" "deq_u=16" "rt_u=2" "grid_np=2"; do b1 "$t"; done; done
