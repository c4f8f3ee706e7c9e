#!/bin/bash
# N = 1 under the world-1 carveout: LSU stores for the dequantize (fbd=0) + bulk stores for the
# bf16 round trip (fbb=1), alternated with the current defaults
mkdir -p gpurun_out
b1() {
  HZ_TUNE=$1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e41_b1.log 2>&1
  echo "N1 [$1] $(grep '^{' gpurun_out/e41_b1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})')"
}
for r in 1 2 3; do b1 ""; b1 "fbd=0,fbb=1"; done
b1 "fbd=0,fbb=1,carve1=-1"
