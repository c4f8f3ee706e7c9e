#!/bin/bash
# N = 2: uniform shared-memory carveout for every launch of a world-2 context (HZ_TUNE carve)
mkdir -p gpurun_out
b2() {
  HZ_TUNE=$1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e37_b2.log 2>&1
  echo "N2 [$1] $(grep '^{' gpurun_out/e37_b2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})')"
}
for c in "" carve=10 carve=25 carve=50 "" carve=10 carve=25; do b2 "$c"; done
