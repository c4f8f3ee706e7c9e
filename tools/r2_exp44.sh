#!/bin/bash
# N = 4 (2,2): level-1 requantizing reduce with 8 warp steps per iteration (rq_u=8, 96 registers)
mkdir -p gpurun_out
b4() {
  HZ_TUNE=$1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29615 bench.py --gpus 4 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e44_b4.log 2>&1
  echo "N4 [$1] $(grep '^{' gpurun_out/e44_b4.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})')"
}
for r in 1 2; do for t in "" "rq_u=8"; do b4 "$t"; done; done
HZ_TUNE=rq_u=8 timeout 600 python -m pytest tests/test_gpu_vworld.py -x -q -m gpu -k hierarchy > gpurun_out/e44_pt.log 2>&1; echo "rq_u=8 vworld rc=$?"; tail -1 gpurun_out/e44_pt.log
