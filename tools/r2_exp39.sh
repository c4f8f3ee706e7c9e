#!/bin/bash
# bulk-store staging of the dual / triple kernels moved to dynamic shared memory (0 bytes when
# off): A/B against the previous build on one box (HZ_LIB=libhz_old.so), N = 2; parity
mkdir -p gpurun_out
b2() {
  HZ_LIB=$1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e39_b2.log 2>&1
  echo "N2 [$1] $(grep '^{' gpurun_out/e39_b2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})')"
}
for r in 1 2 3; do b2 libhz.so; b2 libhz_old.so; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/e39_pt.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/e39_pt.log
HZ_TUNE=dgb=1 timeout 600 python -m pytest tests/test_gpu_vworld.py -x -q -m gpu > gpurun_out/e39_dgb.log 2>&1; echo "dgb=1 vworld rc=$?"; tail -1 gpurun_out/e39_dgb.log
