#!/bin/bash
# Dual-kernel (k_gather_quantize) work split sweep through bench.py at N GPUs (HZ_TUNE gq / gqf).
N=${1:-2}
mkdir -p gpurun_out/gq
export HZ_BENCH_WATCHDOG=200
for tune in gq=0 gq=1 gq=2,gqf=30 gq=2,gqf=50 gq=2,gqf=70; do
  HZ_TUNE=$tune timeout 240 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2968$N bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail --no-flat \
    > gpurun_out/gq/${tune}_n$N.log 2>&1
  echo "$tune rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/gq/${tune}_n$N.log | head -1) $(grep -o '"gather_quantize": {[^}]*' gpurun_out/gq/${tune}_n$N.log | grep -o '"avg_ms": [0-9.]*' | head -1)"
done
