#!/bin/bash
# Dual-kernel (k_gather_quantize) schedule sweep through bench.py at N GPUs (HZ_TUNE gq / gqf / gqc).
# usage: bash tools/gq_sweep.sh N config "tune1 tune2 ..."
N=${1:-2}
CFG=${2:-gpt1.3b}
TUNES=${3:-"gq=0 gq=1 gq=2,gqf=30 gq=2,gqf=50 gq=2,gqf=70"}
mkdir -p gpurun_out/gq
export HZ_BENCH_WATCHDOG=300
for tune in $TUNES; do
  HZ_TUNE=$tune timeout 300 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 \
    --master-port 2968$N bench.py --gpus $N --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-tail \
    --no-flat > gpurun_out/gq/${CFG}_${tune}_n$N.log 2>&1
  echo "$CFG $tune rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/gq/${CFG}_${tune}_n$N.log | head -1) $(grep -o '"gather_quantize": {[^}]*' gpurun_out/gq/${CFG}_${tune}_n$N.log | grep -o '"avg_ms": [0-9.]*' | head -1)"
done
