#!/bin/bash
# A/B of the pipelined one-launch P2P kernels (HZ_TUNE fused=1, pf producer %,
# pk chunks per call) against the two-kernel default: bench.py at 2 and 4 GPUs
# (GPT-1.3B), stage breakdown kept in gpurun_out/ab_*.json.
mkdir -p gpurun_out
for n in ${AB_GPUS:-2 4}; do
  for tune in ${AB_TUNES:-"" fused=1 fused=1,pf=20 fused=1,pf=40 fused=1,pk=8 fused=1,pk=32}; do
    tag=$(echo "n${n}_${tune:-default}" | tr ',=' '_-')
    HZ_TUNE="$tune" timeout 600 python -m torch.distributed.run --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port 2980$n bench.py --gpus $n --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-flat --no-tail \
      > gpurun_out/ab_$tag.log 2>&1 || echo "$tag failed"
    grep '^{' gpurun_out/ab_$tag.log | tail -1 > gpurun_out/ab_$tag.json
  done
done
