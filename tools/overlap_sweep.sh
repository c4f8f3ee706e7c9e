#!/bin/bash
# N3 overlap sweep: tools/train_step.py over tokens x libhz grid limits (4 and 2 GPUs).
mkdir -p gpurun_out
set -x
for T in 1024 2048; do
 for lim in 0 16 32 64; do
  modes="hz"; [ $lim = 0 ] && modes="compute,hz,flat"
  timeout 300 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 tools/train_step.py --tokens $T --grid-limit $lim --modes $modes --steps 5 2>&1 | grep '^{' >> gpurun_out/sweep4.jsonl
 done
done
for lim in 0 32; do
  timeout 300 python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 tools/train_step.py --tokens 1024 --grid-limit $lim --steps 5 2>&1 | grep '^{' >> gpurun_out/sweep2.jsonl
done
