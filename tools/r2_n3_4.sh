#!/bin/bash
# N3 at N = 4 (the verdict's configuration): GPT-1.3B, 1024 tokens/GPU, compute / hz / flat
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 $B --master-port 29851 tools/train_step.py --tokens 1024 --steps 5 --warmup 3 --modes compute,hz,flat > gpurun_out/n3_4_a.log 2>&1; echo "rc=$?"
grep '^{' gpurun_out/n3_4_a.log | tail -1
timeout 900 $B --master-port 29852 tools/train_step.py --tokens 2048 --steps 5 --warmup 3 --modes compute,hz,flat > gpurun_out/n3_4_b.log 2>&1; echo "rc=$?"
grep '^{' gpurun_out/n3_4_b.log | tail -1
