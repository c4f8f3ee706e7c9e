#!/bin/bash
# config 5 message sweep at 2 and 4 GPUs (P2P transport, and NCCL transport at 4)
mkdir -p gpurun_out
for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2962$n \
    tools/msg_sweep.py --out gpurun_out/sweep_r02_${n}gpu_p2p.jsonl > gpurun_out/sweep_r02_${n}.log 2>&1 || echo "n=$n failed"
done
timeout 900 python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29629 \
  tools/msg_sweep.py --transport nccl --out gpurun_out/sweep_r02_4gpu_nccl.jsonl > gpurun_out/sweep_r02_4n.log 2>&1 || echo "nccl failed"
