#!/bin/bash
# the design space the paper tabulates, through bench.py at N GPUs
# (default 4, hierarchy (2,2)), GPT-1.3B: role levels (sec-degree 2 vs P, setting Z),
# int4 vs int8 qgZ, block sizes.  One JSON line per variant in gpurun_out/variants/.
N=${1:-4}
mkdir -p gpurun_out/variants
run() {
  tag=$1; shift
  timeout 600 python -m torch.distributed.run --nproc-per-node $N --master-addr 127.0.0.1 --master-port 2975$N \
    bench.py --gpus $N --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail --no-flat "$@" \
    > gpurun_out/variants/${tag}_n$N.log 2>&1 || echo "$tag failed"
  grep '^{' gpurun_out/variants/${tag}_n$N.log | tail -1 > gpurun_out/variants/${tag}_n$N.json
}
run base
run roles12 --roles 1,2
run roles10 --roles 1,0
run roles21 --roles 2,1
run roles22 --roles 2,2
run qgz8 --qgz-bits 8
run block64 --block 64
run block1024 --block 1024
run block2048 --block 2048
run nccl --transport nccl
