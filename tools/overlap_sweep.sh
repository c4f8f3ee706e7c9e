#!/bin/bash
# N3 overlap sweep: tools/train_step.py (4 GPUs) over tokens x communication SM
# partition (CUDA green context of K SMs for the communication stream, libhz grids
# sized to it), with / without stream priorities.
mkdir -p gpurun_out
out=${SWEEP_OUT:-gpurun_out/overlap4.jsonl}
for T in ${SWEEP_TOKENS:-1024 2048}; do
  for flags in "" "--green 32" "--green 48" "--green 64" "--green 48 --prio"; do
    modes="hz"; [ -z "$flags" ] && modes="compute,hz,flat"
    timeout 300 python -m torch.distributed.run --nproc-per-node ${SWEEP_GPUS:-4} --master-addr 127.0.0.1 \
      --master-port 29611 tools/train_step.py --tokens $T --modes $modes --steps 5 $flags 2>&1 | grep '^{' >> $out
  done
done
