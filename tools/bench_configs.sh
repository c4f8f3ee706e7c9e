#!/bin/bash
# BASELINE.json configs 3 and 4 (GPT 6.7B, NeoX 20B) through bench.py at 2 and 4 GPUs
mkdir -p gpurun_out
for cfg in gpt6.7b neox20b; do
  for n in 4 2; do
    timeout 900 python -m torch.distributed.run --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2970$n \
      bench.py --gpus $n --config $cfg --steps 5 --warmup 3 --no-cpu-baseline --no-e2e \
      > gpurun_out/bench_${cfg}_${n}.log 2>&1 || echo "$cfg n=$n failed"
    grep '^{' gpurun_out/bench_${cfg}_${n}.log | tail -1 > gpurun_out/bench_${cfg}_${n}.json
  done
done
