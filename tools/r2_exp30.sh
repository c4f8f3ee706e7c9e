#!/bin/bash
# backward triple kernel job order (gqro) at N=2 (GPT-1.3B, GPT-6.7B)
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for cfg in "gpt1.3b:gqro=0" "gpt1.3b:gqro=1" "gpt1.3b:gqro=2" "gpt1.3b:gqro=3" "gpt6.7b:gqro=0" "gpt6.7b:gqro=1" "gpt6.7b:gqro=3"; do
  i=$((i+1)); m=${cfg%%:*}; t=${cfg#*:}
  HZ_TUNE=$t timeout 600 $B --master-port 2978$i bench.py --gpus 2 --config $m --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e30_$i.log 2>&1; echo "[$cfg] rc=$?"
  echo "[$cfg] $(grep '^{' gpurun_out/e30_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})')"
done
