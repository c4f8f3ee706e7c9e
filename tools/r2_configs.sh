#!/bin/bash
# BASELINE configs 3 / 4 (GPT-6.7B, NeoX-20B) at N = 2 and 4, round 2 code
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "2 gpt6.7b" "4 gpt6.7b" "4 neox20b" "2 neox20b"; do
  set -- $cfg; i=$((i+1))
  timeout 1200 $B --nproc-per-node $1 --master-port 2990$i bench.py --gpus $1 --config $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cfg_$2_$1.log 2>&1; echo "$2 N=$1 rc=$?"
  grep '^{' gpurun_out/cfg_$2_$1.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["config"]["workload"][:30], d["ms_per_step"], round(d["value"]), round(d["roofline"]["frac"],3), round(d["step_model"]["frac_of_model_bidir_probe"],3), (d.get("flat_zero3_baseline") or {}).get("ms_per_step"), (d.get("step_tail") or {}).get("ms_per_step"))'
done
