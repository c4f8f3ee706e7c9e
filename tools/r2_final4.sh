#!/bin/bash
# End-of-round check on a 4-GPU box with the final library: full GPU suite (1-, 2-, 4-rank),
# N = 2 / 4 bench lines, configs 3 / 4 at N = 2 / 4
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -q -m gpu > gpurun_out/f4_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/f4_pytest.log
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $B --nproc-per-node 2 --master-port 29872 bench.py --gpus 2 > gpurun_out/f4_bench2.log 2>&1; echo "bench2 rc=$?"
timeout 900 $B --nproc-per-node 4 --master-port 29874 bench.py --gpus 4 > gpurun_out/f4_bench4.log 2>&1; echo "bench4 rc=$?"
i=0
for cfg in "2 gpt6.7b" "4 gpt6.7b" "2 neox20b" "4 neox20b"; do
  set -- $cfg; i=$((i+1))
  timeout 1200 $B --nproc-per-node $1 --master-port 2988$i bench.py --gpus $1 --config $2 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f4_cfg_$2_$1.log 2>&1; echo "$2 N=$1 rc=$?"
done
for f in f4_bench2 f4_bench4 f4_cfg_gpt6.7b_2 f4_cfg_gpt6.7b_4 f4_cfg_neox20b_2 f4_cfg_neox20b_4; do
  grep '^{' gpurun_out/$f.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["config"]["workload"][:12], round(d["ms_per_step"],3), round(d["value"]), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), round(d["step_model"]["frac_of_model_bidir_probe"],3), (d.get("e2e") or {}).get("ms_per_step"), (d.get("flat_zero3_baseline") or {}).get("ms_per_step"), d["clocks"]["reasons"])'
done
