#!/bin/bash
# N3: synthetic GPT-1.3B training step at N GPUs, 1024 tokens/GPU: how much of the communication
# hides behind the layer GEMMs as the libhz grids shrink to leave room for GEMM CTAs on every SM
N=${1:-2}
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
run() {  # budget tune modes
  i=$((i+1))
  HZ_TUNE=$2 timeout 900 $B --master-port 2980$i tools/train_step.py --tokens 1024 --steps 5 --warmup 3 --budget $1 --modes $3 > gpurun_out/n3_${N}_$i.log 2>&1
  echo "budget=$1 tune=[$2] $(grep '^{' gpurun_out/n3_${N}_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(v["ms_per_step"],2) if isinstance(v,dict) else round(v,3)) for k,v in d["results"].items()})')"
}
run 0 "" compute,hz,flat
run 37 "" hz
run 74 "" hz
run 37 "deq_u=16,q_u=8,gqu=8,rf_u=4" hz
run 74 "deq_u=16,q_u=8,gqu=8,rf_u=4" hz
run 0 "deq_u=16,q_u=8,gqu=8,rf_u=4" hz
