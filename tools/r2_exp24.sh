#!/bin/bash
# chunked vs one-pass dual kernel at the large layers (N=2 and N=4)
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "2:neox20b:" "2:neox20b:gqc=1" "4:gpt6.7b:" "4:gpt6.7b:gqc=1" "4:neox20b:" "4:neox20b:gqc=1"; do
  i=$((i+1)); IFS=: read n m t <<< "$cfg"
  HZ_TUNE=$t timeout 900 $B --nproc-per-node $n --master-port 2974$i bench.py --gpus $n --config $m --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e24_$i.log 2>&1; echo "[$cfg] rc=$?"
  echo "[$cfg] $(grep '^{' gpurun_out/e24_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})')"
done
