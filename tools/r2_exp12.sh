#!/bin/bash
# mixed-queue link dual kernel + TMA reduce: parity, then N=2 A/B
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for t in "tma=0,lk=0,rt=0" "tma=1,lk=0,rt=0" "tma=1,ts=2,lk=0,rt=0" "tma=1,tte=4096,ts=2,tsm=57344,lk=0,rt=0"; do
  i=$((i+1))
  HZ_TUNE=$t timeout 600 $B --master-port 2966$i bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e12_b2_$i.log 2>&1; echo "$t rc=$?"
  echo "$t $(grep '^{' gpurun_out/e12_b2_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2), round(v.get("avg_publish_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"
done
