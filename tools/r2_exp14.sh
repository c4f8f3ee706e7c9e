#!/bin/bash
# piece rotation in the gather loop: parity (vworld, 2-process) + N=2 bench
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for t in "" "pub=1" "pub=2"; do
  i=$((i+1))
  HZ_TUNE=$t timeout 600 $B --master-port 2968$i bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e14_b2_$i.log 2>&1; echo "[$t] rc=$?"
  echo "[$t] $(grep '^{' gpurun_out/e14_b2_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["step_model"]["frac_of_model_bidir_probe"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2), round(v.get("avg_publish_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"
done
