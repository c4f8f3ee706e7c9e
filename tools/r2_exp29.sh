#!/bin/bash
# low-register dual kernel (gql=1): parity (vworld under HZ_TUNE) + N=2 A/B
mkdir -p gpurun_out
HZ_TUNE=gql=1 timeout 900 python -m pytest tests/test_gpu_vworld.py -q -x -k "hierarchy or paired" > gpurun_out/e29_vw.log 2>&1; echo "vworld gql rc=$?"; tail -n 2 gpurun_out/e29_vw.log
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "2:" "2:gql=1" "2:" "2:gql=1"; do
  i=$((i+1)); n=${cfg%%:*}; t=${cfg#*:}
  HZ_TUNE=$t timeout 600 $B --nproc-per-node $n --master-port 2977$i bench.py --gpus $n --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e29_$i.log 2>&1; echo "[N$n $t] rc=$?"
  echo "[N$n $t] $(grep '^{' gpurun_out/e29_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})')"
done
