#!/bin/bash
# link ring geometry sweep at N=2 + ncu --set full of the dual kernel (old vs warp-specialised) in one process
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for t in "lk=0" "lk=-2,lte=4096,ls=3" "lk=-2,lte=8192,ls=2" "lk=-2,lte=4096,ls=2" "lk=-2,lte=2048,ls=4" "lk=-1,lte=4096,ls=3" "lk=0,rt_te=2048,rt_s=2"; do
  i=$((i+1))
  HZ_TUNE=$t timeout 600 $B --master-port 2965$i bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e7_b2_$i.log 2>&1; echo "$t rc=$?"
  echo "$t $(grep '^{' gpurun_out/e7_b2_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2), round(v.get("avg_publish_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"
done
timeout 300 python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/e7_vwp.log 2>&1 && \
HZ_TUNE=lk=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_quantize -c 2 -o gpurun_out/e7_dual_old -f python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/e7_ncu_old.log 2>&1; echo "ncu old rc=$?"
HZ_TUNE=lk=-2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_quantize -c 2 -o gpurun_out/e7_dual_ws -f python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/e7_ncu_ws.log 2>&1; echo "ncu ws rc=$?"
