#!/bin/bash
# mixed-queue link dual kernel + TMA reduce: parity, then N=2 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vworld.py -q -x > gpurun_out/e6_vw.log 2>&1; echo "vworld rc=$?"; tail -n 2 gpurun_out/e6_vw.log
timeout 900 python -m pytest tests/test_gpu_collectives.py -q -x -k "test_multi_gpu and 2" > gpurun_out/e6_mp.log 2>&1; echo "mp rc=$?"; tail -n 2 gpurun_out/e6_mp.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for t in "lk=-2" "lk=0" "lk=-2,lw=1" "lk=-2,lw=3" "lk=-2,rt=0"; do
  i=$((i+1))
  HZ_TUNE=$t timeout 600 $B --master-port 2964$i bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e6_b2_$i.log 2>&1; echo "$t rc=$?"
  echo "$t $(grep '^{' gpurun_out/e6_b2_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2), round(v.get("avg_publish_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"
done
