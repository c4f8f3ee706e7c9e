#!/bin/bash
# deferred last qgZ hop + backward triple kernel: parity (vworld incl. step_host, 2-process), N=2 A/B
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/e19_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 1 gpurun_out/e19_smoke.log
timeout 1200 python -m pytest tests/test_gpu_vworld.py -q -x > gpurun_out/e19_vw.log 2>&1; echo "vworld rc=$?"; tail -n 3 gpurun_out/e19_vw.log
timeout 900 python -m pytest tests/test_gpu_collectives.py -q -x -k "test_multi_gpu and 2" > gpurun_out/e19_mp.log 2>&1; echo "mp rc=$?"; tail -n 3 gpurun_out/e19_mp.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for t in "" "defer=0"; do
  i=$((i+1))
  HZ_TUNE=$t timeout 600 $B --master-port 2972$i bench.py --gpus 2 --no-cpu-baseline --no-tail --no-flat > gpurun_out/e19_b2_$i.log 2>&1; echo "[$t] rc=$?"
  echo "[$t] $(grep '^{' gpurun_out/e19_b2_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["gpu_launches"], d["step_model"]["frac_of_model_bidir_probe"], d["e2e"]["ms_per_step"], d["e2e"]["host_shards_equal_device_run"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2), round(v.get("avg_publish_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"
done
