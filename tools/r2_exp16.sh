#!/bin/bash
# balanced dual-kernel schedule: parity + N=2 A/B (schedule, register bound)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_vworld.py -q -x > gpurun_out/e16_vw.log 2>&1; echo "vworld rc=$?"; tail -n 2 gpurun_out/e16_vw.log
timeout 900 python -m pytest tests/test_gpu_collectives.py -q -x -k "test_multi_gpu and 2" > gpurun_out/e16_mp.log 2>&1; echo "mp rc=$?"; tail -n 2 gpurun_out/e16_mp.log
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for cfg in "libhz.so:" "libhz.so:gq=0" "libhz_b4.so:" "libhz_b4.so:gq=0"; do
  i=$((i+1)); lib=${cfg%%:*}; t=${cfg#*:}
  HZ_LIB=$lib HZ_TUNE=$t timeout 600 $B --master-port 2969$i bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e16_b2_$i.log 2>&1; echo "[$cfg] rc=$?"
  echo "[$cfg] $(grep '^{' gpurun_out/e16_b2_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["step_model"]["frac_of_model_bidir_probe"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2), round(v.get("avg_publish_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"
done
