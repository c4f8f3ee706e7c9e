#!/bin/bash
# gathered layer by TMA bulk stores in the dual / triple kernels: parity + N=2 / N=4 A/B
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_vworld.py -q -x > gpurun_out/e28_vw.log 2>&1; echo "vworld rc=$?"; tail -n 2 gpurun_out/e28_vw.log
timeout 1200 python -m pytest tests/test_gpu_collectives.py -q -x -k "test_multi_gpu and (2 or 4)" > gpurun_out/e28_mp.log 2>&1; echo "mp rc=$?"; tail -n 2 gpurun_out/e28_mp.log
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
i=0
for cfg in "2:" "2:dgb=0" "4:" "4:dgb=0" "2:" "2:dgb=0"; do
  i=$((i+1)); n=${cfg%%:*}; t=${cfg#*:}
  HZ_TUNE=$t timeout 600 $B --nproc-per-node $n --master-port 2976$i bench.py --gpus $n --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e28_$i.log 2>&1; echo "[N$n $t] rc=$?"
  echo "[N$n $t] $(grep '^{' gpurun_out/e28_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})')"
done
