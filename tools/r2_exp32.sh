#!/bin/bash
# cp.async-pipelined gather+dequantize (dqa=1): parity, N=1 and N=2 A/B
mkdir -p gpurun_out
HZ_TUNE=dqa=1 timeout 900 python -m pytest tests/test_gpu_codec.py tests/test_gpu_vworld.py -q -x -k "dequantize or hierarchy or full_size" > gpurun_out/e32_pt.log 2>&1; echo "parity dqa rc=$?"; tail -n 2 gpurun_out/e32_pt.log
for t in "" "dqa=1" "" "dqa=1"; do
  HZ_TUNE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e32.log 2>&1; echo "[N1 $t] rc=$?"
  echo "[N1 $t] $(grep '^{' gpurun_out/e32.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:round(v["avg_ms"]*1e3,2) for k,v in d["stages"].items()})')"
done
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for t in "" "dqa=1"; do
  i=$((i+1))
  HZ_TUNE=$t timeout 600 $B --master-port 2979$i bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e32_b2.log 2>&1; echo "[N2 $t] rc=$?"
  echo "[N2 $t] $(grep '^{' gpurun_out/e32_b2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})')"
done
