#!/bin/bash
# dequantize / gather output by TMA bulk stores: parity + N=1 and N=2 A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/e27_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/e27_pytest.log
for t in "" "fbd=0" "" "fbd=0"; do
  HZ_TUNE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e27.log 2>&1; echo "[$t] rc=$?"
  echo "[$t] $(grep '^{' gpurun_out/e27.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1e3,2) for k,v in d["stages"].items()})')"
done
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for t in "" "fbd=0"; do
  i=$((i+1))
  HZ_TUNE=$t timeout 600 $B --master-port 2975$i bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e27_b2.log 2>&1; echo "[N2 $t] rc=$?"
  echo "[N2 $t] $(grep '^{' gpurun_out/e27_b2.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})')"
done
