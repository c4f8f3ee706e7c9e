#!/bin/bash
# fp32 round trip with TMA stores (OUT=4): parity + N=1 A/B
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/e26_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/e26_pytest.log
for t in "" "fb=0" "" "fb=0"; do
  HZ_TUNE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e26.log 2>&1; echo "[$t] rc=$?"
  echo "[$t] $(grep '^{' gpurun_out/e26.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1e3,2) for k,v in d["stages"].items()})')"
done
