#!/bin/bash
# TMA tile engine: full 1-GPU parity suite, then the N=1 bench with the engine on / off
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/e10_smoke.log 2>&1; echo "smoke rc=$?"; tail -n 2 gpurun_out/e10_smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/e10_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/e10_pytest.log
for t in "tma=1" "tma=0" "tma=1,tte=8192,ts=2" "tma=1,ts=2"; do
  HZ_TUNE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e10_b1_$t.log 2>&1; echo "$t rc=$?"
  echo "$t $(grep '^{' gpurun_out/e10_b1_$t.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], d["roofline"]["frac"], {k:(round(v["avg_ms"]*1e3,1)) for k,v in d["stages"].items()})')"
done
