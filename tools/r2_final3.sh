#!/bin/bash
# N = 1 evidence after the world-1 carveout scope: smoke, the full bench line, GPU suite, and the
# ncu launch list of the same bench command (plain run first)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f3_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f3_smoke.log
timeout 900 python bench.py > gpurun_out/f3_bench1.log 2>&1; echo "bench1 rc=$?"
grep '^{' gpurun_out/f3_bench1.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["value"]), d["roofline"]["kernel"], round(d["roofline"]["frac"],4), round(d["step_model"]["frac_of_model"],4), d["e2e"]["ms_per_step"], d["gpu_launches"], d["clocks"])'
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-tail"
$C > gpurun_out/f3_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02c_launches.csv $C > gpurun_out/f3_ncu.log 2>&1; echo "launch list rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f3_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/f3_pytest.log
