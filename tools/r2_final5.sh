#!/bin/bash
# N = 1 after the store-mode defaults flip (fbd=0, fbb=1 under the world-1 carveout): GPU suite,
# smoke, the full bench line, the ncu launch list of the same command
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/f5_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/f5_pytest.log
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f5_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f5_smoke.log
timeout 900 python bench.py > gpurun_out/f5_bench1.log 2>&1; echo "bench1 rc=$?"
grep '^{' gpurun_out/f5_bench1.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["value"]), d["roofline"]["kernel"], round(d["roofline"]["frac"],4), round(d["step_model"]["frac_of_model"],4), d["e2e"]["ms_per_step"], d["gpu_launches"], d["clocks"], {k:round(v["avg_ms"]*1000,2) for k,v in d["stages"].items()})'
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-tail"
$C > gpurun_out/f5_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02d_launches.csv $C > gpurun_out/f5_ncu.log 2>&1; echo "launch list rc=$?"
