#!/bin/bash
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/c1_smi.log 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c1_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/c1_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 3 gpurun_out/c1_pytest.log
timeout 600 python bench.py > gpurun_out/c1_bench1.log 2>&1; echo "bench1 rc=$?"
grep '^{' gpurun_out/c1_bench1.log | tail -n 1 | cut -c1-600
