#!/bin/bash
# round-2 ncu evidence at N = 1: launch list of the bench step (same command, plain run first),
# and one full capture of the dominant kernel (the fused round trip) with source counters
mkdir -p gpurun_out /tmp/ncu
C="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-tail"
$C > gpurun_out/n1b_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02b_launches.csv $C > gpurun_out/n1b_ncu_launch.log 2>&1; echo "launch list rc=$?"
python tools/kbench.py --step1 --once > gpurun_out/n1b_kb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_quantize -c 2 -o /tmp/ncu/rt -f \
  python tools/kbench.py --step1 --once > gpurun_out/n1b_ncu_full.log 2>&1; echo "full rc=$?"
ncu -i /tmp/ncu/rt.ncu-rep --page details --csv > gpurun_out/r02b_rt_details.csv 2>/dev/null
ncu -i /tmp/ncu/rt.ncu-rep --page raw --csv > gpurun_out/r02b_rt_raw.csv 2>/dev/null
ls -la /tmp/ncu
