#!/bin/bash
# N=1: fp32 round trip register bound / unroll
mkdir -p gpurun_out
for cfg in "libhz.so:" "libhz_rt4.so:" "libhz.so:rt_u=2" "libhz.so:" "libhz_rt4.so:"; do
  lib=${cfg%%:*}; t=${cfg#*:}
  HZ_LIB=$lib HZ_TUNE=$t timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e20.log 2>&1; echo "[$cfg] rc=$?"
  echo "[$cfg] $(grep '^{' gpurun_out/e20.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["roofline"]["frac"],4), {k:round(v["avg_ms"]*1e3,2) for k,v in d["stages"].items()})')"
done
