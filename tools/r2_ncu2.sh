#!/bin/bash
# ncu metrics pass of the P2P kernels of a real 2-GPU exchange (incl. the backward triple kernel), one process
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum
timeout 300 python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/n2_vwp.log 2>&1 && \
timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/r02_vwp2_triple_ncu.csv \
  python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/n2_vwp_ncu.log 2>&1; echo "ncu rc=$?"
