#!/bin/bash
# does the virtual-world ncu stall depend on the deferred last hop?
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum
timeout 300 python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/n3_vwp.log 2>&1
HZ_TUNE=defer=0 timeout 420 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/n3_nodefer.csv \
  python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/n3_nodefer.log 2>&1; echo "ncu defer=0 rc=$?"
timeout 420 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/n3_defer_l2.csv \
  python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/n3_defer_l2.log 2>&1; echo "ncu defer 2 layers rc=$?"
