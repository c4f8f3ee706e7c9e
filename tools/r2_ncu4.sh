#!/bin/bash
# virtual-world ncu metrics pass with application replay (no per-kernel memory save/restore,
# which can revert a peer's flag writes into this GPU's pool during a replayed kernel)
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum
HZ_TUNE=vwserial=1 timeout 300 python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/n4_vwp.log 2>&1
HZ_TUNE=vwserial=1 timeout 600 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/n4_ser2.csv \
  python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/n4_ser2.log 2>&1; echo "ncu app N=2 rc=$?"
HZ_TUNE=vwserial=1 timeout 300 python tools/vw_profile.py --gpus 4 --layers 3 --steps 1 > gpurun_out/n4_vwp4.log 2>&1
HZ_TUNE=vwserial=1 timeout 600 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/n4_ser4.csv \
  python tools/vw_profile.py --gpus 4 --layers 3 --steps 1 > gpurun_out/n4_ser4.log 2>&1; echo "ncu app N=4 rc=$?"
