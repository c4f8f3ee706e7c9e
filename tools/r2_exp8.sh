#!/bin/bash
# ncu --set full of the N=2 dual kernel (all-warps vs warp-specialised), reports kept under /tmp, CSV pages exported
mkdir -p gpurun_out /tmp/ncu
timeout 300 python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/e8_vwp.log 2>&1 && \
HZ_TUNE=lk=0 timeout 900 ncu --set full --metrics nvlrx__bytes.sum,nvltx__bytes.sum --clock-control none --import-source on -k regex:k_gather_quantize -c 2 -o /tmp/ncu/old -f python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/e8_ncu_old.log 2>&1; echo "ncu old rc=$?"
HZ_TUNE=lk=-2,lte=4096,ls=3 timeout 900 ncu --set full --metrics nvlrx__bytes.sum,nvltx__bytes.sum --clock-control none --import-source on -k regex:k_gather_quantize -c 2 -o /tmp/ncu/ws -f python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/e8_ncu_ws.log 2>&1; echo "ncu ws rc=$?"
HZ_TUNE=lk=0 timeout 900 ncu --set full --metrics nvlrx__bytes.sum,nvltx__bytes.sum --clock-control none --import-source on -k regex:k_reduce -c 2 -o /tmp/ncu/red -f python tools/vw_profile.py --gpus 2 --layers 2 --steps 1 > gpurun_out/e8_ncu_red.log 2>&1; echo "ncu red rc=$?"
for r in old ws red; do
  ncu -i /tmp/ncu/$r.ncu-rep --page raw --csv > gpurun_out/e8_${r}_raw.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page details --csv > gpurun_out/e8_${r}_details.csv 2>/dev/null
  ncu -i /tmp/ncu/$r.ncu-rep --page source --csv > gpurun_out/e8_${r}_source.csv 2>/dev/null
  ls -la /tmp/ncu/$r.ncu-rep
done
du -sh gpurun_out
