#!/bin/bash
# N = 2 / 4 bench lines with the complete N>1 ncu traffic table; ncu --set full of the backward
# triple kernel at N = 2 (virtual world, serial launches)
mkdir -p gpurun_out /tmp/ncu
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $B --nproc-per-node 2 --master-port 29862 bench.py --gpus 2 > gpurun_out/final2_bench2.log 2>&1; echo "bench2 rc=$?"
timeout 900 $B --nproc-per-node 4 --master-port 29864 bench.py --gpus 4 > gpurun_out/final2_bench4.log 2>&1; echo "bench4 rc=$?"
HZ_TUNE=vwserial=1 timeout 300 python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/final2_vwp.log 2>&1 && \
HZ_TUNE=vwserial=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gather_quantize_reduce -c 1 \
  -o /tmp/ncu/triple -f python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/final2_ncu.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/ncu/triple.ncu-rep --page details --csv > gpurun_out/r02_triple_details.csv 2>/dev/null
ncu -i /tmp/ncu/triple.ncu-rep --page source --csv > gpurun_out/r02_triple_source.csv 2>/dev/null
for f in final2_bench2 final2_bench4; do grep '^{' gpurun_out/$f.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); r=d["roofline"]; print(d["n_gpus"], d["ms_per_step"], r["kernel"], round(r["frac"],3), r.get("traffic"), r.get("nvlink_traffic"))'; done
