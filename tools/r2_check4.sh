#!/bin/bash
# 4-GPU validation: multi-process parity at 2 and 4 ranks (all transports), multi-device vworld,
# N=2 / N=4 bench lines, and the ncu metrics pass of the P2P kernels over real NVLink (one process).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_collectives.py tests/test_gpu_vworld.py -q -m multigpu > gpurun_out/c4_mp.log 2>&1; echo "mp rc=$?"; tail -n 3 gpurun_out/c4_mp.log
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $B --nproc-per-node 2 --master-port 29702 bench.py --gpus 2 > gpurun_out/c4_bench2.log 2>&1; echo "bench2 rc=$?"
timeout 900 $B --nproc-per-node 4 --master-port 29704 bench.py --gpus 4 > gpurun_out/c4_bench4.log 2>&1; echo "bench4 rc=$?"
for n in 2 4; do grep '^{' gpurun_out/c4_bench$n.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["ms_per_step"], d["value"], d["roofline"]["kernel"], round(d["roofline"]["frac"],3), round(d["step_model"]["frac_of_model_bidir_probe"],3), {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})'; done
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum
for n in 2 4; do
  timeout 300 python tools/vw_profile.py --gpus $n --layers 3 --steps 1 > gpurun_out/c4_vwp$n.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none -k regex:k_ --csv --log-file gpurun_out/c4_vwp${n}_ncu.csv \
    python tools/vw_profile.py --gpus $n --layers 3 --steps 1 > gpurun_out/c4_vwp${n}_ncu.log 2>&1; echo "ncu vwp$n rc=$?"
done
