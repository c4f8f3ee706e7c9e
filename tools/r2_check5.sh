#!/bin/bash
# 4-GPU validation of the final round-2 library: multi-process parity at 2/4 ranks (all transports),
# multi-device virtual world, N=1/2/4 bench lines (default + defer=0 at N=4)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_collectives.py tests/test_gpu_vworld.py -q -m multigpu > gpurun_out/c5_mp.log 2>&1; echo "mp rc=$?"; tail -n 3 gpurun_out/c5_mp.log
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python bench.py > gpurun_out/c5_bench1.log 2>&1; echo "bench1 rc=$?"
timeout 900 $B --nproc-per-node 2 --master-port 29712 bench.py --gpus 2 > gpurun_out/c5_bench2.log 2>&1; echo "bench2 rc=$?"
timeout 900 $B --nproc-per-node 4 --master-port 29714 bench.py --gpus 4 > gpurun_out/c5_bench4.log 2>&1; echo "bench4 rc=$?"
HZ_TUNE=defer=0 timeout 900 $B --nproc-per-node 4 --master-port 29715 bench.py --gpus 4 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/c5_bench4_nodefer.log 2>&1; echo "bench4 defer=0 rc=$?"
for f in c5_bench1 c5_bench2 c5_bench4 c5_bench4_nodefer; do grep '^{' gpurun_out/$f.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["n_gpus"], d["ms_per_step"], round(d["value"]), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), round(d["step_model"]["frac_of_model_bidir_probe"],3), (d.get("e2e") or {}).get("ms_per_step"), d["gpu_launches"], {k:round(v["avg_ms"]*1e3,1) for k,v in d["stages"].items()})'; done
