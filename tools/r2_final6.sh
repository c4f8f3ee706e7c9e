#!/bin/bash
# 2-GPU sanity after the store-mode defaults flip: the multi-process GPU tests and the N = 2 line
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_collectives.py tests/test_gpu_tiles.py -m gpu -x -q > gpurun_out/f6_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/f6_pytest.log
B="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 $B --nproc-per-node 2 --master-port 29882 bench.py --gpus 2 > gpurun_out/f6_bench2.log 2>&1; echo "bench2 rc=$?"
grep '^{' gpurun_out/f6_bench2.log | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["value"]), d["roofline"]["kernel"], round(d["roofline"]["frac"],4), round(d["step_model"]["frac_of_model_bidir_probe"],4), d["e2e"]["ms_per_step"], d["clocks"]["reasons"])'
