#!/bin/bash
# 2/4-GPU validation: real multi-process parity (P2P + NCCL transports) and the N>1 bench lines.
N=${1:-2}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/c2_topo.log 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/c2_build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_collectives.py -q -m multigpu -x --timeout 900 > gpurun_out/c2_mp_pytest.log 2>&1; echo "mp pytest rc=$?"; tail -n 3 gpurun_out/c2_mp_pytest.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29602 \
  bench.py --gpus $N > gpurun_out/c2_bench${N}.log 2>&1; echo "bench$N rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29603 \
  bench.py --gpus $N --transport nccl --no-cpu-baseline --no-e2e > gpurun_out/c2_bench${N}_nccl.log 2>&1; echo "bench$N nccl rc=$?"
for f in gpurun_out/c2_bench${N}.log gpurun_out/c2_bench${N}_nccl.log; do grep '^{' $f | tail -n 1 | cut -c1-400; done
