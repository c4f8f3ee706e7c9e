#!/bin/bash
# Round-end validation on a 4-GPU box: build, smoke, full GPU test suite, and the
# bench contract (N = 1 default line, --impl reference, N = 2 and 4 under torchrun).
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/rc_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/rc_pytest.log
timeout 600 python bench.py > gpurun_out/rc_bench1.log 2>&1; echo "bench1 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/rc_ref1.log 2>&1; echo "ref rc=$?"
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2990$n bench.py --gpus $n > gpurun_out/rc_bench$n.log 2>&1; echo "bench$n rc=$?"
done
for f in gpurun_out/rc_bench1.log gpurun_out/rc_ref1.log gpurun_out/rc_bench2.log gpurun_out/rc_bench4.log; do
  grep '^{' $f | tail -n 1 | cut -c1-400
done
