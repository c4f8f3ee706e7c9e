#!/bin/bash
# Round-end validation: build, smoke, full GPU test suite, and the bench contract
# (N = 1 default line, --impl reference, N = 2 / 4 under torchrun when the box has them),
# plus the ncu evidence of this round (N = 1 launch list, dual-kernel full capture).
# usage: bash tools/round_check.sh [max_gpus]
NMAX=${1:-4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/rc_pytest.log 2>&1; echo "pytest rc=$?"; tail -n 2 gpurun_out/rc_pytest.log
timeout 600 python bench.py > gpurun_out/rc_bench1.log 2>&1; echo "bench1 rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/rc_ref1.log 2>&1; echo "ref rc=$?"
for n in 2 4; do
  [ $n -gt $NMAX ] && continue
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
    --master-port 2990$n bench.py --gpus $n > gpurun_out/rc_bench$n.log 2>&1; echo "bench$n rc=$?"
done
timeout 300 python tools/kbench.py --pair > gpurun_out/rc_pair.log 2>&1; echo "pair rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file gpurun_out/rc_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
  --no-tail > gpurun_out/rc_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gather_quantize -c 2 \
  -o gpurun_out/rc_pair_full -f python tools/kbench.py --pair --once > gpurun_out/rc_ncu_pair.log 2>&1; echo "ncu pair rc=$?"
for f in gpurun_out/rc_bench1.log gpurun_out/rc_ref1.log gpurun_out/rc_bench2.log gpurun_out/rc_bench4.log; do
  [ -f $f ] && grep '^{' $f | tail -n 1 | cut -c1-300
done
