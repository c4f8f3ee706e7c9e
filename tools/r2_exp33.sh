#!/bin/bash
# N3: shared-memory carveout of the libhz kernels (HZ_TUNE carve) so cuBLAS GEMM CTAs (~213-221 KB
# dynamic smem, 168 regs x 256 threads) can be co-resident with libhz CTAs; N = 2, 1024 tokens/GPU
N=2
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
run() {  # budget tune modes
  i=$((i+1))
  HZ_TUNE=$2 timeout 600 $B --master-port 2990$i tools/train_step.py --tokens 1024 --steps 5 --warmup 3 --budget $1 --modes $3 > gpurun_out/e33_$i.log 2>&1
  echo "budget=$1 tune=[$2] $(grep '^{' gpurun_out/e33_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print({k:(round(v["ms_per_step"],2) if isinstance(v,dict) else round(v,3)) for k,v in d["results"].items()})')"
}
run 0 "" compute,hz,flat
run 0 "carve=100" hz
run 37 "carve=100" hz
run 74 "carve=100" hz
run 37 "carve=100,grid_np=4" hz
run 0 "carve=100,grid_np=4" hz
run 37 "" hz
for t in "" "carve=100"; do
  HZ_TUNE=$t timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-tail > gpurun_out/e33_b1_$t.log 2>&1
  echo "bench1 [$t] $(grep '^{' gpurun_out/e33_b1_$t.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], round(d["roofline"]["frac"],4))')"
done
