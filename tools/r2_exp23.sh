#!/bin/bash
# GPT-6.7B at N=2: round-1 17.7 ms vs round-2 19.3 ms — which change?
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
i=0
for cfg in "libhz.so:" "libhz_nc.so:" "libhz.so:defer=0" "libhz.so:gqc=1" "libhz.so:"; do
  i=$((i+1)); lib=${cfg%%:*}; t=${cfg#*:}
  HZ_LIB=$lib HZ_TUNE=$t timeout 900 $B --master-port 2973$i bench.py --gpus 2 --config gpt6.7b --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e23_$i.log 2>&1; echo "[$cfg] rc=$?"
  echo "[$cfg] $(grep '^{' gpurun_out/e23_$i.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"
done
