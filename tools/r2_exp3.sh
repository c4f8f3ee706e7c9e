#!/bin/bash
# N=2 experiments: coherent vs non-coherent peer loads, one-process NVLink ncu of the P2P kernels.
mkdir -p gpurun_out
B="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 600 $B --master-port 29611 bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e3_bench2_a.log 2>&1; echo "a rc=$?"
HZ_LIB=libhz_nc.so timeout 600 $B --master-port 29612 bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e3_bench2_nc.log 2>&1; echo "nc rc=$?"
timeout 600 $B --master-port 29613 bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e3_bench2_b.log 2>&1; echo "b rc=$?"
HZ_TUNE=pdl=1 timeout 600 $B --master-port 29614 bench.py --gpus 2 --no-cpu-baseline --no-e2e --no-tail --no-flat > gpurun_out/e3_bench2_pdl.log 2>&1; echo "pdl rc=$?"
for f in a nc b pdl; do echo "$f $(grep '^{' gpurun_out/e3_bench2_$f.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["ms_per_step"], {k:(round(v["avg_ms"]*1e3,1), round(v.get("avg_wait_ms",0)*1e3,2), round(v.get("avg_publish_ms",0)*1e3,2)) for k,v in d["stages"].items()})')"; done
timeout 900 python -m pytest tests/test_gpu_vworld.py -q -m multigpu -x > gpurun_out/e3_vw_pytest.log 2>&1; echo "vw mp pytest rc=$?"; tail -n 2 gpurun_out/e3_vw_pytest.log
timeout 300 python tools/vw_profile.py --gpus 2 --layers 3 --time > gpurun_out/e3_vwp.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum,lts__t_sectors_srcunit_ltcfabric.sum \
  --clock-control none -k regex:k_ --csv --log-file gpurun_out/e3_vwp_ncu.csv python tools/vw_profile.py --gpus 2 --layers 3 --steps 1 > gpurun_out/e3_vwp_ncu.log 2>&1; echo "vwp ncu rc=$?"
tail -n 3 gpurun_out/e3_vwp.log
