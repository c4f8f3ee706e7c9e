#!/bin/bash
# N3 diagnostic: launch statistics and occupancy limiters of the cuBLAS GEMMs of the synthetic
# GPT-1.3B layer (1024 tokens), to see whether a libhz CTA can be co-resident beside them
mkdir -p gpurun_out
timeout 600 ncu --section LaunchStats --section Occupancy --clock-control none -c 60 --csv --page details \
  --log-file gpurun_out/gemm_occ.csv python tools/train_step.py --tokens 1024 --layers 2 --steps 1 --warmup 1 \
  --modes compute > gpurun_out/gemm_occ.log 2>&1
echo "ncu rc=$?"
python - <<'PY'
import csv, collections
rows = list(csv.reader(open("gpurun_out/gemm_occ.csv")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
want = ("Registers Per Thread", "Shared Memory Configuration Size", "Dynamic Shared Memory Per Block",
        "Static Shared Memory Per Block", "Block Size", "Grid Size", "Block Limit Registers",
        "Block Limit Shared Mem", "Theoretical Occupancy", "Waves Per SM")
k = collections.OrderedDict()
for r in rows[hdr + 1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        k.setdefault((d["Kernel Name"][:90]), {})[d["Metric Name"]] = d["Metric Value"] + " " + d.get("Metric Unit", "")
for name, m in k.items():
    print(name, m)
PY
