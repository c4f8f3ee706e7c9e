#!/usr/bin/env python
"""Per-kernel-kind DRAM and NVLink bytes per element from an ncu metrics CSV (tool).

Reads the CSV of an `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum,nvlrx__bytes.sum,nvltx__bytes.sum --csv` run of
tools/vw_profile.py (one process, rank r on GPU r: the P2P kernels of a real N-GPU
exchange, launches serialised by ncu) and merges, per kernel kind, the summed bytes and
the summed element counts into profiles/ncu_traffic.json under the key "<kind>@N<n>"
(bench.py looks this key up first for an N-GPU line; "traffic" = bytes per element x
the launch's elements).  Element counts come from the launch arguments the library
traces (one vw_profile pass with HZ trace stamps), so they are given here per kernel
name: --elems 'regex=count,...' (';'-separated; the number of elements one launch of that kernel
processes: gathered + quantized).

    python tools/ncu_traffic_update.py gpurun_out/e8_vwp_ncu.csv --n 2 \\
        --kind 'k_gather_quantize=gather_quantize' --elems 'quantize<__nv_bfloat16, 8=75537408;quantize<__nv_bfloat16, 4=100716544'
"""

import argparse
import csv
import json
import os
import re
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: i for i, h in enumerate(hdr)}
    launches = defaultdict(dict)
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        key = (r[ix["ID"]], r[ix["Kernel Name"]])
        v = r[ix["Metric Value"]].replace(",", "")
        try:
            launches[key][r[ix["Metric Name"]]] = float(v)
        except ValueError:
            pass
    return launches


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--n", type=int, required=True, help="GPUs of the profiled exchange")
    ap.add_argument("--kind", required=True, help="kernel-name regex=kind;...")
    ap.add_argument("--elems", required=True, help="kernel-name regex=elements per launch;...")
    ap.add_argument("--source", default="")
    args = ap.parse_args()
    kinds = [kv.split("=", 1) for kv in args.kind.split(";")]
    elems = [(k, int(v)) for k, v in (kv.split("=", 1) for kv in args.elems.split(";"))]
    acc = defaultdict(lambda: defaultdict(float))
    for (_, name), m in read(args.csv).items():
        kind = next((k for rx, k in kinds if re.search(rx, name)), None)
        if kind is None:
            continue
        ne = next((n for rx, n in elems if re.search(rx, name)), None)
        if ne is None:
            continue
        a = acc[kind]
        a["dram"] += m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
        a["nvlrx"] += m.get("nvlrx__bytes.sum", 0)
        a["nvltx"] += m.get("nvltx__bytes.sum", 0)
        a["ns"] += m.get("gpu__time_duration.sum", 0)
        a["elems"] += ne
        a["launches"] += 1
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    d = json.load(open(path)) if os.path.exists(path) else {}
    for kind, a in acc.items():
        d[f"{kind}@N{args.n}"] = {
            "dram_bytes": a["dram"], "nvlink_rx_bytes": a["nvlrx"], "nvlink_tx_bytes": a["nvltx"],
            "elems": a["elems"], "launches": int(a["launches"]), "ncu_ns": a["ns"],
            "source": args.source or os.path.basename(args.csv),
            "how": "ncu metrics pass over tools/vw_profile.py (one process, one rank per GPU, launches serialised: "
                   "the peer is idle while a kernel runs, so NVLink carries one direction at a time)",
        }
        print(kind, json.dumps(d[f"{kind}@N{args.n}"]))
    with open(path, "w") as f:
        json.dump(d, f, indent=1)


if __name__ == "__main__":
    main()
