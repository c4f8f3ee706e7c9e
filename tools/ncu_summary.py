#!/usr/bin/env python
"""Summarise ncu captures for profiles/ (run here, on the CPU box, on files that
gpurun brought back):

  python tools/ncu_summary.py --launches gpurun_out/launches_rNN.csv \
      --rep gpurun_out/prof_rNN.ncu-rep --out profiles/rNN

writes <out>_launches.md (per-kernel share of the timed step from the launch list),
<out>_kernels.md (key metrics of the full capture) and updates profiles/ncu_traffic.json
(DRAM bytes per element of each kernel kind, read by bench.py's roofline block)."""

import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

KIND = [  # (regex on the demangled kernel name, kind used by the library trace)
    (r"k_gather_quantize_reduce", "gather_quantize_reduce"),
    (r"k_gather_quantize", "gather_quantize"),
    (r"k_tiles", "tiles"),
    (r"k_quantize<[^,<>]+, \d+, \d+, \d+, [1-6]\b", "quantize_dequantize"),
    (r"k_quantize", "quantize"),
    (r"k_dequantize", "dequantize"),
    (r"k_reduce_requant", "reduce_requant"),
    (r"k_reduce_f32", "reduce"),
    (r"k_adamw", "adamw"),
    (r"k_gather_copy", "gather_copy"),
]


def kind_of(name):
    for rx, k in KIND:
        if re.search(rx, name):
            return k
    return None


def read_csv(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    return list(csv.DictReader(io.StringIO("".join(lines))))


def launches(path, last):
    rows = read_csv(path)
    per = collections.OrderedDict()
    for r in rows:
        key = r["ID"]
        d = per.setdefault(key, {"name": r["Kernel Name"], "grid": r["Grid Size"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    ours = [v for v in per.values() if kind_of(v["name"])]
    ours = ours[-last:] if last else ours
    agg = collections.OrderedDict()
    for v in ours:
        k = kind_of(v["name"])
        a = agg.setdefault(k, {"launches": 0, "ns": 0.0, "dram": 0.0})
        a["launches"] += 1
        a["ns"] += v.get("gpu__time_duration.sum", 0.0)
        a["dram"] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    return ours, agg


def rep_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = read_csv_text(out)
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Theoretical Occupancy",
            "Registers Per Thread", "Issue Slots Busy", "Executed Ipc Active", "L2 Hit Rate", "Grid Size",
            "Compute (SM) Throughput", "Warp Cycles Per Issued Instruction", "No Eligible"]
    per = collections.OrderedDict()
    for r in rows:
        d = per.setdefault(r["ID"], {"name": r["Kernel Name"]})
        if r["Metric Name"] in want:
            d[r["Metric Name"]] = f'{r["Metric Value"]} {r["Metric Unit"]}'.strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    lines = [l for l in raw.splitlines() if l and not l.startswith("==")]
    hdr = next(csv.reader([lines[0]]))
    units = dict(zip(hdr, next(csv.reader([lines[1]]))))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for row in csv.reader(lines[2:]):
        r = dict(zip(hdr, row))
        d = per.get(r.get("ID"))
        if d is None:
            continue
        try:
            rd = float(r["dram__bytes_read.sum"].replace(",", "")) * scale[units["dram__bytes_read.sum"]]
            wr = float(r["dram__bytes_write.sum"].replace(",", "")) * scale[units["dram__bytes_write.sum"]]
            d["dram_read_bytes"] = rd
            d["dram_write_bytes"] = wr
            d["dram_bytes"] = rd + wr
        except (KeyError, ValueError):
            pass
    return per


def read_csv_text(text, header_skip=False):
    lines = [l for l in text.splitlines() if l and not l.startswith("==")]
    if header_skip and len(lines) > 1:
        # raw page: second line holds units
        hdr = next(csv.reader([lines[0]]))
        body = lines[2:]
        return [dict(zip(hdr, row)) for row in csv.reader(body)]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--last", type=int, default=0, help="keep only the last N launches of our kernels")
    ap.add_argument("--rep")
    ap.add_argument("--rep-elems", default="", help="comma list: element count per captured launch")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    if a.launches:
        ours, agg = launches(a.launches, a.last)
        tot = sum(v["ns"] for v in agg.values()) or 1
        with open(a.out + "_launches.md", "w") as f:
            f.write(f"# ncu launch list ({os.path.basename(a.launches)}), last {len(ours)} launches of libhz kernels\n\n")
            f.write("cold-cache, serialised replay (`--metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                    "dram__bytes_write.sum --clock-control none`): compare SHARES, not absolutes\n\n")
            f.write("| kernel kind | launches | total us | share | avg us | DRAM MB / launch |\n|---|---|---|---|---|---|\n")
            for k, v in agg.items():
                f.write(f"| {k} | {v['launches']} | {v['ns']/1e3:.1f} | {v['ns']/tot:.3f} | {v['ns']/v['launches']/1e3:.2f} |"
                        f" {v['dram']/v['launches']/1e6:.2f} |\n")
        print(open(a.out + "_launches.md").read())
    if a.rep:
        per = rep_metrics(a.rep)
        elems = [int(x) for x in a.rep_elems.split(",") if x]
        traffic_path = os.path.join(os.path.dirname(a.out) or ".", "ncu_traffic.json")
        traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
        with open(a.out + "_kernels.md", "w") as f:
            f.write(f"# ncu --set full ({os.path.basename(a.rep)})\n\n")
            for i, (kid, d) in enumerate(per.items()):
                f.write(f"## {kid}: {d['name'][:140]}\n\n")
                for k, v in d.items():
                    if k not in ("name",):
                        f.write(f"- {k}: {v}\n")
                if i < len(elems) and "dram_bytes" in d:
                    f.write(f"- elements: {elems[i]}; DRAM bytes / element: {d['dram_bytes']/elems[i]:.4f} "
                            f"(read {d['dram_read_bytes']/elems[i]:.4f}, write {d['dram_write_bytes']/elems[i]:.4f}; "
                            "writes still dirty in L2 at kernel end are not counted)\n")
                    k = kind_of(d["name"])
                    if k:
                        # several variants of one kind in one capture: average bytes per element
                        prev = traffic.get(k) if traffic.get(k, {}).get("source") == os.path.basename(a.rep) else None
                        if prev:
                            prev["dram_bytes"] = (prev["dram_bytes"] / prev["elems"] + d["dram_bytes"] / elems[i]) / 2 * elems[i]
                            prev["elems"] = elems[i]
                            prev["kernel"] += " | " + d["name"][:120]
                        elif k not in traffic or traffic[k].get("source") != os.path.basename(a.rep):
                            traffic[k] = {"dram_bytes": d["dram_bytes"], "elems": elems[i],
                                          "source": os.path.basename(a.rep), "kernel": d["name"][:160]}
                f.write("\n")
        json.dump(traffic, open(traffic_path, "w"), indent=1)
        print(open(a.out + "_kernels.md").read()[:6000])


if __name__ == "__main__":
    main()
