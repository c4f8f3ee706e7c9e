#!/usr/bin/env python
"""Render tools/msg_sweep.py JSONL files as markdown tables (median ms, algbw GB/s,
wire GB/s per rank, and the flat/hz time ratios)."""
import json
import sys


def table(path):
    rows = {}
    for line in open(path):
        d = json.loads(line)
        rows.setdefault(d["bytes"], {})[d["op"]] = d
    first = next(iter(rows.values()))
    d0 = next(iter(first.values()))
    out = [f"### {d0['n_gpus']} GPUs, hierarchy {tuple(d0['hierarchy'])}, hz transport "
           f"{first['hz_allgather_fwd']['transport']}  (`{path.split('/')[-1]}`)", "",
           "| logical bytes | hz AG fwd ms (algbw) | hz AG bwd ms (algbw, wire/rank) | hz RS ms (algbw) "
           "| flat AG ms (algbw, wire) | flat RS ms (algbw) | AG fwd speedup | AG bwd speedup | RS speedup "
           "| back-to-back ms: hz fwd / bwd / RS, flat AG / RS |",
           "|---|---|---|---|---|---|---|---|---|---|"]
    for S, r in sorted(rows.items()):
        f, b, rs = r["hz_allgather_fwd"], r["hz_allgather_bwd"], r["hz_reduce_scatter"]
        fa, fr = r["flat_allgather"], r["flat_reduce_scatter"]
        size = f"{S >> 20} MB" if S < 1 << 30 else f"{S >> 30} GB"
        out.append(f"| {size} | {f['ms_median']:.3f} ({f['algbw_GBps']:.0f}) "
                   f"| {b['ms_median']:.3f} ({b['algbw_GBps']:.0f}, {b['wire_GBps_per_rank']:.0f}) "
                   f"| {rs['ms_median']:.3f} ({rs['algbw_GBps']:.0f}) "
                   f"| {fa['ms_median']:.3f} ({fa['algbw_GBps']:.0f}, {fa['wire_GBps_per_rank']:.0f}) "
                   f"| {fr['ms_median']:.3f} ({fr['algbw_GBps']:.0f}) "
                   f"| {fa['ms_median'] / f['ms_median']:.2f} | {fa['ms_median'] / b['ms_median']:.2f} "
                   f"| {fr['ms_median'] / rs['ms_median']:.2f} "
                   + ("| " + " / ".join(f"{r_['ms_loop']:.3f}" for r_ in (f, b, rs)) + ", "
                      + " / ".join(f"{r_['ms_loop']:.3f}" for r_ in (fa, fr)) + " |" if "ms_loop" in f else "| — |"))
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print("\n".join(table(p) for p in sys.argv[1:]))
