#!/usr/bin/env python
"""Benchmark of the hierarchical ZeRO++ data-parallel hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config gpt1.3b] [--impl hz|reference]

N > 1 is launched by the driver as
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P bench.py --gpus N --steps K --warmup W
(one rank per GPU; if started without torchrun and --gpus > 1 this script re-launches
itself that way).

A step = one pass of the whole hot path over every parameter tensor of the model
(GA = 1, setting T of the paper): per tensor, in forward order, the qwZ all-gather
(quantize primary -> per-level NCCL all-gather -> dequantize, keeping the hpZ
secondary), then in backward order the all-gather from the secondary and the qgZ
reduce-scatter (quantize -> per-level all-to-all -> dequantize+sum(+requantize) ->
fp32 gradient shard).  Inputs are resident in HBM before the timed region; every
step touches several GB (> 126 MB L2), so no L2 flush is needed between steps.

value = logical bytes of all ranks / time, logical bytes per tensor per rank =
2*psi (forward gathered bf16) + 2*psi (backward gathered bf16) + 2*psi (bf16
gradient in): 6*psi.  Weak scaling: per-rank work is fixed as N grows.

The calls are issued in a training step's order with adjacent layers paired
(--pipelined, default): hz_allgather_params_next gathers layer k and prefetches
the quantize of layer k+1 in the same launch; hz_backward_step reduce-scatters
layer i while gathering layer i-1 (one dual kernel on the NVLink transport).
--no-pipelined issues one call per collective.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "param all-gather + grad reduce-scatter GB/s per step at 1/2/4/8 B200, % roofline"
UNIT = "GB/s"
HIERARCHY = {
    "gpt1.3b": {1: (1,), 2: (2,), 4: (2, 2), 8: (2, 4)},
    "gpt6.7b": {1: (1,), 2: (2,), 4: (2, 2), 8: (2, 2, 2)},
    "neox20b": {1: (1,), 2: (2,), 4: (2, 2), 8: (2, 2, 2)},
}
KERNEL_KINDS = ("quantize", "dequantize", "gather_dequantize", "gather_quantize", "gather_quantize_reduce",
                "dequantize_roundtrip",
                "quantize_dequantize", "reduce",
                "reduce_requant")
NVLINK_NOMINAL_GBS = 900.0  # NVLink 5, per direction (north_star denominator)
NVLINK_PEER_GBS = 770.0     # fallback: measured peer copy per direction (B200_PROFILING.md)
NVLINK_BIDIR_PROBE_GBS = 620.0   # fallback: both GPUs of a pair pulling at once (profiles/bulk_probe_r01.txt)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["hz", "reference"], default="hz")
    ap.add_argument("--config", choices=sorted(HIERARCHY), default="gpt1.3b")
    ap.add_argument("--qwz-bits", type=int, default=8)
    ap.add_argument("--qgz-bits", type=int, default=4)
    ap.add_argument("--block", type=int, default=256)
    ap.add_argument("--roles", default="1,1",
                    help="w,s role levels (primary, hpZ secondary); 1,1 = the paper's ZeRO-topo (setting T); "
                         "L,1 or L,2 = ZeRO++ inside the hierarchy (setting Z); s=0 keeps a replicated secondary")
    ap.add_argument("--pipelined", action=argparse.BooleanOptionalAction, default=True,
                    help="issue the step through hz_allgather_params_next / hz_backward_step (adjacent layers "
                         "paired in one launch on the P2P transport); --no-pipelined: one call per collective")
    ap.add_argument("--layers", type=int, default=0, help="limit the tensor count (debug only)")
    ap.add_argument("--hierarchy", default="",
                    help="override the hierarchy, e.g. 4 = one level over all ranks (ZeRO++-style flat "
                         "qwZ / hpZ / qgZ) instead of the default 2,2")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flat", action="store_true")
    ap.add_argument("--no-alt", action="store_true", help="at 8 GPUs: skip the second hierarchy")
    ap.add_argument("--no-tail", action="store_true", help="skip the step-tail (AdamW + post-update gather) timing")
    ap.add_argument("--transport", choices=["p2p", "nccl"], default="p2p",
                    help="N>1 collective transport: fused NVLink peer-memory kernels (p2p) or NCCL")
    ap.add_argument("--cpu-sample-layers", type=int, default=4)
    ap.add_argument("--no-trace", action="store_true", help="no per-launch events (overhead check)")
    ap.add_argument("--graph", action=argparse.BooleanOptionalAction, default=True,
                    help="capture one step in a CUDA graph and time graph replays (--no-graph: eager)")
    args = ap.parse_args()
    args.w, args.s = (int(x) for x in args.roles.split(","))
    return args


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def relaunch_under_torchrun(args):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", "29533",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ------------------------------------------------------------------ measurement
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 50 ms from the warm-up through the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, devices):
        self.devices = set(devices)
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8 or not f[0].isdigit() or int(f[0]) not in self.devices:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        loaded = [s for s in sm if s > 0]
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (torch copy, read+write, measured)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def ncu_traffic():
    """Per-element DRAM bytes of each kernel kind from the committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


MIX_PROBE_ELEMS = 50358272
MIX_PROBE_KINDS = {   # kernel kind -> probe mixes (tools/hbm_mix_probe.cu) it averages over
    "quantize_dequantize": ("quantize_dequantize_bf16", "quantize_dequantize_f32"),
    "dequantize": ("dequantize",),
    "quantize": ("quantize",),
    # world-1 backward pair: dequantize of layer i-1 + qgZ round trip of layer i (equal sizes
    # except the embedding, so the per-element average of the two mixes)
    "dequantize_roundtrip": ("dequantize", "quantize_dequantize_f32"),
}


def same_mix_probe(kind, avg_elems, avg_ms):
    """Time a plain streaming kernel with this kind's read:write byte mix takes for the
    same element count (committed probe, profiles/hbm_mix_r01.json), and our kernel's
    fraction of it (> 1: faster than the plain streaming kernel)."""
    try:
        with open(os.path.join(ROOT, "profiles", "hbm_mix_r01.json")) as f:
            probe = json.load(f)
        keys = MIX_PROBE_KINDS[kind]
        us = sum(probe[k]["us"] for k in keys) / len(keys) * avg_elems / MIX_PROBE_ELEMS
    except (OSError, ValueError, KeyError):
        return {}
    return {"same_mix_probe_us": us, "frac_of_same_mix_probe": us / (avg_ms * 1e3),
            "same_mix_probe_source": "profiles/hbm_mix_r01.json (tools/hbm_mix_probe.cu)"}


# --------------------------------------------------------------------- the step
class Model:
    def __init__(self, hz, ctx, torch, config, rank, world, args, device):
        from paper_2501_04266_b200 import synth
        self.hz, self.ctx, self.torch = hz, ctx, torch
        self.args = args
        tensors = synth.model_tensors(config)
        if args.layers:
            tensors = tensors[:args.layers]
        self.tensors = []
        L = ctx.levels
        B = args.block
        max_np = 0
        self.p2p = ctx.p2p
        for i, (name, numel) in enumerate(tensors):
            p = ctx.partition(numel, B, w=args.w, s=args.s, gl=L)
            Np = p.padded_numel
            off_w, len_w = p.range(args.w)
            seed = 2000 + 97 * rank + i
            full_p = synth.torch_normal(Np, 7000 + i, 0.02, torch.bfloat16, device, outlier_every=0)
            full_p[numel:] = 0                                       # zero padding (O2)
            primary = full_p[off_w:off_w + len_w].clone()
            del full_p
            grad = synth.torch_normal(Np, seed, 1e-3, torch.bfloat16, device)
            grad[numel:] = 0
            _, len_s = p.range(args.s)
            _, len_l = p.range(L)
            t = {
                "name": name, "numel": numel, "p": p, "primary": primary, "grad": grad,
                "sec_c": self.alloc(len_s * args.qwz_bits // 8, torch.uint8, device),
                "sec_s": self.alloc(len_s // B, torch.float32, device),
                "shard": torch.empty(len_l, dtype=torch.float32, device=device),
            }
            self.tensors.append(t)
            max_np = max(max_np, Np)
        self.full = [torch.empty(max_np, dtype=torch.bfloat16, device=device) for _ in range(2)]
        self.bits = [args.qgz_bits] * L
        self.logical_bytes = sum(6 * t["numel"] for t in self.tensors)

    def alloc(self, numel, dtype, device):
        """hpZ secondaries must be peer-readable (symmetric pool) in P2P mode."""
        if self.p2p:
            return self.ctx.sym_alloc(numel, dtype)
        return self.torch.empty(numel, dtype=dtype, device=device)

    def step(self, stream):
        ctx, bits, T = self.ctx, self.args.qwz_bits, self.tensors
        if not self.args.pipelined:
            for i, t in enumerate(T):                                # forward: qwZ + hpZ
                ctx.allgather_params(t["p"], t["primary"], t["sec_c"], t["sec_s"], self.full[i & 1], bits=bits,
                                     stream=stream)
            for i, t in reversed(list(enumerate(T))):               # backward: gather from secondary, qgZ
                ctx.allgather_params(t["p"], None, t["sec_c"], t["sec_s"], self.full[i & 1], bits=bits,
                                     backward=True, stream=stream)
                ctx.reduce_scatter_grads(t["p"], t["grad"], t["shard"], self.bits, stream=stream)
            return
        # the same calls in a training step's issue order, adjacent layers paired
        # (hz_allgather_params_next / hz_backward_step: one launch per pair on the P2P transport)
        n = len(T)
        for i, t in enumerate(T):                                    # forward: gather i, prefetch quantize i+1
            nx = T[i + 1] if i + 1 < n else None
            ctx.allgather_params_next(t["p"], t["primary"], t["sec_c"], t["sec_s"], self.full[i & 1], bits=bits,
                                      p_next=nx["p"] if nx else None, next_primary=nx["primary"] if nx else None,
                                      next_sec_codes=nx["sec_c"] if nx else None,
                                      next_sec_scales=nx["sec_s"] if nx else None, stream=stream)
        t = T[n - 1]
        ctx.allgather_params(t["p"], None, t["sec_c"], t["sec_s"], self.full[(n - 1) & 1], bits=bits, backward=True,
                             stream=stream)
        for i in range(n - 1, -1, -1):                               # backward: qgZ of i || gather of i-1
            t, pv = T[i], (T[i - 1] if i > 0 else None)
            ctx.backward_step(t["p"], t["grad"], t["shard"], self.bits, p_prev=pv["p"] if pv else None,
                              prev_sec_codes=pv["sec_c"] if pv else None, prev_sec_scales=pv["sec_s"] if pv else None,
                              prev_full_out=self.full[(i - 1) & 1] if pv else None, prev_bits=bits, stream=stream)


def hierarchy_of(args, world):
    if args.hierarchy:
        g = tuple(int(x) for x in args.hierarchy.split(","))
        if math.prod(g) != world:
            raise SystemExit(f"--hierarchy {args.hierarchy}: product != {world} ranks")
        return g
    return HIERARCHY[args.config].get(world)


def p2p_pool_bytes(args, group):
    """Symmetric pool: every tensor's hpZ secondary + the library's per-level send slots."""
    from paper_2501_04266_b200 import synth
    W = math.prod(group)
    B = args.block
    unit = W * 4 * B
    total = 0
    max_np = 0
    for _, numel in synth.model_tensors(args.config):
        Np = -(-numel // unit) * unit
        len_s = Np // math.prod(group[:args.s])
        len_w = Np // math.prod(group[:args.w])
        total += len_s * args.qwz_bits // 8 + len_s // B * 4 + 512
        if args.s != args.w:                                      # quantized-primary slot
            total += len_w * args.qwz_bits // 8 + len_w // B * 4 + 512
        max_np = max(max_np, Np)
    total += 2 * (len(group) + 1) * (max_np + max_np // B * 4 + 512)   # slots + the last hop's 2nd (may grow once)
    total += 2 * (max_np // W) * 4 + 1024                       # step-tail update slot
    top = max_np // (W // group[-1])                             # len_{L-1}
    total += 2 * top * 4 + 1024                                 # allreduce + select ping-pong
    return int(total * 1.1) + (64 << 20)                        # bump-allocator slack


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def step_model(recs, steps, hbm_peak, nvl_peak=NVLINK_PEER_GBS, nvl_bidir=NVLINK_BIDIR_PROBE_GBS):
    """the modeled minimum of one step = the sum over the step's
    launches of each launch's roofline time, max(local HBM bytes / HBM peak, peer bytes /
    NVLink peak) (NCCL calls: bytes sent / NVLink peak) — every kernel at its roofline,
    back to back, no synchronisation.  Local HBM bytes include the bytes the group's peers
    read from this GPU (served bytes; equal to the bytes it reads from them, the
    exchanges being symmetric).  Returned per step, with the NVLink term at the one-way
    and at the bidirectional peer-read peak (both GPUs of a group pull at once), both
    measured in this run when N > 1 (hz_nvlink_probe)."""
    t, tb = 0.0, 0.0
    for r in recs:
        b, rem = float(r["bytes"]), float(r.get("remote_bytes", 0) or 0)
        if r["kind"].startswith("nccl"):
            b, rem = 0.0, b
        # the exchanges are symmetric: the members read from this GPU's HBM as many bytes
        # as it reads from theirs (served bytes), so its HBM moves bytes + rem
        t += max((b + rem) / (hbm_peak * 1e9), rem / (nvl_peak * 1e9))
        tb += max((b + rem) / (hbm_peak * 1e9), rem / (nvl_bidir * 1e9))
    return {"model_ms": t / steps * 1e3, "model_ms_bidir_probe": tb / steps * 1e3,
            "hbm_peak_GBps": hbm_peak, "nvlink_peak_GBps": nvl_peak, "nvlink_bidir_probe_GBps": nvl_bidir}


def nvlink_probe(ctx, rank, world, stream, nbytes=256 << 20):
    """The NVLink denominators of this run (hz_nvlink_probe: the fused kernels' own load
    path): one way (rank 0 pulls from rank 1 while the others idle) and bidirectional
    (every rank pulls from its partner r^1 at once; min over ranks), GB/s per direction."""
    if world < 2:
        return None
    try:
        out = {}
        barrier(world)
        ms = ctx.nvlink_probe(1, nbytes, 5, stream=stream) if rank == 0 else 0.0
        one = nbytes / (ms * 1e-3) / 1e9 if rank == 0 else 0.0
        out["one_way_GBps"] = max_over_ranks(one, world)
        barrier(world)
        ms = ctx.nvlink_probe(rank ^ 1, nbytes, 5, stream=stream)
        out["bidirectional_GBps"] = -max_over_ranks(-(nbytes / (ms * 1e-3) / 1e9), world)
        out["bytes"] = nbytes
        out["what"] = "hz_nvlink_probe: full-grid 16-byte coherent loads of a peer's pool (the gather/reduce load path)"
        return out
    except Exception as e:  # noqa: BLE001
        return {"error": str(e)[:200], "one_way_GBps": NVLINK_PEER_GBS, "bidirectional_GBps": NVLINK_BIDIR_PROBE_GBS}


def summarize_trace(recs, steps):
    kinds = {}
    for r in recs:
        r = dict(r)
        if r["ms"] < 0:                      # stamps-only trace: device-clock duration
            r["ms"] = r.get("stamp_ms", -1.0)
        if r["ms"] < 0:
            continue
        key = r["kind"]
        if key.startswith("reduce") or key.startswith("nccl"):
            key = f"{key}@L{r['level']}"          # per-level rows of the qgZ levels / hops
        k = kinds.setdefault(key, {"launches": 0, "ms": 0.0, "bytes": 0, "elems": 0, "remote": 0,
                                         "wait_ms": 0.0, "work_ms": 0.0, "publish_ms": 0.0, "stamped": 0})
        k["launches"] += 1
        k["ms"] += r["ms"]
        if r.get("wait_ms", -1) >= 0:
            k["stamped"] += 1
            k["wait_ms"] += r["wait_ms"]
            k["work_ms"] += r["work_ms"]
            k["publish_ms"] += max(r.get("publish_ms", 0.0), 0.0)
        k["bytes"] += r["bytes"]
        k["remote"] += r.get("remote_bytes", 0)
        k["elems"] += r["elems"]
    total_ms = sum(v["ms"] for v in kinds.values()) or 1.0
    out = {}
    for name, v in kinds.items():
        out[name] = {
            "launches_per_step": v["launches"] / steps,
            "avg_ms": v["ms"] / v["launches"],
            "avg_bytes": v["bytes"] / v["launches"],
            "avg_elems": v["elems"] / v["launches"],
            "GBps": v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else None,
            "share": v["ms"] / total_ms,
        }
        if v["remote"]:
            out[name]["avg_remote_bytes"] = v["remote"] / v["launches"]
            out[name]["nvlink_GBps"] = v["remote"] / (v["ms"] * 1e-3) / 1e9
        if v["stamped"]:
            out[name]["avg_wait_ms"] = v["wait_ms"] / v["stamped"]
            out[name]["avg_work_ms"] = v["work_ms"] / v["stamped"]
            out[name]["avg_publish_ms"] = v["publish_ms"] / v["stamped"]
    return out


def run_hz(args):
    import torch
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    from paper_2501_04266_b200 import hz

    group = hierarchy_of(args, world)
    if group is None:
        raise SystemExit(f"no hierarchy for {world} GPUs")
    if not (1 <= args.w <= len(group) and 0 <= args.s <= len(group)):
        raise SystemExit(f"--roles {args.roles}: need 1 <= w <= L and 0 <= s <= L (L = {len(group)})")
    uid = hz.get_uid() if rank == 0 else None
    if world > 1:
        import torch.distributed as dist
        box = [uid]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]
    ctx = hz.Context(rank, world, uid, group, local)
    transport = args.transport if world > 1 else "local"
    if transport == "p2p":
        ctx.enable_p2p(p2p_pool_bytes(args, group))
    model = Model(hz, ctx, torch, args.config, rank, world, args, device)
    stream = torch.cuda.current_stream()
    use_graph = args.graph

    # clocks are sampled from the start of the warm-up (under the same load) through
    # the end of the timed region: the timed region alone is often shorter than the
    # sampling period
    sampler = ClockSampler([local] if world == 1 else range(world)) if rank == 0 else None
    if sampler:
        sampler.start()
    for _ in range(max(args.warmup, 3)):
        model.step(stream)
    torch.cuda.synchronize()
    t_end = time.time() + 0.5                      # extra untimed steps: >= 0.5 s under load
    while max_over_ranks(time.time(), world) < t_end:
        model.step(stream)
        torch.cuda.synchronize()

    per_step_kernels = 5 * len(model.tensors)
    if not args.no_trace:
        # in-kernel device-clock stamps only: no stream operations inside the timed region
        hz.trace_begin(capacity=(args.steps + 1) * per_step_kernels * 4 + 64, events=False, stamps=True)
    graph = None
    if use_graph:
        # one step captured into a CUDA graph (the library's kernels, NCCL calls and
        # trace events become graph nodes); each timed step is one replay
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cs):
            if transport == "p2p":
                ctx.p2p_capture_begin()
            model.step(cs)
            if transport == "p2p":
                ctx.p2p_capture_end(cs)
        torch.cuda.synchronize()
        for _ in range(2):
            graph.replay()
        if transport == "p2p":
            ctx.p2p_replayed(2)
        torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0, e1 = ev[0], ev[-1]
    e0.record(stream)
    for k in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            model.step(stream)
        ev[k + 1].record(stream)
    torch.cuda.synchronize()
    per_step = sorted(ev[k].elapsed_time(ev[k + 1]) for k in range(args.steps))
    pct = {f"p{q}": max_over_ranks(per_step[min(len(per_step) - 1, int(round(q / 100 * (len(per_step) - 1))))], world)
           for q in (10, 50, 90)}
    if graph is not None and transport == "p2p":
        ctx.p2p_replayed(args.steps)
    barrier(world)
    hz.trace_end()
    clocks = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1)
    ms = max_over_ranks(ms, world)
    ms_per_step = ms / args.steps
    recs = hz.trace_read()
    # with a graph the trace holds one step's launches (events re-recorded by every replay)
    stages = summarize_trace(recs, 1 if graph is not None else args.steps)
    peak0, _ = measured_peaks()
    nvl = nvlink_probe(ctx, rank, world, stream) if transport == "p2p" else None
    nvl_uni = nvl["one_way_GBps"] if nvl else NVLINK_PEER_GBS
    nvl_bi = nvl["bidirectional_GBps"] if nvl else NVLINK_BIDIR_PROBE_GBS
    smodel = step_model(recs, 1 if graph is not None else args.steps, peak0, nvl_uni, nvl_bi) if recs else None
    if smodel:
        smodel["frac_of_model"] = smodel["model_ms"] / ms_per_step
        smodel["frac_of_model_bidir_probe"] = smodel["model_ms_bidir_probe"] / ms_per_step
    gpu_launches = sum(1 for r in recs if r["kind"] in KERNEL_KINDS) * (args.steps if graph is not None else 1)
    value = world * model.logical_bytes / (ms_per_step * 1e-3) / 1e9

    # roofline: the kernel kind with the largest share of device time
    peak, peak_src = measured_peaks()
    kern = {k: v for k, v in stages.items() if k.split("@")[0] in KERNEL_KINDS}
    roofline = None
    if kern:
        dom = max(kern, key=lambda k: kern[k]["share"])
        d = kern[dom]
        base = dom.split("@")[0]
        traffic = None
        nt = ncu_traffic()
        # N > 1: the per-element bytes of the same kernel captured in an N-GPU exchange
        # (tools/vw_profile.py under ncu, key "<kind>@N<n>"); N = 1: the world-1 capture
        tr = (nt.get(f"{dom}@N{world}") or nt.get(f"{base}@N{world}")) if world > 1 else (nt.get(dom) or nt.get(base))
        nvl_traffic = None
        if tr and tr.get("elems"):
            traffic = tr["dram_bytes"] / tr["elems"] * d["avg_elems"]
            if tr.get("nvlink_rx_bytes") is not None:
                nvl_traffic = {"rx": tr["nvlink_rx_bytes"] / tr["elems"] * d["avg_elems"],
                               "tx": tr["nvlink_tx_bytes"] / tr["elems"] * d["avg_elems"],
                               "source": tr.get("source")}
        roofline = {"bound": "hbm", "kernel": dom, "achieved": d["GBps"], "peak": peak, "unit": "GB/s",
                    "frac": d["GBps"] / peak, "traffic": traffic, "algorithmic_bytes_per_launch": d["avg_bytes"],
                    "avg_launch_ms": d["avg_ms"], "peak_source": peak_src}
        if nvl_traffic:
            roofline["nvlink_traffic"] = nvl_traffic   # ncu nvlrx/nvltx bytes per launch (protocol included)
        roofline.update(same_mix_probe(base, d["avg_elems"], d["avg_ms"]))
        rb = d.get("avg_remote_bytes", 0)
        if rb:
            # fused NVLink kernel: local HBM moves its own bytes plus the bytes the peers
            # read from it (served = remote, symmetric exchange); NVLink moves rb each way
            # at once, so the floor is the slower of (bytes + served) / HBM peak and rb /
            # the bidirectional peer-read peak measured in this run
            hbm_b = d["avg_bytes"] + rb
            t_hbm = hbm_b / (peak * 1e9)
            t_nvl = rb / (nvl_bi * 1e9)
            hbm_ach = hbm_b / (d["avg_ms"] * 1e-3) / 1e9
            roofline.update({"achieved": hbm_ach, "frac": hbm_ach / peak, "hbm_frac": hbm_ach / peak,
                             "served_bytes_per_launch": rb, "remote_bytes_per_launch": rb,
                             "nvlink_achieved": d["nvlink_GBps"],
                             "nvlink_peak_measured_bidirectional": nvl_bi, "nvlink_peak_measured_one_way": nvl_uni,
                             "nvlink_frac": d["nvlink_GBps"] / nvl_bi,
                             "nvlink_frac_of_one_way": d["nvlink_GBps"] / nvl_uni,
                             "nvlink_frac_of_900": d["nvlink_GBps"] / NVLINK_NOMINAL_GBS,
                             "floor_ms": max(t_hbm, t_nvl) * 1e3, "frac_of_floor": max(t_hbm, t_nvl) * 1e3 / d["avg_ms"]})
            if t_nvl > t_hbm:
                roofline.update({"bound": "nvlink", "achieved": d["nvlink_GBps"], "peak": nvl_bi,
                                 "frac": d["nvlink_GBps"] / nvl_bi,
                                 "peak_source": ("hz_nvlink_probe in this run: both GPUs of each pair pulling "
                                                 "at once, per direction" if nvl else "fallback bidirectional probe")})
    nccl = {k: v for k, v in stages.items() if k.startswith("nccl")}
    for v in nccl.values():
        v["frac_of_nvlink_one_way"] = (v["GBps"] or 0) / nvl_uni

    # cross-check of the per-kernel durations with CUDA events on the launching stream
    # (a separate eager pass: the events add stream operations between launches)
    if roofline is not None and not args.no_trace:
        hz.trace_begin(capacity=(args.steps + 1) * per_step_kernels * 4 + 64, events=True, stamps=False)
        barrier(world)
        for _ in range(args.steps):
            model.step(stream)
        torch.cuda.synchronize()
        hz.trace_end()
        ev = summarize_trace(hz.trace_read(), args.steps).get(roofline["kernel"])
        if ev:
            roofline["events_avg_launch_ms"] = ev["avg_ms"]
            roofline["events_achieved_hbm_GBps"] = ev["GBps"]
            roofline["timer"] = ("in-kernel %globaltimer stamps (CTA 0 entry -> last CTA exit) over the timed "
                                 "region; CUDA events on the launching stream in a second eager pass: events_*")

    # step tail, timed separately: AdamW on every optimizer shard and
    # the post-update all-gather of the updated weights into the primaries
    tail = None
    if not args.no_tail:
        tail = extra(step_tail, hz, ctx, torch, model, stream, world, args)

    # A10 cross-node step both ways (default qgZ reduce-scatter vs paper-literal
    # allreduce + select), on fp32 range_{L-1} shards
    a10 = None
    if world > 1 and not args.no_tail:
        a10 = extra(cross_node_step, hz, ctx, torch, model, stream, world, args)

    # flat ZeRO-3 baseline on the same logical bytes (context, not timed with the step)
    flat = None
    if world > 1 and not args.no_flat:
        flat = extra(flat_baseline, hz, ctx, torch, model, stream, world, args)

    # eight GPUs: the other 8-rank hierarchy of BASELINE configs 2-4 in the same command
    # ((2,4) and (2,2,2)), its own context and tensors, same timing discipline
    alt = None
    if world == 8 and not args.hierarchy and not args.no_alt:
        other = (2, 2, 2) if tuple(group) == (2, 4) else (2, 4)
        alt = extra(alt_hierarchy, hz, torch, args, other, rank, world, local, device)

    e2e = None
    if not args.no_e2e:
        e2e = extra(run_e2e, hz, ctx, torch, model, stream, world, args)

    cpu = None
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, group, model)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "ms_per_step_pct": pct, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded torch.Generator on device: params N(0,0.02^2), grads N(0,1e-6) with 1/1024 x64 outliers)",
        "config": {
            "workload": f"{args.config}: {len(model.tensors)} flat per-tensor buffers ({model.logical_bytes // 6:,} params), "
                        f"{'setting T' if (args.w, args.s) == (1, 1) else 'roles'} (w={args.w}, s={args.s}, gl=L), GA=1",
            "hierarchy": list(group), "block": args.block, "qwz_bits": args.qwz_bits, "qgz_bits": args.qgz_bits,
            "io": "bf16 params/grads in, bf16 gathered layers out, fp32 scales, fp32 gradient shard",
            "l2": "inputs larger than L2 (each step streams several GB); no flush",
            "parallelism": f"dp{world} hierarchical ({'x'.join(map(str, group))})",
            "transport": transport,
            "cuda_graph": graph is not None,
            "pipelined": args.pipelined,
        },
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": gpu_launches,
        "clocks": clocks,
        "stages": stages,
        "step_model": smodel,
        "nvlink_probe": nvl,
        "flat_zero3_baseline": flat,
        "step_tail": tail,
        "a10_cross_node_step": a10,
        "alt_hierarchy": alt,
        "topology": topology(world) if rank == 0 else None,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    # a CUDA graph that captured NCCL calls must be destroyed before its communicators
    # (ncclCommDestroy waits for the graph's resources otherwise)
    del graph
    torch.cuda.synchronize()
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def extra(fn, *a):
    """Secondary measurements never take the headline line down with them."""
    try:
        return fn(*a)
    except Exception as e:  # noqa: BLE001
        return {"error": f"{type(e).__name__}: {e}"[:300]}


def topology(world):
    """nvidia-smi topo -m row of GPU0 (link class to every peer) — a box whose GPUs talk
    over PCIe instead of NVLink would make the N > 1 numbers meaningless."""
    if world < 2:
        return None
    try:
        out = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True, timeout=20).stdout
        for line in out.splitlines():
            f = line.split()
            if f and f[0].endswith("GPU0"):
                return {"gpu0_row": f[1:1 + world]}
    except (OSError, subprocess.SubprocessError):
        pass
    return None


def alt_hierarchy(hz, torch, args, group, rank, world, local, device):
    """One more 8-rank hierarchy in the same process: its own hz context (P2P), tensors
    and captured step; K replays timed with CUDA events, max over ranks; per-level stages
    from the in-kernel stamps."""
    uid = hz.get_uid() if rank == 0 else None
    import torch.distributed as dist
    box = [uid]
    dist.broadcast_object_list(box, src=0)
    ctx = hz.Context(rank, world, box[0], group, local)
    try:
        ctx.enable_p2p(p2p_pool_bytes(args, group))
        model = Model(hz, ctx, torch, args.config, rank, world, args, device)
        stream = torch.cuda.current_stream()
        for _ in range(max(args.warmup, 3)):
            model.step(stream)
        torch.cuda.synchronize()
        hz.trace_begin(capacity=5 * len(model.tensors) * 4 + 64, events=False, stamps=True)
        cs = torch.cuda.Stream()
        cs.wait_stream(stream)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=cs):
            ctx.p2p_capture_begin()
            model.step(cs)
            ctx.p2p_capture_end(cs)
        torch.cuda.synchronize()
        graph.replay()
        ctx.p2p_replayed(1)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        ctx.p2p_replayed(args.steps)
        hz.trace_end()
        ms = max_over_ranks(e0.elapsed_time(e1), world) / args.steps
        stages = summarize_trace(hz.trace_read(), 1)
        del graph
        torch.cuda.synchronize()
        return {"hierarchy": list(group), "ms_per_step": ms, "unit": UNIT,
                "value": world * model.logical_bytes / (ms * 1e-3) / 1e9, "stages": stages}
    finally:
        ctx.close()


def flat_baseline(hz, ctx, torch, model, stream, world, args):
    """Plain NCCL bf16 all-gather (x2) + reduce-scatter on the world communicator over the
    same tensors: the ZeRO-3 rows of Tables VII/VIII."""
    bufs = []
    for t in model.tensors:
        Np = t["p"].padded_numel
        bufs.append((torch.empty(Np // world, dtype=torch.bfloat16, device=t["grad"].device), t["grad"],
                     torch.empty(Np // world, dtype=torch.bfloat16, device=t["grad"].device)))

    def step():
        for chunk, g, _ in bufs:
            ctx.flat_allgather(chunk, model.full[0][:g.numel()], stream=stream)
        for chunk, g, rs in reversed(bufs):
            ctx.flat_allgather(chunk, model.full[1][:g.numel()], stream=stream)
            ctx.flat_reduce_scatter(g, rs, stream=stream)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    barrier(world)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    n = max(1, min(args.steps, 5))
    e0.record(stream)
    for _ in range(n):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world) / n
    return {"ms_per_step": ms, "value": world * model.logical_bytes / (ms * 1e-3) / 1e9, "unit": UNIT,
            "what": "ncclAllGather x2 + ncclReduceScatter, bf16, world communicator"}


def step_tail(hz, ctx, torch, model, stream, world, args):
    """AdamW (fp32 master, m, v over range_L; the qgZ shard is the gradient) + post-update
    all-gather of every tensor, eager, CUDA events around K steps, max over ranks."""
    states = []
    for t in model.tensors:
        n = t["shard"].numel()
        states.append((torch.randn(n, device=t["shard"].device).mul_(0.02),
                       torch.zeros(n, device=t["shard"].device), torch.zeros(n, device=t["shard"].device)))
    hp = hz.adamw_params(1e-4, 0.9, 0.95, 1e-8, 0.1, 1)

    def one():
        for t, (th, m, v) in zip(model.tensors, states):
            ctx.adamw_step(t["p"], t["shard"], th, m, v, hp, t["primary"], stream=stream)

    one()
    torch.cuda.synchronize()
    barrier(world)
    n = max(1, min(args.steps, 5))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        one()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world) / n
    opt_elems = sum(t["shard"].numel() for t in model.tensors)
    del states
    torch.cuda.empty_cache()
    return {"ms_per_step": ms, "optimizer_elems_per_rank": opt_elems,
            "adamw_hbm_bytes_per_step": opt_elems * 30,
            "what": "AdamW on the fp32 optimizer shards + post-update all-gather of the bf16 weights into the "
                    "primaries (eager; not part of the headline metric)"}


def cross_node_step(hz, ctx, torch, model, stream, world, args):
    """A10, the once-per-step top-level reduction of every tensor's fp32 range_{L-1}
    shard, two ways: the default qgZ reduce-scatter of level L (quantized, R12) and
    the paper-literal fp32 allreduce over level L + select of range_L (P:361,
    hz_allreduce_select).  CUDA events around K steps, max over ranks."""
    L = ctx.levels
    lens = [t["p"].range(L - 1)[1] for t in model.tensors]
    src = torch.empty(max(lens), dtype=torch.float32, device=model.tensors[0]["grad"].device).normal_(0, 1e-3)
    gL = ctx.group[L - 1]

    def rs():
        for t, n in zip(model.tensors, lens):
            ctx.reduce_scatter_grads(t["p"], src[:n], t["shard"], model.bits, from_level=L, to_level=L, stream=stream)

    def ar():
        for t, n in zip(model.tensors, lens):
            ctx.allreduce_select(t["p"], src[:n], t["shard"], L, L, stream=stream)

    out = {}
    for name, fn in (("qgz_reduce_scatter", rs), ("allreduce_select", ar)):
        fn()
        torch.cuda.synchronize()
        barrier(world)
        n = max(1, min(args.steps, 5))
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(n):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        out[name + "_ms"] = max_over_ranks(e0.elapsed_time(e1), world) / n
    total = sum(lens)
    bits = model.bits[L - 1]
    out["peer_bytes_per_rank"] = {
        "qgz_reduce_scatter": int((gL - 1) * (total // gL) * (bits / 8 + 4 / args.block)),
        "allreduce_select": int((gL - 1) * total * 4)}
    out["what"] = ("level-L reduction of fp32 range_{L-1} shards of every tensor: qgZ int%d reduce-scatter "
                   "(default, R12) vs fp32 allreduce + select (P:361)" % bits)
    del src
    return out


def _host_registered(torch, numel, dtype):
    """Page-locked host tensor of exactly numel elements (cudaHostRegister on a plain
    CPU allocation; torch's pinned allocator would round each buffer up to a power
    of two)."""
    h = torch.empty(numel, dtype=dtype)
    rc = torch.cuda.cudart().cudaHostRegister(h.data_ptr(), h.numel() * h.element_size(), 0)
    if int(rc) != 0:
        raise RuntimeError(f"cudaHostRegister failed ({rc})")
    return h


def _host_unregister(torch, h):
    torch.cuda.cudart().cudaHostUnregister(h.data_ptr())


def _pcie_probe(torch, h, d, stream):
    """H2D alone, D2H alone and both at once on two streams: the copy floor of e2e."""
    nb = min(h.numel() * h.element_size(), d.numel() * d.element_size())
    hb, db = h.view(torch.uint8)[:nb], d.view(torch.uint8)[:nb]
    hb2 = hb.clone().pin_memory() if nb <= (1 << 30) else None
    out = {}
    s2 = torch.cuda.Stream()
    for name in ("h2d", "d2h", "both"):
        best = None
        for _ in range(3):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            with torch.cuda.stream(stream):
                if name in ("h2d", "both"):
                    db.copy_(hb, non_blocking=True)
            if name in ("d2h", "both"):
                s2.wait_event(e0)
                with torch.cuda.stream(s2):
                    (hb2 if (name == "both" and hb2 is not None) else hb).copy_(db, non_blocking=True)
                stream.wait_stream(s2)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            best = ms if best is None else min(best, ms)
        out[name + "_GBps"] = (2 if name == "both" else 1) * nb / (best * 1e-3) / 1e9
    out["probe_bytes"] = nb
    return out


def run_e2e(hz, ctx, torch, model, stream, world, args):
    """The same step end to end through the C-ABI with HOST buffers: hz_step_host
    (csrc/executor.cpp) uploads every tensor's primary and gradient from page-locked
    host memory, runs the gathers and the qgZ reduce-scatter, and downloads every fp32
    gradient shard, the copies on the library's two copy streams overlapping each
    other and the kernels.  Timed with CUDA events on the kernel stream (which waits
    for the last download), back-to-back steps, max over ranks.  The host shards are
    compared bitwise with the device-resident run's shards."""
    L = ctx.levels
    tens = model.tensors
    h_p = _host_registered(torch, sum(t["primary"].numel() for t in tens), torch.bfloat16)
    h_g = _host_registered(torch, sum(t["grad"].numel() for t in tens), torch.bfloat16)
    h_s = _host_registered(torch, sum(t["shard"].numel() for t in tens), torch.float32)
    free = torch.cuda.mem_get_info()[0]
    fresh = free > h_s.numel() * 4 + (4 << 30)
    io = []
    op = og = os_ = 0
    for t in tens:
        npr, ngr, nsh = t["primary"].numel(), t["grad"].numel(), t["shard"].numel()
        hp, hg, hs = h_p[op:op + npr], h_g[og:og + ngr], h_s[os_:os_ + nsh]
        op, og, os_ = op + npr, og + ngr, os_ + nsh
        hp.copy_(t["primary"])
        hg.copy_(t["grad"])
        io.append({"p": t["p"], "h_primary": hp, "d_primary": t["primary"], "h_grad": hg, "d_grad": t["grad"],
                   "sec_codes": t["sec_c"], "sec_scales": t["sec_s"],
                   "d_shard": torch.empty_like(t["shard"]) if fresh else t["shard"], "h_shard": hs})
    h2d = sum(t["primary"].numel() * 2 + t["grad"].numel() * 2 for t in tens)
    d2h = sum(t["shard"].numel() * 4 for t in tens)
    sargs = ctx.step_host_args(io, model.bits)

    def step():
        ctx.step_host(sargs, model.full, qwz_bits=args.qwz_bits, stream=stream)

    step()
    model.step(stream)        # device-resident step on the same inputs: reference shards in t["shard"]
    torch.cuda.synchronize()
    match = None
    if fresh:
        match = all(torch.equal(io[i]["h_shard"].view(torch.int32), t["shard"].cpu().view(torch.int32))
                    for i, t in enumerate(tens))
    barrier(world)
    n = max(1, min(args.steps, 5))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(n):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world) / n
    probe = _pcie_probe(torch, h_s, io[0]["d_shard"] if fresh else model.full[0], stream)
    floor_ms = max(h2d / (probe["h2d_GBps"] * 1e9), d2h / (probe["d2h_GBps"] * 1e9),
                   (h2d + d2h) / (probe["both_GBps"] * 1e9)) * 1e3
    for h in (h_p, h_g, h_s):
        _host_unregister(torch, h)
    return {"value": world * model.logical_bytes / (ms * 1e-3) / 1e9, "unit": UNIT, "ms_per_step": ms,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "api": "hz_step_host (C-ABI, host buffers; copies on two library streams overlapping the kernels)",
            "host_shards_equal_device_run": match,
            "pcie_probe": probe, "pcie_floor_ms": floor_ms, "frac_of_pcie_floor": floor_ms / ms}


# ------------------------------------------------------------------ CPU oracle
def _host_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"affinity_cores": len(os.sched_getaffinity(0)), "cpu_count": os.cpu_count(), "cpu_model": model}


def _oracle_layer(g, numel, seed, args):
    """Inputs of one tensor for all W simulated ranks, then the timed oracle step."""
    import ml_dtypes
    import numpy as np
    from oracle import collectives as col
    from oracle import partition as pm
    from paper_2501_04266_b200 import synth
    W = pm.world_of(g)
    L = len(g)
    B = args.block
    Np = pm.padded_numel(numel, g, B)
    full = np.zeros(Np, np.float32)
    full[:numel] = synth.params_like(numel, seed, block=B, specials=False)
    full = full.astype(ml_dtypes.bfloat16)
    prim = {}
    for r in range(W):
        off, ln = pm.range_at(r, g, Np, 1)
        prim[r] = full[off:off + ln]
    grads = {}
    for r in range(W):
        x = np.zeros(Np, np.float32)
        x[:numel] = synth.gradient_like(numel, seed + 1 + r, block=B, specials=False)
        grads[r] = x.astype(ml_dtypes.bfloat16)
    bpl = {l: args.qgz_bits for l in range(1, L + 1)}
    t0 = time.perf_counter()
    _, sec = col.allgather_forward(prim, g, Np, B, 1, 1, bits=args.qwz_bits)
    col.allgather_backward(sec, g, Np, B, 1, bits=args.qwz_bits)
    col.reduce_scatter(grads, g, Np, B, 1, L, bpl)
    return time.perf_counter() - t0, W * 6 * numel


def cpu_baseline(args, group, model):
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    from paper_2501_04266_b200 import synth
    numel = synth.layer_numel(synth.GPT_CONFIGS[args.config]["hidden"])
    secs, byts = 0.0, 0
    n = max(1, args.cpu_sample_layers)
    for i in range(n):
        s, b = _oracle_layer(group, numel, 31 + i, args)
        secs += s
        byts += b
    info = _host_info()
    # BASELINE config 1 as well: the flat 1M-element tensor over 8 simulated ranks (2,2,2)
    s1, b1 = _oracle_layer((2, 2, 2), 1 << 20, 11, args)
    # and SURVEY §8(d)'s CPU sample of config 2: one GPT-1.3B layer over the 8 simulated
    # ranks of the (2,4) hierarchy the config names (8 x 50.4 M elements)
    s2, b2 = _oracle_layer((2, 4), numel, 41, args)
    return {"value": byts / secs / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{n} tensors of {numel:,} params ({args.config} layer size), all {math.prod(group)} simulated "
                      f"rank(s) of hierarchy {list(group)}: fwd+bwd qwZ all-gather + qgZ reduce-scatter, NumPy "
                      f"single thread; {secs:.1f} s",
            "config1": {"value": b1 / s1 / 1e9, "unit": UNIT, "seconds": s1,
                        "sample": "BASELINE config 1: 1,048,576 elements, 8 simulated ranks as (2,2,2), same step"},
            "config2_layer_2x4": {"value": b2 / s2 / 1e9, "unit": UNIT, "seconds": s2,
                                  "sample": f"one {args.config} layer ({numel:,} params) over the 8 simulated ranks of "
                                            "hierarchy (2,4) (SURVEY 8(d)), same step, NumPy single thread"},
            **info}


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, on this arm's config / metric, each step
    a bounded sample (one tensor split over the N simulated ranks).  Rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_2501_04266_b200 import synth
    n = args.gpus
    group = hierarchy_of(args, n)
    numel = synth.layer_numel(synth.GPT_CONFIGS[args.config]["hidden"])
    numel = max(1, numel // n)
    for i in range(max(args.warmup, 3)):
        _oracle_layer(group, min(numel, 1 << 20), 100 + i, args)
    secs, byts = 0.0, 0
    for i in range(args.steps):
        s, b = _oracle_layer(group, numel, 200 + i, args)
        secs += s
        byts += b
    value = byts / secs / 1e9
    info = _host_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": secs / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded numpy)",
        "config": {"workload": f"{args.config}: per step one tensor of {numel:,} params per simulated rank "
                               f"(layer size / N), setting T, GA=1",
                   "hierarchy": list(group), "block": args.block, "qwz_bits": args.qwz_bits,
                   "qgz_bits": args.qgz_bits},
        "cpu_baseline": {"value": value, "unit": UNIT, "kind": "oracle", "cores": 1,
                         "sample": f"{args.steps} steps x {numel:,} params x {n} simulated ranks", **info},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    wd = float(os.environ.get("HZ_BENCH_WATCHDOG", "0"))
    if wd > 0:
        # debug aid: dump every thread's Python stack and exit if the run exceeds wd seconds
        import faulthandler
        faulthandler.dump_traceback_later(wd, exit=True)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_hz(args)


if __name__ == "__main__":
    main()
