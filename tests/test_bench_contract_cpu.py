"""bench.py's reference arm runs on CPU (it times the oracle): its JSON line carries the
contract keys (metric / value / unit / impl / e2e with zero copied bytes / cpu_baseline)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    p = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["metric"].startswith("param all-gather + grad reduce-scatter GB/s")
    assert d["unit"] == "GB/s" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] >= 3
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert "workload" in d["config"]


def test_reference_arm_under_torchrun_prints_once():
    """N > 1 (torchrun, gloo on CPU here): rank 0 alone runs the reference arm and prints
    one line; the other ranks exit 0 without work."""
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29791", "bench.py", "--impl", "reference",
                        "--gpus", "2", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0


def test_step_model_sums_launch_rooflines():
    """bench.step_model: per launch max(HBM bytes / HBM peak, peer bytes / NVLink peak),
    NCCL calls on the link only, summed and divided by the steps the trace covers."""
    sys.path.insert(0, ROOT)
    import bench
    recs = [{"kind": "quantize", "bytes": 6e9, "remote_bytes": 0},             # 1 ms at 6000 GB/s
            {"kind": "gather_dequantize", "bytes": 3e9, "remote_bytes": 1.5e9},  # max(0.5, 2.0) ms at 750
            {"kind": "nccl_allgather", "bytes": 0.75e9, "remote_bytes": 0}]      # 1 ms on the link
    m = bench.step_model(recs, 2, 6000.0, nvl_peak=750.0, nvl_bidir=500.0)
    assert abs(m["model_ms"] - (1.0 + 2.0 + 1.0) / 2) < 1e-9
    assert abs(m["model_ms_bidir_probe"] - (1.0 + 3.0 + 1.5) / 2) < 1e-9
