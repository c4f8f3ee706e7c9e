"""NCCL path parity (hz_init / hz_allgather_params / hz_reduce_scatter_grads) against
the oracle.  World 1 (hierarchy (1,)) runs in-process on one GPU; with >= 2 GPUs
the same worker runs under torchrun on 2, 4 and (if present) 8 GPUs, one process
per GPU, covering every hierarchy of that size (tests/mp_parity.py)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_world1_context():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests import mp_parity
    errors = mp_parity.run(0, 1, 0)
    assert not errors, "\n".join(errors)


@pytest.mark.multigpu
@pytest.mark.parametrize("n", [2, 4, 8])
def test_multi_gpu(n):
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + n),
           os.path.join(ROOT, "tests", "mp_parity.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]


@pytest.mark.multigpu
@pytest.mark.parametrize("n", [2, 4])
@pytest.mark.parametrize("tune", ["gqc=4", "gq=2,gqf=60", "nofuse=1"])
def test_multi_gpu_transport_variants(n, tune):
    """The alternative P2P kernel schedules selected with HZ_TUNE: the dual kernel's
    chunked interleave (gqc=4, the default for large layers only), its role split
    (gq=2), and the unpaired two-call path (nofuse=1)."""
    if not torch.cuda.is_available() or torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(29520 + n),
           os.path.join(ROOT, "tests", "mp_parity.py")]
    env = dict(os.environ, HZ_TUNE=tune)
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]


def test_world1_pair1_variant():
    """World 1 with HZ_TUNE pair1=1: hz_backward_step runs the previous layer's dequantize
    and this layer's qgZ round trip as one dual kernel (off by default); same results."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1",
           "--master-addr", "127.0.0.1", "--master-port", "29519", os.path.join(ROOT, "tests", "mp_parity.py")]
    env = dict(os.environ, HZ_TUNE="pair1=1")
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-4000:]


def test_world1_full_size_neox20b():
    """NeoX-20B layer (453 M parameters) through hz_allgather_params / hz_reduce_scatter_grads
    in the bench configuration, checked on sampled blocks."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_04266_b200 import hz, synth
    from tests import mp_parity
    numel = synth.layer_numel(synth.GPT_CONFIGS["neox20b"]["hidden"])
    errors = mp_parity.check_full_size(hz, 0, 1, (1,), hz.get_uid(), 0, numel, p2p=False)
    assert not errors, "\n".join(errors)
    torch.cuda.empty_cache()


def test_step_host_validation():
    """hz_step_host rejects bad arguments on the host, naming the tensor and field,
    and enqueues nothing."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2501_04266_b200 import hz
    ctx = hz.Context(0, 1, hz.get_uid(), (1,), 0)
    try:
        p = ctx.partition(4096, 256, 1, 1, 1)
        d = lambda n, dt: torch.empty(n, dtype=dt, device="cuda")
        t = {"p": p, "h_primary": torch.empty(4096, dtype=torch.bfloat16).pin_memory(),
             "d_primary": d(p.range(1)[1], torch.bfloat16),
             "h_grad": torch.empty(p.padded_numel, dtype=torch.bfloat16).pin_memory(),
             "d_grad": d(p.padded_numel, torch.bfloat16), "sec_codes": d(p.range(1)[1], torch.uint8),
             "sec_scales": d(p.range(1)[1] // 256, torch.float32), "d_shard": d(p.range(1)[1], torch.float32),
             "h_shard": None}
        full = [d(p.padded_numel, torch.bfloat16) for _ in range(2)]
        with pytest.raises(hz.HZError) as ei:
            ctx.step_host([t], full)
        assert ei.value.status == hz.ERR_INVALID and "t[0].h_shard" in str(ei.value)
        t["h_shard"] = torch.empty(p.range(1)[1], dtype=torch.float32).pin_memory()
        with pytest.raises(hz.HZError) as ei:
            ctx.step_host([t], full, qwz_bits=5)
        assert "qwz_bits" in str(ei.value)
        bad = dict(t, d_grad=t["d_grad"][1:])                      # misaligned device pointer
        with pytest.raises(hz.HZError) as ei:
            ctx.step_host([t, bad], full)
        assert "t[1].d_grad" in str(ei.value)
        ctx.step_host([t], full)                                   # valid call still works
        torch.cuda.synchronize()
    finally:
        ctx.close()
