"""The TMA tile engine (csrc/tiles.cuh, k_tiles.cu; HZ_TUNE tma=1, off by default because
it measured slower — profiles/tma_r02.md) stays parity-tested: the codec kernels'
bitwise tests and the multi-rank virtual-world checks rerun in a subprocess with the
engine on, so every quantize / round trip / gather / dual / reduce the engine takes is
compared with the oracle bit for bit."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tile_engine_parity():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, HZ_TUNE="tma=1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_codec.py"),
           os.path.join(ROOT, "tests", "test_gpu_vworld.py") + "::test_vworld_hierarchy",
           os.path.join(ROOT, "tests", "test_gpu_collectives.py") + "::test_world1_context"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]


def test_bulk_store_gather_parity():
    """The non-default store modes stay parity-tested (profiles/tma_r02.md): HZ_TUNE dgb=1 (the
    dual and triple kernels store the gathered layer by TMA bulk stores from dynamic shared
    memory), fbd=1 (the world-1 dequantize by bulk stores) and fbb=0 (the bf16 round trip by
    st.global).  The codec tests, the paired virtual-world schedule (dual + triple kernels)
    and the hierarchy checks rerun with them, bitwise against the oracle."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, HZ_TUNE="dgb=1,fbd=1,fbb=0")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_codec.py"),
           os.path.join(ROOT, "tests", "test_gpu_vworld.py") + "::test_vworld_hierarchy",
           os.path.join(ROOT, "tests", "test_gpu_vworld.py") + "::test_vworld_trace_shows_multi_rank_kernels",
           os.path.join(ROOT, "tests", "test_gpu_vworld.py") + "::test_deferred_last_hop_completes_on_flush"]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=1200, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-4000:] + p.stderr[-2000:]
