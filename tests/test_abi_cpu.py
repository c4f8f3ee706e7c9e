"""CPU-side checks of the C-ABI boundary (no GPU): libhz.so loads, exports exactly
the entry points include/hz.h declares, hz_partition_ex is bit-identical to the
oracle's O1-O3 map, and host validation rejects bad arguments naming the field."""

import ctypes
import os
import re
import subprocess

import pytest

from oracle import partition as pm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hz.h")


@pytest.fixture(scope="module")
def hz():
    from paper_2501_04266_b200 import build
    build.build()
    from paper_2501_04266_b200 import hz as mod
    return mod


def _declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^HZ_API [^(]*?\b(hz_\w+)\(", src, flags=re.M)))


def test_exports_match_header(hz):
    declared = _declared()
    assert len(declared) >= 19
    assert sorted(hz.exported_symbols()) == declared
    lib = hz.lib_handle()
    for name in declared:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", hz.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if " T " in l)
    assert exported == declared                   # nothing else leaks out of the .so
    assert "sm_100a" in hz.version()


def test_sm100a_code_only(hz):
    out = subprocess.run(["cuobjdump", "--list-elf", hz.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


HIERS = [(1,), (2,), (2, 2), (2, 4), (4, 2), (2, 2, 2), (8,), (3, 2), (2, 2, 2, 2)]


@pytest.mark.parametrize("g", HIERS)
def test_partition_parity_with_oracle(hz, g):
    W = pm.world_of(g)
    L = len(g)
    for numel in (0, 1, 1000, 50_358_272, 453_064_704):
        for block in (32, 256, 2048):
            Np = pm.padded_numel(numel, g, block)
            for r in range(W):
                for w, s, gl in ((1, 1, L), (L, min(2, L), L), (0, 0, 0), (1, L, L)):
                    p = hz.partition_ex(r, g, numel, block, w, s, gl)
                    assert p.padded_numel == Np
                    off, ln = pm.ranges(r, g, Np)
                    assert list(p.off[:L + 1]) == off
                    assert list(p.len[:L + 1]) == ln
                    assert list(p.digit[:L]) == pm.digits(r, g)
                    assert (p.w, p.s, p.gl, p.world, p.rank) == (w, s, gl, W, r)


def test_partition_validation(hz):
    bad = [
        (dict(rank=0, group=(2, 2), numel=10, block=100), "block"),
        (dict(rank=4, group=(2, 2), numel=10, block=256), "rank"),
        (dict(rank=0, group=(2, 0), numel=10, block=256), "group"),
        (dict(rank=0, group=(2, 2), numel=-1, block=256), "numel"),
        (dict(rank=0, group=(2, 2), numel=10, block=256, w=3), "w"),
        (dict(rank=0, group=(2, 2), numel=10, block=256, s=-1), "s"),
        (dict(rank=0, group=(2, 2, 2, 2, 2), numel=10, block=256), "levels"),
    ]
    for kw, field in bad:
        with pytest.raises(hz.HZError) as ei:
            hz.partition_ex(**kw)
        assert ei.value.status == hz.ERR_INVALID
        assert str(ei.value).split(": ", 1)[1].startswith(field), (kw, str(ei.value))


def test_collective_validation_without_context(hz):
    lib = hz.lib_handle()
    p = hz.partition_ex(0, (2, 2), 1000)
    # no context: rejected on the host, message names the field
    assert lib.hz_allreduce_select(None, ctypes.byref(p), None, 1, 2, None, None) == hz.ERR_INVALID
    assert lib.hz_last_error().startswith(b"ctx")
    assert lib.hz_set_sm_budget(-1) == hz.ERR_INVALID
    assert lib.hz_set_sm_budget(0) == hz.OK
    bits = (ctypes.c_int * 2)(4, 4)
    assert lib.hz_step_host(None, 1, None, hz.BF16, 8, bits, None, None, hz.BF16, None) == hz.ERR_INVALID
    assert lib.hz_last_error().startswith(b"ctx")
    # the paired-layer entry points validate like the calls they pair
    assert lib.hz_allgather_params_next(None, ctypes.byref(p), None, hz.BF16, 8, None, None, None, hz.BF16, None,
                                        None, None, None, None) == hz.ERR_INVALID
    assert lib.hz_last_error().startswith(b"ctx")
    assert lib.hz_backward_step(None, ctypes.byref(p), None, hz.BF16, 1, 2, bits, None, 0, None, None, None, 8, None,
                                hz.BF16, None) == hz.ERR_INVALID
    assert lib.hz_last_error().startswith(b"ctx")


def test_codec_validation_without_gpu(hz):
    lib = hz.lib_handle()
    # rejected on the host before any CUDA call
    assert lib.hz_quantize(None, hz.BF16, 256, 3, 256, None, None, None) == hz.ERR_INVALID
    assert b"bits" in lib.hz_last_error()
    assert lib.hz_quantize(None, hz.BF16, 300, 8, 256, None, None, None) == hz.ERR_INVALID
    assert b"n:" in lib.hz_last_error()
    assert lib.hz_quantize(None, hz.BF16, 256, 8, 256, None, None, None) == hz.ERR_INVALID
    assert b"x:" in lib.hz_last_error()
    assert lib.hz_quantize(8, hz.BF16, 256, 8, 256, 16, 16, None) == hz.ERR_INVALID   # misaligned x
    assert lib.hz_dequantize(None, None, 256, 8, 256, None, 7, None) == hz.ERR_INVALID
    assert b"out_dt" in lib.hz_last_error()
    assert lib.hz_quantize(None, hz.BF16, 0, 8, 256, None, None, None) == hz.OK       # n == 0: no-op
    arr = (ctypes.c_void_p * 1)(None)
    assert lib.hz_reduce_chunks(0, arr, arr, 256, 4, 256, 0, None, None, None, 0, None) == hz.ERR_INVALID
    assert lib.hz_reduce_chunks(1, arr, arr, 256, 4, 256, 3, None, None, None, 0, None) == hz.ERR_INVALID
    assert b"bits_out" in lib.hz_last_error()
    assert lib.hz_init(None, 0, 1, None, 1, None, 0, 0) == hz.ERR_INVALID
    assert lib.hz_finalize(None) == hz.OK
    assert lib.hz_trace_begin(0, 3) == hz.ERR_INVALID
    assert lib.hz_trace_begin(16, 0) == hz.ERR_INVALID


def test_binding_fails_loudly_without_the_library(tmp_path):
    """No CPU fallback: the binding raises ImportError when libhz.so is missing."""
    import shutil
    import subprocess
    import sys
    pkg = tmp_path / "paper_2501_04266_b200"
    pkg.mkdir()
    src = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2501_04266_b200")
    for f in ("__init__.py", "hz.py"):
        shutil.copy(os.path.join(src, f), pkg / f)
    code = ("import sys\n"
            "try:\n"
            "    from paper_2501_04266_b200 import hz\n"
            "except ImportError as e:\n"
            "    print('ImportError', e); sys.exit(0)\n"
            "sys.exit(1)\n")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=tmp_path, timeout=120,
                       env=dict(os.environ, PYTHONPATH=str(tmp_path)))
    assert p.returncode == 0, p.stdout + p.stderr
    assert "no CPU fallback" in p.stdout


def test_product_package_never_touches_the_oracle():
    """The oracle is test infrastructure: nothing in the product package (binding,
    build, synthetic inputs, CUDA / C++ sources) imports or includes it."""
    root = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2501_04266_b200")
    pat = re.compile(r"^\s*(import\s+oracle|from\s+oracle|#\s*include\s+\S*oracle)", re.M)
    for dirpath, _, files in os.walk(root):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                with open(os.path.join(dirpath, f)) as fh:
                    assert not pat.search(fh.read()), os.path.join(dirpath, f)
