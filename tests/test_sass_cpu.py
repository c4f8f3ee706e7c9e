"""Static checks of the built libhz.so (no GPU): what the parity tests rely on and what
the performance design assumes, read from the sm_100a SASS with cuobjdump.

* R10 / O9 (no FMA in the summation): the elementwise dequantize and the fp32 level
  reduce contain no FFMA — every product and sum rounds on its own, as in the oracle.
  (Kernels that divide — the quantize scale, AdamW — do contain FFMA, inside the
  IEEE-exact division / square-root sequences only.)
* No kernel touches local memory (register spills would turn the streaming kernels
  into local-memory traffic).
* The codec kernels and the dual kernel are sm_100a code.
"""

import os
import re
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2501_04266_b200", "libhz.so")
CUOBJDUMP = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"

pytestmark = pytest.mark.skipif(not (os.path.exists(LIB) and os.path.exists(CUOBJDUMP)),
                                reason="needs the built libhz.so and cuobjdump")


def _run(*args):
    return subprocess.run([CUOBJDUMP, *args, LIB], capture_output=True, text=True, timeout=600).stdout


@pytest.fixture(scope="module")
def sass():
    funcs = {}
    cur = None
    for line in _run("-sass").splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur is not None:
            funcs[cur].append(line)
    return funcs


@pytest.fixture(scope="module")
def resources():
    out = {}
    cur = None
    for line in _run("-res-usage").splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            cur = m.group(1)
        elif cur and "REG:" in line:
            out[cur] = {k: int(v) for k, v in re.findall(r"(REG|STACK|SHARED|LOCAL):(\d+)", line)}
    return out


def test_arch_is_sm100a():
    elf = _run("-lelf")
    assert "sm_100a" in elf


def _tile_kind(f, kind):
    return "k_tiles" in f and kind in f and "DualJob" not in f


def test_no_fma_in_dequantize_and_fp32_reduce(sass):
    names = [f for f in sass if "k_dequantize" in f or "k_reduce_f32" in f or _tile_kind(f, "GatherJob")
             or (_tile_kind(f, "ReduceJob") and re.search(r"ReduceJobILi[48]ELi\d+ELi[01]ELi0E", f))]
    assert names, "kernels not found in the SASS"
    bad = [f for f in names if any("FFMA" in l for l in sass[f])]
    assert not bad, f"FFMA in {bad[:3]}"


def test_no_local_memory(resources):
    assert resources
    bad = [f for f, r in resources.items() if r.get("LOCAL", 0) != 0]
    assert not bad, f"local memory in {bad[:3]}"


def test_dual_kernel_default_variant_fits_64_registers(resources):
    """The one-pass k_gather_quantize (the default below 32 gather tiles per warp) keeps
    the 64 registers of the kernels it merges (4 CTAs of 256 threads per SM)."""
    one_pass = [r for f, r in resources.items() if "k_gather_quantize" in f and "Li0ELb0ELi4E" in f]
    assert one_pass
    assert all(r["REG"] <= 64 and r.get("STACK", 0) == 0 for r in one_pass), one_pass


def test_tile_engine_kernels_are_tma_pipelines(sass, resources):
    """Every instantiation of the tile engine (k_tiles: quantize, round trip, gather,
    dual, reduce) moves its tiles with bulk copies both ways — cp.async.bulk global ->
    shared (SASS UBLKCP) completed on mbarriers (SYNCS.ARRIVE.TRANS64 / SYNCS.PHASECHK)
    and shared -> global bulk stores — and fits 4 CTAs per SM (<= 64 registers)."""
    names = [f for f in sass if "k_tiles" in f]
    assert len(names) >= 40, len(names)
    for f in names:
        text = "\n".join(sass[f])
        assert text.count("UBLKCP") >= 2, f"no bulk load + store in {f}"
        assert "SYNCS.ARRIVE.TRANS64" in text and "SYNCS.PHASECHK" in text, f"no mbarrier in {f}"
        assert resources[f]["REG"] <= 64, (f, resources[f])


def test_backward_triple_kernel_keeps_four_ctas_per_sm(sass, resources):
    """The backward triple kernel (gather || quantize || deferred fp32 reduce) keeps the
    dual kernel's 4 CTAs of 256 threads per SM (<= 64 registers; its three jobs are
    separate non-inlined functions) and touches no local memory."""
    names = [f for f in resources if "k_gather_quantize_reduce" in f]
    assert names, "k_gather_quantize_reduce not in the library"
    assert all(resources[f]["REG"] <= 64 and resources[f].get("LOCAL", 0) == 0 for f in names), \
        {f: resources[f] for f in names}
