"""Build libhz.so in-tree: nvcc for sm_100a, NCCL from the torch-bundled wheel.

    python -m paper_2501_04266_b200.build [--force] [-v]

Every translation unit under csrc/ is compiled to an object in csrc/_obj/ (in
parallel) and linked into ``paper_2501_04266_b200/libhz.so``.  Exactness flags:
--fmad=false (no FMA contraction: the sums and products must round like the
oracle's), -ftz=false, -prec-div=true, -prec-sqrt=true.  The CUDA runtime is
linked statically; NCCL is the venv's libnccl.so.2 (the 2.28.9 copy torch loads,
so one process never holds two NCCLs), found through an rpath.
"""

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
# HZ_BUILD_VARIANT=name HZ_NVCC_DEFS="-DX=Y ...": an experimental build into
# libhz_<name>.so (objects in csrc/_obj_<name>), loaded with HZ_LIB=libhz_<name>.so
_VAR = os.environ.get("HZ_BUILD_VARIANT", "")
OBJ = os.path.join(CSRC, "_obj" + ("_" + _VAR if _VAR else ""))
LIB = os.path.join(PKG, "libhz" + ("_" + _VAR if _VAR else "") + ".so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    cands = []
    if spec and spec.submodule_search_locations:
        for loc in spec.submodule_search_locations:
            cands.append(os.path.join(loc, "nccl"))
    for c in cands:
        if os.path.exists(os.path.join(c, "include", "nccl.h")):
            return c
    raise RuntimeError("NCCL headers not found under the nvidia wheel namespace")


def _flags():
    nd = nccl_dir()
    return [
        *ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-ftz=false", "-prec-div=true",
        "-prec-sqrt=true", "-Xcompiler", "-fPIC,-O2,-Wall,-fvisibility=hidden", "-I", os.path.join(ROOT, "include"),
        "-I", os.path.join(nd, "include"), *os.environ.get("HZ_NVCC_DEFS", "").split(),
    ], nd


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _deps():
    return sources() + glob.glob(os.path.join(CSRC, "*.h")) + [os.path.join(ROOT, "include", "hz.h"),
                                                              os.path.abspath(__file__)]


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    flags, nd = _flags()
    jobs = []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src) + ".o")
        cmd = [NVCC, *flags, "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC, *flags, "-x", "cu", "-c", src, "-o", obj]
        jobs.append((src, obj, cmd))

    def run(job):
        src, obj, cmd = job
        hdr_t = max(os.path.getmtime(d) for d in _deps() if d.endswith(".h") or d.endswith(".py"))
        if not force and os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_t):
            return src, 0, ""
        p = subprocess.run(cmd, capture_output=True, text=True)
        return src, p.returncode, p.stdout + p.stderr

    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        results = list(ex.map(run, jobs))
    for src, rc, out in results:
        if verbose and out:
            print(out, file=sys.stderr)
        if rc:
            raise RuntimeError(f"nvcc failed on {os.path.basename(src)}:\n{out}")
    lib_dir = os.path.join(nd, "lib")
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB + ".tmp",
            *[j[1] for j in jobs], "-L", lib_dir, "-l:libnccl.so.2",
            "-Xlinker", f"-rpath,{lib_dir}", "-Xlinker", "--no-undefined", "-lpthread", "-ldl", "-lrt"]
    p = subprocess.run(link, capture_output=True, text=True)
    if p.returncode:
        raise RuntimeError("link failed:\n" + p.stdout + p.stderr)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    lib = build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(lib)
