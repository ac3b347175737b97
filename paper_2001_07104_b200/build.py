"""Build librfgpu.so in-tree with nvcc for sm_100a (no GPU needed to compile).

    python -m paper_2001_07104_b200.build [--force] [-j N]

Each csrc/*.cu is compiled to build/<name>.o with
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo`` and the objects are
linked into ``paper_2001_07104_b200/librfgpu.so`` (cudart linked statically).
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INC = os.path.join(os.path.dirname(HERE), "include")
# RF_PHASE_TIMING=1: profiling build (per-phase clock64 counters in the tree kernel,
# rf_debug_phase_cycles) into build_pt/ and librfgpu_pt.so; load it with RFGPU_LIB.
PHASE_TIMING = os.environ.get("RF_PHASE_TIMING", "0") == "1"
# RF_VARIANT=<tag> with RF_DEFS="-DX ...": an experimental variant (A/B timing) in
# build_<tag>/ and librfgpu_<tag>.so; never the product library.
VARIANT = os.environ.get("RF_VARIANT", "pt" if PHASE_TIMING else "")
BUILD = os.path.join(os.path.dirname(HERE), f"build_{VARIANT}" if VARIANT else "build")
LIB = os.path.join(HERE, f"librfgpu_{VARIANT}.so" if VARIANT else "librfgpu.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "-I" + INC, "--expt-relaxed-constexpr"] + (["-DRF_PHASE_TIMING"] if PHASE_TIMING else []) + \
    (os.environ.get("RF_DEFS", "").split() if VARIANT else [])


def _deps_mtime():
    files = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(INC, "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(src):
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    if os.path.exists(obj) and os.path.getmtime(obj) >= _deps_mtime():
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj


def build(force: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= _deps_mtime():
        return LIB
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for f in glob.glob(os.path.join(BUILD, "*.o")):
            os.remove(f)
    with cf.ThreadPoolExecutor(max_workers=jobs or min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(_compile, srcs))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-cudart", "static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    a = ap.parse_args()
    print(build(a.force, a.j))
    sys.exit(0)
