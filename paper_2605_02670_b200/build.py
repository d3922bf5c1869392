"""Build libgrf.so in-tree for sm_100a with nvcc (no torch extension machinery).

    python -m paper_2605_02670_b200.build [--force] [--verbose]

Every .cu is compiled with ``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3``;
noise.cu additionally with ``--fmad=false`` (its bit-exact Box-Muller must not be
contracted into FMAs).  The C-ABI host code (grf_api.cpp) is compiled by nvcc's host
compiler.  The CUDA runtime is linked statically; NCCL is dlopen'ed at
grf_comm_init, so the library has no link-time NCCL dependency.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
OUTDIR = os.path.join(HERE, "lib")
BUILDDIR = os.path.join(OUTDIR, "obj")
LIB = os.path.join(OUTDIR, "libgrf.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
          "-Xptxas", "-v", "--expt-relaxed-constexpr"]
PER_FILE = {"noise.cu": ["--fmad=false"]}
SOURCES = ["noise.cu", "edge_setup.cu", "sweep.cu", "sweep_c0.cu", "sweep_r0k.cu", "sweep_r1k.cu", "sweep_r2k.cu", "sweep2_c16.cu", "sweep2_c32.cu",
           "sweep2_r16.cu", "sweep2_r32.cu", "sweep3_r32.cu", "sweep3_c32.cu", "pcg.cu", "pcg_warp.cu", "pcg_global.cu", "dist.cu", "refine.cu", "grf_api.cpp"]
HEADERS = ["grf_internal.h", "thomas.cuh", "sweep_impl.cuh", "sweep2_impl.cuh", "sweep3_impl.cuh"]


def nvcc() -> str:
    p = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(p):
        raise RuntimeError("nvcc not found: the CUDA toolkit is required to build libgrf.so")
    return p


def _stale(target, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src: str, force: bool, verbose: bool) -> tuple[str, str]:
    path = os.path.join(CSRC, src)
    obj = os.path.join(BUILDDIR, src + ".o")
    deps = [path, os.path.join(INCLUDE, "grf.h")] + [os.path.join(CSRC, h) for h in HEADERS]
    if not force and not _stale(obj, deps + [__file__]):
        return obj, ""
    cmd = [nvcc()] + ARCH + COMMON + PER_FILE.get(src, [])
    if src.endswith(".cpp"):
        cmd += ["-x", "cu"] if False else []
    cmd += ["-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return obj, (r.stdout + r.stderr) if verbose else ""


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILDDIR, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, force, verbose), SOURCES))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            print(log, file=sys.stderr)
    if force or _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-ldl", "-cudart", "static"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    a = ap.parse_args()
    print(build(a.force, a.verbose))
