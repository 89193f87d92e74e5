"""Build libcsrk_cuda.so in-tree for sm_100a.

``python -m paper_2203_05096_b200.build`` (or ``__graft_entry__.build()``)
compiles every CUDA / C++ source under ``csrc/`` with nvcc
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` and links
``paper_2203_05096_b200/lib/libcsrk_cuda.so``.  Objects are rebuilt only
when a source or header is newer than the library.  nvcc cross-compiles, so
this works on a machine without a GPU.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB_DIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIB_DIR, "libcsrk_cuda.so")

CUDA_SOURCES = ["abi.cu", "spmv.cu", "listing.cu", "construct.cu", "cg.cu", "sort.cu", "graph.cu", "rcm.cu", "coarsen.cu", "bandk_dev.cu", "mg.cu"]
CXX_SOURCES = ["bandk.cpp", "mmio.cpp"]
HEADERS = [os.path.join(CSRC, "internal.h"), os.path.join(REPO, "include", "csrk.h")]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-Wall", "--expt-relaxed-constexpr"]
CXX_FLAGS = ["-O3", "-std=c++17", "-fPIC", "-Wall", "-fopenmp"]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the CUDA toolkit is required to build")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    return res


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile (if needed) and return the path of libcsrk_cuda.so."""
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIB_DIR, exist_ok=True)
    nvcc = _nvcc()
    jobs = []
    objs = []
    for src in CUDA_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + HEADERS):
            jobs.append([nvcc, *ARCH, *NVCC_FLAGS, "-c", path, "-o", obj])
    for src in CXX_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(BUILD, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + HEADERS):
            jobs.append(["g++", *CXX_FLAGS, "-c", path, "-o", obj])
    with ThreadPoolExecutor(max_workers=max(1, len(jobs))) as pool:
        list(pool.map(lambda c: _run(c, verbose), jobs))
    if force or jobs or _stale(LIB, objs):
        _run([nvcc, *ARCH, "-shared", "-o", LIB, *objs, "-Xcompiler", "-fopenmp",
              "-lgomp", "-ldl"], verbose)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
