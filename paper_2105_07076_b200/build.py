"""Build the sm_100a C-ABI library in-tree: paper_2105_07076_b200/libidkit_b200.so.

nvcc cross-compiles for B200 without a GPU.  Every .cu under csrc/ is compiled
with -gencode arch=compute_100a,code=sm_100a -lineinfo and linked into one
shared library exporting the symbols declared in include/idkit_b200.h.
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libidkit_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I" + os.path.join(ROOT, "include")]


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def headers():
    out = [os.path.join(ROOT, "include", "idkit_b200.h")]
    out += [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    return out


def up_to_date(target, deps):
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def build(verbose: bool = False, force: bool = False, trace: bool = False) -> str:
    """trace=True: a separate debug library (libidkit_b200_trace.so) whose
    resident CPQR records per-step phase marks for tools/trace_cpqr.py
    (-DIDK_CPQR_TRACE; the product library carries no trace code)."""
    objdir = os.path.join(PKG, "build_trace" if trace else "build")
    lib = os.path.join(PKG, "libidkit_b200_trace.so") if trace else LIB
    flags = FLAGS + (["-DIDK_CPQR_TRACE"] if trace else [])
    os.makedirs(objdir, exist_ok=True)
    objs, jobs = [], []
    hdrs = headers()
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if not force and up_to_date(obj, [src] + hdrs):
            continue
        cmd = [NVCC] + ARCH + flags + ["-c", src, "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        jobs.append(cmd)
    # translation units compile independently: one nvcc per core
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as pool:
        list(pool.map(lambda c: subprocess.run(c, check=True), jobs))
    if force or not up_to_date(lib, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-o", lib] + objs + ["-lcudart_static", "-lrt", "-ldl", "-lpthread"]
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv, trace="--trace" in sys.argv))
