"""Build libchainserve_b200.so (hand-written sm_100a CUDA + the C-ABI) in-tree.

    python -m paper_2604_14993_b200.build [--verbose]

nvcc cross-compiles for sm_100a without a GPU.  -fmad=false keeps every
a*b+c of the reference as two IEEE operations (Python never fuses); the few
FMAs glibc's log1p uses are explicit __fma_rn calls.
"""

from __future__ import annotations

import argparse
import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "csrc")
LIB = os.path.join(PKG, "libchainserve_b200.so")
SOURCES = ["capi.cu", "exp_stream.cu", "jffc_sim.cu", "jffc_seg.cu", "stats.cu", "compose.cu", "dist.cu", "bounds.cu", "sim_ext.cu"]


def nccl_dirs():
    """NCCL 2.28 shipped with the torch wheels (nvidia-nccl-cu12)."""
    import importlib.util

    spec = importlib.util.find_spec("nvidia")
    for base in (list(spec.submodule_search_locations) if spec else []):
        inc, lib = os.path.join(base, "nccl", "include"), os.path.join(base, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("nccl.h not found (expected nvidia/nccl from the torch wheels)")


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the CUDA engine")


def flags(verbose: bool):
    f = [
        "-gencode", "arch=compute_100a,code=sm_100a",
        "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
        "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
        "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-I", nccl_dirs()[0],
    ]
    if verbose:
        f += ["-Xptxas", "-v"]
    return f


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    deps = [src] + [os.path.join(CSRC, h) for h in os.listdir(CSRC) if h.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "chainserve_b200.h"))
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    cc = nvcc()
    objs = []
    jobs = []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s.replace(".cu", ".o"))
        objs.append(obj)
        if force or _stale(obj, src):
            jobs.append([cc, *flags(verbose), "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4) or 1) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
            if verbose or res.returncode:
                sys.stderr.write(res.stdout + res.stderr)
            if res.returncode:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}")
    if force or jobs or not os.path.exists(LIB):
        nccl_lib = nccl_dirs()[1]
        link = [cc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB, *objs,
                "-lcudart", "-L", nccl_lib, "-l:libnccl.so.2", "-Xlinker", f"-rpath={nccl_lib}"]
        res = subprocess.run(link, capture_output=True, text=True)
        if res.returncode:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link of libchainserve_b200.so failed")
    return LIB


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--force", action="store_true")
    a = ap.parse_args()
    print(build(verbose=a.verbose, force=a.force))
