"""Build liblrq.so (the CUDA engine + C ABI) in-tree for sm_100a.

    python -m paper_2604_26423_b200.build        # or __graft_entry__.build()

The shared library is written to paper_2604_26423_b200/_lib/liblrq.so so it
travels with the repository snapshot to the GPU box (it is git-ignored).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "_lib")
LIB = os.path.join(LIBDIR, "liblrq.so")
SOURCES = ["lrq_engine.cu"]
HEADERS = sorted(f for f in os.listdir(CSRC) if f.endswith((".cuh", ".h")))

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-DLRQ_EXPLICIT_FFMA2", "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "--expt-relaxed-constexpr"]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found; the LR-QAOA engine needs the CUDA toolkit to build")


def _stale(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "lrq.h"))
    return any(os.path.exists(d) and os.path.getmtime(d) > t for d in deps)


LIB_CHECKED = os.path.join(LIBDIR, "liblrq_checked.so")


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """checked=True: the bounds-checked build (-DLRQ_CHECKED, device asserts;
    load it with LRQ_LIB=<path>).  The product build is the default."""
    lib = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib):
        return lib
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = lib + ".tmp"
    cmd = [_nvcc(), *ARCH, *FLAGS, *(["-DLRQ_CHECKED"] if checked else []), "-o", tmp,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, checked="--checked" in sys.argv))
