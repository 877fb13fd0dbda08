"""Build libhybridsort.so in-tree with nvcc for sm_100a (B200).

One shared library holds every kernel of the path plus the C ABI of
include/hs.h.  cudart is linked statically so the library does not depend on
which libcudart the host process (torch) has loaded; streams are driver
objects and are shared across runtimes.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libhybridsort.so")
SO_DEBUG = os.path.join(HERE, "libhybridsort_debug.so")  # -DHS_DEBUG: device invariant checks
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the CUDA 12.9 toolkit is required to build libhybridsort.so")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _inputs() -> list[str]:
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))


def needs_build() -> bool:
    return needs_build_at(SO)


def needs_build_at(so: str) -> bool:
    if not os.path.exists(so):
        return True
    t = os.path.getmtime(so)
    return any(os.path.getmtime(p) > t for p in _inputs())


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    """Build libhybridsort.so (or, debug=True, libhybridsort_debug.so with -DHS_DEBUG)."""
    so = SO_DEBUG if debug else SO
    if not force and not needs_build_at(so):
        return so
    cmd = [_nvcc(), *NVCC_FLAGS, *(["-DHS_DEBUG"] if debug else []), "-I", INCLUDE, "-I", CSRC, "-o", so + ".tmp",
           *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    os.replace(so + ".tmp", so)
    return so


if __name__ == "__main__":
    build(force=True, verbose=True)
