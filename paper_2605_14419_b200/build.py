"""In-tree build of the C-ABI library ``libzsort_b200.so`` for sm_100a.

The library is plain CUDA C++ behind ``extern "C"`` entry points
(include/zsort_b200.h); Python binds it with ctypes, so no torch extension
ABI is involved.  ``python -m paper_2605_14419_b200.build`` rebuilds it.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libzsort_b200.so")
SOURCES = [os.path.join(CSRC, "zsort_b200.cu")]
HEADERS = [os.path.join(CSRC, "common.cuh"), os.path.join(CSRC, "sort_kernels.cuh"),
           os.path.join(CSRC, "dist_kernels.cuh"), os.path.join(CSRC, "gen_kernels.cuh"),
           os.path.join(REPO, "include", "zsort_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    extra = ["-DZSB_PHASE_PROFILE"] if os.environ.get("ZSB_PHASE_PROFILE") == "1" else []
    extra += os.environ.get("ZSB_NVCC_EXTRA", "").split()
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(REPO, "include"), "-o", LIB + ".tmp", *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
