"""Build the native library in-tree:  python -m paper_2402_02273_b200.build

nvcc cross-compiles for sm_100a (B200) without a GPU.  Output:
paper_2402_02273_b200/libgliosim_b200.so (git-ignored; travels to the GPU box with
the repo snapshot).  Flags that matter for parity: -fmad=false (no FMA contraction in
device code) and -ffp-contract=off for the host side (seed_initial, select_params).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libgliosim_b200.so")
SOURCES = ["gs_kernels.cu", "gs_solve.cu", "gs_cluster.cu", "gs_vtkfmt.cu", "gs_capi.cu", "gs_io.cpp"]
HEADERS = ["gs_device.cuh", "gs_kernels.cuh", "gs_tma.cuh", "gs_io.hpp", "gs_vtkfmt.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-O2",
    "-Xptxas", "-v",
    "-shared",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "gliosim_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale() and "GS_LIB_OUT" not in os.environ:
        return LIB
    # GS_NVCC_EXTRA (e.g. "-DGS_TILE8") and GS_LIB_OUT build A/B variants of the library
    extra = os.environ.get("GS_NVCC_EXTRA", "").split()
    out = os.environ.get("GS_LIB_OUT", LIB)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-o", out,
           *[os.path.join(CSRC, s) for s in SOURCES]]
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(CSRC, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed ({res.returncode}); see {log}")
    if verbose:
        sys.stderr.write(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
