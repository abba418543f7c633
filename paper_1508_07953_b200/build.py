"""Build the in-tree CUDA library (sm_100a) that backs the package.

    python -m paper_1508_07953_b200.build

Produces paper_1508_07953_b200/_lib/libriann_b200.so with nvcc
(-gencode arch=compute_100a,code=sm_100a, -lineinfo, -fmad=false so no
float64 expression is contracted into an FMA).  The .so is git-ignored but
travels to the GPU box with the gpurun snapshot.
"""

from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB_DIR = os.path.join(PKG, "_lib")
LIB = os.environ.get("RIANN_LIB") or os.path.join(LIB_DIR, "libriann_b200.so")  # RIANN_LIB: development A/B builds
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the CUDA library")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(REPO, "include", "riann_b200.h")])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    tmp = LIB + ".tmp"
    cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-fmad=false",
           "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(REPO, "include"),
           "-o", tmp, os.path.join(CSRC, "riann_b200.cu"),
           "-Xlinker", "-rpath,/usr/local/cuda/lib64"]
    if os.environ.get("RIANN_HANG_DEBUG"):
        cmd.insert(1, "-DRIANN_HANG_DEBUG")
    for d in os.environ.get("RIANN_NVCC_DEFS", "").split():  # development A/B builds
        cmd.insert(1, d)
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{r.stdout}\n{r.stderr}")
    if verbose:
        print(r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
