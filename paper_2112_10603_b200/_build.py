"""Build the C-ABI shared library (libfvv_b200.so) in-tree with nvcc for sm_100a.

No JIT cache, no torch extension: the .so sits next to this file so it
travels to the GPU box with the repo snapshot and is what the tests, smoke()
and bench.py load (paper_2112_10603_b200/_lib.py).
"""
from __future__ import annotations

import os
import shutil
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIB = PKG / "libfvv_b200.so"
SOURCES = ["interp_kernels.cu", "tile_kernels.cu", "conv_tc.cu", "vinet_kernels.cu", "api.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "--fmad=false",            # the reference never contracts a*b+c
    "-Xcompiler", "-fPIC", "-shared",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: the B200 path has no fallback")


def stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.h")) + [PKG.parent / "include" / "fvv_b200.h"]
    return any(d.stat().st_mtime > t for d in deps if d.exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return LIB
    extra = os.environ.get("FVV_NVCC_EXTRA", "").split()  # tuning sweeps only (e.g. -DFVV_MINB_MASK=8)
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-o", str(LIB) + ".tmp", *[str(CSRC / s) for s in SOURCES]]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":  # pragma: no cover
    print(build(force=True, verbose=True))
