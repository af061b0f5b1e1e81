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
SOURCES = ["interp_kernels.cu", "tile_kernels.cu", "conv_tc.cu", "vinet_kernels.cu", "refine_kernels.cu", "encode_kernels.cu", "deflate_kernels.cu", "ts_mux.cpp", "diag_kernels.cu", "literal_kernels.cu", "api.cu"]
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
    """Compile every translation unit to an object in parallel, then link the .so."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    extra = os.environ.get("FVV_NVCC_EXTRA", "").split()  # tuning sweeps only (e.g. -DFVV_MINB_MASK=8)
    objdir = PKG / "_obj"
    objdir.mkdir(exist_ok=True)
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def one(src: str) -> Path:
        obj = objdir / (Path(src).stem + ".o")
        if src.endswith(".cpp"):  # host-only translation unit
            cmd = [shutil.which("g++") or "g++", "-O2", "-std=c++17", "-fPIC", "-c", "-o", str(obj), str(CSRC / src)]
        else:
            cmd = [nvcc(), *compile_flags, *extra, "-c", "-o", str(obj), str(CSRC / src)]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(one, SOURCES))
    cmd = [nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-Xcompiler", "-fPIC",
           "-o", str(LIB) + ".tmp", *map(str, objs)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(str(LIB) + ".tmp", LIB)
    return LIB


if __name__ == "__main__":  # pragma: no cover
    print(build(force=True, verbose=True))
