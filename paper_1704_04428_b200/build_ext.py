"""In-tree build of libconvlab_b200.so (sm_100a only).

    python -m paper_1704_04428_b200.build_ext [--force]

nvcc -gencode arch=compute_100a,code=sm_100a (NOT -arch=sm_100a, which also embeds
compute_100 PTX that ptxas rejects for tcgen05).  cudart is linked statically so the
library loads on a CPU-only host (its entry points then return CL_ENODEVICE).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "_build"
LIB = PKG / "libconvlab_b200.so"

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
                  "-I", str(ROOT / "include"), "-I", str(CSRC)]
CU_SOURCES = ["prepass.cu", "tc_conv.cu", "tc_direct.cu", "direct.cu", "api.cu"]
CXX_SOURCES = ["facade.cpp"]
HEADERS = ["ptx.cuh", "tc_conv.cuh", "split_tile.cuh", "internal.hpp"]


def _stale(obj: Path, deps) -> bool:
    if not obj.exists():
        return True
    t = obj.stat().st_mtime
    return any(Path(d).stat().st_mtime > t for d in deps if Path(d).exists())


def build(force: bool = False, verbose: bool = False) -> Path:
    BUILD.mkdir(exist_ok=True)
    hdrs = [CSRC / h for h in HEADERS] + list((ROOT / "include").glob("*.h*"))
    objs = []
    for src in CU_SOURCES:
        obj = BUILD / (Path(src).stem + ".o")
        if force or _stale(obj, [CSRC / src, *hdrs]):
            cmd = [NVCC, *NVFLAGS, "-c", str(CSRC / src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
        objs.append(obj)
    for src in CXX_SOURCES:
        if not (CSRC / src).exists():
            continue
        obj = BUILD / (Path(src).stem + ".o")
        if force or _stale(obj, [CSRC / src, *hdrs]):
            cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-fvisibility=hidden", "-I", str(ROOT / "include"),
                   "-c", str(CSRC / src), "-o", str(obj)]
            if verbose:
                print(" ".join(cmd))
            subprocess.run(cmd, check=True)
        objs.append(obj)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", str(LIB), *map(str, objs), "-ldl", "-lrt",
               "-lpthread"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
