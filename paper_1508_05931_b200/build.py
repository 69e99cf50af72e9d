"""In-tree build of the native library (libgscan.so) for sm_100a.

nvcc cross-compiles without a GPU, so this runs in the CPU container and the
resulting .so travels to the GPU box with the repo snapshot.

Flags:
  -gencode arch=compute_100a,code=sm_100a   B200 only (tcgen05-era ISA)
  --fmad=false                               no silent a*b+c contraction anywhere:
                                             the reference's predicates and
                                             dist2 are un-fused
  -lineinfo                                  ncu source view
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "_lib"
LIB = LIBDIR / "libgscan.so"
ROOT = PKG.parent

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-std=c++17", "--fmad=false", "-lineinfo", "-Xcompiler", "-fPIC",
              "-Xptxas", "-O3"] + ARCH
CXX_FLAGS = ["-std=c++20", "-O2", "-fPIC", "-ffp-contract=off"]

CU_SOURCES = ["gscan.cu"]
CXX_SOURCES = ["datagen.cpp", "mt64_jump.cpp", "io.cpp"]


def _run(cmd: list[str]) -> None:
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)


def _stale(target: Path, deps: list[Path]) -> bool:
    if not target.exists():
        return True
    t = target.stat().st_mtime
    return any(d.stat().st_mtime > t for d in deps)


def build(force: bool = False, verbose_ptxas: bool = False) -> Path:
    LIBDIR.mkdir(exist_ok=True)
    headers = sorted(CSRC.glob("*.cuh")) + sorted(CSRC.glob("*.h")) + [ROOT / "include/gscan.h"]
    objs = []
    for src in CU_SOURCES:
        obj = LIBDIR / (Path(src).stem + ".cu.o")
        if force or _stale(obj, [CSRC / src] + headers):
            extra = ["-Xptxas", "-v"] if verbose_ptxas else []
            _run([NVCC, *NVCC_FLAGS, *extra, "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(obj)
    for src in CXX_SOURCES:
        obj = LIBDIR / (Path(src).stem + ".cpp.o")
        if force or _stale(obj, [CSRC / src] + headers):
            _run(["g++", *CXX_FLAGS, "-c", str(CSRC / src), "-o", str(obj)])
        objs.append(obj)
    if force or _stale(LIB, objs):
        _run([NVCC, *ARCH, "-shared", "-o", str(LIB), *map(str, objs), "-lcudart_static"])
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
