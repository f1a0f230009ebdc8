"""Build liblk.so in-tree: the sm_100a kernels, the host runtime and the
native trace validator, linked into one shared library behind include/lk.h.

    python -m paper_2310_01212_b200.build

Objects are rebuilt only when a source or header is newer than the library.
"""
from __future__ import annotations

import os
import subprocess
import sys
import sysconfig
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIB = PKG / "liblk.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", str(ROOT / "include")]

SOURCES = ["lk_kernels.cu", "lk_host.cu", "lk_validate.cpp"]
# CPython fast path for trigger/wait (csrc/lk_pyfast.c); binds liblk.so's
# entry points at run time, so it links no CUDA library
PYFAST = PKG / ("_lkfast" + sysconfig.get_config_var("EXT_SUFFIX"))
HEADERS = ["lk_internal.h", "lk_protocol.cuh"]


def _stale() -> bool:
    if not LIB.exists():
        return True
    t = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES + HEADERS] + [ROOT / "include" / "lk.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build_pyfast(force: bool = False, verbose: bool = False) -> Path:
    src = CSRC / "lk_pyfast.c"
    if not force and PYFAST.exists() and PYFAST.stat().st_mtime > max(src.stat().st_mtime,
                                                                       Path(__file__).stat().st_mtime):
        return PYFAST
    tmp = PYFAST.with_suffix(".tmp")
    cmd = [os.environ.get("CC", "gcc"), "-O2", "-shared", "-fPIC", "-Wall", "-Werror",
           "-I", sysconfig.get_paths()["include"], str(src), "-o", str(tmp)]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, PYFAST)
    return PYFAST


def build(force: bool = False, verbose: bool = False) -> Path:
    build_pyfast(force, verbose)
    if not force and not _stale():
        return LIB
    objdir = PKG / "build"
    objdir.mkdir(exist_ok=True)
    objs = []
    for src in SOURCES:
        obj = objdir / (src + ".o")
        cmd = [NVCC, *ARCH, *COMMON, "-c", str(CSRC / src), "-o", str(obj)]
        if src.endswith(".cu"):
            cmd[1:1] = ["-Xptxas", "-v"] if verbose else []
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        objs.append(str(obj))
    tmp = LIB.with_suffix(".so.tmp")
    link = [NVCC, *ARCH, "-shared", "-o", str(tmp), *objs, "-lpthread"]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.run(link, check=True)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
