"""In-tree build of the native library `libsplbm_b200.so` (sm_100a kernels + C++ host runtime).

Everything is compiled by nvcc for `-gencode arch=compute_100a,code=sm_100a`; the shared object
lands next to this file so it travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsplbm_b200.so")
BUILD = os.path.join(ROOT, "build", "native")
# the tolerance-mode build: same sources with SPLBM_FMA=1 (contracted multiply-adds)
FMA_LIB = os.path.join(PKG, "libsplbm_b200_fma.so")
FMA_BUILD = os.path.join(ROOT, "build", "native_fma")
SOURCES = ["kernels.cu", "engine.cpp", "tiling.cpp", "tiling_gpu.cu", "geometry.cpp", "geometry_gpu.cu", "nccl_api.cpp",
           "mrt.cpp"]
HEADERS = ["kernels.h", "lattice.cuh", "common.h", "tiling.h", "tiling_gpu.h", "nccl_api.h", "mrt.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr",
                     "-Xcompiler", "-fPIC,-O3,-Wall", "-I", CSRC, "-I", os.path.join(ROOT, "include")]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _newer(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps)


def build(force: bool = False, verbose: bool = False, defines: list[str] | None = None,
          lib: str | None = None, build_dir: str | None = None) -> str:
    """Compile the sources; `defines`/`lib`/`build_dir` build an experiment variant elsewhere."""
    out_lib = lib or LIB
    bdir = build_dir or BUILD
    os.makedirs(bdir, exist_ok=True)
    extra = [f"-D{d}" for d in (defines or [])]
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "splbm_b200.h")]
    objs = []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(bdir, src + ".o")
        objs.append(o)
        if not force and _newer(o, [s] + hdrs):
            continue
        cmd = [nvcc()] + NVCC_FLAGS + extra + ["-c", s, "-o", o]
        if src.endswith(".cpp"):
            cmd = [nvcc()] + NVCC_FLAGS + extra + ["-x", "cu", "-c", s, "-o", o]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    if force or not _newer(out_lib, objs):
        tmp = out_lib + ".tmp"
        subprocess.run([nvcc()] + ARCH + ["-shared", "-o", tmp] + objs + ["-lpthread", "-ldl"], check=True)
        os.replace(tmp, out_lib)
    return out_lib


def build_all(force: bool = False, verbose: bool = False) -> list[str]:
    """The bit-exact library and the tolerance-mode (SPLBM_FMA=1) library."""
    return [build(force, verbose),
            build(force, verbose, defines=["SPLBM_FMA=1"], lib=FMA_LIB, build_dir=FMA_BUILD)]


if __name__ == "__main__":
    print(build_all(force="--force" in sys.argv, verbose=True))
