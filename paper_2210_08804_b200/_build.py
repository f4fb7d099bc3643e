"""Builds the in-tree native library libhps_b200.so with nvcc for sm_100a.

All translation units (CUDA kernels, the host runtime and the C ABI) are
compiled by nvcc (`-x cu` for the .cpp files, which share the device
headers) and linked into one shared object next to this file, so the GPU box
receives it with the repo snapshot. Incremental: objects are rebuilt only
when a source or header is newer.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
BUILD = PKG / "build"
LIB = PKG / "libhps_b200.so"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++20", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
         "--expt-relaxed-constexpr", f"-I{ROOT / 'include'}", f"-I{CSRC}"]

SOURCES = ["cache_kernels.cu", "lookup_kernels.cu", "shard_kernels.cu", "wire.cu", "device_cache.cpp", "volatile_store.cpp", "segment_store.cpp",
           "peer.cpp", "engine.cpp", "capi.cpp"]


def _newest_header() -> float:
    hs = list(CSRC.glob("*.cuh")) + list(CSRC.glob("*.hpp")) + list((ROOT / "include").glob("*.h"))
    return max(h.stat().st_mtime for h in hs)


def build(verbose: bool = False, variant: str | None = None, defines: tuple = ()) -> Path:
    """Builds libhps_b200.so; with `variant`, libhps_b200.<variant>.so from the
    same sources plus `-D` `defines` (compile-time A/B builds, loaded with
    HPSB_LIB_VARIANT=<variant>; tools/build_variant.py)."""
    bdir = BUILD / variant if variant else BUILD
    lib = PKG / f"libhps_b200.{variant}.so" if variant else LIB
    bdir.mkdir(parents=True, exist_ok=True)
    hdr = _newest_header()
    objs = []
    for src in SOURCES:
        s = CSRC / src
        o = bdir / (src + ".o")
        objs.append(o)
        if o.exists() and o.stat().st_mtime >= max(s.stat().st_mtime, hdr):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, *(f"-D{d}" for d in defines)]
        if src.endswith(".cpp"):
            cmd += ["-x", "cu"]
        cmd += ["-c", str(s), "-o", str(o)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    if not lib.exists() or lib.stat().st_mtime < max(o.stat().st_mtime for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", str(lib), *map(str, objs), "-lcudart_static",
               "-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return lib


if __name__ == "__main__":
    print(build(verbose=True))
