"""Harness input: the reference's PowerLawSampler (workload.cpp:24-70),
bit-exact, from tools/libhps_workload.so (tools/workload.cpp). Used by
bench.py, the tests and the tools to draw the same key streams the reference
draws; not part of the product library."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
SRC = HERE / "workload.cpp"
SO = HERE / "libhps_workload.so"
_lib = None


def build() -> Path:
    if not SO.exists() or SO.stat().st_mtime < SRC.stat().st_mtime:
        subprocess.run(["g++", "-std=c++20", "-O2", "-fPIC", "-shared", str(SRC), "-o", str(SO)],
                       check=True)
    return SO


def _l():
    global _lib
    if _lib is None:
        if not SO.exists():
            build()
        _lib = C.CDLL(str(SO))
        _lib.hps_powerlaw_sample.restype = C.c_int
        _lib.hps_powerlaw_sample.argtypes = [C.c_double, C.c_uint64, C.c_uint64, C.c_uint64,
                                             C.c_size_t, C.c_void_p]
    return _lib


def powerlaw_sample(alpha: float, keyspace: int, permute_seed: int, draw_seed: int,
                    count: int) -> np.ndarray:
    """PowerLawSampler::sample (workload.cpp:24-70), bit-exact."""
    out = np.empty(count, dtype=np.uint64)
    rc = _l().hps_powerlaw_sample(alpha, keyspace, permute_seed, draw_seed, count,
                                  out.ctypes.data)
    if rc != 0:
        raise ValueError("powerlaw_sample: keyspace and alpha must be positive")
    return out
