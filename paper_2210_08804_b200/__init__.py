"""B200-native HPS lookup path: Python mirror of the reference interface.

The product is the native library ``libhps_b200.so`` (CUDA kernels for
sm_100a + the C++ host runtime) behind the C ABI in ``include/hps_b200.h``.
This module binds that ABI with ctypes and mirrors the reference's C++ API
(``/root/reference/proj/core/include/hps/*.hpp``) with the same names,
argument meaning and error behaviour, so tests read like the reference's own:

=====================  ==================================================
Python                 reference
=====================  ==================================================
SlabCacheConfig        SlabCacheConfig        slab_cache.hpp:27-34
SlabCache              SlabCache              slab_cache.hpp:41-116
CacheMiss              CacheMiss              slab_cache.hpp:36-39
VolatileStore          VolatileStore          volatile_store.hpp:45-137
VolatileTableConfig    VolatileTableConfig    volatile_store.hpp:31-40
EngineConfig           EngineConfig           lookup_engine.hpp:29-37
LookupEngine           LookupEngine           lookup_engine.hpp:152-196
LookupOutcome          LookupOutcome          lookup_engine.hpp:145-150
LookupResult           LookupResult           types.hpp:41-48
FetchResult            FetchResult            types.hpp:51-55
tier_fetch             tier_fetch             lookup_engine.hpp:125-127
dedup_keys             dedup_keys             types.hpp:57-64
xxh64 / xxh64_key      xxh64 / xxh64_key      xxhash64.hpp:60-124
partition_of           partition_of           volatile_store.hpp:43
=====================  ==================================================

Errors: ``InvalidArgument`` (a ``ValueError``) where the reference throws
``std::invalid_argument``; ``LogicError`` for ``std::logic_error``;
``TierFault`` for ``hps::TierFault``; ``HpsError`` for CUDA / internal
failures. There is no CPU fallback: if the native library is missing or no
GPU is present, cache and engine calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from pathlib import Path
from typing import List, NamedTuple, Optional, Sequence

import numpy as np

_PKG = Path(__file__).resolve().parent
# HPSB_LIB_VARIANT=<name> loads libhps_b200.<name>.so built next to it (same-box
# A/B of two builds, tools/ab.sh); the default is the in-tree build.
LIB_PATH = _PKG / (f"libhps_b200.{os.environ['HPSB_LIB_VARIANT']}.so"
                   if os.environ.get("HPSB_LIB_VARIANT") else "libhps_b200.so")

kSlotsPerSlab = 32
kSlabsetSeed = 0x5EED5E7
kSlabSeed = 0x51AB
kPartitionSeed = 0

HPS_MEM_HOST = 0
HPS_MEM_DEVICE = 1
HPS_REPLACE_EXACT = 0
HPS_REPLACE_RELAXED = 1


class HpsError(RuntimeError):
    """CUDA / internal failure inside the native library."""


class InvalidArgument(ValueError):
    """std::invalid_argument in the reference."""


class LogicError(RuntimeError):
    """std::logic_error in the reference (check_invariants)."""


class TierFault(RuntimeError):
    """hps::TierFault in the reference (types.hpp:14-20)."""


class OutOfMemory(MemoryError):
    pass


_ERR = {1: InvalidArgument, 2: HpsError, 3: OutOfMemory, 4: LogicError, 5: TierFault}

_lib: Optional[C.CDLL] = None


class _CacheConfig(C.Structure):
    _fields_ = [("slabset_count", C.c_uint64), ("slabs_per_set", C.c_uint32),
                ("dimension", C.c_uint32), ("worker_pool_size", C.c_uint32),
                ("tasks_per_worker", C.c_uint32)]


class _CacheInfo(C.Structure):
    _fields_ = [("dimension", C.c_uint32), ("slabs_per_set", C.c_uint32),
                ("slabset_count", C.c_uint64), ("capacity", C.c_uint64),
                ("occupied", C.c_uint64), ("recency_clock", C.c_uint64),
                ("device", C.c_int), ("reserved", C.c_int)]


class _EngineConfig(C.Structure):
    _fields_ = [("hit_rate_threshold", C.c_double), ("default_vector", C.POINTER(C.c_float)),
                ("default_vector_len", C.c_uint32), ("workspace_pool_size", C.c_uint32),
                ("async_worker_count", C.c_uint32), ("volatile_tier_enabled", C.c_int),
                ("max_batch", C.c_uint32)]


class _Outcome(C.Structure):
    _fields_ = [("sync_branch", C.c_int), ("unique_hit_rate", C.c_double),
                ("unique_count", C.c_uint64), ("defaults_returned", C.c_uint64)]


class _Stats(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "queries", "queried_keys", "unique_keys", "cache_hits", "cache_misses", "sync_batches",
        "async_batches", "defaults_returned", "vdb_hits", "pdb_hits", "tier_missing",
        "async_faults")]


COLD_FETCH_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_size_t,
                            C.POINTER(C.c_uint64), C.POINTER(C.c_float), C.POINTER(C.c_size_t),
                            C.POINTER(C.c_uint64), C.POINTER(C.c_size_t))

# name -> (restype, argtypes); mirrors include/hps_b200.h
_P = C.c_void_p
_U64P = C.POINTER(C.c_uint64)
_SZP = C.POINTER(C.c_size_t)
SIGNATURES = {
    "hps_last_error": (C.c_char_p, []),
    "hps_kernel_launch_count": (C.c_uint64, []),
    "hps_xxh64": (C.c_uint64, [_P, C.c_size_t, C.c_uint64]),
    "hps_xxh64_key": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "hps_slabset_of": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "hps_first_slab_of": (C.c_uint32, [C.c_uint64, C.c_uint32]),
    "hps_partition_of": (C.c_uint32, [C.c_uint64, C.c_uint32]),
    "hps_dedup_keys": (C.c_int, [C.c_int, _P, C.c_size_t, _P, _P, _SZP, C.c_int, _P]),
    "hps_cache_create": (C.c_int, [C.POINTER(_CacheConfig), C.c_int, C.POINTER(_P)]),
    "hps_cache_destroy": (C.c_int, [_P]),
    "hps_cache_get_info": (C.c_int, [_P, C.POINTER(_CacheInfo)]),
    "hps_cache_stream": (_P, [_P]),
    "hps_cache_query": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t, _P, _P, _SZP, C.c_int, _P]),
    "hps_cache_lookup_device": (C.c_int, [_P, _P, C.c_size_t, _P, _P, _P, _P, _P, _P, _P]),
    "hps_cache_set_profile_events": (C.c_int, [_P, _P, _P]),
    "hps_stream_begin_capture": (C.c_int, [_P]),
    "hps_stream_end_capture": (C.c_int, [_P, C.POINTER(_P)]),
    "hps_graph_launch": (C.c_int, [_P, _P]),
    "hps_graph_destroy": (C.c_int, [_P]),
    "hps_event_record": (C.c_int, [_P, _P]),
    "hps_cache_replace": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t, C.c_int, _P]),
    "hps_cache_replace_device_async": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t, _P]),
    "hps_cache_set_replace_mode": (C.c_int, [_P, C.c_int]),
    "hps_peer_blob_size": (C.c_size_t, []),
    "hps_cache_peer_export": (C.c_int, [_P, C.c_uint64, _P, C.c_size_t, _SZP]),
    "hps_peer_group_create": (C.c_int, [_P, C.c_uint32, C.c_uint32, _P, C.c_size_t,
                                        C.POINTER(_P)]),
    "hps_peer_group_destroy": (C.c_int, [_P]),
    "hps_peer_lookup_device": (C.c_int, [_P, _P, C.c_size_t, _P, _P, _P, _P]),
    "hps_cache_peer_drain": (C.c_int, [_P, _P, C.c_size_t, _SZP]),
    "hps_cache_get_replace_mode": (C.c_int, [_P, C.POINTER(C.c_int), C.POINTER(C.c_uint64)]),
    "hps_cache_update": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t, _SZP, C.c_int, _P]),
    "hps_cache_dump": (C.c_int, [_P, C.c_uint64, C.c_uint64, _P, C.c_size_t, _SZP]),
    "hps_cache_check_invariants": (C.c_int, [_P]),
    "hps_cache_export_state": (C.c_int, [_P, _P, _P, _P, _P]),
    "hps_cache_debug_trace": (C.c_int, [_P, _P, C.c_size_t, _U64P]),
    "hps_cache_update_device": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t, _P, _P]),
    "hps_shard_of": (C.c_uint32, [C.c_uint64, C.c_uint32]),
    "hps_engine_lookup_multi": (C.c_int, [_P, C.c_size_t, _P, _P, _P, _P, _P, C.c_int]),
    "hps_cache_dump_device": (C.c_int, [_P, C.c_uint64, C.c_uint64, _P, _P, _P]),
    "hps_cache_create_shared": (C.c_int, [_P, C.c_int, _P, C.POINTER(_P)]),
    "hps_wire_lookup_frame": (C.c_int, [C.c_int, _P, _P, C.c_uint32, C.c_uint32, C.c_int, _P,
                                        C.c_size_t, _SZP, _P]),
    "hps_multi_create": (C.c_int, [_P, C.c_size_t, C.c_size_t, C.POINTER(_P)]),
    "hps_multi_destroy": (C.c_int, [_P]),
    "hps_multi_lookup": (C.c_int, [_P, _P, _P, _P, _P, _P]),
    "hps_refresh_cache": (C.c_int, [_P, _P, C.c_char_p, _P, _P, C.c_size_t, _U64P, _P,
                                    C.c_size_t, _SZP]),
    "hps_shard_count": (C.c_int, [C.c_int, _P, C.c_size_t, C.c_uint32, _P, _P]),
    "hps_shard_scatter": (C.c_int, [C.c_int, _P, C.c_size_t, C.c_uint32, _P, _P, _P, _P]),
    "hps_shard_unroute": (C.c_int, [C.c_int, C.c_size_t, C.c_uint32, _P, _P, _P, _P, _P, _P]),
    "hps_vdb_create": (C.c_int, [C.c_uint32, C.POINTER(_P)]),
    "hps_vdb_destroy": (C.c_int, [_P]),
    "hps_vdb_register_table": (C.c_int, [_P, C.c_char_p, C.c_uint32, C.c_uint32, C.c_uint64]),
    "hps_vdb_has_table": (C.c_int, [_P, C.c_char_p]),
    "hps_vdb_insert": (C.c_int, [_P, C.c_char_p, _P, C.c_size_t, _P, C.c_size_t, _P, C.c_size_t,
                                 _SZP]),
    "hps_vdb_insert_async": (C.c_int, [_P, C.c_char_p, _P, C.c_size_t, _P, C.c_size_t]),
    "hps_vdb_lookup": (C.c_int, [_P, C.c_char_p, _P, C.c_size_t, _P, _P, _SZP, _P, _SZP]),
    "hps_vdb_drain": (C.c_int, [_P]),
    "hps_vdb_table_size": (C.c_int, [_P, C.c_char_p, _U64P]),
    "hps_vdb_partition_size": (C.c_int, [_P, C.c_char_p, C.c_uint32, _U64P]),
    "hps_vdb_table_clock": (C.c_int, [_P, C.c_char_p, _U64P]),
    "hps_vdb_last_access": (C.c_int, [_P, C.c_char_p, C.c_uint64, _U64P, C.POINTER(C.c_int)]),
    "hps_vdb_evict": (C.c_int, [_P, C.c_char_p, C.c_uint32, _P, C.c_size_t, _SZP]),
    "hps_vdb_last_evicted": (C.c_int, [_P, C.c_size_t, _SZP]),
    "hps_pdb_open": (C.c_int, [C.c_char_p, C.c_uint32, C.POINTER(_P)]),
    "hps_pdb_destroy": (C.c_int, [_P]),
    "hps_pdb_attach": (C.c_int, [_P, C.c_char_p]),
    "hps_pdb_refresh": (C.c_int, [_P, C.c_char_p]),
    "hps_pdb_info": (C.c_int, [_P, C.c_char_p, C.POINTER(C.c_uint32), _U64P, _U64P]),
    "hps_pdb_get": (C.c_int, [_P, C.c_char_p, _P, C.c_size_t, _P, _P, _SZP, _P, _SZP]),
    "hps_pdb_table_ctx": (C.c_int, [_P, C.c_char_p, C.POINTER(_P)]),
    "hps_pdb_cold_fetch": (C.c_int, [_P, _P, C.c_size_t, _P, _P, _SZP, _P, _SZP]),
    "hps_vdb_dimension": (C.c_int, [_P, C.c_char_p, C.POINTER(C.c_uint32)]),
    "hps_vdb_partition_count": (C.c_int, [_P, C.c_char_p, C.POINTER(C.c_uint32)]),
    "hps_vdb_keys": (C.c_int, [_P, C.c_char_p, _P, C.c_size_t, _SZP]),
    "hps_tier_fetch": (C.c_int, [_P, C.c_char_p, C.c_uint32, COLD_FETCH_FN, _P, _P, C.c_size_t,
                                 _P, _P, _SZP, _P, _SZP, _P]),
    "hps_engine_create": (C.c_int, [C.c_char_p, C.c_uint32, _P, _P, COLD_FETCH_FN, _P,
                                    C.POINTER(_EngineConfig), C.POINTER(_P)]),
    "hps_engine_destroy": (C.c_int, [_P]),
    "hps_engine_lookup": (C.c_int, [_P, _P, C.c_size_t, _P, C.c_size_t, _P, C.POINTER(_Outcome),
                                    C.c_int, _P]),
    "hps_engine_drain_async": (C.c_int, [_P]),
    "hps_engine_get_stats": (C.c_int, [_P, C.POINTER(_Stats)]),
    "hps_engine_reserve": (C.c_int, [_P, C.c_size_t]),
    "hps_replicas_create": (C.c_int, [_P, C.c_size_t, C.POINTER(_P)]),
    "hps_replicas_destroy": (C.c_int, [_P]),
    "hps_replicas_lookup": (C.c_int, [_P, _P, _P, _P, _P, _P, C.c_int]),
    "hps_engine_pool_info": (C.c_int, [_P, _U64P, _U64P, _U64P]),
}


def lib() -> C.CDLL:
    """Loads the in-tree native library (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2210_08804_b200._build)")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().hps_last_error().decode(errors="replace")
        raise _ERR.get(rc, HpsError)(msg)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------- vocabulary --
def kernel_launch_count() -> int:
    """Kernels launched by libhps_b200 in this process so far."""
    return int(lib().hps_kernel_launch_count())


def xxh64(data: bytes, seed: int = 0) -> int:
    buf = C.create_string_buffer(bytes(data), len(data))
    return int(lib().hps_xxh64(buf, len(data), seed))


def xxh64_key(key: int, seed: int) -> int:
    return int(lib().hps_xxh64_key(key, seed))


class StreamGraph:
    """CUDA graph captured from library calls on `stream` (see
    hps_stream_begin_capture in include/hps_b200.h)."""

    def __init__(self, stream: int):
        self.stream = stream
        self.exec = C.c_void_p()

    def __enter__(self):
        _check(lib().hps_stream_begin_capture(self.stream))
        return self

    def __exit__(self, et, ev, tb):
        rc = lib().hps_stream_end_capture(self.stream, C.byref(self.exec))
        if et is None:
            _check(rc)

    def launch(self, stream: int = 0):
        _check(lib().hps_graph_launch(self.exec, stream or self.stream))

    def __del__(self):
        try:
            if self.exec:
                lib().hps_graph_destroy(self.exec)
        except Exception:
            pass


def event_record(event: int, stream: int) -> None:
    """Records a cudaEvent_t on a stream (an external record node inside a
    capture, so it can time a region of a replayed graph)."""
    _check(lib().hps_event_record(event, stream))


def partition_of(key: int, partition_count: int) -> int:
    return int(lib().hps_partition_of(key, partition_count))


@dataclass
class TableId:
    name: str
    dimension: int


@dataclass
class DedupResult:
    unique_keys: np.ndarray
    inverse_indices: np.ndarray


def dedup_keys(keys, device: int = 0) -> DedupResult:
    """GPU dedup: unique keys in first-occurrence order + u32 inverse."""
    k = _u64(keys)
    uniq = np.empty(len(k), dtype=np.uint64)
    inv = np.empty(len(k), dtype=np.uint32)
    nu = C.c_size_t(0)
    _check(lib().hps_dedup_keys(device, _ptr(k), len(k), _ptr(uniq), _ptr(inv), C.byref(nu),
                                HPS_MEM_HOST, None))
    return DedupResult(uniq[: nu.value].copy(), inv)


@dataclass
class FetchResult:
    found_keys: np.ndarray
    found_vectors: np.ndarray
    missing_keys: np.ndarray


# ------------------------------------------------------------------ cache --
@dataclass
class SlabCacheConfig:
    slabset_count: int = 1
    slabs_per_set: int = 2
    dimension: int = 0
    worker_pool_size: int = 1
    tasks_per_worker: int = 8


class CacheMiss(NamedTuple):
    position: int
    key: int


class SlabCache:
    """HBM-resident set-associative embedding cache (slab_cache.hpp:41-116)."""

    def __init__(self, config: SlabCacheConfig, device: int = 0,
                 share_stream_with: Optional["SlabCache"] = None):
        """share_stream_with: join that cache's CACHE GROUP (one stream; the
        tables of one model) so a MultiLookup can run them in one launch."""
        self._h = C.c_void_p()
        cfg = _CacheConfig(config.slabset_count, config.slabs_per_set, config.dimension,
                           config.worker_pool_size, config.tasks_per_worker)
        if share_stream_with is None:
            _check(lib().hps_cache_create(C.byref(cfg), device, C.byref(self._h)))
        else:
            _check(lib().hps_cache_create_shared(C.byref(cfg), device, share_stream_with.handle,
                                                 C.byref(self._h)))
            self._group_anchor = share_stream_with
        self._dim = int(config.dimension)
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_cache_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    # -- operations ---------------------------------------------------------
    def query(self, keys, out_vectors: np.ndarray) -> List[CacheMiss]:
        """Copies hit rows into out_vectors (float32, modified in place; miss
        rows untouched) and returns misses in ascending position order."""
        k = _u64(keys)
        if not (isinstance(out_vectors, np.ndarray) and out_vectors.dtype == np.float32
                and out_vectors.flags.c_contiguous):
            raise InvalidArgument("out_vectors must be a contiguous float32 ndarray")
        n = len(k)
        pos = np.empty(max(n, 1), dtype=np.uint32)
        mk = np.empty(max(n, 1), dtype=np.uint64)
        nm = C.c_size_t(0)
        _check(lib().hps_cache_query(self._h, _ptr(k), n, _ptr(out_vectors), out_vectors.size,
                                     _ptr(pos), _ptr(mk), C.byref(nm), HPS_MEM_HOST, None))
        m = nm.value
        return [CacheMiss(int(p), int(q)) for p, q in zip(pos[:m], mk[:m])]

    def query_arrays(self, keys, out_vectors: np.ndarray):
        """query() returning (miss_positions, miss_keys) arrays."""
        k = _u64(keys)
        n = len(k)
        pos = np.empty(max(n, 1), dtype=np.uint32)
        mk = np.empty(max(n, 1), dtype=np.uint64)
        nm = C.c_size_t(0)
        _check(lib().hps_cache_query(self._h, _ptr(k), n, _ptr(out_vectors), out_vectors.size,
                                     _ptr(pos), _ptr(mk), C.byref(nm), HPS_MEM_HOST, None))
        return pos[: nm.value].copy(), mk[: nm.value].copy()

    def query_device(self, keys_ptr: int, n: int, out_ptr: int, miss_pos_ptr: int,
                     miss_keys_ptr: int, stream: int = 0) -> int:
        """Device-pointer query (e.g. torch tensors' data_ptr()); returns the
        miss count."""
        nm = C.c_size_t(0)
        _check(lib().hps_cache_query(self._h, keys_ptr, n, out_ptr, n * self._dim, miss_pos_ptr,
                                     miss_keys_ptr, C.byref(nm), HPS_MEM_DEVICE,
                                     stream or None))
        return nm.value

    def lookup_device(self, keys_ptr: int, n: int, out_ptr: int, flags_ptr: int,
                      default_row_ptr: int, miss_keys_ptr: int, miss_firsts_ptr: int,
                      counts_ptr: int, stream: int = 0) -> None:
        """hps_cache_lookup_device: the lookup hot path on device pointers,
        stream-ordered (no host sync). Unique misses come back as (key, first
        position) in claim order; sort by position for the reference order."""
        _check(lib().hps_cache_lookup_device(self._h, keys_ptr, n, out_ptr, flags_ptr,
                                             default_row_ptr, miss_keys_ptr, miss_firsts_ptr,
                                             counts_ptr, stream or None))

    def set_profile_events(self, start_event: int = 0, end_event: int = 0) -> None:
        _check(lib().hps_cache_set_profile_events(self._h, start_event or None,
                                                  end_event or None))

    def replace(self, keys, vectors) -> None:
        k = _u64(keys)
        v = _f32(vectors)
        _check(lib().hps_cache_replace(self._h, _ptr(k), len(k), _ptr(v), v.size, HPS_MEM_HOST,
                                       None))

    def replace_device(self, keys_ptr: int, n: int, rows_ptr: int, stream: int = 0) -> None:
        _check(lib().hps_cache_replace(self._h, keys_ptr, n, rows_ptr, n * self._dim,
                                       HPS_MEM_DEVICE, stream or None))

    def replace_fill(self, keys_ptr: int, n: int, rows_ptr: int, stream: int = 0) -> None:
        """Stream-ordered replace of DISTINCT device keys (the engine's miss
        fill; hps_cache_replace_device_async): no duplicate check, no sync."""
        _check(lib().hps_cache_replace_device_async(self._h, keys_ptr, n, rows_ptr, n * self._dim,
                                                    stream or None))

    def set_replace_mode(self, mode: int) -> None:
        """HPS_REPLACE_EXACT (default, slot-exact with the reference) or
        HPS_REPLACE_RELAXED (atomicCAS slot claims for distinct-key replaces;
        see include/hps_b200.h)."""
        _check(lib().hps_cache_set_replace_mode(self._h, int(mode)))

    def replace_mode(self) -> int:
        m = C.c_int(0)
        _check(lib().hps_cache_get_replace_mode(self._h, C.byref(m), None))
        return m.value

    def peer_export(self, inbox_cap: int = 1 << 20) -> bytes:
        """This shard's peer-mapping blob (CUDA IPC handles + geometry + a miss
        inbox of inbox_cap keys): ship it to the other ranks."""
        n = lib().hps_peer_blob_size()
        buf = C.create_string_buffer(n)
        ln = C.c_size_t(0)
        _check(lib().hps_cache_peer_export(self._h, inbox_cap, buf, n, C.byref(ln)))
        return buf.raw[: ln.value]

    def peer_drain(self, cap: int = 1 << 20) -> np.ndarray:
        """Keys peers appended to this shard's miss inbox since the last
        drain (input order unspecified, duplicates possible); empties it."""
        out = np.empty(max(cap, 1), dtype=np.uint64)
        n = C.c_size_t(0)
        _check(lib().hps_cache_peer_drain(self._h, _ptr(out), cap, C.byref(n)))
        return out[: min(n.value, cap)].copy()

    def relaxed_dropped(self) -> int:
        """Keys the relaxed mode has not admitted so far."""
        d = C.c_uint64(0)
        _check(lib().hps_cache_get_replace_mode(self._h, None, C.byref(d)))
        return d.value

    def update(self, keys, vectors) -> int:
        k = _u64(keys)
        v = _f32(vectors)
        w = C.c_size_t(0)
        _check(lib().hps_cache_update(self._h, _ptr(k), len(k), _ptr(v), v.size, C.byref(w),
                                      HPS_MEM_HOST, None))
        return w.value

    def update_device(self, keys_ptr: int, n: int, rows_ptr: int, stream: int = 0) -> int:
        w = C.c_size_t(0)
        _check(lib().hps_cache_update(self._h, keys_ptr, n, rows_ptr, n * self._dim, C.byref(w),
                                      HPS_MEM_DEVICE, stream or None))
        return w.value

    def update_device_async(self, keys_ptr: int, n: int, rows_ptr: int, written_ptr: int = 0,
                            stream: int = 0) -> None:
        """hps_cache_update_device: stream-ordered update on device pointers;
        the written count lands in device memory at written_ptr (optional)."""
        _check(lib().hps_cache_update_device(self._h, keys_ptr, n, rows_ptr, n * self._dim,
                                             written_ptr or None, stream or None))

    def dump_device_async(self, set_begin: int, set_end: int, out_ptr: int, n_out_ptr: int,
                          stream: int = 0) -> None:
        """hps_cache_dump_device: stream-ordered dump into device memory."""
        _check(lib().hps_cache_dump_device(self._h, set_begin, set_end, out_ptr, n_out_ptr,
                                           stream or None))

    def dump(self, batch_size: int) -> "DumpCursor":
        if batch_size == 0:
            raise InvalidArgument("dump batch size must be positive")
        return DumpCursor(self, batch_size)

    def dump_range(self, set_begin: int, set_end: int) -> np.ndarray:
        cap = max(0, (min(set_end, self.slabset_count()) - set_begin)) * self.slabs_per_set() * 32
        out = np.empty(max(cap, 1), dtype=np.uint64)
        n = C.c_size_t(0)
        _check(lib().hps_cache_dump(self._h, set_begin, set_end, _ptr(out), cap, C.byref(n)))
        return out[: n.value].copy()

    def dump_all(self) -> np.ndarray:
        return self.dump_range(0, self.slabset_count())

    def check_invariants(self) -> None:
        _check(lib().hps_cache_check_invariants(self._h))

    def export_state(self):
        """(keys, counters, masks, rows) host copies of the device table."""
        cap = self.capacity()
        keys = np.empty(cap, dtype=np.uint64)
        ctr = np.empty(cap, dtype=np.uint64)
        masks = np.empty(self.slabset_count() * self.slabs_per_set(), dtype=np.uint32)
        rows = np.empty(cap * self._dim, dtype=np.float32)
        _check(lib().hps_cache_export_state(self._h, _ptr(keys), _ptr(ctr), _ptr(masks),
                                            _ptr(rows)))
        return keys, ctr, masks, rows

    def debug_trace(self) -> np.ndarray:
        """Per-call lookup phase timeline (HPSB_TRACE=1), absolute globaltimer
        ns: rows of [first block start, last A done, last block start, first
        A done, first copy done, last copy done, finish start, finish end],
        oldest first; resets the ring."""
        ring = np.empty(4096 * 8, dtype=np.uint64)
        n = C.c_uint64(0)
        _check(lib().hps_cache_debug_trace(self._h, _ptr(ring), ring.size, C.byref(n)))
        k = min(int(n.value), 4096)
        r = ring.reshape(-1, 8)
        idx = [(int(n.value) - k + i) % 4096 for i in range(k)]
        r = r[idx].copy()
        for f in (1, 2, 5):
            r[:, f] = ~r[:, f]
        return r.astype(np.int64)

    # -- accessors (slab_cache.hpp:95-106) ----------------------------------
    def _info(self) -> _CacheInfo:
        i = _CacheInfo()
        _check(lib().hps_cache_get_info(self._h, C.byref(i)))
        return i

    def dimension(self) -> int:
        return self._dim

    def slabset_count(self) -> int:
        return int(self._info().slabset_count)

    def slabs_per_set(self) -> int:
        return int(self._info().slabs_per_set)

    def capacity(self) -> int:
        return int(self._info().capacity)

    def occupied(self) -> int:
        return int(self._info().occupied)

    def recency_clock(self) -> int:
        return int(self._info().recency_clock)

    def stream(self) -> int:
        return int(lib().hps_cache_stream(self._h) or 0)

    @staticmethod
    def slabset_of(key: int, slabset_count: int) -> int:
        return int(lib().hps_slabset_of(key, slabset_count))

    @staticmethod
    def first_slab_of(key: int, slabs_per_set: int) -> int:
        return int(lib().hps_first_slab_of(key, slabs_per_set))


class DumpCursor:
    """SlabCache::DumpCursor (slab_cache.hpp:74-90): batches of resident keys,
    reading a bounded range of slabsets per device call."""

    _SETS_PER_CALL = 4096

    def __init__(self, cache: SlabCache, batch_size: int):
        self._c = cache
        self._bs = batch_size
        self._next_set = 0
        self._staged = np.empty(0, dtype=np.uint64)
        self._pos = 0
        self._S = cache.slabset_count()

    def next(self) -> Optional[np.ndarray]:
        out: List[np.ndarray] = []
        have = 0
        while True:
            take = min(self._bs - have, len(self._staged) - self._pos)
            if take > 0:
                out.append(self._staged[self._pos: self._pos + take])
                self._pos += take
                have += take
            if have == self._bs:
                return np.concatenate(out)
            if self._next_set >= self._S:
                return np.concatenate(out) if have else None
            end = min(self._S, self._next_set + self._SETS_PER_CALL)
            self._staged = self._c.dump_range(self._next_set, end)
            self._pos = 0
            self._next_set = end


# -------------------------------------------------------------------- vdb --
@dataclass
class VolatileTableConfig:
    partition_count: int = 16
    overflow_margin: int = 1 << 20
    initial_cache_rate: float = 1.0


class VolatileStore:
    """Host volatile DB tier (volatile_store.hpp:45-137)."""

    def __init__(self, lookup_threads: int = 0):
        self._h = C.c_void_p()
        _check(lib().hps_vdb_create(lookup_threads, C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_vdb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def register_table(self, table: TableId, config: VolatileTableConfig = VolatileTableConfig()):
        _check(lib().hps_vdb_register_table(self._h, table.name.encode(), table.dimension,
                                            config.partition_count, config.overflow_margin))

    def has_table(self, name: str) -> bool:
        return bool(lib().hps_vdb_has_table(self._h, name.encode()))

    def partition_count(self, name: str) -> int:
        v = C.c_uint32(0)
        _check(lib().hps_vdb_partition_count(self._h, name.encode(), C.byref(v)))
        return v.value

    def _dim(self, name: str) -> int:
        v = C.c_uint32(0)
        _check(lib().hps_vdb_dimension(self._h, name.encode(), C.byref(v)))
        return v.value

    @staticmethod
    def _evicted(ev: np.ndarray, n: int) -> np.ndarray:
        if n > len(ev):
            ev = np.empty(n, dtype=np.uint64)
            ne = C.c_size_t(0)
            _check(lib().hps_vdb_last_evicted(_ptr(ev), n, C.byref(ne)))
        return ev[:n].copy()

    def insert(self, name: str, keys, vectors) -> np.ndarray:
        k = _u64(keys)
        v = _f32(vectors)
        cap = len(k) + 64
        ev = np.empty(cap, dtype=np.uint64)
        ne = C.c_size_t(0)
        _check(lib().hps_vdb_insert(self._h, name.encode(), _ptr(k), len(k), _ptr(v), v.size,
                                    _ptr(ev), cap, C.byref(ne)))
        return self._evicted(ev, ne.value)

    def keys(self, name: str) -> np.ndarray:
        n = C.c_size_t(0)
        _check(lib().hps_vdb_keys(self._h, name.encode(), None, 0, C.byref(n)))
        out = np.empty(n.value + 1024, dtype=np.uint64)
        _check(lib().hps_vdb_keys(self._h, name.encode(), _ptr(out), len(out), C.byref(n)))
        if n.value > len(out):
            out = np.empty(n.value, dtype=np.uint64)
            _check(lib().hps_vdb_keys(self._h, name.encode(), _ptr(out), len(out), C.byref(n)))
        return out[: min(n.value, len(out))].copy()

    def insert_async(self, name: str, keys, vectors) -> None:
        k = _u64(keys)
        v = _f32(vectors)
        _check(lib().hps_vdb_insert_async(self._h, name.encode(), _ptr(k), len(k), _ptr(v),
                                          v.size))

    def lookup(self, name: str, keys) -> FetchResult:
        k = _u64(keys)
        d = self._dim(name)
        n = len(k)
        fk = np.empty(max(n, 1), dtype=np.uint64)
        fv = np.empty(max(n, 1) * d, dtype=np.float32)
        mk = np.empty(max(n, 1), dtype=np.uint64)
        nf, nm = C.c_size_t(0), C.c_size_t(0)
        _check(lib().hps_vdb_lookup(self._h, name.encode(), _ptr(k), n, _ptr(fk), _ptr(fv),
                                    C.byref(nf), _ptr(mk), C.byref(nm)))
        return FetchResult(fk[: nf.value].copy(), fv[: nf.value * d].copy(), mk[: nm.value].copy())

    def evict(self, name: str, partition: int) -> np.ndarray:
        cap = 1024
        ev = np.empty(cap, dtype=np.uint64)
        ne = C.c_size_t(0)
        _check(lib().hps_vdb_evict(self._h, name.encode(), partition, _ptr(ev), cap, C.byref(ne)))
        return self._evicted(ev, ne.value)

    def drain(self) -> None:
        _check(lib().hps_vdb_drain(self._h))

    def partition_size(self, name: str, partition: int) -> int:
        v = C.c_uint64(0)
        _check(lib().hps_vdb_partition_size(self._h, name.encode(), partition, C.byref(v)))
        return v.value

    def table_size(self, name: str) -> int:
        v = C.c_uint64(0)
        _check(lib().hps_vdb_table_size(self._h, name.encode(), C.byref(v)))
        return v.value

    def table_clock(self, name: str) -> int:
        v = C.c_uint64(0)
        _check(lib().hps_vdb_table_clock(self._h, name.encode(), C.byref(v)))
        return v.value

    def last_access(self, name: str, key: int) -> Optional[int]:
        v = C.c_uint64(0)
        f = C.c_int(0)
        _check(lib().hps_vdb_last_access(self._h, name.encode(), key, C.byref(v), C.byref(f)))
        return v.value if f.value else None


# ------------------------------------------------------------- cold tier --
class ColdTier:
    """Adapter turning any object with ``get(keys) -> FetchResult`` (the
    reference's PersistentStore::get contract, persistent_store.cpp:405-439)
    into the C callback the engine calls for VDB leftovers."""

    def __init__(self, store, dimension: int):
        self.store = store
        self.dim = dimension

        def _cb(ctx, keys, n, fk, fv, nf, mk, nm):
            try:
                ks = np.ctypeslib.as_array(keys, shape=(n,)).copy() if n else np.empty(0, np.uint64)
                r = self.store.get(ks)
                f = _u64(r.found_keys)
                v = _f32(r.found_vectors)
                m = _u64(r.missing_keys)
                if len(f):
                    C.memmove(fk, f.ctypes.data, f.nbytes)
                    C.memmove(fv, v.ctypes.data, v.nbytes)
                if len(m):
                    C.memmove(mk, m.ctypes.data, m.nbytes)
                nf[0] = len(f)
                nm[0] = len(m)
                return 0
            except Exception:  # surfaces as TierFault in the engine
                return 1

        self.fn = COLD_FETCH_FN(_cb)


class SegmentStore:
    """Batched cold reads over the reference's persistent-store files
    (hps_pdb_*): <root>/<escaped table>/{MANIFEST,
    seg-<n>.log} indexed the way PersistentStore's open does
    (persistent_store.cpp:229-268), memory-mapped, a batch's probes and row
    copies spread over host threads -- in place of PersistentStore::get's one
    pread per key (persistent_store.cpp:405-439). Read-only."""

    def __init__(self, root, threads: int = 0):
        self._h = C.c_void_p()
        _check(lib().hps_pdb_open(str(root).encode(), threads, C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_pdb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def attach(self, name: str) -> None:
        _check(lib().hps_pdb_attach(self._h, name.encode()))

    def refresh(self, name: str) -> None:
        _check(lib().hps_pdb_refresh(self._h, name.encode()))

    def _info(self, name: str):
        d, k, sg = C.c_uint32(0), C.c_uint64(0), C.c_uint64(0)
        _check(lib().hps_pdb_info(self._h, name.encode(), C.byref(d), C.byref(k), C.byref(sg)))
        return d.value, k.value, sg.value

    def dimension(self, name: str) -> int:
        return self._info(name)[0]

    def key_count(self, name: str) -> int:
        return self._info(name)[1]

    def segment_count(self, name: str) -> int:
        return self._info(name)[2]

    def get(self, name: str, keys) -> FetchResult:
        k = _u64(keys)
        n = len(k)
        d = self.dimension(name)
        fk = np.empty(max(n, 1), dtype=np.uint64)
        fv = np.empty(max(n, 1) * d, dtype=np.float32)
        mk = np.empty(max(n, 1), dtype=np.uint64)
        nf, nm = C.c_size_t(0), C.c_size_t(0)
        _check(lib().hps_pdb_get(self._h, name.encode(), _ptr(k), n, _ptr(fk), _ptr(fv),
                                 C.byref(nf), _ptr(mk), C.byref(nm)))
        return FetchResult(fk[: nf.value].copy(), fv[: nf.value * d].copy(), mk[: nm.value].copy())

    def table(self, name: str) -> "SegmentTable":
        return SegmentTable(self, name)


class SegmentTable:
    """One table of a SegmentStore as an engine cold tier: passed as `pdb`
    to LookupEngine / tier_fetch / refresh_cache it is called NATIVELY
    (hps_pdb_cold_fetch), no Python callback on the miss path."""

    def __init__(self, store: SegmentStore, name: str):
        self.store = store
        self.name = name
        self.ctx = C.c_void_p()
        _check(lib().hps_pdb_table_ctx(store._h, name.encode(), C.byref(self.ctx)))
        self.fn = C.cast(lib().hps_pdb_cold_fetch, COLD_FETCH_FN)

    def get(self, keys) -> FetchResult:
        return self.store.get(self.name, keys)


def _cold(pdb, dim):
    """(callback, ctx, keep-alive) of a cold tier: native for a SegmentTable,
    a ctypes adapter for any object with get(keys) -> FetchResult."""
    if pdb is None:
        return _NULL_COLD, None, None
    if isinstance(pdb, SegmentTable):
        return pdb.fn, pdb.ctx, pdb
    ct = ColdTier(pdb, dim)
    return ct.fn, None, ct


class DictStore:
    """Minimal in-memory cold tier with the PersistentStore::get contract
    (found keys / rows and missing keys in input order)."""

    def __init__(self, dimension: int):
        self.dim = dimension
        self.rows = {}

    def put(self, keys, vectors):
        v = _f32(vectors).reshape(-1, self.dim)
        for k, r in zip(_u64(keys), v):
            self.rows[int(k)] = r.copy()

    def get(self, keys) -> FetchResult:
        fk, fv, mk = [], [], []
        for k in _u64(keys):
            r = self.rows.get(int(k))
            if r is None:
                mk.append(int(k))
            else:
                fk.append(int(k))
                fv.append(r)
        return FetchResult(np.array(fk, dtype=np.uint64),
                           np.concatenate(fv).astype(np.float32) if fv else np.empty(0, np.float32),
                           np.array(mk, dtype=np.uint64))


_NULL_COLD = COLD_FETCH_FN()


def tier_fetch(table: TableId, keys, vdb: Optional[VolatileStore], pdb=None,
               counters: Optional[dict] = None) -> FetchResult:
    """lookup_engine.cpp:50-89: VDB first, then the cold tier (pdb)."""
    k = _u64(keys)
    n = len(k)
    d = table.dimension
    cfn, cctx, _keep = _cold(pdb, d)
    fk = np.empty(max(n, 1), dtype=np.uint64)
    fv = np.empty(max(n, 1) * d, dtype=np.float32)
    mk = np.empty(max(n, 1), dtype=np.uint64)
    nf, nm = C.c_size_t(0), C.c_size_t(0)
    cnt = np.zeros(3, dtype=np.uint64)
    _check(lib().hps_tier_fetch(vdb.handle if vdb else None, table.name.encode(), d,
                                cfn, cctx, _ptr(k), n, _ptr(fk),
                                _ptr(fv), C.byref(nf), _ptr(mk), C.byref(nm), _ptr(cnt)))
    if counters is not None:
        counters["vdb_hits"] = counters.get("vdb_hits", 0) + int(cnt[0])
        counters["pdb_hits"] = counters.get("pdb_hits", 0) + int(cnt[1])
        counters["missing"] = counters.get("missing", 0) + int(cnt[2])
    return FetchResult(fk[: nf.value].copy(), fv[: nf.value * d].copy(), mk[: nm.value].copy())


@dataclass
class RefreshOutcome:
    """refresh_engine.hpp:30-33"""
    refreshed: int = 0
    unresolved: np.ndarray = field(default_factory=lambda: np.empty(0, np.uint64))


def refresh_cache(cache: "SlabCache", table: TableId, vdb: Optional[VolatileStore], pdb=None,
                  dump_batch_size: int = 65536) -> RefreshOutcome:
    """refresh_engine.cpp:5-22 on the B200 cache (hps_refresh_cache): dump,
    tier fetch (VDB, then pdb), non-admitting update; the host fetch of one
    batch overlaps the device update of the previous one."""
    cfn, cctx, _keep = _cold(pdb, table.dimension)
    cap = cache.capacity()
    un = np.empty(max(cap, 1), dtype=np.uint64)
    refreshed = C.c_uint64(0)
    nu = C.c_size_t(0)
    _check(lib().hps_refresh_cache(cache.handle, vdb.handle if vdb else None,
                                   table.name.encode(), cfn, cctx,
                                   dump_batch_size, C.byref(refreshed), _ptr(un), cap,
                                   C.byref(nu)))
    return RefreshOutcome(int(refreshed.value), un[: nu.value].copy())


# ----------------------------------------------------------------- engine --
@dataclass
class EngineConfig:
    hit_rate_threshold: float = 0.8
    default_vector: Sequence[float] = field(default_factory=list)
    workspace_pool_size: int = 16
    async_worker_count: int = 2
    volatile_tier_enabled: bool = True
    max_batch: int = 0  # largest accepted batch (0 = no limit below 2^32)


@dataclass
class LookupOutcome:
    sync_branch: bool = False
    unique_hit_rate: float = 0.0
    unique_count: int = 0
    defaults_returned: int = 0


@dataclass
class LookupResult:
    dimension: int
    vectors: np.ndarray
    miss_flags: np.ndarray


@dataclass
class EngineStatsSnapshot:
    queries: int = 0
    queried_keys: int = 0
    unique_keys: int = 0
    cache_hits: int = 0
    cache_misses: int = 0
    sync_batches: int = 0
    async_batches: int = 0
    defaults_returned: int = 0
    vdb_hits: int = 0
    pdb_hits: int = 0
    tier_missing: int = 0
    async_faults: int = 0


@dataclass
class PoolInfo:
    size: int
    outstanding: int
    peak_outstanding: int


class LookupEngine:
    """lookup_engine.hpp:152-196, device-backed."""

    def __init__(self, table: TableId, cache: SlabCache, vdb: Optional[VolatileStore],
                 pdb=None, config: EngineConfig = EngineConfig()):
        self._h = C.c_void_p()
        self.table = table
        self.cache = cache
        self.vdb = vdb
        cfn, cctx, self._cold = _cold(pdb, table.dimension)
        dv = _f32(list(config.default_vector))
        self._dv = dv
        cfg = _EngineConfig(float(config.hit_rate_threshold),
                            dv.ctypes.data_as(C.POINTER(C.c_float)) if dv.size else None,
                            dv.size, config.workspace_pool_size, config.async_worker_count,
                            1 if config.volatile_tier_enabled else 0, config.max_batch)
        _check(lib().hps_engine_create(table.name.encode(), table.dimension, cache.handle,
                                       vdb.handle if vdb else None,
                                       cfn, cctx, C.byref(cfg), C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_engine_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup(self, keys, outcome: Optional[LookupOutcome] = None) -> LookupResult:
        k = _u64(keys)
        n = len(k)
        d = self.table.dimension
        out = np.empty(n * d, dtype=np.float32)
        flags = np.empty(max(n, 1), dtype=np.uint8)
        o = _Outcome()
        _check(lib().hps_engine_lookup(self._h, _ptr(k), n, _ptr(out), out.size, _ptr(flags),
                                       C.byref(o), HPS_MEM_HOST, None))
        if outcome is not None:
            outcome.sync_branch = bool(o.sync_branch)
            outcome.unique_hit_rate = float(o.unique_hit_rate)
            outcome.unique_count = int(o.unique_count)
            outcome.defaults_returned = int(o.defaults_returned)
        return LookupResult(d, out, flags[:n].copy())

    def lookup_ptrs(self, keys_ptr: int, n: int, out_ptr: int, flags_ptr: int, mem: int,
                    stream: int = 0) -> LookupOutcome:
        """Pointer-level lookup (device pointers with mem=HPS_MEM_DEVICE, or
        pinned host pointers with mem=HPS_MEM_HOST)."""
        o = _Outcome()
        _check(lib().hps_engine_lookup(self._h, keys_ptr, n, out_ptr, n * self.table.dimension,
                                       flags_ptr, C.byref(o), mem, stream or None))
        return LookupOutcome(bool(o.sync_branch), float(o.unique_hit_rate), int(o.unique_count),
                             int(o.defaults_returned))

    @staticmethod
    def lookup_multi_ptrs(engines, keys_ptrs, ns, out_ptrs, flags_ptrs, mem: int):
        """hps_engine_lookup_multi over pointers (one entry per engine/table);
        returns the per-table LookupOutcome list."""
        t = len(engines)
        PA = C.c_void_p * t
        outs = (_Outcome * t)()
        _check(lib().hps_engine_lookup_multi(
            PA(*[e._h for e in engines]), t, PA(*keys_ptrs), (C.c_size_t * t)(*ns),
            PA(*out_ptrs), PA(*flags_ptrs), outs, mem))
        return [LookupOutcome(bool(o.sync_branch), float(o.unique_hit_rate), int(o.unique_count),
                              int(o.defaults_returned)) for o in outs]

    def drain_async(self) -> None:
        _check(lib().hps_engine_drain_async(self._h))

    def reserve(self, max_keys: int) -> None:
        """Allocate every workspace for batches of up to max_keys now."""
        _check(lib().hps_engine_reserve(self._h, max_keys))

    def stats(self) -> EngineStatsSnapshot:
        s = _Stats()
        _check(lib().hps_engine_get_stats(self._h, C.byref(s)))
        return EngineStatsSnapshot(*[int(getattr(s, f)) for f, _ in _Stats._fields_])

    def workspace_pool(self) -> PoolInfo:
        a, b, c = C.c_uint64(), C.c_uint64(), C.c_uint64()
        _check(lib().hps_engine_pool_info(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return PoolInfo(a.value, b.value, c.value)


class ReplicaGroup:
    """The paper's concurrent deployment in one process: one
    cache replica + engine per GPU in `devices`, every engine over the SAME
    host VolatileStore (and cold tier), each replica serving its own batch on
    its own host thread (hps_replicas_*). No collective."""

    def __init__(self, devices: Sequence[int], cache_config: "SlabCacheConfig", table: TableId,
                 vdb: Optional[VolatileStore], pdb=None,
                 config: EngineConfig = EngineConfig()):
        self.caches = [SlabCache(cache_config, device=d) for d in devices]
        self.engines = [LookupEngine(table, c, vdb, pdb, config) for c in self.caches]
        self.table = table
        PA = C.c_void_p * len(self.engines)
        self._h = C.c_void_p()
        _check(lib().hps_replicas_create(PA(*[e._h for e in self.engines]), len(self.engines),
                                         C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_replicas_destroy(self._h)
            self._h = None
        for e in getattr(self, "engines", []):
            e.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __len__(self):
        return len(self.engines)

    def lookup_ptrs(self, keys_ptrs, ns, out_ptrs, flags_ptrs, mem: int = HPS_MEM_HOST):
        g = len(self.engines)
        PA = C.c_void_p * g
        outs = (_Outcome * g)()
        _check(lib().hps_replicas_lookup(self._h, PA(*keys_ptrs), (C.c_size_t * g)(*ns),
                                         PA(*out_ptrs), PA(*flags_ptrs), outs, mem))
        return [LookupOutcome(bool(o.sync_branch), float(o.unique_hit_rate), int(o.unique_count),
                              int(o.defaults_returned)) for o in outs]

    def lookup(self, batches) -> List[LookupResult]:
        """batches[r] = replica r's keys; returns one LookupResult each."""
        ks = [_u64(b) for b in batches]
        d = self.table.dimension
        outs = [np.empty(max(len(k), 1) * d, dtype=np.float32) for k in ks]
        fls = [np.empty(max(len(k), 1), dtype=np.uint8) for k in ks]
        self.lookup_ptrs([k.ctypes.data for k in ks], [len(k) for k in ks],
                         [o.ctypes.data for o in outs], [f.ctypes.data for f in fls])
        return [LookupResult(d, o[: len(k) * d], f[: len(k)]) for k, o, f in zip(ks, outs, fls)]


class MultiLookup:
    """hps_multi_*: one lookup of several tables (engines whose caches form one
    cache group) with one H2D, one kernel launch, one D2H and one host wait;
    per-table semantics of LookupEngine.lookup."""

    def __init__(self, engines: Sequence["LookupEngine"], max_batch: int):
        self.engines = list(engines)
        self._h = C.c_void_p()
        t = len(self.engines)
        _check(lib().hps_multi_create((C.c_void_p * t)(*[e._h for e in self.engines]), t,
                                      max_batch, C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup_ptrs(self, keys_ptrs, ns, out_ptrs, flags_ptrs) -> List[LookupOutcome]:
        t = len(self.engines)
        PA = C.c_void_p * t
        outs = (_Outcome * t)()
        _check(lib().hps_multi_lookup(self._h, PA(*keys_ptrs), (C.c_size_t * t)(*ns),
                                      PA(*out_ptrs), PA(*flags_ptrs), outs))
        return [LookupOutcome(bool(o.sync_branch), float(o.unique_hit_rate), int(o.unique_count),
                              int(o.defaults_returned)) for o in outs]

    def lookup(self, keys_per_table) -> List["LookupResult"]:
        ks = [_u64(k) for k in keys_per_table]
        res = [LookupResult(e.table.dimension, np.zeros(len(k) * e.table.dimension, np.float32),
                            np.zeros(len(k), np.uint8)) for e, k in zip(self.engines, ks)]
        self.lookup_ptrs([k.ctypes.data for k in ks], [len(k) for k in ks],
                         [r.vectors.ctypes.data for r in res], [r.miss_flags.ctypes.data for r in res])
        return res


def wire_lookup_frame(rows, miss_flags, dim: int) -> bytes:
    """hps_wire_lookup_frame on host arrays: the reference's LOOKUP response
    frame (wire.cpp:174-188), byte-exact."""
    r = _f32(rows)
    f = np.ascontiguousarray(miss_flags, dtype=np.uint8)
    count = len(f)
    n = C.c_size_t(0)
    _check(lib().hps_wire_lookup_frame(0, None, None, count, dim, HPS_MEM_HOST, None, 0,
                                       C.byref(n), None))
    buf = np.empty(n.value, dtype=np.uint8)
    _check(lib().hps_wire_lookup_frame(0, _ptr(r), _ptr(f), count, dim, HPS_MEM_HOST, _ptr(buf),
                                       buf.size, C.byref(n), None))
    return buf.tobytes()


def wire_lookup_frame_device(rows_ptr: int, flags_ptr: int, count: int, dim: int, frame_ptr: int,
                             cap: int, device: int = 0, stream: int = 0) -> int:
    """Device-mode frame (rows / flags in HBM, frame ideally pinned); returns
    the frame length."""
    n = C.c_size_t(0)
    _check(lib().hps_wire_lookup_frame(device, rows_ptr, flags_ptr, count, dim, HPS_MEM_DEVICE,
                                       frame_ptr, cap, C.byref(n), stream or None))
    return n.value


def bench_draw_seed(seed: int) -> int:
    """bench.cpp:33-35"""
    return (seed ^ 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
