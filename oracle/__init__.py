"""Parity oracle for the B200 lookup path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package, and only as the checker
or the timed CPU baseline; the product path (paper_2210_08804_b200) never
imports it.

* ``OracleCache`` -- ctypes over liboracle.so, the C restatement of the
  reference cache (hps_oracle.c; file:line citations there).
* ``EngineOracle`` -- pure-Python restatement of LookupEngine::lookup
  (lookup_engine.cpp:130-241) and tier_fetch (:50-89) over OracleCache and a
  dict VDB; for small cases.
* ``RefCache`` / ``RefModel`` / ``RefEngine`` / ``ref_*`` -- the UNMODIFIED
  reference compiled from its own sources into _ref/libhps_ref.so
  (Makefile), used to pin the restatement and as the CPU baseline.

Parity status: pinned (see hps_oracle.c header and tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path
from typing import List, Optional

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libhps_ref.so"
# the reference's tests/unit/test_slab_cache.cpp built against include/hps/slab_cache.hpp
REF_CACHE_TEST = HERE / "_ref" / "test_slab_cache_b200"
# tests/unit/test_lookup_engine.cpp built against include/hps/lookup_engine.hpp
REF_ENGINE_TEST = HERE / "_ref" / "test_lookup_engine_b200"
# tests/unit/test_refresh_engine.cpp + the reference's refresh_engine.cpp over the B200 cache
REF_REFRESH_TEST = HERE / "_ref" / "test_refresh_engine_b200"
# tests/unit/test_volatile_store.cpp built against include/hps/volatile_store.hpp
REF_VDB_TEST = HERE / "_ref" / "test_volatile_store_b200"
# the reference's acceptance suite (c1-c10) against the B200 cache + engine
REF_ACCEPTANCE = HERE / "_ref" / "acceptance_b200"
REF_SRC = Path("/root/reference/proj")

_P = C.c_void_p
_SZ = C.c_size_t


def build(quiet: bool = True) -> None:
    """Builds liboracle.so and (when the reference sources are present)
    _ref/libhps_ref.so."""
    subprocess.run(["make", "-C", str(HERE)], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


_olib = None
_rlib = None


def olib() -> C.CDLL:
    global _olib
    if _olib is None:
        if not ORACLE_SO.exists():
            build()
        l = C.CDLL(str(ORACLE_SO))
        l.orc_xxh64.restype = C.c_uint64
        l.orc_xxh64.argtypes = [_P, _SZ, C.c_uint64]
        l.orc_xxh64_key.restype = C.c_uint64
        l.orc_xxh64_key.argtypes = [C.c_uint64, C.c_uint64]
        l.orc_slabset_of.restype = C.c_uint64
        l.orc_slabset_of.argtypes = [C.c_uint64, C.c_uint64]
        l.orc_first_slab_of.restype = C.c_uint32
        l.orc_first_slab_of.argtypes = [C.c_uint64, C.c_uint32]
        l.orc_partition_of.restype = C.c_uint32
        l.orc_partition_of.argtypes = [C.c_uint64, C.c_uint32]
        l.orc_dedup.restype = _SZ
        l.orc_dedup.argtypes = [_P, _SZ, _P, _P]
        l.orc_cache_create.restype = _P
        l.orc_cache_create.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        l.orc_cache_destroy.argtypes = [_P]
        l.orc_cache_clock.restype = C.c_uint64
        l.orc_cache_clock.argtypes = [_P]
        l.orc_cache_occupied.restype = _SZ
        l.orc_cache_occupied.argtypes = [_P]
        l.orc_cache_query.argtypes = [_P, _P, _SZ, _P, _P]
        l.orc_cache_replace.restype = C.c_int
        l.orc_cache_replace.argtypes = [_P, _P, _SZ, _P]
        l.orc_cache_update.restype = _SZ
        l.orc_cache_update.argtypes = [_P, _P, _SZ, _P]
        l.orc_cache_dump.restype = _SZ
        l.orc_cache_dump.argtypes = [_P, C.c_uint64, C.c_uint64, _P, _SZ]
        l.orc_cache_state.argtypes = [_P, _P, _P, _P, _P]
        l.orc_powerlaw_sample.restype = C.c_int
        l.orc_powerlaw_sample.argtypes = [C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, _SZ, _P]
        l.orc_mt64_first.restype = C.c_uint64
        l.orc_mt64_first.argtypes = [C.c_uint64, _SZ]
        _olib = l
    return _olib


def ref_available() -> bool:
    return REF_SO.exists()


def rlib() -> C.CDLL:
    global _rlib
    if _rlib is None:
        if not REF_SO.exists():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference sources)")
        l = C.CDLL(str(REF_SO))
        l.ref_last_error.restype = C.c_char_p
        l.ref_wire_lookup_frame.restype = _SZ
        l.ref_wire_lookup_frame.argtypes = [_P, _P, C.c_uint32, C.c_uint32, _P, _SZ]
        l.ref_pdb_open.argtypes = [C.c_char_p, C.POINTER(_P)]
        l.ref_pdb_destroy.argtypes = [_P]
        l.ref_pdb_create_table.argtypes = [_P, C.c_char_p, C.c_uint32]
        l.ref_pdb_put.argtypes = [_P, C.c_char_p, _P, _SZ, _P]
        l.ref_pdb_flush.argtypes = [_P, C.c_char_p]
        l.ref_pdb_compact.argtypes = [_P, C.c_char_p]
        l.ref_pdb_get.argtypes = [_P, C.c_char_p, _P, _SZ, _P, _P, C.POINTER(_SZ), _P,
                                  C.POINTER(_SZ)]
        l.ref_pdb_segment_count.restype = _SZ
        l.ref_pdb_segment_count.argtypes = [_P, C.c_char_p]
        l.ref_pdb_key_count.restype = _SZ
        l.ref_pdb_key_count.argtypes = [_P, C.c_char_p]
        l.ref_xxh64.restype = C.c_uint64
        l.ref_xxh64.argtypes = [_P, _SZ, C.c_uint64]
        l.ref_xxh64_key.restype = C.c_uint64
        l.ref_xxh64_key.argtypes = [C.c_uint64, C.c_uint64]
        l.ref_partition_of.restype = C.c_uint32
        l.ref_partition_of.argtypes = [C.c_uint64, C.c_uint32]
        l.ref_dedup.restype = _SZ
        l.ref_dedup.argtypes = [_P, _SZ, _P, _P]
        l.ref_cache_create.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.POINTER(_P)]
        l.ref_cache_destroy.argtypes = [_P]
        l.ref_cache_query.argtypes = [_P, _P, _SZ, _P, _SZ, _P, _P, C.POINTER(_SZ)]
        l.ref_cache_replace.argtypes = [_P, _P, _SZ, _P, _SZ]
        l.ref_cache_update.argtypes = [_P, _P, _SZ, _P, _SZ, C.POINTER(_SZ)]
        l.ref_cache_dump_all.restype = _SZ
        l.ref_cache_dump_all.argtypes = [_P, _P, _SZ]
        l.ref_cache_clock.restype = C.c_uint64
        l.ref_cache_clock.argtypes = [_P]
        l.ref_cache_occupied.restype = _SZ
        l.ref_cache_occupied.argtypes = [_P]
        l.ref_cache_check.argtypes = [_P]
        l.ref_model_create.restype = _P
        l.ref_model_create.argtypes = [C.c_uint64, C.c_uint32, C.c_uint32]
        l.ref_model_destroy.argtypes = [_P]
        l.ref_model_query.argtypes = [_P, _P, _SZ, _P, _SZ, _P]
        l.ref_model_replace.argtypes = [_P, _P, _SZ, _P, _SZ]
        l.ref_model_update.restype = _SZ
        l.ref_model_update.argtypes = [_P, _P, _SZ, _P, _SZ]
        l.ref_model_resident.restype = _SZ
        l.ref_model_resident.argtypes = [_P, _P, _SZ]
        l.ref_model_clock.restype = C.c_uint64
        l.ref_model_clock.argtypes = [_P]
        l.ref_powerlaw_sample.argtypes = [C.c_double, C.c_uint64, C.c_uint64, C.c_uint64, _SZ, _P]
        l.ref_engine_create.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32,
                                        C.c_double, C.c_uint32, C.c_int, _P, C.c_uint32,
                                        C.c_uint32, C.c_uint32, C.POINTER(_P)]
        l.ref_engine_destroy.argtypes = [_P]
        l.ref_engine_vdb_insert.argtypes = [_P, _P, _SZ, _P]
        l.ref_engine_pdb_put.argtypes = [_P, _P, _SZ, _P]
        l.ref_engine_cache_replace.argtypes = [_P, _P, _SZ, _P]
        l.ref_engine_lookup.argtypes = [_P, _P, _SZ, _P, _P, _P, C.POINTER(C.c_double)]
        l.ref_engine_drain.argtypes = [_P]
        l.ref_engine_stats.argtypes = [_P, _P]
        l.ref_engine_cache.restype = _P
        l.ref_engine_cache.argtypes = [_P]
        l.ref_hw_threads.restype = C.c_uint
        _rlib = l
    return _rlib


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64).reshape(-1))


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(-1))


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ------------------------------------------------------------- restatement --
def xxh64(data: bytes, seed: int = 0) -> int:
    b = C.create_string_buffer(bytes(data), len(data))
    return int(olib().orc_xxh64(b, len(data), seed))


def xxh64_key(key: int, seed: int) -> int:
    return int(olib().orc_xxh64_key(key, seed))


def slabset_of(key: int, S: int) -> int:
    return int(olib().orc_slabset_of(key, S))


def first_slab_of(key: int, W: int) -> int:
    return int(olib().orc_first_slab_of(key, W))


def partition_of(key: int, P: int) -> int:
    return int(olib().orc_partition_of(key, P))


def dedup(keys):
    k = _u64(keys)
    u = np.empty(max(len(k), 1), dtype=np.uint64)
    inv = np.empty(max(len(k), 1), dtype=np.uint32)
    n = olib().orc_dedup(_p(k), len(k), _p(u), _p(inv))
    return u[:n].copy(), inv[: len(k)].copy()


def powerlaw_sample(alpha, keyspace, permute_seed, draw_seed, count) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    rc = olib().orc_powerlaw_sample(alpha, keyspace, permute_seed, draw_seed, count, _p(out))
    if rc:
        raise ValueError("bad sampler spec")
    return out


class OracleCache:
    """C restatement of the slot-exact cache model."""

    def __init__(self, S: int, W: int, d: int):
        self.S, self.W, self.d = S, W, d
        self._h = olib().orc_cache_create(S, W, d)
        if not self._h:
            raise ValueError("bad geometry")

    def __del__(self):
        if getattr(self, "_h", None):
            olib().orc_cache_destroy(self._h)
            self._h = None

    def query(self, keys, out: np.ndarray) -> np.ndarray:
        """clock++; hit rows into out (in place); returns u8 hit flags."""
        k = _u64(keys)
        hit = np.zeros(max(len(k), 1), dtype=np.uint8)
        olib().orc_cache_query(self._h, _p(k), len(k), _p(out), _p(hit))
        return hit[: len(k)]

    def replace(self, keys, vectors) -> bool:
        """False (and no mutation) on duplicate keys."""
        k = _u64(keys)
        v = _f32(vectors)
        return olib().orc_cache_replace(self._h, _p(k), len(k), _p(v)) == 0

    def update(self, keys, vectors) -> int:
        k = _u64(keys)
        v = _f32(vectors)
        return int(olib().orc_cache_update(self._h, _p(k), len(k), _p(v)))

    def dump(self, set_begin: int = 0, set_end: Optional[int] = None) -> np.ndarray:
        set_end = self.S if set_end is None else set_end
        cap = (set_end - set_begin) * self.W * 32
        out = np.empty(max(cap, 1), dtype=np.uint64)
        n = olib().orc_cache_dump(self._h, set_begin, set_end, _p(out), cap)
        return out[:n].copy()

    def clock(self) -> int:
        return int(olib().orc_cache_clock(self._h))

    def occupied(self) -> int:
        return int(olib().orc_cache_occupied(self._h))

    def state(self):
        cap = self.S * self.W * 32
        keys = np.empty(cap, dtype=np.uint64)
        ctr = np.empty(cap, dtype=np.uint64)
        masks = np.empty(self.S * self.W, dtype=np.uint32)
        rows = np.empty(cap * self.d, dtype=np.float32)
        olib().orc_cache_state(self._h, _p(keys), _p(ctr), _p(masks), _p(rows))
        return keys, ctr, masks, rows


class EngineOracle:
    """Python restatement of LookupEngine::lookup (lookup_engine.cpp:130-241)
    with tier_fetch (:50-89) over a dict VDB and a dict cold tier. Async
    fills are applied on drain_async() in submission order (the reference's
    background timing is nondeterministic; tests drain after each lookup)."""

    def __init__(self, S, W, d, threshold=0.8, default_vector=(), vdb_enabled=True):
        self.cache = OracleCache(S, W, d)
        self.d = d
        self.threshold = threshold
        dv = list(default_vector)[:d]
        self.default = np.array(dv + [0.0] * (d - len(dv)), dtype=np.float32)
        self.vdb = {}
        self.cold = {}
        self.vdb_enabled = vdb_enabled
        self.pending: List[np.ndarray] = []
        self.stats = dict(queries=0, queried_keys=0, unique_keys=0, cache_hits=0, cache_misses=0,
                          sync_batches=0, async_batches=0, defaults_returned=0, vdb_hits=0,
                          pdb_hits=0, tier_missing=0, async_faults=0)

    def tier_fetch(self, keys, counters):
        found_k, found_v, remaining = [], [], []
        for k in keys:
            k = int(k)
            if self.vdb_enabled and k in self.vdb:
                found_k.append(k)
                found_v.append(self.vdb[k])
            else:
                remaining.append(k)
        counters["vdb_hits"] += len(found_k)
        missing = []
        promote = []
        for k in remaining:
            if k in self.cold:
                found_k.append(k)
                found_v.append(self.cold[k])
                counters["pdb_hits"] += 1
                promote.append(k)
            else:
                missing.append(k)
                counters["missing"] += 1
        if self.vdb_enabled:
            for k in promote:
                self.vdb[k] = self.cold[k]
        return found_k, found_v, missing

    def lookup(self, keys):
        keys = _u64(keys)
        d = self.d
        uniq, inv = dedup(keys)
        nu = len(uniq)
        ws = np.zeros(nu * d, dtype=np.float32)
        hit = self.cache.query(uniq, ws)
        miss_rows = np.nonzero(hit == 0)[0]
        misses = uniq[miss_rows]
        h = 1.0 if nu == 0 else 1.0 - len(misses) / nu
        sync = h < self.threshold
        udef = np.zeros(nu, dtype=np.uint8)
        c = dict(vdb_hits=0, pdb_hits=0, missing=0)
        defaults = 0
        if sync:
            fk, fv, mk = self.tier_fetch(misses, c)
            row_of = {int(k): int(r) for k, r in zip(misses, miss_rows)}
            for k, v in zip(fk, fv):
                ws[row_of[k] * d:(row_of[k] + 1) * d] = v
            for k in mk:
                r = row_of[k]
                ws[r * d:(r + 1) * d] = self.default
                udef[r] = 1
                defaults += 1
            if fk:
                self.cache.replace(np.array(fk, dtype=np.uint64),
                                   np.concatenate(fv).astype(np.float32))
        else:
            for r in miss_rows:
                ws[r * d:(r + 1) * d] = self.default
                udef[r] = 1
                defaults += 1
        out = ws.reshape(max(nu, 1), d)[inv].reshape(-1) if len(keys) else np.empty(0, np.float32)
        flags = udef[inv] if len(keys) else np.empty(0, np.uint8)
        s = self.stats
        s["queries"] += 1
        s["queried_keys"] += len(keys)
        s["unique_keys"] += nu
        s["cache_hits"] += nu - len(misses)
        s["cache_misses"] += len(misses)
        s["defaults_returned"] += defaults
        if sync:
            s["sync_batches"] += 1
            s["vdb_hits"] += c["vdb_hits"]
            s["pdb_hits"] += c["pdb_hits"]
            s["tier_missing"] += c["missing"]
        else:
            s["async_batches"] += 1
            if len(misses):
                self.pending.append(misses.copy())
        outcome = dict(sync_branch=sync, unique_hit_rate=h, unique_count=nu,
                       defaults_returned=defaults)
        return out, flags, outcome

    def drain_async(self):
        for misses in self.pending:
            c = dict(vdb_hits=0, pdb_hits=0, missing=0)
            fk, fv, _ = self.tier_fetch(misses, c)
            if fk:
                self.cache.replace(np.array(fk, dtype=np.uint64),
                                   np.concatenate(fv).astype(np.float32))
            self.stats["vdb_hits"] += c["vdb_hits"]
            self.stats["pdb_hits"] += c["pdb_hits"]
            self.stats["tier_missing"] += c["missing"]
        self.pending = []


# ------------------------------------------------------ reference (as-is) --
def _rcheck(rc):
    if rc == 1:
        raise ValueError(rlib().ref_last_error().decode())
    if rc:
        raise RuntimeError(rlib().ref_last_error().decode())


class RefCache:
    """The reference hps::SlabCache itself."""

    def __init__(self, S, W, d, workers=1, tasks_per_worker=8):
        self.d = d
        self._h = C.c_void_p()
        _rcheck(rlib().ref_cache_create(S, W, d, workers, tasks_per_worker, C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().ref_cache_destroy(self._h)
            self._h = None

    def query(self, keys, out: np.ndarray):
        k = _u64(keys)
        pos = np.empty(max(len(k), 1), dtype=np.uint64)
        mk = np.empty(max(len(k), 1), dtype=np.uint64)
        nm = C.c_size_t(0)
        _rcheck(rlib().ref_cache_query(self._h, _p(k), len(k), _p(out), out.size, _p(pos), _p(mk),
                                       C.byref(nm)))
        return pos[: nm.value].copy(), mk[: nm.value].copy()

    def replace(self, keys, vectors):
        k = _u64(keys)
        v = _f32(vectors)
        _rcheck(rlib().ref_cache_replace(self._h, _p(k), len(k), _p(v), v.size))

    def update(self, keys, vectors) -> int:
        k = _u64(keys)
        v = _f32(vectors)
        w = C.c_size_t(0)
        _rcheck(rlib().ref_cache_update(self._h, _p(k), len(k), _p(v), v.size, C.byref(w)))
        return w.value

    def dump_all(self) -> np.ndarray:
        n = rlib().ref_cache_dump_all(self._h, None, 0)
        out = np.empty(max(n, 1), dtype=np.uint64)
        n = rlib().ref_cache_dump_all(self._h, _p(out), n)
        return out[:n].copy()

    def clock(self) -> int:
        return int(rlib().ref_cache_clock(self._h))

    def occupied(self) -> int:
        return int(rlib().ref_cache_occupied(self._h))

    def check_invariants(self):
        _rcheck(rlib().ref_cache_check(self._h))


class RefModel:
    """The reference's own slot-exact test model (reference_cache.hpp)."""

    def __init__(self, S, W, d):
        self._h = rlib().ref_model_create(S, W, d)

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().ref_model_destroy(self._h)
            self._h = None

    def query(self, keys, out):
        k = _u64(keys)
        hit = np.zeros(max(len(k), 1), dtype=np.uint8)
        rlib().ref_model_query(self._h, _p(k), len(k), _p(out), out.size, _p(hit))
        return hit[: len(k)]

    def replace(self, keys, vectors):
        k = _u64(keys)
        v = _f32(vectors)
        rlib().ref_model_replace(self._h, _p(k), len(k), _p(v), v.size)

    def update(self, keys, vectors):
        k = _u64(keys)
        v = _f32(vectors)
        return int(rlib().ref_model_update(self._h, _p(k), len(k), _p(v), v.size))

    def resident(self):
        n = rlib().ref_model_resident(self._h, None, 0)
        out = np.empty(max(n, 1), dtype=np.uint64)
        rlib().ref_model_resident(self._h, _p(out), n)
        return out[:n].copy()

    def clock(self):
        return int(rlib().ref_model_clock(self._h))


class RefEngine:
    """The reference LookupEngine over its VolatileStore (+ empty PDB)."""

    def __init__(self, dim, S, W=2, workers=2, threshold=0.8, partitions=16, use_vdb=True,
                 default_vector=(), pool=16, async_workers=2):
        self.d = dim
        dv = _f32(list(default_vector))
        self._h = C.c_void_p()
        _rcheck(rlib().ref_engine_create(dim, S, W, workers, threshold, partitions,
                                         1 if use_vdb else 0, _p(dv) if dv.size else None,
                                         dv.size, pool, async_workers, C.byref(self._h)))

    def __del__(self):
        if getattr(self, "_h", None):
            rlib().ref_engine_destroy(self._h)
            self._h = None

    def vdb_insert(self, keys, vectors):
        k = _u64(keys)
        v = _f32(vectors)
        _rcheck(rlib().ref_engine_vdb_insert(self._h, _p(k), len(k), _p(v)))

    def pdb_put(self, keys, vectors):
        k = _u64(keys)
        v = _f32(vectors)
        _rcheck(rlib().ref_engine_pdb_put(self._h, _p(k), len(k), _p(v)))

    def cache_replace(self, keys, vectors):
        k = _u64(keys)
        v = _f32(vectors)
        _rcheck(rlib().ref_engine_cache_replace(self._h, _p(k), len(k), _p(v)))

    def lookup(self, keys):
        k = _u64(keys)
        out = np.empty(max(len(k), 1) * self.d, dtype=np.float32)
        flags = np.empty(max(len(k), 1), dtype=np.uint8)
        oc = np.zeros(3, dtype=np.uint64)
        h = C.c_double(0)
        _rcheck(rlib().ref_engine_lookup(self._h, _p(k), len(k), _p(out), _p(flags), _p(oc),
                                         C.byref(h)))
        outcome = dict(sync_branch=bool(oc[0]), unique_hit_rate=h.value,
                       unique_count=int(oc[1]), defaults_returned=int(oc[2]))
        return out[: len(k) * self.d], flags[: len(k)], outcome

    def drain(self):
        rlib().ref_engine_drain(self._h)

    def stats(self):
        s = np.zeros(12, dtype=np.uint64)
        rlib().ref_engine_stats(self._h, _p(s))
        names = ["queries", "queried_keys", "unique_keys", "cache_hits", "cache_misses",
                 "sync_batches", "async_batches", "defaults_returned", "vdb_hits", "pdb_hits",
                 "tier_missing", "async_faults"]
        return {n: int(v) for n, v in zip(names, s)}


def ref_powerlaw_sample(alpha, keyspace, permute_seed, draw_seed, count) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    _rcheck(rlib().ref_powerlaw_sample(alpha, keyspace, permute_seed, draw_seed, count, _p(out)))
    return out


def ref_xxh64(data: bytes, seed: int = 0) -> int:
    b = C.create_string_buffer(bytes(data), len(data))
    return int(rlib().ref_xxh64(b, len(data), seed))


def ref_wire_lookup_frame(rows, flags, dim: int) -> bytes:
    r = _f32(rows)
    f = np.ascontiguousarray(flags, dtype=np.uint8)
    cap = 13 + r.size * 4 + (len(f) + 7) // 8
    out = np.empty(max(cap, 1), dtype=np.uint8)
    n = rlib().ref_wire_lookup_frame(_p(r), _p(f), len(f), dim, _p(out), out.size)
    return out[:n].tobytes()


def ref_dedup(keys):
    k = _u64(keys)
    u = np.empty(max(len(k), 1), dtype=np.uint64)
    inv = np.empty(max(len(k), 1), dtype=np.uint32)
    n = rlib().ref_dedup(_p(k), len(k), _p(u), _p(inv))
    return u[:n].copy(), inv[: len(k)].copy()


class RefPersistentStore:
    """The reference's own hps::PersistentStore (oracle/_ref) -- the writer of
    the segment files and the parity partner of the native batched reader."""

    def __init__(self, root):
        self._h = C.c_void_p()
        _rcheck(rlib().ref_pdb_open(str(root).encode(), C.byref(self._h)))

    def close(self):
        if self._h:
            rlib().ref_pdb_destroy(self._h)
            self._h = None

    def create_table(self, name, dim):
        _rcheck(rlib().ref_pdb_create_table(self._h, name.encode(), dim))
        self.dims = getattr(self, "dims", {})
        self.dims[name] = dim

    def put(self, name, keys, rows):
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        v = np.ascontiguousarray(rows, dtype=np.float32)
        _rcheck(rlib().ref_pdb_put(self._h, name.encode(), k.ctypes.data, len(k), v.ctypes.data))

    def flush(self, name):
        _rcheck(rlib().ref_pdb_flush(self._h, name.encode()))

    def compact(self, name):
        _rcheck(rlib().ref_pdb_compact(self._h, name.encode()))

    def segment_count(self, name):
        return rlib().ref_pdb_segment_count(self._h, name.encode())

    def key_count(self, name):
        return rlib().ref_pdb_key_count(self._h, name.encode())

    def get(self, name, keys, dim):
        k = np.ascontiguousarray(keys, dtype=np.uint64)
        n = len(k)
        fk = np.empty(max(n, 1), np.uint64)
        fv = np.empty(max(n, 1) * dim, np.float32)
        mk = np.empty(max(n, 1), np.uint64)
        nf, nm = _SZ(0), _SZ(0)
        _rcheck(rlib().ref_pdb_get(self._h, name.encode(), k.ctypes.data, n, fk.ctypes.data,
                                   fv.ctypes.data, C.byref(nf), mk.ctypes.data, C.byref(nm)))
        return fk[: nf.value].copy(), fv[: nf.value * dim].copy(), mk[: nm.value].copy()
