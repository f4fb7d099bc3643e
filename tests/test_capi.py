"""CPU: the C-ABI library loads and exports every symbol include/hps_b200.h
declares; host-only pieces (hashes, sampler, the volatile DB and tier_fetch)
behave like the reference (test_volatile_store.cpp, test_lookup_engine.cpp
:53-93). No GPU compute is called here."""
import re
from pathlib import Path

import numpy as np
import pytest

import oracle
import paper_2210_08804_b200 as hps

ROOT = Path(__file__).resolve().parent.parent


def test_library_exports_every_declared_symbol():
    header = (ROOT / "include" / "hps_b200.h").read_text()
    declared = set(re.findall(r"\b(hps_[a-z0-9_]+)\s*\(", header))
    declared -= {"hps_cold_fetch_fn"}
    assert len(declared) >= 38
    l = hps.lib()
    for name in sorted(declared):
        assert hasattr(l, name), name
    assert set(hps.SIGNATURES) == declared


def test_product_host_hashes_match_oracle():
    rng = np.random.default_rng(1)
    for k in rng.integers(0, 2**64 - 1, 300, dtype=np.uint64):
        k = int(k)
        for s in (0, hps.kSlabsetSeed, hps.kSlabSeed):
            assert hps.xxh64_key(k, s) == oracle.xxh64_key(k, s)
        assert hps.SlabCache.slabset_of(k, 977) == oracle.slabset_of(k, 977)
        assert hps.SlabCache.first_slab_of(k, 4) == oracle.first_slab_of(k, 4)
        assert hps.partition_of(k, 7) == oracle.partition_of(k, 7)
    assert hps.partition_of(0, 16) == 11
    for data in (b"", b"abc", bytes(range(37)), bytes(range(100)), bytes(range(255)) * 3):
        for s in (0, 1, 0x51AB):
            assert hps.xxh64(data, s) == oracle.xxh64(data, s)


def rows(keys, dim, salt=0.0):
    # test_volatile_store.cpp:16-25
    return np.array([[float(k) + salt + 0.125 * c for c in range(dim)] for k in keys],
                    dtype=np.float32).reshape(-1)


T = hps.TableId


def test_vdb_register_insert_lookup_round_trip():
    vdb = hps.VolatileStore()
    vdb.register_table(T("t", 2), hps.VolatileTableConfig(partition_count=4, overflow_margin=100))
    assert vdb.has_table("t") and not vdb.has_table("other")
    assert vdb.partition_count("t") == 4
    keys = [1, 2, 3]
    assert len(vdb.insert("t", keys, rows(keys, 2))) == 0
    assert vdb.table_size("t") == 3
    for k in keys:
        assert vdb.partition_size("t", hps.partition_of(k, 4)) >= 1
    r = vdb.lookup("t", [2, 9, 1])
    assert r.found_keys.tolist() == [2, 1]
    assert r.missing_keys.tolist() == [9]
    assert r.found_vectors.size == 4 and r.found_vectors[0] == 2.0 and r.found_vectors[2] == 1.0


def test_vdb_reregister_and_bad_input():
    vdb = hps.VolatileStore()
    vdb.register_table(T("t", 8))
    vdb.register_table(T("t", 8))
    with pytest.raises(hps.InvalidArgument):
        vdb.register_table(T("t", 16))
    vdb.register_table(T("u", 2))
    with pytest.raises(hps.InvalidArgument):
        vdb.lookup("nope", [1])
    with pytest.raises(hps.InvalidArgument):
        vdb.insert("u", [1], [1.0])  # wrong buffer size
    with pytest.raises(hps.InvalidArgument):
        vdb.insert("u", [1], [1.0, float("nan")])
    assert vdb.table_size("u") == 0
    with pytest.raises(hps.InvalidArgument):
        vdb.register_table(T("", 2))
    with pytest.raises(hps.InvalidArgument):
        vdb.register_table(T("z", 2), hps.VolatileTableConfig(partition_count=0))


def test_vdb_clock_once_per_call():
    vdb = hps.VolatileStore()
    vdb.register_table(T("t", 1), hps.VolatileTableConfig(partition_count=2))
    assert vdb.table_clock("t") == 0
    vdb.insert("t", [1, 2, 3, 4], rows([1, 2, 3, 4], 1))
    assert vdb.table_clock("t") == 1
    vdb.lookup("t", [1, 2, 3, 4])
    assert vdb.table_clock("t") == 2
    vdb.lookup("t", [999])
    assert vdb.table_clock("t") == 3


def test_vdb_refresh_is_monotone():
    vdb = hps.VolatileStore()
    vdb.register_table(T("t", 1), hps.VolatileTableConfig(partition_count=1))
    vdb.insert("t", [5, 6], rows([5, 6], 1))
    assert vdb.last_access("t", 5) == 1
    vdb.lookup("t", [5])
    vdb.drain()
    assert vdb.last_access("t", 5) == 2
    assert vdb.last_access("t", 6) == 1
    assert vdb.last_access("t", 7) is None
    vdb2 = hps.VolatileStore()
    vdb2.register_table(T("t", 1), hps.VolatileTableConfig(partition_count=1))
    vdb2.insert("t", [5], rows([5], 1))
    vdb2.lookup("t", [5])
    vdb2.insert("t", [5], rows([5], 1, 0.5))
    vdb2.drain()
    assert vdb2.last_access("t", 5) == 3


def test_vdb_evicts_oldest_beyond_margin_with_key_tie_break():
    vdb = hps.VolatileStore()
    vdb.register_table(T("t", 1), hps.VolatileTableConfig(partition_count=1, overflow_margin=3))
    vdb.insert("t", [10, 11], rows([10, 11], 1))      # clock 1
    vdb.insert("t", [12], rows([12], 1))              # clock 2
    vdb.lookup("t", [10])                             # 10 -> 3
    ev = vdb.insert("t", [13, 14], rows([13, 14], 1))  # clock 4, 5 entries > 3
    # oldest: 11 (1), 12 (2); then 10 (3)
    assert ev.tolist() == [11, 12]
    assert vdb.table_size("t") == 3
    # ties broken by the smaller key
    vdb2 = hps.VolatileStore()
    vdb2.register_table(T("t", 1), hps.VolatileTableConfig(partition_count=1, overflow_margin=2))
    ev = vdb2.insert("t", [9, 4, 7, 1], rows([9, 4, 7, 1], 1))
    assert ev.tolist() == [1, 4]


def test_vdb_matches_reference_partitioned_lookup_order():
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built")
    d = 4
    vdb = hps.VolatileStore(4)
    vdb.register_table(T("t", d), hps.VolatileTableConfig(partition_count=16))
    ref = oracle.RefEngine(d, S=4, partitions=16)
    rng = np.random.default_rng(3)
    keys = rng.choice(100000, 20000, replace=False).astype(np.uint64)
    v = rng.standard_normal(len(keys) * d).astype(np.float32)
    vdb.insert("t", keys, v)
    q = rng.integers(0, 100000, 50000, dtype=np.uint64)
    r = vdb.lookup("t", q)
    present = set(keys.tolist())
    want_found = [k for k in q.tolist() if k in present]
    assert r.found_keys.tolist() == want_found
    assert r.missing_keys.tolist() == [k for k in q.tolist() if k not in present]
    row_of = {int(k): i for i, k in enumerate(keys)}
    got = r.found_vectors.reshape(-1, d)
    idx = np.array([row_of[k] for k in want_found])
    assert np.array_equal(got, v.reshape(-1, d)[idx])


def test_tier_fetch_reads_volatile_first_then_cold_then_promotes():
    """test_lookup_engine.cpp:53-93 with a dict cold tier."""
    vdb = hps.VolatileStore()
    table = T("t", 1)
    vdb.register_table(table, hps.VolatileTableConfig(partition_count=2))
    pdb = hps.DictStore(1)
    pdb.put([1], [100.0])
    pdb.put([2], [200.0])
    vdb.insert("t", [1], [111.0])
    c = {}
    r = hps.tier_fetch(table, [1, 2, 3], vdb, pdb, c)
    assert r.found_keys.tolist() == [1, 2]
    assert r.found_vectors.tolist() == [111.0, 200.0]
    assert r.missing_keys.tolist() == [3]
    assert c == {"vdb_hits": 1, "pdb_hits": 1, "missing": 1}
    vdb.drain()
    p = vdb.lookup("t", [2])
    assert p.found_keys.tolist() == [2] and p.found_vectors.tolist() == [200.0]
    c2 = {}
    r2 = hps.tier_fetch(table, [1, 2], None, pdb, c2)
    assert r2.found_vectors.tolist() == [100.0, 200.0]
    assert c2 == {"vdb_hits": 0, "pdb_hits": 2, "missing": 0}
    r3 = hps.tier_fetch(table, [], vdb, pdb)
    assert len(r3.found_keys) == 0 and len(r3.missing_keys) == 0


def test_cache_without_gpu_fails_loudly():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises((hps.HpsError, hps.OutOfMemory)):
        hps.SlabCache(hps.SlabCacheConfig(slabset_count=4, slabs_per_set=2, dimension=4))


def test_cache_config_validation_precedes_device_use():
    for cfg in (hps.SlabCacheConfig(slabset_count=0, dimension=4),
                hps.SlabCacheConfig(slabset_count=1, slabs_per_set=0, dimension=4),
                hps.SlabCacheConfig(slabset_count=1, dimension=0),
                hps.SlabCacheConfig(slabset_count=1, dimension=4, worker_pool_size=0)):
        with pytest.raises(hps.InvalidArgument):
            hps.SlabCache(cfg)


def test_vdb_parallel_lookups_from_several_threads():
    """Large lookups fan out over the store's thread pool (chunks of >= 512
    keys); several caller threads at once (the engine's async fill next to a
    sync-branch fetch) share that pool. Every result must be exact -- a
    regression guard for the pool's completion countdown, which once let a
    caller return while the last worker was still signalling it."""
    import threading

    d = 4
    vdb = hps.VolatileStore(8)
    vdb.register_table(T("t", d), hps.VolatileTableConfig(partition_count=16))
    keys = np.arange(0, 200000, 2, dtype=np.uint64)
    vdb.insert("t", keys, rows(keys, d))
    errors = []

    def worker(seed):
        rng = np.random.default_rng(seed)
        for _ in range(150):
            q = rng.integers(0, 200000, 3000, dtype=np.uint64)
            r = vdb.lookup("t", q)
            want = q[q % 2 == 0]
            if not (np.array_equal(r.found_keys, want) and
                    r.found_vectors.tobytes() == rows(want, d).tobytes() and
                    np.array_equal(r.missing_keys, q[q % 2 == 1])):
                errors.append(seed)
                return

    ts = [threading.Thread(target=worker, args=(s,)) for s in range(4)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errors


def test_round2_entry_points_validate_arguments_without_a_gpu():
    """Replace-mode, peer-memory and drain entry points reject null handles /
    bad sizes with HPS_INVALID_ARGUMENT and a thread-local message, before
    touching a device (the C ABI's error contract, hps_b200.h)."""
    import ctypes as C

    L = hps.lib()
    assert L.hps_peer_blob_size() >= 64
    assert L.hps_cache_set_replace_mode(None, 1) == 1  # HPS_INVALID_ARGUMENT
    assert b"null" in L.hps_last_error()
    assert L.hps_cache_get_replace_mode(None, None, None) == 1
    n = C.c_size_t(0)
    assert L.hps_cache_peer_drain(None, None, 0, C.byref(n)) == 1
    blob = C.create_string_buffer(L.hps_peer_blob_size())
    ln = C.c_size_t(0)
    assert L.hps_cache_peer_export(None, 16, blob, len(blob), C.byref(ln)) == \
        1
    g = C.c_void_p()
    assert L.hps_peer_group_create(None, 0, 1, blob, len(blob), C.byref(g)) == \
        1
    assert L.hps_peer_lookup_device(None, None, 0, None, None, None, None) == \
        1
    assert L.hps_peer_group_destroy(None) == 0
