"""GPU parity for the lookup engine (calls through the C ABI).

Port of /root/reference/proj/tests/unit/test_lookup_engine.cpp (the cold
tier is a DictStore with PersistentStore::get's contract) plus lockstep
sessions against the reference-generated fixture and the Python engine
oracle."""
import hashlib
import json
from pathlib import Path

import numpy as np

from tools import workload
import pytest

import oracle
import paper_2210_08804_b200 as hps
from opstream import row_values

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
T = hps.TableId


def rows(keys, dim, salt=0.0):
    # test_lookup_engine.cpp:23-32
    return np.array([[float(k) * 10.0 + salt + c for c in range(dim)] for k in keys],
                    dtype=np.float32).reshape(-1)


class Fixture:
    def __init__(self, pdb_keys=20):
        self.table = T("t", 2)
        self.pdb = hps.DictStore(2)
        keys = list(range(pdb_keys))
        self.pdb.put(keys, rows(keys, 2))
        self.cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=8, slabs_per_set=2,
                                                       dimension=2))


def test_cold_lookup_takes_sync_branch_and_admits():
    fx = Fixture()
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, hps.EngineConfig(hit_rate_threshold=0.75))
    o = hps.LookupOutcome()
    keys = [0, 1, 2, 3]
    r = e.lookup(keys, o)
    assert o.sync_branch and o.unique_hit_rate == 0.0 and o.unique_count == 4
    assert o.defaults_returned == 0
    assert r.dimension == 2 and r.miss_flags.tolist() == [0] * 4
    assert r.vectors.tolist() == rows(keys, 2).tolist()
    r2 = e.lookup(keys, o)
    assert o.unique_hit_rate == 1.0 and not o.sync_branch
    assert r2.vectors.tolist() == rows(keys, 2).tolist()
    assert fx.cache.occupied() == 4


def test_async_branch_ships_defaults_and_fills_in_background():
    fx = Fixture()
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb,
                         hps.EngineConfig(hit_rate_threshold=0.75, default_vector=[9.0, 9.0]))
    e.lookup([0, 1, 2, 3, 4, 5])
    o = hps.LookupOutcome()
    r = e.lookup([0, 1, 2, 3, 4, 5, 10, 11], o)
    assert not o.sync_branch and o.unique_hit_rate == 0.75 and o.defaults_returned == 2
    assert r.miss_flags.tolist() == [0] * 6 + [1, 1]
    assert r.vectors[12] == 9.0 and r.vectors[15] == 9.0
    e.drain_async()
    r2 = e.lookup([10, 11], o)
    assert o.unique_hit_rate == 1.0
    assert r2.miss_flags.tolist() == [0, 0]
    assert r2.vectors.tolist() == rows([10, 11], 2).tolist()


def test_duplicate_keys_expand_to_identical_rows():
    fx = Fixture()
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, hps.EngineConfig(hit_rate_threshold=0.75))
    o = hps.LookupOutcome()
    r = e.lookup([5, 5, 6, 5], o)
    assert o.unique_count == 2
    v5, v6 = rows([5], 2).tolist(), rows([6], 2).tolist()
    assert r.vectors.tolist() == v5 + v5 + v6 + v5


def test_empty_query_returns_empty_result():
    fx = Fixture()
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, hps.EngineConfig())
    clock = fx.cache.recency_clock()
    o = hps.LookupOutcome()
    r = e.lookup([], o)
    assert len(r.vectors) == 0 and len(r.miss_flags) == 0
    assert o.unique_count == 0 and o.unique_hit_rate == 1.0 and not o.sync_branch
    assert fx.cache.recency_clock() == clock + 1  # the cache query still ticks


def test_threshold_comparison_is_strict():
    def run(t):
        fx = Fixture()
        e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, hps.EngineConfig(hit_rate_threshold=t))
        e.lookup([0])
        o = hps.LookupOutcome()
        e.lookup([0, 1], o)
        return o

    at = run(0.5)
    assert at.unique_hit_rate == 0.5 and not at.sync_branch
    below = run(0.5625)
    assert below.unique_hit_rate == 0.5 and below.sync_branch and below.defaults_returned == 0


def test_absent_keys_come_back_as_flagged_defaults():
    fx = Fixture()
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb,
                         hps.EngineConfig(hit_rate_threshold=0.75, default_vector=[7.0]))
    o = hps.LookupOutcome()
    r = e.lookup([500, 501], o)
    assert o.sync_branch and o.defaults_returned == 2
    assert r.miss_flags.tolist() == [1, 1]
    assert r.vectors.tolist() == [7.0, 0.0, 7.0, 0.0]
    assert fx.cache.occupied() == 0
    assert e.stats().tier_missing == 2


def test_engine_stats_add_up_over_a_deterministic_sequence():
    fx = Fixture()
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, hps.EngineConfig(hit_rate_threshold=0.75))
    e.lookup([0, 1, 2, 3])
    e.lookup([0, 1, 2, 3, 4, 5, 6, 7])
    e.lookup([0, 1, 2, 3, 4, 5, 6, 7])
    e.lookup([0, 1, 2, 3, 4, 5, 10, 11])
    e.drain_async()
    e.lookup([10, 11])
    e.drain_async()
    s = e.stats()
    assert (s.queries, s.queried_keys, s.unique_keys) == (5, 30, 30)
    assert (s.cache_hits, s.cache_misses) == (20, 10)
    assert (s.sync_batches, s.async_batches, s.defaults_returned) == (2, 3, 2)
    assert (s.pdb_hits, s.vdb_hits, s.tier_missing, s.async_faults) == (10, 0, 0, 0)


def test_volatile_tier_values_win_when_enabled_and_are_skipped_when_not():
    table = T("t", 1)
    pdb = hps.DictStore(1)
    pdb.put([3], [30.0])
    vdb = hps.VolatileStore()
    vdb.register_table(table)
    vdb.insert("t", [3], [33.0])
    c1 = hps.SlabCache(hps.SlabCacheConfig(slabset_count=4, slabs_per_set=2, dimension=1))
    e1 = hps.LookupEngine(table, c1, vdb, pdb, hps.EngineConfig(hit_rate_threshold=0.75))
    assert e1.lookup([3]).vectors.tolist() == [33.0]
    assert e1.stats().vdb_hits == 1
    c2 = hps.SlabCache(hps.SlabCacheConfig(slabset_count=4, slabs_per_set=2, dimension=1))
    e2 = hps.LookupEngine(table, c2, vdb, pdb,
                          hps.EngineConfig(hit_rate_threshold=0.75, volatile_tier_enabled=False))
    assert e2.lookup([3]).vectors.tolist() == [30.0]
    assert e2.stats().vdb_hits == 0 and e2.stats().pdb_hits == 1


def test_workspace_pool_bounds_in_flight_batches():
    fx = Fixture(200)
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb,
                         hps.EngineConfig(hit_rate_threshold=0.0, workspace_pool_size=2,
                                          async_worker_count=1))
    for i in range(30):
        e.lookup([i * 3 % 200, (i * 3 + 1) % 200])
    e.drain_async()
    p = e.workspace_pool()
    assert p.size == 2 and p.outstanding == 0 and 1 <= p.peak_outstanding <= 2


def test_engine_shuts_down_cleanly_with_queued_work():
    fx = Fixture(100)
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb,
                         hps.EngineConfig(hit_rate_threshold=0.0, workspace_pool_size=8))
    for i in range(20):
        e.lookup([i * 2, i * 2 + 1])
    e.close()


def test_configuration_is_validated():
    fx = Fixture()
    for cfg in (hps.EngineConfig(hit_rate_threshold=-0.1), hps.EngineConfig(hit_rate_threshold=1.5),
                hps.EngineConfig(async_worker_count=0), hps.EngineConfig(workspace_pool_size=0)):
        with pytest.raises(hps.InvalidArgument):
            hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, cfg)
    wrong = hps.SlabCache(hps.SlabCacheConfig(slabset_count=2, slabs_per_set=2, dimension=5))
    with pytest.raises(hps.InvalidArgument):
        hps.LookupEngine(fx.table, wrong, None, fx.pdb, hps.EngineConfig())


def test_reference_engine_session_fixture():
    """40 lookups through the reference LookupEngine (engine.json) replayed
    through the device engine: outcomes, every output byte, flags, stats."""
    e = json.loads((GOLD / "engine.json").read_text())
    d = e["dim"]
    table = T("t", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table, hps.VolatileTableConfig(partition_count=e["partitions"]))
    vk = np.arange(e["vdb_keys"], dtype=np.uint64)
    vdb.insert("t", vk, row_values(vk, d, e["vdb_salt"]))
    c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=e["S"], slabs_per_set=e["W"], dimension=d))
    eng = hps.LookupEngine(table, c, vdb, None,
                           hps.EngineConfig(hit_rate_threshold=e["threshold"],
                                            default_vector=e["default_vector"]))
    rng = np.random.default_rng(e["batch_seed"])
    for step in e["steps"]:
        keys = rng.integers(0, e["key_range"], 1 + int(rng.integers(300)), dtype=np.uint64)
        o = hps.LookupOutcome()
        r = eng.lookup(keys, o)
        eng.drain_async()
        assert o.__dict__ == step["outcome"]
        assert hashlib.sha256(r.vectors.tobytes()).hexdigest() == step["out_sha"]
        assert hashlib.sha256(r.miss_flags.tobytes()).hexdigest() == step["flags_sha"]
    assert eng.stats().__dict__ == e["stats"]


@pytest.mark.parametrize("threshold", [0.0, 0.7, 0.95, 1.0])
def test_lockstep_with_engine_oracle_power_law(threshold):
    d, S = 32, 64
    eo = oracle.EngineOracle(S, 2, d, threshold=threshold, default_vector=[1.5])
    table = T("t", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table)
    vk = np.arange(0, 40000, 2, dtype=np.uint64)  # odd keys are absent everywhere
    vv = row_values(vk, d, 3)
    vdb.insert("t", vk, vv)
    for k, r in zip(vk, vv.reshape(-1, d)):
        eo.vdb[int(k)] = r
    c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d))
    eng = hps.LookupEngine(table, c, vdb, None,
                           hps.EngineConfig(hit_rate_threshold=threshold, default_vector=[1.5]))
    stream = workload.powerlaw_sample(1.2, 40000, 7, 8, 30 * 2048)
    for b in range(30):
        keys = stream[b * 2048:(b + 1) * 2048]
        o = hps.LookupOutcome()
        r = eng.lookup(keys, o)
        eng.drain_async()
        out, flags, oc = eo.lookup(keys)
        eo.drain_async()
        assert o.__dict__ == oc
        assert r.vectors.tobytes() == out.tobytes()
        assert (r.miss_flags == flags).all()
    s = eng.stats().__dict__
    assert s == eo.stats
    c.check_invariants()


def test_device_and_pinned_pointer_lookups_match_host_lookup():
    import torch

    d = 128
    table = T("t", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table)
    vk = np.arange(100000, dtype=np.uint64)
    vdb.insert("t", vk, row_values(vk, d, 2))

    def mk():
        c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=1024, slabs_per_set=2, dimension=d))
        return c, hps.LookupEngine(table, c, vdb, None, hps.EngineConfig(hit_rate_threshold=0.8))

    ch, eh = mk()
    cd, ed = mk()
    cp, ep = mk()
    stream = workload.powerlaw_sample(1.2, 100000, 1, 2, 8 * 16384)
    for b in range(8):
        keys = stream[b * 16384:(b + 1) * 16384]
        r = eh.lookup(keys)
        eh.drain_async()
        kt = torch.from_numpy(keys.view(np.int64)).cuda()
        out = torch.empty(len(keys) * d, device="cuda")
        fl = torch.empty(len(keys), dtype=torch.uint8, device="cuda")
        ed.lookup_ptrs(kt.data_ptr(), len(keys), out.data_ptr(), fl.data_ptr(), hps.HPS_MEM_DEVICE,
                       torch.cuda.current_stream().cuda_stream)
        torch.cuda.current_stream().synchronize()
        ed.drain_async()
        assert out.cpu().numpy().tobytes() == r.vectors.tobytes()
        assert (fl.cpu().numpy() == r.miss_flags).all()
        kp = torch.from_numpy(keys.view(np.int64)).pin_memory()
        op = torch.empty(len(keys) * d).pin_memory()
        fp = torch.empty(len(keys), dtype=torch.uint8).pin_memory()
        ep.lookup_ptrs(kp.data_ptr(), len(keys), op.data_ptr(), fp.data_ptr(), hps.HPS_MEM_HOST)
        ep.drain_async()
        assert op.numpy().tobytes() == r.vectors.tobytes()
        assert (fp.numpy() == r.miss_flags).all()


def test_multi_table_lookup_equals_per_table_lookups():
    """hps_engine_lookup_multi (all tables' device work in flight before the
    first host wait) must give every table exactly what a per-table
    hps_engine_lookup gives: rows, flags, outcomes, cache state, stats --
    over sync and async branches, with the tables' VDBs and cold tiers."""
    import torch

    d, T_, n = 16, 5, 3000

    def build():
        vdb = hps.VolatileStore(4)
        engines, caches = [], []
        for t in range(T_):
            table = T(f"m{t}", d)
            vdb.register_table(table)
            keys = np.arange(t * 100000, t * 100000 + 20000, dtype=np.uint64)
            vdb.insert(table.name, keys, row_values(keys, d, t))
            c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=64, slabs_per_set=2, dimension=d))
            caches.append(c)
            engines.append(hps.LookupEngine(table, c, vdb, None,
                                            hps.EngineConfig(hit_rate_threshold=0.6,
                                                             default_vector=[float(t)] * d)))
        return vdb, caches, engines

    va, ca, ea = build()
    vb, cb, eb = build()
    rng = np.random.default_rng(9)
    for r in range(6):
        batches = [workload.powerlaw_sample(1.1, 26000, t, 50 * r + t, n) + np.uint64(t * 100000)
                   for t in range(T_)]
        pk = [torch.from_numpy(b.view(np.int64)).pin_memory() for b in batches]
        po = [torch.empty(n * d).pin_memory() for _ in range(T_)]
        pf = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(T_)]
        outs = hps.LookupEngine.lookup_multi_ptrs(ea, [p.data_ptr() for p in pk], [n] * T_,
                                                  [p.data_ptr() for p in po],
                                                  [p.data_ptr() for p in pf], hps.HPS_MEM_HOST)
        for t in range(T_):
            o = hps.LookupOutcome()
            want = eb[t].lookup(batches[t], o)
            assert po[t].numpy().tobytes() == want.vectors.tobytes(), (r, t)
            assert (pf[t].numpy() == want.miss_flags).all(), (r, t)
            assert outs[t] == o, (r, t)
        for e in ea + eb:
            e.drain_async()
    for t in range(T_):
        assert ca[t].dump_all().tolist() == cb[t].dump_all().tolist()
        assert ea[t].stats() == eb[t].stats()
    for e in ea + eb:
        e.close()


@pytest.mark.parametrize("dump_batch", [1, 97, 4096])
def test_native_refresh_matches_reference_semantics(dump_batch):
    """hps_refresh_cache = refresh_cache (refresh_engine.cpp:5-22): every
    resident key in dump order, VDB value first, then the cold tier; found
    rows written back with update (nothing admitted, recency untouched),
    keys absent from both reported unresolved in dump order."""
    d = 8
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=32, slabs_per_set=2, dimension=d))
    o = oracle.OracleCache(32, 2, d)
    rng = np.random.default_rng(dump_batch)
    keys = rng.choice(100000, 1500, replace=False).astype(np.uint64)
    cache.replace(keys, row_values(keys, d, 0))
    o.replace(keys, row_values(keys, d, 0))
    resident = cache.dump_all()
    assert (resident == o.dump()).all()
    table = T("r", d)
    vdb = hps.VolatileStore(2)
    vdb.register_table(table)
    in_vdb = resident[rng.random(len(resident)) < 0.5]
    vdb.insert("r", in_vdb, row_values(in_vdb, d, 1))
    rest = np.setdiff1d(resident, in_vdb)
    in_cold = rest[rng.random(len(rest)) < 0.6]
    pdb = hps.DictStore(d)
    pdb.put(in_cold, row_values(in_cold, d, 2))
    clock = cache.recency_clock()
    out = hps.refresh_cache(cache, table, vdb, pdb, dump_batch_size=dump_batch)
    found = np.concatenate([in_vdb, in_cold])
    want_un = resident[~np.isin(resident, found)]
    assert out.refreshed == len(found)
    assert out.unresolved.tolist() == want_un.tolist()
    vset = set(in_vdb.tolist())
    for b in range(0, len(resident), dump_batch):
        bk = resident[b:b + dump_batch]
        fv = [k for k in bk if int(k) in vset]
        fc = [k for k in bk if int(k) not in vset and k in set(in_cold.tolist())]
        if fv:
            o.update(np.array(fv, np.uint64), row_values(np.array(fv, np.uint64), d, 1))
        if fc:
            o.update(np.array(fc, np.uint64), row_values(np.array(fc, np.uint64), d, 2))
    gk, gc, gm, gr = cache.export_state()
    ok, oc, om, orow = o.state()
    occ = (np.repeat(gm, 32).reshape(-1, 32) >> np.arange(32, dtype=np.uint32) & 1).reshape(-1) == 1
    assert (gm == om).all() and (gk[occ] == ok[occ]).all() and (gc[occ] == oc[occ]).all()
    assert gr.reshape(-1, d)[occ].tobytes() == orow.reshape(-1, d)[occ].tobytes()
    assert cache.recency_clock() == clock and cache.occupied() == len(resident)


def test_native_refresh_tier_fault_keeps_finished_batches():
    d = 4
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=16, slabs_per_set=2, dimension=d))
    keys = np.arange(600, dtype=np.uint64)
    cache.replace(keys, row_values(keys, d, 0))
    resident = cache.dump_all()

    class Flaky:
        calls = 0

        def get(self, ks):
            Flaky.calls += 1
            if Flaky.calls > 2:
                raise IOError("segment unreadable")
            return hps.FetchResult(ks, row_values(ks, d, 5), np.empty(0, np.uint64))

    with pytest.raises(hps.TierFault):
        hps.refresh_cache(cache, T("f", d), None, Flaky(), dump_batch_size=100)
    got = np.zeros(len(resident) * d, np.float32)
    cache.query(resident, got)
    got = got.reshape(-1, d)
    assert got[:200].tobytes() == row_values(resident[:200], d, 5).tobytes()
    assert got[200:].tobytes() == row_values(resident[200:], d, 0).tobytes()


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("dims", [(16, 16, 16, 16), (8, 12, 16, 20, 4), (3, 5)])
def test_group_multi_lookup_one_launch_equals_per_table_lookups(dims, pinned):
    """MultiLookup (cache group, ONE kernel launch for all tables) must give
    every table exactly what a per-table hps_engine_lookup gives on an
    identical twin: rows, flags, outcomes, cache contents, stats -- with
    different dims per table, ragged and empty per-table batches, and both
    the sync and the async branch; pinned caller outputs get the rows written
    straight into them (zero-copy), pageable ones through the staging mirror."""
    import torch

    T_ = len(dims)

    def build(grouped):
        vdb = hps.VolatileStore(4)
        caches, engines = [], []
        for t, d in enumerate(dims):
            table = T(f"g{t}", d)
            vdb.register_table(table)
            keys = np.arange(t * 100000, t * 100000 + 9000, dtype=np.uint64)
            vdb.insert(table.name, keys, row_values(keys, d, t))
            cfg = hps.SlabCacheConfig(slabset_count=32, slabs_per_set=2, dimension=d)
            c = hps.SlabCache(cfg, share_stream_with=caches[0] if (grouped and caches) else None)
            caches.append(c)
            engines.append(hps.LookupEngine(table, c, vdb, None,
                                            hps.EngineConfig(hit_rate_threshold=0.55,
                                                             default_vector=[1.5 + t] * d)))
        return vdb, caches, engines

    va, ca, ea = build(True)
    vb, cb, eb = build(False)
    m = hps.MultiLookup(ea, max_batch=4096)
    for r in range(6):
        ns = [(700 + 311 * t + 97 * r) % 4097 for t in range(T_)]
        if r == 2:
            ns[0] = 0
        batches = [workload.powerlaw_sample(1.1, 11000, t, 70 * r + t, ns[t]) + np.uint64(t * 100000)
                   for t in range(T_)]
        if pinned:
            pk = [torch.from_numpy(b.view(np.int64)).pin_memory() for b in batches]
            po = [torch.zeros(max(ns[t], 1) * dims[t]).pin_memory() for t in range(T_)]
            pf = [torch.zeros(max(ns[t], 1), dtype=torch.uint8).pin_memory() for t in range(T_)]
            m.lookup_ptrs([k.data_ptr() for k in pk], ns, [o.data_ptr() for o in po],
                          [f.data_ptr() for f in pf])
            got = [hps.LookupResult(dims[t], po[t].numpy()[: ns[t] * dims[t]].copy(),
                                    pf[t].numpy()[: ns[t]].copy()) for t in range(T_)]
        else:
            got = m.lookup(batches)
        for t in range(T_):
            o = hps.LookupOutcome()
            want = eb[t].lookup(batches[t], o)
            assert got[t].vectors.tobytes() == want.vectors.tobytes(), (r, t)
            assert (got[t].miss_flags == want.miss_flags).all(), (r, t)
        for e in ea + eb:
            e.drain_async()
    for t in range(T_):
        assert ca[t].dump_all().tolist() == cb[t].dump_all().tolist()
        sa, sb = ea[t].stats(), eb[t].stats()
        assert sa == sb, (t, sa, sb)
        ca[t].check_invariants()
    m.close()
    for e in ea + eb:
        e.close()


@pytest.mark.parametrize("threshold", [0.7, 1.0])
def test_zero_copy_small_calls_pinned_and_pageable_match_oracle(threshold):
    """Host-buffer calls of <= 4,096 keys run zero-copy (the kernels read the
    keys from and write rows, flags, counts and claims to pinned host memory;
    the sync branch's scatter and fill read the host-staged rows). Pinned
    caller buffers (rows written straight into the caller's memory), pageable
    ones, and sizes across the zero-copy limit (4,096 / 4,097) must all match
    the engine oracle call for call: outcomes, rows, flags, and the final
    engine stats."""
    import torch

    d, S = 16, 96
    eo = oracle.EngineOracle(S, 2, d, threshold=threshold, default_vector=[0.25, -1.0])
    table = T("t", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table)
    vk = np.arange(0, 60000, 3, dtype=np.uint64)  # other keys are absent everywhere
    vv = row_values(vk, d, 5)
    vdb.insert("t", vk, vv)
    for k, r in zip(vk, vv.reshape(-1, d)):
        eo.vdb[int(k)] = r
    c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d))
    eng = hps.LookupEngine(table, c, vdb, None,
                           hps.EngineConfig(hit_rate_threshold=threshold,
                                            default_vector=[0.25, -1.0]))
    maxn = 4097
    pk = torch.empty(maxn, dtype=torch.int64).pin_memory()
    po = torch.empty(maxn * d).pin_memory()
    pf = torch.empty(maxn, dtype=torch.uint8).pin_memory()
    sizes = [1, 7, 1024, 4096, 4097, 300, 4096, 2048, 33, 4097, 1500, 4000]
    stream = workload.powerlaw_sample(1.15, 60000, 11, 12, sum(sizes))
    at = 0
    for b, n in enumerate(sizes):
        keys = stream[at:at + n]
        at += n
        if b % 2 == 0:
            pk.numpy().view(np.uint64)[:n] = keys
            o = eng.lookup_ptrs(pk.data_ptr(), n, po.data_ptr(), pf.data_ptr(), hps.HPS_MEM_HOST)
            got_rows, got_flags = po.numpy()[: n * d].copy(), pf.numpy()[:n].copy()
            got = (o.sync_branch, o.unique_hit_rate, o.unique_count, o.defaults_returned)
        else:
            oo = hps.LookupOutcome()
            r = eng.lookup(keys, oo)
            got_rows, got_flags = r.vectors, r.miss_flags
            got = (oo.sync_branch, oo.unique_hit_rate, oo.unique_count, oo.defaults_returned)
        eng.drain_async()
        out, flags, oc = eo.lookup(keys)
        eo.drain_async()
        assert got == (oc["sync_branch"], oc["unique_hit_rate"], oc["unique_count"],
                       oc["defaults_returned"]), (b, n)
        assert got_rows.tobytes() == out.tobytes(), (b, n)
        assert (got_flags == flags).all(), (b, n)
    assert eng.stats().__dict__ == eo.stats
    c.check_invariants()
    eng.close()


def test_group_multi_lookup_with_empty_tables_over_many_calls():
    """An empty per-table batch takes no lookup view (no block would ever
    release it): more than kLookupViews (8) group calls with table 0 empty
    every time, and some calls with every table empty, must keep matching
    the per-table twin (a leaked view would hang its next use on the device)."""
    dims = (8, 16)
    T_ = len(dims)

    def build(grouped):
        vdb = hps.VolatileStore(2)
        caches, engines = [], []
        for t, d in enumerate(dims):
            table = T(f"e{t}", d)
            vdb.register_table(table)
            keys = np.arange(t * 100000, t * 100000 + 5000, dtype=np.uint64)
            vdb.insert(table.name, keys, row_values(keys, d, t))
            cfg = hps.SlabCacheConfig(slabset_count=16, slabs_per_set=2, dimension=d)
            c = hps.SlabCache(cfg, share_stream_with=caches[0] if (grouped and caches) else None)
            caches.append(c)
            engines.append(hps.LookupEngine(table, c, vdb, None,
                                            hps.EngineConfig(hit_rate_threshold=0.6)))
        return vdb, caches, engines

    va, ca, ea = build(True)
    vb, cb, eb = build(False)
    m = hps.MultiLookup(ea, max_batch=2048)
    for r in range(20):
        ns = [0, 0 if r % 5 == 4 else 200 + 37 * r]
        batches = [workload.powerlaw_sample(1.1, 6000, t, 90 * r + t, ns[t]) + np.uint64(t * 100000)
                   for t in range(T_)]
        got = m.lookup(batches)
        for t in range(T_):
            want = eb[t].lookup(batches[t])
            assert got[t].vectors.tobytes() == want.vectors.tobytes(), (r, t)
            assert (got[t].miss_flags == want.miss_flags).all(), (r, t)
        for e in ea + eb:
            e.drain_async()
    for t in range(T_):
        assert ca[t].recency_clock() == cb[t].recency_clock()
        assert ca[t].dump_all().tolist() == cb[t].dump_all().tolist()
        assert ea[t].stats() == eb[t].stats()
    m.close()
    for e in ea + eb:
        e.close()


def test_engine_lookup_multi_device_mode_orders_against_default_stream():
    """hps_engine_lookup_multi with HPS_MEM_DEVICE orders against the legacy
    default stream (like hps_engine_lookup with a NULL stream): keys written
    by a default-stream kernel right before the call are the ones looked up,
    and default-stream reads right after it see the final rows and flags --
    including the sync branch's scatter."""
    import torch

    d, T_, n = 32, 3, 20000

    def build():
        vdb = hps.VolatileStore(4)
        engines = []
        for t in range(T_):
            table = T(f"dm{t}", d)
            vdb.register_table(table)
            keys = np.arange(t * 100000, t * 100000 + 50000, dtype=np.uint64)
            vdb.insert(table.name, keys, row_values(keys, d, t))
            c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=128, slabs_per_set=2, dimension=d))
            engines.append((c, hps.LookupEngine(table, c, vdb, None,
                                                hps.EngineConfig(hit_rate_threshold=0.9))))
        return vdb, engines

    va, ea = build()
    vb, eb = build()
    for r in range(4):
        batches = [workload.powerlaw_sample(1.05, 60000, t, 11 * r + t, n) + np.uint64(t * 100000)
                   for t in range(T_)]
        # keys land on the device through a default-stream kernel (x + 0)
        src = [torch.from_numpy(b.view(np.int64)).cuda() for b in batches]
        torch.cuda.synchronize()
        torch.cuda.set_stream(torch.cuda.default_stream())
        big = torch.empty(1 << 26, device="cuda")
        big.uniform_()  # queue default-stream work ahead of the key writes
        dk = [s + 0 for s in src]
        out = [torch.full((n * d,), -7.0, device="cuda") for _ in range(T_)]
        fl = [torch.full((n,), 9, dtype=torch.uint8, device="cuda") for _ in range(T_)]
        hps.LookupEngine.lookup_multi_ptrs([e for _, e in ea], [k.data_ptr() for k in dk], [n] * T_,
                                           [o.data_ptr() for o in out], [f.data_ptr() for f in fl],
                                           hps.HPS_MEM_DEVICE)
        got = [(o.cpu().numpy(), f.cpu().numpy()) for o, f in zip(out, fl)]  # default stream
        for t in range(T_):
            want = eb[t][1].lookup(batches[t])
            assert got[t][0].tobytes() == want.vectors.tobytes(), (r, t)
            assert (got[t][1] == want.miss_flags).all(), (r, t)
        for (_, e) in ea + eb:
            e.drain_async()
    for (_, e) in ea + eb:
        e.close()


def test_max_batch_is_enforced():
    fx = Fixture(200)
    e = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, hps.EngineConfig(max_batch=64))
    e.lookup(np.arange(64, dtype=np.uint64) % 200)
    with pytest.raises(hps.InvalidArgument):
        e.lookup(np.arange(65, dtype=np.uint64) % 200)
    e.close()
    unlimited = hps.LookupEngine(fx.table, fx.cache, None, fx.pdb, hps.EngineConfig())
    assert unlimited.lookup(np.arange(5000, dtype=np.uint64) % 200).vectors.size == 5000 * 2
    unlimited.close()


@pytest.mark.parametrize("threshold", [0.5, 0.95])
def test_large_pageable_batches_lockstep_with_engine_oracle(threshold):
    """Batches whose rows come back through the chunked staging + parallel
    copy-on (pageable numpy output, 40,000 x 64 floats = 10 MB, 5 chunks),
    both branches, in lock-step with the engine oracle."""
    d, S = 64, 512
    eo = oracle.EngineOracle(S, 2, d, threshold=threshold, default_vector=[0.5])
    table = T("t", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table)
    vk = np.arange(0, 60000, 3, dtype=np.uint64)
    vv = row_values(vk, d, 5)
    vdb.insert("t", vk, vv)
    for k, r in zip(vk, vv.reshape(-1, d)):
        eo.vdb[int(k)] = r
    c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d))
    eng = hps.LookupEngine(table, c, vdb, None,
                           hps.EngineConfig(hit_rate_threshold=threshold, default_vector=[0.5]))
    stream = workload.powerlaw_sample(1.05, 60000, 3, 4, 6 * 40000)
    branches = set()
    for b in range(6):
        keys = stream[b * 40000:(b + 1) * 40000]
        o = hps.LookupOutcome()
        r = eng.lookup(keys, o)
        eng.drain_async()
        out, flags, oc = eo.lookup(keys)
        eo.drain_async()
        branches.add(o.sync_branch)
        assert o.__dict__ == oc
        assert r.vectors.tobytes() == out.tobytes()
        assert (r.miss_flags == flags).all()
    assert eng.stats().__dict__ == eo.stats
    c.check_invariants()


def test_async_fills_on_the_side_stream_interleave_with_lookups():
    """Back-to-back large lookups with background fills in flight (their
    uploads on the engine's copy stream, replaces enqueued after): every
    unflagged row is the stored row, every flagged row the default, and the
    cache ends consistent with every fetched key resident or evicted."""
    d, S = 128, 1024
    table = T("t", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table)
    vk = np.arange(200000, dtype=np.uint64)
    vv = row_values(vk, d, 9)
    vdb.insert("t", vk, vv)
    vv = vv.reshape(-1, d)
    c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d))
    eng = hps.LookupEngine(table, c, vdb, None,
                           hps.EngineConfig(hit_rate_threshold=0.0, default_vector=[-2.0]))
    stream = workload.powerlaw_sample(1.1, 200000, 11, 12, 12 * 32768)
    for b in range(12):
        keys = stream[b * 32768:(b + 1) * 32768]
        o = hps.LookupOutcome()
        r = eng.lookup(keys, o)
        assert not o.sync_branch
        got = r.vectors.reshape(-1, d)
        hit = r.miss_flags == 0
        assert (got[hit] == vv[keys[hit].astype(np.int64)]).all()
        dv = np.zeros(d, np.float32)
        dv[0] = -2.0  # the default vector, zero-padded to the dimension
        assert (got[~hit] == dv).all()
    eng.drain_async()
    c.check_invariants()
    assert eng.stats().async_faults == 0


def test_native_segment_cold_tier_engine_matches_python_cold_tier(tmp_path):
    """The engine with the native batched reader (hps_pdb_cold_fetch, §8 row
    f4) behind a partial VDB behaves exactly like the engine over a Python
    cold tier holding the same rows: outcomes, rows, flags, stats (PDB hits
    promoted into the VDB included)."""
    from test_segment_store import write_table

    d, S = 16, 64
    table = T("cold", d)
    keys = np.arange(0, 30000, 3, dtype=np.uint64)
    vals = row_values(keys, d, 4)
    write_table(tmp_path, "cold", d, {0: [(int(k), d, v) for k, v in
                                         zip(keys, vals.reshape(-1, d))]})
    native = hps.SegmentStore(tmp_path).table("cold")
    py = hps.DictStore(d)
    py.put(keys, vals)
    engines = []
    for cold in (native, py):
        vdb = hps.VolatileStore()
        vdb.register_table(table)
        vk = keys[::4]
        vdb.insert("cold", vk, row_values(vk, d, 4))
        c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d))
        engines.append((hps.LookupEngine(table, c, vdb, cold,
                                         hps.EngineConfig(hit_rate_threshold=0.9)), c, vdb))
    stream = workload.powerlaw_sample(1.1, 33000, 5, 6, 10 * 4000)
    for b in range(10):
        q = stream[b * 4000:(b + 1) * 4000]
        res = []
        for e, _, vdb in engines:
            o = hps.LookupOutcome()
            r = e.lookup(q, o)
            e.drain_async()
            vdb.drain()
            res.append((o.__dict__, r.vectors.tobytes(), r.miss_flags.tobytes()))
        assert res[0] == res[1]
    s0, s1 = engines[0][0].stats().__dict__, engines[1][0].stats().__dict__
    assert s0 == s1 and s0["pdb_hits"] > 0
    assert engines[0][2].table_size("cold") == engines[1][2].table_size("cold")


def test_reserve_preallocates_and_lookups_are_unchanged():
    d = 32
    table = T("t", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table)
    vk = np.arange(50000, dtype=np.uint64)
    vdb.insert("t", vk, row_values(vk, d, 1))
    outs = []
    for mode in ("lazy", "reserve", "max_batch"):
        c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=256, slabs_per_set=2, dimension=d))
        e = hps.LookupEngine(table, c, vdb, None, hps.EngineConfig(
            hit_rate_threshold=0.7, workspace_pool_size=4,
            max_batch=20000 if mode == "max_batch" else 0))
        if mode == "reserve":
            e.reserve(20000)
        stream = workload.powerlaw_sample(1.1, 50000, 2, 3, 6 * 20000)
        got = []
        for b in range(6):
            r = e.lookup(stream[b * 20000:(b + 1) * 20000])
            e.drain_async()
            got.append((r.vectors.tobytes(), r.miss_flags.tobytes()))
        outs.append((got, e.stats().__dict__))
        c.check_invariants()
    assert outs[0] == outs[1] == outs[2]


def test_replica_group_shares_one_vdb_and_matches_independent_engines():
    """ReplicaGroup (hps_replicas_*): replicas on their own threads over ONE
    shared VDB give every replica exactly what an independent engine gives
    for its own stream (the GPU box has one GPU: both replicas on device 0)."""
    d, S = 32, 128
    table = T("t", d)
    vk = np.arange(0, 60000, 2, dtype=np.uint64)
    vv = row_values(vk, d, 7)

    def vdb_full():
        v = hps.VolatileStore()
        v.register_table(table)
        v.insert("t", vk, vv)
        return v

    shared = vdb_full()
    cfg = hps.EngineConfig(hit_rate_threshold=0.85, default_vector=[0.5])
    grp = hps.ReplicaGroup([0, 0], hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2,
                                                       dimension=d), table, shared, None, cfg)
    solo = []
    for r in range(2):
        c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d))
        solo.append((c, hps.LookupEngine(table, c, vdb_full(), None, cfg)))
    streams = [workload.powerlaw_sample(1.15, 60000, 20 + r, 30 + r, 8 * 6000) for r in range(2)]
    for b in range(8):
        batches = [s[b * 6000:(b + 1) * 6000] for s in streams]
        got = grp.lookup(batches)
        for e in grp.engines:
            e.drain_async()
        for r in range(2):
            want = solo[r][1].lookup(batches[r])
            solo[r][1].drain_async()
            assert got[r].vectors.tobytes() == want.vectors.tobytes()
            assert (got[r].miss_flags == want.miss_flags).all()
    for r in range(2):
        assert grp.engines[r].stats().__dict__ == solo[r][1].stats().__dict__
        grp.caches[r].check_invariants()
    grp.close()
