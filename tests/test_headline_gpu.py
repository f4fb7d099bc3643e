"""GPU parity of the HEADLINE path exactly as bench.py times it, and of
captured-graph replays.

* The timed kernel path: hps_cache_lookup_device at cfg 2 (S = 31,250, W = 2,
  d = 128, batch 65,536, the persisting L2 window on), 20 calls chained as
  programmatic dependents and captured into ONE CUDA graph, at unique-key hit
  rates 0.5 / 0.9 / 0.99 drawn by bench.py's own Workload. Every call's rows,
  miss flags, claims (keys + first positions), per-call counts, and the
  recency stamps after the run are checked against the oracle applying the
  same lookups one after another (LookupEngine::lookup's dedup -> query ->
  expand, lookup_engine.cpp:130-203; SlabCache::query, slab_cache.cpp:69-91).
* The same at a cfg-5-scale geometry (1.6 M slabsets = 102.4 M slots).
* Replays: a captured graph launched several times is exactly the same
  lookups issued again -- fresh recency stamps in stream order (paper Alg. 1,
  PAPER.md:296-297), unique hits counted on every replay, views reused only
  after release.
"""
import numpy as np
import pytest

import bench
import oracle
import paper_2210_08804_b200 as hps
from tools import workload

pytestmark = pytest.mark.gpu


def _first_positions(q, keys):
    u, idx = np.unique(q, return_index=True)
    return idx[np.searchsorted(u, keys)]


def check_lookup(o, q, default, d, out, fl, mk, mf, cnt, tag):
    """One lookup-level call against the oracle applying it now."""
    uniq, inv = oracle.dedup(q)
    ws = np.zeros(len(uniq) * d, np.float32)
    hit = o.query(uniq, ws)
    ws = ws.reshape(-1, d)
    ws[hit == 0] = default
    assert out.tobytes() == ws[inv].reshape(-1).tobytes(), tag
    assert (fl == (1 - hit)[inv]).all(), tag
    um = int((hit == 0).sum())
    assert cnt.tolist() == [len(uniq) - um, um], tag
    ck = mk[:um].view(np.uint64)
    cf = mf[:um]
    # claims sorted by first position = the reference's miss order
    assert (ck[np.argsort(cf, kind="stable")] == uniq[hit == 0]).all(), tag
    assert (cf.astype(np.int64) == _first_positions(q, ck)).all(), tag
    return len(uniq) - um, um


def check_state(c, o):
    gk, gc, gm, _ = c.export_state()
    ok, oc, om, _ = o.state()
    occ = (np.repeat(gm, 32).reshape(-1, 32) >> np.arange(32, dtype=np.uint32) & 1).reshape(-1) == 1
    assert (gm == om).all() and (gk[occ] == ok[occ]).all() and (gc[occ] == oc[occ]).all()
    assert c.recency_clock() == o.clock()


class Bufs:
    def __init__(self, torch, K, n, d):
        self.out = [torch.empty(n * d, device="cuda") for _ in range(K)]
        self.fl = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(K)]
        self.mk = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(K)]
        self.mf = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(K)]
        self.cnt = torch.zeros(K, 2, dtype=torch.int64, device="cuda")

    def issue(self, c, j, qt, n, dr, stream):
        c.lookup_device(qt.data_ptr(), n, self.out[j].data_ptr(), self.fl[j].data_ptr(),
                        dr.data_ptr(), self.mk[j].data_ptr(), self.mf[j].data_ptr(),
                        self.cnt[j].data_ptr(), stream)

    def check(self, o, j, q, default, d, tag):
        return check_lookup(o, q, default, d, self.out[j].cpu().numpy(), self.fl[j].cpu().numpy(),
                            self.mk[j].cpu().numpy(), self.mf[j].cpu().numpy(),
                            self.cnt[j].cpu().numpy(), tag)


@pytest.mark.parametrize("own_stream", [True, False])
def test_captured_graph_replays_like_reissued_lookups(own_stream):
    """One captured 10-call graph (more calls than lookup views, so views are
    reused inside a replay) launched three times, with an eager lookup between
    two launches: every replay's rows, flags, claims and unique counts match
    the oracle applying 30 (+2) fresh queries in order; recency clock and
    stamps match at the end. Captured on the cache's own stream and on a
    separate user stream (the launch orders the cache stream around it)."""
    import torch

    S, W, d, K, n = 512, 2, 64, 10, 12000
    c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=W, dimension=d))
    o = oracle.OracleCache(S, W, d)
    rng = np.random.default_rng(5 + own_stream)
    keys = rng.choice(100000, 30000, replace=False).astype(np.uint64)
    v = bench.table_rows(keys, d)
    c.replace(keys, v)
    o.replace(keys, v)
    default = np.full(d, 0.5, np.float32)
    dr = torch.from_numpy(default).cuda()
    qs = [workload.powerlaw_sample(1.2, 100000, 3, 40 + b, n) for b in range(K)]
    qt = [torch.from_numpy(q.view(np.int64)).cuda() for q in qs]
    b = Bufs(torch, K, n, d)
    user = torch.cuda.Stream()
    sp = c.stream() if own_stream else user.cuda_stream
    b.issue(c, 0, qt[0], n, dr, sp)  # sizes the scratch (no allocation inside a capture)
    torch.cuda.synchronize()
    b.check(o, 0, qs[0], default, d, "warm")
    g = hps.StreamGraph(sp)
    with g:
        for j in range(K):
            b.issue(c, j, qt[j], n, dr, sp)
    # the capture itself consumed no clock ticks
    assert c.recency_clock() == o.clock()
    extra = workload.powerlaw_sample(1.2, 100000, 9, 9, n)
    et = torch.from_numpy(extra.view(np.int64)).cuda()
    hits = []
    for rep in range(3):
        g.launch(sp)
        torch.cuda.synchronize()
        for j in range(K):
            hits.append(b.check(o, j, qs[j], default, d, (rep, j))[0])
        if rep == 0:
            # an eager lookup between replays, on the cache's own stream
            b.issue(c, 0, et, n, dr, c.stream())
            torch.cuda.synchronize()
            b.check(o, 0, extra, default, d, "between")
    assert min(hits) > 0  # replays count their unique hits
    check_state(c, o)
    c.check_invariants()


def _headline_cache(wl, d):
    return hps.SlabCache(hps.SlabCacheConfig(slabset_count=wl.S, slabs_per_set=wl.W, dimension=d,
                                             worker_pool_size=8, tasks_per_worker=8))


@pytest.mark.parametrize("h", [0.5, 0.9, 0.99])
def test_headline_cfg2_pipelined_graph_parity(h):
    """bench.py's timed configuration, its workload generator and its call
    sequence: preload through the device replace in 64K chunks, 20 lookups
    PDL-chained in one captured graph, launched twice."""
    import torch

    wl = bench.Workload()
    d, n, K = wl.dim, wl.batch, 20
    c = _headline_cache(wl, d)
    o = oracle.OracleCache(wl.S, wl.W, d)
    for i in range(0, len(wl.preload), n):
        k = wl.preload[i:i + n]
        r = bench.table_rows(k, d)
        kt = torch.from_numpy(k.view(np.int64)).cuda()
        rt = torch.from_numpy(r).cuda()
        c.replace_device(kt.data_ptr(), len(k), rt.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert o.replace(k, r)
    torch.cuda.synchronize()
    resident = c.dump_all()
    assert (resident == o.dump()).all()
    wl.set_resident(resident)
    batches, _, h_draw = wl.batches(h, K, seed=7000 + int(h * 100))
    assert abs(h_draw - h) < 0.02
    qt = [torch.from_numpy(q.view(np.int64)).cuda() for q in batches]
    dr = torch.zeros(d, device="cuda")
    default = np.zeros(d, np.float32)
    b = Bufs(torch, K, n, d)
    sp = c.stream()
    b.issue(c, 0, qt[0], n, dr, sp)
    torch.cuda.synchronize()
    b.check(o, 0, batches[0], default, d, "warm")
    g = hps.StreamGraph(sp)
    with g:
        for j in range(K):
            b.issue(c, j, qt[j], n, dr, sp)
    meas = []
    for rep in range(2):
        g.launch(sp)
        torch.cuda.synchronize()
        for j in range(K):
            uh, um = b.check(o, j, batches[j], default, d, (h, rep, j))
            meas.append(uh / (uh + um))
    assert abs(np.mean(meas) - h) < 0.02
    check_state(c, o)


def test_cfg5_scale_geometry_pipelined_lookups():
    """A cfg-5-scale table geometry (1.6 M slabsets x 2 slabs = 102.4 M slots;
    d = 4 keeps the oracle's host copy small): 8 M preloaded keys from a 1 B
    keyspace, then 20 PDL-chained 65,536-key lookups in one graph, checked
    call by call against the oracle."""
    import torch

    S, W, d, n, K = 1_600_000, 2, 4, 65536, 20
    c = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=W, dimension=d,
                                          worker_pool_size=8, tasks_per_worker=8))
    assert c.capacity() >= 100_000_000
    o = oracle.OracleCache(S, W, d)
    rng = np.random.default_rng(1_000_000_000)
    pre = np.unique(rng.integers(0, 1_000_000_000, 8_400_000, dtype=np.uint64))[:8_000_000]
    rng.shuffle(pre)
    chunk = 1 << 20
    for i in range(0, len(pre), chunk):
        k = pre[i:i + chunk]
        r = bench.table_rows(k, d)
        kt = torch.from_numpy(k.view(np.int64)).cuda()
        rt = torch.from_numpy(r).cuda()
        c.replace_device(kt.data_ptr(), len(k), rt.data_ptr(), torch.cuda.current_stream().cuda_stream)
        assert o.replace(k, r)
    torch.cuda.synchronize()
    assert c.occupied() == o.occupied()
    qs = []
    for j in range(K):
        idx = workload.powerlaw_sample(1.2, len(pre), 11, 100 + j, n).astype(np.int64)
        q = pre[idx]
        absent = rng.random(n) < 0.3
        q[absent] = rng.integers(1_000_000_000, 2_000_000_000, int(absent.sum()), dtype=np.uint64)
        qs.append(q)
    qt = [torch.from_numpy(q.view(np.int64)).cuda() for q in qs]
    dr = torch.full((d,), -1.0, device="cuda")
    default = np.full(d, -1.0, np.float32)
    b = Bufs(torch, K, n, d)
    sp = c.stream()
    b.issue(c, 0, qt[0], n, dr, sp)
    torch.cuda.synchronize()
    b.check(o, 0, qs[0], default, d, "warm")
    g = hps.StreamGraph(sp)
    with g:
        for j in range(K):
            b.issue(c, j, qt[j], n, dr, sp)
    g.launch(sp)
    torch.cuda.synchronize()
    for j in range(K):
        b.check(o, j, qs[j], default, d, j)
    assert c.recency_clock() == o.clock()
    gk, gc, gm, _ = c.export_state()
    ok, oc, om, _ = o.state()
    assert (gm == om).all()
    occ = (np.repeat(gm, 32).reshape(-1, 32) >> np.arange(32, dtype=np.uint32) & 1).reshape(-1) == 1
    assert (gk[occ] == ok[occ]).all() and (gc[occ] == oc[occ]).all()
