"""Key-hash-sharded mode and the multi-rank path.

* CPU, gloo, world size 2 (and 3): the collective orchestration of
  paper_2210_08804_b200/sharded.py with CPU stand-ins for the routing kernels
  and an oracle-backed shard lookup per rank -- every rank's rows and miss
  flags must equal what the owner shards hold, whatever the routing order.
* GPU: the routing kernels (count / scatter / unroute) against numpy, and a
  world-size-1 NCCL run of the whole path against the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2210_08804_b200 as hps
from paper_2210_08804_b200 import sharded

D = 8
KEYSPACE = 4000


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def key_rows(keys):
    k = np.asarray(keys, dtype=np.float64)
    return (k[:, None] * 0.5 + np.arange(D)[None, :]).astype(np.float32).reshape(-1)


class CpuOps:
    """CPU stand-ins for ShardOps (same contract; owners from the product's
    host hash hps_shard_of)."""

    def count(self, keys, world):
        own = sharded.shard_of(keys.numpy().view(np.uint64), world)
        return torch.from_numpy(np.bincount(own, minlength=world).astype(np.int64))

    def scatter(self, keys, world, offsets):
        k = keys.numpy().view(np.uint64)
        own = sharded.shard_of(k, world)
        # deliberately NOT input order inside a segment: the carried
        # positions must undo any order
        order = np.lexsort((-np.arange(len(k)), own))
        return (torch.from_numpy(k[order].view(np.int64).copy()),
                torch.from_numpy(order.astype(np.int32)))

    def unroute(self, send_pos, rows, flags_in, out, flags_out, dim):
        p = send_pos.numpy().astype(np.int64)
        out.view(-1, dim)[torch.from_numpy(p)] = rows.view(-1, dim)
        flags_out[torch.from_numpy(p)] = flags_in


def oracle_shard_lookup(shard: "oracle.OracleCache", default):
    def run(keys, default_row):
        k = keys.numpy().view(np.uint64)
        uniq, inv = oracle.dedup(k)
        ws = np.zeros(len(uniq) * D, np.float32)
        hit = shard.query(uniq, ws)
        ws = ws.reshape(-1, D)
        ws[hit == 0] = default
        rows = torch.from_numpy(ws[inv].reshape(-1).copy())
        flags = torch.from_numpy((1 - hit)[inv].astype(np.uint8))
        miss = uniq[hit == 0]
        cnt = torch.tensor([int(hit.sum()), len(miss)], dtype=torch.int64)
        return rows, flags, torch.from_numpy(miss.view(np.int64).copy()), None, cnt
    return run


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        table = rng.choice(KEYSPACE, 1500, replace=False).astype(np.uint64)
        own = sharded.shard_of(table, world)
        mine = table[own == rank]
        shard = oracle.OracleCache(64, 2, D)
        shard.replace(mine, key_rows(mine))
        default = np.full(D, -1.0, np.float32)
        sl = sharded.ShardedLookup(D, oracle_shard_lookup(shard, default), ops=CpuOps())
        resident = set(int(k) for k in table)  # every key lives on exactly one owner
        ok = True
        for b in range(3):
            brng = np.random.default_rng(100 * rank + b)
            batch = brng.integers(0, KEYSPACE, 700 + 97 * rank, dtype=np.uint64)
            batch[:5] = batch[5:10]  # duplicates within the batch
            out, flags, (mk, _, cnt) = sl.lookup(torch.from_numpy(batch.view(np.int64)),
                                                 torch.from_numpy(default))
            # each owner's shard must hold the keys it owns (capacity is
            # 4096 slots, no eviction at 1500 keys)
            in_cache = np.array([int(k) in resident for k in batch])
            want = key_rows(batch).reshape(-1, D)
            want[~in_cache] = default
            ok &= out.numpy().reshape(-1, D).tobytes() == want.tobytes()
            ok &= (flags.numpy() == (~in_cache).astype(np.uint8)).all()
            # owner-side unique misses are keys this rank owns
            ok &= bool((sharded.shard_of(mk.numpy().view(np.uint64), world) == rank).all())
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


def engine_oracle_lookup(eo: "oracle.EngineOracle"):
    """CPU stand-in for engine_local_lookup: the owner's whole LookupEngine
    (EngineOracle: dedup, query, hit-rate switch, tier fetch, replace)."""
    def run(keys, default_row):
        out, flags, oc = eo.lookup(keys.numpy().view(np.uint64))
        eo.drain_async()
        return torch.from_numpy(out.copy()), torch.from_numpy(flags.astype(np.uint8)), oc
    return run


def _engine_worker(rank, world, port, threshold, q):
    """Owner-side miss fill: every owner runs an engine over its shard with
    the VDB behind it; the requester's rows must be the VDB rows (flag 0) or
    the default (flag 1: absent, or an async-branch miss), and the owners
    must have admitted the keys they fetched."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        default = np.full(D, -2.0, np.float32)
        eo = oracle.EngineOracle(256, 2, D, threshold=threshold, default_vector=list(default))
        vdb_keys = np.arange(0, KEYSPACE, 2, dtype=np.uint64)  # odd keys absent everywhere
        mine = vdb_keys[sharded.shard_of(vdb_keys, world) == rank]
        for k, r in zip(mine, key_rows(mine).reshape(-1, D)):
            eo.vdb[int(k)] = r
        sl = sharded.ShardedLookup(D, engine_oracle_lookup(eo), ops=CpuOps())
        ok = True
        for b in range(4):
            brng = np.random.default_rng(1000 * rank + b)
            batch = brng.integers(0, KEYSPACE, 500 + 61 * rank, dtype=np.uint64)
            out, flags, (oc,) = sl.lookup(torch.from_numpy(batch.view(np.int64)),
                                          torch.from_numpy(default))
            got = out.numpy().reshape(-1, D)
            fl = flags.numpy()
            want = key_rows(batch).reshape(-1, D)
            present = batch % 2 == 0
            ok &= bool((got[fl == 0] == want[fl == 0]).all())
            ok &= bool((got[fl == 1] == default).all())
            ok &= bool((fl[~present] == 1).all())
            if threshold >= 1.0:  # every batch with a miss takes the sync branch
                ok &= bool((fl[present] == 0).all())
        # owner-side fill: every present key this rank owns that was looked
        # up (by anyone) is resident in its shard now (no eviction at 512 slots)
        ok &= eo.cache.occupied() > 0 and eo.stats["vdb_hits"] == eo.cache.occupied()
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("threshold", [1.0, 0.6])
def test_sharded_engine_owner_side_fill_gloo(threshold):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = free_port()
    procs = [ctx.Process(target=_engine_worker, args=(r, world, port, threshold, q))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get() for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_lookup_orchestration_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get() for _ in range(world))
    assert all(p.exitcode == 0 for p in procs)
    assert all(res[r] for r in range(world)), res


def test_shard_hash_is_balanced_and_independent_of_placement():
    """Owners spread evenly, and the owner hash is not the slabset hash: a
    shard's keys still fill all of its slabsets."""
    keys = np.arange(200000, dtype=np.uint64) * 2654435761 % (1 << 40)
    for world in (2, 4, 8):
        own = sharded.shard_of(keys, world)
        frac = np.bincount(own, minlength=world) / len(keys)
        assert np.all(np.abs(frac - 1 / world) < 0.01)
    own = sharded.shard_of(keys, 8)
    sets = np.array([oracle.slabset_of(int(k), 64) for k in keys[own == 3][:20000]])
    assert len(np.unique(sets)) == 64


@pytest.mark.gpu
def test_routing_kernels_match_numpy():
    ops = sharded.ShardOps(0)
    rng = np.random.default_rng(3)
    for n, world in [(1, 4), (1000, 2), (65536, 8), (4097, 5)]:
        k = rng.integers(0, 2**63, n, dtype=np.uint64)
        kt = torch.from_numpy(k.view(np.int64)).cuda()
        counts = ops.count(kt, world)
        own = sharded.shard_of(k, world)
        assert (counts.cpu().numpy() == np.bincount(own, minlength=world)).all()
        offsets = torch.zeros_like(counts)
        offsets[1:] = torch.cumsum(counts, 0)[:-1]
        sk, sp = ops.scatter(kt, world, offsets)
        sk, sp = sk.cpu().numpy().view(np.uint64), sp.cpu().numpy()
        assert (sk == k[sp]).all() and (np.sort(sp) == np.arange(n)).all()
        off = offsets.cpu().numpy()
        for o in range(world):
            seg = sk[off[o]: off[o] + counts[o].item()]
            assert (sharded.shard_of(seg, world) == o).all()
        rows = torch.from_numpy(key_rows(sk)).cuda()
        fl_in = torch.from_numpy((sk % 2).astype(np.uint8)).cuda()
        out = torch.empty(n * D, device="cuda")
        fl = torch.empty(n, dtype=torch.uint8, device="cuda")
        ops.unroute(torch.from_numpy(sp).cuda(), rows, fl_in, out, fl, D)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == key_rows(k).tobytes()
        assert (fl.cpu().numpy() == (k % 2)).all()


@pytest.mark.gpu
def test_sharded_lookup_world_one_nccl_matches_oracle():
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        S, W = 64, 2
        cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=W, dimension=D))
        o = oracle.OracleCache(S, W, D)
        rng = np.random.default_rng(5)
        keys = rng.choice(KEYSPACE, 1500, replace=False).astype(np.uint64)
        cache.replace(keys, key_rows(keys))
        o.replace(keys, key_rows(keys))
        default = np.full(D, 3.0, np.float32)
        sl = sharded.ShardedLookup(D, sharded.cache_local_lookup(cache))
        for b in range(3):
            q = rng.integers(0, KEYSPACE, 3000, dtype=np.uint64)
            out, fl, (mk, mf, cnt) = sl.lookup(torch.from_numpy(q.view(np.int64)).cuda(),
                                               torch.from_numpy(default).cuda())
            torch.cuda.synchronize()
            uniq, inv = oracle.dedup(q)
            ws = np.zeros(len(uniq) * D, np.float32)
            hit = o.query(uniq, ws)
            ws = ws.reshape(-1, D)
            ws[hit == 0] = default
            assert out.cpu().numpy().tobytes() == ws[inv].reshape(-1).tobytes()
            assert (fl.cpu().numpy() == (1 - hit)[inv]).all()
            um = int((hit == 0).sum())
            assert cnt.cpu().tolist() == [len(uniq) - um, um]
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_engine_lookup_world_one_nccl_matches_engine_oracle():
    """engine_local_lookup on B200 (NCCL, world 1): the owner's engine
    fetches its misses from the host VDB and admits them; outcomes, rows and
    flags equal the engine oracle's (no eviction, so the routing order inside
    a segment does not change which keys are resident)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        S, W, thr = 256, 2, 0.7
        table = hps.TableId("t", D)
        vdb = hps.VolatileStore()
        vdb.register_table(table)
        vk = np.arange(0, KEYSPACE, 2, dtype=np.uint64)
        vdb.insert("t", vk, key_rows(vk))
        eo = oracle.EngineOracle(S, W, D, threshold=thr, default_vector=[4.0])
        for k, r in zip(vk, key_rows(vk).reshape(-1, D)):
            eo.vdb[int(k)] = r
        cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=W, dimension=D))
        eng = hps.LookupEngine(table, cache, vdb, None,
                               hps.EngineConfig(hit_rate_threshold=thr, default_vector=[4.0]))
        sl = sharded.ShardedLookup(D, sharded.engine_local_lookup(eng))
        rng = np.random.default_rng(9)
        dflt = torch.zeros(D, device="cuda")
        for b in range(6):
            q = rng.integers(0, KEYSPACE // 4, 2000, dtype=np.uint64)
            out, fl, (oc,) = sl.lookup(torch.from_numpy(q.view(np.int64)).cuda(), dflt)
            eng.drain_async()
            torch.cuda.synchronize()
            want, wflags, woc = eo.lookup(q)
            eo.drain_async()
            assert oc.__dict__ == woc
            assert out.cpu().numpy().tobytes() == want.tobytes()
            assert (fl.cpu().numpy() == wflags).all()
        cache.check_invariants()
        assert cache.occupied() == eo.cache.occupied()
    finally:
        dist.destroy_process_group()


def _peer_worker(rank, world, port, q):
    """Peer-memory sharded lookup (hps_peer_*): `world` processes on cuda:0,
    each owning one shard; the shards are mapped through CUDA IPC (NVLink peer
    memory on a multi-GPU node). Every position's row / flag must equal what
    its owner shard holds; the owners admit their inboxes between steps."""
    import faulthandler
    import sys
    import traceback

    # a stuck worker dumps its stack and exits instead of hanging the suite
    faulthandler.dump_traceback_later(150, exit=True, file=sys.stderr)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=__import__("datetime").timedelta(seconds=120))
    try:
        torch.cuda.set_device(0)
        cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=64, slabs_per_set=2, dimension=D))
        peer = sharded.PeerShardedLookup(cache, inbox_cap=1 << 14)
        vdb = {int(k): r for k, r in zip(range(0, KEYSPACE, 2),
                                         key_rows(np.arange(0, KEYSPACE, 2)).reshape(-1, D))}

        def fetch(keys):
            fk = np.array([k for k in keys if int(k) in vdb], dtype=np.uint64)
            rows = (np.concatenate([vdb[int(k)] for k in fk]) if len(fk)
                    else np.empty(0, np.float32))
            return fk, rows.astype(np.float32)

        default = torch.full((D,), -7.0, device="cuda")
        resident = set()
        ok = True
        for step in range(4):
            rng = np.random.default_rng(500 * rank + step)
            batch = rng.integers(0, KEYSPACE, 1500 + 111 * rank, dtype=np.uint64)
            batch[:4] = [0, 2, 4, 6]  # shared across ranks: duplicates across requesters
            out, fl = peer.lookup(torch.from_numpy(batch.view(np.int64)).cuda(), default)
            torch.cuda.synchronize()
            got = out.cpu().numpy().reshape(-1, D)
            flags = fl.cpu().numpy()
            res = np.array([int(k) in resident for k in batch])
            want = key_rows(batch).reshape(-1, D)
            want[~res] = -7.0
            ok &= got.tobytes() == want.tobytes()
            ok &= bool((flags == (~res).astype(np.uint8)).all())
            admitted = peer.fill(fetch)
            # recency: every call ticked this shard's clock once (all ranks
            # looked up `step + 1` times), the fill stamped with it, and no
            # counter is newer than the clock
            ok &= cache.recency_clock() == world * (step + 1)
            _, ctrs, masks, _ = cache.export_state()
            occ = (np.repeat(masks, 32).reshape(-1, 32)
                   >> np.arange(32, dtype=np.uint32) & 1).reshape(-1) == 1
            if occ.any():
                top = int(ctrs[occ].max())
                ok &= top <= cache.recency_clock()
                if admitted:
                    ok &= top == cache.recency_clock()
            every = [None] * world
            dist.all_gather_object(every, [int(k) for k in batch])
            new_even = set(k for b in every for k in b if k % 2 == 0) - resident
            owners = sharded.shard_of(np.array(sorted(new_even), dtype=np.uint64), world)
            ok &= admitted == int((owners == rank).sum())
            resident |= new_even
        cache.check_invariants()
        # the shard holds exactly the even keys it owns that anyone asked for
        mine = set(int(k) for k in cache.dump_all())
        ok &= mine == set(k for k in resident
                          if sharded.shard_of(np.array([k], np.uint64), world)[0] == rank)
        peer.close()
        q.put((rank, bool(ok)))
    except Exception:
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3])
def test_peer_memory_sharded_lookup_two_processes_one_gpu(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, v = q.get(timeout=240)
            res[r] = v
    finally:
        for p in procs:
            p.join(30)
            if p.is_alive():
                p.kill()
    assert all(res.get(r) is True for r in range(world)), res
    assert all(p.exitcode == 0 for p in procs)


@pytest.mark.gpu
def test_peer_inbox_overflow_is_counted_and_bounded():
    """An owner's inbox holds inbox_cap keys between drains: appends beyond it
    are dropped but counted (the drain reports how many were appended), and
    the inbox is empty again after the drain."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=8, slabs_per_set=2, dimension=D))
        peer = sharded.PeerShardedLookup(cache, inbox_cap=16)
        keys = torch.arange(1000, dtype=torch.int64, device="cuda") * 7 + 3
        default = torch.zeros(D, device="cuda")
        out, fl = peer.lookup(keys, default)
        torch.cuda.synchronize()
        assert int(fl.sum().item()) == 1000  # empty shard: every key misses
        import ctypes as C

        buf = np.empty(16, dtype=np.uint64)
        n = C.c_size_t(0)
        assert hps.lib().hps_cache_peer_drain(cache.handle, buf.ctypes.data, 16, C.byref(n)) == 0
        assert n.value == 1000  # one append per distinct key of a warp: all distinct here
        assert set(int(k) for k in buf) <= set(range(3, 7000, 7))
        assert len(cache.peer_drain(16)) == 0  # empty after the drain
        peer.close()
    finally:
        dist.destroy_process_group()
