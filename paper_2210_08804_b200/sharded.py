"""Key-hash-sharded lookup over torch.distributed.

For tables larger than one GPU's HBM: rank r of G holds the shard of keys
with ``shard_of(key, G) == r`` (``hps_shard_of``; its own seed, not the
slabset seed) in its own :class:`SlabCache`. A lookup is collective -- every
rank calls it with its own batch:

1. route: per-owner counts and the keys scattered into per-owner segments
   (CUDA kernels ``hps_shard_count`` / ``hps_shard_scatter``; original
   positions ride along);
2. exchange: the counts, then the keys (all-to-all; NCCL over NVLink on the
   GPU box, gloo in the CPU tests);
3. each owner runs ONE lookup of everything it received -- either the bare
   cache lookup (``cache_local_lookup``: ``hps_cache_lookup_device``, probe,
   recency, rows, default rows for misses, the owner's unique misses handed
   back), or the whole lookup engine (``engine_local_lookup``:
   ``hps_engine_lookup`` on device pointers -- dedup, query, the hit-rate
   switch, the tier fetch of the owner's unique misses from the host VDB,
   scatter, replace or background fill: the owner fills its own shard with
   the reference's LookupEngine semantics, lookup_engine.cpp:130-241);
4. exchange back: rows and miss flags (reverse all-to-all);
5. unroute: rows to the requester's original positions
   (``hps_shard_unroute``).

One host synchronisation per lookup: the per-owner counts are exchanged on
the device and read back together (the all-to-all split sizes must be host
values). The only collectives are these exchanges; the replica mode (one full cache
per GPU, ``bench.py --gpus N``) has none. There is no reference counterpart:
the reference is single-process and the paper deploys replicas
(PAPER.md:809).

The device ops and the local lookup are injectable (``ops``,
``local_lookup``) so the orchestration runs under gloo on CPU in the tests.
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np

from . import HPS_MEM_DEVICE, _check, lib  # noqa: F401  (re-exported helpers)


def shard_of(keys, world: int) -> np.ndarray:
    """Owner rank of each key (host; same function as the device kernels)."""
    k = np.ascontiguousarray(keys, dtype=np.uint64)
    f = lib().hps_shard_of
    return np.fromiter((f(int(x), world) for x in k), dtype=np.int64, count=len(k))


class ShardOps:
    """Routing kernels of one rank (device pointers, torch CUDA tensors)."""

    def __init__(self, device: int = 0):
        self.device = device

    def _stream(self):
        import torch

        return torch.cuda.current_stream(self.device).cuda_stream

    def count(self, keys, world: int):
        import torch

        counts = torch.empty(world, dtype=torch.int64, device=keys.device)
        _check(lib().hps_shard_count(self.device, keys.data_ptr(), keys.numel(), world,
                                     counts.data_ptr(), self._stream()))
        return counts

    def scatter(self, keys, world: int, offsets):
        import torch

        send_keys = torch.empty_like(keys)
        send_pos = torch.empty(keys.numel(), dtype=torch.int32, device=keys.device)
        cursor = offsets.clone()
        _check(lib().hps_shard_scatter(self.device, keys.data_ptr(), keys.numel(), world,
                                       cursor.data_ptr(), send_keys.data_ptr(),
                                       send_pos.data_ptr(), self._stream()))
        return send_keys, send_pos

    def unroute(self, send_pos, rows, flags_in, out, flags_out, dim: int):
        _check(lib().hps_shard_unroute(self.device, send_pos.numel(), dim, send_pos.data_ptr(),
                                       rows.data_ptr(), flags_in.data_ptr(), out.data_ptr(),
                                       flags_out.data_ptr(), self._stream()))


def cache_local_lookup(cache, device: int = 0) -> Callable:
    """The owner-side lookup on a local shard: one hps_cache_lookup_device on
    the received keys. Returns (rows, flags, miss_keys, miss_firsts, counts)."""

    def run(keys, default_row):
        import torch

        n = keys.numel()
        d = cache.dimension()
        rows = torch.empty(max(n, 1) * d, device=keys.device)
        flags = torch.empty(max(n, 1), dtype=torch.uint8, device=keys.device)
        mk = torch.empty(max(n, 1), dtype=torch.int64, device=keys.device)
        mf = torch.empty(max(n, 1), dtype=torch.int32, device=keys.device)
        cnt = torch.zeros(2, dtype=torch.int64, device=keys.device)
        st = torch.cuda.current_stream(device).cuda_stream
        cache.lookup_device(keys.data_ptr(), n, rows.data_ptr(), flags.data_ptr(),
                            default_row.data_ptr(), mk.data_ptr(), mf.data_ptr(), cnt.data_ptr(),
                            st)
        return rows[: n * d], flags[:n], mk, mf, cnt

    return run


def engine_local_lookup(engine, device: int = 0) -> Callable:
    """The owner-side lookup through a full LookupEngine over the owner's
    shard cache (hps_engine_lookup, HPS_MEM_DEVICE): misses are fetched from
    the engine's tiers and admitted into the owner's shard (sync branch) or
    filled in the background (async branch), exactly as a single-GPU engine
    does (lookup_engine.cpp:130-241). The engine's configured default vector
    is used for absent keys. Returns (rows, flags, outcome)."""

    def run(keys, default_row):
        import torch

        n = keys.numel()
        d = engine.table.dimension
        rows = torch.empty(max(n, 1) * d, device=keys.device)
        flags = torch.empty(max(n, 1), dtype=torch.uint8, device=keys.device)
        st = torch.cuda.current_stream(device).cuda_stream
        o = engine.lookup_ptrs(keys.data_ptr(), n, rows.data_ptr(), flags.data_ptr(),
                               HPS_MEM_DEVICE, st)
        return rows[: n * d], flags[:n], o

    return run


class ShardedLookup:
    """Collective lookup over a key-hash-sharded cache (see module doc)."""

    def __init__(self, dim: int, local_lookup: Callable, group=None, ops=None, device: int = 0):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.dim = dim
        self.local_lookup = local_lookup
        self.ops = ops if ops is not None else ShardOps(device)

    def lookup(self, keys, default_row):
        """keys: int64 tensor of this rank's batch. Returns (rows [n*dim],
        miss flags [n], owner_side) where owner_side is what THIS rank's
        shard lookup returned besides rows and flags: (miss_keys,
        miss_firsts, counts) for cache_local_lookup (its unique misses, to be
        fetched and replaced by this rank), (outcome,) for
        engine_local_lookup (misses already fetched / admitted)."""
        import torch

        dist, G, d = self.dist, self.world, self.dim
        n = keys.numel()
        counts = self.ops.count(keys, G)
        recv_counts = torch.empty_like(counts)
        dist.all_to_all_single(recv_counts, counts, group=self.group)
        offsets = torch.zeros_like(counts)
        if G > 1:
            offsets[1:] = torch.cumsum(counts, 0)[:-1]
        send_keys, send_pos = self.ops.scatter(keys, G, offsets)
        # the one host synchronisation: both split vectors at once
        splits = torch.cat([counts, recv_counts]).cpu().tolist()
        send_splits, recv_splits = splits[:G], splits[G:]
        recv_keys = torch.empty(sum(recv_splits), dtype=keys.dtype, device=keys.device)
        dist.all_to_all_single(recv_keys, send_keys, recv_splits, send_splits, group=self.group)
        rows, flags, *owner_side = self.local_lookup(recv_keys, default_row)
        back_rows = torch.empty(n * d, dtype=rows.dtype, device=keys.device)
        dist.all_to_all_single(back_rows.view(-1, d) if n else back_rows,
                               rows.view(-1, d) if rows.numel() else rows,
                               send_splits, recv_splits, group=self.group)
        back_flags = torch.empty(n, dtype=torch.uint8, device=keys.device)
        dist.all_to_all_single(back_flags, flags.contiguous(), send_splits, recv_splits,
                               group=self.group)
        out = torch.empty(n * d, dtype=rows.dtype, device=keys.device)
        flags_out = torch.empty(n, dtype=torch.uint8, device=keys.device)
        self.ops.unroute(send_pos, back_rows, back_flags, out, flags_out, d)
        return out, flags_out, tuple(owner_side)


class PeerShardedLookup:
    """The key-hash-sharded lookup over PEER MEMORY (SURVEY §8e's B200-native
    alternative; include/hps_b200.h hps_peer_*): each rank exports its shard
    cache, the blobs are exchanged once (``all_gather_object``), and every
    rank maps every shard. A lookup is then ONE kernel on the requester --
    route, probe the owner's slabs, stamp, copy the owner's row over NVLink
    into the local output, append misses to the owner's inbox -- with no
    collective on the data path. ``fill`` is the owner side: between lookup
    phases (a barrier on each side) every owner drains its inbox, fetches the
    keys from its tiers and admits them into its shard."""

    def __init__(self, cache, group=None, inbox_cap: int = 1 << 20, device: int = 0):
        import ctypes as C

        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.cache = cache
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = device
        self.inbox_cap = inbox_cap
        blob = cache.peer_export(inbox_cap)
        blobs = [None] * self.world
        dist.all_gather_object(blobs, blob, group=group)
        self._blobs = b"".join(blobs)
        self._h = C.c_void_p()
        _check(lib().hps_peer_group_create(cache.handle, self.rank, self.world, self._blobs,
                                           len(blob), C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None):
            lib().hps_peer_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def lookup(self, keys, default_row, stream: int = 0):
        """keys: int64 CUDA tensor of this rank's batch; default_row: float32
        CUDA tensor of dim floats. Returns (rows [n*dim], miss flags [n]) --
        stream-ordered on `stream` (default: the current stream)."""
        import torch

        n = keys.numel()
        d = self.cache.dimension()
        out = torch.empty(max(n, 1) * d, device=keys.device)
        flags = torch.empty(max(n, 1), dtype=torch.uint8, device=keys.device)
        st = stream or torch.cuda.current_stream(self.device).cuda_stream
        _check(lib().hps_peer_lookup_device(self._h, keys.data_ptr(), n, out.data_ptr(),
                                            flags.data_ptr(), default_row.data_ptr(), st))
        return out[: n * d], flags[:n]

    def fill(self, fetch: Callable) -> int:
        """Owner side, collective: after every rank's lookups (barrier), drain
        this shard's inbox, fetch its unique keys (``fetch(keys) -> (found
        keys, rows)``, e.g. a VolatileStore lookup) and admit them; a second
        barrier before anyone looks up again. Returns the keys admitted."""
        import torch

        torch.cuda.synchronize(self.device)
        self.dist.barrier(group=self.group)
        keys = np.unique(self.cache.peer_drain(self.inbox_cap))
        admitted = 0
        if len(keys):
            fk, rows = fetch(keys)
            if len(fk):
                self.cache.replace(fk, rows)
                admitted = len(fk)
        self.dist.barrier(group=self.group)
        return admitted
