#!/usr/bin/env python
"""Peer-memory sharded lookup timing (hps_peer_*): WORLD
processes, rank r on GPU r % device_count (all on GPU 0 on a one-GPU box,
where the "peer" accesses are CUDA-IPC mappings of the same HBM). Each rank
owns 1/WORLD of the key space in a shard cache (cfg-2 geometry split over
the ranks), the shards are preloaded with every key they own from a 10 M-key
power-law table's hot ranks, and each rank then times --steps lookups of its
own 65,536-key power-law batches (CUDA events on its stream, after a
barrier). Prints one JSON line per rank (rank 0 adds the aggregate).

  python tools/bench_peer.py --world 2
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def worker(rank, a, port, q):
    import torch
    import torch.distributed as dist

    import bench
    import paper_2210_08804_b200 as hps
    from paper_2210_08804_b200 import sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=a.world)
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    wl = bench.Workload()
    d, n = wl.dim, wl.batch
    S = (wl.S + a.world - 1) // a.world
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=wl.W, dimension=d),
                          device=dev)
    own = sharded.shard_of(wl.preload, a.world) == rank
    mine = wl.preload[own]
    for i in range(0, len(mine), 65536):
        k = mine[i:i + 65536]
        cache.replace(k, bench.table_rows(k, d))
    peer = sharded.PeerShardedLookup(cache, inbox_cap=1 << 22, device=dev)
    parts = [None] * a.world
    dist.all_gather_object(parts, cache.dump_all())
    wl.set_resident(np.concatenate(parts))
    batches, _, _ = wl.batches(0.9, 16, seed=77 + rank)
    dk = [torch.from_numpy(b.view(np.int64)).cuda(dev) for b in batches]
    default = torch.zeros(d, device=f"cuda:{dev}")
    st = torch.cuda.current_stream(dev)
    for s in range(a.warmup):
        peer.lookup(dk[s % 16], default)
    torch.cuda.synchronize(dev)
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time

    e0.record(st)
    h0 = time.perf_counter()
    for s in range(a.steps):
        out, fl = peer.lookup(dk[s % 16], default)
    host_us = (time.perf_counter() - h0) * 1e6 / a.steps
    e1.record(st)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1) / a.steps
    miss = float(fl.float().mean().item())
    dist.barrier()
    peer.close()
    q.put({"rank": rank, "device": dev, "ms_per_step": ms, "keys_per_s": n / (ms * 1e-3),
           "host_issue_us_per_call": host_us,
           "miss_fraction_positions": miss})
    dist.destroy_process_group()


def main():
    import torch.multiprocessing as mp

    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=2)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    a = ap.parse_args()
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    procs = [ctx.Process(target=worker, args=(r, a, port, q)) for r in range(a.world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join()
    res = sorted([q.get() for _ in range(a.world)], key=lambda r: r["rank"])
    agg = sum(r["keys_per_s"] for r in res)
    print(json.dumps({"world": a.world, "per_rank": res, "aggregate_keys_per_s": agg,
                      "note": "ranks share one GPU when the box has fewer GPUs than ranks"}))


if __name__ == "__main__":
    main()
