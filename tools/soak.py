#!/usr/bin/env python
"""Soak test of the serving path (one GPU): several host threads drive ONE
lookup engine concurrently (host and pinned buffers, batch sizes 1 .. 65,536,
power-law keys, every hit-rate branch), while other threads update resident
rows (stream-ordered device updates of rows that stay equal to the table's),
run refresh passes and dump the cache. Every returned row whose flag is 0 is
compared with the table row of its key (rows are a pure function of the
key, so the check holds whatever the interleaving), flagged rows with the
default row; the cache invariants are checked periodically. Runs for
--seconds and prints one JSON line (calls, keys, errors).

  python tools/soak.py --seconds 300
"""
from __future__ import annotations

import argparse
import json
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2210_08804_b200 as hps

    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--keys", type=int, default=2_000_000)
    ap.add_argument("--dim", type=int, default=64)
    ap.add_argument("--threads", type=int, default=4)
    a = ap.parse_args()
    d = a.dim
    K = a.keys
    S = (K // 10) // 64
    table = hps.TableId("soak", d)
    vdb = hps.VolatileStore()
    vdb.register_table(table, hps.VolatileTableConfig(partition_count=16, overflow_margin=1 << 40))
    present = np.arange(0, K, dtype=np.uint64) * np.uint64(3)  # keys 3i; 3i+1 absent everywhere
    for i in range(0, len(present), 1 << 18):
        k = present[i:i + (1 << 18)]
        vdb.insert("soak", k, bench.table_rows(k, d))
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d))
    default = np.full(d, -9.0, np.float32)
    eng = hps.LookupEngine(table, cache, vdb, None,
                           hps.EngineConfig(hit_rate_threshold=0.8, default_vector=list(default)))
    eng.reserve(65536)
    ranks = np.arange(1, K + 1, dtype=np.float64) ** -1.1
    cdf = np.cumsum(ranks)
    cdf /= cdf[-1]
    stop = time.monotonic() + a.seconds
    lock = threading.Lock()
    stats = dict(lookup_calls=0, lookup_keys=0, row_errors=0, flag_errors=0, updates=0,
                 refreshes=0, dumps=0, invariant_checks=0, exceptions=[])

    def record(**kw):
        with lock:
            for k, v in kw.items():
                if k == "exceptions":
                    stats[k].extend(v)
                else:
                    stats[k] += v

    def looker(tid):
        rng = np.random.default_rng(100 + tid)
        sizes = [1, 7, 256, 1024, 4096, 16384, 65536]
        while time.monotonic() < stop:
            try:
                n = int(rng.choice(sizes))
                r = np.searchsorted(cdf, rng.random(n))
                keys = (r.astype(np.uint64) * np.uint64(3) + (rng.random(n) < 0.05).astype(np.uint64))
                pinned = rng.random() < 0.5
                if pinned:
                    kt = torch.from_numpy(keys.view(np.int64)).pin_memory()
                    out = torch.empty(n * d).pin_memory()
                    fl = torch.empty(n, dtype=torch.uint8).pin_memory()
                    eng.lookup_ptrs(kt.data_ptr(), n, out.data_ptr(), fl.data_ptr(),
                                    hps.HPS_MEM_HOST)
                    rows, flags = out.numpy().reshape(-1, d), fl.numpy()
                else:
                    res = eng.lookup(keys)
                    rows, flags = res.vectors.reshape(-1, d), res.miss_flags
                want = bench.table_rows(keys, d).reshape(-1, d)
                ok_rows = flags == 0
                row_err = int((rows[ok_rows] != want[ok_rows]).any(axis=1).sum())
                row_err += int((rows[~ok_rows] != default).any(axis=1).sum())
                flag_err = int(((keys % 3 != 0) & ok_rows).sum())  # absent keys are never hits
                record(lookup_calls=1, lookup_keys=n, row_errors=row_err, flag_errors=flag_err)
            except Exception as e:  # noqa: BLE001
                record(exceptions=[f"lookup: {e!r}"])
                return

    def updater():
        rng = np.random.default_rng(7)
        while time.monotonic() < stop:
            try:
                res = cache.dump_all()
                record(dumps=1)
                if len(res):
                    k = rng.choice(res, min(len(res), 20000), replace=False)
                    # rewrite resident rows with their own (unchanged) values:
                    # concurrent lookups must never see anything else
                    kt = torch.from_numpy(k.view(np.int64)).cuda()
                    rt = torch.from_numpy(bench.table_rows(k, d)).cuda()
                    cache.update_device(kt.data_ptr(), len(k), rt.data_ptr())
                    record(updates=1)
                time.sleep(0.01)
            except Exception as e:  # noqa: BLE001
                record(exceptions=[f"update: {e!r}"])
                return

    def refresher():
        while time.monotonic() < stop:
            try:
                hps.refresh_cache(cache, table, vdb, None, dump_batch_size=65536)
                record(refreshes=1)
                cache.check_invariants()
                record(invariant_checks=1)
                time.sleep(0.5)
            except Exception as e:  # noqa: BLE001
                record(exceptions=[f"refresh: {e!r}"])
                return

    ts = [threading.Thread(target=looker, args=(t,)) for t in range(a.threads)]
    ts += [threading.Thread(target=updater), threading.Thread(target=refresher)]
    t0 = time.monotonic()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    eng.drain_async()
    cache.check_invariants()
    stats["invariant_checks"] += 1
    stats["seconds"] = time.monotonic() - t0
    stats["engine_stats"] = eng.stats().__dict__
    stats["ok"] = (stats["row_errors"] == 0 and stats["flag_errors"] == 0
                   and not stats["exceptions"])
    print(json.dumps(stats))
    return 0 if stats["ok"] else 1


if __name__ == "__main__":
    sys.exit(main())
