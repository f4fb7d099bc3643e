#!/usr/bin/env python
"""cfg 1 (BASELINE.json configs[0]): the reference's own benchmark shape,
run_bench (core/src/bench.cpp:37-168) -- power-law (alpha 1.2) stream over a
1M-key table, dim 16, cache 10 % of the table (bench.cpp:63-69:
slabsets = ceil(keys / 10 / 64) = 1,563, W = 2), batch 1024, 20,000 batches,
steady state = the last 10 % (bench.cpp:94-95) -- through BOTH lookup
engines on the IDENTICAL key stream:

  * the B200 engine (hps_engine_lookup = LookupEngine::lookup, pinned host
    keys / rows / flags, H2D + D2H inside every call), and
  * the reference LookupEngine compiled from its own sources (oracle/_ref),
    cache worker pool 2 (run_bench's default).

The stream is the reference sampler's (PowerLawSampler, permute seed 42,
draw seed 42 ^ 0x9E3779B97F4A7C15, bench.cpp:33-35, restated bit-exactly
by workload.powerlaw_sample). Both volatile DBs hold the whole table up front
(run_bench starts with the rows in its persistent store and promotes them
into the VDB on first miss; which tier serves a miss does not change the
cache's trajectory). Per threshold (1.0: every batch with a miss takes the
synchronous branch -- deterministic; 0.8: the run_bench default mix of sync
and async batches):

  * per-batch unique-key hit rates of the two engines: exactly equal at
    t = 1.0 (returned rows compared bit-exactly batch by batch too); at
    t = 0.8 the async fill's timing decides which later batch hits, so the
    steady-state hit rate is compared with a tolerance (0.5 points);
  * steady-state latency per batch (host wall clock around the lookup call,
    as run_bench measures), p50 / p99, and keys/s.

  python tools/bench_cfg1.py [--batches 20000] > profiles/r01_cfg1.json
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from tools import workload  # noqa: E402

KEYS, DIM, BATCH, ALPHA, SEED = 1_000_000, 16, 1024, 1.2, 42


def cfg1_stream(batches: int) -> np.ndarray:
    import paper_2210_08804_b200 as hps

    return workload.powerlaw_sample(ALPHA, KEYS, SEED, SEED ^ 0x9E3779B97F4A7C15, batches * BATCH)


def run(threshold: float, batches: int, compare_rows: bool, stream: np.ndarray,
        table_rows: np.ndarray, workers: int = 2) -> dict:
    import torch

    import oracle
    import paper_2210_08804_b200 as hps

    S = max(1, (KEYS // 10 + 63) // 64)
    all_keys = np.arange(KEYS, dtype=np.uint64)
    # ---- B200 engine
    vdb = hps.VolatileStore(os.cpu_count() or 8)
    table = hps.TableId("cfg1", DIM)
    vdb.register_table(table, hps.VolatileTableConfig(partition_count=16, overflow_margin=KEYS))
    vdb.insert("cfg1", all_keys, table_rows)
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=DIM),
                          device=0)
    eng = hps.LookupEngine(table, cache, vdb, None,
                           hps.EngineConfig(hit_rate_threshold=threshold))
    keys_h = torch.empty(BATCH, dtype=torch.int64).pin_memory()
    out_h = torch.empty(BATCH * DIM, dtype=torch.float32).pin_memory()
    flags_h = torch.empty(BATCH, dtype=torch.uint8).pin_memory()
    kv = keys_h.numpy().view(np.uint64)
    # ---- reference engine (its own sources, oracle/_ref)
    ref = oracle.RefEngine(DIM, S, 2, workers, threshold, 16)
    ref.vdb_insert(all_keys, table_rows)

    lat_g = np.empty(batches)
    lat_r = np.empty(batches)
    h_g = np.empty(batches)
    h_r = np.empty(batches)
    sync_g = sync_r = 0
    rows_equal = True
    first_row_mismatch = None
    for it in range(batches):
        b = stream[it * BATCH:(it + 1) * BATCH]
        kv[:] = b
        t0 = time.perf_counter_ns()
        o = eng.lookup_ptrs(keys_h.data_ptr(), BATCH, out_h.data_ptr(), flags_h.data_ptr(),
                            hps.HPS_MEM_HOST)
        t1 = time.perf_counter_ns()
        rout, rflags, ro = ref.lookup(b)
        t2 = time.perf_counter_ns()
        lat_g[it] = (t1 - t0) / 1e3
        lat_r[it] = (t2 - t1) / 1e3
        h_g[it] = o.unique_hit_rate
        h_r[it] = ro["unique_hit_rate"]
        sync_g += int(o.sync_branch)
        sync_r += int(ro["sync_branch"])
        if compare_rows and rows_equal:
            if (out_h.numpy().tobytes() != rout.tobytes()
                    or not np.array_equal(flags_h.numpy(), rflags)):
                rows_equal = False
                first_row_mismatch = it
    eng.drain_async()
    ref.drain()
    steady = slice(batches - max(1, batches // 10), batches)

    def summary(lat, h, sync):
        s = lat[steady]
        return {"steady_latency_us_mean": float(s.mean()),
                "steady_latency_us_p50": float(np.median(s)),
                "steady_latency_us_p99": float(np.percentile(s, 99)),
                "steady_keys_per_s": BATCH / (float(s.mean()) * 1e-6),
                "steady_unique_hit_rate": float(h[steady].mean()),
                "overall_unique_hit_rate": float(h.mean()),
                "sync_batches": sync, "async_batches": batches - sync}

    res = {"threshold": threshold, "batches": batches,
           "b200": summary(lat_g, h_g, sync_g),
           "reference_cpu": dict(summary(lat_r, h_r, sync_r), cache_worker_pool=workers),
           "per_batch_hit_rate_equal": bool(np.array_equal(h_g, h_r)),
           "max_abs_hit_rate_delta": float(np.abs(h_g - h_r).max()),
           "steady_hit_rate_delta": float(h_g[steady].mean() - h_r[steady].mean())}
    if compare_rows:
        res["rows_and_flags_bit_exact_every_batch"] = rows_equal
        res["first_row_mismatch_batch"] = first_row_mismatch
    res["b200_vs_reference_latency"] = (res["reference_cpu"]["steady_latency_us_mean"] /
                                        res["b200"]["steady_latency_us_mean"])
    eng.close()
    return res


def main():
    import bench

    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", type=int, default=20000)
    ap.add_argument("--thresholds", default="1.0,0.8")
    a = ap.parse_args()
    stream = cfg1_stream(a.batches)
    rows = bench.table_rows(np.arange(KEYS, dtype=np.uint64), DIM)
    out = {"config": "cfg1: run_bench shape (bench.cpp:37-168) -- 1M keys, alpha 1.2, dim 16, "
                     "cache 10 % (1,563 x 2 slabsets), batch 1024, steady = last 10 %",
           "host_cores": os.cpu_count(),
           "latency": "host wall clock around one engine lookup call (pinned host buffers; "
                      "H2D, kernels, VDB miss fetch, D2H inside), as run_bench times it",
           "runs": [run(float(t), a.batches, float(t) >= 1.0, stream, rows)
                    for t in a.thresholds.split(",")]}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
