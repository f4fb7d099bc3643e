#!/usr/bin/env python
"""Replace and Update at the cfg-2 geometry (S = 31,250 x 2 slabsets, d = 128,
2 M slots) -- the cache-mutation kernels behind the miss path and the
online-update path (SlabCache::replace / update, slab_cache.cpp:93-125).

  python tools/bench_replace.py > profiles/<round>_replace.json

After the bench's preload (2.2 M keys through 64K-key device replaces), timed
with CUDA events on the cache stream:
  replace_fill   -- engine-fill replace (unvalidated, unique keys), 65,536
                    keys per call: half fresh keys (insert / evict), a quarter
                    already resident (recency refresh only), a quarter fresh
                    keys hashing into sets other keys of the call also touch
  replace_user   -- the same through hps_cache_replace (device mode: duplicate
                    check before mutation, host reads the flag)
  replace_relaxed -- the engine-fill replace in the opt-in relaxed mode
                    (hps_cache_set_replace_mode(HPS_REPLACE_RELAXED):
                    atomicCAS slot claims, every key at once), same batch
                    shape, then the invariants checked and the dropped keys
                    counted (run after everything else)
  update_all     -- hps_cache_update_device of every resident row
and the cache state is checked against the oracle at the end when --check.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import torch

    import bench
    import paper_2210_08804_b200 as hps

    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--check", action="store_true")
    ap.add_argument("--only", choices=["all", "relaxed"], default="all",
                    help="relaxed: preload, then only the relaxed leg (profiling)")
    a = ap.parse_args()
    wl = bench.Workload()
    d, n = wl.dim, a.batch
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=wl.S, slabs_per_set=wl.W, dimension=d,
                                              worker_pool_size=8, tasks_per_worker=8))
    st = torch.cuda.ExternalStream(cache.stream())
    sp = st.cuda_stream
    o = None
    if a.check:
        import oracle

        o = oracle.OracleCache(wl.S, wl.W, d)
    for i in range(0, len(wl.preload), 65536):
        k = wl.preload[i:i + 65536]
        r = bench.table_rows(k, d)
        cache.replace_device(torch.from_numpy(k.view(np.int64)).cuda().data_ptr(), len(k),
                             torch.from_numpy(r).cuda().data_ptr(), sp)
        if o is not None:
            o.replace(k, r)
    torch.cuda.synchronize()
    resident = cache.dump_all()
    rng = np.random.default_rng(5)
    fresh = wl.rank_to_key[len(wl.preload):]
    batches = []
    for b in range(2 * a.reps + 3):
        f = fresh[b * n: b * n + n // 2 + n // 4]
        rres = rng.choice(resident, n // 4, replace=False)
        k = np.concatenate([f, rres])
        k = np.unique(k)[:n]
        rng.shuffle(k)
        batches.append((k, bench.table_rows(k, d)))
    dk = [(torch.from_numpy(k.view(np.int64)).cuda(), torch.from_numpy(r).cuda()) for k, r in batches]
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    res = {"geometry": {"S": wl.S, "W": wl.W, "d": d}, "batch": n}

    def timed(fn, reps):
        torch.cuda.synchronize()
        ev[0].record(st)
        for j in range(reps):
            fn(j)
        ev[1].record(st)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) * 1e3 / reps

    if a.only == "relaxed":
        return relaxed_leg(a, cache, batches, dk, sp, timed, res, hps)
    # warm
    cache.replace_fill(dk[0][0].data_ptr(), len(batches[0][0]), dk[0][1].data_ptr(), sp)
    if o is not None:
        o.replace(*batches[0])
    t_fill = timed(lambda j: cache.replace_fill(dk[1 + j][0].data_ptr(), len(batches[1 + j][0]),
                                                dk[1 + j][1].data_ptr(), sp), a.reps)
    if o is not None:
        for j in range(a.reps):
            o.replace(*batches[1 + j])
    res["replace_fill_us"] = t_fill
    res["replace_fill_row_gbs"] = n * d * 4 * 2 / (t_fill * 1e-6) / 1e9
    u = a.reps + 1
    k, r = batches[u]
    t_user = timed(lambda j: cache.replace_device(dk[u][0].data_ptr(), len(k), dk[u][1].data_ptr(),
                                                  sp), 1)
    if o is not None:
        o.replace(k, r)
    res["replace_user_us"] = t_user
    resident = cache.dump_all()
    R = len(resident)
    rk = torch.from_numpy(resident.view(np.int64)).cuda()
    rows = torch.from_numpy(bench.table_rows(resident, d)).cuda()
    written = torch.zeros(1, dtype=torch.int64, device="cuda")
    cache.update_device_async(rk.data_ptr(), R, rows.data_ptr(), written.data_ptr(), sp)
    t_upd = timed(lambda j: cache.update_device_async(rk.data_ptr(), R, rows.data_ptr(),
                                                      written.data_ptr(), sp), 5)
    res["update_all"] = {"rows": R, "us": t_upd, "row_gbs": R * d * 4 / (t_upd * 1e-6) / 1e9}
    if o is not None:
        o.update(resident, bench.table_rows(resident, d))
        gk, gc, gm, gr = cache.export_state()
        ok, oc, om, orow = o.state()
        occ = (np.repeat(gm, 32).reshape(-1, 32) >> np.arange(32, dtype=np.uint32) & 1).reshape(-1) == 1
        res["state_equal"] = bool((gm == om).all() and (gk[occ] == ok[occ]).all()
                                  and (gc[occ] == oc[occ]).all()
                                  and gr.reshape(-1, d)[occ].tobytes() == orow.reshape(-1, d)[occ].tobytes())
    relaxed_leg(a, cache, batches, dk, sp, timed, res, hps)


def relaxed_leg(a, cache, batches, dk, sp, timed, res, hps):
    n = a.batch
    d = cache.dimension()
    # relaxed mode last (the exact-mode state check above is done)
    cache.set_replace_mode(hps.HPS_REPLACE_RELAXED)
    base = a.reps + 2
    cache.replace_fill(dk[base][0].data_ptr(), len(batches[base][0]), dk[base][1].data_ptr(), sp)
    t_rel = timed(lambda j: cache.replace_fill(dk[base + 1 + j][0].data_ptr(),
                                               len(batches[base + 1 + j][0]),
                                               dk[base + 1 + j][1].data_ptr(), sp), a.reps)
    cache.check_invariants()
    res["replace_relaxed_us"] = t_rel
    res["replace_relaxed_row_gbs"] = n * d * 4 * 2 / (t_rel * 1e-6) / 1e9
    res["replace_relaxed_dropped"] = cache.relaxed_dropped()
    res["replace_relaxed_keys"] = int(sum(len(batches[base + j][0]) for j in range(a.reps + 1)))
    print(json.dumps(res))


if __name__ == "__main__":
    main()
