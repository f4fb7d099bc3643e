"""Diagnostic: native refresh timing vs VDB lookup threads (cfg-2 sized)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2210_08804_b200 as hps

wl = bench.Workload()
d = wl.dim
cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=wl.S, slabs_per_set=2, dimension=d), device=0)
for i in range(0, len(wl.preload), 65536):
    k = wl.preload[i:i + 65536]
    cache.replace(k, bench.table_rows(k, d))
res = cache.dump_all()
for threads in (8, 16):
    v = hps.VolatileStore(threads)
    t = hps.TableId("r", d)
    v.register_table(t, hps.VolatileTableConfig(partition_count=16, overflow_margin=1 << 40))
    for i in range(0, len(res), 1 << 18):
        k = res[i:i + (1 << 18)]
        v.insert("r", k, bench.table_rows(k, d))
    for rep in range(2):
        t0 = time.perf_counter()
        out = hps.refresh_cache(cache, t, v, None, dump_batch_size=65536)
        print(f"threads {threads} rep {rep}: {(time.perf_counter() - t0) * 1e3:.1f} ms, refreshed {out.refreshed}")
    v.close()
