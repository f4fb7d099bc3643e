#!/usr/bin/env python
"""CUPTI trace (torch.profiler) of 50 steady-state cfg-1 engine lookups: every
kernel and copy of the small-batch engine path with its duration.

  mkdir -p gpurun_out/c1; python tools/prof_engine_cfg1.py <threshold>
"""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
import paper_2210_08804_b200 as hps
from tools.bench_cfg1 import cfg1_stream, KEYS, DIM, BATCH
thr = float(sys.argv[1])
S = (KEYS // 10 + 63) // 64
stream = cfg1_stream(3000)
rows = bench.table_rows(np.arange(KEYS, dtype=np.uint64), DIM)
vdb = hps.VolatileStore(os.cpu_count() or 8)
table = hps.TableId("cfg1", DIM)
vdb.register_table(table, hps.VolatileTableConfig(partition_count=16, overflow_margin=KEYS))
vdb.insert("cfg1", np.arange(KEYS, dtype=np.uint64), rows)
cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=DIM), device=0)
eng = hps.LookupEngine(table, cache, vdb, None, hps.EngineConfig(hit_rate_threshold=thr))
kh = torch.empty(BATCH, dtype=torch.int64).pin_memory(); oh = torch.empty(BATCH*DIM).pin_memory(); fh = torch.empty(BATCH, dtype=torch.uint8).pin_memory()
kv = kh.numpy().view(np.uint64)
def one(it):
    kv[:] = stream[it*BATCH:(it+1)*BATCH]
    t0 = time.perf_counter_ns()
    eng.lookup_ptrs(kh.data_ptr(), BATCH, oh.data_ptr(), fh.data_ptr(), hps.HPS_MEM_HOST)
    return (time.perf_counter_ns() - t0) / 1e3
for it in range(2900): one(it)
from torch.profiler import profile, ProfilerActivity
lat = []
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as p:
    for it in range(2900, 2950): lat.append(one(it))
print("lat us", np.median(lat))
p.export_chrome_trace(f"gpurun_out/c1/trace_{thr}.json")
