#!/usr/bin/env python
"""Host VDB batch-lookup throughput (the miss path's fetch): a 2M-key d = 128
table (1 GB of rows), 65,536 random keys per call into a pinned destination,
swept over lookup-thread counts.

  python tools/vdb_probe.py [--keys N] > gpurun_out/<tag>/vdb.json
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2210_08804_b200 as hps  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--keys", type=int, default=2_000_000)
    ap.add_argument("--batch", type=int, default=65536)
    a = ap.parse_args()
    import torch

    d = 128
    keys = np.arange(a.keys, dtype=np.uint64) * np.uint64(2654435761)
    rng = np.random.default_rng(0)
    q = np.ascontiguousarray(keys[rng.integers(0, len(keys), a.batch)])
    fk = torch.empty(a.batch, dtype=torch.int64).pin_memory()
    fv = torch.empty(a.batch * d).pin_memory()
    mk = torch.empty(a.batch, dtype=torch.int64).pin_memory()
    nf, nm = C.c_size_t(0), C.c_size_t(0)
    res = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
           "table_keys": a.keys, "batch": a.batch, "dim": d, "by_threads": {}}
    for th in (1, 2, 4, 8, 16, 32, 0):
        if th > 0 and th > 2 * res["affinity"]:
            continue
        v = hps.VolatileStore(th)
        t = hps.TableId("x", d)
        v.register_table(t, hps.VolatileTableConfig(partition_count=16, overflow_margin=1 << 40))
        for i in range(0, len(keys), 1 << 18):
            k = keys[i:i + (1 << 18)]
            v.insert("x", k, bench.table_rows(k, d))
        f = hps.lib().hps_vdb_lookup
        for _ in range(3):
            f(v.handle, b"x", q.ctypes.data, len(q), fk.data_ptr(), fv.data_ptr(), C.byref(nf),
              mk.data_ptr(), C.byref(nm))
        reps = 20
        t0 = time.perf_counter()
        for _ in range(reps):
            f(v.handle, b"x", q.ctypes.data, len(q), fk.data_ptr(), fv.data_ptr(), C.byref(nf),
              mk.data_ptr(), C.byref(nm))
        ms = (time.perf_counter() - t0) * 1e3 / reps
        res["by_threads"][str(th)] = {"ms": ms, "rows_gbs": a.batch * d * 4 / ms / 1e6}
        v.close() if hasattr(v, "close") else None
        del v
    print(json.dumps(res))


if __name__ == "__main__":
    main()
