#!/usr/bin/env python
"""Phase timeline of the lookup kernel inside the bench's graph (diagnostic).

  HPSB_TRACE=1 python tools/trace_lookup.py [--steps 200] [--hit 0.9]

Runs the bench.py cfg-2 workload through hps_cache_lookup_device, captured
in one CUDA graph like the bench, and prints the median per-call timeline
(us, relative to the call's first block start) and the start-to-start gap
between consecutive calls."""
import argparse
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
if "--no-trace" in sys.argv:  # just run the graph once (e.g. under ncu --graph-profiling graph)
    os.environ.pop("HPSB_TRACE", None)
else:
    os.environ.setdefault("HPSB_TRACE", "1")


def main():
    import torch

    import bench
    import paper_2210_08804_b200 as hps

    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--hit", type=float, default=0.9)
    ap.add_argument("--no-trace", action="store_true")
    a = ap.parse_args()
    wl = bench.Workload()
    d, n = wl.dim, wl.batch
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=wl.S, slabs_per_set=wl.W, dimension=d),
                          device=0)
    for i in range(0, len(wl.preload), n):
        k = wl.preload[i:i + n]
        cache.replace(k, bench.table_rows(k, d))
    wl.set_resident(cache.dump_all())
    batches, _, _ = wl.batches(a.hit, 32, 7)
    dk = [torch.from_numpy(b.view(np.int64)).cuda() for b in batches]
    outs = [torch.empty(n * d, device="cuda") for _ in range(8)]
    fl = torch.empty(n, dtype=torch.uint8, device="cuda")
    mk = torch.empty(n, dtype=torch.int64, device="cuda")
    mf = torch.empty(n, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(2 * a.steps, dtype=torch.int64, device="cuda")
    dr = torch.zeros(d, device="cuda")
    sp = cache.stream()
    for s in range(10):
        cache.lookup_device(dk[s % 32].data_ptr(), n, outs[s % 8].data_ptr(), fl.data_ptr(),
                            dr.data_ptr(), mk.data_ptr(), mf.data_ptr(), cnt.data_ptr(), sp)
    torch.cuda.synchronize()
    cache.debug_trace()
    g = hps.StreamGraph(sp)
    with g:
        for s in range(a.steps):
            cache.lookup_device(dk[s % 32].data_ptr(), n, outs[s % 8].data_ptr(), fl.data_ptr(),
                                dr.data_ptr(), mk.data_ptr(), mf.data_ptr(),
                                cnt[2 * s:].data_ptr(), sp)
    g.launch()
    torch.cuda.synchronize()
    if a.no_trace:
        return
    t = cache.debug_trace()[-a.steps:]
    rel = (t[:, 1:] - t[:, :1]) / 1e3
    names = ["last A done", "last block start", "first A done", "first copy done",
             "last copy done", "finish start", "finish end"]
    print(f"{len(t)} calls; per-call timeline (us from the call's first block start), median [p10, p90]:")
    for j, nm in enumerate(names):
        col = rel[:, j]
        print(f"  {nm:16s} {np.median(col):7.2f}  [{np.percentile(col, 10):6.2f}, {np.percentile(col, 90):6.2f}]")
    gap = np.diff(t[:, 0]) / 1e3
    end_to_start = (t[1:, 0] - t[:-1, 7]) / 1e3
    print(f"  start-to-start gap      {np.median(gap):7.2f}  [{np.percentile(gap, 10):6.2f}, {np.percentile(gap, 90):6.2f}]")
    print(f"  next start - finish end {np.median(end_to_start):7.2f}")
    print(f"  next start - last A done {np.median((t[1:, 0] - t[:-1, 1]) / 1e3):7.2f}")
    print(f"  next start - last copy done {np.median((t[1:, 0] - t[:-1, 5]) / 1e3):7.2f}")


if __name__ == "__main__":
    main()
