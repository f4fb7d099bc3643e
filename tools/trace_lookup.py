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
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--no-trace", action="store_true")
    ap.add_argument("--isolated", action="store_true",
                    help="one call at a time (host sync between calls): single-call timeline")
    ap.add_argument("--graph-events", action="store_true",
                    help="the bench's p50 arrangement: one graph, CUDA events around every "
                         "lookup (no overlap); also times an empty event pair and a tiny "
                         "kernel the same way (the launch floor)")
    ap.add_argument("--update-frac", type=float, default=0.0,
                    help="cfg 4: stream-ordered update of this fraction of the resident rows "
                         "after every lookup")
    ap.add_argument("--per-call", action="store_true",
                    help="also print every call's first block start, last phase A, last copy "
                         "and finish end relative to the first call's start (fill / drain)")
    a = ap.parse_args()
    wl = bench.Workload(batch=a.batch, dim=a.dim)
    d, n = wl.dim, wl.batch
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=wl.S, slabs_per_set=wl.W, dimension=d),
                          device=0)
    for i in range(0, len(wl.preload), n):
        k = wl.preload[i:i + n]
        cache.replace(k, bench.table_rows(k, d))
    resident = cache.dump_all()
    wl.set_resident(resident)
    upd = []
    if a.update_frac > 0:
        u = max(1, int(len(resident) * a.update_frac))
        rng = np.random.default_rng(77)
        for j in range(8):
            idx = rng.choice(len(resident), u, replace=False)
            upd.append((torch.from_numpy(resident[idx].view(np.int64)).cuda(),
                        torch.empty(u * d, device="cuda").uniform_(-1, 1), u))
    written = torch.zeros(1, dtype=torch.int64, device="cuda")
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
        if upd:
            k, r, u = upd[s % 8]
            cache.update_device_async(k.data_ptr(), u, r.data_ptr(), written.data_ptr(), sp)
    torch.cuda.synchronize()
    cache.debug_trace()
    if a.graph_events:
        st = torch.cuda.ExternalStream(sp)
        kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(a.steps)]
        fev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(a.steps)]
        for x, y in kev + fev:
            x.record(st)
            y.record(st)
        torch.cuda.synchronize()
        g = hps.StreamGraph(sp)
        if True:
            with g:
                for s in range(a.steps):
                    cache.set_profile_events(kev[s][0].cuda_event, kev[s][1].cuda_event)
                    cache.lookup_device(dk[s % 32].data_ptr(), n, outs[s % 8].data_ptr(),
                                        fl.data_ptr(), dr.data_ptr(), mk.data_ptr(), mf.data_ptr(),
                                        cnt[2 * s:].data_ptr(), sp)
                    # the floor: the same event pair around a 32-key lookup (one block)
                    cache.set_profile_events(fev[s][0].cuda_event, fev[s][1].cuda_event)
                    cache.lookup_device(dk[s % 32].data_ptr(), 32, outs[s % 8].data_ptr(),
                                        fl.data_ptr(), dr.data_ptr(), mk.data_ptr(), mf.data_ptr(),
                                        cnt[2 * s:].data_ptr(), sp)
                    cache.set_profile_events(0, 0)
        g.launch()
        torch.cuda.synchronize()
        k1 = np.array([x.elapsed_time(y) for x, y in kev]) * 1e3
        f1 = np.array([x.elapsed_time(y) for x, y in fev]) * 1e3
        print(f"graph with events: lookup p50 {np.median(k1):.2f} us, 32-key lookup (floor) p50 "
              f"{np.median(f1):.2f} us")
    elif a.isolated:
        st = torch.cuda.ExternalStream(sp)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(a.steps)]
        for s in range(a.steps):
            ev[s][0].record(st)
            cache.lookup_device(dk[s % 32].data_ptr(), n, outs[s % 8].data_ptr(), fl.data_ptr(),
                                dr.data_ptr(), mk.data_ptr(), mf.data_ptr(),
                                cnt[2 * s:].data_ptr(), sp)
            ev[s][1].record(st)
            torch.cuda.synchronize()
        el = np.array([x.elapsed_time(y) for x, y in ev]) * 1e3
        print(f"isolated calls: event-bracketed median {np.median(el):.2f} us "
              f"[p10 {np.percentile(el, 10):.2f}, p90 {np.percentile(el, 90):.2f}]")
    else:
        g = hps.StreamGraph(sp)
        with g:
            for s in range(a.steps):
                cache.lookup_device(dk[s % 32].data_ptr(), n, outs[s % 8].data_ptr(), fl.data_ptr(),
                                    dr.data_ptr(), mk.data_ptr(), mf.data_ptr(),
                                    cnt[2 * s:].data_ptr(), sp)
                if upd:
                    k, r, u = upd[s % 8]
                    cache.update_device_async(k.data_ptr(), u, r.data_ptr(), written.data_ptr(), sp)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        st = torch.cuda.ExternalStream(sp)
        t0.record(st)
        g.launch()
        t1.record(st)
        torch.cuda.synchronize()
        print(f"graph: {t0.elapsed_time(t1) * 1e3 / a.steps:.2f} us per step")
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
    if a.per_call:
        z = t[0, 0]
        print("  call   start  lastA  lastcopy  finish_end  (us from call 0 start)")
        for i in range(len(t)):
            print(f"  {i:4d} {(t[i, 0] - z) / 1e3:7.2f} {(t[i, 1] - z) / 1e3:6.2f} "
                  f"{(t[i, 5] - z) / 1e3:8.2f} {(t[i, 7] - z) / 1e3:10.2f}")
    gap = np.diff(t[:, 0]) / 1e3
    end_to_start = (t[1:, 0] - t[:-1, 7]) / 1e3
    print(f"  start-to-start gap      {np.median(gap):7.2f}  [{np.percentile(gap, 10):6.2f}, {np.percentile(gap, 90):6.2f}]")
    print(f"  next start - finish end {np.median(end_to_start):7.2f}")
    print(f"  next start - last A done {np.median((t[1:, 0] - t[:-1, 1]) / 1e3):7.2f}")
    print(f"  next start - last copy done {np.median((t[1:, 0] - t[:-1, 5]) / 1e3):7.2f}")


if __name__ == "__main__":
    main()
