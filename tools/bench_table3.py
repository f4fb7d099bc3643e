#!/usr/bin/env python
"""Cache Update and Dump at the sizes of the paper's Table 3 (PAPER.md:
527-533) -- the only published numbers that measure the
cache API itself (A100-80GB: Update 1 / 10 / 40 GB in 5.152 / 50.262 /
200.345 ms = 194.2 / 198.96 / 199.73 GB/s; Dump 1 / 40 GB in 0.064 / 1.19 ms).

  python tools/bench_table3.py [--sizes 1,10,40] > profiles/<round>_table3.json

Per size: a cache whose rows take SIZE GB (d = 128, W = 2), filled through
replace with SIZE-GB-worth of distinct keys; then, timed with CUDA events on
the cache stream, (a) hps_cache_update_device of every resident key with new
device-resident rows (GB of rows rewritten per second, the paper's metric)
and (b) hps_cache_dump_device of the whole key set into device memory.
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

PAPER = {1: {"update_ms": 5.152, "dump_ms": 0.064}, 10: {"update_ms": 50.262},
         40: {"update_ms": 200.345, "dump_ms": 1.19}}


def main():
    import torch

    import paper_2210_08804_b200 as hps

    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1,10,40")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    d, W = 128, 2
    out = {"metric": "cache Update / Dump time and GB/s at the paper's Table 3 sizes",
           "dim": d, "slabs_per_set": W, "points": []}
    for gb in [int(x) for x in a.sizes.split(",")]:
        slots = int(gb * 1e9) // (d * 4)
        S = slots // (W * 32)
        cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=W, dimension=d),
                              device=0)
        st = torch.cuda.ExternalStream(cache.stream())
        sp = st.cuda_stream
        n_keys = S * W * 32
        chunk = 1 << 20
        with torch.cuda.stream(st):
            for i in range(0, n_keys, chunk):
                m = min(chunk, n_keys - i)
                # distinct keys, scattered over the sets (odd multiplier mod 2^63)
                k = (torch.arange(i, i + m, dtype=torch.int64, device="cuda")
                     * 0x9E3779B97F4A7C1) & ((1 << 63) - 1)
                r = torch.rand(m * d, device="cuda")
                cache.replace_device(k.data_ptr(), m, r.data_ptr(), sp)
            resident = torch.empty(n_keys, dtype=torch.int64, device="cuda")
            n_res = torch.zeros(1, dtype=torch.int64, device="cuda")
            cache.dump_device_async(0, S, resident.data_ptr(), n_res.data_ptr(), sp)
        torch.cuda.synchronize()
        R = int(n_res.item())
        rows = torch.rand(R * d, device="cuda")
        written = torch.zeros(1, dtype=torch.int64, device="cuda")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

        def timed(fn):
            fn()
            torch.cuda.synchronize()
            ev[0].record(st)
            for _ in range(a.reps):
                fn()
            ev[1].record(st)
            torch.cuda.synchronize()
            return ev[0].elapsed_time(ev[1]) / a.reps

        upd_ms = timed(lambda: cache.update_device_async(resident.data_ptr(), R, rows.data_ptr(),
                                                         written.data_ptr(), sp))
        assert int(written.item()) == R
        dump_ms = timed(lambda: cache.dump_device_async(0, S, resident.data_ptr(),
                                                        n_res.data_ptr(), sp))
        row_bytes = R * d * 4
        p = {"cache_gb": gb, "slabsets": S, "resident_keys": R, "row_bytes": row_bytes,
             "update_ms": upd_ms, "update_gb_per_s": row_bytes / (upd_ms * 1e-3) / 1e9,
             "dump_ms": dump_ms, "dump_keys_per_s": R / (dump_ms * 1e-3)}
        ref = PAPER.get(gb, {})
        if "update_ms" in ref:
            p["paper_a100_update_ms"] = ref["update_ms"]
            p["update_speedup_vs_paper_a100"] = ref["update_ms"] / upd_ms
        if "dump_ms" in ref:
            p["paper_a100_dump_ms"] = ref["dump_ms"]
            p["dump_speedup_vs_paper_a100"] = ref["dump_ms"] / dump_ms
        out["points"].append(p)
        print(json.dumps(p), file=sys.stderr)
        del cache, rows, resident
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
