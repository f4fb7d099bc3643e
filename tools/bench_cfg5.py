#!/usr/bin/env python
"""cfg 5 (BASELINE.json configs[4]) on one B200: a 1B-key table, one cache
replica per GPU -- here the replica of one GPU. The cache holds 20 % of the
table (200M slots, d = 128: 102 GB of rows in HBM); keys follow a power law
(alpha 1.2) over all 1B keys, so the hit rate is whatever the cache earns
(no calibration). Everything is generated on the device: rank -> key is a
bijective 64-bit mix (no 8 GB permutation), the power-law inverse CDF is a
1B-entry device array (torch.searchsorted).

  python tools/bench_cfg5.py [--keys 1000000000] [--cache-frac 0.2] [--steps 300]

Per step = one hps_cache_lookup_device of a 65,536-key batch (graph-captured
like bench.py); reports keys/s, the measured unique-key hit rate and the
roofline fraction with the same algorithmic-bytes formula (the unique
counts from the kernel; slabs probed estimated as 1 + P(first slab full)).
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def mix64(x):
    """Bijective 64-bit finalizer (rank -> key), int64 torch arithmetic."""
    import torch

    m1 = -49064778989728563  # 0xff51afd7ed558ccd as int64
    m2 = -4265267296055464877  # 0xc4ceb9fe1a85ec53 as int64
    x = x ^ ((x >> 33) & ((1 << 31) - 1))
    x = x * m1
    x = x ^ ((x >> 33) & ((1 << 31) - 1))
    x = x * m2
    x = x ^ ((x >> 33) & ((1 << 31) - 1))
    return x


def main():
    import torch

    import bench
    import paper_2210_08804_b200 as hps

    ap = argparse.ArgumentParser()
    ap.add_argument("--keys", type=int, default=1_000_000_000)
    ap.add_argument("--cache-frac", type=float, default=0.2)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--steps", type=int, default=300)
    a = ap.parse_args()
    K, d, n = a.keys, a.dim, a.batch
    S = int(-(-int(K * a.cache_frac) // 64))
    t0 = time.perf_counter()
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=S, slabs_per_set=2, dimension=d),
                          device=0)
    st = torch.cuda.ExternalStream(cache.stream())
    sp = st.cuda_stream
    # power-law CDF over K ranks on the device (float64: 8 GB at 1B)
    cdf = torch.empty(K, dtype=torch.float64, device="cuda")
    step = 1 << 26
    acc = 0.0
    for i in range(0, K, step):
        r = torch.arange(i + 1, min(K, i + step) + 1, dtype=torch.float64, device="cuda")
        c = torch.cumsum(r.pow(-1.2), 0) + acc
        acc = float(c[-1].item())
        cdf[i:i + len(r)] = c
    cdf /= acc
    # preload: the hottest ranks through replace (1.1x capacity, like bench.py)
    cap = S * 64
    with torch.cuda.stream(st):
        for i in range(0, int(cap * 1.1), 1 << 20):
            m = min(1 << 20, int(cap * 1.1) - i)
            keys = mix64(torch.arange(i, i + m, dtype=torch.int64, device="cuda"))
            rows = torch.rand(m * d, device="cuda")
            cache.replace_device(keys.data_ptr(), m, rows.data_ptr(), sp)
    torch.cuda.synchronize()
    setup_s = time.perf_counter() - t0
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    pool = 32
    batches = []
    for _ in range(pool):
        u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g)
        ranks = torch.searchsorted(cdf, u).clamp_(max=K - 1)
        batches.append(mix64(ranks))
    del cdf
    torch.cuda.empty_cache()
    outs = [torch.empty(n * d, device="cuda") for _ in range(8)]
    fl = torch.empty(n, dtype=torch.uint8, device="cuda")
    mk = torch.empty(n, dtype=torch.int64, device="cuda")
    mf = torch.empty(n, dtype=torch.int32, device="cuda")
    dr = torch.zeros(d, device="cuda")
    steps = a.steps
    cnt = torch.zeros(2 * steps, dtype=torch.int64, device="cuda")
    for s in range(10):
        cache.lookup_device(batches[s % pool].data_ptr(), n, outs[s % 8].data_ptr(), fl.data_ptr(),
                            dr.data_ptr(), mk.data_ptr(), mf.data_ptr(), cnt.data_ptr(), sp)
    torch.cuda.synchronize()
    gr = hps.StreamGraph(sp)
    with gr:
        for s in range(steps):
            cache.lookup_device(batches[s % pool].data_ptr(), n, outs[s % 8].data_ptr(),
                                fl.data_ptr(), dr.data_ptr(), mk.data_ptr(), mf.data_ptr(),
                                cnt[2 * s:].data_ptr(), sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    gr.launch()
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    c = cnt.cpu().numpy().reshape(-1, 2)[:steps]
    uh, um = c[:, 0].mean(), c[:, 1].mean()
    # algorithmic bytes, slabs probed ~ 1.1 per unique key
    b = 8 * n + 260 * 1.1 * (uh + um) + 8 * uh + 4 * d * uh + 4 * d * n
    peak = bench.hbm_peak()[0]
    out = {"workload": f"cfg5 replica: {K} keys, cache {a.cache_frac:.0%} ({S} slabsets x 2, "
                       f"{S * 64 * d * 4 / 1e9:.1f} GB of rows), d {d}, batch {n}, power-law 1.2, "
                       "natural hit rate",
           "keys_per_s": n / (ms * 1e-3), "ms_per_step": ms,
           "unique_keys_per_batch": float(uh + um), "unique_hit_rate": float(uh / (uh + um)),
           "algorithmic_bytes_per_batch": b, "achieved_gbs": b / (ms * 1e-3) / 1e9,
           "roofline_frac": b / (ms * 1e-3) / 1e9 / peak, "setup_s": setup_s,
           "occupied": cache.occupied(), "capacity": cache.capacity()}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
