"""Diagnostic: does graph-captured lookup_device serialise, and how long is
one lookup when steps run back to back? (not part of the product)"""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
import paper_2210_08804_b200 as hps  # noqa: E402


def main():
    wl = bench.Workload()
    d, n = wl.dim, wl.batch
    cache = hps.SlabCache(hps.SlabCacheConfig(slabset_count=wl.S, slabs_per_set=2, dimension=d))
    st = torch.cuda.ExternalStream(cache.stream())
    for i in range(0, len(wl.preload), n):
        k = wl.preload[i:i + n]
        kt = torch.from_numpy(k.view(np.int64)).cuda()
        rt = torch.from_numpy(bench.table_rows(k, d)).cuda()
        cache.replace_device(kt.data_ptr(), len(k), rt.data_ptr(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    wl.set_resident(cache.dump_all())
    batches, _, _ = wl.batches(0.9, 32, 5)
    dk = [torch.from_numpy(b.view(np.int64)).cuda() for b in batches]
    outs = [torch.empty(n * d, device="cuda") for _ in range(8)]
    fl = [torch.empty(n, dtype=torch.uint8, device="cuda") for _ in range(8)]
    mk = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(8)]
    mf = [torch.empty(n, dtype=torch.int32, device="cuda") for _ in range(8)]
    dr = torch.zeros(d, device="cuda")
    K = 200
    counts = torch.zeros(2 * K, dtype=torch.int64, device="cuda")
    sp = st.cuda_stream

    def step(s):
        cache.lookup_device(dk[s % 32].data_ptr(), n, outs[s % 8].data_ptr(), fl[s % 8].data_ptr(),
                            dr.data_ptr(), mk[s % 8].data_ptr(), mf[s % 8].data_ptr(), counts[2 * s:].data_ptr(), sp)

    for s in range(10):
        step(s)
    torch.cuda.synchronize()
    # (a) plain launches, timed on the stream
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    t0 = time.perf_counter()
    for s in range(K):
        step(s)
    t_host = time.perf_counter() - t0
    b.record(st)
    torch.cuda.synchronize()
    print(f"plain: {a.elapsed_time(b) * 1e3 / K:.2f} us/step (host enqueue {t_host * 1e6 / K:.2f} us/step)")
    # (b) graph without events
    g = hps.StreamGraph(sp)
    with g:
        for s in range(K):
            step(s)
    torch.cuda.synchronize()
    a.record(st)
    g.launch()
    b.record(st)
    torch.cuda.synchronize()
    print(f"graph: {a.elapsed_time(b) * 1e3 / K:.2f} us/step")
    c = counts.cpu().numpy().reshape(-1, 2)
    print("counts first/last", c[0], c[K - 1], "h", np.mean(1 - c[:, 1] / c.sum(1)))
    # (c) correctness of the last graph step vs an eager lookup of the same batch
    ref_out = torch.empty(n * d, device="cuda")
    rfl = torch.empty(n, dtype=torch.uint8, device="cuda")
    rmk = torch.empty(n, dtype=torch.int64, device="cuda")
    rmf = torch.empty(n, dtype=torch.int32, device="cuda")
    rc = torch.zeros(2, dtype=torch.int64, device="cuda")
    s = K - 1
    cache.lookup_device(dk[s % 32].data_ptr(), n, ref_out.data_ptr(), rfl.data_ptr(), dr.data_ptr(),
                        rmk.data_ptr(), rmf.data_ptr(), rc.data_ptr(), sp)
    torch.cuda.synchronize()
    print("rows equal:", torch.equal(ref_out, outs[s % 8]), "flags equal:", torch.equal(rfl, fl[s % 8]))


if __name__ == "__main__":
    main()
