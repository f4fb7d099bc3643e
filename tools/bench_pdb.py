#!/usr/bin/env python
"""Cold-tier fetch: the reference's PersistentStore::get (one pread per key,
persistent_store.cpp:405-439; oracle/_ref) against the native batched reader
(hps_pdb_get / SegmentStore) on the SAME segment files, written by the
reference itself. Host code on the box's cores; files in the page cache (the
serving steady state) after one untimed pass.

  python tools/bench_pdb.py [--keys 2000000] [--dim 128] [--batch 65536]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def main():
    import oracle
    import paper_2210_08804_b200 as hps

    ap = argparse.ArgumentParser()
    ap.add_argument("--keys", type=int, default=2_000_000)
    ap.add_argument("--dim", type=int, default=128)
    ap.add_argument("--batch", type=int, default=65536)
    ap.add_argument("--reps", type=int, default=10)
    a = ap.parse_args()
    d, name = a.dim, "cold"
    with tempfile.TemporaryDirectory(dir=os.environ.get("TMPDIR", "/tmp")) as td:
        ref = oracle.RefPersistentStore(td)
        ref.create_table(name, d)
        t0 = time.perf_counter()
        step = 1 << 17
        for i in range(0, a.keys, step):
            k = np.arange(i, min(a.keys, i + step), dtype=np.uint64)
            v = ((k[:, None] * 3 + np.arange(d)[None, :]) % 1000).astype(np.float32) / 7.0
            ref.put(name, k, v.reshape(-1))
        ref.flush(name)
        write_s = time.perf_counter() - t0
        rng = np.random.default_rng(1)
        batches = [rng.integers(0, int(a.keys * 1.1), a.batch).astype(np.uint64)
                   for _ in range(a.reps)]
        st = hps.SegmentStore(td)
        t0 = time.perf_counter()
        st.attach(name)
        attach_s = time.perf_counter() - t0
        # warm the page cache (both read the same files)
        st.get(name, np.arange(a.keys, dtype=np.uint64))
        res = {}
        # the engine's use: the reader fills reused (pinned staging) buffers
        import ctypes as C

        fk = np.empty(a.batch, np.uint64)
        fv = np.empty(a.batch * d, np.float32)
        mk = np.empty(a.batch, np.uint64)
        fv.fill(0)
        nf, nm = C.c_size_t(0), C.c_size_t(0)

        def native_into(b):
            hps._check(hps.lib().hps_pdb_get(st._h, name.encode(), b.ctypes.data, len(b),
                                             fk.ctypes.data, fv.ctypes.data, C.byref(nf),
                                             mk.ctypes.data, C.byref(nm)))

        for label, fn in (("reference_pread_per_key", lambda b: ref.get(name, b, d)),
                          ("native_batched", native_into)):
            fn(batches[0])
            t0 = time.perf_counter()
            for b in batches:
                fn(b)
            el = (time.perf_counter() - t0) / a.reps
            res[label] = {"ms_per_batch": el * 1e3, "keys_per_s": a.batch / el,
                          "row_gb_per_s": a.batch * (1 / 1.1) * d * 4 / el / 1e9}
        # bit-exact on every batch
        for b in batches[:3]:
            w = ref.get(name, b, d)
            g = st.get(name, b)
            assert np.array_equal(g.found_keys, w[0]) and np.array_equal(g.missing_keys, w[2])
            assert g.found_vectors.tobytes() == w[1].tobytes()
        ref.close()
    print(json.dumps({"table_keys": a.keys, "dim": d, "batch": a.batch,
                      "host_cores": os.cpu_count(), "write_s_reference": write_s,
                      "attach_index_s": attach_s, **res,
                      "speedup": res["reference_pread_per_key"]["ms_per_batch"]
                      / res["native_batched"]["ms_per_batch"], "parity": "bit-exact"}))


if __name__ == "__main__":
    main()
