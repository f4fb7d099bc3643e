"""Generates the golden fixtures in this directory FROM THE REFERENCE ITSELF.

Run in the build container (needs /root/reference and oracle/_ref):
    python tests/golden/gen_golden.py

* xxh64_vectors.json   -- the reference's KATs (test_core.cpp:26-95) plus
                          100 random keys hashed by the reference build.
* cache_streams.json   -- digests of acceptance-c1-shaped op streams
                          (tests/opstream.py) driven through the reference
                          hps::SlabCache (slab_cache.cpp) for 5 geometries.
* sampler.json         -- head of the cfg-1 / cfg-2 power-law streams from
                          the reference PowerLawSampler (workload.cpp:24-70).
* dedup.json           -- reference dedup_keys on the KAT and a random batch.
* engine.json          -- a deterministic LookupEngine session (reference
                          lookup_engine.cpp over its VolatileStore).
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402
from opstream import run_stream  # noqa: E402

STREAMS = [
    # name, (S, W, d), seed, n_ops, keyspace
    ("c1_8x2_d4", (8, 2, 4), 0xACCE5501, 20000, 2000),
    ("single_set_heavy_evict", (1, 2, 4), 0xC0FFEE, 3000, 150),
    ("wider_4x4_d2", (4, 4, 2), 0xB0BA, 3000, 700),
    ("odd_d3_16x2", (16, 2, 3), 99, 3000, 2000),
    ("d16_64x2", (64, 2, 16), 7, 3000, 20000),
]

# test_core.cpp:26-48 (python xxhash 3.8.1 vectors) and :60-95
KEY_VECTORS = [
    (0x0000000000000000, 0x0, 0x34c96acdcadb1bbb), (0x0000000000000000, 0x5eed5e7, 0x745edad0b55c7529),
    (0x0000000000000000, 0x51ab, 0x1ad3c98ac1007642), (0x0000000000000001, 0x0, 0x9f29cb17a2a49995),
    (0x0000000000000001, 0x5eed5e7, 0x31216ea572261b87), (0x0000000000000001, 0x51ab, 0xa5a92c269add42ac),
    (0x000000000000002a, 0x0, 0xb556806fb6d14353), (0x000000000000002a, 0x5eed5e7, 0x0ecee854a20b3c97),
    (0x000000000000002a, 0x51ab, 0xd5383bb7d12dd9bb), (0x00000000deadbeef, 0x0, 0x3396f1a59cb00c78),
    (0x00000000deadbeef, 0x5eed5e7, 0x3f015bb63d32533b), (0x00000000deadbeef, 0x51ab, 0xe1ce647702f7cfee),
    (0xffffffffffffffff, 0x0, 0x85d136adb773c6c9), (0xffffffffffffffff, 0x5eed5e7, 0xb381e2275c0d2bfc),
    (0xffffffffffffffff, 0x51ab, 0xd0403fac826f0e81), (0x00000000075bcd15, 0x0, 0xcb7c2941b198004d),
    (0x00000000075bcd15, 0x5eed5e7, 0x10259bc427113c9e), (0x00000000075bcd15, 0x51ab, 0x24150e02a606d7cc),
    (0x0db4da5f44d20b4e, 0x0, 0xd893cc247c28555b), (0x0db4da5f44d20b4e, 0x5eed5e7, 0x47f234a72e49907a),
    (0x0db4da5f44d20b4e, 0x51ab, 0x14892f29321ae82d),
]


def byte_vectors():
    ramp = bytes(range(37))
    hundred = bytes(range(100))
    strided = bytes((i * 7 + 3) % 256 for i in range(257))
    sentence = b"xxhash is a fast non-cryptographic hash"
    return [
        ("", 0, 0xef46db3751d8e999), ("", 1, 0xd5afba1336a3be4b), ("abc", 0, 0x44bc2cf5ad770999),
        (sentence.hex(), 2654435761, 0x8d2f75313a0b23b2), (ramp.hex(), 0, 0xd93fa2dfee5c24c9),
        (ramp.hex(), 0x9E3779B185EBCA87, 0x938d1db91225bf4d), (hundred.hex(), 0, 0x6ac1e58032166597),
        (hundred.hex(), 0x51AB, 0xc43ed1d0392fd432), (strided.hex(), 0, 0xb7b604f7e4f822fa),
        (strided.hex(), 0x5EED5E7, 0x0a02478f8fb4c8a2),
    ]


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle)"
    rng = np.random.default_rng(2026)
    rand = [int(x) for x in rng.integers(0, 2**63, 100, dtype=np.uint64)] + [2**64 - 2]
    kv = {
        "source": "reference test_core.cpp:26-95 + reference build (oracle/_ref)",
        "key_vectors": [[hex(k), hex(s), hex(e)] for k, s, e in KEY_VECTORS],
        "byte_vectors": [[("hex:" + d) if i >= 3 else d, hex(s), hex(e)]
                         for i, (d, s, e) in enumerate(byte_vectors())],
        "random_keys": [[hex(k), hex(s), hex(oracle.rlib().ref_xxh64_key(k, s))]
                        for k in rand for s in (0, 0x5EED5E7, 0x51AB)],
        "partition_of_0_16": int(oracle.rlib().ref_partition_of(0, 16)),
    }
    (HERE / "xxh64_vectors.json").write_text(json.dumps(kv, indent=1))

    streams = []
    for name, geo, seed, n_ops, keyspace in STREAMS:
        c = oracle.RefCache(*geo, workers=2, tasks_per_worker=2)
        dig, clock, occ, resident = run_stream(c, geo, seed, n_ops, keyspace, "ref")
        c.check_invariants()
        order = c.dump_all()
        streams.append(dict(name=name, geometry=list(geo), seed=seed, n_ops=n_ops,
                            keyspace=keyspace, digest=dig, clock=clock, occupied=occ,
                            resident_sha=hashlib.sha256(resident.tobytes()).hexdigest(),
                            dump_order_sha=hashlib.sha256(order.tobytes()).hexdigest()))
        print(name, dig[:16], clock, occ)
    (HERE / "cache_streams.json").write_text(json.dumps(
        {"source": "reference hps::SlabCache via oracle/_ref", "streams": streams}, indent=1))

    samp = {}
    for name, (alpha, ks, seed) in {"cfg1": (1.2, 1_000_000, 42), "cfg2": (1.2, 10_000_000, 42)}.items():
        draw = seed ^ 0x9E3779B97F4A7C15
        n = 1 << 16
        keys = oracle.ref_powerlaw_sample(alpha, ks, seed, draw, n)
        samp[name] = dict(alpha=alpha, keyspace=ks, permute_seed=seed, draw_seed=draw, count=n,
                          head=[int(x) for x in keys[:64]],
                          sha256=hashlib.sha256(keys.tobytes()).hexdigest(),
                          unique_fraction_1024=len(np.unique(keys[:1024])) / 1024.0)
    (HERE / "sampler.json").write_text(json.dumps(
        {"source": "reference PowerLawSampler via oracle/_ref", **samp}, indent=1))

    kat = [7, 3, 7, 9, 3, 3, 1, 9]
    u, inv = oracle.ref_dedup(kat)
    batch = rng.integers(0, 5000, 20000, dtype=np.uint64)
    bu, binv = oracle.ref_dedup(batch)
    (HERE / "dedup.json").write_text(json.dumps({
        "source": "reference dedup_keys via oracle/_ref (types.cpp:20-34)",
        "kat": {"keys": kat, "unique": [int(x) for x in u], "inverse": [int(x) for x in inv]},
        "random": {"seed": 2026, "n": 20000, "keyspace": 5000,
                   "unique_sha": hashlib.sha256(bu.tobytes()).hexdigest(),
                   "inverse_sha": hashlib.sha256(binv.tobytes()).hexdigest(),
                   "n_unique": int(len(bu))}}, indent=1))

    # engine session: VDB holds keys [0, 3000); batches draw from [0, 3500)
    d = 8
    e = oracle.RefEngine(d, S=16, W=2, workers=2, threshold=0.6, partitions=4,
                         default_vector=[9.0, 8.0])
    vk = np.arange(3000, dtype=np.uint64)
    from opstream import row_values
    e.vdb_insert(vk, row_values(vk, d, 1))
    erng = np.random.default_rng(11)
    steps = []
    for b in range(40):
        keys = erng.integers(0, 3500, 1 + int(erng.integers(300)), dtype=np.uint64)
        out, flags, oc = e.lookup(keys)
        e.drain()
        steps.append(dict(n=int(len(keys)), outcome=oc,
                          out_sha=hashlib.sha256(out.tobytes()).hexdigest(),
                          flags_sha=hashlib.sha256(flags.tobytes()).hexdigest()))
    (HERE / "engine.json").write_text(json.dumps({
        "source": "reference LookupEngine via oracle/_ref",
        "dim": d, "S": 16, "W": 2, "threshold": 0.6, "partitions": 4,
        "default_vector": [9.0, 8.0], "vdb_keys": 3000, "vdb_salt": 1, "batch_seed": 11,
        "batches": 40, "key_range": 3500, "steps": steps, "stats": e.stats()}, indent=1))


if __name__ == "__main__":
    main()
