"""Deterministic cache op streams shared by fixtures, oracle tests and GPU
parity tests (shape of acceptance c1, acceptance_main.cpp:105-208: 45%
query with duplicates, 35% replace of distinct keys, 20% update with
duplicates; rows = (key*31 + c*7 + salt*13) % 9973)."""
from __future__ import annotations

import hashlib

import numpy as np


def row_values(keys: np.ndarray, dim: int, salt: int) -> np.ndarray:
    k = keys.astype(np.uint64)[:, None]
    c = np.arange(dim, dtype=np.uint64)[None, :]
    v = (k * np.uint64(31) + c * np.uint64(7) + np.uint64(salt * 13)) % np.uint64(9973)
    return v.astype(np.float32).reshape(-1)


def ops(seed: int, n_ops: int, keyspace: int, dim: int, max_query: int = 64,
        max_write: int = 48):
    rng = np.random.default_rng(seed)
    for op in range(n_ops):
        roll = int(rng.integers(100))
        if roll < 45:
            keys = rng.integers(0, keyspace, 1 + int(rng.integers(max_query)), dtype=np.uint64)
            yield ("q", keys, None)
        elif roll < 80:
            n = 1 + int(rng.integers(max_write))
            keys = rng.choice(keyspace, size=min(n, keyspace), replace=False).astype(np.uint64)
            yield ("r", keys, row_values(keys, dim, op))
        else:
            keys = rng.integers(0, keyspace, 1 + int(rng.integers(max_write)), dtype=np.uint64)
            yield ("u", keys, row_values(keys, dim, op + 7))


class Digest:
    """Rolling sha256 over every observable result of an op stream."""

    def __init__(self):
        self.h = hashlib.sha256()

    def query(self, hit: np.ndarray, rows: np.ndarray):
        self.h.update(b"q")
        self.h.update(np.ascontiguousarray(hit, dtype=np.uint8).tobytes())
        self.h.update(np.ascontiguousarray(rows, dtype=np.float32).tobytes())

    def update(self, written: int):
        self.h.update(b"u%d" % written)

    def state(self, clock: int, occupied: int):
        self.h.update(b"s%d,%d" % (clock, occupied))

    def hexdigest(self) -> str:
        return self.h.hexdigest()


def run_stream(cache, geometry, seed, n_ops, keyspace, kind):
    """Drives `cache` (kind: 'ref' = oracle.RefCache, 'oracle' =
    oracle.OracleCache, 'gpu' = paper_2210_08804_b200.SlabCache) through the
    stream and returns (digest, clock, occupied, sorted resident keys)."""
    S, W, d = geometry
    dg = Digest()
    for kind_op, keys, vecs in ops(seed, n_ops, keyspace, d):
        n = len(keys)
        if kind_op == "q":
            out = np.zeros(n * d, dtype=np.float32)
            if kind == "oracle":
                hit = cache.query(keys, out)
            else:
                if kind == "ref":
                    pos, _ = cache.query(keys, out)
                else:
                    pos, _ = cache.query_arrays(keys, out)
                hit = np.ones(n, dtype=np.uint8)
                hit[pos.astype(np.int64)] = 0
            dg.query(hit, out)
        elif kind_op == "r":
            cache.replace(keys, vecs)
        else:
            dg.update(int(cache.update(keys, vecs)))
        clock = cache.clock() if kind != "gpu" else cache.recency_clock()
        dg.state(clock, cache.occupied())
    if kind == "ref":
        res = cache.dump_all()
    elif kind == "oracle":
        res = cache.dump()
    else:
        res = cache.dump_all()
    clock = cache.clock() if kind != "gpu" else cache.recency_clock()
    return dg.hexdigest(), clock, cache.occupied(), np.sort(res)
