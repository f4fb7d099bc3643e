"""CPU: pin the oracle (C restatement) against the reference's golden
vectors, against fixtures generated from the reference build, and -- when
oracle/_ref is present -- against the live reference library.

Mirrors /root/reference/proj/tests/unit/test_core.cpp and the
slab-cache parts of test_slab_cache.cpp / acceptance c1."""
import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

import oracle
from tools import workload
from opstream import ops, row_values, run_stream

GOLD = Path(__file__).resolve().parent / "golden"


def _load(name):
    return json.loads((GOLD / name).read_text())


def _bytes(spec: str) -> bytes:
    return bytes.fromhex(spec[4:]) if spec.startswith("hex:") else spec.encode()


def test_xxh64_key_vectors_match_canonical():
    kv = _load("xxh64_vectors.json")
    for k, s, e in kv["key_vectors"] + kv["random_keys"]:
        assert oracle.xxh64_key(int(k, 16), int(s, 16)) == int(e, 16), (k, s)


def test_xxh64_byte_vectors_cover_every_tail_path():
    for d, s, e in _load("xxh64_vectors.json")["byte_vectors"]:
        assert oracle.xxh64(_bytes(d), int(s, 16)) == int(e, 16), d


def test_xxh64_independent_python_xxhash():
    xxhash = pytest.importorskip("xxhash")
    rng = np.random.default_rng(5)
    for k in rng.integers(0, 2**64 - 1, 200, dtype=np.uint64):
        for s in (0, 0x5EED5E7, 0x51AB):
            want = xxhash.xxh64_intdigest(int(k).to_bytes(8, "little"), seed=s)
            assert oracle.xxh64_key(int(k), s) == want


def test_placement_seeds_and_partition_example():
    assert oracle.partition_of(0, 16) == 11  # test_core.cpp:105
    assert _load("xxh64_vectors.json")["partition_of_0_16"] == 11
    assert oracle.slabset_of(0, 1024) == oracle.xxh64_key(0, 0x5EED5E7) % 1024
    assert oracle.first_slab_of(0, 2) == oracle.xxh64_key(0, 0x51AB) % 2


def test_dedup_preserves_first_occurrence_order():
    kat = _load("dedup.json")["kat"]
    u, inv = oracle.dedup(kat["keys"])
    assert u.tolist() == kat["unique"] == [7, 3, 9, 1]
    assert inv.tolist() == kat["inverse"]
    u, inv = oracle.dedup([])
    assert len(u) == 0 and len(inv) == 0
    keys = np.arange(100, dtype=np.uint64) * 31 + 5
    u, inv = oracle.dedup(keys)
    assert (u == keys).all() and (inv == np.arange(100)).all()


def test_dedup_random_matches_reference_fixture():
    r = _load("dedup.json")["random"]
    rng = np.random.default_rng(r["seed"])
    # gen_golden draws the KAT first from a fresh rng(2026) used for xxh64 keys
    rng.integers(0, 2**63, 100, dtype=np.uint64)
    batch = rng.integers(0, r["keyspace"], r["n"], dtype=np.uint64)
    u, inv = oracle.dedup(batch)
    assert len(u) == r["n_unique"]
    assert hashlib.sha256(u.tobytes()).hexdigest() == r["unique_sha"]
    assert hashlib.sha256(inv.tobytes()).hexdigest() == r["inverse_sha"]


@pytest.mark.parametrize("stream", _load("cache_streams.json")["streams"], ids=lambda s: s["name"])
def test_oracle_cache_reproduces_reference_stream(stream):
    geo = tuple(stream["geometry"])
    c = oracle.OracleCache(*geo)
    dig, clock, occ, resident = run_stream(c, geo, stream["seed"], stream["n_ops"],
                                           stream["keyspace"], "oracle")
    assert dig == stream["digest"]
    assert clock == stream["clock"] and occ == stream["occupied"]
    assert hashlib.sha256(resident.tobytes()).hexdigest() == stream["resident_sha"]
    assert hashlib.sha256(c.dump().tobytes()).hexdigest() == stream["dump_order_sha"]


def test_eviction_tie_break_worked_example():
    """test_slab_cache.cpp:193-237 on the oracle."""
    c = oracle.OracleCache(1, 2, 1)
    s0, s1 = [], []
    k = 0
    while len(s0) < 32 or len(s1) < 32:
        if oracle.first_slab_of(k, 2) == 0:
            if len(s0) < 32:
                s0.append(k)
        elif len(s1) < 32:
            s1.append(k)
        k += 1
    fill = np.array(s0 + s1, dtype=np.uint64)
    assert c.replace(fill, row_values(fill, 1, 0))
    assert c.occupied() == 64
    assert c.replace([1000000], [7.0])
    out = np.zeros(1, np.float32)
    assert c.query([s0[0]], out)[0] == 0
    assert c.query([1000000], out)[0] == 1 and out[0] == 7.0
    assert c.query([s0[1]], out)[0] == 1
    assert c.replace([1000001], [8.0])
    assert c.query([s0[2]], out)[0] == 0
    assert c.query([1000001], out)[0] == 1


def test_replace_duplicates_rejected_before_mutation():
    c = oracle.OracleCache(2, 2, 1)
    assert not c.replace([3, 4, 3], [1, 2, 3])
    assert c.occupied() == 0


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_matches_live_reference_and_its_model_op_for_op():
    geo = (8, 2, 4)
    ref = oracle.RefCache(*geo, workers=3, tasks_per_worker=2)
    model = oracle.RefModel(*geo)
    orc = oracle.OracleCache(*geo)
    for kind, keys, vecs in ops(0xFACADE, 1500, 900, geo[2]):
        n = len(keys)
        if kind == "q":
            a = np.full(n * 4, np.nan, np.float32)
            b = np.full(n * 4, np.nan, np.float32)
            m = np.full(n * 4, np.nan, np.float32)
            pos, mk = ref.query(keys, a)
            hit_o = orc.query(keys, b)
            hit_m = model.query(keys, m)
            hit_r = np.ones(n, np.uint8)
            hit_r[pos.astype(np.int64)] = 0
            assert (np.diff(pos.astype(np.int64)) > 0).all()
            assert (hit_r == hit_o).all() and (hit_o == hit_m).all()
            assert (mk == keys[pos.astype(np.int64)]).all()
            assert a.tobytes() == b.tobytes() == m.tobytes()  # NaN rows untouched
        elif kind == "r":
            ref.replace(keys, vecs)
            model.replace(keys, vecs)
            assert orc.replace(keys, vecs)
        else:
            assert ref.update(keys, vecs) == orc.update(keys, vecs) == model.update(keys, vecs)
        assert ref.clock() == orc.clock() == model.clock()
        assert ref.occupied() == orc.occupied()
    assert (ref.dump_all() == orc.dump()).all()
    assert (np.sort(model.resident()) == np.sort(orc.dump())).all()


def test_product_sampler_matches_reference_fixture():
    import paper_2210_08804_b200 as hps

    s = _load("sampler.json")
    for name in ("cfg1", "cfg2"):
        f = s[name]
        keys = workload.powerlaw_sample(f["alpha"], f["keyspace"], f["permute_seed"], f["draw_seed"],
                                   f["count"])
        assert keys[:64].tolist() == f["head"]
        assert hashlib.sha256(keys.tobytes()).hexdigest() == f["sha256"]
    f = s["cfg1"]
    o = oracle.powerlaw_sample(f["alpha"], f["keyspace"], f["permute_seed"], f["draw_seed"], 4096)
    assert o[:64].tolist() == f["head"]


def test_engine_oracle_reproduces_reference_session():
    e = _load("engine.json")
    d = e["dim"]
    eo = oracle.EngineOracle(e["S"], e["W"], d, threshold=e["threshold"],
                             default_vector=e["default_vector"])
    vk = np.arange(e["vdb_keys"], dtype=np.uint64)
    for k, r in zip(vk, row_values(vk, d, e["vdb_salt"]).reshape(-1, d)):
        eo.vdb[int(k)] = r
    rng = np.random.default_rng(e["batch_seed"])
    for step in e["steps"]:
        keys = rng.integers(0, e["key_range"], 1 + int(rng.integers(300)), dtype=np.uint64)
        out, flags, oc = eo.lookup(keys)
        eo.drain_async()
        assert len(keys) == step["n"]
        assert oc == step["outcome"]
        assert hashlib.sha256(out.tobytes()).hexdigest() == step["out_sha"]
        assert hashlib.sha256(flags.tobytes()).hexdigest() == step["flags_sha"]
    assert eo.stats == e["stats"]
