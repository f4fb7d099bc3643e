"""batched cold reads (hps_pdb_* / SegmentStore) over the
reference's persistent-store files, against the reference's own
PersistentStore::get (persistent_store.cpp:405-439, oracle/_ref) on segments
the reference itself wrote -- found keys, rows (bit-exact) and missing keys
in input order -- plus hand-made directories for the scan rules
(persistent_store.cpp:229-268: ascending segment numbers, newest record
wins, a segment's scan stops at its first incomplete or foreign-dimension
record). Host code: runs without a GPU."""
import struct

import numpy as np
import pytest

import oracle
import paper_2210_08804_b200 as hps

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def rows_for(keys, d, salt):
    k = np.asarray(keys, dtype=np.float64)
    return (k[:, None] * 0.25 + salt + np.arange(d)[None, :] * 0.125).astype(np.float32).reshape(-1)


def compare(root, name, d, probe):
    ref = oracle.RefPersistentStore(root)
    try:
        want = ref.get(name, probe, d)
    finally:
        ref.close()
    st = hps.SegmentStore(root, threads=4)
    st.attach(name)
    got = st.get(name, probe)
    assert np.array_equal(got.found_keys, want[0])
    assert got.found_vectors.tobytes() == want[1].tobytes()
    assert np.array_equal(got.missing_keys, want[2])
    return st, got


@needs_ref
def test_reference_written_segments_with_overwrites_and_compaction(tmp_path):
    d, name = 16, "emb"
    ref = oracle.RefPersistentStore(tmp_path)
    ref.create_table(name, d)
    k0 = np.arange(5000, dtype=np.uint64) * 7
    ref.put(name, k0, rows_for(k0, d, 0.0))
    ref.flush(name)
    k1 = k0[::5]
    ref.put(name, k1, rows_for(k1, d, 1.0))  # overwrites
    ref.flush(name)
    ref.compact(name)  # a new, higher-numbered segment with the live records
    k2 = np.concatenate([k0[1::9], np.arange(100000, 102000, dtype=np.uint64)])
    ref.put(name, k2, rows_for(k2, d, 2.0))
    ref.close()  # flushes
    rng = np.random.default_rng(3)
    probe = np.concatenate([rng.choice(k0, 3000), rng.integers(0, 110000, 3000).astype(np.uint64),
                            k2[:500]]).astype(np.uint64)
    rng.shuffle(probe)
    st, got = compare(tmp_path, name, d, probe)
    assert st.key_count(name) == 5000 + 2000
    assert len(got.found_keys) > 3000 and len(got.missing_keys) > 0


@needs_ref
def test_torn_tail_is_ignored_like_the_reference(tmp_path):
    d, name = 8, "t"
    ref = oracle.RefPersistentStore(tmp_path)
    ref.create_table(name, d)
    k = np.arange(300, dtype=np.uint64)
    ref.put(name, k, rows_for(k, d, 0.5))
    ref.close()
    seg = sorted((tmp_path / name).glob("seg-*.log"))[-1]
    with open(seg, "ab") as f:  # a crash mid-append: header + part of a row
        f.write(struct.pack("<QI", 999, d) + b"\x00" * 10)
    st = hps.SegmentStore(tmp_path)
    st.attach(name)
    got = st.get(name, np.array([999, 5, 299], np.uint64))
    assert got.missing_keys.tolist() == [999]
    # the reference opened afterwards (it truncates the torn bytes) agrees
    compare(tmp_path, name, d, np.array([999, 5, 299, 1000], np.uint64))


def write_table(root, name, d, segments):
    """segments: {number: [(key, dim, row or raw bytes)]} in the reference's
    record format [u64 key][u32 dim][dim f32] (persistent_store.cpp:376)."""
    tdir = root / hps_escape(name)
    tdir.mkdir(parents=True)
    (tdir / "MANIFEST").write_text(f"name={name}\ndim={d}\nversion=1\n")
    for num, recs in segments.items():
        with open(tdir / f"seg-{num}.log", "wb") as f:
            for key, rdim, row in recs:
                f.write(struct.pack("<QI", key, rdim))
                f.write(row if isinstance(row, bytes) else np.asarray(row, np.float32).tobytes())


def hps_escape(name):
    safe = set("abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789._-")
    if name in (".", ".."):
        return "%2E" * len(name)
    return "".join(c if c in safe else "%{:02X}".format(ord(c)) for c in name)


@needs_ref
def test_scan_rules_segment_order_newest_wins_and_stop_at_bad_record(tmp_path):
    d, name = 4, "a b/c"  # escaped directory name
    r = lambda v: [float(v)] * d  # noqa: E731
    write_table(tmp_path, name, d, {
        # seg-10 sorts after seg-2 numerically (not lexically)
        10: [(1, d, r(10)), (2, d, r(10))],
        2: [(1, d, r(2)), (3, d, r(2)), (4, 3, b"\x00" * 12), (5, d, r(2))],  # bad dim: 5 ignored
        0: [(3, d, r(0)), (6, d, r(0)), (7, d, r(0))],
    })
    # open the reader first: the reference's open truncates the LAST segment
    st = hps.SegmentStore(tmp_path)
    st.attach(name)
    probe = np.array([1, 2, 3, 4, 5, 6, 7, 8], np.uint64)
    got = st.get(name, probe)
    assert got.found_keys.tolist() == [1, 2, 3, 6, 7]
    assert got.found_vectors.reshape(-1, d)[:, 0].tolist() == [10, 10, 2, 0, 0]
    assert got.missing_keys.tolist() == [4, 5, 8]
    assert st.segment_count(name) == 3
    compare(tmp_path, name, d, probe)


@needs_ref
def test_refresh_follows_flushed_appends_and_compactions(tmp_path):
    d, name = 8, "t"
    ref = oracle.RefPersistentStore(tmp_path)
    ref.create_table(name, d)
    k = np.arange(1000, dtype=np.uint64)
    ref.put(name, k, rows_for(k, d, 0.0))
    ref.flush(name)
    st = hps.SegmentStore(tmp_path)
    st.attach(name)
    k2 = np.arange(1000, 1500, dtype=np.uint64)
    ref.put(name, k2, rows_for(k2, d, 0.0))
    ref.put(name, k[:10], rows_for(k[:10], d, 9.0))
    assert len(st.get(name, k2).found_keys) == 0  # unflushed, not yet refreshed
    ref.flush(name)
    st.refresh(name)
    g = st.get(name, np.concatenate([k[:10], k2]))
    assert len(g.found_keys) == 510
    assert g.found_vectors[:10 * d].tobytes() == rows_for(k[:10], d, 9.0).tobytes()  # newest
    assert g.found_vectors[10 * d:].tobytes() == rows_for(k2, d, 0.0).tobytes()
    ref.compact(name)
    st.refresh(name)  # the old segments are gone: re-indexed from scratch
    probe = np.arange(0, 1600, 3, dtype=np.uint64)
    want = ref.get(name, probe, d)
    got = st.get(name, probe)
    ref.close()
    assert np.array_equal(got.found_keys, want[0])
    assert got.found_vectors.tobytes() == want[1].tobytes()
    assert np.array_equal(got.missing_keys, want[2])


def test_missing_table_and_malformed_manifest(tmp_path):
    st = hps.SegmentStore(tmp_path)
    with pytest.raises(hps.InvalidArgument, match="persistent store has no table named nope"):
        st.attach("nope")
    (tmp_path / "bad").mkdir()
    (tmp_path / "bad" / "MANIFEST").write_text("name=bad\ndim=0\nversion=1\n")
    with pytest.raises(hps.TierFault, match="malformed MANIFEST"):
        st.attach("bad")
    with pytest.raises(hps.InvalidArgument):
        st.get("nope", np.array([1], np.uint64))


def test_native_cold_tier_in_tier_fetch_matches_a_python_cold_tier(tmp_path):
    """tier_fetch (VDB first, then the cold tier; cold hits promoted to the
    VDB) with the native reader as the cold tier equals the same call over
    a Python cold tier holding the same rows."""
    d, name = 8, "t"
    r = lambda k: rows_for(k, d, 3.0)  # noqa: E731
    keys = np.arange(0, 4000, 2, dtype=np.uint64)
    write_table(tmp_path, name, d, {0: [(int(k), d, r([k])) for k in keys]})
    st = hps.SegmentStore(tmp_path)
    cold_native = st.table(name)
    cold_py = hps.DictStore(d)
    cold_py.put(keys, r(keys))
    table = hps.TableId(name, d)
    probe = np.random.default_rng(5).integers(0, 4400, 3000).astype(np.uint64)
    out = []
    for cold in (cold_native, cold_py):
        vdb = hps.VolatileStore()
        vdb.register_table(table)
        vk = keys[::7]
        vdb.insert(name, vk, r(vk) + np.float32(1.0))
        cnt = {}
        f = hps.tier_fetch(table, probe, vdb, cold, cnt)
        vdb.drain()
        out.append((f, cnt, vdb.table_size(name)))
    (fa, ca, na), (fb, cb, nb) = out
    assert np.array_equal(fa.found_keys, fb.found_keys)
    assert fa.found_vectors.tobytes() == fb.found_vectors.tobytes()
    assert np.array_equal(fa.missing_keys, fb.missing_keys)
    assert ca == cb and ca["pdb_hits"] > 0 and na == nb
