"""Host-side mirror of the reference API (CPU only): arithmetic pinned to the
reference's golden values, argument validation with the reference's exception
types, and the API surface (names, enum values, dataclass fields)."""

import dataclasses

import numpy as np
import pytest

import paper_2605_25040_b200 as cafs
from conftest import load_json
from oracle import gen as ogen
from paper_2605_25040_b200 import datagen


def test_fast_hash_matches_reference(known_answers):
    for row in known_answers["fast_hash"]:
        v, m, want = row[:3]
        mult = row[3] if len(row) > 3 else None
        assert cafs.fast_hash(v, m, mult) == want
    assert cafs.fast_hash(1, 9) == 316  # tests/test_buckets.py:38-40
    xs = np.arange(4096, dtype=np.uint64)
    assert cafs.fast_hash(xs, 12).tolist() == [cafs.fast_hash(int(v), 12) for v in xs]
    for bad in (0, 64, -3):
        with pytest.raises(ValueError):
            cafs.fast_hash(1, bad)


def test_table_size_matches_reference(known_answers):
    for k_hat, n, cap, want in known_answers["table_size_for"]:
        assert cafs.table_size_for(k_hat, n, cap) == want
    for args in ((0, 10, 4), (1, 0, 4), (1, 10, 5)):
        with pytest.raises(ValueError):
            cafs.table_size_for(*args)


def test_chao1_matches_reference(known_answers):
    for u, f1, f2, n, sat, want in known_answers["chao1"]:
        assert cafs.chao1(u, f1, f2, n, sat) == want
    with pytest.raises(ValueError):
        cafs.chao1(0, 0, 0, 10, False)


def test_check_hash_mult():
    assert cafs.check_hash_mult(None) == 0x9E3779B97F4A7C15
    assert cafs.check_hash_mult(3) == 3
    for bad in (2, 0, -1, 1 << 64):
        with pytest.raises(ValueError):
            cafs.check_hash_mult(bad)


def test_validation_errors_match_reference_types():
    """sorter.py:302-314: raised before any device work."""
    with pytest.raises(TypeError):
        cafs.cafs_sort([3, 1, 2])
    with pytest.raises(TypeError):
        cafs.cafs_sort(np.zeros(4, np.float64))
    with pytest.raises(ValueError):
        cafs.cafs_sort(np.zeros((2, 2), np.uint64))
    ro = np.zeros(4, np.uint64)
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        cafs.cafs_sort(ro)
    with pytest.raises(ValueError):
        cafs.cafs_sort(np.zeros(4, np.uint64), hash_mult=4)
    import torch
    with pytest.raises(TypeError):
        cafs.cafs_sort(torch.zeros(4, dtype=torch.float32))
    with pytest.raises(ValueError):
        cafs.cafs_sort(torch.zeros((2, 2), dtype=torch.int64))


def test_api_surface_mirrors_reference():
    # sorter.py:44-49 Route values, :52-57 DispatchDecision, :60-81 SortTelemetry,
    # cardinality.py:76-82 CardinalityEstimate
    assert [r.value for r in cafs.Route] == [
        "already_sorted", "fallback_small_n", "tiny_count", "fallback_high_entropy", "main"]
    assert [f.name for f in dataclasses.fields(cafs.DispatchDecision)] == [
        "route", "keys", "k_hat", "estimate"]
    assert [f.name for f in dataclasses.fields(cafs.CardinalityEstimate)] == [
        "k_hat", "u", "f1", "f2", "saturated"]
    ref_tel = ["n", "decision", "spill_len", "guard_fired", "stage_ms", "counted_total",
               "updates", "tiny_count_failed", "table"]
    assert [f.name for f in dataclasses.fields(cafs.SortTelemetry)][:len(ref_tel)] == ref_tel
    assert cafs.SortTelemetry().route is None
    assert (cafs.SMALL_N_CUTOFF, cafs.TINY_MAX_KEYS, cafs.SAMPLE_TARGET) == (2048, 8, 1024)
    pl = cafs.PairList.from_pairs([(5, 2), (1, 3)])
    assert pl.to_pairs() == [(5, 2), (1, 3)] and len(pl) == 2


def test_package_configs_match_oracle_configs():
    for name, c in datagen.CONFIGS.items():
        o = ogen.CONFIGS[name]
        assert (c.n, c.k, c.dist, c.s, c.palette, c.seed) == (o.n, o.k, o.dist, o.s, o.palette,
                                                              o.seed)
        if c.dist == "zipf":
            assert np.array_equal(datagen.zipf_cdf(c.k, c.s), o.cdf())


def test_config_seeds_route_as_intended():
    rec = {r["name"]: r["route"] for r in load_json("config_cases.json")}
    assert rec == {"cfg1": "main", "cfg2": "tiny_count", "cfg3": "main",
                   "cfg5": "fallback_high_entropy", "cfg4": "main"}


def test_distributed_fallback_bucket_ranges():
    """Bucket ranges of the distributed fallback (sharded._exchange_sort)."""
    from paper_2605_25040_b200.sharded import bucket_ranges, msd_shift
    assert msd_shift(0, 0) == 0
    assert msd_shift(0, 0xFFF) == 0
    assert msd_shift(0, 0x1FFF) == 1
    assert msd_shift(0, (1 << 64) - 1) == 52
    assert msd_shift(0x8000_0000_0000_0000, 0x8000_0000_0000_00FF) == 0
    # sign-extended int32 keys: a 2^32 span although all 32 high bits vary
    assert msd_shift(0x7FFF_FFFF_8000_0000, 0x8000_0000_7FFF_FFFF) == 20
    rng = np.random.default_rng(3)
    for _ in range(200):
        totals = rng.integers(0, 5, 16) * rng.integers(0, 2, 16)
        n = int(totals.sum())
        cuts = np.sort(rng.integers(0, n + 1, rng.integers(1, 5)))
        sizes = np.diff(np.concatenate([[0], cuts, [n]])).tolist()
        P = np.concatenate([[0], np.cumsum(totals)])
        off = 0
        for (lo, hi), s in zip(bucket_ranges(totals, sizes), sizes):
            if s == 0:
                assert lo == hi
            else:
                # the received buckets cover the slice, and no bucket is needless
                assert P[lo] <= off and P[hi] >= off + s
                assert totals[lo] > 0 and totals[hi - 1] > 0
            off += s


def test_host_tables_match_oracle_telemetry():
    """The exported host BucketTable / FreqSet (the reference API's counting
    structures) reproduce the oracle's (= the reference's) table statistics and
    estimate on the same inputs."""
    from oracle import cafs_oracle as orc
    from oracle import gen as ogen

    for n, k, seed in ((20_000, 300, 1), (30_000, 3000, 2), (9_000, 40, 3)):
        x = ogen.gen_input(n, k, seed).view(np.int64)
        ot = orc.cafs_sort(x.copy())
        assert ot.route == "main"
        xu = x.view(np.uint64) ^ np.uint64(1 << 63)
        t = cafs.BucketTable(int(ot.table_buckets).bit_length() - 1)
        t.count_sequence(xu)
        s = t.stats
        assert (s.updates, s.hits, s.claims, s.spill_pushes, s.spill_len) == (
            ot.updates, ot.hits, ot.claims, ot.spill_pushes, ot.spill_len)
        assert t.counted_total() == ot.counted_total
        assert t.spill.shape[0] == ot.spill_len
        keys, counts = t.occupied_pairs()
        assert int(counts.sum()) + ot.spill_len == n
        fs = cafs.FreqSet()
        stride = n // 1024
        for v in xu[: 1024 * stride: stride]:
            fs.insert(int(v))
        e = ot.decision.estimate
        assert fs.spectrum() == (e.u, e.f1, e.f2)


def test_bucket_update_rules():
    b = cafs.Bucket.empty()
    assert b.cap == 4
    assert cafs.bucket_update(b, 0)          # a zero key matches the empty slot 0
    assert b.counts.tolist() == [1, 0, 0, 0]
    for v in (5, 6, 7):
        assert cafs.bucket_update(b, v, 2)
    assert not cafs.bucket_update(b, 8)       # full: the caller spills
    assert cafs.bucket_update(b, 6)
    assert b.keys.tolist() == [0, 5, 6, 7] and b.counts.tolist() == [1, 2, 3, 2]
    with pytest.raises(ValueError):
        cafs.bucket_update(b, 5, 0)
    assert cafs.Bucket.empty(np.uint32).cap == 8
