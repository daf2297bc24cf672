"""Pin the CPU oracle to the reference's own outputs (CPU only).

The golden fixtures were produced by running the real reference package
(tests/golden/make_golden.py).  The oracle is trusted as the GPU parity checker
only because every case here matches: the sorted bytes, the dispatch tuple
(route, k_hat, u, f1, f2, saturated, tiny keys) and the reference's telemetry
counters (spill_len, guard_fired, counted_total, updates, hits, claims).
"""

import hashlib

import numpy as np
import pytest

from conftest import dtype32_input, load_json, special_input, sweep_input
from oracle import cafs_oracle as orc
from oracle import gen as ogen


def _sha(x):
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def _check(rec, x, mult=orc.HASH_MULT):
    n = x.shape[0]
    d = orc.dispatch(x, mult) if n > 1 else None
    if d is not None:
        assert d.route == rec["dispatch_route"]
        if rec.get("tiny_keys") is not None:
            assert d.keys == rec["tiny_keys"]
    y = x.copy()
    tel = orc.cafs_sort(y, mult)
    assert _sha(y) == rec["sha256"]
    assert tel.route == rec["route"]
    if rec["k_hat"] is not None:
        e = tel.decision.estimate
        assert (e.k_hat, e.u, e.f1, e.f2, e.saturated) == (
            rec["k_hat"], rec["u"], rec["f1"], rec["f2"], rec["saturated"])
    assert tel.spill_len == rec["spill_len"]
    assert tel.guard_fired == rec["guard_fired"]
    assert tel.tiny_count_failed == rec["tiny_count_failed"]
    if "table_buckets" in rec:
        assert tel.counted_total == rec["counted_total"]
        assert tel.updates == rec["updates"]
        assert (tel.table_buckets, tel.hits, tel.claims, tel.spill_pushes) == (
            rec["table_buckets"], rec["hits"], rec["claims"], rec["spill_pushes"])


def test_known_answer_hash(known_answers):
    for row in known_answers["fast_hash"]:
        v, m, want = row[:3]
        mult = row[3] if len(row) > 3 else orc.HASH_MULT
        assert orc.fast_hash(v, m, mult) == want


def test_known_answer_table_size(known_answers):
    for k_hat, n, cap, want in known_answers["table_size_for"]:
        assert orc.table_size_for(k_hat, n, cap) == want


def test_known_answer_chao1(known_answers):
    for u, f1, f2, n, sat, want in known_answers["chao1"]:
        assert orc.chao1(u, f1, f2, n, sat) == want  # bit-exact float64


def test_known_answer_mix(known_answers):
    m = known_answers["mix_outputs"]
    assert ogen.mix_outputs(m["seed"], len(m["outputs"])).tolist() == m["outputs"]


@pytest.mark.parametrize("rec", load_json("special_cases.json"), ids=lambda r: r["name"])
def test_special_cases(rec):
    x = special_input(rec["name"])
    _check(rec, x, rec.get("hash_mult", orc.HASH_MULT))


def test_reference_sweep():
    cases = load_json("sweep_cases.json")
    assert len(cases) == 250
    routes = set()
    for rec in cases:
        _check(rec, sweep_input(rec))
        routes.add(rec["route"])
    assert routes == set(orc.ROUTES)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_baseline_configs(name):
    rec = {r["name"]: r for r in load_json("config_cases.json")}[name]
    x = ogen.CONFIGS[name].generate()
    _check(rec, x)


def test_cfg4_dispatch_sparse():
    """cfg4 is 2^30 rows: check its dispatch from the rows dispatch reads."""
    rec = {r["name"]: r for r in load_json("config_cases.json")}["cfg4"]
    c = ogen.CONFIGS["cfg4"]
    stride = c.n // 1024
    head = c.generate(65536, 0)
    assert not orc.is_monotone(head)
    samples = np.concatenate([c.generate(1, i * stride) for i in range(1024)])
    # sample_and_estimate of exactly the 1024 sampled rows, with n = 2^30
    e = orc.sample_and_estimate(samples)
    k_hat = orc.chao1(e.u, e.f1, e.f2, c.n, e.saturated)
    assert (k_hat, e.u, e.f1, e.f2, e.saturated) == (
        rec["k_hat"], rec["u"], rec["f1"], rec["f2"], rec["saturated"])
    assert orc.table_size_for(k_hat, c.n, 4) == rec["table_buckets"]


@pytest.mark.parametrize("rec", load_json("dtype32_cases.json"), ids=lambda r: r["name"])
def test_dtype32_cases_match_widened_oracle(rec):
    """A 32-bit column sorts and dispatches exactly as its int64 widening: the
    premise of the device's 32-bit path (keys widened in registers).  The
    bucket-table counters hash in the 32-bit unsigned domain and are checked
    against these goldens on the GPU (tests/test_gpu_parity.py)."""
    x = dtype32_input(rec["name"])
    w = x.astype(np.int64)
    y = w.copy()
    tel = orc.cafs_sort(y, rec.get("hash_mult", orc.HASH_MULT))
    assert _sha(y.astype(x.dtype)) == rec["sha256"]
    assert tel.route == rec["route"]  # the guard keeps the route MAIN (sorter.py:264-273)
    if rec["k_hat"] is not None:
        e = tel.decision.estimate
        assert (e.k_hat, e.u, e.f1, e.f2, e.saturated) == (
            rec["k_hat"], rec["u"], rec["f1"], rec["f2"], rec["saturated"])
    assert tel.tiny_count_failed == rec["tiny_count_failed"]


def test_checker_fails_on_an_injected_fault():
    """Negative control (the reference's fault_point pattern, selftest.py:84-105):
    one corrupted output element, a wrong dispatch tuple or a wrong telemetry
    counter must each make the golden check fail."""
    recs = load_json("special_cases.json")
    rec = next(r for r in recs if r["route"] == "main" and "table_buckets" in r)
    x = special_input(rec["name"])
    _check(rec, x)  # the clean case passes
    y = x.copy()
    orc.cafs_sort(y)
    y[y.shape[0] // 2] ^= 1  # one flipped bit in the sorted output
    assert _sha(y) != rec["sha256"]
    for field, bad in (("route", "tiny_count"), ("u", rec["u"] + 1),
                       ("spill_len", rec["spill_len"] + 1)):
        with pytest.raises(AssertionError):
            _check(dict(rec, **{field: bad}), x)


def test_c_generator_matches_numpy_generator():
    """oracle.cafs_oracle.generate (the C generator the CPU baseline uses at full
    size) is bit-identical to oracle/gen.py on every config, threaded and not."""
    from oracle import cafs_oracle as orc
    from oracle import gen as ogen

    for c in ogen.CONFIGS.values():
        for start, n, thr in ((0, 70_000, 1), (987_654, 200_001, 5)):
            assert np.array_equal(orc.generate(c, n, start, threads=thr), c.generate(n, start)), c.name
