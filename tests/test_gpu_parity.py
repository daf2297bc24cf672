"""GPU parity: the sm_100a pipeline against the oracle and the reference's goldens.

Every case compares the sorted bytes (bit-exact) and the dispatch tuple
(route, k_hat, u, f1, f2, saturated, tiny keys, tiny_count_failed) with the
values the real reference produced (tests/golden/*.json), and where useful
with the C oracle run on the same box.  All calls go through the package's
public API and therefore the C ABI of libcafs_b200.so.
"""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import dtype32_input, load_json, special_input, sweep_input  # noqa: E402
from oracle import cafs_oracle as orc  # noqa: E402
from oracle import gen as ogen  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_25040_b200 as cafs  # noqa: E402
from paper_2605_25040_b200 import Route, SortTelemetry  # noqa: E402


def sha(a) -> str:
    if isinstance(a, torch.Tensor):
        a = a.cpu().numpy()
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def to_dev(x: np.ndarray):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def check_decision(tel: SortTelemetry, rec: dict):
    assert tel.route.value == rec["route"]
    assert tel.tiny_count_failed == rec.get("tiny_count_failed", False)
    if rec["k_hat"] is None:
        assert tel.decision.estimate is None
    else:
        e = tel.decision.estimate
        assert (e.k_hat, e.u, e.f1, e.f2, e.saturated) == (
            rec["k_hat"], rec["u"], rec["f1"], rec["f2"], rec["saturated"])
    if rec["route"] == "main" and "table_buckets" in rec:
        assert tel.table_buckets == rec["table_buckets"]


def check_exact(tel: SortTelemetry, rec: dict):
    """The reference's bucket-table telemetry, computed on device."""
    assert tel.exact
    assert (tel.spill_len, tel.guard_fired, tel.updates) == (
        rec["spill_len"], rec["guard_fired"], rec["updates"])
    if "table_buckets" in rec:
        assert tel.counted_total == rec["counted_total"]
        t = tel.table
        assert (t.n_buckets, t.hits, t.claims, t.spill_pushes) == (
            rec["table_buckets"], rec["hits"], rec["claims"], rec["spill_pushes"])


def run_case(x: np.ndarray, rec: dict, mult=None, exact=True):
    t = to_dev(x)
    tel = SortTelemetry()
    cafs.cafs_sort(t, telemetry=tel, hash_mult=mult, exact_telemetry=exact)
    torch.cuda.synchronize()
    assert sha(t) == rec["sha256"], "sorted bytes differ from the reference"
    check_decision(tel, rec)
    if exact:
        check_exact(tel, rec)
    if x.shape[0] > 1:
        # the reference's dispatch takes the unsigned-domain copy (sorter.py:357)
        xu = x.view(np.uint64) ^ np.uint64(1 << 63) if x.dtype == np.int64 else x
        d = cafs.dispatch(to_dev(xu), hash_mult=mult)
        assert d.route.value == rec["dispatch_route"]
        if rec.get("tiny_keys") is not None:
            assert d.keys.tolist() == rec["tiny_keys"]
            if x.dtype == np.int64:
                # signed input as it is: the keys are the values' raw bits,
                # ascending as unsigned (the reference's uint64 FreqSet)
                ds = cafs.dispatch(to_dev(x), hash_mult=mult)
                want = sorted(int(k) ^ (1 << 63) for k in rec["tiny_keys"])
                assert ds.keys.tolist() == want
    assert set(tel.stage_ms) <= {"count", "sort_k", "emit"}
    return tel


@pytest.mark.parametrize("rec", load_json("special_cases.json"), ids=lambda r: r["name"])
def test_special_cases(rec):
    x = special_input(rec["name"])
    tel = run_case(x, rec, rec.get("hash_mult"))
    # stage labels as the reference records them (the GPU guard is its own)
    if not tel.guard_fired and not rec["guard_fired"]:
        assert sorted(tel.stage_ms) == rec["stage_keys"]


def test_reference_sweep():
    cases = load_json("sweep_cases.json")
    routes = set()
    for i, rec in enumerate(cases):
        # alternate: the fused fast path, and the exact-telemetry path
        tel = run_case(sweep_input(rec), rec, exact=bool(i % 2))
        routes.add(tel.route)
    assert routes == set(Route)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_baseline_config(name):
    rec = {r["name"]: r for r in load_json("config_cases.json")}[name]
    x = ogen.CONFIGS[name].generate()
    run_case(x, rec)


def _device_config(name, n=None, start=0):
    c = ogen.CONFIGS[name]
    n = c.n - start if n is None else n
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    pal = None if c.palette == "codes" else to_dev(c.palette_values())
    cdf = None if c.dist != "zipf" else to_dev(c.cdf())
    lib = cafs.sorter._lib.load()
    rc = lib.cafs_gen_draw(out.data_ptr(), n, start, c.seed, 0 if pal is None else pal.data_ptr(),
                           c.k, 0 if cdf is None else cdf.data_ptr(),
                           torch.cuda.current_stream().cuda_stream)
    assert rc == 0
    return out


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_device_generator_matches_numpy(name):
    c = ogen.CONFIGS[name]
    for start in (0, c.n // 3, c.n - 5000):
        d = _device_config(name, 5000, start).cpu().numpy()
        assert np.array_equal(d, c.generate(5000, start))


def test_cfg4_full_size_properties():
    """N = 2^30: sortedness, per-code histogram and the dispatch tuple."""
    rec = {r["name"]: r for r in load_json("config_cases.json")}["cfg4"]
    x = _device_config("cfg4")
    hist_in = torch.bincount(x, minlength=4096)
    tel = SortTelemetry()
    cafs.cafs_sort(x, telemetry=tel)
    torch.cuda.synchronize()
    check_decision(tel, rec)
    assert not tel.guard_fired and tel.counted_total == x.shape[0]
    assert bool((x[1:] >= x[:-1]).all())
    assert torch.equal(torch.bincount(x, minlength=4096), hist_in)
    del x


def test_numpy_dropin_matches_reference():
    """numpy input takes the host entry point (H2D, device pipeline, D2H)."""
    for rec in load_json("special_cases.json")[:8]:
        x = special_input(rec["name"])
        tel = SortTelemetry()
        cafs.cafs_sort(x, telemetry=tel, hash_mult=rec.get("hash_mult"))
        assert sha(x) == rec["sha256"]
        check_decision(tel, rec)


@pytest.mark.parametrize("dtype", [np.int64, np.uint64, np.int32, np.uint32])
@pytest.mark.parametrize("seed", range(3))
def test_all_dtypes_torch_and_numpy(dtype, seed):
    rng = np.random.default_rng(seed * 31 + 1)
    info = np.iinfo(dtype)
    n = int(rng.integers(2, 200_000))
    k = int(rng.integers(1, min(n, 3000)))
    pal = rng.integers(info.min, int(info.max) + 1, k, dtype=dtype)
    x = pal[rng.integers(0, k, n)]
    want = np.sort(x)
    y = x.copy()
    cafs.cafs_sort(y)
    assert np.array_equal(y, want)
    t = torch.from_numpy(x.copy()).cuda()
    cafs.cafs_sort(t)
    assert np.array_equal(t.cpu().numpy(), want)


def test_strided_views():
    base = ogen.gen_input(40_000, 32)
    x = base[::2]
    want = np.sort(x)
    cafs.cafs_sort(x)
    assert np.array_equal(x, want)
    t = torch.from_numpy(ogen.gen_input(40_000, 32).view(np.int64)).cuda()[::2]
    want = np.sort(t.cpu().numpy())
    cafs.cafs_sort(t)
    assert np.array_equal(t.cpu().numpy(), want)


def test_empty_singleton_and_two():
    for x in (np.empty(0, np.int64), np.array([9], np.int64)):
        tel = SortTelemetry()
        cafs.cafs_sort(x, telemetry=tel)
        assert tel.route is Route.ALREADY_SORTED
    t = torch.tensor([5, -3], dtype=torch.int64, device="cuda")
    tel = SortTelemetry()
    cafs.cafs_sort(t, telemetry=tel)
    assert t.tolist() == [-3, 5] and tel.route is Route.FALLBACK_SMALL_N


def test_sliced_unaligned_tensor():
    """x[1:] is 8-byte but not 16-byte aligned: head/tail paths of every kernel."""
    for name in ("cfg1", "cfg2", "cfg5"):
        full = torch.from_numpy(ogen.CONFIGS[name].generate(300_001)).cuda()
        t = full[1:]
        want = np.sort(t.cpu().numpy())
        cafs.cafs_sort(t)
        assert np.array_equal(t.cpu().numpy(), want)
        assert full[0].item() == ogen.CONFIGS[name].generate(1)[0]


def test_stage_apis_against_oracle():
    x = ogen.CONFIGS["cfg1"].generate(200_000)
    est = cafs.sample_and_estimate(to_dev(x))
    oe = orc.sample_and_estimate(x)
    assert (est.k_hat, est.u, est.f1, est.f2, est.saturated) == (
        oe.k_hat, oe.u, oe.f1, oe.f2, oe.saturated)
    e = cafs.sample_and_estimate(np.array([3, 3, 5], np.uint64))
    assert (e.u, e.f1, e.f2, e.k_hat) == (2, 1, 1, min(2 + 1 / 4, 3))
    e = cafs.sample_and_estimate(np.full(1024, 7, np.uint64))
    assert (e.k_hat, e.u, e.f1, e.f2, e.saturated) == (1.0, 1, 0, 0, False)
    # tiny counts (keys in the unsigned domain of the array)
    x2 = ogen.CONFIGS["cfg2"].generate(100_000)
    vals = np.unique(x2)  # int64, the array's own domain
    got = cafs.tiny_counts(to_dev(x2), vals)
    assert got.tolist() == orc.tiny_counts(x2, vals.view(np.uint64) ^ np.uint64(1 << 63)).tolist()
    assert int(got.sum()) == x2.shape[0]
    # monotone
    assert cafs.is_monotone(to_dev(np.arange(200_000, dtype=np.int64)))
    y = np.arange(200_000, dtype=np.int64)
    y[150_000] = -1
    assert not cafs.is_monotone(to_dev(y))
    assert cafs.is_monotone(np.array([-5, -1, 0, 3], np.int64))
    assert not cafs.is_monotone(np.array([0, -1], np.int64))


def test_tiny_count_sort_semantics():
    rng = np.random.default_rng(1)
    keys = np.arange(1, 9, dtype=np.uint64)
    x = keys[rng.integers(0, 8, 5000)]
    x[17] = 1000
    out = np.full_like(x, 77)
    assert not cafs.tiny_count_sort(x, keys, out)
    assert np.all(out == 77)
    x = np.array([2, 1, 2, 1, 1], np.uint64)
    assert cafs.tiny_count_sort(x, np.array([1, 2], np.uint64), x)
    assert x.tolist() == [1, 1, 1, 2, 2]
    with pytest.raises(ValueError):
        cafs.tiny_count_sort(np.zeros(4, np.uint64), np.arange(9, dtype=np.uint64),
                             np.zeros(4, np.uint64))


@pytest.mark.parametrize("n", [1, 5, 255, 256, 8192, 8193, 100_000, 1_500_000])
def test_pair_sort_and_emit(n):
    rng = np.random.default_rng(n)
    keys = np.unique(rng.integers(0, 1 << 64, n, dtype=np.uint64))
    rng.shuffle(keys)
    counts = rng.integers(1, 5, keys.shape[0]).astype(np.int64)
    pl = cafs.pair_sort(cafs.PairList(keys, counts))
    order = np.argsort(keys)
    assert np.array_equal(pl.keys, keys[order]) and np.array_equal(pl.counts, counts[order])
    out = np.empty(int(counts.sum()), np.uint64)
    cafs.emit(pl, out)
    assert np.array_equal(out, np.repeat(keys[order], counts[order]))
    with pytest.raises(ValueError):
        cafs.emit(pl, np.empty(int(counts.sum()) + 1, np.uint64))


def test_fallback_sort_large_random():
    for n in (8191, 8192, 8193, 1_000_003, 12_000_000):
        x = ogen.mix_outputs(n, n).view(np.int64)
        want = np.sort(x)
        t = to_dev(x)
        cafs.fallback_sort(t)
        assert np.array_equal(t.cpu().numpy(), want)


def test_fallback_sort_few_negative_keys():
    """The key span must see a handful of sign changes among millions of keys."""
    x = (ogen.mix_outputs(31, 3_000_000) >> np.uint64(1)).view(np.int64).copy()
    x[[5, 1_000_001, 2_999_998]] = [-1, -(1 << 62), -7]
    want = np.sort(x)
    t = to_dev(x)
    cafs.fallback_sort(t)
    assert np.array_equal(t.cpu().numpy(), want)


def test_fallback_sort_clustered_and_repeated():
    """Buckets whose sub-buckets are large (repeats, clusters) take the byte passes."""
    rng = np.random.default_rng(12)
    n = 4_000_000
    x = ogen.mix_outputs(21, n).view(np.int64).copy()
    x[rng.integers(0, n, n // 3)] = 77                      # one heavy key
    x[rng.integers(0, n, n // 5)] = rng.integers(0, 3000, n // 5) << 20  # low-entropy cluster
    for arr in (x, x.view(np.uint64)):
        want = np.sort(arr)
        t = torch.from_numpy(arr.copy()).cuda() if arr.dtype == np.int64 else arr.copy()
        cafs.fallback_sort(t)
        got = t.cpu().numpy() if isinstance(t, torch.Tensor) else t
        assert np.array_equal(got, want)


def test_guard_reroutes_to_fallback():
    """More distinct keys than the global table holds (16 Mi), under a low estimate."""
    n = 20_000_000
    x = ogen.mix_outputs(77, n).view(np.int64).copy()
    stride = n // 1024
    x[::stride][:1024] = np.arange(1024, dtype=np.int64) % 100  # sample sees 100 keys
    want = np.sort(x)
    t = to_dev(x)
    tel = SortTelemetry()
    cafs.cafs_sort(t, telemetry=tel)
    assert tel.route is Route.MAIN and tel.guard_fired
    assert np.array_equal(t.cpu().numpy(), want)


def test_hash_mult_validation_and_override():
    x = to_dev(ogen.gen_input(100_000, 300).view(np.int64))
    with pytest.raises(ValueError):
        cafs.cafs_sort(x, hash_mult=2)
    want = np.sort(x.cpu().numpy())
    cafs.cafs_sort(x, hash_mult=0xC2B2AE3D27D4EB4F)
    assert np.array_equal(x.cpu().numpy(), want)


def test_direct_range_off_matches():
    x = ogen.CONFIGS["cfg4"].generate(3_000_000)
    want = np.sort(x)
    for direct in (True, False):
        t = to_dev(x)
        cafs.cafs_sort(t, direct_range=direct)
        assert np.array_equal(t.cpu().numpy(), want)


def test_determinism_and_repeat_calls():
    x = ogen.CONFIGS["cfg3"].generate(2_000_000)
    outs = set()
    for _ in range(3):
        t = to_dev(x)
        cafs.cafs_sort(t)
        outs.add(sha(t))
    assert len(outs) == 1 and outs == {sha(np.sort(x))}


def _dense_mix(kind: str) -> np.ndarray:
    """Dictionary codes (inside the dense window) plus out-of-window keys."""
    rng = np.random.default_rng(len(kind))
    x = rng.integers(-2000, 2000, 1_500_000, dtype=np.int64)
    if kind == "outliers":  # append mode: hash pairs + dense pairs, one sort
        x[rng.integers(0, x.shape[0], 3000)] = rng.integers(-(1 << 62), 1 << 62, 3000)
    elif kind == "sentinel":  # the key whose order-mapped value is ~0
        x[::1000] = np.iinfo(np.int64).max
    elif kind == "many_outliers":  # > kSmallSortMax pairs in total: the large sort
        x[rng.integers(0, x.shape[0], 40_000)] = rng.integers(-(1 << 62), 1 << 62, 40_000)
    return x


@pytest.mark.parametrize("kind", ["codes", "outliers", "sentinel", "many_outliers"])
@pytest.mark.parametrize("exact", [False, True])
def test_dense_window_paths(kind, exact):
    x = _dense_mix(kind)
    want = x.copy()
    ot = orc.cafs_sort(want)
    t = to_dev(x)
    tel = SortTelemetry()
    cafs.cafs_sort(t, telemetry=tel, exact_telemetry=exact)
    assert sha(t) == sha(want)
    assert tel.route.value == ot.route
    if exact:
        assert (tel.spill_len, tel.guard_fired, tel.updates, tel.counted_total) == (
            ot.spill_len, ot.guard_fired, ot.updates, ot.counted_total)
        t_ = tel.table
        assert (t_.hits, t_.claims, t_.spill_pushes) == (ot.hits, ot.claims, ot.spill_pushes)
    # the stage API the sharded sort uses (count -> pairs) sees the same pairs
    from paper_2605_25040_b200.sharded import DeviceOps
    keys, counts = np.unique(x, return_counts=True)
    k, c = DeviceOps(0).count_pairs(to_dev(x), cafs.HASH_MULT)
    order_mapped = keys.view(np.uint64) ^ np.uint64(1 << 63)
    assert np.array_equal(k.cpu().numpy().view(np.uint64), order_mapped)
    assert np.array_equal(c.cpu().numpy(), counts)


def test_guard_then_dense_window():
    """A guard that fires mid-count must not leave dense-window counts behind."""
    n = 24_000_000
    x = ogen.mix_outputs(78, n).view(np.int64).copy()
    stride = n // 1024
    x[::stride][:1024] = np.arange(1024, dtype=np.int64) % 100  # low estimate + a window
    x[:n // 4] = np.arange(n // 4) % 100  # many rows land in the window
    tel = SortTelemetry()
    t = to_dev(x)
    cafs.cafs_sort(t, telemetry=tel)
    assert tel.guard_fired and np.array_equal(t.cpu().numpy(), np.sort(x))
    y = ogen.CONFIGS["cfg4"].generate(1_000_000)
    t = to_dev(y)
    cafs.cafs_sort(t)
    assert np.array_equal(t.cpu().numpy(), np.sort(y))


@pytest.mark.parametrize("rec", load_json("dtype32_cases.json"), ids=lambda r: r["name"])
def test_dtype32_native_path(rec):
    """int32 / uint32 columns on the 4-byte-key path (cafs_sort_i32): sorted
    bytes, decision and the reference's bucket-table telemetry (hashed in the
    32-bit unsigned domain) against the reference's own outputs."""
    x = dtype32_input(rec["name"])
    mult = rec.get("hash_mult")
    for exact in (False, True):
        t = to_dev(x)
        tel = SortTelemetry()
        cafs.cafs_sort(t, telemetry=tel, hash_mult=mult, exact_telemetry=exact)
        torch.cuda.synchronize()
        assert sha(t) == rec["sha256"]
        check_decision(tel, rec)
        if exact:
            check_exact(tel, rec)
    y = x.copy()  # numpy: 4 bytes per key over PCIe (cafs_sort_i32_host)
    cafs.cafs_sort(y, hash_mult=mult)
    assert sha(y) == rec["sha256"]
    if x.shape[0] > 4:  # a view 4 bytes past a 16-byte boundary: head/tail paths
        full = to_dev(np.concatenate([x[:1], x]))
        v = full[1:]
        cafs.cafs_sort(v, hash_mult=mult)
        assert np.array_equal(v.cpu().numpy(), np.sort(x)) and full[0].item() == x[0]


@pytest.mark.parametrize("dtype", [np.int32, np.uint32])
def test_dtype32_routes_at_scale(dtype):
    """Large 32-bit columns through every route, including the guard."""
    info = np.iinfo(dtype)
    rng = np.random.default_rng(77)
    cases = {
        "tiny": np.array([info.min, 0, 5, info.max], dtype)[rng.integers(0, 4, 8_000_000)],
        "dense": (np.minimum(rng.zipf(1.2, 6_000_000), 4000) + (0 if dtype == np.uint32 else -2000)).astype(dtype),
        "hash": rng.integers(info.min, info.max, 200_000, dtype=dtype)[rng.integers(0, 200_000, 5_000_000)],
        "fallback": rng.integers(info.min, info.max, 3_000_001, dtype=dtype),
    }
    z = np.minimum(rng.zipf(1.2, 3_000_000), 3000).astype(np.int64)
    # dense windows at the edges of the 32-bit domain (the 32-bit window test
    # applies only when the window lies inside it)
    cases["dense_top"] = (int(info.max) - z).astype(dtype)
    cases["dense_bottom"] = (int(info.min) + z).astype(dtype)
    cases["dense_mid"] = (z + (1 << 20)).astype(dtype)
    g = ogen.mix_outputs(5, 20_000_000).astype(dtype)  # ~all distinct (> 16 Mi) ...
    g[::20_000_000 // 1024][:1024] = (np.arange(1024) % 100).astype(dtype)  # ... low estimate
    cases["guard"] = g
    for name, x in cases.items():
        t = to_dev(x)
        tel = SortTelemetry()
        cafs.cafs_sort(t, telemetry=tel)
        assert np.array_equal(t.cpu().numpy(), np.sort(x)), name
        if name == "guard":
            assert tel.route is Route.MAIN and tel.guard_fired


@pytest.mark.parametrize("direct", [True, False])
def test_graph_replay_every_route(direct):
    """Repeated sorts of one buffer: the 1st call runs the gated pipeline, the
    2nd captures a CUDA graph with conditional route bodies, later calls replay
    it -- for every route, including a tiny-count miss and the 32-bit path."""
    rng = np.random.default_rng(99)
    tiny = np.array([-5, 3, 1 << 40], np.int64)[rng.integers(0, 3, 500_000)]
    miss = tiny.copy()
    miss[7] = 11  # never sampled: the tiny route re-enters MAIN
    inputs = {
        "tiny": tiny, "tiny_miss": miss,
        "dense": (np.minimum(rng.zipf(1.3, 800_000), 3000)).astype(np.int64),
        "hash": ogen.CONFIGS["cfg3"].generate(600_000),
        "fallback": ogen.mix_outputs(3, 400_000).view(np.int64).copy(),
        "sorted": np.arange(-100_000, 100_000, dtype=np.int64),
        "dense_i32": (np.minimum(rng.zipf(1.3, 800_000), 3000) - 1500).astype(np.int32),
        "hash_i32": rng.integers(-2**31, 2**31 - 1, 50_000, dtype=np.int32)[rng.integers(0, 50_000, 700_000)],
    }
    for name, x in inputs.items():
        want = np.sort(x)
        pristine = to_dev(x)
        t = torch.empty_like(pristine)
        for it in range(4):
            t.copy_(pristine)
            cafs.cafs_sort(t, direct_range=direct)
            assert np.array_equal(t.cpu().numpy(), want), (name, it)
        tel = SortTelemetry()  # and a telemetry call on the same buffer (timed graph)
        t.copy_(pristine)
        cafs.cafs_sort(t, telemetry=tel, direct_range=direct)
        assert np.array_equal(t.cpu().numpy(), want), name
        assert tel.tiny_count_failed == (name == "tiny_miss")


@pytest.mark.parametrize("dtype", [np.int64, np.int32])
def test_no_writes_outside_the_column(dtype):
    """Canary rows on both sides of a sorted slice stay untouched, on every
    route and alignment (no memory checker on the pool: bounds by test)."""
    rng = np.random.default_rng(2024)
    info = np.iinfo(dtype)
    cases = {
        "tiny": np.array([info.min, 0, 9], dtype)[rng.integers(0, 3, 300_007)],
        "dense": (np.minimum(rng.zipf(1.3, 300_011), 3000)).astype(dtype),
        "hash": rng.integers(info.min, info.max, 30_000, dtype=dtype)[rng.integers(0, 30_000, 5_000_003)],
        "fallback": rng.integers(info.min, info.max, 200_003, dtype=dtype),
        "small": rng.integers(-50, 50, 1_999).astype(dtype),
    }
    canary = np.array(0x5A5A5A5A, dtype=dtype)
    for name, x in cases.items():
        for lead in (0, 1, 3):
            buf = np.full(lead + x.shape[0] + 8, canary, dtype)
            buf[lead:lead + x.shape[0]] = x
            full = to_dev(buf)
            t = full[lead:lead + x.shape[0]]
            cafs.cafs_sort(t)
            got = full.cpu().numpy()
            assert np.array_equal(got[lead:lead + x.shape[0]], np.sort(x)), (name, lead)
            assert np.all(got[:lead] == canary) and np.all(got[lead + x.shape[0]:] == canary), (name, lead)


def test_large_pageable_numpy_staged_transfers():
    """Pageable numpy arrays above the staging threshold go through the
    multi-threaded pinned staging in both directions (int64 and int32)."""
    rng = np.random.default_rng(77)
    for x in (rng.integers(-3000, 3000, 40_000_003).astype(np.int64),
              rng.integers(-2**31, 2**31 - 1, 30_000_001, dtype=np.int32),
              ogen.mix_outputs(9, 12_000_000).view(np.int64).copy()):
        want = np.sort(x)
        cafs.cafs_sort(x)
        assert np.array_equal(x, want)


def _fuzz_input(rng):
    kind = rng.integers(0, 6)
    n = int(rng.choice([0, 1, 2, 3, 100, 2047, 2048, 2049, 5000, 16385, 16386, 70_000, 300_000]))
    if kind == 0:    # tiny alphabet
        pal = rng.integers(-2**63, 2**63 - 1, int(rng.integers(1, 9)), dtype=np.int64)
    elif kind == 1:  # dictionary codes around a random base
        base = int(rng.integers(-2**62, 2**62))
        pal = base + np.arange(int(rng.integers(2, 6000)), dtype=np.int64)
    elif kind == 2:  # random palette
        pal = rng.integers(-2**63, 2**63 - 1, int(rng.integers(9, 50_000)), dtype=np.int64)
    elif kind == 3:  # all distinct
        return rng.permutation(rng.integers(-2**63, 2**63 - 1, n, dtype=np.int64))
    elif kind == 4:  # sorted, with maybe one inversion
        x = np.sort(rng.integers(-1000, 1000, n).astype(np.int64))
        if n > 2 and rng.integers(0, 2):
            i = int(rng.integers(0, n - 1))
            x[i], x[i + 1] = x[i + 1] + 1, x[i]
        return x
    else:            # extremes
        info = np.iinfo(np.int64)
        pal = np.array([info.min, info.min + 1, -1, 0, 1, info.max - 1, info.max], np.int64)
    if n == 0:
        return np.empty(0, np.int64)
    w = rng.zipf(1.2, pal.shape[0]).astype(np.float64) if rng.integers(0, 2) else None
    p = None if w is None else w / w.sum()
    return pal[rng.choice(pal.shape[0], n, p=p)]


@pytest.mark.parametrize("seed", range(6))
def test_fuzz_against_oracle(seed):
    """Seeded random columns over every route, size edge and dtype: sorted
    bytes equal np.sort and the decision equals the C oracle's."""
    rng = np.random.default_rng(1000 + seed)
    for _ in range(40):
        x = _fuzz_input(rng)
        dt = [np.int64, np.uint64, np.int32, np.uint32][int(rng.integers(0, 4))]
        if dt == np.uint64:
            x = x.view(np.uint64)
        elif dt in (np.int32, np.uint32):
            x = x.astype(dt)  # wraps: a different but valid column
        want = np.sort(x)
        t = to_dev(x)
        tel = SortTelemetry()
        cafs.cafs_sort(t, telemetry=tel)
        assert np.array_equal(t.cpu().numpy(), want), (x.dtype, x.shape)
        if x.shape[0] > 1:
            xo = x.astype(np.int64) if x.dtype in (np.int32, np.uint32) else x.copy()
            ot = orc.cafs_sort(xo)
            assert tel.route.value == ot.route, (x.dtype, x.shape, tel.route, ot.route)
            if ot.decision.estimate is not None and tel.decision.estimate is not None:
                e, oe = tel.decision.estimate, ot.decision.estimate
                assert (e.k_hat, e.u, e.f1, e.f2) == (oe.k_hat, oe.u, oe.f1, oe.f2)


def test_main_route_beyond_two_million_keys():
    """2.3 M distinct keys on the main route (a skewed column the dispatcher
    sends to MAIN): the 16 Mi-key device table counts them without the guard,
    and the exact telemetry still matches the oracle's bucket table."""
    rng = np.random.default_rng(5)
    K = 6_000_000
    pal = ogen.mix_outputs(11, K).view(np.int64)
    x = pal[np.minimum(rng.zipf(1.05, 40_000_000), K) - 1]
    ot = orc.cafs_sort(x.copy())
    t = to_dev(x)
    tel = SortTelemetry()
    cafs.cafs_sort(t, telemetry=tel, exact_telemetry=True)
    assert np.array_equal(t.cpu().numpy(), np.sort(x))
    assert tel.route is Route.MAIN and ot.route == "main"
    assert not tel.device_guard_fired and tel.pairs == np.unique(x).shape[0] > 2_200_000
    assert (tel.spill_len, tel.guard_fired, tel.updates) == (ot.spill_len, ot.guard_fired, ot.updates)
    assert (tel.table.hits, tel.table.claims, tel.table.spill_pushes) == (ot.hits, ot.claims,
                                                                          ot.spill_pushes)


def test_parity_checks_catch_an_injected_fault():
    """Negative control for the GPU checks (the reference's fault_point pattern,
    selftest.py:84-105): a device result with one flipped bit, or a golden
    record with a wrong route / estimate / spill count, must fail run_case."""
    rec = next(r for r in load_json("special_cases.json")
               if r["route"] == "main" and "table_buckets" in r)
    x = special_input(rec["name"])
    run_case(x, rec)  # clean
    t = to_dev(x)
    cafs.cafs_sort(t)
    t[t.shape[0] // 2] ^= 1
    assert sha(t) != rec["sha256"]
    for field, bad in (("route", "tiny_count"), ("u", rec["u"] + 1),
                       ("spill_len", rec["spill_len"] + 1)):
        with pytest.raises(AssertionError):
            run_case(x, dict(rec, **{field: bad}))


def _checksums(t):
    """Permutation-invariant fingerprints of an int64 column (sum and sum of
    squares mod 2^64), computed on the device in 2^28-row slices."""
    s = q = 0
    for i in range(0, t.shape[0], 1 << 28):
        c = t[i:i + (1 << 28)]
        s = (s + int(c.sum().item())) % (1 << 64)
        q = (q + int((c * c).sum().item())) % (1 << 64)
    return s, q


@pytest.mark.parametrize("route", ["main", "fallback"])
def test_beyond_two_billion_rows(route):
    """Maximum-size edge: 2^31 + 12345 rows (past every 32-bit row index), on the
    dense-window main route and on the fallback route (LSD onesweep: more rows
    than the MSD buckets take); sortedness plus permutation-invariant checksums
    (and the per-code histogram for the codes) at full size."""
    n = (1 << 31) + 12345
    lib = cafs.sorter._lib.load()
    st = torch.cuda.current_stream().cuda_stream
    x = torch.empty(n, dtype=torch.int64, device="cuda")
    if route == "main":  # dictionary codes 0..999, uniform
        assert lib.cafs_gen_draw(x.data_ptr(), n, 0, 77, 0, 1000, 0, st) == 0
        hist_in = torch.bincount(x, minlength=1000)
    else:  # random 64-bit keys
        assert lib.cafs_gen_mix(x.data_ptr(), n, 78, 0, st) == 0
    sums = _checksums(x)
    tel = SortTelemetry()
    cafs.cafs_sort(x, telemetry=tel)
    torch.cuda.synchronize()
    assert tel.route.value == ("main" if route == "main" else "fallback_high_entropy")
    assert bool((x[1:] >= x[:-1]).all())
    assert _checksums(x) == sums
    if route == "main":
        assert torch.equal(torch.bincount(x, minlength=1000), hist_in)
    del x
    torch.cuda.empty_cache()
