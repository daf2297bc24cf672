"""GPU parity of the partitioned main count (csrc/hashpart.cu).

Columns of at least 2^20 rows whose sample shows no dense key window are
counted by per-SM tables plus key-range partitions reduced on chip (no global
hash table, no pair sort).  That path runs when no reference-exact telemetry
is requested (the exact statistics need the unsorted input, which the
partitioned count overwrites with its spill), so these tests call the API
without telemetry or with ``exact_telemetry=False``, check
``telemetry.count_path``, and compare the sorted bytes with ``np.sort`` and the
dispatch tuple with the reference's goldens.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import load_json  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2605_25040_b200 as cafs  # noqa: E402
from paper_2605_25040_b200 import datagen  # noqa: E402


def sort_partitioned(x: torch.Tensor, expect_path="partitioned"):
    y = x.clone()
    tel = cafs.SortTelemetry()
    cafs.cafs_sort(y, telemetry=tel, exact_telemetry=False)
    torch.cuda.synchronize()
    if expect_path is not None:
        assert tel.count_path == expect_path, (tel.count_path, tel.route)
    return y, tel


def check_sorted_equal(y: torch.Tensor, x: torch.Tensor):
    want = np.sort(x.cpu().numpy(), kind="stable")
    got = y.cpu().numpy()
    assert got.dtype == want.dtype
    assert np.array_equal(got, want)


def test_cfg3_through_the_partitioned_count():
    """BASELINE config 3 (Zipf 1.1 over 130k random keys): the reference's
    sorted bytes and dispatch tuple (tests/golden/config_cases.json)."""
    import hashlib

    rec = next(r for r in load_json("config_cases.json") if r["name"] == "cfg3")
    x = datagen.generate("cfg3")
    y, tel = sort_partitioned(x)
    assert hashlib.sha256(y.cpu().numpy().tobytes()).hexdigest() == rec["sha256"]
    e = tel.decision.estimate
    assert tel.route.value == rec["route"]
    assert (e.k_hat, e.u, e.f1, e.f2, e.saturated) == (
        rec["k_hat"], rec["u"], rec["f1"], rec["f2"], rec["saturated"])
    assert tel.pairs == 129998 and tel.counted_total == x.numel()
    assert 0 < tel.global_updates < x.numel()  # some keys spilled past the SM tables


@pytest.mark.parametrize("k,dist,s", [(2, "uniform", 0), (1000, "uniform", 0),
                                      (4096, "uniform", 0), (50_000, "zipf", 0.8),
                                      (200_000, "uniform", 0), (120_000, "zipf", 1.4)])
def test_key_families(k, dist, s):
    cfg = datagen.Config("t", 3_000_000, k, dist, s=s, seed=1000 + k)
    x = datagen.generate(cfg)
    y, tel = sort_partitioned(x, expect_path=None)
    check_sorted_equal(y, x)
    if tel.route.value == "main":
        assert tel.count_path == "partitioned"
        assert tel.pairs == np.unique(x.cpu().numpy()).size


@pytest.mark.parametrize("dtype", [np.int64, np.uint64, np.int32, np.uint32])
def test_dtypes(dtype):
    """numpy columns of every supported dtype (the host entry points)."""
    cfg = datagen.Config("t", 2_500_000, 30_000, "zipf", s=1.05, seed=77)
    x64 = datagen.generate(cfg).cpu().numpy()
    x = (x64 & 0xFFFFFFFF).astype(dtype) if np.dtype(dtype).itemsize == 4 else x64.view(dtype)
    y = x.copy()
    tel = cafs.SortTelemetry()
    cafs.cafs_sort(y, telemetry=tel, exact_telemetry=False)
    assert tel.count_path == "partitioned"
    assert np.array_equal(y, np.sort(x))


@pytest.mark.parametrize("lo,hi", [(1, 0), (3, 1), (2, 5), (0, 3)])
def test_unaligned_views(lo, hi):
    """Head and tail keys outside the 16-byte body (CTA 0 inserts them)."""
    cfg = datagen.Config("t", 2_000_011, 20_000, "zipf", s=1.0, seed=12)
    base = datagen.generate(cfg)
    x = base[lo:base.numel() - hi]
    y = x.clone()
    tel = cafs.SortTelemetry()
    cafs.cafs_sort(y, telemetry=tel, exact_telemetry=False)
    assert tel.count_path == "partitioned"
    check_sorted_equal(y, x)
    # the rows around the view are untouched
    assert torch.equal(base[:lo], datagen.generate(cfg)[:lo])


def test_extreme_keys_and_sentinel():
    """INT64_MAX maps to the all-ones key (the old path's empty marker) and
    INT64_MIN to zero; both are ordinary keys here."""
    cfg = datagen.Config("t", 2_000_000, 20_000, "zipf", s=1.0, seed=14)
    x = datagen.generate(cfg)
    x[::7] = 2**63 - 1
    x[::11] = -2**63
    x[5::13] = -1
    y, tel = sort_partitioned(x)
    check_sorted_equal(y, x)


def test_heavy_spill():
    """Uniform keys far beyond the per-SM tables: most rows spill, every
    partition still fits."""
    cfg = datagen.Config("t", 4_000_000, 300_000, "uniform", seed=9)
    x = datagen.generate(cfg)
    y, tel = sort_partitioned(x)
    check_sorted_equal(y, x)
    assert tel.global_updates > x.numel() // 3


def test_partition_overflow_recovers():
    """Half one key, half unique keys: the sample's Chao1 (~1.5e5) admits the
    partitioned count, but the partitions overflow; the column is rebuilt from
    the cells and the spill and sorted by the fallback."""
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    n = 4_000_000
    x = torch.randint(-2**62, 2**62, (n,), device="cuda", generator=g)
    x[torch.rand(n, device="cuda", generator=g) < 0.5] = 12345
    y, tel = sort_partitioned(x)
    assert tel.guard_fired
    check_sorted_equal(y, x)


def test_repeat_calls_and_graph_replay():
    """The same buffer sorted repeatedly (captured, then replayed) and a
    second buffer of another size in between."""
    cfg = datagen.Config("t", 2_000_000, 5_000, "uniform", seed=21)
    x = datagen.generate(cfg)
    x2 = datagen.generate(datagen.Config("t2", 3_000_001, 40_000, "zipf", s=0.9, seed=22))
    want = np.sort(x.cpu().numpy())
    want2 = np.sort(x2.cpu().numpy())
    y, y2 = x.clone(), x2.clone()
    for _ in range(4):
        y.copy_(x)
        cafs.cafs_sort(y)
        y2.copy_(x2)
        cafs.cafs_sort(y2)
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), want)
        assert np.array_equal(y2.cpu().numpy(), want2)


def test_exact_telemetry_keeps_the_table_path():
    """Reference-exact telemetry needs the unsorted input after the count:
    those calls count on the global-table path and match the reference."""
    x = datagen.generate("cfg3")
    y = x.clone()
    tel = cafs.SortTelemetry()
    cafs.cafs_sort(y, telemetry=tel)
    assert tel.exact and tel.count_path == "table"
    rec = next(r for r in load_json("config_cases.json") if r["name"] == "cfg3")
    assert tel.spill_len == rec["spill_len"]


def test_host_numpy_column():
    """numpy input (the reference's own type) through the host entry point."""
    cfg = datagen.Config("t", 2_000_000, 9_000, "zipf", s=1.2, seed=31)
    xn = datagen.generate(cfg).cpu().numpy()
    y = xn.copy()
    cafs.cafs_sort(y)
    assert np.array_equal(y, np.sort(xn))


def test_route_changes_on_one_buffer():
    """The graph cached for a buffer holds only the kernels of the route its
    last call took; a call whose data needs another route must notice and run
    the whole pipeline.  One buffer, same length, data cycling through every
    route and count path, several times (direct, captured, replayed)."""
    n = 2_100_000
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    cols = {
        "tiny": datagen.generate(datagen.Config("t1", n, 5, "uniform", seed=41)),
        "dense": datagen.generate(datagen.Config("t2", n, 3000, "zipf", s=0.9,
                                                 palette="codes", seed=42)),
        "partitioned": datagen.generate(datagen.Config("t3", n, 20_000, "zipf", s=1.1, seed=43)),
        "fallback": torch.randint(-2**62, 2**62, (n,), device="cuda", generator=g),
        "sorted": torch.arange(n, device="cuda", dtype=torch.int64) * 3 - n,
    }
    # dictionary codes with a few keys outside the window the sample opens: a
    # pipeline cached for in-window codes holds no compaction / pair sort and
    # must be re-run with them (and the next in-window column must not see
    # leftovers in the global table)
    outl = cols["dense"].clone()
    outl[11::300_007] = 2**55 + torch.arange(outl[11::300_007].shape[0], device="cuda")
    cols["dense_outliers"] = outl
    want = {k: np.sort(v.cpu().numpy()) for k, v in cols.items()}
    buf = torch.empty(n, dtype=torch.int64, device="cuda")
    order = ["tiny", "dense", "dense", "partitioned", "partitioned", "tiny", "fallback",
             "dense", "sorted", "partitioned", "tiny", "tiny", "fallback", "dense",
             "dense", "dense_outliers", "dense", "dense", "dense_outliers", "dense_outliers",
             "dense_outliers", "dense"]
    for rep in range(2):
        for name in order:
            buf.copy_(cols[name])
            cafs.cafs_sort(buf)
            torch.cuda.synchronize()
            assert np.array_equal(buf.cpu().numpy(), want[name]), (rep, name)
