"""Launch-mode parity: the same columns sorted with programmatic dependent
launch off / on for every kernel, with and without CUDA-graph replay, and the
two-phase estimate kernel's self-resetting arrival counter exercised by
interleaved calls of different shapes (estimate.cu, common.cuh EstScratch).

Each mode runs in a fresh process because CAFS_PDL / CAFS_GRAPHS are read once.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import hashlib, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_2605_25040_b200 as cafs
from oracle import cafs_oracle as orc
rng = np.random.default_rng(11)
cols = {
    "tiny": rng.choice(rng.integers(-2**62, 2**62, 5), 300_000),
    "dense_outliers": np.where(rng.random(400_000) < 0.01, rng.integers(-2**62, 2**62, 400_000),
                               rng.integers(0, 3000, 400_000)),
    "hash": rng.choice(rng.integers(-2**62, 2**62, 20_000), 600_000),
    "big_hash": rng.choice(rng.integers(-2**62, 2**62, 50_000), 5_000_000),
    "fallback": rng.integers(-2**62, 2**62, 200_000),
    "small_n": rng.integers(-9, 9, 1500),
    "sorted": np.arange(100_000, dtype=np.int64),
}
bad = []
for name, x in cols.items():
    x = x.astype(np.int64)
    want = np.sort(x)
    route = orc.cafs_sort(x.copy()).route
    t = torch.empty(x.shape[0], dtype=torch.int64, device="cuda")
    for rep in range(3):  # direct, capture, replay
        t.copy_(torch.from_numpy(x))
        tel = cafs.SortTelemetry()
        cafs.cafs_sort(t, telemetry=tel)
        torch.cuda.synchronize()
        if not np.array_equal(t.cpu().numpy(), want) or tel.route.value != route:
            bad.append((name, rep, tel.route.value, route))
print("BAD", bad)
sys.exit(1 if bad else 0)
"""


@pytest.mark.parametrize("env", [{"CAFS_PDL": "0"}, {"CAFS_PDL": "0x1ff"},
                                 {"CAFS_PDL": "0", "CAFS_GRAPHS": "0"},
                                 {"CAFS_GRAPHS": "0"}])
def test_launch_modes_sort_identically(env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", _CHILD, ROOT], env=e, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_estimate_interleaved_shapes_against_oracle():
    """Sorts and stage-API estimates of different sizes back to back on one
    context: every call's dispatch must equal the oracle's (a stale arrival
    count in the two-phase estimate would elect the wrong CTA or none)."""
    import paper_2605_25040_b200 as cafs
    from oracle import cafs_oracle as orc

    rng = np.random.default_rng(5)
    sizes = [2048, 16_384, 16_385, 16_386, 70_000, 1_000_003, 3000, 5_000_000]
    for i in range(3):
        for n in sizes:
            k = int(rng.integers(2, 5000))
            x = rng.choice(rng.integers(-2**62, 2**62, k), n).astype(np.int64)
            if i == 1:
                x[: min(n, 16_385)] = np.sort(x[: min(n, 16_385)])  # sorted prefix
            otel = orc.cafs_sort(x.copy())
            t = torch.from_numpy(x).cuda()
            d = cafs.dispatch(t)
            assert d.route.value == otel.route, (n, d.route, otel.route)
            tel = cafs.SortTelemetry()
            cafs.cafs_sort(t, telemetry=tel)
            torch.cuda.synchronize()
            assert tel.route.value == otel.route
            e, oe = tel.decision.estimate, otel.decision.estimate
            if oe is not None:
                assert (e.k_hat, e.u, e.f1, e.f2) == (oe.k_hat, oe.u, oe.f1, oe.f2)
            assert np.array_equal(t.cpu().numpy(), np.sort(x))


def test_concurrent_threads_on_two_streams_share_one_context():
    """Two host threads, each sorting on its own CUDA stream through the one
    per-device context: the context serialises the calls (host lock plus a
    wait for the previous stream on a switch), so both threads get exact results."""
    import threading

    import paper_2605_25040_b200 as cafs

    rng = np.random.default_rng(9)
    cols = [rng.choice(rng.integers(-2**62, 2**62, k), n).astype(np.int64)
            for k, n in ((5, 700_000), (3000, 900_000), (60_000, 1_200_000), (4, 500_000))]
    want = [np.sort(c) for c in cols]
    errors = []

    def worker(idx):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(6):
                    c = idx * 2 + rep % 2
                    t = torch.from_numpy(cols[c]).cuda(non_blocking=False)
                    cafs.cafs_sort(t)
                    s.synchronize()
                    if not np.array_equal(t.cpu().numpy(), want[c]):
                        errors.append((idx, rep))
        except Exception as e:  # pragma: no cover
            errors.append(repr(e))

    ths = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors


def test_large_pair_sort_bucket_overflow_recovers():
    """> 8192 pairs whose keys cluster in one MSD bucket of the pair span: the
    unchecked bucket sort flags the overflow and the call re-sorts the pairs
    by LSD and re-emits (abi.cu sort_pairs_large_unchecked); the output and the
    route still match the oracle."""
    import paper_2605_25040_b200 as cafs
    from oracle import cafs_oracle as orc

    rng = np.random.default_rng(21)
    hot = rng.integers(-2**62, 2**62, 300)
    n_hot, n_cold = 2_700_000, 300_000
    x = np.concatenate([rng.choice(hot, n_hot), rng.integers(0, 60_000, n_cold)]).astype(np.int64)
    rng.shuffle(x)
    otel = orc.cafs_sort(x.copy())
    assert otel.route == "main"
    for _ in range(2):  # direct and graph-replayed pipelines
        t = torch.from_numpy(x).cuda()
        tel = cafs.SortTelemetry()
        cafs.cafs_sort(t, telemetry=tel)
        torch.cuda.synchronize()
        assert tel.route.value == "main" and tel.pairs > 8192
        assert np.array_equal(t.cpu().numpy(), np.sort(x))
