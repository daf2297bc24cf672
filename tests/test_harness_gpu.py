"""The reference harness's run_point contract (cafs/bench.py:102-136) driven
against the B200 sort through a registry: every algorithm sorts a fresh copy
of gen_input(GenSpec(n, k, seed_base)) per replicate and must equal np.sort.
The reference package is not available on the GPU box, so the loop and the
generator are restated here (oracle/gen.gen_input is pinned to the reference's
own generator in tests/test_oracle_golden.py)."""

import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import gen as ogen  # noqa: E402
from paper_2605_25040_b200 import harness  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def run_point(n, k, algos, reps=2, seed_base=42, registry=None):
    data = ogen.gen_input(n, k, seed_base)
    want = np.sort(data)
    rows = []
    for name in algos:
        fn = registry[name]
        best, correct = float("inf"), True
        for _ in range(reps):
            buf = data.copy()
            t0 = time.perf_counter()
            fn(buf)
            best = min(best, (time.perf_counter() - t0) * 1e3)
            correct &= bool(np.array_equal(buf, want))
        rows.append((name, n, k, best, correct))
    return rows


@pytest.mark.parametrize("n,k", [(1_000, 2), (50_000, 7), (1_000_000, 200), (2_000_000, 130_000),
                                 (3_000_000, 2_500_000), (10_000_000, 8)])
def test_run_point_with_b200_registry(n, k):
    reg = harness.register({"stdsort": lambda x: x.sort(kind="quicksort")})
    rows = run_point(n, k, ["stdsort", harness.NAME], registry=reg)
    assert [r[0] for r in rows] == ["stdsort", "cafs_b200"]
    assert all(r[4] for r in rows), rows
    # the registry callable sorts numpy views in place, like the reference's
    x = ogen.gen_input(n, k, 7).view(np.int64)
    y = x.copy()
    reg[harness.NAME](y)
    assert np.array_equal(y, np.sort(x))
