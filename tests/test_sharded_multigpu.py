"""The native multi-GPU sort across real NCCL ranks: world = min(8, GPUs).

One process per GPU (torchrun, NCCL over NVLink); every rank holds a
contiguous row shard of the same column, calls ``cafs_sort_sharded`` and must
end up holding exactly its rows [off_r, off_r + n_r) of ``np.sort`` of the
whole column -- bit-exact -- with the route the oracle (the reference
restated) takes on the whole column.  Columns: cfg4-style dictionary codes,
a tiny column, random keys with more than 8192 distinct values (the pair
exchange continuation), a skewed column that trips the device guard, a
high-entropy column (the distributed fallback) and an already sorted one.
Skipped when fewer than two GPUs are visible (this build's pool gives one GPU
per call; the same code path runs at one NCCL rank in test_sharded_nccl.py and
as two gloo ranks in test_sharded_gpu.py).
"""

import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available() or torch.cuda.device_count() < 2:  # pragma: no cover
    pytest.skip("needs at least two CUDA devices", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import os, sys
import numpy as np, torch, torch.distributed as dist
sys.path.insert(0, sys.argv[1])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
local = int(os.environ.get("LOCAL_RANK", rank))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
import paper_2605_25040_b200 as cafs
from paper_2605_25040_b200.sharded import cafs_sort_sharded
from oracle import cafs_oracle as orc
from oracle import gen as ogen
rng = np.random.default_rng(11)
codes = ogen.Config("c", 3_000_000, 4096, "zipf", s=0.8, palette="codes", seed=4).generate()
skew = rng.integers(-2**62, 2**62, 5_000_000)
skew[: 3_000_000] = rng.integers(0, 3, 3_000_000)
outl = codes.copy()
outl[7::600_000] = 2**50 + np.arange(outl[7::600_000].shape[0])  # keys outside the dense window
cols = {
    "codes": codes,
    "codes_outliers": outl,  # on one or two ranks only: every rank must re-run alike
    "tiny": rng.choice(rng.integers(-2**62, 2**62, 6), 1_000_003),
    "many_pairs": rng.choice(rng.integers(-2**62, 2**62, 50_000), 3_000_000),
    "skew_guard": rng.permutation(skew),
    # main route, more distinct keys than the device merge takes: exchanged and
    # sorted inside the library like a fallback column
    "main_too_many_pairs": rng.permutation(np.concatenate([
        rng.choice(rng.integers(-2**62, 2**62, 100), 4_000_000),
        rng.integers(-2**62, 2**62, 1_500_000)[rng.integers(0, 1_500_000, 4_000_000)]])),
    "fallback": rng.integers(-2**62, 2**62, 2_000_000),
    "sorted": np.arange(-100_000, 100_001, dtype=np.int64),
}
bad = []
for name, x in cols.items():
    x = x.astype(np.int64)
    want = np.sort(x)
    route = orc.cafs_sort(x.copy()).route
    n = x.shape[0]
    per = n // world
    lo = rank * per
    hi = n if rank == world - 1 else lo + per
    t = torch.from_numpy(x[lo:hi].copy()).cuda()
    # direct, captured, replayed with every route class's kernels, then with the
    # predicted class's only (dictionary codes: the all-reduce of the window counts)
    for rep in range(6):
        t.copy_(torch.from_numpy(x[lo:hi]))
        tel = cafs.SortTelemetry()
        cafs_sort_sharded(t, telemetry=tel)
        torch.cuda.synchronize()
        if not np.array_equal(t.cpu().numpy(), want[lo:hi]) or tel.route.value != route:
            bad.append((name, rep, tel.route.value, route, tel.sharded_path))
ok = torch.tensor([0 if bad else 1], device="cuda")
dist.all_reduce(ok, op=dist.ReduceOp.MIN)
if bad:
    print("RANK", rank, "FAILED", bad, flush=True)
dist.destroy_process_group()
sys.exit(0 if ok.item() == 1 else 1)
"""


def test_native_sharded_sort_on_all_gpus(tmp_path):
    world = min(8, torch.cuda.device_count())
    child = tmp_path / "child.py"
    child.write_text(_CHILD)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), str(child), ROOT]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
