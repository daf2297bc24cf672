"""The sharded sort with the REAL device kernels (DeviceOps through the C ABI).

Two ranks share the one GPU of the test box; their collectives run under gloo
through host memory, so no kernel ever waits on another rank (the multi-rank
NCCL path differs only in where the collective buffers live).  The
concatenated shards must equal np.sort of the whole column and every rank must
take the reference's decision.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from conftest import load_json  # noqa: E402
from oracle import cafs_oracle as orc  # noqa: E402
from oracle import gen as ogen  # noqa: E402

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)


def _cases():
    main = ogen.gen_input(400_000, 300, 3).view(np.int64)
    tiny = ogen.gen_input(600_000, 6, 4).view(np.int64)
    fail = tiny.copy()
    fail[1] = 12345
    return {
        "main": (main, [150_001]),
        "cfg3_slice": (ogen.CONFIGS["cfg3"].generate(1_000_000), [400_000]),
        "cfg4_slice": (ogen.CONFIGS["cfg4"].generate(2_000_000), [1_000_000]),
        "tiny": (tiny, [300_000]),
        "tiny_fail": (fail, [3]),
        "distinct": (ogen.distinct_values(200_000, 9).view(np.int64), [90_000]),
        "ramp": (np.arange(-100_000, 100_000, dtype=np.int64), [100_000]),
        "small": (ogen.gen_input(1500, 50, 5).view(np.int64), [700]),
        "empty_shard": (main[:50_000], [50_000]),
        "distinct_uneven": (ogen.distinct_values(300_000, 10).view(np.int64), [1_001]),
        "skew": (_skew(), [100_001]),
        "guard": (_guard_input(), [10_000_000]),
        "int32": (np.minimum(np.random.default_rng(8).zipf(1.3, 700_000), 3000).astype(np.int32)
                  - 1500, [250_000]),
    }


def _skew():
    x = ogen.distinct_values(200_000, 11).view(np.int64).copy()
    x[::2] = 123456789  # one bucket straddles both output slices
    return x


def _guard_input():
    """More distinct keys than the device table holds (16 Mi), under a low estimate."""
    n = 20_000_000
    x = ogen.mix_outputs(77, n).view(np.int64).copy()
    x[::n // 1024][:1024] = np.arange(1024, dtype=np.int64) % 100
    return x


def _worker(rank, world, port, name, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_25040_b200 import SortTelemetry
        from paper_2605_25040_b200.sharded import cafs_sort_sharded

        x, cuts = _cases()[name]
        b = [0] + cuts + [x.shape[0]]
        local = torch.from_numpy(x[b[rank]:b[rank + 1]].copy()).cuda()
        tel = SortTelemetry()
        cafs_sort_sharded(local, telemetry=tel)
        torch.cuda.synchronize()
        assert tel.kernels_launched > 0  # the device kernels ran (C ABI accounting)
        # columns the stream-ordered path can finish on device must not fall back
        if name in ("main", "cfg4_slice", "tiny", "ramp", "empty_shard"):
            assert tel.sharded_path == "streamed", (name, tel.sharded_path)
        e = tel.decision.estimate
        q.put((rank, local.cpu().numpy(), tel.route.value, tel.tiny_count_failed,
               None if e is None else (e.k_hat, e.u, e.f1, e.f2, e.saturated), tel.guard_fired))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name", list(_cases()))
def test_sharded_two_ranks_device_kernels(name):
    import torch.multiprocessing as mp
    x, _ = _cases()[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    got = np.concatenate([r[1] for r in res])
    assert np.array_equal(got, np.sort(x))
    otel = orc.cafs_sort(x.astype(np.int64) if x.dtype == np.int32 else x.copy())
    for r in res:
        assert r[2] == otel.route and r[3] == otel.tiny_count_failed
        assert r[5] == (name == "guard")  # device guard: the distributed fallback ran
        if r[4] is not None:
            oe = otel.decision.estimate
            assert r[4] == (oe.k_hat, oe.u, oe.f1, oe.f2, oe.saturated)
