"""The row-sharded multi-GPU orchestration, run as world_size-2 gloo on CPU.

``cafs_sort_sharded`` takes its local steps from an ``ops`` object; on the GPU
that is the C ABI (``DeviceOps``).  Here a numpy restatement of those local
steps (test-only) stands in, so the host logic -- global sample positions
across shards, the all-gathered monotone test, the identical decision on every
rank, the pair-table exchange and merge, and each rank's output slice -- is
checked against the single-process oracle on CPU.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import cafs_oracle as orc
from oracle import gen as ogen

SIGN = np.uint64(1 << 63)


class NumpyOps:
    """Local pipeline steps as numpy (test double of sharded.DeviceOps)."""

    signed = True
    pair_cap = None  # set: count_pairs reports a table overflow above this many keys

    def _u(self, x):
        return x.numpy().view(np.uint64) ^ SIGN

    def is_monotone(self, x):
        return bool(orc.is_monotone(x.numpy())) if x.shape[0] > 1 else True

    def estimate(self, samples):
        vals, cnts = np.unique(self._u(samples), return_counts=True)
        u = int(vals.shape[0])
        keys = [int(v) for v in vals] if u <= 8 else []
        return u, int((cnts == 1).sum()), int((cnts == 2).sum()), u == 1024, keys

    def tiny_counts(self, x, keys):
        xu = self._u(x)
        return np.array([int((xu == np.uint64(k)).sum()) for k in keys], np.int64)

    def count_pairs(self, x, mult):
        vals, cnts = np.unique(self._u(x), return_counts=True)
        if self.pair_cap is not None and vals.shape[0] > self.pair_cap:
            return None
        return torch.from_numpy(vals.view(np.int64).copy()), torch.from_numpy(cnts.astype(np.int64))

    def merge_pairs(self, keys, counts):
        k = keys.numpy().view(np.uint64)
        vals, inv = np.unique(k, return_inverse=True)
        tot = np.zeros(vals.shape[0], np.int64)
        np.add.at(tot, inv, counts.numpy())
        return torch.from_numpy(vals.view(np.int64).copy()), torch.from_numpy(tot)

    def emit_slice(self, keys, counts, out, begin, end, total):
        full = np.repeat(keys.numpy().view(np.uint64), counts.numpy())
        assert full.shape[0] == total
        out.copy_(torch.from_numpy((full[begin:end] ^ SIGN).view(np.int64).copy()))

    def fallback_sort(self, x):
        x.copy_(torch.from_numpy(np.sort(x.numpy())))

    def key_span(self, x):
        u = self._u(x)
        if u.shape[0] == 0:
            return (1 << 64) - 1, 0
        return int(u.min()), int(u.max())

    def partition(self, x, g_min, g_max):
        from paper_2605_25040_b200.sharded import PARTITION_BUCKETS, msd_shift
        sh = np.uint64(msd_shift(g_min, g_max))
        d = (((self._u(x) - np.uint64(g_min)) >> sh) & np.uint64(4095)).astype(np.int64)
        order = np.argsort(d, kind="stable")
        return (torch.from_numpy(x.numpy()[order].copy()),
                np.bincount(d, minlength=PARTITION_BUCKETS).astype(np.int64))

    def keys_tensor(self, keys, counts):
        return (torch.from_numpy(np.array(keys, np.uint64).view(np.int64)),
                torch.from_numpy(np.asarray(counts, np.int64)))


def _cases():
    rng = np.random.default_rng(7)
    main = ogen.gen_input(200_000, 200, 3).view(np.int64)
    tiny = ogen.gen_input(300_000, 4, 4).view(np.int64)
    fail = tiny.copy()
    fail[1] = 12345  # never sampled: tiny count misses -> MAIN
    distinct = ogen.distinct_values(100_000, 9).view(np.int64)
    ramp = np.arange(-50_000, 50_000, dtype=np.int64)
    small = ogen.gen_input(1000, 50, 5).view(np.int64)
    zipf = ogen.CONFIGS["cfg3"].generate(400_000)
    skew = ogen.distinct_values(100_000, 11).view(np.int64).copy()
    skew[::2] = 123456789  # one huge bucket across both slices, still high-entropy
    return {"main": (main, [120_003]), "tiny": (tiny, [150_000]), "tiny_fail": (fail, [7]),
            "distinct": (distinct, [60_000]), "ramp": (ramp, [50_000]),
            "small": (small, [400]), "zipf": (zipf, [200_000]),
            "empty_shard": (main[:100_000], [100_000]),
            "uneven": (rng.permutation(main), [33]),
            "distinct_uneven": (distinct, [999]), "distinct_empty": (distinct, [0]),
            "skew": (skew, [50_001]), "guard": (main, [90_000])}


def _worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2605_25040_b200 import SortTelemetry
        from paper_2605_25040_b200.sharded import cafs_sort_sharded

        x, cuts = _cases()[name]
        bounds = [0] + cuts + [x.shape[0]]
        local = torch.from_numpy(x[bounds[rank]:bounds[rank + 1]].copy())
        tel = SortTelemetry()
        ops = NumpyOps()
        if name == "guard":
            ops.pair_cap = 100  # the device table "overflows": guard -> distributed fallback
        cafs_sort_sharded(local, ops=ops, telemetry=tel)
        e = tel.decision.estimate
        q.put((rank, local.numpy(), tel.route.value, tel.tiny_count_failed, tel.guard_fired,
               None if e is None else (e.k_hat, e.u, e.f1, e.f2, e.saturated)))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name", list(_cases()))
def test_sharded_world2_matches_single_process_oracle(name):
    x, _ = _cases()[name]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    got = np.concatenate([r[1] for r in res])
    assert np.array_equal(got, np.sort(x))
    # every rank took the decision the single-process reference takes
    y = x.copy()
    otel = orc.cafs_sort(y) if x.shape[0] > 1 else None
    for r in res:
        assert r[2] == otel.route
        assert r[3] == otel.tiny_count_failed
        assert r[4] == (name == "guard")
        if r[5] is not None:
            oe = otel.decision.estimate
            assert r[5] == (oe.k_hat, oe.u, oe.f1, oe.f2, oe.saturated)
