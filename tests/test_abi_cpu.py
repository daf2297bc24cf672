"""The C ABI library without a GPU: it loads, exports every declared symbol, its
struct layouts match the ctypes mirror, and device calls fail cleanly."""

import ctypes
import os
import re
import subprocess

import pytest

from paper_2605_25040_b200 import _lib
from paper_2605_25040_b200 import build as pkg_build

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
HEADER = os.path.join(ROOT, "include", "cafs_b200.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        pkg_build.build()
    return _lib.load()


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|uint64_t|const char\*)\s+(cafs_\w+)\(", text, re.M)))


def test_header_declares_the_abi():
    syms = declared_symbols()
    assert "cafs_sort_i64" in syms and "cafs_emit_i64" in syms
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table and header disagree"


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (cafs_\w+)$", out, re.M))
    missing = set(declared_symbols()) - exported
    assert not missing, f"not exported: {missing}"
    for name in declared_symbols():
        assert getattr(lib, name) is not None


def test_abi_version_and_status_strings(lib):
    assert lib.cafs_abi_version() == 2
    assert lib.cafs_status_string(0) == b"ok"
    assert b"invalid" in lib.cafs_status_string(-1)


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include "cafs_b200.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                   "int main(){printf(\"%zu %zu %zu %zu %zu\\n\", sizeof(cafs_estimate_t),"
                   " sizeof(cafs_decision_t), sizeof(cafs_telemetry_t),"
                   " offsetof(cafs_telemetry_t, stage_ms), offsetof(cafs_telemetry_t,"
                   " kernels_launched));return 0;}\n")
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_lib.Estimate), ctypes.sizeof(_lib.Decision),
            ctypes.sizeof(_lib.Telemetry), _lib.Telemetry.stage_ms.offset,
            _lib.Telemetry.kernels_launched.offset]
    assert got == want


def test_device_calls_fail_cleanly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    rc = lib.cafs_ctx_create(0, ctypes.byref(h))
    assert rc != 0 and not h.value
    assert lib.cafs_sort_i64(None, None, 0, 1, 1, 0, None, None) == _lib.EINVAL


def test_fallback_exchange_plan_sorts_a_sharded_column(lib):
    """cafs_shard_fallback_plan (the native distributed fallback's host step)
    against sharded.bucket_ranges and an end-to-end numpy simulation of the
    exchange: every rank's received buckets, sorted, hold its rows of the sorted
    column at the planned offset.  Uneven and empty shards, skewed buckets."""
    import ctypes

    import numpy as np

    from paper_2605_25040_b200.sharded import bucket_ranges, msd_shift

    B = 4096
    rng = np.random.default_rng(5)
    cases = [
        [rng.integers(0, 2**63, n, dtype=np.uint64) for n in (5000, 7000, 1, 9000)],
        [rng.integers(0, 2**63, n, dtype=np.uint64) for n in (4000, 0, 6000)],          # empty shard
        [np.full(3000, 7, np.uint64), rng.integers(0, 50, 2000).astype(np.uint64)],     # one bucket
        [rng.integers(0, 2**63, 3000, dtype=np.uint64)],                                 # one rank
        [np.concatenate([np.full(4000, 2**62, np.uint64),
                         rng.integers(0, 2**63, 100, dtype=np.uint64)]) for _ in range(8)],  # straddling
    ]
    for shards in cases:
        W = len(shards)
        allk = np.concatenate(shards)
        g_min, g_max = int(allk.min()), int(allk.max())
        shift = msd_shift(g_min, g_max)
        parts, counts = [], np.zeros((W, B), np.uint32)
        for r, x in enumerate(shards):
            d = ((x - np.uint64(g_min)) >> np.uint64(shift)).astype(np.int64)
            order = np.argsort(d, kind="stable")
            parts.append(x[order])
            counts[r] = np.bincount(d, minlength=B)
        sizes = [int(x.shape[0]) for x in shards]
        ranges = bucket_ranges(counts.sum(0).astype(np.int64), sizes)
        want = np.sort(allk)
        plans = []
        for r in range(W):
            sa, sn, rn = (np.zeros(W, np.uint64) for _ in range(3))
            start = ctypes.c_uint64(0)
            rc = lib.cafs_shard_fallback_plan(W, r, counts.ctypes.data, sa.ctypes.data,
                                              sn.ctypes.data, rn.ctypes.data, ctypes.byref(start))
            assert rc == 0
            plans.append((sa, sn, rn, int(start.value)))
            L = np.concatenate([[0], np.cumsum(counts[r], dtype=np.int64)])
            for d, (lo, hi) in enumerate(ranges):  # the Python host path's splits
                assert int(sn[d]) == int(L[hi] - L[lo])
                if sn[d]:
                    assert int(sa[d]) == int(L[lo])
        off = 0
        for d in range(W):
            for s_ in range(W):  # what s sends to d is what d expects from s
                assert int(plans[s_][1][d]) == int(plans[d][2][s_])
            recv = np.concatenate([parts[s_][int(plans[s_][0][d]):int(plans[s_][0][d] + plans[s_][1][d])]
                                   for s_ in range(W)])
            recv.sort()
            st = plans[d][3]
            assert np.array_equal(recv[st:st + sizes[d]], want[off:off + sizes[d]])
            off += sizes[d]
    bad = np.zeros(B, np.uint32)
    assert lib.cafs_shard_fallback_plan(0, 0, bad.ctypes.data, None, None, None, None) != 0
