"""ctypes binding of the C oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Mirrors the reference's observable results for one ``cafs_sort`` call
(``/root/reference/pkg/src/cafs/sorter.py:335-386``): the sorted array, the
dispatch decision (route, k_hat, u, f1, f2, saturated, tiny keys) and the
telemetry counters (spill_len, guard_fired, counted_total, updates, ...).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libcafs_oracle.so")

HASH_MULT = 0x9E3779B97F4A7C15
ROUTES = ("already_sorted", "fallback_small_n", "tiny_count", "fallback_high_entropy", "main")


class _Estimate(ctypes.Structure):
    _fields_ = [("k_hat", ctypes.c_double), ("u", ctypes.c_int64), ("f1", ctypes.c_int64),
                ("f2", ctypes.c_int64), ("saturated", ctypes.c_int32), ("nkeys", ctypes.c_int32),
                ("keys", ctypes.c_uint64 * 8)]


class _Decision(ctypes.Structure):
    _fields_ = [("route", ctypes.c_int32), ("has_estimate", ctypes.c_int32), ("est", _Estimate)]


class _Telemetry(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("decision", _Decision), ("spill_len", ctypes.c_uint64),
                ("guard_fired", ctypes.c_int32), ("tiny_count_failed", ctypes.c_int32),
                ("counted_total", ctypes.c_uint64), ("updates", ctypes.c_uint64),
                ("hits", ctypes.c_uint64), ("claims", ctypes.c_uint64),
                ("spill_pushes", ctypes.c_uint64), ("table_buckets", ctypes.c_uint64),
                ("pairs", ctypes.c_uint64)]


def build() -> str:
    """Compile the oracle with its Makefile (gcc); returns the library path."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        p64 = ctypes.POINTER(ctypes.c_int64)
        L.orc_fast_hash.restype = ctypes.c_uint64
        L.orc_fast_hash.argtypes = [ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64]
        L.orc_table_size_for.restype = ctypes.c_uint64
        L.orc_table_size_for.argtypes = [ctypes.c_double, ctypes.c_uint64, ctypes.c_int]
        L.orc_chao1.restype = ctypes.c_double
        L.orc_chao1.argtypes = [ctypes.c_int64] * 3 + [ctypes.c_uint64, ctypes.c_int]
        L.orc_is_monotone.restype = ctypes.c_int
        L.orc_is_monotone.argtypes = [p64, ctypes.c_uint64, ctypes.c_int]
        L.orc_dispatch.restype = None
        L.orc_dispatch.argtypes = [p64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                   ctypes.POINTER(_Decision)]
        L.orc_sample_estimate.restype = None
        L.orc_sample_estimate.argtypes = [p64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                          ctypes.POINTER(_Estimate)]
        L.orc_tiny_counts.restype = None
        L.orc_tiny_counts.argtypes = [p64, ctypes.c_uint64, ctypes.c_int,
                                      ctypes.POINTER(ctypes.c_uint64), ctypes.c_int, p64]
        L.orc_fallback_sort.restype = None
        L.orc_fallback_sort.argtypes = [p64, ctypes.c_uint64, ctypes.c_int]
        L.orc_cafs_sort.restype = ctypes.c_int
        L.orc_cafs_sort.argtypes = [p64, ctypes.c_uint64, ctypes.c_int, ctypes.c_uint64,
                                    ctypes.POINTER(_Telemetry)]
        L.orc_gen_draw.restype = None
        L.orc_gen_draw.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, p64,
                                   ctypes.c_uint64, ctypes.POINTER(ctypes.c_double), p64]
        _lib = L
    return _lib


def _as_i64(x: np.ndarray) -> tuple[np.ndarray, int]:
    if x.dtype == np.int64:
        return x, 1
    if x.dtype == np.uint64:
        return x.view(np.int64), 0
    raise TypeError(f"oracle handles int64/uint64, got {x.dtype}")


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


@dataclass
class Estimate:
    k_hat: float
    u: int
    f1: int
    f2: int
    saturated: bool


@dataclass
class Decision:
    route: str
    estimate: Estimate | None = None
    keys: list[int] | None = None  # tiny route: ascending, unsigned domain

    def as_tuple(self):
        e = self.estimate
        if e is None:
            return (self.route,)
        return (self.route, e.k_hat, e.u, e.f1, e.f2, e.saturated)


@dataclass
class Telemetry:
    n: int
    decision: Decision
    spill_len: int = 0
    guard_fired: bool = False
    tiny_count_failed: bool = False
    counted_total: int = 0
    updates: int = 0
    hits: int = 0
    claims: int = 0
    spill_pushes: int = 0
    table_buckets: int = 0
    pairs: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def route(self) -> str:
        return self.decision.route


def _estimate(e: _Estimate) -> Estimate:
    return Estimate(float(e.k_hat), int(e.u), int(e.f1), int(e.f2), bool(e.saturated))


def _decision(d: _Decision) -> Decision:
    route = ROUTES[d.route]
    if not d.has_estimate:
        return Decision(route)
    keys = [int(d.est.keys[i]) for i in range(d.est.nkeys)] if route == "tiny_count" else None
    return Decision(route, _estimate(d.est), keys)


def fast_hash(x: int, m_log2: int, mult: int = HASH_MULT) -> int:
    return int(lib().orc_fast_hash(x, m_log2, mult))


def table_size_for(k_hat: float, n: int, cap: int = 4) -> int:
    return int(lib().orc_table_size_for(float(k_hat), n, cap))


def chao1(u, f1, f2, n, saturated) -> float:
    return float(lib().orc_chao1(u, f1, f2, n, int(saturated)))


def is_monotone(x: np.ndarray) -> bool:
    x = np.ascontiguousarray(x)
    xi, signed = _as_i64(x)
    return bool(lib().orc_is_monotone(_ptr(xi), xi.shape[0], signed))


def sample_and_estimate(x: np.ndarray, mult: int = HASH_MULT) -> Estimate:
    x = np.ascontiguousarray(x)
    xi, signed = _as_i64(x)
    e = _Estimate()
    lib().orc_sample_estimate(_ptr(xi), xi.shape[0], signed, mult, ctypes.byref(e))
    return _estimate(e)


def dispatch(x: np.ndarray, mult: int = HASH_MULT) -> Decision:
    x = np.ascontiguousarray(x)
    xi, signed = _as_i64(x)
    d = _Decision()
    lib().orc_dispatch(_ptr(xi), xi.shape[0], signed, mult, ctypes.byref(d))
    return _decision(d)


def tiny_counts(x: np.ndarray, keys) -> np.ndarray:
    x = np.ascontiguousarray(x)
    xi, signed = _as_i64(x)
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    out = np.zeros(k.shape[0], np.int64)
    lib().orc_tiny_counts(_ptr(xi), xi.shape[0], signed,
                          k.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), k.shape[0], _ptr(out))
    return out


def cafs_sort(x: np.ndarray, mult: int = HASH_MULT) -> Telemetry:
    """In-place oracle sort of a contiguous int64/uint64 array; returns telemetry."""
    if not x.flags.c_contiguous:
        raise ValueError("oracle sorts contiguous arrays")
    xi, signed = _as_i64(x)
    t = _Telemetry()
    rc = lib().orc_cafs_sort(_ptr(xi), xi.shape[0], signed, mult, ctypes.byref(t))
    if rc != 0:
        raise RuntimeError(f"oracle cafs_sort failed: {rc}")
    return Telemetry(n=int(t.n), decision=_decision(t.decision), spill_len=int(t.spill_len),
                     guard_fired=bool(t.guard_fired), tiny_count_failed=bool(t.tiny_count_failed),
                     counted_total=int(t.counted_total), updates=int(t.updates), hits=int(t.hits),
                     claims=int(t.claims), spill_pushes=int(t.spill_pushes),
                     table_buckets=int(t.table_buckets), pairs=int(t.pairs))


def fallback_sort(x: np.ndarray) -> None:
    xi, signed = _as_i64(x)
    lib().orc_fallback_sort(_ptr(xi), xi.shape[0], signed)


def generate(config, n: int | None = None, start: int = 0, threads: int | None = None) -> np.ndarray:
    """Rows [start, start+n) of a BASELINE config (oracle/gen.py Config) by the C
    generator, split over host threads (ctypes releases the GIL); bit-identical
    to ``config.generate`` (tests/test_oracle_golden.py)."""
    import threading

    n = config.n - start if n is None else n
    out = np.empty(n, np.int64)
    pal = None if config.palette == "codes" else np.ascontiguousarray(config.palette_values())
    cdf = config.cdf()
    cdf_p = None if cdf is None else cdf.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    pal_p = None if pal is None else _ptr(pal)
    T = max(1, min(threads or os.cpu_count() or 1, (n >> 16) or 1))
    share = (n + T - 1) // T

    def work(t):
        lo = t * share
        hi = min(n, lo + share)
        if hi > lo:
            lib().orc_gen_draw(config.seed, hi - lo, start + lo, pal_p, config.k, cdf_p,
                               _ptr(out[lo:hi]))

    ths = [threading.Thread(target=work, args=(t,)) for t in range(T)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    return out
