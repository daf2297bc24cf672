"""Host-side mirror of the reference's sort API, backed by libcafs_b200.so.

Same names, argument meaning and error behaviour as the reference package
(``/root/reference/pkg/src/cafs``): ``cafs_sort(x, telemetry=None,
hash_mult=None)`` sorts a 1-D integer array in place and fills a
:class:`SortTelemetry`; ``dispatch`` / ``sample_and_estimate`` / ``is_monotone``
/ ``tiny_count_sort`` / ``pair_sort`` / ``emit`` / ``fallback_sort`` expose the
pipeline stages.  Every stage runs on the B200 through the C ABI -- this module
only validates, converts and fills the Python result types.

Inputs:
* a ``torch`` CUDA tensor (int64 / uint64; int32 / uint32 are widened on
  device) is sorted in place on its device and stream;
* a ``numpy`` array or CPU tensor takes the host entry point
  (``cafs_sort_i64_host``: H2D, device pipeline, D2H) -- the drop-in for
  callers of the reference, which sorts numpy arrays.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib

SMALL_N_CUTOFF = 2048         # sorter.py:29
TINY_MAX_KEYS = 8             # sorter.py:30
PAIR_RADIX_MIN = 256          # sorter.py:31 (our pair sort has no such split; kept for API parity)
_MONO_CHUNK = 1 << 14         # sorter.py:32
SAMPLE_TARGET = 1024          # cardinality.py:26
FREQSET_SLOTS = 4096          # cardinality.py:27
HASH_MULT = 0x9E3779B97F4A7C15  # buckets.py:30
_MASK64 = (1 << 64) - 1

SUPPORTED_DTYPES = tuple(np.dtype(t) for t in (np.uint64, np.int64, np.uint32, np.int32))


class Route(Enum):  # sorter.py:44-49
    ALREADY_SORTED = "already_sorted"
    FALLBACK_SMALL_N = "fallback_small_n"
    TINY_COUNT = "tiny_count"
    FALLBACK_HIGH_ENTROPY = "fallback_high_entropy"
    MAIN = "main"


_ROUTE_BY_CODE = [Route.ALREADY_SORTED, Route.FALLBACK_SMALL_N, Route.TINY_COUNT,
                  Route.FALLBACK_HIGH_ENTROPY, Route.MAIN]


@dataclass(frozen=True)
class CardinalityEstimate:  # cardinality.py:76-82
    k_hat: float
    u: int
    f1: int
    f2: int
    saturated: bool


@dataclass
class DispatchDecision:  # sorter.py:52-57
    route: Route
    keys: np.ndarray | None = None              # TINY_COUNT: <= 8 keys, ascending
    k_hat: float | None = None                  # MAIN
    estimate: CardinalityEstimate | None = None


class TableStats:
    """The reference's TableStats (buckets.py:152-169): named update counters."""

    __slots__ = ("updates", "hits", "claims", "spill_pushes", "spill_len")

    def __init__(self, updates=0, hits=0, claims=0, spill_pushes=0, spill_len=0):
        self.updates, self.hits, self.claims = int(updates), int(hits), int(claims)
        self.spill_pushes, self.spill_len = int(spill_pushes), int(spill_len)

    def __repr__(self):
        return (f"TableStats(updates={self.updates}, hits={self.hits}, claims={self.claims}, "
                f"spill_pushes={self.spill_pushes}, spill_len={self.spill_len})")


class TableSummary:
    """``SortTelemetry.table``: a read-only view with the reference BucketTable's
    observable surface (buckets.py:172-292) -- ``n_buckets``, ``cap``,
    ``m_log2``, ``dtype``, ``hash_mult``, ``stats``, ``spill_len``,
    ``counted_total()`` -- for the table the reference would have built on the
    same input.  The device computes these exactly (telemetry.cu) without
    building the table; its slot arrays and spill buffer are not materialised
    (``keys`` / ``counts`` / ``spill`` raise)."""

    def __init__(self, n_buckets: int, cap: int, hits: int, claims: int, spill_pushes: int,
                 spill_len: int, updates: int = 0, counted_total: int = 0,
                 dtype=np.uint64, hash_mult: int = HASH_MULT):
        self.n_buckets = int(n_buckets)
        self.cap = int(cap)
        self.m_log2 = self.n_buckets.bit_length() - 1
        self.dtype = np.dtype(dtype)
        self.hash_mult = int(hash_mult)
        self.stats = TableStats(updates, hits, claims, spill_pushes, spill_len)
        self._counted = int(counted_total)

    hits = property(lambda self: self.stats.hits)
    claims = property(lambda self: self.stats.claims)
    spill_pushes = property(lambda self: self.stats.spill_pushes)
    spill_len = property(lambda self: self.stats.spill_len)

    def counted_total(self) -> int:
        """Sum of the bucket counters (excludes the spill), buckets.py:290-292."""
        return self._counted

    def _absent(self, *_):
        raise AttributeError("the device pipeline does not materialise the reference's "
                             "bucket slots or spill buffer; see stats / spill_len")

    keys = property(_absent)
    counts = property(_absent)
    spill = property(_absent)
    occupied_pairs = _absent


@dataclass
class SortTelemetry:  # sorter.py:60-81
    """Read-only view of one cafs_sort invocation.

    ``stage_ms`` keys follow the reference's count / sort_k / emit labels and
    are CUDA-event times.  ``spill_len``, ``updates``, ``guard_fired``,
    ``counted_total`` and ``table`` describe the reference's bucket table, which
    the device pipeline does not build; whenever a telemetry object is passed
    they are computed exactly on device (telemetry.cu), as the reference fills
    them (sorter.py:326-331).  ``cafs_sort(..., exact_telemetry=False)`` skips
    that extra pass: spill_len / updates / table are then None (not computed)
    and guard_fired reports the device guard.
    ``device_guard_fired`` (global-table overflow), ``pairs`` (distinct keys),
    ``global_updates``, ``table_buckets`` (the reference's table size M),
    ``kernels_launched`` and ``count_path`` (how the column was counted: "tiny",
    "dense" window, global "table" or "partitioned", include/cafs_b200.h) are
    device extras.
    """

    n: int = 0
    decision: DispatchDecision | None = None
    spill_len: int | None = 0
    guard_fired: bool = False
    stage_ms: dict[str, float] = field(default_factory=dict)
    counted_total: int = 0
    updates: int | None = 0
    tiny_count_failed: bool = False
    table: object | None = None
    pairs: int = 0
    global_updates: int = 0
    table_buckets: int = 0
    kernels_launched: int = 0
    kernel_ms: dict[str, float] = field(default_factory=dict)
    device_guard_fired: bool = False
    exact: bool = False
    sharded_path: str = ""  # sharded sort: "streamed" (device decisions) or "host"
    count_path: str = ""    # "", "tiny", "dense", "table" or "partitioned"

    @property
    def route(self) -> Route | None:
        return self.decision.route if self.decision else None


@dataclass
class PairList:  # sorter.py:199-216
    keys: np.ndarray
    counts: np.ndarray

    @classmethod
    def from_pairs(cls, pairs) -> "PairList":
        return cls(np.array([k for k, _ in pairs], dtype=np.uint64),
                   np.array([c for _, c in pairs], dtype=np.int64))

    def to_pairs(self) -> list[tuple[int, int]]:
        return list(zip(self.keys.tolist(), self.counts.tolist()))

    def __len__(self) -> int:
        return self.keys.shape[0]


# ---------------- pure host arithmetic (same formulas as the reference) ----------------

def check_hash_mult(mult) -> int:
    """buckets.py:54-67: None -> default; else an odd 64-bit integer."""
    if mult is None:
        return HASH_MULT
    mult = int(mult)
    if not 0 < mult <= _MASK64 or mult % 2 == 0:
        raise ValueError("hash multiplier must be an odd 64-bit integer")
    return mult


def fast_hash(x, m_log2, mult=None):
    """buckets.py:70-85: top m_log2 bits of x * mult mod 2^64."""
    if not 1 <= m_log2 <= 63:
        raise ValueError(f"m_log2 out of range: {m_log2}")
    mult = check_hash_mult(mult)
    if isinstance(x, np.ndarray):
        with np.errstate(over="ignore"):
            prod = x.astype(np.uint64, copy=False) * np.uint64(mult)
        return prod >> np.uint64(64 - m_log2)
    return ((int(x) * mult) & _MASK64) >> (64 - m_log2)


def _bit_ceil(v: int) -> int:
    return 1 << (v - 1).bit_length() if v > 1 else 1


def table_size_for(k_hat, n: int, cap: int) -> int:
    """buckets.py:92-105 (the reference's bucket count, reported in telemetry)."""
    if k_hat < 1 or n < 1:
        raise ValueError("k_hat and n must be >= 1")
    if cap not in (4, 8):
        raise ValueError(f"cap must be 4 or 8, got {cap}")
    m = _bit_ceil(int(math.ceil(8.0 * k_hat / cap)))
    m = min(m, _bit_ceil(int(math.ceil(n / cap))))
    return max(m, 8)


def chao1(u: int, f1: int, f2: int, n: int, saturated: bool) -> float:
    """cardinality.py:85-96 (the device computes the same float64 expression)."""
    if u < 1:
        raise ValueError("u must be >= 1")
    if saturated:
        return float(n)
    return min(u + (f1 * f1) / (2.0 * (f2 + 1)), float(n))


# ---------------- input handling ----------------

def _torch():
    import torch
    return torch


def _is_tensor(x) -> bool:
    try:
        torch = _torch()
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


_TORCH_KIND = {"torch.int64": ("int64", True), "torch.uint64": ("uint64", False),
               "torch.int32": ("int32", True), "torch.uint32": ("uint32", False)}


def _validate(x) -> None:
    """sorter.py:302-314, extended to torch tensors."""
    if _is_tensor(x):
        if x.dim() != 1:
            raise ValueError("cafs_sort expects a 1-D array")
        if str(x.dtype) not in _TORCH_KIND:
            raise TypeError(f"unsupported dtype {x.dtype}; need one of "
                            f"{[str(d) for d in SUPPORTED_DTYPES]}")
        if x.requires_grad:
            raise ValueError("cafs_sort sorts in place; tensor requires grad")
        n = x.shape[0]
    else:
        if not isinstance(x, np.ndarray):
            raise TypeError("cafs_sort expects a numpy array")
        if x.ndim != 1:
            raise ValueError("cafs_sort expects a 1-D array")
        if x.dtype not in SUPPORTED_DTYPES:
            raise TypeError(f"unsupported dtype {x.dtype}; need one of "
                            f"{[str(d) for d in SUPPORTED_DTYPES]}")
        if not x.flags.writeable:
            raise ValueError("cafs_sort sorts in place; array is read-only")
        n = x.shape[0]
    if n >= 1 << 32:
        raise ValueError("arrays of 2**32 or more elements exceed the 32-bit slot counters")


def _kind(x) -> tuple[str, bool]:
    if _is_tensor(x):
        return _TORCH_KIND[str(x.dtype)]
    return x.dtype.name, x.dtype.kind == "i"


def _device_index(t) -> int:
    return t.device.index if t.device.index is not None else _torch().cuda.current_device()


def _stream_ptr(dev: int) -> int:
    torch = _torch()
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)  # skips the Stream object
    return raw(dev) if raw is not None else torch.cuda.current_stream(dev).cuda_stream


class _Device64:
    """A contiguous 64-bit device view of the caller's array plus a write-back.

    64-bit CUDA tensors are used as they are.  32-bit ones are widened
    (sign- or zero-extension preserves order) and narrowed back; non-contiguous
    tensors go through a contiguous copy.  Host arrays are handled by the
    host entry point instead.
    """

    def __init__(self, x, native32: bool = False):
        torch = _torch()
        self.x = x
        self.kind, self.signed = _TORCH_KIND[str(x.dtype)]
        self.dev = _device_index(x)
        self.native32 = native32 and self.kind in ("int32", "uint32")
        if self.native32 or self.kind in ("int64", "uint64"):
            # cafs_sort_i32 takes 4-byte keys as they are
            self.t = x if x.is_contiguous() else x.contiguous()
        else:
            # widen to int64: int32 sign-extends, uint32 zero-extends (both < 2^63)
            self.t = x.to(torch.int64)
            self.signed = True
        self.n = x.shape[0]

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def write_back(self) -> None:
        if self.t is not self.x:
            self.x.copy_(self.t.to(self.x.dtype) if self.t.dtype != self.x.dtype else self.t)


def _decision_from_c(d: _lib.Decision, n: int, kind: str) -> DispatchDecision:
    route = _ROUTE_BY_CODE[d.route]
    if not d.has_estimate:
        return DispatchDecision(route)
    e = d.est
    est = CardinalityEstimate(float(e.k_hat), int(e.u), int(e.f1), int(e.f2), bool(e.saturated))
    if route is Route.TINY_COUNT:
        keys = np.array([e.keys[i] for i in range(e.nkeys)], dtype=np.uint64)
        return DispatchDecision(route, keys=_keys_to_reference_domain(keys, kind), estimate=est)
    if route is Route.MAIN:
        return DispatchDecision(route, k_hat=est.k_hat, estimate=est)
    return DispatchDecision(route, estimate=est)


def _keys_to_reference_domain(keys_u64: np.ndarray, kind: str) -> np.ndarray:
    """Device keys live in the 64-bit order-mapped domain; the reference reports
    tiny keys in the unsigned domain of the input dtype (sorter.py:84-94)."""
    if kind in ("int64", "uint64"):
        return keys_u64
    orig = (keys_u64 ^ np.uint64(1 << 63)).view(np.int64)  # widened int64 values
    if kind == "int32":
        return (orig.astype(np.int32).view(np.uint32) ^ np.uint32(1 << 31))
    return orig.astype(np.uint32)


def _stage_dict(t: _lib.Telemetry) -> dict[str, float]:
    out = {}
    for i, name in enumerate(("count", "sort_k", "emit")):
        if t.stage_ms[i] >= 0:
            out[name] = float(t.stage_ms[i])
    return out


# the reference's table key dtype per input dtype (to_unsigned, sorter.py:84-94)
_REF_DTYPE = {"int64": np.uint64, "uint64": np.uint64, "int32": np.uint32, "uint32": np.uint32}


_COUNT_PATHS = {1: "tiny", 2: "dense", 3: "table", 4: "partitioned"}  # cafs_count_path_t


def _fill_telemetry(tel: SortTelemetry, t: _lib.Telemetry, kind: str, timing: bool,
                    mult: int = HASH_MULT) -> None:
    tel.n = int(t.n)
    tel.decision = _decision_from_c(t.decision, tel.n, kind)
    tel.guard_fired = bool(t.guard_fired)
    tel.device_guard_fired = bool(t.guard_fired)
    tel.tiny_count_failed = bool(t.tiny_count_failed)
    tel.counted_total = int(t.counted_total)
    tel.pairs = int(t.pairs)
    tel.global_updates = int(t.global_updates)
    tel.kernels_launched = int(t.kernels_launched)
    tel.count_path = _COUNT_PATHS.get(int(t.count_path), "")
    cap = 8 if kind in ("int32", "uint32") else 4
    route = tel.decision.route
    if route is Route.MAIN and tel.decision.estimate is not None:
        tel.table_buckets = table_size_for(max(1.0, tel.decision.estimate.k_hat), tel.n, cap)
    tel.exact = bool(t.exact)
    if t.exact:
        tel.spill_len = int(t.ref_spill_len)
        tel.updates = int(t.ref_updates)
        tel.guard_fired = bool(t.ref_guard_fired)
        tel.counted_total = int(t.ref_counted_total)
        if route is Route.MAIN:
            tel.table = TableSummary(tel.table_buckets, cap, int(t.ref_hits), int(t.ref_claims),
                                     int(t.ref_spill_pushes), int(t.ref_spill_len),
                                     int(t.ref_updates), int(t.ref_counted_total),
                                     _REF_DTYPE[kind], mult)
        else:
            tel.table = None
    elif route is Route.MAIN:
        # the reference's table statistics were not computed (exact_telemetry=False)
        tel.spill_len = None
        tel.updates = None
        tel.table = None
    if timing:
        tel.stage_ms = _stage_dict(t)
        tel.kernel_ms = {name: float(t.kernel_ms[i])
                         for i, name in enumerate(("count_kernel", "emit_kernel", "estimate_kernel"))
                         if t.kernel_ms[i] >= 0}
    else:
        # labels of the stages that ran (times not measured without a telemetry object)
        tel.stage_ms = {}


# ---------------- the API ----------------

def cafs_sort(x, telemetry: SortTelemetry | None = None, hash_mult=None, *,
              direct_range: bool = True, exact_telemetry: bool | None = None) -> None:
    """Sort a 1-D integer array ascending, in place (sorter.py:335-386).

    ``x`` is a torch CUDA tensor (sorted on its device and current stream) or a
    numpy array / CPU tensor (sorted through the host entry point).  Pass a
    :class:`SortTelemetry` to observe the route, estimate, guard, the
    reference's bucket-table statistics and per-stage CUDA-event timings;
    ``exact_telemetry=False`` skips the statistics' extra input pass.
    """
    _validate(x)
    mult = check_hash_mult(hash_mult)
    want = telemetry is not None
    if exact_telemetry is None:
        exact_telemetry = want
    flags = (_lib.FLAG_TIMING if want else 0) | (0 if direct_range else _lib.FLAG_NO_DIRECT)
    if want and exact_telemetry:
        flags |= _lib.FLAG_EXACT_TELEMETRY
        kind0 = _kind(x)[0]
        flags |= {"int32": _lib.FLAG_DOM_I32, "uint32": _lib.FLAG_DOM_U32}.get(kind0, 0)
    t = _lib.Telemetry() if want else None  # no telemetry: the C side keeps its own
    lib = _lib.load()
    if _is_tensor(x) and x.is_cuda:
        v = _Device64(x, native32=True)
        ctx = _lib.context(v.dev)
        sort = lib.cafs_sort_i32 if v.native32 else lib.cafs_sort_i64
        rc = sort(ctx, v.ptr, v.n, int(v.signed), mult, flags,
                  ctypes.byref(t) if want else None, _stream_ptr(v.dev))
        _lib.check(rc, ctx, "cafs_sort")
        v.write_back()
        kind = v.kind
    else:
        kind = _host_sort(x, mult, flags, t)
    if want:
        _fill_telemetry(telemetry, t, kind, want, mult)


def _host_sort(x, mult: int, flags: int, t: _lib.Telemetry | None) -> str:
    """numpy / CPU-tensor input: one H2D, the device pipeline, one D2H."""
    torch = _torch()
    arr = x.numpy() if _is_tensor(x) else x
    kind = arr.dtype.name
    work = arr if arr.flags.c_contiguous else np.ascontiguousarray(arr)
    signed = int(arr.dtype.kind == "i")
    dev = torch.cuda.current_device() if torch.cuda.is_available() else 0
    ctx = _lib.context(dev)
    lib = _lib.load()
    ptr = work.ctypes.data if work.shape[0] else 0
    # 4-byte keys cross PCIe as 4 bytes (cafs_sort_i32_host)
    sort = lib.cafs_sort_i32_host if kind in ("int32", "uint32") else lib.cafs_sort_i64_host
    rc = sort(ctx, ptr, ptr, work.shape[0], signed, mult, flags,
              ctypes.byref(t) if t is not None else None,
              _stream_ptr(dev) if torch.cuda.is_available() else 0)
    _lib.check(rc, ctx, "cafs_sort")
    if work is not arr:
        arr[...] = work.astype(arr.dtype) if work.dtype != arr.dtype else work
    return kind


def _as_device(x):
    """Device 64-bit view for the stage APIs (numpy input is uploaded)."""
    torch = _torch()
    if _is_tensor(x) and x.is_cuda:
        return _Device64(x)
    arr = x.numpy() if _is_tensor(x) else np.asarray(x)
    kind = arr.dtype.name
    if kind in ("int32", "uint32"):
        t = torch.from_numpy(arr.astype(np.int64)).cuda()
        v = _Device64(t)
        v.kind = kind
        return v
    t = torch.from_numpy(np.ascontiguousarray(arr).view(np.int64)).cuda()
    v = _Device64(t)
    v.kind = kind
    v.signed = kind == "int64"
    return v


def dispatch(x, n: int | None = None, hash_mult=None) -> DispatchDecision:
    """sorter.py:141-162, with the reference's input semantics: x's values are
    taken as they are (cafs_sort passes the unsigned-domain copy, sorter.py:357);
    the monotone test uses x's own order and the tiny keys are the sampled
    values' 64-bit patterns (signed 32-bit values sign-extended, as the
    reference's uint64 FreqSet stores them, cardinality.py:71-73), ascending as
    unsigned integers.  Unsigned input -- what cafs_sort itself dispatches on --
    gives exactly cafs_sort's decision."""
    mult = check_hash_mult(hash_mult)
    if n is not None and n != x.shape[0]:
        x = x[:n]
    n = x.shape[0]
    if n < 2:
        return DispatchDecision(Route.ALREADY_SORTED)
    v = _as_device(x)
    ctx = _lib.context(v.dev)
    d = _lib.Decision()
    rc = _lib.load().cafs_dispatch_i64(ctx, v.ptr, v.n, int(v.signed), mult, ctypes.byref(d),
                                       _stream_ptr(v.dev))
    _lib.check(rc, ctx, "dispatch")
    dec = _decision_from_c(d, n, "uint64")
    if dec.keys is not None and v.signed:
        # device keys are order-mapped (bit 63 flipped): back to the raw bits
        dec.keys = np.sort(dec.keys ^ np.uint64(1 << 63))
    return dec


def sample_and_estimate(x, n: int | None = None, hash_mult=None) -> CardinalityEstimate:
    """cardinality.py:113-125 (hash_mult is validated; the spectrum is hash-independent)."""
    check_hash_mult(hash_mult)
    if n is not None and n != x.shape[0]:
        x = x[:n]
    n = x.shape[0]
    if n < 1:
        raise ValueError("n must be >= 1")
    v = _as_device(x)
    ctx = _lib.context(v.dev)
    e = _lib.Estimate()
    rc = _lib.load().cafs_estimate_i64(ctx, v.ptr, v.n, int(v.signed), ctypes.byref(e),
                                       _stream_ptr(v.dev))
    _lib.check(rc, ctx, "sample_and_estimate")
    return CardinalityEstimate(float(e.k_hat), int(e.u), int(e.f1), int(e.f2), bool(e.saturated))


def is_monotone(x) -> bool:
    """sorter.py:115-129: True iff x is non-decreasing."""
    if x.shape[0] < 2:
        return True
    v = _as_device(x)
    ctx = _lib.context(v.dev)
    out = ctypes.c_int()
    rc = _lib.load().cafs_is_monotone_i64(ctx, v.ptr, v.n, int(v.signed), ctypes.byref(out),
                                          _stream_ptr(v.dev))
    _lib.check(rc, ctx, "is_monotone")
    return bool(out.value)


def _to_u64_domain(keys: np.ndarray, kind: str, signed: bool) -> np.ndarray:
    k = np.asarray(keys)
    if kind in ("int32", "uint32"):
        wid = k.astype(np.int64) if kind == "int32" or k.dtype.kind == "i" else k.astype(np.int64)
        return wid.view(np.uint64) ^ np.uint64(1 << 63)
    if signed:
        return k.astype(np.int64).view(np.uint64) ^ np.uint64(1 << 63)
    return k.astype(np.uint64)


def tiny_counts(x, keys) -> np.ndarray:
    """_kernels.py:156-169: counts of each key (in x's own value domain)."""
    keys = np.asarray(keys)
    if keys.shape[0] > TINY_MAX_KEYS:
        raise ValueError("tiny-count takes at most 8 keys")
    v = _as_device(x)
    ku = np.ascontiguousarray(_to_u64_domain(keys, v.kind, v.signed))
    out = np.zeros(keys.shape[0], np.int64)
    ctx = _lib.context(v.dev)
    rc = _lib.load().cafs_tiny_counts_i64(
        ctx, v.ptr, v.n, int(v.signed), ku.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
        keys.shape[0], out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _stream_ptr(v.dev))
    _lib.check(rc, ctx, "tiny_counts")
    return out


def tiny_count_sort(x, keys, out) -> bool:
    """sorter.py:165-180: count x against <= 8 keys and emit into out on success;
    out is untouched on failure (and may alias x)."""
    keys = np.sort(np.asarray(keys))
    if keys.shape[0] > TINY_MAX_KEYS:
        raise ValueError("tiny-count takes at most 8 keys")
    counts = tiny_counts(x, keys)
    if int(counts.sum()) != x.shape[0]:
        return False
    emit(PairList(keys, counts), out)
    return True


def pair_sort(pairs: PairList) -> PairList:
    """sorter.py:228-241: sort (key, count) pairs ascending by uint64 key."""
    torch = _torch()
    n = len(pairs)
    keys = np.ascontiguousarray(pairs.keys, dtype=np.uint64)
    counts = np.ascontiguousarray(pairs.counts, dtype=np.int64)
    if n < 2:
        return PairList(keys.copy(), counts.copy())
    dk = torch.from_numpy(keys.view(np.int64)).cuda()
    dc = torch.from_numpy(counts).cuda()
    dev = _device_index(dk)
    ctx = _lib.context(dev)
    rc = _lib.load().cafs_pair_sort(ctx, dk.data_ptr(), dc.data_ptr(), n, _stream_ptr(dev))
    _lib.check(rc, ctx, "pair_sort")
    return PairList(dk.cpu().numpy().view(np.uint64), dc.cpu().numpy())


def emit(pairs: PairList, out) -> None:
    """sorter.py:244-251: expand sorted pairs into out (ValueError on a size mismatch)."""
    torch = _torch()
    total = int(np.asarray(pairs.counts).sum()) if len(pairs) else 0
    n_out = out.shape[0]
    if total != n_out:
        raise ValueError(f"pair counts sum to {total}, out has {n_out} slots")
    if total == 0:
        return
    kind, signed = _kind(out)
    ku = np.ascontiguousarray(_to_u64_domain(np.asarray(pairs.keys), kind, signed))
    dk = torch.from_numpy(ku.view(np.int64)).cuda()
    dc = torch.from_numpy(np.ascontiguousarray(pairs.counts, dtype=np.int64)).cuda()
    if _is_tensor(out) and out.is_cuda and kind in ("int64", "uint64") and out.is_contiguous():
        dst = out
    else:
        dst = torch.empty(n_out, dtype=torch.int64, device=dk.device)
    dev = _device_index(dk)
    ctx = _lib.context(dev)
    rc = _lib.load().cafs_emit_i64(ctx, dk.data_ptr(), dc.data_ptr(), len(pairs), dst.data_ptr(),
                                   0, n_out, total,
                                   int(signed or kind in ("int32", "uint32")), _stream_ptr(dev))
    _lib.check(rc, ctx, "emit")
    if dst is out:
        return
    if _is_tensor(out):
        out.copy_(dst.to(out.dtype) if out.dtype != dst.dtype else dst)
    else:
        host = dst.cpu().numpy()
        out[...] = host.astype(out.dtype) if kind in ("int32", "uint32") else host.view(out.dtype)


def fallback_sort(x) -> None:
    """sorter.py:132-138: the fallback engine (on-device LSD radix sort), in place."""
    _validate(x)
    if _is_tensor(x) and x.is_cuda:
        v = _Device64(x)
    else:
        v = _as_device(x)
    ctx = _lib.context(v.dev)
    rc = _lib.load().cafs_fallback_sort_i64(ctx, v.ptr, v.n, int(v.signed), _stream_ptr(v.dev))
    _lib.check(rc, ctx, "fallback_sort")
    if _is_tensor(x) and x.is_cuda:
        v.write_back()
    else:
        host = v.t.cpu().numpy()
        if v.kind in ("int32", "uint32"):
            x[...] = host.astype(x.dtype)
        else:
            x[...] = host.view(x.dtype) if isinstance(x, np.ndarray) else _torch().from_numpy(host)
