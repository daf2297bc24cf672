"""ctypes binding of libcafs_b200.so (the C ABI declared in include/cafs_b200.h).

The library is the product: there is no Python or CPU fallback.  Importing
works without it (so the package and its pure host logic import on a CPU-only
machine), but every call that needs the device raises ``RuntimeError`` when the
library is missing or no sm_100 device is present.
"""

from __future__ import annotations

import atexit
import ctypes
import os
import threading

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libcafs_b200.so")

TINY_MAX = 8

# status codes (cafs_status_t)
OK, EINVAL, ECUDA, ENOMEM, ESUM, EINTERNAL = 0, -1, -2, -3, -4, -5
FLAG_TIMING = 1
FLAG_NO_DIRECT = 2
FLAG_EXACT_TELEMETRY = 4
FLAG_DOM_I32 = 8
FLAG_DOM_U32 = 16


class Estimate(ctypes.Structure):
    _fields_ = [("k_hat", ctypes.c_double), ("u", ctypes.c_int64), ("f1", ctypes.c_int64),
                ("f2", ctypes.c_int64), ("saturated", ctypes.c_int32), ("nkeys", ctypes.c_int32),
                ("keys", ctypes.c_uint64 * TINY_MAX)]


class Decision(ctypes.Structure):
    _fields_ = [("route", ctypes.c_int32), ("has_estimate", ctypes.c_int32), ("est", Estimate)]


class Telemetry(ctypes.Structure):
    _fields_ = [("n", ctypes.c_uint64), ("decision", Decision),
                ("tiny_count_failed", ctypes.c_int32), ("guard_fired", ctypes.c_int32),
                ("counted_total", ctypes.c_uint64), ("pairs", ctypes.c_uint64),
                ("table_buckets", ctypes.c_uint64), ("global_updates", ctypes.c_uint64),
                ("stage_ms", ctypes.c_float * 3), ("kernel_ms", ctypes.c_float * 4),
                ("kernels_launched", ctypes.c_uint32), ("exact", ctypes.c_int32),
                ("ref_guard_fired", ctypes.c_int32), ("ref_spill_len", ctypes.c_uint64),
                ("ref_updates", ctypes.c_uint64), ("ref_hits", ctypes.c_uint64),
                ("ref_claims", ctypes.c_uint64), ("ref_spill_pushes", ctypes.c_uint64),
                ("ref_counted_total", ctypes.c_uint64), ("count_path", ctypes.c_int32),
                ("_reserved", ctypes.c_int32)]


# every symbol include/cafs_b200.h declares, with its ctypes signature
_P = ctypes.c_void_p
_U64 = ctypes.c_uint64
_I = ctypes.c_int
SIGNATURES = {
    "cafs_abi_version": (_I, []),
    "cafs_status_string": (ctypes.c_char_p, [_I]),
    "cafs_last_error": (ctypes.c_char_p, [_P]),
    "cafs_ctx_create": (_I, [_I, ctypes.POINTER(_P)]),
    "cafs_ctx_destroy": (None, [_P]),
    "cafs_sort_i64": (_I, [_P, _P, _U64, _I, _U64, ctypes.c_uint32, ctypes.POINTER(Telemetry), _P]),
    "cafs_sort_i64_host": (_I, [_P, _P, _P, _U64, _I, _U64, ctypes.c_uint32,
                                ctypes.POINTER(Telemetry), _P]),
    "cafs_sort_i32": (_I, [_P, _P, _U64, _I, _U64, ctypes.c_uint32, ctypes.POINTER(Telemetry), _P]),
    "cafs_sort_i32_host": (_I, [_P, _P, _P, _U64, _I, _U64, ctypes.c_uint32,
                                ctypes.POINTER(Telemetry), _P]),
    "cafs_dispatch_i64": (_I, [_P, _P, _U64, _I, _U64, ctypes.POINTER(Decision), _P]),
    "cafs_estimate_i64": (_I, [_P, _P, _U64, _I, ctypes.POINTER(Estimate), _P]),
    "cafs_is_monotone_i64": (_I, [_P, _P, _U64, _I, ctypes.POINTER(_I), _P]),
    "cafs_tiny_counts_i64": (_I, [_P, _P, _U64, _I, ctypes.POINTER(_U64), _I,
                                  ctypes.POINTER(ctypes.c_int64), _P]),
    "cafs_count_pairs_i64": (_I, [_P, _P, _U64, _I, _U64, _P, _P, _U64, ctypes.POINTER(_U64), _P]),
    "cafs_merge_pairs": (_I, [_P, _P, _P, _U64, _P, _P, _U64, ctypes.POINTER(_U64), _P]),
    "cafs_pair_sort": (_I, [_P, _P, _P, _U64, _P]),
    "cafs_emit_i64": (_I, [_P, _P, _P, _U64, _P, _U64, _U64, _U64, _I, _P]),
    "cafs_fallback_sort_i64": (_I, [_P, _P, _U64, _I, _P]),
    "cafs_ctx_kernel_count": (_U64, [_P]),
    "cafs_shard_begin_i64": (_I, [_P, _P, _U64, _I, _P, _P]),
    "cafs_shard_local_pairs_i64": (_I, [_P, _P, _P, _U64, ctypes.POINTER(_U64), _P]),
    "cafs_nccl_unique_id": (_I, [ctypes.c_char_p]),
    "cafs_comm_create": (_I, [_I, ctypes.c_char_p, _I, _I, ctypes.POINTER(_P)]),
    "cafs_comm_destroy": (_I, [_P]),
    "cafs_sort_i64_sharded": (_I, [_P, _P, _P, _U64, _I, _U64, ctypes.POINTER(Telemetry),
                                   ctypes.POINTER(_I), _P]),
    "cafs_sort_i32_sharded": (_I, [_P, _P, _P, _U64, _I, _U64, ctypes.POINTER(Telemetry),
                                   ctypes.POINTER(_I), _P]),
    "cafs_shard_sample_i64": (_I, [_P, _P, _U64, _I, _P, _I, _I, _P, _P]),
    "cafs_shard_count_i64": (_I, [_P, _P, _U64, _I, _U64, _P, _I, _P, _P, _P, _U64, _P]),
    "cafs_shard_finish_i64": (_I, [_P, _P, _U64, _I, _P, _P, _I, _U64, ctypes.POINTER(Telemetry),
                                   ctypes.POINTER(_I), _P]),
    "cafs_key_span_i64": (_I, [_P, _P, _U64, _I, ctypes.POINTER(_U64), ctypes.POINTER(_U64), _P]),
    "cafs_partition_i64": (_I, [_P, _P, _U64, _I, _U64, _U64, _P, ctypes.POINTER(_U64), _P]),
    "cafs_shard_fallback_plan": (_I, [_I, _I, _P, _P, _P, _P, ctypes.POINTER(_U64)]),
    "cafs_gen_mix": (_I, [_P, _U64, _U64, _U64, _P]),
    "cafs_gen_draw": (_I, [_P, _U64, _U64, _U64, _P, _U64, _P, _P]),
}

_lib = None
_lock = threading.Lock()
_ctx: dict[int, int] = {}


class LibraryMissing(RuntimeError):
    pass


def load(path: str = LIB_PATH):
    """Load the shared library (CPU-safe: loading needs no GPU)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise LibraryMissing(
                    f"{path} is not built; run `python -m paper_2605_25040_b200.build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(path)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def context(device: int) -> int:
    """Per-device native context (control block, global table, scratch)."""
    lib = load()
    h = _ctx.get(device)
    if h is None:
        with _lock:
            h = _ctx.get(device)
            if h is None:
                out = _P()
                rc = lib.cafs_ctx_create(device, ctypes.byref(out))
                if rc != OK:
                    raise RuntimeError(
                        f"cafs_ctx_create(device={device}) failed: "
                        f"{lib.cafs_status_string(rc).decode()} (needs an sm_100 B200)")
                h = out.value
                _ctx[device] = h
    return h


def check(rc: int, ctx: int | None = None, what: str = "call") -> None:
    if rc == OK:
        return
    lib = load()
    msg = lib.cafs_status_string(rc).decode()
    detail = lib.cafs_last_error(ctx).decode() if ctx else ""
    text = f"{what}: {msg}" + (f" ({detail})" if detail else "")
    if rc in (EINVAL, ESUM):
        raise ValueError(text)
    raise RuntimeError(text)


@atexit.register
def _cleanup():
    if _lib is None:
        return
    for h in list(_ctx.values()):
        try:
            _lib.cafs_ctx_destroy(h)
        except Exception:
            pass
    _ctx.clear()
