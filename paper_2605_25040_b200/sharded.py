"""Row-sharded multi-GPU CAFS sort over torch.distributed (NCCL on NVLink/NVSwitch).

One process per GPU.  The global column is the concatenation of every rank's
``x_local`` in rank order; afterwards rank r's ``x_local`` holds rows
``[off_r, off_r + n_r)`` of the globally sorted column (same shard sizes), so the
concatenated result is bit-identical to a single-GPU ``cafs_sort`` (and to the
reference) on the whole column.

The reference is single-threaded; the paper names a parallel CAFS with
per-thread tables and a final merge as future work.  Here:

1. dispatch, globally identical on every rank (sorter.py:141-162):
   * monotone: each shard's full non-decreasing check plus its first/last key,
     all-gathered (global monotone <=> every shard monotone and the shard
     boundaries ordered);
   * samples: the global positions ``i * (N // 1024)`` that fall in a shard
     are gathered locally and all-gathered (1024 x 8 B in total), then every
     rank runs the estimate kernel on the same 1024 values and the same
     float64 Chao1 with the global N;
2. TINY: local tiny counts, all-reduce of <= 8 counters; a miss anywhere
   re-enters MAIN on all ranks (sorter.py:378-385);
3. MAIN: local hash count into sorted (key, count) pairs, all-gather of the
   pair tables (<= K x 16 B per rank), the merge (union + fold, sorter.py:276-285)
   on every rank, then each rank emits only its own output slice from the
   global prefix sum;
4. FALLBACK / guard: a distributed MSD sort (:func:`_exchange_sort`, SURVEY.md
   §8(f)2): one partition pass on a globally agreed 4096-way digit, an
   all-to-all of bucket ranges over NCCL, a local sort of the received range;
   inputs under 2048 rows are gathered and sorted everywhere.

Local steps go through :class:`DeviceOps` (the C ABI); collectives through
``torch.distributed``.  Tests inject a CPU ``ops`` object with the same
interface to check this orchestration under ``gloo``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .sorter import (
    SAMPLE_TARGET,
    SMALL_N_CUTOFF,
    TINY_MAX_KEYS,
    CardinalityEstimate,
    DispatchDecision,
    Route,
    SortTelemetry,
    check_hash_mult,
    chao1,
    table_size_for,
)

_SIGN = 1 << 63
PARTITION_BUCKETS = 4096  # CAFS_PARTITION_BUCKETS


def _torch():
    import torch
    return torch


# the device's pair capacity: global table + the ~0 sentinel + the dense window
_PAIR_CAP = (1 << 24) + 1 + 8192


class DeviceOps:
    """Local pipeline steps on this rank's GPU, through libcafs_b200.so."""

    def __init__(self, device: int, signed: bool = True):
        self.device = device
        self.signed = signed
        self.ctx = _lib.context(device)
        self.lib = _lib.load()

    def _stream(self):
        return _torch().cuda.current_stream(self.device).cuda_stream

    def kernel_count(self) -> int:
        """Kernels launched so far by this rank's context (C ABI accounting)."""
        return int(self.lib.cafs_ctx_kernel_count(self.ctx))

    def is_monotone(self, x) -> bool:
        if x.shape[0] < 2:
            return True
        out = ctypes.c_int()
        _lib.check(self.lib.cafs_is_monotone_i64(self.ctx, x.data_ptr(), x.shape[0],
                                                 int(self.signed), ctypes.byref(out),
                                                 self._stream()), self.ctx, "is_monotone")
        return bool(out.value)

    def estimate(self, samples) -> tuple[int, int, int, bool, list[int]]:
        """(u, f1, f2, saturated, ascending distinct keys if u <= 8) of the samples."""
        e = _lib.Estimate()
        _lib.check(self.lib.cafs_estimate_i64(self.ctx, samples.data_ptr(), samples.shape[0],
                                              int(self.signed), ctypes.byref(e), self._stream()),
                   self.ctx, "estimate")
        keys = [int(e.keys[i]) for i in range(e.nkeys)]
        return int(e.u), int(e.f1), int(e.f2), bool(e.saturated), keys

    def tiny_counts(self, x, keys_u64: list[int]) -> np.ndarray:
        k = np.array(keys_u64, dtype=np.uint64)
        out = np.zeros(len(keys_u64), np.int64)
        if x.shape[0]:
            _lib.check(self.lib.cafs_tiny_counts_i64(
                self.ctx, x.data_ptr(), x.shape[0], int(self.signed),
                k.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), len(keys_u64),
                out.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), self._stream()),
                self.ctx, "tiny_counts")
        return out

    def _pairs_out(self, cap):
        torch = _torch()
        dev = torch.device("cuda", self.device)
        return (torch.empty(cap, dtype=torch.int64, device=dev),
                torch.empty(cap, dtype=torch.int64, device=dev))

    def count_pairs(self, x, mult: int):
        """Sorted distinct (key, count) pairs of the shard, or None on table overflow."""
        cap = _PAIR_CAP
        k, c = self._pairs_out(cap)
        if x.shape[0] == 0:
            return k[:0], c[:0]
        npairs = ctypes.c_uint64()
        rc = self.lib.cafs_count_pairs_i64(self.ctx, x.data_ptr(), x.shape[0], int(self.signed),
                                           mult, k.data_ptr(), c.data_ptr(), cap,
                                           ctypes.byref(npairs), self._stream())
        if rc == _lib.EINVAL:
            return None
        _lib.check(rc, self.ctx, "count_pairs")
        return k[:npairs.value], c[:npairs.value]

    def merge_pairs(self, keys, counts):
        cap = _PAIR_CAP
        k, c = self._pairs_out(cap)
        npairs = ctypes.c_uint64()
        rc = self.lib.cafs_merge_pairs(self.ctx, keys.data_ptr(), counts.data_ptr(), keys.shape[0],
                                       k.data_ptr(), c.data_ptr(), cap, ctypes.byref(npairs),
                                       self._stream())
        if rc == _lib.EINVAL:
            return None
        _lib.check(rc, self.ctx, "merge_pairs")
        return k[:npairs.value], c[:npairs.value]

    def emit_slice(self, keys, counts, out, begin: int, end: int, total: int) -> None:
        if end <= begin:
            return
        _lib.check(self.lib.cafs_emit_i64(self.ctx, keys.data_ptr(), counts.data_ptr(),
                                          keys.shape[0], out.data_ptr(), begin, end, total,
                                          int(self.signed), self._stream()), self.ctx, "emit")

    def fallback_sort(self, x) -> None:
        if x.shape[0] < 2:
            return
        _lib.check(self.lib.cafs_fallback_sort_i64(self.ctx, x.data_ptr(), x.shape[0],
                                                   int(self.signed), self._stream()),
                   self.ctx, "fallback_sort")

    def key_span(self, x) -> tuple[int, int]:
        """(min, max) of the order-mapped keys; (2**64-1, 0) for an empty shard."""
        lo, hi = ctypes.c_uint64(), ctypes.c_uint64()
        _lib.check(self.lib.cafs_key_span_i64(self.ctx, x.data_ptr(), x.shape[0], int(self.signed),
                                              ctypes.byref(lo), ctypes.byref(hi),
                                              self._stream()), self.ctx, "key_span")
        return int(lo.value), int(hi.value)

    def partition(self, x, g_min: int, g_max: int):
        """x grouped by the global bucket digit; (grouped tensor, counts[4096])."""
        torch = _torch()
        out = torch.empty_like(x)
        counts = np.zeros(PARTITION_BUCKETS, np.uint64)
        _lib.check(self.lib.cafs_partition_i64(
            self.ctx, x.data_ptr(), x.shape[0], int(self.signed), g_min, g_max, out.data_ptr(),
            counts.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)), self._stream()),
            self.ctx, "partition")
        return out, counts.astype(np.int64)

    # ---- the stream-ordered pipeline (cafs_shard_*): no host sync until finish ----
    def shard_begin(self, x, hdr) -> None:
        _lib.check(self.lib.cafs_shard_begin_i64(self.ctx, x.data_ptr(), x.shape[0],
                                                 int(self.signed), hdr.data_ptr(), self._stream()),
                   self.ctx, "shard_begin")

    def shard_sample(self, x, hdr_all, world: int, rank: int, samples) -> None:
        _lib.check(self.lib.cafs_shard_sample_i64(self.ctx, x.data_ptr(), x.shape[0],
                                                  int(self.signed), hdr_all.data_ptr(), world,
                                                  rank, samples.data_ptr(), self._stream()),
                   self.ctx, "shard_sample")

    def shard_count(self, x, mult: int, hdr_all, world: int, samples, tiny, send, cap: int):
        _lib.check(self.lib.cafs_shard_count_i64(self.ctx, x.data_ptr(), x.shape[0],
                                                 int(self.signed), mult, hdr_all.data_ptr(), world,
                                                 samples.data_ptr(), tiny.data_ptr(),
                                                 send.data_ptr(), cap, self._stream()),
                   self.ctx, "shard_count")

    def shard_finish(self, x, tiny_sum, recv, world: int, cap: int):
        """(status, telemetry): status 0 = sorted, 1 = needs the host-driven path."""
        t = _lib.Telemetry()
        status = ctypes.c_int()
        _lib.check(self.lib.cafs_shard_finish_i64(self.ctx, x.data_ptr(), x.shape[0],
                                                  int(self.signed), tiny_sum.data_ptr(),
                                                  recv.data_ptr(), world, cap, ctypes.byref(t),
                                                  ctypes.byref(status), self._stream()),
                   self.ctx, "shard_finish")
        return int(status.value), t

    def sort_native(self, x, ncomm: int, mult: int):
        """The whole stream-ordered sharded sort with the library's own NCCL
        communicator (cafs_sort_i64_sharded, or cafs_sort_i32_sharded for
        4-byte shards): (status, telemetry)."""
        t = _lib.Telemetry()
        status = ctypes.c_int()
        torch = _torch()
        if x.dtype in (torch.int32, torch.uint32):
            fn, signed = self.lib.cafs_sort_i32_sharded, x.dtype == torch.int32
        else:
            fn, signed = self.lib.cafs_sort_i64_sharded, self.signed
        _lib.check(fn(self.ctx, ncomm, x.data_ptr(), x.shape[0], int(signed), mult,
                      ctypes.byref(t), ctypes.byref(status), self._stream()),
                   self.ctx, "sort_sharded")
        return int(status.value), t

    def shard_local_pairs(self):
        """This shard's pairs from the streamed count phase; None on overflow."""
        k, c = self._pairs_out(_PAIR_CAP)
        npairs = ctypes.c_uint64()
        _lib.check(self.lib.cafs_shard_local_pairs_i64(self.ctx, k.data_ptr(), c.data_ptr(),
                                                       _PAIR_CAP, ctypes.byref(npairs),
                                                       self._stream()), self.ctx, "shard_pairs")
        if npairs.value == (1 << 64) - 1:
            return None
        return k[:npairs.value], c[:npairs.value]

    def keys_tensor(self, keys_u64: list[int], counts: np.ndarray):
        torch = _torch()
        dev = torch.device("cuda", self.device)
        k = torch.from_numpy(np.array(keys_u64, dtype=np.uint64).view(np.int64)).to(dev)
        c = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int64)).to(dev)
        return k, c


class Comm:
    """The few collectives the sharded sort needs, over torch.distributed.

    With NCCL the collective buffers live on the GPU; with gloo (CPU tests, or
    several ranks sharing one GPU) they are staged through host memory."""

    def __init__(self, group=None, device=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        host_only = dist.get_backend(group) == "gloo"
        self.device = None if host_only else device  # where collective buffers live

    def _t(self, a, dtype=None):
        torch = _torch()
        t = torch.as_tensor(a, dtype=dtype or torch.int64)
        return t.to(self.device) if self.device is not None else t

    def all_gather_ints(self, vals: list[int]) -> list[list[int]]:
        """u64 values of every rank, rank order; one collective, one copy back."""
        torch = _torch()
        t = self._t(np.array(vals, dtype=np.uint64).view(np.int64))
        if self.device is not None:  # NCCL: one [world, k] device tensor
            out = torch.empty((self.world, t.shape[0]), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            rows = out.cpu().numpy()
        else:
            outs = [torch.empty_like(t) for _ in range(self.world)]
            self.dist.all_gather(outs, t, group=self.group)
            rows = torch.stack(outs).numpy()
        return rows.view(np.uint64).astype(object).tolist()

    def all_reduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self._t(np.array(a, dtype=np.int64))  # a copy: the reduction is in place
        self.dist.all_reduce(t, group=self.group)
        return t.cpu().numpy()

    def all_to_all_var(self, send, in_splits: list[int], out_splits: list[int]):
        """Variable-size all-to-all of a 1-D int64 tensor (send is split in rank order)."""
        torch = _torch()
        stage = self.device is None and send.is_cuda
        src = send.cpu() if stage else send
        out = torch.empty(int(sum(out_splits)), dtype=send.dtype, device=src.device)
        self.dist.all_to_all_single(out, src, out_splits, in_splits, group=self.group)
        return out.to(send.device) if stage else out

    def all_gather_into(self, out, t) -> None:
        """out[world * k] <- every rank's t[k] in rank order (stream-ordered on NCCL)."""
        if self.device is not None:
            self.dist.all_gather_into_tensor(out, t, group=self.group)
            return
        torch = _torch()
        src = t.cpu()
        parts = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(parts, src, group=self.group)
        out.copy_(torch.cat(parts).to(out.device))

    def all_reduce_inplace(self, t) -> None:
        """t <- SUM over ranks (stream-ordered on NCCL)."""
        if self.device is not None:
            self.dist.all_reduce(t, group=self.group)
            return
        w = t.cpu()
        self.dist.all_reduce(w, group=self.group)
        t.copy_(w.to(t.device))

    def all_reduce_tensor(self, t):
        """Element-wise SUM across ranks of a fixed-shape tensor (a new tensor)."""
        stage = self.device is None and t.is_cuda
        w = t.cpu() if stage else t.clone()
        self.dist.all_reduce(w, group=self.group)
        return w.to(t.device) if stage else w

    def all_gather_pairs(self, keys, counts, sizes: list[int]):
        """All-gather every rank's (keys, counts) in rank order, sizes known: one
        collective of a [2, max] tensor per rank."""
        torch = _torch()
        m = max(sizes) if sizes else 0
        dev = keys.device if self.device is not None or not keys.is_cuda else torch.device("cpu")
        pack = torch.zeros((2, max(m, 1)), dtype=keys.dtype, device=dev)
        pack[0, :keys.shape[0]] = keys.to(dev)
        pack[1, :counts.shape[0]] = counts.to(dev)
        out = [torch.empty_like(pack) for _ in range(self.world)]
        self.dist.all_gather(out, pack, group=self.group)
        k = torch.cat([o[0, :s] for o, s in zip(out, sizes)]).to(keys.device)
        c = torch.cat([o[1, :s] for o, s in zip(out, sizes)]).to(keys.device)
        return k, c

    def all_gather_var(self, t, sizes: list[int] | None = None):
        """All-gather 1-D int64 tensors of different lengths (pad to the max)."""
        torch = _torch()
        if sizes is None:
            sizes = [s[0] for s in self.all_gather_ints([int(t.shape[0])])]
        m = max(sizes) if sizes else 0
        dev = t.device if self.device is not None or not t.is_cuda else torch.device("cpu")
        pad = torch.zeros(m, dtype=t.dtype, device=dev)
        pad[:t.shape[0]] = t.to(dev)
        out = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(out, pad, group=self.group)
        return torch.cat([o[:s] for o, s in zip(out, sizes)]).to(t.device)


_OPS: dict = {}
_COMMS: dict = {}


def _device_ops(device: int, signed: bool) -> DeviceOps:
    """One DeviceOps per (device, signedness): the context and library handles
    are per process anyway, and building them costs host time on every call."""
    ops = _OPS.get((device, signed))
    if ops is None:
        ops = _OPS[(device, signed)] = DeviceOps(device, signed)
    return ops


def _comm(group, device) -> Comm:
    """One Comm per (process group, device); a destroyed default group is
    replaced by a new object, so the key includes the group's identity."""
    import torch.distributed as dist
    g = group if group is not None else dist.group.WORLD
    key = (id(g), str(device))
    c = _COMMS.get(key)
    if (c is None or c.group is not group or c.world != dist.get_world_size(group)
            or c.rank != dist.get_rank(group)):
        c = _COMMS[key] = Comm(group, device)
    return c


def msd_shift(g_min: int, g_max: int, bits: int = 12) -> int:
    """Shift that fits the span [g_min, g_max] into a `bits`-bit digit
    (k - g_min) >> shift (msd.cu msd_shift)."""
    if g_max <= g_min:
        return 0
    hb = (g_max - g_min).bit_length() - 1
    return hb + 1 - bits if hb + 1 > bits else 0


def bucket_ranges(totals: np.ndarray, sizes: list[int]) -> list[tuple[int, int]]:
    """Bucket range [lo, hi) each rank needs for its output slice.

    Rank d owns sorted rows [off_d, off_d + n_d); bucket b holds rows
    [P[b], P[b+1]) of the sorted column.  A bucket straddling two slices goes to
    both ranks (each sorts it and keeps its part)."""
    P = np.concatenate([[0], np.cumsum(totals, dtype=np.int64)])
    out, off = [], 0
    for n_d in sizes:
        if n_d == 0:
            out.append((0, 0))
        else:
            lo = int(np.searchsorted(P[1:], off, side="right"))
            hi = int(np.searchsorted(P[:-1], off + n_d, side="left"))
            out.append((lo, hi))
        off += n_d
    return out


def _exchange_sort(x_local, sizes: list[int], comm, ops) -> None:
    """Distributed fallback sort: one MSD partition pass, an
    all-to-all of bucket ranges, a local sort of the received range.

    1. global span: all-gather of each shard's min/max of the order-mapped
       keys -> one 4096-way digit (k - min) >> shift, the same on every rank
       (so bucket b precedes bucket b+1 globally);
    2. local partition by that digit (cafs_partition_i64) and an all-reduce of
       the bucket counts -> the global row range of every bucket;
    3. rank d receives, from every rank, the buckets overlapping its output
       slice (all_to_all_single with per-rank splits), sorts them locally with
       the single-GPU fallback and keeps its rows.
    Traffic per key: ~8 B over NVLink plus the local partition and sort; every
    rank sorts ~1/N of the column (versus all of it when gathering)."""
    torch = _torch()
    rank, world = comm.rank, comm.world
    n_local = int(x_local.shape[0])
    off = int(sum(sizes[:rank]))
    spans = comm.all_gather_ints(list(ops.key_span(x_local)))
    g_min, g_max = (1 << 64) - 1, 0
    for (lo, hi), n_r in zip(spans, sizes):
        if n_r:
            g_min = min(g_min, lo)
            g_max = max(g_max, hi)
    part, counts = ops.partition(x_local, g_min, g_max)
    totals = comm.all_reduce_sum(counts)
    ranges = bucket_ranges(totals, sizes)
    L = np.concatenate([[0], np.cumsum(counts, dtype=np.int64)])
    in_splits = [int(L[hi] - L[lo]) for lo, hi in ranges]
    matrix = comm.all_gather_ints(in_splits)  # matrix[s][d]: rows s sends to d
    out_splits = [int(matrix[s][rank]) for s in range(world)]
    pieces = [part[int(L[lo]):int(L[hi])] for lo, hi in ranges]
    send = torch.cat(pieces) if pieces else part[:0]
    recv = comm.all_to_all_var(send, in_splits, out_splits)
    if n_local == 0:
        return
    ops.fallback_sort(recv)
    P = np.concatenate([[0], np.cumsum(totals, dtype=np.int64)])
    start = off - int(P[ranges[rank][0]])
    x_local.copy_(recv[start:start + n_local])


def cafs_sort_sharded(x_local, group=None, hash_mult=None, telemetry: SortTelemetry | None = None,
                      ops=None, signed: bool | None = None) -> None:
    """Sort the row-sharded global column in place; see the module docstring.

    int64 / uint64 shards run as they are; contiguous int32 / uint32 CUDA
    shards run natively at 4 bytes per key (cafs_sort_i32_sharded); other
    4-byte shards (strided views, the host-driven continuation) are sorted
    through a contiguous int64 copy -- widening preserves the order and every
    rank's decision (the keys' identities are unchanged)."""
    torch = _torch()
    mult = check_hash_mult(hash_mult)
    if x_local.dim() != 1:
        raise ValueError("cafs_sort_sharded expects a 1-D shard")
    if (x_local.dtype in (torch.int32, torch.uint32) and x_local.is_cuda
            and x_local.is_contiguous() and ops is None and _native_enabled()
            and _sort_sharded_native32(x_local, group, mult, telemetry)):
        return
    if x_local.dtype not in (torch.int64, torch.uint64) or not x_local.is_contiguous():
        if x_local.dtype not in (torch.int64, torch.uint64, torch.int32, torch.uint32):
            raise TypeError(f"unsupported dtype {x_local.dtype}")
        wide = x_local.to(torch.int64) if x_local.dtype != torch.uint64 else x_local.contiguous()
        cafs_sort_sharded(wide, group, hash_mult, telemetry, ops,
                          signed if x_local.dtype == torch.uint64 else True)
        x_local.copy_(wide.to(x_local.dtype) if wide.dtype != x_local.dtype else wide)
        if (telemetry is not None and x_local.dtype in (torch.int32, torch.uint32)
                and telemetry.route is Route.MAIN and telemetry.decision.estimate is not None):
            # the reference's table for 4-byte keys has 8-slot buckets (buckets.py:33-43)
            telemetry.table_buckets = table_size_for(
                max(1.0, telemetry.decision.estimate.k_hat), telemetry.n, 8)
        return
    if ops is None:
        if signed is None:
            signed = x_local.dtype == torch.int64
        dev = x_local.device.index if x_local.device.index is not None else torch.cuda.current_device()
        ops = _device_ops(dev, signed)
    else:
        signed = ops.signed if signed is None else signed
    comm = _comm(group, x_local.device if x_local.is_cuda else None)
    tel = telemetry if telemetry is not None else SortTelemetry()
    k0 = ops.kernel_count() if hasattr(ops, "kernel_count") else 0
    try:
        fast = (hasattr(ops, "shard_begin") and x_local.is_cuda and x_local.is_contiguous()
                and x_local.dtype in (torch.int64, torch.uint64))
        native = (fast and comm.device is not None and hasattr(ops, "sort_native")
                  and _native_enabled())
        if native and _sort_sharded_native(x_local, comm, ops, tel, mult):
            pass  # "native", or "native+host" when the merge continued on the host
        elif not native and fast and _sort_sharded_streamed(x_local, comm, ops, tel, mult):
            tel.sharded_path = "streamed"
        else:
            tel.sharded_path = "host"
            _sort_sharded(x_local, comm, ops, tel, mult, signed)
    finally:
        if hasattr(ops, "kernel_count"):
            tel.kernels_launched = ops.kernel_count() - k0


SHARD_PAIR_CAP = 8192  # pairs per rank in the stream-ordered exchange (the pair sort's capacity)

_NATIVE_COMMS: dict = {}


def _native_enabled() -> bool:
    import os
    return os.environ.get("CAFS_SHARD_NATIVE", "1") != "0"


def _native_comm(comm, device: int):
    """The library's NCCL communicator for this process group (cafs_comm_create),
    made once: rank 0's unique id is broadcast over the group itself."""
    torch = _torch()
    dist = comm.dist
    key = (id(comm.group if comm.group is not None else dist.group.WORLD), device, comm.world,
           comm.rank)
    h = _NATIVE_COMMS.get(key)
    if h is not None:
        return h
    lib = _lib.load()
    buf = ctypes.create_string_buffer(128)
    if comm.rank == 0:
        _lib.check(lib.cafs_nccl_unique_id(buf), None, "nccl_unique_id")
    idt = torch.frombuffer(bytearray(buf.raw), dtype=torch.uint8).to(comm.device)
    src = 0 if comm.group is None else dist.get_global_rank(comm.group, 0)
    dist.broadcast(idt, src=src, group=comm.group)
    out = ctypes.c_void_p()
    _lib.check(lib.cafs_comm_create(device, bytes(idt.cpu().numpy().tobytes()), comm.world,
                                    comm.rank, ctypes.byref(out)), None, "comm_create")
    _NATIVE_COMMS[key] = out.value
    return out.value


def _sort_sharded_native(x_local, comm, ops, tel, mult: int) -> bool:
    """cafs_sort_i64_sharded: every phase and the three NCCL collectives in one
    graph-replayed enqueue.  False when the column needs the host-driven path
    (every rank agrees; the column is untouched)."""
    from .sorter import _decision_from_c
    ncomm = _native_comm(comm, ops.device)
    status, t = ops.sort_native(x_local, ncomm, mult)
    tel.n = int(t.n)
    tel.decision = _decision_from_c(t.decision, tel.n, "int64" if ops.signed else "uint64")
    if status != 0:
        if tel.decision.route is not Route.MAIN:
            return False
        sizes = [int(v[0]) for v in comm.all_gather_ints([int(x_local.shape[0])])]
        tel.table_buckets = table_size_for(max(1.0, tel.decision.estimate.k_hat), tel.n, 4)
        _main_exchange(x_local, comm, ops, tel, ops.shard_local_pairs(), sizes, tel.decision)
        tel.sharded_path = "native+host"  # counted natively, merged on the host-driven path
        return True
    tel.sharded_path = "native"
    tel.counted_total = int(t.counted_total)
    tel.pairs = int(t.pairs)
    tel.tiny_count_failed = bool(t.tiny_count_failed)  # re-entered MAIN inside the call
    if tel.decision.route is Route.MAIN:
        tel.table_buckets = table_size_for(max(1.0, tel.decision.estimate.k_hat), tel.n, 4)
    return True


def _sort_sharded_native32(x_local, group, mult: int, telemetry) -> bool:
    """A 4-byte shard through cafs_sort_i32_sharded.  False (column untouched,
    every rank agrees) when the column needs the host-driven continuation; the
    caller then sorts it through the widened int64 copy."""
    from .sorter import _decision_from_c
    torch = _torch()
    dev = x_local.device.index if x_local.device.index is not None else torch.cuda.current_device()
    signed = x_local.dtype == torch.int32
    ops = _device_ops(dev, signed)
    comm = _comm(group, x_local.device)
    if comm.device is None:
        return False
    k0 = ops.kernel_count()
    status, t = ops.sort_native(x_local, _native_comm(comm, ops.device), mult)
    if status != 0:
        return False
    tel = telemetry if telemetry is not None else SortTelemetry()
    tel.n = int(t.n)
    tel.decision = _decision_from_c(t.decision, tel.n, "int32" if signed else "uint32")
    tel.sharded_path = "native"
    tel.counted_total = int(t.counted_total)
    tel.pairs = int(t.pairs)
    tel.tiny_count_failed = bool(t.tiny_count_failed)
    if tel.decision.route is Route.MAIN:
        # the reference's table for 4-byte keys has 8-slot buckets (buckets.py:33-43)
        tel.table_buckets = table_size_for(max(1.0, tel.decision.estimate.k_hat), tel.n, 8)
    tel.kernels_launched = ops.kernel_count() - k0
    return True


_SHARD_BUFS: dict = {}


def _shard_buffers(dev, world: int, cap: int):
    """The stream-ordered path's exchange buffers, allocated once per (device,
    world size, stream): header, gathered headers, samples, tiny counters, the
    send row and the gathered rows.  Every phase fully rewrites what it reads
    next, and calls on one stream are ordered, so reuse across them is safe."""
    torch = _torch()
    key = (str(dev), world, cap, torch.cuda.current_stream(dev).cuda_stream)
    bufs = _SHARD_BUFS.get(key)
    if bufs is None:
        i64 = torch.int64
        bufs = (torch.empty(8, dtype=i64, device=dev),
                torch.empty(world * 8, dtype=i64, device=dev),
                torch.empty(SAMPLE_TARGET, dtype=i64, device=dev),
                torch.empty(32, dtype=i64, device=dev),
                torch.empty(1 + 2 * cap, dtype=i64, device=dev),
                torch.empty(world * (1 + 2 * cap), dtype=i64, device=dev))
        _SHARD_BUFS[key] = bufs
    return bufs


def _sort_sharded_streamed(x_local, comm, ops, tel, mult: int) -> bool:
    """The stream-ordered path: four local phases (cafs_shard_*) around four
    stream-ordered collectives, the decisions taken on device, one host sync.
    False when the column needs the host-driven path (every rank agrees)."""
    torch = _torch()
    from .sorter import _decision_from_c
    dev = x_local.device
    world, rank = comm.world, comm.rank
    cap = SHARD_PAIR_CAP
    hdr, hdr_all, samples, tiny, send, recv = _shard_buffers(dev, world, cap)
    ops.shard_begin(x_local, hdr)
    comm.all_gather_into(hdr_all, hdr)
    ops.shard_sample(x_local, hdr_all, world, rank, samples)
    comm.all_reduce_inplace(samples)
    ops.shard_count(x_local, mult, hdr_all, world, samples, tiny, send, cap)
    comm.all_reduce_inplace(tiny)
    comm.all_gather_into(recv, send)
    status, t = ops.shard_finish(x_local, tiny, recv, world, cap)
    tel.n = int(t.n)
    tel.decision = _decision_from_c(t.decision, tel.n, "int64" if ops.signed else "uint64")
    if status != 0:
        if tel.decision.route is not Route.MAIN:
            return False  # fallback routes and tiny misses: the host-driven path
        # too many pairs for the device merge: continue from this shard's
        # pairs (the count is not repeated)
        sizes = [int(v) for v in hdr_all.view(world, 8)[:, 0].cpu().tolist()]
        tel.table_buckets = table_size_for(max(1.0, tel.decision.estimate.k_hat), tel.n, 4)
        _main_exchange(x_local, comm, ops, tel, ops.shard_local_pairs(), sizes, tel.decision)
        tel.sharded_path = "native+host"  # counted natively, merged on the host-driven path
        return True
    tel.sharded_path = "native"
    tel.counted_total = int(t.counted_total)
    tel.pairs = int(t.pairs)
    if tel.decision.route is Route.MAIN:
        tel.table_buckets = table_size_for(max(1.0, tel.decision.estimate.k_hat), tel.n, 4)
    return True


def _sort_sharded(x_local, comm, ops, tel, mult: int, signed: bool) -> None:
    """Four collectives on the MAIN route (header, samples, pair sizes, pairs)."""
    torch = _torch()
    flip = _SIGN if signed else 0
    m64 = (1 << 64) - 1

    # ---- one header all-gather: shard size, local monotone, first/last key ----
    n_local = int(x_local.shape[0])
    mono = ops.is_monotone(x_local) if n_local > 1 else True
    first = last = 0
    if n_local:
        fl = torch.stack([x_local[0], x_local[-1]]).cpu().numpy()  # one D2H
        first, last = ((int(v) & m64) ^ flip for v in fl)
    hdr = comm.all_gather_ints([n_local, int(mono), first, last])
    sizes = [int(h[0]) for h in hdr]
    N = int(sum(sizes))
    off = int(sum(sizes[:comm.rank]))
    tel.n = N
    if N <= 1:
        tel.decision = DispatchDecision(Route.ALREADY_SORTED)
        return

    # ---- monotone (sorter.py:115-129): every shard sorted, boundaries ordered ----
    g_mono = all(h[1] for h in hdr)
    prev = None
    for n_r, _, f_, l_ in hdr:
        if n_r:
            if prev is not None and f_ < prev:
                g_mono = False
            prev = l_
    if g_mono:
        tel.decision = DispatchDecision(Route.ALREADY_SORTED)
        return

    def _fallback(route_decision: DispatchDecision, guard: bool = False):
        tel.decision = route_decision
        tel.guard_fired = guard
        if N < SMALL_N_CUTOFF:  # a few KB: gather and sort everywhere
            full = comm.all_gather_var(x_local, sizes)
            ops.fallback_sort(full)
            x_local.copy_(full[off:off + n_local])
            return
        _exchange_sort(x_local, sizes, comm, ops)

    if N < SMALL_N_CUTOFF:
        _fallback(DispatchDecision(Route.FALLBACK_SMALL_N))
        return

    # ---- strided samples (cardinality.py:99-110): each rank fills the global
    # positions in its shard, one all-reduce assembles all 1024 ----
    stride = N // SAMPLE_TARGET
    lo = (off + stride - 1) // stride
    hi = min(SAMPLE_TARGET, (off + n_local + stride - 1) // stride)
    buf = torch.zeros(SAMPLE_TARGET, dtype=x_local.dtype, device=x_local.device)
    if hi > lo:
        pos = torch.arange(lo, hi, device=x_local.device, dtype=torch.int64) * stride - off
        buf[lo:hi] = x_local.index_select(0, pos)
    samples = comm.all_reduce_tensor(buf)
    u, f1, f2, saturated, keys = ops.estimate(samples)
    k_hat = chao1(u, f1, f2, N, saturated)
    est = CardinalityEstimate(k_hat, u, f1, f2, saturated)

    if k_hat <= TINY_MAX_KEYS and u <= TINY_MAX_KEYS:
        # ---- TINY (sorter.py:367-385) ----
        cnt = ops.tiny_counts(x_local, keys)
        tot = comm.all_reduce_sum(cnt)
        if int(tot.sum()) == N:
            tel.decision = DispatchDecision(Route.TINY_COUNT, keys=np.array(keys, np.uint64),
                                            estimate=est)
            kt, ct = ops.keys_tensor(keys, tot)
            ops.emit_slice(kt, ct, x_local, off, off + n_local, N)
            tel.counted_total = N
            tel.pairs = len(keys)
            return
        tel.tiny_count_failed = True
    elif k_hat * 2 > N:
        _fallback(DispatchDecision(Route.FALLBACK_HIGH_ENTROPY, estimate=est))
        return

    # ---- MAIN: local count, all-gather of pair tables, merge, slice emit ----
    decision = DispatchDecision(Route.MAIN, k_hat=k_hat, estimate=est)
    tel.table_buckets = table_size_for(max(1.0, k_hat), N, 4)
    _main_exchange(x_local, comm, ops, tel, ops.count_pairs(x_local, mult), sizes, decision)


def _main_exchange(x_local, comm, ops, tel, pairs, sizes: list[int], decision) -> None:
    """MAIN after the local count: all-gather of the pair tables, merge, slice
    emit; `pairs` None = this shard's table overflowed (the guard)."""
    N = int(sum(sizes))
    off = int(sum(sizes[:comm.rank]))
    n_local = int(x_local.shape[0])
    meta = comm.all_gather_ints([int(pairs is None), 0 if pairs is None else int(pairs[0].shape[0])])
    merged = None
    if not any(m[0] for m in meta):
        counts = [int(m[1]) for m in meta]
        keys_all, cnts_all = comm.all_gather_pairs(pairs[0], pairs[1], counts)
        # every rank merges the same tables: the overflow outcome is the same everywhere
        merged = ops.merge_pairs(keys_all, cnts_all)
    if merged is None:  # the guard: the distributed fallback (sorter.py:264-273)
        tel.decision = decision
        tel.guard_fired = True
        _exchange_sort(x_local, sizes, comm, ops)
        return
    tel.decision = decision
    ops.emit_slice(merged[0], merged[1], x_local, off, off + n_local, N)
    tel.counted_total = N
    tel.pairs = int(merged[0].shape[0])
