"""Host-side counting structures of the reference API (not on the device path).

The reference package exports its scalar counting cell, bucket table and
sampling multiset (``cafs/__init__.py:12-54``); callers use them to inspect or
re-run the reference semantics on small inputs.  The B200 pipeline never builds
these structures (the device counts with its own shared/global tables,
csrc/hashcount.cu), so they are provided here with the reference's semantics,
in numpy, for API completeness:

* :class:`Bucket` / :func:`bucket_update` -- one cache-line counting record and
  its update rule (buckets.py:108-149): the lowest slot holding the value (a
  zero key matches an empty slot) gains the increment, else the lowest empty
  slot is claimed, else the update is rejected;
* :class:`BucketTable` -- ``2**m_log2`` buckets plus the raw spill buffer
  (buckets.py:172-292), with ``update`` / ``count_sequence`` (run-folded) /
  ``update_many`` / ``occupied_pairs`` / ``counted_total`` and the
  :class:`~.sorter.TableStats` counters;
* :class:`FreqSet` -- the 4096-slot sample multiset of the cardinality
  estimator (cardinality.py:31-73); the device estimator computes the same
  (u, f1, f2) without it (the spectrum does not depend on the hash).
"""

from __future__ import annotations

import numpy as np

from .sorter import FREQSET_SLOTS, TableStats, check_hash_mult, fast_hash

_SLOTS_BY_WIDTH = {8: 4, 4: 8}  # keys per 64-byte bucket (buckets.py:33-43)


def bucket_cap(dtype) -> int:
    w = np.dtype(dtype).itemsize
    if w not in _SLOTS_BY_WIDTH:
        raise ValueError(f"unsupported key width: {w * 8} bits")
    return _SLOTS_BY_WIDTH[w]


class Bucket:
    """Parallel key / counter slots of one bucket (views into a table row)."""

    __slots__ = ("keys", "counts")

    def __init__(self, keys: np.ndarray, counts: np.ndarray):
        self.keys = keys
        self.counts = counts

    @classmethod
    def empty(cls, dtype=np.uint64) -> "Bucket":
        c = bucket_cap(dtype)
        return cls(np.zeros(c, dtype=dtype), np.zeros(c, dtype=np.uint32))

    @property
    def cap(self) -> int:
        return int(self.keys.shape[0])

    def occupied(self) -> int:
        return int(np.count_nonzero(self.counts))


def bucket_update(bucket: Bucket, val: int, inc: int = 1) -> bool:
    """Apply one (val, inc) update to `bucket`; False = full (the caller spills)."""
    if inc < 1:
        raise ValueError("inc must be >= 1")
    v = int(val)
    hit = np.flatnonzero(bucket.keys.astype(object) == v) if bucket.cap else []
    if len(hit):
        bucket.counts[hit[0]] += np.uint32(inc)
        return True
    free = np.flatnonzero(bucket.counts == 0)
    if len(free):
        j = free[0]
        bucket.keys[j] = v
        bucket.counts[j] = np.uint32(inc)
        return True
    return False


class BucketTable:
    """The reference's fixed-capacity counting table, on the host."""

    def __init__(self, m_log2: int, dtype=np.uint64, hash_mult=None):
        if m_log2 < 3:
            raise ValueError("table needs at least 8 buckets (m_log2 >= 3)")
        self.m_log2 = int(m_log2)
        self.dtype = np.dtype(dtype)
        self.hash_mult = check_hash_mult(hash_mult)
        c = bucket_cap(self.dtype)
        self.keys = np.zeros((1 << self.m_log2, c), dtype=self.dtype)
        self.counts = np.zeros((1 << self.m_log2, c), dtype=np.uint32)
        self.stats = TableStats()
        self._spill: list[np.ndarray] = []

    @property
    def n_buckets(self) -> int:
        return int(self.keys.shape[0])

    @property
    def cap(self) -> int:
        return int(self.keys.shape[1])

    @property
    def spill_len(self) -> int:
        return self.stats.spill_len

    def bucket(self, i: int) -> Bucket:
        return Bucket(self.keys[i], self.counts[i])

    def update(self, val: int, inc: int = 1) -> None:
        b = self.bucket(fast_hash(int(val), self.m_log2, self.hash_mult))
        present = bool(np.any((b.keys.astype(object) == int(val)) & (b.counts > 0)))
        if bucket_update(b, val, inc):
            if present:
                self.stats.hits += 1
            else:
                self.stats.claims += 1
        else:
            self._spill.append(np.full(inc, val, dtype=self.dtype))
            self.stats.spill_pushes += 1
            self.stats.spill_len += inc
        self.stats.updates += 1

    def count_sequence(self, x: np.ndarray) -> None:
        """One update per maximal run of equal adjacent values."""
        if x.dtype != self.dtype:
            raise ValueError(f"expected {self.dtype} values, got {x.dtype}")
        if not x.size:
            return
        starts = np.flatnonzero(np.concatenate(([True], x[1:] != x[:-1])))
        lens = np.diff(np.append(starts, x.shape[0]))
        for s, ln in zip(starts.tolist(), lens.tolist()):
            self.update(int(x[s]), ln)

    def update_many(self, vals: np.ndarray, lens: np.ndarray | None = None) -> None:
        if vals.dtype != self.dtype:
            raise ValueError(f"expected {self.dtype} values, got {vals.dtype}")
        if lens is None:
            lens = np.ones(vals.shape[0], dtype=np.int64)
        elif np.any(np.asarray(lens) < 1):
            raise ValueError("inc must be >= 1")
        for v, ln in zip(vals.tolist(), np.asarray(lens).tolist()):
            self.update(int(v), int(ln))

    @property
    def spill(self) -> np.ndarray:
        """Spilled raw keys in push order."""
        if not self._spill:
            return np.empty(0, dtype=self.dtype)
        if len(self._spill) > 1:
            self._spill = [np.concatenate(self._spill)]
        return self._spill[0]

    def occupied_pairs(self) -> tuple[np.ndarray, np.ndarray]:
        m = self.counts > 0
        return self.keys[m].astype(np.uint64, copy=False), self.counts[m].astype(np.int64)

    def counted_total(self) -> int:
        return int(self.counts.sum(dtype=np.int64))


class FreqSet:
    """4096-slot linear-probing multiset of sampled keys (load <= 1/4)."""

    __slots__ = ("keys", "counters", "occupied", "hash_mult")

    def __init__(self, hash_mult=None):
        self.keys = np.zeros(FREQSET_SLOTS, dtype=np.uint64)
        self.counters = np.zeros(FREQSET_SLOTS, dtype=np.uint32)
        self.occupied = 0
        self.hash_mult = check_hash_mult(hash_mult)

    def insert(self, key: int) -> None:
        k = int(key) & ((1 << 64) - 1)
        j = fast_hash(k, 12, self.hash_mult)
        while self.counters[j] != 0 and int(self.keys[j]) != k:
            j = (j + 1) & (FREQSET_SLOTS - 1)
        if self.counters[j] == 0:
            self.keys[j] = k
            self.occupied += 1
        self.counters[j] += np.uint32(1)

    def spectrum(self) -> tuple[int, int, int]:
        c = self.counters
        return int(np.count_nonzero(c)), int(np.count_nonzero(c == 1)), int(np.count_nonzero(c == 2))

    def distinct_keys(self) -> np.ndarray:
        return np.sort(self.keys[self.counters > 0])
