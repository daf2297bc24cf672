"""B200-native CAFS: cardinality-aware frequency sort on sm_100a.

Drop-in for the reference package's sort path (``cafs``, arxiv 2605.25040):
the same entry point ``cafs_sort(x, telemetry=None, hash_mult=None)``, the same
dispatcher routes and result types, executed by hand-written CUDA kernels in
``libcafs_b200.so`` (C ABI: ``include/cafs_b200.h``).  Row-sharded multi-GPU
sorting over torch.distributed/NCCL lives in :mod:`.sharded`.
"""

from .sorter import (
    FREQSET_SLOTS,
    HASH_MULT,
    PAIR_RADIX_MIN,
    SAMPLE_TARGET,
    SMALL_N_CUTOFF,
    SUPPORTED_DTYPES,
    TINY_MAX_KEYS,
    CardinalityEstimate,
    DispatchDecision,
    PairList,
    Route,
    SortTelemetry,
    TableStats,
    TableSummary,
    cafs_sort,
    chao1,
    check_hash_mult,
    dispatch,
    emit,
    fallback_sort,
    fast_hash,
    is_monotone,
    pair_sort,
    sample_and_estimate,
    table_size_for,
    tiny_count_sort,
    tiny_counts,
)

from .tables import Bucket, BucketTable, FreqSet, bucket_update

__version__ = "0.1.0"

__all__ = [
    "Bucket", "BucketTable", "FreqSet", "TableStats", "bucket_update",
    "CardinalityEstimate", "DispatchDecision", "PairList", "Route", "SortTelemetry", "TableSummary",
    "cafs_sort", "chao1", "check_hash_mult", "dispatch", "emit", "fallback_sort", "fast_hash",
    "is_monotone", "pair_sort", "sample_and_estimate", "table_size_for", "tiny_count_sort",
    "tiny_counts", "FREQSET_SLOTS", "HASH_MULT", "PAIR_RADIX_MIN", "SAMPLE_TARGET",
    "SMALL_N_CUTOFF", "SUPPORTED_DTYPES", "TINY_MAX_KEYS", "__version__",
]
