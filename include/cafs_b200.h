/*
 * cafs_b200.h -- C ABI of libcafs_b200.so, the B200 (sm_100a) CAFS sort.
 *
 * Plain pointers, sizes and status codes; no torch or CUDA types in the
 * signatures (streams travel as `void*` = cudaStream_t).  Every call is
 * stream-ordered on the given stream and thread-safe: calls on distinct contexts run
 * concurrently; calls sharing a context are serialised (a per-context lock, and a
 * call on a different stream than the previous one first waits for that stream).
 *
 * Each entry point replaces one interface of the reference package
 * (paths relative to /root/reference/pkg/src/cafs):
 *
 *   cafs_sort_i64            sorter.py:335-386   cafs_sort(x, telemetry, hash_mult)
 *   cafs_sort_i64_host       sorter.py:335-386   same call on host (numpy) buffers
 *   cafs_dispatch_i64        sorter.py:141-162   dispatch(x, n, hash_mult)
 *   cafs_estimate_i64        cardinality.py:113-125  sample_and_estimate(x, n, hash_mult)
 *                            (+ _kernels.py:131-153 freqset_insert_many, cardinality.py:63-69)
 *   cafs_is_monotone_i64     sorter.py:115-129   is_monotone(x)
 *   cafs_tiny_counts_i64     _kernels.py:156-169 tiny_counts(x, keys)
 *   cafs_count_pairs_i64     sorter.py:183-196 + 254-288  main_count_loop -> reconstruct's
 *                            sorted (key, count) pairs (count_sequence _kernels.py:25-81,
 *                            fold_sorted :219-225, pair_sort :228-241)
 *   cafs_merge_pairs         sorter.py:276-285   spill fold + union of pair lists (sharded merge)
 *   cafs_pair_sort           _kernels.py:185-214 radix_sort_pairs / sorter.py:228-241 pair_sort
 *   cafs_emit_i64            sorter.py:244-251 + _kernels.py:172-182  emit / emit_fill
 *   cafs_fallback_sort_i64   sorter.py:132-138   fallback_sort(x)
 *   cafs_sort_i32(_host)     sorter.py:335-386   cafs_sort on int32 / uint32 arrays
 *   cafs_key_span_i64,       (no reference counterpart: the distributed
 *   cafs_partition_i64        fallback of SURVEY.md §8(f)2, sharded.py)
 *   cafs_shard_*_i64,        (no reference counterpart: the reference is single-process,
 *   cafs_sort_i64_sharded,    PAPER.md:714 names a parallel CAFS as future work) the
 *   cafs_comm_create          row-sharded multi-GPU sort of SURVEY.md §8(e); the native
 *                             call runs its collectives on the library's NCCL communicator
 *
 * Keys are 64-bit.  `is_signed` = 1 for int64 (order-mapped by flipping bit 63,
 * sorter.py:84-94, folded into the kernels' loads/stores), 0 for uint64.
 * Errors: the reference raises TypeError/ValueError from Python; here the same
 * conditions return CAFS_EINVAL and the Python layer raises the reference's
 * exception type.
 */
#ifndef CAFS_B200_H
#define CAFS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CAFS_ABI_VERSION 2
#define CAFS_TINY_MAX_KEYS 8      /* sorter.py:30  TINY_MAX_KEYS */
#define CAFS_SMALL_N_CUTOFF 2048  /* sorter.py:29  SMALL_N_CUTOFF */
#define CAFS_SAMPLE_TARGET 1024   /* cardinality.py:26 */
#define CAFS_DEFAULT_HASH_MULT 0x9E3779B97F4A7C15ull /* buckets.py:30 */

/* cafs.sorter.Route (sorter.py:44-49), same order */
typedef enum {
  CAFS_ALREADY_SORTED = 0,
  CAFS_FALLBACK_SMALL_N = 1,
  CAFS_TINY_COUNT = 2,
  CAFS_FALLBACK_HIGH_ENTROPY = 3,
  CAFS_MAIN = 4
} cafs_route_t;

typedef enum {
  CAFS_OK = 0,
  CAFS_EINVAL = -1,    /* bad argument (reference: ValueError/TypeError) */
  CAFS_ECUDA = -2,     /* CUDA runtime error */
  CAFS_ENOMEM = -3,    /* device allocation failed */
  CAFS_ESUM = -4,      /* pair counts do not sum to n (reference emit ValueError) */
  CAFS_EINTERNAL = -5
} cafs_status_t;

/* cafs.cardinality.CardinalityEstimate (cardinality.py:76-82) + the sampled
 * distinct keys (FreqSet.distinct_keys, ascending, unsigned domain) when u <= 8 */
typedef struct {
  double k_hat;
  int64_t u, f1, f2;
  int32_t saturated;
  int32_t nkeys;
  uint64_t keys[CAFS_TINY_MAX_KEYS];
} cafs_estimate_t;

/* cafs.sorter.DispatchDecision (sorter.py:52-57) */
typedef struct {
  int32_t route;
  int32_t has_estimate;
  cafs_estimate_t est;
} cafs_decision_t;

/* Stage indices of cafs_telemetry_t.stage_ms (sorter.py:64-66 labels) */
enum { CAFS_STAGE_COUNT = 0, CAFS_STAGE_SORT_K = 1, CAFS_STAGE_EMIT = 2 };
/* Kernel indices of cafs_telemetry_t.kernel_ms (single-kernel CUDA-event times) */
enum { CAFS_KERNEL_COUNT = 0, CAFS_KERNEL_EMIT = 1, CAFS_KERNEL_ESTIMATE = 2 };

/* cafs.sorter.SortTelemetry (sorter.py:60-81).  stage_ms[i] < 0: stage not run. */
typedef struct {
  uint64_t n;
  cafs_decision_t decision;      /* final decision (MAIN after a tiny-count failure) */
  int32_t tiny_count_failed;
  int32_t guard_fired;           /* device guard: global table overflow -> fallback */
  uint64_t counted_total;        /* elements counted into (key, count) pairs */
  uint64_t pairs;                /* distinct keys emitted (K') */
  uint64_t table_buckets;        /* reference table_size_for(max(1,k_hat), n, 4) on MAIN */
  uint64_t global_updates;       /* device: elements resolved in the L2 global table */
  float stage_ms[3];
  float kernel_ms[4];            /* count kernel (hash or tiny), emit kernel, estimate kernel */
  uint32_t kernels_launched;     /* kernels this call put on the stream */
  /* CAFS_FLAG_EXACT_TELEMETRY: the reference bucket table's statistics
   * (buckets.py:152-169, sorter.py:326-331), computed exactly on device */
  int32_t exact;                 /* 1 when the ref_* fields are valid */
  int32_t ref_guard_fired;       /* 2 * ref_spill_len > n (sorter.py:264) */
  uint64_t ref_spill_len, ref_updates, ref_hits, ref_claims, ref_spill_pushes;
  uint64_t ref_counted_total;
  int32_t count_path;            /* cafs_count_path_t: how the column was counted */
  int32_t _reserved;
} cafs_telemetry_t;

/* cafs_telemetry_t.count_path (B200-side; the reference has one bucket table) */
typedef enum {
  CAFS_COUNT_NONE = 0,         /* no count: sorted input or a fallback route */
  CAFS_COUNT_TINY = 1,         /* tiny route: <= 8 sampled keys, one pass */
  CAFS_COUNT_DENSE = 2,        /* main route: dense key window (dictionary codes) */
  CAFS_COUNT_TABLE = 3,        /* main route: CTA tables + the global (L2) hash table */
  CAFS_COUNT_PARTITIONED = 4   /* main route: CTA tables + key-range partitions (hashpart.cu) */
} cafs_count_path_t;

typedef struct cafs_ctx cafs_ctx_t;

/* Context: per-device persistent state (control block, the L2-resident global
 * (key, count) table, pair buffers).  One context per device and stream user. */
int cafs_ctx_create(int device, cafs_ctx_t** out);
void cafs_ctx_destroy(cafs_ctx_t* ctx);
int cafs_abi_version(void);
const char* cafs_status_string(int status);
const char* cafs_last_error(cafs_ctx_t* ctx);

/* Flags for cafs_sort_i64 */
#define CAFS_FLAG_TIMING 1u      /* fill stage_ms with CUDA-event timings */
#define CAFS_FLAG_NO_DIRECT 2u   /* disable the dense-range direct-count path */
#define CAFS_FLAG_EXACT_TELEMETRY 4u  /* compute the reference's bucket-table statistics */
#define CAFS_FLAG_DOM_I32 8u     /* keys are widened int32 (reference domain: u32, cap 8) */
#define CAFS_FLAG_DOM_U32 16u    /* keys are widened uint32 */

/* cafs_sort(x) in place on device memory (sorter.py:335-386).  n < 2^32. */
int cafs_sort_i64(cafs_ctx_t* ctx, int64_t* d_x, uint64_t n, int is_signed,
                  uint64_t hash_mult, uint32_t flags, cafs_telemetry_t* tel, void* stream);

/* Same on host memory: h_in -> device -> sort -> h_out (h_out may equal h_in).
 * Page-locked buffers give full PCIe bandwidth; pageable ones work too. */
int cafs_sort_i64_host(cafs_ctx_t* ctx, const int64_t* h_in, int64_t* h_out, uint64_t n,
                       int is_signed, uint64_t hash_mult, uint32_t flags,
                       cafs_telemetry_t* tel, void* stream);

/* cafs_sort for 4-byte keys (SUPPORTED_DTYPES int32 / uint32, sorter.py:34):
 * is_signed = 1 for int32 (the reference's order map flips bit 31,
 * sorter.py:84-94), 0 for uint32.  Same routes, estimate and telemetry as the
 * int64 widening of the column (keys are widened in registers), but the count
 * reads and the emit writes 4 B per key.  d_x must be 4-byte aligned. */
int cafs_sort_i32(cafs_ctx_t* ctx, int32_t* d_x, uint64_t n, int is_signed, uint64_t hash_mult,
                  uint32_t flags, cafs_telemetry_t* tel, void* stream);
int cafs_sort_i32_host(cafs_ctx_t* ctx, const int32_t* h_in, int32_t* h_out, uint64_t n,
                       int is_signed, uint64_t hash_mult, uint32_t flags,
                       cafs_telemetry_t* tel, void* stream);

/* dispatch(x) -> decision (sorter.py:141-162); requires n >= 2 */
int cafs_dispatch_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                      uint64_t hash_mult, cafs_decision_t* out, void* stream);

/* sample_and_estimate(x, n) (cardinality.py:113-125); n >= 1 */
int cafs_estimate_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                      cafs_estimate_t* out, void* stream);

/* is_monotone(x) (sorter.py:115-129) */
int cafs_is_monotone_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         int* out, void* stream);

/* tiny_counts(x, keys) (_kernels.py:156-169): keys in the unsigned domain, distinct,
 * nk <= 8; h_counts[j] = #{i : x_u[i] == keys[j]} */
int cafs_tiny_counts_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         const uint64_t* h_keys, int nk, int64_t* h_counts, void* stream);

/* Count x into distinct (key, count) pairs sorted by unsigned key (the count +
 * reconstruct stages of the main route).  d_keys/d_counts hold `cap` entries;
 * *h_npairs receives K'.  Returns CAFS_EINVAL if K' > cap. */
int cafs_count_pairs_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         uint64_t hash_mult, uint64_t* d_keys, uint64_t* d_counts,
                         uint64_t cap, uint64_t* h_npairs, void* stream);

/* Merge (key, count) pairs whose keys may repeat (e.g. the all-gathered tables
 * of a sharded sort) into distinct pairs sorted by key with summed counts --
 * the union + fold of reconstruct (sorter.py:276-285) across shards. */
int cafs_merge_pairs(cafs_ctx_t* ctx, const uint64_t* d_keys_in, const uint64_t* d_counts_in,
                     uint64_t m, uint64_t* d_keys, uint64_t* d_counts, uint64_t cap,
                     uint64_t* h_npairs, void* stream);

/* pair_sort: sort (key, count) pairs by unsigned key in place (keys distinct) */
int cafs_pair_sort(cafs_ctx_t* ctx, uint64_t* d_keys, uint64_t* d_counts, uint64_t npairs,
                   void* stream);

/* emit: expand sorted pairs into out[0 .. sum(counts)) restricted to the output
 * slice [out_begin, out_end) of the global sorted order (whole array:
 * 0 .. total); d_out receives out_end - out_begin keys.  Keys are unsigned-domain;
 * is_signed un-flips them on store.  Sum check as sorter.py:247-248. */
int cafs_emit_i64(cafs_ctx_t* ctx, const uint64_t* d_keys, const uint64_t* d_counts,
                  uint64_t npairs, int64_t* d_out, uint64_t out_begin, uint64_t out_end,
                  uint64_t total, int is_signed, void* stream);

/* fallback_sort(x): on-device LSD radix sort (sorter.py:132-138 replaced) */
int cafs_fallback_sort_i64(cafs_ctx_t* ctx, int64_t* d_x, uint64_t n, int is_signed,
                           void* stream);

/* ---- distributed fallback (sharded high-entropy / guard routes) ----
 * The reference is single-process; its fallback_sort (sorter.py:132-138) is
 * what a multi-GPU caller replaces with: global span -> one bucket digit ->
 * local partition -> all-to-all of bucket ranges -> local sort of the received
 * range.  These two calls are the local steps. */
/* min and max of the order-mapped keys (h_min = ~0, h_max = 0 when n == 0) */
int cafs_key_span_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                      uint64_t* h_min, uint64_t* h_max, void* stream);
/* Group x into 4096 buckets by ((k - g_min) >> shift), the shift fitting the
 * GLOBAL span [g_min, g_max] of order-mapped keys into 12 bits:
 * d_out[0..n) = the keys (same representation as x) in ascending bucket
 * order, h_counts[4096] = keys per bucket. */
#define CAFS_PARTITION_BUCKETS 4096
int cafs_partition_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                       uint64_t g_min, uint64_t g_max, int64_t* d_out, uint64_t* h_counts,
                       void* stream);

/* The exchange plan of the distributed fallback, from every rank's bucket
 * counts (counts[r * 4096 + b], all-gathered): rank `rank` sends rows
 * [send_at[d], send_at[d] + send_n[d]) of its partitioned shard to rank d,
 * receives recv_n[s] rows from rank s (stored in rank order), sorts what it
 * received and keeps rows [*start, *start + its row count).  Pure host
 * arithmetic (sharded.py bucket_ranges / _exchange_sort); the native sharded
 * sort calls it between its two collectives. */
int cafs_shard_fallback_plan(int world, int rank, const uint32_t* counts, uint64_t* send_at,
                             uint64_t* send_n, uint64_t* recv_n, uint64_t* start);

/* ---- stream-ordered sharded sort (one process per GPU, row shards) ----
 * The host-driven sharded path (sharded.py) synchronises between every
 * collective; these four calls enqueue the local phases on `stream` with the
 * decisions taken on device, so a rank synchronises once (in finish).  The
 * caller runs the collectives in between (NCCL, stream-ordered):
 *   begin(x) -> d_hdr[8]                       all-gather -> d_hdr_all[world*8]
 *   sample(x, d_hdr_all) -> d_samples[1024]    all-reduce SUM
 *   count(x, d_samples) -> d_tiny[32], d_send[1+2*cap]
 *                      all-reduce SUM d_tiny; all-gather d_send -> d_recv
 *   finish(x, d_tiny, d_recv) -> x = this rank's rows of the sorted column
 * *h_status = 0: done (route and estimate in tel); 1: this column needs the
 * host-driven path (fallback routes, tiny miss, table overflow, more than
 * cap pairs on a rank or 8192 merged) -- every rank returns the same status.
 * int64 / uint64 only.  The dispatch is sorter.py:141-162 on the global
 * column. */
#define CAFS_SHARD_HDR_WORDS 8
#define CAFS_SHARD_TINY_WORDS 32
int cafs_shard_begin_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         uint64_t* d_hdr, void* stream);
int cafs_shard_sample_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                          const uint64_t* d_hdr_all, int world, int rank, uint64_t* d_samples,
                          void* stream);
int cafs_shard_count_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         uint64_t hash_mult, const uint64_t* d_hdr_all, int world,
                         const uint64_t* d_samples, uint64_t* d_tiny, uint64_t* d_send,
                         uint64_t cap, void* stream);
int cafs_shard_finish_i64(cafs_ctx_t* ctx, int64_t* d_x, uint64_t n, int is_signed,
                          const uint64_t* d_tiny_sum, const uint64_t* d_recv, int world,
                          uint64_t cap, cafs_telemetry_t* tel, int* h_status, void* stream);

/* ---- native multi-GPU sort (the library's own NCCL communicator) ----
 * The stream-ordered sharded sort above with the collectives inside the
 * library: cafs_sort_i64_sharded enqueues header -> ncclAllGather -> samples
 * -> ncclAllReduce -> estimate + local count -> ncclAllGather of the pair
 * tables (the tiny counters ride in the same rows) -> merge -> slice emit,
 * captured as one CUDA graph per (column, rows, flags) and replayed, and
 * synchronises once.  Same results and *h_status as cafs_shard_finish_i64
 * (1: the caller continues on the host-driven path; the column is untouched).
 * Replaces the per-phase torch.distributed orchestration of sharded.py for
 * NCCL process groups; the reference has no multi-GPU sort.
 * Communicator setup: rank 0 calls cafs_nccl_unique_id, the caller
 * broadcasts the bytes, every rank calls cafs_comm_create (collective). */
#define CAFS_NCCL_ID_BYTES 128
#define CAFS_SHARD_PAIR_CAP 8192 /* pairs per rank in the exchange (as sharded.py) */
typedef struct cafs_comm_t cafs_comm_t;
int cafs_nccl_unique_id(unsigned char* out /* CAFS_NCCL_ID_BYTES */);
int cafs_comm_create(int device, const unsigned char* id, int world, int rank,
                     cafs_comm_t** out);
int cafs_comm_destroy(cafs_comm_t* comm);
int cafs_sort_i64_sharded(cafs_ctx_t* ctx, cafs_comm_t* comm, int64_t* d_x, uint64_t n,
                          int is_signed, uint64_t hash_mult, cafs_telemetry_t* tel, int* h_status,
                          void* stream);
/* The same for int32 (is_signed = 1) / uint32 (is_signed = 0) shards: 4 bytes
 * per key read and written on every rank (the tables and the exchange hold
 * the keys' 64-bit order-mapped widening, as cafs_sort_i32 does). */
int cafs_sort_i32_sharded(cafs_ctx_t* ctx, cafs_comm_t* comm, int32_t* d_x, uint64_t n,
                          int is_signed, uint64_t hash_mult, cafs_telemetry_t* tel, int* h_status,
                          void* stream);

/* After finish returned status 1 on the main route: this shard's (key, count)
 * pairs from the count phase, for the host-driven merge; *h_npairs = ~0 when
 * they were lost to a table overflow (the guard). */
int cafs_shard_local_pairs_i64(cafs_ctx_t* ctx, uint64_t* d_keys, uint64_t* d_counts,
                               uint64_t cap, uint64_t* h_npairs, void* stream);

/* Kernels this context has launched since it was created (monotone; the
 * per-call count of cafs_sort_i64 is also in cafs_telemetry_t.kernels_launched).
 * No reference counterpart: launch accounting for the multi-GPU bench. */
uint64_t cafs_ctx_kernel_count(const cafs_ctx_t* ctx);

/* ---- synthetic inputs (bench / tests; bit-identical to oracle/gen.py) ---- */
/* out[i] = fmix64(seed + (skip + i + 1) * 0x9E3779B97F4A7C15) */
int cafs_gen_mix(uint64_t* d_out, uint64_t count, uint64_t seed, uint64_t skip, void* stream);
/* rows [start, start+n): out[i] = palette[idx(start+i)], idx uniform (mulhi) or,
 * when d_cdf != NULL, Zipf by searchsorted(cdf, u, 'right'); palette NULL = codes */
int cafs_gen_draw(int64_t* d_out, uint64_t n, uint64_t start, uint64_t seed,
                  const int64_t* d_palette, uint64_t k, const double* d_cdf, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CAFS_B200_H */
