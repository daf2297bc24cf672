// abi.cu -- the C ABI of libcafs_b200.so and the native pipeline orchestrator.
//
// cafs_sort_i64 is the B200 restatement of cafs_sort (sorter.py:335-386):
//
//   n <= 1                        -> ALREADY_SORTED                 (:353-355)
//   K0/K1 estimate kernel         -> route, k_hat, u, f1, f2, keys  (:141-162)
//     prefix sorted and n > 64 Ki -> full monotone scan kernel
//   FALLBACK_SMALL_N / HIGH_ENT.  -> on-device sort (radix.cu)      (:362-366)
//   TINY_COUNT                    -> K2 count, finalize, K5 emit    (:367-377)
//     any miss                    -> MAIN with the same k_hat       (:378-385)
//   MAIN                          -> K3 hash count, compact, K4 pair sort + scan,
//                                    K5 emit; global-table overflow -> guard
//                                    -> fallback sort               (:317-332, :254-293)
//
// Host round trips: one after the estimate kernel (the route decides which
// kernels exist) and one at the end of the call (telemetry, guard).  Every
// stage in between is stream-ordered and gated on the device control block.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

using namespace cafs;

struct cafs_ctx {
  int device = 0;
  int num_sms = 148;
  // calls on one context are serialised: a host lock, and a call on a stream
  // other than the previous call's first waits for that stream (the control
  // block, tables and scratch are per context)
  std::recursive_mutex mu;
  cudaStream_t last_stream = nullptr;
  bool has_last = false;
  DevCtl* d_ctl = nullptr;
  DevCtl* h_ctl = nullptr;  // pinned mirror
  // main route: global table + pair buffers
  u64* gkeys = nullptr;
  u64* gcnt = nullptr;
  u32* glist = nullptr;
  u64* pk_a = nullptr;  // compacted pairs (unsorted)
  u64* pk_t = nullptr;  // MSD bucket buffers of the large pair sort (lazy)
  u32* tile_map = nullptr;  // emit tile -> pair map for large pair sets (lazy)
  u64 tile_map_len = 0;
  u64* pc_t = nullptr;
  u64* pc_a = nullptr;
  u64* pk_b = nullptr;  // sorted pairs
  u64* pc_b = nullptr;
  u64* poffs = nullptr;  // exclusive offsets, npairs + 1
  u64* bsum = nullptr;
  u64* dense = nullptr;  // dense-window counts (zero between calls)
  // radix sort scratch
  u32* ghist = nullptr;  // [8][256]
  u32* gbase = nullptr;  // [8][256]
  int* trivial = nullptr;
  int* h_trivial = nullptr;
  u32* tile_counters = nullptr;  // [8]
  u64* tile_state = nullptr;
  size_t tile_state_words = 0;
  u64* tmp = nullptr;
  size_t tmp_elems = 0;
  void* msd = nullptr;  // MSD bucket-sort state
  // exact-telemetry scratch (telemetry.cu), allocated on first use
  u64* tl_keys = nullptr;
  u32* tl_idx = nullptr;
  u32* tl_first = nullptr;
  u32* tl_runs = nullptr;
  u64* tl_comp = nullptr;   // [4][kPairCap]: comp, cidx, comp2, cidx2
  u64* tl_offs = nullptr;
  void* tl_acc = nullptr;
  u64* stage = nullptr;  // host-path device staging buffer
  size_t stage_elems = 0;
  u32 epoch = 0;
  int32_t* h_scratch = nullptr;  // pinned (64 B + a partition histogram)
  cudaEvent_t ev[32] = {};
  std::string last_error;
  uint64_t launches = 0;  // kernels this context has launched (monotone)
  u64* wide = nullptr;    // int64 copy of a 32-bit column (host-driven fallback routes)
  u64 wide_elems = 0;
  // partitioned count (hashpart.cu): the partitioned spill (n keys) and its scratch
  void* hp_part = nullptr;
  size_t hp_part_bytes = 0;
  void* hp_scratch = nullptr;
  void* hp_mscratch = nullptr;  // the sharded merge's (the local count's stays for a restore)
  // pageable host transfers: per worker thread a stream and two pinned buffers
  cudaStream_t xfer_stream[32] = {};
  cudaEvent_t xfer_event[32][4] = {};
  unsigned char* xfer_buf = nullptr;  // pinned, kXferThreads x 2 x kXferChunk
  // CUDA Graphs of the fused pipeline (estimate + gated route kernels), keyed by
  // the call's arguments; captured on the second call with the same key
  cudaStream_t cap_stream = nullptr;
  struct GraphEntry {
    u64 x = 0, n = 0, flip = 0, mult = 0;
    uint32_t flags = 0;
    int timing = 0;
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
    int tn = 0, mark = 0, label[16] = {}, cond[16] = {};
    uint64_t launches = 0;  // kernels in the captured graph
    uint64_t stamp = 0;
    int kk = 0;             // key kind the graph was captured for
    int exact = 0;          // exact-telemetry calls leave the emit out of the graph
    uint32_t groups = ~0u;  // kernel groups the graph holds (the route the last call took)
  } graphs[16];
  uint64_t graph_clock = 0;
  uint64_t buf_gen = 0;  // bumped when a buffer captured graphs point to is reallocated
};

namespace cafs {
bool pdl_enabled(unsigned which) {  // programmatic dependent launch (common.cuh)
  static const unsigned mask = [] {
    const char* e = getenv("CAFS_PDL");
    // default: not the compaction -- measured on cfg3, its early-launched CTAs
    // cost 45 us (the other kernels gain 2-5 us)
    return e ? (unsigned)strtoul(e, nullptr, 0) : 0x1ffu & ~kPdlCompact;
  }();
  return (mask & which) != 0;
}
}  // namespace cafs

namespace {

// hash-table pairs + the ~0 sentinel pair + dense-window pairs appended after them
constexpr u64 kPairCap = kGlobalCap + 1 + 8192;

int fail(cafs_ctx_t* c, int code, const char* what, cudaError_t e = cudaSuccess) {
  if (c) {
    c->last_error = what;
    if (e != cudaSuccess) {
      c->last_error += ": ";
      c->last_error += cudaGetErrorString(e);
    }
  }
  return code;
}

#define CK(call)                                                              \
  do {                                                                        \
    cudaError_t e_ = (call);                                                  \
    if (e_ != cudaSuccess) return fail(ctx, CAFS_ECUDA, #call, e_);           \
  } while (0)

#define CKL()                                                                 \
  do {                                                                        \
    cudaError_t e_ = cudaGetLastError();                                      \
    if (e_ != cudaSuccess) return fail(ctx, CAFS_ECUDA, "kernel launch", e_); \
  } while (0)

#define TRY(expr)             \
  do {                        \
    int r_ = (expr);          \
    if (r_ != CAFS_OK) return r_; \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// One per entry-point call (see cafs_ctx::mu).
// A stream switch waits (on the host) for the previous stream's work: nothing
// is recorded on the common same-stream path.
struct CallGuard {
  cafs_ctx_t* c;
  cudaStream_t st;
  std::unique_lock<std::recursive_mutex> lk;
  CallGuard(cafs_ctx_t* ctx, void* stream) : c(ctx), st((cudaStream_t)stream), lk(ctx->mu) {
    if (c->has_last && c->last_stream != st) cudaStreamSynchronize(c->last_stream);
  }
  ~CallGuard() {
    c->last_stream = st;
    c->has_last = true;
  }
};

u64 bit_ceil(u64 v) { return v <= 1 ? 1 : 1ull << (64 - __builtin_clzll(v - 1)); }

// buckets.py:92-105 (reported in telemetry; the GPU tables are sized on their own)
u64 table_size_for(double k_hat, u64 n, int cap) {
  u64 m = bit_ceil((u64)std::ceil(8.0 * k_hat / cap));
  u64 m2 = bit_ceil((u64)std::ceil((double)n / cap));
  if (m2 < m) m = m2;
  return m < 8 ? 8 : m;
}

int ensure_main(cafs_ctx_t* ctx) {
  if (ctx->gkeys) return CAFS_OK;
  CK(cudaMalloc(&ctx->gkeys, kGlobalSlots * 8));
  CK(cudaMalloc(&ctx->gcnt, kGlobalSlots * 8));
  CK(cudaMalloc(&ctx->glist, (size_t)kListStripes * kStripeCap * 4));
  CK(cudaMemset(ctx->gkeys, 0xFF, kGlobalSlots * 8));
  CK(cudaMemset(ctx->gcnt, 0, kGlobalSlots * 8));
  CK(cudaMalloc(&ctx->pk_a, kPairCap * 8));
  CK(cudaMalloc(&ctx->pc_a, kPairCap * 8));
  CK(cudaMalloc(&ctx->pk_b, kPairCap * 8));
  CK(cudaMalloc(&ctx->pc_b, kPairCap * 8));
  CK(cudaMalloc(&ctx->poffs, (kPairCap + 1) * 8));
  CK(cudaMalloc(&ctx->bsum, (kPairCap / 8192 + 2) * 8));
  CK(cudaMalloc(&ctx->dense, dense_window_len() * 8));
  CK(cudaMemset(ctx->dense, 0, dense_window_len() * 8));
  return CAFS_OK;
}

// Drop every captured pipeline graph (a buffer they reference was reallocated).
void drop_graphs(cafs_ctx_t* ctx) {
  ++ctx->buf_gen;  // the sharded calls' graphs (per communicator) check it
  for (auto& g : ctx->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g = cafs_ctx_t::GraphEntry();
  }
}

// Columns from this many rows take the partitioned count when the sample shows
// no dense window (smaller ones: the TMA queued shape of hashcount.cu).
constexpr u64 kHpMinRows = 1ull << 20;

bool hp_allowed(u64 n, bool exact) { return !exact && n >= kHpMinRows; }

// The emit's tile -> pair map (emit.cu): one u32 per 8 KB output tile.
int ensure_tile_map(cafs_ctx_t* ctx, u64 n, int kk) {
  const u64 tiles = emit_tiles(n, kk);
  if (tiles > ctx->tile_map_len) {
    CK(cudaDeviceSynchronize());
    if (ctx->tile_map) CK(cudaFree(ctx->tile_map));
    ctx->tile_map = nullptr;
    ctx->tile_map_len = 0;
    drop_graphs(ctx);
    CK(cudaMalloc(&ctx->tile_map, tiles * sizeof(u32)));
    ctx->tile_map_len = tiles;
  }
  return CAFS_OK;
}

int ensure_hp(cafs_ctx_t* ctx, u64 n, int kk) {
  const size_t bytes = (size_t)n * (kk ? 4 : 8) + 64;
  if (bytes > ctx->hp_part_bytes) {
    CK(cudaDeviceSynchronize());
    if (ctx->hp_part) CK(cudaFree(ctx->hp_part));
    ctx->hp_part = nullptr;
    ctx->hp_part_bytes = 0;
    drop_graphs(ctx);
    CK(cudaMalloc(&ctx->hp_part, bytes));
    ctx->hp_part_bytes = bytes;
  }
  if (!ctx->hp_scratch) CK(cudaMalloc(&ctx->hp_scratch, hp_scratch_bytes(ctx->num_sms)));
  return ensure_tile_map(ctx, n, kk);  // the emit's tile -> pair map (hp_place's pairs)
}

HpBufs hp_bufs(cafs_ctx_t* ctx) { return HpBufs{ctx->hp_part, ctx->hp_scratch, ctx->pk_a, ctx->pc_a}; }

int ensure_radix(cafs_ctx_t* ctx, u64 n, bool need_tmp) {
  if (!ctx->ghist) {
    CK(cudaMalloc(&ctx->ghist, 8 * 256 * 4));
    CK(cudaMalloc(&ctx->gbase, 8 * 256 * 4));
    CK(cudaMalloc(&ctx->trivial, 8 * sizeof(int)));
    CK(cudaMallocHost(&ctx->h_trivial, 8 * sizeof(int)));
    CK(cudaMalloc(&ctx->tile_counters, 8 * 4));
  }
  const size_t words = (size_t)onesweep_tiles(n) * 256;
  if (words > ctx->tile_state_words) {
    if (ctx->tile_state) CK(cudaFree(ctx->tile_state));
    ctx->tile_state = nullptr;
    size_t w = words < (size_t)65536 ? (size_t)65536 : words;
    CK(cudaMalloc(&ctx->tile_state, w * 8));
    CK(cudaMemset(ctx->tile_state, 0, w * 8));  // epoch 0 is never used
    ctx->tile_state_words = w;
  }
  if (!ctx->msd) CK(cudaMalloc(&ctx->msd, msd_state_bytes()));
  if (need_tmp && n > ctx->tmp_elems) {
    if (ctx->tmp) CK(cudaFree(ctx->tmp));
    ctx->tmp = nullptr;
    CK(cudaMalloc(&ctx->tmp, n * 8));
    ctx->tmp_elems = n;
  }
  return CAFS_OK;
}

u32 next_epoch(cafs_ctx_t* ctx) {
  ctx->epoch = (ctx->epoch + 1) & 0x3FFFFFFFu;
  if (ctx->epoch == 0) ctx->epoch = 1;
  return ctx->epoch;
}

// LSD radix sort of keys (optionally with a u64 payload) -> result in (k_out, v_out).
// k_in may equal k_out (in place via the ctx temp buffer) for keys-only sorts.
int radix_sort(cafs_ctx_t* ctx, u64* keys, u64* vals, u64* kalt, u64* valt, u64 n, u64 flip,
               cudaStream_t st, u64** result_k, u64** result_v) {
  CK(cudaMemsetAsync(ctx->ghist, 0, 8 * 256 * 4, st));
  CK(cudaMemsetAsync(ctx->tile_counters, 0, 8 * 4, st));
  launch_radix_hist(keys, n, flip, ctx->ghist, ctx->num_sms, st);
  launch_radix_prep(ctx->ghist, n, ctx->gbase, ctx->trivial, st);
  ctx->launches += 2;
  CKL();
  CK(cudaMemcpyAsync(ctx->h_trivial, ctx->trivial, 8 * sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  int passes[8], np = 0;
  for (int p = 0; p < 8; ++p)
    if (!ctx->h_trivial[p]) passes[np++] = p;
  u64 *sk = keys, *sv = vals, *dk = kalt, *dv = valt;
  for (int i = 0; i < np; ++i) {
    const u64 fin = i == 0 ? flip : 0, fout = i == np - 1 ? flip : 0;
    cudaError_t e = launch_onesweep(sk, sv, dk, dv, n, passes[i], fin, fout,
                                    ctx->gbase + passes[i] * 256, ctx->tile_state,
                                    ctx->tile_counters + i, next_epoch(ctx), st);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "onesweep", e);
    ctx->launches++;
    u64* t = sk; sk = dk; dk = t;
    t = sv; sv = dv; dv = t;
  }
  *result_k = sk;
  *result_v = sv;
  return CAFS_OK;
}

int try_msd(cafs_ctx_t* ctx, const u64* keys, const u64* vals, u64 n, u64 flip, u64* tk, u64* tv,
            u64* dk, u64* dv, cudaStream_t st, bool* done);

// More than kSmallSortMax pairs: (pk_a, pc_a) -> (pk_b, pc_b) sorted by key.
// MSD buckets when they fit (pk_b/pc_b double as the bucket buffers, the result
// is copied back), else LSD onesweep.
int sort_pairs_large(cafs_ctx_t* ctx, u64 np, cudaStream_t st) {
  TRY(ensure_radix(ctx, np, false));
  if (!ctx->pk_t) {
    CK(cudaMalloc(&ctx->pk_t, kPairCap * 8));
    CK(cudaMalloc(&ctx->pc_t, kPairCap * 8));
  }
  bool done;
  TRY(try_msd(ctx, ctx->pk_a, ctx->pc_a, np, 0, ctx->pk_t, ctx->pc_t, ctx->pk_b, ctx->pc_b, st,
              &done));
  if (done) return CAFS_OK;
  u64 *rk, *rv;
  TRY(radix_sort(ctx, ctx->pk_a, ctx->pc_a, ctx->pk_b, ctx->pc_b, np, 0, st, &rk, &rv));
  if (rk != ctx->pk_b) {
    CK(cudaMemcpyAsync(ctx->pk_b, rk, np * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->pc_b, rv, np * 8, cudaMemcpyDeviceToDevice, st));
  }
  return CAFS_OK;
}

// The main route's > kSmallSortMax pairs without the host's bucket-size round
// trip: the MSD bucket sorts go out with the largest cap, and a bucket above it
// raises MsdState::overflow, checked after the call's final synchronisation
// (then the pairs are re-sorted by LSD and re-emitted).  *check: such an
// unchecked MSD sort was enqueued.
int sort_pairs_large_unchecked(cafs_ctx_t* ctx, u64 np, cudaStream_t st, bool* check) {
  *check = false;
  TRY(ensure_radix(ctx, np, false));
  if (!ctx->pk_t) {
    CK(cudaMalloc(&ctx->pk_t, kPairCap * 8));
    CK(cudaMalloc(&ctx->pc_t, kPairCap * 8));
  }
  if (!launch_msd_count(ctx->pk_a, np, 0, ctx->msd, ctx->num_sms, st))
    return sort_pairs_large(ctx, np, st);  // too many pairs for MSD buckets: LSD
  launch_msd_sort(ctx->pk_a, ctx->pc_a, np, 0, ctx->msd, ctx->pk_t, ctx->pc_t, ctx->pk_b,
                  ctx->pc_b, msd_bucket_cap(), ctx->num_sms, st);
  ctx->launches += 6;
  CKL();
  *check = true;
  return CAFS_OK;
}

// MSD bucket sort (msd.cu) when every bucket fits a CTA; returns false (nothing
// written) when some bucket is too large, leaving the LSD path to the caller.
int try_msd(cafs_ctx_t* ctx, const u64* keys, const u64* vals, u64 n, u64 flip, u64* tk, u64* tv,
            u64* dk, u64* dv, cudaStream_t st, bool* done) {
  *done = false;
  if (!launch_msd_count(keys, n, flip, ctx->msd, ctx->num_sms, st)) return CAFS_OK;  // LSD
  ctx->launches += 3;
  CKL();
  CK(cudaMemcpyAsync(ctx->h_scratch, (char*)ctx->msd + msd_maxb_offset(), sizeof(u32),
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const u32 maxb = (u32)ctx->h_scratch[0];
  if (maxb > msd_bucket_cap()) return CAFS_OK;
  launch_msd_sort(keys, vals, n, flip, ctx->msd, tk, tv, dk, dv, maxb, ctx->num_sms, st);
  ctx->launches += maxb > 128 ? 3 : 2;
  CKL();
  *done = true;
  return CAFS_OK;
}

// fallback_sort (sorter.py:132-138) on device, in place
int fallback_sort(cafs_ctx_t* ctx, u64* x, u64 n, u64 flip, cudaStream_t st) {
  if (n < 2) return CAFS_OK;
  if (n <= kSmallSortMax) {
    cudaError_t e = launch_small_sort_keys(x, n, flip, st);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "small sort", e);
    ctx->launches++;
    return CAFS_OK;
  }
  TRY(ensure_radix(ctx, n, true));
  bool done;
  TRY(try_msd(ctx, x, nullptr, n, flip, ctx->tmp, nullptr, x, nullptr, st, &done));
  if (done) return CAFS_OK;
  u64 *rk, *rv;
  TRY(radix_sort(ctx, x, nullptr, ctx->tmp, nullptr, n, flip, st, &rk, &rv));
  if (rk != x) CK(cudaMemcpyAsync(x, rk, n * 8, cudaMemcpyDeviceToDevice, st));
  return CAFS_OK;
}

// fallback for any key kind: a 32-bit column is widened to int64, sorted by the
// 64-bit fallback and narrowed back (rare routes: high entropy, small n, guard)
int fallback_any(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, cudaStream_t st, int kk) {
  if (kk == 0) return fallback_sort(ctx, (u64*)x, n, flip, st);
  if (n < 2) return CAFS_OK;
  if (n > ctx->wide_elems) {
    if (ctx->wide) CK(cudaFree(ctx->wide));
    ctx->wide = nullptr;
    ctx->wide_elems = 0;
    CK(cudaMalloc(&ctx->wide, n * 8));
    ctx->wide_elems = n;
  }
  launch_widen(x, n, kk, ctx->wide, ctx->num_sms, st);
  TRY(fallback_sort(ctx, ctx->wide, n, kSign, st));
  launch_narrow(ctx->wide, n, kk, x, ctx->num_sms, st);
  ctx->launches += 2;
  CKL();
  return CAFS_OK;
}

// ---- host <-> device transfers for pageable (unregistered) host memory ----
// The driver stages pageable copies through its own pinned buffers at ~7 GB/s
// per direction on the test host; here host threads each copy a contiguous
// share through a small ring of pinned buffers of their own (host memcpy into
// one while the DMAs of the others run on the thread's stream).  Threads,
// chunk bytes and buffers per thread: 16 x 4 MB x 3 measured 3.0-3.1 Gkeys/s
// for a 2^30-row numpy sort (16 x 8 MB x 2: 2.6-2.8; pinned host memory: 3.5);
// CAFS_XFER_T / _MB / _NB override them (tuning knobs).
constexpr int kXferMax = 32;
static int xfer_threads() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("CAFS_XFER_T"); v = e ? atoi(e) : 16; if (v < 1 || v > 32) v = 16; }
  return v;
}
static size_t xfer_chunk() {
  static size_t v = 0;
  if (!v) {
    const char* e = getenv("CAFS_XFER_MB");
    const int mb = e ? atoi(e) : 4;
    v = (size_t)(mb >= 1 && mb <= 64 ? mb : 4) << 20;
  }
  return v;
}
static int xfer_bufs() {
  static int v = -1;
  if (v < 0) { const char* e = getenv("CAFS_XFER_NB"); v = e ? atoi(e) : 3; if (v < 2 || v > 4) v = 3; }
  return v;
}
#define kXferThreads xfer_threads()
#define kXferChunk xfer_chunk()
#define kXferBufs xfer_bufs()

bool host_is_pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}

int ensure_xfer(cafs_ctx_t* ctx) {
  if (ctx->xfer_buf) return CAFS_OK;
  for (int t = 0; t < kXferThreads; ++t) {
    CK(cudaStreamCreateWithFlags(&ctx->xfer_stream[t], cudaStreamNonBlocking));
    for (int b = 0; b < 4; ++b)
      CK(cudaEventCreateWithFlags(&ctx->xfer_event[t][b], cudaEventDisableTiming));
  }
  CK(cudaMallocHost(&ctx->xfer_buf, (size_t)kXferThreads * kXferBufs * kXferChunk));
  return CAFS_OK;
}

// bytes from pageable host memory to the device (to_device) or back; returns
// the first CUDA error of any worker (cudaSuccess otherwise)
cudaError_t staged_copy(cafs_ctx_t* ctx, void* dev, void* host, size_t bytes, bool to_device) {
  std::vector<std::thread> workers;
  cudaError_t errs[kXferMax] = {};
  const int T = kXferThreads, NB = kXferBufs;
  const size_t C = kXferChunk;
  const size_t share = ((bytes + T - 1) / T + 15) & ~(size_t)15;
  const int device = ctx->device;
  for (int t = 0; t < T; ++t) {
    const size_t lo = (size_t)t * share;
    if (lo >= bytes) break;
    const size_t hi = lo + share < bytes ? lo + share : bytes;
    workers.emplace_back([=, &errs]() {
      cudaError_t e = cudaSetDevice(device);
      cudaStream_t st = ctx->xfer_stream[t];
      unsigned char* base = ctx->xfer_buf + (size_t)t * NB * C;  // NB pinned buffers, a ring
      unsigned char* hp = (unsigned char*)host;
      unsigned char* dp = (unsigned char*)dev;
      const size_t nch = (hi - lo + C - 1) / C;
      auto len_of = [&](size_t c) { const size_t o = lo + c * C; return hi - o < C ? hi - o : C; };
      if (to_device) {  // memcpy into buffer c % NB once its previous DMA is done, then DMA it
        for (size_t c = 0; c < nch && e == cudaSuccess; ++c) {
          const int k = (int)(c % NB);
          if (c >= (size_t)NB) e = cudaEventSynchronize(ctx->xfer_event[t][k]);
          if (e != cudaSuccess) break;
          memcpy(base + k * C, hp + lo + c * C, len_of(c));
          e = cudaMemcpyAsync(dp + lo + c * C, base + k * C, len_of(c), cudaMemcpyHostToDevice, st);
          if (e == cudaSuccess) e = cudaEventRecord(ctx->xfer_event[t][k], st);
        }
      } else {  // DMAs run NB - 1 chunks ahead of the memcpy out of the pinned ring
        for (size_t c = 0; c < nch && c < (size_t)NB - 1 && e == cudaSuccess; ++c) {
          e = cudaMemcpyAsync(base + (c % NB) * C, dp + lo + c * C, len_of(c), cudaMemcpyDeviceToHost, st);
          if (e == cudaSuccess) e = cudaEventRecord(ctx->xfer_event[t][c % NB], st);
        }
        for (size_t c = 0; c < nch && e == cudaSuccess; ++c) {
          const size_t nx = c + NB - 1;
          if (nx < nch) {
            e = cudaMemcpyAsync(base + (nx % NB) * C, dp + lo + nx * C, len_of(nx),
                                cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaEventRecord(ctx->xfer_event[t][nx % NB], st);
            if (e != cudaSuccess) break;
          }
          e = cudaEventSynchronize(ctx->xfer_event[t][c % NB]);
          if (e == cudaSuccess) memcpy(hp + lo + c * C, base + (c % NB) * C, len_of(c));
        }
      }
      if (e == cudaSuccess) e = cudaStreamSynchronize(st);
      errs[t] = e;
    });
  }
  for (auto& w : workers) w.join();
  for (int t = 0; t < T; ++t)
    if (errs[t] != cudaSuccess) return errs[t];
  return cudaSuccess;
}

// host buffer -> device (the caller's stream waits for it) and back
int host_to_device(cafs_ctx_t* ctx, void* dev, const void* host, size_t bytes, cudaStream_t st) {
  if (!bytes) return CAFS_OK;
  if (bytes >= 4 * kXferChunk && host_is_pageable(host)) {
    TRY(ensure_xfer(ctx));
    CK(cudaStreamSynchronize(st));  // the device buffer is free
    cudaError_t e = staged_copy(ctx, dev, (void*)host, bytes, true);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "staged host-to-device copy", e);
    return CAFS_OK;
  }
  CK(cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st));
  return CAFS_OK;
}

int device_to_host(cafs_ctx_t* ctx, void* host, const void* dev, size_t bytes, cudaStream_t st) {
  if (!bytes) return CAFS_OK;
  if (bytes >= 4 * kXferChunk && host_is_pageable(host)) {
    TRY(ensure_xfer(ctx));
    CK(cudaStreamSynchronize(st));  // the sort has finished
    cudaError_t e = staged_copy(ctx, (void*)dev, host, bytes, false);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "staged device-to-host copy", e);
    return CAFS_OK;
  }
  CK(cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st));
  return CAFS_OK;
}

int sync_ctl(cafs_ctx_t* ctx, cudaStream_t st) {
  CK(cudaMemcpyAsync(ctx->h_ctl, ctx->d_ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

void fill_decision(const DevCtl& c, int route, bool has_est, cafs_decision_t* d) {
  memset(d, 0, sizeof(*d));
  d->route = route;
  d->has_estimate = has_est ? 1 : 0;
  if (!has_est) return;
  d->est.k_hat = c.k_hat;
  d->est.u = c.u;
  d->est.f1 = c.f1;
  d->est.f2 = c.f2;
  d->est.saturated = c.saturated;
  d->est.nkeys = c.u <= CAFS_TINY_MAX_KEYS ? (int)c.u : 0;
  for (int j = 0; j < d->est.nkeys; ++j) d->est.keys[j] = c.keys[j];
}

// Non-blocking stage/kernel timer: event pairs are recorded on the stream and
// read after the call's final synchronize, so timing does not perturb the run.
enum { L_STAGE_COUNT = 0, L_STAGE_SORT_K = 1, L_STAGE_EMIT = 2, L_K_COUNT = 3, L_K_EMIT = 4,
       L_K_EST = 5, L_K_PAIR = 6 };
constexpr int kMaxTimed = 16;

// Conditions under which a timed interval is reported (the fused pipeline
// launches every route's kernels; gated-off ones must not show up as stages).
enum { C_ALWAYS = 0, C_TINY = 1, C_MAIN = 2, C_EMIT = 3 };

struct StageTimer {
  cafs_ctx_t* ctx;
  cudaStream_t st;
  bool on;
  cafs_telemetry_t* tel;
  int n = 0;
  int label[kMaxTimed] = {};
  int cond[kMaxTimed] = {};
  bool capturing = false;  // inside stream capture: record external event nodes
  void rec(cudaEvent_t e) {
    if (capturing) cudaEventRecordWithFlags(e, st, cudaEventRecordExternal);
    else cudaEventRecord(e, st);
  }
  int begin() {
    if (!on || n >= kMaxTimed) return -1;
    rec(ctx->ev[2 * n]);
    return n++;
  }
  void end(int i, int lab, int c = C_ALWAYS) {
    if (i < 0) return;
    rec(ctx->ev[2 * i + 1]);
    label[i] = lab;
    cond[i] = c;
  }
  // call after the stream is synchronized; tiny_ran / main_ran / emitted say
  // which gated groups actually executed
  void finish(bool tiny_ran, bool main_ran, bool emitted) {
    for (int i = 0; i < n; ++i) {
      if ((cond[i] == C_TINY && !tiny_ran) || (cond[i] == C_MAIN && !main_ran) ||
          (cond[i] == C_EMIT && !emitted))
        continue;
      float ms = 0;
      if (cudaEventElapsedTime(&ms, ctx->ev[2 * i], ctx->ev[2 * i + 1]) != cudaSuccess) continue;
      float* slot = label[i] < 3 ? &tel->stage_ms[label[i]] : &tel->kernel_ms[label[i] - 3];
      *slot = (*slot < 0 ? 0.f : *slot) + ms;
    }
    n = 0;
  }
};

// K0/K1 (+ the full monotone scan when the prefix is sorted).  Leaves the
// device control block filled and *monotone / *route set.
int run_dispatch(cafs_ctx_t* ctx, const void* x, u64 n, u64 flip, cudaStream_t st, bool* monotone,
                 int* route, StageTimer* tm = nullptr, int kk = 0) {
  const int te = tm ? tm->begin() : -1;
  launch_estimate(x, n, flip, 1, ctx->d_ctl, st, kk);
  if (tm) tm->end(te, L_K_EST);
  ctx->launches++;
  CKL();
  TRY(sync_ctl(ctx, st));
  *monotone = false;
  if (ctx->h_ctl->prefix_sorted) {
    if (n <= kMonoPrefix) {
      *monotone = true;
    } else {
      launch_monotone_scan(x, n, flip, ctx->d_ctl, ctx->num_sms, st, kk);
      ctx->launches++;
      CKL();
      TRY(sync_ctl(ctx, st));
      *monotone = !ctx->h_ctl->scan_inversion;
    }
  }
  *route = *monotone ? CAFS_ALREADY_SORTED : ctx->h_ctl->route;
  return CAFS_OK;
}

// Kernel groups of the fused pipeline.  Every group's kernels check the device
// decision, so launching all of them is always correct; a call whose buffer
// and shape were sorted before launches only the groups the previous call's
// route used (its captured graph holds just those), and the host re-runs the
// full pipeline when the device decision needs a group that was left out
// (the left-out kernels never touch the column, so nothing is lost).
enum : uint32_t {
  kGrpTiny = 1, kGrpDense = 2, kGrpHp = 4, kGrpTable = 8, kGrpOld = 16, kGrpDensePairs = 32,
  kGrpAll = 63
};

uint32_t groups_needed(const DevCtl& c) {
  const int r = c.eff_route;
  // (a dense-window column whose keys all fell inside the window needs neither
  // the compaction nor the pair sort: its window counts are the sorted pairs)
  uint32_t main = c.range_len > 0
                      ? (kGrpDense | kGrpDensePairs | ((c.dense_outside || c.overflow) ? kGrpOld : 0u))
                  : c.hp_ok ? kGrpHp
                            : (kGrpTable | kGrpOld);
  if (r == CAFS_TINY_COUNT) return kGrpTiny | (c.tiny_failed ? main : 0u);
  if (r == CAFS_MAIN) return main;
  return 0;  // sorted input (or its scan), fallback routes: the host's
}

// The fused pipeline (sorter.py:357-386 as one stream of gated kernels):
// tiny count -> tiny finalize -> hash count (dense or queued variant) ->
// compact -> pair sort -> emit.  Each kernel reads the device decision of the
// estimate kernel and exits unless its route is active, so the host needs no
// round trip between the dispatch and the emit.
int launch_fused(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, u64 mult, uint32_t flags,
                 StageTimer& tm, cudaStream_t st, bool with_emit = true, int kk = 0,
                 uint32_t groups = kGrpAll) {
  TRY(ensure_main(ctx));
  DevCtl* c = ctx->d_ctl;
  int ts, tk;
  // CAFS_EMIT_MAP=1 (experiment): the map for every route-specific pipeline
  static const int force_map = getenv("CAFS_EMIT_MAP") ? atoi(getenv("CAFS_EMIT_MAP")) : 0;
  if (groups & kGrpTiny) {
    ts = tm.begin();
    tk = tm.begin();
    launch_tiny_count(x, n, flip, c, ctx->num_sms, st, kGateTiny, kk, ctx->pk_b, ctx->pc_b,
                      ctx->poffs);
    tm.end(tk, L_K_COUNT, C_TINY);
    tm.end(ts, L_STAGE_COUNT, C_TINY);
    ctx->launches++;
  }
  const bool direct = !(flags & CAFS_FLAG_NO_DIRECT);
  const bool hp = hp_allowed(n, !with_emit) && (groups & kGrpHp);
  const bool any_main = groups & (kGrpDense | kGrpHp | kGrpTable | kGrpOld);
  if (any_main) {
    ts = tm.begin();
    tk = tm.begin();
    if (hp) TRY(ensure_hp(ctx, n, kk));
    cudaError_t e = cudaSuccess;
    if (direct && (groups & kGrpDense)) {
      e = launch_hash_count(x, n, flip, mult, c, ctx->gkeys, ctx->gcnt, ctx->glist, 1,
                            ctx->num_sms, st, 0, kGateMainDense, ctx->dense, kk);
      ctx->launches++;
    }
    if (hp && e == cudaSuccess) {  // the partitioned count: the sorted pairs, no pair sort
      // a pipeline that holds only the partitioned count (its route predicted)
      // also gets the emit's tile -> pair map, written with the pairs' offsets
      e = launch_hp_count(hp_bufs(ctx), x, n, flip, c, ctx->pk_b, ctx->pc_b, ctx->poffs,
                          ctx->num_sms, st, kGateMainHP, kk,
                          (with_emit && groups == kGrpHp && !force_map) ? ctx->tile_map : nullptr);
      ctx->launches += 3;
    }
    if (e == cudaSuccess && (groups & kGrpTable)) {
      e = launch_hash_count(x, n, flip, mult, c, ctx->gkeys, ctx->gcnt, ctx->glist,
                            direct ? 1 : 0, ctx->num_sms, st, 1,
                            direct ? kGateMainHash : kGateMainOld, ctx->dense, kk);
      ctx->launches++;
    }
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "hash_count", e);
    tm.end(tk, L_K_COUNT, C_MAIN);
    // a pipeline that holds only the table route (predicted) and emits: the
    // pair sort gathers the pairs from the table itself, no compaction kernel
    const bool gather = with_emit && groups == (kGrpTable | kGrpOld);
    if ((groups & kGrpOld) && !gather) {
      launch_compact(c, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a, ctx->num_sms, st,
                     kGateMainOld);
      ctx->launches++;
    }
    if (direct && (groups & kGrpDensePairs)) {
      launch_dense_pairs(c, ctx->dense, ctx->pk_a, ctx->pc_a, ctx->pk_b, ctx->pc_b, ctx->poffs, n,
                         st, kGateMainDense);
      ctx->launches++;
    }
    tm.end(ts, L_STAGE_COUNT, C_MAIN);
    if (groups & kGrpOld) {
      ts = tm.begin();
      e = launch_small_sort_pairs(ctx->pk_a, ctx->pc_a, 0, c, n, ctx->pk_b, ctx->pc_b, ctx->poffs,
                                  st, kGateMainOld, gather ? ctx->gkeys : nullptr,
                                  gather ? ctx->gcnt : nullptr, gather ? ctx->glist : nullptr);
      if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "pair sort", e);
      tm.end(ts, L_STAGE_SORT_K, C_MAIN);
      ctx->launches++;
    }
  }
  // a pipeline that holds only the partitioned count (its route predicted)
  // also writes the emit's tile -> pair map: its pair sets are large
  bool map = hp && groups == kGrpHp;  // written by hp_place
  const bool map_kernel = force_map && with_emit && groups != kGrpAll && groups != 0 &&
                          !(groups & kGrpTiny);
  if (map_kernel) {
    TRY(ensure_tile_map(ctx, n, kk));
    map = true;
  }
  if (with_emit && map_kernel) {
    launch_emit_map(ctx->poffs, c, x, 0, n, ctx->tile_map, (u64)ctx->num_sms * 8 * 256,
                    ctx->num_sms, st, kk);
    ctx->launches++;
  }
  if (with_emit && groups != 0) {
    ts = tm.begin();
    tk = tm.begin();
    launch_emit(ctx->pk_b, ctx->poffs, 0, c, x, 0, n, flip, ctx->num_sms, st, kSmallSortMax, kk,
                false, map ? ctx->tile_map : nullptr);
    tm.end(tk, L_K_EMIT, C_EMIT);
    tm.end(ts, L_STAGE_EMIT, C_EMIT);
    ctx->launches++;
  }
  CKL();
  return CAFS_OK;
}

// Reference-exact bucket-table statistics (telemetry.cu), from the compacted
// pairs (pk_a, pc_a) and the still-unsorted input x.
int exact_telemetry(cafs_ctx_t* ctx, const void* x, u64 n, u64 flip, u64 mult, double k_hat,
                    uint32_t flags, cafs_telemetry_t* tel, cudaStream_t st, int kk = 0) {
  const DevCtl c = *ctx->h_ctl;
  const u64 np = c.npairs;
  // the key -> pair lookup table: a power of two >= 2 x pairs (load <= 1/2)
  u64 tl_slots = 1024;
  while (tl_slots < 2 * kPairCap) tl_slots <<= 1;
  if (!ctx->tl_keys) {
    CK(cudaMalloc(&ctx->tl_keys, tl_slots * 8));
    CK(cudaMalloc(&ctx->tl_idx, tl_slots * 4));
    CK(cudaMalloc(&ctx->tl_first, kPairCap * 4));
    CK(cudaMalloc(&ctx->tl_runs, kPairCap * 4));
    CK(cudaMalloc(&ctx->tl_comp, 4 * kPairCap * 8));
    CK(cudaMalloc(&ctx->tl_offs, (kPairCap + 1) * 8));
    CK(cudaMalloc(&ctx->tl_acc, tel_accum_bytes()));
  }
  TRY(ensure_radix(ctx, np, false));
  int log2s = 10;
  while ((1ull << log2s) < 2 * np) ++log2s;
  CK(cudaMemsetAsync(ctx->tl_acc, 0, tel_accum_bytes(), st));
  // all np pairs: sorted in pk_b when the pair sort (or the dense path)
  // finished, else the compacted list in pk_a
  const u64* pk = c.pairs_ready ? ctx->pk_b : ctx->pk_a;
  const u64* pc = c.pairs_ready ? ctx->pc_b : ctx->pc_a;
  launch_tel_build(pk, np, ctx->tl_keys, ctx->tl_idx, log2s, ctx->tl_first, ctx->tl_runs,
                   ctx->tl_acc, ctx->num_sms, st);
  launch_tel_runs(x, n, flip, ctx->tl_keys, ctx->tl_idx, log2s, ctx->tl_first, ctx->tl_runs,
                  ctx->tl_acc, ctx->num_sms, st, kk);
  const bool dom32 = flags & (CAFS_FLAG_DOM_I32 | CAFS_FLAG_DOM_U32);
  const int cap = dom32 ? 8 : 4;
  const u64 M = table_size_for(k_hat > 1.0 ? k_hat : 1.0, n, cap);
  const int m_log2 = 63 - __builtin_clzll(M);
  const int dom = kk ? kk : (flags & CAFS_FLAG_DOM_I32) ? 1 : (flags & CAFS_FLAG_DOM_U32) ? 2 : 0;
  u64 *comp = ctx->tl_comp, *cidx = comp + kPairCap, *comp2 = cidx + kPairCap,
      *cidx2 = comp2 + kPairCap;
  launch_tel_comp(pk, np, ctx->tl_first, mult, m_log2, dom, comp, cidx, ctx->num_sms, st);
  ctx->launches += 3;
  u64 *sk = comp, *sv = cidx;
  if (np <= kSmallSortMax) {
    cudaError_t e = launch_small_sort_pairs(comp, cidx, np, nullptr, 0, comp2, cidx2, ctx->tl_offs,
                                            st, kGateNone);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "telemetry sort", e);
    sk = comp2;
    sv = cidx2;
  } else {
    bool done;
    TRY(try_msd(ctx, comp, cidx, np, 0, comp2, cidx2, comp, cidx, st, &done));
    if (!done) TRY(radix_sort(ctx, comp, cidx, comp2, cidx2, np, 0, st, &sk, &sv));
  }
  launch_tel_classify(sk, sv, np, cap, pc, ctx->tl_runs, ctx->tl_acc, ctx->num_sms, st);
  ctx->launches += 2;
  CKL();
  unsigned long long acc[6];
  CK(cudaMemcpyAsync(acc, ctx->tl_acc, sizeof(acc), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  // TelAccum: runs, spill_len, spill_pushes, claims, stored_runs
  tel->exact = 1;
  tel->ref_updates = acc[0];
  tel->ref_spill_len = acc[1];
  tel->ref_spill_pushes = acc[2];
  tel->ref_claims = acc[3];
  tel->ref_hits = acc[4] - acc[3];
  tel->ref_counted_total = n - acc[1];
  tel->ref_guard_fired = acc[1] * 2 > n;
  return CAFS_OK;
}

// After the fused pipeline: the guard (overflow -> fallback, sorter.py:264-273),
// the large-pair-set path, and the sum check (sorter.py:247-248).
int fallback_any(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, cudaStream_t st, int kk);

int main_finish(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, cafs_telemetry_t* tel,
                StageTimer& tm, cudaStream_t st, bool* emitted, int kk = 0) {
  DevCtl& c = *ctx->h_ctl;
  tel->global_updates = c.g_updates;
  static const bool debug = getenv("CAFS_DEBUG") != nullptr;
  if (debug)
    fprintf(stderr, "[cafs] route=%d eff=%d hp_ok=%d hp_ovf=%u range_len=%u npairs=%llu total=%llu ready=%d need_large=%d ovf=%d k_hat=%f\n",
            c.route, c.eff_route, c.hp_ok, c.hp_overflow, c.range_len, (unsigned long long)c.npairs,
            (unsigned long long)c.total, c.pairs_ready, c.need_large, c.overflow, c.k_hat);
  if (c.hp_overflow) {
    // a partition of the partitioned count held more distinct keys than its
    // table: put the column back together from the cells and the spill (its
    // streamed part was overwritten by the spill), then sort it like the guard
    launch_hp_restore(hp_bufs(ctx), x, n, flip, ctx->num_sms, st, kk);
    ctx->launches++;
    CKL();
    tel->guard_fired = 1;
    *emitted = false;
    const int ts = tm.begin();
    TRY(fallback_any(ctx, x, n, flip, st, kk));
    tm.end(ts, L_STAGE_SORT_K);
    return CAFS_OK;
  }
  if (c.overflow) {
    CK(cudaMemsetAsync(ctx->gkeys, 0xFF, kGlobalSlots * 8, st));
    CK(cudaMemsetAsync(ctx->gcnt, 0, kGlobalSlots * 8, st));
    tel->guard_fired = 1;
    *emitted = false;
    const int ts = tm.begin();
    TRY(fallback_any(ctx, x, n, flip, st, kk));
    tm.end(ts, L_STAGE_SORT_K);
    return CAFS_OK;
  }
  if (c.need_large) {
    if (c.need_compact) {
      // the pipeline held no compaction and its pair sort found too many pairs
      // to gather: compact now (npairs is read back with the next sync)
      launch_compact(ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a,
                     ctx->num_sms, st, kGateNone);
      ctx->launches++;
      CKL();
      TRY(sync_ctl(ctx, st));
    }
    const u64 np = c.npairs;
    bool check = false;
    for (int pass = 0; pass < 2; ++pass) {
      int ts = tm.begin();
      if (pass == 0) {
        TRY(sort_pairs_large_unchecked(ctx, np, st, &check));
      } else {  // a bucket overflowed the unchecked MSD sort: LSD, then the same scan + emit
        u64 *rk, *rv;
        TRY(radix_sort(ctx, ctx->pk_a, ctx->pc_a, ctx->pk_b, ctx->pc_b, np, 0, st, &rk, &rv));
        if (rk != ctx->pk_b) {
          CK(cudaMemcpyAsync(ctx->pk_b, rk, np * 8, cudaMemcpyDeviceToDevice, st));
          CK(cudaMemcpyAsync(ctx->pc_b, rv, np * 8, cudaMemcpyDeviceToDevice, st));
        }
        check = false;
      }
      launch_scan(ctx->pc_b, np, ctx->bsum, ctx->poffs, ctx->d_ctl, n, st);
      ctx->launches += 3;
      CKL();
      tm.end(ts, L_STAGE_SORT_K);
      ts = tm.begin();
      const u64 tiles = emit_tiles(n, kk);
      if (tiles > ctx->tile_map_len) {
        if (ctx->tile_map) CK(cudaFree(ctx->tile_map));
        ctx->tile_map = nullptr;
        ctx->tile_map_len = 0;
        CK(cudaMalloc(&ctx->tile_map, tiles * sizeof(u32)));
        ctx->tile_map_len = tiles;
      }
      launch_emit_map(ctx->poffs, ctx->d_ctl, x, 0, n, ctx->tile_map, np, ctx->num_sms, st, kk);
      const int tk = tm.begin();
      launch_emit(ctx->pk_b, ctx->poffs, 0, ctx->d_ctl, x, 0, n, flip, ctx->num_sms, st, np, kk,
                  false, ctx->tile_map);
      tm.end(tk, L_K_EMIT);
      ctx->launches += 2;
      CKL();
      tm.end(ts, L_STAGE_EMIT);
      if (check)
        CK(cudaMemcpyAsync(ctx->h_scratch, (char*)ctx->msd + msd_overflow_offset(), sizeof(u32),
                           cudaMemcpyDeviceToHost, st));
      TRY(sync_ctl(ctx, st));
      if (!check || ctx->h_scratch[0] == 0) break;
    }
    *emitted = true;
  }
  if (c.sum_error || !c.pairs_ready) return fail(ctx, CAFS_ESUM, "pair counts do not sum to n");
  tel->counted_total = c.total;
  tel->pairs = c.npairs;
  return CAFS_OK;
}

void pipeline_direct(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, u64 mult, uint32_t flags,
                     StageTimer& tm, cudaStream_t st, bool exact, int* mark, int* rc, int kk,
                     uint32_t groups = kGrpAll) {
  const int te = tm.begin();
  launch_estimate(x, n, flip, 1, ctx->d_ctl, st, kk,
                  (hp_allowed(n, exact) ? kEstHp : 0) |
                      ((flags & CAFS_FLAG_NO_DIRECT) ? kEstNoWindow : 0));
  tm.end(te, L_K_EST);
  ctx->launches++;
  *mark = tm.n;
  *rc = launch_fused(ctx, x, n, flip, mult, flags, tm, st, !exact, kk, groups);
}

// The estimate + fused kernels, replayed from a cached CUDA Graph when the same
// (buffer, n, flags) was sorted before: one graph launch instead of ~9 kernel
// launches (the small-input latency).  The graph's kernels are the same; only
// the launch path differs.
int launch_pipeline(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, u64 mult, uint32_t flags,
                    StageTimer& tm, cudaStream_t st, bool exact, int* mark, int kk,
                    uint32_t* used, cafs_ctx_t::GraphEntry** entry) {
  *used = kGrpAll;
  *entry = nullptr;
  static int use_graphs = -1;
  if (use_graphs < 0) {
    const char* e = getenv("CAFS_GRAPHS");
    use_graphs = e ? atoi(e) != 0 : 1;
  }
  int rc = CAFS_OK;
  if (!use_graphs || !ctx->cap_stream) {
    pipeline_direct(ctx, x, n, flip, mult, flags, tm, st, exact, mark, &rc, kk);
    CKL();
    return rc;
  }
  const int timing = tm.on ? 1 : 0;
  cafs_ctx_t::GraphEntry* hit = nullptr;
  cafs_ctx_t::GraphEntry* lru = &ctx->graphs[0];
  for (auto& g : ctx->graphs) {
    if (g.seen && g.x == (u64)x && g.n == n && g.flip == flip && g.mult == mult &&
        g.flags == flags && g.timing == timing && g.kk == kk && g.exact == (int)exact) {
      hit = &g;
      break;
    }
    if (g.stamp < lru->stamp) lru = &g;
  }
  if (hit && hit->exec) {
    *used = hit->groups;
    *entry = hit;
    CK(cudaGraphLaunch(hit->exec, st));
    tm.n = hit->tn;
    for (int i = 0; i < hit->tn; ++i) { tm.label[i] = hit->label[i]; tm.cond[i] = hit->cond[i]; }
    *mark = hit->mark;
    ctx->launches += hit->launches;
    hit->stamp = ++ctx->graph_clock;
    return CAFS_OK;
  }
  if (!hit) {  // first sighting: run directly, capture next time
    if (lru->exec) cudaGraphExecDestroy(lru->exec);
    *lru = cafs_ctx_t::GraphEntry();
    lru->x = (u64)x; lru->n = n; lru->flip = flip; lru->mult = mult; lru->flags = flags;
    lru->timing = timing; lru->seen = 1; lru->stamp = ++ctx->graph_clock; lru->kk = kk;
    lru->exact = exact ? 1 : 0;
    *entry = lru;
    pipeline_direct(ctx, x, n, flip, mult, flags, tm, st, exact, mark, &rc, kk);
    CKL();
    return rc;
  }
  // second sighting: capture on the context's stream, then launch on the caller's
  const uint64_t l0 = ctx->launches;
  StageTimer ct = tm;
  ct.st = ctx->cap_stream;
  ct.capturing = true;
  cudaGraph_t graph = nullptr;
  *used = hit->groups;
  *entry = hit;
  CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
  pipeline_direct(ctx, x, n, flip, mult, flags, ct, ctx->cap_stream, exact, mark, &rc, kk,
                  hit->groups);
  cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &graph);
  if (rc != CAFS_OK) { if (graph) cudaGraphDestroy(graph); return rc; }
  if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "graph capture", e);
  e = cudaGraphInstantiate(&hit->exec, graph, 0);
  cudaGraphDestroy(graph);
  if (e != cudaSuccess) { hit->exec = nullptr; return fail(ctx, CAFS_ECUDA, "graph instantiate", e); }
  hit->tn = ct.n;
  hit->mark = *mark;
  for (int i = 0; i < ct.n; ++i) { hit->label[i] = ct.label[i]; hit->cond[i] = ct.cond[i]; }
  hit->launches = ctx->launches - l0;
  hit->stamp = ++ctx->graph_clock;
  CK(cudaGraphLaunch(hit->exec, st));
  tm.n = ct.n;
  for (int i = 0; i < ct.n; ++i) { tm.label[i] = ct.label[i]; tm.cond[i] = ct.cond[i]; }
  return CAFS_OK;
}

int check_common(cafs_ctx_t* ctx, const void* p, u64 n, u64 align = 8) {
  if (!ctx) return CAFS_EINVAL;
  if (n >= (1ull << 32)) return fail(ctx, CAFS_EINVAL, "arrays of 2**32 or more elements");
  if (n > 0 && !p) return fail(ctx, CAFS_EINVAL, "null data pointer");
  if (((uintptr_t)p) & (align - 1))
    return fail(ctx, CAFS_EINVAL, align == 8 ? "data must be 8-byte aligned"
                                             : "data must be 4-byte aligned");
  return CAFS_OK;
}

// host-side perfect hash for caller-given tiny keys (same family as estimate.cu)
u64 host_fmix64(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// ---- the sharded pipeline's device phases (shard.cu), shared by the
// cafs_shard_* calls (collectives by the caller) and cafs_sort_i64_sharded
// (collectives here, over the library's own NCCL communicator) ----

// Route classes of the sharded pipeline.  The route, the dense window and so
// the class of a column are the same on every rank (all decide from the same
// all-reduced samples and gathered headers), so a communicator can predict the
// next column's class from the last ones and leave the other classes' kernels
// out of its graph -- the collectives stay the same three on every rank; a
// wrong prediction is seen by every rank alike and all re-run the full
// pipeline (the left-out kernels never touch the column).
// kClsWindowSum: the window class's own pipeline -- every rank counts into the
// same dense window (its base comes from the all-reduced samples), so the
// merge is the element-wise sum of the count arrays: one all-reduce of 64 KB
// in place of the pair tables' all-gather and the merge of the gathered lists.
// A key outside the window on any rank leaves the summed counts short of the
// column's rows on every rank: all re-run the full pipeline.
enum : uint32_t { kClsTiny = 1, kClsWindow = 2, kClsNoWindow = 4, kClsAll = 7, kClsWindowSum = 8 };

uint32_t shard_class(const DevCtl& h) {
  if (h.eff_route == CAFS_TINY_COUNT) return kClsTiny;
  if (h.eff_route == CAFS_MAIN) return h.range_len > 0 ? kClsWindow : kClsNoWindow;
  return 0;  // sorted, fallback routes: no device count
}

// estimate on the gathered samples -> route; tiny count or local hash count ->
// sorted local pairs -> this rank's send row [np, keys[cap], counts[cap]]
int shard_count_enqueue(cafs_ctx_t* ctx, const void* x, u64 n, u64 flip, u64 mult,
                        const u64* hdr_all, int world, const u64* samples, u64* tiny, u64* send,
                        u64 cap, cudaStream_t st, int kk = 0, uint32_t cls = kClsAll,
                        int est_opts = 0) {
  DevCtl* c = ctx->d_ctl;
  // the partitioned count gives this shard's pairs sorted on device for any
  // number of keys (the table path's pair sort stops at 8192)
  const bool hp = hp_allowed(n, false);
  if (hp) TRY(ensure_hp(ctx, n, kk));
  launch_estimate_sharded(samples, hdr_all, world, c, st, (hp ? kEstHp : 0) | est_opts);
  ctx->launches++;
  if (cls & kClsTiny) {
    launch_tiny_count(x, n, flip, c, ctx->num_sms, st, kGateTiny, kk);
    launch_shard_tiny_pack(c, tiny, st);
    ctx->launches += 2;
  }
  const bool any_main = cls & (kClsWindow | kClsNoWindow);
  cudaError_t e = cudaSuccess;
  if (cls & kClsWindow) {
    e = launch_hash_count(x, n, flip, mult, c, ctx->gkeys, ctx->gcnt, ctx->glist, 1, ctx->num_sms,
                          st, 0, kGateMainDense, ctx->dense, kk);
    ctx->launches++;
  }
  if (hp && (cls & kClsNoWindow) && e == cudaSuccess) {
    e = launch_hp_count(hp_bufs(ctx), x, n, flip, c, ctx->pk_b, ctx->pc_b, ctx->poffs,
                        ctx->num_sms, st, kGateMainHP, kk);
    ctx->launches += 3;
  }
  if ((cls & kClsNoWindow) && e == cudaSuccess) {
    e = launch_hash_count(x, n, flip, mult, c, ctx->gkeys, ctx->gcnt, ctx->glist, 1,
                          ctx->num_sms, st, 1, kGateMainHash, ctx->dense, kk);
    ctx->launches++;
  }
  if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "hash_count", e);
  if (any_main) {
    launch_compact(c, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a, ctx->num_sms, st,
                   kGateMainOld);
    ctx->launches++;
  }
  if (cls & kClsWindow) {
    launch_dense_pairs(c, ctx->dense, ctx->pk_a, ctx->pc_a, ctx->pk_b, ctx->pc_b, ctx->poffs, n,
                       st, kGateMainDense);
    ctx->launches++;
  }
  if (any_main) {
    e = launch_small_sort_pairs(ctx->pk_a, ctx->pc_a, 0, c, n, ctx->pk_b, ctx->pc_b, ctx->poffs,
                                st, kGateMainOld);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "pair sort", e);
    launch_shard_pack_pairs(c, ctx->pk_b, ctx->pc_b, send, cap, st);
    ctx->launches += 2;
  }
  CKL();
  return CAFS_OK;
}

// tiny totals or the merge of every rank's row -> sorted global pairs -> this
// rank's slice emit (every kernel gated on the device decision)
int shard_finish_enqueue(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, const u64* tiny_sum,
                         const u64* recv, int world, u64 cap, u64 row, cudaStream_t st,
                         int kk = 0, uint32_t cls = kClsAll) {
  DevCtl* c = ctx->d_ctl;
  if (cls & kClsTiny) {
    launch_shard_tiny_finish(c, tiny_sum, ctx->pk_b, ctx->pc_b, ctx->poffs, st);
    ctx->launches++;
  }
  if (cls & (kClsWindow | kClsNoWindow)) {
    // the union of every rank's sorted list (sorter.py:276-285): key-range
    // partitions of the gathered lists reduced on device into the global sorted
    // pairs and offsets -- no hash table, no pair sort, any number of pairs
    if (!ctx->hp_mscratch) CK(cudaMalloc(&ctx->hp_mscratch, hp_scratch_bytes(ctx->num_sms)));
    launch_shard_merge_check(c, recv, world, cap, row, st);
    HpBufs mb = hp_bufs(ctx);
    mb.scratch = ctx->hp_mscratch;
    cudaError_t e = launch_hp_shard_merge(mb, recv, world, cap, row, c, ctx->pk_b, ctx->pc_b,
                                          ctx->poffs, st);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "sharded merge", e);
    ctx->launches += 4;
  }
  launch_emit(ctx->pk_b, ctx->poffs, 0, c, x, 0, n, flip, ctx->num_sms, st, 0, kk, true);
  ctx->launches++;
  CKL();
  return CAFS_OK;
}

// after the control block reached the host mirror: the status every rank agrees
// on (same gathered data) and the telemetry
int shard_result(cafs_ctx_t* ctx, void* x, u64 n, u64 flip, cafs_telemetry_t* tel, int* h_status,
                 cudaStream_t st, int kk = 0) {
  const DevCtl& h = *ctx->h_ctl;
  const int eff = h.eff_route;
  int status = 1;  // 1: the caller runs the host-driven sharded path
  if (eff == CAFS_ALREADY_SORTED) status = 0;
  else if ((eff == CAFS_TINY_COUNT || eff == CAFS_MAIN) && h.pairs_ready && !h.overflow) status = 0;
  if (status != 0 && eff == CAFS_MAIN && h.local_hp) {
    // the partitioned count spilled into this shard: rebuild it from the cells
    // and the spill for the host-driven path (which may sort the rows again)
    launch_hp_restore(hp_bufs(ctx), x, n, flip, ctx->num_sms, st, kk);
    ctx->launches++;
    CKL();
    CK(cudaStreamSynchronize(st));
  }
  if (status != 0 && eff == CAFS_MAIN && !h.merge_bad && h.hp_overflow) {
    // the merge itself overflowed over this shard's sorted pairs: they are gone
    ctx->h_ctl->local_overflow = 1;
    CK(cudaMemcpyAsync(&ctx->d_ctl->local_overflow, &ctx->h_ctl->local_overflow,
                       sizeof(int32_t), cudaMemcpyHostToDevice, st));
    CK(cudaStreamSynchronize(st));
  }
  if (eff == CAFS_MAIN && h.overflow) {  // a local overflow left this rank's table dirty
    CK(cudaMemsetAsync(ctx->gkeys, 0xFF, kGlobalSlots * 8, st));
    CK(cudaMemsetAsync(ctx->gcnt, 0, kGlobalSlots * 8, st));
    CK(cudaStreamSynchronize(st));
  }
  *h_status = status;
  if (tel) {
    memset(tel, 0, sizeof(*tel));
    tel->n = h.n_global;
    fill_decision(h, eff, eff != CAFS_ALREADY_SORTED && h.n_global >= CAFS_SMALL_N_CUTOFF,
                  &tel->decision);
    tel->counted_total = status == 0 && eff != CAFS_ALREADY_SORTED ? h.n_global : 0;
    tel->pairs = h.npairs;
    for (int i = 0; i < 3; ++i) tel->stage_ms[i] = -1.f;
    for (int i = 0; i < 4; ++i) tel->kernel_ms[i] = -1.f;
  }
  return CAFS_OK;
}

}  // namespace

extern "C" {

int cafs_abi_version(void) { return CAFS_ABI_VERSION; }

const char* cafs_status_string(int s) {
  switch (s) {
    case CAFS_OK: return "ok";
    case CAFS_EINVAL: return "invalid argument";
    case CAFS_ECUDA: return "CUDA error";
    case CAFS_ENOMEM: return "out of device memory";
    case CAFS_ESUM: return "pair counts do not sum to the output length";
    default: return "internal error";
  }
}

const char* cafs_last_error(cafs_ctx_t* ctx) { return ctx ? ctx->last_error.c_str() : ""; }

int cafs_ctx_create(int device, cafs_ctx_t** out) {
  if (!out) return CAFS_EINVAL;
  *out = nullptr;
  cafs_ctx_t* ctx = new (std::nothrow) cafs_ctx_t();
  if (!ctx) return CAFS_ENOMEM;
  ctx->device = device;
  DeviceGuard g(device);
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) { delete ctx; return CAFS_ECUDA; }
  cudaDeviceProp prop;
  e = cudaGetDeviceProperties(&prop, device);
  if (e != cudaSuccess) { delete ctx; return CAFS_ECUDA; }
  if (prop.major != 10) { delete ctx; return CAFS_EINVAL; }  // sm_100a only
  ctx->num_sms = prop.multiProcessorCount;
  if (cudaMalloc(&ctx->d_ctl, kDevCtlAlloc) != cudaSuccess ||
      cudaMallocHost(&ctx->h_ctl, sizeof(DevCtl)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_scratch, 64 + CAFS_PARTITION_BUCKETS * 4) != cudaSuccess ||
      cudaMemset(ctx->d_ctl, 0, kDevCtlAlloc) != cudaSuccess) {
    cafs_ctx_destroy(ctx);
    return CAFS_ENOMEM;
  }
  for (int i = 0; i < 32; ++i) cudaEventCreate(&ctx->ev[i]);
  cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking);
  *out = ctx;
  return CAFS_OK;
}

void cafs_ctx_destroy(cafs_ctx_t* ctx) {
  if (!ctx) return;
  DeviceGuard g(ctx->device);
  { std::lock_guard<std::recursive_mutex> lk(ctx->mu); }  // no call in flight on the host
  cudaDeviceSynchronize();
  void* dev[] = {ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a,
                 ctx->pk_b, ctx->pc_b, ctx->poffs, ctx->bsum, ctx->dense, ctx->ghist, ctx->gbase,
                 ctx->trivial, ctx->tile_counters, ctx->tile_state, ctx->tmp, ctx->stage, ctx->msd,
                 ctx->tl_keys, ctx->tl_idx, ctx->tl_first, ctx->tl_runs, ctx->tl_comp,
                 ctx->tl_offs, ctx->tl_acc, ctx->pk_t, ctx->pc_t, ctx->wide, ctx->tile_map,
                 ctx->hp_part, ctx->hp_scratch, ctx->hp_mscratch};
  for (void* p : dev)
    if (p) cudaFree(p);
  if (ctx->h_ctl) cudaFreeHost(ctx->h_ctl);
  if (ctx->h_scratch) cudaFreeHost(ctx->h_scratch);
  if (ctx->h_trivial) cudaFreeHost(ctx->h_trivial);
  for (int i = 0; i < 32; ++i)
    if (ctx->ev[i]) cudaEventDestroy(ctx->ev[i]);
  for (auto& g : ctx->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
  for (int t = 0; t < kXferThreads; ++t) {
    if (ctx->xfer_stream[t]) cudaStreamDestroy(ctx->xfer_stream[t]);
    for (int b = 0; b < 4; ++b)
      if (ctx->xfer_event[t][b]) cudaEventDestroy(ctx->xfer_event[t][b]);
  }
  if (ctx->xfer_buf) cudaFreeHost(ctx->xfer_buf);
  delete ctx;
}

// The whole sort for key kind kk (0: 64-bit, 1: int32, 2: uint32; the flip of
// 32-bit kinds is implied).
static int sort_impl(cafs_ctx_t* ctx, void* d_x, uint64_t n, int is_signed, uint64_t hash_mult,
                     uint32_t flags, cafs_telemetry_t* tel, void* stream, int kk) {
  TRY(check_common(ctx, d_x, n, kk ? 4 : 8));
  if ((hash_mult & 1) == 0) return fail(ctx, CAFS_EINVAL, "hash multiplier must be odd");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t launches0 = ctx->launches;
  cafs_telemetry_t local;
  const bool want_tel = tel != nullptr;
  if (!tel) tel = &local;
  memset(tel, 0, sizeof(*tel));
  tel->n = n;
  for (int i = 0; i < 3; ++i) tel->stage_ms[i] = -1.f;
  for (int i = 0; i < 4; ++i) tel->kernel_ms[i] = -1.f;
  if (n <= 1) {
    tel->decision.route = CAFS_ALREADY_SORTED;
    return CAFS_OK;
  }
  StageTimer tm{ctx, st, want_tel && (flags & CAFS_FLAG_TIMING), tel};
  void* x = d_x;
  const u64 flip = (is_signed || kk) ? kSign : 0;
  // K0/K1 then every route's kernels, gated on the device decision; one sync
  const bool exact = want_tel && (flags & CAFS_FLAG_EXACT_TELEMETRY);
  TRY(ensure_main(ctx));
  int mark = 0;
  uint32_t used = kGrpAll;
  cafs_ctx_t::GraphEntry* entry = nullptr;
  TRY(launch_pipeline(ctx, x, n, flip, hash_mult, flags, tm, st, exact, &mark, kk, &used, &entry));
  TRY(sync_ctl(ctx, st));
  {
    const uint32_t need = groups_needed(*ctx->h_ctl);
    if (need & ~used) {
      // the cached pipeline left out a group this input's route needs: run
      // the whole pipeline (nothing was written to the column)
      tm.n = 0;
      int rc2 = CAFS_OK;
      if ((used & kGrpDense) && !(used & kGrpOld) && ctx->h_ctl->dense_outside &&
          !ctx->h_ctl->overflow) {
        // the window-only pipeline counted keys outside the window into the
        // global table and held no compaction: empty the table first
        launch_compact(ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a,
                       ctx->num_sms, st, kGateNone);
        ctx->launches++;
      }
      pipeline_direct(ctx, x, n, flip, hash_mult, flags, tm, st, exact, &mark, &rc2, kk);
      TRY(rc2);
      CKL();
      TRY(sync_ctl(ctx, st));
    }
    // the next call on this buffer and shape launches what this route used
    const uint32_t next = groups_needed(*ctx->h_ctl);
    if (entry && entry->groups != next && ctx->h_ctl->eff_route != kNeedScan) {
      if (entry->exec) cudaGraphExecDestroy(entry->exec);
      entry->exec = nullptr;
      entry->groups = next;
    }
  }
  int eff = ctx->h_ctl->eff_route;
  bool mono = eff == CAFS_ALREADY_SORTED;
  if (eff == kNeedScan) {
    // the first 16385 rows are sorted: scan the rest, then rerun the gated
    // pipeline with the resolved route (the first pass was all no-ops)
    tm.n = mark;
    launch_monotone_scan(x, n, flip, ctx->d_ctl, ctx->num_sms, st, kk);
    ctx->launches++;
    CKL();
    TRY(sync_ctl(ctx, st));
    mono = !ctx->h_ctl->scan_inversion;
    eff = mono ? CAFS_ALREADY_SORTED : ctx->h_ctl->route;
    if (!mono && (eff == CAFS_TINY_COUNT || eff == CAFS_MAIN)) {
      ctx->h_scratch[0] = eff;
      CK(cudaMemcpyAsync(&ctx->d_ctl->eff_route, ctx->h_scratch, sizeof(int32_t),
                         cudaMemcpyHostToDevice, st));
      TRY(launch_fused(ctx, x, n, flip, hash_mult, flags, tm, st, !exact, kk));
      TRY(sync_ctl(ctx, st));
    }
  }
  if (exact) {
    // the reference's table statistics need the unsorted input: compute them
    // now, then run the emit the fused pipeline left out
    const DevCtl& cc = *ctx->h_ctl;
    const bool main_ran_ = eff == CAFS_MAIN || (eff == CAFS_TINY_COUNT && cc.tiny_failed);
    if (main_ran_ && !cc.overflow)
      TRY(exact_telemetry(ctx, x, n, flip, hash_mult, cc.k_hat, flags, tel, st, kk));
    if ((eff == CAFS_MAIN || eff == CAFS_TINY_COUNT) && cc.pairs_ready) {
      const int ts = tm.begin();
      launch_emit(ctx->pk_b, ctx->poffs, 0, ctx->d_ctl, x, 0, n, flip, ctx->num_sms, st,
                  kSmallSortMax, kk);
      tm.end(ts, L_STAGE_EMIT, C_EMIT);
      ctx->launches++;
      CKL();
    }
    if (main_ran_ && cc.overflow) {
      // the device guard sorts with the fallback; the reference statistics
      // still follow from the pairs the count saw -- not available, so report
      // them as not exact
      tel->exact = 0;
    }
  }
  const DevCtl c = *ctx->h_ctl;
  fill_decision(c, eff, !mono && n >= CAFS_SMALL_N_CUTOFF, &tel->decision);
  bool tiny_ran = false, main_ran = false, emitted = false;
  int rc = CAFS_OK;
  switch (eff) {
    case CAFS_ALREADY_SORTED:
      break;
    case CAFS_FALLBACK_SMALL_N:
    case CAFS_FALLBACK_HIGH_ENTROPY: {
      const int ts = tm.begin();
      rc = fallback_any(ctx, x, n, flip, st, kk);
      tm.end(ts, L_STAGE_SORT_K);
      break;
    }
    case CAFS_TINY_COUNT:
      tiny_ran = true;
      if (!c.tiny_failed) {
        if (!c.pairs_ready) return fail(ctx, CAFS_ESUM, "tiny counts do not sum to n");
        emitted = true;
        tel->counted_total = n;
        tel->pairs = (u64)c.nkeys;
        break;
      }
      // the sample missed a value: MAIN with the same k_hat (sorter.py:378-385)
      tel->tiny_count_failed = 1;
      tel->decision.route = CAFS_MAIN;
      /* fall through */
    default:
      main_ran = true;
      emitted = true;
      tel->table_buckets = table_size_for(c.k_hat > 1.0 ? c.k_hat : 1.0, n, kk ? 8 : 4);  // bucket_cap, buckets.py:33-43
      rc = main_finish(ctx, x, n, flip, tel, tm, st, &emitted, kk);
      break;
  }
  if (rc != CAFS_OK) return rc;
  if (tiny_ran && !c.tiny_failed) tel->count_path = CAFS_COUNT_TINY;
  else if (main_ran)
    tel->count_path = c.range_len > 0 ? CAFS_COUNT_DENSE
                      : c.hp_ok       ? CAFS_COUNT_PARTITIONED
                                      : CAFS_COUNT_TABLE;
  CK(cudaStreamSynchronize(st));
  tm.finish(tiny_ran, main_ran, emitted);
  if (exact && !main_ran) {
    // no bucket table in the reference either: all statistics are zero
    tel->exact = 1;
    tel->ref_counted_total = tel->counted_total;
  }
  tel->kernels_launched = (uint32_t)(ctx->launches - launches0);
  return CAFS_OK;
}

int cafs_sort_i64(cafs_ctx_t* ctx, int64_t* d_x, uint64_t n, int is_signed, uint64_t hash_mult,
                  uint32_t flags, cafs_telemetry_t* tel, void* stream) {
  return sort_impl(ctx, d_x, n, is_signed, hash_mult, flags, tel, stream, 0);
}

int cafs_sort_i32(cafs_ctx_t* ctx, int32_t* d_x, uint64_t n, int is_signed, uint64_t hash_mult,
                  uint32_t flags, cafs_telemetry_t* tel, void* stream) {
  return sort_impl(ctx, d_x, n, is_signed, hash_mult, flags, tel, stream, is_signed ? 1 : 2);
}

int cafs_sort_i32_host(cafs_ctx_t* ctx, const int32_t* h_in, int32_t* h_out, uint64_t n,
                       int is_signed, uint64_t hash_mult, uint32_t flags, cafs_telemetry_t* tel,
                       void* stream) {
  if (!ctx) return CAFS_EINVAL;
  if (n >= (1ull << 32)) return fail(ctx, CAFS_EINVAL, "arrays of 2**32 or more elements");
  if (n > 0 && (!h_in || !h_out)) return fail(ctx, CAFS_EINVAL, "null host pointer");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  if (n > ctx->stage_elems) {  // the stage holds n 8-byte words: room for n 4-byte keys
    if (ctx->stage) CK(cudaFree(ctx->stage));
    ctx->stage = nullptr;
    ctx->stage_elems = 0;
    CK(cudaMalloc(&ctx->stage, (n ? n : 1) * 8));
    ctx->stage_elems = n;
  }
  TRY(host_to_device(ctx, ctx->stage, h_in, n * 4, st));
  TRY(cafs_sort_i32(ctx, (int32_t*)ctx->stage, n, is_signed, hash_mult, flags, tel, stream));
  TRY(device_to_host(ctx, h_out, ctx->stage, n * 4, st));
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

int cafs_sort_i64_host(cafs_ctx_t* ctx, const int64_t* h_in, int64_t* h_out, uint64_t n,
                       int is_signed, uint64_t hash_mult, uint32_t flags, cafs_telemetry_t* tel,
                       void* stream) {
  if (!ctx) return CAFS_EINVAL;
  if (n >= (1ull << 32)) return fail(ctx, CAFS_EINVAL, "arrays of 2**32 or more elements");
  if (n > 0 && (!h_in || !h_out)) return fail(ctx, CAFS_EINVAL, "null host pointer");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  if (n > ctx->stage_elems) {
    if (ctx->stage) CK(cudaFree(ctx->stage));
    ctx->stage = nullptr;
    ctx->stage_elems = 0;
    CK(cudaMalloc(&ctx->stage, (n ? n : 1) * 8));
    ctx->stage_elems = n;
  }
  TRY(host_to_device(ctx, ctx->stage, h_in, n * 8, st));
  TRY(cafs_sort_i64(ctx, (int64_t*)ctx->stage, n, is_signed, hash_mult, flags, tel, stream));
  TRY(device_to_host(ctx, h_out, ctx->stage, n * 8, st));
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

int cafs_dispatch_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                      uint64_t hash_mult, cafs_decision_t* out, void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!out || n < 2) return fail(ctx, CAFS_EINVAL, "dispatch needs n >= 2");
  if ((hash_mult & 1) == 0) return fail(ctx, CAFS_EINVAL, "hash multiplier must be odd");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  bool mono;
  int route;
  TRY(run_dispatch(ctx, (const u64*)d_x, n, is_signed ? kSign : 0, (cudaStream_t)stream, &mono,
                   &route));
  fill_decision(*ctx->h_ctl, route, !mono && n >= CAFS_SMALL_N_CUTOFF, out);
  return CAFS_OK;
}

int cafs_estimate_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                      cafs_estimate_t* out, void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!out || n < 1) return fail(ctx, CAFS_EINVAL, "n must be >= 1");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  launch_estimate((const u64*)d_x, n, is_signed ? kSign : 0, 0, ctx->d_ctl, st);
  ctx->launches++;
  CKL();
  TRY(sync_ctl(ctx, st));
  cafs_decision_t d;
  fill_decision(*ctx->h_ctl, 0, true, &d);
  *out = d.est;
  return CAFS_OK;
}

int cafs_is_monotone_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed, int* out,
                         void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!out) return CAFS_EINVAL;
  if (n < 2) { *out = 1; return CAFS_OK; }
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  bool mono;
  int route;
  TRY(run_dispatch(ctx, (const u64*)d_x, n, is_signed ? kSign : 0, (cudaStream_t)stream, &mono,
                   &route));
  *out = mono ? 1 : 0;
  return CAFS_OK;
}

int cafs_tiny_counts_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         const uint64_t* h_keys, int nk, int64_t* h_counts, void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (nk < 0 || nk > CAFS_TINY_MAX_KEYS || (nk && (!h_keys || !h_counts)))
    return fail(ctx, CAFS_EINVAL, "tiny-count takes at most 8 keys");
  if (nk == 0) return CAFS_OK;
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  // distinct keys -> perfect hash into 16 slots
  u64 uk[CAFS_TINY_MAX_KEYS];
  int nu = 0, map[CAFS_TINY_MAX_KEYS];
  for (int j = 0; j < nk; ++j) {
    int f = -1;
    for (int q = 0; q < nu; ++q)
      if (uk[q] == h_keys[j]) f = q;
    if (f < 0) { uk[nu] = h_keys[j]; f = nu++; }
    map[j] = f;
  }
  DevCtl& c = *ctx->h_ctl;
  memset(&c, 0, sizeof(c));
  c.nkeys = nu;
  for (int q = 0; q < nu; ++q) c.keys[q] = uk[q];
  for (u64 t = 0;; ++t) {
    const u64 m = host_fmix64(t + 0x5851F42D4C957F2Dull) | 1ull;
    u32 used = 0;
    bool ok = true;
    for (int q = 0; q < nu; ++q) {
      const u32 s = (u32)((uk[q] * m) >> 60);
      ok &= !((used >> s) & 1u);
      used |= 1u << s;
    }
    if (ok) {
      c.tiny_mult = m;
      for (int q = 0; q < nu; ++q) c.tiny_slot[q] = (int)((uk[q] * m) >> 60);
      break;
    }
  }
  CK(cudaMemcpyAsync(ctx->d_ctl, &c, sizeof(DevCtl), cudaMemcpyHostToDevice, st));
  if (n)
    launch_tiny_count((const u64*)d_x, n, is_signed ? kSign : 0, ctx->d_ctl, ctx->num_sms, st,
                      kGateNone);
  ctx->launches += n ? 1 : 0;
  CKL();
  TRY(sync_ctl(ctx, st));
  for (int j = 0; j < nk; ++j) h_counts[j] = (int64_t)ctx->h_ctl->tiny_counts[c.tiny_slot[map[j]]];
  return CAFS_OK;
}

int cafs_count_pairs_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         uint64_t hash_mult, uint64_t* d_keys, uint64_t* d_counts, uint64_t cap,
                         uint64_t* h_npairs, void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!h_npairs || (hash_mult & 1) == 0) return fail(ctx, CAFS_EINVAL, "bad arguments");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  *h_npairs = 0;
  if (n == 0) return CAFS_OK;
  TRY(ensure_main(ctx));
  // the estimate kernel resets the per-call control block and sets the range window
  launch_estimate((const u64*)d_x, n, is_signed ? kSign : 0, 0, ctx->d_ctl, st);
  // both count shapes, each gated on the estimate's window (no host round trip)
  cudaError_t e = launch_hash_count((const u64*)d_x, n, is_signed ? kSign : 0, hash_mult,
                                    ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, 1,
                                    ctx->num_sms, st, 0, kGateDense, ctx->dense);
  if (e == cudaSuccess)
    e = launch_hash_count((const u64*)d_x, n, is_signed ? kSign : 0, hash_mult, ctx->d_ctl,
                          ctx->gkeys, ctx->gcnt, ctx->glist, 1, ctx->num_sms, st, 1, kGateHash,
                          ctx->dense);
  if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "hash_count", e);
  launch_compact(ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a,
                 ctx->num_sms, st, kGateNone);
  launch_dense_pairs(ctx->d_ctl, ctx->dense, ctx->pk_a, ctx->pc_a, ctx->pk_b, ctx->pc_b,
                     ctx->poffs, n, st, kGateNone);
  e = launch_small_sort_pairs(ctx->pk_a, ctx->pc_a, 0, ctx->d_ctl, n, ctx->pk_b, ctx->pc_b,
                              ctx->poffs, st, kGateNone);
  ctx->launches += 6;
  if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "pair sort", e);
  TRY(sync_ctl(ctx, st));
  DevCtl c = *ctx->h_ctl;
  if (c.overflow) {
    CK(cudaMemsetAsync(ctx->gkeys, 0xFF, kGlobalSlots * 8, st));
    CK(cudaMemsetAsync(ctx->gcnt, 0, kGlobalSlots * 8, st));
    CK(cudaStreamSynchronize(st));
    return fail(ctx, CAFS_EINVAL, "more distinct keys than the global table holds");
  }
  const u64 np = c.npairs;
  if (c.need_large) TRY(sort_pairs_large(ctx, np, st));
  *h_npairs = np;
  if (np > cap) return fail(ctx, CAFS_EINVAL, "output capacity too small");
  CK(cudaMemcpyAsync(d_keys, ctx->pk_b, np * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(d_counts, ctx->pc_b, np * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

int cafs_merge_pairs(cafs_ctx_t* ctx, const uint64_t* d_keys_in, const uint64_t* d_counts_in,
                     uint64_t m, uint64_t* d_keys, uint64_t* d_counts, uint64_t cap,
                     uint64_t* h_npairs, void* stream) {
  if (!ctx || !h_npairs || (m && (!d_keys_in || !d_counts_in))) return CAFS_EINVAL;
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  *h_npairs = 0;
  TRY(ensure_main(ctx));
  launch_insert_pairs((const u64*)d_keys_in, (const u64*)d_counts_in, m, CAFS_DEFAULT_HASH_MULT,
                      ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->num_sms, st);
  launch_compact(ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a,
                 ctx->num_sms, st, kGateNone);
  cudaError_t e = launch_small_sort_pairs(ctx->pk_a, ctx->pc_a, 0, ctx->d_ctl, ~0ull, ctx->pk_b,
                                          ctx->pc_b, ctx->poffs, st, kGateNone);
  ctx->launches += 4;
  if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "pair sort", e);
  CKL();
  TRY(sync_ctl(ctx, st));
  DevCtl c = *ctx->h_ctl;
  if (c.overflow) {
    CK(cudaMemsetAsync(ctx->gkeys, 0xFF, kGlobalSlots * 8, st));
    CK(cudaMemsetAsync(ctx->gcnt, 0, kGlobalSlots * 8, st));
    CK(cudaStreamSynchronize(st));
    return fail(ctx, CAFS_EINVAL, "more distinct keys than the global table holds");
  }
  const u64 np = c.npairs;
  if (c.need_large) TRY(sort_pairs_large(ctx, np, st));
  *h_npairs = np;
  if (np > cap) return fail(ctx, CAFS_EINVAL, "output capacity too small");
  CK(cudaMemcpyAsync(d_keys, ctx->pk_b, np * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(d_counts, ctx->pc_b, np * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

int cafs_pair_sort(cafs_ctx_t* ctx, uint64_t* d_keys, uint64_t* d_counts, uint64_t npairs,
                   void* stream) {
  if (!ctx) return CAFS_EINVAL;
  if (npairs > kGlobalCap) return fail(ctx, CAFS_EINVAL, "too many pairs");
  if (npairs < 2) return CAFS_OK;
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(ensure_main(ctx));
  if (npairs <= kSmallSortMax) {
    CK(cudaMemcpyAsync(ctx->pk_a, d_keys, npairs * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(ctx->pc_a, d_counts, npairs * 8, cudaMemcpyDeviceToDevice, st));
    cudaError_t e = launch_small_sort_pairs(ctx->pk_a, ctx->pc_a, npairs, nullptr, 0, (u64*)d_keys,
                                            (u64*)d_counts, ctx->poffs, st, kGateNone);
    ctx->launches++;
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "pair sort", e);
  } else {
    TRY(ensure_radix(ctx, npairs, false));
    u64 *rk, *rv;
    TRY(radix_sort(ctx, (u64*)d_keys, (u64*)d_counts, ctx->pk_b, ctx->pc_b, npairs, 0, st, &rk,
                   &rv));
    if (rk != (u64*)d_keys) {
      CK(cudaMemcpyAsync(d_keys, rk, npairs * 8, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(d_counts, rv, npairs * 8, cudaMemcpyDeviceToDevice, st));
    }
  }
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

int cafs_emit_i64(cafs_ctx_t* ctx, const uint64_t* d_keys, const uint64_t* d_counts,
                  uint64_t npairs, int64_t* d_out, uint64_t out_begin, uint64_t out_end,
                  uint64_t total, int is_signed, void* stream) {
  if (!ctx) return CAFS_EINVAL;
  if (out_begin > out_end || out_end > total || npairs > kGlobalCap)
    return fail(ctx, CAFS_EINVAL, "bad output slice");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(ensure_main(ctx));
  DevCtl& c = *ctx->h_ctl;
  memset(&c, 0, sizeof(c));
  CK(cudaMemcpyAsync(ctx->d_ctl, &c, sizeof(DevCtl), cudaMemcpyHostToDevice, st));
  launch_scan((const u64*)d_counts, npairs, ctx->bsum, ctx->poffs, ctx->d_ctl, total, st);
  ctx->launches += 3;
  if (npairs && out_end > out_begin) {
    launch_emit((const u64*)d_keys, ctx->poffs, 0, ctx->d_ctl, (u64*)d_out, out_begin, out_end,
                is_signed ? kSign : 0, ctx->num_sms, st, npairs);
    ctx->launches++;
  }
  CKL();
  TRY(sync_ctl(ctx, st));
  if (ctx->h_ctl->sum_error)
    return fail(ctx, CAFS_ESUM, "pair counts do not sum to the output length");
  return CAFS_OK;
}

int cafs_fallback_sort_i64(cafs_ctx_t* ctx, int64_t* d_x, uint64_t n, int is_signed,
                           void* stream) {
  TRY(check_common(ctx, d_x, n));
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(fallback_sort(ctx, (u64*)d_x, n, is_signed ? kSign : 0, st));
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

int cafs_key_span_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                      uint64_t* h_min, uint64_t* h_max, void* stream) {
  if (!h_min || !h_max) return CAFS_EINVAL;
  TRY(check_common(ctx, d_x, n));
  *h_min = ~0ull;
  *h_max = 0;
  if (n == 0) return CAFS_OK;
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(ensure_radix(ctx, n, false));
  launch_msd_span((const u64*)d_x, n, is_signed ? kSign : 0, ctx->msd, ctx->num_sms, st);
  ctx->launches++;
  CKL();
  CK(cudaMemcpyAsync(ctx->h_scratch, (char*)ctx->msd + msd_span_offset(), 16,
                     cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const u64* v = (const u64*)ctx->h_scratch;
  *h_min = v[0];
  *h_max = v[1];
  return CAFS_OK;
}

int cafs_partition_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                       uint64_t g_min, uint64_t g_max, int64_t* d_out, uint64_t* h_counts,
                       void* stream) {
  if (!h_counts || (n && !d_out)) return CAFS_EINVAL;
  TRY(check_common(ctx, d_x, n));
  if (n >> 32) return fail(ctx, CAFS_EINVAL, "partition: more than 2^32 keys per rank");
  for (int b = 0; b < CAFS_PARTITION_BUCKETS; ++b) h_counts[b] = 0;
  if (n == 0) return CAFS_OK;
  const u64 flip = is_signed ? kSign : 0;
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(ensure_radix(ctx, n, false));
  launch_msd_partition((const u64*)d_x, n, flip, ctx->msd, g_min, g_max, (u64*)d_out,
                       ctx->num_sms, st);
  ctx->launches += 4;
  CKL();
  const u32* hc = (const u32*)ctx->h_scratch;  // pinned, 64 + 4096 x 4 bytes
  cudaError_t e = cudaMemcpyAsync(ctx->h_scratch, (char*)ctx->msd + msd_hist_offset(),
                                  CAFS_PARTITION_BUCKETS * 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess)
    for (int b = 0; b < CAFS_PARTITION_BUCKETS; ++b) h_counts[b] = hc[b];
  if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "partition", e);
  return CAFS_OK;
}

uint64_t cafs_ctx_kernel_count(const cafs_ctx_t* ctx) { return ctx ? ctx->launches : 0; }

// After cafs_shard_finish_i64 returned status 1 on the main route: this shard's
// (key, count) pairs from the count phase, for the host-driven exchange and
// merge (sorted when they fitted the device pair sort).  *h_npairs = ~0 when
// they were lost to a global-table overflow (the guard).
int cafs_shard_local_pairs_i64(cafs_ctx_t* ctx, uint64_t* d_keys, uint64_t* d_counts,
                               uint64_t cap, uint64_t* h_npairs, void* stream) {
  if (!ctx || !h_npairs) return CAFS_EINVAL;
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(ensure_main(ctx));
  TRY(sync_ctl(ctx, st));
  const DevCtl& c = *ctx->h_ctl;
  if (c.local_overflow) { *h_npairs = ~0ull; return CAFS_OK; }
  const u64 np = c.local_npairs;
  *h_npairs = np;
  if (np > cap) return fail(ctx, CAFS_EINVAL, "output capacity too small");
  const u64* k = c.local_sorted ? ctx->pk_b : ctx->pk_a;
  const u64* v = c.local_sorted ? ctx->pc_b : ctx->pc_a;
  if (np) {
    CK(cudaMemcpyAsync(d_keys, k, np * 8, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(d_counts, v, np * 8, cudaMemcpyDeviceToDevice, st));
  }
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

// ---- stream-ordered sharded pipeline (shard.cu); no host synchronisation
// until cafs_shard_finish_i64 ----
int cafs_shard_begin_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         uint64_t* d_hdr, void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!d_hdr) return fail(ctx, CAFS_EINVAL, "null header buffer");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  launch_shard_header((const u64*)d_x, n, is_signed ? kSign : 0, (u64*)d_hdr, ctx->num_sms,
                      (cudaStream_t)stream);
  ctx->launches += 2;
  CKL();
  return CAFS_OK;
}

int cafs_shard_sample_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                          const uint64_t* d_hdr_all, int world, int rank, uint64_t* d_samples,
                          void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!d_hdr_all || !d_samples || world < 1 || rank < 0 || rank >= world)
    return fail(ctx, CAFS_EINVAL, "bad shard arguments");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  TRY(ensure_main(ctx));
  launch_shard_samples((const u64*)d_x, n, is_signed ? kSign : 0, (const u64*)d_hdr_all, world,
                       rank, (u64*)d_samples, ctx->d_ctl, (cudaStream_t)stream);
  ctx->launches++;
  CKL();
  return CAFS_OK;
}

int cafs_shard_count_i64(cafs_ctx_t* ctx, const int64_t* d_x, uint64_t n, int is_signed,
                         uint64_t hash_mult, const uint64_t* d_hdr_all, int world,
                         const uint64_t* d_samples, uint64_t* d_tiny, uint64_t* d_send,
                         uint64_t cap, void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!d_hdr_all || !d_samples || !d_tiny || !d_send || world < 1 || (hash_mult & 1) == 0)
    return fail(ctx, CAFS_EINVAL, "bad shard arguments");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  TRY(ensure_main(ctx));
  return shard_count_enqueue(ctx, (const u64*)d_x, n, is_signed ? kSign : 0, hash_mult,
                             (const u64*)d_hdr_all, world, (const u64*)d_samples, (u64*)d_tiny,
                             (u64*)d_send, cap, (cudaStream_t)stream);
}

int cafs_shard_finish_i64(cafs_ctx_t* ctx, int64_t* d_x, uint64_t n, int is_signed,
                          const uint64_t* d_tiny_sum, const uint64_t* d_recv, int world,
                          uint64_t cap, cafs_telemetry_t* tel, int* h_status, void* stream) {
  TRY(check_common(ctx, d_x, n));
  if (!d_tiny_sum || !d_recv || !h_status || world < 1)
    return fail(ctx, CAFS_EINVAL, "bad shard arguments");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(ensure_main(ctx));
  TRY(shard_finish_enqueue(ctx, (u64*)d_x, n, is_signed ? kSign : 0, (const u64*)d_tiny_sum,
                           (const u64*)d_recv, world, cap, 1 + 2 * cap, st));
  TRY(sync_ctl(ctx, st));
  return shard_result(ctx, (u64*)d_x, n, is_signed ? kSign : 0, tel, h_status, st);
}

int cafs_gen_mix(uint64_t* d_out, uint64_t count, uint64_t seed, uint64_t skip, void* stream) {
  if (count && !d_out) return CAFS_EINVAL;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (count) launch_gen_mix((u64*)d_out, count, seed, skip, sms, (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? CAFS_OK : CAFS_ECUDA;
}

int cafs_gen_draw(int64_t* d_out, uint64_t n, uint64_t start, uint64_t seed,
                  const int64_t* d_palette, uint64_t k, const double* d_cdf, void* stream) {
  if ((n && !d_out) || k == 0 || k >= (1ull << 32)) return CAFS_EINVAL;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (n)
    launch_gen_draw((u64*)d_out, n, start, seed, (const u64*)d_palette, k, d_cdf, sms,
                    (cudaStream_t)stream);
  return cudaGetLastError() == cudaSuccess ? CAFS_OK : CAFS_ECUDA;
}


// ---- native multi-GPU sort: the library's own NCCL communicator ----
// One call enqueues the whole stream-ordered sharded pipeline (shard.cu
// phases + three NCCL collectives over NVLink/NVSwitch), captured once per
// (column, rows, flags) as a CUDA graph with the collectives inside, then
// replayed: one graph launch and one host synchronisation per call.

struct cafs_comm_t {
  ncclComm_t nc = nullptr;
  int world = 0, rank = 0, device = 0;
  u64 cap = 0, row = 0;  // pairs per rank in the exchange; words per gathered row
  u64 *hdr = nullptr, *hdr_all = nullptr, *samples = nullptr, *send = nullptr, *recv = nullptr,
      *tiny_sum = nullptr;
  struct Graph {
    u64 x = 0, n = 0, flip = 0, mult = 0;
    int seen = 0;
    uint64_t launches = 0, stamp = 0;
    uint64_t gen = 0;  // the context's buf_gen at capture
    int kk = 0;        // key kind
    uint32_t cls = 0;  // route classes whose kernels the graph holds
    cudaGraphExec_t exec = nullptr;
  } graphs[8];
  uint64_t clock = 0;
  // the route classes the next call's pipeline holds: one class after two
  // columns of that class in a row, else all (the same on every rank)
  uint32_t pred = 7, last_cls = 0;
  int sum_penalty = 0;  // calls left before the window class's sum pipeline is tried again
  // distributed fallback (sharded_fallback): global span, every rank's bucket
  // counts, this shard partitioned by bucket, the buckets received
  u64* fb_span = nullptr;
  u32* fb_counts = nullptr;
  u32* h_counts = nullptr;  // pinned mirror of fb_counts
  u64 *fb_part = nullptr, *fb_recv = nullptr;
  u64 fb_part_len = 0, fb_recv_len = 0;
};

int cafs_nccl_unique_id(unsigned char* out) {
  if (!out) return CAFS_EINVAL;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CAFS_ECUDA;
  static_assert(sizeof(id) == CAFS_NCCL_ID_BYTES, "ncclUniqueId size");
  memcpy(out, &id, sizeof(id));
  return CAFS_OK;
}

int cafs_comm_destroy(cafs_comm_t* comm) {
  if (!comm) return CAFS_OK;
  DeviceGuard g(comm->device);
  for (auto& g : comm->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (comm->nc) ncclCommDestroy(comm->nc);
  for (u64* p : {comm->hdr, comm->hdr_all, comm->samples, comm->send, comm->recv, comm->tiny_sum,
                 comm->fb_span, (u64*)comm->fb_counts, comm->fb_part, comm->fb_recv})
    if (p) cudaFree(p);
  if (comm->h_counts) cudaFreeHost(comm->h_counts);
  delete comm;
  return CAFS_OK;
}

int cafs_comm_create(int device, const unsigned char* id, int world, int rank,
                     cafs_comm_t** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return CAFS_EINVAL;
  *out = nullptr;
  DeviceGuard g(device);
  cafs_comm_t* c = new (std::nothrow) cafs_comm_t();
  if (!c) return CAFS_ENOMEM;
  c->world = world;
  c->rank = rank;
  c->device = device;
  c->cap = CAFS_SHARD_PAIR_CAP;
  c->row = 1 + 2 * c->cap + CAFS_SHARD_TINY_WORDS;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  if (ncclCommInitRank(&c->nc, world, uid, rank) != ncclSuccess) {
    c->nc = nullptr;
    cafs_comm_destroy(c);
    return CAFS_ECUDA;
  }
  if (cudaMalloc(&c->hdr, kShardHdrWords * 8) != cudaSuccess ||
      cudaMalloc(&c->hdr_all, (size_t)world * kShardHdrWords * 8) != cudaSuccess ||
      cudaMalloc(&c->samples, kSampleTarget * 8) != cudaSuccess ||
      cudaMalloc(&c->send, c->row * 8) != cudaSuccess ||
      cudaMalloc(&c->recv, (size_t)world * c->row * 8) != cudaSuccess ||
      cudaMalloc(&c->tiny_sum, CAFS_SHARD_TINY_WORDS * 8) != cudaSuccess ||
      cudaMemset(c->send, 0, c->row * 8) != cudaSuccess) {  // unused tiny words stay 0
    cafs_comm_destroy(c);
    return CAFS_ENOMEM;
  }
  *out = c;
  return CAFS_OK;
}

}  // extern "C"

extern "C" int cafs_shard_fallback_plan(int world, int rank, const uint32_t* counts,
                                        uint64_t* send_at, uint64_t* send_n, uint64_t* recv_n,
                                        uint64_t* start) {
  if (world < 1 || rank < 0 || rank >= world || !counts || !send_at || !send_n || !recv_n || !start)
    return CAFS_EINVAL;
  constexpr int B = CAFS_PARTITION_BUCKETS;
  const int W = world, me = rank;
  // rows of the sorted column before bucket b, and every rank's rows
  std::vector<u64> P(B + 1, 0), rows(W, 0);
  // L[r][b]: rows of rank r's partitioned shard before bucket b
  std::vector<u64> L((size_t)W * (B + 1), 0);
  for (int r = 0; r < W; ++r)
    for (int b = 0; b < B; ++b)
      L[(size_t)r * (B + 1) + b + 1] = L[(size_t)r * (B + 1) + b] + counts[(size_t)r * B + b];
  for (int r = 0; r < W; ++r) rows[r] = L[(size_t)r * (B + 1) + B];
  for (int b = 0; b < B; ++b) {
    u64 t = 0;
    for (int r = 0; r < W; ++r) t += counts[(size_t)r * B + b];
    P[b + 1] = P[b] + t;
  }
  // the bucket range [lo, hi) overlapping rank d's rows [off_d, off_d + n_d): a
  // bucket straddling two ranks' rows is in both ranges
  std::vector<int> lo(W, 0), hi(W, 0);
  u64 off = 0, my_off = 0;
  for (int d = 0; d < W; ++d) {
    if (d == me) my_off = off;
    if (rows[d]) {
      lo[d] = (int)(std::upper_bound(P.begin() + 1, P.end(), off) - (P.begin() + 1));
      hi[d] = (int)(std::lower_bound(P.begin(), P.end() - 1, off + rows[d]) - P.begin());
    }
    off += rows[d];
  }
  for (int d = 0; d < W; ++d) {
    send_at[d] = L[(size_t)me * (B + 1) + lo[d]];
    send_n[d] = L[(size_t)me * (B + 1) + hi[d]] - send_at[d];
    recv_n[d] = L[(size_t)d * (B + 1) + hi[me]] - L[(size_t)d * (B + 1) + lo[me]];
  }
  *start = rows[me] ? my_off - P[lo[me]] : 0;
  return CAFS_OK;
}

namespace {

// largest exchange row (pairs per rank) the native sharded sort grows to; a
// longer list continues on the host-driven path
constexpr u64 kShardCapMax = 1ull << 20;

// the pair tables' all-gather, the merge and this rank's slice emit; again
// (from_local) after the row grew: the rows are re-packed from the count's pairs
int sharded_exchange(cafs_ctx_t* ctx, cafs_comm_t* cm, void* x, u64 n, u64 flip, cudaStream_t st,
                     int from_local, int kk, uint32_t cls) {
  const u64 cap = cm->cap, row = cm->row, tiny_off = 1 + 2 * cap;
  if (from_local) {
    launch_shard_pack_pairs(ctx->d_ctl, ctx->pk_b, ctx->pc_b, cm->send, cap, st, 1);
    ctx->launches++;
  }
  if (ncclAllGather(cm->send, cm->recv, row, ncclUint64, cm->nc, st) != ncclSuccess)
    return fail(ctx, CAFS_ECUDA, "ncclAllGather (pair tables)");
  if (cls & kClsTiny) {
    launch_shard_tiny_gather(cm->recv, cm->world, row, tiny_off, cm->tiny_sum, st);
    ctx->launches++;
  }
  TRY(shard_finish_enqueue(ctx, x, n, flip, cm->tiny_sum, cm->recv, cm->world, cap, row, st, kk,
                           cls));
  CK(cudaMemcpyAsync(ctx->h_ctl, ctx->d_ctl, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
  CKL();
  return CAFS_OK;
}

// a larger exchange row for this communicator (the captured graphs go)
int comm_resize(cafs_ctx_t* ctx, cafs_comm_t* c, u64 cap) {
  CK(cudaDeviceSynchronize());
  for (auto& g : c->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g = cafs_comm_t::Graph();
  }
  if (c->send) CK(cudaFree(c->send));
  if (c->recv) CK(cudaFree(c->recv));
  c->send = c->recv = nullptr;
  c->cap = cap;
  c->row = 1 + 2 * cap + CAFS_SHARD_TINY_WORDS;
  CK(cudaMalloc(&c->send, c->row * 8));
  CK(cudaMalloc(&c->recv, (size_t)c->world * c->row * 8));
  CK(cudaMemset(c->send, 0, c->row * 8));
  return CAFS_OK;
}

int sharded_enqueue(cafs_ctx_t* ctx, cafs_comm_t* cm, void* x, u64 n, u64 flip, u64 mult,
                    cudaStream_t st, int kk, uint32_t cls, int est_opts = 0) {
  const u64 cap = cm->cap, row = cm->row, tiny_off = 1 + 2 * cap;
  launch_shard_header(x, n, flip, cm->hdr, ctx->num_sms, st, kk);
  if (ncclAllGather(cm->hdr, cm->hdr_all, kShardHdrWords, ncclUint64, cm->nc, st) != ncclSuccess)
    return fail(ctx, CAFS_ECUDA, "ncclAllGather (headers)");
  launch_shard_samples(x, n, flip, cm->hdr_all, cm->world, cm->rank, cm->samples, ctx->d_ctl, st,
                       kk);
  if (ncclAllReduce(cm->samples, cm->samples, kSampleTarget, ncclUint64, ncclSum, cm->nc, st) !=
      ncclSuccess)
    return fail(ctx, CAFS_ECUDA, "ncclAllReduce (samples)");
  if (cls == kClsWindowSum) {
    DevCtl* c = ctx->d_ctl;
    launch_estimate_sharded(cm->samples, cm->hdr_all, cm->world, c, st, est_opts);
    cudaError_t e = launch_hash_count(x, n, flip, mult, c, ctx->gkeys, ctx->gcnt, ctx->glist, 1,
                                      ctx->num_sms, st, 0, kGateMainDense, ctx->dense, kk);
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "hash_count", e);
    if (ncclAllReduce(ctx->dense, ctx->dense, dense_window_len(), ncclUint64, ncclSum, cm->nc,
                      st) != ncclSuccess)
      return fail(ctx, CAFS_ECUDA, "ncclAllReduce (window counts)");
    // the summed counts -> the column's sorted pairs and offsets on every rank
    launch_dense_pairs(c, ctx->dense, ctx->pk_a, ctx->pc_a, ctx->pk_b, ctx->pc_b, ctx->poffs,
                       ~0ull, st, kGateMainDense);
    launch_emit(ctx->pk_b, ctx->poffs, 0, c, x, 0, n, flip, ctx->num_sms, st, 0, kk, true);
    CK(cudaMemcpyAsync(ctx->h_ctl, c, sizeof(DevCtl), cudaMemcpyDeviceToHost, st));
    ctx->launches += 7;  // header (2), samples, estimate, count, pairs, emit
    CKL();
    return CAFS_OK;
  }
  TRY(shard_count_enqueue(ctx, x, n, flip, mult, cm->hdr_all, cm->world, cm->samples,
                          cm->send + tiny_off, cm->send, cap, st, kk, cls, est_opts));
  ctx->launches += 3;  // header (2), samples
  return sharded_exchange(ctx, cm, x, n, flip, st, 0, kk, cls);
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

// The distributed fallback inside the library (fallback_sort, sorter.py:132-138,
// over row shards), on the communicator's own NCCL ranks:
//   1. the column's key span: all-reduce (min, max) of the shards' spans;
//   2. this shard grouped into 4096 buckets by (key - min) >> shift -- the same
//      digit on every rank, so bucket b precedes bucket b + 1 in the sorted
//      column -- and an all-gather of every rank's bucket counts;
//   3. each rank receives, from every rank, the buckets that overlap its rows
//      of the sorted column (grouped ncclSend / ncclRecv of contiguous bucket
//      ranges; a bucket straddling two ranks' rows goes to both), sorts them
//      with the single-GPU fallback and keeps its rows.
// ~8 B per key cross NVLink once; every rank sorts ~1/world of the column.
// Two host synchronisations (span, counts): the transfer sizes are data.
int sharded_fallback(cafs_ctx_t* ctx, cafs_comm_t* cm, u64* x, u64 n, u64 flip, cudaStream_t st) {
  const int W = cm->world, me = cm->rank;
  constexpr int B = CAFS_PARTITION_BUCKETS;
  if (!cm->fb_span) {
    CK(cudaMalloc(&cm->fb_span, 4 * 8));
    CK(cudaMalloc(&cm->fb_counts, (size_t)W * B * 4));
    CK(cudaMallocHost(&cm->h_counts, (size_t)W * B * 4 + 32));
  }
  TRY(ensure_radix(ctx, n ? n : 1, false));
  // 1. span (an empty shard contributes [~0, 0])
  u64* loc = cm->fb_span + 2;
  if (n) {
    launch_msd_span(x, n, flip, ctx->msd, ctx->num_sms, st);
    ctx->launches++;
    CKL();
    CK(cudaMemcpyAsync(loc, (char*)ctx->msd + msd_span_offset(), 16, cudaMemcpyDeviceToDevice, st));
  } else {
    CK(cudaMemsetAsync(loc, 0xFF, 8, st));
    CK(cudaMemsetAsync(loc + 1, 0, 8, st));
  }
  if (ncclGroupStart() != ncclSuccess ||
      ncclAllReduce(loc, cm->fb_span, 1, ncclUint64, ncclMin, cm->nc, st) != ncclSuccess ||
      ncclAllReduce(loc + 1, cm->fb_span + 1, 1, ncclUint64, ncclMax, cm->nc, st) != ncclSuccess ||
      ncclGroupEnd() != ncclSuccess)
    return fail(ctx, CAFS_ECUDA, "ncclAllReduce (key span)");
  u64* hs = (u64*)((char*)cm->h_counts + (size_t)W * B * 4);
  CK(cudaMemcpyAsync(hs, cm->fb_span, 16, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const u64 g_min = hs[0], g_max = hs[1];
  // 2. partition and every rank's bucket counts
  if (n > cm->fb_part_len) {
    if (cm->fb_part) CK(cudaFree(cm->fb_part));
    cm->fb_part = nullptr;
    cm->fb_part_len = 0;
    CK(cudaMalloc(&cm->fb_part, n * 8));
    cm->fb_part_len = n;
  }
  u32* hist = (u32*)((char*)ctx->msd + msd_hist_offset());
  if (n) {
    launch_msd_partition(x, n, flip, ctx->msd, g_min, g_max, cm->fb_part, ctx->num_sms, st);
    ctx->launches += 4;
    CKL();
  } else {
    CK(cudaMemsetAsync(hist, 0, B * 4, st));
  }
  if (ncclAllGather(hist, cm->fb_counts, B, ncclUint32, cm->nc, st) != ncclSuccess)
    return fail(ctx, CAFS_ECUDA, "ncclAllGather (bucket counts)");
  CK(cudaMemcpyAsync(cm->h_counts, cm->fb_counts, (size_t)W * B * 4, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::vector<uint64_t> send_at(W), send_n(W), recv_n(W), recv_at(W + 1, 0);
  uint64_t start = 0;
  if (cafs_shard_fallback_plan(W, me, cm->h_counts, send_at.data(), send_n.data(), recv_n.data(),
                               &start) != CAFS_OK)
    return fail(ctx, CAFS_EINTERNAL, "sharded fallback: plan");
  u64 mine = 0;
  for (int b = 0; b < B; ++b) mine += cm->h_counts[(size_t)me * B + b];
  if (mine != n) return fail(ctx, CAFS_EINTERNAL, "sharded fallback: bucket counts");
  for (int r = 0; r < W; ++r) recv_at[r + 1] = recv_at[r] + recv_n[r];
  const u64 R = recv_at[W];
  if (R > cm->fb_recv_len) {
    if (cm->fb_recv) CK(cudaFree(cm->fb_recv));
    cm->fb_recv = nullptr;
    cm->fb_recv_len = 0;
    CK(cudaMalloc(&cm->fb_recv, R * 8));
    cm->fb_recv_len = R;
  }
  // 3. the exchange: contiguous bucket ranges of the partitioned shard
  if (ncclGroupStart() != ncclSuccess) return fail(ctx, CAFS_ECUDA, "ncclGroupStart");
  bool nccl_ok = true;
  for (int d = 0; d < W; ++d) {
    const u64 a = send_at[d], cnt = send_n[d];
    if (d == me) {
      if (cnt)
        CK(cudaMemcpyAsync(cm->fb_recv + recv_at[me], cm->fb_part + a, cnt * 8,
                           cudaMemcpyDeviceToDevice, st));
      continue;
    }
    if (cnt) nccl_ok &= ncclSend(cm->fb_part + a, cnt, ncclUint64, d, cm->nc, st) == ncclSuccess;
    if (recv_n[d])
      nccl_ok &= ncclRecv(cm->fb_recv + recv_at[d], recv_n[d], ncclUint64, d, cm->nc, st) ==
                 ncclSuccess;
  }
  if (ncclGroupEnd() != ncclSuccess || !nccl_ok)
    return fail(ctx, CAFS_ECUDA, "ncclSend / ncclRecv (bucket ranges)");
  if (n == 0) return CAFS_OK;
  // the received buckets sorted; this rank's rows start at `start`
  TRY(fallback_sort(ctx, cm->fb_recv, R, flip, st));
  if (start + n > R) return fail(ctx, CAFS_EINTERNAL, "sharded fallback: slice outside the received rows");
  CK(cudaMemcpyAsync(x, cm->fb_recv + start, n * 8, cudaMemcpyDeviceToDevice, st));
  CK(cudaStreamSynchronize(st));
  return CAFS_OK;
}

static int sharded_impl(cafs_ctx_t* ctx, cafs_comm_t* comm, void* d_x, uint64_t n, int is_signed,
                        uint64_t hash_mult, cafs_telemetry_t* tel, int* h_status, void* stream,
                        int kk) {
  TRY(check_common(ctx, d_x, n, kk ? 4 : 8));
  if (!comm || !h_status || (hash_mult & 1) == 0) return fail(ctx, CAFS_EINVAL, "bad arguments");
  if (comm->device != ctx->device) return fail(ctx, CAFS_EINVAL, "comm and context devices differ");
  DeviceGuard g(ctx->device);
  CallGuard cg(ctx, stream);
  cudaStream_t st = (cudaStream_t)stream;
  TRY(ensure_main(ctx));
  const u64 flip = (is_signed || kk) ? kSign : 0;
  void* x = d_x;
  static int use_graphs = -1;
  if (use_graphs < 0) {
    const char* e = getenv("CAFS_GRAPHS");
    use_graphs = e ? atoi(e) != 0 : 1;
  }
  static int predict = -1;  // CAFS_SHARD_PREDICT=0: every call holds every class's kernels
  if (predict < 0) {
    const char* e = getenv("CAFS_SHARD_PREDICT");
    predict = e ? atoi(e) != 0 : 1;
  }
  uint32_t used = predict ? comm->pred : (uint32_t)kClsAll;
  if (used == kClsWindow && comm->sum_penalty == 0) used = kClsWindowSum;
  if (comm->sum_penalty > 0) --comm->sum_penalty;
  cafs_comm_t::Graph* hit = nullptr;
  cafs_comm_t::Graph* lru = &comm->graphs[0];
  for (auto& gr : comm->graphs) {
    if (gr.seen && gr.x == (u64)x && gr.n == n && gr.flip == flip && gr.mult == hash_mult &&
        gr.kk == kk && gr.cls == used) {
      hit = &gr;
      if (gr.exec && gr.gen != ctx->buf_gen) {  // captured before a buffer moved
        cudaGraphExecDestroy(gr.exec);
        gr.exec = nullptr;
      }
      break;
    }
    if (gr.stamp < lru->stamp) lru = &gr;
  }
  if (!use_graphs || !ctx->cap_stream) {
    TRY(sharded_enqueue(ctx, comm, x, n, flip, hash_mult, st, kk, used));
  } else if (hit && hit->exec) {  // replay
    CK(cudaGraphLaunch(hit->exec, st));
    ctx->launches += hit->launches;
    hit->stamp = ++comm->clock;
  } else if (!hit) {  // first sighting: direct, capture next time
    if (lru->exec) cudaGraphExecDestroy(lru->exec);
    *lru = cafs_comm_t::Graph();
    lru->x = (u64)x; lru->n = n; lru->flip = flip; lru->mult = hash_mult;
    lru->seen = 1; lru->stamp = ++comm->clock; lru->kk = kk; lru->cls = used;
    TRY(sharded_enqueue(ctx, comm, x, n, flip, hash_mult, st, kk, used));
  } else {  // second sighting: capture on the context's stream, launch on the caller's
    const uint64_t l0 = ctx->launches;
    cudaGraph_t graph = nullptr;
    CK(cudaStreamBeginCapture(ctx->cap_stream, cudaStreamCaptureModeThreadLocal));
    const int rc = sharded_enqueue(ctx, comm, x, n, flip, hash_mult, ctx->cap_stream, kk, used);
    cudaError_t e = cudaStreamEndCapture(ctx->cap_stream, &graph);
    if (rc != CAFS_OK) { if (graph) cudaGraphDestroy(graph); return rc; }
    if (e != cudaSuccess) return fail(ctx, CAFS_ECUDA, "graph capture (sharded)", e);
    e = cudaGraphInstantiate(&hit->exec, graph, 0);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) { hit->exec = nullptr; return fail(ctx, CAFS_ECUDA, "graph instantiate", e); }
    hit->launches = ctx->launches - l0;
    hit->stamp = ++comm->clock;
    hit->gen = ctx->buf_gen;
    CK(cudaGraphLaunch(hit->exec, st));
  }
  CK(cudaStreamSynchronize(st));
  const DevCtl& h = *ctx->h_ctl;
  {
    uint32_t now = shard_class(h);
    bool redo = now & ~(used == kClsWindowSum ? (uint32_t)kClsWindow : used);
    if (used == kClsWindowSum && now == kClsWindow && !h.pairs_ready) {
      // the summed window counts are short: a rank met keys outside the window
      // (they sit in its global table) or lost its table -- clean up, and use
      // the pair-table pipeline for this communicator's next columns
      if (h.overflow) {
        CK(cudaMemsetAsync(ctx->gkeys, 0xFF, kGlobalSlots * 8, st));
        CK(cudaMemsetAsync(ctx->gcnt, 0, kGlobalSlots * 8, st));
      } else {
        launch_compact(ctx->d_ctl, ctx->gkeys, ctx->gcnt, ctx->glist, ctx->pk_a, ctx->pc_a,
                       ctx->num_sms, st, kGateNone);
        ctx->launches++;
      }
      comm->sum_penalty = 32;
      redo = true;
    }
    if (redo) {
      // the prediction left this column's class out (on every rank alike):
      // all re-run the full pipeline, collectives included
      used = kClsAll;
      TRY(sharded_enqueue(ctx, comm, x, n, flip, hash_mult, st, kk, used));
      CK(cudaStreamSynchronize(st));
      now = shard_class(h);
    }
    if (now) {
      comm->pred = now == comm->last_cls ? now : (uint32_t)kClsAll;
      comm->last_cls = now;
    }
  }
  bool tiny_retry = false;
  if (h.eff_route == CAFS_TINY_COUNT && h.tiny_failed) {
    // some rank met a value the sample missed (every rank sees it in the
    // gathered counters): MAIN with the same estimate (sorter.py:378-385), the
    // full pipeline again with the route forced
    used = kClsAll;
    TRY(sharded_enqueue(ctx, comm, x, n, flip, hash_mult, st, kk, used, kEstForceMain));
    CK(cudaStreamSynchronize(st));
    tiny_retry = true;
  }
  if (h.eff_route == CAFS_MAIN && h.merge_bad && h.shard_grow > comm->cap &&
      h.shard_grow <= kShardCapMax) {
    // some rank's sorted pairs did not fit the exchange row: every rank saw it
    // in the same gathered rows, so all grow the row and exchange again from
    // the pairs their count left on device (later calls use the larger row)
    u64 cap = comm->cap;
    while (cap < h.shard_grow) cap <<= 1;
    TRY(comm_resize(ctx, comm, cap));
    TRY(sharded_exchange(ctx, comm, x, n, flip, st, 1, kk, used));
    CK(cudaStreamSynchronize(st));
  }
  TRY(shard_result(ctx, x, n, flip, tel, h_status, st, kk));
  if (tiny_retry && tel) tel->tiny_count_failed = 1;
  static int native_fb = -1;  // CAFS_SHARD_FALLBACK=0: fallback columns return status 1
  if (native_fb < 0) {
    const char* e = getenv("CAFS_SHARD_FALLBACK");
    native_fb = e ? atoi(e) != 0 : 1;
  }
  const int eff = ctx->h_ctl->eff_route;
  if (*h_status == 1 && native_fb &&
      (eff == CAFS_FALLBACK_SMALL_N || eff == CAFS_FALLBACK_HIGH_ENTROPY || eff == CAFS_MAIN)) {
    // the dispatcher's fallback branch (every rank takes it: the route is
    // global) -- and a main-route column whose tables the device could not
    // merge (a rank's lost table: the guard, sorter.py:264-273; a list over
    // 2^20 pairs; a merge partition over 2048 keys): every rank saw that in
    // the same gathered rows and its shard is intact (shard_result rebuilt a
    // shard the partitioned count spilled into), so the column is exchanged
    // and sorted like a fallback column
    if (kk == 0) {
      TRY(sharded_fallback(ctx, comm, (u64*)x, n, flip, st));
    } else {
      // 4-byte shards: exchanged and sorted as their order-preserving 64-bit
      // widening (like the single-GPU fallback of 4-byte columns)
      if (n > ctx->wide_elems) {
        if (ctx->wide) CK(cudaFree(ctx->wide));
        ctx->wide = nullptr;
        ctx->wide_elems = 0;
        CK(cudaMalloc(&ctx->wide, (n ? n : 1) * 8));
        ctx->wide_elems = n ? n : 1;
      }
      if (n) launch_widen(x, n, kk, ctx->wide, ctx->num_sms, st);
      TRY(sharded_fallback(ctx, comm, ctx->wide, n, kSign, st));
      if (n) {
        launch_narrow(ctx->wide, n, kk, x, ctx->num_sms, st);
        ctx->launches += 2;
        CKL();
        CK(cudaStreamSynchronize(st));
      }
    }
    *h_status = 0;
  }
  return CAFS_OK;
}

}  // namespace

extern "C" {

int cafs_sort_i64_sharded(cafs_ctx_t* ctx, cafs_comm_t* comm, int64_t* d_x, uint64_t n,
                          int is_signed, uint64_t hash_mult, cafs_telemetry_t* tel, int* h_status,
                          void* stream) {
  return sharded_impl(ctx, comm, d_x, n, is_signed, hash_mult, tel, h_status, stream, 0);
}

int cafs_sort_i32_sharded(cafs_ctx_t* ctx, cafs_comm_t* comm, int32_t* d_x, uint64_t n,
                          int is_signed, uint64_t hash_mult, cafs_telemetry_t* tel, int* h_status,
                          void* stream) {
  return sharded_impl(ctx, comm, d_x, n, is_signed, hash_mult, tel, h_status, stream,
                      is_signed ? 1 : 2);
}

}  // extern "C"
