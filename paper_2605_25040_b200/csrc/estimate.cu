// estimate.cu -- K0 monotone probe + K1 Chao1 cardinality estimate and route.
//
// One CTA of 1024 threads replaces the reference's dispatch pre-pass
// (sorter.py:141-162):
//   * is_monotone (sorter.py:115-129): the first kMonoPrefix rows are checked
//     here; only a prefix that is already sorted triggers the full-array scan
//     kernel below (random inputs pay ~0 extra bytes);
//   * _sample (cardinality.py:99-110): samples x[i * (n // 1024)], i < 1024;
//   * FreqSet spectrum (cardinality.py:31-73): a 2048-slot linear
//     probing table of the multiplicative hash (the reference: 4096), built in smem
//     by all 1024 samples at once (CAS claims).  Concurrent insertion can place
//     a key in a different slot than the sequential reference, but
//     (u, f1, f2) and the sorted distinct keys are hash- and order-independent
//     (the reference's own test, tests/test_cardinality.py:139-152);
//   * chao1 (cardinality.py:85-96) in IEEE float64 with explicit _rn ops;
//   * route chain of sorter.py:153-162 and, for the tiny route, the ascending
//     distinct sampled keys (FreqSet.distinct_keys).
// It also derives two B200-side parameters from the sorted sample: a perfect
// hash for the <= 8 tiny keys and the dense-range window of the main count.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr u32 kRangeCap = 8192;  // dense direct-count window (must match hashcount.cu)

__device__ __forceinline__ int warp_incl_max(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = max(v, t);
  }
  return v;
}

__device__ __forceinline__ int warp_incl_sum(int v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

__device__ __forceinline__ u64 warp_min_u64(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t < v ? t : v;
  }
  return v;
}
__device__ __forceinline__ u64 warp_max_u64(u64 v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 t = __shfl_xor_sync(0xffffffffu, v, o);
    v = t > v ? t : v;
  }
  return v;
}

constexpr int kFreqSlots = 2048;  // <= 50% load for 1024 samples (reference: 4096, cardinality.py:27)

// Phase A runs on kEstCtas CTAs: each loads its 1024 / kEstCtas samples and
// checks its stretch of the prefix, so the ~140 KB of scattered reads take one
// DRAM round trip per SM instead of ~16 on one SM.  The last CTA to arrive
// (threadfence + arrival counter, self-resetting) runs phase B: FreqSet,
// spectrum, Chao1, route.
constexpr int kEstCtas = 16;

template <int KK>
__global__ void __launch_bounds__(1024, 1)
    estimate_kernel(const typename KeyT<KK>::T* __restrict__ x, u64 n, u64 flip, int check_prefix,
                    DevCtl* ctl, const u64* __restrict__ ghdr, int world, int opts) {
  // ghdr != null: sharded mode -- x holds the 1024 all-reduced samples
  // (order-mapped, flip 0) and the column's rows, monotone state and N come
  // from the all-gathered shard headers (kShardHdrWords words per rank)
  using K = typename KeyT<KK>::T;
  __shared__ u64 fkeys[kFreqSlots];
  __shared__ u32 fcnt[kFreqSlots];
  __shared__ u64 rmin[32], rmax[32];
  __shared__ long long red[3][32];
  __shared__ u32 n_max_key;  // occurrences of the sentinel value ~0 among the samples
  __shared__ int am_last, inv;
  __shared__ int best_t;
  __shared__ u32 nlist;
  __shared__ u64 klist[CAFS_TINY_MAX_KEYS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  pdl_begin();
  EstScratch* es = est_scratch(ctl);
  u64 nn = n;  // rows of the column
  if (ghdr) {
    nn = 0;
    for (int r = 0; r < world; ++r) nn += ghdr[r * kShardHdrWords];
  }
  const u64 m = nn < (u64)kSampleTarget ? nn : (u64)kSampleTarget;
  u64 stride = ghdr ? 1 : n / kSampleTarget;
  if (stride < 1) stride = 1;

  // ---- phase A (every CTA): this CTA's strided samples (cardinality.py:102-104)
  // and its (x[r], x[r+1]) pairs of the reference's first chunk (sorter.py:115-129),
  // all loads in flight together ----
  const int G = gridDim.x;
  const int per = kSampleTarget / G;
  u64 sv = 0;
  const u64 si = (u64)blockIdx.x * per + tid;
  if (tid < per && si < m) sv = key_map<KK>(x[si * stride], flip);
  int found = 0;
  if (check_prefix) {
    const u64 P = n < kMonoPrefix ? n : kMonoPrefix;
    for (u64 r = (u64)blockIdx.x * 1024 + tid; r + 1 < P; r += (u64)G * 1024)
      found |= key_map<KK>(x[r + 1], flip) < key_map<KK>(x[r], flip);
  }
  if (tid < per) {  // publish (only the writers fence: a fence costs ~1k cycles)
    __stcg(&es->samples[si], sv);
    __threadfence();
  }
  found = __syncthreads_or(found);
  if (tid == 0) {  // arrivals in the low 16 bits, CTAs that saw an inversion above
    const u32 old = atomicAdd(&es->arrive, 1u + (found ? 0x10000u : 0u));
    am_last = (old & 0xffffu) == (u32)(G - 1);
    inv = (old >> 16) + (u32)found > 0;
  }
  __syncthreads();
  if (!am_last) return;

  // ---- phase B (the last CTA) ----
  for (int i = tid; i < kFreqSlots; i += 1024) { fkeys[i] = kEmpty; fcnt[i] = 0; }
  if (tid == 0) {
    best_t = 0x7fffffff;
    n_max_key = 0;
    nlist = 0;
    // per-call state of the later stages
    ctl->scan_inversion = 0;
    ctl->tiny_miss = 0;
    ctl->g_updates = 0;
    ctl->empty_key_count = 0;
    ctl->overflow = 0;
    ctl->need_large = 0;
    ctl->need_compact = 0;
    ctl->npairs = 0;
    ctl->total = 0;
    ctl->pairs_ready = 0;
    ctl->sum_error = 0;
    ctl->tiny_failed = 0;
    ctl->tiny_done = 0;
    ctl->dense_outside = 0;
    ctl->hp_overflow = 0;
    ctl->merge_bad = 0;
    ctl->local_hp = 0;
    ctl->shard_grow = 0;
  }
  if (tid < 16) ctl->tiny_counts[tid] = 0;
  if (tid < kListStripes) ctl->g_fill[tid] = 0;
  const bool valid = (u64)tid < m;
  const u64 v = valid ? __ldcg(&es->samples[tid]) : 0ull;
  __syncthreads();
  if (tid == 0) es->arrive = 0;  // ready for the next call (every CTA has arrived)
  // insert the sample into the FreqSet
  // (merging a warp's equal samples first with __match_any_sync cost 2 us:
  // 0.26 lanes/clk/SM; 128 contending shared atomics per slot are cheaper)
  if (valid) {
    const u32 c = 1;
    if (v == kEmpty) {
      atomicAdd(&n_max_key, c);
    } else {
      u32 j = (u32)((v * kGamma) >> 53);  // fast_hash(v, 11); the reference uses 12 bits (cardinality.py:47-61)
      while (true) {
        const u64 old = atomicCAS(&fkeys[j], kEmpty, v);
        if (old == kEmpty || old == v) { atomicAdd(&fcnt[j], c); break; }
        j = (j + 1) & (kFreqSlots - 1);
      }
    }
  }
  u64 lo = warp_min_u64(valid ? v : kEmpty), hi = warp_max_u64(valid ? v : 0ull);
  if (lane == 0) { rmin[wid] = lo; rmax[wid] = hi; }
  __syncthreads();
  // ---- spectrum (cardinality.py:63-69): u, f1, f2 ----
  long long cu = 0, c1 = 0, c2 = 0;
  for (int i = tid; i < kFreqSlots; i += 1024) {
    const u32 c = fcnt[i];
    cu += c > 0;
    c1 += c == 1;
    c2 += c == 2;
  }
  if (tid == 0 && n_max_key) { cu += 1; c1 += n_max_key == 1; c2 += n_max_key == 2; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cu += __shfl_xor_sync(0xffffffffu, cu, o);
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
  }
  if (lane == 0) { red[0][wid] = cu; red[1][wid] = c1; red[2][wid] = c2; }
  __syncthreads();
  if (wid == 0) {  // totals by one warp, broadcast through shared memory
    long long a0 = red[0][lane], a1 = red[1][lane], a2 = red[2][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    }
    __syncwarp();
    if (lane == 0) { red[0][0] = a0; red[1][0] = a1; red[2][0] = a2; }
  }
  __syncthreads();
  const long long u = red[0][0], f1 = red[1][0], f2 = red[2][0];
  // distinct keys (FreqSet.distinct_keys) when u <= 8: collect, then sort
  if (u <= CAFS_TINY_MAX_KEYS) {
    for (int i = tid; i < kFreqSlots; i += 1024)
      if (fcnt[i]) klist[atomicAdd(&nlist, 1u)] = fkeys[i];
    if (tid == 0 && n_max_key) klist[atomicAdd(&nlist, 1u)] = kEmpty;
  }
  __syncthreads();
  if (tid == 0 && u <= CAFS_TINY_MAX_KEYS) {
    for (int a = 1; a < (int)u; ++a) {  // insertion sort, <= 8 keys
      const u64 k = klist[a];
      int b = a - 1;
      while (b >= 0 && klist[b] > k) { klist[b + 1] = klist[b]; --b; }
      klist[b + 1] = k;
    }
    for (int a = 0; a < (int)u; ++a) ctl->keys[a] = klist[a];
  }

  // ---- chao1 (cardinality.py:85-96), bit-exact float64 ----
  const bool saturated = (u == kSampleTarget);
  double k_hat;
  if (saturated) {
    k_hat = (double)nn;
  } else {
    double q = __ddiv_rn((double)(f1 * f1), __dmul_rn(2.0, (double)(f2 + 1)));
    k_hat = __dadd_rn((double)u, q);
    if (!(k_hat < (double)nn)) k_hat = (double)nn;  // min(k_hat, float(n))
  }
  // ---- route (sorter.py:155-162), assuming not monotone ----
  int route;
  if (nn < CAFS_SMALL_N_CUTOFF) route = CAFS_FALLBACK_SMALL_N;
  else if (k_hat <= 8.0 && u <= 8) route = CAFS_TINY_COUNT;
  else if (__dmul_rn(k_hat, 2.0) > (double)nn) route = CAFS_FALLBACK_HIGH_ENTROPY;
  else route = CAFS_MAIN;
  if ((opts & kEstForceMain) && route == CAFS_TINY_COUNT) route = CAFS_MAIN;

  // ---- tiny route: perfect hash of the <= 8 keys into 16 slots ----
  if (route == CAFS_TINY_COUNT) {
    __syncthreads();
    const int nk = (int)u;
    const u64 mult = fmix64((u64)tid + 0x5851F42D4C957F2Dull) | 1ull;
    u32 used = 0;
    bool ok = true;
    for (int j = 0; j < nk; ++j) {
      const u32 sl = (u32)((klist[j] * mult) >> 60);
      ok &= !((used >> sl) & 1u);
      used |= 1u << sl;
    }
    const u32 okm = __ballot_sync(0xffffffffu, ok);  // one atomic per warp, not per thread
    if (okm && lane == __ffs(okm) - 1) atomicMin(&best_t, tid);
    __syncthreads();
    if (tid == best_t) {
      ctl->tiny_mult = mult;
      for (int j = 0; j < nk; ++j) ctl->tiny_slot[j] = (int)((klist[j] * mult) >> 60);
    }
  }

  // the sample's span by warp 0's shuffles (a 32-step loop on thread 0 cost ~1 us)
  u64 span_lo = kEmpty, span_hi = 0;
  if (wid == 0) {
    span_lo = warp_min_u64(rmin[lane]);
    span_hi = warp_max_u64(rmax[lane]);
  }
  if (tid == 0) {
    ctl->prefix_sorted = !inv;
    ctl->route = route;
    int eff = (check_prefix && !inv) ? (n <= kMonoPrefix ? CAFS_ALREADY_SORTED : kNeedScan)
                                     : route;
    if (ghdr) {  // globally sorted iff every shard is and the boundaries are ordered
      bool mono = true, have = false;
      u64 prev = 0;
      for (int r = 0; r < world; ++r) {
        const u64* h = ghdr + r * kShardHdrWords;
        if (h[0] == 0) continue;
        if (!(h[1] == 1 || (h[1] == 2 && h[4] == 0))) mono = false;
        if (have && h[2] < prev) mono = false;
        prev = h[3];
        have = true;
      }
      eff = (nn <= 1 || mono) ? CAFS_ALREADY_SORTED : route;
      ctl->n_global = nn;
    }
    ctl->eff_route = eff;
    ctl->u = u;
    ctl->f1 = f1;
    ctl->f2 = f2;
    ctl->k_hat = k_hat;
    ctl->saturated = saturated;
    ctl->nkeys = (int)(u < CAFS_TINY_MAX_KEYS ? u : CAFS_TINY_MAX_KEYS);
    // dense-range window for the main count: centred on the sample's span
    const u64 smin = span_lo, smax = span_hi;
    const u64 width = smax - smin;
    if (!(opts & kEstNoWindow) && m > 0 && smax >= smin && width < kRangeCap / 2) {
      const u64 margin = (kRangeCap - 1 - width) / 2;
      u64 base = smin >= margin ? smin - margin : 0ull;
      if (base > kEmpty - (kRangeCap - 1)) base = kEmpty - (kRangeCap - 1);
      ctl->range_base = base;
      ctl->range_len = kRangeCap;
    } else {
      ctl->range_base = 0;
      ctl->range_len = 0;
    }
    // the partitioned count (hashpart.cu): columns without a window whose
    // estimated key count fits its 256 partitions of <= 4096 keys
    ctl->hp_ok = (opts & kEstHp) && m == kSampleTarget && ctl->range_len == 0 &&
                 k_hat <= kHpMaxKhat;
  }
}

// Full-array non-decreasing check; only launched when the prefix was sorted.
template <int KK>
__global__ void monotone_scan_kernel(const typename KeyT<KK>::T* __restrict__ x, u64 n, u64 flip,
                                     DevCtl* ctl) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  int found = 0;
  u64 it = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i + 1 < n; i += stride, ++it) {
    found |= key_map<KK>(x[i + 1], flip) < key_map<KK>(x[i], flip);
    if ((it & 63) == 63) {
      if (found) break;
      if (*((volatile int*)&ctl->scan_inversion)) return;
    }
  }
  if (found) ctl->scan_inversion = 1;
}

void launch_estimate(const void* x, u64 n, u64 flip, int check_prefix, DevCtl* ctl,
                     cudaStream_t st, int kk, int opts) {
  switch (kk) {
    case 1:
      launch_pdl(kPdlEstimate, estimate_kernel<1>, kEstCtas, 1024, 0, st, (const u32*)x, n, flip, check_prefix,
                 ctl, (const u64*)nullptr, 0, opts);
      break;
    case 2:
      launch_pdl(kPdlEstimate, estimate_kernel<2>, kEstCtas, 1024, 0, st, (const u32*)x, n, flip, check_prefix,
                 ctl, (const u64*)nullptr, 0, opts);
      break;
    default:
      launch_pdl(kPdlEstimate, estimate_kernel<0>, kEstCtas, 1024, 0, st, (const u64*)x, n, flip, check_prefix,
                 ctl, (const u64*)nullptr, 0, opts);
  }
}

void launch_estimate_sharded(const u64* samples, const u64* ghdr, int world, DevCtl* ctl,
                             cudaStream_t st, int opts) {
  estimate_kernel<0><<<1, 1024, 0, st>>>(samples, kSampleTarget, 0, 0, ctl, ghdr, world, opts);
}

void launch_monotone_scan(const void* x, u64 n, u64 flip, DevCtl* ctl, int num_sms,
                          cudaStream_t st, int kk) {
  const dim3 g(num_sms * 4), b(512);
  switch (kk) {
    case 1: monotone_scan_kernel<1><<<g, b, 0, st>>>((const u32*)x, n, flip, ctl); break;
    case 2: monotone_scan_kernel<2><<<g, b, 0, st>>>((const u32*)x, n, flip, ctl); break;
    default: monotone_scan_kernel<0><<<g, b, 0, st>>>((const u64*)x, n, flip, ctl);
  }
}

}  // namespace cafs
