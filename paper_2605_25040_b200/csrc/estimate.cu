// estimate.cu -- K0 monotone probe + K1 Chao1 cardinality estimate and route.
//
// One CTA of 1024 threads replaces the reference's dispatch pre-pass
// (sorter.py:141-162):
//   * is_monotone (sorter.py:115-129): the first kMonoPrefix rows are checked
//     here; only a prefix that is already sorted triggers the full-array scan
//     kernel below (random inputs pay ~0 extra bytes);
//   * _sample (cardinality.py:99-110): samples x[i * (n // 1024)], i < 1024;
//   * FreqSet spectrum (cardinality.py:63-73): instead of a 4096-slot linear
//     probing table the 1024 samples are bitonic-sorted in shared memory and
//     run lengths counted.  (u, f1, f2) are hash-independent, so this is exact
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

__global__ void __launch_bounds__(1024, 1)
    estimate_kernel(const u64* __restrict__ x, u64 n, u64 flip, int check_prefix, DevCtl* ctl) {
  __shared__ u64 s[kSampleTarget];
  __shared__ int warp_a[32], warp_b[32];
  __shared__ int inv;
  __shared__ int best_t;
  __shared__ long long red[3][32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  if (tid == 0) {
    inv = 0;
    best_t = 0x7fffffff;
    // per-call state of the later stages
    ctl->scan_inversion = 0;
    ctl->tiny_miss = 0;
    ctl->g_used = 0;
    ctl->g_updates = 0;
    ctl->empty_key_count = 0;
    ctl->overflow = 0;
    ctl->need_large = 0;
    ctl->npairs = 0;
    ctl->total = 0;
    ctl->pairs_ready = 0;
    ctl->sum_error = 0;
  }
  if (tid < 16) ctl->tiny_counts[tid] = 0;
  __syncthreads();

  // ---- K0: prefix monotone probe (exact: any inversion => not monotone) ----
  if (check_prefix) {
    const u64 P = n < kMonoPrefix ? n : kMonoPrefix;
    int found = 0;
    for (u64 i = tid; i + 1 < P; i += blockDim.x) found |= ((x[i + 1] ^ flip) < (x[i] ^ flip));
    if (__syncthreads_or(found) && tid == 0) inv = 1;
  }

  // ---- K1: 1024 strided samples (cardinality.py:102-104) ----
  const u64 m = n < (u64)kSampleTarget ? n : (u64)kSampleTarget;
  u64 stride = n / kSampleTarget;
  if (stride < 1) stride = 1;
  s[tid] = (u64)tid < m ? (x[(u64)tid * stride] ^ flip) : kEmpty;
  __syncthreads();
  // bitonic sort, 1024 keys, one per thread
  for (int k = 2; k <= kSampleTarget; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      int p = tid ^ j;
      if (p > tid) {
        u64 a = s[tid], b = s[p];
        bool up = (tid & k) == 0;
        if ((a > b) == up) { s[tid] = b; s[p] = a; }
      }
      __syncthreads();
    }
  }
  // ---- spectrum over the first m sorted samples ----
  const bool valid = (u64)tid < m;
  const u64 v = s[tid];
  const bool start = valid && (tid == 0 || s[tid - 1] != v);
  const bool last = valid && ((u64)tid == m - 1 || s[tid + 1] != v);
  // run start index (inclusive max-scan of start ? tid : 0)
  int rs = warp_incl_max(start ? tid : 0);
  if (lane == 31) warp_a[wid] = rs;
  // distinct-key rank (inclusive sum of start flags)
  int rk = warp_incl_sum(start ? 1 : 0);
  if (lane == 31) warp_b[wid] = rk;
  __syncthreads();
  if (wid == 0) {
    int a = warp_incl_max(warp_a[lane]);
    int b = warp_incl_sum(warp_b[lane]);
    warp_a[lane] = a;  // inclusive
    warp_b[lane] = b;
  }
  __syncthreads();
  if (wid > 0) {
    rs = max(rs, warp_a[wid - 1]);
    rk += warp_b[wid - 1];
  }
  const int len = tid - rs + 1;
  long long cu = start ? 1 : 0;
  long long c1 = (last && len == 1) ? 1 : 0;
  long long c2 = (last && len == 2) ? 1 : 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cu += __shfl_xor_sync(0xffffffffu, cu, o);
    c1 += __shfl_xor_sync(0xffffffffu, c1, o);
    c2 += __shfl_xor_sync(0xffffffffu, c2, o);
  }
  if (lane == 0) { red[0][wid] = cu; red[1][wid] = c1; red[2][wid] = c2; }
  __syncthreads();
  if (wid == 0) {
    cu = red[0][lane]; c1 = red[1][lane]; c2 = red[2][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      cu += __shfl_xor_sync(0xffffffffu, cu, o);
      c1 += __shfl_xor_sync(0xffffffffu, c1, o);
      c2 += __shfl_xor_sync(0xffffffffu, c2, o);
    }
    if (lane == 0) { red[0][0] = cu; red[1][0] = c1; red[2][0] = c2; }
  }
  __syncthreads();
  const long long u = red[0][0], f1 = red[1][0], f2 = red[2][0];
  // distinct keys ascending (FreqSet.distinct_keys)
  if (start && rk - 1 < CAFS_TINY_MAX_KEYS) ctl->keys[rk - 1] = v;

  // ---- chao1 (cardinality.py:85-96), bit-exact float64 ----
  const bool saturated = (u == kSampleTarget);
  double k_hat;
  if (saturated) {
    k_hat = (double)n;
  } else {
    double q = __ddiv_rn((double)(f1 * f1), __dmul_rn(2.0, (double)(f2 + 1)));
    k_hat = __dadd_rn((double)u, q);
    if (!(k_hat < (double)n)) k_hat = (double)n;  // min(k_hat, float(n))
  }
  // ---- route (sorter.py:155-162), assuming not monotone ----
  int route;
  if (n < CAFS_SMALL_N_CUTOFF) route = CAFS_FALLBACK_SMALL_N;
  else if (k_hat <= 8.0 && u <= 8) route = CAFS_TINY_COUNT;
  else if (__dmul_rn(k_hat, 2.0) > (double)n) route = CAFS_FALLBACK_HIGH_ENTROPY;
  else route = CAFS_MAIN;

  // ---- tiny route: perfect hash of the <= 8 keys into 16 slots ----
  if (route == CAFS_TINY_COUNT) {
    const int nk = (int)u;
    const u64 mult = fmix64((u64)tid + 0x5851F42D4C957F2Dull) | 1ull;
    u32 used = 0;
    bool ok = true;
    for (int j = 0; j < nk; ++j) {
      u32 sl = (u32)((ctl->keys[j] * mult) >> 60);
      ok &= !((used >> sl) & 1u);
      used |= 1u << sl;
    }
    if (ok) atomicMin(&best_t, tid);
    __syncthreads();
    if (tid == best_t) {
      ctl->tiny_mult = mult;
      for (int j = 0; j < nk; ++j) ctl->tiny_slot[j] = (int)((ctl->keys[j] * mult) >> 60);
    }
  }

  if (tid == 0) {
    ctl->prefix_sorted = !inv;
    ctl->route = route;
    ctl->u = u;
    ctl->f1 = f1;
    ctl->f2 = f2;
    ctl->k_hat = k_hat;
    ctl->saturated = saturated;
    ctl->nkeys = (int)(u < CAFS_TINY_MAX_KEYS ? u : CAFS_TINY_MAX_KEYS);
    // dense-range window for the main count: centred on the sample's span
    const u64 lo = s[0], hi = s[m - 1];
    const u64 width = hi - lo;
    if (width < kRangeCap / 2) {
      const u64 margin = (kRangeCap - 1 - width) / 2;
      u64 base = lo >= margin ? lo - margin : 0ull;
      if (base > kEmpty - (kRangeCap - 1)) base = kEmpty - (kRangeCap - 1);
      ctl->range_base = base;
      ctl->range_len = kRangeCap;
    } else {
      ctl->range_base = 0;
      ctl->range_len = 0;
    }
  }
}

// Full-array non-decreasing check; only launched when the prefix was sorted.
__global__ void monotone_scan_kernel(const u64* __restrict__ x, u64 n, u64 flip, DevCtl* ctl) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  int found = 0;
  u64 it = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i + 1 < n; i += stride, ++it) {
    found |= ((x[i + 1] ^ flip) < (x[i] ^ flip));
    if ((it & 63) == 63) {
      if (found) break;
      if (*((volatile int*)&ctl->scan_inversion)) return;
    }
  }
  if (found) ctl->scan_inversion = 1;
}

void launch_estimate(const u64* x, u64 n, u64 flip, int check_prefix, DevCtl* ctl,
                     cudaStream_t st) {
  estimate_kernel<<<1, 1024, 0, st>>>(x, n, flip, check_prefix, ctl);
}

void launch_monotone_scan(const u64* x, u64 n, u64 flip, DevCtl* ctl, int num_sms,
                          cudaStream_t st) {
  monotone_scan_kernel<<<num_sms * 4, 512, 0, st>>>(x, n, flip, ctl);
}

}  // namespace cafs
