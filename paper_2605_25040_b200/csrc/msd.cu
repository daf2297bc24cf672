// msd.cu -- MSD bucket sort: the fallback engine and the large pair sort.
//
// Replaces fallback_sort (sorter.py:132-138) and, for more than 8192 pairs,
// radix_sort_pairs (_kernels.py:185-214).  An LSD radix sort of 64-bit keys
// moves 16 B/key per digit pass (8 passes for random keys); here one pass
// partitions the keys into 4096 buckets by (k - min) >> shift over the keys'
// numeric span (a min/max reduction, so dictionary codes, clustered and
// sign-extended 32-bit keys still spread), and each bucket is then sorted in
// shared memory: one warp for <= 128 keys (rank sort), else a 256-thread CTA
// (a second split on 10 more bits + rank sort, or stable byte passes).
// DRAM traffic: 8 (span) + 8 (histogram) + 16 (scatter) + 16 (bucket sort) =
// 48 B/key.  Buckets larger than kBucketCap (skewed keys, or n ~ 2^30) are
// left to the onesweep LSD path (radix.cu) by the host.
#include <cstddef>

#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kMsdBits = 12;
constexpr u32 kMsdBuckets = 1u << kMsdBits;
constexpr int kBsThreads = 256;
constexpr int kBsWarps = kBsThreads / 32;
constexpr u32 kBucketCap = 4096;                       // keys per bucket sorted in smem
constexpr int kBsRounds = kBucketCap / kBsThreads;     // 16 rounds of 32 per warp
constexpr u32 kWarpBucketMax = 128;                    // buckets sorted by one warp
constexpr int kSubBits = 11;                           // second-level split inside a bucket
constexpr u32 kSubBins = 1u << kSubBits;               // (overlays the warp counters)
constexpr u32 kSubMax = 64;                            // largest sub-bucket rank-sorted
constexpr size_t kBsCounterBytes = (size_t)kSubBins * 4 > (size_t)kBsWarps * 256 * 4
                                       ? (size_t)kSubBins * 4 : (size_t)kBsWarps * 256 * 4;
constexpr int kScThreads = 256;
constexpr int kScItems = 16;                           // keys per thread in the scatter
constexpr u64 kScChunk = (u64)kScThreads * kScItems;   // 4096

// The sort's scatter gives each chunk of keys a fixed slice of every bucket
// (reserved by the histogram kernel), so it writes without global atomics.
constexpr u32 kMsdMaxChunks = 512;
constexpr u64 kMsdMaxN = (u64)kMsdBuckets * kBucketCap;  // beyond: some bucket > kBucketCap

struct MsdState {
  unsigned long long kmin, kmax;  // span of the order-mapped keys (adjacent: read as a pair)
  u32 hist[kMsdBuckets];
  u32 base[kMsdBuckets + 1];
  u32 cursor[kMsdBuckets];
  u32 maxb;
  int shift;
  u32 overflow;  // a bucket larger than the bucket sort's cap (unchecked launches)
  u32 offs[kMsdMaxChunks][kMsdBuckets];  // chunk c's offset inside bucket b (not memset)
};
constexpr size_t kMsdClear = offsetof(MsdState, offs);

// keys per chunk: about two chunks per SM, a multiple of 4096, at most 64K
static u64 msd_chunk(u64 n, int num_sms) {
  u64 c = (n + 2ull * num_sms - 1) / (2ull * num_sms);
  c = (c + 4095) & ~4095ull;
  if (c < 4096) c = 4096;
  if (c > 65536) c = 65536;
  return c;
}

__device__ __forceinline__ u32 msd_digit(u64 k, u64 base, int shift) {
  return (u32)((k - base) >> shift) & (kMsdBuckets - 1);
}

__global__ void __launch_bounds__(512) msd_reduce_kernel(const u64* __restrict__ keys, u64 n,
                                                         u64 flip, MsdState* ms) {
  pdl_begin();
  u64 lo = ~0ull, hi = 0;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  auto take = [&](u64 k) {
    lo = k < lo ? k : lo;
    hi = k > hi ? k : hi;
  };
  for (; i + 3 * stride < n; i += 4 * stride) {  // four loads in flight per thread
    const u64 a = keys[i] ^ flip, b = keys[i + stride] ^ flip, c = keys[i + 2 * stride] ^ flip,
              d = keys[i + 3 * stride] ^ flip;
    take(a); take(b); take(c); take(d);
  }
  for (; i < n; i += stride) take(keys[i] ^ flip);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&ms->kmin, lo);
    atomicMax(&ms->kmax, hi);
  }
}

// shift so the bucket digit (k - kmin) >> shift covers the span in 4096 steps
// (the numeric span, not the varying bits: sign-extended 32-bit keys vary in
// all 32 high bits while spanning only 2^32 values)
__device__ __forceinline__ int msd_shift(const MsdState* ms) {
  if (ms->kmax <= ms->kmin) return 0;
  const u64 span = ms->kmax - ms->kmin;
  const int hb = 63 - __clzll(span);
  return hb + 1 > kMsdBits ? hb + 1 - kMsdBits : 0;
}

__global__ void __launch_bounds__(512) msd_hist_kernel(const u64* __restrict__ keys, u64 n,
                                                       u64 flip, MsdState* ms) {
  __shared__ u32 h[kMsdBuckets];
  for (u32 i = threadIdx.x; i < kMsdBuckets; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int shift = msd_shift(ms);
  const u64 kbase = ms->kmin;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(&h[msd_digit(keys[i] ^ flip, kbase, shift)], 1u);
  __syncthreads();
  for (u32 i = threadIdx.x; i < kMsdBuckets; i += blockDim.x)
    if (h[i]) atomicAdd(&ms->hist[i], h[i]);
}

__global__ void __launch_bounds__(1024) msd_scan_kernel(MsdState* ms) {
  pdl_begin();
  __shared__ u32 ws[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr int IT = kMsdBuckets / 1024;
  u32 c[IT], local = 0, mx = 0;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    c[q] = ms->hist[tid * IT + q];
    local += c[q];
    mx = c[q] > mx ? c[q] : mx;
  }
  u32 incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u32 t = __shfl_xor_sync(0xffffffffu, mx, o);
    mx = t > mx ? t : mx;
  }
  if (lane == 31) ws[wid] = incl;
  if (lane == 0) atomicMax(&ms->maxb, mx);
  __syncthreads();
  if (wid == 0) {
    u32 w = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    ws[lane] = w;
  }
  __syncthreads();
  u32 run = incl - local + (wid ? ws[wid - 1] : 0);
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    ms->base[tid * IT + q] = run;
    ms->cursor[tid * IT + q] = run;
    run += c[q];
  }
  if (tid == 1023) ms->base[kMsdBuckets] = run;
  if (tid == 0) ms->shift = msd_shift(ms);
}

// Chunk histograms (the sort's first pass after the span): chunk c counts its
// keys per bucket in shared memory, then reserves its slice of every bucket
// with one atomic per non-empty bucket; offs[c][b] = that slice's offset,
// hist[b] = the bucket's total.
__global__ void __launch_bounds__(1024) msd_chunk_hist_kernel(const u64* __restrict__ keys, u64 n,
                                                              u64 flip, MsdState* ms, u64 chunk) {
  pdl_begin();
  __shared__ u32 h[kMsdBuckets];
  for (u32 i = threadIdx.x; i < kMsdBuckets; i += 1024) h[i] = 0;
  __syncthreads();
  const int shift = msd_shift(ms);
  const u64 kbase = ms->kmin;
  const u64 c0 = blockIdx.x * chunk;
  const u64 c1 = c0 + chunk < n ? c0 + chunk : n;
  u64 i = c0 + threadIdx.x;
  for (; i + 3 * 1024 < c1; i += 4 * 1024) {
    const u64 a = keys[i], b = keys[i + 1024], c = keys[i + 2048], d = keys[i + 3072];
    atomicAdd(&h[msd_digit(a ^ flip, kbase, shift)], 1u);
    atomicAdd(&h[msd_digit(b ^ flip, kbase, shift)], 1u);
    atomicAdd(&h[msd_digit(c ^ flip, kbase, shift)], 1u);
    atomicAdd(&h[msd_digit(d ^ flip, kbase, shift)], 1u);
  }
  for (; i < c1; i += 1024) atomicAdd(&h[msd_digit(keys[i] ^ flip, kbase, shift)], 1u);
  __syncthreads();
  u32* row = ms->offs[blockIdx.x];
  for (u32 b = threadIdx.x; b < kMsdBuckets; b += 1024) {
    const u32 c = h[b];
    row[b] = c ? atomicAdd(&ms->hist[b], c) : 0u;
  }
}

// Scatter with the reserved slices: position = bucket base + chunk offset +
// the key's rank among the chunk's keys of that bucket (shared atomics; order
// inside a bucket is not preserved -- the bucket sort follows).
template <bool HAS_VAL>
__global__ void __launch_bounds__(1024)
    msd_scatter_chunk_kernel(const u64* __restrict__ keys, const u64* __restrict__ vals, u64 n,
                             u64 flip, const MsdState* ms, u64 chunk, u64* __restrict__ tk,
                             u64* __restrict__ tv) {
  pdl_begin();
  __shared__ u32 lc[kMsdBuckets];
  __shared__ u32 gb[kMsdBuckets];
  const u32* row = ms->offs[blockIdx.x];
  for (u32 b = threadIdx.x; b < kMsdBuckets; b += 1024) {
    lc[b] = 0;
    gb[b] = ms->base[b] + row[b];
  }
  __syncthreads();
  const int shift = ms->shift;
  const u64 kbase = ms->kmin;
  const u64 c0 = blockIdx.x * chunk;
  const u64 c1 = c0 + chunk < n ? c0 + chunk : n;
  u64 i = c0 + threadIdx.x;
  for (; i + 3 * 1024 < c1; i += 4 * 1024) {
    u64 k[4], v[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      k[j] = keys[i + j * 1024] ^ flip;
      if (HAS_VAL) v[j] = vals[i + j * 1024];
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const u32 d = msd_digit(k[j], kbase, shift);
      const u32 pos = gb[d] + atomicAdd(&lc[d], 1u);
      tk[pos] = k[j];
      if (HAS_VAL) tv[pos] = v[j];
    }
  }
  for (; i < c1; i += 1024) {
    const u64 k = keys[i] ^ flip;
    const u32 d = msd_digit(k, kbase, shift);
    const u32 pos = gb[d] + atomicAdd(&lc[d], 1u);
    tk[pos] = k;
    if (HAS_VAL) tv[pos] = vals[i];
  }
}

// Key-only scatter staged through shared memory: each 16384-key tile of the
// chunk is counting-sorted by bucket in shared memory first, then written out
// by consecutive threads, so the ~4 keys a tile holds per bucket leave as one
// contiguous run instead of ~4 scattered 8-byte stores (the unstaged scatter
// is bound by L2 write transactions: ~1 TB/s).
constexpr int kStTile = 16384;
constexpr size_t kStSmem = (size_t)kStTile * 8 + (size_t)kMsdBuckets * 4 * 3;

__global__ void __launch_bounds__(1024, 1)
    msd_scatter_staged_kernel(const u64* __restrict__ keys, u64 n, u64 flip, const MsdState* ms,
                              u64 chunk, u64* __restrict__ tk) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char st_smem[];
  u64* stage = (u64*)st_smem;                    // [kStTile] keys in bucket order
  u32* gpos = (u32*)(stage + kStTile);           // [4096] next global position per bucket
  u32* th = gpos + kMsdBuckets;                  // [4096] tile counts -> ranks
  u32* toff = th + kMsdBuckets;                  // [4096] tile offsets (exclusive)
  __shared__ u32 wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u32* row = ms->offs[blockIdx.x];
  for (u32 b = tid; b < kMsdBuckets; b += 1024) {
    gpos[b] = ms->base[b] + row[b];
    th[b] = 0;
  }
  __syncthreads();
  const int shift = ms->shift;
  const u64 kbase = ms->kmin;
  const u64 c0 = blockIdx.x * chunk;
  const u64 c1 = c0 + chunk < n ? c0 + chunk : n;
  constexpr int IPT = kStTile / 1024;  // keys per thread per tile
  for (u64 t0 = c0; t0 < c1; t0 += kStTile) {
    const u32 tn = (u32)((c1 - t0) < (u64)kStTile ? (c1 - t0) : (u64)kStTile);
    u64 k[IPT];
    u32 r[IPT], d[IPT];
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const u32 i = tid + j * 1024;
      k[j] = i < tn ? keys[t0 + i] ^ flip : 0;
    }
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const u32 i = tid + j * 1024;
      d[j] = msd_digit(k[j], kbase, shift);
      if (i < tn) r[j] = atomicAdd(&th[d[j]], 1u);
    }
    __syncthreads();
    {  // exclusive scan of the tile counts (4 bins per thread)
      u32 c[4], loc = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) { c[q] = th[tid * 4 + q]; loc += c[q]; }
      u32 incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 tt = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += tt;
      }
      if (lane == 31) wsum[wid] = incl;
      __syncthreads();
      if (wid == 0) {
        u32 w = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 tt = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += tt;
        }
        wsum[lane] = w;
      }
      __syncthreads();
      u32 run = incl - loc + (wid ? wsum[wid - 1] : 0);
#pragma unroll
      for (int q = 0; q < 4; ++q) { toff[tid * 4 + q] = run; run += c[q]; }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const u32 i = tid + j * 1024;
      if (i < tn) stage[toff[d[j]] + r[j]] = k[j];
    }
    __syncthreads();
    // consecutive threads write consecutive staged keys: a bucket's run is contiguous
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
      const u32 i = tid + j * 1024;
      if (i < tn) {
        const u64 key = stage[i];
        const u32 dd = msd_digit(key, kbase, shift);
        tk[gpos[dd] + (i - toff[dd])] = key;
      }
    }
    __syncthreads();
    for (u32 b = tid; b < kMsdBuckets; b += 1024) {  // advance the bucket cursors
      gpos[b] += th[b];
      th[b] = 0;
    }
    __syncthreads();
  }
}

// Scatter a 4096-key chunk into its buckets: local counts (shared atomics give
// each key its rank), one global reservation per non-empty bucket, then the
// writes.  Order inside a bucket is not preserved: keys are sorted afterwards
// and pair keys are distinct, so stability is not needed.
template <bool HAS_VAL>
__global__ void __launch_bounds__(kScThreads)
    msd_scatter_kernel(const u64* __restrict__ keys, const u64* __restrict__ vals, u64 n, u64 flip,
                       MsdState* ms, u64* __restrict__ tk, u64* __restrict__ tv,
                       u64 out_xor = 0) {
  __shared__ u32 h[kMsdBuckets];
  __shared__ u32 g[kMsdBuckets];
  for (u32 i = threadIdx.x; i < kMsdBuckets; i += kScThreads) h[i] = 0;
  __syncthreads();
  const int shift = ms->shift;
  const u64 kbase = ms->kmin;
  const u64 c0 = (u64)blockIdx.x * kScChunk;
  u64 k[kScItems];
  u32 r[kScItems];
#pragma unroll
  for (int j = 0; j < kScItems; ++j) {
    const u64 i = c0 + threadIdx.x + (u64)j * kScThreads;
    k[j] = i < n ? keys[i] ^ flip : 0;
  }
#pragma unroll
  for (int j = 0; j < kScItems; ++j) {
    const u64 i = c0 + threadIdx.x + (u64)j * kScThreads;
    if (i < n) r[j] = atomicAdd(&h[msd_digit(k[j], kbase, shift)], 1u);
  }
  __syncthreads();
  for (u32 b = threadIdx.x; b < kMsdBuckets; b += kScThreads)
    if (h[b]) g[b] = atomicAdd(&ms->cursor[b], h[b]);
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kScItems; ++j) {
    const u64 i = c0 + threadIdx.x + (u64)j * kScThreads;
    if (i < n) {
      const u32 pos = g[msd_digit(k[j], kbase, shift)] + r[j];
      tk[pos] = k[j] ^ out_xor;
      if (HAS_VAL) tv[pos] = vals[i];
    }
  }
}

// Buckets of at most kWarpBucketMax keys (the common case when the 4096
// buckets split a few hundred thousand keys): one warp per bucket, a rank sort
// -- each key's destination is the number of keys that precede it (smaller,
// or equal and earlier: stable) -- from a broadcast scan of the bucket in
// shared memory.  No block barriers, no digit passes, 32 buckets per CTA wave.
template <bool HAS_VAL>
__global__ void __launch_bounds__(256)
    bucket_small_kernel(const u64* __restrict__ tk, const u64* __restrict__ tv,
                        const MsdState* ms, u64 flip, u64* __restrict__ dk,
                        u64* __restrict__ dv) {
  pdl_begin();
  constexpr int R = kWarpBucketMax / 32;
  __shared__ u64 sk[8][kWarpBucketMax];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const u32 b = blockIdx.x * 8 + wid;
  if (b >= kMsdBuckets) return;
  const u32 base = ms->base[b];
  const u32 n = ms->base[b + 1] - base;
  if (n == 0 || n > kWarpBucketMax) return;
  u64 k[R], v[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const u32 i = lane + 32 * r;
    k[r] = i < n ? tk[base + i] : ~0ull;
    v[r] = (HAS_VAL && i < n) ? tv[base + i] : 0;
  }
#pragma unroll
  for (int r = 0; r < R; ++r)
    if (lane + 32 * r < n) sk[wid][lane + 32 * r] = k[r];
  __syncwarp();
  u32 rank[R];
#pragma unroll
  for (int r = 0; r < R; ++r) rank[r] = 0;
  for (u32 j = 0; j < n; ++j) {
    const u64 kj = sk[wid][j];
#pragma unroll
    for (int r = 0; r < R; ++r)
      rank[r] += (kj < k[r]) || (kj == k[r] && j < (u32)(lane + 32 * r));
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (lane + 32 * r < n) {
      dk[base + rank[r]] = k[r] ^ flip;
      if (HAS_VAL) dv[base + rank[r]] = v[r];
    }
  }
}

// One CTA per bucket: load it into shared memory, LSD radix over the bytes that
// vary inside the bucket (stable 8-ballot multisplit, warp-contiguous
// segments), write it back sorted (un-flipping the keys; pairs carry their
// value through a 16-bit index).  `cap` (>= the largest bucket, a multiple of
// kBsThreads) sizes the shared buffers, so small buckets leave room for more
// CTAs per SM.
__host__ __device__ constexpr size_t bs_smem_bytes(u32 cap, bool has_val) {
  return (size_t)cap * 16 + (has_val ? (size_t)cap * 4 : 0) + kBsCounterBytes;
}

template <bool HAS_VAL>
__global__ void __launch_bounds__(kBsThreads, 5)  // latency-bound phases: more CTAs per SM
    bucket_sort_kernel(const u64* __restrict__ tk, const u64* __restrict__ tv,
                       const MsdState* ms, u64 flip, u64* __restrict__ dk, u64* __restrict__ dv,
                       u32 cap) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char bs_smem[];
  u64* kb[2] = {(u64*)bs_smem, (u64*)bs_smem + cap};
  unsigned short* ib[2] = {(unsigned short*)((u64*)bs_smem + 2 * cap),
                           (unsigned short*)((u64*)bs_smem + 2 * cap) + cap};
  u32 (*wcnt)[256] =
      (u32 (*)[256])(bs_smem + (size_t)cap * 16 + (HAS_VAL ? (size_t)cap * 4 : 0));  // [warps]
  __shared__ u32 dstart[256];
  __shared__ u32 wsum8[8];
  __shared__ u64 red_or[kBsWarps], red_and[kBsWarps];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u32 b = blockIdx.x;
  const u32 base = ms->base[b];
  const u32 n = ms->base[b + 1] - base;
  if (n <= kWarpBucketMax) return;  // bucket_small_kernel's
  if (n > cap) {  // launched without the host's maxb check: the caller redoes the sort
    if (tid == 0) atomicOr(&((MsdState*)ms)->overflow, 1u);
    return;
  }
  u64 vor = 0, vand = ~0ull, vmin = ~0ull, vmax = 0;
  {  // all loads in flight before any use (one DRAM round trip, not n/256)
    u64 lk[kBsRounds];
#pragma unroll
    for (int j = 0; j < kBsRounds; ++j) {
      const u32 i = tid + j * kBsThreads;
      lk[j] = i < n ? tk[base + i] : 0;
    }
#pragma unroll
    for (int j = 0; j < kBsRounds; ++j) {
      const u32 i = tid + j * kBsThreads;
      if (i < n) {
        kb[0][i] = lk[j];
        if (HAS_VAL) ib[0][i] = (unsigned short)i;
        vor |= lk[j];
        vand &= lk[j];
        vmin = lk[j] < vmin ? lk[j] : vmin;
        vmax = lk[j] > vmax ? lk[j] : vmax;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vor |= __shfl_xor_sync(0xffffffffu, vor, o);
    vand &= __shfl_xor_sync(0xffffffffu, vand, o);
    const u64 a = __shfl_xor_sync(0xffffffffu, vmin, o), b = __shfl_xor_sync(0xffffffffu, vmax, o);
    vmin = a < vmin ? a : vmin;
    vmax = b > vmax ? b : vmax;
  }
  __shared__ u64 red_min[kBsWarps], red_max[kBsWarps];
  if (lane == 0) { red_or[wid] = vor; red_and[wid] = vand; red_min[wid] = vmin; red_max[wid] = vmax; }
  __syncthreads();
  vor = 0; vand = ~0ull; vmin = ~0ull; vmax = 0;
  for (int w = 0; w < kBsWarps; ++w) {
    vor |= red_or[w];
    vand &= red_and[w];
    vmin = red_min[w] < vmin ? red_min[w] : vmin;
    vmax = red_max[w] > vmax ? red_max[w] : vmax;
  }
  const u64 vary = vor ^ vand;
  // ---- two-level path: split the bucket's numeric span [vmin, vmax] into
  // 2^kSubBits sub-buckets (shared-memory counting sort), then rank-sort each
  // sub-bucket -- a few keys each when the keys are spread -- instead of up to
  // 7 byte passes.  Buckets with a sub-bucket over kSubMax keys (clustered or
  // repeated keys) take the LSD passes below.
  if (vmax > vmin) {
    const int hb = 63 - __clzll(vmax - vmin);
    const int nbits = hb + 1 < kSubBits ? hb + 1 : kSubBits;
    const int sh = hb + 1 - nbits;
    const u32 dmask = (1u << nbits) - 1;
    // one array: counts -> starts (scan) -> ends (the scatter's cursors);
    // afterwards sub-bucket d is [d ? c2[d-1] : 0, c2[d])
    u32* c2 = &wcnt[0][0];          // [kSubBins] (overlays the warp counters)
    __shared__ u32 maxsub;
    for (u32 i = tid; i < kSubBins; i += kBsThreads) c2[i] = 0;
    if (tid == 0) maxsub = 0;
    __syncthreads();
    for (u32 i = tid; i < n; i += kBsThreads)
      atomicAdd(&c2[(u32)((kb[0][i] - vmin) >> sh) & dmask], 1u);
    __syncthreads();
    {  // exclusive scan of the kSubBins counts (kSubBins / kBsThreads per thread)
      constexpr int PT = kSubBins / kBsThreads;
      u32 c[PT], loc = 0, mx = 0;
#pragma unroll
      for (int q = 0; q < PT; ++q) {
        c[q] = c2[tid * PT + q];
        loc += c[q];
        mx = c[q] > mx ? c[q] : mx;
      }
      u32 incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const u32 t = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = t > mx ? t : mx;
      }
      if (lane == 31) wsum8[wid] = incl;
      if (lane == 0) atomicMax(&maxsub, mx);
      __syncthreads();
      u32 run = incl - loc;
      for (int w = 0; w < wid; ++w) run += wsum8[w];
#pragma unroll
      for (int q = 0; q < PT; ++q) {
        c2[tid * PT + q] = run;
        run += c[q];
      }
    }
    __syncthreads();
    if (maxsub <= kSubMax) {
      for (u32 i = tid; i < n; i += kBsThreads) {
        const u64 k = kb[0][i];
        const u32 p = atomicAdd(&c2[(u32)((k - vmin) >> sh) & dmask], 1u);
        kb[1][p] = k;
        if (HAS_VAL) ib[1][p] = ib[0][i];
      }
      __syncthreads();
      for (u32 p = tid; p < n; p += kBsThreads) {
        const u64 k = kb[1][p];
        const u32 d = (u32)((k - vmin) >> sh) & dmask;
        const u32 s0 = d ? c2[d - 1] : 0u, e0 = c2[d];
        u32 r = 0;
        for (u32 j = s0; j < e0; ++j) {
          const u64 kj = kb[1][j];
          r += (kj < k) || (kj == k && j < p);
        }
        dk[base + s0 + r] = k ^ flip;
        if (HAS_VAL) dv[base + s0 + r] = tv[base + ib[1][p]];
      }
      return;
    }
    __syncthreads();  // the LSD passes reuse wcnt
  }
  // warp-contiguous segments of whole rounds
  const u32 rounds = ((n + 31) / 32 + kBsWarps - 1) / kBsWarps;  // rounds per warp
  const u32 w0 = wid * rounds * 32;
  int cur = 0;
  for (int p = 0; p < 8; ++p) {
    if (((vary >> (8 * p)) & 0xFF) == 0) continue;
    const int shift = 8 * p;
    const u64* src = kb[cur];
    u64* dst = kb[cur ^ 1];
    const unsigned short* isrc = ib[cur];
    unsigned short* idst = ib[cur ^ 1];
    u32* my = wcnt[wid];
    for (int i = lane; i < 256; i += 32) my[i] = 0;
    __syncwarp();
    u32 rank[kBsRounds];
    u32 dig[kBsRounds];
#pragma unroll
    for (int r = 0; r < kBsRounds; ++r) {
      if ((u32)r >= rounds) break;
      const u32 idx = w0 + r * 32 + lane;
      const bool valid = idx < n;
      const u32 d = valid ? (u32)(src[idx] >> shift) & 255u : 0u;
      u32 peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int bb = 0; bb < 8; ++bb) {
        const u32 bal = __ballot_sync(0xffffffffu, (d >> bb) & 1u);
        peers &= ((d >> bb) & 1u) ? bal : ~bal;
      }
      u32 before = 0;
      if (valid) before = my[d];
      __syncwarp();
      if (valid) {
        rank[r] = before + __popc(peers & lanemask_lt());
        if (lane == 31 - __clz(peers)) my[d] = before + __popc(peers);
      }
      dig[r] = d;
      __syncwarp();
    }
    __syncthreads();
    {  // per digit: exclusive prefix over warps, then over digits (256 threads)
      u32 acc = 0;
#pragma unroll
      for (int w = 0; w < kBsWarps; ++w) {
        const u32 c = wcnt[w][tid];
        wcnt[w][tid] = acc;
        acc += c;
      }
      u32 incl = acc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum8[wid] = incl;
      __syncthreads();
      u32 pre = 0;
      for (int w = 0; w < wid; ++w) pre += wsum8[w];
      dstart[tid] = pre + incl - acc;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kBsRounds; ++r) {
      if ((u32)r >= rounds) break;
      const u32 idx = w0 + r * 32 + lane;
      if (idx < n) {
        const u32 pos = dstart[dig[r]] + wcnt[wid][dig[r]] + rank[r];
        dst[pos] = src[idx];
        if (HAS_VAL) idst[pos] = isrc[idx];
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  if (HAS_VAL) {
    u64 lv[kBsRounds];
#pragma unroll
    for (int j = 0; j < kBsRounds; ++j) {
      const u32 i = tid + j * kBsThreads;
      lv[j] = i < n ? tv[base + ib[cur][i]] : 0;
    }
#pragma unroll
    for (int j = 0; j < kBsRounds; ++j) {
      const u32 i = tid + j * kBsThreads;
      if (i < n) dv[base + i] = lv[j];
    }
  }
  for (u32 i = tid; i < n; i += kBsThreads) dk[base + i] = kb[cur][i] ^ flip;
}

// ---------------- host side ----------------
size_t msd_state_bytes() { return sizeof(MsdState); }
u32 msd_bucket_cap() { return kBucketCap; }

// false: the keys cannot all fit kBucketCap-sized buckets (n too large)
bool launch_msd_count(const u64* keys, u64 n, u64 flip, void* state, int num_sms,
                      cudaStream_t st) {
  if (n > kMsdMaxN) return false;
  const u64 chunk = msd_chunk(n, num_sms);
  const u64 nchunks = (n + chunk - 1) / chunk;
  if (nchunks > kMsdMaxChunks) return false;
  MsdState* ms = (MsdState*)state;
  cudaMemsetAsync(ms, 0, kMsdClear, st);
  cudaMemsetAsync(&ms->kmin, 0xFF, sizeof(u64), st);
  u64 blocks = (n + 512 * 8 - 1) / (512 * 8);
  if (blocks > (u64)num_sms * 4) blocks = (u64)num_sms * 4;
  if (blocks < 1) blocks = 1;
  msd_reduce_kernel<<<(unsigned)blocks, 512, 0, st>>>(keys, n, flip, ms);
  launch_pdl(kPdlMsd, msd_chunk_hist_kernel, (unsigned)nchunks, 1024, 0, st, keys, n, flip, ms, chunk);
  launch_pdl(kPdlMsd, msd_scan_kernel, 1, 1024, 0, st, ms);
  return true;
}

__global__ void msd_set_span_kernel(MsdState* ms, u64 kmin, u64 kmax) {
  ms->kmin = kmin;
  ms->kmax = kmax;
}

// Local min/max of the order-mapped keys (the distributed fallback all-gathers
// them to fix one bucket digit for every rank).
void launch_msd_span(const u64* keys, u64 n, u64 flip, void* state, int num_sms, cudaStream_t st) {
  MsdState* ms = (MsdState*)state;
  cudaMemsetAsync(ms, 0, kMsdClear, st);
  cudaMemsetAsync(&ms->kmin, 0xFF, sizeof(u64), st);
  u64 blocks = (n + 512 * 8 - 1) / (512 * 8);
  if (blocks > (u64)num_sms * 4) blocks = (u64)num_sms * 4;
  if (blocks < 1) blocks = 1;
  msd_reduce_kernel<<<(unsigned)blocks, 512, 0, st>>>(keys, n, flip, ms);
}
size_t msd_span_offset() { return offsetof(MsdState, kmin); }  // kmin, kmax adjacent
size_t msd_hist_offset() { return offsetof(MsdState, hist); }

// Group keys by the bucket digit of a GLOBAL span [kmin, kmax]: out holds the
// keys (original representation) in ascending digit order; hist = counts.
void launch_msd_partition(const u64* keys, u64 n, u64 flip, void* state, u64 kmin, u64 kmax,
                          u64* out, int num_sms, cudaStream_t st) {
  MsdState* ms = (MsdState*)state;
  cudaMemsetAsync(ms, 0, kMsdClear, st);
  msd_set_span_kernel<<<1, 1, 0, st>>>(ms, kmin, kmax);
  u64 blocks = (n + 512 * 8 - 1) / (512 * 8);
  if (blocks > (u64)num_sms * 4) blocks = (u64)num_sms * 4;
  if (blocks < 1) blocks = 1;
  msd_hist_kernel<<<(unsigned)blocks, 512, 0, st>>>(keys, n, flip, ms);
  msd_scan_kernel<<<1, 1024, 0, st>>>(ms);
  const u64 chunks = (n + kScChunk - 1) / kScChunk;
  if (chunks)
    msd_scatter_kernel<false><<<(unsigned)chunks, kScThreads, 0, st>>>(keys, nullptr, n, flip, ms,
                                                                       out, nullptr, flip);
}

size_t msd_maxb_offset() { return offsetof(MsdState, maxb); }
size_t msd_overflow_offset() { return offsetof(MsdState, overflow); }

// keys (and vals) -> tmp (bucketed) -> dk/dv sorted; dk may equal keys
constexpr size_t kBsSmem = bs_smem_bytes(kBucketCap, true);

void launch_msd_sort(const u64* keys, const u64* vals, u64 n, u64 flip, void* state, u64* tk,
                     u64* tv, u64* dk, u64* dv, u32 maxb, int num_sms, cudaStream_t st) {
  MsdState* ms = (MsdState*)state;
  const u64 chunk = msd_chunk(n, num_sms);
  const u64 chunks = (n + chunk - 1) / chunk;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(bucket_sort_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBsSmem);
    cudaFuncSetAttribute(bucket_sort_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBsSmem);
    cudaFuncSetAttribute(msd_scatter_staged_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kStSmem);
    attr_dev = dev;
  }
  const bool large = maxb > kWarpBucketMax;
  const u32 cap = (maxb + kBsThreads - 1) / kBsThreads * kBsThreads;  // <= kBucketCap
  if (vals) {
    launch_pdl(kPdlMsd, msd_scatter_chunk_kernel<true>, (unsigned)chunks, 1024, 0, st, keys, vals,
               n, flip, (const MsdState*)ms, chunk, tk, tv);
    launch_pdl(kPdlMsd, bucket_small_kernel<true>, kMsdBuckets / 8, 256, 0, st, (const u64*)tk,
               (const u64*)tv, (const MsdState*)ms, flip, dk, dv);
    if (large)
      launch_pdl(kPdlMsd, bucket_sort_kernel<true>, kMsdBuckets, kBsThreads,
                 bs_smem_bytes(cap, true), st, (const u64*)tk, (const u64*)tv,
                 (const MsdState*)ms, flip, dk, dv, cap);
  } else {
    launch_pdl(kPdlMsd, msd_scatter_staged_kernel, (unsigned)chunks, 1024, kStSmem, st, keys, n,
               flip, (const MsdState*)ms, chunk, tk);
    launch_pdl(kPdlMsd, bucket_small_kernel<false>, kMsdBuckets / 8, 256, 0, st, (const u64*)tk,
               (const u64*)nullptr, (const MsdState*)ms, flip, dk, (u64*)nullptr);
    if (large)
      launch_pdl(kPdlMsd, bucket_sort_kernel<false>, kMsdBuckets, kBsThreads,
                 bs_smem_bytes(cap, false), st, (const u64*)tk, (const u64*)nullptr,
                 (const MsdState*)ms, flip, dk, (u64*)nullptr, cap);
  }
}

}  // namespace cafs
