// radix.cu -- K6: on-device LSD radix sort (the fallback engine) and the
// single-CTA small sorts.
//
// Replaces fallback_sort (sorter.py:132-138, numpy's host introsort) and, for
// more than kSmallSortMax pairs, radix_sort_pairs (_kernels.py:185-214).
//
// Onesweep-style LSD: one read computes all eight 8-bit digit histograms
// (digits constant over the array are skipped), then one kernel per digit
// pass: 8192-key tiles taken in launch order from an atomic counter, stable
// in-tile ranking with 8-ballot warp multisplit (no __match_any_sync -- it
// measured ~0.26 lanes/clk/SM on B200), a decoupled look-back over per-tile
// digit aggregates for the global offsets, and a shared-memory staged scatter
// so runs of equal digits leave the SM as coalesced stores.  Look-back state
// words carry a per-pass epoch, so no buffer is cleared between passes/calls.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kOsThreads = 512;
constexpr int kOsWarps = kOsThreads / 32;
constexpr int kOsItems = 16;
constexpr int kOsTile = kOsThreads * kOsItems;  // 8192 keys

// ---------------- histograms of all 8 digits in one read ----------------
__global__ void __launch_bounds__(512)
    radix_hist_kernel(const u64* __restrict__ keys, u64 n, u64 flip, u32* ghist) {
  __shared__ u32 h[8][256];
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 v = keys[i] ^ flip;
#pragma unroll
    for (int p = 0; p < 8; ++p) atomicAdd(&h[p][(v >> (8 * p)) & 255], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 256; i += blockDim.x) {
    const u32 c = (&h[0][0])[i];
    if (c) atomicAdd(&ghist[i], c);
  }
}

// exclusive digit offsets per pass + "digit constant over the array" flags
__global__ void radix_prep_kernel(const u32* ghist, u64 n, u32* gbase, int* trivial) {
  const int p = blockIdx.x;  // 8 blocks of 256 threads
  const int d = threadIdx.x;
  __shared__ u32 s[256];
  __shared__ int triv;
  if (d == 0) triv = 0;
  const u32 c = ghist[p * 256 + d];
  s[d] = c;
  __syncthreads();
  if ((u64)c == n) triv = 1;
  // inclusive scan (Hillis-Steele, 256 entries)
  for (int o = 1; o < 256; o <<= 1) {
    u32 t = d >= o ? s[d - o] : 0;
    __syncthreads();
    s[d] += t;
    __syncthreads();
  }
  gbase[p * 256 + d] = s[d] - c;
  __syncthreads();
  if (d == 0) trivial[p] = triv;
}

// state word: [63:34] epoch | [33:32] flag | [31:0] value
constexpr u64 kFlagAgg = 1, kFlagIncl = 2;
// epoch: 1 .. 2^30-1, never 0 (the buffer is zeroed once at allocation)
__device__ __forceinline__ u64 pack_state(u32 epoch, u64 flag, u32 v) {
  return ((u64)(epoch & 0x3FFFFFFFu) << 34) | (flag << 32) | (u64)v;
}

template <bool HAS_VAL>
__global__ void __launch_bounds__(kOsThreads)
    onesweep_kernel(const u64* __restrict__ src, const u64* __restrict__ srcv, u64* __restrict__ dst,
                    u64* __restrict__ dstv, u64 n, int shift, u64 flip_in, u64 flip_out,
                    const u32* __restrict__ gbase, u64* tile_state, u32* tile_counter, u32 epoch) {
  extern __shared__ __align__(16) unsigned char smem[];
  u64* buf = (u64*)smem;                                             // [kOsTile]
  u64* vbuf = buf + kOsTile;                                         // [kOsTile] if HAS_VAL
  u32* wcnt = (u32*)(HAS_VAL ? (vbuf + kOsTile) : (buf + kOsTile));  // [kOsWarps][256]
  __shared__ u32 tot[256], dstart[256], gpos[256];
  __shared__ u32 tile_sh;
  __shared__ u32 wsum[8];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) tile_sh = atomicAdd(tile_counter, 1u);
  for (int i = lane; i < 256; i += 32) wcnt[wid * 256 + i] = 0;
  __syncthreads();
  const u32 tile = tile_sh;
  const u64 tbase = (u64)tile * kOsTile;
  const u64 wbase = tbase + (u64)wid * (kOsItems * 32);

  u64 k[kOsItems];
  u64 v[HAS_VAL ? kOsItems : 1];
  u32 rank[kOsItems];
#pragma unroll
  for (int j = 0; j < kOsItems; ++j) {
    const u64 idx = wbase + j * 32 + lane;
    if (idx < n) {
      k[j] = src[idx] ^ flip_in;
      if (HAS_VAL) v[j] = srcv[idx];
    } else {
      k[j] = 0;
      if (HAS_VAL) v[j] = 0;
    }
  }
  u32* my = wcnt + wid * 256;
#pragma unroll
  for (int j = 0; j < kOsItems; ++j) {
    const u64 idx = wbase + j * 32 + lane;
    const bool valid = idx < n;
    const u32 d = (u32)(k[j] >> shift) & 255u;
    u32 peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const u32 bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
      peers &= ((d >> b) & 1u) ? bb : ~bb;
    }
    u32 before = 0;
    if (valid) before = my[d];
    __syncwarp();
    if (valid) {
      rank[j] = before + __popc(peers & lanemask_lt());
      const int leader = 31 - __clz(peers);
      if (lane == leader) my[d] = before + __popc(peers);
    }
    __syncwarp();
  }
  __syncthreads();

  // per digit: tile total, exclusive prefix across warps
  u32 acc = 0, lane_incl = 0;
  if (tid < 256) {
#pragma unroll 4
    for (int w = 0; w < kOsWarps; ++w) {
      const u32 c = wcnt[w * 256 + tid];
      wcnt[w * 256 + tid] = acc;
      acc += c;
    }
    tot[tid] = acc;
    // publish this tile's aggregate (or inclusive prefix for tile 0)
    *((volatile u64*)(tile_state + (u64)tile * 256 + tid)) =
        pack_state(epoch, tile == 0 ? kFlagIncl : kFlagAgg, acc);
    lane_incl = acc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 t = __shfl_up_sync(0xffffffffu, lane_incl, o);
      if (lane >= o) lane_incl += t;
    }
    if (lane == 31) wsum[wid] = lane_incl;
  }
  __syncthreads();
  if (tid < 256) {
    u32 pre = 0;
    for (int w = 0; w < wid; ++w) pre += wsum[w];
    dstart[tid] = pre + lane_incl - acc;
    // decoupled look-back over the preceding tiles' digit counts
    // windowed: the states of 8 predecessors are loaded in one round trip and
    // consumed nearest-first until an inclusive prefix is found; an unpublished
    // state stops the window and is polled again
    u32 excl = 0;
    if (tile > 0) {
      int t = (int)tile - 1;
      bool done = false;
      while (!done) {
        u64 stw[8];
#pragma unroll
        for (int w = 0; w < 8; ++w)
          stw[w] = t - w >= 0 ? *((volatile u64*)(tile_state + (u64)(t - w) * 256 + tid)) : 0ull;
        int used = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) {
          if (done || used != w) break;
          const u64 sv = stw[w];
          if ((u32)(sv >> 34) != epoch) break;  // not yet published in this pass
          excl += (u32)sv;
          used = w + 1;
          if (((sv >> 32) & 3) == kFlagIncl) done = true;
        }
        t -= used;
      }
      *((volatile u64*)(tile_state + (u64)tile * 256 + tid)) =
          pack_state(epoch, kFlagIncl, excl + acc);
    }
    gpos[tid] = gbase[tid] + excl;
  }
  __syncthreads();

  // stage in tile order, then scatter with coalesced runs
#pragma unroll
  for (int j = 0; j < kOsItems; ++j) {
    const u64 idx = wbase + j * 32 + lane;
    if (idx < n) {
      const u32 d = (u32)(k[j] >> shift) & 255u;
      const u32 lp = dstart[d] + wcnt[wid * 256 + d] + rank[j];
      buf[lp] = k[j];
      if (HAS_VAL) vbuf[lp] = v[j];
    }
  }
  __syncthreads();
  const u32 tn = (u32)((n - tbase) < (u64)kOsTile ? (n - tbase) : (u64)kOsTile);
  for (u32 i = tid; i < tn; i += kOsThreads) {
    const u64 key = buf[i];
    const u32 d = (u32)(key >> shift) & 255u;
    const u64 g = (u64)gpos[d] + (i - dstart[d]);
    dst[g] = key ^ flip_out;
    if (HAS_VAL) dstv[g] = vbuf[i];
  }
}

// ---------------- single-CTA sorts (<= kSmallSortMax) ----------------
// LSD radix sort of up to 8192 keys in shared memory (the reference's own
// pair-sort algorithm, _kernels.py:185-214: stable 8-bit digits), carrying a
// 16-bit index so pairs keep their counts.  Bytes that are equal across all
// keys (OR == AND) are skipped: dictionary codes need 2 passes, not 8.  Each
// warp ranks a contiguous segment with the 8-ballot multisplit, so the sort is
// stable.  Used for the small-n fallback route and the main route's
// (key, count) pairs, which also get their exclusive offsets (emit's input).
template <bool PAIRS>
__global__ void __launch_bounds__(1024, 1)
    small_sort_kernel(u64* keys_io, const u64* in_cnt, u64 n_arg, u64 flip, DevCtl* ctl,
                      u64 expect_total, u64* out_keys, u64* out_cnt, u64* out_offs, int gate,
                      u64* gkeys, u64* gcnt, const u32* glist) {
  pdl_begin();
  extern __shared__ __align__(16) unsigned char smem[];
  u64* kb = (u64*)smem;                                       // [2][kSmallSortMax]
  unsigned short* ib = (unsigned short*)(kb + 2 * kSmallSortMax);  // [2][kSmallSortMax]
  u32* wcnt = (u32*)(ib + 2 * kSmallSortMax);                 // [32][256]
  __shared__ u32 dstart[256], wsum8[8];
  __shared__ u64 red_or[32], red_and[32];
  __shared__ u64 wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  u64 n = n_arg;
  if (ctl && expect_total == kExpectCtlN) expect_total = ctl->n_global;  // sharded merge
  if (PAIRS && ctl) {
    if (ctl->overflow || ctl->pairs_ready || !gate_open(ctl, gate)) return;  // ready: dense path
    if (gkeys) {
      // gather mode (the pipeline holds no compaction kernel): the table's
      // claimed slots, listed per stripe, become the pairs in keys_io / in_cnt
      // (what compact_kernel writes) and are re-zeroed; too many for this
      // kernel: the host compacts before its large sort
      __shared__ u32 spre[kListStripes + 1];
      __shared__ u32 wtot[4];
      u32 f = 0;
      if (tid < (int)kListStripes) {
        const u32 g = ctl->g_fill[tid];
        f = g < kStripeCap ? g : (u32)kStripeCap;
      }
      u32 inc = f;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
      }
      if (tid < (int)kListStripes && lane == 31) wtot[wid] = inc;
      __syncthreads();
      if (tid < (int)kListStripes) {
        u32 pre = 0;
        for (int w = 0; w < wid; ++w) pre += wtot[w];
        spre[tid] = pre + inc - f;
        if (tid == (int)kListStripes - 1) spre[kListStripes] = pre + inc;
      }
      __syncthreads();
      const u64 tot = spre[kListStripes];
      const u64 e = ctl->empty_key_count;
      if (tot > kGlobalCap) {  // stripes have headroom; the table's capacity is the guard
        if (tid == 0) ctl->overflow = 1;
        return;
      }
      if (tot + (e ? 1 : 0) > (u64)kSmallSortMax) {
        if (tid == 0) { ctl->need_large = 1; ctl->need_compact = 1; }
        return;
      }
      u64* cnt_io = const_cast<u64*>(in_cnt);
      for (u32 i = tid; i < (u32)tot; i += 1024) {
        u32 s2 = 0;  // the stripe holding pair i
#pragma unroll
        for (u32 st2 = kListStripes / 2; st2 > 0; st2 >>= 1)
          if (spre[s2 + st2] <= i) s2 += st2;
        const u32 h = glist[(u64)s2 * kStripeCap + (i - spre[s2])];
        keys_io[i] = gkeys[h];
        cnt_io[i] = gcnt[h];
        gkeys[h] = kEmpty;
        gcnt[h] = 0;
      }
      if (tid == 0 && e) { keys_io[tot] = kEmpty; cnt_io[tot] = e; }
      n = tot + (e ? 1 : 0);
      __syncthreads();  // the pairs are read back below by other threads
    } else {
      n = ctl->npairs;
      if (n > (u64)kSmallSortMax) {
        if (tid == 0) ctl->need_large = 1;
        return;
      }
    }
  }
  u64 vor = 0, vand = ~0ull;
  {  // all loads in flight before any use (one round trip, not n/1024)
    u64 lk[kSmallSortMax / 1024];
#pragma unroll
    for (int j = 0; j < (int)(kSmallSortMax / 1024); ++j) {
      const u32 i = tid + j * 1024;
      lk[j] = i < n ? keys_io[i] ^ flip : 0;
    }
#pragma unroll
    for (int j = 0; j < (int)(kSmallSortMax / 1024); ++j) {
      const u32 i = tid + j * 1024;
      if (i < n) {
        kb[i] = lk[j];
        ib[i] = (unsigned short)i;
        vor |= lk[j];
        vand &= lk[j];
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    vor |= __shfl_xor_sync(0xffffffffu, vor, o);
    vand &= __shfl_xor_sync(0xffffffffu, vand, o);
  }
  if (lane == 0) { red_or[wid] = vor; red_and[wid] = vand; }
  __syncthreads();
  vor = 0; vand = ~0ull;
  for (int w = 0; w < 32; ++w) { vor |= red_or[w]; vand &= red_and[w]; }
  const u64 vary = vor ^ vand;  // bits that differ between some keys

  int cur = 0;
  int nvary = 0;
  for (int p = 0; p < 8; ++p) nvary += ((vary >> (8 * p)) & 0xFF) != 0;
  if (n <= 1024 && nvary > 0) {
    // up to 1024 keys: a rank sort -- thread i counts the keys before its own
    // (smaller, or equal and earlier: stable) with broadcast reads, then
    // writes it to the other buffer; one barrier instead of a bitonic network
    u64 k = 0;
    u32 r = 0;
    if ((u64)tid < n) {
      k = kb[tid];
#pragma unroll 8
      for (u32 j = 0; j < (u32)n; ++j) {
        const u64 kj = kb[j];
        r += (kj < k || (kj == k && j < (u32)tid)) ? 1u : 0u;
      }
      kb[kSmallSortMax + r] = k;
      ib[kSmallSortMax + r] = ib[tid];
    }
    __syncthreads();
    cur = 1;
    nvary = 0;
  } else if (n <= kBitonicMax && nvary > 2) {
    // few keys, many varying bytes: one bitonic network (log2(P)(log2(P)+1)/2
    // barrier steps) beats up to 8 radix passes of fixed cost each
    u32 P = 2;
    while (P < n) P <<= 1;
    for (u32 i = n + tid; i < P; i += 1024) { kb[i] = kEmpty; ib[i] = 0xFFFF; }
    __syncthreads();
    for (u32 k = 2; k <= P; k <<= 1) {
      for (u32 j = k >> 1; j > 0; j >>= 1) {
        for (u32 i = tid; i < P; i += 1024) {
          const u32 q = i ^ j;
          if (q > i) {
            const u64 a = kb[i], b = kb[q];
            const u32 ia = ib[i], iq = ib[q];
            const bool gt = a > b || (a == b && ia > iq);  // (key, index) order: stable
            if (gt == ((i & k) == 0)) {
              kb[i] = b; kb[q] = a;
              ib[i] = (unsigned short)iq; ib[q] = (unsigned short)ia;
            }
          }
        }
        __syncthreads();
      }
    }
    nvary = 0;  // sorted: skip the radix passes
  }
  // each warp owns a contiguous, 32-aligned segment of at most 8 rounds
  const u32 seg = (u32)(((n + 31) / 32 + 31) / 32) * 32;  // items per warp (multiple of 32)
  const u32 w0 = wid * seg;
  for (int p = 0; p < 8 && nvary > 0; ++p) {
    if (((vary >> (8 * p)) & 0xFF) == 0) continue;
    const int shift = 8 * p;
    u64* src = kb + cur * kSmallSortMax;
    u64* dst = kb + (cur ^ 1) * kSmallSortMax;
    unsigned short* isrc = ib + cur * kSmallSortMax;
    unsigned short* idst = ib + (cur ^ 1) * kSmallSortMax;
    u32* my = wcnt + wid * 256;
    for (int i = lane; i < 256; i += 32) my[i] = 0;
    __syncwarp();
    u32 rank[8], dig[8];
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if ((u32)(r * 32) >= seg) break;  // uniform across the block
      const u32 idx = w0 + r * 32 + lane;
      const bool valid = (u32)(r * 32) < seg && idx < n;
      const u32 d = valid ? (u32)(src[idx] >> shift) & 255u : 0u;
      u32 peers = __ballot_sync(0xffffffffu, valid);
#pragma unroll
      for (int b = 0; b < 8; ++b) {
        const u32 bb = __ballot_sync(0xffffffffu, (d >> b) & 1u);
        peers &= ((d >> b) & 1u) ? bb : ~bb;
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
    if (tid < 256) {  // exclusive prefix over warps, then over digits
      u32 acc = 0;
      for (int w = 0; w < 32; ++w) {
        const u32 c = wcnt[w * 256 + tid];
        wcnt[w * 256 + tid] = acc;
        acc += c;
      }
      u32 incl = acc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum8[wid] = incl;
      dstart[tid] = incl - acc;
    }
    __syncthreads();
    if (tid < 256) {
      u32 pre = 0;
      for (int w = 0; w < wid; ++w) pre += wsum8[w];
      dstart[tid] += pre;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if ((u32)(r * 32) >= seg) break;
      const u32 idx = w0 + r * 32 + lane;
      if (idx < n) {
        const u32 pos = dstart[dig[r]] + wcnt[wid * 256 + dig[r]] + rank[r];
        dst[pos] = src[idx];
        idst[pos] = isrc[idx];
      }
    }
    __syncthreads();
    cur ^= 1;
  }
  const u64* sk = kb + cur * kSmallSortMax;
  const unsigned short* si = ib + cur * kSmallSortMax;
  if (!PAIRS) {
    for (u32 i = tid; i < n; i += 1024) keys_io[i] = sk[i] ^ flip;
    return;
  }
  // gather counts in key order and take the exclusive scan (8 items/thread)
  constexpr int IT = kSmallSortMax / 1024;
  u64 c[IT];
  u64 local = 0;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const u32 i = tid * IT + q;
    c[q] = i < n ? in_cnt[si[i]] : 0;
    local += c[q];
  }
  u64 incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u64 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    u64 w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u64 t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  u64 run = incl - local + (wid ? wsum[wid - 1] : 0);
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const u32 i = tid * IT + q;
    if (i < n) {
      out_keys[i] = sk[i];
      out_cnt[i] = c[q];
      out_offs[i] = run;
    }
    run += c[q];
  }
  if (tid == 1023) {
    const u64 total = wsum[31];
    out_offs[n] = total;
    if (ctl) {
      ctl->total = total;
      ctl->npairs = n;
      ctl->sum_error = (total != expect_total);
      ctl->pairs_ready = (total == expect_total);
    }
  }
}

// ---------------- multi-block exclusive scan (large pair sets) ----------------
constexpr int kScanItems = 8192;  // per block: 1024 threads x 8

__global__ void __launch_bounds__(1024) scan_reduce_kernel(const u64* in, u64 n, u64* bsum) {
  pdl_begin();
  __shared__ u64 w[32];
  const u64 b0 = (u64)blockIdx.x * kScanItems;
  u64 s = 0;
  for (int q = 0; q < 8; ++q) {
    const u64 i = b0 + threadIdx.x + q * 1024;
    if (i < n) s += in[i];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) w[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    u64 t = 0;
    for (int i = 0; i < 32; ++i) t += w[i];
    bsum[blockIdx.x] = t;
  }
}

__global__ void scan_top_kernel(u64* bsum, u64 nb, u64 n, u64* offs_end, DevCtl* ctl,
                                u64 expect_total) {
  pdl_begin();
  if (threadIdx.x != 0) return;
  u64 run = 0;
  for (u64 b = 0; b < nb; ++b) { const u64 c = bsum[b]; bsum[b] = run; run += c; }
  *offs_end = run;
  if (ctl) {
    ctl->total = run;
    ctl->npairs = n;
    ctl->sum_error = (run != expect_total);
    ctl->pairs_ready = (run == expect_total);
  }
}

__global__ void __launch_bounds__(1024)
    scan_apply_kernel(const u64* in, u64 n, const u64* bsum, u64* out) {
  pdl_begin();
  __shared__ u64 w[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u64 b0 = (u64)blockIdx.x * kScanItems + (u64)tid * 8;
  u64 c[8], local = 0;
  for (int q = 0; q < 8; ++q) { c[q] = (b0 + q < n) ? in[b0 + q] : 0; local += c[q]; }
  u64 incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    u64 t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) w[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    u64 x = w[lane];
    for (int o = 1; o < 32; o <<= 1) {
      u64 t = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += t;
    }
    w[lane] = x;
  }
  __syncthreads();
  u64 run = bsum[blockIdx.x] + incl - local + (wid ? w[wid - 1] : 0);
  for (int q = 0; q < 8; ++q) {
    if (b0 + q < n) out[b0 + q] = run;
    run += c[q];
  }
}

// ---------------- host-side launchers ----------------
size_t onesweep_smem(bool has_val) {
  return (size_t)kOsTile * 8 * (has_val ? 2 : 1) + (size_t)kOsWarps * 256 * 4;
}
u64 onesweep_tiles(u64 n) { return (n + kOsTile - 1) / kOsTile; }

void launch_radix_hist(const u64* keys, u64 n, u64 flip, u32* ghist, int num_sms,
                       cudaStream_t st) {
  u64 blocks = (n + 512 * 16 - 1) / (512 * 16);
  if (blocks > (u64)num_sms * 4) blocks = (u64)num_sms * 4;
  if (blocks < 1) blocks = 1;
  radix_hist_kernel<<<(unsigned)blocks, 512, 0, st>>>(keys, n, flip, ghist);
}

void launch_radix_prep(const u32* ghist, u64 n, u32* gbase, int* trivial, cudaStream_t st) {
  radix_prep_kernel<<<8, 256, 0, st>>>(ghist, n, gbase, trivial);
}

cudaError_t launch_onesweep(const u64* src, const u64* srcv, u64* dst, u64* dstv, u64 n, int pass,
                            u64 flip_in, u64 flip_out, const u32* gbase, u64* tile_state,
                            u32* tile_counter, u32 epoch, cudaStream_t st) {
  const bool hv = srcv != nullptr;
  const size_t sm = onesweep_smem(hv);
  const u64 tiles = onesweep_tiles(n);
  cudaError_t e;
  if (hv) {
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      e = cudaFuncSetAttribute(onesweep_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sm);
      if (e != cudaSuccess) return e;
      attr_dev = dev;
    }
    onesweep_kernel<true><<<(unsigned)tiles, kOsThreads, sm, st>>>(
        src, srcv, dst, dstv, n, 8 * pass, flip_in, flip_out, gbase, tile_state, tile_counter,
        epoch);
  } else {
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      e = cudaFuncSetAttribute(onesweep_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sm);
      if (e != cudaSuccess) return e;
      attr_dev = dev;
    }
    onesweep_kernel<false><<<(unsigned)tiles, kOsThreads, sm, st>>>(
        src, nullptr, dst, nullptr, n, 8 * pass, flip_in, flip_out, gbase, tile_state,
        tile_counter, epoch);
  }
  return cudaGetLastError();
}

size_t small_sort_smem() { return (size_t)kSmallSortMax * (16 + 4) + 32 * 256 * 4; }

cudaError_t launch_small_sort_keys(u64* keys, u64 n, u64 flip, cudaStream_t st) {
  const size_t sm = small_sort_smem();
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(small_sort_kernel<false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  small_sort_kernel<false><<<1, 1024, sm, st>>>(keys, nullptr, n, flip, nullptr, 0, nullptr,
                                                nullptr, nullptr, kGateNone, nullptr, nullptr,
                                                nullptr);
  return cudaGetLastError();
}

cudaError_t launch_small_sort_pairs(u64* keys, const u64* cnt, u64 n, DevCtl* ctl, u64 expect,
                                    u64* out_keys, u64* out_cnt, u64* out_offs, cudaStream_t st,
                                    int gate, u64* gkeys, u64* gcnt, const u32* glist) {
  const size_t sm = small_sort_smem();
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(small_sort_kernel<true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  return launch_pdl(kPdlPairSort, small_sort_kernel<true>, 1, 1024, sm, st, keys, cnt, n, (u64)0, ctl, expect,
                    out_keys, out_cnt, out_offs, gate, gkeys, gcnt, glist);
}

void launch_scan(const u64* in, u64 n, u64* bsum, u64* out_offs, DevCtl* ctl, u64 expect,
                 cudaStream_t st) {
  const u64 nb = (n + kScanItems - 1) / kScanItems;
  launch_pdl(kPdlMsd, scan_reduce_kernel, (unsigned)(nb ? nb : 1), 1024, 0, st, in, n, bsum);
  launch_pdl(kPdlMsd, scan_top_kernel, 1, 32, 0, st, bsum, nb, n, out_offs + n, ctl, expect);
  launch_pdl(kPdlMsd, scan_apply_kernel, (unsigned)(nb ? nb : 1), 1024, 0, st, in, n,
             (const u64*)bsum, out_offs);
}

}  // namespace cafs
