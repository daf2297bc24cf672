// hashpart.cu -- K3 for columns without a dense window: a partitioned count
// whose output is the sorted (key, count) pairs, with no global hash table and
// no pair sort.
//
// Replaces count_sequence + BucketTable (_kernels.py:25-81, buckets.py:172-292)
// and reconstruct's pair sort (sorter.py:228-241, 276-285) on the MAIN route
// when the sample saw no dense key window.  The reference folds runs into a
// 4-slot bucket cache and spills what does not fit; this path keeps that
// contract (every element lands in exactly one partial (key, count) cell or
// in the spill) and then finishes the spill exactly, on chip:
//
//   hp_count_kernel, one persistent CTA per SM, 1024 threads
//     * warp 0 streams the CTA's contiguous row range through a 3 x 31 KB TMA
//       ring (cp.async.bulk + mbarrier complete_tx);
//     * 31 consumer warps look every key up in a two-choice table of 2-slot
//       buckets in shared memory (8192 slots): two independent LDS.128, four
//       compares, one shared atomic per hit.  No sentinel test: an empty slot
//       holds a marker that is never one of the probing key's two buckets'
//       keys (the marker of E0's buckets is E1, E1's buckets are disjoint);
//     * a miss goes to the warp's queue.  While the table has room, 32 queued
//       misses are resolved together (CAS claims); once it is nearly full a
//       miss is spilled without probing: 32 keys at a time, coalesced, into the
//       part of the CTA's own input range it has already streamed (the emit
//       overwrites the input anyway) -- no extra memory, no global atomics;
//     * tail: the CTA's cells (occupied slots) and its spill are counting-sorted
//       by key-range partition (512 partitions, monotone in the key) into its
//       region of the cell buffer and of `part` (laid out like x).
//   hp_reduce_kernel, one CTA per partition (two per SM)
//     * gathers the partition's segments of every CTA's cells and spill into an
//       exact shared-memory table and sorts its distinct keys (bitonic) -- in
//       global key order, since partitions are key ranges;
//   hp_place_kernel, one CTA per partition
//     * prefix of the partitions' (pairs, rows), then the pairs at their global
//       positions with their emit offsets; the last one publishes npairs /
//       total / pairs_ready for the emit.
//   A partition with more than kHpPartCap distinct keys sets hp_overflow; the
//   host then writes the column back from the (intact) cells and spill and
//   sorts it with the fallback (abi.cu: main_finish).
//
// Partition map: 4096 fine bins over the sample's span [min, max] (keys
// outside clamp to the end bins), bin -> partition = half the sample mass
// before the bin + half the bin's position in the span, so that a partition
// holds at most ~2x its share of the rows (heavy keys) or of the value range
// (spread-out distinct keys).
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kHpThreads = 1024;
constexpr int kHpUnroll = 4;                 // 16-byte loads in flight per thread
constexpr u64 kHpRound = (u64)kHpUnroll * kHpThreads;  // vectors per CTA round
constexpr int kHpSLog2 = 14;
constexpr u32 kHpS = 1u << kHpSLog2;         // table slots
constexpr u32 kHpNB = kHpS / 2;              // 2-slot buckets
constexpr int kHpNBLog2 = kHpSLog2 - 1;
constexpr int kHpD = 2;                      // buckets a key may sit in (home, second choice)
constexpr u32 kHpFullClaims = kHpS - kHpS / 16;  // from here on a miss spills without probing
constexpr int kHpQ = 64;                     // per-warp miss queue
constexpr int kHpP = kHpParts;               // key-range partitions
constexpr int kHpFine = 2048;                // fine bins of the partition map
constexpr u32 kHpCellCap = kHpS + 16;        // cells per CTA (+ CTA 0's head / tail keys)
constexpr u32 kHpPartSlots = 4096;           // hp_reduce exact table
constexpr u32 kHpPartCap = 2048;             // distinct keys per partition (load <= 1/2)
constexpr u32 kHpListCap = kHpPartCap + kHpThreads;  // claims may overshoot by one per thread
constexpr u32 kHpStage = kHpPartCap + 1;     // staged pairs per partition (+ the ~0 sentinel)
static_assert(kHpP % 2 == 0 && kHpP <= 1024, "partition map: half by mass, half by position");

constexpr size_t kHpQueueBytes = (size_t)32 * kHpQ * 8;
constexpr size_t kHpCountSmem = (size_t)kHpS * 12 + kHpQueueBytes + (size_t)kHpFine * 2;
static_assert(kHpCountSmem + 11 * 1024 <= 232448, "shared memory budget");
constexpr size_t kHpReduceSmem = (size_t)kHpPartSlots * 12 + (size_t)kHpListCap * 16;

// the home bucket of a key (a cache of partial counts: a weak hash costs
// spills, never correctness)
__host__ __device__ __forceinline__ u32 hp_t(u64 v) {
  return (u32)(v >> 32) * 0x9E3779B1u + (u32)v;
}
__host__ __device__ __forceinline__ u32 hp_b1(u32 t) { return (t * 0x85EBCA77u) >> (32 - kHpNBLog2); }
// the second choice: an independent bucket (adjacent buckets would make the
// same few keys overflow in every CTA, piling their rows into one partition)
__host__ __device__ __forceinline__ u32 hp_b2(u32 t) { return (t * 0xC2B2AE3Du) >> (32 - kHpNBLog2); }

struct HpArgs {
  const void* x;   // column (keys of kind KK); its streamed part receives the spill
  u64 n;
  u64 flip;
  DevCtl* ctl;
  void* part;      // partitioned spill, same layout and key type as x
  u64* cellk;      // [grid][kHpCellCap] cells (key, count), grouped by partition
  u32* cellw;
  u32* cpofs;      // [grid][kHpP + 1] cell segment starts per partition
  u32* spofs;      // [grid][kHpP + 1] spill segment starts per partition
  u64* pd;         // [kHpP] pairs of each partition (hp_reduce -> hp_place)
  u64* pr;         // [kHpP] rows of each partition
  u64* pk_stage;   // [kHpP][kHpStage] each partition's sorted pairs (hp_reduce)
  u64* pc_stage;
  u64* pk;         // sorted pairs: keys, counts, offsets (npairs + 1)
  u64* pc;
  u64* poffs;
  u64 e0, e1;      // empty-slot markers: e1 in E0's two buckets ma, mb, e0 elsewhere
  u32 ma, mb;
  int gate;
  // the sharded merge (hp_reduce<KK, true>): every rank's sorted (key, count)
  // list gathered in rows [np, keys[cap], counts[cap]] of `row` words
  const u64* recv;
  u64 row, cap;
  int shard;
  // the emit's tile -> pair map (emit.cu), written by hp_place for the
  // single-GPU pipeline's emit of the whole column; null: not wanted
  u32* tile_pair;
  int kk;
};

__device__ __forceinline__ u64 hp_marker(const HpArgs& a, u32 b) {
  return (b == a.ma || b == a.mb) ? a.e1 : a.e0;
}

// Partition of a key: its fine bin over the sample span, mapped (pmap).
__device__ __forceinline__ u32 hp_part(u64 v, u64 lo, int sh, const unsigned short* pmap) {
  const u64 d = (v - lo) >> sh;
  const u32 f = v < lo ? 0u : (d < (u64)kHpFine ? (u32)d : (u32)(kHpFine - 1));
  return pmap[f];
}

// CTA c's rows: a contiguous range of whole stages of the 16-byte-aligned body.
__device__ __forceinline__ void hp_range(u64 body_keys, u64 skk, u32 c, u32 G, u64* k0, u64* k1) {
  const u64 chunks = (body_keys + skk - 1) / skk;
  const u64 per = (chunks + G - 1) / G;
  const u64 a = (u64)c * per * skk, b = a + per * skk;
  *k0 = a < body_keys ? a : body_keys;
  *k1 = b < body_keys ? b : body_keys;
}

// Exclusive scan of the kHpP partition counters by one warp (kHpScanPer per
// lane; the arrays are padded to a multiple of 32 with zeros); out[kHpP] = total.
constexpr int kHpScanPer = (kHpP + 31) / 32;
constexpr int kHpPad = 32 * kHpScanPer + 1;  // padded length of the per-partition arrays
__device__ __forceinline__ void hp_scan_parts(const u32* in, u32* out) {
  const int lane = threadIdx.x & 31;
  u32 v[kHpScanPer], s = 0;
#pragma unroll
  for (int j = 0; j < kHpScanPer; ++j) { v[j] = in[lane * kHpScanPer + j]; s += v[j]; }
  u32 inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  u32 run = inc - s;
#pragma unroll
  for (int j = 0; j < kHpScanPer; ++j) { out[lane * kHpScanPer + j] = run; run += v[j]; }
  // (counters past kHpP are zero, so out[kHpP] is already the total when padded)
  if (lane == 31) out[32 * kHpScanPer] = run;
}

// The spill of warp w lives in the vectors w itself has streamed: its j-th
// spilled key goes to chunk j / (32 * KPV) of its own (round, unroll) chunks.
template <int KPV>
__device__ __forceinline__ u64 hp_spill_pos(u64 v0, u32 w, u32 j) {
  const u32 ci = j / (32 * KPV), within = j % (32 * KPV);
  const u32 r = ci / kHpUnroll, q = ci % kHpUnroll;
  return (v0 + (u64)r * kHpRound + (u64)q * kHpThreads + (u64)w * 32) * KPV + within;
}

// The partition map from the estimate's 1024 order-mapped samples, by a whole
// 1024-thread CTA: span [lo, hi] -> shift sh (2^sh-wide fine bins), fine-bin
// histogram, bin -> partition (half sample mass before the bin, half its
// position in the span).  `fh` is kHpFine u32 of scratch, `rl` 128 u64.
__device__ void hp_build_pmap(const u64* samp, unsigned short* pmap, u32* fh, u64* rl, u64* s_lo,
                              int* s_sh) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (u32 i = tid; i < kHpFine; i += kHpThreads) fh[i] = 0;
  const u64 sv = __ldcg(&samp[tid]);
  u64 lo = sv, hi = sv;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const u64 l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  if (lane == 0) { rl[wid] = lo; rl[32 + wid] = hi; }
  __syncthreads();
  if (wid == 0) {
    lo = rl[lane];
    hi = rl[32 + lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const u64 l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
      lo = l2 < lo ? l2 : lo;
      hi = h2 > hi ? h2 : hi;
    }
    if (lane == 0) {
      int sh = 0;
      while (sh < 63 && ((hi - lo) >> sh) >= (u64)kHpFine) ++sh;
      *s_lo = lo;
      *s_sh = sh;
    }
  }
  __syncthreads();
  const u64 d = (sv - *s_lo) >> *s_sh;
  atomicAdd(&fh[d < (u64)kHpFine ? (u32)d : kHpFine - 1], 1u);
  __syncthreads();
  // exclusive scan of the fine bins: kHpFine / 1024 per thread
  constexpr int FPT = kHpFine / kHpThreads;
  u32 vf[FPT], s = 0;
#pragma unroll
  for (int j = 0; j < FPT; ++j) { vf[j] = fh[tid * FPT + j]; s += vf[j]; }
  u32 inc = s;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  u32* ws = (u32*)(rl + 64);
  if (lane == 31) ws[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    u32 w = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    ws[32 + lane] = w;
  }
  __syncthreads();
  u32 run = inc - s + (wid ? ws[32 + wid - 1] : 0);
#pragma unroll
  for (int j = 0; j < FPT; ++j) {
    const u32 f = tid * FPT + j;
    const u32 p = (run * (kHpP / 2)) / kSampleTarget + (f * (kHpP / 2)) / kHpFine;
    pmap[f] = (unsigned short)(p < (u32)kHpP ? p : kHpP - 1);
    run += vf[j];
  }
  __syncthreads();
}

template <int KK>
__global__ void __launch_bounds__(kHpThreads, 1) hp_count_kernel(HpArgs a) {
  pdl_begin();
  if (!gate_open(a.ctl, a.gate)) return;
  using K = typename KeyT<KK>::T;
  constexpr int KPV = 16 / sizeof(K);  // keys per 16-byte vector
  constexpr int KPT = kHpUnroll * KPV;  // keys per thread per round
  extern __shared__ __align__(128) unsigned char smem[];
  u64* tkeys = (u64*)smem;                              // [kHpS]
  u32* tcnt = (u32*)(tkeys + kHpS);                     // [kHpS]
  u64* queue = (u64*)(tcnt + kHpS);                     // [32][kHpQ]
  unsigned short* pmap = (unsigned short*)(queue + 32 * kHpQ);  // [kHpFine]
  __shared__ u32 shist[kHpPad], hstart[kHpPad], lhist[kHpPad], lstart[kHpPad];
  __shared__ u32 wsp[33];  // spilled keys per warp, then their prefix
  __shared__ u32 ncell_extra, sclaims;
  __shared__ u64 extra_k[16];
  __shared__ u64 s_lo;
  __shared__ int s_sh;

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u32 c = blockIdx.x, G = gridDim.x;
  const u64 flip = a.flip, n = a.n;
  const K* xk = (const K*)a.x;
  const u64 mis = (((uintptr_t)a.x) & 15) / sizeof(K);
  const u64 head0 = mis ? (u64)KPV - mis : 0;
  const u64 head = head0 < n ? head0 : n;
  const u64 body = (n - head) / KPV * KPV;
  K* xb = (K*)(xk + head);
  const ulonglong2* xv = (const ulonglong2*)xb;
  u64 v0, v1;  // this CTA's vectors (whole rounds)
  hp_range(body / KPV, kHpRound, c, G, &v0, &v1);

  if (tid == 0) { ncell_extra = 0; sclaims = 0; }
  if (tid < 33) wsp[tid] = 0;
  // ---- prologue: partition map from the estimate's 1024 samples ----
  hp_build_pmap(est_scratch(a.ctl)->samples, pmap, tcnt, queue, &s_lo, &s_sh);
  for (u32 i = tid; i < kHpS; i += kHpThreads) {
    tkeys[i] = hp_marker(a, i >> 1);
    tcnt[i] = 0;
  }
  for (u32 i = tid; i < kHpPad; i += kHpThreads) shist[i] = 0;
  __syncthreads();
  const u64 plo = s_lo;
  const int psh = s_sh;
  const u32 tbase = smem_u32(tkeys), cbase = smem_u32(tcnt);
  u64* wq = queue + (size_t)wid * kHpQ;
  u32 qn = 0;   // warp-uniform queue length
  u32 nsw = 0;  // warp-uniform: keys this warp has spilled

  // 32 queued misses (one per active lane) with the whole warp: while the
  // table has room, look again in the key's kHpD buckets and claim an empty
  // slot; what remains is spilled into vectors this warp has streamed
  auto resolve = [&](bool active, u64 u) {
    bool done = !active;
    if (*((volatile u32*)&sclaims) < kHpFullClaims && __any_sync(0xffffffffu, active)) {
      const u32 t = hp_t(u);
#pragma unroll
      for (int d = 0; d < kHpD; ++d) {
        if (!done) {
          const u32 bb = d ? hp_b2(t) : hp_b1(t);
          u64 t0, t1;
          asm volatile("ld.volatile.shared.v2.u64 {%0,%1}, [%2];"
                       : "=l"(t0), "=l"(t1) : "r"(tbase + bb * 16));
          const u64 mk = hp_marker(a, bb);
          int hit = t0 == u ? 0 : (t1 == u ? 1 : -1);
          if (hit < 0 && t0 == mk) {
            const u64 o = atomicCAS(&tkeys[2 * bb], mk, u);
            if (o == mk) atomicAdd(&sclaims, 1u);
            if (o == mk || o == u) hit = 0;
          }
          if (hit < 0 && t1 == mk) {
            const u64 o = atomicCAS(&tkeys[2 * bb + 1], mk, u);
            if (o == mk) atomicAdd(&sclaims, 1u);
            if (o == mk || o == u) hit = 1;
          }
          if (hit >= 0) { atomicAdd(&tcnt[2 * bb + hit], 1u); done = true; }
        }
      }
    }
    const bool sp = !done;
    const u32 m = __ballot_sync(0xffffffffu, sp);
    if (m) {
      if (sp) {
        xb[hp_spill_pos<KPV>(v0, wid, nsw + __popc(m & lanemask_lt()))] = key_unmap<KK>(u, flip);
        atomicAdd(&shist[hp_part(u, plo, psh, pmap)], 1u);
      }
      nsw += __popc(m);
    }
  };

  for (u64 r0v = v0; r0v < v1; r0v += kHpRound) {  // CTA-uniform rounds
    ulonglong2 w[kHpUnroll];
    u32 vmask = 0;
#pragma unroll
    for (int q = 0; q < kHpUnroll; ++q) {
      const u64 i = r0v + (u64)q * kHpThreads + tid;
      w[q] = make_ulonglong2(0, 0);
      if (i < v1) { w[q] = ld_stream_v2(xv + i); vmask |= ((1u << KPV) - 1) << (q * KPV); }
    }
    u64 v[KPT];
#pragma unroll
    for (int q = 0; q < kHpUnroll; ++q) {
      if constexpr (KPV == 2) {
        v[q * 2] = key_map<KK>((K)w[q].x, flip);
        v[q * 2 + 1] = key_map<KK>((K)w[q].y, flip);
      } else {
        v[q * 4] = key_map<KK>((K)w[q].x, flip);
        v[q * 4 + 1] = key_map<KK>((K)(w[q].x >> 32), flip);
        v[q * 4 + 2] = key_map<KK>((K)w[q].y, flip);
        v[q * 4 + 3] = key_map<KK>((K)(w[q].y >> 32), flip);
      }
    }
    u32 mm = 0;  // this thread's misses
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      // one LDS.128 of the home bucket, a predicated RED on a hit
      const u32 b = hp_b1(hp_t(v[k]));
      u64 a0, a1;
      asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(a0), "=l"(a1) : "r"(tbase + b * 16));
      const bool hx = a0 == v[k], hy = a1 == v[k];
      const u32 live = (vmask >> k) & 1u;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p red.shared.add.u32 [%0], 1;\n\t}"
                   ::"r"(cbase + (2 * b + (u32)hy) * 4), "r"((u32)(hx | hy) & live) : "memory");
      mm |= (((u32)!(hx | hy)) & live) << k;
    }
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const bool miss = (mm >> k) & 1u;
      const u32 m = __ballot_sync(0xffffffffu, miss);
      if (m) {
        if (miss) wq[qn + __popc(m & lanemask_lt())] = v[k];
        qn += __popc(m);
        if (qn >= 32) {
          __syncwarp();
          const u64 u = wq[qn - 32 + lane];
          __syncwarp();
          qn -= 32;
          resolve(true, u);
        }
      }
    }
  }
  __syncwarp();
  {
    const u64 u = (u32)lane < qn ? wq[lane] : 0ull;
    __syncwarp();
    resolve((u32)lane < qn, u);
  }
  if (lane == 0) wsp[wid] = nsw;
  __syncthreads();
  // head and tail keys (< KPV each, CTA 0): the table, else extra cells
  if (c == 0 && wid == 1) {
    const u64 tail0 = head + body;
    const bool hv = (u64)lane < head, tv = (u64)lane < n - tail0;
    for (int r = 0; r < 2; ++r) {
      const bool act = r == 0 ? hv : tv;
      const u64 u = act ? key_map<KK>(xk[r == 0 ? lane : tail0 + lane], flip) : 0ull;
      bool done = !act;
      const u32 t = hp_t(u);
      for (int d = 0; d < kHpD && !done; ++d) {
        const u32 bb = d ? hp_b2(t) : hp_b1(t);
        const u64 mk = hp_marker(a, bb);
        for (int s2 = 0; s2 < 2 && !done; ++s2) {
          const u32 slot = 2 * bb + s2;
          u64 k = atomicCAS(&tkeys[slot], mk, u);
          if (k == mk) k = u;
          if (k == u) { atomicAdd(&tcnt[slot], 1u); done = true; }
        }
      }
      if (!done) extra_k[atomicAdd(&ncell_extra, 1u)] = u;
    }
  }
  if (wid == 0) {  // prefix of the warps' spills
    const u32 x = wsp[lane];
    u32 inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    __syncwarp();
    wsp[lane] = inc - x;
    if (lane == 31) wsp[32] = inc;
  }
  for (u32 i = tid; i < kHpPad; i += kHpThreads) lhist[i] = 0;
  __syncthreads();

  // ---- tail 1: the cells, counting-sorted by partition into this CTA's region.
  // A thread keeps its slots' destinations and counts in registers, which
  // frees the count array as the staging area: the keys go through it in two
  // passes, the counts in one, every global store coalesced ----
  constexpr int kCpt = kHpS / kHpThreads;  // slots per thread
  u32 cpos[kCpt + 1], ccnt[kCpt];  // destination (partition | rank << 16, then the position)
#pragma unroll
  for (int j = 0; j < kCpt; ++j) {
    const u32 slot = tid + j * kHpThreads;
    const u64 k = tkeys[slot];
    ccnt[j] = tcnt[slot];
    cpos[j] = ~0u;
    if (k != hp_marker(a, slot >> 1)) {
      const u32 pp = hp_part(k, plo, psh, pmap);
      cpos[j] = pp | (atomicAdd(&lhist[pp], 1u) << 16);
    }
  }
  cpos[kCpt] = ~0u;
  if ((u32)tid < ncell_extra) {
    const u32 pp = hp_part(extra_k[tid], plo, psh, pmap);
    cpos[kCpt] = pp | (atomicAdd(&lhist[pp], 1u) << 16);
  }
  __syncthreads();
  if (wid == 0) hp_scan_parts(lhist, lstart);
  else if (wid == 1) hp_scan_parts(shist, hstart);  // the spill's histogram, taken while spilling
  __syncthreads();
  for (u32 i = tid; i <= kHpP; i += kHpThreads) {
    a.cpofs[(size_t)c * (kHpP + 1) + i] = lstart[i];
    a.spofs[(size_t)c * (kHpP + 1) + i] = hstart[i];
  }
#pragma unroll
  for (int j = 0; j <= kCpt; ++j)
    if (cpos[j] != ~0u) cpos[j] = lstart[cpos[j] & 0xffffu] + (cpos[j] >> 16);
  const u32 ncells = lstart[kHpP];
  u64* gck = a.cellk + (size_t)c * kHpCellCap;
  u32* gcw = a.cellw + (size_t)c * kHpCellCap;
  u64* stk = (u64*)tcnt;  // staging: kHpS / 2 keys, or kHpS counts
  for (u32 lo = 0; lo < ncells; lo += kHpS / 2) {
    const u32 hi = lo + kHpS / 2 < ncells ? lo + kHpS / 2 : ncells;
#pragma unroll
    for (int j = 0; j <= kCpt; ++j)
      if (cpos[j] >= lo && cpos[j] < hi)
        stk[cpos[j] - lo] = j < kCpt ? tkeys[tid + j * kHpThreads] : extra_k[tid];
    __syncthreads();
    for (u32 i = lo + tid; i < hi; i += kHpThreads) gck[i] = stk[i - lo];
    __syncthreads();
  }
  {
    const u32 lo = 0, hi = ncells < kHpS ? ncells : kHpS;  // the (<= 16) cells past kHpS below
#pragma unroll
    for (int j = 0; j <= kCpt; ++j)
      if (cpos[j] < hi) tcnt[cpos[j]] = j < kCpt ? ccnt[j] : 1u;
    __syncthreads();
    for (u32 i = lo + tid; i < hi; i += kHpThreads) gcw[i] = tcnt[i];
#pragma unroll
    for (int j = 0; j <= kCpt; ++j)
      if (cpos[j] != ~0u && cpos[j] >= kHpS) gcw[cpos[j]] = j < kCpt ? ccnt[j] : 1u;
  }
  // ---- tail 2: the spill, grouped by partition in this CTA's rows of `part`:
  // a key's place is its partition's start (the histogram taken while
  // spilling) + its arrival rank (the order inside a partition is free); a
  // warp moves the keys it spilled itself ----
  __syncthreads();
  for (u32 i = tid; i < kHpP; i += kHpThreads) lhist[i] = 0;
  __syncthreads();
  K* outp = (K*)a.part + head + v0 * KPV;
  constexpr int kSpU = 4;
  for (u32 g0 = 0; g0 < nsw; g0 += 32 * kSpU) {
    K kv[kSpU];
#pragma unroll
    for (int j = 0; j < kSpU; ++j) {
      const u32 g = g0 + j * 32 + lane;
      if (g < nsw) kv[j] = *((volatile K*)&xb[hp_spill_pos<KPV>(v0, wid, g)]);
    }
#pragma unroll
    for (int j = 0; j < kSpU; ++j) {
      const u32 g = g0 + j * 32 + lane;
      if (g < nsw) {
        const u32 pp = hp_part(key_map<KK>(kv[j], flip), plo, psh, pmap);
        outp[hstart[pp] + atomicAdd(&lhist[pp], 1u)] = kv[j];
      }
    }
  }
  const u32 ns = wsp[32];
  if (tid == 0 && ns) atomicAdd(&a.ctl->g_updates, (u64)ns);
}

// ---- hp_reduce: one CTA per partition ----
// The partition's items are the segments [cpofs[c][p], cpofs[c][p+1]) of every
// CTA c's cells and [spofs[c][p], spofs[c][p+1]) of its spill, read as one flat
// list (a segment table in shared memory): a warp takes 128 consecutive items
// with kRdUnroll loads per lane in flight.  Output:
// the partition's sorted distinct keys and counts in its staging slot, and its
// (pairs, rows) in pd / pr for hp_place.
constexpr int kRdUnroll = 4;
template <int KK, bool SH>
__global__ void __launch_bounds__(kHpThreads, 2) hp_reduce_kernel(HpArgs a, u32 G) {
  pdl_begin();
  if (!gate_open(a.ctl, a.gate)) return;
  if (SH && a.ctl->merge_bad) return;
  using K = typename KeyT<KK>::T;
  constexpr int KPV = 16 / sizeof(K);
  extern __shared__ __align__(128) unsigned char smem[];
  u64* hk = (u64*)smem;                        // [kHpPartSlots]
  u32* hc = (u32*)(hk + kHpPartSlots);         // [kHpPartSlots]
  u64* lk = (u64*)(hc + kHpPartSlots);         // [kHpListCap]
  u64* lc = lk + kHpListCap;                   // [kHpListCap]
  __shared__ u32 segs[2 * 160 + 1];            // flat start of segment j (cells, then spill)
  __shared__ u32 sbeg[2 * 160];                // its first index in the source array
  __shared__ u32 rk[512];                      // rank sort: a key's rank
  __shared__ u32 claims, nd, ovf;
  __shared__ unsigned long long sent;
  __shared__ u64 wsum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u32 p = blockIdx.x;
  for (u32 i = tid; i < kHpPartSlots; i += kHpThreads) { hk[i] = kEmpty; hc[i] = 0; }
  if (tid == 0) { claims = 0; nd = 0; ovf = 0; sent = 0; }
  const u64 n = a.n;
  const u64 mis = (((uintptr_t)a.x) & 15) / sizeof(K);
  const u64 head0 = mis ? (u64)KPV - mis : 0;
  const u64 head = head0 < n ? head0 : n;
  const u64 body = (n - head) / KPV * KPV;
  const K* part = (const K*)a.part + head;
  // segment table: j < G cells of CTA j, G <= j < 2G spill of CTA j - G
  // (sharded merge: one segment per rank's list); segs = their flat starts
  const u32 nseg = SH ? G : 2 * G;
  u32 len = 0;
  if ((u32)tid < nseg) {
    const bool cell = (u32)tid < G;
    const u32 c = cell ? tid : tid - G;
    const u32* o = (cell ? a.cpofs : a.spofs) + (size_t)c * (kHpP + 1);
    const u32 b0 = o[p], b1 = o[p + 1];
    len = b1 - b0;
    u64 v0 = 0, v1;
    if (!cell) hp_range(body / KPV, kHpRound, c, G, &v0, &v1);
    // cells: index into cellk / cellw; spill: index into part (CTA range + segment)
    sbeg[tid] = cell ? (SH ? b0 : c * kHpCellCap + b0) : (u32)(v0 * KPV + b0);
  }
  u32 inc = len;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    u64 w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 t = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += t;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  if ((u32)tid <= nseg) segs[tid] = inc - len + (wid ? (u32)wsum[wid - 1] : 0u);
  __syncthreads();

  auto insert = [&](u64 k, u32 w) {
    if (k == kEmpty) { atomicAdd(&sent, (unsigned long long)w); return; }
    u32 h = (u32)((k * kGamma) >> (64 - 12));
    for (u32 pr = 0; pr < kHpPartSlots; ++pr) {
      u64 cur = *((volatile u64*)&hk[h]);
      if (cur == kEmpty) {
        if (*((volatile u32*)&claims) >= kHpPartCap) { ovf = 1; return; }
        cur = atomicCAS(&hk[h], kEmpty, k);
        if (cur == kEmpty) { atomicAdd(&claims, 1u); cur = k; }
      }
      if (cur == k) { atomicAdd(&hc[h], w); return; }
      h = (h + 1) & (kHpPartSlots - 1);
    }
    ovf = 1;
  };
  // Equal single-row items in a warp (a spilled heavy key fills whole
  // segments) are added once by their first lane instead of 32 serialised
  // shared atomics on one address.
  auto insert_agg = [&](u64 k, u32 w) {
    const bool one = w == 1;
    const u32 m1 = __ballot_sync(0xffffffffu, one);
    if (m1) {
      const int ld = __ffs(m1) - 1;
      const u64 kl = __shfl_sync(0xffffffffu, k, ld);
      const u32 me = __ballot_sync(0xffffffffu, one && k == kl);
      if (one && k == kl) w = lane == ld ? (u32)__popc(me) : 0u;
    }
    if (w) insert(k, w);
  };
  // The segments as one flat list: thread t takes items t, t + 1024, ... with
  // kRdUnroll loads in flight (an item's segment by binary search of the
  // table, mostly a broadcast: neighbours share a segment), so a partition
  // costs a few global round trips however its rows are spread over segments.
  const u32 total = segs[nseg];
  for (u32 i0 = 0; i0 < total; i0 += kHpThreads * kRdUnroll) {  // CTA-uniform
    u64 k[kRdUnroll];
    u32 w[kRdUnroll];
    u32 j = 0;  // the segment of this thread's previous item (its items ascend)
#pragma unroll
    for (int r = 0; r < kRdUnroll; ++r) {
      // a warp takes 128 consecutive items, 32 per step: the first item's
      // segment by binary search, the next ones' by a short walk from it
      const u32 i = i0 + (u32)wid * (32 * kRdUnroll) + r * 32 + lane;
      w[r] = 0;
      k[r] = 0;
      if (i < total) {
        bool found = false;
        if (r > 0) {
#pragma unroll
          for (int s2 = 0; s2 < 6 && !found; ++s2) {
            if (segs[j + 1] > i) found = true;
            else ++j;
          }
        }
        if (!found) {
          j = 0;
#pragma unroll
          for (u32 st = SH ? 16 : 256; st > 0; st >>= 1)  // sharded: nseg < 32 ranks
            if (j + st < nseg && segs[j + st] <= i) j += st;
        }
        const u32 off = sbeg[j] + (i - segs[j]);
        if (SH) {
          const u64* L = a.recv + (size_t)j * a.row;
          k[r] = L[1 + off];
          w[r] = (u32)L[1 + a.cap + off];
        } else if (j < G) {
          k[r] = a.cellk[off];
          w[r] = a.cellw[off];
        } else {
          k[r] = key_map<KK>(part[off], a.flip);
          w[r] = 1;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < kRdUnroll; ++r) insert_agg(k[r], w[r]);
  }
  __syncthreads();
  // compact the distinct keys (order is irrelevant: they are sorted next)
  for (u32 j = tid; j < kHpPartSlots; j += kHpThreads) {
    const u64 kk = hk[j];
    if (kk != kEmpty) {
      const u32 q = atomicAdd(&nd, 1u);
      if (q < kHpListCap) { lk[q] = kk; lc[q] = hc[j]; }
    }
  }
  __syncthreads();
  const bool bad = ovf || nd > kHpPartCap;
  const u32 d = bad ? 0u : nd;
  if (d <= 512) {
    // rank sort (the keys are distinct): key q moves to the number of keys
    // below it.  1024 / dpad threads share a key, each counting over its
    // slice of the list (every step reads one key by broadcast: a warp's
    // lanes hold consecutive keys and the same slice); no barrier per step,
    // where the bitonic network needs 36-45
    u32 dpad = 32;
    while (dpad < d) dpad <<= 1;
    const u32 T = kHpThreads / dpad, q = tid & (dpad - 1), sl = tid / dpad;
    if ((u32)tid < 512) rk[tid] = 0;
    __syncthreads();
    u64 mk = 0, mc = 0;
    if (q < d) {
      mk = lk[q];
      if (sl == 0) mc = lc[q];
      const u32 j0 = (u32)(((u64)d * sl) / T), j1 = (u32)(((u64)d * (sl + 1)) / T);
      u32 rank = 0;
#pragma unroll 8
      for (u32 j = j0; j < j1; ++j) rank += lk[j] < mk ? 1u : 0u;
      if (rank) atomicAdd(&rk[q], rank);
    }
    __syncthreads();
    if (q < d && sl == 0) { const u32 r = rk[q]; lk[r] = mk; lc[r] = mc; }
    __syncthreads();
  } else {
    // bitonic sort (padded to a power of two with ~0)
    u32 np2 = 1;
    while (np2 < d) np2 <<= 1;
    for (u32 j = d + tid; j < np2; j += kHpThreads) { lk[j] = kEmpty; lc[j] = 0; }
    __syncthreads();
    for (u32 k2 = 2; k2 <= np2; k2 <<= 1) {
      for (u32 j = k2 >> 1; j > 0; j >>= 1) {
        for (u32 q = tid; q < np2; q += kHpThreads) {
          const u32 l = q ^ j;
          if (l > q) {
            const u64 ki = lk[q], kl = lk[l];
            const bool up = (q & k2) == 0;
            if ((ki > kl) == up) {
              lk[q] = kl; lk[l] = ki;
              const u64 t = lc[q]; lc[q] = lc[l]; lc[l] = t;
            }
          }
        }
        __syncthreads();
      }
    }
  }
  // the sentinel key ~0 (the largest) goes last
  const u64 snt = bad ? 0ull : (u64)sent;
  const u32 dd = d + (snt ? 1u : 0u);
  if (tid == 0 && snt) { lk[d] = kEmpty; lc[d] = snt; }
  __syncthreads();
  u64 rows = 0;
  u64* sk = a.pk_stage + (size_t)p * kHpStage;
  u64* sc = a.pc_stage + (size_t)p * kHpStage;
  for (u32 j = tid; j < dd; j += kHpThreads) {
    sk[j] = lk[j];
    sc[j] = lc[j];
    rows += lc[j];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) rows += __shfl_xor_sync(0xffffffffu, rows, o);
  __syncthreads();
  if (lane == 0) wsum[wid] = rows;
  __syncthreads();
  if (tid == 0) {
    u64 r = 0;
    for (int w2 = 0; w2 < 32; ++w2) r += wsum[w2];
    a.pd[p] = dd;
    a.pr[p] = r;
    if (bad) atomicExch((unsigned*)&a.ctl->hp_overflow, 1u);
  }
}

// ---- hp_place: the partitions' staged pairs -> their global positions ----
// Block p sums (pairs, rows) of the partitions before it, copies its pairs to
// pk / pc and writes their emit offsets; the last block publishes the totals.
__global__ void __launch_bounds__(256) hp_place_kernel(HpArgs a) {
  pdl_begin();
  if (!gate_open(a.ctl, a.gate)) return;
  if (a.shard && a.ctl->merge_bad) return;
  __shared__ u64 wd[8], wr[8], wsc[8];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u32 p = blockIdx.x;
  u64 d0 = 0, r0 = 0;
  for (u32 q = tid; q < p; q += 256) { d0 += a.pd[q]; r0 += a.pr[q]; }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    d0 += __shfl_xor_sync(0xffffffffu, d0, o);
    r0 += __shfl_xor_sync(0xffffffffu, r0, o);
  }
  if (lane == 0) { wd[wid] = d0; wr[wid] = r0; }
  __syncthreads();
  u64 D = 0, R = 0;
#pragma unroll
  for (int w2 = 0; w2 < 8; ++w2) { D += wd[w2]; R += wr[w2]; }
  const u32 dd = (u32)a.pd[p];
  const u64* sk = a.pk_stage + (size_t)p * kHpStage;
  const u64* sc = a.pc_stage + (size_t)p * kHpStage;
  u64 run = R;
  for (u32 b0 = 0; b0 < dd; b0 += 256) {
    const u32 i = b0 + tid;
    const u64 cnt = i < dd ? sc[i] : 0;
    u64 inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u64 t = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += t;
    }
    if (lane == 31) wsc[wid] = inc;
    __syncthreads();
    u64 before = 0, all = 0;
#pragma unroll
    for (int w2 = 0; w2 < 8; ++w2) {
      before += w2 < wid ? wsc[w2] : 0;
      all += wsc[w2];
    }
    const u64 rs = run + before + inc - cnt;  // the pair's first row
    if (i < dd) {
      a.pk[D + i] = sk[i];
      a.pc[D + i] = cnt;
      a.poffs[D + i] = rs;
    }
    if (a.tile_pair) {
      // tile_pair[t] = the pair holding the first key of the emit's tile t
      // (the emit of rows [0, n) into x: same head / tile geometry as emit.cu)
      const u64 TK = a.kk ? 2048 : 1024, VK = a.kk ? 8 : 4, ksz = a.kk ? 4 : 8;
      const u64 mis = (((uintptr_t)a.x) & 31) / ksz;
      const u64 hd = mis ? ((VK - mis) < a.n ? (VK - mis) : a.n) : 0;
      const u64 nkeys = (a.n - hd) / VK * VK;
      const u64 ntiles = (nkeys + TK - 1) / TK;
      u64 t_lo = 0, t_hi = 0;
      if (i < dd && cnt) {
        const u64 re = rs + cnt;
        t_lo = rs <= hd ? 0 : (rs - hd + TK - 1) / TK;
        t_hi = re <= hd ? 0 : (re - hd + TK - 1) / TK;
        if (t_hi > ntiles) t_hi = ntiles;
      }
      const bool longrun = t_hi > t_lo + 32;
      if (!longrun)
        for (u64 t = t_lo; t < t_hi; ++t) a.tile_pair[t] = (u32)(D + i);
      for (u32 m = __ballot_sync(0xffffffffu, longrun); m; m &= m - 1) {
        const int r = __ffs(m) - 1;
        const u64 lo = __shfl_sync(0xffffffffu, t_lo, r), hi = __shfl_sync(0xffffffffu, t_hi, r);
        const u32 pr = (u32)(D + b0 + (u32)(wid * 32 + r));
        for (u64 t = lo + lane; t < hi; t += 32) a.tile_pair[t] = pr;
      }
    }
    run += all;
    __syncthreads();
  }
  if (p == gridDim.x - 1 && tid == 0) {
    const u64 tot_d = D + dd, tot_r = run;
    const bool bad = *((volatile u32*)&a.ctl->hp_overflow) != 0;
    const u64 expect = a.shard ? a.ctl->n_global : a.n;  // sharded merge: the column's N
    a.poffs[tot_d] = tot_r;
    a.ctl->npairs = tot_d;
    a.ctl->total = tot_r;
    a.ctl->sum_error = !bad && tot_r != expect;
    a.ctl->pairs_ready = !bad && tot_r == expect;
  }
}

// The recovery after a partition overflow: every CTA's rows are exactly its
// spill plus its cells (CTA 0's also hold the unaligned head and tail keys),
// so each CTA writes them back over its own range of the column, which the
// general fallback sort then sorts.
template <int KK>
__global__ void __launch_bounds__(1024) hp_restore_kernel(HpArgs a, u32 G) {
  using K = typename KeyT<KK>::T;
  constexpr int KPV = 16 / sizeof(K);
  __shared__ u64 woff[1025];
  const u32 c = blockIdx.x;
  const int tid = threadIdx.x;
  const u64 n = a.n;
  const u64 mis = (((uintptr_t)a.x) & 15) / sizeof(K);
  const u64 head0 = mis ? (u64)KPV - mis : 0;
  const u64 head = head0 < n ? head0 : n;
  const u64 body = (n - head) / KPV * KPV;
  const u64 tail0 = head + body;
  u64 v0, v1;
  hp_range(body / KPV, kHpRound, c, G, &v0, &v1);
  const u64 r0 = v0 * KPV, r1 = v1 * KPV;
  K* x = (K*)a.x;
  const u64 span = r1 - r0;
  auto pos = [&](u64 q) -> u64 {  // q-th row of this CTA -> its index in the column
    if (q < span) return head + r0 + q;
    q -= span;
    return q < head ? q : tail0 + (q - head);
  };
  const u32 ns = a.spofs[(size_t)c * (kHpP + 1) + kHpP];
  const u32 nc = a.cpofs[(size_t)c * (kHpP + 1) + kHpP];
  const K* src = (const K*)a.part + head + r0;
  for (u32 i = tid; i < ns; i += blockDim.x) x[pos(i)] = src[i];
  const u64* ck = a.cellk + (size_t)c * kHpCellCap;
  const u32* cw = a.cellw + (size_t)c * kHpCellCap;
  u64 base = ns;
  for (u32 c0 = 0; c0 < nc; c0 += 1024) {
    const u32 m = nc - c0 < 1024u ? nc - c0 : 1024u;
    if (tid == 0) {
      u64 run = base;
      for (u32 j = 0; j < m; ++j) { woff[j] = run; run += cw[c0 + j]; }
      woff[m] = run;
    }
    __syncthreads();
    for (u32 j = 0; j < m; ++j) {
      const K k = key_unmap<KK>(ck[c0 + j], a.flip);
      for (u64 q = woff[j] + tid; q < woff[j + 1]; q += blockDim.x) x[pos(q)] = k;
    }
    base = woff[m];
    __syncthreads();
  }
}

// The sharded merge's segment table: every rank's gathered list (sorted,
// order-mapped keys) cut at the partitions' key boundaries, which follow
// from the partition map of the (identical, all-reduced) samples: partition
// p starts at the first fine bin mapped to p or above.  CTA r: list r.
__global__ void __launch_bounds__(kHpThreads, 1) hp_shard_bounds_kernel(HpArgs a) {
  pdl_begin();
  if (!gate_open(a.ctl, kGateMain) || a.ctl->merge_bad) return;
  __shared__ unsigned short pmap[kHpFine];
  __shared__ u32 fh[kHpFine];
  __shared__ u64 rl[128];
  __shared__ u64 bound[kHpP + 1];
  __shared__ unsigned char has[kHpP + 1];  // a bin starts partition p (else: past every key)
  __shared__ u64 s_lo;
  __shared__ int s_sh;
  const int tid = threadIdx.x;
  const u32 r = blockIdx.x;
  if (r == 0 && tid == 0) a.ctl->hp_overflow = 0;  // the merge's own overflow flag
  hp_build_pmap(est_scratch(a.ctl)->samples, pmap, fh, rl, &s_lo, &s_sh);
  for (u32 p = tid; p <= kHpP; p += kHpThreads) has[p] = 0;
  __syncthreads();
  const u64 lo = s_lo;
  const int sh = s_sh;
  if (tid == 0) { bound[0] = 0; has[0] = 1; }
  for (u32 f = 1 + tid; f < (u32)kHpFine; f += kHpThreads) {
    const u32 p0 = pmap[f - 1], p1 = pmap[f];
    const u64 off = (u64)f << sh;
    if (off > ~0ull - lo) continue;  // the bin starts past the largest key: holds none
    for (u32 q = p0 + 1; q <= p1; ++q) { bound[q] = lo + off; has[q] = 1; }
  }
  __syncthreads();
  const u64* L = a.recv + (size_t)r * a.row;
  const u64 np = L[0];
  u32* out = a.cpofs + (size_t)r * (kHpP + 1);
  for (u32 p = tid; p <= kHpP; p += kHpThreads) {
    u64 pos = np;
    if (p < (u32)kHpP && has[p]) {  // the first index with key >= bound[p]
      u64 lo2 = 0, hi2 = np;
      const u64 kb = bound[p];
      while (lo2 < hi2) {
        const u64 mid = (lo2 + hi2) >> 1;
        if (L[1 + mid] < kb) lo2 = mid + 1; else hi2 = mid;
      }
      pos = lo2;
    }
    out[p] = (u32)pos;
  }
}

// ---- host side ----
static void hp_markers(u64* e0, u64* e1, u32* ma, u32* mb) {
  const u64 E0 = 0x5DEECE66D1234567ull;
  const u32 t0 = hp_t(E0), a0 = hp_b1(t0), b0 = hp_b2(t0);
  u64 E1 = E0;
  for (u64 t = 1;; ++t) {  // E1's two buckets clear of E0's
    E1 = E0 + t * 0x9E3779B97F4A7C15ull;
    const u32 t1 = hp_t(E1), a1 = hp_b1(t1), b1 = hp_b2(t1);
    if (a1 != a0 && a1 != b0 && b1 != a0 && b1 != b0) break;
  }
  *e0 = E0;
  *e1 = E1;
  *ma = a0;
  *mb = b0;
}

int hp_grid(u64 n, int kk, int num_sms) {
  const u64 chunks = (n / (kk ? 4 : 2) + kHpRound - 1) / kHpRound;
  const u64 g = num_sms < 160 ? (u64)num_sms : 160;  // hp_reduce's segment table holds 2 x 160
  return (int)(chunks < g ? (chunks ? chunks : 1) : g);
}

size_t hp_scratch_bytes(int num_sms) {
  return (size_t)num_sms * kHpCellCap * 12 + (size_t)num_sms * (kHpP + 1) * 8 + kHpP * 16 + 16;
}

// G: the count's grid (the scratch is laid out per CTA of it)
static HpArgs hp_args(const HpBufs& b, const void* x, u64 n, u64 flip, DevCtl* ctl, u64* pk,
                      u64* pc, u64* poffs, int gate, int G) {
  HpArgs a{};
  a.x = x;
  a.n = n;
  a.flip = flip;
  a.ctl = ctl;
  a.part = b.part;
  char* s = (char*)b.scratch;
  a.cellk = (u64*)s;
  s += (size_t)G * kHpCellCap * 8;
  a.cellw = (u32*)s;
  s += (size_t)G * kHpCellCap * 4;
  a.cpofs = (u32*)s;
  s += (size_t)G * (kHpP + 1) * 4;
  a.spofs = (u32*)s;
  s += (size_t)G * (kHpP + 1) * 4;
  a.pd = (u64*)(((uintptr_t)s + 7) & ~(uintptr_t)7);
  a.pr = a.pd + kHpP;
  a.pk_stage = b.pk_stage;
  a.pc_stage = b.pc_stage;
  a.pk = pk;
  a.pc = pc;
  a.poffs = poffs;
  hp_markers(&a.e0, &a.e1, &a.ma, &a.mb);
  a.gate = gate;
  return a;
}

template <typename F>
static cudaError_t hp_attr(F* f, size_t smem) {
  return cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int KK>
static cudaError_t hp_launch_t(const HpArgs& a, int G, cudaStream_t st) {
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = hp_attr(hp_count_kernel<KK>, kHpCountSmem);
    if (e == cudaSuccess) e = hp_attr(hp_reduce_kernel<KK, false>, kHpReduceSmem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  cudaError_t e = launch_pdl(kPdlCount, hp_count_kernel<KK>, G, kHpThreads, kHpCountSmem, st, a);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kPdlCount, hp_reduce_kernel<KK, false>, kHpP, kHpThreads, kHpReduceSmem, st, a,
                 (u32)G);
  if (e != cudaSuccess) return e;
  return launch_pdl(kPdlCount, hp_place_kernel, kHpP, 256, 0, st, a);
}

cudaError_t launch_hp_count(const HpBufs& b, const void* x, u64 n, u64 flip, DevCtl* ctl,
                            u64* pk, u64* pc, u64* poffs, int num_sms, cudaStream_t st, int gate,
                            int kk, u32* tile_pair) {
  const int G = hp_grid(n, kk, num_sms);
  HpArgs a = hp_args(b, x, n, flip, ctl, pk, pc, poffs, gate, G);
  a.tile_pair = tile_pair;
  a.kk = kk;
  if (kk == 1) return hp_launch_t<1>(a, G, st);
  if (kk == 2) return hp_launch_t<2>(a, G, st);
  return hp_launch_t<0>(a, G, st);
}

// The sharded merge: the gathered sorted lists -> the global sorted pairs and
// their offsets in pk / pc / poffs (every rank, the same result).
cudaError_t launch_hp_shard_merge(const HpBufs& b, const u64* recv, int world, u64 cap, u64 row,
                                  DevCtl* ctl, u64* pk, u64* pc, u64* poffs, cudaStream_t st) {
  HpArgs a = hp_args(b, nullptr, 0, 0, ctl, pk, pc, poffs, kGateMain, world);
  a.recv = recv;
  a.row = row;
  a.cap = cap;
  a.shard = 1;
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = hp_attr(hp_reduce_kernel<0, true>, kHpReduceSmem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  cudaError_t e = launch_pdl(kPdlCount, hp_shard_bounds_kernel, world, kHpThreads, 0, st, a);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kPdlCount, hp_reduce_kernel<0, true>, kHpP, kHpThreads, kHpReduceSmem, st, a,
                 (u32)world);
  if (e != cudaSuccess) return e;
  return launch_pdl(kPdlCount, hp_place_kernel, kHpP, 256, 0, st, a);
}

void launch_hp_restore(const HpBufs& b, void* x, u64 n, u64 flip, int num_sms, cudaStream_t st,
                       int kk) {
  const int G = hp_grid(n, kk, num_sms);
  const HpArgs a = hp_args(b, x, n, flip, nullptr, nullptr, nullptr, nullptr, kGateNone, G);
  if (kk == 1) hp_restore_kernel<1><<<G, 1024, 0, st>>>(a, (u32)G);
  else if (kk == 2) hp_restore_kernel<2><<<G, 1024, 0, st>>>(a, (u32)G);
  else hp_restore_kernel<0><<<G, 1024, 0, st>>>(a, (u32)G);
}

}  // namespace cafs
