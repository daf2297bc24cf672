// hashcount.cu -- K3: the main-route counting pass and its compaction.
//
// Replaces count_sequence (_kernels.py:25-81) / main_count_loop
// (sorter.py:183-196).  The reference folds runs and probes a 4-slot
// cache-line bucket per update, spilling overflow keys to a side buffer.  The
// B200 design keeps the same contract -- every element lands in exactly one
// (key, count) cell, cells are merged by key, the spill guard re-routes to the
// fallback -- with a layout for 148 SMs:
//
//   * persistent CTAs (one per SM, 1024 threads); warp 0's lane 0 is the TMA
//     producer that streams 16-32 KB chunks of the int64 column into a
//     shared-memory ring (cp.async.bulk + mbarrier complete_tx; 9 x 15.5 KB for
//     the dense-window shape, 143 KB in flight per SM); warps 1..31 consume;
//   * per element (bit-63 flip in registers):
//       - dense-range window (dictionary-encoded columns): one shared atomic
//         into counts[v - base]; the window is set by the estimate kernel from
//         the sample's span, exact for any key because out-of-window keys take
//         the hash path;
//       - otherwise a per-CTA shared open-addressing (u64 key, u32 count) table,
//         first probe inline, linear probing + CAS claims on the slow path,
//         claims capped at load 1/2;
//       - keys that find no shared slot go to the global L2-resident table
//         (global_insert in common.cuh): the analogue of the reference's spill;
//   * one flush per CTA of its shared cells into the global table;
//   * the guard: global table overflow (more than kGlobalCap distinct keys or
//     a probe chain over kGlobalMaxProbe) sets ctl->overflow and the pipeline
//     re-routes to the fallback radix sort (reference guard: sorter.py:264-273).
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kHcThreads = 1024;
constexpr u32 kRange = 8192;              // dense window (u32 counters, 32 KB)
constexpr int kSLog2 = 13;                // shared table: 8192 slots (64 KB keys + 32 KB counts)
constexpr int kSMaxProbe = 4;             // a longer chain spills: the table is only a cache
                                          // of partial counts, so a key found in two places
                                          // (or in a slot and the spill) still sums right
template <int STAGES, int STAGE_KEYS, int QCAP, bool RANGE, int SLOG2 = kSLog2>
constexpr size_t hc_smem() {
  return (RANGE ? (size_t)kRange * 4 : 0) + ((size_t)12 << SLOG2) +
         (size_t)STAGES * STAGE_KEYS * 8 + (size_t)32 * QCAP * 8 + (size_t)2 * STAGES * 8 + 16;
}

struct HcArgs {
  const void* x;  // keys of kind KK (common.cuh)
  u64 n;
  u64 flip;
  u64 mult;
  DevCtl* ctl;
  u64* gkeys;
  u64* gcnt;
  u32* glist;
  int use_range;
  int gate;
  u64* dense;   // global dense-window counts [kRange] (zero on entry)
};

// key -> global table, keeping the sentinel value out of it
__device__ __forceinline__ void table_add(const HcArgs& a, u64 key, u64 inc) {
  if (key == kEmpty) atomicAdd(&a.ctl->empty_key_count, inc);
  else global_insert(a.gkeys, a.gcnt, a.glist, a.ctl, key, inc, a.mult);
}

// Shared-table miss: linear probing with claims capped at load 1/2.  True when
// resolved.  SLOG2: the table's size.
template <int SLOG2 = kSLog2>
__device__ __noinline__ bool probe_smem(u64 v, u64* skeys, u32* scnt, u32* sclaims, u64 mult) {
  constexpr u32 S = 1u << SLOG2;
  u32 h = mhash(v, mult, 64 - SLOG2);
  for (int p = 0; p < kSMaxProbe; ++p) {
    const u64 k = *((volatile u64*)&skeys[h]);
    if (k == v) { atomicAdd(&scnt[h], 1u); return true; }
    if (k == kEmpty) {
      if (*((volatile u32*)sclaims) >= S / 2) return false;
      const u64 old = atomicCAS(&skeys[h], kEmpty, v);
      if (old == kEmpty) {
        atomicAdd(sclaims, 1u);
        atomicAdd(&scnt[h], 1u);
        return true;
      }
      if (old == v) { atomicAdd(&scnt[h], 1u); return true; }
    }
    h = (h + 1) & (S - 1);
  }
  return false;
}

// Inline slow path (rare misses): shared probe, else the global table.
template <int SLOG2 = kSLog2>
__device__ __forceinline__ u32 count_slow(u64 v, u64* skeys, u32* scnt, u32* sclaims,
                                          const HcArgs& a) {
  if (probe_smem<SLOG2>(v, skeys, scnt, sclaims, a.mult)) return 0;
  global_insert(a.gkeys, a.gcnt, a.glist, a.ctl, v, 1, a.mult);
  return 1;
}

// Warp-convergent slow path of the queued shapes: the warp's queued misses are
// probed in the CTA's table 32 at a time, and those it cannot take go straight
// to the L2-resident global table -- the reference's spill (buckets.py:273-282)
// without the spill buffer: a fold pass over spilled keys cost more (cfg3:
// +100 us) than the inline L2 round trips it saves in the count (+45 us).
// Returns 1 on the lanes whose key went to the global table.
template <int SLOG2 = kSLog2>
__device__ __forceinline__ u32 resolve_miss(bool active, u64 v, u64* skeys, u32* scnt, u32* sclaims,
                                            const HcArgs& a) {
  const bool miss = active && !probe_smem<SLOG2>(v, skeys, scnt, sclaims, a.mult);
  if (miss) global_insert(a.gkeys, a.gcnt, a.glist, a.ctl, v, 1, a.mult);
  return miss ? 1u : 0u;
}

// STAGES x STAGE_KEYS TMA ring fed by a dedicated producer warp (warp 0);
// warps 1..31 consume.  STAGE_KEYS / 2 is a multiple of the 992 consumers so
// every consumer takes the same number of 16-byte vectors per stage.
// QCAP > 0: first-probe misses are queued per warp and resolved 32 at a time
// with the whole warp active (the slow path is otherwise run by a few lanes
// of a diverged warp, leaving its L2 round trips unoverlapped).
// RANGE = false: no dense window (launched only when the window is closed).
// STAGE_KEYS counts 8-byte words; a stage holds STAGE_KEYS * 8 / sizeof(K) keys.
// SLOG2: log2 of the shared table's slots (the dense-window shape gives some
// of them to a deeper ring: its keys rarely reach the table).
template <int STAGES, int STAGE_KEYS, int QCAP, bool RANGE, int KK, int SLOG2 = kSLog2>
__global__ void __launch_bounds__(kHcThreads, 1) hash_count_kernel(HcArgs a) {
  constexpr u32 kS = 1u << SLOG2;
  using K = typename KeyT<KK>::T;
  constexpr int KPV = 16 / sizeof(K);                         // keys per 16-byte vector
  constexpr u64 SK = (u64)STAGE_KEYS * 8 / sizeof(K);         // keys per stage
  constexpr int kConsumers = kHcThreads - 32;
  static_assert((STAGE_KEYS / 2) % kConsumers == 0, "balanced stages");
  constexpr u32 kVpt = STAGE_KEYS / 2 / kConsumers;
  extern __shared__ __align__(128) unsigned char smem[];
  u64* stage = (u64*)smem;                                        // [STAGES][STAGE_KEYS]
  u64* skeys = stage + (size_t)STAGES * STAGE_KEYS;               // [kS]
  u32* scnt = (u32*)(skeys + kS);                                 // [kS]
  u32* dcnt = scnt + kS;                                          // [kRange] if RANGE
  u64* queue = (u64*)(dcnt + (RANGE ? kRange : 0));               // [32][QCAP]
  u64* full = queue + 32 * QCAP;                                  // [STAGES]
  u64* empty = full + STAGES;                                     // [STAGES]
  __shared__ u32 sclaims;
  __shared__ u64 red_empty[32], red_glob[32];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u64 flip = a.flip, mult = a.mult;

  // ---- before the programmatic dependency resolves (the estimate kernel may
  // still be running): nothing here reads what it writes -- the tables are
  // cleared and the ring's first stages are already on their way from HBM ----
  for (u32 i = tid; i < kS; i += kHcThreads) { skeys[i] = kEmpty; scnt[i] = 0; }
  if (RANGE)
    for (u32 i = tid; i < kRange; i += kHcThreads) dcnt[i] = 0;
  if (tid == 0) {
    sclaims = 0;
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // body = 16-byte aligned stretch of whole vectors; head/tail keys scalar
  const u64 n = a.n;
  const K* xk = (const K*)a.x;
  const u64 mis = (((uintptr_t)a.x) & 15) / sizeof(K);
  const u64 head0 = mis ? (u64)KPV - mis : 0;
  const u64 head = head0 < n ? head0 : n;
  const u64 body = (n - head) / KPV * KPV;
  const K* xb = xk + head;
  const u64 nchunks = (body + SK - 1) / SK;
  const u64 my_chunks =
      nchunks > blockIdx.x ? (nchunks - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
  const u64 pre_chunks = my_chunks < (u64)STAGES ? my_chunks : (u64)STAGES;
  if (tid == 0) {
    for (u64 it = 0; it < pre_chunks; ++it) {
      const u64 off = (blockIdx.x + it * gridDim.x) * SK;
      const u32 bytes = (u32)(((body - off) < SK ? (body - off) : SK) * sizeof(K));
      mbar_arrive_expect_tx(&full[it], bytes);
      tma_load_1d(stage + (size_t)it * STAGE_KEYS, xb + off, bytes, &full[it]);
    }
  }
  pdl_begin();
  if (!gate_open(a.ctl, a.gate)) {
    // not this column's shape: let the stages in flight land before the CTA
    // (and its shared memory) goes
    if (tid == 0)
      for (u64 it = 0; it < pre_chunks; ++it) mbar_wait(&full[it], 0);
    return;
  }
  const u64 base = (RANGE && a.use_range) ? a.ctl->range_base : 0ull;
  const u64 rlen = (RANGE && a.use_range) ? a.ctl->range_len : 0u;

  u64 empty_cnt = 0;
  u32 glob_cnt = 0;

  // direct window or first shared probe; false = unresolved (slow path)
  auto fast = [&](u64 v) -> bool {
    const u64 d = v - base;
    if (RANGE && d < rlen) { atomicAdd(&dcnt[d], 1u); return true; }
    if (v == kEmpty) { empty_cnt++; return true; }
    const u32 h = mhash(v, mult, 64 - SLOG2);
    if (skeys[h] == v) { atomicAdd(&scnt[h], 1u); return true; }
    return false;
  };
  auto count1 = [&](u64 v) {
    if (!fast(v)) glob_cnt += count_slow<SLOG2>(v, skeys, scnt, &sclaims, a);
  };

  if (wid == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      u32 s = 0, ph = 1;  // the first STAGES chunks were issued above: one lap done
      for (u64 it = pre_chunks; it < my_chunks; ++it) {
        if (it >= (u64)STAGES) mbar_wait(&empty[s], ph ^ 1);
        const u64 off = (blockIdx.x + it * gridDim.x) * SK;
        const u32 bytes = (u32)(((body - off) < SK ? (body - off) : SK) * sizeof(K));
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_1d(stage + (size_t)s * STAGE_KEYS, xb + off, bytes, &full[s]);
        if (++s == STAGES) { s = 0; ph ^= 1; }
      }
    }
  } else {
    const int ctid = tid - 32;
    u64* wq = queue + (size_t)wid * QCAP;
    u32 qn = 0;  // warp-uniform queue length
    auto enqueue = [&](bool miss, u64 v) {
      const u32 m = __ballot_sync(0xffffffffu, miss);
      if (m == 0) return;
      if (miss) wq[qn + __popc(m & lanemask_lt())] = v;
      qn += __popc(m);
      if (qn >= 32) {
        __syncwarp();
        const u64 u = wq[qn - 32 + lane];
        __syncwarp();
        qn -= 32;
        glob_cnt += resolve_miss<SLOG2>(true, u, skeys, scnt, &sclaims, a);
      }
    };
    // 32-bit keys: is the dense window inside the 32-bit domain?  Then a key
    // is in it iff (u32)(x - base) < kRange (no wrap-around false positives)
    bool w32 = false;
    u32 base32 = 0;
    if constexpr (KK != 0 && RANGE) {
      const long long B = (long long)(base ^ kSign);  // the window's first key, as int64
      const long long lo = KK == 1 ? -2147483648ll : 0ll;
      const long long hi = (KK == 1 ? 2147483647ll : 4294967295ll) - (long long)kRange;
      w32 = rlen == kRange && B >= lo && B <= hi;
      base32 = (u32)B;
    }
    u32 s = 0, ph = 0;
    u64 off = (u64)blockIdx.x * SK;
    const u64 off_step = (u64)gridDim.x * SK;
    for (u64 it = 0; it < my_chunks; ++it, off += off_step) {
      mbar_wait(&full[s], ph);
      const u32 nv = (u32)(((body - off) < SK ? (body - off) : SK) / KPV);
      const ulonglong2* sv = (const ulonglong2*)(stage + (size_t)s * STAGE_KEYS);
#pragma unroll
      for (u32 q = 0; q < kVpt; ++q) {
        const u32 i = ctid + q * kConsumers;
        const bool valid = i < nv;
        ulonglong2 w = make_ulonglong2(0, 0);
        if (valid) w = sv[i];
        if constexpr (KK != 0 && RANGE && QCAP == 0) {
          // 32-bit keys inside a window that lies in the 32-bit domain: the
          // window test in 32-bit arithmetic (exact there), no widening
          if (w32) {
            const u32 d0 = (u32)w.x - base32, d1 = (u32)(w.x >> 32) - base32;
            const u32 d2 = (u32)w.y - base32, d3 = (u32)(w.y >> 32) - base32;
            if (valid && max(max(d0, d1), max(d2, d3)) < kRange) {
              atomicAdd(&dcnt[d0], 1u);
              atomicAdd(&dcnt[d1], 1u);
              atomicAdd(&dcnt[d2], 1u);
              atomicAdd(&dcnt[d3], 1u);
              continue;
            }
          }
        }
        u64 v[KPV];
        if constexpr (KPV == 2) {
          v[0] = key_map<KK>((K)w.x, flip);
          v[1] = key_map<KK>((K)w.y, flip);
        } else {
          v[0] = key_map<KK>((K)w.x, flip);
          v[1] = key_map<KK>((K)(w.x >> 32), flip);
          v[2] = key_map<KK>((K)w.y, flip);
          v[3] = key_map<KK>((K)(w.y >> 32), flip);
        }
        bool all_in = RANGE;
        if constexpr (RANGE) {
#pragma unroll
          for (int k = 0; k < KPV; ++k) all_in = all_in && (v[k] - base) < rlen;
        }
        if (QCAP == 0) {
          if (valid) {
            if (all_in) {
#pragma unroll
              for (int k = 0; k < KPV; ++k) atomicAdd(&dcnt[v[k] - base], 1u);
            } else {
#pragma unroll
              for (int k = 0; k < KPV; ++k) count1(v[k]);
            }
          }
        } else {
          bool m[KPV];
#pragma unroll
          for (int k = 0; k < KPV; ++k) m[k] = false;
          if (valid) {
            if (all_in) {
#pragma unroll
              for (int k = 0; k < KPV; ++k) atomicAdd(&dcnt[v[k] - base], 1u);
            } else {
#pragma unroll
              for (int k = 0; k < KPV; ++k) m[k] = !fast(v[k]);
            }
          }
#pragma unroll
          for (int k = 0; k < KPV; ++k) enqueue(m[k], v[k]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == STAGES) { s = 0; ph ^= 1; }
    }
    if (QCAP > 0) {
      __syncwarp();
      glob_cnt += resolve_miss<SLOG2>((u32)lane < qn, (u32)lane < qn ? wq[lane] : 0ull, skeys, scnt,
                                      &sclaims, a);
    }
    if (blockIdx.x == 0 && ctid < 32) {  // head and tail keys (< KPV each)
      const u64 tail0 = head + body;
      if ((u64)ctid < head) count1(key_map<KK>(xk[ctid], flip));
      if ((u64)ctid < n - tail0) count1(key_map<KK>(xk[tail0 + ctid], flip));
    }
  }
  __syncthreads();

  // ---- flush the CTA's shared cells into the global table ----
  for (u32 d = tid; RANGE && d < (u32)rlen; d += kHcThreads) {
    const u32 c = dcnt[d];
    if (c) atomicAdd(&a.dense[d], (u64)c);  // key base + d: no hashing, no claims
  }
  constexpr int kFlushBatch = 2;  // first probes in flight per thread (register budget)
#pragma unroll 1
  for (u32 h0 = tid; h0 < kS; h0 += kFlushBatch * kHcThreads) {
    constexpr int R = kFlushBatch;
    u64 key[R], inc[R];
    bool ok[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const u32 h = h0 + r * kHcThreads;
      inc[r] = scnt[h];
      key[r] = skeys[h];
      if (inc[r] && key[r] == kEmpty) {  // cannot happen: the sentinel is counted aside
        atomicAdd(&a.ctl->empty_key_count, inc[r]);
        inc[r] = 0;
      }
      ok[r] = inc[r] != 0;
    }
    global_insert_batch<R>(a.gkeys, a.gcnt, a.glist, a.ctl, key, inc, ok);
  }
  u64 g = glob_cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    empty_cnt += __shfl_xor_sync(0xffffffffu, empty_cnt, o);
    g += __shfl_xor_sync(0xffffffffu, g, o);
  }
  if (lane == 0) { red_empty[wid] = empty_cnt; red_glob[wid] = g; }
  __syncthreads();
  if (tid == 0) {
    u64 e = 0, gg = 0;
    for (int w = 0; w < kHcThreads / 32; ++w) { e += red_empty[w]; gg += red_glob[w]; }
    if (e) atomicAdd(&a.ctl->empty_key_count, e);
    if (gg) atomicAdd(&a.ctl->g_updates, gg);
  }
}

// The high-cardinality shape (no dense window): the whole shared memory holds
// the table -- 16384 slots, twice the TMA shapes' -- and the column is read
// with direct 16-byte streaming loads (this shape is bound by the table work,
// ~1.5 TB/s, not by HBM, so the TMA ring buys nothing while taking 93 KB).
// With twice the slots, a skewed column misses the CTA's table on ~13 % of its
// keys instead of ~21 % (cfg3), and every miss costs a probe and an L2
// round trip into the global table.
constexpr int kBigSLog2 = 14;
constexpr u32 kBigS = 1u << kBigSLog2;
constexpr int kBigQcap = 64;
constexpr size_t kBigSmem = (size_t)kBigS * 12 + (size_t)32 * kBigQcap * 8;
constexpr int kBigThreads = kHcThreads;  // 32 warps: the shape is latency-bound per warp
                                         // (512 threads with 8 loads each: 1.4x slower)
constexpr int kBigUnroll = 4;  // 16-byte loads in flight per thread
constexpr int kBigBatchVecs = 1;  // vectors whose first probes are issued together (2 or 4:
                                  // register spills at the 64-register cap, 5-30 % slower)
constexpr u64 kBigMinRows = 1ull << 22;  // below: the 8192-slot queued shape

template <int KK>
__global__ void __launch_bounds__(kBigThreads, 1) hash_count_big_kernel(HcArgs a) {
  pdl_begin();
  if (!gate_open(a.ctl, a.gate)) return;
  using K = typename KeyT<KK>::T;
  constexpr int KPV = 16 / sizeof(K);
  extern __shared__ __align__(128) unsigned char smem[];
  u64* skeys = (u64*)smem;                      // [kBigS]
  u32* scnt = (u32*)(skeys + kBigS);            // [kBigS]
  u64* queue = (u64*)(scnt + kBigS);            // [32][kBigQcap]
  __shared__ u32 sclaims;
  __shared__ u64 red_empty[32], red_glob[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u64 flip = a.flip, mult = a.mult;
  for (u32 i = tid; i < kBigS; i += kBigThreads) { skeys[i] = kEmpty; scnt[i] = 0; }
  if (tid == 0) sclaims = 0;
  __syncthreads();

  const u64 n = a.n;
  const K* xk = (const K*)a.x;
  const u64 mis = (((uintptr_t)a.x) & 15) / sizeof(K);
  const u64 head0 = mis ? (u64)KPV - mis : 0;
  const u64 head = head0 < n ? head0 : n;
  const u64 nvec = (n - head) / KPV;
  const ulonglong2* xv = (const ulonglong2*)(xk + head);
  // this CTA's contiguous range of vectors
  const u64 per = (nvec + gridDim.x - 1) / gridDim.x;
  const u64 v0 = blockIdx.x * per;
  const u64 v1 = v0 + per < nvec ? v0 + per : nvec;

  u64 empty_cnt = 0;
  u32 glob_cnt = 0;
  u64* wq = queue + (size_t)wid * kBigQcap;
  u32 qn = 0;  // warp-uniform
  auto enqueue = [&](bool miss, u64 v) {
    const u32 m = __ballot_sync(0xffffffffu, miss);
    if (m == 0) return;
    if (miss) wq[qn + __popc(m & lanemask_lt())] = v;
    qn += __popc(m);
    if (qn >= 32) {
      __syncwarp();
      const u64 u = wq[qn - 32 + lane];
      __syncwarp();
      qn -= 32;
      glob_cnt += resolve_miss<kBigSLog2>(true, u, skeys, scnt, &sclaims, a);
    }
  };
  auto fast = [&](u64 v) -> bool {
    if (v == kEmpty) { empty_cnt++; return true; }
    const u32 h = mhash(v, mult, 64 - kBigSLog2);
    if (skeys[h] == v) { atomicAdd(&scnt[h], 1u); return true; }
    return false;
  };
  for (u64 r0 = v0; r0 < v1; r0 += (u64)kBigUnroll * kBigThreads) {  // CTA-uniform rounds
    ulonglong2 w[kBigUnroll];
    bool ok[kBigUnroll];
#pragma unroll
    for (int q = 0; q < kBigUnroll; ++q) {
      const u64 i = r0 + (u64)q * kBigThreads + tid;
      ok[q] = i < v1;
      w[q] = ok[q] ? ld_stream_v2(xv + i) : make_ulonglong2(0, 0);
    }
    // branch-free first probes, BATCH keys at a time: hashes, then the shared
    // loads, then predicated increments; the miss queue (a ballot per key)
    // only when some lane of the warp missed (the per-key branchy form: +2 %)
    constexpr int BV = kBigBatchVecs;          // vectors per batch
    constexpr int BATCH = BV * KPV;            // keys per batch
#pragma unroll
    for (int q0 = 0; q0 < kBigUnroll; q0 += BV) {
      u64 v[BATCH];
      bool act[BATCH];
#pragma unroll
      for (int b = 0; b < BV; ++b) {
        const ulonglong2 ww = w[q0 + b];
        if constexpr (KPV == 2) {
          v[b * 2] = key_map<KK>((K)ww.x, flip);
          v[b * 2 + 1] = key_map<KK>((K)ww.y, flip);
        } else {
          v[b * 4] = key_map<KK>((K)ww.x, flip);
          v[b * 4 + 1] = key_map<KK>((K)(ww.x >> 32), flip);
          v[b * 4 + 2] = key_map<KK>((K)ww.y, flip);
          v[b * 4 + 3] = key_map<KK>((K)(ww.y >> 32), flip);
        }
#pragma unroll
        for (int k = 0; k < KPV; ++k) act[b * KPV + k] = ok[q0 + b];
      }
      u32 h[BATCH];
      u64 sk[BATCH];
#pragma unroll
      for (int j = 0; j < BATCH; ++j) h[j] = mhash(v[j], mult, 64 - kBigSLog2);
#pragma unroll
      for (int j = 0; j < BATCH; ++j) sk[j] = skeys[h[j]];
      u32 mm = 0;
#pragma unroll
      for (int j = 0; j < BATCH; ++j) {
        const bool sentinel = v[j] == kEmpty;  // counted aside (never a table key)
        const bool hit = act[j] && !sentinel && sk[j] == v[j];
        if (hit) atomicAdd(&scnt[h[j]], 1u);
        empty_cnt += (act[j] && sentinel) ? 1u : 0u;
        mm |= (act[j] && !sentinel && !hit) ? (1u << j) : 0u;
      }
      if (__any_sync(0xffffffffu, mm != 0)) {
#pragma unroll
        for (int j = 0; j < BATCH; ++j) enqueue((mm >> j) & 1u, v[j]);
      }
    }
  }
  __syncwarp();
  glob_cnt += resolve_miss<kBigSLog2>((u32)lane < qn, (u32)lane < qn ? wq[lane] : 0ull, skeys,
                                      scnt, &sclaims, a);
  if (blockIdx.x == 0 && tid < 32) {  // head and tail keys (< KPV each)
    const u64 tail0 = head + nvec * KPV;
    if ((u64)tid < head) {
      const u64 v = key_map<KK>(xk[tid], flip);
      if (!fast(v)) glob_cnt += count_slow<kBigSLog2>(v, skeys, scnt, &sclaims, a);
    }
    if ((u64)tid < n - tail0) {
      const u64 v = key_map<KK>(xk[tail0 + tid], flip);
      if (!fast(v)) glob_cnt += count_slow<kBigSLog2>(v, skeys, scnt, &sclaims, a);
    }
  }
  __syncthreads();
  // ---- flush the CTA's shared cells into the global table ----
#pragma unroll 1
  for (u32 h0 = tid; h0 < kBigS; h0 += 2 * kBigThreads) {
    u64 key[2], inc[2];
    bool okf[2];
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const u32 h = h0 + r * kBigThreads;
      inc[r] = scnt[h];
      key[r] = skeys[h];
      okf[r] = inc[r] != 0;
    }
    global_insert_batch<2>(a.gkeys, a.gcnt, a.glist, a.ctl, key, inc, okf);
  }
  u64 g = glob_cnt;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    empty_cnt += __shfl_xor_sync(0xffffffffu, empty_cnt, o);
    g += __shfl_xor_sync(0xffffffffu, g, o);
  }
  if (lane == 0) { red_empty[wid] = empty_cnt; red_glob[wid] = g; }
  __syncthreads();
  if (tid == 0) {
    u64 e = 0, gg = 0;
    for (int w2 = 0; w2 < kBigThreads / 32; ++w2) { e += red_empty[w2]; gg += red_glob[w2]; }
    if (e) atomicAdd(&a.ctl->empty_key_count, e);
    if (gg) atomicAdd(&a.ctl->g_updates, gg);
  }
}

template <int KK>
static cudaError_t launch_hc_big(const HcArgs& a, u64 n, int num_sms, cudaStream_t st) {
  static_assert(kBigSmem <= 232448 - 2048, "shared memory budget");
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(hash_count_big_kernel<KK>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)kBigSmem);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const u64 kpv = KK ? 4 : 2;
  const u64 rounds = (n / kpv + (u64)kBigUnroll * kBigThreads - 1) / ((u64)kBigUnroll * kBigThreads);
  const int grid = (int)(rounds < (u64)num_sms ? (rounds ? rounds : 1) : (u64)num_sms);
  return launch_pdl(kPdlCount, hash_count_big_kernel<KK>, grid, kBigThreads, kBigSmem, st, a);
  return cudaGetLastError();
}

// Occupied global slots -> dense (key, count) pairs; re-zero the slots so the
// table is clean for the next call.  Block s compacts claim-list stripe s to
// the offset of the stripes before it.  The sentinel key's count becomes the
// last pair.
__global__ void __launch_bounds__(256) compact_kernel(DevCtl* ctl, u64* gkeys, u64* gcnt,
                                                      const u32* glist, u64* pkeys, u64* pcnt,
                                                      int gate) {
  pdl_begin();
  if (ctl->overflow || !gate_open(ctl, gate)) return;
  __shared__ u64 pre_sh, tot_sh;
  const u32 s = blockIdx.x;
  if (threadIdx.x < 32) {
    u64 pre = 0, tot = 0;
    for (u32 t = threadIdx.x; t < kListStripes; t += 32) {
      const u64 f = ctl->g_fill[t] < kStripeCap ? ctl->g_fill[t] : kStripeCap;
      tot += f;
      if (t < s) pre += f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      pre += __shfl_xor_sync(0xffffffffu, pre, o);
      tot += __shfl_xor_sync(0xffffffffu, tot, o);
    }
    if (threadIdx.x == 0) { pre_sh = pre; tot_sh = tot; }
  }
  __syncthreads();
  if (tot_sh > kGlobalCap) {  // stripes have headroom; the table's capacity is the guard
    if (s == 0 && threadIdx.x == 0) ctl->overflow = 1;
    return;
  }
  const u64 pre = pre_sh;
  const u32 m = ctl->g_fill[s] < kStripeCap ? ctl->g_fill[s] : (u32)kStripeCap;
  const u32* lst = glist + (u64)s * kStripeCap;
  for (u32 i = threadIdx.x; i < m; i += blockDim.x) {
    const u32 h = lst[i];
    pkeys[pre + i] = gkeys[h];
    pcnt[pre + i] = gcnt[h];
    gkeys[h] = kEmpty;
    gcnt[h] = 0;
  }
  if (s == 0 && threadIdx.x == 0) {
    const u64 tot = tot_sh;
    const u64 e = ctl->empty_key_count;
    if (e) { pkeys[tot] = kEmpty; pcnt[tot] = e; }
    ctl->npairs = tot + (e ? 1 : 0);
  }
}

// Dense-window counts -> (key, count) pairs in key order (the window is a key
// range), re-zeroing the array.  When nothing else was counted (no hash-table
// pairs), these ARE the sorted pairs: offsets are written and the pair sort is
// skipped; otherwise they are appended to the compacted pairs for the sort.
__global__ void __launch_bounds__(1024) dense_pairs_kernel(DevCtl* ctl, u64* dense, u64* pkeys,
                                                           u64* pcnt, u64* skeys, u64* scnt,
                                                           u64* soffs, u64 n_expect, int gate) {
  pdl_begin();
  __shared__ u32 wsum[32];
  __shared__ unsigned long long csum[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  // one round trip: the control words and the whole window are loaded together
  // (the window is kRange words whatever its open length, zero outside it),
  // the gate is checked afterwards
  constexpr int IT = kRange / 1024;
  u64 c[IT];
  {
    const ulonglong2* dv = (const ulonglong2*)(dense + tid * IT);
#pragma unroll
    for (int q = 0; q < IT / 2; ++q) {
      const ulonglong2 w = __ldcg(dv + q);
      c[2 * q] = w.x;
      c[2 * q + 1] = w.y;
    }
  }
  const u64 base = ctl->range_base;
  const u32 rlen = ctl->range_len;
  const int ovf = ctl->overflow;
  const u64 m = ctl->npairs;  // pairs compacted from the hash table
  // ~0: the counts were all-reduced over the ranks of a sharded sort and must
  // sum to the whole column
  const u64 ng = ctl->n_global;
  if (n_expect == ~0ull) n_expect = ng;
  if (!gate_open(ctl, gate)) return;  // the count kernel was gated off too: dense untouched
  if (ovf) {  // guard: the fallback sorts; leave the window zeroed for the next call
    for (u32 d = threadIdx.x; d < rlen; d += blockDim.x) dense[d] = 0;
    return;
  }
  u32 nz = 0;
  u64 local = 0;
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const u32 d = tid * IT + q;
    if (d >= rlen) c[q] = 0;
    nz += c[q] != 0;
    local += c[q];
  }
  // exclusive scans of the non-zero flags (output slot) and counts (offsets)
  u32 inz = nz;
  u64 icnt = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const u32 t = __shfl_up_sync(0xffffffffu, inz, o);
    const u64 t2 = __shfl_up_sync(0xffffffffu, icnt, o);
    if (lane >= o) { inz += t; icnt += t2; }
  }
  if (lane == 31) { wsum[wid] = inz; csum[wid] = icnt; }
  __syncthreads();
  if (wid == 0) {
    u32 w = wsum[lane];
    u64 w2 = csum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const u32 t = __shfl_up_sync(0xffffffffu, w, o);
      const u64 t2 = __shfl_up_sync(0xffffffffu, w2, o);
      if (lane >= o) { w += t; w2 += t2; }
    }
    wsum[lane] = w;
    csum[lane] = w2;
  }
  __syncthreads();
  const u32 ndense = wsum[31];
  const u64 dtotal = csum[31];
  const bool direct = (m == 0);
  u32 slot = inz - nz + (wid ? wsum[wid - 1] : 0);
  u64 off = icnt - local + (wid ? csum[wid - 1] : 0);
#pragma unroll
  for (int q = 0; q < IT; ++q) {
    const u32 d = tid * IT + q;
    if (c[q]) {
      if (direct) {
        skeys[slot] = base + d;
        scnt[slot] = c[q];
        soffs[slot] = off;
      } else {
        pkeys[m + slot] = base + d;
        pcnt[m + slot] = c[q];
      }
      dense[d] = 0;
      ++slot;
      off += c[q];
    }
  }
  __syncthreads();
  if (tid == 0) {
    ctl->npairs = m + ndense;
    if (direct) {
      soffs[ndense] = dtotal;
      ctl->total = dtotal;
      ctl->sum_error = (dtotal != n_expect);
      ctl->pairs_ready = (dtotal == n_expect);
    }
    // keys outside the window: compacted pairs, or (when the pipeline held no
    // compaction) window counts short of the rows
    ctl->dense_outside = (m != 0) || dtotal != n_expect;
  }
}

void launch_dense_pairs(DevCtl* ctl, u64* dense, u64* pkeys, u64* pcnt, u64* skeys, u64* scnt,
                        u64* soffs, u64 n_expect, cudaStream_t st, int gate) {
  launch_pdl(kPdlDense, dense_pairs_kernel, 1, 1024, 0, st, ctl, dense, pkeys, pcnt, skeys, scnt, soffs,
             n_expect, gate);
}

size_t dense_window_len() { return kRange; }

// (key, count) pairs -> global table (the merge step of the sharded sort)
__global__ void insert_pairs_kernel(const u64* __restrict__ keys, const u64* __restrict__ cnts,
                                    u64 m, u64 mult, DevCtl* ctl, u64* gkeys, u64* gcnt,
                                    u32* glist) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += stride) {
    const u64 k = keys[i], c = cnts[i];
    if (c == 0) continue;
    if (k == kEmpty) atomicAdd(&ctl->empty_key_count, c);
    else global_insert(gkeys, gcnt, glist, ctl, k, c, mult);
  }
}

// zero the per-call fields of the control block (estimate_kernel does the same)
__global__ void reset_ctl_kernel(DevCtl* ctl) {
  for (u32 t = threadIdx.x; t < kListStripes; t += blockDim.x) ctl->g_fill[t] = 0;
  if (threadIdx.x == 0) {
    ctl->g_updates = 0;
    ctl->empty_key_count = 0;
    ctl->overflow = 0;
    ctl->need_large = 0;
    ctl->npairs = 0;
    ctl->total = 0;
    ctl->pairs_ready = 0;
    ctl->sum_error = 0;
    ctl->range_len = 0;
  }
}

void launch_insert_pairs(const u64* keys, const u64* cnts, u64 m, u64 mult, DevCtl* ctl,
                         u64* gkeys, u64* gcnt, u32* glist, int num_sms, cudaStream_t st) {
  reset_ctl_kernel<<<1, 32, 0, st>>>(ctl);
  u64 blocks = (m + 255) / 256;
  if (blocks > (u64)num_sms * 8) blocks = (u64)num_sms * 8;
  if (blocks < 1) blocks = 1;
  insert_pairs_kernel<<<(unsigned)blocks, 256, 0, st>>>(keys, cnts, m, mult, ctl, gkeys, gcnt,
                                                         glist);
}

template <int ST, int SK, int QC, bool RG, int KK = 0, int SL = kSLog2>
static cudaError_t launch_hc(const HcArgs& a, u64 n, int num_sms, cudaStream_t st) {
  constexpr size_t sm = hc_smem<ST, SK, QC, RG, SL>();
  static_assert(sm <= 232448 - 2048, "shared memory budget");
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(hash_count_kernel<ST, SK, QC, RG, KK, SL>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    attr_dev = dev;
  }
  const u64 keys_per_stage = (u64)SK * 8 / (KK ? 4 : 8);
  const u64 chunks = (n + keys_per_stage - 1) / keys_per_stage;
  const int grid = (int)(chunks < (u64)num_sms ? (chunks ? chunks : 1) : (u64)num_sms);
  return launch_pdl(kPdlCount, hash_count_kernel<ST, SK, QC, RG, KK, SL>, grid, kHcThreads, sm, st, a);
  return cudaGetLastError();
}

// shapes: 0 = dense window (deep TMA ring, inline slow path, the window's
// counters in shared memory); without the window (the gate guarantees it is
// closed -- kGateMainHash / kGateHash -- or use_range is 0) the big-table
// shape with per-warp miss queues (the TMA queued shape for
// columns under kBigMinRows rows)
cudaError_t launch_hash_count(const void* x, u64 n, u64 flip, u64 mult, DevCtl* ctl, u64* gkeys,
                              u64* gcnt, u32* glist, int use_range, int num_sms,
                              cudaStream_t st, int variant, int gate, u64* dense,
                              int kk) {
  HcArgs a{x, n, flip, mult, ctl, gkeys, gcnt, glist, use_range, gate, dense};
  const bool window = use_range && gate != kGateMainHash && gate != kGateHash;
  (void)variant;
  if (window) {
    // 9 x 15.5 KB ring, 4096-slot table: 143 KB in flight per SM (3 x 31 KB
    // with 8192 slots left the cfg4 count at 6.85 TB/s; this shape 7.19)
    if (kk == 1) return launch_hc<9, 1984, 0, true, 1, 12>(a, n, num_sms, st);
    if (kk == 2) return launch_hc<9, 1984, 0, true, 2, 12>(a, n, num_sms, st);
    return launch_hc<9, 1984, 0, true, 0, 12>(a, n, num_sms, st);
  }
  if (n < kBigMinRows) {  // small columns: the table's init and flush would dominate
    if (kk == 1) return launch_hc<3, 3968, 64, false, 1>(a, n, num_sms, st);
    if (kk == 2) return launch_hc<3, 3968, 64, false, 2>(a, n, num_sms, st);
    return launch_hc<3, 3968, 64, false, 0>(a, n, num_sms, st);
  }
  if (kk == 1) return launch_hc_big<1>(a, n, num_sms, st);
  if (kk == 2) return launch_hc_big<2>(a, n, num_sms, st);
  return launch_hc_big<0>(a, n, num_sms, st);
}

void launch_compact(DevCtl* ctl, u64* gkeys, u64* gcnt, const u32* glist, u64* pkeys, u64* pcnt,
                    int num_sms, cudaStream_t st, int gate) {
  launch_pdl(kPdlCompact, compact_kernel, kListStripes, 256, 0, st, ctl, gkeys, gcnt, glist, pkeys, pcnt, gate);
}

}  // namespace cafs
