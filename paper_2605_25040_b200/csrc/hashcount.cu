// hashcount.cu -- K3: the main-route counting pass and its compaction.
//
// Replaces count_sequence (_kernels.py:25-81) / main_count_loop
// (sorter.py:183-196).  The reference folds runs and probes a 4-slot
// cache-line bucket per update, spilling overflow keys to a side buffer.  The
// B200 design keeps the same contract -- every element lands in exactly one
// (key, count) cell, cells are merged by key, the spill guard re-routes to the
// fallback -- with a layout for 148 SMs:
//
//   * persistent CTAs (one per SM, 1024 threads); warp 0 is a TMA producer
//     that streams 16 KB chunks of the int64 column into a 6-stage shared
//     memory ring (cp.async.bulk + mbarrier complete_tx), warps 1..31 consume;
//   * per element (bit-63 flip in registers):
//       - dense-range window (dictionary-encoded columns): one shared atomic
//         into counts[v - base]; the window is set by the estimate kernel from
//         the sample's span, exact for any key because out-of-window keys take
//         the hash path;
//       - otherwise a per-CTA shared open-addressing (u64 key, u32 count) table,
//         first probe inline, linear probing + CAS claims on the slow path,
//         claims capped at 3/4 load;
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
constexpr int kHcConsumers = kHcThreads - 32;
constexpr u32 kRange = 8192;              // dense window (u32 counters, 32 KB)
constexpr int kSLog2 = 13;                // shared table: 8192 slots (64 KB keys + 32 KB counts)
constexpr u32 kS = 1u << kSLog2;
constexpr u32 kSClaimCap = kS * 3 / 4;
constexpr int kSMaxProbe = 32;
constexpr int kStages = 6;
constexpr u32 kStageKeys = 2048;          // 16 KB per stage
constexpr size_t kHcSmem =
    (size_t)kRange * 4 + (size_t)kS * 8 + (size_t)kS * 4 + (size_t)kStages * kStageKeys * 8 +
    (size_t)2 * kStages * 8 + 16;

struct HcArgs {
  const u64* x;
  u64 n;
  u64 flip;
  u64 mult;
  DevCtl* ctl;
  u64* gkeys;
  u64* gcnt;
  u32* glist;
  int use_range;
};

// key -> global table, keeping the sentinel value out of it
__device__ __forceinline__ void table_add(const HcArgs& a, u64 key, u64 inc) {
  if (key == kEmpty) atomicAdd(&a.ctl->empty_key_count, inc);
  else global_insert(a.gkeys, a.gcnt, a.glist, a.ctl, key, inc, a.mult);
}

__global__ void __launch_bounds__(kHcThreads, 1) hash_count_kernel(HcArgs a) {
  extern __shared__ __align__(128) unsigned char smem[];
  u64* stage = (u64*)smem;                                        // [kStages][kStageKeys]
  u64* skeys = stage + (size_t)kStages * kStageKeys;              // [kS]
  u32* scnt = (u32*)(skeys + kS);                                 // [kS]
  u32* dcnt = scnt + kS;                                          // [kRange]
  u64* full = (u64*)(dcnt + kRange);                              // [kStages]
  u64* empty = full + kStages;                                    // [kStages]
  __shared__ u32 sclaims;
  __shared__ u64 red_empty[32], red_glob[32];

  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u64 flip = a.flip, mult = a.mult;
  const u64 base = a.use_range ? a.ctl->range_base : 0ull;
  const u32 rlen = a.use_range ? a.ctl->range_len : 0u;

  for (u32 i = tid; i < kS; i += kHcThreads) { skeys[i] = kEmpty; scnt[i] = 0; }
  for (u32 i = tid; i < kRange; i += kHcThreads) dcnt[i] = 0;
  if (tid == 0) {
    sclaims = 0;
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kHcConsumers / 32);
    }
    fence_mbar_init();
  }
  __syncthreads();

  // body = 16-byte aligned, even-length stretch of x; head/tail elements scalar
  const u64 n = a.n;
  const u64 head = (((uintptr_t)a.x) & 15) ? 1 : 0;
  const u64 body = n > head ? ((n - head) & ~1ull) : 0;
  const u64* xb = a.x + head;
  const u64 nchunks = (body + kStageKeys - 1) / kStageKeys;

  u64 empty_cnt = 0, glob_cnt = 0;

  auto count1 = [&](u64 raw) {
    const u64 v = raw ^ flip;
    const u64 d = v - base;
    if (d < rlen) {
      atomicAdd(&dcnt[d], 1u);
      return;
    }
    if (v == kEmpty) { empty_cnt++; return; }
    u32 h = mhash(v, mult, 64 - kSLog2);
    u64 k = skeys[h];
    if (k == v) { atomicAdd(&scnt[h], 1u); return; }
    // slow path: linear probing with capped claims
    for (int p = 0; p < kSMaxProbe; ++p) {
      if (k == v) { atomicAdd(&scnt[h], 1u); return; }
      if (k == kEmpty) {
        if (*((volatile u32*)&sclaims) >= kSClaimCap) break;
        u64 old = atomicCAS(&skeys[h], kEmpty, v);
        if (old == kEmpty) {
          atomicAdd(&sclaims, 1u);
          atomicAdd(&scnt[h], 1u);
          return;
        }
        if (old == v) { atomicAdd(&scnt[h], 1u); return; }
      }
      h = (h + 1) & (kS - 1);
      k = *((volatile u64*)&skeys[h]);
    }
    glob_cnt++;
    global_insert(a.gkeys, a.gcnt, a.glist, a.ctl, v, 1, mult);
  };

  if (wid == 0) {
    // ---- TMA producer ----
    if (lane == 0) {
      u32 it = 0;
      for (u64 c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
        const u32 s = it % kStages;
        const u32 ph = (it / kStages) & 1;
        if (it >= (u32)kStages) mbar_wait(&empty[s], ph ^ 1);
        const u64 off = c * kStageKeys;
        const u64 cnt = (body - off) < kStageKeys ? (body - off) : kStageKeys;
        const u32 bytes = (u32)(cnt * 8);
        mbar_arrive_expect_tx(&full[s], bytes);
        tma_load_1d(stage + (size_t)s * kStageKeys, xb + off, bytes, &full[s]);
      }
    }
  } else {
    // ---- consumers ----
    const int ctid = tid - 32;
    u32 it = 0;
    for (u64 c = blockIdx.x; c < nchunks; c += gridDim.x, ++it) {
      const u32 s = it % kStages;
      const u32 ph = (it / kStages) & 1;
      mbar_wait(&full[s], ph);
      const u64 off = c * kStageKeys;
      const u32 cnt = (u32)((body - off) < kStageKeys ? (body - off) : kStageKeys);
      const ulonglong2* sv = (const ulonglong2*)(stage + (size_t)s * kStageKeys);
      for (u32 i = ctid; i < cnt / 2; i += kHcConsumers) {
        ulonglong2 v = sv[i];
        count1(v.x);
        count1(v.y);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (blockIdx.x == 0 && ctid == 0) {
      if (head && n > 0) count1(a.x[0]);
      if (n > head && ((n - head) & 1)) count1(a.x[n - 1]);
    }
  }
  __syncthreads();

  // ---- flush the CTA's shared cells into the global table ----
  for (u32 d = tid; d < rlen; d += kHcThreads) {
    const u32 c = dcnt[d];
    if (c) table_add(a, base + d, c);
  }
  for (u32 h = tid; h < kS; h += kHcThreads) {
    const u32 c = scnt[h];
    if (c) table_add(a, skeys[h], c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    empty_cnt += __shfl_xor_sync(0xffffffffu, empty_cnt, o);
    glob_cnt += __shfl_xor_sync(0xffffffffu, glob_cnt, o);
  }
  if (lane == 0) { red_empty[wid] = empty_cnt; red_glob[wid] = glob_cnt; }
  __syncthreads();
  if (tid == 0) {
    u64 e = 0, g = 0;
    for (int w = 0; w < kHcThreads / 32; ++w) { e += red_empty[w]; g += red_glob[w]; }
    if (e) atomicAdd(&a.ctl->empty_key_count, e);
    if (g) atomicAdd(&a.ctl->g_updates, g);
  }
}

// Occupied global slots -> dense (key, count) pairs; re-zero the slots so the
// table is clean for the next call.  The sentinel key's count becomes the last
// pair.
__global__ void compact_kernel(DevCtl* ctl, u64* gkeys, u64* gcnt, const u32* glist, u64* pkeys,
                               u64* pcnt) {
  if (ctl->overflow) return;
  const u64 m = ctl->g_used;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < m; i += stride) {
    const u32 h = glist[i];
    pkeys[i] = gkeys[h];
    pcnt[i] = gcnt[h];
    gkeys[h] = kEmpty;
    gcnt[h] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const u64 e = ctl->empty_key_count;
    if (e) { pkeys[m] = kEmpty; pcnt[m] = e; }
    ctl->npairs = m + (e ? 1 : 0);
  }
}

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
  if (threadIdx.x == 0) {
    ctl->g_used = 0;
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

size_t hash_count_smem() { return kHcSmem; }

cudaError_t launch_hash_count(const u64* x, u64 n, u64 flip, u64 mult, DevCtl* ctl, u64* gkeys,
                              u64* gcnt, u32* glist, int use_range, int num_sms,
                              cudaStream_t st) {
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(hash_count_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kHcSmem);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  HcArgs a{x, n, flip, mult, ctl, gkeys, gcnt, glist, use_range};
  u64 chunks = (n + kStageKeys - 1) / kStageKeys;
  int grid = (int)(chunks < (u64)num_sms ? (chunks ? chunks : 1) : (u64)num_sms);
  hash_count_kernel<<<grid, kHcThreads, kHcSmem, st>>>(a);
  return cudaGetLastError();
}

void launch_compact(DevCtl* ctl, u64* gkeys, u64* gcnt, const u32* glist, u64* pkeys, u64* pcnt,
                    int num_sms, cudaStream_t st) {
  compact_kernel<<<num_sms, 256, 0, st>>>(ctl, gkeys, gcnt, glist, pkeys, pcnt);
}

}  // namespace cafs
