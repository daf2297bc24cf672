// emit.cu -- K5: run-length emit of sorted (key, offset) pairs.
//
// Replaces emit / emit_fill (sorter.py:244-251, _kernels.py:172-182): the
// reference walks the pairs and fills out[p : p + c] = key.  Here the OUTPUT
// is partitioned into warp tiles of 1024 keys (8 KB): every warp works alone
// (no block-level barrier), finds the pairs covering its tile with a binary
// search of the offsets (staged once per CTA in shared memory when there are
// at most kSmemOffs pairs), and writes with 256-bit stores (STG.256, one
// 1 KB contiguous run per warp instruction).  A tile inside one run -- the
// common case for low-cardinality columns -- is a pure store stream; a
// fragmented tile resolves each lane's 4 keys by a search + forward walk.  The
// bit-63 flip back to int64 happens in the store.  [begin, end) selects a
// slice of the global sorted order: each GPU of a sharded sort writes only
// its own rows.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kEmitThreads = 512;
constexpr int kEmitVpl = 8;                       // 32-byte vectors per lane per tile
constexpr u64 kTileKeys = 32ull * kEmitVpl * 4;  // 1024 keys per warp tile
constexpr u64 kSmemOffs = 8192;                  // pairs whose offsets fit in smem

__device__ __forceinline__ void st_v4(void* p, u64 a, u64 b, u64 c, u64 d) {
  asm volatile("st.global.L1::no_allocate.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b),
               "l"(c), "l"(d)
               : "memory");
}

// largest p in [lo, hi] with offs[p] <= g  (offs non-decreasing, offs[lo] <= g)
__device__ __forceinline__ u64 find_pair(const u64* offs, u64 lo, u64 hi, u64 g) {
  while (lo < hi) {
    const u64 mid = (lo + hi + 1) >> 1;
    if (offs[mid] <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

template <bool SMEM>
__global__ void __launch_bounds__(kEmitThreads)
    emit_kernel(const u64* __restrict__ keys, const u64* __restrict__ goffs, u64 npairs_arg,
                const DevCtl* ctl, u64* __restrict__ out, u64 begin, u64 end, u64 flip) {
  extern __shared__ __align__(16) u64 soffs[];
  u64 npairs = npairs_arg;
  if (ctl) {
    if (!ctl->pairs_ready) return;
    npairs = ctl->npairs;
  }
  if (npairs == 0 || end <= begin) return;
  if (SMEM && npairs > kSmemOffs) return;  // host picks the variant; guard anyway
  const u64* offs = goffs;
  if (SMEM) {
    for (u64 i = threadIdx.x; i <= npairs; i += kEmitThreads) soffs[i] = goffs[i];
    __syncthreads();
    offs = soffs;
  }
  const int lane = threadIdx.x & 31;
  const u64 L = end - begin;
  // 32-byte aligned body; up to 3 head and 3 tail keys are scalar
  const u64 mis = (((uintptr_t)out) >> 3) & 3;
  const u64 head = mis ? ((4 - mis) < L ? (4 - mis) : L) : 0;
  const u64 nvec = (L - head) / 4;
  const u64 body_end = head + nvec * 4;
  if (blockIdx.x == 0 && threadIdx.x < 8) {
    const u64 j = threadIdx.x < 4 ? threadIdx.x : body_end + (threadIdx.x - 4);
    if ((threadIdx.x < 4 && j < head) || (threadIdx.x >= 4 && j < L)) {
      const u64 p = find_pair(offs, 0, npairs - 1, begin + j);
      out[j] = keys[p] ^ flip;
    }
  }
  if (nvec == 0) return;
  u64* ob = out + head;
  const u64 gb = begin + head;  // global position of ob[0]
  const u64 ntiles = (nvec * 4 + kTileKeys - 1) / kTileKeys;
  const u64 nwarps = (u64)gridDim.x * (kEmitThreads / 32);
  const u64 gw = (u64)blockIdx.x * (kEmitThreads / 32) + (threadIdx.x >> 5);
  u64 p = 0;  // pair cursor: tiles are visited in increasing order per warp
  for (u64 t = gw; t < ntiles; t += nwarps) {
    const u64 e0 = t * kTileKeys;
    const u64 e1 = (e0 + kTileKeys) < nvec * 4 ? (e0 + kTileKeys) : nvec * 4;
    u64 p0 = 0, p1 = 0;
    if (lane == 0) p0 = find_pair(offs, p, npairs - 1, gb + e0);
    if (lane == 1) p1 = find_pair(offs, p, npairs - 1, gb + e1 - 1);
    p0 = __shfl_sync(0xffffffffu, p0, 0);
    p1 = __shfl_sync(0xffffffffu, p1, 1);
    p = p0;
    if (p0 == p1) {
      const u64 k = keys[p0] ^ flip;
#pragma unroll
      for (int j = 0; j < kEmitVpl; ++j) {
        const u64 e = e0 + ((u64)j * 32 + lane) * 4;
        if (e < e1) st_v4(ob + e, k, k, k, k);
      }
    } else {
      u64 q = p0;
#pragma unroll 1
      for (int j = 0; j < kEmitVpl; ++j) {
        const u64 e = e0 + ((u64)j * 32 + lane) * 4;
        if (e < e1) {
          const u64 g = gb + e;
          q = find_pair(offs, q, p1, g);
          u64 kv[4];
          u64 qq = q;
          u64 nb = offs[qq + 1];
          kv[0] = keys[qq] ^ flip;
#pragma unroll
          for (int r = 1; r < 4; ++r) {
            while (g + r >= nb) { ++qq; nb = offs[qq + 1]; }
            kv[r] = keys[qq] ^ flip;
          }
          st_v4(ob + e, kv[0], kv[1], kv[2], kv[3]);
        }
      }
    }
  }
}

void launch_emit(const u64* keys, const u64* offs, u64 npairs, const DevCtl* ctl, u64* out,
                 u64 begin, u64 end, u64 flip, int num_sms, cudaStream_t st, u64 npairs_bound) {
  const u64 L = end > begin ? end - begin : 0;
  const u64 wtiles = (L + kTileKeys - 1) / kTileKeys;
  u64 grid = (u64)num_sms * 4;
  const u64 need = (wtiles + (kEmitThreads / 32) - 1) / (kEmitThreads / 32);
  if (need < grid) grid = need ? need : 1;
  // npairs_bound: an upper bound of the pair count known on the host (the device
  // count may be smaller); smem staging when it fits
  static int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(emit_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)((kSmemOffs + 1) * 8));
    attr_dev = dev;
  }
  if (npairs_bound <= kSmemOffs) {
    const size_t sm = (size_t)(npairs_bound + 1) * 8;
    emit_kernel<true><<<(unsigned)grid, kEmitThreads, sm, st>>>(keys, offs, npairs, ctl, out,
                                                                begin, end, flip);
  } else {
    emit_kernel<false><<<(unsigned)grid, kEmitThreads, 0, st>>>(keys, offs, npairs, ctl, out,
                                                                 begin, end, flip);
  }
}

}  // namespace cafs
