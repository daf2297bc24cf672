// emit.cu -- K5: run-length emit of sorted (key, offset) pairs.
//
// Replaces emit / emit_fill (sorter.py:244-251, _kernels.py:172-182): the
// reference walks pairs and fills out[p : p + c] = key.  Here the OUTPUT is
// partitioned: each CTA owns a contiguous span of 16-byte vectors, finds its
// first pair once with a 32-ary warp search over the offsets, then walks
// 8192-element tiles.  A tile covered by a single run (the common case for
// low-cardinality columns) is a pure streaming fill with 128-bit stores; a
// fragmented tile gives each thread 16 consecutive positions, one binary
// search and a forward walk.  The sign-bit flip back to int64 happens in the
// store.  `begin/end` select a slice of the global sorted order, which is how
// each GPU of a sharded sort writes only its own output rows.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kEmitThreads = 512;
constexpr u64 kEmitTileV = 4096;  // 16-byte vectors per tile (8192 keys)

// largest p in [lo, hi) with offs[p] <= g (offs non-decreasing, offs[lo] <= g)
__device__ u64 warp_search(const u64* offs, u64 lo, u64 hi, u64 g) {
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const u64 step = (hi - lo + 31) / 32;
    u64 probe = lo + (u64)lane * step;
    bool pred = probe < hi && offs[probe] <= g;
    const u32 b = __ballot_sync(0xffffffffu, pred);
    const int last = 31 - __clz(b);  // lane 0 always true (offs[lo] <= g)
    lo = lo + (u64)last * step;
    const u64 nh = lo + step;
    hi = nh < hi ? nh : hi;
  }
  const u64 probe = lo + lane;
  const bool pred = probe < hi && offs[probe] <= g;
  const u32 b = __ballot_sync(0xffffffffu, pred);
  return lo + (31 - __clz(b));
}

__device__ __forceinline__ u64 bsearch_pair(const u64* offs, u64 lo, u64 hi, u64 g) {
  // largest p in [lo, hi] with offs[p] <= g
  while (lo < hi) {
    const u64 mid = (lo + hi + 1) >> 1;
    if (offs[mid] <= g) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kEmitThreads)
    emit_kernel(const u64* __restrict__ keys, const u64* __restrict__ offs, u64 npairs_arg,
                const DevCtl* ctl, u64* __restrict__ out, u64 begin, u64 end, u64 flip) {
  __shared__ u64 sp[2][2];
  u64 npairs = npairs_arg;
  if (ctl) {
    if (!ctl->pairs_ready) return;
    npairs = ctl->npairs;
  }
  if (npairs == 0 || end <= begin) return;
  const int tid = threadIdx.x, wid = tid >> 5;
  const u64 L = end - begin;
  const u64 head = (((uintptr_t)out) & 15) ? 1 : 0;
  const u64 nvec = L > head ? (L - head) / 2 : 0;
  // scalar head / tail element
  if (blockIdx.x == 0 && tid == 0) {
    if (head) {
      const u64 p = bsearch_pair(offs, 0, npairs - 1, begin);
      out[0] = keys[p] ^ flip;
    }
    if (L > head && ((L - head) & 1)) {
      const u64 p = bsearch_pair(offs, 0, npairs - 1, end - 1);
      out[L - 1] = keys[p] ^ flip;
    }
  }
  if (nvec == 0) return;
  // this CTA's vector span, a whole number of tiles
  const u64 ntiles = (nvec + kEmitTileV - 1) / kEmitTileV;
  const u64 tpb = (ntiles + gridDim.x - 1) / gridDim.x;
  const u64 t_begin = (u64)blockIdx.x * tpb;
  u64 t_end = t_begin + tpb;
  if (t_end > ntiles) t_end = ntiles;
  if (t_begin >= t_end) return;
  ulonglong2* ov = (ulonglong2*)(out + head);
  const u64 gbase = begin + head;  // global position of vector 0's first element

  u64 p = 0;  // running pair cursor (warp 0)
  if (wid == 0) p = warp_search(offs, 0, npairs, gbase + t_begin * kEmitTileV * 2);
  int par = 0;
  for (u64 t = t_begin; t < t_end; ++t, par ^= 1) {
    const u64 v0 = t * kEmitTileV;
    const u64 v1 = (v0 + kEmitTileV) < nvec ? (v0 + kEmitTileV) : nvec;
    const u64 g0 = gbase + v0 * 2, glast = gbase + v1 * 2 - 1;
    if (wid == 0) {
      const int lane = tid & 31;
      // advance p to the pair containing g0 (offs[npairs] = total > glast stops the scan)
      while (true) {
        const u64 q = p + 1 + lane;
        const bool le = q <= npairs && offs[q] <= g0;
        const u32 b = __ballot_sync(0xffffffffu, le);
        p += __popc(b);
        if (b != 0xffffffffu) break;
      }
      u64 p1 = p;
      while (true) {
        const u64 q = p1 + 1 + lane;
        const bool le = q <= npairs && offs[q] <= glast;
        const u32 b = __ballot_sync(0xffffffffu, le);
        p1 += __popc(b);
        if (b != 0xffffffffu) break;
      }
      if (lane == 0) { sp[par][0] = p; sp[par][1] = p1; }
    }
    __syncthreads();
    const u64 p0 = sp[par][0], p1 = sp[par][1];
    if (p0 == p1) {
      const u64 k = keys[p0] ^ flip;
      for (u64 v = v0 + tid; v < v1; v += kEmitThreads) st_stream_v2(ov + v, k, k);
    } else {
      // 8 vectors (16 keys) per thread: one search, then walk forward
      const u64 va = v0 + (u64)tid * 8;
      if (va < v1) {
        const u64 g = gbase + va * 2;
        u64 q = bsearch_pair(offs, p0, p1, g);
        u64 nb = offs[q + 1];
        u64 kq = keys[q] ^ flip;
        const int nv = (int)((v1 - va) < 8 ? (v1 - va) : 8);
        for (int e = 0; e < nv; ++e) {
          const u64 ga = g + 2 * e;
          while (ga >= nb) { ++q; nb = offs[q + 1]; kq = keys[q] ^ flip; }
          const u64 ka = kq;
          while (ga + 1 >= nb) { ++q; nb = offs[q + 1]; kq = keys[q] ^ flip; }
          st_stream_v2(ov + va + e, ka, kq);
        }
      }
    }
  }
}

void launch_emit(const u64* keys, const u64* offs, u64 npairs, const DevCtl* ctl, u64* out,
                 u64 begin, u64 end, u64 flip, int num_sms, cudaStream_t st) {
  const u64 L = end > begin ? end - begin : 0;
  u64 tiles = (L / 2 + kEmitTileV - 1) / kEmitTileV;
  u64 grid = (u64)num_sms * 4;
  if (tiles < grid) grid = tiles ? tiles : 1;
  emit_kernel<<<(unsigned)grid, kEmitThreads, 0, st>>>(keys, offs, npairs, ctl, out, begin, end,
                                                       flip);
}

}  // namespace cafs
