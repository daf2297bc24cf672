// emit.cu -- K5: run-length emit of sorted (key, offset) pairs.
//
// Replaces emit / emit_fill (sorter.py:244-251, _kernels.py:172-182): the
// reference walks the pairs and fills out[p : p + c] = key.  Here the OUTPUT
// is partitioned into 1024-key warp tiles, grid-strided; every warp works
// alone (no block-level barrier), caches the run it is in, and otherwise finds
// its tile's pairs with a 32-ary warp search of the offsets (staged once per
// CTA in shared memory, or a sampled index of them for large pair sets).  It
// writes with 256-bit stores (STG.256, one 1 KB contiguous run per warp
// instruction).  A tile inside one run -- the
// common case for low-cardinality columns -- is a pure store stream; a
// fragmented tile is walked in windows of 32 run boundaries kept in registers
// (shuffle search, one coalesced 256 B store per warp instruction).  The
// bit-63 flip back to int64 (or the narrowing to 32-bit keys) happens in the
// store.  [begin, end) selects a
// slice of the global sorted order: each GPU of a sharded sort writes only
// its own rows.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kEmitThreads = 128;                 // a CTA lives as long as its slowest warp (one
                                                  // fragmented tile): 4 warps, not 16 (cfg4 / 8:
                                                  // emit 178 -> 160 us; cfg4: 1163 -> 1153 us)
constexpr int kEmitVpl = 8;                       // 32-byte vectors per lane per tile
constexpr u64 kTileBytes = 32ull * kEmitVpl * 32;  // 8 KB per warp tile (1024 int64 keys)
constexpr u64 kIdxEntries = 4096;                // max shared index of the offsets (32 KB)
constexpr int kIdxDefault = 256;                 // measured best (64..1024 within noise)

__device__ __forceinline__ void st_v4(void* p, u64 a, u64 b, u64 c, u64 d) {
  asm volatile("st.global.L1::no_allocate.v4.u64 [%0], {%1,%2,%3,%4};" ::"l"(p), "l"(a), "l"(b),
               "l"(c), "l"(d)
               : "memory");
}

// Warp-cooperative 32-ary search: the largest p in [lo, hi] with offs[p] <= g
// (offs non-decreasing, offs[lo] <= g).  Every lane returns it.
__device__ __forceinline__ u64 warp_find(const u64* offs, u64 lo, u64 hi, u64 g) {
  const int lane = threadIdx.x & 31;
  while (hi - lo >= 32) {
    const u64 step = (hi - lo + 32) / 32;
    u64 probe = lo + (u64)lane * step;
    if (probe > hi) probe = hi;
    const u32 m = __ballot_sync(0xffffffffu, offs[probe] <= g);  // lane 0 always set
    const u64 at = lo + (u64)(31 - __clz(m)) * step;  // last probe with offs <= g
    const u64 nh = at + step - 1;                       // the next probe is > g
    if (nh < hi) hi = nh;
    lo = at < hi ? at : hi;                              // probes past hi were clamped to hi
  }
  const u64 probe = lo + lane;
  const u32 m = __ballot_sync(0xffffffffu, probe <= hi && offs[probe] <= g);
  return lo + (31 - __clz(m));
}

// MAP: tiles find their pairs in a tile -> pair map (large pair sets) instead
// of searching the offsets; a template flag so the common path's code (and its
// 48 registers) is unchanged -- a runtime flag cost cfg4 70 us (60 registers).
template <int KK, bool MAP>
__global__ void __launch_bounds__(kEmitThreads)
    emit_kernel(const u64* __restrict__ keys, const u64* __restrict__ goffs, u64 npairs_arg,
                const DevCtl* ctl, typename KeyT<KK>::T* __restrict__ out, u64 begin, u64 end,
                u64 flip, u64 tpw, u64 idx_entries, int ctl_slice,
                const u32* __restrict__ tile_pair) {
  pdl_begin();
  using K = typename KeyT<KK>::T;
  constexpr u64 VK = 32 / sizeof(K);             // keys per 32-byte vector
  constexpr u64 kTileKeys = kTileBytes / sizeof(K);
  // a uniform 32-byte vector of key k
  auto splat = [](K k) -> u64 {
    if constexpr (sizeof(K) == 8) return (u64)k;
    else return (u64)k | ((u64)k << 32);
  };
  extern __shared__ __align__(16) u64 soffs[];
  u64 npairs = npairs_arg;
  if (ctl) {
    if (!ctl->pairs_ready) return;
    npairs = ctl->npairs;
    if (ctl_slice) {  // a sharded rank's rows, known on device only
      begin = ctl->slice[0];
      end = ctl->slice[1];
    }
  }
  if (npairs == 0 || end <= begin) return;
  const u64* offs = goffs;
  // index of the offsets in shared memory: soffs[j] = offs[j * stride]; with at
  // most kIdxEntries pairs (stride 1) it is the offsets themselves, otherwise it
  // narrows each search to `stride` global entries
  // (with a tile map the tiles' pairs are looked up, not searched: no index)
  const u64 stride = MAP ? 0 : (npairs + idx_entries) / idx_entries;
  const u64 nidx = MAP ? 0 : npairs / stride + 1;
  for (u64 i = threadIdx.x; i < nidx; i += blockDim.x) soffs[i] = goffs[i * stride];
  if (!MAP) __syncthreads();
  if (stride == 1) offs = soffs;
  // pair containing global position g, searching from pair lo (offs[lo] <= g)
  auto locate = [&](u64 lo, u64 g) -> u64 {
    if (MAP) return warp_find(goffs, lo, npairs - 1, g);  // head / tail keys only
    if (stride == 1) return warp_find(soffs, lo, npairs - 1, g);
    const u64 j = warp_find(soffs, lo / stride, nidx - 1, g);
    u64 a = j * stride, b = a + stride - 1;
    if (a < lo) a = lo;
    if (b > npairs - 1) b = npairs - 1;
    return warp_find(goffs, a, b, g);
  };
  const int lane = threadIdx.x & 31;
  const u64 L = end - begin;
  // 32-byte aligned body; up to VK-1 head and VK-1 tail keys are scalar
  const u64 mis = (((uintptr_t)out) & 31) / sizeof(K);
  const u64 head = mis ? ((VK - mis) < L ? (VK - mis) : L) : 0;
  const u64 nvec = (L - head) / VK;
  const u64 body_end = head + nvec * VK;
  if (blockIdx.x == 0 && threadIdx.x < 32) {
    // warp 0: scalar head and tail keys (lanes [0, VK) head, [VK, 2 VK) tail)
    const u64 j = (u64)lane < VK ? (u64)lane : body_end + (lane - VK);
    const bool act = ((u64)lane < VK && j < head) || ((u64)lane >= VK && (u64)lane < 2 * VK && j < L);
    for (int r = 0; r < (int)(2 * VK); ++r) {  // each active lane's search, warp-cooperatively
      const bool mine = __shfl_sync(0xffffffffu, act, r);
      const u64 jj = __shfl_sync(0xffffffffu, j, r);
      if (mine) {
        const u64 p = locate(0, begin + jj);
        if (lane == r) out[jj] = key_unmap<KK>(keys[p], flip);
      }
    }
  }
  if (nvec == 0) return;
  K* ob = out + head;
  const u64 gb = begin + head;  // global position of ob[0]
  const u64 ntiles = (nvec * VK + kTileKeys - 1) / kTileKeys;
  const u64 gw = (u64)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  // each warp takes `tpw` consecutive tiles; CTAs are many and short-lived, so
  // the tiles being written at any moment form one moving window of the output
  // in launch order (measured: 7.3 TB/s vs 6.2-6.4 TB/s for persistent
  // grid-strided warps).  The run a warp is in is cached across its tiles.
  const u64 t0 = gw * tpw;
  const u64 t1 = (t0 + tpw) < ntiles ? (t0 + tpw) : ntiles;
  u64 p = 0;             // pair cursor (pairs only move forward)
  u64 rs = 1, re = 0;    // cached run [rs, re) of pair p (empty)
  u64 rk = 0;            // the run's key as a uniform 8-byte word
  for (u64 t = t0; t < t1; ++t) {
    const u64 e0 = t * kTileKeys;
    const u64 e1 = (e0 + kTileKeys) < nvec * VK ? (e0 + kTileKeys) : nvec * VK;
    const u64 g0 = gb + e0, glast = gb + e1 - 1;
    if (!(g0 >= rs && glast < re)) {
      p = MAP ? (u64)tile_pair[t] : locate(p, g0);
      rs = offs[p];
      re = offs[p + 1];
      rk = splat(key_unmap<KK>(keys[p], flip));
    }
    if (glast < re) {
#pragma unroll
      for (int j = 0; j < kEmitVpl; ++j) {
        const u64 e = e0 + ((u64)j * 32 + lane) * VK;
        if (e < e1) st_v4(ob + e, rk, rk, rk, rk);
      }
      continue;
    }
    // fragmented tile: walk its pairs in windows of 32 run boundaries held in
    // registers (as 32-bit positions relative to the tile).  Each lane takes a
    // whole 32-byte vector: one 5-step shuffle search for the vector's first
    // key; a chunk of 32 vectors no boundary cuts through is written like a
    // uniform tile, otherwise the remaining keys of each vector are searched
    // too -- either way the warp writes 1 KB per store instruction
    u64 q = p;
    u32 g = 0;
    const u32 gend = (u32)(glast + 1 - g0);
    K* ot = ob + e0;  // the tile's first key (32-byte aligned)
    while (true) {
      const u64 qi = q + lane;
      u32 wr = 0xffffffffu;  // end of pair qi, relative to the tile
      K wk = 0;
      if (qi < npairs) {
        const u64 d = offs[qi + 1] - g0;
        wr = d > 0xfffffffeull ? 0xffffffffu : (u32)d;
        wk = key_unmap<KK>(keys[qi], flip);
      }
      const u32 wtop = __shfl_sync(0xffffffffu, wr, 31);
      const u32 wend = wtop < gend ? wtop : gend;
      // number of the window's boundaries <= pos (pos < wtop): the pair of pos
      auto find = [&](u32 pos) -> int {
        int i = 0;
#pragma unroll
        for (int st = 16; st >= 1; st >>= 1) {
          const u32 b = __shfl_sync(0xffffffffu, wr, i + st - 1);
          if (b <= pos) i += st;
        }
        return i;
      };
      u32 a = g;
      // keys before the first whole vector (only after a window change)
      u32 ha = (a + (u32)VK - 1) / (u32)VK * (u32)VK;
      if (ha > wend) ha = wend;
      if (a < ha) {
        const u32 pos = a + lane;
        const K k = __shfl_sync(0xffffffffu, wk, find(pos));
        if (pos < ha) ot[pos] = k;
        a = ha;
      }
      const u32 vend = a + (wend - a) / (u32)VK * (u32)VK;
      for (; a < vend; a += 32 * (u32)VK) {
        const u32 pos = a + lane * (u32)VK;
        const bool act = pos < vend;
        const int i = find(pos);
        const u32 b = __shfl_sync(0xffffffffu, wr, i);
        K kv[VK];
        kv[0] = __shfl_sync(0xffffffffu, wk, i);
        if (__any_sync(0xffffffffu, act && b < pos + (u32)VK)) {
#pragma unroll
          for (int e = 1; e < (int)VK; ++e) kv[e] = __shfl_sync(0xffffffffu, wk, find(pos + e));
        } else {
#pragma unroll
          for (int e = 1; e < (int)VK; ++e) kv[e] = kv[0];
        }
        if (act) {
          if constexpr (sizeof(K) == 8)
            st_v4(ot + pos, (u64)kv[0], (u64)kv[1], (u64)kv[2], (u64)kv[3]);
          else
            st_v4(ot + pos, (u64)kv[0] | ((u64)kv[1] << 32), (u64)kv[2] | ((u64)kv[3] << 32),
                  (u64)kv[4] | ((u64)kv[5] << 32), (u64)kv[6] | ((u64)kv[7] << 32));
        }
      }
      a = vend;
      if (a < wend) {  // keys after the last whole vector (the window ends inside one)
        const u32 pos = a + lane;
        const K k = __shfl_sync(0xffffffffu, wk, find(pos));
        if (pos < wend) ot[pos] = k;
      }
      g = wend;
      if (g >= gend) {
        // the tile's last key is in the window: its pair is the next tile's cursor
        p = q + (u64)find(gend - 1);
        break;
      }
      q += 32;
    }
    if (t + 1 >= t1) break;  // the warp's last tile: no cursor needed
    rs = offs[p];
    re = offs[p + 1];
    rk = splat(key_unmap<KK>(keys[p], flip));
  }
}

// Tile -> pair map for large pair sets: tile_pair[t] = the pair holding the
// first key of emit tile t.  One warp per pair writes the tiles that start
// inside its run (long runs: 32 tiles per store instruction), so the emit's
// warps look their tiles' pairs up instead of searching the offsets (a search
// costs ~4 dependent L2 round trips per tile: 27 % of the emit's warp time on
// cfg3, plus 7 % for each CTA's shared index of the offsets).
template <int KK>
__global__ void __launch_bounds__(256)
    emit_map_kernel(const u64* __restrict__ goffs, const DevCtl* ctl, const void* out, u64 begin,
                    u64 end, u32* __restrict__ tile_pair) {
  pdl_begin();
  using K = typename KeyT<KK>::T;
  constexpr u64 VK = 32 / sizeof(K);
  constexpr u64 kTileKeys = kTileBytes / sizeof(K);
  if (!ctl->pairs_ready) return;
  const u64 npairs = ctl->npairs;
  const u64 L = end - begin;
  const u64 mis = (((uintptr_t)out) & 31) / sizeof(K);  // the emit's head (same formula)
  const u64 head = mis ? ((VK - mis) < L ? (VK - mis) : L) : 0;
  const u64 nkeys = (L - head) / VK * VK;
  const u64 ntiles = (nkeys + kTileKeys - 1) / kTileKeys;
  const u64 gb = begin + head;
  // a thread per pair writes its (usually 0 or 1) tiles; a run covering more
  // than 32 tiles is written by its whole warp, 32 entries per instruction
  const int lane = threadIdx.x & 31;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 p0 = (u64)blockIdx.x * blockDim.x + (threadIdx.x & ~31u); p0 < npairs;
       p0 += stride) {  // warp-uniform: p0 is the warp's first pair
    const u64 p = p0 + lane;
    u64 t_lo = 0, t_hi = 0;
    if (p < npairs) {
      const u64 s = goffs[p], e = goffs[p + 1];
      // tiles whose first position gb + t * TK lies in [s, e)
      t_lo = s <= gb ? 0 : (s - gb + kTileKeys - 1) / kTileKeys;
      t_hi = e <= gb ? 0 : (e - gb + kTileKeys - 1) / kTileKeys;
      if (t_hi > ntiles) t_hi = ntiles;
    }
    const bool longrun = t_hi > t_lo + 32;
    if (!longrun)
      for (u64 t = t_lo; t < t_hi; ++t) tile_pair[t] = (u32)p;
    for (u32 m = __ballot_sync(0xffffffffu, longrun); m; m &= m - 1) {
      const int r = __ffs(m) - 1;
      const u64 lo = __shfl_sync(0xffffffffu, t_lo, r), hi = __shfl_sync(0xffffffffu, t_hi, r);
      const u32 pr = (u32)(p0 + r);
      for (u64 t = lo + lane; t < hi; t += 32) tile_pair[t] = pr;
    }
  }
}

u64 emit_tiles(u64 L, int kk) { return (L + kTileBytes / (kk ? 4 : 8) - 1) / (kTileBytes / (kk ? 4 : 8)); }

void launch_emit_map(const u64* offs, const DevCtl* ctl, const void* out, u64 begin, u64 end,
                     u32* tile_pair, u64 npairs_bound, int num_sms, cudaStream_t st, int kk) {
  u64 grid = (npairs_bound + 255) / 256;  // a thread per pair
  const u64 maxg = (u64)num_sms * 8;
  if (grid > maxg) grid = maxg;
  if (grid < 1) grid = 1;
  if (kk)
    launch_pdl(kPdlEmit, emit_map_kernel<1>, (unsigned)grid, 256, 0, st, offs, ctl, out, begin,
               end, tile_pair);
  else
    launch_pdl(kPdlEmit, emit_map_kernel<0>, (unsigned)grid, 256, 0, st, offs, ctl, out, begin,
               end, tile_pair);
}

void launch_emit(const u64* keys, const u64* offs, u64 npairs, const DevCtl* ctl, void* out,
                 u64 begin, u64 end, u64 flip, int num_sms, cudaStream_t st, u64 /*npairs_bound*/,
                 int kk, bool ctl_slice, const u32* tile_pair) {
  const u64 L = end > begin ? end - begin : 0;
  const u64 tile_keys = kTileBytes / (kk ? 4 : 8);
  const u64 wtiles = (L + tile_keys - 1) / tile_keys;
  static int tpw = -1, idx = -1, thr = 0;  // CAFS_EMIT_TPW / CAFS_EMIT_IDX / CAFS_EMIT_THREADS: tuning knobs
  if (tpw < 0) {
    const char* e = getenv("CAFS_EMIT_THREADS");
    thr = e ? atoi(e) : 0;
    e = getenv("CAFS_EMIT_TPW");
    tpw = e ? atoi(e) : 2;
    if (tpw < 1 || tpw > 4096) tpw = 2;
    e = getenv("CAFS_EMIT_IDX");
    idx = e ? atoi(e) : kIdxDefault;
    if (idx < 32 || idx > (int)kIdxEntries) idx = kIdxDefault;
  }
  // small outputs: one tile per warp and smaller CTAs, so the work still
  // spreads over every SM (1M keys = 977 tiles: 31 CTAs of 16 warps x 2 tiles)
  u64 tpw_use = (u64)tpw, threads = kEmitThreads;
  const u64 spread = (u64)num_sms * 4;
  if ((wtiles + tpw_use * 4 - 1) / (tpw_use * 4) < spread * 4) tpw_use = 1;
  if (thr == 64 || thr == 128) threads = thr;
  const u64 wpb = threads / 32;
  u64 grid = (wtiles + tpw_use * wpb - 1) / (tpw_use * wpb);
  if (grid < 1) grid = 1;
  const size_t sm = ((u64)idx + 1) * 8;
  switch (kk) {
    case 1:
      if (tile_pair)
        launch_pdl(kPdlEmit, emit_kernel<1, true>, (unsigned)grid, (unsigned)threads, sm, st, keys,
                   offs, npairs, ctl, (u32*)out, begin, end, flip, tpw_use, (u64)idx,
                   ctl_slice ? 1 : 0, tile_pair);
      else
        launch_pdl(kPdlEmit, emit_kernel<1, false>, (unsigned)grid, (unsigned)threads, sm, st, keys,
                   offs, npairs, ctl, (u32*)out, begin, end, flip, tpw_use, (u64)idx,
                   ctl_slice ? 1 : 0, tile_pair);
      break;
    case 2:
      if (tile_pair)
        launch_pdl(kPdlEmit, emit_kernel<2, true>, (unsigned)grid, (unsigned)threads, sm, st, keys,
                   offs, npairs, ctl, (u32*)out, begin, end, flip, tpw_use, (u64)idx,
                   ctl_slice ? 1 : 0, tile_pair);
      else
        launch_pdl(kPdlEmit, emit_kernel<2, false>, (unsigned)grid, (unsigned)threads, sm, st, keys,
                   offs, npairs, ctl, (u32*)out, begin, end, flip, tpw_use, (u64)idx,
                   ctl_slice ? 1 : 0, tile_pair);
      break;
    default:
      if (tile_pair)
        launch_pdl(kPdlEmit, emit_kernel<0, true>, (unsigned)grid, (unsigned)threads, sm, st, keys,
                   offs, npairs, ctl, (u64*)out, begin, end, flip, tpw_use, (u64)idx,
                   ctl_slice ? 1 : 0, tile_pair);
      else
        launch_pdl(kPdlEmit, emit_kernel<0, false>, (unsigned)grid, (unsigned)threads, sm, st, keys,
                   offs, npairs, ctl, (u64*)out, begin, end, flip, tpw_use, (u64)idx,
                   ctl_slice ? 1 : 0, tile_pair);
  }
}

}  // namespace cafs
