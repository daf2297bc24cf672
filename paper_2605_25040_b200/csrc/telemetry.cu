// telemetry.cu -- reference-exact bucket-table telemetry (opt-in).
//
// The device pipeline never builds the reference's 4-slot bucket table
// (buckets.py:172-292), so spill_len / updates / hits / claims / spill_pushes /
// guard_fired are not by-products of the sort.  They are nevertheless an
// order-independent function of the input (SURVEY.md §8(a) note):
//
//   * count_sequence (_kernels.py:25-81) applies one update per run of equal
//     adjacent values; a bucket's slots are claimed permanently by the first
//     <= cap distinct keys (by first occurrence) that hash to it; any other key
//     finds the bucket full on every one of its runs and spills;
//   * so: updates = #runs; a key is stored iff fewer than cap keys of its
//     bucket occur earlier; claims = #stored keys; hits = runs of stored keys -
//     claims; spill_pushes = runs of spilled keys; spill_len = occurrences of
//     spilled keys; counted_total = n - spill_len; the guard fires iff
//     2 * spill_len > n (sorter.py:264).
//
// Kernels: (1) a lookup table key -> pair index over the distinct keys;
// (2) one pass over the UNSORTED input: every run start adds a run to its key
// and offers its index to the key's first occurrence (atomicMin);
// (3) composite keys (bucket << 32 | first) are sorted (msd/small sort) and a
// key is stored iff it is among the first `cap` of its bucket segment.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

struct TelAccum {
  unsigned long long runs, spill_len, spill_pushes, claims, stored_runs;
  unsigned long long empty_idx;  // pair index of the sentinel key value ~0, if present
};

__device__ __forceinline__ u32 tl_hash(u64 k, int log2s) {
  return (u32)(fmix64(k) >> (64 - log2s));  // mixer: robust to multiplicative colliders
}

__global__ void tl_build_kernel(const u64* __restrict__ keys, u64 np, u64* tkeys, u32* tidx,
                                int log2s, u32* first, u32* runs, TelAccum* acc) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u32 mask = (1u << log2s) - 1;
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < np; j += stride) {
    const u64 k = keys[j];
    first[j] = 0xFFFFFFFFu;
    runs[j] = 0;
    if (k == kEmpty) { acc->empty_idx = j; continue; }  // looked up by index, not hashed
    u32 h = tl_hash(k, log2s);
    while (true) {  // keys are distinct; load <= 1/2
      const u64 old = atomicCAS(&tkeys[h], kEmpty, k);
      if (old == kEmpty) { tidx[h] = (u32)j; break; }
      h = (h + 1) & mask;
    }
  }
}

__device__ __forceinline__ u32 tl_lookup(const u64* tkeys, const u32* tidx, int log2s, u64 k,
                                         u64 empty_idx) {
  if (k == kEmpty) return (u32)empty_idx;  // the sentinel value has no table slot
  const u32 mask = (1u << log2s) - 1;
  u32 h = tl_hash(k, log2s);
  while (tkeys[h] != k) h = (h + 1) & mask;
  return tidx[h];
}

template <int KK>
__global__ void __launch_bounds__(512)
    tl_runs_kernel(const typename KeyT<KK>::T* __restrict__ x, u64 n, u64 flip, const u64* tkeys,
                   const u32* tidx, int log2s, u32* first, u32* runs, TelAccum* acc) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 empty_idx = acc->empty_idx;
  u64 local = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 v = key_map<KK>(x[i], flip);
    if (i > 0 && key_map<KK>(x[i - 1], flip) == v) continue;
    ++local;
    const u32 j = tl_lookup(tkeys, tidx, log2s, v, empty_idx);
    atomicAdd(&runs[j], 1u);
    atomicMin(&first[j], (u32)i);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
  if ((threadIdx.x & 31) == 0 && local) atomicAdd(&acc->runs, local);
}

// composite sort key: reference bucket of the key (in the reference's unsigned
// domain of the input dtype), then first occurrence
__global__ void tl_comp_kernel(const u64* __restrict__ keys, u64 np, const u32* first, u64 mult,
                               int m_log2, int dom, u64* comp, u64* cidx) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < np; j += stride) {
    u64 k = keys[j];
    // dom 0: 64-bit (key already in the reference domain); 1: int32 widened to
    // int64 then order-mapped -> reference u32 domain; 2: uint32 widened likewise
    if (dom == 1) k = (u64)((u32)(int)(long long)(k ^ kSign) ^ 0x80000000u);
    else if (dom == 2) k = (u64)(u32)(k ^ kSign);
    const u64 b = (k * mult) >> (64 - m_log2);
    comp[j] = (b << 32) | first[j];
    cidx[j] = j;
  }
}

__global__ void tl_classify_kernel(const u64* __restrict__ comp, const u64* __restrict__ cidx,
                                   u64 np, int cap, const u64* __restrict__ counts,
                                   const u32* runs, TelAccum* acc) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  u64 sl = 0, sp = 0, cl = 0, sr = 0;
  for (u64 q = blockIdx.x * (u64)blockDim.x + threadIdx.x; q < np; q += stride) {
    const bool stored = q < (u64)cap || (comp[q - cap] >> 32) != (comp[q] >> 32);
    const u64 j = cidx[q];
    if (stored) { cl += 1; sr += runs[j]; }
    else { sl += counts[j]; sp += runs[j]; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    sl += __shfl_xor_sync(0xffffffffu, sl, o);
    sp += __shfl_xor_sync(0xffffffffu, sp, o);
    cl += __shfl_xor_sync(0xffffffffu, cl, o);
    sr += __shfl_xor_sync(0xffffffffu, sr, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (sl) atomicAdd(&acc->spill_len, sl);
    if (sp) atomicAdd(&acc->spill_pushes, sp);
    if (cl) atomicAdd(&acc->claims, cl);
    if (sr) atomicAdd(&acc->stored_runs, sr);
  }
}

size_t tel_accum_bytes() { return sizeof(TelAccum); }

void launch_tel_build(const u64* keys, u64 np, u64* tkeys, u32* tidx, int log2s, u32* first,
                      u32* runs, void* acc, int num_sms, cudaStream_t st) {
  cudaMemsetAsync(tkeys, 0xFF, (size_t(1) << log2s) * 8, st);
  u64 blocks = (np + 255) / 256;
  if (blocks > (u64)num_sms * 8) blocks = (u64)num_sms * 8;
  tl_build_kernel<<<(unsigned)(blocks ? blocks : 1), 256, 0, st>>>(keys, np, tkeys, tidx, log2s,
                                                                   first, runs, (TelAccum*)acc);
}

void launch_tel_runs(const void* x, u64 n, u64 flip, const u64* tkeys, const u32* tidx, int log2s,
                     u32* first, u32* runs, void* acc, int num_sms, cudaStream_t st, int kk) {
  const dim3 g(num_sms * 4), b(512);
  TelAccum* ac = (TelAccum*)acc;
  switch (kk) {
    case 1:
      tl_runs_kernel<1><<<g, b, 0, st>>>((const u32*)x, n, flip, tkeys, tidx, log2s, first, runs, ac);
      break;
    case 2:
      tl_runs_kernel<2><<<g, b, 0, st>>>((const u32*)x, n, flip, tkeys, tidx, log2s, first, runs, ac);
      break;
    default:
      tl_runs_kernel<0><<<g, b, 0, st>>>((const u64*)x, n, flip, tkeys, tidx, log2s, first, runs, ac);
  }
}

void launch_tel_comp(const u64* keys, u64 np, const u32* first, u64 mult, int m_log2, int dom,
                     u64* comp, u64* cidx, int num_sms, cudaStream_t st) {
  u64 blocks = (np + 255) / 256;
  if (blocks > (u64)num_sms * 8) blocks = (u64)num_sms * 8;
  tl_comp_kernel<<<(unsigned)(blocks ? blocks : 1), 256, 0, st>>>(keys, np, first, mult, m_log2,
                                                                  dom, comp, cidx);
}

void launch_tel_classify(const u64* comp, const u64* cidx, u64 np, int cap, const u64* counts,
                         const u32* runs, void* acc, int num_sms, cudaStream_t st) {
  u64 blocks = (np + 255) / 256;
  if (blocks > (u64)num_sms * 8) blocks = (u64)num_sms * 8;
  tl_classify_kernel<<<(unsigned)(blocks ? blocks : 1), 256, 0, st>>>(comp, cidx, np, cap, counts,
                                                                      runs, (TelAccum*)acc);
}

}  // namespace cafs
