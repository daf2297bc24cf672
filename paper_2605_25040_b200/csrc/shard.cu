// shard.cu -- kernels of the stream-ordered sharded pipeline (abi.cu:
// cafs_shard_*).  One process per GPU holds a row shard of the column; the
// reference is single-process (the paper leaves a parallel CAFS as future
// work).  Every decision the host would otherwise make between
// collectives is taken on device from all-gathered data, so a rank enqueues
//   header -> all-gather -> samples -> all-reduce -> estimate + local count ->
//   all-reduce (tiny counts) + all-gather (pair tables) -> merge -> slice emit
// and synchronises once.  The dispatch is the reference's (sorter.py:141-162)
// evaluated on the GLOBAL column: N and the monotone test come from the shard
// headers, the 1024 strided samples from the shards that hold their positions.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

// Header of this shard (kShardHdrWords words): rows, monotone state of the
// first kMonoPrefix rows (0 inversion, 1 sorted, 2 sorted prefix of a longer
// shard -> word 4 holds the full scan's verdict), first and last key.
template <int KK>
__global__ void __launch_bounds__(1024) shard_header_kernel(const typename KeyT<KK>::T* __restrict__ x,
                                                            u64 n, u64 flip, u64* hdr) {
  __shared__ int inv;
  if (threadIdx.x == 0) inv = 0;
  __syncthreads();
  const u64 P = n < kMonoPrefix ? n : kMonoPrefix;
  // thread t checks rows [16t, 16t + 16]: 17 loads in flight at once (one
  // DRAM round trip for the reference's first chunk, not 16)
  const u64 i0 = (u64)threadIdx.x * 16;
  // (thread 0's first / last key ride in the same round trip)
  u64 kfirst = 0, klast = 0;
  if (threadIdx.x == 0 && n) {
    kfirst = key_map<KK>(x[0], flip);
    klast = key_map<KK>(x[n - 1], flip);
  }
  u64 a[17];
#pragma unroll
  for (int j = 0; j < 17; ++j) a[j] = i0 + j < P ? key_map<KK>(x[i0 + j], flip) : 0;
  int found = 0;
#pragma unroll
  for (int j = 0; j < 16; ++j) found |= (i0 + j + 1 < P) && a[j + 1] < a[j];
  if (found) inv = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    hdr[0] = n;
    hdr[1] = n <= 1 ? 1 : (inv ? 0 : (n <= kMonoPrefix ? 1 : 2));
    hdr[2] = kfirst;
    hdr[3] = klast;
    hdr[4] = 0;
    hdr[5] = hdr[6] = hdr[7] = 0;
  }
}

// The rest of a shard whose prefix is sorted (state 2): any inversion -> word 4.
template <int KK>
__global__ void shard_scan_kernel(const typename KeyT<KK>::T* __restrict__ x, u64 n, u64 flip,
                                  u64* hdr) {
  pdl_begin();
  if (hdr[1] != 2) return;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  int found = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i + 1 < n; i += stride)
    found |= key_map<KK>(x[i + 1], flip) < key_map<KK>(x[i], flip);
  if (found) hdr[4] = 1;
}

// The global sample positions i * (N // 1024) (cardinality.py:102-104) that
// fall in this shard; zeros elsewhere, so an all-reduce SUM assembles the
// sample.  Also records this rank's slice of the sorted output.
template <int KK>
__global__ void __launch_bounds__(1024) shard_samples_kernel(const typename KeyT<KK>::T* __restrict__ x,
                                                             u64 n, u64 flip, const u64* ghdr, int world,
                                                             int rank, u64* samples,
                                                             DevCtl* ctl) {
  u64 N = 0, off = 0;
  for (int r = 0; r < world; ++r) {
    const u64 nr = ghdr[r * kShardHdrWords];
    if (r < rank) off += nr;
    N += nr;
  }
  const u64 i = threadIdx.x;
  u64 stride = N / kSampleTarget;
  if (stride < 1) stride = 1;
  const u64 m = N < (u64)kSampleTarget ? N : (u64)kSampleTarget;
  const u64 pos = i * stride;
  u64 v = 0;
  if (i < m && pos >= off && pos < off + n) v = key_map<KK>(x[pos - off], flip);
  samples[i] = v;
  if (threadIdx.x == 0) {
    ctl->slice[0] = off;
    ctl->slice[1] = off + n;
  }
}

// Local tiny counts (per perfect-hash slot) and misses, for the all-reduce.
__global__ void shard_tiny_pack_kernel(const DevCtl* ctl, u64* out) {
  const int t = threadIdx.x;
  if (t < 16) out[t] = ctl->tiny_counts[t];
  if (t == 16) out[16] = ctl->tiny_miss;
}

// This rank's sorted (key, count) table for the all-gather: [np, keys[cap],
// counts[cap]]; np = ~0 when the pairs are lost or unsorted (table overflow);
// np > cap: sorted, but too many for this exchange row (the pairs are not
// sent; the caller may grow the row and exchange again, from_local).
__global__ void shard_pack_pairs_kernel(DevCtl* ctl, const u64* keys, const u64* cnts,
                                        u64* send, u64 cap, int from_local) {
  const bool main = gate_open(ctl, kGateMain);
  bool sorted;
  u64 np;
  if (from_local) {  // a second exchange: the count's state was saved by the first
    sorted = ctl->local_sorted && !ctl->local_overflow;
    np = ctl->local_npairs;
  } else {
    sorted = main && !ctl->overflow && !ctl->hp_overflow && ctl->pairs_ready;
    np = ctl->npairs;
  }
  const bool ok = main && sorted && np <= cap;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    send[0] = main ? (sorted ? np : ~0ull) : 0ull;
    if (!from_local) {
      ctl->local_npairs = main ? ctl->npairs : 0;
      ctl->local_sorted = main && ctl->pairs_ready && !ctl->hp_overflow;
      ctl->local_overflow = main && (ctl->overflow || ctl->hp_overflow);
      ctl->local_hp = main && ctl->hp_ok && ctl->range_len == 0;
    }
  }
  if (!ok) return;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < np; j += stride) {
    send[1 + j] = keys[j];
    send[1 + cap + j] = cnts[j];
  }
}

// Tiny route on the all-reduced counts: the keys' global counts must sum to N
// and no rank may have seen another value (sorter.py:367-385); else the
// caller re-runs the column on the host-driven path.
__global__ void shard_tiny_finish_kernel(DevCtl* ctl, const u64* tiny_sum, u64* pkeys, u64* pcnt,
                                         u64* poffs) {
  if (threadIdx.x != 0 || !gate_open(ctl, kGateTiny)) return;
  const u64 N = ctl->n_global;
  const int nk = ctl->nkeys;
  u64 off = 0;
  for (int j = 0; j < nk; ++j) {
    const u64 c = tiny_sum[ctl->tiny_slot[j]];
    pkeys[j] = ctl->keys[j];
    pcnt[j] = c;
    poffs[j] = off;
    off += c;
  }
  poffs[nk] = off;
  const bool ok = tiny_sum[16] == 0 && off == N;
  ctl->npairs = nk;
  ctl->total = off;
  ctl->pairs_ready = ok;
  ctl->tiny_failed = !ok;
}

// Merge: the union of every rank's table (sorter.py:276-285) in the global
// table -- reset its per-call counters first; a rank that could not exchange
// its table (np = ~0) or a local overflow skips the merge on this rank (the
// caller then takes the host-driven path on all ranks: every rank sees the same
// gathered np values).
__global__ void shard_merge_reset_kernel(DevCtl* ctl, const u64* recv, int world, u64 row) {
  if (!gate_open(ctl, kGateMain)) return;
  __shared__ int bad;
  if (threadIdx.x == 0) bad = ctl->overflow;
  __syncthreads();
  for (int r = threadIdx.x; r < world; r += blockDim.x)
    if (recv[(u64)r * row] == ~0ull) bad = 1;
  for (u32 t = threadIdx.x; t < kListStripes; t += blockDim.x) ctl->g_fill[t] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl->npairs = 0;
    ctl->total = 0;
    ctl->pairs_ready = 0;
    ctl->sum_error = 0;
    ctl->need_large = 0;
    ctl->empty_key_count = 0;
    ctl->overflow = bad;  // gates the merge kernels below off
  }
}

// Before the sorted merge: reset the per-call merge state; a rank whose list
// is missing (np = ~0) or longer than the row (np > cap) gates the merge off
// on every rank (they all see the same rows); shard_grow = the longest list
// that did not fit, for the caller to grow the row.
__global__ void shard_merge_check_kernel(DevCtl* ctl, const u64* recv, int world, u64 cap, u64 row) {
  if (!gate_open(ctl, kGateMain)) return;
  __shared__ int bad;
  __shared__ unsigned long long grow;
  if (threadIdx.x == 0) { bad = 0; grow = 0; }
  __syncthreads();
  for (int r = threadIdx.x; r < world; r += blockDim.x) {
    const u64 np = recv[(u64)r * row];
    if (np == ~0ull || np > cap) atomicOr(&bad, 1);
    if (np != ~0ull && np > cap) atomicMax(&grow, (unsigned long long)np);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl->npairs = 0;
    ctl->total = 0;
    ctl->pairs_ready = 0;
    ctl->sum_error = 0;
    ctl->need_large = 0;
    ctl->merge_bad = bad;
    ctl->shard_grow = grow;
  }
}

void launch_shard_merge_check(DevCtl* ctl, const u64* recv, int world, u64 cap, u64 row,
                              cudaStream_t st) {
  shard_merge_check_kernel<<<1, 256, 0, st>>>(ctl, recv, world, cap, row);
}

__global__ void shard_merge_insert_kernel(DevCtl* ctl, const u64* recv, int world, u64 cap,
                                          u64 row, u64* gkeys, u64* gcnt, u32* glist) {
  if (!gate_open(ctl, kGateMain) || ctl->overflow) return;
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (int r = 0; r < world; ++r) {
    const u64* t = recv + (u64)r * row;
    const u64 np = t[0];
    for (u64 j = blockIdx.x * (u64)blockDim.x + threadIdx.x; j < np; j += stride) {
      const u64 k = t[1 + j], c = t[1 + cap + j];
      if (k == kEmpty) atomicAdd(&ctl->empty_key_count, c);
      else global_insert(gkeys, gcnt, glist, ctl, k, c, 0);
    }
  }
}

void launch_shard_header(const void* x, u64 n, u64 flip, u64* hdr, int num_sms, cudaStream_t st,
                         int kk) {
  if (kk == 1) {
    shard_header_kernel<1><<<1, 1024, 0, st>>>((const u32*)x, n, flip, hdr);
    launch_pdl(kPdlEstimate, shard_scan_kernel<1>, num_sms * 4, 512, 0, st, (const u32*)x, n, flip, hdr);
  } else if (kk == 2) {
    shard_header_kernel<2><<<1, 1024, 0, st>>>((const u32*)x, n, flip, hdr);
    launch_pdl(kPdlEstimate, shard_scan_kernel<2>, num_sms * 4, 512, 0, st, (const u32*)x, n, flip, hdr);
  } else {
    shard_header_kernel<0><<<1, 1024, 0, st>>>((const u64*)x, n, flip, hdr);
    launch_pdl(kPdlEstimate, shard_scan_kernel<0>, num_sms * 4, 512, 0, st, (const u64*)x, n, flip, hdr);
  }
}

void launch_shard_samples(const void* x, u64 n, u64 flip, const u64* ghdr, int world, int rank,
                          u64* samples, DevCtl* ctl, cudaStream_t st, int kk) {
  if (kk == 1)
    shard_samples_kernel<1><<<1, kSampleTarget, 0, st>>>((const u32*)x, n, flip, ghdr, world, rank,
                                                         samples, ctl);
  else if (kk == 2)
    shard_samples_kernel<2><<<1, kSampleTarget, 0, st>>>((const u32*)x, n, flip, ghdr, world, rank,
                                                         samples, ctl);
  else
    shard_samples_kernel<0><<<1, kSampleTarget, 0, st>>>((const u64*)x, n, flip, ghdr, world, rank,
                                                         samples, ctl);
}

void launch_shard_tiny_pack(const DevCtl* ctl, u64* out, cudaStream_t st) {
  shard_tiny_pack_kernel<<<1, 32, 0, st>>>(ctl, out);
}

void launch_shard_pack_pairs(DevCtl* ctl, const u64* keys, const u64* cnts, u64* send,
                             u64 cap, cudaStream_t st, int from_local) {
  const u64 g = cap / 8192 + 1;
  shard_pack_pairs_kernel<<<(unsigned)(g < 148 ? g : 148), 1024, 0, st>>>(ctl, keys, cnts, send,
                                                                          cap, from_local);
}

void launch_shard_tiny_finish(DevCtl* ctl, const u64* tiny_sum, u64* pkeys, u64* pcnt, u64* poffs,
                              cudaStream_t st) {
  shard_tiny_finish_kernel<<<1, 32, 0, st>>>(ctl, tiny_sum, pkeys, pcnt, poffs);
}

void launch_shard_merge(DevCtl* ctl, const u64* recv, int world, u64 cap, u64 row, u64* gkeys,
                        u64* gcnt, u32* glist, int num_sms, cudaStream_t st) {
  shard_merge_reset_kernel<<<1, 256, 0, st>>>(ctl, recv, world, row);
  shard_merge_insert_kernel<<<num_sms * 2, 256, 0, st>>>(ctl, recv, world, cap, row, gkeys, gcnt,
                                                         glist);
}

// The tiny counters every rank packed at `tiny_off` of its gathered row, summed
// (the native sharded path carries them in the pair-table all-gather instead
// of a separate all-reduce).
__global__ void shard_tiny_gather_kernel(const u64* recv, int world, u64 row, u64 tiny_off,
                                         u64* tiny_sum) {
  const int t = threadIdx.x;
  u64 s = 0;
  for (int r = 0; r < world; ++r) s += recv[(u64)r * row + tiny_off + t];
  tiny_sum[t] = s;
}

void launch_shard_tiny_gather(const u64* recv, int world, u64 row, u64 tiny_off, u64* tiny_sum,
                              cudaStream_t st) {
  shard_tiny_gather_kernel<<<1, CAFS_SHARD_TINY_WORDS, 0, st>>>(recv, world, row, tiny_off,
                                                                tiny_sum);
}

}  // namespace cafs
