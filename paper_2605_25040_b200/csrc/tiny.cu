// tiny.cu -- K2: one-pass count of x against the <= 8 sampled keys.
//
// Replaces _kernels.tiny_counts (_kernels.py:156-169) and the TINY branch of
// cafs_sort (sorter.py:367-385).  The reference compares every element with
// every key (the paper's cmpeq/movemask/tzcnt bucket).  On
// B200 that is 8 x 64-bit compares per element -- more ALU issue than the
// HBM stream leaves room for -- so the keys are placed by a perfect
// multiplicative hash (found by the estimate kernel) into 16 slots: each
// element costs one multiply, one broadcast-free shared-memory key probe
// (16 x 8 B = 128 B spans the 32 banks exactly) and one add into a
// lane-private shared counter (counter[warp][slot][lane]: bank == lane, no
// atomics, no conflicts).  An element whose probed key differs is a miss; any
// miss means the sample missed a value and the caller re-enters the main route
// with the same k_hat, exactly as sorter.py:378-385.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr int kTinyThreads = 512;
constexpr int kTinyWarps = kTinyThreads / 32;

// Success check (sum == n <=> no miss) and the <= 8 sorted pairs + offsets;
// run by one thread of the count's last CTA (the counters are read from L2).
__device__ void tiny_finalize(DevCtl* ctl, u64 n, u64* pkeys, u64* pcnt, u64* poffs) {
  if (__ldcg(&ctl->tiny_miss) != 0) {
    ctl->pairs_ready = 0;
    ctl->tiny_failed = 1;
    return;
  }
  const int nk = ctl->nkeys;
  u64 off = 0;
  for (int j = 0; j < nk; ++j) {
    const u64 c = __ldcg(&ctl->tiny_counts[ctl->tiny_slot[j]]);
    pkeys[j] = ctl->keys[j];
    pcnt[j] = c;
    poffs[j] = off;
    off += c;
  }
  poffs[nk] = off;
  ctl->npairs = nk;
  ctl->total = off;
  ctl->sum_error = (off != n);
  ctl->pairs_ready = (off == n);
}

template <int KK>
__global__ void __launch_bounds__(kTinyThreads, 4)  // 2048 threads per SM: more loads in flight
    tiny_count_kernel(const typename KeyT<KK>::T* __restrict__ x, u64 n, u64 flip, DevCtl* ctl,
                      int gate, u64* pkeys, u64* pcnt, u64* poffs) {
  pdl_begin();
  using K = typename KeyT<KK>::T;
  constexpr int KPV = 16 / sizeof(K);  // keys per 16-byte vector
  if (!gate_open(ctl, gate)) return;
  __shared__ u64 skey[16];
  __shared__ u32 cnt[kTinyWarps][16][32];
  __shared__ u64 wmiss[kTinyWarps];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const u64 mult = ctl->tiny_mult;
  const int nk = ctl->nkeys;
  if (tid < 16) {
    u64 k = ctl->keys[0];  // never hashes to an empty slot, so it can stand in
    for (int j = 0; j < nk; ++j)
      if (ctl->tiny_slot[j] == tid) k = ctl->keys[j];
    skey[tid] = k;
  }
  for (int i = lane; i < 16 * 32; i += 32) (&cnt[wid][0][0])[i] = 0;
  __syncthreads();

  u32* mycnt = &cnt[wid][0][lane];
  u64 miss = 0;
  auto count1 = [&](K raw) {
    const u64 v = key_map<KK>(raw, flip);
    const u32 sl = (u32)((v * mult) >> 60);
    const u32 eq = (skey[sl] == v);
    mycnt[sl * 32] += eq;
    miss += 1u - eq;
  };

  // a 16-byte vector's keys
  auto count_vec = [&](ulonglong2 w) {
    if constexpr (KPV == 2) {
      count1(w.x); count1(w.y);
    } else {
      count1((u32)w.x); count1((u32)(w.x >> 32)); count1((u32)w.y); count1((u32)(w.y >> 32));
    }
  };
  // 16-byte aligned body, scalar head/tail (x may be an element-aligned view)
  const u64 mis = (((uintptr_t)x) & 15) / sizeof(K);
  const u64 head0 = mis ? (u64)KPV - mis : 0;
  const u64 head = head0 < n ? head0 : n;
  const u64 nb = (n - head) / KPV;  // 16-byte vectors in the body
  const ulonglong2* xv = (const ulonglong2*)(x + head);
  const u64 gtid = blockIdx.x * (u64)blockDim.x + tid;
  const u64 gstride = (u64)gridDim.x * blockDim.x;
  u64 i = gtid;
  for (; i + 3 * gstride < nb; i += 4 * gstride) {
    ulonglong2 a = ld_stream_v2(xv + i);
    ulonglong2 b = ld_stream_v2(xv + i + gstride);
    ulonglong2 c = ld_stream_v2(xv + i + 2 * gstride);
    ulonglong2 d = ld_stream_v2(xv + i + 3 * gstride);
    count_vec(a); count_vec(b); count_vec(c); count_vec(d);
  }
  for (; i < nb; i += gstride) count_vec(ld_stream_v2(xv + i));
  if (gtid < head) count1(x[gtid]);  // head keys
  const u64 tail0 = head + nb * KPV;
  if (gtid < n - tail0) count1(x[tail0 + gtid]);  // tail keys
  // ---- reduce: per slot over warps and lanes ----
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) miss += __shfl_xor_sync(0xffffffffu, miss, o);
  if (lane == 0) wmiss[wid] = miss;
  __syncthreads();
  if (wid < 16) {  // warp `wid` reduces slot `wid`
    u64 sum = 0;
    for (int w = 0; w < kTinyWarps; ++w) sum += cnt[w][wid][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0 && sum) atomicAdd(&ctl->tiny_counts[wid], sum);
  }
  if (tid == 0) {
    u64 m = 0;
    for (int w = 0; w < kTinyWarps; ++w) m += wmiss[w];
    if (m) atomicAdd(&ctl->tiny_miss, m);
  }
  if (pkeys) {  // the last CTA to finish runs the finalize (no separate launch)
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (tid == 0) last = atomicAdd(&ctl->tiny_done, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last && tid == 0) {
      __threadfence();
      tiny_finalize(ctl, n, pkeys, pcnt, poffs);
      ctl->tiny_done = 0;
    }
  }
}

void launch_tiny_count(const void* x, u64 n, u64 flip, DevCtl* ctl, int num_sms,
                       cudaStream_t st, int gate, int kk, u64* pkeys, u64* pcnt, u64* poffs) {
  const u64 kpv = kk ? 4 : 2;
  u64 blocks = (n / kpv + kTinyThreads * 8 - 1) / (kTinyThreads * 8);
  u64 maxb = (u64)num_sms * 4;
  if (blocks > maxb) blocks = maxb;
  if (blocks < 1) blocks = 1;
  const unsigned g = (unsigned)blocks;
  switch (kk) {
    case 1:
      launch_pdl(kPdlTiny, tiny_count_kernel<1>, g, kTinyThreads, 0, st, (const u32*)x, n, flip, ctl, gate,
                 pkeys, pcnt, poffs);
      break;
    case 2:
      launch_pdl(kPdlTiny, tiny_count_kernel<2>, g, kTinyThreads, 0, st, (const u32*)x, n, flip, ctl, gate,
                 pkeys, pcnt, poffs);
      break;
    default:
      launch_pdl(kPdlTiny, tiny_count_kernel<0>, g, kTinyThreads, 0, st, (const u64*)x, n, flip, ctl, gate,
                 pkeys, pcnt, poffs);
  }
}

}  // namespace cafs
