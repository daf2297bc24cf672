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

__global__ void __launch_bounds__(kTinyThreads)
    tiny_count_kernel(const u64* __restrict__ x, u64 n, u64 flip, DevCtl* ctl, int gate) {
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
  auto count1 = [&](u64 raw) {
    const u64 v = raw ^ flip;
    const u32 sl = (u32)((v * mult) >> 60);
    const u32 eq = (skey[sl] == v);
    mycnt[sl * 32] += eq;
    miss += 1u - eq;
  };

  // 16-byte aligned body, scalar head/tail (x may be an 8-byte aligned view)
  const u64 head = (((uintptr_t)x) & 15) ? 1 : 0;
  const u64 nb = n > head ? (n - head) / 2 : 0;  // 16-byte vectors in the body
  const ulonglong2* xv = (const ulonglong2*)(x + head);
  const u64 gtid = blockIdx.x * (u64)blockDim.x + tid;
  const u64 gstride = (u64)gridDim.x * blockDim.x;
  u64 i = gtid;
  for (; i + 3 * gstride < nb; i += 4 * gstride) {
    ulonglong2 a = ld_stream_v2(xv + i);
    ulonglong2 b = ld_stream_v2(xv + i + gstride);
    ulonglong2 c = ld_stream_v2(xv + i + 2 * gstride);
    ulonglong2 d = ld_stream_v2(xv + i + 3 * gstride);
    count1(a.x); count1(a.y); count1(b.x); count1(b.y);
    count1(c.x); count1(c.y); count1(d.x); count1(d.y);
  }
  for (; i < nb; i += gstride) {
    ulonglong2 a = ld_stream_v2(xv + i);
    count1(a.x); count1(a.y);
  }
  if (gtid == 0) {
    if (head && n > 0) count1(x[0]);
    if (n > head && ((n - head) & 1)) count1(x[n - 1]);
  }
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
}

// Success check (sum == n <=> no miss) and the <= 8 sorted pairs + offsets.
__global__ void tiny_finalize_kernel(DevCtl* ctl, u64 n, u64* pkeys, u64* pcnt, u64* poffs,
                                     int gate) {
  if (threadIdx.x != 0 || !gate_open(ctl, gate)) return;
  if (ctl->tiny_miss != 0) {
    ctl->pairs_ready = 0;
    ctl->tiny_failed = 1;
    return;
  }
  const int nk = ctl->nkeys;
  u64 off = 0;
  for (int j = 0; j < nk; ++j) {
    const u64 c = ctl->tiny_counts[ctl->tiny_slot[j]];
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

void launch_tiny_count(const u64* x, u64 n, u64 flip, DevCtl* ctl, int num_sms,
                       cudaStream_t st, int gate) {
  u64 blocks = (n / 2 + kTinyThreads * 8 - 1) / (kTinyThreads * 8);
  u64 maxb = (u64)num_sms * 4;
  if (blocks > maxb) blocks = maxb;
  if (blocks < 1) blocks = 1;
  tiny_count_kernel<<<(unsigned)blocks, kTinyThreads, 0, st>>>(x, n, flip, ctl, gate);
}

void launch_tiny_finalize(DevCtl* ctl, u64 n, u64* pkeys, u64* pcnt, u64* poffs,
                          cudaStream_t st, int gate) {
  tiny_finalize_kernel<<<1, 32, 0, st>>>(ctl, n, pkeys, pcnt, poffs, gate);
}

}  // namespace cafs
