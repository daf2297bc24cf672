// Microbenchmarks to choose the hash-count design (scratch; not product code).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); exit(1);} } while (0)
typedef unsigned long long u64;
typedef unsigned int u32;

__device__ __forceinline__ u64 fmix(u64 z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gen(u64* x, u64 n, u32 K, int skew) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += (u64)gridDim.x * blockDim.x) {
    u64 r = fmix(12345 + (i + 1) * 0x9E3779B97F4A7C15ull);
    u64 idx;
    if (skew) { double u = (r >> 11) * (1.0 / 9007199254740992.0); idx = (u64)(K * u * u * u); if (idx >= K) idx = K - 1; }
    else idx = __umul64hi(r, K);
    x[i] = fmix(777 + (idx + 1) * 0x9E3779B97F4A7C15ull);
  }
}

__global__ void stream_read(const ulonglong2* __restrict__ x, u64 n2, u64* out) {
  u64 acc = 0;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n2; i += (u64)gridDim.x * blockDim.x) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(x + i));
    acc ^= v.x + v.y;
  }
  if (acc == 0x1234567) out[0] = acc;
}

__global__ void stream_copy(const ulonglong2* __restrict__ x, ulonglong2* __restrict__ y, u64 n2) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n2; i += (u64)gridDim.x * blockDim.x) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(x + i));
    y[i] = v;
  }
}

__global__ void stream_write(ulonglong2* __restrict__ y, u64 n2) {
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n2; i += (u64)gridDim.x * blockDim.x) {
    y[i] = make_ulonglong2(i, i);
  }
}

constexpr u64 EMPTY = ~0ull;
constexpr u64 MULT = 0x9E3779B97F4A7C15ull;

// MODE 0: atomicAdd per element; 1: match_any aggregated; 2: plain (racy) add; 3: probe only
template <int LOG2S, int MODE>
__global__ void __launch_bounds__(512) hcount(const ulonglong2* __restrict__ x, u64 n2, u64* gout, u32* miss) {
  constexpr int S = 1 << LOG2S;
  extern __shared__ __align__(16) unsigned char sm[];
  u64* sk = (u64*)sm;
  u32* sc = (u32*)(sm + S * 8);
  for (int i = threadIdx.x; i < S; i += blockDim.x) { sk[i] = EMPTY; sc[i] = 0; }
  __syncthreads();
  u32 lmiss = 0;
  const int lane = threadIdx.x & 31;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n2; i += (u64)gridDim.x * blockDim.x) {
    ulonglong2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.u64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "l"(x + i));
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      u64 key = e ? v.y : v.x;
      u32 h = (u32)((key * MULT) >> (64 - LOG2S));
      int slot = -1;
#pragma unroll 1
      for (int p = 0; p < 16; ++p) {
        u64 k = sk[h];
        if (k == key) { slot = h; break; }
        if (k == EMPTY) {
          u64 old = atomicCAS(&sk[h], EMPTY, key);
          if (old == EMPTY || old == key) { slot = h; break; }
        }
        h = (h + 1) & (S - 1);
      }
      if (MODE == 0) { if (slot >= 0) atomicAdd(&sc[slot], 1u); else lmiss++; }
      else if (MODE == 1) {
        u32 grp = __match_any_sync(0xffffffffu, key);
        int leader = __ffs(grp) - 1;
        if (lane == leader) { if (slot >= 0) atomicAdd(&sc[slot], (u32)__popc(grp)); else lmiss += __popc(grp); }
      } else if (MODE == 2) { if (slot >= 0) sc[slot] += 1; else lmiss++; }
      else { if (slot < 0) lmiss++; else lmiss += (slot == 77777); }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < S; i += blockDim.x) if (sc[i]) atomicAdd(&gout[i], (u64)sc[i]);
  if (lmiss) atomicAdd(miss, lmiss);
}

// pure smem atomics throughput
__global__ void __launch_bounds__(512) atoms_pure(u32* out, int iters, int spread) {
  __shared__ u32 t[8192];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) t[i] = 0;
  __syncthreads();
  u32 h = threadIdx.x * 2654435761u + blockIdx.x;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    u32 a = spread ? (h >> 19) : (threadIdx.x & 31) * 1;
    atomicAdd(&t[a], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t[5];
}

__global__ void __launch_bounds__(512) lds_pure(u32* out, int iters) {
  __shared__ u64 t[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) t[i] = i;
  __syncthreads();
  u32 h = threadIdx.x * 2654435761u + blockIdx.x;
  u64 acc = 0;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    acc += t[(h >> 20)];
  }
  if (acc == 12345) out[blockIdx.x] = (u32)acc;
}

__global__ void __launch_bounds__(512) match_pure(u32* out, int iters) {
  u32 h = threadIdx.x * 2654435761u + blockIdx.x;
  u32 acc = 0;
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    u64 key = (u64)(h >> 20) * 0x100000001ull;
    acc += __match_any_sync(0xffffffffu, key);
  }
  if (acc == 12345) out[blockIdx.x] = acc;
}

__global__ void gatomic(u64* tbl, u32 logsz, u64 n, int iters) {
  u64 h = blockIdx.x * (u64)blockDim.x + threadIdx.x;
  for (int it = 0; it < iters; ++it) {
    u64 r = fmix(h * 1000003 + it);
    atomicAdd(&tbl[r >> (64 - logsz)], 1ull);
  }
}

int main() {
  int dev = 0; CK(cudaSetDevice(dev));
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  const int SMS = prop.multiProcessorCount;
  const u64 n = 1ull << 30;
  u64 *x, *y, *gout; u32* miss; u32* o32;
  CK(cudaMalloc(&x, n * 8)); CK(cudaMalloc(&y, n * 8)); CK(cudaMalloc(&gout, 1 << 20)); CK(cudaMalloc(&miss, 4)); CK(cudaMalloc(&o32, 1 << 16));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  auto timeit = [&](auto fn, int reps) {
    fn(); CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int r = 0; r < reps; ++r) { cudaEventRecord(a); fn(); cudaEventRecord(b); CK(cudaEventSynchronize(b)); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
    CK(cudaGetLastError());
    return best;
  };
  for (int blocks_per_sm : {2, 4, 8}) {
    float ms = timeit([&] { stream_read<<<SMS * blocks_per_sm, 512>>>((ulonglong2*)x, n / 2, gout); }, 5);
    printf("stream_read bps=%d: %.3f ms  %.1f GB/s\n", blocks_per_sm, ms, n * 8 / ms / 1e6);
    ms = timeit([&] { stream_copy<<<SMS * blocks_per_sm, 512>>>((ulonglong2*)x, (ulonglong2*)y, n / 2); }, 5);
    printf("stream_copy bps=%d: %.3f ms  %.1f GB/s (r+w)\n", blocks_per_sm, ms, n * 16 / ms / 1e6);
    ms = timeit([&] { stream_write<<<SMS * blocks_per_sm, 512>>>((ulonglong2*)y, n / 2); }, 5);
    printf("stream_write bps=%d: %.3f ms  %.1f GB/s\n", blocks_per_sm, ms, n * 8 / ms / 1e6);
  }
  for (int iters : {4096}) {
    float ms = timeit([&] { atoms_pure<<<SMS * 4, 512>>>(o32, iters, 1); }, 3);
    double ops = (double)SMS * 4 * 512 * iters;
    printf("atoms spread: %.3f ms  %.2f lane-atomics/clk/SM (@1.9GHz)\n", ms, ops / (ms * 1e-3) / SMS / 1.9e9);
    ms = timeit([&] { atoms_pure<<<SMS * 4, 512>>>(o32, iters, 0); }, 3);
    printf("atoms lane-distinct (bank=lane): %.3f ms  %.2f lane-atomics/clk/SM\n", ms, ops / (ms * 1e-3) / SMS / 1.9e9);
    ms = timeit([&] { lds_pure<<<SMS * 4, 512>>>(o32, iters); }, 3);
    printf("lds64 random: %.3f ms  %.2f lane-loads/clk/SM\n", ms, ops / (ms * 1e-3) / SMS / 1.9e9);
    ms = timeit([&] { match_pure<<<SMS * 4, 512>>>(o32, iters); }, 3);
    printf("match_any u64: %.3f ms  %.2f lane-ops/clk/SM\n", ms, ops / (ms * 1e-3) / SMS / 1.9e9);
  }
  {
    u64* tbl; CK(cudaMalloc(&tbl, (1ull << 22) * 8)); CK(cudaMemset(tbl, 0, (1ull << 22) * 8));
    int iters = 64; u64 threads = (u64)SMS * 8 * 512;
    float ms = timeit([&] { gatomic<<<SMS * 8, 512>>>(tbl, 22, 0, iters); }, 3);
    printf("global atomics 4M-slot: %.3f ms  %.2f G atomics/s\n", ms, threads * iters / (ms * 1e-3) / 1e9);
    ms = timeit([&] { gatomic<<<SMS * 8, 512>>>(tbl, 16, 0, iters); }, 3);
    printf("global atomics 64k-slot: %.3f ms  %.2f G atomics/s\n", ms, threads * iters / (ms * 1e-3) / 1e9);
  }
  for (int skew : {0, 1}) for (u32 K : {200u, 4096u}) {
    gen<<<SMS * 8, 512>>>(x, n, K, skew); CK(cudaDeviceSynchronize());
    auto run = [&](auto kern, int log2s, const char* name) {
      size_t smem = (size_t(1) << log2s) * 12;
      CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      for (int threads : {256, 512}) {
        int occ = 0; CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, threads, smem));
        CK(cudaMemset(gout, 0, 1 << 20)); CK(cudaMemset(miss, 0, 4));
        float ms = timeit([&] { kern<<<SMS * occ, threads, smem>>>((ulonglong2*)x, n / 2, gout, miss); }, 3);
        u32 hm; CK(cudaMemcpy(&hm, miss, 4, cudaMemcpyDeviceToHost));
        printf("K=%u skew=%d %s S=2^%d thr=%d occ=%d: %.3f ms  %.1f Gkeys/s  %.1f GB/s read  miss=%u\n", K, skew, name, log2s, threads, occ, ms, n / ms / 1e6, n * 8 / ms / 1e6, hm);
      }
    };
    run(hcount<13, 0>, 13, "atomic");
    run(hcount<13, 1>, 13, "match ");
    run(hcount<13, 2>, 13, "racy  ");
    run(hcount<13, 3>, 13, "probe ");
    run(hcount<14, 0>, 14, "atomic");
  }
  return 0;
}
