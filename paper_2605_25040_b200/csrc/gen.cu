// gen.cu -- synthetic inputs for the BASELINE configs, generated in HBM.
//
// Bit-identical to oracle/gen.py (the numpy restatement): the counter-based
// SplitMix stream of the reference's datagen.py:26-53,
//   r(seed, i) = fmix64(seed + (i + 1) * 0x9E3779B97F4A7C15),
// uniform draws by multiply-high (datagen.py:88-92) and Zipf draws by
// searchsorted(cdf, u, 'right') over a float64 CDF uploaded from the host.
// Row i of a config depends only on i, so each GPU generates its own shard.
#include "common.cuh"
#include "kernels.cuh"

namespace cafs {

constexpr u64 kElXor = 0xD1B54A32D192ED03ull;

__global__ void gen_mix_kernel(u64* out, u64 count, u64 seed, u64 skip) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < count; i += stride)
    out[i] = fmix64(seed + (skip + i + 1) * kGamma);
}

__global__ void gen_draw_kernel(u64* out, u64 n, u64 start, u64 seed, const u64* palette, u64 k,
                                const double* cdf) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  const u64 s = seed ^ kElXor;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride) {
    const u64 r = fmix64(s + (start + i + 1) * kGamma);
    u64 idx;
    if (cdf) {
      const double u = __dmul_rn((double)(r >> 11), 1.0 / 9007199254740992.0);
      u64 lo = 0, hi = k;  // count of cdf[j] <= u
      while (lo < hi) {
        const u64 mid = (lo + hi) >> 1;
        if (cdf[mid] <= u) lo = mid + 1; else hi = mid;
      }
      idx = lo;
    } else {
      idx = __umul64hi(r, k);
    }
    out[i] = palette ? palette[idx] : idx;
  }
}

void launch_gen_mix(u64* out, u64 count, u64 seed, u64 skip, int num_sms, cudaStream_t st) {
  gen_mix_kernel<<<num_sms * 8, 256, 0, st>>>(out, count, seed, skip);
}

void launch_gen_draw(u64* out, u64 n, u64 start, u64 seed, const u64* palette, u64 k,
                     const double* cdf, int num_sms, cudaStream_t st) {
  gen_draw_kernel<<<num_sms * 8, 256, 0, st>>>(out, n, start, seed, palette, k, cdf);
}

// 32-bit keys <-> their int64 widening (value-preserving: int32 sign-extends,
// uint32 zero-extends), for the routes that run on a 64-bit copy
__global__ void widen_kernel(const void* __restrict__ x, u64 n, int kk, u64* __restrict__ out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride) {
    const u32 v = ((const u32*)x)[i];
    out[i] = kk == 1 ? (u64)(long long)(int)v : (u64)v;
  }
}
__global__ void narrow_kernel(const u64* __restrict__ x, u64 n, void* __restrict__ out) {
  const u64 stride = (u64)gridDim.x * blockDim.x;
  for (u64 i = blockIdx.x * (u64)blockDim.x + threadIdx.x; i < n; i += stride)
    ((u32*)out)[i] = (u32)x[i];
}
void launch_widen(const void* x, u64 n, int kk, u64* out, int num_sms, cudaStream_t st) {
  if (n) widen_kernel<<<num_sms * 8, 512, 0, st>>>(x, n, kk, out);
}
void launch_narrow(const u64* x, u64 n, int kk, void* out, int num_sms, cudaStream_t st) {
  (void)kk;
  if (n) narrow_kernel<<<num_sms * 8, 512, 0, st>>>(x, n, out);
}

}  // namespace cafs
