// Shared device/host helpers for the nmg library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "nmg kernels are written for sm_100a only"
#endif

#define NMG_HD __host__ __device__ __forceinline__
#define NMG_D __device__ __forceinline__

namespace nmg {

constexpr int kWarp = 32;

NMG_HD int ceil_div(int a, int b) { return (a + b - 1) / b; }
NMG_HD int64_t ceil_div64(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Deterministic block-wide sum of one double per thread (fixed tree; blockDim.x a
// multiple of 32, <= 1024).  All threads receive the total.
NMG_D double block_sum_f64(double v, double* scratch /* >= 32 doubles */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  const int nw = blockDim.x >> 5;
  double t = (lane < nw) ? scratch[lane] : 0.0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  return t;
}

// 2D level-filter input, paired layout: right-hand sides 2p and 2p + 1 are the real and the
// imaginary part of complex image p (F' is a real symmetric operator, so one complex 2D FFT
// filters both, see filter2d).  N = n * n pixels per image.
NMG_D void zput(float2* Z, int64_t N, int b, int64_t pix, float v) {
  reinterpret_cast<float*>(Z)[((int64_t)(b >> 1) * N + pix) * 2 + (b & 1)] = v;
}

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is a per-DEVICE property: set it once per
// (call site, device).  `done` is the call site's bitmask of devices already configured (a
// concurrent double set is harmless: the call is idempotent).
inline cudaError_t smem_optin(const void* fn, int bytes, std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_acquire) & bit) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.fetch_or(bit, std::memory_order_acq_rel);
  return e;
}
#define NMG_SMEM_OPTIN(fn, bytes)                                         \
  do {                                                                    \
    static std::atomic<uint64_t> nmg_optin_done_{0};                      \
    ::nmg::smem_optin((const void*)(fn), (int)(bytes), nmg_optin_done_); \
  } while (0)

}  // namespace nmg
