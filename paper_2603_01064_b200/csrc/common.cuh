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

// 2D level-filter input, per-RHS packing: rows 2r and 2r + 1 of RHS b's image (`rows` x n real
// values, rows even) are the real and the imaginary part of complex row r of its spectrum
// buffer Z_b = [rows / 2][n] complex (one real 2D DFT done as n/2 complex row FFTs plus a
// Hermitian unmixing in the column pass, see level2d.cu).  Each RHS keeps its own buffer, so
// right-hand sides never share a transform (per-RHS independence, SURVEY pin P14).
NMG_D void zput(float2* Z, int rows, int n, int b, int y, int x, float v) {
  reinterpret_cast<float*>(Z)[(int64_t)b * rows * n + (int64_t)(y >> 1) * 2 * n + 2 * x + (y & 1)] = v;
}

// 2D CNN output h(y, x) = b3 + Q0(x - 1) + Q1(x) + Q2(x + 1) (conv_strip.cu): the strip kernel
// stores v = the sum without the terms that cross its 128-pixel strip boundary and, per (image
// row, strip), the edge record E = {Q2(X0), Q0(X0 + 127), Q2(X0 + 1)}; this completes pixel x of
// a row whose records start at E (the same additions in the same order as a whole-row sum)
constexpr int kStripSeg = 128;
NMG_D float strip_h_fix(float v, const float4* __restrict__ E, int n, int x) {
  if (n < kStripSeg) return v;
  const int m = x & (kStripSeg - 1), st = x / kStripSeg;
  if (m == 0 && x > 0) return (v + __ldg(&E[st - 1].y)) + __ldg(&E[st].z);
  if (m == kStripSeg - 1 && x < n - 1) return v + __ldg(&E[st + 1].x);
  return v;
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
