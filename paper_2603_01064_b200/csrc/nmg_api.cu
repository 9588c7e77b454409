// C-ABI implementation: hierarchy construction (host fp64), device workspaces,
// and the NMGF cycle orchestration on one stream.
//
// Paper mapping (PAPER.md = P):
//   Galerkin chain  A^(l+1) = I_l^{l+1} A^(l) I_{l+1}^l        Alg 1, Alg 3
//   smoothing step  b = y - A x*, h = N(b/|b|)|b|, x = x*+F'(h)  Alg 3
//   restriction     y_{l+1} = I_l^{l+1}(y_l - A x)
//   correction      x += I_{l+1}^l NMGF(0, y_{l+1})
//   coarse          x_L = (A^(L))^{-1} y_L
//   outer loop      x^tau = NMGF(x^{tau-1}, y), relres <= tol
// Implementation choices that differ from a literal transcription:
//   * correction form x + NMGF(0, y - A x) with an fp64 outer residual (pin P11);
//   * the post-smoothing residual is b = r_l - (A_l P_l) e  (A_l P_l precomputed),
//     which equals y_l - A_l (x_l + P_l e) exactly and halves that GEMM.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>

#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/nmg.h"
#include "comm.h"
#include "kernels.h"

using namespace nmg;

namespace {

thread_local std::string g_err;

nmg_status fail(nmg_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

}  // namespace

nmg_status nmg::comm_fail(nmg_status st, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}

namespace {

#define NMG_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess) {                                                               \
      return fail(_e == cudaErrorMemoryAllocation ? NMG_ERR_OOM : NMG_ERR_CUDA, "%s: %s (%s:%d)", \
                  #expr, cudaGetErrorString(_e), __FILE__, __LINE__);                       \
    }                                                                                      \
  } while (0)

#define NMG_TRY(expr)                 \
  do {                                \
    nmg_status _s = (expr);           \
    if (_s != NMG_OK) return _s;      \
  } while (0)

template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  ~DevBuf() { if (p) cudaFree(p); }
  nmg_status alloc(size_t count) {
    if (p) { cudaFree(p); p = nullptr; }
    n = count;
    if (count == 0) return NMG_OK;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) return fail(NMG_ERR_OOM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
    return NMG_OK;
  }
  nmg_status upload(const T* h, size_t count) {
    NMG_TRY(alloc(count));
    NMG_CUDA(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice));
    return NMG_OK;
  }
};

// ---------------------------------------------------------------- host Ozaki digits
// rows of A (n x n, row-major): exponent e_r with max_k |a_rk| < 2^{e_r}, then S truncation
// digits of a 2^{-e_r} (ozaki.cu); dig [S][n][n]
void host_digits(const std::vector<double>& A, int n, int S, std::vector<int8_t>& dig, std::vector<int>& ew) {
  dig.assign((size_t)S * n * n, 0);
  ew.assign(n, 0);
  for (int r = 0; r < n; ++r) {
    double mx = 0.0;
    for (int k = 0; k < n; ++k) mx = std::max(mx, std::fabs(A[(size_t)r * n + k]));
    int e = 0;
    if (mx > 0.0) std::frexp(mx, &e);
    ew[r] = e;
    for (int k = 0; k < n; ++k) {
      double v = std::ldexp(A[(size_t)r * n + k], -e);
      for (int i = 0; i < S; ++i) {
        v *= 128.0;
        const double dg = std::trunc(v);
        v -= dg;
        dig[((size_t)i * n + r) * n + k] = (int8_t)(int)dg;
      }
    }
  }
}

// K-block range per row tile of digit planes dig [S][rows][K]: [first, last + 1) of the bk-wide
// K blocks holding a nonzero digit of the tile's bn rows in any plane.  The Gaussian operators
// decay below 2^-49 of their row maximum a few hundred points off the diagonal, where every
// truncation digit is zero: the contraction may skip those blocks exactly (int32 zeros).  An
// all-zero tile keeps one block so that its accumulators are written.
std::vector<int2> digit_kranges(const std::vector<int8_t>& dig, int S, int rows, int K, int bn, int bk) {
  std::vector<int2> kr(rows / bn);
  for (int t = 0; t < rows / bn; ++t) {
    int lo = K / bk, hi = 0;
    for (int kb = 0; kb < K / bk; ++kb) {
      bool nz = false;
      for (int i = 0; i < S && !nz; ++i)
        for (int r = t * bn; r < (t + 1) * bn && !nz; ++r) {
          const int8_t* row = dig.data() + ((size_t)i * rows + r) * K + (size_t)kb * bk;
          for (int k = 0; k < bk; ++k)
            if (row[k]) { nz = true; break; }
        }
      if (nz) { lo = std::min(lo, kb); hi = kb + 1; }
    }
    if (hi <= lo) { lo = 0; hi = 1; }
    kr[t] = make_int2(lo, hi);
  }
  return kr;
}

// per 64-row tile of a split operator (hi/lo planes [rows][cols], fp32 bit patterns): the K
// elements [first, last + 1) holding a nonzero hi or lo value, rounded out to `gran`
std::vector<int2> zero_kranges_f32(const std::vector<float>& hi, const std::vector<float>& lo, int rows, int cols,
                                   int gran) {
  std::vector<int2> kr(rows / 64);
  for (int t = 0; t < rows / 64; ++t) {
    int a = cols, b = 0;
    for (int r = t * 64; r < (t + 1) * 64; ++r)
      for (int c = 0; c < cols; ++c) {
        const size_t i = (size_t)r * cols + c;
        if (hi[i] != 0.0f || lo[i] != 0.0f) { a = std::min(a, c); b = std::max(b, c + 1); }
      }
    if (b <= a) { a = 0; b = gran; }
    kr[t] = make_int2(a / gran * gran, (b + gran - 1) / gran * gran);
  }
  return kr;
}

// ---------------------------------------------------------------- host fp64 transfers
// R (n_f/2 x n_f) applied to the rows of a column block: out = R * A  (A: n_f x cols)
void host_restrict_rows(const std::vector<double>& A, int n_f, int cols, std::vector<double>& out) {
  const int n_c = n_f / 2;
  out.assign((size_t)n_c * cols, 0.0);
  for (int j = 0; j < n_c; ++j) {
    const int taps[4] = {std::max(2 * j - 1, 0), 2 * j, 2 * j + 1, std::min(2 * j + 2, n_f - 1)};
    const double wts[4] = {1.0 / 8, 3.0 / 8, 3.0 / 8, 1.0 / 8};
    double* o = &out[(size_t)j * cols];
    for (int t = 0; t < 4; ++t) {
      const double* a = &A[(size_t)taps[t] * cols];
      for (int c = 0; c < cols; ++c) o[c] += wts[t] * a[c];
    }
  }
}
// out = A * P  (A: rows x n_f, P: n_f x n_f/2)
void host_prolong_cols(const std::vector<double>& A, int rows, int n_f, std::vector<double>& out) {
  const int n_c = n_f / 2;
  out.assign((size_t)rows * n_c, 0.0);
  for (int r = 0; r < rows; ++r) {
    const double* a = &A[(size_t)r * n_f];
    double* o = &out[(size_t)r * n_c];
    for (int i = 0; i < n_f; ++i) {
      const int j = i >> 1;
      const int k = std::min(std::max((i & 1) ? j + 1 : j - 1, 0), n_c - 1);
      o[j] += 0.75 * a[i];
      o[k] += 0.25 * a[i];
    }
  }
}
// Galerkin: R A P for square A (n_f x n_f)
void host_galerkin(const std::vector<double>& A, int n_f, std::vector<double>& out) {
  std::vector<double> AP;
  host_prolong_cols(A, n_f, n_f, AP);          // n_f x n_c
  host_restrict_rows(AP, n_f, n_f / 2, out);   // n_c x n_c
}

bool host_cholesky(std::vector<double>& A, int n, int* bad_pivot) {   // in place, lower
  for (int j = 0; j < n; ++j) {
    double d = A[(size_t)j * n + j];
    for (int k = 0; k < j; ++k) d -= A[(size_t)j * n + k] * A[(size_t)j * n + k];
    if (!(d > 0.0)) { *bad_pivot = j; return false; }
    const double ljj = std::sqrt(d);
    A[(size_t)j * n + j] = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = A[(size_t)i * n + j];
      for (int k = 0; k < j; ++k) s -= A[(size_t)i * n + k] * A[(size_t)j * n + k];
      A[(size_t)i * n + j] = s / ljj;
    }
    for (int i = 0; i < j; ++i) A[(size_t)i * n + j] = 0.0;
  }
  return true;
}

std::vector<float> to_f32(const std::vector<double>& v) {
  std::vector<float> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = (float)v[i];
  return o;
}

// Host emulation of cvt.rna.tf32.f32 (round to nearest, ties away from zero).
float tf32_rna(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) { u += 0x1000u; u &= 0xFFFFE000u; }
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
void split_host(const std::vector<double>& v, std::vector<float>& hi, std::vector<float>& lo) {
  hi.resize(v.size());
  lo.resize(v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    const float f = (float)v[i];
    hi[i] = tf32_rna(f);
    lo[i] = tf32_rna(f - hi[i]);
  }
}

uint16_t f16_rn(float x) {
  const __half h = __float2half_rn(x);
  uint16_t b;
  std::memcpy(&b, &h, 2);
  return b;
}
float f16_f(uint16_t b) {
  __half h;
  std::memcpy(&h, &b, 2);
  return __half2float(h);
}
// largest power of two S with S * bound <= 2^14 (f16 hi parts keep 2 bits of headroom)
float pow2_scale(double bound) {
  if (!(bound > 0.0) || !std::isfinite(bound)) return 1.0f;
  const int e = (int)std::floor(std::log2(16384.0 / bound));
  return std::ldexp(1.0f, std::max(-60, std::min(60, e)));
}

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

nmg_status get_encoder() {
  if (g_encode) return NMG_OK;
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !fn)
    return fail(NMG_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable");
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return NMG_OK;
}

// 2D fp32 row-major [rows][cols] tensor map, box {16, box_rows}, SWIZZLE_64B.
nmg_status make_map(CUtensorMap* m, const float* p, int64_t rows, int64_t cols, int box_rows) {
  NMG_TRY(get_encoder());
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * sizeof(float)};
  cuuint32_t box[2] = {16u, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, (void*)p, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NMG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%lld", (int)r,
                                     (long long)rows, (long long)cols);
  return NMG_OK;
}

// f16 [rows][cols], box {32, box_rows} (64-byte rows), SWIZZLE_64B
nmg_status make_map16(CUtensorMap* m, const uint16_t* p, int64_t rows, int64_t cols, int box_rows) {
  NMG_TRY(get_encoder());
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2u};
  cuuint32_t box[2] = {32u, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1u, 1u};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, (void*)p, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NMG_ERR_CUDA, "cuTensorMapEncodeTiled (f16) failed (%d)", (int)r);
  return NMG_OK;
}

// digit planes [S][rows][K] int8, box {ozaki_bk(), box_rows, S}, SWIZZLE_32B / _64B (32- / 64-byte rows)
nmg_status make_digit_map(CUtensorMap* m, const int8_t* p, int S, int64_t rows, int64_t K, int box_rows,
                          int box_digits = 0) {
  NMG_TRY(get_encoder());
  const int bk = ozaki_bk();
  cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)rows, (cuuint64_t)S};
  cuuint64_t strides[2] = {(cuuint64_t)K, (cuuint64_t)(rows * K)};
  cuuint32_t box[3] = {(cuuint32_t)bk, (cuuint32_t)box_rows, (cuuint32_t)(box_digits > 0 ? box_digits : S)};
  cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, (void*)p, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, bk == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NMG_ERR_CUDA, "cuTensorMapEncodeTiled (digits) failed (%d)", (int)r);
  return NMG_OK;
}

// padded activation tensor [rows][Wp][32] fp32 (rows = nrhs * Wp), box {16, 32, 10}, SWIZZLE_64B
nmg_status make_act_map(CUtensorMap* m, const float* p, int64_t rows, int Wp) {
  NMG_TRY(get_encoder());
  cuuint64_t dims[3] = {32u, (cuuint64_t)Wp, (cuuint64_t)rows};
  cuuint64_t strides[2] = {32u * sizeof(float), (cuuint64_t)Wp * 32u * sizeof(float)};
  cuuint32_t box[3] = {16u, 32u, 10u};
  cuuint32_t es[3] = {1u, 1u, 1u};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)p, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NMG_ERR_CUDA, "cuTensorMapEncodeTiled (3D) failed (%d)", (int)r);
  return NMG_OK;
}

// a2 activations f16 [rhs][y][x][C] viewed as 5D {8 ch, x, C/8 chunk, y, rhs}; box
// {8, 130, C/8, 1, 1} lands as the canonical no-swizzle K-major row buffer [C/8][130][8];
// x = -1 and x = n are out of bounds and zero-filled (the conv's zero padding).
nmg_status make_a2_map(CUtensorMap* m, const uint16_t* p, int n, int C, int64_t nrhs, int hg = 0) {
  NMG_TRY(get_encoder());
  if (hg <= 0) hg = n;   // image height (slab mode: R + 2 halo rows)
  cuuint64_t dims[5] = {8u, (cuuint64_t)n, (cuuint64_t)(C / 8), (cuuint64_t)hg, (cuuint64_t)nrhs};
  cuuint64_t strides[4] = {(cuuint64_t)C * 2u, 16u, (cuuint64_t)n * C * 2u, (cuuint64_t)hg * n * C * 2u};
  cuuint32_t box[5] = {8u, 130u, (cuuint32_t)(C / 8), 1u, 1u};
  cuuint32_t es[5] = {1u, 1u, 1u, 1u, 1u};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5, (void*)p, dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(NMG_ERR_CUDA, "cuTensorMapEncodeTiled (a2 5D) failed (%d)", (int)r);
  return NMG_OK;
}

// FNO layer input, channels-last fp32 (tf32 hi or lo plane): 1D [rhs][n][c] as {c, x, rhs} with box
// {16, 128, 1}; 2D [rhs][n][n][c] as {c, x, y, rhs} with box {16, bx, by, 1}; SWIZZLE_64B.  Points
// outside the image (tap shifts) are zero-filled: the convolution's "same" padding.
nmg_status make_fno_x_map(CUtensorMap* m, const float* p, int dim, int n, int c, int64_t nrhs, int bx, int by,
                          int halo_ks = 0) {
  NMG_TRY(get_encoder());
  CUresult r;
  if (halo_ks > 0) {
    // row-halo variant (fno_conv_rows_kernel): {4 ch, x, c/4 chunk, y, rhs}, box {4, 128 + ks - 1, 4, 1, 1}
    // lands as the no-swizzle K-major tile [4 chunks][128 + ks - 1 pixels][4 tf32]
    cuuint64_t dims[5] = {4u, (cuuint64_t)n, (cuuint64_t)(c / 4), (cuuint64_t)n, (cuuint64_t)nrhs};
    cuuint64_t strides[4] = {(cuuint64_t)c * 4u, 16u, (cuuint64_t)n * c * 4u, (cuuint64_t)n * n * c * 4u};
    cuuint32_t box[5] = {4u, (cuuint32_t)(128 + halo_ks - 1), 4u, 1u, 1u};
    cuuint32_t es[5] = {1u, 1u, 1u, 1u, 1u};
    r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, (void*)p, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (dim == 1) {
    cuuint64_t dims[3] = {(cuuint64_t)c, (cuuint64_t)n, (cuuint64_t)nrhs};
    cuuint64_t strides[2] = {(cuuint64_t)c * 4u, (cuuint64_t)n * c * 4u};
    cuuint32_t box[3] = {16u, 128u, 1u};
    cuuint32_t es[3] = {1u, 1u, 1u};
    r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)p, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    cuuint64_t dims[4] = {(cuuint64_t)c, (cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)nrhs};
    cuuint64_t strides[3] = {(cuuint64_t)c * 4u, (cuuint64_t)n * c * 4u, (cuuint64_t)n * n * c * 4u};
    cuuint32_t box[4] = {16u, (cuuint32_t)bx, (cuuint32_t)by, 1u};
    cuuint32_t es[4] = {1u, 1u, 1u, 1u};
    r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)p, dims, strides, box, es,
                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) return fail(NMG_ERR_CUDA, "cuTensorMapEncodeTiled (FNO input, %dD) failed (%d)", dim, (int)r);
  return NMG_OK;
}

}  // namespace

// ======================================================================= handle
struct nmg_hierarchy {
  nmg_problem_desc d{};
  nmg_tuning tune{};                                     // copied from desc.tuning (zeros = defaults)
  int L = 0;
  std::vector<int> n;      // points per axis, level 0 = finest
  std::vector<int64_t> N;  // unknowns per level
  // level-1 fp64 operator (1D: A; 2D: B, C)
  DevBuf<double> A64, B64, C64;
  std::vector<std::unique_ptr<DevBuf<double>>> A64l;     // fp64 A_l by level (1 .. L-2) for cycle64:
                                                         // every level in NMG_PREC_FP64, the fused
                                                         // coarse levels (n_l <= 512) in the mixed path
  int l_fuse = -1;                                       // first level of the fused coarse sub-cycle
  // per smoothed level (l < L-1) fp32 operators (SIMT path) and tf32 hi/lo splits (tcgen05)
  std::vector<std::unique_ptr<DevBuf<float>>> A32, AP32, A32h, A32l, AP32h, AP32l;
  std::vector<CUtensorMap> mAh, mAl, mAPh, mAPl;        // W operand maps per level (box 256)
  std::vector<CUtensorMap> mAh64, mAl64, mAPh64, mAPl64; // same with box 64
  std::vector<std::unique_ptr<DevBuf<float>>> sxh, sxl;  // X splits per level [max_rhs][n_l]
  std::vector<CUtensorMap> mXh, mXl;
  std::vector<char> split_fresh;                         // sxh/sxl[l] hold the split of wx[l]
  // 1D inner operator applies in FP16x3 (kind::f16): per-row-scaled f16 hi/lo planes
  bool gemm_f16 = false;
  struct F16Op { DevBuf<uint16_t> h, l; DevBuf<float> winv; DevBuf<int2> kr; CUtensorMap m256h, m256l, m64h, m64l, m128h, m128l; };
  bool gemm_mc = true;                                   // 256-wide FP16x3 tiles multicast W over CTA pairs
  std::vector<std::unique_ptr<F16Op>> A16, AP16;         // per smoothed level
  std::vector<std::unique_ptr<DevBuf<uint16_t>>> sx16h, sx16l;
  std::vector<std::unique_ptr<DevBuf<float>>> sxinv;
  std::vector<CUtensorMap> mX16h, mX16l;
  bool use_tc = true;
  bool smooth_f16 = false;                               // 1D smoother layer 2 on tcgen05 FP16x3 (default)
  std::vector<std::unique_ptr<DevBuf<uint16_t>>> W1b;    // per level: stacked f16 layer-2 weights
  std::vector<float> s1d_sc;                             // per level: S1, T1
  std::vector<Smooth1dW> s1d_w;                          // per level: host copy of the 1D CNN weights
  // fp64 outer residual via int8 digit products (Ozaki-style), 1D
  bool ozaki = false;
  DevBuf<int8_t> wdig, xdig;
  DevBuf<int> wexp, xexp;
  CUtensorMap mWd{}, mXd{};
  // 2D: the Kronecker pair (C then B) of the fp64 outer residual on the same int8 scheme
  bool ozaki2d = false;
  DevBuf<int8_t> wdigB;
  DevBuf<int> wexpB;
  CUtensorMap mWdB{};
  // per ozaki_bn()-row tile of the W digits: the K blocks holding a nonzero digit (C / A, then B)
  DevBuf<int2> wkr, wkrB;
  // 2D: A_l = B_l (x) C_l + alpha Q_l (x) Q_l; fp32 factors (SIMT), tf32 hi/lo (tcgen05)
  std::vector<std::unique_ptr<DevBuf<float>>> B32, C32, B32h, B32l, C32h, C32l, Q32;
  std::vector<std::unique_ptr<DevBuf<int2>>> Bkr, Ckr;   // per level: nonzero K ranges of B_l, C_l
  std::vector<int> qhb;                                  // Q_l half-bandwidth
  std::vector<CUtensorMap> mBh, mBl, mCh, mCl, mTh, mTl;
  std::vector<CUtensorMap> mBh64, mBl64, mCh64, mCl64;
  std::vector<CUtensorMap> mKBh, mKBl, mKCh, mKCl;      // W maps for kron_tc (box rows kron_tile_n)
  bool use_kron = false;
  std::vector<std::unique_ptr<DevBuf<float>>> tth, ttl;  // step-1 output (transposed blocks), hi/lo
  DevBuf<float2> Z;                                      // filter spectrum workspace
  DevBuf<double> snorm, spart;                           // smoother norms
  DevBuf<double> T64;                                    // fp64 outer step-1 output
  int rows_per_rhs = 1;
  int num_sms = 148;
  // 2D CNN on tcgen05 FP16x3 column-strip kernels (levels with n % 128 == 0 or 16 <= n < 128,
  // C = 32 / 48); other levels and tune.ffma_cnn use the FFMA kernel cnn2d
  bool conv_bf = false;
  int bf_C = 0, bf_chunk = 0;
  bool fuse_combine = true;                              // strip combine fused with the forward row FFT
  int64_t bf_px = 0;                                     // pixels per RHS the a2 / q workspaces hold
  std::vector<float> strip_sc;                           // per level: S1, T1, S2, T2
  DevBuf<uint16_t> a2h, a2l;                             // [chunk][n][n][C] f16 hi / lo (scaled by S2)
  DevBuf<float> qbuf;                                    // CNN output h [chunk][px], then edge records
  std::vector<CUtensorMap> mA2h, mA2l;                   // per level
  std::vector<std::unique_ptr<DevBuf<uint16_t>>> WB;     // per level: hidden 1 hi, lo, hidden 2 hi, lo
  // coarse Cholesky factor (row-major L and L^T)
  DevBuf<double> Lrow, Lcol;
  DevBuf<double> Ainv;                                   // explicit A_L^{-1} (default coarse apply)
  bool coarse_inv = true;
  int nc = 0;
  // FNO smoothers (nmg_load_fno_weights): per level arch + device parameters; shared workspaces
  struct FnoLevel {
    nmg_fno_arch arch{}; DevBuf<float> p; float proj_b = 0.f;
    // tensor-core W-convolution (fno_tc.cu): W as [layer][o][tap][c] tf32 hi/lo + one map per layer
    bool tc = false;
    DevBuf<float> w2h, w2l;
    std::vector<CUtensorMap> mWh, mWl;
  };
  std::vector<std::unique_ptr<FnoLevel>> fno;            // null = the level has a CNN
  DevBuf<float> fz0, fz1;
  DevBuf<float> fXh[2], fXl[2];                          // channels-last tf32 hi/lo layer inputs (ping-pong)
  DevBuf<float2> fT, fZh, fYh;
  int fno_chunk = 0;
  // smoother weights per level
  std::vector<std::unique_ptr<DevBuf<float>>> W;
  std::vector<int> w_loaded;
  nmg_cnn_arch arch{};
  DevBuf<float2> tw;
  int tw_n = 0;
  // workspaces
  std::vector<std::unique_ptr<DevBuf<float>>> wy, wx, wr, wb;
  DevBuf<double> part, ynorm, relres, ywork;
  DevBuf<uint8_t> active;
  DevBuf<double> hy, hx;   // staging for nmg_vcycles_host (allocated at create); nmg_solve's
                           // compacted active set reuses them
  DevBuf<int32_t> cmap;    // nmg_solve: compacted index -> RHS
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;         // copy streams of nmg_vcycles_host
  std::vector<cudaEvent_t> hev;                          // its chunk events
  int ntiles = 0;        // ||r||^2 partials per row: DMMA residual (64-wide tiles)
  int ntiles_oz = 0;     // ... Ozaki residual (ozaki_bn()-wide tiles)
  int64_t launches = 0;
  bool poisoned = false;
  // profiling (nmg_profile): event pairs per kernel class
  bool prof_on = false;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  struct Rec { int cls, nk; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  // CUDA graphs of one cycle, keyed by (nrhs, y, x, stream); a few entries so that the chunks
  // of nmg_vcycles_host each replay their own graph
  bool use_graph = true;
  struct GraphEntry {
    int nrhs; const void* y; void* x; cudaStream_t s; bool lanes;
    int seen; cudaGraphExec_t exec; int64_t launches; uint64_t used;
  };
  std::vector<GraphEntry> graphs;
  uint64_t g_clock = 0;
  // RHS lanes: a second hierarchy (same operators and weights) cycles the second half of a
  // large batch on a forked stream, so the two halves' kernels overlap (fills the last wave of
  // each launch and the small coarse-level grids); both halves are captured in one graph
  std::vector<std::unique_ptr<nmg_hierarchy>> lanes;     // lanes 1 .. K-1 (lane 0 is this handle)
  int lane_mult = 1;                                     // K while the lanes run (GEMM tile choice)
  bool lane_tiles = true;                                // GEMM tile width chosen for the whole batch
  std::vector<cudaStream_t> ls;                          // one forked stream per extra lane
  cudaEvent_t evf = nullptr;
  std::vector<cudaEvent_t> evj;
  // slab-sharded single-system mode (nmg_create_hierarchy_slab)
  bool slab = false;
  nmg_comm* comm = nullptr;                              // not owned
  int nw = 1, rank = 0, Ls = 0;                          // world; levels 0..Ls-1 sharded, the rest replicated
  static constexpr int HS = 4;                           // halo rows (the 4-layer 3x3 CNN's reach)
  std::vector<int> R;                                    // slab rows per sharded level
  std::vector<std::unique_ptr<DevBuf<float>>> sy, sx, sr, sb;   // [B][R + 2 HS][n_l] per sharded level
  std::vector<CUtensorMap> mKBhS, mKBlS;                 // B_l hi/lo maps, box rows kron_tile_n(R_l)
  DevBuf<float> tsend, trecv, hsend, hrecv, csend, crecv;
  DevBuf<double> t64send, t64recv, dscratch, ssum, rsum, ysq;
  DevBuf<float2> zs, za, zb;
  ~nmg_hierarchy() {
    for (auto x : ls) cudaStreamDestroy(x);
    if (evf) cudaEventDestroy(evf);
    for (auto e : evj) cudaEventDestroy(e);
    for (auto e : ev_pool) cudaEventDestroy(e);
    for (auto& g : graphs) if (g.exec) cudaGraphExecDestroy(g.exec);
    for (auto e : hev) cudaEventDestroy(e);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
  }
};

namespace {

// levels served by the column-strip CNN kernels (conv_strip.cu)
constexpr int kMaxHostChunks = 16;   // host-entry pipeline: RHS chunks / lanes (events per handle)
inline bool strip_level(int n) { return n % 128 == 0 || (n >= 16 && n < 128); }
// strip-edge records of the CNN output (after the chunk's h images in qbuf, see strip_h_fix)
inline float4* qedge(nmg_hierarchy* h) {
  return reinterpret_cast<float4*>(h->qbuf.p + (size_t)h->bf_chunk * h->bf_px);
}

void coarse_solve(nmg_hierarchy* h, int nrhs, const float* y, int64_t ldy, float* x, int64_t ldx, cudaStream_t s,
                  float* xh = nullptr, float* xl = nullptr) {
  if (h->coarse_inv) coarse_inv_apply(h->nc, nrhs, h->Ainv.p, y, ldy, x, ldx, s, xh, xl);
  else coarse_chol_solve(h->nc, nrhs, h->Lrow.p, h->Lcol.p, y, ldy, x, ldx, s, xh, xl);
}

nmg_status check_launch(nmg_hierarchy* h) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    h->poisoned = true;
    return fail(NMG_ERR_CUDA, "kernel launch failed: %s", cudaGetErrorString(e));
  }
  return NMG_OK;
}

cudaEvent_t prof_event(nmg_hierarchy* h) {
  if (h->ev_used == h->ev_pool.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    h->ev_pool.push_back(e);
  }
  return h->ev_pool[h->ev_used++];
}

// Counts the `nk` library kernel launches of one launcher call of class `cls`; when profiling,
// brackets them with events.
struct Prof {
  nmg_hierarchy* h; int cls; cudaStream_t s; int nk; cudaEvent_t a = nullptr;
  Prof(nmg_hierarchy* h_, int cls_, cudaStream_t s_, int nk_ = 1) : h(h_), cls(cls_), s(s_), nk(nk_) {
    h->launches += nk;
    if (h->prof_on && (a = prof_event(h))) cudaEventRecord(a, s);
  }
  ~Prof() {
    if (!a) return;
    cudaEvent_t b = prof_event(h);
    if (!b) return;
    cudaEventRecord(b, s);
    h->recs.push_back({cls, nk, a, b});
  }
};

// ---------------------------------------------------------------- 1D level operations
void launch_smooth1d(nmg_hierarchy* h, int l, Smooth1dArgs& a, cudaStream_t s) {
  if (h->smooth_f16 && a.n % 128 == 0 && h->W1b.size() > (size_t)l && h->W1b[l]->p) {
    a.wb = h->W1b[l]->p;
    // |u| <= 1 when normalised (||u||_2 = 1); the debug entry allows |u| <= 16
    const float S1 = h->s1d_sc[2 * l] * (a.normalize ? 1.f : 1.f / 16.f);
    a.in_scale = S1;
    a.d_scale = 1.f / (S1 * h->s1d_sc[2 * l + 1]);
    a.w = h->s1d_w[l];
    for (int c = 0; c < 16; ++c) a.w.b0[c] *= S1;
    // layer-2 output scale folded into layer 3 (d_scale a power of two: exact)
    for (int c = 0; c < 16; ++c) a.w.b1[c] /= a.d_scale;
    for (int i = 0; i < 80; ++i) a.w.w2[i] *= a.d_scale;
    smooth1d_f16(a, s);
  } else {
    smooth1d(a, s);
  }
}

// FNO smoother at level l (NEXT-2): x (+)= ||b|| F'_l(N(b / ||b||)) in RHS chunks (normalize =
// false: the raw network output of the debug CNN op; filter = false: no F').  norms: ||b|| per
// RHS already in h->snorm when normalize.
nmg_status run_fno(nmg_hierarchy* h, int l, int nrhs, const float* b, float* x, bool normalize, bool filter,
                   bool accumulate, cudaStream_t s) {
  const nmg_hierarchy::FnoLevel& F = *h->fno[l];
  const nmg_fno_arch& ar = F.arch;
  const int dim = h->d.dim, n = h->n[l], c = ar.width, k = ar.modes, ks = ar.ksize;
  const int64_t N = h->N[l];
  const float* P = F.p.p;
  FnoArgs a{};
  a.dim = dim; a.n = n; a.c = c; a.L = ar.n_layers; a.k = k; a.ks = ks;
  a.lift_w = P; a.lift_b = P + c;
  size_t off = 2 * (size_t)c;
  const size_t spec = (dim == 1 ? (size_t)k : (size_t)2 * k * k) * c * c * 2;
  const size_t conv = (size_t)c * c * (dim == 1 ? ks : ks * ks);
  for (int i = 0; i < ar.n_layers; ++i) {
    a.layer[i].R = reinterpret_cast<const float2*>(P + off); off += spec;
    a.layer[i].W = P + off; off += conv;
    a.layer[i].B = P + off; off += c;
    if (F.tc) { a.layer[i].tWh = &F.mWh[i]; a.layer[i].tWl = &F.mWl[i]; }
  }
  CUtensorMap mXh[2], mXl[2];
  if (F.tc) {
    int bx, by;
    fno_tc_box(n, &bx, &by);
    a.tc_rows = h->tune.simt_fno != 2 && fno_tc_rows(dim, n, ks);
    const int hks = a.tc_rows ? ks : 0;
    for (int q = 0; q < 2; ++q) {
      NMG_TRY(make_fno_x_map(&mXh[q], h->fXh[q].p, dim, n, c, h->fno_chunk, bx, by, hks));
      NMG_TRY(make_fno_x_map(&mXl[q], h->fXl[q].p, dim, n, c, h->fno_chunk, bx, by, hks));
      a.tXh[q] = &mXh[q]; a.tXl[q] = &mXl[q];
      a.Xh[q] = h->fXh[q].p; a.Xl[q] = h->fXl[q].p;
    }
  }
  a.proj_w = P + off;
  a.proj_b = F.proj_b;
  a.Z0 = h->fz0.p; a.Z1 = h->fz1.p; a.T = h->fT.p; a.Zh = h->fZh.p; a.Yh = h->fYh.p;
  a.tw = h->tw.p; a.tw_n = h->tw_n;
  a.filter = filter && h->d.level_filter != 0;
  a.accumulate = accumulate;
  const bool zf = dim == 2 && a.filter;
  for (int r0 = 0; r0 < nrhs; r0 += h->fno_chunk) {
    const int cnt = std::min(h->fno_chunk, nrhs - r0);
    a.nrhs = cnt;
    a.in = b + (int64_t)r0 * N;
    a.norms = normalize ? h->snorm.p + r0 : nullptr;
    a.x = x + (int64_t)r0 * N;
    a.Zf = zf ? h->Z.p : nullptr;
    a.zb0 = r0;
    { Prof p(h, NMG_K_SMOOTH, s, fno_launches(dim, ar.n_layers, F.tc)); fno_forward(a, s); }
    NMG_TRY(check_launch(h));
  }
  if (zf) {
    { Prof p(h, NMG_K_FILTER, s, 3);
      filter2d(nrhs, n, h->Z.p, h->tw.p, h->tw_n, x, accumulate, s, normalize ? h->snorm.p : nullptr); }
    NMG_TRY(check_launch(h));
  }
  return NMG_OK;
}

nmg_status smooth_level(nmg_hierarchy* h, int l, int nrhs, const float* b, float* x, bool accumulate,
                        cudaStream_t s) {
  if (h->fno.size() > (size_t)l && h->fno[l]) {
    const int n = h->n[l];
    { Prof p(h, NMG_K_FILTER, s, 2); norms_f32(nrhs, n, b, h->spart.p, 1, h->snorm.p, s); }
    NMG_TRY(check_launch(h));
    NMG_TRY(run_fno(h, l, nrhs, b, x, true, true, accumulate, s));
    if (h->split_fresh.size() > (size_t)l) h->split_fresh[l] = 0;
    return NMG_OK;
  }
  Smooth1dArgs a{};
  a.n = h->n[l]; a.nrhs = nrhs;
  a.b = b; a.ldb = a.n;
  a.x = x; a.ldx = a.n;
  a.params = h->W[l]->p;
  a.twiddle = h->tw.p; a.tw_n = h->tw_n;
  a.normalize = true;
  a.filter = h->d.level_filter != 0;
  a.accumulate = accumulate;
  bool split = !h->gemm_f16 && x == h->wx[l]->p && h->sxh.size() > (size_t)l && h->sxh[l]->p;
  if (split) { a.xh = h->sxh[l]->p; a.xl = h->sxl[l]->p; }
  if (h->gemm_f16 && a.filter && x == h->wx[l]->p && h->smooth_f16 && a.n % 128 == 0 && h->sx16h.size() > (size_t)l &&
      h->sx16h[l]->p) {
    a.x16h = h->sx16h[l]->p; a.x16l = h->sx16l[l]->p; a.xinv = h->sxinv[l]->p;
    split = true;
  }
  { Prof p(h, NMG_K_SMOOTH, s); launch_smooth1d(h, l, a, s); }
  if (h->split_fresh.size() > (size_t)l) h->split_fresh[l] = split ? 1 : 0;
  return check_launch(h);
}

// D = C - X * W^T-ish  (W: [N][K] K-major), fp32
nmg_status resid_gemm(nmg_hierarchy* h, int M, int N, int K, const float* X, const float* W, const float* C,
                      float* D, cudaStream_t s, bool negate = true) {
  Gemm32Args g{};
  g.M = M; g.N = N; g.K = K; g.batch = 1;
  g.X = X; g.ldx = K; g.sx = 0;
  g.W = W; g.ldw = K; g.sw = 0; g.w_kmajor = true;
  g.C = C; g.ldc = N; g.sc = 0;
  g.D = D; g.ldd = N; g.sd = 0;
  g.negate = negate;
  { Prof p(h, NMG_K_GEMM32, s); gemm_f32(g, s); }
  return check_launch(h);
}

// D = C - A_l X   (which = 0: W = A_l, K = n_l;  which = 1: W = A_l P_l, K = n_l / 2)
// X lives in wx[lx] (lx = l for A_l, l + 1 for A_l P_l).  tcgen05 3xTF32 when the
// shape allows, else the SIMT kernel.
nmg_status level_resid(nmg_hierarchy* h, int l, int which, int nrhs, const float* C, float* D, cudaStream_t s,
                       bool negate = true) {
  const int n = h->n[l];
  const int K = which == 0 ? n : n / 2;
  const int lx = which == 0 ? l : l + 1;
  const float* X = h->wx[lx]->p;
  const bool tc = h->use_tc && n % 16 == 0 && K % 16 == 0 && K >= 16;
  if (!tc) return resid_gemm(h, nrhs, n, K, X, which == 0 ? h->A32[l]->p : h->AP32[l]->p, C, D, s, negate);
  if (h->gemm_f16) {
    if (!h->split_fresh[lx]) {
      { Prof p(h, NMG_K_MISC, s); split_f16_rows(nrhs, K, X, h->sx16h[lx]->p, h->sx16l[lx]->p, h->sxinv[lx]->p, s); }
      NMG_TRY(check_launch(h));
      h->split_fresh[lx] = 1;
    }
    const nmg_hierarchy::F16Op& W = which == 0 ? *h->A16[l] : *h->AP16[l];
    TcGemmArgs g{};
    g.M = nrhs; g.N = n; g.K = K;
    g.C = C; g.ldc = n; g.D = D; g.ldd = n; g.negate = negate;
    g.xinv = h->sxinv[lx]->p; g.winv = W.winv.p;
    g.krange = h->tune.dense_k ? nullptr : W.kr.p;
    if (h->gemm_mc) { g.wh_mc = &W.m128h; g.wl_mc = &W.m128l; }
    {
      Prof p(h, NMG_K_GEMM32, s);
      const int bn = tc_pick_bn(nrhs * h->lane_mult, n, h->num_sms);
      tc_gemm_f16(&h->mX16h[lx], &h->mX16l[lx], bn == 256 ? &W.m256h : &W.m64h, bn == 256 ? &W.m256l : &W.m64l, g, s,
                  bn);
    }
    return check_launch(h);
  }
  if (!h->split_fresh[lx]) {
    { Prof p(h, NMG_K_MISC, s); split_tf32((int64_t)nrhs * K, X, h->sxh[lx]->p, h->sxl[lx]->p, s); }
    NMG_TRY(check_launch(h));
    h->split_fresh[lx] = 1;
  }
  TcGemmArgs g{};
  g.M = nrhs; g.N = n; g.K = K;
  g.C = C; g.ldc = n; g.D = D; g.ldd = n; g.negate = negate;
  {
    Prof p(h, NMG_K_GEMM32, s);
    const int bn = tc_pick_bn(nrhs * h->lane_mult, n, h->num_sms);
    if (which == 0)
      tc_gemm(&h->mXh[lx], &h->mXl[lx], bn == 256 ? &h->mAh[l] : &h->mAh64[l], bn == 256 ? &h->mAl[l] : &h->mAl64[l],
              g, s, bn);
    else
      tc_gemm(&h->mXh[lx], &h->mXl[lx], bn == 256 ? &h->mAPh[l] : &h->mAPh64[l],
              bn == 256 ? &h->mAPl[l] : &h->mAPl64[l], g, s, bn);
  }
  return check_launch(h);
}

// NMGF(0, y_l) at level l (0-based): input wy[l], output wx[l].
// the coarse levels l0 .. L-1 as one fp64 sub-cycle launch (cycle64.cu): x_l0 = NMGF(0, y_l0)
bool fused_coarse_ok(const nmg_hierarchy* h, int l) {
  if (h->l_fuse < 0 || l != h->l_fuse) return false;
  for (int q = l; q < h->L - 1; ++q)
    if (h->fno.size() > (size_t)q && h->fno[q]) return false;   // CNN smoothers only
  return true;
}

nmg_status cycle_level_1d(nmg_hierarchy* h, int l, int nrhs, cudaStream_t s) {
  const int n = h->n[l];
  float* y = h->wy[l]->p;
  float* x = h->wx[l]->p;
  if (fused_coarse_ok(h, l)) {
    Cycle64Args a{};
    a.n = n; a.L = h->L - l; a.nrhs = nrhs; a.nu1 = h->d.nu1; a.nu2 = h->d.nu2;
    a.filter = h->d.level_filter != 0;
    for (int q = l; q < h->L - 1; ++q) {
      a.A[q - l] = q == 0 ? h->A64.p : h->A64l[q]->p;
      a.W[q - l] = h->W[q]->p;
    }
    a.Ainv = h->Ainv.p;
    a.yf = y; a.xf = x; a.do_cycle = true;
    { Prof p(h, NMG_K_COARSE, s); cycle64(a, s); }
    h->split_fresh[l] = 0;
    return check_launch(h);
  }
  if (l == h->L - 1) {
    float* xh = (!h->gemm_f16 && h->sxh.size() > (size_t)l && h->sxh[l]->p && h->nc <= 128) ? h->sxh[l]->p : nullptr;
    { Prof p(h, NMG_K_COARSE, s);
      coarse_solve(h, nrhs, y, n, x, n, s, xh, xh ? h->sxl[l]->p : nullptr); }
    h->split_fresh[l] = xh ? 1 : 0;
    return check_launch(h);
  }
  float* r = h->wr[l]->p;
  float* b = h->wb[l]->p;
  const int nu1 = h->d.nu1, nu2 = h->d.nu2;
  const float* rl = y;
  if (nu1 >= 1) {
    NMG_TRY(smooth_level(h, l, nrhs, y, x, false, s));           // x = x* + F'(h), x* = 0
    for (int k = 1; k < nu1; ++k) {
      NMG_TRY(level_resid(h, l, 0, nrhs, y, b, s));              // b = y - A x
      NMG_TRY(smooth_level(h, l, nrhs, b, x, true, s));
    }
    NMG_TRY(level_resid(h, l, 0, nrhs, y, r, s));                 // r_l = y - A x
    rl = r;
  } else {
    NMG_CUDA(cudaMemsetAsync(x, 0, sizeof(float) * (size_t)nrhs * n, s));
    h->split_fresh[l] = 0;
  }
  { Prof p(h, NMG_K_TRANSFER, s); restrict1d(nrhs, n, rl, n, h->wy[l + 1]->p, n / 2, s); }   // y_{l+1} = R r_l
  NMG_TRY(check_launch(h));
  NMG_TRY(cycle_level_1d(h, l + 1, nrhs, s));
  const float* e = h->wx[l + 1]->p;
  if (nu2 >= 1) {
    NMG_TRY(level_resid(h, l, 1, nrhs, rl, b, s));                // b = r_l - (A P) e
  }
  { Prof p(h, NMG_K_TRANSFER, s); prolong_add1d(nrhs, n / 2, e, n / 2, x, n, s); }   // x += P e
  h->split_fresh[l] = 0;
  NMG_TRY(check_launch(h));
  if (nu2 >= 1) {
    NMG_TRY(smooth_level(h, l, nrhs, b, x, true, s));
    for (int k = 1; k < nu2; ++k) {
      NMG_TRY(level_resid(h, l, 0, nrhs, y, b, s));
      NMG_TRY(smooth_level(h, l, nrhs, b, x, true, s));
    }
  }
  return NMG_OK;
}

// ---------------------------------------------------------------- 2D level operations
// D = Cin -/+ A_l X,  A_l X = Mat(hat A Vec X) = C_l X B_l^T + alpha Q_l X Q_l^T.
// On the row-major [i2][i1] arrays (arr = X^T) this is B arr C^T + alpha Q arr Q^T:
//   step 1: Tt = blockT(arr C^T)   (M = nrhs*n rows, transposed store within n x n blocks)
//   stencil: D = Cin -/+ alpha Q arr Q^T
//   step 2: D = D -/+ blockT(Tt B^T)
nmg_status apply2d(nmg_hierarchy* h, int l, int nrhs, const float* X, const float* Cin, float* D, cudaStream_t s,
                   bool negate = true) {
  const int n = h->n[l];
  const int M = nrhs * n;
  if (h->use_kron && kron_supported(n, h->qhb[l])) {
    // fused path (kron_tc.cu): pass 1 T = blockT(arr C^T); pass 2 D = Cin -/+ (blockT(T B^T) + alpha QXQ^T)
    CUtensorMap mx;
    NMG_TRY(make_map(&mx, X, (int64_t)M, n, tc_gemm_block_m()));
    KronArgs k{};
    k.M = M; k.n = n; k.mode = KRON_T; k.D = h->tth[l]->p;
    k.krange = h->tune.dense_k ? nullptr : h->Ckr[l]->p;
    { Prof p(h, NMG_K_GEMM32, s); kron_tc(&mx, &h->mKCh[l], &h->mKCl[l], k, h->num_sms, s); }
    NMG_TRY(check_launch(h));
    KronArgs k2{};
    k2.M = M; k2.n = n; k2.mode = KRON_RESID; k2.D = D; k2.X = X; k2.Cin = Cin; k2.Q = h->Q32[l]->p;
    k2.hb = h->qhb[l]; k2.alpha = (float)h->d.alpha; k2.negate = negate;
    k2.krange = h->tune.dense_k ? nullptr : h->Bkr[l]->p;
    { Prof p(h, NMG_K_GEMM32, s); kron_tc(&h->mTh[l], &h->mKBh[l], &h->mKBl[l], k2, h->num_sms, s); }
    return check_launch(h);
  }
  const bool tc = h->use_tc && n % 16 == 0;
  if (tc) {
    { Prof p(h, NMG_K_MISC, s); split_tf32((int64_t)M * n, X, h->sxh[l]->p, h->sxl[l]->p, s); }
    TcGemmArgs g{};
    g.M = M; g.N = n; g.K = n; g.tblock = n; g.Dh = h->tth[l]->p; g.Dl = h->ttl[l]->p; g.negate = false;
    const int bn = tc_pick_bn(M, n, h->num_sms);
    { Prof p(h, NMG_K_GEMM32, s);
      tc_gemm(&h->mXh[l], &h->mXl[l], bn == 256 ? &h->mCh[l] : &h->mCh64[l], bn == 256 ? &h->mCl[l] : &h->mCl64[l],
              g, s, bn); }
  } else {
    Gemm32Args g{};
    g.M = M; g.N = n; g.K = n; g.batch = 1;
    g.X = X; g.ldx = n; g.W = h->C32[l]->p; g.ldw = n; g.w_kmajor = true;
    g.C = nullptr; g.D = h->tth[l]->p; g.ldd = n; g.negate = false; g.tblock = n;
    { Prof p(h, NMG_K_GEMM32, s); gemm_f32(g, s); }
  }
  NMG_TRY(check_launch(h));
  { Prof p(h, NMG_K_MISC, s);
    qstencil(nrhs, n, h->qhb[l], negate ? (float)h->d.alpha : -(float)h->d.alpha, h->Q32[l]->p, X, Cin, D, s); }
  NMG_TRY(check_launch(h));
  if (tc) {
    TcGemmArgs g{};
    g.M = M; g.N = n; g.K = n; g.tblock = n; g.C = D; g.D = D; g.negate = negate;
    const int bn = tc_pick_bn(M, n, h->num_sms);
    { Prof p(h, NMG_K_GEMM32, s);
      tc_gemm(&h->mTh[l], &h->mTl[l], bn == 256 ? &h->mBh[l] : &h->mBh64[l], bn == 256 ? &h->mBl[l] : &h->mBl64[l],
              g, s, bn); }
  } else {
    Gemm32Args g{};
    g.M = M; g.N = n; g.K = n; g.batch = 1;
    g.X = h->tth[l]->p; g.ldx = n; g.W = h->B32[l]->p; g.ldw = n; g.w_kmajor = true;
    g.C = D; g.D = D; g.ldd = n; g.negate = negate; g.tblock = n;
    { Prof p(h, NMG_K_GEMM32, s); gemm_f32(g, s); }
  }
  return check_launch(h);
}

// x = x* + hat F'(||b|| N(b/||b||))   (Alg 4)
nmg_status smooth2d(nmg_hierarchy* h, int l, int nrhs, const float* b, float* x, bool accumulate, cudaStream_t s,
                    bool normalize = true, bool filter = true) {
  const int n = h->n[l];
  const int64_t N = (int64_t)n * n;
  const int chunks = (int)std::min<int64_t>(64, std::max<int64_t>(1, N / 4096));
  if (normalize) {
    { Prof p(h, NMG_K_FILTER, s, 2); norms_f32(nrhs, N, b, h->spart.p, chunks, h->snorm.p, s); }
    NMG_TRY(check_launch(h));
  }
  const bool filt = filter && h->d.level_filter != 0;
  if (h->fno.size() > (size_t)l && h->fno[l]) return run_fno(h, l, nrhs, b, x, normalize, filter, accumulate, s);
  if (h->conv_bf && strip_level(n) && h->bf_C == h->arch.channels) {
    const int C = h->arch.channels;
    const float* P = h->W[l]->p;
    const float* b1 = P + C * 9 + C + C * C * 9;
    const float* b2 = b1 + C + C * C * 9;
    const float* w3 = b2 + C;
    const float* b3 = w3 + C * 9;
    const size_t plane = (size_t)9 * C * C;
    const uint16_t* wb = h->WB[l]->p;
    const float* sc = &h->strip_sc[(size_t)6 * l];
    const double* nrm = normalize ? h->snorm.p : nullptr;
    for (int r0 = 0; r0 < nrhs; r0 += h->bf_chunk) {
      const int cnt = std::min(h->bf_chunk, nrhs - r0);
      const int64_t off = (int64_t)r0 * N;
      StripArgs a{};
      a.n = n; a.nrhs = cnt; a.C = C; a.ysplit = strip_ysplit(n, cnt, h->num_sms);
      a.b = b + off; a.norms = nrm ? nrm + r0 : nullptr;
      a.w_in = P; a.w_out = w3;
      a.wh = wb; a.wl = wb + plane; a.bias = b1;
      // |u| <= 1 when normalised (||u||_2 = 1); the debug entry allows |u| <= 16
      const float dbg = normalize ? 1.0f : 1.0f / 16.0f;
      a.in_scale = sc[0] * dbg; a.out_scale = sc[2] * dbg; a.d_scale = 1.0f / (sc[0] * dbg * sc[1]);
      a.out_h = h->a2h.p; a.out_l = h->a2l.p; a.q = h->qbuf.p; a.qe = qedge(h); a.b3 = b3;
      { Prof p(h, NMG_K_SMOOTH, s); strip_l12(a, h->num_sms, s); }
      a.wh = wb + 2 * plane; a.wl = wb + 3 * plane; a.bias = b2;
      a.d_scale = 1.0f / (sc[2] * dbg * sc[3]);
      a.w4 = wb + 4 * plane; a.a3_scale = sc[4] * dbg; a.d4_scale = 1.0f / (sc[4] * dbg * sc[5]);
      { Prof p(h, NMG_K_SMOOTH, s); strip_l34(&h->mA2h[l], &h->mA2l[l], a, h->num_sms, s); }
      if (filt && h->fuse_combine) {
        // h = s (b3 + Q0 + Q1 + Q2) for the chunk's RHS pairs, straight into the forward row FFT
        { Prof p(h, NMG_K_FILTER, s);
          combine_rows_fft(n, cnt, h->qbuf.p, a.qe, a.norms, h->Z.p, r0, h->tw.p, h->tw_n, s); }
      } else {
        { Prof p(h, NMG_K_FILTER, s);
          strip_combine(n, cnt, h->qbuf.p, a.qe, a.norms, filt ? h->Z.p : nullptr, r0, x + off, accumulate, s); }
      }
      NMG_TRY(check_launch(h));
    }
    if (filt) {
      { Prof p(h, NMG_K_FILTER, s, h->fuse_combine ? 2 : 3);
        filter2d(nrhs, n, h->Z.p, h->tw.p, h->tw_n, x, accumulate, s, normalize ? h->snorm.p : nullptr,
                 h->fuse_combine); }
      NMG_TRY(check_launch(h));
    }
    return NMG_OK;
  }
  Cnn2dArgs a{};
  a.n = n; a.nrhs = nrhs; a.C = h->arch.channels;
  a.b = b; a.norms = normalize ? h->snorm.p : nullptr; a.params = h->W[l]->p;
  a.Z = filt ? h->Z.p : nullptr; a.x = x; a.accumulate = accumulate;
  { Prof p(h, NMG_K_SMOOTH, s); cnn2d(a, s); }
  NMG_TRY(check_launch(h));
  if (filt) {
    { Prof p(h, NMG_K_FILTER, s, 3); filter2d(nrhs, n, h->Z.p, h->tw.p, h->tw_n, x, accumulate, s, normalize ? h->snorm.p : nullptr); }
    NMG_TRY(check_launch(h));
  }
  return NMG_OK;
}

nmg_status cycle_level_2d(nmg_hierarchy* h, int l, int nrhs, cudaStream_t s) {
  const int n = h->n[l];
  float* y = h->wy[l]->p;
  float* x = h->wx[l]->p;
  if (l == h->L - 1) {
    { Prof p(h, NMG_K_COARSE, s); coarse_solve(h, nrhs, y, h->nc, x, h->nc, s); }
    return check_launch(h);
  }
  float* r = h->wr[l]->p;
  float* b = h->wb[l]->p;
  const size_t bytes = sizeof(float) * (size_t)nrhs * n * n;
  if (h->d.nu1 >= 1) {
    NMG_TRY(smooth2d(h, l, nrhs, y, x, false, s));
    for (int k = 1; k < h->d.nu1; ++k) {
      NMG_TRY(apply2d(h, l, nrhs, x, y, b, s));
      NMG_TRY(smooth2d(h, l, nrhs, b, x, true, s));
    }
    NMG_TRY(apply2d(h, l, nrhs, x, y, r, s));
  } else {
    NMG_CUDA(cudaMemsetAsync(x, 0, bytes, s));
    NMG_CUDA(cudaMemcpyAsync(r, y, bytes, cudaMemcpyDeviceToDevice, s));
  }
  { Prof p(h, NMG_K_TRANSFER, s); restrict2d(nrhs, n, r, h->wy[l + 1]->p, s); }
  NMG_TRY(check_launch(h));
  NMG_TRY(cycle_level_2d(h, l + 1, nrhs, s));
  { Prof p(h, NMG_K_TRANSFER, s); prolong_add2d(nrhs, n / 2, h->wx[l + 1]->p, x, s); }
  NMG_TRY(check_launch(h));
  for (int k = 0; k < h->d.nu2; ++k) {
    NMG_TRY(apply2d(h, l, nrhs, x, y, b, s));
    NMG_TRY(smooth2d(h, l, nrhs, b, x, true, s));
  }
  return NMG_OK;
}

// ---------------------------------------------------------------- slab-sharded mode (§8(e))
// Every sharded level keeps its vectors as this rank's slab of R_l rows plus HS halo rows per
// side, [b][R_l + 2 HS][n_l]; "global row g" of image b lives at slab + b img + (HS - r0 + g) n.
inline int64_t slab_img(const nmg_hierarchy* h, int l) { return (int64_t)(h->R[l] + 2 * h->HS) * h->n[l]; }

// fill the halo rows of x (level l) from the neighbouring ranks (zeros at the image borders)
nmg_status halo_exchange(nmg_hierarchy* h, int l, int nrhs, float* x, cudaStream_t s) {
  const int n = h->n[l], R = h->R[l], H = h->HS;
  { Prof p(h, NMG_K_MISC, s); halo_pack(nrhs, n, R, H, x, h->hsend.p, s); }
  NMG_TRY(check_launch(h));
  NMG_TRY(h->comm->all_gather(h->hsend.p, h->hrecv.p, sizeof(float) * (size_t)2 * nrhs * H * n, s));
  { Prof p(h, NMG_K_MISC, s); halo_unpack(nrhs, n, R, H, h->rank, h->nw, h->hrecv.p, x, s); }
  return check_launch(h);
}

// recv = [W][rows_per_rank] blocks of `width` elements per row -> full rows: dst row m, columns
// q w .. q w + w - 1 = rank q's block row m  (unpack of an all-gathered slab-major array)
template <typename T>
nmg_status unpack_gathered(nmg_hierarchy* h, const T* recv, T* dst, int64_t rows, int64_t width, int64_t dpitch,
                           cudaStream_t s) {
  for (int q = 0; q < h->nw; ++q)
    NMG_CUDA(cudaMemcpy2DAsync(dst + q * width, sizeof(T) * dpitch, recv + (int64_t)q * rows * width, sizeof(T) * width,
                               sizeof(T) * width, rows, cudaMemcpyDeviceToDevice, s));
  return NMG_OK;
}

// D = Cin -/+ A_l X on the slab (X's halo rows must hold the neighbours' rows when hb > 0):
// pass 1 T = C_l X[:, slab] (local), all-gather T, pass 2 D[:, slab] = T B_l[slab]^T + alpha QXQ^T
nmg_status apply_slab(nmg_hierarchy* h, int l, int nrhs, const float* X, const float* Cin, float* D, cudaStream_t s,
                      bool negate = true) {
  const int n = h->n[l], R = h->R[l], H = h->HS;
  CUtensorMap mx;
  NMG_TRY(make_map(&mx, X, (int64_t)nrhs * (R + 2 * H), n, tc_gemm_block_m()));
  KronArgs k{};
  k.M = nrhs * (R + 2 * H); k.n = n; k.mode = KRON_T; k.D = h->tsend.p;
  k.R = R; k.H = H; k.r0 = h->rank * R; k.img = slab_img(h, l);
  k.krange = h->tune.dense_k ? nullptr : h->Ckr[l]->p;
  { Prof p(h, NMG_K_GEMM32, s); kron_tc(&mx, &h->mKCh[l], &h->mKCl[l], k, h->num_sms, s); }
  NMG_TRY(check_launch(h));
  NMG_TRY(h->comm->all_gather(h->tsend.p, h->trecv.p, sizeof(float) * (size_t)nrhs * n * R, s));
  NMG_TRY(unpack_gathered<float>(h, h->trecv.p, h->tth[l]->p, (int64_t)nrhs * n, R, n, s));
  KronArgs k2{};
  k2.M = nrhs * n; k2.n = n; k2.mode = KRON_RESID; k2.D = D; k2.X = X; k2.Cin = Cin; k2.Q = h->Q32[l]->p;
  k2.hb = h->qhb[l]; k2.alpha = (float)h->d.alpha; k2.negate = negate;
  k2.R = R; k2.H = H; k2.r0 = h->rank * R; k2.img = slab_img(h, l);
  k2.krange = (h->tune.dense_k || (h->rank * R) % 64) ? nullptr : h->Bkr[l]->p;
  { Prof p(h, NMG_K_GEMM32, s); kron_tc(&h->mTh[l], &h->mKBhS[l], &h->mKBlS[l], k2, h->num_sms, s); }
  return check_launch(h);
}

// x = x* + F'(||b|| N(b/||b||)) on the slab; b's halo rows are filled here (CNN reach 4 rows)
nmg_status smooth_slab(nmg_hierarchy* h, int l, int nrhs, float* b, float* x, bool accumulate, cudaStream_t s) {
  const int n = h->n[l], R = h->R[l], H = h->HS, C = h->arch.channels;
  const int64_t img = slab_img(h, l);
  if (!(h->conv_bf && h->bf_C == C && strip_level(n)))
    return fail(NMG_ERR_UNSUPPORTED, "slab mode needs the strip-kernel CNN (C = 32 / 48, n %% 128 == 0)");
  // ||b|| over the whole image: local sums of squares, summed over the ranks (fixed order)
  {
    const int chunks = (int)std::min<int64_t>(64, std::max<int64_t>(1, (int64_t)R * n / 4096));
    { Prof p(h, NMG_K_FILTER, s, 2); sumsq_f32(nrhs, (int64_t)R * n, b, img, (int64_t)H * n, h->spart.p, chunks, h->snorm.p, s); }
    NMG_TRY(check_launch(h));
    NMG_TRY(h->comm->sum_f64(h->snorm.p, nrhs, h->dscratch.p, s));
    { Prof p(h, NMG_K_MISC, s); sqrt_inplace(nrhs, h->snorm.p, s); }
  }
  NMG_TRY(halo_exchange(h, l, nrhs, b, s));
  const bool filt = h->d.level_filter != 0;
  const float* P = h->W[l]->p;
  const float* b1 = P + C * 9 + C + C * C * 9;
  const float* b2 = b1 + C + C * C * 9;
  const float* w3 = b2 + C;
  const float* b3 = w3 + C * 9;
  const size_t plane = (size_t)9 * C * C;
  const uint16_t* wb = h->WB[l]->p;
  const float* sc = &h->strip_sc[(size_t)6 * l];
  const int hg = R + 2 * H;
  // RHS per CNN chunk: the a2 / q workspaces hold bf_chunk images of bf_px pixels
  const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(h->bf_chunk, h->bf_chunk * h->bf_px / ((int64_t)hg * n)));
  CUtensorMap m2h, m2l;
  NMG_TRY(make_a2_map(&m2h, h->a2h.p, n, C, chunk, hg));
  NMG_TRY(make_a2_map(&m2l, h->a2l.p, n, C, chunk, hg));
  for (int c0 = 0; c0 < nrhs; c0 += chunk) {
    const int cnt = std::min(chunk, nrhs - c0);
    const int64_t off = (int64_t)c0 * img;
    StripArgs a{};
    a.n = n; a.h = hg; a.nrhs = cnt; a.C = C; a.ysplit = strip_ysplit(n, cnt, h->num_sms, hg);
    a.ylo = h->rank == 0 ? H : 0;                       // the global image border is zero padding
    a.yhi = h->rank == h->nw - 1 ? hg - H : hg;
    a.b = b + off; a.norms = h->snorm.p + c0;
    a.w_in = P; a.w_out = w3;
    a.wh = wb; a.wl = wb + plane; a.bias = b1;
    a.in_scale = sc[0]; a.out_scale = sc[2]; a.d_scale = 1.0f / (sc[0] * sc[1]);
    a.out_h = h->a2h.p; a.out_l = h->a2l.p; a.q = h->qbuf.p; a.qe = qedge(h); a.b3 = b3;
    { Prof p(h, NMG_K_SMOOTH, s); strip_l12(a, h->num_sms, s); }
    a.wh = wb + 2 * plane; a.wl = wb + 3 * plane; a.bias = b2;
    a.d_scale = 1.0f / (sc[2] * sc[3]);
    a.w4 = wb + 4 * plane; a.a3_scale = sc[4]; a.d4_scale = 1.0f / (sc[4] * sc[5]);
    { Prof p(h, NMG_K_SMOOTH, s); strip_l34(&m2h, &m2l, a, h->num_sms, s); }
    { Prof p(h, NMG_K_FILTER, s);
      strip_combine(n, cnt, h->qbuf.p, a.qe, a.norms, filt ? h->zs.p : nullptr, c0, x + off, accumulate, s, hg, H); }
    NMG_TRY(check_launch(h));
  }
  if (filt) {
    // rows local; columns after an all-to-all transpose; back; inverse rows + update
    const size_t chunk = sizeof(float2) * (size_t)nrhs * (R / 2) * filter2d_slab_chunk(n, h->nw);
    { Prof p(h, NMG_K_FILTER, s); filter2d_slab_rows(n, nrhs, R, h->zs.p, h->tw.p, h->tw_n, s); }
    { Prof p(h, NMG_K_MISC, s); filter2d_slab_pack(n, nrhs, R, h->nw, h->zs.p, h->za.p, false, s); }
    NMG_TRY(check_launch(h));
    NMG_TRY(h->comm->all_to_all(h->za.p, h->zb.p, chunk, s));
    { Prof p(h, NMG_K_FILTER, s); filter2d_slab_cols(n, nrhs, R, h->nw, h->rank, h->zb.p, h->tw.p, h->tw_n, s); }
    NMG_TRY(check_launch(h));
    NMG_TRY(h->comm->all_to_all(h->zb.p, h->za.p, chunk, s));
    { Prof p(h, NMG_K_MISC, s); filter2d_slab_pack(n, nrhs, R, h->nw, h->zs.p, h->za.p, true, s); }
    { Prof p(h, NMG_K_FILTER, s);
      filter2d_slab_inverse(n, nrhs, R, h->zs.p, h->tw.p, h->tw_n, x, img, (int64_t)H * n, accumulate, h->snorm.p, s); }
    NMG_TRY(check_launch(h));
  }
  return NMG_OK;
}

nmg_status cycle_level_2d(nmg_hierarchy* h, int l, int nrhs, cudaStream_t s);

// NMGF(0, y_l) on the slab of sharded level l: input sy[l] (own rows), output sx[l] (own rows)
nmg_status cycle_slab(nmg_hierarchy* h, int l, int nrhs, cudaStream_t s) {
  const int n = h->n[l], R = h->R[l], H = h->HS, r0 = h->rank * R;
  const int64_t img = slab_img(h, l);
  float* y = h->sy[l]->p;
  float* x = h->sx[l]->p;
  float* r = h->sr[l]->p;
  float* b = h->sb[l]->p;
  const bool hx = h->qhb[l] > 0;   // the mass stencil reads x rows +- hb
  if (h->d.nu1 >= 1) {
    NMG_TRY(smooth_slab(h, l, nrhs, y, x, false, s));
    for (int k = 1; k < h->d.nu1; ++k) {
      if (hx) NMG_TRY(halo_exchange(h, l, nrhs, x, s));
      NMG_TRY(apply_slab(h, l, nrhs, x, y, b, s));
      NMG_TRY(smooth_slab(h, l, nrhs, b, x, true, s));
    }
    if (hx) NMG_TRY(halo_exchange(h, l, nrhs, x, s));
    NMG_TRY(apply_slab(h, l, nrhs, x, y, r, s));
  } else {
    NMG_CUDA(cudaMemsetAsync(x, 0, sizeof(float) * (size_t)nrhs * img, s));
    NMG_CUDA(cudaMemcpyAsync(r, y, sizeof(float) * (size_t)nrhs * img, cudaMemcpyDeviceToDevice, s));
  }
  NMG_TRY(halo_exchange(h, l, nrhs, r, s));   // full weighting reads fine rows 2 j2 - 1 .. 2 j2 + 2
  const int nc = n / 2, Rc = R / 2, r0c = r0 / 2;
  const int64_t foff = (int64_t)(H - r0) * n;
  if (l + 1 < h->Ls) {
    { Prof p(h, NMG_K_TRANSFER, s);
      restrict_slab(nrhs, nc, Rc, r0c, r, img, foff, h->sy[l + 1]->p, slab_img(h, l + 1), (int64_t)H * nc, s); }
    NMG_TRY(check_launch(h));
    NMG_TRY(cycle_slab(h, l + 1, nrhs, s));
    NMG_TRY(halo_exchange(h, l + 1, nrhs, h->sx[l + 1]->p, s));
    { Prof p(h, NMG_K_TRANSFER, s);
      prolong_slab(nrhs, nc, R, r0, h->sx[l + 1]->p, slab_img(h, l + 1), (int64_t)(H - r0c) * nc, x, img,
                   (int64_t)H * n, s); }
  } else {
    // replicated coarse sub-cycle: gather the restricted RHS, run the levels >= l + 1 on every rank
    const int Rq = nc / h->nw;
    { Prof p(h, NMG_K_TRANSFER, s);
      restrict_slab(nrhs, nc, Rq, h->rank * Rq, r, img, foff, h->csend.p, (int64_t)Rq * nc, 0, s); }
    NMG_TRY(check_launch(h));
    NMG_TRY(h->comm->all_gather(h->csend.p, h->crecv.p, sizeof(float) * (size_t)nrhs * Rq * nc, s));
    NMG_TRY(unpack_gathered<float>(h, h->crecv.p, h->wy[l + 1]->p, nrhs, (int64_t)Rq * nc, (int64_t)nc * nc, s));
    NMG_TRY(cycle_level_2d(h, l + 1, nrhs, s));
    { Prof p(h, NMG_K_TRANSFER, s);
      prolong_slab(nrhs, nc, R, r0, h->wx[l + 1]->p, (int64_t)nc * nc, 0, x, img, (int64_t)H * n, s); }
  }
  NMG_TRY(check_launch(h));
  for (int k = 0; k < h->d.nu2; ++k) {
    if (hx) NMG_TRY(halo_exchange(h, l, nrhs, x, s));
    NMG_TRY(apply_slab(h, l, nrhs, x, y, b, s));
    NMG_TRY(smooth_slab(h, l, nrhs, b, x, true, s));
  }
  return NMG_OK;
}

// fp64 outer residual on the slab: pass 1 T = C X[:, slab] (DMMA), all-gather T, pass 2
// r[:, slab] = y - (T B[slab]^T + alpha x); r32 -> sy[0] (own rows), ||r||^2 partials -> part
nmg_status outer_residual_slab(nmg_hierarchy* h, int nrhs, const double* y, const double* x, double* r64,
                               bool want_part, cudaStream_t s) {
  const int n = h->n[0], R = h->R[0], H = h->HS, r0 = h->rank * R;
  if (h->ozaki2d && R % 128 == 0) {
    // the same two passes on the int8 tensor cores (Ozaki digits, as outer_residual 2D)
    const int64_t plane = (int64_t)h->d.max_rhs * n * n;
    { Prof p(h, NMG_K_GEMM64, s); ozaki_split_rows(nrhs * R, n, x, n, h->xdig.p, plane, h->xexp.p, s); }
    NMG_TRY(check_launch(h));
    OzakiArgs o{};
    o.M = nrhs * R; o.N = n; o.K = n;
    o.r64 = h->t64send.p; o.plus = true;
    o.tblock = n; o.tb_R = R; o.tb_S = R; o.tb_img = (int64_t)n * R;
    o.ex = h->xexp.p; o.ew = h->wexp.p; o.krange = h->tune.dense_k ? nullptr : h->wkr.p;
    { Prof p(h, NMG_K_GEMM64, s); ozaki_resid(&h->mXd, &h->mWd, o, s); }
    NMG_TRY(check_launch(h));
    NMG_TRY(h->comm->all_gather(h->t64send.p, h->t64recv.p, sizeof(double) * (size_t)nrhs * n * R, s));
    NMG_TRY(unpack_gathered<double>(h, h->t64recv.p, h->T64.p, (int64_t)nrhs * n, R, n, s));
    { Prof p(h, NMG_K_GEMM64, s); ozaki_split_rows(nrhs * n, n, h->T64.p, n, h->xdig.p, plane, h->xexp.p, s); }
    NMG_TRY(check_launch(h));
    OzakiArgs q{};
    q.M = nrhs * n; q.N = R; q.K = n;
    q.Y = y; q.ax = x; q.alpha = h->d.alpha;
    q.r32 = h->sy[0]->p; q.r32_img = slab_img(h, 0); q.r32_off = (int64_t)H * n;
    q.r64 = r64; q.part = want_part ? h->part.p : nullptr;
    q.tblock = n; q.tb_R = n; q.tb_S = n; q.tb_img = (int64_t)R * n;
    q.ex = h->xexp.p; q.ew = h->wexpB.p; q.wrow0 = r0;
    q.krange = (h->tune.dense_k || r0 % (2 * ozaki_bn())) ? nullptr : h->wkrB.p;
    { Prof p(h, NMG_K_GEMM64, s); ozaki_resid(&h->mXd, &h->mWdB, q, s); }
    return check_launch(h);
  }
  Gemm64Args g{};
  g.M = nrhs * R; g.N = n; g.K = n;
  g.X = x; g.ldx = n; g.W = h->C64.p; g.ldw = n;
  g.Y = nullptr; g.r32 = nullptr; g.r64 = h->t64send.p; g.part = nullptr; g.negate = false;
  g.tblock = n; g.tb_R = R; g.tb_S = R; g.tb_img = (int64_t)n * R;
  { Prof p(h, NMG_K_GEMM64, s); gemm_f64(g, s); }
  NMG_TRY(check_launch(h));
  NMG_TRY(h->comm->all_gather(h->t64send.p, h->t64recv.p, sizeof(double) * (size_t)nrhs * n * R, s));
  NMG_TRY(unpack_gathered<double>(h, h->t64recv.p, h->T64.p, (int64_t)nrhs * n, R, n, s));
  Gemm64Args q{};
  q.M = nrhs * n; q.N = R; q.K = n;
  q.X = h->T64.p; q.ldx = n; q.W = h->B64.p + (int64_t)r0 * n; q.ldw = n;
  q.Y = y; q.r32 = h->sy[0]->p; q.r64 = r64; q.part = want_part ? h->part.p : nullptr;
  q.negate = true; q.ax = x; q.alpha = h->d.alpha;
  q.tblock = n; q.tb_R = n; q.tb_S = n; q.tb_img = (int64_t)R * n;
  q.r32_img = slab_img(h, 0); q.r32_off = (int64_t)H * n;
  { Prof p(h, NMG_K_GEMM64, s); gemm_f64(q, s); }
  return check_launch(h);
}

nmg_status inner_cycle(nmg_hierarchy* h, int nrhs, cudaStream_t s) {
  if (h->slab) return cycle_slab(h, 0, nrhs, s);
  if (h->d.dim == 1) return cycle_level_1d(h, 0, nrhs, s);
  return cycle_level_2d(h, 0, nrhs, s);
}

// fp64 residual at level 1: r32 = y - A x -> wy[0]; optional r64; norm partials -> part
nmg_status outer_residual(nmg_hierarchy* h, int nrhs, const double* y, const double* x, double* r64,
                          bool want_part, cudaStream_t s) {
  if (h->slab) return outer_residual_slab(h, nrhs, y, x, r64, want_part, s);
  if (h->d.dim == 2 && h->ozaki2d) {
    const int n = h->n[0];
    const int M = nrhs * n;
    const int64_t plane = (int64_t)h->d.max_rhs * n * n;
    { Prof p(h, NMG_K_GEMM64, s); ozaki_split_rows(M, n, x, n, h->xdig.p, plane, h->xexp.p, s); }
    NMG_TRY(check_launch(h));
    OzakiArgs o{};
    o.M = M; o.N = n; o.K = n;
    o.r64 = h->T64.p; o.tblock = n; o.plus = true;
    o.ex = h->xexp.p; o.ew = h->wexp.p; o.krange = h->tune.dense_k ? nullptr : h->wkr.p;
    { Prof p(h, NMG_K_GEMM64, s); ozaki_resid(&h->mXd, &h->mWd, o, s); }
    NMG_TRY(check_launch(h));
    { Prof p(h, NMG_K_GEMM64, s); ozaki_split_rows(M, n, h->T64.p, n, h->xdig.p, plane, h->xexp.p, s); }
    NMG_TRY(check_launch(h));
    OzakiArgs q{};
    q.M = M; q.N = n; q.K = n;
    q.Y = y; q.r32 = h->wy[0]->p; q.r64 = r64; q.part = want_part ? h->part.p : nullptr;
    q.tblock = n; q.ax = x; q.alpha = h->d.alpha;
    q.ex = h->xexp.p; q.ew = h->wexpB.p; q.krange = h->tune.dense_k ? nullptr : h->wkrB.p;
    { Prof p(h, NMG_K_GEMM64, s); ozaki_resid(&h->mXd, &h->mWdB, q, s); }
    return check_launch(h);
  }
  if (h->d.dim == 2) {
    const int n = h->n[0];
    Gemm64Args g{};
    g.M = nrhs * n; g.N = n; g.K = n;
    g.X = x; g.ldx = n; g.W = h->C64.p; g.ldw = n;
    g.Y = nullptr; g.r32 = nullptr; g.r64 = h->T64.p; g.part = nullptr; g.negate = false; g.tblock = n;
    { Prof p(h, NMG_K_GEMM64, s); gemm_f64(g, s); }
    NMG_TRY(check_launch(h));
    Gemm64Args q{};
    q.M = nrhs * n; q.N = n; q.K = n;
    q.X = h->T64.p; q.ldx = n; q.W = h->B64.p; q.ldw = n;
    q.Y = y; q.r32 = h->wy[0]->p; q.r64 = r64; q.part = want_part ? h->part.p : nullptr;
    q.negate = true; q.tblock = n; q.ax = x; q.alpha = h->d.alpha;
    { Prof p(h, NMG_K_GEMM64, s); gemm_f64(q, s); }
    return check_launch(h);
  }
  if (h->ozaki && nrhs > 64) {   // small batches: one DMMA tile row beats the digit pipeline
    const int n = h->n[0];
    { Prof p(h, NMG_K_GEMM64, s);
      ozaki_split_rows(nrhs, n, x, n, h->xdig.p, (int64_t)h->d.max_rhs * n, h->xexp.p, s); }
    NMG_TRY(check_launch(h));
    OzakiArgs o{};
    o.M = nrhs; o.N = n; o.K = n;
    o.Y = y; o.ldy = n;
    o.r32 = h->wy[0]->p; o.ldr32 = n;
    o.r64 = r64; o.ldr64 = n;
    o.part = want_part ? h->part.p : nullptr;
    o.ex = h->xexp.p; o.ew = h->wexp.p; o.krange = h->tune.dense_k ? nullptr : h->wkr.p;
    { Prof p(h, NMG_K_GEMM64, s); ozaki_resid(&h->mXd, &h->mWd, o, s); }
    return check_launch(h);
  }
  Gemm64Args g{};
  const int n = h->n[0];
  g.M = nrhs; g.N = n; g.K = n;
  g.X = x; g.ldx = n;
  g.W = h->A64.p; g.ldw = n;
  g.Y = y; g.ldy = n;
  g.r32 = h->wy[0]->p; g.ldr32 = n;
  g.r64 = r64; g.ldr64 = n;
  g.part = want_part ? h->part.p : nullptr;
  g.negate = true;
  { Prof p(h, NMG_K_GEMM64, s); gemm_f64(g, s); }
  return check_launch(h);
}

// ||y|| per RHS (slab mode: local sums of squares summed over the ranks)
nmg_status ynorms(nmg_hierarchy* h, int nrhs, const double* y, cudaStream_t s) {
  if (!h->slab) {
    { Prof p(h, NMG_K_MISC, s, 2); row_norms_f64(nrhs, (int)h->N[0], y, h->N[0], h->ynorm.p, h->ywork.p, s); }
    return check_launch(h);
  }
  { Prof p(h, NMG_K_MISC, s, 2); sumsq_f64(nrhs, (int64_t)h->R[0] * h->n[0], y, h->ywork.p, h->ysq.p, s); }
  NMG_TRY(check_launch(h));
  return h->comm->sum_f64(h->ysq.p, nrhs, h->dscratch.p, s);
}
// relres = ||r|| / ||y|| from the outer residual's partials; active = relres > tol
nmg_status relres_fin(nmg_hierarchy* h, int nrhs, double tol, uint8_t* active, double* relres, cudaStream_t s) {
  if (!h->slab) {
    const bool oz = h->d.dim == 1 ? (h->ozaki && nrhs > 64) : h->ozaki2d;   // as outer_residual
    { Prof p(h, NMG_K_MISC, s);
      relres_finalize(nrhs, oz ? h->ntiles_oz : h->ntiles, h->part.p, h->ynorm.p, relres, tol, active, s, h->rows_per_rhs); }
    return check_launch(h);
  }
  const int64_t cnt = (int64_t)((h->ozaki2d && h->R[0] % 128 == 0) ? h->R[0] / ozaki_bn() : gemm_f64_ntiles(h->R[0])) *
                      h->n[0];
  { Prof p(h, NMG_K_MISC, s); part_sums(nrhs, cnt, h->part.p, h->rsum.p, s); }
  NMG_TRY(check_launch(h));
  NMG_TRY(h->comm->sum_f64(h->rsum.p, nrhs, h->dscratch.p, s));
  { Prof p(h, NMG_K_MISC, s); relres_sums(nrhs, h->rsum.p, h->ysq.p, relres, tol, active, s); }
  return check_launch(h);
}
// x += inner correction (fp64)
nmg_status outer_update(nmg_hierarchy* h, int nrhs, double* x, const uint8_t* active, cudaStream_t s) {
  if (!h->slab) {
    const int64_t N = h->N[0];
    { Prof p(h, NMG_K_MISC, s); update_x(nrhs, (int)N, x, N, h->wx[0]->p, N, active, s); }
    return check_launch(h);
  }
  { Prof p(h, NMG_K_MISC, s);
    update_slab(nrhs, (int64_t)h->R[0] * h->n[0], x, h->sx[0]->p, slab_img(h, 0), (int64_t)h->HS * h->n[0], active, s); }
  return check_launch(h);
}

nmg_status check_ready(nmg_hierarchy* h, int nrhs) {
  if (!h) return fail(NMG_ERR_INVALID_ARG, "null handle");
  if (h->poisoned) return fail(NMG_ERR_CUDA, "handle poisoned by an earlier CUDA error");
  if (nrhs < 0 || nrhs > h->d.max_rhs) return fail(NMG_ERR_INVALID_ARG, "nrhs %d outside [0, max_rhs=%d]", nrhs, h->d.max_rhs);
  for (int l = 0; l < h->L - 1; ++l)
    if (!h->w_loaded[l]) return fail(NMG_ERR_NO_WEIGHTS, "level %d has no smoother weights", l + 1);
  NMG_CUDA(cudaSetDevice(h->d.device));
  return NMG_OK;
}

// one outer step: residual (+relres/active), inner cycle, masked update
// (relres: where the relative residuals go, default h->relres; a lane writes its slice of the
// parent's array)
nmg_status outer_step(nmg_hierarchy* h, int nrhs, const double* y, double* x, double tol, bool use_active,
                      cudaStream_t s, double* relres = nullptr) {
  NMG_TRY(outer_residual(h, nrhs, y, x, nullptr, true, s));
  NMG_TRY(relres_fin(h, nrhs, tol, h->active.p, relres ? relres : h->relres.p, s));
  NMG_TRY(inner_cycle(h, nrhs, s));
  return outer_update(h, nrhs, x, use_active ? h->active.p : nullptr, s);
}

nmg_status debug_2d(nmg_hierarchy* h, int l, int op, int nrhs, const float* fin, float* fout, cudaStream_t s) {
  const int n = h->n[l];
  const bool smoothed = l < h->L - 1;
  const size_t bytes = sizeof(float) * (size_t)nrhs * n * n;
  switch (op) {
    case NMG_OP_APPLY:
    case NMG_OP_RESIDUAL:
      if (!smoothed) return fail(NMG_ERR_INVALID_ARG, "no fp32 operator stored at the coarsest level");
      return apply2d(h, l, nrhs, fin, op == NMG_OP_RESIDUAL ? fout : nullptr, fout, s, op == NMG_OP_RESIDUAL);
    case NMG_OP_RESTRICT:
      if (!smoothed) return fail(NMG_ERR_INVALID_ARG, "no coarser level");
      { Prof p(h, NMG_K_TRANSFER, s); restrict2d(nrhs, n, fin, fout, s); }
      return check_launch(h);
    case NMG_OP_PROLONG:
      if (!smoothed) return fail(NMG_ERR_INVALID_ARG, "no coarser level");
      { Prof p(h, NMG_K_TRANSFER, s); prolong_add2d(nrhs, n / 2, fin, fout, s); }
      return check_launch(h);
    case NMG_OP_FILTER:
      if (!smoothed) return fail(NMG_ERR_INVALID_ARG, "no filter at the coarsest level");
      { Prof p(h, NMG_K_FILTER, s); real_to_complex(nrhs, n, fin, h->Z.p, s); }
      { Prof p(h, NMG_K_FILTER, s, 3); filter2d(nrhs, n, h->Z.p, h->tw.p, h->tw_n, fout, false, s, nullptr); }
      return check_launch(h);
    case NMG_OP_CNN:
    case NMG_OP_SMOOTH:
      if (!smoothed || !h->w_loaded[l]) return fail(NMG_ERR_NO_WEIGHTS, "no smoother at level %d", l + 1);
      return smooth2d(h, l, nrhs, fin, fout, op == NMG_OP_SMOOTH, s, op == NMG_OP_SMOOTH, op == NMG_OP_SMOOTH);
    case NMG_OP_COARSE:
      if (smoothed) return fail(NMG_ERR_INVALID_ARG, "COARSE needs level == L");
      { Prof p(h, NMG_K_COARSE, s); coarse_solve(h, nrhs, fin, h->nc, fout, h->nc, s); }
      return check_launch(h);
    case NMG_OP_CYCLE0:
      for (int q = l; q < h->L - 1; ++q)
        if (!h->w_loaded[q]) return fail(NMG_ERR_NO_WEIGHTS, "level %d has no smoother", q + 1);
      NMG_CUDA(cudaMemcpyAsync(h->wy[l]->p, fin, bytes, cudaMemcpyDeviceToDevice, s));
      NMG_TRY(cycle_level_2d(h, l, nrhs, s));
      NMG_CUDA(cudaMemcpyAsync(fout, h->wx[l]->p, bytes, cudaMemcpyDeviceToDevice, s));
      return NMG_OK;
    default:
      return fail(NMG_ERR_INVALID_ARG, "unknown op %d", op);
  }
}

}  // namespace

// ======================================================================= C ABI
namespace {

// set while nmg_create_hierarchy builds a lane or a slab handle: no RHS lanes of its own
thread_local bool t_no_lanes = false;

// One cycle through a cached CUDA graph: the first call with a given (nrhs, y, x, stream) runs
// eagerly, the second captures the whole cycle, later calls replay it (launch-latency bound
// small configs and coarse levels).
void drop_graphs(nmg_hierarchy* h) {
  for (auto& g : h->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  h->graphs.clear();
  for (auto& hk : h->lanes) drop_graphs(hk.get());
}

// NMG_PREC_FP64: one fused launch (cycle64.cu)
nmg_status cycle_fp64(nmg_hierarchy* h, int nrhs, const double* y, double* x, bool do_cycle, bool relres_after,
                      double tol, const uint8_t* active_in, uint8_t* active_out, cudaStream_t s) {
  Cycle64Args a{};
  a.n = h->d.n; a.L = h->L; a.nrhs = nrhs; a.nu1 = h->d.nu1; a.nu2 = h->d.nu2; a.filter = h->d.level_filter != 0;
  for (int l = 0; l < h->L - 1; ++l) {
    a.A[l] = l == 0 ? h->A64.p : h->A64l[l]->p;
    a.W[l] = h->W[l]->p;
  }
  a.Ainv = h->Ainv.p;
  a.y = y; a.x = x; a.relres = h->relres.p; a.tol = tol;
  a.active_in = active_in; a.active_out = active_out;
  a.do_cycle = do_cycle; a.relres_after = relres_after;
  { Prof p(h, NMG_K_SMOOTH, s); cycle64(a, s); }
  return check_launch(h);
}

// allow_lanes = false: the whole batch runs on this handle alone (the host-buffer pipeline runs
// its lane 0 this way while lanes 1..K-1 cycle their own RHS on the lane handles concurrently,
// so a lane handle is never used by two graphs at once).
nmg_status graph_cycle(nmg_hierarchy* h, int nrhs, const double* y, double* x, cudaStream_t s,
                       bool allow_lanes = true) {
  auto body = [&]() -> nmg_status {
    if (h->d.precision == NMG_PREC_FP64) return cycle_fp64(h, nrhs, y, x, true, false, -1.0, nullptr, nullptr, s);
    const int K = (int)h->lanes.size() + 1;
    const int gr = h->d.dim == 1 ? 128 : 2;             // lane granularity (1D: GEMM M tiles)
    if (K == 1 || !allow_lanes || h->prof_on || nrhs < K * gr || s == nullptr) {
      NMG_TRY(ynorms(h, nrhs, y, s));
      return outer_step(h, nrhs, y, x, -1.0, false, s);
    }
    // K lanes: RHS [off_k, off_k+1) on lane k (lane 0 = this handle on s, lane k > 0 on its
    // forked stream); the RHS are independent, so the lanes' kernels overlap
    int off[kMaxHostChunks + 1];
    for (int k = 0; k <= K; ++k) off[k] = std::min(nrhs, (nrhs * k / K + gr - 1) / gr * gr);
    off[K] = nrhs;
    const int64_t N = h->N[0];
    NMG_CUDA(cudaEventRecord(h->evf, s));
    nmg_status st = NMG_OK;
    const int mult = h->lane_tiles ? K : 1;     // concurrent GEMMs: tile width for the whole batch
    h->lane_mult = mult;
    for (int k = 1; k < K && st == NMG_OK; ++k) {
      nmg_hierarchy* hk = h->lanes[k - 1].get();
      const int cnt = off[k + 1] - off[k];
      if (cnt <= 0) continue;
      NMG_CUDA(cudaStreamWaitEvent(h->ls[k - 1], h->evf, 0));
      const int64_t l0 = hk->launches;
      hk->lane_mult = mult;
      st = ynorms(hk, cnt, y + off[k] * N, h->ls[k - 1]);
      if (st == NMG_OK)
        st = outer_step(hk, cnt, y + off[k] * N, x + off[k] * N, -1.0, false, h->ls[k - 1], h->relres.p + off[k]);
      hk->lane_mult = 1;
      h->launches += hk->launches - l0;
    }
    if (st == NMG_OK) st = ynorms(h, off[1], y, s);
    if (st == NMG_OK) st = outer_step(h, off[1], y, x, -1.0, false, s);
    h->lane_mult = 1;
    NMG_TRY(st);
    for (int k = 1; k < K; ++k) {
      NMG_CUDA(cudaEventRecord(h->evj[k - 1], h->ls[k - 1]));
      NMG_CUDA(cudaStreamWaitEvent(s, h->evj[k - 1], 0));
    }
    return NMG_OK;
  };
  if (!h->use_graph || h->slab || s == nullptr || h->prof_on) return body();
  nmg_hierarchy::GraphEntry* g = nullptr;
  for (auto& e : h->graphs)
    if (e.nrhs == nrhs && e.y == y && e.x == x && e.s == s && e.lanes == allow_lanes) g = &e;
  if (!g) {
    if (h->graphs.size() >= 24) {   // host-entry chunks (up to 16) + the device-entry batch
      auto old = h->graphs.begin();
      for (auto it = h->graphs.begin(); it != h->graphs.end(); ++it)
        if (it->used < old->used) old = it;
      if (old->exec) cudaGraphExecDestroy(old->exec);
      h->graphs.erase(old);
    }
    h->graphs.push_back({nrhs, y, x, s, allow_lanes, 0, nullptr, 0, 0});
    g = &h->graphs.back();
  }
  g->used = ++h->g_clock;
  if (g->exec) {
    NMG_CUDA(cudaGraphLaunch(g->exec, s));
    h->launches += g->launches;
    return NMG_OK;
  }
  if (g->seen++ == 0) return body();
  const int64_t l0 = h->launches;
  if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    h->use_graph = false;
    return body();
  }
  nmg_status st = body();
  cudaGraph_t gr = nullptr;
  cudaError_t e = cudaStreamEndCapture(s, &gr);
  if (st != NMG_OK || e != cudaSuccess || !gr) {
    if (gr) cudaGraphDestroy(gr);
    cudaGetLastError();
    h->use_graph = false;
    h->launches = l0;
    h->poisoned = false;
    return body();
  }
  g->launches = h->launches - l0;
  h->launches = l0;
  e = cudaGraphInstantiate(&g->exec, gr, 0);
  cudaGraphDestroy(gr);
  if (e != cudaSuccess) {
    cudaGetLastError();
    g->exec = nullptr;
    h->use_graph = false;
    return body();
  }
  NMG_CUDA(cudaGraphLaunch(g->exec, s));
  h->launches += g->launches;
  return NMG_OK;
}

}  // namespace

extern "C" {

const char* nmg_last_error(void) { return g_err.c_str(); }
const char* nmg_version(void) { return "nmg-b200 0.1 (sm_100a)"; }
int64_t nmg_launch_count(const nmg_hierarchy* h) { return h ? h->launches : 0; }

nmg_status nmg_create_hierarchy(const nmg_problem_desc* desc, const double* factors, nmg_hierarchy** out) {
  g_err.clear();
  if (!desc || !factors || !out) return fail(NMG_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  const nmg_problem_desc& d = *desc;
  if (d.dim != 1 && d.dim != 2) return fail(NMG_ERR_INVALID_ARG, "dim must be 1 or 2 (got %d)", d.dim);
  if (d.n < 2 || (d.n & (d.n - 1))) return fail(NMG_ERR_INVALID_ARG, "n must be a power of two >= 2 (got %d)", d.n);
  if (d.levels < 1 || (d.n >> (d.levels - 1)) < 2)
    return fail(NMG_ERR_INVALID_ARG, "levels %d too deep for n = %d", d.levels, d.n);
  if (!(d.alpha > 0.0)) return fail(NMG_ERR_INVALID_ARG, "alpha must be > 0");
  if (d.nu1 < 0 || d.nu2 < 0 || d.max_rhs < 1) return fail(NMG_ERR_INVALID_ARG, "bad nu1/nu2/max_rhs");
  const int nc = d.n >> (d.levels - 1);
  const int Nc = d.dim == 1 ? nc : nc * nc;
  if (Nc > 256) return fail(NMG_ERR_UNSUPPORTED, "coarsest system %d > 256 unknowns", Nc);
  if (d.dim == 1 && d.n > 8192) return fail(NMG_ERR_UNSUPPORTED, "1D n > 8192");
  if (d.dim == 2 && d.n > 1024) return fail(NMG_ERR_UNSUPPORTED, "2D n > 1024");

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= d.device || d.device < 0)
    return fail(NMG_ERR_CUDA, "no CUDA device %d visible (no CPU fallback exists)", d.device);
  cudaDeviceProp prop;
  NMG_CUDA(cudaGetDeviceProperties(&prop, d.device));
  if (prop.major != 10) return fail(NMG_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a", d.device, prop.major, prop.minor);
  NMG_CUDA(cudaSetDevice(d.device));

  if (d.precision != NMG_PREC_MIXED && d.precision != NMG_PREC_FP64)
    return fail(NMG_ERR_INVALID_ARG, "precision must be NMG_PREC_MIXED or NMG_PREC_FP64 (got %d)", d.precision);
  if (d.precision == NMG_PREC_FP64 && (d.dim != 1 || d.n > 1024))
    return fail(NMG_ERR_UNSUPPORTED, "NMG_PREC_FP64 is implemented for 1D problems with n <= 1024");

  auto h = std::make_unique<nmg_hierarchy>();
  h->d = d;
  if (d.tuning) h->tune = *d.tuning;
  h->d.tuning = nullptr;                                 // the caller's struct is not kept
  h->L = d.levels;
  for (int l = 0; l < h->L; ++l) {
    h->n.push_back(d.n >> l);
    h->N.push_back(d.dim == 1 ? (int64_t)(d.n >> l) : (int64_t)(d.n >> l) * (d.n >> l));
  }
  h->nc = Nc;
  {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d.device);
    h->num_sms = sms > 0 ? sms : 148;
  }
  const int n = d.n;
  const size_t nn = (size_t)n * n;

  std::vector<double> Acoarse;
  if (d.dim == 1 && d.precision == NMG_PREC_MIXED && h->tune.fused_coarse > 0) {
    // opt-in: the coarse levels (n_l <= tune.fused_coarse) run as one fused fp64 sub-cycle
    // kernel per RHS (cycle64.cu).  Measured slower for the BASELINE shapes (cfg 1, n_l <= 512:
    // 2.57 vs 1.42 ms per step at 1024 RHS, 0.66 vs 0.58 ms at 128): one CTA per RHS streams
    // the fp64 operator from L2 for every matvec, where the batched GEMMs read it once per tile
    for (int l = 0; l < h->L - 1; ++l)
      if (h->n[l] <= h->tune.fused_coarse) { h->l_fuse = l; break; }
  }
  if (d.dim == 1) {
    std::vector<double> A(factors, factors + nn);
    for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += d.alpha;
    NMG_TRY(h->A64.upload(A.data(), nn));
    for (int l = 0; l < h->L - 1; ++l) {
      const int nl = h->n[l];
      h->A32.emplace_back(new DevBuf<float>());
      h->AP32.emplace_back(new DevBuf<float>());
      NMG_TRY(h->A32.back()->upload(to_f32(A).data(), (size_t)nl * nl));
      std::vector<double> AP, Ac;
      host_prolong_cols(A, nl, nl, AP);                 // A_l P_l : nl x nl/2
      NMG_TRY(h->AP32.back()->upload(to_f32(AP).data(), (size_t)nl * (nl / 2)));
      {
        std::vector<float> hi, lo;
        h->A32h.emplace_back(new DevBuf<float>()); h->A32l.emplace_back(new DevBuf<float>());
        h->AP32h.emplace_back(new DevBuf<float>()); h->AP32l.emplace_back(new DevBuf<float>());
        split_host(A, hi, lo);
        NMG_TRY(h->A32h.back()->upload(hi.data(), hi.size()));
        NMG_TRY(h->A32l.back()->upload(lo.data(), lo.size()));
        split_host(AP, hi, lo);
        NMG_TRY(h->AP32h.back()->upload(hi.data(), hi.size()));
        NMG_TRY(h->AP32l.back()->upload(lo.data(), lo.size()));
      }
      {
        // f16 hi/lo planes with a power-of-two scale per row (FP16x3 GEMM operand W)
        auto f16op = [&](const std::vector<double>& M, int rows, int cols) -> std::unique_ptr<nmg_hierarchy::F16Op> {
          std::unique_ptr<nmg_hierarchy::F16Op> op(new nmg_hierarchy::F16Op());
          std::vector<uint16_t> hi((size_t)rows * cols), lo((size_t)rows * cols);
          std::vector<float> winv(rows);
          for (int r = 0; r < rows; ++r) {
            double mx = 0.0;
            for (int c = 0; c < cols; ++c) mx = std::max(mx, std::fabs(M[(size_t)r * cols + c]));
            const float T = pow2_scale(mx);
            winv[r] = 1.0f / T;
            for (int c = 0; c < cols; ++c) {
              const float v = (float)M[(size_t)r * cols + c] * T;
              hi[(size_t)r * cols + c] = f16_rn(v);
              lo[(size_t)r * cols + c] = f16_rn(v - f16_f(hi[(size_t)r * cols + c]));
            }
          }
          // per 64-row tile: the 32-element K blocks holding a nonzero hi or lo value (the
          // Gaussian operators' far off-diagonal entries flush to zero in both f16 planes: the
          // FP16x3 GEMM skips those blocks, whose products are exact zeros)
          std::vector<int2> kr(rows / 64);
          for (int t = 0; t < rows / 64; ++t) {
            int lo_k = cols, hi_k = 0;
            for (int r = t * 64; r < (t + 1) * 64; ++r)
              for (int c = 0; c < cols; ++c)
                if ((hi[(size_t)r * cols + c] | lo[(size_t)r * cols + c]) & 0x7fffu) {
                  lo_k = std::min(lo_k, c);
                  hi_k = std::max(hi_k, c + 1);
                }
            if (hi_k <= lo_k) { lo_k = 0; hi_k = 32; }
            kr[t] = make_int2(lo_k / 32 * 32, (hi_k + 31) / 32 * 32);
          }
          if (op->h.upload(hi.data(), hi.size()) != NMG_OK || op->l.upload(lo.data(), lo.size()) != NMG_OK ||
              op->winv.upload(winv.data(), winv.size()) != NMG_OK ||
              (rows % 64 == 0 && op->kr.upload(kr.data(), kr.size()) != NMG_OK))
            return nullptr;
          return op;
        };
        h->A16.push_back(f16op(A, nl, nl));
        h->AP16.push_back(f16op(AP, nl, nl / 2));
        if (!h->A16.back() || !h->AP16.back()) return fail(NMG_ERR_OOM, "f16 operator planes");
      }
      host_restrict_rows(AP, nl, nl / 2, Ac);           // R A P
      A.swap(Ac);
      while ((int)h->A64l.size() < l + 2) h->A64l.emplace_back(new DevBuf<double>());
      if (l + 1 < h->L - 1 && (d.precision == NMG_PREC_FP64 || (h->l_fuse >= 0 && l + 1 >= h->l_fuse)))
        NMG_TRY(h->A64l[l + 1]->upload(A.data(), A.size()));
    }
    Acoarse = A;
  } else {
    std::vector<double> B(factors, factors + nn), C(factors + nn, factors + 2 * nn), Q(nn, 0.0);
    for (int i = 0; i < n; ++i) Q[(size_t)i * n + i] = 1.0;
    NMG_TRY(h->B64.upload(B.data(), nn));
    NMG_TRY(h->C64.upload(C.data(), nn));
    for (int l = 0; l < h->L - 1; ++l) {
      const int nl = h->n[l];
      const size_t nn2 = (size_t)nl * nl;
      auto up = [&](std::vector<std::unique_ptr<DevBuf<float>>>& v, const float* src) -> nmg_status {
        v.emplace_back(new DevBuf<float>());
        return v.back()->upload(src, nn2);
      };
      NMG_TRY(up(h->B32, to_f32(B).data()));
      NMG_TRY(up(h->C32, to_f32(C).data()));
      NMG_TRY(up(h->Q32, to_f32(Q).data()));
      std::vector<float> hi, lo;
      split_host(B, hi, lo);
      NMG_TRY(up(h->B32h, hi.data()));
      NMG_TRY(up(h->B32l, lo.data()));
      auto kr_up = [&](std::vector<std::unique_ptr<DevBuf<int2>>>& v) -> nmg_status {
        v.emplace_back(new DevBuf<int2>());
        if (nl % 64) return NMG_OK;
        const std::vector<int2> kr = zero_kranges_f32(hi, lo, nl, nl, 16);
        return v.back()->upload(kr.data(), kr.size());
      };
      NMG_TRY(kr_up(h->Bkr));
      split_host(C, hi, lo);
      NMG_TRY(up(h->C32h, hi.data()));
      NMG_TRY(up(h->C32l, lo.data()));
      NMG_TRY(kr_up(h->Ckr));
      int hb = 0;
      for (int i = 0; i < nl; ++i)
        for (int j = 0; j < nl; ++j)
          if (Q[(size_t)i * nl + j] != 0.0) hb = std::max(hb, std::abs(i - j));
      h->qhb.push_back(hb);
      std::vector<double> t;
      host_galerkin(B, nl, t); B.swap(t);
      host_galerkin(C, nl, t); C.swap(t);
      host_galerkin(Q, nl, t); Q.swap(t);
    }
    Acoarse.assign((size_t)Nc * Nc, 0.0);
    for (int i2 = 0; i2 < nc; ++i2)
      for (int i1 = 0; i1 < nc; ++i1)
        for (int j2 = 0; j2 < nc; ++j2)
          for (int j1 = 0; j1 < nc; ++j1)
            Acoarse[(size_t)(i1 + nc * i2) * Nc + (j1 + nc * j2)] =
                B[(size_t)i2 * nc + j2] * C[(size_t)i1 * nc + j1] +
                d.alpha * Q[(size_t)i2 * nc + j2] * Q[(size_t)i1 * nc + j1];
  }
  int bad = -1;
  if (!host_cholesky(Acoarse, Nc, &bad))
    return fail(NMG_ERR_NOT_SPD, "coarsest operator not SPD: Cholesky pivot %d <= 0", bad);
  std::vector<double> Lt((size_t)Nc * Nc);
  for (int i = 0; i < Nc; ++i)
    for (int j = 0; j < Nc; ++j) Lt[(size_t)j * Nc + i] = Acoarse[(size_t)i * Nc + j];
  NMG_TRY(h->Lrow.upload(Acoarse.data(), Acoarse.size()));
  NMG_TRY(h->Lcol.upload(Lt.data(), Lt.size()));
  {
    // explicit inverse A_L^{-1} = L^{-T} L^{-1} (fp64, symmetric), column by column
    h->coarse_inv = h->tune.coarse_subst == 0 || d.precision == NMG_PREC_FP64 || h->l_fuse >= 0;
    if (h->coarse_inv) {
      std::vector<double> inv((size_t)Nc * Nc), z(Nc);
      for (int j = 0; j < Nc; ++j) {
        for (int i = 0; i < Nc; ++i) {           // L z = e_j
          double v = (i == j) ? 1.0 : 0.0;
          for (int k = 0; k < i; ++k) v -= Acoarse[(size_t)i * Nc + k] * z[k];
          z[i] = v / Acoarse[(size_t)i * Nc + i];
        }
        for (int i = Nc - 1; i >= 0; --i) {      // L^T x = z
          double v = z[i];
          for (int k = i + 1; k < Nc; ++k) v -= Acoarse[(size_t)k * Nc + i] * z[k];
          z[i] = v / Acoarse[(size_t)i * Nc + i];
        }
        for (int i = 0; i < Nc; ++i) inv[(size_t)i * Nc + j] = z[i];
      }
      for (int i = 0; i < Nc; ++i)               // symmetrise (exact inverse is symmetric)
        for (int j = i + 1; j < Nc; ++j) {
          const double v = 0.5 * (inv[(size_t)i * Nc + j] + inv[(size_t)j * Nc + i]);
          inv[(size_t)i * Nc + j] = inv[(size_t)j * Nc + i] = v;
        }
      NMG_TRY(h->Ainv.upload(inv.data(), inv.size()));
    }
  }

  // twiddles exp(-2 pi i k / tw_n), k < tw_n / 2
  h->tw_n = n;
  {
    std::vector<float2> tw(std::max(1, n / 2));
    for (int k = 0; k < n / 2; ++k) {
      const double ang = -2.0 * M_PI * (double)k / (double)n;
      tw[k] = make_float2((float)std::cos(ang), (float)std::sin(ang));
    }
    NMG_TRY(h->tw.upload(tw.data(), tw.size()));
  }
  // weights slots
  h->w_loaded.assign(std::max(0, h->L - 1), 0);
  for (int l = 0; l < h->L - 1; ++l) h->W.emplace_back(new DevBuf<float>());
  // workspaces
  const size_t B = (size_t)d.max_rhs;
  for (int l = 0; l < h->L; ++l) {
    for (auto* v : {&h->wy, &h->wx, &h->wr, &h->wb}) {
      v->emplace_back(new DevBuf<float>());
      const bool need = (v == &h->wy || v == &h->wx) || l < h->L - 1;
      if (need) NMG_TRY(v->back()->alloc(B * (size_t)h->N[l]));
    }
  }
  h->use_tc = h->tune.simt_gemm == 0;
  h->use_graph = h->tune.no_graphs == 0;
  h->smooth_f16 = h->use_tc && h->tune.ffma_cnn == 0;
  if (d.dim == 1) h->gemm_f16 = h->use_tc;            // 1D inner applies: FP16x3 on tcgen05
  if (d.dim == 1) {
    h->mAh.resize(h->L); h->mAl.resize(h->L); h->mAPh.resize(h->L); h->mAPl.resize(h->L);
    h->mAh64.resize(h->L); h->mAl64.resize(h->L); h->mAPh64.resize(h->L); h->mAPl64.resize(h->L);
    h->mXh.resize(h->L); h->mXl.resize(h->L);
    h->mX16h.resize(h->L); h->mX16l.resize(h->L);
    for (int l = 0; l < h->L; ++l) {
      const int nl = h->n[l];
      h->sxh.emplace_back(new DevBuf<float>());
      h->sxl.emplace_back(new DevBuf<float>());
      h->sx16h.emplace_back(new DevBuf<uint16_t>());
      h->sx16l.emplace_back(new DevBuf<uint16_t>());
      h->sxinv.emplace_back(new DevBuf<float>());
      if (nl % 16 != 0) continue;   // small levels use the SIMT kernel
      if (h->gemm_f16) {
        NMG_TRY(h->sx16h.back()->alloc(B * nl));
        NMG_TRY(h->sx16l.back()->alloc(B * nl));
        NMG_TRY(h->sxinv.back()->alloc(B));
        NMG_TRY(make_map16(&h->mX16h[l], h->sx16h.back()->p, (int64_t)B, nl, tc_gemm_block_m()));
        NMG_TRY(make_map16(&h->mX16l[l], h->sx16l.back()->p, (int64_t)B, nl, tc_gemm_block_m()));
        if (l < h->L - 1) {
          for (auto* op : {h->A16[l].get(), h->AP16[l].get()}) {
            const int cols = op == h->A16[l].get() ? nl : nl / 2;
            NMG_TRY(make_map16(&op->m256h, op->h.p, nl, cols, 256));
            NMG_TRY(make_map16(&op->m256l, op->l.p, nl, cols, 256));
            NMG_TRY(make_map16(&op->m64h, op->h.p, nl, cols, 64));
            NMG_TRY(make_map16(&op->m64l, op->l.p, nl, cols, 64));
            NMG_TRY(make_map16(&op->m128h, op->h.p, nl, cols, 128));
            NMG_TRY(make_map16(&op->m128l, op->l.p, nl, cols, 128));
          }
        }
      }
      NMG_TRY(h->sxh.back()->alloc(B * nl));
      NMG_TRY(h->sxl.back()->alloc(B * nl));
      NMG_TRY(make_map(&h->mXh[l], h->sxh.back()->p, (int64_t)B, nl, tc_gemm_block_m()));
      NMG_TRY(make_map(&h->mXl[l], h->sxl.back()->p, (int64_t)B, nl, tc_gemm_block_m()));
      if (l < h->L - 1) {
        NMG_TRY(make_map(&h->mAh[l], h->A32h[l]->p, nl, nl, 256));
        NMG_TRY(make_map(&h->mAl[l], h->A32l[l]->p, nl, nl, 256));
        NMG_TRY(make_map(&h->mAh64[l], h->A32h[l]->p, nl, nl, 64));
        NMG_TRY(make_map(&h->mAl64[l], h->A32l[l]->p, nl, nl, 64));
        if ((nl / 2) % 16 == 0) {
          NMG_TRY(make_map(&h->mAPh[l], h->AP32h[l]->p, nl, nl / 2, 256));
          NMG_TRY(make_map(&h->mAPl[l], h->AP32l[l]->p, nl, nl / 2, 256));
          NMG_TRY(make_map(&h->mAPh64[l], h->AP32h[l]->p, nl, nl / 2, 64));
          NMG_TRY(make_map(&h->mAPl64[l], h->AP32l[l]->p, nl, nl / 2, 64));
        }
      }
    }
  }
  if (d.dim == 2) {
    h->mBh.resize(h->L); h->mBl.resize(h->L); h->mCh.resize(h->L); h->mCl.resize(h->L);
    h->mTh.resize(h->L); h->mTl.resize(h->L); h->mXh.resize(h->L); h->mXl.resize(h->L);
    h->mBh64.resize(h->L); h->mBl64.resize(h->L); h->mCh64.resize(h->L); h->mCl64.resize(h->L);
    h->mKBh.resize(h->L); h->mKBl.resize(h->L); h->mKCh.resize(h->L); h->mKCl.resize(h->L);
    h->use_kron = h->use_tc && h->tune.no_kron == 0;
    for (int l = 0; l < h->L; ++l) {
      const int nl = h->n[l];
      for (auto* v : {&h->sxh, &h->sxl, &h->tth, &h->ttl}) {
        v->emplace_back(new DevBuf<float>());
        if (l < h->L - 1) NMG_TRY(v->back()->alloc(B * (size_t)nl * nl));
      }
      if (l >= h->L - 1 || nl % 16 != 0) continue;
      const int64_t rows = (int64_t)B * nl;
      NMG_TRY(make_map(&h->mXh[l], h->sxh[l]->p, rows, nl, tc_gemm_block_m()));
      NMG_TRY(make_map(&h->mXl[l], h->sxl[l]->p, rows, nl, tc_gemm_block_m()));
      NMG_TRY(make_map(&h->mTh[l], h->tth[l]->p, rows, nl, tc_gemm_block_m()));
      NMG_TRY(make_map(&h->mTl[l], h->ttl[l]->p, rows, nl, tc_gemm_block_m()));
      NMG_TRY(make_map(&h->mBh[l], h->B32h[l]->p, nl, nl, 256));
      NMG_TRY(make_map(&h->mBl[l], h->B32l[l]->p, nl, nl, 256));
      NMG_TRY(make_map(&h->mCh[l], h->C32h[l]->p, nl, nl, 256));
      NMG_TRY(make_map(&h->mCl[l], h->C32l[l]->p, nl, nl, 256));
      NMG_TRY(make_map(&h->mBh64[l], h->B32h[l]->p, nl, nl, 64));
      NMG_TRY(make_map(&h->mBl64[l], h->B32l[l]->p, nl, nl, 64));
      NMG_TRY(make_map(&h->mCh64[l], h->C32h[l]->p, nl, nl, 64));
      NMG_TRY(make_map(&h->mCl64[l], h->C32l[l]->p, nl, nl, 64));
      if (kron_supported(nl, h->qhb[l])) {
        const int kb = kron_tile_n(nl);
        NMG_TRY(make_map(&h->mKBh[l], h->B32h[l]->p, nl, nl, kb));
        NMG_TRY(make_map(&h->mKBl[l], h->B32l[l]->p, nl, nl, kb));
        NMG_TRY(make_map(&h->mKCh[l], h->C32h[l]->p, nl, nl, kb));
        NMG_TRY(make_map(&h->mKCl[l], h->C32l[l]->p, nl, nl, kb));
      }
    }
    NMG_TRY(h->Z.alloc(B * (size_t)h->N[0] / 2));          // level filter: [B][n/2][n] complex
    NMG_TRY(h->snorm.alloc(B));
    NMG_TRY(h->spart.alloc(B * 64));
    NMG_TRY(h->T64.alloc(B * (size_t)h->N[0]));
    h->rows_per_rhs = n;
    // FP16x3 column-strip kernels for the levels strip_level() accepts; the rest FFMA (cnn2d)
    h->conv_bf = h->use_tc && h->tune.ffma_cnn == 0;
    if (h->conv_bf) {
      h->mA2h.resize(h->L); h->mA2l.resize(h->L);
      for (int l = 0; l < h->L - 1; ++l) h->WB.emplace_back(new DevBuf<uint16_t>());
    }
  }
  if (d.dim == 1) {
    h->ozaki = h->use_tc && n % 128 == 0 && /* CTA pairs along N */ h->tune.fp64_dmma == 0;
    if (h->ozaki) {
      // W digits of A (rows n, K = n), host: exponent per row, S truncation digits
      const int S = ozaki_digits();
      std::vector<double> A(factors, factors + nn);
      for (int i = 0; i < n; ++i) A[(size_t)i * n + i] += d.alpha;
      std::vector<int8_t> dig;
      std::vector<int> ew;
      host_digits(A, n, S, dig, ew);
      NMG_TRY(h->wdig.upload(dig.data(), dig.size()));
      NMG_TRY(h->wexp.upload(ew.data(), ew.size()));
      const std::vector<int2> kr = digit_kranges(dig, S, n, n, ozaki_bn(), ozaki_bk());
      NMG_TRY(h->wkr.upload(kr.data(), kr.size()));
      NMG_TRY(h->xdig.alloc((size_t)S * B * n));
      NMG_TRY(h->xexp.alloc(B));
      NMG_TRY(make_digit_map(&h->mWd, h->wdig.p, S, n, n, ozaki_bn()));
      NMG_TRY(make_digit_map(&h->mXd, h->xdig.p, S, (int64_t)B, n, 64, 1));   // half tiles, one digit per box
    }
  }
  if (d.dim == 2) {
    // fp64 outer residual as two Ozaki int8 passes (T = X C^T, then y - T B^T - alpha x);
    // tune.fp64_dmma keeps the DMMA kernel
    h->ozaki2d = h->use_tc && n % 128 == 0 && h->tune.fp64_dmma == 0;
    if (h->ozaki2d) {
      const int S = ozaki_digits();
      std::vector<int8_t> dig;
      std::vector<int> ew;
      std::vector<double> Bm(factors, factors + nn), Cm(factors + nn, factors + 2 * nn);
      host_digits(Cm, n, S, dig, ew);
      NMG_TRY(h->wdig.upload(dig.data(), dig.size()));
      NMG_TRY(h->wexp.upload(ew.data(), ew.size()));
      std::vector<int2> kr = digit_kranges(dig, S, n, n, ozaki_bn(), ozaki_bk());
      NMG_TRY(h->wkr.upload(kr.data(), kr.size()));
      host_digits(Bm, n, S, dig, ew);
      NMG_TRY(h->wdigB.upload(dig.data(), dig.size()));
      NMG_TRY(h->wexpB.upload(ew.data(), ew.size()));
      kr = digit_kranges(dig, S, n, n, ozaki_bn(), ozaki_bk());
      NMG_TRY(h->wkrB.upload(kr.data(), kr.size()));
      NMG_TRY(h->xdig.alloc((size_t)S * B * nn));
      NMG_TRY(h->xexp.alloc(B * n));
      NMG_TRY(make_digit_map(&h->mWd, h->wdig.p, S, n, n, ozaki_bn()));
      NMG_TRY(make_digit_map(&h->mWdB, h->wdigB.p, S, n, n, ozaki_bn()));
      NMG_TRY(make_digit_map(&h->mXd, h->xdig.p, S, (int64_t)B * n, n, 64, 1));
    }
  }
  h->split_fresh.assign(h->L, 0);
  h->ntiles = gemm_f64_ntiles(d.dim == 1 ? (int)h->N[0] : n);
  h->ntiles_oz = (d.dim == 1 ? (int)h->N[0] : n) / ozaki_bn();
  NMG_TRY(h->part.alloc(B * (size_t)std::max(h->ntiles, h->ntiles_oz) * (size_t)h->rows_per_rhs));
  NMG_TRY(h->ynorm.alloc(B));
  NMG_TRY(h->ywork.alloc(B * 64));
  NMG_TRY(h->relres.alloc(B));
  NMG_TRY(h->active.alloc(B));
  {
    const int tl = h->tune.lanes;
    int K = (t_no_lanes || d.precision == NMG_PREC_FP64) ? 1 : tl > 0 ? std::min(8, tl) : 4;
    if (d.dim != 1 && K > 1) {
      // 2D: two lanes by default while the batch is small enough that a second set of lane
      // workspaces is cheap (cfg 2, 4: same device time, the host entry overlaps more)
      if (tl == 0) K = (int64_t)d.max_rhs * h->N[0] <= ((int64_t)1 << 26) ? 2 : 1;
      while (K > 1 && d.max_rhs < K * 16) --K;            // lanes of >= 16 RHS
    }
    while (d.dim == 1 && K > 1 && d.max_rhs < K * 256) --K;   // 1D lanes of >= 256 RHS
    if (K > 1) {
      nmg_problem_desc d2 = d;
      d2.max_rhs = (d.max_rhs + K - 1) / K + (d.dim == 1 ? 128 : 2);   // a lane's share (rounded up)
      d2.tuning = &h->tune;
      t_no_lanes = true;                                 // a lane itself has no lanes
      nmg_status st = NMG_OK;
      for (int k = 1; k < K && st == NMG_OK; ++k) {
        nmg_hierarchy* raw = nullptr;
        st = nmg_create_hierarchy(&d2, factors, &raw);
        if (st == NMG_OK) h->lanes.emplace_back(raw);
      }
      t_no_lanes = false;
      NMG_TRY(st);
      NMG_CUDA(cudaEventCreateWithFlags(&h->evf, cudaEventDisableTiming));
      for (int k = 1; k < K; ++k) {
        cudaStream_t x;
        cudaEvent_t e;
        NMG_CUDA(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking));
        h->ls.push_back(x);
        NMG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        h->evj.push_back(e);
      }
    }
  }
  if (!t_no_lanes) {
    // staging and copy streams of the host-buffer entry nmg_vcycles_host (no lazy allocation)
    const size_t cnt = (size_t)d.max_rhs * h->N[0];
    NMG_TRY(h->hy.alloc(cnt));
    NMG_TRY(h->hx.alloc(cnt));
    NMG_TRY(h->cmap.alloc((size_t)d.max_rhs));
    NMG_CUDA(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
    NMG_CUDA(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
    h->hev.resize(2 * kMaxHostChunks + 2);
    for (auto& e : h->hev) NMG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  NMG_CUDA(cudaDeviceSynchronize());
  *out = h.release();
  return NMG_OK;
}

nmg_status nmg_create_hierarchy_slab(const nmg_problem_desc* desc, const double* factors, nmg_comm* comm,
                                     nmg_hierarchy** out) {
  g_err.clear();
  if (!desc || !factors || !comm || !out) return fail(NMG_ERR_INVALID_ARG, "null argument");
  *out = nullptr;
  if (desc->dim != 2) return fail(NMG_ERR_UNSUPPORTED, "the slab-sharded mode is 2D only");
  const int W = comm->world;
  if (desc->n % W != 0 || desc->n / W < 32 || (desc->n / W) % 32 != 0)
    return fail(NMG_ERR_UNSUPPORTED, "slab mode needs n / world to be a multiple of 32 (n = %d, world = %d)", desc->n, W);
  nmg_hierarchy* raw = nullptr;
  t_no_lanes = true;                                     // the slab cycle has no RHS lanes
  const nmg_status cst = nmg_create_hierarchy(desc, factors, &raw);
  t_no_lanes = false;
  NMG_TRY(cst);
  std::unique_ptr<nmg_hierarchy> h(raw);
  if (!h->use_kron) return fail(NMG_ERR_UNSUPPORTED, "slab mode needs the tcgen05 Kronecker apply (NMG_KRON != 0)");
  h->slab = true;
  h->comm = comm;
  h->nw = W;
  h->rank = comm->rank;
  h->use_graph = false;
  // sharded levels: smoothed levels whose slab keeps >= 32 rows and whose width the strip CNN serves
  h->Ls = 0;
  for (int l = 0; l < h->L - 1; ++l) {
    const int nl = h->n[l];
    if (nl % W != 0 || nl / W < 32 || nl % 128 != 0 || !kron_supported(nl, h->qhb[l]) || (nl / 2) % W != 0) break;
    h->R.push_back(nl / W);
    h->Ls = l + 1;
  }
  if (h->Ls == 0) return fail(NMG_ERR_UNSUPPORTED, "no level can be sharded (n = %d, world = %d)", desc->n, W);
  const size_t B = (size_t)h->d.max_rhs;
  const int H = h->HS;
  const int n0 = h->n[0], R0 = h->R[0];
  h->mKBhS.resize(h->Ls); h->mKBlS.resize(h->Ls);
  for (int l = 0; l < h->Ls; ++l) {
    const int nl = h->n[l], R = h->R[l];
    for (auto* v : {&h->sy, &h->sx, &h->sr, &h->sb}) {
      v->emplace_back(new DevBuf<float>());
      NMG_TRY(v->back()->alloc(B * (size_t)(R + 2 * H) * nl));
      NMG_CUDA(cudaMemset(v->back()->p, 0, sizeof(float) * v->back()->n));
    }
    NMG_TRY(make_map(&h->mKBhS[l], h->B32h[l]->p, nl, nl, kron_tile_n(R)));
    NMG_TRY(make_map(&h->mKBlS[l], h->B32l[l]->p, nl, nl, kron_tile_n(R)));
  }
  NMG_TRY(h->tsend.alloc(B * n0 * R0));
  NMG_TRY(h->trecv.alloc(B * n0 * n0));
  NMG_TRY(h->t64send.alloc(B * n0 * R0));
  NMG_TRY(h->t64recv.alloc(B * n0 * n0));
  NMG_TRY(h->hsend.alloc(2 * B * H * n0));
  NMG_TRY(h->hrecv.alloc((size_t)W * 2 * B * H * n0));
  // level filter: per-RHS [R/2][n] complex rows; all-to-all chunks of n / W + 1 slots per rank
  NMG_TRY(h->zs.alloc(B * (R0 / 2) * n0));
  NMG_TRY(h->za.alloc((size_t)W * B * (R0 / 2) * filter2d_slab_chunk(n0, W)));
  NMG_TRY(h->zb.alloc((size_t)W * B * (R0 / 2) * filter2d_slab_chunk(n0, W)));
  const int nq = h->n[h->Ls];
  NMG_TRY(h->csend.alloc(B * (nq / W) * nq));
  NMG_TRY(h->crecv.alloc(B * nq * nq));
  NMG_TRY(h->dscratch.alloc((size_t)W * B));
  NMG_TRY(h->ssum.alloc(B));
  NMG_TRY(h->rsum.alloc(B));
  NMG_TRY(h->ysq.alloc(B));
  NMG_CUDA(cudaDeviceSynchronize());
  *out = h.release();
  return NMG_OK;
}

// Exact rebalancing of the CNN's hidden channels before the FP16x3 splits.  ReLU is positively
// homogeneous, so scaling hidden channel c of layer k (its weights and bias) by a power of two
// lambda_c and the next layer's input-channel-c weights by 1 / lambda_c leaves every fp32 value
// of the network bitwise unchanged up to the factor lambda_c on a_k[c] (power-of-two products and
// sums round identically; exponents are clamped far from the fp32 range ends).  A channel whose
// activation bound B_k[c] = |b_k[c]| + sum |w_k[c]| B_{k-1} lies more than 2^4 below the layer's
// largest is lifted into the largest one's binade: the layer's split scale S_k = 2^14 / max_c
// B_k[c] would otherwise leave such a channel only a few bits in its f16 hi/lo parts (the spread
// moves to the next layer's weights, whose split scale comes from their actual maximum).  Layers
// whose channels all lie within 2^4 of each other (the seeded and the trained smoothers) are
// left as given, so their splits are unchanged.
void balance_cnn(std::vector<float>& p, int n_layers, int C, int kk) {
  std::vector<double> bin(1, 1.0);   // |u| <= 1 (||u||_2 = 1 after the normalisation)
  size_t off = 0;
  int cin = 1;
  for (int layer = 0; layer + 1 < n_layers; ++layer) {
    const int cout = C;
    float* w = p.data() + off;
    float* b = w + (size_t)cout * cin * kk;
    const size_t next = off + (size_t)cout * cin * kk + cout;   // next layer's weights [o'][c][t]
    const int cout_next = layer + 2 == n_layers ? 1 : C;
    std::vector<double> bout(cout, 0.0);
    double bmax = 0.0;
    for (int o = 0; o < cout; ++o) {
      double B = std::fabs((double)b[o]);
      for (int c = 0; c < cin; ++c)
        for (int t = 0; t < kk; ++t) B += std::fabs((double)w[((size_t)o * cin + c) * kk + t]) * bin[c];
      bout[o] = B;
      if (std::isfinite(B)) bmax = std::max(bmax, B);
    }
    int emax = 0;
    if (bmax > 0.0) std::frexp(bmax, &emax);
    for (int o = 0; o < cout; ++o) {
      const double B = bout[o];
      if (!(B > 0.0) || !(B < std::ldexp(bmax, -4))) continue;
      int e = 0;
      std::frexp(B, &e);
      const int sh = std::min(40, emax - e);                     // B 2^sh in bmax's binade
      const float lam = std::ldexp(1.0f, sh), inv = std::ldexp(1.0f, -sh);
      for (int i = 0; i < cin * kk; ++i) w[(size_t)o * cin * kk + i] *= lam;
      b[o] *= lam;
      for (int o2 = 0; o2 < cout_next; ++o2)
        for (int t = 0; t < kk; ++t) p[next + ((size_t)o2 * cout + o) * kk + t] *= inv;
      bout[o] = std::ldexp(B, sh);
    }
    bin.swap(bout);
    off = next;
    cin = cout;
  }
}

nmg_status nmg_load_smoother_weights(nmg_hierarchy* h, int32_t level, const nmg_cnn_arch* arch,
                                     const float* params_in, size_t n_params) {
  const float* params = params_in;
  g_err.clear();
  if (!h || !arch || !params) return fail(NMG_ERR_INVALID_ARG, "null argument");
  if (level < 1 || level > h->L - 1) return fail(NMG_ERR_INVALID_ARG, "level %d outside 1..%d", level, h->L - 1);
  const bool ok1 = h->d.dim == 1 && arch->n_layers == 3 && arch->channels == 16 && arch->ksize == 5;
  const bool ok2 = h->d.dim == 2 && arch->n_layers == 4 && (arch->channels == 32 || arch->channels == 48) &&
                   arch->ksize == 3;
  if (!ok1 && !ok2)
    return fail(NMG_ERR_UNSUPPORTED, "CNN arch (%d layers, %d ch, k %d) not supported for dim %d",
                arch->n_layers, arch->channels, arch->ksize, h->d.dim);
  const int C = arch->channels, k = arch->ksize, kk = h->d.dim == 1 ? k : k * k;
  size_t want = 0;
  int cin = 1;
  for (int i = 0; i < arch->n_layers; ++i) {
    const int cout = (i == arch->n_layers - 1) ? 1 : C;
    want += (size_t)cout * cin * kk + cout;
    cin = cout;
  }
  if (n_params != want) return fail(NMG_ERR_SHAPE, "expected %zu parameters, got %zu", want, n_params);
  std::vector<float> balanced(params, params + n_params);
  if (!h->tune.no_balance) {
    balance_cnn(balanced, arch->n_layers, C, kk);
    params = balanced.data();
  }
  NMG_CUDA(cudaSetDevice(h->d.device));
  // captured cycle graphs bake in weight pointers, tensor maps and by-value weights: drop them
  // (after the device is idle) so the next cycle re-captures with the new smoother
  NMG_CUDA(cudaDeviceSynchronize());
  drop_graphs(h);
  if (h->d.dim == 2) {
    // device layout: hidden-layer weights transposed to [c][t2][t1][o] (see cnn2d_kernel)
    std::vector<float> dev(params, params + n_params);
    size_t off = (size_t)C * 9 + C;                        // after w0, b0
    for (int layer = 1; layer <= 2; ++layer) {
      for (int o = 0; o < C; ++o)
        for (int c = 0; c < C; ++c)
          for (int t = 0; t < 9; ++t) dev[off + ((size_t)c * 9 + t) * C + o] = params[off + ((size_t)o * C + c) * 9 + t];
      off += (size_t)C * C * 9 + C;
    }
    NMG_TRY(h->W[level - 1]->upload(dev.data(), n_params));
    if (h->conv_bf) {
      // Scales (powers of two) from rigorous bounds: |u| <= 1 (||u||_2 = 1), |a1| <= B1,
      // |a2| <= B2; weights of each hidden layer scaled by T so max |w T| <= 2^14.
      double B1 = 0.0;
      for (int c = 0; c < C; ++c) {
        double sacc = std::fabs((double)params[(size_t)C * 9 + c]);
        for (int t = 0; t < 9; ++t) sacc += std::fabs((double)params[(size_t)c * 9 + t]);
        B1 = std::max(B1, sacc);
      }
      const size_t L1 = (size_t)C * 9 + C, L2 = L1 + (size_t)C * C * 9 + C;
      double B2 = 0.0, wm1 = 0.0, wm2 = 0.0;
      for (int o = 0; o < C; ++o) {
        double sacc = 0.0;
        for (size_t i = 0; i < (size_t)C * 9; ++i) {
          const double w = std::fabs((double)params[L1 + (size_t)o * C * 9 + i]);
          sacc += w;
          wm1 = std::max(wm1, w);
        }
        B2 = std::max(B2, sacc * B1 + std::fabs((double)params[L1 + (size_t)C * C * 9 + o]));
      }
      double B3 = 0.0, wm4 = 0.0;
      for (int o = 0; o < C; ++o) {
        double sacc = 0.0;
        for (size_t i = 0; i < (size_t)C * 9; ++i) {
          const double w = std::fabs((double)params[L2 + (size_t)o * C * 9 + i]);
          sacc += w;
          wm2 = std::max(wm2, w);
        }
        B3 = std::max(B3, sacc * B2 + std::fabs((double)params[L2 + (size_t)C * C * 9 + o]));
      }
      const size_t L3 = L2 + (size_t)C * C * 9 + C;         // w3 [1][C][3][3]
      for (size_t i = 0; i < (size_t)C * 9; ++i) wm4 = std::max(wm4, std::fabs((double)params[L3 + i]));
      const float S1 = pow2_scale(B1), S2 = pow2_scale(B2), T1 = pow2_scale(wm1), T2 = pow2_scale(wm2);
      const float S3 = pow2_scale(B3), T4 = pow2_scale(wm4);
      if (h->strip_sc.size() < (size_t)6 * h->L) h->strip_sc.assign((size_t)6 * h->L, 1.0f);
      float* sc = &h->strip_sc[(size_t)6 * (level - 1)];
      sc[0] = S1; sc[1] = T1; sc[2] = S2; sc[3] = T2; sc[4] = S3; sc[5] = T4;
      // B operand of the strip kernels: W'[n' = t2 C + o][k' = t1 C + c] = w[o][c][t2][t1] T, f16
      // hi/lo, canonical no-swizzle K-major layout: element (n', k') at ((k'/8) N + n') 8 + k' % 8
      const int N = 3 * C;
      const size_t plane = (size_t)N * N;
      std::vector<uint16_t> wb(4 * plane + 2 * 16 * (size_t)C, 0);
      // layer 4 as an MMA B operand: rows t2 * 3 + t1 (9 of 16), K = c: [C/8][16][8]
      for (int c = 0; c < C; ++c)
        for (int t = 0; t < 9; ++t) {
          const float w = params[L3 + (size_t)c * 9 + t] * T4;
          const size_t at = 4 * plane + ((size_t)(c / 8) * 16 + t) * 8 + c % 8;
          wb[at] = f16_rn(w);
          wb[at + 16 * (size_t)C] = f16_rn(w - f16_f(wb[at]));
        }
      size_t woff = L1;
      for (int layer = 0; layer < 2; ++layer) {
        uint16_t* hi = wb.data() + (2 * layer) * plane;
        uint16_t* lo = wb.data() + (2 * layer + 1) * plane;
        const float T = layer == 0 ? T1 : T2;
        for (int t2 = 0; t2 < 3; ++t2)
          for (int o = 0; o < C; ++o)
            for (int t1 = 0; t1 < 3; ++t1)
              for (int c = 0; c < C; ++c) {
                const float w = params[woff + (((size_t)o * C + c) * 3 + t2) * 3 + t1] * T;
                const int np = t2 * C + o, kp = t1 * C + c;
                const size_t at = ((size_t)(kp / 8) * N + np) * 8 + kp % 8;
                hi[at] = f16_rn(w);
                lo[at] = f16_rn(w - f16_f(hi[at]));
              }
        woff += (size_t)C * C * 9 + C;
      }
      NMG_TRY(h->WB[level - 1]->upload(wb.data(), wb.size()));
      if (h->bf_C != C) {
        // activation workspaces for one RHS chunk at the finest strip level
        int nmax = 0;
        for (int l = 0; l < h->L - 1; ++l)
          if (strip_level(h->n[l])) nmax = std::max(nmax, h->n[l]);
        if (nmax > 0) {
          int64_t px = (int64_t)nmax * nmax;
          if (h->slab) px = std::max<int64_t>(px, (int64_t)(h->R[0] + 2 * h->HS) * h->n[0]);   // halo'd slab image
          const int64_t per = px * C * 4 + px * 8;                      // bytes per RHS (a2 hi/lo, h + edges)
          const int64_t budget = (int64_t)16 << 30;
          const int64_t B = h->d.max_rhs;
          const int64_t cmax = std::max<int64_t>(1, std::min<int64_t>(B, budget / per));
          const int64_t nch = (B + cmax - 1) / cmax;
          h->bf_chunk = (int)((B + nch - 1) / nch);
          h->bf_px = px;
          NMG_TRY(h->a2h.alloc((size_t)h->bf_chunk * px * C));
          NMG_TRY(h->a2l.alloc((size_t)h->bf_chunk * px * C));
          // CNN output h [chunk][px] followed by the strip-edge records (px / 32 floats per image)
          NMG_TRY(h->qbuf.alloc((size_t)h->bf_chunk * px * 2));
          for (int l = 0; l < h->L - 1; ++l) {
            if (!strip_level(h->n[l])) continue;
            NMG_TRY(make_a2_map(&h->mA2h[l], h->a2h.p, h->n[l], C, h->bf_chunk));
            NMG_TRY(make_a2_map(&h->mA2l[l], h->a2l.p, h->n[l], C, h->bf_chunk));
          }
        }
        h->bf_C = C;
      }
    }
  } else {
    NMG_TRY(h->W[level - 1]->upload(params, n_params));
    if (h->smooth_f16) {
      // layer-2 B operand per tap t: [chunk kc][row r][j], rows 0..15 = hi(w1[o][c][t] T),
      // rows 16..31 = lo, c = 8 kc + j; scales from |u| <= 1 and max |w1| (see conv_strip.cu)
      const size_t L1 = (size_t)C * k + C;
      double B1 = 0.0, wm = 0.0;
      for (int c = 0; c < C; ++c) {
        double acc = std::fabs((double)params[(size_t)C * k + c]);
        for (int t = 0; t < k; ++t) acc += std::fabs((double)params[(size_t)c * k + t]);
        B1 = std::max(B1, acc);
      }
      for (size_t i = 0; i < (size_t)C * C * k; ++i) wm = std::max(wm, std::fabs((double)params[L1 + i]));
      const float S1 = pow2_scale(B1), T1 = pow2_scale(wm);
      if (h->s1d_sc.size() < (size_t)2 * h->L) h->s1d_sc.assign((size_t)2 * h->L, 1.0f);
      h->s1d_sc[2 * (level - 1)] = S1;
      h->s1d_sc[2 * (level - 1) + 1] = T1;
      std::vector<uint16_t> wb((size_t)k * 2 * 32 * 8);
      for (int t = 0; t < k; ++t)
        for (int o = 0; o < C; ++o)
          for (int c = 0; c < C; ++c) {
            const float w = params[L1 + ((size_t)o * C + c) * k + t] * T1;
            const uint16_t hi = f16_rn(w), lo = f16_rn(w - f16_f(hi));
            const size_t base = (size_t)t * 2 * 32 * 8 + (size_t)(c / 8) * 32 * 8 + c % 8;
            wb[base + (size_t)o * 8] = hi;
            wb[base + (size_t)(16 + o) * 8] = lo;
          }
      if (h->s1d_w.size() < (size_t)h->L) h->s1d_w.resize(h->L);
      {
        Smooth1dW& hw = h->s1d_w[level - 1];
        const float* P = params;
        for (int i = 0; i < C * k; ++i) hw.w0[i] = P[i];
        for (int c = 0; c < C; ++c) hw.b0[c] = P[C * k + c];
        for (int c = 0; c < C; ++c) hw.b1[c] = P[L1 + (size_t)C * C * k + c];
        for (int i = 0; i < C * k; ++i) hw.w2[i] = P[L1 + (size_t)C * C * k + C + i];
        hw.b2 = P[L1 + (size_t)C * C * k + C + C * k];
      }
      while (h->W1b.size() < (size_t)(h->L)) h->W1b.emplace_back(new DevBuf<uint16_t>());
      NMG_TRY(h->W1b[level - 1]->upload(wb.data(), wb.size()));
    }
  }
  h->w_loaded[level - 1] = 1;
  if (h->fno.size() > (size_t)(level - 1)) h->fno[level - 1].reset();   // the CNN replaces an FNO
  for (auto& hk : h->lanes) NMG_TRY(nmg_load_smoother_weights(hk.get(), level, arch, params, n_params));
  h->arch = *arch;
  return NMG_OK;
}

nmg_status nmg_load_fno_weights(nmg_hierarchy* h, int32_t level, const nmg_fno_arch* arch, const float* params,
                                size_t n_params) {
  g_err.clear();
  if (!h || !arch || !params) return fail(NMG_ERR_INVALID_ARG, "null argument");
  if (level < 1 || level > h->L - 1) return fail(NMG_ERR_INVALID_ARG, "level %d outside 1..%d", level, h->L - 1);
  if (h->slab) return fail(NMG_ERR_UNSUPPORTED, "FNO smoothers are not available on a slab-sharded handle");
  if (h->d.precision == NMG_PREC_FP64) return fail(NMG_ERR_UNSUPPORTED, "FNO smoothers run in the mixed-precision cycle only");
  const int dim = h->d.dim, n = h->n[level - 1];
  const int c = arch->width, L = arch->n_layers, k = arch->modes, ks = arch->ksize;
  if (c < 1 || c > 64 || L < 1 || L > 8 || ks < 1 || ks > 7 || (ks & 1) == 0 || k < 1 || (k & (k - 1)) ||
      4 * k > n || n > 4096)
    return fail(NMG_ERR_UNSUPPORTED, "FNO arch (width %d, layers %d, modes %d, ksize %d) not supported at n = %d", c, L,
                k, ks, n);
  const size_t spec = (dim == 1 ? (size_t)k : (size_t)2 * k * k) * c * c * 2;
  const size_t conv = (size_t)c * c * (dim == 1 ? ks : ks * ks);
  const size_t want = 2 * (size_t)c + L * (spec + conv + c) + c + 1;
  if (n_params != want) return fail(NMG_ERR_SHAPE, "expected %zu FNO parameters, got %zu", want, n_params);
  NMG_CUDA(cudaSetDevice(h->d.device));
  NMG_CUDA(cudaDeviceSynchronize());
  drop_graphs(h);
  if (h->fno.size() < (size_t)h->L) h->fno.resize(h->L);
  std::unique_ptr<nmg_hierarchy::FnoLevel> F(new nmg_hierarchy::FnoLevel());
  F->arch = *arch;
  F->proj_b = params[n_params - 1];
  NMG_TRY(F->p.upload(params, n_params));
  F->tc = h->tune.simt_fno != 1 && fno_tc_ok(dim, n, c);   // simt_fno 2: tcgen05 box variant only
  if (F->tc) {
    // W [o][c][tap] -> [layer][o][tap][c], tf32 hi/lo (K index of the implicit GEMM = tap * c + channel)
    const int taps = dim == 1 ? ks : ks * ks;
    std::vector<float> wh((size_t)L * conv), wl((size_t)L * conv);
    for (int i = 0; i < L; ++i) {
      const float* Wi = params + 2 * (size_t)c + i * (spec + conv + c) + spec;
      for (int o = 0; o < c; ++o)
        for (int ch = 0; ch < c; ++ch)
          for (int t = 0; t < taps; ++t) {
            const float w = Wi[((size_t)o * c + ch) * taps + t];
            const size_t at = (size_t)i * conv + ((size_t)o * taps + t) * c + ch;
            wh[at] = tf32_rna(w);
            wl[at] = tf32_rna(w - wh[at]);
          }
    }
    NMG_TRY(F->w2h.upload(wh.data(), wh.size()));
    NMG_TRY(F->w2l.upload(wl.data(), wl.size()));
    F->mWh.resize(L);
    F->mWl.resize(L);
    for (int i = 0; i < L; ++i) {
      NMG_TRY(make_map(&F->mWh[i], F->w2h.p + (size_t)i * conv, c, (int64_t)taps * c, 64));
      NMG_TRY(make_map(&F->mWl[i], F->w2l.p + (size_t)i * conv, c, (int64_t)taps * c, 64));
    }
  }
  h->fno[level - 1] = std::move(F);
  // workspaces for the largest FNO level: RHS chunks with <= 2 GiB of activations per buffer
  int64_t per = 0, tper = 0, hper = 0;
  bool any_tc = false;
  for (int l = 0; l < h->L - 1; ++l) {
    if (!h->fno[l]) continue;
    any_tc = any_tc || h->fno[l]->tc;
    const nmg_fno_arch& a = h->fno[l]->arch;
    per = std::max<int64_t>(per, (int64_t)a.width * h->N[l]);
    if (dim == 2) tper = std::max<int64_t>(tper, (int64_t)a.width * h->n[l] * a.modes);
    hper = std::max<int64_t>(hper, (int64_t)a.width * (dim == 1 ? a.modes : 2 * a.modes * a.modes));
  }
  const int64_t B = h->d.max_rhs;
  const int chunk = (int)std::max<int64_t>(1, std::min<int64_t>(B, ((int64_t)1 << 29) / per));
  if (chunk != h->fno_chunk || (int64_t)h->fz0.n < chunk * per || (int64_t)h->fZh.n < chunk * hper ||
      (int64_t)h->fT.n < chunk * tper || (any_tc && (int64_t)h->fXh[0].n < chunk * per)) {
    h->fno_chunk = chunk;
    if (any_tc)
      for (int q = 0; q < 2; ++q) {
        NMG_TRY(h->fXh[q].alloc((size_t)chunk * per));
        NMG_TRY(h->fXl[q].alloc((size_t)chunk * per));
      }
    NMG_TRY(h->fz0.alloc((size_t)chunk * per));
    NMG_TRY(h->fz1.alloc((size_t)chunk * per));
    NMG_TRY(h->fZh.alloc((size_t)chunk * hper));
    NMG_TRY(h->fYh.alloc((size_t)chunk * hper));
    if (tper) NMG_TRY(h->fT.alloc((size_t)chunk * tper));
  }
  if (!h->snorm.p) NMG_TRY(h->snorm.alloc(B));
  if (!h->spart.p) NMG_TRY(h->spart.alloc(B * 64));
  h->w_loaded[level - 1] = 1;
  for (auto& hk : h->lanes) NMG_TRY(nmg_load_fno_weights(hk.get(), level, arch, params, n_params));
  return NMG_OK;
}

nmg_status nmg_residual(nmg_hierarchy* h, int32_t nrhs, const double* y, const double* x, double* r,
                        double* relres, void* stream) {
  g_err.clear();
  if (!h) return fail(NMG_ERR_INVALID_ARG, "null handle");
  if (nrhs < 0 || nrhs > h->d.max_rhs) return fail(NMG_ERR_INVALID_ARG, "bad nrhs");
  if (nrhs == 0) return NMG_OK;
  if (!y || !x) return fail(NMG_ERR_INVALID_ARG, "null argument");
  NMG_CUDA(cudaSetDevice(h->d.device));
  cudaStream_t s = (cudaStream_t)stream;
  NMG_TRY(outer_residual(h, nrhs, y, x, r, relres != nullptr, s));
  if (relres) {
    NMG_TRY(ynorms(h, nrhs, y, s));
    NMG_TRY(relres_fin(h, nrhs, -1.0, nullptr, relres, s));
  }
  return check_launch(h);
}

nmg_status nmg_vcycle(nmg_hierarchy* h, int32_t nrhs, const double* y, double* x, void* stream) {
  g_err.clear();
  NMG_TRY(check_ready(h, nrhs));
  if (nrhs == 0) return NMG_OK;
  if (!y || !x) return fail(NMG_ERR_INVALID_ARG, "null y/x");
  return graph_cycle(h, nrhs, y, x, (cudaStream_t)stream);
}

nmg_status nmg_solve(nmg_hierarchy* h, int32_t nrhs, const double* y, double* x, double tol, int32_t max_cycles,
                     nmg_report* rep, void* stream) {
  g_err.clear();
  NMG_TRY(check_ready(h, nrhs));
  cudaStream_t s = (cudaStream_t)stream;
  if (rep) { rep->fail_cycle = -1; rep->fail_rhs = -1; rep->total_cycles = 0; rep->wall_seconds = 0; }
  if (nrhs == 0) return NMG_OK;
  if (!y || !x || max_cycles < 0) return fail(NMG_ERR_INVALID_ARG, "bad arguments");
  const int64_t N = h->N[0];
  std::vector<double> rr(nrhs), rr0(nrhs, 0.0);
  std::vector<uint8_t> act(nrhs, 1);
  std::vector<int32_t> cyc(nrhs, 0), above(nrhs, 0);
  if (rep && rep->history)
    for (size_t i = 0; i < (size_t)nrhs * (max_cycles + 1); ++i) rep->history[i] = NAN;
  cudaEvent_t e0, e1;
  NMG_CUDA(cudaEventCreate(&e0));
  NMG_CUDA(cudaEventCreate(&e1));
  const bool f64 = h->d.precision == NMG_PREC_FP64;
  NMG_CUDA(cudaEventRecord(e0, s));
  if (f64) {
    NMG_TRY(cycle_fp64(h, nrhs, y, x, false, false, tol, nullptr, h->active.p, s));
  } else {
    NMG_TRY(ynorms(h, nrhs, y, s));
    NMG_TRY(outer_residual(h, nrhs, y, x, nullptr, true, s));
    NMG_TRY(relres_fin(h, nrhs, tol, h->active.p, h->relres.p, s));
  }
  nmg_status st = NMG_OK;
  int tau = 0;
  // Active-set compaction (the RHS are independent; each RHS's arithmetic does not
  // depend on the batch it runs in): once the converged RHS would leave enough work undone, the
  // still-active ones are gathered into the handle's staging buffers and cycle as a smaller batch;
  // x goes back to the caller's rows before each regathering and at the end.  cur = rows cycling,
  // cmap[i] = the RHS in row i (identity while yc == y).
  const double* yc = y;
  double* xc = x;
  int cur = nrhs;
  std::vector<int32_t> map(nrhs);
  for (int b = 0; b < nrhs; ++b) map[b] = b;
  const bool can_compact = !f64 && !h->slab && h->hy.p && h->cmap.p && h->tune.no_compaction != 1;
  for (;; ++tau) {
    NMG_CUDA(cudaMemcpyAsync(rr.data(), h->relres.p, sizeof(double) * cur, cudaMemcpyDeviceToHost, s));
    NMG_CUDA(cudaStreamSynchronize(s));
    if (h->slab) {
      st = h->comm->check_async();
      if (st != NMG_OK) break;
    }
    int nact = 0;
    for (int i = 0; i < cur; ++i) {
      const int b = map[i];
      if (!act[b]) continue;
      const double rb = rr[i];
      if (!std::isfinite(rb)) {
        if (rep) { rep->fail_cycle = tau; rep->fail_rhs = b; }
        st = fail(NMG_ERR_NONFINITE, "non-finite residual at cycle %d, rhs %d", tau, b);
        break;
      }
      if (rep && rep->history) rep->history[(size_t)b * (max_cycles + 1) + tau] = rb;
      if (tau == 0) rr0[b] = rb;
      // divergence = relres above 10x the initial relres for 5 consecutive cycles
      above[b] = (tau > 0 && rb > 10.0 * rr0[b]) ? above[b] + 1 : 0;
      if (h->d.divergence_check && above[b] >= 5) {
        if (rep) { rep->fail_cycle = tau; rep->fail_rhs = b; }
        st = fail(NMG_ERR_DIVERGED, "rhs %d diverged: relres %.3e > 10 x initial %.3e for 5 cycles (cycle %d)", b,
                  rb, rr0[b], tau);
        break;
      }
      if (rb <= tol) act[b] = 0; else ++nact;
    }
    if (st != NMG_OK || nact == 0 || tau == max_cycles) break;
    for (int b = 0; b < nrhs; ++b) if (act[b]) cyc[b] = tau + 1;
    if (f64) {
      NMG_TRY(cycle_fp64(h, nrhs, y, x, true, true, tol, h->active.p, h->active.p, s));
      continue;
    }
    // compact when the converged rows are at least 1/8 of the batch and 2^22 values of work
    // (no_compaction = 2, for the parity tests: whenever one has converged)
    const bool compact = h->tune.no_compaction == 2
                             ? nact < cur
                             : nact <= cur - cur / 8 && (int64_t)(cur - nact) * N >= ((int64_t)1 << 22);
    if (can_compact && compact) {
      if (xc != x) permute_rows(cur, N, xc, x, h->cmap.p, true, s);            // x back to its rows
      std::vector<int32_t> nmap;
      nmap.reserve(nact);
      for (int i = 0; i < cur; ++i) if (act[map[i]]) nmap.push_back(map[i]);
      map.swap(nmap);
      cur = nact;
      NMG_CUDA(cudaMemcpyAsync(h->cmap.p, map.data(), sizeof(int32_t) * cur, cudaMemcpyHostToDevice, s));
      permute_rows(cur, N, y, h->hy.p, h->cmap.p, false, s);
      permute_rows(cur, N, x, h->hx.p, h->cmap.p, false, s);
      NMG_TRY(check_launch(h));
      yc = h->hy.p;
      xc = h->hx.p;
      // the residual of the compacted batch (the same values, now in rows 0 .. cur - 1)
      NMG_TRY(ynorms(h, cur, yc, s));
      NMG_TRY(outer_residual(h, cur, yc, xc, nullptr, true, s));
      NMG_TRY(relres_fin(h, cur, tol, h->active.p, h->relres.p, s));
      NMG_CUDA(cudaStreamSynchronize(s));   // map (pageable host memory) consumed before it changes
    }
    NMG_TRY(inner_cycle(h, cur, s));
    NMG_TRY(outer_update(h, cur, xc, h->active.p, s));
    NMG_TRY(outer_residual(h, cur, yc, xc, nullptr, true, s));
    NMG_TRY(relres_fin(h, cur, tol, h->active.p, h->relres.p, s));
  }
  if (xc != x) {
    permute_rows(cur, N, xc, x, h->cmap.p, true, s);
    NMG_TRY(check_launch(h));
  }
  NMG_CUDA(cudaEventRecord(e1, s));
  NMG_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rep) {
    rep->wall_seconds = ms * 1e-3;
    rep->total_cycles = tau;
    for (int b = 0; b < nrhs; ++b) {
      if (rep->cycles) rep->cycles[b] = cyc[b];
      if (rep->converged) rep->converged[b] = act[b] ? 0 : 1;
    }
  }
  return st;
}

nmg_status nmg_vcycles_host(nmg_hierarchy* h, int32_t nrhs, const double* y_host, double* x_host, int32_t cycles,
                            double* relres_host, void* stream) {
  g_err.clear();
  NMG_TRY(check_ready(h, nrhs));
  if (nrhs == 0) return NMG_OK;
  if (!y_host || !x_host || cycles < 0) return fail(NMG_ERR_INVALID_ARG, "bad arguments");
  if (h->slab) return fail(NMG_ERR_UNSUPPORTED, "nmg_vcycles_host: not available on a slab-sharded handle");
  cudaStream_t s = (cudaStream_t)stream;
  if (!h->hy.p || !h->s_h2d) return fail(NMG_ERR_UNSUPPORTED, "nmg_vcycles_host: handle has no host staging");
  const int64_t N0 = h->N[0];
  cudaEvent_t ev_start = h->hev[2 * kMaxHostChunks], ev_end = h->hev[2 * kMaxHostChunks + 1];
  NMG_CUDA(cudaEventRecord(ev_start, s));                 // staging buffers free after prior work on s
  NMG_CUDA(cudaStreamWaitEvent(h->s_h2d, ev_start, 0));
  NMG_CUDA(cudaStreamWaitEvent(h->s_d2h, ev_start, 0));
  const int K = (int)h->lanes.size() + 1;
  const int gr = h->d.dim == 1 ? 128 : 2;
  if (K > 1 && nrhs >= K * gr && !h->prof_on && s != nullptr && h->tune.host_chunks == 0) {
    // Lane-pipelined (the RHS are independent): lane k's RHS are copied in on s_h2d,
    // its stream starts cycling as soon as they land (the lanes overlap on the GPU while later
    // lanes are still in flight over PCIe), and its x goes back on s_d2h when it finishes.
    int off[kMaxHostChunks + 1];
    for (int k = 0; k <= K; ++k) off[k] = std::min(nrhs, (nrhs * k / K + gr - 1) / gr * gr);
    off[K] = nrhs;
    for (int k = 0; k < K; ++k) {
      const size_t b = sizeof(double) * (size_t)(off[k + 1] - off[k]) * N0;
      if (!b) continue;
      NMG_CUDA(cudaMemcpyAsync(h->hy.p + off[k] * N0, y_host + off[k] * N0, b, cudaMemcpyHostToDevice, h->s_h2d));
      NMG_CUDA(cudaMemcpyAsync(h->hx.p + off[k] * N0, x_host + off[k] * N0, b, cudaMemcpyHostToDevice, h->s_h2d));
      NMG_CUDA(cudaEventRecord(h->hev[k], h->s_h2d));
    }
    const int mult = h->lane_tiles ? K : 1;
    for (int k = 0; k < K; ++k) {
      const int cnt = off[k + 1] - off[k];
      if (cnt <= 0) continue;
      nmg_hierarchy* hk = k == 0 ? h : h->lanes[k - 1].get();
      cudaStream_t sk = k == 0 ? s : h->ls[k - 1];
      const double* yc = h->hy.p + off[k] * N0;
      double* xc = h->hx.p + off[k] * N0;
      NMG_CUDA(cudaStreamWaitEvent(sk, h->hev[k], 0));
      const int64_t l0 = hk->launches;
      hk->lane_mult = mult;
      nmg_status st = NMG_OK;
      // lane k runs its RHS on its own handle and stream only (no sub-lanes: lane 0's batch must
      // not fork onto lanes 1..K-1, which are cycling their own RHS concurrently)
      for (int c = 0; c < cycles && st == NMG_OK; ++c) st = graph_cycle(hk, cnt, yc, xc, sk, false);
      hk->lane_mult = 1;
      if (k > 0) h->launches += hk->launches - l0;
      NMG_TRY(st);
      if (relres_host && cycles > 0)
        NMG_CUDA(cudaMemcpyAsync(relres_host + off[k], hk->relres.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, sk));
      NMG_CUDA(cudaEventRecord(h->hev[kMaxHostChunks + k], sk));
      NMG_CUDA(cudaStreamWaitEvent(h->s_d2h, h->hev[kMaxHostChunks + k], 0));
      NMG_CUDA(cudaMemcpyAsync(x_host + off[k] * N0, xc, sizeof(double) * (size_t)cnt * N0, cudaMemcpyDeviceToHost,
                               h->s_d2h));
    }
    NMG_CUDA(cudaEventRecord(ev_end, h->s_d2h));
    NMG_CUDA(cudaStreamWaitEvent(s, ev_end, 0));
    NMG_CUDA(cudaStreamSynchronize(s));
    return NMG_OK;
  }
  // Pipelined over RHS chunks (the RHS are independent): host->device copies of
  // chunk c + 1 and the device->host copy of chunk c - 1 run on two copy streams while chunk c
  // cycles on the caller's stream.  One plain cudaMemcpyAsync per buffer and chunk.
  // two chunks keep each chunk's kernels near full occupancy (measured: cfg 1 in 4 chunks of
  // 256 RHS runs at 64% of the batch efficiency); for very large batches the copy of the first
  // chunk and the return of the last one are the exposed part, so more chunks: config 3 (2048
  // RHS of 512^2, 12.9 GB over PCIe per cycle) e2e 4,652 / 4,782 / 4,928 RHS cycles/s at 4 / 6 / 8
  // equal chunks, ~4,980 with the ramped 12-chunk schedule below (vs 4,850 for 8 equal ones)
  int nch = nrhs < 256 ? 1 : ((int64_t)nrhs * N0 / 4 < ((int64_t)1 << 25) ? 2
                             : ((int64_t)nrhs * N0 < ((int64_t)1 << 29) ? 4 : 8));
  if (h->tune.host_chunks > 0)
    nch = std::max(1, std::min(kMaxHostChunks, std::min(nrhs, (int)h->tune.host_chunks)));
  int off[kMaxHostChunks + 1];
  for (int c = 0; c <= nch; ++c) off[c] = (int)((int64_t)nrhs * c / nch);
  if (h->tune.host_chunks == 0 && nch == 8) {
    // ramped chunk sizes (1 2 4 8 16 16 16 16 8 4 2 1) / 94: the exposed parts of the pipeline
    // are the first chunk's copy-in and the last chunk's copy-out, and a chunk's copy-in (2 x 8 B
    // per value at PCIe rate) fits under the previous chunk's cycle as long as it at most doubles
    static const int w[12] = {1, 2, 4, 8, 16, 16, 16, 16, 8, 4, 2, 1};
    nch = 12;
    int acc = 0;
    for (int c = 0; c <= nch; ++c) {
      off[c] = (int)((int64_t)nrhs * acc / 94);
      if (c < nch) acc += w[c];
    }
  }
  for (int c = 0; c < nch; ++c) {
    const size_t b = sizeof(double) * (size_t)(off[c + 1] - off[c]) * N0;
    NMG_CUDA(cudaMemcpyAsync(h->hy.p + off[c] * N0, y_host + off[c] * N0, b, cudaMemcpyHostToDevice, h->s_h2d));
    NMG_CUDA(cudaMemcpyAsync(h->hx.p + off[c] * N0, x_host + off[c] * N0, b, cudaMemcpyHostToDevice, h->s_h2d));
    NMG_CUDA(cudaEventRecord(h->hev[c], h->s_h2d));
  }
  for (int c = 0; c < nch; ++c) {
    const int cnt = off[c + 1] - off[c];
    double* yc = h->hy.p + off[c] * N0;
    double* xc = h->hx.p + off[c] * N0;
    NMG_CUDA(cudaStreamWaitEvent(s, h->hev[c], 0));
    for (int k = 0; k < cycles; ++k) NMG_TRY(graph_cycle(h, cnt, yc, xc, s));
    if (relres_host && cycles > 0)
      NMG_CUDA(cudaMemcpyAsync(relres_host + off[c], h->relres.p, sizeof(double) * cnt, cudaMemcpyDeviceToHost, s));
    NMG_CUDA(cudaEventRecord(h->hev[kMaxHostChunks + c], s));
    NMG_CUDA(cudaStreamWaitEvent(h->s_d2h, h->hev[kMaxHostChunks + c], 0));
    NMG_CUDA(cudaMemcpyAsync(x_host + off[c] * N0, xc, sizeof(double) * (size_t)cnt * N0, cudaMemcpyDeviceToHost,
                             h->s_d2h));
  }
  NMG_CUDA(cudaEventRecord(ev_end, h->s_d2h));
  NMG_CUDA(cudaStreamWaitEvent(s, ev_end, 0));
  NMG_CUDA(cudaStreamSynchronize(s));
  return NMG_OK;
}

nmg_status nmg_debug_level_op(nmg_hierarchy* h, int32_t level, int32_t op, int32_t nrhs, const void* in, void* out,
                              void* stream) {
  g_err.clear();
  if (!h) return fail(NMG_ERR_INVALID_ARG, "null handle");
  if (h->slab) return fail(NMG_ERR_UNSUPPORTED, "nmg_debug_level_op: not available on a slab-sharded handle");
  if (level < 1 || level > h->L) return fail(NMG_ERR_INVALID_ARG, "level %d outside 1..%d", level, h->L);
  if (nrhs < 0 || nrhs > h->d.max_rhs) return fail(NMG_ERR_INVALID_ARG, "bad nrhs");
  if (nrhs == 0) return NMG_OK;
  if (!in || !out) return fail(NMG_ERR_INVALID_ARG, "null argument");
  NMG_CUDA(cudaSetDevice(h->d.device));
  cudaStream_t s = (cudaStream_t)stream;
  const int l = level - 1;
  const float* fin = (const float*)in;
  float* fout = (float*)out;
  if (h->d.dim == 2) return debug_2d(h, l, op, nrhs, fin, fout, s);
  const int n = h->n[l];
  const bool smoothed = l < h->L - 1;
  switch (op) {
    case NMG_OP_APPLY:
    case NMG_OP_RESIDUAL: {
      if (!smoothed) return fail(NMG_ERR_INVALID_ARG, "no fp32 operator stored at the coarsest level");
      if (h->use_tc && n % 16 == 0) {
        NMG_CUDA(cudaMemcpyAsync(h->wx[l]->p, fin, sizeof(float) * (size_t)nrhs * n, cudaMemcpyDeviceToDevice, s));
        h->split_fresh[l] = 0;
        NMG_TRY(level_resid(h, l, 0, nrhs, op == NMG_OP_RESIDUAL ? fout : nullptr, fout, s, op == NMG_OP_RESIDUAL));
        return NMG_OK;
      }
      Gemm32Args g{};
      g.M = nrhs; g.N = n; g.K = n; g.batch = 1;
      g.X = fin; g.ldx = n; g.W = h->A32[l]->p; g.ldw = n; g.w_kmajor = true;
      g.C = op == NMG_OP_RESIDUAL ? fout : nullptr; g.ldc = n;
      g.D = fout; g.ldd = n;
      g.negate = op == NMG_OP_RESIDUAL;
      gemm_f32(g, s);
      break;
    }
    case NMG_OP_RESTRICT:
      if (!smoothed) return fail(NMG_ERR_INVALID_ARG, "no coarser level");
      restrict1d(nrhs, n, fin, n, fout, n / 2, s);
      break;
    case NMG_OP_PROLONG:
      if (!smoothed) return fail(NMG_ERR_INVALID_ARG, "no coarser level");
      prolong_add1d(nrhs, n / 2, fin, n / 2, fout, n, s);
      break;
    case NMG_OP_FILTER:
      filter1d(n, nrhs, fin, fout, h->tw.p, h->tw_n, s);
      break;
    case NMG_OP_CNN:
    case NMG_OP_SMOOTH: {
      if (!smoothed || !h->w_loaded[l]) return fail(NMG_ERR_NO_WEIGHTS, "no smoother at level %d", level);
      if (h->fno.size() > (size_t)l && h->fno[l]) {
        if (op == NMG_OP_SMOOTH) return smooth_level(h, l, nrhs, fin, fout, true, s);
        return run_fno(h, l, nrhs, fin, fout, false, false, false, s);
      }
      Smooth1dArgs a{};
      a.n = n; a.nrhs = nrhs; a.b = fin; a.ldb = n; a.x = fout; a.ldx = n;
      a.params = h->W[l]->p; a.twiddle = h->tw.p; a.tw_n = h->tw_n;
      a.normalize = op == NMG_OP_SMOOTH;
      a.filter = op == NMG_OP_SMOOTH && h->d.level_filter != 0;
      a.accumulate = op == NMG_OP_SMOOTH;
      launch_smooth1d(h, l, a, s);
      break;
    }
    case NMG_OP_COARSE:
      if (smoothed) return fail(NMG_ERR_INVALID_ARG, "COARSE needs level == L");
      coarse_solve(h, nrhs, fin, n, fout, n, s);
      break;
    case NMG_OP_CYCLE0: {
      for (int q = l; q < h->L - 1; ++q)
        if (!h->w_loaded[q]) return fail(NMG_ERR_NO_WEIGHTS, "level %d has no smoother", q + 1);
      NMG_CUDA(cudaMemcpyAsync(h->wy[l]->p, fin, sizeof(float) * (size_t)nrhs * n, cudaMemcpyDeviceToDevice, s));
      NMG_TRY(cycle_level_1d(h, l, nrhs, s));
      NMG_CUDA(cudaMemcpyAsync(fout, h->wx[l]->p, sizeof(float) * (size_t)nrhs * n, cudaMemcpyDeviceToDevice, s));
      break;
    }
    default:
      return fail(NMG_ERR_INVALID_ARG, "unknown op %d", op);
  }
  h->launches++;
  return check_launch(h);
}

nmg_status nmg_profile(nmg_hierarchy* h, int32_t enable) {
  if (!h) return fail(NMG_ERR_INVALID_ARG, "null handle");
  if (enable) { h->recs.clear(); h->ev_used = 0; }
  h->prof_on = enable != 0;
  return NMG_OK;
}

nmg_status nmg_profile_query(nmg_hierarchy* h, int32_t kclass, double* total_ms, int64_t* launches) {
  if (!h || !total_ms || !launches) return fail(NMG_ERR_INVALID_ARG, "null argument");
  double tot = 0.0;
  int64_t cnt = 0;
  for (auto& r : h->recs) {
    if (r.cls != kclass) continue;
    NMG_CUDA(cudaEventSynchronize(r.b));
    float ms = 0.f;
    NMG_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    tot += ms;
    cnt += r.nk;
  }
  *total_ms = tot;
  *launches = cnt;
  return NMG_OK;
}

void nmg_destroy_hierarchy(nmg_hierarchy* h) {
  if (!h) return;
  cudaSetDevice(h->d.device);
  cudaDeviceSynchronize();
  delete h;
}

}  // extern "C"
