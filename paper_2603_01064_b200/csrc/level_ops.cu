// Memory-bound level passes: transfers (reading R4), coarse Cholesky solve
// (Alg 3 P:324 exact coarse solve; BASELINE "dense Cholesky"), and the
// fp64 outer-iteration helpers (stop rule P:479).
#include "common.cuh"
#include "kernels.h"

#include <algorithm>

namespace nmg {
namespace {

// ---- restriction I_l^{l+1}: full weighting on the cell-centred grid --------------
// r[j] = ((f[2j-1] + f[2j+2]) + 3 (f[2j] + f[2j+1])) / 8 with clamped end taps,
// evaluated in this fixed order without FMA contraction (bit-exact index-map parity).
__global__ void restrict1d_kernel(int nrhs, int n_c, const float* __restrict__ f, int64_t ldf,
                                  float* __restrict__ c, int64_t ldc) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nrhs * n_c) return;
  const int b = (int)(idx / n_c), j = (int)(idx - (int64_t)b * n_c);
  const int n_f = 2 * n_c;
  const float* fr = f + (int64_t)b * ldf;
  const float fm = fr[max(2 * j - 1, 0)];
  const float f0 = fr[2 * j];
  const float f1 = fr[2 * j + 1];
  const float fp = fr[min(2 * j + 2, n_f - 1)];
  const float outer = __fadd_rn(fm, fp);
  const float inner = __fmul_rn(3.0f, __fadd_rn(f0, f1));
  c[(int64_t)b * ldc + j] = __fmul_rn(__fadd_rn(outer, inner), 0.125f);
}

// vectorised: thread = coarse outputs 2s, 2s + 1 from fine 4s - 1 .. 4s + 4 (one float4 load
// + two scalars); same expression order as restrict1d_kernel (bitwise)
__global__ void restrict1d_x2_kernel(int nrhs, int n_c, const float* __restrict__ f, int64_t ldf,
                                     float* __restrict__ c, int64_t ldc) {
  const int hc = n_c >> 1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nrhs * hc) return;
  const int b = (int)(idx / hc), sidx = (int)(idx - (int64_t)b * hc);
  const int n_f = 2 * n_c;
  const float* fr = f + (int64_t)b * ldf;
  const float4 m = *reinterpret_cast<const float4*>(fr + 4 * sidx);
  const float fm = fr[max(4 * sidx - 1, 0)];
  const float fp = fr[min(4 * sidx + 4, n_f - 1)];
  float2 o;
  o.x = __fmul_rn(__fadd_rn(__fadd_rn(fm, m.z), __fmul_rn(3.0f, __fadd_rn(m.x, m.y))), 0.125f);
  o.y = __fmul_rn(__fadd_rn(__fadd_rn(m.y, fp), __fmul_rn(3.0f, __fadd_rn(m.z, m.w))), 0.125f);
  *reinterpret_cast<float2*>(c + (int64_t)b * ldc + 2 * sidx) = o;
}

// ---- interpolation I_{l+1}^l and correction: f[i] += 3/4 c[i>>1] + 1/4 c[k] ----------
// vectorised: thread = fine 4t .. 4t + 3 from coarse 2t - 1 .. 2t + 2 (bitwise prolong_add1d)
__global__ void prolong_add1d_x4_kernel(int nrhs, int n_c, const float* __restrict__ c, int64_t ldc,
                                        float* __restrict__ f, int64_t ldf) {
  const int q = n_c >> 1;                          // fine quads per row
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nrhs * q) return;
  const int b = (int)(idx / q), t = (int)(idx - (int64_t)b * q);
  const float* cr = c + (int64_t)b * ldc;
  const float c0 = cr[2 * t], c1 = cr[2 * t + 1];
  const float cm = cr[max(2 * t - 1, 0)], cp = cr[min(2 * t + 2, n_c - 1)];
  float4* fq = reinterpret_cast<float4*>(f + (int64_t)b * ldf) + t;
  float4 v = *fq;
  v.x = __fadd_rn(v.x, __fadd_rn(__fmul_rn(0.75f, c0), __fmul_rn(0.25f, cm)));
  v.y = __fadd_rn(v.y, __fadd_rn(__fmul_rn(0.75f, c0), __fmul_rn(0.25f, c1)));
  v.z = __fadd_rn(v.z, __fadd_rn(__fmul_rn(0.75f, c1), __fmul_rn(0.25f, c0)));
  v.w = __fadd_rn(v.w, __fadd_rn(__fmul_rn(0.75f, c1), __fmul_rn(0.25f, cp)));
  *fq = v;
}

__global__ void prolong_add1d_kernel(int nrhs, int n_c, const float* __restrict__ c, int64_t ldc,
                                     float* __restrict__ f, int64_t ldf) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n_f = 2 * n_c;
  if (idx >= (int64_t)nrhs * n_f) return;
  const int b = (int)(idx / n_f), i = (int)(idx - (int64_t)b * n_f);
  const int j = i >> 1;
  const int k = min(max((i & 1) ? j + 1 : j - 1, 0), n_c - 1);
  const float* cr = c + (int64_t)b * ldc;
  const float v = __fadd_rn(__fmul_rn(0.75f, cr[j]), __fmul_rn(0.25f, cr[k]));
  float* fr = f + (int64_t)b * ldf;
  fr[i] = __fadd_rn(fr[i], v);
}

// ---- coarse solve: x = L^{-T} L^{-1} y with the host Cholesky factor (fp64) ----------
// One warp per RHS (8 per CTA); lane owns entries j = q*32 + lane of the fp64 iterate.
// Blocked substitution over 32-wide diagonal blocks.  The CTA stages the 32-row panel
// of the factor each block needs (forward: rows i0.. of Lcol = L^T, columns i0..nc;
// backward: rows i0.. of Lrow, columns 0..i0+32) in shared memory with cp.async, double
// buffered, so the next panel streams in while the current one is used.  Inside a block
// the 32 sequential steps keep the block's column (forward) / row (backward) of L in
// registers (dependent chain per step: shfl -> mul -> fma); the update of the other blocks
// is an accumulation over independent shared-memory reads.
NMG_D void cp_async8(double* dst, const double* src) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}

template <int NQ>
NMG_D void coarse_issue_panel(int p, int nc, const double* Lrow, const double* Lcol, double* P) {
  constexpr int PS = NQ * 32;
  const bool fwd = p < NQ;
  const int q0 = fwd ? p : 2 * NQ - 1 - p;
  const int i0 = q0 * 32;
  const int rows = min(32, nc - i0);
  const int len = fwd ? nc - i0 : min(i0 + 32, nc);
  const double* src = fwd ? Lcol + (int64_t)i0 * nc + i0 : Lrow + (int64_t)i0 * nc;
  for (int e = threadIdx.x; e < rows * len; e += blockDim.x) {
    const int il = e / len, jj = e - il * len;
    cp_async8(P + il * PS + jj, src + (int64_t)il * nc + jj);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
}

constexpr int kCoarseWarps = 4;   // RHS per CTA: few, so that many SMs share the issue load

// x = A_L^{-1} y with the explicit fp64 inverse (symmetric, computed once from the Cholesky
// factor at setup): thread j forms x_j for CR right-hand sides; the Ainv[k][j] loads of a warp
// are coalesced and independent of the accumulation, so there is no sequential substitution
// chain.  Fixed summation order k = 0 .. nc - 1 (deterministic).
constexpr int kCoarseRhs = 8;
__global__ void __launch_bounds__(256) coarse_inv_kernel(int nc, int nrhs, const double* __restrict__ Ainv,
                                                         const float* __restrict__ y, int64_t ldy,
                                                         float* __restrict__ x, int64_t ldx,
                                                         float* __restrict__ xh, float* __restrict__ xl) {
  __shared__ double ys[kCoarseRhs][256];
  const int b0 = blockIdx.x * kCoarseRhs;
  for (int i = threadIdx.x; i < kCoarseRhs * nc; i += blockDim.x) {
    const int r = i / nc, k = i - r * nc;
    ys[r][k] = (b0 + r < nrhs) ? (double)y[(int64_t)(b0 + r) * ldy + k] : 0.0;
  }
  __syncthreads();
  const int j = blockIdx.y * blockDim.x + threadIdx.x;   // output index (column slice per CTA)
  if (j < nc) {
    double acc[kCoarseRhs];
#pragma unroll
    for (int r = 0; r < kCoarseRhs; ++r) acc[r] = 0.0;
    // register double buffer: the next 8 Ainv values are in flight while 8 are used
    double av[8], an[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) av[i] = __ldg(Ainv + (int64_t)min(i, nc - 1) * nc + j);
    for (int k0 = 0; k0 < nc; k0 += 8) {
#pragma unroll
      for (int i = 0; i < 8; ++i) an[i] = __ldg(Ainv + (int64_t)min(k0 + 8 + i, nc - 1) * nc + j);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (k0 + i >= nc) break;
#pragma unroll
        for (int r = 0; r < kCoarseRhs; ++r) acc[r] = fma(av[i], ys[r][k0 + i], acc[r]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) av[i] = an[i];
    }
#pragma unroll
    for (int r = 0; r < kCoarseRhs; ++r) {
      if (b0 + r >= nrhs) break;
      const float v = (float)acc[r];
      x[(int64_t)(b0 + r) * ldx + j] = v;
      if (xh) {
        uint32_t hh, ll;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(hh) : "f"(v));
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(ll) : "f"(v - __uint_as_float(hh)));
        xh[(int64_t)(b0 + r) * ldx + j] = __uint_as_float(hh);
        xl[(int64_t)(b0 + r) * ldx + j] = __uint_as_float(ll);
      }
    }
  }
}

template <int NQ>
__global__ void __launch_bounds__(kCoarseWarps * 32) coarse_kernel(int nc, int nrhs, const double* __restrict__ Lrow,
                                                     const double* __restrict__ Lcol,
                                                     const float* __restrict__ y, int64_t ldy,
                                                     float* __restrict__ x, int64_t ldx,
                                                     float* __restrict__ xh, float* __restrict__ xl) {
  constexpr int PS = NQ * 32;
  extern __shared__ double Pbuf[];   // 2 x [32][PS] panels, dinv[NQ*32], zs[warps][32]
  double* dinv = Pbuf + 2 * 32 * PS;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* zs = dinv + PS + warp * 32;
  const int b = blockIdx.x * kCoarseWarps + warp;
  const bool live = b < nrhs;
  for (int i = threadIdx.x; i < nc; i += blockDim.x) dinv[i] = 1.0 / Lrow[(int64_t)i * nc + i];
  double z[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int j = q * 32 + lane;
    z[q] = (live && j < nc) ? (double)y[(int64_t)b * ldy + j] : 0.0;
  }
  coarse_issue_panel<NQ>(0, nc, Lrow, Lcol, Pbuf);
  // forward: L z = y.  Within a block the undivided values z'_i are broadcast and the
  // column is pre-scaled by 1 / L_ii (z_j -= (L_ji / L_ii) z'_i), so a step is shfl -> fma.
#pragma unroll
  for (int q0 = 0; q0 < NQ; ++q0) {
    const int p = q0;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    coarse_issue_panel<NQ>(p + 1, nc, Lrow, Lcol, Pbuf + ((p + 1) & 1) * 32 * PS);
    const double* P = Pbuf + (p & 1) * 32 * PS;   // P[il][jj] = L[i0 + jj][i0 + il]
    const int i0 = q0 * 32;
    const bool okj = i0 + lane < nc;
    double Lb[32];
#pragma unroll
    for (int il = 0; il < 32; ++il) Lb[il] = (okj && il < lane) ? P[il * PS + lane] * dinv[i0 + il] : 0.0;
#pragma unroll
    for (int il = 0; il < 32; ++il) z[q0] = fma(-Lb[il], __shfl_sync(0xffffffffu, z[q0], il), z[q0]);
    if (okj) z[q0] *= dinv[i0 + lane];
    zs[lane] = z[q0];
    __syncwarp();
#pragma unroll
    for (int q = q0 + 1; q < NQ; ++q) {
      const int jj = (q - q0) * 32 + lane;
      const bool ok = q * 32 + lane < nc;
      double acc = z[q];
#pragma unroll
      for (int il = 0; il < 32; ++il)
        if (ok) acc = fma(-P[il * PS + jj], zs[il], acc);
      z[q] = acc;
    }
  }
  // backward: L^T x = z, same scheme on the rows of L
#pragma unroll
  for (int q0 = NQ - 1; q0 >= 0; --q0) {
    const int p = 2 * NQ - 1 - q0;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    if (p + 1 < 2 * NQ) coarse_issue_panel<NQ>(p + 1, nc, Lrow, Lcol, Pbuf + ((p + 1) & 1) * 32 * PS);
    const double* P = Pbuf + (p & 1) * 32 * PS;   // P[il][j] = L[i0 + il][j]
    const int i0 = q0 * 32;
    const bool okj = i0 + lane < nc;
    double Lb[32];
#pragma unroll
    for (int il = 0; il < 32; ++il)
      Lb[il] = (okj && il > lane && i0 + il < nc) ? P[il * PS + i0 + lane] * dinv[i0 + il] : 0.0;
#pragma unroll
    for (int il = 31; il >= 0; --il) z[q0] = fma(-Lb[il], __shfl_sync(0xffffffffu, z[q0], il), z[q0]);
    if (okj) z[q0] *= dinv[i0 + lane];
    zs[lane] = z[q0];
    __syncwarp();
    const int rows = min(32, nc - i0);
#pragma unroll
    for (int q = 0; q < q0; ++q) {
      double acc = z[q];
#pragma unroll
      for (int il = 0; il < 32; ++il)
        if (il < rows) acc = fma(-P[il * PS + q * 32 + lane], zs[il], acc);
      z[q] = acc;
    }
  }
  if (!live) return;
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int j = q * 32 + lane;
    if (j < nc) {
      const float v = (float)z[q];
      x[(int64_t)b * ldx + j] = v;
      if (xh) {
        uint32_t hh, ll;
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(hh) : "f"(v));
        asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(ll) : "f"(v - __uint_as_float(hh)));
        xh[(int64_t)b * ldx + j] = __uint_as_float(hh);
        xl[(int64_t)b * ldx + j] = __uint_as_float(ll);
      }
    }
  }
}

// ---- fp64 outer helpers ----------------------------------------------------------
// per-RHS ||y||_2 in fp64: stage 1 chunk partials (grid chunks x nrhs), stage 2 fixed-order sum
__global__ void __launch_bounds__(256) row_sumsq_partial_kernel(int64_t N, int chunks, const double* __restrict__ y,
                                                                int64_t ldy, double* __restrict__ part) {
  __shared__ double red[32];
  const int b = blockIdx.y, ch = blockIdx.x;
  const int64_t len = ceil_div64(N, chunks);
  const int64_t lo = ch * len, hi = min(N, lo + len);
  const double* r = y + (int64_t)b * ldy;
  double s = 0.0;
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) s += r[j] * r[j];
  s = block_sum_f64(s, red);
  if (threadIdx.x == 0) part[(int64_t)b * chunks + ch] = s;
}
__global__ void __launch_bounds__(256) row_norms_final_kernel(int chunks, const double* __restrict__ part,
                                                              double* __restrict__ out) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  double s = 0.0;
  for (int c = threadIdx.x; c < chunks; c += blockDim.x) s += part[(int64_t)b * chunks + c];
  s = block_sum_f64(s, red);
  if (threadIdx.x == 0) out[b] = sqrt(s);
}

// relres = sqrt(sum of the residual GEMM's ||r||^2 partials) / ||y||, one block per RHS
// (fixed-order tree => deterministic)
__global__ void __launch_bounds__(256) relres_kernel(int ntiles, const double* __restrict__ part,
                                                     const double* __restrict__ ynorm, double* __restrict__ relres,
                                                     double tol, uint8_t* __restrict__ active, int rows_per_rhs) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  const int64_t cnt = (int64_t)ntiles * rows_per_rhs;
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < cnt; t += blockDim.x) s += part[(int64_t)b * cnt + t];
  s = block_sum_f64(s, red);
  if (threadIdx.x != 0) return;
  const double yn = ynorm[b];
  // y = 0: converged at x = 0; a non-finite ||y|| or residual propagates as NaN/Inf
  const double rr = (yn > 0.0) ? sqrt(s) / yn : (yn == 0.0 && s == 0.0 ? 0.0 : sqrt(s) / yn);
  relres[b] = rr;
  if (active) active[b] = (rr > tol || rr != rr) ? 1 : 0;
}

__global__ void update_x_kernel(int nrhs, int N, double* __restrict__ x, int64_t ldx,
                                const float* __restrict__ d, int64_t ldd, const uint8_t* __restrict__ active) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nrhs * N) return;
  const int b = (int)(idx / N), j = (int)(idx - (int64_t)b * N);
  if (active && !active[b]) return;
  x[(int64_t)b * ldx + j] += (double)d[(int64_t)b * ldd + j];
}

// active-set compaction of nmg_solve: dst row i = src row map[i] (gather) or dst row map[i] =
// src row i (scatter); rows of N doubles, 16-byte vectors when N is even
__global__ void permute_rows_kernel(int rows, int64_t N, const double* __restrict__ src, double* __restrict__ dst,
                                    const int32_t* __restrict__ map, int scatter) {
  for (int i = blockIdx.y; i < rows; i += gridDim.y) {
    const int64_t si = scatter ? i : map[i], di = scatter ? map[i] : i;
    if (N % 2 == 0) {
      const double2* s2 = reinterpret_cast<const double2*>(src + si * N);
      double2* d2 = reinterpret_cast<double2*>(dst + di * N);
      for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N / 2; k += (int64_t)gridDim.x * blockDim.x)
        d2[k] = s2[k];
    } else {
      for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x)
        dst[di * N + k] = src[si * N + k];
    }
  }
}

__global__ void f64_to_f32_kernel(int64_t count, const double* __restrict__ in, float* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = (float)in[i];
}
__global__ void f32_to_f64_kernel(int64_t count, const float* __restrict__ in, double* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < count) out[i] = (double)in[i];
}

inline int nblk(int64_t n, int t) { return (int)ceil_div64(n, t); }

}  // namespace

void restrict1d(int nrhs, int n_f, const float* f, int64_t ldf, float* c, int64_t ldc, cudaStream_t s) {
  const int n_c = n_f / 2;
  if (n_c % 2 == 0 && ldf % 4 == 0 && ldc % 2 == 0 && ((uintptr_t)f & 15) == 0 && ((uintptr_t)c & 7) == 0)
    restrict1d_x2_kernel<<<nblk((int64_t)nrhs * (n_c / 2), 256), 256, 0, s>>>(nrhs, n_c, f, ldf, c, ldc);
  else
    restrict1d_kernel<<<nblk((int64_t)nrhs * n_c, 256), 256, 0, s>>>(nrhs, n_c, f, ldf, c, ldc);
}

void prolong_add1d(int nrhs, int n_c, const float* c, int64_t ldc, float* f, int64_t ldf, cudaStream_t s) {
  if (n_c % 2 == 0 && ldf % 4 == 0 && ((uintptr_t)f & 15) == 0)
    prolong_add1d_x4_kernel<<<nblk((int64_t)nrhs * (n_c / 2), 256), 256, 0, s>>>(nrhs, n_c, c, ldc, f, ldf);
  else
    prolong_add1d_kernel<<<nblk((int64_t)nrhs * 2 * n_c, 256), 256, 0, s>>>(nrhs, n_c, c, ldc, f, ldf);
}

void coarse_inv_apply(int nc, int nrhs, const double* Ainv, const float* y, int64_t ldy, float* x, int64_t ldx,
                      cudaStream_t s, float* xh, float* xl) {
  const int bt = std::min(64, ceil_div(nc, 32) * 32);
  coarse_inv_kernel<<<dim3(ceil_div(nrhs, kCoarseRhs), ceil_div(nc, bt)), bt, 0, s>>>(nc, nrhs, Ainv, y, ldy, x, ldx,
                                                                                     xh, xl);
}

void coarse_chol_solve(int nc, int nrhs, const double* Lrow, const double* Lcol, const float* y, int64_t ldy,
                       float* x, int64_t ldx, cudaStream_t s, float* xh, float* xl) {
  const int grid = ceil_div(nrhs, kCoarseWarps);
  const int nq = ceil_div(nc, 32);
#define NMG_COARSE(Q)                                                                                   \
  case Q: {                                                                                             \
    const int smem = (2 * 32 * Q * 32 + Q * 32 + kCoarseWarps * 32) * (int)sizeof(double);           \
    NMG_SMEM_OPTIN(coarse_kernel<Q>, smem);                                                           \
    coarse_kernel<Q><<<grid, kCoarseWarps * 32, smem, s>>>(nc, nrhs, Lrow, Lcol, y, ldy, x, ldx, xh, xl);           \
  } break;
  switch (nq) {
    NMG_COARSE(1) NMG_COARSE(2) NMG_COARSE(3) NMG_COARSE(4)
    NMG_COARSE(5) NMG_COARSE(6) NMG_COARSE(7) NMG_COARSE(8)
    default: break;
  }
#undef NMG_COARSE
}

void row_norms_f64(int nrhs, int N, const double* y, int64_t ldy, double* out, double* part, cudaStream_t s) {
  // a few chunks per RHS so that small batches of long vectors still fill the GPU; part: [nrhs][64]
  const int chunks = (int)std::min<int64_t>(64, std::max<int64_t>(1, N / 8192));
  row_sumsq_partial_kernel<<<dim3(chunks, nrhs), 256, 0, s>>>(N, chunks, y, ldy, part);
  row_norms_final_kernel<<<nrhs, 64, 0, s>>>(chunks, part, out);
}

void relres_finalize(int nrhs, int ntiles, const double* part, const double* ynorm, double* relres, double tol,
                     uint8_t* active, cudaStream_t s, int rows_per_rhs) {
  relres_kernel<<<nrhs, rows_per_rhs > 1 ? 256 : 32, 0, s>>>(ntiles, part, ynorm, relres, tol, active, rows_per_rhs);
}

void update_x(int nrhs, int N, double* x, int64_t ldx, const float* d, int64_t ldd, const uint8_t* active,
              cudaStream_t s) {
  update_x_kernel<<<nblk((int64_t)nrhs * N, 256), 256, 0, s>>>(nrhs, N, x, ldx, d, ldd, active);
}

void permute_rows(int rows, int64_t N, const double* src, double* dst, const int32_t* map, bool scatter,
                  cudaStream_t s) {
  if (rows <= 0) return;
  const int bx = (int)std::min<int64_t>(64, (N / 2 + 255) / 256 + 1);
  permute_rows_kernel<<<dim3(bx, std::min(rows, 65535)), 256, 0, s>>>(rows, N, src, dst, map, scatter ? 1 : 0);
}
void f64_to_f32(int64_t count, const double* in, float* out, cudaStream_t s) {
  f64_to_f32_kernel<<<nblk(count, 256), 256, 0, s>>>(count, in, out);
}
void f32_to_f64(int64_t count, const float* in, double* out, cudaStream_t s) {
  f32_to_f64_kernel<<<nblk(count, 256), 256, 0, s>>>(count, in, out);
}

}  // namespace nmg
