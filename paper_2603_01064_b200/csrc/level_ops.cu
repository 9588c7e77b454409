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

// ---- interpolation I_{l+1}^l and correction: f[i] += 3/4 c[i>>1] + 1/4 c[k] ----------
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
// One warp per RHS; lane owns entries j = q*32 + lane of the fp64 iterate.  Blocked
// substitution over 32-wide diagonal blocks: inside a block the 32 sequential steps keep
// the block's column (forward) / row (backward) of L in registers, so the dependent chain
// per step is shfl -> mul -> fma; the off-diagonal update of the other blocks is a plain
// accumulation of independent coalesced loads (Lcol[i*nc + j] = L[j][i]).
NMG_D double coarse_ld(const double* p) { return __ldg(p); }

template <int NQ>
__global__ void __launch_bounds__(256) coarse_kernel(int nc, int nrhs, const double* __restrict__ Lrow,
                                                     const double* __restrict__ Lcol,
                                                     const float* __restrict__ y, int64_t ldy,
                                                     float* __restrict__ x, int64_t ldx,
                                                     float* __restrict__ xh, float* __restrict__ xl) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= nrhs) return;
  double z[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const int j = q * 32 + lane;
    z[q] = (j < nc) ? (double)y[(int64_t)b * ldy + j] : 0.0;
  }
  // forward: L z = y
#pragma unroll
  for (int q0 = 0; q0 < NQ; ++q0) {
    const int i0 = q0 * 32, jd = i0 + lane;
    const bool okj = jd < nc;
    double Lb[32];
#pragma unroll
    for (int il = 0; il < 32; ++il)
      Lb[il] = (okj && i0 + il < nc && il < lane) ? coarse_ld(Lcol + (int64_t)(i0 + il) * nc + jd) : 0.0;
    const double dv = okj ? 1.0 / coarse_ld(Lcol + (int64_t)jd * nc + jd) : 1.0;
#pragma unroll
    for (int il = 0; il < 32; ++il) {
      const double zi = __shfl_sync(0xffffffffu, z[q0], il) * __shfl_sync(0xffffffffu, dv, il);
      z[q0] = (lane == il) ? zi : fma(-Lb[il], zi, z[q0]);
    }
#pragma unroll
    for (int q = q0 + 1; q < NQ; ++q) {
      const int j = q * 32 + lane;
      double acc = z[q];
#pragma unroll 8
      for (int il = 0; il < 32; ++il) {
        const double zi = __shfl_sync(0xffffffffu, z[q0], il);
        if (j < nc && i0 + il < nc) acc = fma(-coarse_ld(Lcol + (int64_t)(i0 + il) * nc + j), zi, acc);
      }
      z[q] = acc;
    }
  }
  // backward: L^T x = z
#pragma unroll
  for (int q0 = NQ - 1; q0 >= 0; --q0) {
    const int i0 = q0 * 32, jd = i0 + lane;
    const bool okj = jd < nc;
    double Lb[32];
#pragma unroll
    for (int il = 0; il < 32; ++il)
      Lb[il] = (okj && i0 + il < nc && il > lane) ? coarse_ld(Lrow + (int64_t)(i0 + il) * nc + jd) : 0.0;
    const double dv = okj ? 1.0 / coarse_ld(Lrow + (int64_t)jd * nc + jd) : 1.0;
#pragma unroll
    for (int il = 31; il >= 0; --il) {
      const double xi = __shfl_sync(0xffffffffu, z[q0], il) * __shfl_sync(0xffffffffu, dv, il);
      z[q0] = (lane == il) ? xi : fma(-Lb[il], xi, z[q0]);
    }
#pragma unroll
    for (int q = 0; q < q0; ++q) {
      const int j = q * 32 + lane;
      double acc = z[q];
#pragma unroll 8
      for (int il = 0; il < 32; ++il) {
        const double xi = __shfl_sync(0xffffffffu, z[q0], il);
        if (i0 + il < nc) acc = fma(-coarse_ld(Lrow + (int64_t)(i0 + il) * nc + j), xi, acc);
      }
      z[q] = acc;
    }
  }
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
  restrict1d_kernel<<<nblk((int64_t)nrhs * n_c, 256), 256, 0, s>>>(nrhs, n_c, f, ldf, c, ldc);
}

void prolong_add1d(int nrhs, int n_c, const float* c, int64_t ldc, float* f, int64_t ldf, cudaStream_t s) {
  prolong_add1d_kernel<<<nblk((int64_t)nrhs * 2 * n_c, 256), 256, 0, s>>>(nrhs, n_c, c, ldc, f, ldf);
}

void coarse_chol_solve(int nc, int nrhs, const double* Lrow, const double* Lcol, const float* y, int64_t ldy,
                       float* x, int64_t ldx, cudaStream_t s, float* xh, float* xl) {
  const int grid = ceil_div(nrhs, 8);
  const int nq = ceil_div(nc, 32);
#define NMG_COARSE(Q) \
  case Q: coarse_kernel<Q><<<grid, 256, 0, s>>>(nc, nrhs, Lrow, Lcol, y, ldy, x, ldx, xh, xl); break;
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

void f64_to_f32(int64_t count, const double* in, float* out, cudaStream_t s) {
  f64_to_f32_kernel<<<nblk(count, 256), 256, 0, s>>>(count, in, out);
}
void f32_to_f64(int64_t count, const float* in, double* out, cudaStream_t s) {
  f32_to_f64_kernel<<<nblk(count, 256), 256, 0, s>>>(count, in, out);
}

}  // namespace nmg
