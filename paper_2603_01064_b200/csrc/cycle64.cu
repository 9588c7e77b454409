// NMG_PREC_FP64 (reading R14, BASELINE configs[0] "fp64" system): the whole NMGF cycle of one
// right-hand side in ONE kernel launch, one CTA per RHS, every step in fp64 except the CNN's
// own arithmetic (fp32 weights and activations, as the smoother is specified):
//   relres_in = ||y - A x|| / ||y||                                      (outer test)
//   x <- NMGF1d(x, y, A, 1, L)   (Alg 3 P:315-339 with nu1 pre / nu2 post steps, reading R9):
//     level l < L: nu1 x { b = y_l - A_l x_l; h = ||b|| N(b / ||b||); x_l += F'_l(h) }
//                  y_{l+1} = R_l (y_l - A_l x_l)
//     level L:     x_L = (A^(L))^{-1} y_L  (explicit fp64 inverse from the Cholesky factor)
//     back up:     x_l += P_l x_{l+1}; nu2 smoothing steps
//   relres_out = ||y - A x|| / ||y||  (nmg_solve's test after the cycle)
// Levels live in shared memory (y_l, x_l fp64 for every level; n <= 1024), the dense fp64
// Galerkin operators A_l and A_L^{-1} are read from L2 by warp-per-row dot products (fixed
// order, deterministic).  The level filter is an fp64 complex FFT of the real row.  For the
// latency-bound small problems (config 0: n = 256, 8 RHS) one launch replaces the ~50 kernel
// launches of the mixed-precision cycle.  The same kernel runs the COARSE SUB-CYCLE of the mixed
// path (yf / xf set): NMGF(0, y_l0) over the levels with n_l <= 512, fp32 in and out, every step
// in between in fp64 -- one launch instead of ~8 per coarse level (latency-bound at small batches).
#include <cmath>

#include "common.cuh"
#include "kernels.h"

namespace nmg {
namespace {

constexpr int NT = 512;
constexpr int C = 16, KS = 5, HK = 2;

struct Smem {
  float* w;         // the level's CNN parameters (1473 floats)
  double2* tw;      // exp(-2 pi i k / n0), k < n0 / 2 (fp64 twiddles of the finest level)
  double* y[8];
  double* x[8];
  double* r;        // n
  double* b;        // n
  float* u;         // n + 4 (zero padded by 2 each side)
  float* a1;        // [C][n + 4]
  float* a2;        // [C][n + 4]
  double2* z;       // n complex (FFT)
  double* red;      // 32
};

// out[i] = (sub ? y[i] : 0) - sum_j A[i][j] v[j]   (warp per 4 rows, lanes over j, fixed order;
// the 4 rows' loads of 4 consecutive j-steps are issued together to hide the L2 latency)
NMG_D void matvec(const double* __restrict__ A, int n, const double* v, const double* y, double* out) {
  constexpr int RW = 4;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i0 = warp * RW; i0 < n; i0 += (NT / 32) * RW) {
    double acc[RW];
#pragma unroll
    for (int r = 0; r < RW; ++r) acc[r] = 0.0;
    const int nr = min(RW, n - i0);
    for (int j0 = 0; j0 < n; j0 += 128) {
      double a[RW][4], vv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = j0 + 32 * q + lane;
        vv[q] = j < n ? v[j] : 0.0;
#pragma unroll
        for (int r = 0; r < RW; ++r) a[r][q] = (j < n && r < nr) ? __ldg(A + (int64_t)(i0 + r) * n + j) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q)
#pragma unroll
        for (int r = 0; r < RW; ++r) acc[r] = fma(a[r][q], vv[q], acc[r]);
    }
#pragma unroll
    for (int r = 0; r < RW; ++r) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[r] += __shfl_xor_sync(0xffffffffu, acc[r], o);
      if (lane == 0 && r < nr) out[i0 + r] = (y ? y[i0 + r] : 0.0) - acc[r];
    }
  }
  __syncthreads();
}

NMG_D double norm2(const double* v, int n, double* red) {
  double ss = 0.0;
  for (int j = threadIdx.x; j < n; j += NT) ss = fma(v[j], v[j], ss);
  return sqrt(block_sum_f64(ss, red));
}

// fp64 complex FFT of length n in shared memory (radix 2, DIF forward natural -> bit-reversed,
// DIT inverse bit-reversed -> natural); twiddles exp(-+2 pi i pos / len) = tw[pos n0 / len]
NMG_D void fft64(double2* z, int n, bool inverse, const double2* tw, int n0) {
  if (!inverse) {
    for (int len = n; len >= 2; len >>= 1) {
      const int half = len >> 1, step = n0 / len;
      for (int i = threadIdx.x; i < (n >> 1); i += NT) {
        const int pos = i & (half - 1), j0 = ((i - pos) << 1) + pos, j1 = j0 + half;
        const double2 w = tw[pos * step];
        const double c = w.x, s = w.y;
        const double2 a = z[j0], b = z[j1];
        z[j0] = make_double2(a.x + b.x, a.y + b.y);
        const double dx = a.x - b.x, dy = a.y - b.y;
        z[j1] = make_double2(dx * c - dy * s, dx * s + dy * c);
      }
      __syncthreads();
    }
  } else {
    for (int len = 2; len <= n; len <<= 1) {
      const int half = len >> 1, step = n0 / len;
      for (int i = threadIdx.x; i < (n >> 1); i += NT) {
        const int pos = i & (half - 1), j0 = ((i - pos) << 1) + pos, j1 = j0 + half;
        const double2 w = tw[pos * step];
        const double c = w.x, s = -w.y;                 // conjugate twiddle
        const double2 a = z[j0], bb = z[j1];
        const double2 b = make_double2(bb.x * c - bb.y * s, bb.x * s + bb.y * c);
        z[j0] = make_double2(a.x + b.x, a.y + b.y);
        z[j1] = make_double2(a.x - b.x, a.y - b.y);
      }
      __syncthreads();
    }
  }
}

// x += F'_l(s N(b / s))   (b in S.b; s = ||b||; s = 0 -> no change)
NMG_D void smooth_step(const Cycle64Args& a, int l, int n, double* x, const Smem& S) {
  const double s = norm2(S.b, n, S.red);
  if (s == 0.0) return;
  // the level's parameters in shared memory: w0 [16][1][5], b0, w1 [16][16][5], b1, w2 [1][16][5], b2
  for (int i = threadIdx.x; i < 1473; i += NT) S.w[i] = __ldg(a.W[l] + i);
  __syncthreads();
  const float* P = S.w;
  const float* w0 = P;
  const float* b0 = w0 + C * KS;
  const float* w1 = b0 + C;
  const float* b1 = w1 + C * C * KS;
  const float* w2 = b1 + C;
  const float b2 = w2[C * KS];
  const int np = n + 2 * HK;
  for (int j = threadIdx.x; j < np; j += NT) {
    const int p = j - HK;
    S.u[j] = (p >= 0 && p < n) ? (float)(S.b[p] / s) : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C * np; i += NT) {     // layer 1 (1 -> 16) + ReLU, zero padding
    const int c = i / np, j = i - c * np, p = j - HK;
    float v = 0.f;
    if (p >= 0 && p < n) {
      float acc = b0[c];
#pragma unroll
      for (int t = 0; t < KS; ++t) acc = fmaf(w0[c * KS + t], S.u[j + t - HK], acc);
      v = fmaxf(acc, 0.f);
    }
    S.a1[i] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < C * np; i += NT) {     // layer 2 (16 -> 16) + ReLU
    const int o = i / np, j = i - o * np, p = j - HK;
    float v = 0.f;
    if (p >= 0 && p < n) {
      float acc = b1[o];
      for (int c = 0; c < C; ++c) {
        const float* wr = w1 + (o * C + c) * KS;
        const float* ar = S.a1 + c * np + j - HK;
#pragma unroll
        for (int t = 0; t < KS; ++t) acc = fmaf(wr[t], ar[t], acc);
      }
      v = fmaxf(acc, 0.f);
    }
    S.a2[i] = v;
  }
  __syncthreads();
  for (int p = threadIdx.x; p < n; p += NT) {          // layer 3 (16 -> 1), h = s N(u) in fp64
    float acc = b2;
    for (int c = 0; c < C; ++c) {
      const float* ar = S.a2 + c * np + p;
#pragma unroll
      for (int t = 0; t < KS; ++t) acc = fmaf(w2[c * KS + t], ar[t], acc);
    }
    S.z[p] = make_double2(s * (double)acc, 0.0);
  }
  __syncthreads();
  if (!a.filter) {
    for (int p = threadIdx.x; p < n; p += NT) x[p] += S.z[p].x;
    __syncthreads();
    return;
  }
  fft64(S.z, n, false, S.tw, a.n);                       // bit-reversed spectrum
  const int lg = 31 - __clz(n);
  for (int j = threadIdx.x; j < n; j += NT) {
    const int k = (int)(__brev((unsigned)j) >> (32 - lg));
    const double m = sqrt(2.0 * (double)min(k, n - k) / (double)n);   // m'_l, reading R5
    S.z[j] = make_double2(S.z[j].x * m, S.z[j].y * m);
  }
  __syncthreads();
  fft64(S.z, n, true, S.tw, a.n);
  for (int p = threadIdx.x; p < n; p += NT) x[p] += S.z[p].x / (double)n;   // Re(IDFT), 1/n
  __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) cycle64_kernel(const __grid_constant__ Cycle64Args a) {
  extern __shared__ __align__(16) double sm64[];
  const int b = blockIdx.x;
  const int n0 = a.n;
  Smem S;
  double* p = sm64;
  for (int l = 0; l < a.L; ++l) { S.y[l] = p; p += n0 >> l; S.x[l] = p; p += n0 >> l; }
  S.r = p; p += n0;
  S.b = p; p += n0;
  S.red = p; p += 32;
  S.z = reinterpret_cast<double2*>(p); p += 2 * n0;
  S.tw = reinterpret_cast<double2*>(p); p += n0;
  S.u = reinterpret_cast<float*>(p);
  S.a1 = S.u + n0 + 2 * HK + 4;
  S.a2 = S.a1 + C * (n0 + 2 * HK);
  S.w = S.a2 + C * (n0 + 2 * HK);
  for (int k = threadIdx.x; k < n0 / 2; k += NT) {
    double sn, cs;
    sincospi(-2.0 * k / n0, &sn, &cs);
    S.tw[k] = make_double2(cs, sn);
  }
  const bool sub = a.yf != nullptr;                     // coarse sub-cycle: NMGF(0, y) of fp32 y
  const double* yg = sub ? nullptr : a.y + (int64_t)b * n0;
  double* xg = sub ? nullptr : a.x + (int64_t)b * n0;
  for (int j = threadIdx.x; j < n0; j += NT) {
    S.y[0][j] = sub ? (double)a.yf[(int64_t)b * n0 + j] : yg[j];
    S.x[0][j] = sub ? 0.0 : xg[j];
  }
  __syncthreads();
  const double ny = sub ? 1.0 : norm2(S.y[0], n0, S.red);
  auto relres = [&]() -> double {
    matvec(a.A[0], n0, S.x[0], S.y[0], S.r);
    const double nr = norm2(S.r, n0, S.red);
    return ny > 0.0 ? nr / ny : 0.0;
  };
  const bool active = a.active_in ? a.active_in[b] != 0 : true;
  if (!sub && !a.relres_after) {
    const double rr = relres();
    if (threadIdx.x == 0) {
      if (a.relres) a.relres[b] = rr;
      if (a.active_out) a.active_out[b] = rr > a.tol ? 1 : 0;
    }
  }
  if (a.do_cycle && active) {
    const int L = a.L;
    for (int l = 0; l < L - 1; ++l) {                    // down: pre-smoothing, restriction
      const int n = n0 >> l;
      if (l > 0)
        for (int j = threadIdx.x; j < n; j += NT) S.x[l][j] = 0.0;
      __syncthreads();
      for (int k = 0; k < a.nu1; ++k) {
        matvec(a.A[l], n, S.x[l], S.y[l], S.b);
        smooth_step(a, l, n, S.x[l], S);
      }
      matvec(a.A[l], n, S.x[l], S.y[l], S.r);            // r_l = y_l - A_l x_l
      const int nc = n >> 1;
      for (int j = threadIdx.x; j < nc; j += NT) {       // full weighting (reading R4)
        const double fm = S.r[max(2 * j - 1, 0)], f0 = S.r[2 * j], f1 = S.r[2 * j + 1],
                     fp = S.r[min(2 * j + 2, n - 1)];
        S.y[l + 1][j] = ((fm + fp) + 3.0 * (f0 + f1)) * 0.125;
      }
      __syncthreads();
    }
    {                                                    // coarsest: x_L = A_L^{-1} y_L
      const int nc = n0 >> (L - 1);
      matvec(a.Ainv, nc, S.y[L - 1], nullptr, S.x[L - 1]);
      for (int j = threadIdx.x; j < nc; j += NT) S.x[L - 1][j] = -S.x[L - 1][j];
      __syncthreads();
    }
    for (int l = L - 2; l >= 0; --l) {                   // up: prolongation, post-smoothing
      const int n = n0 >> l, nc = n >> 1;
      for (int i = threadIdx.x; i < n; i += NT) {        // linear interpolation (reading R4)
        const int j = i >> 1;
        const int k = min(max(j + ((i & 1) ? 1 : -1), 0), nc - 1);
        S.x[l][i] += 0.75 * S.x[l + 1][j] + 0.25 * S.x[l + 1][k];
      }
      __syncthreads();
      for (int k = 0; k < a.nu2; ++k) {
        matvec(a.A[l], n, S.x[l], S.y[l], S.b);
        smooth_step(a, l, n, S.x[l], S);
      }
    }
    for (int j = threadIdx.x; j < n0; j += NT) {
      if (sub) a.xf[(int64_t)b * n0 + j] = (float)S.x[0][j];
      else xg[j] = S.x[0][j];
    }
  }
  if (!sub && a.relres_after) {
    const double rr = relres();
    if (threadIdx.x == 0) {
      if (a.relres) a.relres[b] = rr;
      if (a.active_out) a.active_out[b] = (rr > a.tol && active) ? 1 : 0;
    }
  }
}

}  // namespace

size_t cycle64_smem(int n, int L) {
  size_t d = 0;
  for (int l = 0; l < L; ++l) d += 2 * (size_t)(n >> l);
  d += 2 * (size_t)n + 32 + 2 * (size_t)n + (size_t)n;
  return d * sizeof(double) + sizeof(float) * ((size_t)n + 2 * HK + 4 + 2 * (size_t)C * (n + 2 * HK) + 1476) + 64;
}

void cycle64(const Cycle64Args& a, cudaStream_t s) {
  NMG_SMEM_OPTIN(cycle64_kernel, cycle64_smem(1024, 8));
  cycle64_kernel<<<a.nrhs, NT, cycle64_smem(a.n, a.L), s>>>(a);
}

}  // namespace nmg
