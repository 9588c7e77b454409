// FNO neural smoother (section 3.1, Appendix A P:651-657,
// hyperparameters per grid Table 6):
//   N(u) = proj o f_L o ... o f_1 o lift(u),   f(Z) = GELU( DFT^{-1}(R (.) DFT(Z)) + W * Z + B ),
// R a complex c x c channel mixing on the k lowest modes per axis (the rest zeroed), W a
// convolution (kernel ks, zero "same" padding), lift / proj pointwise 1 -> c -> 1 (reading R24:
// sigma = exact GELU).  fp32 SIMT kernels, RHS-major activations Z [b][c][N_l]:
//   fno_lift       Z0 = lift(b / ||b||)
//   per layer      spectral forward (row FFTs in shared memory, fft.cuh; 2D: rows then columns)
//                  -> Zh [b][mode][c] (complex) -> mode mixing Yh = Zh R -> inverse (Hermitian
//                  completion, real output) into Z1 -> Z1 = GELU(Z1 + B + W * Z0) -> swap
//                  (the W convolution: fno_conv_tc, 3xTF32 implicit GEMM on tcgen05 over channels-last
//                  tf32 hi/lo copies of the layer input, fno_tc.cu; the fp32 SIMT fno_conv1d/2d
//                  kernels below serve the shapes it does not take: c % 16 != 0, 1D n < 128, 2D n < 16)
//   fno_proj       h = proj(Z) -> 1D: x (+)= ||b|| F'_l(h) (fused level filter); 2D: the level
//                  filter's input buffer (zput), filter2d finishes.
#include <algorithm>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"

namespace nmg {
namespace {

inline int nblk(int64_t n, int t) { return (int)ceil_div64(n, t); }
constexpr int NT = 256;

NMG_D float gelu(float z) { return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f)); }

// Z0[b][c][p] = lw[c] u + lb[c], u = in[b][p] / s_b (s_b = 0: u = 0)
__global__ void fno_lift_kernel(int nrhs, int c, int64_t N, const float* __restrict__ in,
                                const double* __restrict__ norms, const float* __restrict__ lw,
                                const float* __restrict__ lb, float* __restrict__ Z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nrhs * c * N) return;
  const int64_t p = i % N;
  const int64_t bc = i / N;
  const int ch = (int)(bc % c), b = (int)(bc / c);
  const double s = norms ? norms[b] : 1.0;
  const float u = s != 0.0 ? (float)((double)in[(int64_t)b * N + p] / s) : 0.f;
  Z[i] = fmaf(__ldg(lw + ch), u, __ldg(lb + ch));
}

// forward row DFTs of length n over `rows` rows of Z (row r = Z + r n, real); keep modes
// m < k: out[(r / per) * ostride_b + m * ostride_m + (r % per) * ostride_r] (complex).
// 1D: rows = (b, c), per = c, out = Zh [b][m][c]  (ostride_b = k c, ostride_m = c, ostride_r = 1)
// 2D row pass: rows = (b, c, i2), per = c n, out = T [b][c][i2][m] (ostride_b = c n k, ostride_m = 1,
//   ostride_r = k)
__global__ void __launch_bounds__(NT) fno_rows_fwd_kernel(int n, int64_t rows, int k, const float* __restrict__ Z,
                                                          float2* __restrict__ out, int64_t per, int64_t ostride_b,
                                                          int64_t ostride_m, int64_t ostride_r,
                                                          const float2* __restrict__ tw, int tw_n) {
  // real rows 2q and 2q + 1 travel as one complex row z = x_a + i x_b (half the FFT work); the kept
  // modes are unmixed by the Hermitian symmetry of real rows: X_a[m] = (Z[m] + conj Z[n-m]) / 2,
  // X_b[m] = (Z[m] - conj Z[n-m]) / 2i
  extern __shared__ __align__(16) float2 cb[];
  const int R = max(1, 4096 / n);                      // complex rows per CTA
  const int64_t r0 = (int64_t)blockIdx.x * 2 * R;      // first real row
  const int cnt = (int)min((int64_t)2 * R, rows - r0);
  const int cntc = (cnt + 1) >> 1;
  const int log2n = 31 - __clz(n);
  for (int i = threadIdx.x; i < cntc * n; i += NT) {
    const int q = i >> log2n, p = i & (n - 1);
    const float* za = Z + (r0 + 2 * q) * n + p;
    cb[i] = make_float2(za[0], 2 * q + 1 < cnt ? za[n] : 0.f);
  }
  __syncthreads();
  fft_dif_forward_batch(cb, n, cntc, n, 1, tw, tw_n, threadIdx.x, NT);
  for (int i = threadIdx.x; i < cntc * k; i += NT) {
    const int q = i / k, m = i - q * k;
    const float2 A = cb[q * n + bitrev(m, log2n)], B = cb[q * n + bitrev((n - m) & (n - 1), log2n)];
    const int64_t ra = r0 + 2 * q;
    out[(ra / per) * ostride_b + m * ostride_m + (ra % per) * ostride_r] =
        make_float2(0.5f * (A.x + B.x), 0.5f * (A.y - B.y));
    if (2 * q + 1 < cnt) {
      const int64_t rb = ra + 1;
      out[(rb / per) * ostride_b + m * ostride_m + (rb % per) * ostride_r] =
          make_float2(0.5f * (A.y + B.y), -0.5f * (A.x - B.x));
    }
  }
}

// 2D forward column pass: T [b][c][i2][k] -> Zh [b][(j2, m1)][c], j2 < k: i2-mode j2, j2 >= k:
// i2-mode n - 2k + j2.  CTA = (group of G i1-modes, channel c, RHS b).
__global__ void __launch_bounds__(NT) fno_cols_fwd_kernel(int n, int k, int c, int G, const float2* __restrict__ T,
                                                          float2* __restrict__ Zh, const float2* __restrict__ tw,
                                                          int tw_n) {
  extern __shared__ __align__(16) float2 cb[];   // [n][G]
  const int m0 = blockIdx.x * G, ch = blockIdx.y, b = blockIdx.z;
  const int log2n = 31 - __clz(n);
  const float2* Tb = T + (((int64_t)b * c + ch) * n) * k;
  for (int i = threadIdx.x; i < n * G; i += NT) {
    const int r = i / G, g = i - r * G;
    cb[i] = Tb[(int64_t)r * k + m0 + g];
  }
  __syncthreads();
  fft_dif_forward_batch(cb, n, G, 1, G, tw, tw_n, threadIdx.x, NT);
  const int modes = 2 * k * k;
  for (int i = threadIdx.x; i < 2 * k * G; i += NT) {
    const int j2 = i / G, g = i - j2 * G;
    const int m2 = j2 < k ? j2 : n - 2 * k + j2;
    Zh[((int64_t)b * modes + (int64_t)j2 * k + m0 + g) * c + ch] = cb[bitrev(m2, log2n) * G + g];
  }
}

// Yh[b][m][o] = sum_c Zh[b][m][c] R[m][c][o] (complex); CTA = (mode m, 16 RHS), c <= 64
__global__ void __launch_bounds__(NT) fno_mix_kernel(int nrhs, int modes, int c, const float2* __restrict__ Zh,
                                                     const float2* __restrict__ R, float2* __restrict__ Yh) {
  __shared__ float2 Rs[64 * 64];
  __shared__ float2 Zs[16 * 64];
  const int m = blockIdx.x, b0 = blockIdx.y * 16;
  const int nb = min(16, nrhs - b0);
  const float2* Rm = R + (int64_t)m * c * c;
  for (int i = threadIdx.x; i < c * c; i += NT) Rs[i] = Rm[i];
  for (int i = threadIdx.x; i < nb * c; i += NT) {
    const int bb = i / c, ch = i - bb * c;
    Zs[bb * 64 + ch] = Zh[((int64_t)(b0 + bb) * modes + m) * c + ch];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb * c; i += NT) {
    const int bb = i / c, o = i - bb * c;
    float2 acc = make_float2(0.f, 0.f);
    for (int ch = 0; ch < c; ++ch) {
      const float2 z = Zs[bb * 64 + ch], r = Rs[ch * c + o];
      acc.x = fmaf(z.x, r.x, fmaf(-z.y, r.y, acc.x));
      acc.y = fmaf(z.x, r.y, fmaf(z.y, r.x, acc.y));
    }
    Yh[((int64_t)(b0 + bb) * modes + m) * c + o] = acc;
  }
}

// 2D inverse column pass: Yh [b][(j2, m1)][o] -> T [b][o][i2][m1] (complex inverse DFT along i2 of
// the spectrum with the kept i2-modes, zero elsewhere).  CTA = (group of G i1-modes, o, b).
__global__ void __launch_bounds__(NT) fno_cols_inv_kernel(int n, int k, int c, int G, const float2* __restrict__ Yh,
                                                          float2* __restrict__ T, const float2* __restrict__ tw,
                                                          int tw_n) {
  extern __shared__ __align__(16) float2 cb[];   // [n][G]
  const int m0 = blockIdx.x * G, o = blockIdx.y, b = blockIdx.z;
  const int log2n = 31 - __clz(n);
  const int modes = 2 * k * k;
  for (int i = threadIdx.x; i < n * G; i += NT) cb[i] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int i = threadIdx.x; i < 2 * k * G; i += NT) {
    const int j2 = i / G, g = i - j2 * G;
    const int m2 = j2 < k ? j2 : n - 2 * k + j2;
    cb[bitrev(m2, log2n) * G + g] = Yh[((int64_t)b * modes + (int64_t)j2 * k + m0 + g) * c + o];
  }
  __syncthreads();
  fft_dit_inverse_batch(cb, n, G, 1, G, tw, tw_n, threadIdx.x, NT);
  float2* Tb = T + (((int64_t)b * c + o) * n) * k;
  for (int i = threadIdx.x; i < n * G; i += NT) {
    const int r = i / G, g = i - r * G;
    Tb[(int64_t)r * k + m0 + g] = cb[i];
  }
}

// inverse real row DFTs: row r has modes X[m] = in[(r / per) * istride_b + m * istride_m +
// (r % per) * istride_r], m < k; the real signal is (Re X0 + 2 sum_{0<m<k} Re(X_m e^{2 pi i m p/n})) * scale
// (Hermitian completion; the DC term's imaginary part is dropped as in irfft) -> Z[r][p]
__global__ void __launch_bounds__(NT) fno_rows_inv_kernel(int n, int64_t rows, int k, const float2* __restrict__ in,
                                                          int64_t per, int64_t istride_b, int64_t istride_m,
                                                          int64_t istride_r, float scale, float* __restrict__ Z,
                                                          const float2* __restrict__ tw, int tw_n) {
  // real rows 2q and 2q + 1 as one complex inverse transform of W = Y_a + i Y_b (both Hermitian
  // completed): W[m] = Y_a[m] + i Y_b[m], W[n-m] = conj Y_a[m] + i conj Y_b[m]; y_a = Re, y_b = Im
  extern __shared__ __align__(16) float2 cb[];
  const int R = max(1, 4096 / n);                      // complex rows per CTA
  const int64_t r0 = (int64_t)blockIdx.x * 2 * R;      // first real row
  const int cnt = (int)min((int64_t)2 * R, rows - r0);
  const int cntc = (cnt + 1) >> 1;
  const int log2n = 31 - __clz(n);
  for (int i = threadIdx.x; i < cntc * n; i += NT) cb[i] = make_float2(0.f, 0.f);
  __syncthreads();
  for (int i = threadIdx.x; i < cntc * k; i += NT) {
    const int q = i / k, m = i - q * k;
    const int64_t ra = r0 + 2 * q, rb = ra + 1;
    const float2 A = in[(ra / per) * istride_b + m * istride_m + (ra % per) * istride_r];
    const float2 B = 2 * q + 1 < cnt ? in[(rb / per) * istride_b + m * istride_m + (rb % per) * istride_r]
                                     : make_float2(0.f, 0.f);
    if (m == 0) {
      cb[q * n] = make_float2(A.x, B.x);          // bitrev(0) = 0; DC imaginary parts dropped (irfft)
    } else {
      cb[q * n + bitrev(m, log2n)] = make_float2(A.x - B.y, A.y + B.x);
      cb[q * n + bitrev(n - m, log2n)] = make_float2(A.x + B.y, B.x - A.y);
    }
  }
  __syncthreads();
  fft_dit_inverse_batch(cb, n, cntc, n, 1, tw, tw_n, threadIdx.x, NT);
  for (int i = threadIdx.x; i < cntc * n; i += NT) {
    const int q = i >> log2n, p = i & (n - 1);
    float* za = Z + (r0 + 2 * q) * n + p;
    za[0] = cb[i].x * scale;
    if (2 * q + 1 < cnt) za[n] = cb[i].y * scale;
  }
}

// 1D: Z1[b][o][p] = GELU(Z1[b][o][p] + B[o] + sum_{c,t} W[o][c][t] Z0[b][c][p + t - ks/2])
// CTA = (64-position tile, RHS b); thread = 4 outputs o x 4 positions (c <= 64, ks <= 7)
constexpr int CT1 = 64;
__global__ void __launch_bounds__(NT) fno_conv1d_kernel(int n, int c, int ks, const float* __restrict__ Z0,
                                                        const float* __restrict__ W, const float* __restrict__ B,
                                                        float* __restrict__ Z1) {
  extern __shared__ __align__(16) float sm1[];
  const int h = ks / 2, TW = CT1 + ks - 1;
  float* Ws = sm1;                       // [c][ks][o]   (o fastest)
  float* Xs = Ws + c * ks * c;           // [c][TW]
  const int p0 = blockIdx.x * CT1, b = blockIdx.y;
  for (int i = threadIdx.x; i < c * c * ks; i += NT) {
    const int o = i / (c * ks), r = i - o * c * ks, ch = r / ks, t = r - ch * ks;
    Ws[(ch * ks + t) * c + o] = W[i];
  }
  const float* Zb = Z0 + (int64_t)b * c * n;
  for (int i = threadIdx.x; i < c * TW; i += NT) {
    const int ch = i / TW, q = i - ch * TW, p = p0 - h + q;
    Xs[i] = (p >= 0 && p < n) ? Zb[(int64_t)ch * n + p] : 0.f;
  }
  __syncthreads();
  const int og = threadIdx.x / 16, pg = threadIdx.x % 16;    // 16 o-groups x 16 p-groups
  for (int ob = og * 4; ob < c; ob += 64) {
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][e] = 0.f;
    for (int ch = 0; ch < c; ++ch) {
      for (int t = 0; t < ks; ++t) {
        float w[4], x[4];
#pragma unroll
        for (int a = 0; a < 4; ++a) w[a] = (ob + a < c) ? Ws[(ch * ks + t) * c + ob + a] : 0.f;
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = Xs[ch * TW + pg * 4 + e + t];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[a][e] = fmaf(w[a], x[e], acc[a][e]);
      }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int o = ob + a;
      if (o >= c) continue;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int p = p0 + pg * 4 + e;
        if (p >= n) continue;
        const int64_t at = ((int64_t)b * c + o) * n + p;
        Z1[at] = gelu(Z1[at] + __ldg(B + o) + acc[a][e]);
      }
    }
  }
}

// 2D: same with a ks x ks kernel; CTA = (16 x 16 pixel tile, RHS b); input channels in chunks of
// CC; thread = 4 outputs o x 4 pixels (a 1 x 4 strip along i1)
constexpr int CT2 = 16, CC = 4;
__global__ void __launch_bounds__(NT) fno_conv2d_kernel(int n, int c, int ks, const float* __restrict__ Z0,
                                                        const float* __restrict__ W, const float* __restrict__ B,
                                                        float* __restrict__ Z1) {
  extern __shared__ __align__(16) float sm2[];
  const int h = ks / 2, TW = CT2 + ks - 1, kk = ks * ks;
  float* Ws = sm2;                       // [CC][kk][o]
  float* Xs = Ws + CC * kk * c;          // [CC][TW][TW]
  const int tiles = ceil_div(n, CT2);
  const int ty0 = (blockIdx.x / tiles) * CT2, tx0 = (blockIdx.x % tiles) * CT2, b = blockIdx.y;
  const int og = threadIdx.x / 64, pq = threadIdx.x % 64;    // 4 o-groups x 64 pixel quads
  const int py = pq / 4, px0 = (pq % 4) * 4;
  float acc[16][4];
#pragma unroll
  for (int a = 0; a < 16; ++a)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[a][e] = 0.f;
  const float* Zb = Z0 + (int64_t)b * c * n * n;
  for (int c0 = 0; c0 < c; c0 += CC) {
    __syncthreads();
    for (int i = threadIdx.x; i < CC * kk * c; i += NT) {
      const int o = i % c, r = i / c, t = r % kk, cc = r / kk;
      Ws[i] = (c0 + cc < c) ? W[((int64_t)o * c + c0 + cc) * kk + t] : 0.f;
    }
    for (int i = threadIdx.x; i < CC * TW * TW; i += NT) {
      const int cc = i / (TW * TW), r = i - cc * TW * TW, yy = r / TW, xx = r - yy * TW;
      const int gy = ty0 - h + yy, gx = tx0 - h + xx;
      Xs[i] = (c0 + cc < c && gy >= 0 && gy < n && gx >= 0 && gx < n) ? Zb[((int64_t)(c0 + cc) * n + gy) * n + gx] : 0.f;
    }
    __syncthreads();
    for (int cc = 0; cc < CC; ++cc)
      for (int t2 = 0; t2 < ks; ++t2)
        for (int t1 = 0; t1 < ks; ++t1) {
          float x[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) x[e] = Xs[(cc * TW + py + t2) * TW + px0 + e + t1];
          const float* wr = Ws + (cc * kk + t2 * ks + t1) * c + og * 16;
#pragma unroll
          for (int a = 0; a < 16; ++a) {
            const float w = (og * 16 + a < c) ? wr[a] : 0.f;
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[a][e] = fmaf(w, x[e], acc[a][e]);
          }
        }
  }
  const int gy = ty0 + py;
  if (gy >= n) return;
#pragma unroll
  for (int a = 0; a < 16; ++a) {
    const int o = og * 16 + a;
    if (o >= c) continue;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int gx = tx0 + px0 + e;
      if (gx >= n) continue;
      const int64_t at = (((int64_t)b * c + o) * n + gy) * n + gx;
      Z1[at] = gelu(Z1[at] + __ldg(B + o) + acc[a][e]);
    }
  }
}

// h = proj(Z) (normalised output N(u));  1D: x (+)= s F'_l(h)  (s = ||b||; one CTA per RHS);
// 2D: h -> the level filter's input buffer (zput layout), filter2d applies F' and s
__global__ void __launch_bounds__(NT) fno_proj1d_kernel(int n, int c, const float* __restrict__ Z,
                                                        const float* __restrict__ pw, float pb,
                                                        const double* __restrict__ norms, int filter,
                                                        float* __restrict__ x, int accumulate,
                                                        const float2* __restrict__ tw, int tw_n) {
  extern __shared__ __align__(16) float hb[];
  const int b = blockIdx.x;
  const double s = norms ? norms[b] : 1.0;
  const float* Zb = Z + (int64_t)b * c * n;
  for (int p = threadIdx.x; p < n; p += NT) {
    float acc = pb;
    for (int ch = 0; ch < c; ++ch) acc = fmaf(__ldg(pw + ch), Zb[(int64_t)ch * n + p], acc);
    hb[p] = s != 0.0 ? acc : 0.f;
  }
  if (filter) real_level_filter(hb, n, tw, tw_n, threadIdx.x, NT);   // unnormalised: x 2/n below
  __syncthreads();
  const float sc = filter ? 2.0f / (float)n : 1.0f;
  for (int p = threadIdx.x; p < n; p += NT) {
    const float v = (hb[p] * sc) * (float)s;
    const int64_t at = (int64_t)b * n + p;
    x[at] = accumulate ? x[at] + v : v;
  }
}

__global__ void fno_proj2d_kernel(int nrhs, int n, int c, const float* __restrict__ Z, const float* __restrict__ pw,
                                  float pb, const double* __restrict__ norms, float2* __restrict__ Zf, int zb0,
                                  float* __restrict__ x, int accumulate) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t N = (int64_t)n * n;
  if (i >= (int64_t)nrhs * N) return;
  const int b = (int)(i / N);
  const int64_t p = i - (int64_t)b * N;
  const double s = norms ? norms[b] : 1.0;
  float acc = pb;
  const float* Zb = Z + (int64_t)b * c * N + p;
  for (int ch = 0; ch < c; ++ch) acc = fmaf(__ldg(pw + ch), Zb[(int64_t)ch * N], acc);
  if (s == 0.0) acc = 0.f;
  if (Zf) {
    zput(Zf, n, n, zb0 + b, (int)(p / n), (int)(p % n), acc);
  } else {
    const float v = acc * (float)s;
    x[i] = accumulate ? x[i] + v : v;
  }
}

}  // namespace

size_t fno_conv_smem(int dim, int c, int ks) {
  if (dim == 1) return sizeof(float) * ((size_t)c * ks * c + (size_t)c * (CT1 + ks - 1));
  return sizeof(float) * ((size_t)CC * ks * ks * c + (size_t)CC * (CT2 + ks - 1) * (CT2 + ks - 1));
}

// One FNO forward for `nrhs` RHS of one level (see the file comment).  Z0, Z1: [nrhs][c][N];
// T (2D): [nrhs][c][n][k] complex; Zh, Yh: [nrhs][modes][c] complex.
void fno_forward(const FnoArgs& a, cudaStream_t s) {
  const int n = a.n, c = a.c, k = a.k, ks = a.ks;
  const int64_t N = a.dim == 1 ? (int64_t)n : (int64_t)n * n;
  const int modes = a.dim == 1 ? k : 2 * k * k;
  fno_lift_kernel<<<nblk((int64_t)a.nrhs * c * N, NT), NT, 0, s>>>(a.nrhs, c, N, a.in, a.norms, a.lift_w, a.lift_b,
                                                                  a.Z0);
  const bool tc = a.tXh[0] != nullptr;
  FnoConvArgs ca{};
  if (tc) {
    fno_lift_cl(a.nrhs, c, N, a.in, a.norms, a.lift_w, a.lift_b, a.Xh[0], a.Xl[0], s);
    int bx, by;
    fno_tc_box(n, &bx, &by);
    ca.dim = a.dim; ca.n = n; ca.c = c; ca.ks = ks; ca.nrhs = a.nrhs;
    ca.lbx = 31 - __builtin_clz((unsigned)bx);
    ca.rows = a.tc_rows;
  }
  const int R = std::max(1, 4096 / n);
  const size_t smr = sizeof(float2) * (size_t)R * n;
  const size_t smc = fno_conv_smem(a.dim, c, ks);
  if (tc) {}
  else if (a.dim == 1) NMG_SMEM_OPTIN(fno_conv1d_kernel, fno_conv_smem(1, 64, 7));
  else NMG_SMEM_OPTIN(fno_conv2d_kernel, fno_conv_smem(2, 64, 7));
  float* Z0 = a.Z0;
  float* Z1 = a.Z1;
  for (int l = 0; l < a.L; ++l) {
    const FnoLayer& ly = a.layer[l];
    if (a.dim == 1) {
      const int64_t rows = (int64_t)a.nrhs * c;
      fno_rows_fwd_kernel<<<nblk(rows, 2 * R), NT, smr, s>>>(n, rows, k, Z0, a.Zh, c, (int64_t)k * c, c, 1, a.tw, a.tw_n);
      fno_mix_kernel<<<dim3(modes, ceil_div(a.nrhs, 16)), NT, 0, s>>>(a.nrhs, modes, c, a.Zh, ly.R, a.Yh);
      fno_rows_inv_kernel<<<nblk(rows, 2 * R), NT, smr, s>>>(n, rows, k, a.Yh, c, (int64_t)k * c, c, 1, 1.0f / (float)n,
                                                         Z1, a.tw, a.tw_n);
      if (tc) {
        ca.bias = ly.B; ca.Z1 = Z1;
        ca.Xh_out = l + 1 < a.L ? a.Xh[(l + 1) & 1] : nullptr;
        ca.Xl_out = l + 1 < a.L ? a.Xl[(l + 1) & 1] : nullptr;
        fno_conv_tc(a.tXh[l & 1], a.tXl[l & 1], ly.tWh, ly.tWl, ca, s);
      } else {
        fno_conv1d_kernel<<<dim3(ceil_div(n, CT1), a.nrhs), NT, smc, s>>>(n, c, ks, Z0, ly.W, ly.B, Z1);
      }
    } else {
      const int64_t rows = (int64_t)a.nrhs * c * n;
      const int64_t per = (int64_t)c * n;
      // rows (b, c, i2) -> T[b][c][i2][m1]
      fno_rows_fwd_kernel<<<nblk(rows, 2 * R), NT, smr, s>>>(n, rows, k, Z0, a.T, per, per * k, 1, k, a.tw, a.tw_n);
      const int G = std::min(k, std::max(1, 4096 / n));
      const size_t smg = sizeof(float2) * (size_t)n * G;
      fno_cols_fwd_kernel<<<dim3(k / G, c, a.nrhs), NT, smg, s>>>(n, k, c, G, a.T, a.Zh, a.tw, a.tw_n);
      fno_mix_kernel<<<dim3(modes, ceil_div(a.nrhs, 16)), NT, 0, s>>>(a.nrhs, modes, c, a.Zh, ly.R, a.Yh);
      fno_cols_inv_kernel<<<dim3(k / G, c, a.nrhs), NT, smg, s>>>(n, k, c, G, a.Yh, a.T, a.tw, a.tw_n);
      fno_rows_inv_kernel<<<nblk(rows, 2 * R), NT, smr, s>>>(n, rows, k, a.T, per, per * k, 1, k,
                                                         1.0f / ((float)n * (float)n), Z1, a.tw, a.tw_n);
      if (tc) {
        ca.bias = ly.B; ca.Z1 = Z1;
        ca.Xh_out = l + 1 < a.L ? a.Xh[(l + 1) & 1] : nullptr;
        ca.Xl_out = l + 1 < a.L ? a.Xl[(l + 1) & 1] : nullptr;
        fno_conv_tc(a.tXh[l & 1], a.tXl[l & 1], ly.tWh, ly.tWl, ca, s);
      } else {
        fno_conv2d_kernel<<<dim3(ceil_div(n, CT2) * ceil_div(n, CT2), a.nrhs), NT, smc, s>>>(n, c, ks, Z0, ly.W,
                                                                                             ly.B, Z1);
      }
    }
    std::swap(Z0, Z1);
  }
  if (a.dim == 1) {
    fno_proj1d_kernel<<<a.nrhs, NT, sizeof(float) * (size_t)std::max(n, 4), s>>>(
        n, c, Z0, a.proj_w, a.proj_b, a.norms, a.filter ? 1 : 0, a.x, a.accumulate ? 1 : 0, a.tw, a.tw_n);
  } else {
    fno_proj2d_kernel<<<nblk((int64_t)a.nrhs * N, NT), NT, 0, s>>>(a.nrhs, n, c, Z0, a.proj_w, a.proj_b, a.norms,
                                                                   a.Zf, a.zb0, a.x, a.accumulate ? 1 : 0);
  }
}

int fno_launches(int dim, int L, bool tc) { return 1 + (tc ? 1 : 0) + L * (dim == 1 ? 4 : 6) + 1; }

}  // namespace nmg
