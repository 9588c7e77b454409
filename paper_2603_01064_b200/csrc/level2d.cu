// 2D level operations (Alg 4 "NMGF2d" P:373-401).  Layout: each RHS is an
// n x n column-major matrix X (element (i1, i2) at i1 + n i2, Vec convention P:363),
// i.e. a row-major [i2][i1] array; batches are RHS-major.
//   * restrict2d / prolong_add2d : hat I = I (x) I, tensor products of reading R4
//   * qstencil_resid             : D = C - alpha Q X Q^T (banded Galerkin mass term)
//   * norms_f32                  : ||B_l||_2 Frobenius per RHS in fp64 (R10)
//   * cnn2d_kernel               : fused 4-layer 3x3 CNN smoother N_theta (R7), FFMA
//   * fft2d_*                    : level filter hat F'_l = Re(IDFT2(M' (.) DFT2(.)))
#include <cstdlib>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"

namespace nmg {
namespace {

inline int nblk(int64_t n, int t) { return (int)ceil_div64(n, t); }

NMG_D float r1d(float fm, float f0, float f1, float fp) {
  return __fmul_rn(__fadd_rn(__fadd_rn(fm, fp), __fmul_rn(3.0f, __fadd_rn(f0, f1))), 0.125f);
}

// coarse (b, j2, j1) = R (rows) of R (cols): first along i1 for the 4 fine rows, then i2
__global__ void restrict2d_kernel(int nrhs, int n_c, const float* __restrict__ f, float* __restrict__ c) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)n_c * n_c;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int rem = (int)(idx - b * per);
  const int j2 = rem / n_c, j1 = rem - j2 * n_c;
  const int n_f = 2 * n_c;
  const float* F = f + (int64_t)b * n_f * n_f;
  const int c1[4] = {max(2 * j1 - 1, 0), 2 * j1, 2 * j1 + 1, min(2 * j1 + 2, n_f - 1)};
  const int c2[4] = {max(2 * j2 - 1, 0), 2 * j2, 2 * j2 + 1, min(2 * j2 + 2, n_f - 1)};
  float r[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float* row = F + (int64_t)c2[a] * n_f;
    r[a] = r1d(row[c1[0]], row[c1[1]], row[c1[2]], row[c1[3]]);
  }
  c[idx] = r1d(r[0], r[1], r[2], r[3]);
}

NMG_D float p1d(float cj, float ck) { return __fadd_rn(__fmul_rn(0.75f, cj), __fmul_rn(0.25f, ck)); }

// vectorised restriction: thread = coarse (j2, 2s), (j2, 2s + 1) from 4 fine rows x fine columns
// 4s - 1 .. 4s + 4 (a float4 + two scalars per row); same expression order (bitwise)
__global__ void restrict2d_x2_kernel(int nrhs, int n_c, const float* __restrict__ f, float* __restrict__ c) {
  const int hc = n_c >> 1;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)n_c * hc;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int rem = (int)(idx - b * per);
  const int j2 = rem / hc, sidx = rem - j2 * hc;
  const int n_f = 2 * n_c;
  const float* F = f + (int64_t)b * n_f * n_f;
  const int c2[4] = {max(2 * j2 - 1, 0), 2 * j2, 2 * j2 + 1, min(2 * j2 + 2, n_f - 1)};
  const int xm = max(4 * sidx - 1, 0), xp = min(4 * sidx + 4, n_f - 1);
  float r0[4], r1[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float* row = F + (int64_t)c2[a] * n_f;
    const float4 m = *reinterpret_cast<const float4*>(row + 4 * sidx);
    r0[a] = r1d(row[xm], m.x, m.y, m.z);
    r1[a] = r1d(m.y, m.z, m.w, row[xp]);
  }
  *reinterpret_cast<float2*>(c + ((int64_t)b * n_c + j2) * n_c + 2 * sidx) =
      make_float2(r1d(r0[0], r0[1], r0[2], r0[3]), r1d(r1[0], r1[1], r1[2], r1[3]));
}

// vectorised prolongation: thread = fine (i2, 4t .. 4t + 3) from coarse rows j2, k2 and
// coarse columns 2t - 1 .. 2t + 2 (bitwise prolong_add2d)
__global__ void prolong_add2d_x4_kernel(int nrhs, int n_c, const float* __restrict__ c, float* __restrict__ f) {
  const int q = n_c >> 1;
  const int n_f = 2 * n_c;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)n_f * q;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int rem = (int)(idx - b * per);
  const int i2 = rem / q, t = rem - i2 * q;
  const int j2 = i2 >> 1, k2 = min(max((i2 & 1) ? j2 + 1 : j2 - 1, 0), n_c - 1);
  const float* C = c + (int64_t)b * n_c * n_c;
  const int cm = max(2 * t - 1, 0), cp = min(2 * t + 2, n_c - 1);
  const float* Rj = C + (int64_t)j2 * n_c;
  const float* Rk = C + (int64_t)k2 * n_c;
  const float j0 = Rj[2 * t], j1 = Rj[2 * t + 1], jm = Rj[cm], jp = Rj[cp];
  const float k0 = Rk[2 * t], k1 = Rk[2 * t + 1], km = Rk[cm], kp = Rk[cp];
  float4* fq = reinterpret_cast<float4*>(f + ((int64_t)b * n_f + i2) * n_f) + t;
  float4 v = *fq;
  v.x = __fadd_rn(v.x, p1d(p1d(j0, jm), p1d(k0, km)));
  v.y = __fadd_rn(v.y, p1d(p1d(j0, j1), p1d(k0, k1)));
  v.z = __fadd_rn(v.z, p1d(p1d(j1, j0), p1d(k1, k0)));
  v.w = __fadd_rn(v.w, p1d(p1d(j1, jp), p1d(k1, kp)));
  *fq = v;
}

__global__ void prolong_add2d_kernel(int nrhs, int n_c, const float* __restrict__ c, float* __restrict__ f) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n_f = 2 * n_c;
  const int64_t per = (int64_t)n_f * n_f;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int rem = (int)(idx - b * per);
  const int i2 = rem / n_f, i1 = rem - i2 * n_f;
  const int j1 = i1 >> 1, k1 = min(max((i1 & 1) ? j1 + 1 : j1 - 1, 0), n_c - 1);
  const int j2 = i2 >> 1, k2 = min(max((i2 & 1) ? j2 + 1 : j2 - 1, 0), n_c - 1);
  const float* C = c + (int64_t)b * n_c * n_c;
  const float vj = p1d(C[j2 * n_c + j1], C[j2 * n_c + k1]);
  const float vk = p1d(C[k2 * n_c + j1], C[k2 * n_c + k1]);
  f[idx] = __fadd_rn(f[idx], p1d(vj, vk));
}

// D[b][i2][i1] = C[..] - alpha * sum_{a2, a1} Q[i2][a2] Q[i1][a1] X[b][a2][a1], |a - i| <= hb
__global__ void qstencil_kernel(int nrhs, int n, int hb, float alpha, const float* __restrict__ Q,
                                const float* __restrict__ X, const float* __restrict__ C, float* __restrict__ D) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)n * n;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int rem = (int)(idx - b * per);
  const int i2 = rem / n, i1 = rem - i2 * n;
  const float* Xb = X + (int64_t)b * per;
  float acc = 0.f;
  for (int a2 = max(i2 - hb, 0); a2 <= min(i2 + hb, n - 1); ++a2) {
    const float q2 = Q[(int64_t)i2 * n + a2];
    float t = 0.f;
    for (int a1 = max(i1 - hb, 0); a1 <= min(i1 + hb, n - 1); ++a1) t = fmaf(Q[(int64_t)i1 * n + a1], Xb[(int64_t)a2 * n + a1], t);
    acc = fmaf(q2, t, acc);
  }
  D[idx] = (C ? C[idx] : 0.f) - alpha * acc;
}

// per-RHS sum of squares, fp64, two stages (fixed order => deterministic)
__global__ void __launch_bounds__(256) sumsq_partial_kernel(int64_t N, int chunks, const float* __restrict__ x,
                                                            double* __restrict__ part, int64_t img, int64_t off) {
  __shared__ double red[32];
  const int b = blockIdx.y, ch = blockIdx.x;
  const float* r = x + (int64_t)b * img + off;
  double s = 0.0;
  if ((N & 3) == 0 && (((uintptr_t)r) & 15) == 0) {
    // float4 loads: chunk boundaries on multiples of 4 elements
    const int64_t N4 = N >> 2, len = ceil_div64(N4, chunks);
    const int64_t lo = ch * len, hi = min(N4, lo + len);
    const float4* r4 = reinterpret_cast<const float4*>(r);
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) {
      const float4 v = r4[j];
      s += (double)v.x * (double)v.x + (double)v.y * (double)v.y + (double)v.z * (double)v.z +
           (double)v.w * (double)v.w;
    }
  } else {
    const int64_t len = ceil_div64(N, chunks);
    const int64_t lo = ch * len, hi = min(N, lo + len);
    for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) s += (double)r[j] * (double)r[j];
  }
  s = block_sum_f64(s, red);
  if (threadIdx.x == 0) part[(int64_t)b * chunks + ch] = s;
}
__global__ void sumsq_final_kernel(int nrhs, int chunks, const double* __restrict__ part, double* __restrict__ out,
                                   int take_sqrt) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nrhs) return;
  double s = 0.0;
  for (int c = 0; c < chunks; ++c) s += part[(int64_t)b * chunks + c];
  out[b] = take_sqrt ? sqrt(s) : s;
}

// ------------------------------------------------------------------ fused 2D CNN (FFMA)
// Output tile 16 x 16; 4 layers with 3x3 kernels => halo 4.  Activation planes are
// channel-major [c][y][x] with row stride PS.  Region sizes: in 24, L1 22, L2 20, L3 18.
constexpr int CT = 16;            // output tile
constexpr int PS = 24;            // plane row stride (>= 22 + 2 slack for 4-wide groups)

template <int C>
struct Cnn2dSmem {
  static constexpr int IN = 24 * PS + 8;          // input plane (+ slack)
  static constexpr int A1 = C * 22 * PS + 8;      // layer-1 output; later layer-3 output
  static constexpr int A2 = C * 20 * PS + 8;      // layer-2 output
  static constexpr int W14 = C * 9 + C + C * 9 + 1 + 3;  // layer 1 and 4 params
  static constexpr int FLOATS = IN + A1 + A2 + W14;
};

// one hidden layer C -> C on an output region of w x w (input region w+2), from `in` to `out`.
// Items: (og: C/8 output-channel groups) x (rows w) x (x-groups of 4).  Pixels outside the
// image are written as zeros (zero "same" padding of the next layer).
template <int C>
NMG_D void cnn_hidden_layer(const float* __restrict__ in, float* __restrict__ out, int w,
                            const float* __restrict__ W, const float* __restrict__ Bv, int gy0, int gx0, int n,
                            int tid) {
  const int xg = (w + 3) / 4;
  const int items = (C / 8) * w * xg;
  for (int it = tid; it < items; it += 256) {
    const int og = it / (w * xg);
    const int rem = it - og * (w * xg);
    const int y = rem / xg;
    const int x = (rem - y * xg) * 4;
    float acc[4][8];
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      const float bb = __ldg(Bv + og * 8 + o);
#pragma unroll
      for (int p = 0; p < 4; ++p) acc[p][o] = bb;
    }
#pragma unroll 2
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int t2 = 0; t2 < 3; ++t2) {
        const float* src = in + (c * (w + 2) + y + t2) * PS + x;
        const float4 v0 = *reinterpret_cast<const float4*>(src);
        const float2 v1 = *reinterpret_cast<const float2*>(src + 4);
        const float win[6] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y};
#pragma unroll
        for (int t1 = 0; t1 < 3; ++t1) {
          // weights layout [c][t2][t1][o] (prepared on the host)
          const float4* wp = reinterpret_cast<const float4*>(W + ((c * 3 + t2) * 3 + t1) * C + og * 8);
          const float4 wa = __ldg(wp), wb = __ldg(wp + 1);
          const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
          for (int p = 0; p < 4; ++p)
#pragma unroll
            for (int o = 0; o < 8; ++o) acc[p][o] = fmaf(wv[o], win[p + t1], acc[p][o]);
        }
      }
    }
    const int gy = gy0 + y;
#pragma unroll
    for (int o = 0; o < 8; ++o) {
      float* dst = out + ((og * 8 + o) * w + y) * PS + x;
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int gx = gx0 + x + p;
        const bool inside = gy >= 0 && gy < n && gx >= 0 && gx < n && (x + p) < w;
        dst[p] = inside ? fmaxf(acc[p][o], 0.f) : 0.f;
      }
    }
  }
}

template <int C>
__global__ void __launch_bounds__(256, 1) cnn2d_kernel(Cnn2dArgs a) {
  extern __shared__ __align__(16) float sm[];
  using L = Cnn2dSmem<C>;
  float* in = sm;
  float* act1 = in + L::IN;
  float* act2 = act1 + L::A1;
  float* w14 = act2 + L::A2;
  const int tid = threadIdx.x;
  const int n = a.n;
  const int tiles_x = ceil_div(n, CT);
  const int tile = blockIdx.x, b = blockIdx.y;
  const int ty0 = (tile / tiles_x) * CT, tx0 = (tile % tiles_x) * CT;
  const float* P = a.params;          // [w0 C*9][b0 C][w1' C*C*9][b1 C][w2' C*C*9][b2 C][w3 C*9][b3 1]
  const float* w1t = P + C * 9 + C;   // hidden-layer weights, host-transposed to [c][t2][t1][o]
  const float* b1 = w1t + C * C * 9;
  const float* w2t = b1 + C;
  const float* b2 = w2t + C * C * 9;
  const float* w3 = b2 + C;
  const float b3 = __ldg(w3 + C * 9);
  for (int i = tid; i < C * 9 + C; i += 256) w14[i] = __ldg(P + i);                 // w0, b0
  for (int i = tid; i < C * 9; i += 256) w14[C * 9 + C + i] = __ldg(w3 + i);       // w3
  const double s = a.norms ? a.norms[b] : 1.0;
  const float* X = a.b + (int64_t)b * n * n;
  if (s == 0.0) {   // ||b|| = 0 => h = 0
    if (a.Z || !a.accumulate) {
      for (int i = tid; i < CT * CT; i += 256) {
        const int y = ty0 + i / CT, x = tx0 + i % CT;
        if (y < n && x < n) {
          if (a.Z) zput(a.Z, n, n, b, y, x, 0.f);
          else a.x[((int64_t)b * n + y) * n + x] = 0.f;
        }
      }
    }
    return;
  }
  // input region 24 x 24 at (ty0 - 4, tx0 - 4), scaled by 1/s, zero outside
  for (int i = tid; i < 24 * 24; i += 256) {
    const int y = i / 24, x = i % 24;
    const int gy = ty0 - 4 + y, gx = tx0 - 4 + x;
    float v = 0.f;
    if (gy >= 0 && gy < n && gx >= 0 && gx < n) v = (float)((double)X[(int64_t)gy * n + gx] / s);
    in[y * PS + x] = v;
  }
  __syncthreads();
  // layer 1: 1 -> C on 22 x 22 at (ty0 - 3, tx0 - 3)
  for (int i = tid; i < C * 22 * 22; i += 256) {
    const int c = i / (22 * 22), rem = i - c * 22 * 22, y = rem / 22, x = rem % 22;
    const int gy = ty0 - 3 + y, gx = tx0 - 3 + x;
    float v = 0.f;
    if (gy >= 0 && gy < n && gx >= 0 && gx < n) {
      float acc = w14[C * 9 + c];
#pragma unroll
      for (int t2 = 0; t2 < 3; ++t2)
#pragma unroll
        for (int t1 = 0; t1 < 3; ++t1) acc = fmaf(w14[c * 9 + t2 * 3 + t1], in[(y + t2) * PS + x + t1], acc);
      v = fmaxf(acc, 0.f);
    }
    act1[(c * 22 + y) * PS + x] = v;
  }
  __syncthreads();
  cnn_hidden_layer<C>(act1, act2, 20, w1t, b1, ty0 - 2, tx0 - 2, n, tid);   // layer 2 on 20 x 20
  __syncthreads();
  cnn_hidden_layer<C>(act2, act1, 18, w2t, b2, ty0 - 1, tx0 - 1, n, tid);   // layer 3 on 18 x 18
  __syncthreads();
  // layer 4: C -> 1 on 16 x 16
  {
    const int y = tid / CT, x = tid % CT;
    const int gy = ty0 + y, gx = tx0 + x;
    float acc = b3;
    const float* w3s = w14 + C * 9 + C;
    for (int c = 0; c < C; ++c) {
#pragma unroll
      for (int t2 = 0; t2 < 3; ++t2)
#pragma unroll
        for (int t1 = 0; t1 < 3; ++t1) acc = fmaf(w3s[c * 9 + t2 * 3 + t1], act1[(c * 18 + y + t2) * PS + x + t1], acc);
    }
    if (gy < n && gx < n) {
      const float hv = acc * (float)s;
      const int64_t off = ((int64_t)b * n + gy) * n + gx;
      if (a.Z) zput(a.Z, n, n, b, gy, gx, acc);   // N(u): scaled by s after F'
      else a.x[off] = a.accumulate ? a.x[off] + hv : hv;
    }
  }
}

// ------------------------------------------------------------------ 2D FFT filter passes
// hat F'_l(h) = Re(IDFT2(M' (.) DFT2(h))) of each REAL image h (rows x n) on its own.
// Rows 2r and 2r + 1 travel as one complex row z_r = h_2r + i h_2r+1 (zput, common.cuh):
//   1. forward row FFTs of the rows/2 complex rows (natural-order spectra Z_r[k1]);
//   2. column pass per frequency pair (k1, n - k1), k1 = 0 .. n/2: unmix the two real rows'
//      spectra  H_2r[k1] = (Z_r[k1] + conj Z_r[n-k1]) / 2,  H_2r+1[k1] = (Z_r[k1] - conj Z_r[n-k1]) / 2i
//      (Hermitian symmetry of real rows), FFT along i2, mask M'(k1, k2), inverse FFT along i2,
//      and re-pack  W_r[k1] = Y_2r[k1] + i Y_2r+1[k1],  W_r[n-k1] = conj Y_2r[k1] + i conj Y_2r+1[k1]
//      (the filtered image is real, so Y[n-k1] = conj Y[k1]);
//   3. inverse row FFTs of W_r give y_2r + i y_2r+1 -> scale 1/n^2 (and ||b||) -> x.
// The work equals one complex 2D FFT per RHS PAIR, but no two right-hand sides share a buffer.
// Whole images keep the row spectra in the DIF's bit-reversed order (no permutation pass); the
// mirror of frequency position p (k1 = bitrev(p)) is the reversal of p inside its dyadic block
// [2^j, 2^(j+1)): bitrev(n - bitrev(p)) = 3 * 2^j - 1 - p (p >= 2; positions 0 and 1 hold the
// self-mirrored k1 = 0 and n/2), so a CTA takes a contiguous group of positions and its
// contiguous mirror group.  The slab mode stores natural-order spectra (its all-to-all deals
// mirror-closed frequency chunks to the ranks).

// rows: R complex rows of length n per CTA (R n <= 4096 complex in smem), in place in Z.
// forward: natural in; out bit-reversed (natural = 0) or natural (natural = 1).
// inverse: in bit-reversed (natural = 0) or natural (natural = 1, loaded bit-reversed for the
// DIT pass); complex row Rr = b rpi + r of RHS b writes real rows 2r and 2r + 1 of x at
// b ximg + xoff + (2r) n + col (rpi = rows / 2).
template <int NN>
__global__ void __launch_bounds__(256) fft_rows_kernel(int n_, int64_t nrows, float2* __restrict__ Z,
                                                       const float2* __restrict__ tw, int tw_n, int inverse,
                                                       float* __restrict__ x, int accumulate, float scale,
                                                       const double* __restrict__ norms, int rpi, int64_t ximg,
                                                       int64_t xoff, int natural) {
  const int n = NN > 0 ? NN : n_;   // compile-time for the level sizes (index arithmetic folds)
  extern __shared__ __align__(16) float2 cb[];
  const int R = max(1, 4096 / n);
  const int64_t r0 = (int64_t)blockIdx.x * R;
  const int rows = (int)min((int64_t)R, nrows - r0);
  const int tot = rows * n;
  const int log2n = 31 - __clz(n);
  if (!inverse) {
    for (int i = threadIdx.x; i < tot; i += 256) cb[i] = Z[r0 * n + i];
    __syncthreads();
    fft_dif_forward_batch(cb, n, rows, n, 1, tw, tw_n, threadIdx.x, 256);
    for (int i = threadIdx.x; i < tot; i += 256) {
      const int r = i >> log2n, k = i & (n - 1);
      Z[r0 * n + i] = natural ? cb[r * n + bitrev(k, log2n)] : cb[i];
    }
    return;
  }
  for (int i = threadIdx.x; i < tot; i += 256) {
    const int r = i >> log2n, k = i & (n - 1);
    cb[natural ? r * n + bitrev(k, log2n) : i] = Z[r0 * n + i];
  }
  __syncthreads();
  fft_dit_inverse_batch(cb, n, rows, n, 1, tw, tw_n, threadIdx.x, 256);
  // complex row Rr = r0 + i / n of RHS b = Rr / rpi (rpi = rows per image / 2, a power of two
  // for whole images; the slab mode's R / 2 may not be)
  const bool rp2 = (rpi & (rpi - 1)) == 0;
  const int lrpi = 31 - __clz(rpi);
  for (int i = threadIdx.x; i < tot; i += 256) {
    const int64_t Rr = r0 + (i >> log2n);              // complex row
    const int64_t b = rp2 ? (Rr >> lrpi) : Rr / rpi, r = Rr - b * rpi;
    const int col = i & (n - 1);
    const int64_t o = b * ximg + xoff + 2 * r * n + col;
    const float sb = norms ? (float)norms[b] : 1.f;
    const float v0 = (cb[i].x * scale) * sb, v1 = (cb[i].y * scale) * sb;
    x[o] = accumulate ? x[o] + v0 : v0;
    x[o + n] = accumulate ? x[o + n] + v1 : v1;
  }
}

// combine + forward row FFT: CTA = R complex rows of one RHS; complex row r = (h(2r, .), h(2r+1, .))
// with h the strip kernel's output completed at the strip edges (strip_h_fix), 0 for a RHS with
// ||b|| = 0.  Four consecutive pixels of both rows per thread (two float4 loads).
template <int NN>
__global__ void __launch_bounds__(256) combine_rows_fft_kernel(int n_, int nrhs, const float* __restrict__ q,
                                                               const float4* __restrict__ qe,
                                                               const double* __restrict__ norms,
                                                               float2* __restrict__ Z, int zb0,
                                                               const float2* __restrict__ tw, int tw_n) {
  const int n = NN > 0 ? NN : n_;   // compile-time for the level sizes (index arithmetic folds)
  extern __shared__ __align__(16) float2 cb[];
  const int R = max(1, 4096 / n);
  const int half = n / 2;
  const int rpi = (half + R - 1) / R;                      // CTAs per RHS
  const int b = blockIdx.x / rpi, r0 = (blockIdx.x - b * rpi) * R;
  const int rows = min(R, half - r0);
  const bool on = norms ? norms[b] != 0.0 : true;
  const int64_t per = (int64_t)n * n;
  const int nx = n / kStripSeg;
  if (n % 4 == 0) {
    for (int i4 = threadIdx.x; i4 < rows * n / 4; i4 += 256) {
      const int i = 4 * i4;
      const int r = r0 + i / n, x = i % n;
      float h[2][4];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t row = (int64_t)b * n + 2 * r + e;
        float4 v = on ? __ldg(reinterpret_cast<const float4*>(q + row * n + x)) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (on && n >= kStripSeg) {
          const float4* E = qe + row * nx;
          v.x = strip_h_fix(v.x, E, n, x);          // x % 4 == 0: a possible strip start
          v.w = strip_h_fix(v.w, E, n, x + 3);      // x % 4 == 3: a possible strip end
        }
        h[e][0] = v.x; h[e][1] = v.y; h[e][2] = v.z; h[e][3] = v.w;
      }
      float4* c4 = reinterpret_cast<float4*>(cb + i);
      c4[0] = make_float4(h[0][0], h[1][0], h[0][1], h[1][1]);
      c4[1] = make_float4(h[0][2], h[1][2], h[0][3], h[1][3]);
    }
  } else {
    for (int i = threadIdx.x; i < rows * n; i += 256) {
      const int r = r0 + i / n, x = i % n;
      float h[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t row = (int64_t)b * n + 2 * r + e;
        h[e] = on ? strip_h_fix(__ldg(&q[row * n + x]), qe + row * nx, n, x) : 0.f;
      }
      cb[i] = make_float2(h[0], h[1]);
    }
  }
  __syncthreads();
  fft_dif_forward_batch(cb, n, rows, n, 1, tw, tw_n, threadIdx.x, 256);
  float2* Zp = Z + (int64_t)(zb0 + b) * per / 2 + (int64_t)r0 * n;
  for (int i = threadIdx.x; i < rows * n; i += 256) Zp[i] = cb[i];          // bit-reversed spectra
}

// per-axis profile t[k] = sqrt(2 min(k, n - k) / n); the 2D mask is sqrt(max(q1, q2)) =
// max(t[k1], t[k2]) (sqrt is monotone and correctly rounded, so this is the same value)
NMG_D float mask_axis(int k, int n) { return sqrtf((float)(2 * min(k, n - k)) / (float)n); }

// Column pass on a shared-memory tile cb[i2][c] (n x G): forward along i2, mask M'(k1[c], k2),
// inverse along i2 (unnormalised; the 1/n^2 is applied by the inverse row pass).
NMG_D void cols_filter_tile(float2* cb, int n, int G, const int* k1s, const float2* __restrict__ tw, int tw_n) {
  __shared__ float mt[1024];                                 // the per-axis profile (n <= 1024 here)
  __shared__ float m1s[64];
  const int log2n = 31 - __clz(n);
  for (int k = threadIdx.x; k < n; k += 256) mt[bitrev(k, log2n)] = mask_axis(k, n);   // by DIF position
  for (int c = threadIdx.x; c < G; c += 256) m1s[c] = mask_axis(k1s[c], n);
  fft_dif_forward_batch(cb, n, G, 1, G, tw, tw_n, threadIdx.x, 256);   // ends with __syncthreads
  const int lG = 31 - __clz(G);                              // G a power of two
  for (int i = threadIdx.x; i < n * G; i += 256) {
    const int r = i >> lG, c = i & (G - 1);
    const float m = fmaxf(m1s[c], mt[r]);                   // rows were DIF'd: position r holds k2 = bitrev(r)
    cb[i] = make_float2(cb[i].x * m, cb[i].y * m);
  }
  __syncthreads();
  fft_dit_inverse_batch(cb, n, G, 1, G, tw, tw_n, threadIdx.x, 256);
}

// unmix (step 2): A = Z_r[k1], B = Z_r[n - k1] -> H_2r[k1], H_2r+1[k1]
NMG_D void unmix(float2 A, float2 B, float2& h0, float2& h1) {
  // (A + conj B) / 2 and (A - conj B) / 2i
  h0 = make_float2(0.5f * (A.x + B.x), 0.5f * (A.y - B.y));
  h1 = make_float2(0.5f * (A.y + B.y), -0.5f * (A.x - B.x));
}
// re-pack (step 2): W[k1] = Y0 + i Y1, W[n - k1] = conj Y0 + i conj Y1
NMG_D float2 pack_k(float2 y0, float2 y1) { return make_float2(y0.x - y1.y, y0.y + y1.x); }
NMG_D float2 pack_mirror(float2 y0, float2 y1) { return make_float2(y0.x + y1.y, y1.x - y0.y); }

// whole images: Z_b = [n/2][n] with bit-reversed row spectra.  CTA = (position group, RHS b):
// group 0 = positions {0, 1} (k1 = 0, n/2; self-mirrored); then for each dyadic block
// [2^j, 2^(j+1)), j >= 1, its lower half split in groups of Gs = min(G, 2^(j-1)) positions p,
// each with the mirror positions 3 * 2^j - 1 - p of the upper half.
template <int NN>
__global__ void __launch_bounds__(256) fft_cols_kernel(int n_, int G, float2* __restrict__ Z,
                                                       const float2* __restrict__ tw, int tw_n) {
  const int n = NN > 0 ? NN : n_;   // compile-time for the level sizes (index arithmetic folds)
  extern __shared__ __align__(16) float2 cb[];   // [n][Gc]
  __shared__ int k1s[64];
  const int b = blockIdx.y, half = n / 2;
  const int log2n = 31 - __clz(n);
  int p0 = 0, Gc = 2, S = 1;                      // S = block size (1: the self-mirrored pair)
  {
    int g = blockIdx.x;
    if (g > 0) {
      --g;
      for (S = 2; S < n; S <<= 1) {
        const int cnt = max(1, (S / 2) / G);
        if (g < cnt) { Gc = min(G, S / 2); p0 = S + g * Gc; break; }
        g -= cnt;
      }
    }
  }
  float2* Zb = Z + (int64_t)b * half * n;
  auto mirror = [&](int p) { return S == 1 ? p : 3 * S - 1 - p; };
  for (int c = threadIdx.x; c < Gc; c += 256) k1s[c] = bitrev(p0 + c, log2n);
  const int lGc = 31 - __clz(Gc);                            // Gc a power of two
  for (int i = threadIdx.x; i < half * Gc; i += 256) {
    const int r = i >> lGc, c = i & (Gc - 1);
    const int p = p0 + c;
    float2 h0, h1;
    unmix(Zb[(int64_t)r * n + p], Zb[(int64_t)r * n + mirror(p)], h0, h1);
    cb[(2 * r) * Gc + c] = h0;
    cb[(2 * r + 1) * Gc + c] = h1;
  }
  __syncthreads();
  cols_filter_tile(cb, n, Gc, k1s, tw, tw_n);
  for (int i = threadIdx.x; i < half * Gc; i += 256) {
    const int r = i >> lGc, c = i & (Gc - 1);
    const int p = p0 + c;
    const float2 y0 = cb[(2 * r) * Gc + c], y1 = cb[(2 * r + 1) * Gc + c];
    Zb[(int64_t)r * n + p] = pack_k(y0, y1);
    if (S > 1) Zb[(int64_t)r * n + mirror(p)] = pack_mirror(y0, y1);
  }
}

// ---- slab mode: rank q holds image rows [q R, q R + R) of every RHS: Zs_b = [R/2][n].
// The frequency columns are dealt to the ranks in mirror-closed chunks of CW = 2 h + 1 slots
// (h = n / (2 W)): rank d gets k1 = d h + j (slot j < h), its mirror n - k1 (slot h + j; empty
// for k1 = 0) and, on the last rank, k1 = n/2 (slot 2h; empty elsewhere).
NMG_D int slab_col_of_slot(int d, int j, int h, int n, int W) {   // frequency of slot j, -1 if empty
  if (j < h) return d * h + j;
  if (j < 2 * h) { const int k = d * h + (j - h); return k == 0 ? -1 : n - k; }
  return d == W - 1 ? n / 2 : -1;
}
// dir 0 (pack): buf[d][b][r][j] = Zs[b][r][col(d, j)] (0 for empty slots);  dir 1: the reverse
__global__ void a2a_pack_kernel(int n, int nrhs, int R2, int W, float2* __restrict__ Zs, float2* __restrict__ buf,
                                int dir) {
  const int h = n / (2 * W), CW = 2 * h + 1;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t rows = (int64_t)nrhs * R2;                 // (b, r) pairs
  if (i >= (int64_t)W * rows * CW) return;
  const int j = (int)(i % CW);
  const int64_t br = (i / CW) % rows;
  const int d = (int)(i / (CW * rows));
  const int k = slab_col_of_slot(d, j, h, n, W);
  if (dir == 0) buf[i] = k >= 0 ? Zs[br * n + k] : make_float2(0.f, 0.f);
  else if (k >= 0) Zs[br * n + k] = buf[i];
}
// columns after the all-to-all: buf = [W][nrhs][R2][CW] (chunk q = rank q's complex rows of this
// rank's slots); CTA = (group of G slot pairs j, j + h; RHS b); the last rank's slot 2h (k1 = n/2)
// is one extra group of one column.  Global complex row of (q, r) = q R2 + r.
__global__ void __launch_bounds__(256) fft_cols_slab_kernel(int n, int G, int R2, int W, int rank, int nrhs,
                                                            float2* __restrict__ buf, const float2* __restrict__ tw,
                                                            int tw_n) {
  extern __shared__ __align__(16) float2 cb[];   // [n][Gc]
  __shared__ int k1s[64];
  const int h = n / (2 * W), CW = 2 * h + 1;
  const int b = blockIdx.y;
  const int ng = h / G;
  const bool last = blockIdx.x >= ng;             // the k1 = n/2 slot (last rank only)
  const int Gc = last ? 1 : G;
  const int j0 = last ? 2 * h : blockIdx.x * G;
  const int64_t qstride = (int64_t)nrhs * R2 * CW;
  auto at = [&](int rr, int j) -> int64_t {       // global complex row rr, slot j
    const int q = rr / R2;
    return q * qstride + ((int64_t)b * R2 + (rr - q * R2)) * CW + j;
  };
  for (int c = threadIdx.x; c < Gc; c += 256) k1s[c] = last ? n / 2 : rank * h + j0 + c;
  const int half = n / 2;
  for (int i = threadIdx.x; i < half * Gc; i += 256) {
    const int r = i / Gc, c = i - r * Gc;
    const int j = j0 + c;
    const int k = last ? n / 2 : rank * h + j;
    const float2 A = buf[at(r, j)];
    const float2 B = (last || k == 0) ? A : buf[at(r, j + h)];
    float2 h0, h1;
    unmix(A, B, h0, h1);
    cb[(2 * r) * Gc + c] = h0;
    cb[(2 * r + 1) * Gc + c] = h1;
  }
  __syncthreads();
  cols_filter_tile(cb, n, Gc, k1s, tw, tw_n);
  for (int i = threadIdx.x; i < half * Gc; i += 256) {
    const int r = i / Gc, c = i - r * Gc;
    const int j = j0 + c;
    const int k = last ? n / 2 : rank * h + j;
    const float2 y0 = cb[(2 * r) * Gc + c], y1 = cb[(2 * r + 1) * Gc + c];
    buf[at(r, j)] = pack_k(y0, y1);
    if (!last && k != 0) buf[at(r, j + h)] = pack_mirror(y0, y1);
  }
}

__global__ void real_to_complex_kernel(int nrhs, int n, const float* __restrict__ x, float2* __restrict__ Z) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t N = (int64_t)n * n;
  if (i >= (int64_t)nrhs * N) return;
  const int b = (int)(i / N);
  const int64_t p = i - (int64_t)b * N;
  zput(Z, n, n, b, (int)(p / n), (int)(p % n), x[i]);
}

}  // namespace

void restrict2d(int nrhs, int n_f, const float* f, float* c, cudaStream_t s) {
  const int n_c = n_f / 2;
  if (n_c % 2 == 0 && ((uintptr_t)f & 15) == 0 && ((uintptr_t)c & 7) == 0)
    restrict2d_x2_kernel<<<nblk((int64_t)nrhs * n_c * (n_c / 2), 256), 256, 0, s>>>(nrhs, n_c, f, c);
  else
    restrict2d_kernel<<<nblk((int64_t)nrhs * n_c * n_c, 256), 256, 0, s>>>(nrhs, n_c, f, c);
}
void prolong_add2d(int nrhs, int n_c, const float* c, float* f, cudaStream_t s) {
  if (n_c % 2 == 0 && ((uintptr_t)f & 15) == 0)
    prolong_add2d_x4_kernel<<<nblk((int64_t)nrhs * 2 * n_c * (n_c / 2), 256), 256, 0, s>>>(nrhs, n_c, c, f);
  else
    prolong_add2d_kernel<<<nblk((int64_t)nrhs * 4 * n_c * n_c, 256), 256, 0, s>>>(nrhs, n_c, c, f);
}
void qstencil(int nrhs, int n, int hb, float alpha, const float* Q, const float* X, const float* C, float* D,
              cudaStream_t s) {
  qstencil_kernel<<<nblk((int64_t)nrhs * n * n, 256), 256, 0, s>>>(nrhs, n, hb, alpha, Q, X, C, D);
}
void norms_f32(int nrhs, int64_t N, const float* x, double* part, int chunks, double* out, cudaStream_t s) {
  sumsq_partial_kernel<<<dim3(chunks, nrhs), 256, 0, s>>>(N, chunks, x, part, N, 0);
  sumsq_final_kernel<<<nblk(nrhs, 128), 128, 0, s>>>(nrhs, chunks, part, out, 1);
}
void sumsq_f32(int nrhs, int64_t N, const float* x, int64_t img, int64_t off, double* part, int chunks, double* out,
               cudaStream_t s) {
  sumsq_partial_kernel<<<dim3(chunks, nrhs), 256, 0, s>>>(N, chunks, x, part, img, off);
  sumsq_final_kernel<<<nblk(nrhs, 128), 128, 0, s>>>(nrhs, chunks, part, out, 0);
}
int cnn2d_smem(int C) {
  return (C == 32 ? Cnn2dSmem<32>::FLOATS : Cnn2dSmem<48>::FLOATS) * (int)sizeof(float);
}
void cnn2d(const Cnn2dArgs& a, cudaStream_t s) {
  const int tiles = ceil_div(a.n, CT) * ceil_div(a.n, CT);
  dim3 grid(tiles, a.nrhs);
  const int smem = cnn2d_smem(a.C);
  if (a.C == 32) {
    NMG_SMEM_OPTIN(cnn2d_kernel<32>, smem);
    cnn2d_kernel<32><<<grid, 256, smem, s>>>(a);
  } else {
    NMG_SMEM_OPTIN(cnn2d_kernel<48>, smem);
    cnn2d_kernel<48><<<grid, 256, smem, s>>>(a);
  }
}
// instantiate a kernel for the 2D level sizes (compile-time n), generic otherwise
#define NMG_DISPATCH_N(n, ...)                                     \
  switch (n) {                                                     \
    case 32: { constexpr int NN = 32; __VA_ARGS__; break; }        \
    case 64: { constexpr int NN = 64; __VA_ARGS__; break; }        \
    case 128: { constexpr int NN = 128; __VA_ARGS__; break; }      \
    case 256: { constexpr int NN = 256; __VA_ARGS__; break; }      \
    case 512: { constexpr int NN = 512; __VA_ARGS__; break; }      \
    case 1024: { constexpr int NN = 1024; __VA_ARGS__; break; }    \
    default: { constexpr int NN = 0; __VA_ARGS__; break; }         \
  }
void filter2d(int nrhs, int n, float2* Z, const float2* tw, int tw_n, float* x, bool accumulate, cudaStream_t s,
              const double* norms, bool rows_done) {
  // per-RHS buffers Z_b = [n/2][n] complex (zput); three passes (rows, columns, inverse rows)
  const int64_t nrows = (int64_t)nrhs * (n / 2);
  const int R = std::max(1, 4096 / n);
  const size_t smr = sizeof(float2) * (size_t)R * n;
  if (!rows_done)
    NMG_DISPATCH_N(n, (fft_rows_kernel<NN><<<nblk(nrows, R), 256, smr, s>>>(n, nrows, Z, tw, tw_n, 0, nullptr, 0, 1.f,
                                                                          nullptr, n / 2, (int64_t)n * n, 0, 0)))
  const int G = std::min(std::max(1, n / 2), std::min(64, std::max(2, 4096 / n)));   // 32 KB of columns
  const size_t smc = sizeof(float2) * (size_t)n * std::max(G, 2);
  int groups = 1;
  for (int S = 2; S < n; S <<= 1) groups += std::max(1, (S / 2) / G);
  NMG_DISPATCH_N(n, NMG_SMEM_OPTIN(fft_cols_kernel<NN>, 65536);
                 fft_cols_kernel<NN><<<dim3(groups, nrhs), 256, smc, s>>>(n, G, Z, tw, tw_n))
  NMG_DISPATCH_N(n, (fft_rows_kernel<NN><<<nblk(nrows, R), 256, smr, s>>>(n, nrows, Z, tw, tw_n, 1, x, accumulate ? 1 : 0,
                                                                        1.0f / ((float)n * (float)n), norms, n / 2,
                                                                        (int64_t)n * n, 0, 0)))
}

// ---------------------------------------------------------------- slab-sharded level filter
// Rank `rank` of W holds rows [rank R, rank R + R) of every image: Zs [nrhs][R/2][n].
//   1. row FFTs of the local complex rows (natural-order spectra)
//   2. pack: send chunk d = rank d's mirror-closed frequency slots of every local row
//   3. all-to-all (caller): recv chunk q = rank q's rows of this rank's slots
//   4. unmix, column FFT over i2, mask, inverse, re-pack (in place)
//   5. all-to-all back (caller), unpack into Zs, inverse row FFTs + scale + update of x.
int filter2d_slab_chunk(int n, int W) { return n / W + 1; }   // slots per rank (2 h + 1)
void filter2d_slab_rows(int n, int nrhs, int R, float2* Zs, const float2* tw, int tw_n, cudaStream_t s) {
  const int64_t nrows = (int64_t)nrhs * (R / 2);
  const int RR = std::max(1, 4096 / n);
  const size_t smr = sizeof(float2) * (size_t)RR * n;
  fft_rows_kernel<0><<<nblk(nrows, RR), 256, smr, s>>>(n, nrows, Zs, tw, tw_n, 0, nullptr, 0, 1.f, nullptr, R / 2,
                                                       (int64_t)R * n, 0, 1);
}
void filter2d_slab_inverse(int n, int nrhs, int R, float2* Zs, const float2* tw, int tw_n, float* x, int64_t ximg,
                           int64_t xoff, bool accumulate, const double* norms, cudaStream_t s) {
  const int64_t nrows = (int64_t)nrhs * (R / 2);
  const int RR = std::max(1, 4096 / n);
  const size_t smr = sizeof(float2) * (size_t)RR * n;
  fft_rows_kernel<0><<<nblk(nrows, RR), 256, smr, s>>>(n, nrows, Zs, tw, tw_n, 1, x, accumulate ? 1 : 0,
                                                       1.0f / ((float)n * (float)n), norms, R / 2, ximg, xoff, 1);
}
void filter2d_slab_pack(int n, int nrhs, int R, int W, float2* Zs, float2* buf, bool unpack, cudaStream_t s) {
  const int64_t tot = (int64_t)W * nrhs * (R / 2) * filter2d_slab_chunk(n, W);
  a2a_pack_kernel<<<nblk(tot, 256), 256, 0, s>>>(n, nrhs, R / 2, W, Zs, buf, unpack ? 1 : 0);
}
void filter2d_slab_cols(int n, int nrhs, int R, int W, int rank, float2* buf, const float2* tw, int tw_n,
                        cudaStream_t s) {
  const int h = n / (2 * W);
  const int G = std::min(h, std::min(64, std::max(1, 4096 / n)));
  const size_t smc = sizeof(float2) * (size_t)n * G;
  NMG_SMEM_OPTIN(fft_cols_slab_kernel, 65536);
  const int groups = h / G + (rank == W - 1 ? 1 : 0);
  fft_cols_slab_kernel<<<dim3(groups, nrhs), 256, smc, s>>>(n, G, R / 2, W, rank, nrhs, buf, tw, tw_n);
}
void combine_rows_fft(int n, int nrhs, const float* q, const float4* qe, const double* norms, float2* Z, int zb0,
                      const float2* tw, int tw_n, cudaStream_t s) {
  const int R = std::max(1, 4096 / n);
  const size_t smr = sizeof(float2) * (size_t)R * n;
  NMG_DISPATCH_N(n, (combine_rows_fft_kernel<NN><<<nrhs * ceil_div(n / 2, R), 256, smr, s>>>(n, nrhs, q, qe, norms, Z,
                                                                                           zb0, tw, tw_n)))
}
void real_to_complex(int nrhs, int n, const float* x, float2* Z, cudaStream_t s) {
  real_to_complex_kernel<<<nblk((int64_t)nrhs * n * n, 256), 256, 0, s>>>(nrhs, n, x, Z);
}

}  // namespace nmg
