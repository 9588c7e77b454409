// Shared-memory radix-2 FFTs used by the level filter F'_l
// (F'_l(h) = Re(DFT^{-1}(m'_l (.) DFT(h))); 2D PAPER.md:415).
// Forward: decimation-in-time on bit-reversed input -> natural-order spectrum.
// Inverse: decimation-in-frequency on natural input -> bit-reversed output.
// Unnormalised forward, 1/n applied by the caller on the inverse (reading R6).
#pragma once
#include "common.cuh"

namespace nmg {

NMG_D float2 cmul(float2 a, float2 b) { return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
NMG_D float2 cmulc(float2 a, float2 b) { return make_float2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y); }  // a * conj(b)

NMG_D int bitrev(int v, int log2n) { return (int)(__brev((unsigned)v) >> (32 - log2n)); }

// twiddle table tw[k] = exp(-2 pi i k / tw_n), k < tw_n/2; tw_n >= n, both powers of two.
// Block-cooperative; ends with __syncthreads().
NMG_D void fft_dit_forward(float2* c, int n, const float2* __restrict__ tw, int tw_n, int tid, int nthr) {
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1;
    const int step = tw_n / len;
    for (int i = tid; i < (n >> 1); i += nthr) {
      const int pos = i & (half - 1);
      const int j0 = ((i - pos) << 1) + pos;
      const int j1 = j0 + half;
      const float2 w = __ldg(tw + pos * step);
      const float2 a = c[j0];
      const float2 b = cmul(c[j1], w);
      c[j0] = make_float2(a.x + b.x, a.y + b.y);
      c[j1] = make_float2(a.x - b.x, a.y - b.y);
    }
    __syncthreads();
  }
}

NMG_D void fft_dif_inverse(float2* c, int n, const float2* __restrict__ tw, int tw_n, int tid, int nthr) {
  for (int len = n; len >= 2; len >>= 1) {
    const int half = len >> 1;
    const int step = tw_n / len;
    for (int i = tid; i < (n >> 1); i += nthr) {
      const int pos = i & (half - 1);
      const int j0 = ((i - pos) << 1) + pos;
      const int j1 = j0 + half;
      const float2 w = __ldg(tw + pos * step);
      const float2 a = c[j0];
      const float2 b = c[j1];
      c[j0] = make_float2(a.x + b.x, a.y + b.y);
      c[j1] = cmulc(make_float2(a.x - b.x, a.y - b.y), w);   // inverse: conj twiddle
    }
    __syncthreads();
  }
}

// Forward DIF: natural-order input -> bit-reversed spectrum (no permutation pass).
NMG_D void fft_dif_forward(float2* c, int n, const float2* __restrict__ tw, int tw_n, int tid, int nthr) {
  for (int len = n; len >= 2; len >>= 1) {
    const int half = len >> 1;
    const int step = tw_n / len;
    for (int i = tid; i < (n >> 1); i += nthr) {
      const int pos = i & (half - 1);
      const int j0 = ((i - pos) << 1) + pos;
      const int j1 = j0 + half;
      const float2 w = __ldg(tw + pos * step);
      const float2 a = c[j0];
      const float2 b = c[j1];
      c[j0] = make_float2(a.x + b.x, a.y + b.y);
      c[j1] = cmul(make_float2(a.x - b.x, a.y - b.y), w);
    }
    __syncthreads();
  }
}

// Inverse DIT: bit-reversed input -> natural-order output (conjugate twiddles, no 1/n).
NMG_D void fft_dit_inverse(float2* c, int n, const float2* __restrict__ tw, int tw_n, int tid, int nthr) {
  for (int len = 2; len <= n; len <<= 1) {
    const int half = len >> 1;
    const int step = tw_n / len;
    for (int i = tid; i < (n >> 1); i += nthr) {
      const int pos = i & (half - 1);
      const int j0 = ((i - pos) << 1) + pos;
      const int j1 = j0 + half;
      const float2 w = __ldg(tw + pos * step);
      const float2 a = c[j0];
      const float2 b = cmulc(c[j1], w);
      c[j0] = make_float2(a.x + b.x, a.y + b.y);
      c[j1] = make_float2(a.x - b.x, a.y - b.y);
    }
    __syncthreads();
  }
}

// Radix-2 stages fused R at a time in registers (R = 3, then 2 / 1 for the remainder): the
// same butterflies with the same twiddles in the same order as fft_dif_forward /
// fft_dit_inverse (bit-identical results), but one shared-memory pass and one barrier per R
// stages.  All lengths are powers of two and passed as log2 (llen = log2 len, ltw = log2 tw_n),
// so the index arithmetic is shifts and masks (no integer division).  Block-cooperative; each
// batch / fused driver ends with __syncthreads().
template <int R>
NMG_D void dif_group(float2* c, int llen, int g, const float2* __restrict__ tw, int ltw, int stride = 1) {
  constexpr int E = 1 << R;
  const int lq = llen - R;                      // element spacing q = len >> R in the group
  const int blk = g >> lq, pos = g & ((1 << lq) - 1);
  float2* base = c + ((blk << llen) + pos) * stride;
  const int qs = stride << lq;
  float2 e[E];
#pragma unroll
  for (int i = 0; i < E; ++i) e[i] = base[i * qs];
#pragma unroll
  for (int st = 0; st < R; ++st) {             // stage length len >> st, half = E >> (st + 1) elements
    const int hs = E >> (st + 1);
    const int lstep = ltw - (llen - st);        // twiddle stride tw_n / (len >> st)
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (i & hs) continue;                     // i is the upper element of its pair
      const int posi = pos + ((i & (hs - 1)) << lq);   // position within the current sub-block
      const float2 w = __ldg(tw + (posi << lstep));
      const float2 a = e[i], b = e[i + hs];
      e[i] = make_float2(a.x + b.x, a.y + b.y);
      e[i + hs] = cmul(make_float2(a.x - b.x, a.y - b.y), w);
    }
  }
#pragma unroll
  for (int i = 0; i < E; ++i) base[i * qs] = e[i];
}
template <int R>
NMG_D void dit_group(float2* c, int llen, int g, const float2* __restrict__ tw, int ltw, int stride = 1) {
  // stages len, 2 len, ..., 2^(R-1) len; group = 2^R elements spaced len/2 apart in a block of
  // 2^(R-1) len
  constexpr int E = 1 << R;
  const int lhq = llen - 1;
  const int blk = g >> lhq, pos = g & ((1 << lhq) - 1);
  float2* base = c + ((blk << (lhq + R)) + pos) * stride;
  const int qs = stride << lhq;
  float2 e[E];
#pragma unroll
  for (int i = 0; i < E; ++i) e[i] = base[i * qs];
#pragma unroll
  for (int st = 0; st < R; ++st) {             // stage length len << st, pair distance 2^st elements
    const int hs = 1 << st;
    const int lstep = ltw - (llen + st);        // twiddle stride tw_n / (len << st)
#pragma unroll
    for (int i = 0; i < E; ++i) {
      if (i & hs) continue;
      const int posi = pos + ((i & (hs - 1)) << lhq);
      const float2 w = __ldg(tw + (posi << lstep));
      const float2 a = e[i], b = cmulc(e[i + hs], w);
      e[i] = make_float2(a.x + b.x, a.y + b.y);
      e[i + hs] = make_float2(a.x - b.x, a.y - b.y);
    }
  }
#pragma unroll
  for (int i = 0; i < E; ++i) base[i * qs] = e[i];
}
NMG_D int ilog2(int v) { return 31 - __clz(v); }
// Batched fused passes over `cnt` independent length-n transforms: transform k starts at
// c + k * kstride and its elements are `stride` apart (rows: kstride = n, stride = 1;
// columns of an [n][G] tile: kstride = 1, stride = G).  Same arithmetic as the radix-2 loops.
// Strided (column) transforms put neighbouring transforms on neighbouring threads, so the
// shared-memory accesses stay consecutive; rows put neighbouring groups of one transform there.
template <bool DIT>
NMG_D void fft_batch_pass(float2* c, int ln, int cnt, int kstride, int stride, int llen, int R,
                          const float2* __restrict__ tw, int ltw, int tid, int nthr) {
  const int lper = ln - R;
  const int tot = cnt << lper;
  const bool pow2 = (cnt & (cnt - 1)) == 0;
  const int lcnt = ilog2(max(cnt, 1));
  for (int gg = tid; gg < tot; gg += nthr) {
    int k, g;
    if (stride == 1) { k = gg >> lper; g = gg & ((1 << lper) - 1); }
    else if (pow2) { k = gg & (cnt - 1); g = gg >> lcnt; }
    else { k = gg % cnt; g = gg / cnt; }
    float2* ck = c + k * kstride;
    if (DIT) {
      if (R == 3) dit_group<3>(ck, llen, g, tw, ltw, stride);
      else if (R == 2) dit_group<2>(ck, llen, g, tw, ltw, stride);
      else dit_group<1>(ck, llen, g, tw, ltw, stride);
    } else {
      if (R == 3) dif_group<3>(ck, llen, g, tw, ltw, stride);
      else if (R == 2) dif_group<2>(ck, llen, g, tw, ltw, stride);
      else dif_group<1>(ck, llen, g, tw, ltw, stride);
    }
  }
}
NMG_D void fft_dif_forward_batch(float2* c, int n, int cnt, int kstride, int stride, const float2* __restrict__ tw,
                                 int tw_n, int tid, int nthr) {
  const int ln = ilog2(n), ltw = ilog2(tw_n);
  for (int llen = ln; llen >= 1;) {
    const int R = llen >= 3 ? 3 : llen;
    fft_batch_pass<false>(c, ln, cnt, kstride, stride, llen, R, tw, ltw, tid, nthr);
    llen -= R;
    __syncthreads();
  }
}
NMG_D void fft_dit_inverse_batch(float2* c, int n, int cnt, int kstride, int stride, const float2* __restrict__ tw,
                                 int tw_n, int tid, int nthr) {
  const int ln = ilog2(n), ltw = ilog2(tw_n);
  for (int llen = 1; llen <= ln;) {
    const int left = ln - llen + 1;             // stages remaining (len .. n)
    const int R = left >= 3 ? 3 : left;
    fft_batch_pass<true>(c, ln, cnt, kstride, stride, llen, R, tw, ltw, tid, nthr);
    llen += R;
    __syncthreads();
  }
}
NMG_D void fft_dif_forward_fused(float2* c, int n, const float2* __restrict__ tw, int tw_n, int tid, int nthr) {
  fft_dif_forward_batch(c, n, 1, n, 1, tw, tw_n, tid, nthr);
}
NMG_D void fft_dit_inverse_fused(float2* c, int n, const float2* __restrict__ tw, int tw_n, int tid, int nthr) {
  fft_dit_inverse_batch(c, n, 1, n, 1, tw, tw_n, tid, nthr);
}

// Level mask m'_l in natural DFT order (reading R5): sqrt(2 min(k, n-k) / n).
NMG_D float level_mask_1d(int k, int n) {
  const int m = min(k, n - k);
  return sqrtf((float)(2 * m) / (float)n);
}

// In-place level filter F'(h) = Re(IDFT_n(m' (.) DFT_n(h))) of a REAL row h[0..n) held in
// shared memory, via one n/2-point complex FFT of z[k] = h[2k] + i h[2k+1] (the standard
// real-input packing), the mask applied on the unpacked half spectrum, and one n/2-point
// inverse FFT.  The row is processed alone (no pairing with other right-hand sides).
// Block-cooperative; starts and ends with __syncthreads().
NMG_D void real_level_filter(float* hbuf, int n, const float2* __restrict__ tw, int tw_n, int tid, int nthr) {
  float2* z = reinterpret_cast<float2*>(hbuf);
  const int m = n >> 1;
  __syncthreads();
  if (m >= 2) fft_dif_forward_fused(z, m, tw, tw_n, tid, nthr);   // Z in bit-reversed order
  const int lm = (m >= 2) ? 31 - __clz(m) : 0;
  const int wstep = tw_n / n;                                     // W_n^k = tw[k * wstep]
  const float invn = 1.0f / (float)n;                             // power of two: x invn == x / n
  // pair (k, m - k): unpack H, apply the mask, repack for the inverse
  for (int k = tid; k <= (m >> 1); k += nthr) {
    const int kk = (m - k) & (m - 1);                             // m - k (mod m)
    const int pk = lm ? bitrev(k, lm) : 0, pkk = lm ? bitrev(kk, lm) : 0;
    const float2 Zk = z[pk], Zc = z[pkk];
    const float mk = sqrtf((float)(2 * k) * invn);                // mu[k],   k <= m
    const float mc = sqrtf((float)(2 * (m - k)) * invn);          // mu[m-k]
    const float sp = 0.5f * (mk + mc), sm = 0.5f * (mk - mc);
    // k side: E = (Zk + conj Zc)/2, O = -i (Zk - conj Zc)/2
    float2 E = make_float2(0.5f * (Zk.x + Zc.x), 0.5f * (Zk.y - Zc.y));
    float2 O = make_float2(0.5f * (Zk.y + Zc.y), -0.5f * (Zk.x - Zc.x));
    float2 W = __ldg(tw + k * wstep);                              // e^{-2 pi i k / n}
    float2 WO = cmul(W, O);
    float2 Eg = make_float2(sp * E.x + sm * WO.x, sp * E.y + sm * WO.y);
    float2 WcE = cmulc(E, W);                                      // W^{-k} E
    float2 Og = make_float2(sm * WcE.x + sp * O.x, sm * WcE.y + sp * O.y);
    const float2 Zk2 = make_float2(Eg.x - Og.y, Eg.y + Og.x);      // Eg + i Og
    if (kk != k) {
      // m - k side (same formulas with k -> m - k, mu swapped)
      float2 E2 = make_float2(0.5f * (Zc.x + Zk.x), 0.5f * (Zc.y - Zk.y));
      float2 O2 = make_float2(0.5f * (Zc.y + Zk.y), -0.5f * (Zc.x - Zk.x));
      float2 W2 = __ldg(tw + kk * wstep);
      float2 WO2 = cmul(W2, O2);
      float2 Eg2 = make_float2(sp * E2.x - sm * WO2.x, sp * E2.y - sm * WO2.y);
      float2 WcE2 = cmulc(E2, W2);
      float2 Og2 = make_float2(-sm * WcE2.x + sp * O2.x, -sm * WcE2.y + sp * O2.y);
      z[pkk] = make_float2(Eg2.x - Og2.y, Eg2.y + Og2.x);
    }
    z[pk] = Zk2;
  }
  __syncthreads();
  if (m >= 2) fft_dit_inverse_fused(z, m, tw, tw_n, tid, nthr);  // natural order, unnormalised
}

}  // namespace nmg
