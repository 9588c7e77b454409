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

// Level mask m'_l in natural DFT order (reading R5): sqrt(2 min(k, n-k) / n).
NMG_D float level_mask_1d(int k, int n) {
  const int m = min(k, n - k);
  return sqrtf((float)(2 * m) / (float)n);
}

}  // namespace nmg
