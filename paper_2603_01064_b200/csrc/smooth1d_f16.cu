// Fused 1D neural smoothing step with the 16 -> 16 layer on tcgen05 (FP16x3), one CTA per
// right-hand side (Alg 3; CNN per reading R7; F' per P:305, R5):
//   s = ||b||_2 (fp64)  ->  u = b / s  ->  a1 = ReLU(w0 * u + b0)            (FFMA, producer)
//   a2 = ReLU(w1 * a1 + b1)                                                  (tcgen05, 128-point tiles)
//   h  = s (b2 + w2 * a2)                                                    (FFMA, epilogue)
//   x  = x* + F'(h)                                                          (shared-memory FFT)
//
// Layer 2 puts the positions on the MMA M axis (128 per tile), the output channels on N and
// (tap, input channel) on K.  a1 lives in shared memory in the canonical no-swizzle K-major
// layout [2 chunks][136 rows][8 x f16] (16-byte rows, 8-row core matrices contiguous), so
// tap t is a +16 t byte shift of the A descriptor start: no im2col buffer.  FP16x3 with
// power-of-two scales (see conv_strip.cu): per tap one N = 32 MMA multiplies the hi part of
// a1 by the stacked [W_hi; W_lo] weights and one N = 16 MMA multiplies the lo part by W_hi
// (D[:, 0:16] = Ah Wh + Al Wh, D[:, 16:32] = Ah Wl; the epilogue adds the halves).  Each MMA
// streams its 128 x 16 A tile from shared memory, which makes shared-memory bandwidth the
// tile pipeline's limit: two A reads per tap, not three.
// The CNN weights travel by value in the kernel arguments, so every FFMA of layers 1 and 3
// takes its weight as a constant-bank (uniform-register) operand: no weight registers, no
// shared-memory loads.
// Layer 3 (16 -> 1, k = 5) is split per tap in the epilogue: q_t(p) = sum_c w2[c][t] a2[c](p),
// written to a 512-position ring, and h(p) = b2 + sum_t q_t(p + t - 2) is assembled after the
// next barrier (positions outside [0, n) read zeros) -- no layer-2 halo is recomputed.
//
// Warps: 0-3 epilogue (TMEM lanes = positions), 4-7 layer-1 producer, 8 MMA issuer (the whole
// warp converged, one elected lane issuing, so the stage arithmetic stays in uniform
// registers); the norm, filter and update phases use all 288 threads.  Three CTAs per SM
// overlap the serial phases of one right-hand side with the tile pipelines of the others.
// The level filter is a swizzled Stockham FFT (level_filter_row).  The CNN output row h is written
// into the input-row buffer behind the layer-1 producer and moved into the freed a1 stages for
// the filter (no separate h row: 50 KB per CTA at n = 4096, four CTAs per SM).
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdio>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace nmg {
namespace {

constexpr int C = 16, KS = 5;
constexpr int NT = 288;
constexpr int TP = 128;                 // positions per tile (MMA M)
constexpr int AR = 136;                 // rows of the a1 buffer (132 used: TP + 4 halo)
constexpr int ALBO = AR * 16;           // K-chunk stride of the a1 buffer (bytes)
constexpr int ABYTES = 2 * ALBO;        // one a1 tile, hi or lo (2 chunks)
constexpr int BLBO = 32 * 16;           // K-chunk stride of a stacked weight tap [2][32][8]
constexpr int BTAP = 2 * BLBO;          // bytes per tap
constexpr int QR = 512;                 // q ring (positions)
constexpr int UPAD = 4;
constexpr int NSD = 4;                  // accumulator stages (TMEM, 32 columns each)
constexpr uint32_t IDESC32 = (1u << 4) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(TP >> 4) << 24);
constexpr uint32_t IDESC16 = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(TP >> 4) << 24);

NMG_D bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n.reg .b32 %%rx;\n.reg .pred %%px;\n"
      "elect.sync %%rx|%%px, %1;\n"
      "@%%px mov.s32 %0, 1;\n}\n"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}
NMG_D void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 hv = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
    const float2 hf = __half22float2(hv);   // v - hi per channel pair in one FADD2 (same bits)
    const float2 r = __fadd2_rn(make_float2(v[2 * j], v[2 * j + 1]), make_float2(-hf.x, -hf.y));
    const __half2 lv = __floats2half2_rn(r.x, r.y);
    h[j] = *reinterpret_cast<const uint32_t*>(&hv);
    l[j] = *reinterpret_cast<const uint32_t*>(&lv);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}
NMG_D void tf32_store(float xv, float* xh, float* xl, int64_t at) {
  uint32_t hh, ll;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(hh) : "f"(xv));
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(ll) : "f"(xv - __uint_as_float(hh)));
  xh[at] = __uint_as_float(hh);
  xl[at] = __uint_as_float(ll);
}

// ---- level filter F'_l (reading R5) on the row held in shared memory -----------
// Same mathematics as fft.cuh's real_level_filter (one n/2-point complex FFT of the packed
// row z[k] = h[2k] + i h[2k+1], the mask on the unpacked half spectrum, one inverse), but
// as Stockham autosort passes (natural order in and out, ping-pong between the row buffer
// and a scratch buffer) on a swizzled layout: complex element i lives at sw(i) =
// i ^ ((i >> 3) & 15), a permutation inside aligned 128-element blocks that makes every
// pass's loads and stores, the unpack's (k, m - k) pairs and the row-order accesses of the
// epilogue and update free of shared-memory bank conflicts.
// a1 stages, reused after the tile loop as the FFT scratch (n/2 complex)
NMG_HD int abuf_bytes(int nsa, int n) { return max(2 * nsa * ABYTES, 4 * n); }
NMG_D int sw(int i) { return i ^ ((i >> 3) & 15); }
NMG_D int hsw(int p) { return 2 * sw(p >> 1) + (p & 1); }   // real position p of the row

NMG_D float2 twid(const float2* __restrict__ tw, int tw_n, int k) {   // exp(-2 pi i k / tw_n), k < tw_n
  const int h = tw_n >> 1;
  const float2 w = __ldg(tw + (k & (h - 1)));   // branch-free, so all loads of a pass issue together
  const float sg = k < h ? 1.f : -1.f;
  return make_float2(sg * w.x, sg * w.y);
}
template <bool INV>
NMG_D float2 rot_mi(float2 a) { return INV ? make_float2(-a.y, a.x) : make_float2(a.y, -a.x); }   // a * (-/+ i)
// R-point DFT in registers, natural order in and out (radix-2 DIF, outputs unscrambled)
template <int R, bool INV>
NMG_D void dft_r(float2 (&v)[R]) {
  if constexpr (R == 2) {
    const float2 a = v[0], b = v[1];
    v[0] = make_float2(a.x + b.x, a.y + b.y);
    v[1] = make_float2(a.x - b.x, a.y - b.y);
  } else if constexpr (R == 4) {
    float2 t[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float2 a = v[i], b = v[i + 2];
      t[i] = make_float2(a.x + b.x, a.y + b.y);
      t[i + 2] = make_float2(a.x - b.x, a.y - b.y);
    }
    t[3] = rot_mi<INV>(t[3]);
    v[0] = make_float2(t[0].x + t[1].x, t[0].y + t[1].y);
    v[2] = make_float2(t[0].x - t[1].x, t[0].y - t[1].y);
    v[1] = make_float2(t[2].x + t[3].x, t[2].y + t[3].y);
    v[3] = make_float2(t[2].x - t[3].x, t[2].y - t[3].y);
  } else {
    constexpr float h = 0.70710678118654752440f;
    float2 t[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 a = v[i], b = v[i + 4];
      t[i] = make_float2(a.x + b.x, a.y + b.y);
      t[i + 4] = make_float2(a.x - b.x, a.y - b.y);
    }
    // t[4 + i] *= W8^i
    t[5] = INV ? make_float2(h * (t[5].x - t[5].y), h * (t[5].x + t[5].y))
               : make_float2(h * (t[5].x + t[5].y), h * (t[5].y - t[5].x));
    t[6] = rot_mi<INV>(t[6]);
    t[7] = INV ? make_float2(-h * (t[7].x + t[7].y), h * (t[7].x - t[7].y))
               : make_float2(h * (t[7].y - t[7].x), -h * (t[7].x + t[7].y));
    float2 u[8];
#pragma unroll
    for (int g = 0; g < 8; g += 4) {
      const float2 a0 = t[g], a1 = t[g + 1], b0 = t[g + 2], b1 = t[g + 3];
      u[g] = make_float2(a0.x + b0.x, a0.y + b0.y);
      u[g + 1] = make_float2(a1.x + b1.x, a1.y + b1.y);
      u[g + 2] = make_float2(a0.x - b0.x, a0.y - b0.y);
      u[g + 3] = rot_mi<INV>(make_float2(a1.x - b1.x, a1.y - b1.y));
    }
    // last stage; DIF output index bitrev3: V[0]=u0+u1, V[4]=u0-u1, V[2]=u2+u3, V[6]=u2-u3, ...
    v[0] = make_float2(u[0].x + u[1].x, u[0].y + u[1].y);
    v[4] = make_float2(u[0].x - u[1].x, u[0].y - u[1].y);
    v[2] = make_float2(u[2].x + u[3].x, u[2].y + u[3].y);
    v[6] = make_float2(u[2].x - u[3].x, u[2].y - u[3].y);
    v[1] = make_float2(u[4].x + u[5].x, u[4].y + u[5].y);
    v[5] = make_float2(u[4].x - u[5].x, u[4].y - u[5].y);
    v[3] = make_float2(u[6].x + u[7].x, u[6].y + u[7].y);
    v[7] = make_float2(u[6].x - u[7].x, u[6].y - u[7].y);
  }
}
// one Stockham radix-R pass: sub-transforms of length NS -> NS R (ends with __syncthreads).
// The transform length M and the pass (NS) are compile-time (one instantiation per level
// size), so the group, twiddle and swizzle index arithmetic folds to shifts and masks.
template <int R, int NS, int M, bool INV>
NMG_D void stockham_pass(const float2* src, float2* dst, const float2* __restrict__ tw, int tw_n, int tid) {
  constexpr int q = M / R;
  constexpr float inv = 1.0f / (float)(NS * R);   // a power of two: x inv is bitwise x / (NS R)
  for (int j = tid; j < q; j += NT) {
    const int jm = j & (NS - 1);
    float2 w[R], v[R];
    if constexpr (NS > 1) {   // twiddles first: independent of the data, their latency overlaps the loads
#ifndef NMG_S1D_TWTABLE
      // computed twiddles (no dependent table loads; accurate sincospif, exact arguments):
      // w1 = exp(-2 pi i jm / (NS R)), powers by products
      float sn, cs;
      sincospif(-2.0f * (float)jm * inv, &sn, &cs);
      w[1] = make_float2(cs, sn);
#pragma unroll
      for (int r = 2; r < R; ++r) w[r] = cmul(w[r - 1], w[1]);
#else
      const int tstep = tw_n / (NS * R);
#pragma unroll
      for (int r = 1; r < R; ++r) w[r] = twid(tw, tw_n, jm * r * tstep);
#endif
    }
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = src[sw(j + r * q)];
    if constexpr (NS > 1) {
#pragma unroll
      for (int r = 1; r < R; ++r) v[r] = INV ? cmulc(v[r], w[r]) : cmul(v[r], w[r]);
    }
    dft_r<R, INV>(v);
    const int d = (j - jm) * R + jm;
#pragma unroll
    for (int r = 0; r < R; ++r) dst[sw(d + r * NS)] = v[r];
  }
  __syncthreads();
}
// M-point FFT (M a power of two >= 2) from pass NS on, natural order; returns the buffer
// holding the result (a and b alternate per pass)
template <int M, int NS, bool INV>
NMG_D float2* stockham_fft(float2* a, float2* b, const float2* __restrict__ tw, int tw_n, int tid) {
  if constexpr (NS >= M) {
    return a;
  } else {
    constexpr int REM = M / NS;
    constexpr int R = REM >= 8 ? 8 : (REM == 4 ? 4 : 2);
    stockham_pass<R, NS, M, INV>(a, b, tw, tw_n, tid);
    return stockham_fft<M, NS * R, INV>(b, a, tw, tw_n, tid);
  }
}
// F'(h) of the real row in z (swizzled, n reals = n/2 complex); scratch t of n/2 complex.
// Result (times n/2, unnormalised) back in z.  Starts and ends with __syncthreads().
template <int N>
NMG_D void level_filter_row(float2* z, float2* t, const float2* __restrict__ tw, int tw_n, int tid) {
  constexpr int n = N, m = N >> 1, nthr = NT;
  __syncthreads();
  float2* Z = stockham_fft<m, 1, false>(z, t, tw, tw_n, tid);
  const int wstep = tw_n / n;   // W_n^k = tw[k * wstep]
  constexpr float invn = 1.0f / (float)n;   // n a power of two: x invn is bitwise x / n
  // pair (k, m - k): unpack H, apply the mask, repack for the inverse (as real_level_filter)
  constexpr int UNP = 4;
  for (int k0 = tid; k0 <= (m >> 1); k0 += UNP * nthr) {
    float2 Wv[UNP], W2v[UNP];
#pragma unroll
    for (int u = 0; u < UNP; ++u) {   // twiddle loads of all iterations first
      const int k = min(k0 + u * nthr, m >> 1);
#ifndef NMG_S1D_TWTABLE
      {
        float sn, cs;
        sincospif(-2.0f * (float)k * invn, &sn, &cs);
        Wv[u] = make_float2(cs, sn);
        sincospif(-2.0f * (float)((m - k) & (m - 1)) * invn, &sn, &cs);
        W2v[u] = make_float2(cs, sn);
      }
#else
      Wv[u] = __ldg(tw + k * wstep);
      W2v[u] = __ldg(tw + ((m - k) & (m - 1)) * wstep);
#endif
    }
#pragma unroll
    for (int u = 0; u < UNP; ++u) {
    const int k = k0 + u * nthr;
    if (k > (m >> 1)) break;
    const int kk = (m - k) & (m - 1);
    const float2 Zk = Z[sw(k)], Zc = Z[sw(kk)];
    const float mk = sqrtf((float)(2 * k) * invn);
    const float mc = sqrtf((float)(2 * (m - k)) * invn);
    const float sp = 0.5f * (mk + mc), sm = 0.5f * (mk - mc);
    float2 E = make_float2(0.5f * (Zk.x + Zc.x), 0.5f * (Zk.y - Zc.y));
    float2 O = make_float2(0.5f * (Zk.y + Zc.y), -0.5f * (Zk.x - Zc.x));
    float2 W = Wv[u];
    float2 WO = cmul(W, O);
    float2 Eg = make_float2(sp * E.x + sm * WO.x, sp * E.y + sm * WO.y);
    float2 WcE = cmulc(E, W);
    float2 Og = make_float2(sm * WcE.x + sp * O.x, sm * WcE.y + sp * O.y);
    const float2 Zk2 = make_float2(Eg.x - Og.y, Eg.y + Og.x);
    if (kk != k) {
      float2 E2 = make_float2(0.5f * (Zc.x + Zk.x), 0.5f * (Zc.y - Zk.y));
      float2 O2 = make_float2(0.5f * (Zc.y + Zk.y), -0.5f * (Zc.x - Zk.x));
      float2 W2 = W2v[u];
      float2 WO2 = cmul(W2, O2);
      float2 Eg2 = make_float2(sp * E2.x - sm * WO2.x, sp * E2.y - sm * WO2.y);
      float2 WcE2 = cmulc(E2, W2);
      float2 Og2 = make_float2(-sm * WcE2.x + sp * O2.x, -sm * WcE2.y + sp * O2.y);
      Z[sw(kk)] = make_float2(Eg2.x - Og2.y, Eg2.y + Og2.x);
    }
    Z[sw(k)] = Zk2;
    }
  }
  __syncthreads();
  float2* other = Z == z ? t : z;
  stockham_fft<m, 1, true>(Z, other, tw, tw_n, tid);   // equal pass counts: ends in z
}
// the level sizes the kernel supports (n % 128 == 0, n <= 8192)
NMG_D void level_filter_row(float2* z, float2* t, int n, const float2* __restrict__ tw, int tw_n, int tid) {
  switch (n) {
    case 128: level_filter_row<128>(z, t, tw, tw_n, tid); break;
    case 256: level_filter_row<256>(z, t, tw, tw_n, tid); break;
    case 512: level_filter_row<512>(z, t, tw, tw_n, tid); break;
    case 1024: level_filter_row<1024>(z, t, tw, tw_n, tid); break;
    case 2048: level_filter_row<2048>(z, t, tw, tw_n, tid); break;
    case 4096: level_filter_row<4096>(z, t, tw, tw_n, tid); break;
    default: level_filter_row<8192>(z, t, tw, tw_n, tid); break;
  }
}

// layer-1 producer for channels 8 H .. 8 H + 7 (H compile-time, so the weights are
// constant-bank operands): rows r0, r0 + 64, r0 + 128 of each a1 tile
template <int H>
NMG_D void a1_row(const Smooth1dArgs& a, const float* u, int p, int n, uint4& hi, uint4& lo) {
  float v[8];
  if (p >= 0 && p < n) {
    const float* up = u + p - 2;   // u = b S1 / ||b|| with zero padding
    const float x0 = up[0], x1 = up[1], x2 = up[2], x3 = up[3], x4 = up[4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float* w = a.w.w0 + (8 * H + j) * KS;
      float acc = a.w.b0[8 * H + j];
      acc = fmaf(w[0], x0, acc);
      acc = fmaf(w[1], x1, acc);
      acc = fmaf(w[2], x2, acc);
      acc = fmaf(w[3], x3, acc);
      acc = fmaf(w[4], x4, acc);
      v[j] = fmaxf(acc, 0.f);
    }
  } else {
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = 0.f;
  }
  split8(v, hi, lo);
}

// the same for two positions p0, p1 at once: packed fp32 pairs (FFMA2 with the weight as a
// broadcast operand -- half the FMA issue slots; each lane rounds exactly as the scalar fmaf,
// same order, so the result is bitwise a1_row's)
template <int H>
NMG_D void a1_row2(const Smooth1dArgs& a, const float* u, int p0, int p1, int n, uint4& hi0, uint4& lo0, uint4& hi1,
                   uint4& lo1) {
  const bool ok0 = p0 >= 0 && p0 < n, ok1 = p1 >= 0 && p1 < n;
  const float* u0 = u + (ok0 ? p0 : 2) - 2;   // any in-range window when the position is padding
  const float* u1 = u + (ok1 ? p1 : 2) - 2;
  float2 x[KS];
#pragma unroll
  for (int t = 0; t < KS; ++t) x[t] = make_float2(u0[t], u1[t]);
  float v0[8], v1[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const float* w = a.w.w0 + (8 * H + j) * KS;
    const float b = a.w.b0[8 * H + j];
    float2 acc = make_float2(b, b);
#pragma unroll
    for (int t = 0; t < KS; ++t) acc = __ffma2_rn(x[t], make_float2(w[t], w[t]), acc);
    v0[j] = fmaxf(acc.x, 0.f);
    v1[j] = fmaxf(acc.y, 0.f);
  }
  split8(v0, hi0, lo0);
  split8(v1, hi1, lo1);
  // positions outside [0, n) are zeros of layer 2's input: the caller stores zero words there
}

// Layer-1 producer for channels 8 H .. 8 H + 7 (H compile-time, so the weights are
// constant-bank operands).  Buffer row r of tile k holds position k TP - 2 + r; rows 0..131
// are read by the five tap-shifted MMAs.  Each thread computes rows 4 + r0 and 68 + r0
// (two rows, r0 < 64); rows 0..3 of tile k are rows 128..131 of tile k - 1, which the
// threads r0 = 60..63 carry over in registers (tile 0 computes them).
template <int H, int NSA>
NMG_D void produce_a1(const Smooth1dArgs& a, uint8_t* Abuf, uint64_t* aempty, uint64_t* afull, const float* u,
                      int r0, int ntile, int n, int lane) {
  const bool carry = r0 >= 60;
  uint4 ch, cl;
  if (carry) a1_row<H>(a, u, r0 - 60 - 2, n, ch, cl);   // tile 0 rows 0..3
  for (int k = 0; k < ntile; ++k) {
    const int st = k % NSA;
    const int Q0 = k * TP;
    uint4 h0, l0, h1, l1;
    a1_row2<H>(a, u, Q0 + 2 + r0, Q0 + 66 + r0, n, h0, l0, h1, l1);
    mb_wait(&aempty[st], ((uint32_t)(k / NSA) & 1u) ^ 1u);
    uint4* ah = reinterpret_cast<uint4*>(Abuf + (2 * st) * ABYTES) + H * AR;
    uint4* al = reinterpret_cast<uint4*>(Abuf + (2 * st + 1) * ABYTES) + H * AR;
    // position Q0 + 2 + r0 is always inside the row; Q0 + 66 + r0 passes its end only in the last
    // tile (predicated zero stores instead of selects)
    ah[4 + r0] = h0; al[4 + r0] = l0;
    if (Q0 + 66 + r0 < n) {
      ah[68 + r0] = h1; al[68 + r0] = l1;
    } else {
      ah[68 + r0] = make_uint4(0u, 0u, 0u, 0u); al[68 + r0] = make_uint4(0u, 0u, 0u, 0u);
    }
    if (carry) {
      ah[r0 - 60] = ch; al[r0 - 60] = cl;
      ch = h1; cl = l1;
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) mb_arrive(&afull[st]);
  }
}

#ifdef NMG_S1D_PHASES
#define S1D_TS(i) do { if (threadIdx.x == 0 && blockIdx.x == 0) ts[i] = clock64(); } while (0)
#else
#define S1D_TS(i) do { } while (0)
#endif

template <int NSA>
#ifndef NMG_S1D_MINB
#define NMG_S1D_MINB 4
#endif
__global__ void __launch_bounds__(NT, NMG_S1D_MINB) smooth1d_f16_kernel(const __grid_constant__ Smooth1dArgs a) {
#ifdef NMG_S1D_PHASES
  long long ts[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
  S1D_TS(0);
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u);
  const int n = a.n, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rhs = blockIdx.x;
  uint8_t* Abuf = sm;                                          // [2 stages][hi | lo] ABYTES each
  uint8_t* Bw = Abuf + abuf_bytes(NSA, n);                     // [5 taps][2][32][8] f16
  float* qs = reinterpret_cast<float*>(Bw + KS * BTAP);        // [5][QR]
  // the input row u (b / s) and, in place behind the producer, the CNN output h (plain order):
  // the epilogue of tile k writes h at positions <= k TP + 125, the producer reads u only from
  // the tile it is filling (>= k TP - 2), and tile k + 1 starts at k TP + 126
  float* u = qs + KS * QR;                                     // n + 2 UPAD
  float* hb = reinterpret_cast<float*>(Abuf);                  // filter row (swizzled), after the tiles
  uint64_t* bars = reinterpret_cast<uint64_t*>(u + n + 2 * UPAD);        // afull[2] aempty[2] dfull[2] dempty[2]
  uint64_t* afull = bars;
  uint64_t* aempty = afull + NSA;
  uint64_t* dfull = aempty + NSA;
  uint64_t* dempty = dfull + NSD;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(dempty + NSD);
  __shared__ double red[32];

  // ---------------------------------------------------------------- setup (all threads)
  {
    const uint4* g = reinterpret_cast<const uint4*>(a.wb);
    uint4* d = reinterpret_cast<uint4*>(Bw);
    for (int i = tid; i < KS * BTAP / 16; i += NT) d[i] = __ldg(g + i);
  }
  if (tid == 0) {
    for (int s = 0; s < NSA; ++s) { mb_init(&afull[s], 4); mb_init(&aempty[s], 1); }
    for (int s = 0; s < NSD; ++s) { mb_init(&dfull[s], 1); mb_init(&dempty[s], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)), "r"(32 * NSD));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  const float* brow = a.b + (int64_t)rhs * a.ldb;
  if (tid < UPAD) { u[tid] = 0.f; u[UPAD + n + tid] = 0.f; }
  double ss = 0.0;
  for (int j = tid; j < n; j += NT) {
    const float v = brow[j];
    u[UPAD + j] = v;
    ss += (double)v * (double)v;
  }
  double s = 1.0;
  if (a.normalize) s = sqrt(block_sum_f64(ss, red));   // block-wide, ends with all threads holding s
  if (s != 0.0) {
    // u = b / s with the f16 scale S1 folded in (ReLU(S z) = S ReLU(z), S > 0)
    const float isc = (float)(1.0 / s) * a.in_scale;
    __syncthreads();
    for (int j = tid; j < n; j += NT) u[UPAD + j] *= isc;
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  float* xrow = a.x + (int64_t)rhs * a.ldx;

  if (s == 0.0) {   // ||b|| = 0 => h = 0 (reading R10)
    for (int j = tid; j < n; j += NT) {
      const float xv = a.accumulate ? xrow[j] : 0.f;
      xrow[j] = xv;
      if (a.xh) tf32_store(xv, a.xh, a.xl, (int64_t)rhs * a.ldx + j);
    }
  } else {
    const float sf = (float)s;
    const int ntile = n / TP;
    S1D_TS(1);
    if (warp >= 4 && warp < 8) {
      // ---------------------------------------------------------- layer-1 producer
      const int pt = tid - 128;                 // 0..127
      const int r0 = pt & 63;                   // rows 4 + r0 and 68 + r0 (see produce_a1)
      // u holds b / s times the f16 scale S1 (ReLU(S z) = S ReLU(z), S > 0); b0 arrives
      // pre-multiplied by S1
      if (pt < 64) produce_a1<0, NSA>(a, Abuf, aempty, afull, u + UPAD, r0, ntile, n, lane);
      else produce_a1<1, NSA>(a, Abuf, aempty, afull, u + UPAD, r0, ntile, n, lane);
    } else if (warp == 8) {
      // ---------------------------------------------------------- MMA issuer
      // The whole warp runs the loop converged (waits, stage arithmetic and descriptors stay
      // warp-uniform, so they live in uniform registers); one elected lane issues.
      const uint32_t ab = su32(Abuf), bb = su32(Bw);
      const uint64_t db0 = desc_ns(bb, BLBO), da0 = desc_ns(ab, ALBO);
      for (int k = 0; k < ntile; ++k) {
        const int st = k % NSA, sd = k % NSD;
        mb_wait(&afull[st], (uint32_t)(k / NSA) & 1u);
        mb_wait(&dempty[sd], ((uint32_t)(k / NSD) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        if (elect_one()) {
          const uint32_t d = tmem + (uint32_t)(sd * 32);
          // descriptor start addresses are in 16-byte units: + 1 per tap row shift
          const uint64_t dah = da0 + (uint64_t)((2 * st) * ABYTES >> 4), dal = dah + (ABYTES >> 4);
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const uint64_t db = db0 + (uint64_t)(t * BTAP >> 4);
            mma_f16(d, dah + t, db, IDESC32, t > 0 ? 1u : 0u);
            mma_f16(d, dal + t, db, IDESC16, 1u);
          }
          mma_commit(&aempty[st]);
          mma_commit(&dfull[sd]);
        }
        __syncwarp();
      }
    } else if (warp < 4) {
      // ---------------------------------------------------------- epilogue: layer 3 per tap
      const int m = tid;                        // TMEM lane = position within the tile
      const float b2v = a.w.b2;
      if (m < 2) {
#pragma unroll
        for (int t = 0; t < KS; ++t) qs[t * QR + ((QR - 2 + m) & (QR - 1))] = 0.f;   // positions -2, -1
      }
      auto emit = [&](int p, float hv) {
        if (a.filter) {
          u[UPAD + p] = hv;
        } else {
          const float xv = a.accumulate ? xrow[p] + hv : hv;
          xrow[p] = xv;
          if (a.xh) tf32_store(xv, a.xh, a.xl, (int64_t)rhs * a.ldx + p);
        }
      };
      auto assemble = [&](int p) {
        float acc = b2v;
#pragma unroll
        for (int t = 0; t < KS; ++t) acc += qs[t * QR + ((p + t - 2) & (QR - 1))];
        emit(p, acc * sf);
      };
      // Tiles are consumed in pairs (k, k + 1): each thread holds position k TP + m and
      // (k + 1) TP + m, so layer 3 runs in packed fp32 over the POSITION pair with the weight as
      // a broadcast (uniform) operand.  w2 and b1 arrive scaled by the power of two d_scale
      // (a.w.w2 = w2 d_scale, a.w.b1 = b1 / d_scale: ReLU(d s + b1) w2 = ReLU(s + b1 / d) (w2 d)
      // exactly), so the accumulator only needs its two FP16x3 halves added.
      for (int k = 0; k < ntile; k += 2) {
        const bool two = k + 1 < ntile;
        const int sa = k % NSD, sb = (k + 1) % NSD;
        mb_wait(&dfull[sa], (uint32_t)(k / NSD) & 1u);
        if (two) mb_wait(&dfull[sb], (uint32_t)((k + 1) / NSD) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(sa * 32);
        // an unpaired last tile reads its own columns twice (position B is never stored)
        const uint32_t tb = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)((two ? sb : sa) * 32);
        float2 q2[KS];
#pragma unroll
        for (int t = 0; t < KS; ++t) q2[t] = make_float2(0.f, 0.f);
#pragma unroll
        for (int h4 = 0; h4 < 4; ++h4) {                 // channels 4 h4 .. 4 h4 + 3
          // d[0..3] / d[4..7]: the two FP16x3 halves at position A; d[8..15] the same at B
          uint32_t d[16];
          tld4(ta + 4 * h4, d);
          tld4(ta + 16 + 4 * h4, d + 4);
          tld4(tb + 4 * h4, d + 8);
          tld4(tb + 16 + 4 * h4, d + 12);
          tld_wait16(d);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const int ch = 4 * h4 + c;
            // the halves per position (scalar adds: their results pair up without moves)
            float2 z = make_float2(__uint_as_float(d[c]) + __uint_as_float(d[4 + c]),
                                   __uint_as_float(d[8 + c]) + __uint_as_float(d[12 + c]));
            z = __fadd2_rn(z, make_float2(a.w.b1[ch], a.w.b1[ch]));
            const float2 av = make_float2(fmaxf(z.x, 0.f), fmaxf(z.y, 0.f));
#pragma unroll
            for (int t = 0; t < KS; ++t)
              q2[t] = __ffma2_rn(av, make_float2(a.w.w2[ch * KS + t], a.w.w2[ch * KS + t]), q2[t]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          mb_arrive(&dempty[sa]);
          if (two) mb_arrive(&dempty[sb]);
        }
        const int Q0 = k * TP;
        asm volatile("bar.sync 1, 128;\n" ::: "memory");   // the previous pair's assembly is done
#pragma unroll
        for (int t = 0; t < KS; ++t) {
          qs[t * QR + ((Q0 + m) & (QR - 1))] = q2[t].x;
          if (two) qs[t * QR + ((Q0 + TP + m) & (QR - 1))] = q2[t].y;
        }
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        const int p = Q0 - 2 + m;
        if (p >= 0) assemble(p);
        if (two) assemble(Q0 + TP - 2 + m);
      }
      // positions n, n + 1 are zero padding; finish h(n - 2), h(n - 1)
      if (m < 2) {
#pragma unroll
        for (int t = 0; t < KS; ++t) qs[t * QR + ((n + m) & (QR - 1))] = 0.f;
      }
      asm volatile("bar.sync 1, 128;\n" ::: "memory");
      if (m < 2) assemble(n - 2 + m);
    }
    __syncthreads();
    S1D_TS(2);
    if (a.filter) {
      // ---- level filter F'_l on the whole row (see level_filter_row): h moves from the input-row
      // buffer into the (now free) a1 stages in the swizzled layout; the row buffer is the scratch
      for (int j = tid; j < n; j += NT) hb[hsw(j)] = u[UPAD + j];
      const bool pre = false;
      level_filter_row(reinterpret_cast<float2*>(hb), reinterpret_cast<float2*>(u + UPAD), n, a.twiddle, a.tw_n,
                       tid);
      S1D_TS(3);
      if (pre) {
        asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
      }
      const float scale = 2.0f / (float)n;   // 1/(n/2) of the half-length inverse
      float mx = 0.f;
      for (int j = tid; j < n; j += NT) {
        const float v = hb[hsw(j)] * scale;
        const float xv = a.accumulate ? (pre ? u[UPAD + j] : xrow[j]) + v : v;
        xrow[j] = xv;
        if (a.xh) tf32_store(xv, a.xh, a.xl, (int64_t)rhs * a.ldx + j);
        if (a.x16h) { hb[hsw(j)] = xv; mx = fmaxf(mx, fabsf(xv)); }
      }
      if (a.x16h) {
        // f16 hi/lo split of the updated row for the next FP16x3 operator apply, with the
        // row's power-of-two scale S (S max|x| <= 2^14), as split_f16_rows
        __shared__ float redf[NT / 32];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) redf[warp] = mx;
        __syncthreads();
        mx = redf[0];
#pragma unroll
        for (int w = 1; w < NT / 32; ++w) mx = fmaxf(mx, redf[w]);
        int e = 0;
        if (mx > 0.f) { frexpf(16384.f / mx, &e); e -= 1; }
        e = max(-100, min(100, e));
        const float S = ldexpf(1.f, e);
        if (tid == 0) a.xinv[rhs] = ldexpf(1.f, -e);
        __half* oh = reinterpret_cast<__half*>(a.x16h) + (int64_t)rhs * a.ldx;
        __half* ol = reinterpret_cast<__half*>(a.x16l) + (int64_t)rhs * a.ldx;
        for (int j = tid; j < n; j += NT) {
          const float v = hb[hsw(j)] * S;
          const __half hv = __float2half_rn(v);
          oh[j] = hv;
          ol[j] = __float2half_rn(v - __half2float(hv));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  S1D_TS(4);
#ifdef NMG_S1D_PHASES
  if (threadIdx.x == 0 && blockIdx.x == 0)
    printf("s1d n=%d: setup+norm %lld  tiles %lld  filter %lld  update %lld  (cycles)\n", n, ts[1] - ts[0],
           ts[2] - ts[1], ts[3] - ts[2], ts[4] - ts[3]);
#endif
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(32 * NSD));
}

constexpr int kNSA = 2;   // a1 stages: more buy nothing once shared-memory bandwidth binds

size_t smem_of(int n) {
  return 1024 + abuf_bytes(kNSA, n) + KS * BTAP + sizeof(float) * (KS * QR + n + 2 * UPAD) +
         8 * (2 * kNSA + 2 * NSD) + 16;
}

}  // namespace

size_t smooth1d_f16_smem(int n) { return smem_of(n); }

void smooth1d_f16(const Smooth1dArgs& a, cudaStream_t s) {
  NMG_SMEM_OPTIN(smooth1d_f16_kernel<kNSA>, smem_of(8192));
  smooth1d_f16_kernel<kNSA><<<a.nrhs, NT, smem_of(a.n), s>>>(a);
}

}  // namespace nmg
