// 2D CNN smoother (reading R7: conv(1->C) ReLU conv(C->C) ReLU conv(C->C) ReLU conv(C->1),
// 3x3, zero "same" padding, bias), C = 32 or 48, n % 128 == 0 (n < 128: one strip per image
// row, the 128 - n pixels beyond the row are zero padding and not stored): two persistent
// tcgen05 kernels with FP16x3 products on power-of-two-scaled operands (fp32-accurate).
//
// Pixels sit on the MMA M axis (128 consecutive pixels x = X0..X0+127 of one image row y);
// the N axis stacks the three vertical taps with the output channels, n' = t2*C + o; the K
// axis stacks the horizontal taps with the input channels, k' = t1*C + c:
//
//   D_t2(y, x)[o] = sum_{t1, c} W[o][c][t2][t1] in[c](y, x + t1 - 1)        (one MMA chain)
//   out(y, x)[o]  = b[o] + D_0(y - 1, x) + D_1(y, x) + D_2(y + 1, x)         (epilogue)
//
// The horizontal shift t1 is a 16-byte start-address offset of the A descriptor: the input
// row lives in shared memory in the canonical no-swizzle K-major layout [C/8][130][8 x f16]
// (8-row core matrices contiguous, SBO = 128 B), so pixel x + t1 - 1 is row m + t1 of the
// 130-row buffer.  The vertical combination is temporal: a CTA sweeps down a 128-pixel
// column strip and each epilogue thread (one pixel, a quarter of the channels) carries the
// partial rows in registers.  No output pixel is computed twice, no halo is recomputed.
//
//   strip_l12 : a1 = ReLU(w0 * u + b0) (FFMA, u = b / ||b||) computed row by row by five
//               producer warps straight into the A ring; layer 2 on tcgen05; the epilogue
//               writes a2 (scaled, f16 hi/lo) as pixel-major tensors [b][y][x][C].
//   strip_l34 : TMA loads a2 rows (x halo and image borders zero-filled by the TMA unit);
//               layer 3 on tcgen05; the epilogue applies ReLU and contracts a3 with the last
//               layer's weights into three per-t1 partial sums Q_t1(y, x) (float4 [b][y][x]).
//   combine   : h(y, x) = s (b3 + Q_0(y, x-1) + Q_1(y, x) + Q_2(y, x+1)) -> filter input / x.
//
// FP16x3: v S = hi + lo with hi = f16(v S), lo = f16(v S - hi), S a power of two chosen on
// the host from a rigorous bound on |v| (|u| <= 1 because ||u||_2 = 1; bounds propagate
// through the layers), so hi never overflows and lo stays in the normal range for the values
// that matter; D = Ah Bh + Ah Bl + Al Bh in fp32, rescaled exactly by 1/(S_a S_w).  The
// dropped Al Bl term and the representation error are ~2^-22 relative per product (BF16x3
// would be 2^-17, which the filtered smoothing increment amplifies past 1e-5).
//
// Warp roles (448 threads, one CTA per SM): warps 0 .. 4 NG - 1 epilogue (warp w reads TMEM
// lanes 32 (w % 4).., channel group w / 4), warps 4 NG .. 12 producer, warp 13 MMA issuer;
// NG = 1 for layers 1-2 at C = 32 (9 producer warps), else 2.
#include <cuda.h>
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace nmg {
namespace {

constexpr int SEG = 128;        // pixels per strip (MMA M)
constexpr int RP = SEG + 2;     // rows of the activation buffer (x halo)
constexpr uint32_t IDESC4 = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(SEG >> 4) << 24);  // N = 16
// Warp roles: epilogue warps 0 .. 4 NG - 1 (TMEM lane quarter w % 4, channel group w / 4);
// layers 1-2: producer warps 4 NG .. 12 (FFMA a1, a position pair and C / NQ channels per
// thread), warp 13 MMA issuer; layers 3-4: warp 4 NG TMA, warp 4 NG + 1 layer-4 MMA issuer,
// warp 4 NG + 2 layer-3 MMA issuer.
template <int C, bool FIRST>
struct Roles {
#ifndef NMG_STRIP_NG32
#define NMG_STRIP_NG32 2
#endif
#ifndef NMG_STRIP_P32
#define NMG_STRIP_P32 9
#endif
  // layers 1-2 at C = 32: 8 epilogue warps (two 16-channel groups) and 9 FFMA producer warps
  // with four 8-channel groups per pixel pair (576 threads); layers 3-4: 8 epilogue warps
#ifndef NMG_STRIP_NG48L34
#define NMG_STRIP_NG48L34 2
#endif
  static constexpr int NG = (FIRST && C == 32) ? NMG_STRIP_NG32 : (!FIRST && C == 48) ? NMG_STRIP_NG48L34 : 2;
  // channel groups per producer item (position pair): the 130 row positions x NQ groups
  // spread over the producer threads
#ifndef NMG_STRIP_P48
#define NMG_STRIP_P48 7
#endif
  // layers 1-2 at C = 48: NMG_STRIP_P48 producer warps; 7 warps split a pixel pair's channels
  // in three groups of 16 (195 items)
  static constexpr int NQ = (NG == 1 || (FIRST && C == 32 && NMG_STRIP_P32 >= 9)) ? 4
                            : (FIRST && C == 48 && NMG_STRIP_P48 == 7) ? 3 : 2;
  static constexpr int PROD0 = 4 * NG;                    // first producer warp
  // layers 1-2: FFMA producer warps up to warp 12; layers 3-4: one TMA warp and the layer-4
  // MMA warp only (the rest of the threads go to the epilogue)
  static constexpr int MMAW = FIRST ? (C == 48 ? PROD0 + NMG_STRIP_P48 : (NMG_STRIP_P32 ? PROD0 + NMG_STRIP_P32 : 13))
                                    : PROD0 + 2;   // MMA issuer warp
  static constexpr int NTHR = 32 * (MMAW + 1);
  static constexpr int NPROD = MMAW - PROD0;              // producer warps (FIRST)
};

template <int C>
struct Cfg {
  static constexpr int N = 3 * C;                       // (t2, o)
  static constexpr int K = 3 * C;                       // (t1, c)

  static constexpr int WBYTES = N * K * 2;              // one weight plane (hi or lo)
  static constexpr int ABYTES = ((RP * C * 2) + 127) / 128 * 128;   // one activation row, hi or lo
  static constexpr int ALBO = RP * 16;                  // K-chunk stride of the A buffer
  static constexpr int BLBO = N * 16;                   // K-chunk stride of the B (weight) planes
  // pipeline depths (dev knobs NMG_STRIP_*): activation ring and TMEM D buffers
#ifndef NMG_STRIP_NSTG32
#define NMG_STRIP_NSTG32 5
#endif
#ifndef NMG_STRIP_NSTG48
#define NMG_STRIP_NSTG48 3
#endif
#ifndef NMG_STRIP_NDB
#define NMG_STRIP_NDB 2
#endif
  static constexpr int NSTG = C == 32 ? NMG_STRIP_NSTG32 : NMG_STRIP_NSTG48;
  static constexpr int NDB = NMG_STRIP_NDB;
  static constexpr int TCOLS = NDB * N + 16 <= 256 ? 256 : 512;   // D buffers + D4 (16 columns)
  static constexpr int A4BYTES = SEG * C * 2;           // layer-4 A tile (a3 row), hi or lo
  static constexpr int A4LBO = SEG * 16;
  static constexpr int W4BYTES = 16 * C * 2;            // layer-4 weights [C/8][16][8], hi or lo
  static constexpr int W4LBO = 16 * 16;
  static constexpr int MISC = 8192;                     // barriers, small params
  static constexpr int SMEM = 2 * WBYTES + NSTG * 2 * ABYTES + 2 * A4BYTES + 2 * W4BYTES + MISC + 1024;
  // kind::f16, D f32, A/B f16, K-major both, N, M = 128
  static constexpr uint32_t IDESC = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(SEG >> 4) << 24);
};

template <int CG>
NMG_D void tld_wait(uint32_t* r);
template <>
NMG_D void tld_wait<16>(uint32_t* r) { tld_wait16(r); }
template <>
NMG_D void tld_wait<24>(uint32_t* r) { tld_wait24(r); }
// CG consecutive TMEM columns of this thread's lane
template <int CG>
NMG_D void tload(uint32_t taddr, uint32_t* r) {
#pragma unroll
  for (int j = 0; j < CG / 8; ++j) tld8(taddr + 8 * j, r + 8 * j);
  if constexpr (CG == 32) {
    tld_wait<16>(r);
    tld_wait<16>(r + 16);
  } else {
    tld_wait<CG>(r);
  }
}

// 8 fp32 (already scaled) -> f16 hi (8) and lo (8) packed as uint4; the residual v - hi of a
// channel pair is one packed FADD2 (each lane rounds as the scalar subtraction: same bits)
NMG_D void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 hv = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
    const float2 hf = __half22float2(hv);
    const float2 r = __fadd2_rn(make_float2(v[2 * j], v[2 * j + 1]), make_float2(-hf.x, -hf.y));
    const __half2 lv = __floats2half2_rn(r.x, r.y);
    h[j] = *reinterpret_cast<const uint32_t*>(&hv);
    l[j] = *reinterpret_cast<const uint32_t*>(&lv);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

struct Unit {
  int b, X0, y0, y1;
};
// hg = image height (rows), n = width
NMG_D Unit unit_of(int u, int hg, int nx, int ys) {
  Unit t;
  const int per = nx * ys;
  t.b = u / per;
  const int r = u - t.b * per;
  const int yi = r / nx, xi = r - yi * nx;
  t.X0 = xi * SEG;
  const int rows = (hg + ys - 1) / ys;
  t.y0 = yi * rows;
  t.y1 = min(hg, t.y0 + rows);
  return t;
}

// ------------------------------------------------------------------------------------------
template <int C, bool FIRST>
__global__ void __launch_bounds__(Roles<C, FIRST>::NTHR, 1)
    conv_strip_kernel(const __grid_constant__ CUtensorMap mInH, const __grid_constant__ CUtensorMap mInL,
                      StripArgs a) {
  using G = Cfg<C>;
  using RL = Roles<C, FIRST>;
  constexpr int NSTG = G::NSTG, NDB = G::NDB;
  constexpr int MMAW = RL::MMAW, NTHR = RL::NTHR;
  constexpr int NGRP = RL::NG;
  constexpr int PROD0 = RL::PROD0;
  constexpr int CG = C / NGRP;                           // channels per epilogue thread
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u);
  uint8_t* Wh = sm;
  uint8_t* Wl = Wh + G::WBYTES;
  uint8_t* ring = Wl + G::WBYTES;                        // NSTG x (hi | lo)
  uint8_t* A4 = ring + NSTG * 2 * G::ABYTES;             // !FIRST: a3 row (hi | lo) for layer 4
  uint8_t* W4 = A4 + 2 * G::A4BYTES;                     // !FIRST: layer-4 weights (hi | lo)
  uint8_t* misc = W4 + 2 * G::W4BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(misc);    // [NSTG]
  uint64_t* empty = full + NSTG;                         // [NSTG]
  uint64_t* dfull = empty + NSTG;                        // [NDB]
  uint64_t* dempty = dfull + NDB;                        // [NDB]
  uint64_t* a4full = dempty + NDB;
  uint64_t* d4full = a4full + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(d4full + 1);
  // FIRST: w0 transposed [t][c] then b0 [c];  else: w3 transposed [t][c]
  float* swt = reinterpret_cast<float*>(misc + 512);
  float* sbias = swt + 10 * C;                           // hidden-layer bias [C]

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n;
  const int hg = a.h ? a.h : n;              // stored rows per image (slab mode: R + 2 halo rows)
  // rows [ylo, yhi) are the image; the rest is zero padding of EVERY layer's input (a slab at
  // the top / bottom image border has its outer halo rows outside the image)
  const int ylo = a.ylo, yhi = a.yhi ? a.yhi : hg;
  const int nx = n >= SEG ? n / SEG : 1;   // n < 128: one strip, pixels x >= n are padding
  const int units = a.nrhs * nx * a.ysplit;

  {
    const uint4* gh = reinterpret_cast<const uint4*>(a.wh);
    const uint4* gl = reinterpret_cast<const uint4*>(a.wl);
    uint4* dh = reinterpret_cast<uint4*>(Wh);
    uint4* dl = reinterpret_cast<uint4*>(Wl);
    for (int i = tid; i < G::WBYTES / 16; i += NTHR) { dh[i] = __ldg(gh + i); dl[i] = __ldg(gl + i); }
    // the layer's output scale (a2 S2 / a3 S3, powers of two) folded into the bias and the
    // accumulator scale: ReLU(d acc + b) S = ReLU((d S) acc + b S), bitwise
    const float osc_fold = FIRST ? a.out_scale : a.a3_scale;
    for (int i = tid; i < C; i += NTHR) sbias[i] = __ldg(a.bias + i) * osc_fold;
    if (!FIRST) {
      const uint4* g4 = reinterpret_cast<const uint4*>(a.w4);
      uint4* d4 = reinterpret_cast<uint4*>(W4);
      for (int i = tid; i < 2 * G::W4BYTES / 16; i += NTHR) d4[i] = __ldg(g4 + i);
    }
    const float* wsrc = FIRST ? a.w_in : a.w_out;      // [c][9]
    const float wsc = FIRST ? a.in_scale : 1.f;         // layers 1-2: w0, b0 pre-scaled by S1
    for (int i = tid; i < 9 * C; i += NTHR) {
      const int t = i / C, c = i - t * C;
      swt[i] = __ldg(wsrc + c * 9 + t) * wsc;
    }
    if (FIRST)
      for (int i = tid; i < C; i += NTHR) swt[9 * C + i] = __ldg(a.w_in + 9 * C + i) * wsc;
  }
  if (tid == 0) {
    for (int s = 0; s < NSTG; ++s) { mb_init(&full[s], FIRST ? RL::NPROD : 1); mb_init(&empty[s], 1); }
    for (int s = 0; s < NDB; ++s) { mb_init(&dfull[s], 1); mb_init(&dempty[s], 4 * NGRP); }
    mb_init(a4full, 4 * NGRP);
    mb_init(d4full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == MMAW) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)),
                 "r"(G::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  // virtual input rows of a unit: [y0 - H, y1 + H - 1], H = 1 (layers 1-2) or 2 (layers 3-4)
  constexpr int H = FIRST ? 1 : 2;

  if (warp >= PROD0 && warp < (FIRST ? MMAW : MMAW - 1)) {
    // ------------------------------------------------------------------ producer
    if (FIRST) {
      // item = (position pair p, p + 65 of the row buffer (x = X0 - 1 + p), channel half);
      // 130 items over the 160 producer threads, the weights of a tap loaded once for both
      // positions; 3 x 3 windows of b slide down with the rows, the next row prefetched.
      // w0 and b0 in shared memory are pre-scaled by S1 (ReLU(S z) = S ReLU(z), S > 0).
      constexpr int HC = C / RL::NQ;                       // channels per item
      constexpr int PP = RP / 2;                           // 65 position pairs
      const int pt = tid - PROD0 * 32;
      const int j = pt % PP, half = pt / PP;
      const bool act = pt < RL::NQ * PP;
      const int c0p = half * HC;
      int it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit t = unit_of(u, hg, nx, a.ysplit);
        const double s = a.norms ? a.norms[t.b] : 1.0;
        const float inv = (float)((s != 0.0) ? 1.0 / s : 0.0);
        const float* B = a.b + (int64_t)t.b * hg * n;
        int xs[2];
        bool xin[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          xs[e] = t.X0 - 1 + j + e * PP;
          xin[e] = act && xs[e] >= 0 && xs[e] < n;
        }
        auto ld3 = [&](int yy, float (*w)[3]) {
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const bool ok = xin[e] && yy >= ylo && yy < yhi;
            const float* row = B + (int64_t)yy * n;
#pragma unroll
            for (int t1 = 0; t1 < 3; ++t1) {
              const int xx = xs[e] + t1 - 1;
              w[e][t1] = (ok && xx >= 0 && xx < n) ? __ldg(row + xx) : 0.f;
            }
          }
        };
        const int r0 = max(t.y0 - H, ylo), r1 = min(t.y1 + H - 1, yhi - 1);
        float win[3][2][3];
        ld3(r0 - 1, win[0]);
        ld3(r0, win[1]);
        ld3(r0 + 1, win[2]);
        for (int r = r0; r <= r1; ++r, ++it) {
          float nxt[2][3];
          ld3(r + 2, nxt);                       // in flight while this row is computed
          float uu[2][9];
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int t2 = 0; t2 < 3; ++t2)
#pragma unroll
              for (int t1 = 0; t1 < 3; ++t1) uu[e][t2 * 3 + t1] = win[t2][e][t1] * inv;
          const int st = it % NSTG;
          mb_wait(&empty[st], ((uint32_t)(it / NSTG) & 1u) ^ 1u);
          if (act) {
            uint4* ah = reinterpret_cast<uint4*>(ring + st * 2 * G::ABYTES);
            uint4* al = reinterpret_cast<uint4*>(ring + st * 2 * G::ABYTES + G::ABYTES);
#pragma unroll 1
            for (int g = c0p / 8; g < (c0p + HC) / 8; ++g) {
              // channel pairs in packed fp32 (FFMA2: two FMAs per issue slot, each lane
              // rounded exactly as a scalar fmaf, same order => same bits)
              float2 v2[2][4];
              {
                const float4 b0a = *reinterpret_cast<const float4*>(swt + 9 * C + 8 * g);
                const float4 b0b = *reinterpret_cast<const float4*>(swt + 9 * C + 8 * g + 4);
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  v2[e][0] = make_float2(b0a.x, b0a.y); v2[e][1] = make_float2(b0a.z, b0a.w);
                  v2[e][2] = make_float2(b0b.x, b0b.y); v2[e][3] = make_float2(b0b.z, b0b.w);
                }
              }
#pragma unroll
              for (int q9 = 0; q9 < 9; ++q9) {
                const float4 wa = *reinterpret_cast<const float4*>(swt + q9 * C + 8 * g);
                const float4 wb = *reinterpret_cast<const float4*>(swt + q9 * C + 8 * g + 4);
                const float2 w2[4] = {make_float2(wa.x, wa.y), make_float2(wa.z, wa.w), make_float2(wb.x, wb.y),
                                      make_float2(wb.z, wb.w)};
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                  const float2 u2 = make_float2(uu[e][q9], uu[e][q9]);
#pragma unroll
                  for (int c = 0; c < 4; ++c) v2[e][c] = __ffma2_rn(w2[c], u2, v2[e][c]);
                }
              }
              float v[2][8];
#pragma unroll
              for (int e = 0; e < 2; ++e) {
#pragma unroll
                for (int c = 0; c < 4; ++c) { v[e][2 * c] = v2[e][c].x; v[e][2 * c + 1] = v2[e][c].y; }
#pragma unroll
                for (int c = 0; c < 8; ++c) v[e][c] = fmaxf(v[e][c], 0.f);
                uint4 hi, lo;
                split8(v[e], hi, lo);
                // a position outside the image is zero padding of layer 2's input: predicated
                // zero stores instead of a select per channel
                if (xin[e]) {
                  ah[g * RP + j + e * PP] = hi;
                  al[g * RP + j + e * PP] = lo;
                } else {
                  ah[g * RP + j + e * PP] = make_uint4(0u, 0u, 0u, 0u);
                  al[g * RP + j + e * PP] = make_uint4(0u, 0u, 0u, 0u);
                }
              }
            }
          }
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mb_arrive(&full[st]);
#pragma unroll
          for (int e = 0; e < 2; ++e)
#pragma unroll
            for (int t1 = 0; t1 < 3; ++t1) {
              win[0][e][t1] = win[1][e][t1];
              win[1][e][t1] = win[2][e][t1];
              win[2][e][t1] = nxt[e][t1];
            }
        }
      }
    } else if (tid == PROD0 * 32) {
      int it = 0;
      const uint32_t bytes = 2u * (uint32_t)(RP * C * 2);
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit t = unit_of(u, hg, nx, a.ysplit);
        const int r0 = max(t.y0 - H, ylo), r1 = min(t.y1 + H - 1, yhi - 1);
        for (int r = r0; r <= r1; ++r, ++it) {
          const int st = it % NSTG;
          mb_wait(&empty[st], ((uint32_t)(it / NSTG) & 1u) ^ 1u);
          uint8_t* dst = ring + st * 2 * G::ABYTES;
          mb_expect(&full[st], bytes);
          tma5d(dst, &mInH, &full[st], 0, t.X0 - 1, 0, r, t.b);
          tma5d(dst + G::ABYTES, &mInL, &full[st], 0, t.X0 - 1, 0, r, t.b);
        }
      }
    }
  } else if (warp == MMAW) {
    // ------------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      const uint32_t wh = su32(Wh), wl = su32(Wl), rb = su32(ring);
      int it = 0, k = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit t = unit_of(u, hg, nx, a.ysplit);
        for (int r = t.y0 - H; r <= t.y1 + H - 1; ++r, ++k) {
          const int buf = k % NDB;
          mb_wait(&dempty[buf], ((uint32_t)(k / NDB) & 1u) ^ 1u);
          if (r < ylo || r >= yhi) {      // zero-padding row: nothing to multiply
            mb_arrive(&dfull[buf]);
            continue;
          }
          const int st = it % NSTG;
          mb_wait(&full[st], (uint32_t)(it / NSTG) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t d = tmem + (uint32_t)(buf * G::N);
          const uint32_t ah = rb + st * 2 * G::ABYTES, al = ah + G::ABYTES;
          uint32_t acc = 0;
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            const uint32_t A = pass == 2 ? al : ah;
            const uint32_t Bw = pass == 1 ? wl : wh;
#pragma unroll
            for (int t1 = 0; t1 < 3; ++t1) {
#pragma unroll
              for (int kc = 0; kc < C / 16; ++kc) {
                const uint64_t da = desc_ns(A + (uint32_t)(t1 * 16 + 2 * kc * G::ALBO), G::ALBO);
                const uint64_t db = desc_ns(Bw + (uint32_t)((t1 * (C / 8) + 2 * kc) * G::BLBO), G::BLBO);
                mma_f16(d, da, db, G::IDESC, acc);
                acc = 1;
              }
            }
          }
          mma_commit(&empty[st]);
          mma_commit(&dfull[buf]);
          ++it;
        }
      }
    }
    __syncwarp();
  } else if (!FIRST && warp == MMAW - 1) {
    // ------------------------------------------------------------------ layer-4 MMA issuer
    // (its own thread, so the layer-3 chain of the next row never waits for the epilogue)
    if (lane == 0) {
      const uint32_t a4h = su32(A4), a4l = a4h + G::A4BYTES, w4h = su32(W4), w4l = w4h + G::W4BYTES;
      const uint32_t d4 = tmem + (uint32_t)(NDB * G::N);
      int e4 = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        const Unit t = unit_of(u, hg, nx, a.ysplit);
        for (int r = t.y0 - H; r <= t.y1 + H - 1; ++r, ++e4) {
          // D4[p][t2 * 3 + t1] = sum_c a3[c](p) w3[c][t2][t1] for the a3 row the epilogue wrote
          mb_wait(a4full, (uint32_t)e4 & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          uint32_t acc = 0;
#pragma unroll
          for (int pass = 0; pass < 3; ++pass) {
            const uint32_t A = pass == 2 ? a4l : a4h;
            const uint32_t Bw = pass == 1 ? w4l : w4h;
#pragma unroll
            for (int kc = 0; kc < C / 16; ++kc) {
              mma_f16(d4, desc_ns(A + (uint32_t)(2 * kc * G::A4LBO), G::A4LBO),
                      desc_ns(Bw + (uint32_t)(2 * kc * G::W4LBO), G::W4LBO), IDESC4, acc);
              acc = 1;
            }
          }
          mma_commit(d4full);
        }
      }
    }
    __syncwarp();
  } else if (warp < PROD0) {
    // ------------------------------------------------------------------ epilogue (warps 0-7)
    const int q = warp & 3;                 // TMEM lane quarter
    const int grp = warp >> 2;              // channel half
    const int m = q * 32 + lane;            // pixel within the strip
    const int c0 = grp * CG;
    const float* bv = sbias + c0;
    const float dsc = a.d_scale * (FIRST ? a.out_scale : a.a3_scale);   // output scale folded (see sbias)
    const float b3v = FIRST ? 0.f : __ldg(a.b3);
    float* xch = reinterpret_cast<float*>(misc + 4096);     // [2][4 warps][Q0 of lane 31, Q2 of lane 0]
    int k = 0, e4 = 0;
    float acc4[3][3];                        // layer 4 partial rows h(ya - 1 + i) (FIRST == false)
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) acc4[i][j] = 0.f;
    // a3 row ya went through the layer-4 MMA: h rows ya + 1 (t2 = 0), ya (t2 = 1), ya - 1 (t2 = 2)
    // receive its contributions; h row ya - 1 is then complete
    auto consume_d4 = [&](const Unit& t, int x, int ya) {
      mb_wait(d4full, (uint32_t)e4 & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      ++e4;
      if (grp == 0) {
        uint32_t d[16];
        tld8(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(NDB * G::N), d);
        tld8(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(NDB * G::N + 8), d + 8);
        tld_wait<16>(d);
        const float s4 = a.d4_scale;
#pragma unroll
        for (int t2 = 0; t2 < 3; ++t2)
#pragma unroll
          for (int t1 = 0; t1 < 3; ++t1) acc4[2 - t2][t1] = fmaf(__uint_as_float(d[t2 * 3 + t1]), s4, acc4[2 - t2][t1]);
        // h(yh, x) = b3 + Q0(x - 1) + Q1(x) + Q2(x + 1) (in this order): the x -+ 1 taps of
        // the neighbouring pixels by shuffles inside the warp and through shared memory across
        // the four lane-quarter warps; the strip's first and last pixel lack the term from the
        // neighbouring strip and are finished by strip_combine / combine_rows_fft from the
        // strip-edge records {Q2(X0), Q0(X0 + 127), Q2(X0 + 1)} (same summation order, so the
        // result is bitwise the one of a whole-row combine)
        const int yh = ya - 1;
        const float Q0 = acc4[0][0], Q1 = acc4[0][1], Q2 = acc4[0][2];
        float left = __shfl_up_sync(0xffffffffu, Q0, 1);
        float right = __shfl_down_sync(0xffffffffu, Q2, 1);
        float* xw = xch + 8 * (e4 & 1);
        if (lane == 31) xw[2 * q] = Q0;
        if (lane == 0) xw[2 * q + 1] = Q2;
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        if (lane == 0 && q > 0) left = xw[2 * (q - 1)];
        if (lane == 31 && q < 3) right = xw[2 * (q + 1) + 1];
        if (yh >= t.y0 && yh < t.y1 && x < n) {
          const int64_t row = (int64_t)t.b * hg + yh;
          float* er = reinterpret_cast<float*>(a.qe + row * nx + (t.X0 / SEG));
          float v = b3v + Q1;
          if (m == 0 && x > 0) {            // Q0(x - 1) belongs to the strip on the left
            er[2] = right;
          } else {
            if (x > 0) v += left;
            if (x < n - 1 && m != SEG - 1) v += right;   // else Q2(x + 1) is the right strip's
          }
          a.q[row * n + x] = v;
          if (m == 0) er[0] = Q2;
          if (m == SEG - 1) er[1] = Q0;
        }
#pragma unroll
        for (int t1 = 0; t1 < 3; ++t1) {
          acc4[0][t1] = acc4[1][t1];
          acc4[1][t1] = acc4[2][t1];
          acc4[2][t1] = 0.f;
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    };
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      const Unit t = unit_of(u, hg, nx, a.ysplit);
      const int x = t.X0 + m;
      float2 P0[CG / 2], P1[CG / 2];              // channel pairs (packed fp32 adds)
#pragma unroll
      for (int j = 0; j < CG / 2; ++j) { P0[j] = make_float2(0.f, 0.f); P1[j] = make_float2(0.f, 0.f); }
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) acc4[i][j] = 0.f;
      for (int r = t.y0 - H; r <= t.y1 + H - 1; ++r, ++k) {
        const int buf = k % NDB;
        const bool valid = r >= ylo && r < yhi;
        mb_wait(&dfull[buf], (uint32_t)(k / NDB) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t tb = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(buf * G::N + c0);
        // output row r - 1 is complete: b + D_0(r - 2) + D_1(r - 1) + D_2(r)
        const int yo = r - 1;
        const bool yin = yo >= ylo && yo < yhi;
        // layers 3-4: the previous a3 row's layer-4 result first (it also frees the A4 tile)
        if (!FIRST && r > t.y0 - H) consume_d4(t, x, r - 2);
        const bool store = FIRST && yo >= t.y0 && yo < t.y1 && x < n;
        const int64_t off = (((int64_t)t.b * hg + (store ? yo : 0)) * n + x) * C + c0;
        // 8 channels at a time: D_2 -> this row's activation, D_1 / D_0 -> the carries.  With
        // 16 channels per thread all 48 columns are loaded before one wait (latency once per row)
        constexpr int GB = CG == 16 ? 2 : 1;             // chunks per TMEM wait
        uint32_t DD[GB][24];
#pragma unroll
        for (int g = 0; g < CG / 8; ++g) {
          uint32_t* D = DD[g % GB];
          if (g % GB == 0) {
            if (valid) {
#pragma unroll
              for (int gg = 0; gg < GB; ++gg) {
                tld8(tb + 2 * C + 8 * (g + gg), DD[gg]);
                tld8(tb + C + 8 * (g + gg), DD[gg] + 8);
                tld8(tb + 8 * (g + gg), DD[gg] + 16);
              }
#pragma unroll
              for (int gg = 0; gg < GB; ++gg) tld_wait<24>(DD[gg]);
            } else {
#pragma unroll
              for (int gg = 0; gg < GB; ++gg)
#pragma unroll
                for (int j = 0; j < 24; ++j) DD[gg][j] = 0u;
            }
          }
          float act[8];
          const float2 dsc2 = make_float2(dsc, dsc);
#pragma unroll
          for (int j = 0; j < 8; j += 2) {
            const int c = 8 * g + j;
            const float2 d2 = make_float2(__uint_as_float(D[j]), __uint_as_float(D[j + 1]));
            const float2 t = __ffma2_rn(__fadd2_rn(P1[c / 2], d2), dsc2, make_float2(bv[c], bv[c + 1]));
            // layers 1-2 store only rows inside the image (store implies yin); layers 3-4 feed
            // the a3 row of a padding row to layer 4 as zeros
            act[j] = (FIRST || yin) ? fmaxf(t.x, 0.f) : 0.f;
            act[j + 1] = (FIRST || yin) ? fmaxf(t.y, 0.f) : 0.f;
            P1[c / 2] = __fadd2_rn(P0[c / 2], make_float2(__uint_as_float(D[8 + j]), __uint_as_float(D[9 + j])));
            P0[c / 2] = make_float2(__uint_as_float(D[16 + j]), __uint_as_float(D[17 + j]));
          }
          if (FIRST) {
            if (store) {
              uint4 hi, lo;
              split8(act, hi, lo);
#ifndef NMG_STRIP_NOSTORE
              reinterpret_cast<uint4*>(a.out_h + off)[g] = hi;
              reinterpret_cast<uint4*>(a.out_l + off)[g] = lo;
#else
              if (hi.x == 0x7fffffffu && lo.x == 0x7fffffffu) reinterpret_cast<uint4*>(a.out_h + off)[g] = hi;
#endif
            }
          } else {
            uint4 hi, lo;
            split8(act, hi, lo);
            reinterpret_cast<uint4*>(A4)[(c0 / 8 + g) * SEG + m] = hi;
            reinterpret_cast<uint4*>(A4 + G::A4BYTES)[(c0 / 8 + g) * SEG + m] = lo;
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mb_arrive(&dempty[buf]);
        if (!FIRST) {                                    // a3 row -> layer-4 MMA
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
          __syncwarp();
          if (lane == 0) mb_arrive(a4full);
        }
      }
      if (!FIRST) consume_d4(t, x, t.y1);                 // the unit's last a3 row
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == MMAW) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(G::TCOLS));
  }
}

// h(y, x) = s (b3 + Q0(y, x - 1) + Q1(y, x) + Q2(y, x + 1))  ->  Z = (h, 0) or x (+)= h.  The strip
// kernel stored the sum without the terms that cross a 128-pixel strip boundary; the strip's
// edge record E = {Q2(X0), Q0(X0 + 127), Q2(X0 + 1)} supplies them (strip_h_fix, common.cuh).
// slab mode: images of hg rows whose first and last hh rows are halo (not written)
__global__ void strip_combine_kernel(int n, int nrhs, const float* __restrict__ q, const float4* __restrict__ qe,
                                     const double* __restrict__ norms, float2* __restrict__ Z, int zb0,
                                     float* __restrict__ xo, int accumulate, int hg, int hh) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)hg * n;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int x = (int)(idx % n);
  const int row = (int)((idx - (int64_t)b * per) / n);
  if (row < hh || row >= hg - hh) return;
  const double s = norms ? norms[b] : 1.0;
  float acc = 0.f;
  if (s != 0.0) acc = strip_h_fix(__ldg(&q[idx]), qe + ((int64_t)b * hg + row) * (n / SEG), n, x);
  // the filter path takes N(u) unscaled; filter2d multiplies by s after F'
  if (Z) zput(Z, hg - 2 * hh, n, zb0 + b, row - hh, x, acc);
  else {
    const float hv = acc * (float)s;
    xo[idx] = accumulate ? xo[idx] + hv : hv;
  }
}

template <int C, bool FIRST>
void launch(const CUtensorMap* mh, const CUtensorMap* ml, const StripArgs& a, int num_sms, cudaStream_t s) {
  using G = Cfg<C>;
  NMG_SMEM_OPTIN((conv_strip_kernel<C, FIRST>), G::SMEM);
  const int units = a.nrhs * (a.n >= SEG ? a.n / SEG : 1) * a.ysplit;
  const int grid = std::min(units, num_sms);
  CUtensorMap dummy{};
  conv_strip_kernel<C, FIRST><<<grid, Roles<C, FIRST>::NTHR, G::SMEM, s>>>(mh ? *mh : dummy, ml ? *ml : dummy, a);
}

}  // namespace

int strip_ysplit(int n, int nrhs, int num_sms, int hg) {
  const int strips = nrhs * (n >= SEG ? n / SEG : 1);
  if (hg <= 0) hg = n;
  int ys = 1;
  while (strips * ys < 4 * num_sms && ys < hg / 32) ys *= 2;
  return ys;
}

void strip_l12(const StripArgs& a, int num_sms, cudaStream_t s) {
  if (a.C == 32) launch<32, true>(nullptr, nullptr, a, num_sms, s);
  else launch<48, true>(nullptr, nullptr, a, num_sms, s);
}
void strip_l34(const CUtensorMap* mh, const CUtensorMap* ml, const StripArgs& a, int num_sms, cudaStream_t s) {
  if (a.C == 32) launch<32, false>(mh, ml, a, num_sms, s);
  else launch<48, false>(mh, ml, a, num_sms, s);
}
void strip_combine(int n, int nrhs, const float* q, const float4* qe, const double* norms, float2* Z, int zb0,
                   float* x, bool accumulate, cudaStream_t s, int hg, int hh) {
  if (hg <= 0) hg = n;
  const int64_t tot = (int64_t)nrhs * hg * n;
  strip_combine_kernel<<<(int)ceil_div64(tot, 256), 256, 0, s>>>(n, nrhs, q, qe, norms, Z, zb0, x, accumulate ? 1 : 0,
                                                                 hg, hh);
}

}  // namespace nmg
