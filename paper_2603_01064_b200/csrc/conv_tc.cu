// 2D CNN smoother hidden layers (C -> C, 3x3, zero "same" padding, bias, ReLU; reading R7)
// as a tcgen05 implicit GEMM with 3xTF32 (fp32-accurate) products.
//
//   out[o](y, x) = b[o] + sum_{t2, t1, c} W[o][c][t2][t1] in[c](y + t2 - 1, x + t1 - 1)
//
// GEMM form per 8 x 32 pixel tile (N = 256 pixels, rows r = 0..7, columns xx = 0..31):
//   D[(t1, o)][p] = sum_{t2, c} W[o][c][t2][t1] * in[c](pixel p shifted by t2 - 1 rows)
//   M = 3 * 32 = 96 (padded to 128): taps t1 stacked in M;  K = 3 * C: taps t2 x channels.
// The t2 shift is a row offset of the B-operand descriptor into a 10-row input region held
// in shared memory; the t1 shift is applied in the epilogue (out(x) = D0(x-1) + D1(x) +
// D2(x+1)), so the 32-wide tile yields 30 valid output columns.
//
// Activations live in HBM as padded pixel-major fp32 tensors [b][n+2][n+2][C] (1-pixel
// zero border).  Roles (256 threads, persistent CTAs):
//   warp 0 : TMA producer (weights once; per tile two 16-channel input chunks, SWIZZLE_64B)
//   warps 6-7 : form the tf32 lo part lo = x - trunc_tf32(x) of each landed chunk in smem
//              (the tensor core reads the fp32 chunk itself as the hi part)
//   warp 1 : MMA issuer (tcgen05.mma kind::tf32, M=128 N=256 K=8), double-buffered TMEM
//   warps 2-5 : epilogue (tcgen05.ld -> cross-tap sum through smem -> bias/ReLU -> fp32)
#include <cuda.h>

#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace nmg {
namespace {

constexpr int CC = 32;                      // channels (cfg 2 / cfg 4)
constexpr int TR = 8, TW = 32;              // tile rows x columns (N = 256)
constexpr int RR = TR + 2;                  // input region rows
constexpr int NCH = CC / 16;                // 16-channel chunks
constexpr int AM = 128;                     // padded M
constexpr int A_BLK = AM * 16 * 4;          // one (t2, chunk) weight block, bytes (8 KB)
constexpr int A_BYTES = 3 * NCH * A_BLK;    // 48 KB per hi / lo
constexpr int B_HALF = RR * TW * 16 * 4;    // one chunk region, hi or lo (20 KB)
constexpr int B_STAGE = 2 * B_HALF;         // hi + lo (40 KB)
constexpr int NSTAGE = 2;
constexpr int NGRP = 2;                     // epilogue warp groups (rows r = g, g + 3, ...)
constexpr int SX_BYTES = NGRP * 3 * 32 * 33 * 4;   // epilogue exchange [group][t1][o][xx]
constexpr int CONV_SMEM = 2 * A_BYTES + NSTAGE * B_STAGE + SX_BYTES + 256 + 1024;
constexpr int NTHR = 384;                   // warps 6-7: tf32 lo converters; 2-5, 8-11, 12-15: epilogue

NMG_D uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
NMG_D void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c));
}
NMG_D void mb_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes));
}
NMG_D void mb_arrive(uint64_t* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b))); }
NMG_D void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(su32(b)),
      "r"(ph));
}
NMG_D void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
NMG_D void tma3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(
          su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
NMG_D uint64_t desc_sw64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
constexpr uint32_t kIdescConv = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(256 >> 3) << 17) |
                                ((uint32_t)(AM >> 4) << 24);
NMG_D void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdescConv), "r"(acc));
}
NMG_D void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(b))
               : "memory");
}
NMG_D void tf32_split(float v, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(v));
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(l) : "f"(v - __uint_as_float(h)));
  hi = __uint_as_float(h);
  lo = __uint_as_float(l);
}

struct TileCoord { int b, y0, X0; };
NMG_D TileCoord tile_coord(int t, int tiles_y, int tiles_x) {
  const int per = tiles_y * tiles_x;
  TileCoord c;
  c.b = t / per;
  const int r = t - c.b * per;
  c.y0 = (r / tiles_x) * TR;          // first output image row
  c.X0 = (r % tiles_x) * (TW - 2);    // first padded column of the input region
  return c;
}

__global__ void __launch_bounds__(NTHR, 1)
    conv3x3_tc_kernel(const __grid_constant__ CUtensorMap mAh, const __grid_constant__ CUtensorMap mAl,
                      const __grid_constant__ CUtensorMap mInh, ConvTcArgs a) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  // keep the pointer derived from the __shared__ array (shared-space loads/stores, not generic)
  uint8_t* sm = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u);
  uint8_t* Ah = sm;
  uint8_t* Al = Ah + A_BYTES;
  uint8_t* Bs = Al + A_BYTES;                                  // NSTAGE x (hi | lo)
  float* sx = reinterpret_cast<float*>(Bs + NSTAGE * B_STAGE); // [3][32][33]
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sx) + SX_BYTES);
  uint64_t* a_full = bars;
  uint64_t* b_full = bars + 1;      // [NSTAGE]
  uint64_t* b_empty = bars + 3;     // [NSTAGE]
  uint64_t* t_full = bars + 5;      // [2]
  uint64_t* t_empty = bars + 7;     // [2]
  uint64_t* b_conv = bars + 9;      // [NSTAGE] lo part formed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 11);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n, Wp = n + 2;
  const int tiles_x = ceil_div(n, TW - 2), tiles_y = ceil_div(n, TR);
  const int ntiles = a.nrhs * tiles_x * tiles_y;

  if (tid == 0) {
    mb_init(a_full, 1);
    for (int s = 0; s < NSTAGE; ++s) { mb_init(&b_full[s], 1); mb_init(&b_empty[s], 1); mb_init(&b_conv[s], 2); }
    for (int s = 0; s < 2; ++s) { mb_init(&t_full[s], 1); mb_init(&t_empty[s], 4 * NGRP); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {   // ------------------------------------------------ producer
      mb_expect(a_full, 2 * A_BYTES);
      for (int blk = 0; blk < 3 * NCH; ++blk) {
        tma2d(Ah + blk * A_BLK, &mAh, a_full, 0, blk * AM);
        tma2d(Al + blk * A_BLK, &mAl, a_full, 0, blk * AM);
      }
      int it = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileCoord tc = tile_coord(t, tiles_y, tiles_x);
        const int row0 = tc.b * Wp + tc.y0;          // padded row of the region start (= y0 + 1 - 1)
        for (int ch = 0; ch < NCH; ++ch, ++it) {
          const int s = it % NSTAGE;
          const uint32_t ph = (uint32_t)(it / NSTAGE) & 1u;
          mb_wait(&b_empty[s], ph ^ 1u);
          uint8_t* st = Bs + s * B_STAGE;
          mb_expect(&b_full[s], B_HALF);
          tma3d(st, &mInh, &b_full[s], ch * 16, tc.X0, row0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {   // ------------------------------------------------ MMA issuer
      mb_wait(a_full, 0);
      const uint32_t ah = su32(Ah), al = su32(Al), bs = su32(Bs);
      int it = 0, k = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
        const int ab = k & 1;
        mb_wait(&t_empty[ab], ((uint32_t)(k >> 1) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(ab * 256);
        for (int ch = 0; ch < NCH; ++ch, ++it) {
          const int s = it % NSTAGE;
          mb_wait(&b_conv[s], (uint32_t)(it / NSTAGE) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t bh = bs + s * B_STAGE, bl = bh + B_HALF;
#pragma unroll
          for (int t2 = 0; t2 < 3; ++t2) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t aoff = (uint32_t)((t2 * NCH + ch) * A_BLK + ks * 32);
              const uint32_t boff = (uint32_t)(t2 * TW * 64 + ks * 32);
              const uint64_t dah = desc_sw64(ah + aoff), dal = desc_sw64(al + aoff);
              const uint64_t dbh = desc_sw64(bh + boff), dbl = desc_sw64(bl + boff);
              const uint32_t first = (ch == 0 && t2 == 0 && ks == 0) ? 0u : 1u;
              mma_tf32(d, dah, dbh, first);
              mma_tf32(d, dah, dbl, 1u);
              mma_tf32(d, dal, dbh, 1u);
            }
          }
          mma_commit(&b_empty[s]);
        }
        mma_commit(&t_full[ab]);
      }
    }
    __syncwarp();
  } else if (warp == 6 || warp == 7) {  // --------------------------------- lo converters
    const int ct = tid - 192;         // 0..63
    int it = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
      for (int ch = 0; ch < NCH; ++ch, ++it) {
        const int s = it % NSTAGE;
        mb_wait(&b_full[s], (uint32_t)(it / NSTAGE) & 1u);
        const float4* hi = reinterpret_cast<const float4*>(Bs + s * B_STAGE);
        float4* lo = reinterpret_cast<float4*>(Bs + s * B_STAGE + B_HALF);
#pragma unroll 4
        for (int i = ct; i < B_HALF / 16; i += 64) {
          const float4 v = hi[i];
          float4 r;
          r.x = v.x - __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
          r.y = v.y - __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
          r.z = v.z - __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
          r.w = v.w - __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
          lo[i] = r;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mb_arrive(&b_conv[s]);
      }
    }
  } else {               // ------------------------------------------------ epilogue (warps 2-5, 8-11)
    const int q = warp & 3;            // TMEM lane quarter this warp may access: t1 = q (q = 3: padding)
    const int grp = warp < 8 ? 0 : (warp < 12 ? 1 : 2);   // group g handles tile rows g, g + NGRP, ...
    static_assert(NTHR == 64 + 64 + NGRP * 128, "warp roles: producer, MMA, 2 converters, NGRP x 4 epilogue");
    const int o = lane;                // output channel handled in the combine phase
    const int xw = (warp - (grp == 0 ? 2 : (grp == 1 ? 8 : 12))) & 3;   // combine: columns 1 + xw + 4 k
    float* sxg = sx + grp * 3 * 32 * 33;
    const float bias = __ldg(a.bias + o);
    int k = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++k) {
      const int ab = k & 1;
      const TileCoord tc = tile_coord(t, tiles_y, tiles_x);
      mb_wait(&t_full[ab], (uint32_t)(k >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      for (int r = grp; r < TR; r += NGRP) {
        uint32_t v[32];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(ab * 256 + r * TW);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
              "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]),
              "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]),
              "=r"(v[30]), "=r"(v[31])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        if (q < 3) {
          float* dst = sxg + (q * 32 + lane) * 33;     // [t1][o][xx]
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[j] = __uint_as_float(v[j]);
        }
        asm volatile("bar.sync %0, 128;\n" ::"r"(1 + grp) : "memory");
        const int y = tc.y0 + r;
        if (y < n) {
          const int64_t rowoff = ((int64_t)tc.b * Wp + (y + 1)) * Wp;
          const float* d0 = sxg + o * 33;
          const float* d1 = sxg + (32 + o) * 33;
          const float* d2 = sxg + (64 + o) * 33;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int xx = 1 + xw + 4 * kk;
            const int X = tc.X0 + xx;                   // padded column = image x + 1
            if (xx < TW - 1 && X <= n) {
              const float acc = d0[xx - 1] + d1[xx] + d2[xx + 1] + bias;
              a.out[(rowoff + X) * CC + o] = fmaxf(acc, 0.f);
            }
          }
        }
        asm volatile("bar.sync %0, 128;\n" ::"r"(1 + grp) : "memory");
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      if (lane == 0) mb_arrive(&t_empty[ab]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
  }
}

// ---------------------------------------------------------------- layer 1 (1 -> C), FFMA
// a1(y, x, c) = ReLU(b0[c] + sum_t w0[c][t] u(y + t2 - 1, x + t1 - 1)), u = b / ||b||, into the
// padded hi/lo tensors; border pixels of a1 and a2 (this level's layout) are set to zero.
__global__ void __launch_bounds__(256) conv_in_kernel(int n, const float* __restrict__ b,
                                                      const double* __restrict__ norms,
                                                      const float* __restrict__ w0, const float* __restrict__ b0,
                                                      float* __restrict__ o1, float* __restrict__ z2) {
  // CTA = 256 consecutive padded pixels of one RHS (blockIdx.y); thread = one pixel, all 32
  // channels into shared memory, then fully coalesced float4 stores of the 32 KB block.
  __shared__ float ws[CC * 9 + CC];
  __shared__ float4 tile[256 * (CC / 4) + 32];
  for (int i = threadIdx.x; i < CC * 10; i += blockDim.x) ws[i] = i < CC * 9 ? __ldg(w0 + i) : __ldg(b0 + i - CC * 9);
  __syncthreads();
  const int Wp = n + 2;
  const int per = Wp * Wp;
  const int rb = blockIdx.y;
  const int p0 = blockIdx.x * 256;
  const int p = p0 + threadIdx.x;
  const double s = norms ? norms[rb] : 1.0;
  const double inv = (s != 0.0) ? 1.0 / s : 0.0;
  const float* B = b + (int64_t)rb * n * n;
  float4* trow = tile + threadIdx.x * (CC / 4) + (threadIdx.x >> 3);   // +1 float4 per 8 rows: fewer conflicts
  if (p < per) {
    const int Y = p / Wp, X = p - Y * Wp;
    if (Y == 0 || X == 0 || Y == n + 1 || X == n + 1) {
#pragma unroll
      for (int g = 0; g < CC / 4; ++g) trow[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    } else {
      const int y = Y - 1, x = X - 1;
      float u[9];
#pragma unroll
      for (int t2 = 0; t2 < 3; ++t2)
#pragma unroll
        for (int t1 = 0; t1 < 3; ++t1) {
          const int yy = y + t2 - 1, xx = x + t1 - 1;
          u[t2 * 3 + t1] = (yy >= 0 && yy < n && xx >= 0 && xx < n) ? (float)((double)__ldg(B + yy * n + xx) * inv) : 0.f;
        }
#pragma unroll
      for (int g = 0; g < CC / 4; ++g) {
        float hv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int c = g * 4 + j;
          float acc = ws[CC * 9 + c];
#pragma unroll
          for (int t = 0; t < 9; ++t) acc = fmaf(ws[c * 9 + t], u[t], acc);
          hv[j] = fmaxf(acc, 0.f);
        }
        trow[g] = make_float4(hv[0], hv[1], hv[2], hv[3]);
      }
    }
  }
  __syncthreads();
  const int cnt = min(256, per - p0);
  float4* out = reinterpret_cast<float4*>(o1 + ((int64_t)rb * per + p0) * CC);
  for (int i = threadIdx.x; i < cnt * (CC / 4); i += 256) {
    const int px = i / (CC / 4), g = i - px * (CC / 4);
    out[i] = tile[px * (CC / 4) + (px >> 3) + g];
  }
  // zero border of the second activation tensor (this level's layout)
  if (p < per) {
    const int Y = p / Wp, X = p - Y * Wp;
    if (Y == 0 || X == 0 || Y == n + 1 || X == n + 1) {
      float4* q = reinterpret_cast<float4*>(z2 + ((int64_t)rb * per + p) * CC);
#pragma unroll
      for (int g = 0; g < CC / 4; ++g) q[g] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
  }
}

// ---------------------------------------------------------------- layer 4 (C -> 1), FFMA
// h(y, x) = s * (b3 + sum_{c,t} w3[c][t] a3(y + t2 - 1, x + t1 - 1, c)); 32 x 16 output tile per
// CTA (128 threads, 4 consecutive pixels each), input staged in two 16-channel halves.
constexpr int OW = 32, OH = 16, OPAD = 17;
__global__ void __launch_bounds__(128) conv_out_kernel(int n, const float* __restrict__ ih,
                                                       const double* __restrict__ norms, const float* __restrict__ w3,
                                                       const float* __restrict__ b3, float2* __restrict__ Z,
                                                       int zb0, float* __restrict__ x, int accumulate) {
  __shared__ float tile[(OH + 2) * (OW + 2) * OPAD];
  __shared__ float ws[CC * 9];
  const int tiles_x = ceil_div(n, OW);
  const int ty0 = (blockIdx.x / tiles_x) * OH, tx0 = (blockIdx.x % tiles_x) * OW;
  const int rb = blockIdx.y;
  const int Wp = n + 2;
  for (int i = threadIdx.x; i < CC * 9; i += 128) ws[i] = __ldg(w3 + i);
  const int ly = threadIdx.x >> 3, lx = (threadIdx.x & 7) * 4;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int half = 0; half < 2; ++half) {
    __syncthreads();
    // region padded rows ty0 .. ty0+17, padded cols tx0 .. tx0+33, channels half*16 .. +15
    for (int i = threadIdx.x; i < (OH + 2) * (OW + 2) * 4; i += 128) {
      const int c4 = i & 3, p = i >> 2;
      const int ry = p / (OW + 2), rx = p % (OW + 2);
      const int Y = ty0 + ry, X = tx0 + rx;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (Y < Wp && X < Wp) {
        const int64_t off = (((int64_t)rb * Wp + Y) * Wp + X) * CC + half * 16 + c4 * 4;
        v = *reinterpret_cast<const float4*>(ih + off);
      }
      float* d = tile + p * OPAD + c4 * 4;
      d[0] = v.x; d[1] = v.y; d[2] = v.z; d[3] = v.w;
    }
    __syncthreads();
    for (int cc = 0; cc < 16; ++cc) {
      const int c = half * 16 + cc;
#pragma unroll
      for (int t2 = 0; t2 < 3; ++t2) {
        float win[6];
#pragma unroll
        for (int j = 0; j < 6; ++j) win[j] = tile[((ly + t2) * (OW + 2) + lx + j) * OPAD + cc];
#pragma unroll
        for (int t1 = 0; t1 < 3; ++t1) {
          const float w = ws[c * 9 + t2 * 3 + t1];
#pragma unroll
          for (int p = 0; p < 4; ++p) acc[p] = fmaf(w, win[p + t1], acc[p]);
        }
      }
    }
  }
  const int y = ty0 + ly;
  if (y >= n) return;
  const double s = norms ? norms[rb] : 1.0;
  const float b = __ldg(b3);
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int xx = tx0 + lx + p;
    if (xx >= n) continue;
    const float nv = (s == 0.0) ? 0.f : acc[p] + b;    // N(u); the filter path scales by s after F'
    const int64_t o = ((int64_t)rb * n + y) * n + xx;
    if (Z) zput(Z, (int64_t)n * n, zb0 + rb, (int64_t)y * n + xx, nv);
    else x[o] = accumulate ? x[o] + nv * (float)s : nv * (float)s;
  }
}

__global__ void zero_border_kernel(int n, int nrhs, int C, float* __restrict__ buf) {
  const int Wp = n + 2;
  const int per = 4 * (n + 1);                  // border pixels per padded image
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t total = (int64_t)nrhs * per * C;
  if (idx >= total) return;
  const int c = (int)(idx % C);
  const int64_t pix = idx / C;
  const int rb = (int)(pix / per);
  int k = (int)(pix - (int64_t)rb * per);
  int Y, X;
  if (k < Wp) { Y = 0; X = k; }
  else if ((k -= Wp) < Wp) { Y = n + 1; X = k; }
  else if ((k -= Wp) < n) { Y = k + 1; X = 0; }
  else { k -= n; Y = k + 1; X = n + 1; }
  buf[(((int64_t)rb * Wp + Y) * Wp + X) * C + c] = 0.f;
}

}  // namespace

void zero_border(int n, int nrhs, int C, float* buf, cudaStream_t s) {
  const int64_t total = (int64_t)nrhs * 4 * (n + 1) * C;
  zero_border_kernel<<<(int)ceil_div64(total, 256), 256, 0, s>>>(n, nrhs, C, buf);
}

int conv_tc_smem() { return CONV_SMEM; }

void conv3x3_tc(const CUtensorMap* ah, const CUtensorMap* al, const CUtensorMap* in, const ConvTcArgs& a,
                int num_sms, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(conv3x3_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, CONV_SMEM);
    attr = true;
  }
  const int tiles = a.nrhs * ceil_div(a.n, TW - 2) * ceil_div(a.n, TR);
  const int grid = std::min(tiles, num_sms);
  conv3x3_tc_kernel<<<grid, NTHR, CONV_SMEM, s>>>(*ah, *al, *in, a);
}

void conv_in(int n, int nrhs, const float* b, const double* norms, const float* w0, const float* b0, float* o1,
             float* z2, cudaStream_t s) {
  dim3 grid(ceil_div((n + 2) * (n + 2), 256), nrhs);
  conv_in_kernel<<<grid, 256, 0, s>>>(n, b, norms, w0, b0, o1, z2);
}

void conv_out(int n, int nrhs, const float* in, const double* norms, const float* w3, const float* b3, float2* Z,
              int zb0, float* x, bool accumulate, cudaStream_t s) {
  dim3 grid(ceil_div(n, OW) * ceil_div(n, OH), nrhs);
  conv_out_kernel<<<grid, 128, 0, s>>>(n, in, norms, w3, b3, Z, zb0, x, accumulate ? 1 : 0);
}

}  // namespace nmg
