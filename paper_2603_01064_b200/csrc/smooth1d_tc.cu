// Fused 1D neural smoothing step with the CNN's 16 -> 16 layer on the tensor cores
// (Alg 3; CNN per reading R7), one CTA per right-hand side:
//   s = ||b||_2 (fp64) -> layer 1 (1 -> 16, FFMA) -> layer 2 (16 -> 16, tcgen05 3xTF32)
//   -> layer 3 (16 -> 1, FFMA) -> h = s N(b/s) -> F'_l(h) (real-input FFT) -> x update.
//
// Layer 2 as a GEMM with positions in M:  a2[p][o] = b1[o] + sum_{t, c} a1[p + t][c] W[o][c][t]
//   M = 128 positions (two blocks per 256-wide tile), N = 16 output channels, K = 5 taps x 16.
// a1 is stored K-major without swizzle in "channel-quad planes" [c/4][position][4] (16 B per
// position, 8-position core groups 128 B apart), so the tap shift t is a +16 t byte offset of
// the A-descriptor start address; no im2col buffer is built.
#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"

#include <algorithm>

namespace nmg {
namespace {

constexpr int C = 16, KS = 5, HALO = KS / 2;
constexpr int NT = 256;
constexpr int T3 = 252;                 // h outputs per tile
constexpr int W2 = T3 + 2 * HALO;       // 256 layer-2 positions = 2 MMA M-blocks
constexpr int W1 = W2 + 2 * HALO;       // 260 layer-1 positions
constexpr int A1P = 264;                // positions per channel-quad plane (>= W1 + slack)
constexpr int S2 = W2 + 4;              // layer-2 output row stride (floats)
constexpr int NPARAM = C * KS + C + C * C * KS + C + C * KS + 1;   // 1473
constexpr int UPAD = 3 * HALO;
constexpr int Q3 = T3 / 4;
constexpr int BW = KS * (C / 4) * C * 4;  // weight B operand per hi/lo: [t][c/4][o][4] = 1280 floats

NMG_D uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// SWIZZLE_NONE K-major descriptor: 8-row core groups SBO = 128 B apart, K-quads LBO apart.
NMG_D uint64_t desc_none(uint32_t saddr, uint32_t lbo_bytes) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;                                  // layout type 0 = SWIZZLE_NONE
}
// D f32, A/B tf32, K-major, N = 16, M = 128
constexpr uint32_t kIdesc1d = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(16 >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);

NMG_D void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(kIdesc1d), "r"(acc));
}
NMG_D void tf32_split(float v, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(v));
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(l) : "f"(v - __uint_as_float(h)));
  hi = __uint_as_float(h);
  lo = __uint_as_float(l);
}
NMG_D void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(su32(b)),
      "r"(ph));
}

__global__ void __launch_bounds__(NT, 2) smooth1d_tc_kernel(Smooth1dArgs a) {
  extern __shared__ __align__(16) float sm[];
  const int n = a.n, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rhs = blockIdx.x;
  float* w = sm;                                        // params (1480)
  float* u = w + 1480;                                  // n + 2 UPAD
  float* hb = u + ((n + 2 * UPAD + 3) & ~3);            // h row / filter buffer
  float* a1h = hb + ((n + 3) & ~3);                     // [4][A1P][4]
  float* a1l = a1h + 4 * A1P * 4;
  float* a2 = a1l + 4 * A1P * 4;                        // [16][S2]
  float* bwh = a2 + C * S2;                             // [5][4][16][4]
  float* bwl = bwh + BW;
  uint64_t* mbar = reinterpret_cast<uint64_t*>(bwl + BW);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(mbar + 1);
  __shared__ double red[32];

  const float* w0 = w;
  const float* b0 = w0 + C * KS;
  const float* b1 = b0 + C + C * C * KS;
  const float* w2 = b1 + C;
  const float* b2 = w2 + C * KS;

  for (int i = tid; i < NPARAM; i += NT) w[i] = __ldg(a.params + i);
  // layer-2 weights as the B operand: B_t[o][c] = W[o][c][t], layout [t][c/4][o][4], tf32 hi / lo
  for (int i = tid; i < C * C * KS; i += NT) {
    const int o = i / (C * KS), rem = i - o * C * KS, c = rem / KS, t = rem - c * KS;
    float hi, lo;
    tf32_split(__ldg(a.params + C * KS + C + i), hi, lo);
    const int off = ((t * (C / 4) + c / 4) * C + o) * 4 + (c & 3);
    bwh[off] = hi;
    bwl[off] = lo;
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(su32(mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  const float* brow = a.b + (int64_t)rhs * a.ldb;
  double ss = 0.0;
  for (int j = tid; j < n; j += NT) {
    const float v = brow[j];
    u[UPAD + j] = v;
    ss += (double)v * (double)v;
  }
  if (tid < UPAD) { u[tid] = 0.f; u[UPAD + n + tid] = 0.f; }
  double s = 1.0;
  bool zero = false;
  if (a.normalize) {
    s = sqrt(block_sum_f64(ss, red));
    zero = (s == 0.0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;
  if (zero) {                                   // ||b|| = 0 => h = 0 (reading R10)
    float* xrow = a.x + (int64_t)rhs * a.ldx;
    for (int j = tid; j < n; j += NT) {
      const float xv = a.accumulate ? xrow[j] : 0.f;
      xrow[j] = xv;
      if (a.xh) {
        float hi, lo;
        tf32_split(xv, hi, lo);
        a.xh[(int64_t)rhs * a.ldx + j] = hi;
        a.xl[(int64_t)rhs * a.ldx + j] = lo;
      }
    }
  } else {
    if (a.normalize) {
      for (int j = tid; j < n; j += NT) u[UPAD + j] = (float)((double)u[UPAD + j] / s);
    }
    const float sf = (float)s;
    // layer-1 role: channel quad cq = tid & 3, positions j = (tid >> 2) + 64 k
    const int cq = tid & 3, pj = tid >> 2;
    // layer-3 role
    const int q3 = tid >> 2, cg = tid & 3;
    // layer-2 epilogue role: TMEM lane quarter q = warp & 3, M-block mb = warp >> 2
    const int q = warp & 3, mb = warp >> 2;
    uint32_t phase = 0;
    __syncthreads();
    for (int t0 = 0; t0 < n; t0 += T3) {
      // ---- layer 1 -> a1 (hi / lo) in channel-quad planes; position p = t0 - 4 + j
      for (int j = pj; j < W1; j += NT / 4) {
        const int p = t0 - 2 * HALO + j;
        float r[4] = {0.f, 0.f, 0.f, 0.f};
        if (p >= 0 && p < n) {
          float uw[KS];
#pragma unroll
          for (int t = 0; t < KS; ++t) uw[t] = u[UPAD + p + t - HALO];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int c = cq * 4 + k;
            float acc = b0[c];
#pragma unroll
            for (int t = 0; t < KS; ++t) acc = fmaf(w0[c * KS + t], uw[t], acc);
            r[k] = fmaxf(acc, 0.f);
          }
        }
        float4 hv, lv;
        tf32_split(r[0], hv.x, lv.x); tf32_split(r[1], hv.y, lv.y);
        tf32_split(r[2], hv.z, lv.z); tf32_split(r[3], hv.w, lv.w);
        *reinterpret_cast<float4*>(a1h + (cq * A1P + j) * 4) = hv;
        *reinterpret_cast<float4*>(a1l + (cq * A1P + j) * 4) = lv;
      }
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncthreads();
      // ---- layer 2 on tcgen05: D[mb][m][o] = sum_{t,c} a1[128 mb + m + t][c] W[o][c][t]
      if (tid == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t ah = su32(a1h), al = su32(a1l), bh = su32(bwh), bl = su32(bwl);
        const uint32_t lboA = A1P * 16, lboB = C * 16;
#pragma unroll
        for (int blk = 0; blk < 2; ++blk) {
          const uint32_t d = tmem + (uint32_t)(blk * 16);
#pragma unroll
          for (int t = 0; t < KS; ++t) {
#pragma unroll
            for (int ks = 0; ks < 2; ++ks) {
              const uint32_t aoff = (uint32_t)((2 * ks) * A1P * 16 + (blk * 128 + t) * 16);
              const uint32_t boff = (uint32_t)((t * (C / 4) + 2 * ks) * C * 16);
              const uint64_t dah = desc_none(ah + aoff, lboA), dal = desc_none(al + aoff, lboA);
              const uint64_t dbh = desc_none(bh + boff, lboB), dbl = desc_none(bl + boff, lboB);
              mma_tf32(d, dah, dbh, (t | ks) ? 1u : 0u);
              mma_tf32(d, dah, dbl, 1u);
              mma_tf32(d, dal, dbh, 1u);
            }
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         su32(mbar))
                     : "memory");
      }
      mb_wait(mbar, phase);
      phase ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(mb * 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
        const int m = mb * 128 + q * 32 + lane;         // layer-2 local position, p = t0 - 2 + m
        const int p = t0 - HALO + m;
        const bool inside = p >= 0 && p < n;
#pragma unroll
        for (int o = 0; o < C; ++o) a2[o * S2 + m] = inside ? fmaxf(__uint_as_float(v[o]) + b1[o], 0.f) : 0.f;
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncthreads();
      // ---- layer 3: h[p], p = t0 + 4 q3 + k
      {
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int cc = 0; cc < C / 4; ++cc) {
          const int c = cg * (C / 4) + cc;
          const float4* src = reinterpret_cast<const float4*>(a2 + c * S2 + 4 * q3);
          const float4 v0 = src[0], v1 = src[1];
          const float win[8] = {v0.x, v0.y, v0.z, v0.w, v1.x, v1.y, v1.z, v1.w};
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const float wv = w2[c * KS + t];
#pragma unroll
            for (int k = 0; k < 4; ++k) acc[k] = fmaf(wv, win[k + t], acc[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], 1);
          acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], 2);
        }
        if (cg == 0 && q3 < Q3) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int p = t0 + 4 * q3 + k;
            if (p < n) {
              const float hv = (acc[k] + b2[0]) * sf;
              if (a.filter) {
                hb[p] = hv;
              } else {
                float* xrow = a.x + (int64_t)rhs * a.ldx;
                const float xv = a.accumulate ? xrow[p] + hv : hv;
                xrow[p] = xv;
                if (a.xh) {
                  float hi, lo;
                  tf32_split(xv, hi, lo);
                  a.xh[(int64_t)rhs * a.ldx + p] = hi;
                  a.xl[(int64_t)rhs * a.ldx + p] = lo;
                }
              }
            }
          }
        }
      }
      __syncthreads();
    }
    if (a.filter) {
      real_level_filter(hb, n, a.twiddle, a.tw_n, tid, NT);
      const float scale = 2.0f / (float)n;
      float* xrow = a.x + (int64_t)rhs * a.ldx;
      for (int j = tid; j < n; j += NT) {
        const float v = hb[j] * scale;
        const float xv = a.accumulate ? xrow[j] + v : v;
        xrow[j] = xv;
        if (a.xh) {
          float hi, lo;
          tf32_split(xv, hi, lo);
          a.xh[(int64_t)rhs * a.ldx + j] = hi;
          a.xl[(int64_t)rhs * a.ldx + j] = lo;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tmem));
}

}  // namespace

size_t smooth1d_tc_smem(int n) {
  const size_t f = 1480 + ((n + 2 * UPAD + 3) & ~3) + ((n + 3) & ~3) + 2 * 4 * A1P * 4 + C * S2 + 2 * BW;
  return f * sizeof(float) + 16 + 16;
}

void smooth1d_tc(const Smooth1dArgs& a, cudaStream_t s) {
  const size_t smem = smooth1d_tc_smem(a.n);
  static size_t attr = 0;
  if (smem > attr) {
    const size_t mx = smooth1d_tc_smem(8192);
    cudaFuncSetAttribute(smooth1d_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx);
    attr = mx;
  }
  smooth1d_tc_kernel<<<a.nrhs, NT, smem, s>>>(a);
}

}  // namespace nmg
