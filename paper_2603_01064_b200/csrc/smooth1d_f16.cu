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
// a1 by the stacked [W_hi; W_lo] weights and one N = 16 MMA multiplies the lo part by W_hi,
// so the A tile is read from shared memory twice per tap instead of three times
// (D[:, 0:16] = Ah Wh + Al Wh, D[:, 16:32] = Ah Wl; the epilogue adds the halves).
// Layer 3 (16 -> 1, k = 5) is split per tap in the epilogue: q_t(p) = sum_c w2[c][t] a2[c](p),
// written to a 512-position ring, and h(p) = b2 + sum_t q_t(p + t - 2) is assembled after the
// next barrier (positions outside [0, n) read zeros) -- no layer-2 halo is recomputed.
//
// Warps: 0-3 epilogue (TMEM lanes = positions), 4-7 layer-1 producer, 8 MMA issuer; the
// norm, filter and update phases use all 288 threads.  Two CTAs per SM overlap the serial
// phases of one right-hand side with the tile pipeline of another.
#include <cuda_fp16.h>

#include <algorithm>

#include "common.cuh"
#include "fft.cuh"
#include "kernels.h"

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
constexpr int UPAD = 4;
constexpr int QR = 512;                 // q ring (positions)
constexpr uint32_t IDESC32 = (1u << 4) | ((uint32_t)(32 >> 3) << 17) | ((uint32_t)(TP >> 4) << 24);
constexpr uint32_t IDESC16 = (1u << 4) | ((uint32_t)(16 >> 3) << 17) | ((uint32_t)(TP >> 4) << 24);

NMG_D uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
NMG_D void mb_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c));
}
NMG_D void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
NMG_D void mb_wait(uint64_t* b, uint32_t ph) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
NMG_D uint64_t desc_ns(uint32_t saddr, uint32_t lbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)(128 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
NMG_D void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
NMG_D void mma_commit(uint64_t* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(b))
               : "memory");
}
NMG_D void tld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
// wait::ld with the 32 destination registers threaded through in two groups of 16
NMG_D void tld_wait16(uint32_t* r) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]), "+r"(r[15])
               :
               : "memory");
}
NMG_D void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const __half2 hv = __floats2half2_rn(v[2 * j], v[2 * j + 1]);
    const __half2 lv = __floats2half2_rn(v[2 * j] - __low2float(hv), v[2 * j + 1] - __high2float(hv));
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

__global__ void __launch_bounds__(NT, 3) smooth1d_f16_kernel(Smooth1dArgs a) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u);
  const int n = a.n, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rhs = blockIdx.x;
  uint8_t* Abuf = sm;                                          // [2 stages][hi | lo] ABYTES each
  uint8_t* Bw = Abuf + 4 * ABYTES;                             // [5 taps][2][32][8] f16
  float* par = reinterpret_cast<float*>(Bw + KS * BTAP);       // w0 [c][5], b0, b1, w2t [t][c], b2
  float* w0 = par;
  float* b0 = w0 + C * KS;
  float* b1 = b0 + C;
  float* w2t = b1 + C;
  float* b2 = w2t + KS * C;
  float* qs = par + 256;                                       // [5][QR]
  float* u = qs + KS * QR;                                     // n + 2 UPAD
  float* hb = u + n + 2 * UPAD;                                // n (filter buffer)
  uint64_t* bars = reinterpret_cast<uint64_t*>(hb + n);        // afull[2] aempty[2] dfull[2] dempty[2]
  uint64_t* afull = bars;
  uint64_t* aempty = bars + 2;
  uint64_t* dfull = bars + 4;
  uint64_t* dempty = bars + 6;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
  __shared__ double red[32];

  // ---------------------------------------------------------------- setup (all threads)
  {
    const uint4* g = reinterpret_cast<const uint4*>(a.wb);
    uint4* d = reinterpret_cast<uint4*>(Bw);
    for (int i = tid; i < KS * BTAP / 16; i += NT) d[i] = __ldg(g + i);
    const float* P = a.params;   // w0 [16][1][5], b0 [16], w1 [16][16][5], b1 [16], w2 [1][16][5], b2
    for (int i = tid; i < C * KS + C; i += NT) w0[i] = __ldg(P + i);
    for (int i = tid; i < C; i += NT) b1[i] = __ldg(P + C * KS + C + C * C * KS + i);
    for (int i = tid; i < KS * C; i += NT) {
      const int t = i / C, c = i - t * C;
      w2t[i] = __ldg(P + C * KS + C + C * C * KS + C + c * KS + t);
    }
    if (tid == 0) b2[0] = __ldg(P + C * KS + C + C * C * KS + C + C * KS);
  }
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      mb_init(&afull[s], 4); mb_init(&aempty[s], 1); mb_init(&dfull[s], 1); mb_init(&dempty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)), "r"(64));
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
  if (a.normalize) s = sqrt(block_sum_f64(ss, red));   // block-wide, ends with all threads holding s
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
    const float inv = (float)(1.0 / s);
    const float sf = (float)s;
    const int ntile = n / TP;
    if (warp >= 4 && warp < 8) {
      // ---------------------------------------------------------- layer-1 producer
      const int pt = tid - 128;                 // 0..127
      const int half = pt >> 6;                 // channels 8 half .. 8 half + 7
      const int r0 = pt & 63;                   // rows r0, r0 + 64, r0 + 128 (< AR)
      // weights with u = b / s and the f16 scale S1 folded in (ReLU(S z) = S ReLU(z), S > 0)
      const float sc = a.in_scale;
      float wr[8][KS], br[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        br[j] = b0[8 * half + j] * sc;
#pragma unroll
        for (int t = 0; t < KS; ++t) wr[j][t] = w0[(8 * half + j) * KS + t] * (inv * sc);
      }
      for (int k = 0; k < ntile; ++k) {
        const int st = k & 1;
        mb_wait(&aempty[st], ((uint32_t)(k >> 1) & 1u) ^ 1u);
        uint4* ah = reinterpret_cast<uint4*>(Abuf + (2 * st) * ABYTES) + half * AR;
        uint4* al = reinterpret_cast<uint4*>(Abuf + (2 * st + 1) * ABYTES) + half * AR;
        const int Q0 = k * TP;
        for (int r = r0; r < AR; r += 64) {
          const int p = Q0 - 2 + r;             // a1 position of buffer row r
          float v[8];
          if (r < TP + 4 && p >= 0 && p < n) {
            const float* up = u + UPAD + p - 2;
            const float x0 = up[0], x1 = up[1], x2 = up[2], x3 = up[3], x4 = up[4];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float acc = br[j];
              acc = fmaf(wr[j][0], x0, acc);
              acc = fmaf(wr[j][1], x1, acc);
              acc = fmaf(wr[j][2], x2, acc);
              acc = fmaf(wr[j][3], x3, acc);
              acc = fmaf(wr[j][4], x4, acc);
              v[j] = fmaxf(acc, 0.f);
            }
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = 0.f;
          }
          uint4 hi, lo;
          split8(v, hi, lo);
          ah[r] = hi;
          al[r] = lo;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mb_arrive(&afull[st]);
      }
    } else if (warp == 8) {
      // ---------------------------------------------------------- MMA issuer
      if (lane == 0) {
        const uint32_t ab = su32(Abuf), bb = su32(Bw);
        for (int k = 0; k < ntile; ++k) {
          const int st = k & 1;
          mb_wait(&afull[st], (uint32_t)(k >> 1) & 1u);
          mb_wait(&dempty[st], ((uint32_t)(k >> 1) & 1u) ^ 1u);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t d = tmem + (uint32_t)(st * 32);
          const uint32_t ah = ab + (2 * st) * ABYTES, al = ah + ABYTES;
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            const uint64_t db = desc_ns(bb + t * BTAP, BLBO);
            mma_f16(d, desc_ns(ah + 16 * t, ALBO), db, IDESC32, t > 0 ? 1u : 0u);
            mma_f16(d, desc_ns(al + 16 * t, ALBO), db, IDESC16, 1u);
          }
          mma_commit(&aempty[st]);
          mma_commit(&dfull[st]);
        }
      }
      __syncwarp();
    } else if (warp < 4) {
      // ---------------------------------------------------------- epilogue: layer 3 per tap
      const int m = tid;                        // TMEM lane = position within the tile
      const float dsc = a.d_scale;
      const float b2v = b2[0];
      if (m < 2) {
#pragma unroll
        for (int t = 0; t < KS; ++t) qs[t * QR + ((QR - 2 + m) & (QR - 1))] = 0.f;   // positions -2, -1
      }
      auto emit = [&](int p, float hv) {
        if (a.filter) {
          hb[p] = hv;
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
      for (int k = 0; k < ntile; ++k) {
        const int st = k & 1;
        mb_wait(&dfull[st], (uint32_t)(k >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        uint32_t d[32];
        tld32(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(st * 32), d);
        tld_wait16(d);
        tld_wait16(d + 16);
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mb_arrive(&dempty[st]);
        float q[KS];
#pragma unroll
        for (int t = 0; t < KS; ++t) q[t] = 0.f;
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const float a2 = fmaxf(fmaf(__uint_as_float(d[c]) + __uint_as_float(d[16 + c]), dsc, b1[c]), 0.f);
#pragma unroll
          for (int t = 0; t < KS; ++t) q[t] = fmaf(w2t[t * C + c], a2, q[t]);
        }
        const int Q0 = k * TP;
#pragma unroll
        for (int t = 0; t < KS; ++t) qs[t * QR + ((Q0 + m) & (QR - 1))] = q[t];
        asm volatile("bar.sync 1, 128;\n" ::: "memory");
        const int p = Q0 - 2 + m;
        if (p >= 0) assemble(p);
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
    if (a.filter) {
      // ---- level filter F'_l on the whole row (real-input FFT packing, see fft.cuh)
      real_level_filter(hb, n, a.twiddle, a.tw_n, tid, NT);
      const float scale = 2.0f / (float)n;   // 1/(n/2) of the half-length inverse
      float mx = 0.f;
      for (int j = tid; j < n; j += NT) {
        const float v = hb[j] * scale;
        const float xv = a.accumulate ? xrow[j] + v : v;
        xrow[j] = xv;
        if (a.xh) tf32_store(xv, a.xh, a.xl, (int64_t)rhs * a.ldx + j);
        if (a.x16h) { hb[j] = xv; mx = fmaxf(mx, fabsf(xv)); }
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
          const float v = hb[j] * S;
          const __half hv = __float2half_rn(v);
          oh[j] = hv;
          ol[j] = __float2half_rn(v - __half2float(hv));
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 8) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(64));
}

}  // namespace

size_t smooth1d_f16_smem(int n) {
  return 1024 + 4 * ABYTES + KS * BTAP + sizeof(float) * (256 + KS * QR + n + 2 * UPAD + n) + 8 * 8 + 16;
}

void smooth1d_f16(const Smooth1dArgs& a, cudaStream_t s) {
  static size_t attr = 0;
  const size_t smem = smooth1d_f16_smem(a.n);
  if (smem > attr) {
    cudaFuncSetAttribute(smooth1d_f16_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smooth1d_f16_smem(8192));
    attr = smooth1d_f16_smem(8192);
  }
  smooth1d_f16_kernel<<<a.nrhs, NT, smem, s>>>(a);
}

}  // namespace nmg
