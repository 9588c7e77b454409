// 2D Kronecker operator apply on the 5th-gen tensor cores (3xTF32, fp32-accurate):
//   A_l X = Mat(hat A_l Vec X) = C_l X B_l^T + alpha Q_l X Q_l^T
// on the row-major [i2][i1] image arrays (arr = X^T) as two GEMM passes over all RHS at once:
//   pass 1 (KRON_T)    : T = blockT(arr C^T)                    (M = nrhs * n rows, K = n)
//   pass 2 (KRON_RESID): D = Cin -/+ (blockT(T B^T) + alpha Q arr Q^T)
// blockT = transposed store within each n x n image, so pass 2 again contracts along rows.
// The banded mass term (Q_l has half-bandwidth <= 2, Q_0 = I) and the residual are computed
// in pass 2's epilogue, so one residual costs 24 B/pixel of HBM traffic: pass 1 reads X and
// writes T (fp32), pass 2 reads T, X, Cin and writes D.
//
// Kernel anatomy (persistent, one CTA per SM, 320 threads):
//   warp 8 lane 0 : TMA producer — fp32 A tile (128 rows x 16 K) + W hi/lo tiles per stage
//   warps 4-7     : splitters — A tile -> tf32 hi (in place) + lo (hi = rna(a), lo = rna(a - hi))
//   warp 9 lane 0 : MMA issuer — 3 x tcgen05.mma.kind::tf32 per K=8 (hi*hi + hi*lo + lo*hi),
//                   accumulating into one of two TMEM buffers (tile i uses buffer i & 1)
//   warps 0-3     : epilogue — tcgen05.ld of the other buffer while the next tile's MMAs run
// The hi/lo split of A happens in shared memory, so neither X nor T is ever written split.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace nmg {
namespace {

constexpr int KBM = 128, KBK = 16;
constexpr int KNT = 320;
constexpr int A_BYTES = KBM * KBK * 4;   // 8 KB

template <int TBN> struct KronCfg {
  static constexpr int B_BYTES = TBN * KBK * 4;
  static constexpr int STAGE = 2 * A_BYTES + 2 * B_BYTES;        // A (hi in place), A lo, W hi, W lo
  static constexpr int STAGES = (200 * 1024 / STAGE) > 8 ? 8 : (200 * 1024 / STAGE);
  static constexpr int SMEM = STAGES * STAGE + 1024 /*barriers*/ + 1024 /*align*/;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TBN >> 3) << 17) |
                                    ((uint32_t)(KBM >> 4) << 24);   // D f32, A/B tf32 K-major, M = 128
  static constexpr uint32_t TCOLS = 2 * TBN < 32 ? 32 : 2 * TBN;
};

NMG_D float rna_tf32(float v) {
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(v));
  return __uint_as_float(h);
}

template <int TBN, int HB>
__global__ void __launch_bounds__(KNT, 1)
    kron_tc_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tWh,
                   const __grid_constant__ CUtensorMap tWl, KronArgs a) {
  using Cfg = KronCfg<TBN>;
  constexpr int ST = Cfg::STAGES, STAGE = Cfg::STAGE, B_BYTES = Cfg::B_BYTES;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ST * STAGE);
  uint64_t* split = full + ST;
  uint64_t* empty = split + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n = a.n;
  const int KT = n / KBK;
  // slab mode (R < n): pass 1 rows are the rank's halo'd image rows, pass 2 columns its slab
  const int R = a.R ? a.R : n;
  const int NT = ((a.mode == KRON_T ? n : R) + TBN - 1) / TBN;
  const int wrow0 = a.mode == KRON_T ? 0 : a.r0;
  const int MT = (a.M + KBM - 1) / KBM;
  const int T = MT * NT;
  // K blocks of output-column tile n0: outside the union of its 64-row W ranges every W hi/lo
  // value is zero, so those products are exact zeros (the producer, the splitters and the MMA
  // issuer all walk the same blocks)
  auto krange = [&](int n0, int& kb, int& ke) {
    kb = 0;
    ke = KT;
    if (!a.krange) return;
    int lo = n, hi = 0;
    for (int t = 0; t < TBN / 64 && n0 + 64 * t < (a.mode == KRON_T ? n : R); ++t) {
      const int2 r = __ldg(&a.krange[(wrow0 + n0) / 64 + t]);
      lo = min(lo, r.x);
      hi = max(hi, r.y);
    }
    if (hi <= lo) return;
    kb = lo / KBK;
    ke = max(kb + 1, min(KT, (hi + KBK - 1) / KBK));
  };

  if (tid == 0) {
    for (int s = 0; s < ST; ++s) { mb_init(&full[s], 1); mb_init(&split[s], 4); mb_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mb_init(&tfull[b], 1); mb_init(&tempty[b], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tA) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tWh) : "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(&tWl) : "memory");
  }
  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(Cfg::TCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 8) {
    if (lane == 0) {   // ---------------- TMA producer
      int it = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x) {
        const int m0 = (t / NT) * KBM, n0 = (t % NT) * TBN;
        int kb, ke;
        krange(n0, kb, ke);
        for (int kt = kb; kt < ke; ++kt, ++it) {
          const int s = it % ST;
          mb_wait(&empty[s], ((uint32_t)(it / ST) & 1u) ^ 1u);
          uint8_t* st = sm + s * STAGE;
          mb_expect(&full[s], A_BYTES + 2 * B_BYTES);
          tma2d(st, &tA, &full[s], kt * KBK, m0);
          tma2d(st + 2 * A_BYTES, &tWh, &full[s], kt * KBK, wrow0 + n0);
          tma2d(st + 2 * A_BYTES + B_BYTES, &tWl, &full[s], kt * KBK, wrow0 + n0);
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {   // ---------------- splitters
    const int ct = tid - 128;
    int it = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x) {
      int kb, ke;
      krange((t % NT) * TBN, kb, ke);
      for (int kt = kb; kt < ke; ++kt, ++it) {
        const int s = it % ST;
        mb_wait(&full[s], (uint32_t)(it / ST) & 1u);
        float4* hi = reinterpret_cast<float4*>(sm + s * STAGE);
        float4* lo = reinterpret_cast<float4*>(sm + s * STAGE + A_BYTES);
#pragma unroll
        for (int e = ct; e < A_BYTES / 16; e += 128) {
          const float4 v = hi[e];
          float4 h, l;
          h.x = rna_tf32(v.x); l.x = rna_tf32(v.x - h.x);
          h.y = rna_tf32(v.y); l.y = rna_tf32(v.y - h.y);
          h.z = rna_tf32(v.z); l.z = rna_tf32(v.z - h.z);
          h.w = rna_tf32(v.w); l.w = rna_tf32(v.w - h.w);
          hi[e] = h;
          lo[e] = l;
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mb_arrive(&split[s]);
      }
    }
  } else if (warp == 9) {
    if (lane == 0) {   // ---------------- MMA issuer
      int it = 0, i = 0;
      for (int t = blockIdx.x; t < T; t += gridDim.x, ++i) {
        const int ab = i & 1;
        mb_wait(&tempty[ab], ((uint32_t)(i >> 1) & 1u) ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d = tmem + (uint32_t)(ab * TBN);
        int kb, ke;
        krange((t % NT) * TBN, kb, ke);
        for (int kt = kb; kt < ke; ++kt, ++it) {
          const int s = it % ST;
          const uint32_t ph = (uint32_t)(it / ST) & 1u;
          mb_wait(&full[s], ph);
          mb_wait(&split[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t st = su32(sm + s * STAGE);
#pragma unroll
          for (int ks = 0; ks < 2; ++ks) {
            const uint32_t ko = ks * 32;   // 8 tf32 = 32 bytes along the 64-byte swizzled row
            const uint64_t dah = desc_sw64(st + ko), dal = desc_sw64(st + A_BYTES + ko);
            const uint64_t dwh = desc_sw64(st + 2 * A_BYTES + ko), dwl = desc_sw64(st + 2 * A_BYTES + B_BYTES + ko);
            mma_tf32(d, dah, dwh, Cfg::IDESC, (kt != kb || ks) ? 1u : 0u);
            mma_tf32(d, dah, dwl, Cfg::IDESC, 1u);
            mma_tf32(d, dal, dwh, Cfg::IDESC, 1u);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[ab]);
      }
    }
  } else {   // ---------------- epilogue, warps 0-3 (TMEM lanes 32 w .. 32 w + 31)
    const int64_t img = a.img ? a.img : (int64_t)n * n;   // per-image stride of X, Cin, D
    const int AH = R + 2 * a.H;                            // pass-1 A rows per image
    int i = 0;
    for (int t = blockIdx.x; t < T; t += gridDim.x, ++i) {
      const int ab = i & 1;
      const int m = (t / NT) * KBM + warp * 32 + lane, n0 = (t % NT) * TBN;
      // pass 1: image b, stored row e (slab row e - H; halo rows are not stored);
      // pass 2: image b, row r = i1 of the output
      const int b = a.mode == KRON_T ? m / AH : m / n;
      const int r = a.mode == KRON_T ? m - b * AH - a.H : m - b * n;
      const bool mok = m < a.M && (a.mode != KRON_T || (r >= 0 && r < R));
      const int64_t base = a.mode == KRON_T ? (int64_t)b * n * R + r : b * img + (int64_t)a.H * n + r;
      float q1[2 * HB + 1];
      if (a.mode == KRON_RESID && mok) {
#pragma unroll
        for (int d1 = -HB; d1 <= HB; ++d1) {
          const int a1 = r + d1;
          q1[d1 + HB] = (a1 >= 0 && a1 < n) ? __ldg(a.Q + (int64_t)r * n + a1) : 0.f;
        }
      }
      mb_wait(&tfull[ab], (uint32_t)(i >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t tb = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(ab * TBN);
      if (a.mode == KRON_RESID && HB <= 1) {
        // D = Cin -/+ (acc + alpha S), S[b][i2][i1] = sum_{a2} Q[i2][a2] (sum_{a1} Q[i1][a1] X[b][a2][a1])
        // (|a - i| <= HB; X rows addressed by their global index i2, the slab's halo holds i2 +- HB).
        // Per 16-column chunk: the horizontal pass over the rows i2 - HB .. i2 + 15 + HB, then the
        // vertical pass in registers.  Software-pipelined: the X / Cin loads of chunk c + 1 are in
        // flight while chunk c is combined with its accumulator columns and stored (one DRAM
        // latency per tile instead of one per chunk: the epilogue was latency-bound).  Every load
        // is unconditional (clamped address; out-of-range terms weighted by 0 or dropped by select).
        const float* Xb = a.X + b * img + (int64_t)(a.H - a.r0) * n;
        constexpr int NR = 16 + 2 * HB, NW = 2 * HB + 1;
        const int nch = (min(TBN, R - n0) + 15) / 16;
        float raw[NR][NW], cin[16];       // loads in flight (chunk c + 1)
        float hs[NR], cc[16];             // chunk c, horizontal pass done
        auto load = [&](int c) {
          const int nb = n0 + 16 * c;
#pragma unroll
          for (int k = 0; k < NR; ++k) {
            const float* xrow = Xb + (int64_t)min(max(a.r0 + nb - HB + k, 0), n - 1) * n;
#pragma unroll
            for (int d1 = -HB; d1 <= HB; ++d1) raw[k][d1 + HB] = __ldg(xrow + min(max(r + d1, 0), n - 1));
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) cin[j] = a.Cin ? a.Cin[base + (int64_t)min(nb + j, R - 1) * n] : 0.f;
        };
        auto horizontal = [&](int c) {
          const int nb = n0 + 16 * c;
#pragma unroll
          for (int k = 0; k < NR; ++k) {
            const int a2 = a.r0 + nb - HB + k;
            float t = 0.f;
#pragma unroll
            for (int d1 = -HB; d1 <= HB; ++d1) t = fmaf(q1[d1 + HB], raw[k][d1 + HB], t);
            hs[k] = (a2 >= 0 && a2 < n) ? t : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) cc[j] = cin[j];
        };
        if (mok && nch > 0) { load(0); horizontal(0); }
#pragma unroll 1
        for (int c = 0; c < nch; ++c) {
          if (mok && c + 1 < nch) load(c + 1);
          uint32_t v[16];
          tld16(tb + 16 * c, v);
          tld_wait16(v);
          if (mok) {
            const int nb = n0 + 16 * c;
            float o[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              // columns nb + j >= R are not stored (their clamped terms are never used)
              const int i2 = a.r0 + min(nb + j, R - 1);
              float sq = 0.f;
#pragma unroll
              for (int d2 = -HB; d2 <= HB; ++d2)
                sq = fmaf(__ldg(a.Q + (int64_t)i2 * n + min(max(i2 + d2, 0), n - 1)), hs[j + d2 + HB], sq);
              const float vv = fmaf(a.alpha, sq, __uint_as_float(v[j]));
              o[j] = a.negate ? cc[j] - vv : cc[j] + vv;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j)
              if (nb + j < R) a.D[base + (int64_t)(nb + j) * n] = o[j];
            if (c + 1 < nch) horizontal(c + 1);
          }
        }
      } else {
        // pass 1 (KRON_T), and pass 2 at HB = 2 (levels n <= 128: the pipelined registers would
        // spill there): one chunk at a time
  #pragma unroll 1
        for (int c = 0; c < TBN; c += 16) {
          uint32_t v[16];
          tld16(tb + c, v);
          tld_wait16(v);
          if (!mok) continue;
          const int nb = n0 + c;
          if (a.mode == KRON_T) {
  #pragma unroll
            for (int j = 0; j < 16; ++j)
              if (nb + j < n) a.D[base + (int64_t)(nb + j) * R] = __uint_as_float(v[j]);
          } else {
            // X rows addressed by their global index i2 (the slab's halo holds i2 +- hb).
            // Mass stencil S = Q X Q^T of the chunk: horizontal pass over the rows i2 - HB ..
            // i2 + 15 + HB, then the vertical pass in registers; every load is unconditional
            // (clamped address, out-of-range terms weighted by 0 or dropped by select), so the
            // loads of a chunk issue back to back instead of one dependent miss at a time.
            // S[b][i2][i1] = sum_{a2} Q[i2][a2] (sum_{a1} Q[i1][a1] X[b][a2][a1]), |a - i| <= HB.
            const float* Xb = a.X + b * img + (int64_t)(a.H - a.r0) * n;
            constexpr int NR = 16 + 2 * HB;
            float hs[NR];
  #pragma unroll
            for (int k = 0; k < NR; ++k) {
              const int a2 = a.r0 + nb - HB + k;
              const float* xrow = Xb + (int64_t)min(max(a2, 0), n - 1) * n;
              float t = 0.f;
  #pragma unroll
              for (int d1 = -HB; d1 <= HB; ++d1) t = fmaf(q1[d1 + HB], __ldg(xrow + min(max(r + d1, 0), n - 1)), t);
              hs[k] = (a2 >= 0 && a2 < n) ? t : 0.f;
            }
            float o[16];
  #pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int jj = min(nb + j, R - 1);
              const int i2 = a.r0 + jj;
              float sq = 0.f;
  #pragma unroll
              for (int d2 = -HB; d2 <= HB; ++d2)
                sq = fmaf(__ldg(a.Q + (int64_t)i2 * n + min(max(i2 + d2, 0), n - 1)), hs[jj - nb + d2 + HB], sq);
              const float vv = fmaf(a.alpha, sq, __uint_as_float(v[j]));
              const float cc = a.Cin ? a.Cin[base + (int64_t)jj * n] : 0.f;
              o[j] = a.negate ? cc - vv : cc + vv;
            }
  #pragma unroll
            for (int j = 0; j < 16; ++j)
              if (nb + j < R) a.D[base + (int64_t)(nb + j) * n] = o[j];
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mb_arrive(&tempty[ab]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 9) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(Cfg::TCOLS));
  }
}

template <int TBN, int HB>
void launch_kron(const CUtensorMap* A, const CUtensorMap* Wh, const CUtensorMap* Wl, const KronArgs& a, int sms,
                 cudaStream_t s) {
  NMG_SMEM_OPTIN((kron_tc_kernel<TBN, HB>), KronCfg<TBN>::SMEM);
  const int cols = a.mode == KRON_T ? a.n : (a.R ? a.R : a.n);
  const int tiles = ceil_div(a.M, KBM) * ceil_div(cols, TBN);
  kron_tc_kernel<TBN, HB><<<std::min(tiles, sms), KNT, KronCfg<TBN>::SMEM, s>>>(*A, *Wh, *Wl, a);
}

template <int TBN>
void launch_kron_hb(const CUtensorMap* A, const CUtensorMap* Wh, const CUtensorMap* Wl, const KronArgs& a, int sms,
                    cudaStream_t s) {
  switch (a.mode == KRON_T ? 0 : a.hb) {
    case 0: launch_kron<TBN, 0>(A, Wh, Wl, a, sms, s); break;
    case 1: launch_kron<TBN, 1>(A, Wh, Wl, a, sms, s); break;
    default: launch_kron<TBN, 2>(A, Wh, Wl, a, sms, s); break;
  }
}

}  // namespace

int kron_tile_n(int n) { return n >= 256 ? 256 : n; }

bool kron_supported(int n, int hb) {
  return n % 16 == 0 && n >= 32 && (n <= 256 || n % 256 == 0) && hb <= 2 && (n & (n - 1)) == 0;
}

void kron_tc(const CUtensorMap* A, const CUtensorMap* Wh, const CUtensorMap* Wl, const KronArgs& a, int sms,
             cudaStream_t s) {
  switch (kron_tile_n(a.mode == KRON_T ? a.n : (a.R ? a.R : a.n))) {
    case 32: launch_kron_hb<32>(A, Wh, Wl, a, sms, s); break;
    case 64: launch_kron_hb<64>(A, Wh, Wl, a, sms, s); break;
    case 128: launch_kron_hb<128>(A, Wh, Wl, a, sms, s); break;
    default: launch_kron_hb<256>(A, Wh, Wl, a, sms, s); break;
  }
}

}  // namespace nmg
