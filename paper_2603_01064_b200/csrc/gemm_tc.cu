// fp32-accurate operator apply on the 5th-gen tensor cores (tcgen05, kind::tf32):
//   D = C - X W^T   with  X = Xh + Xl,  W = Wh + Wl  (tf32 hi/lo splits, "3xTF32")
//   X W^T ~= Xh Wh^T + Xh Wl^T + Xl Wh^T, all three accumulated in one TMEM tile.
// This is the inner-cycle residual r_l = y_l - A^(l) x_l (Alg 3, Alg 1
// P:158) and the post-smoothing residual b = r_l - (A^(l) I_{l+1}^l) e.
//
// Kernel anatomy (one 128 x 256 output tile per CTA, 128 threads):
//   warp 0 / lane 0 : TMA producer (cp.async.bulk.tensor, SWIZZLE_64B, 4-stage ring)
//   warp 1 / lane 0 : MMA issuer (tcgen05.mma.cta_group::1.kind::tf32, M=128 N=256 K=8)
//   warp 2          : TMEM allocator (256 fp32 columns)
//   all 4 warps     : epilogue (tcgen05.ld 32x32b.x32 -> registers -> C - acc -> global)
#include <cuda.h>
#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace nmg {
namespace {

#ifndef NMG_GEMM_STAGES64
#define NMG_GEMM_STAGES64 4
#endif
constexpr int TBM = 128, TBK = 16, TNT = 128;
constexpr int A_BYTES = TBM * TBK * 4;                    // 8 KB
template <int TBN> struct TcCfg {
  static constexpr int B_BYTES = TBN * TBK * 4;                     // 16 KB at N = 256
  static constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;     // 48 KB at N = 256
  static constexpr int NST = TBN == 256 ? 4 : NMG_GEMM_STAGES64;   // TMA ring depth
  static constexpr int SMEM = NST * STAGE_BYTES + 1024 /*barriers*/ + 1024 /*align slack*/;
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TBN >> 3) << 17) |
                                    ((uint32_t)(TBM >> 4) << 24);   // D f32, A/B tf32 K-major, M=128
  // FP16x3: the same 64-byte smem rows hold 32 f16 (K per stage 32), kind::f16 with A/B f16
  static constexpr uint32_t IDESC16 = (1u << 4) | ((uint32_t)(TBN >> 3) << 17) | ((uint32_t)(TBM >> 4) << 24);
};

NMG_D void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];\n" ::"l"(map) : "memory");
}

NMG_D void tc_store_chunk(const TcGemmArgs& a, const uint32_t (&v)[32], int m, int nb, const float* crow,
                          float* drow) {
    if (a.tblock) {
      // transposed store within tb x tb blocks: lanes hold consecutive rows -> coalesced
      const int64_t tb = a.tblock;
      const int64_t base = ((int64_t)m / tb) * tb * tb + (m % tb);
#pragma unroll 4
      for (int j = 0; j < 32; ++j) {
        const int n = nb + j;
        if (n >= a.N) break;
        float acc = __uint_as_float(v[j]);
        if (a.negate) acc = -acc;
        const int64_t off = base + (int64_t)n * tb;
        if (a.Dh) {
          uint32_t hh, ll;
          asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(hh) : "f"(acc));
          asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(ll) : "f"(acc - __uint_as_float(hh)));
          a.Dh[off] = __uint_as_float(hh);
          a.Dl[off] = __uint_as_float(ll);
        } else {
          a.D[off] = a.C ? a.C[off] + acc : acc;
        }
      }
      return;
    }
    if (nb + 32 <= a.N && !a.Dh) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float4 o;
        float acc[4] = {__uint_as_float(v[j]), __uint_as_float(v[j + 1]), __uint_as_float(v[j + 2]),
                        __uint_as_float(v[j + 3])};
        if (a.negate) { acc[0] = -acc[0]; acc[1] = -acc[1]; acc[2] = -acc[2]; acc[3] = -acc[3]; }
        if (crow) {
          const float4 cv = *reinterpret_cast<const float4*>(crow + nb + j);
          o = make_float4(cv.x + acc[0], cv.y + acc[1], cv.z + acc[2], cv.w + acc[3]);
        } else {
          o = make_float4(acc[0], acc[1], acc[2], acc[3]);
        }
        *reinterpret_cast<float4*>(drow + nb + j) = o;
      }
    } else {
      for (int j = 0; j < 32 && nb + j < a.N; ++j) {
        float acc = __uint_as_float(v[j]);
        if (a.negate) acc = -acc;
        if (a.Dh) {
          uint32_t hh, ll;
          asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(hh) : "f"(acc));
          asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(ll) : "f"(acc - __uint_as_float(hh)));
          a.Dh[(int64_t)m * a.ldd + nb + j] = __uint_as_float(hh);
          a.Dl[(int64_t)m * a.ldd + nb + j] = __uint_as_float(ll);
        } else {
          drow[nb + j] = crow ? crow[nb + j] + acc : acc;
        }
      }
    }
  }

NMG_D void tma_load_2d_mc(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4}], [%2], %5;\n" ::"r"(su32(dst)),
      "l"(map), "r"(su32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
NMG_D void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
NMG_D uint32_t cta_rank_in_cluster() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}

// MC: CTA pairs along M (cluster 1 x 2) share the W tile -- each loads half of its rows and
// multicasts them to both (W maps with box rows TBN / 2), halving the L2 -> SM traffic of
// the operator, which every M tile re-reads; a stage is refilled only after the MMAs of BOTH
// CTAs released it (commit multicast, empty count 2)
template <int TBN, bool F16 = false, bool MC = false>
__global__ void __launch_bounds__(TNT, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap tXh, const __grid_constant__ CUtensorMap tXl,
                   const __grid_constant__ CUtensorMap tWh, const __grid_constant__ CUtensorMap tWl,
                   TcGemmArgs a) {
  constexpr int KE = F16 ? 2 * TBK : TBK;    // K elements per stage (64-byte rows)
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  constexpr int B_BYTES = TcCfg<TBN>::B_BYTES, STAGE_BYTES = TcCfg<TBN>::STAGE_BYTES;
  constexpr int TSTAGES = TcCfg<TBN>::NST;
  constexpr uint32_t kIdesc = F16 ? TcCfg<TBN>::IDESC16 : TcCfg<TBN>::IDESC;
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + TSTAGES * STAGE_BYTES);
  uint64_t* empty = full + TSTAGES;
  uint64_t* done = empty + TSTAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * TBM, n0 = blockIdx.x * TBN;
  // K blocks [kb, ke): outside the union of the tile's 64-row ranges every W element is zero in
  // both planes, so the skipped products are exact zeros (CTA pairs along M share n0: same range)
  int kb = 0, ke = ceil_div(a.K, KE);
  if (a.krange) {
    int lo = a.K, hi = 0;
#pragma unroll
    for (int t = 0; t < TBN / 64; ++t) {
      if (n0 + 64 * t >= a.N) break;
      const int2 r = __ldg(&a.krange[n0 / 64 + t]);
      lo = min(lo, r.x);
      hi = max(hi, r.y);
    }
    kb = lo / KE;
    ke = max(kb + 1, min(ke, ceil_div(hi, KE)));
  }

  const uint32_t crank = MC ? cta_rank_in_cluster() : 0u;
  if (tid == 0) {
    for (int s = 0; s < TSTAGES; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], MC ? 2 : 1); }
    mb_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    prefetch_tmap(&tXh); prefetch_tmap(&tXl); prefetch_tmap(&tWh); prefetch_tmap(&tWl);
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(TBN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (MC) cluster_sync_all();                  // both CTAs' barriers exist before any multicast
  else __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer
      for (int kt = kb; kt < ke; ++kt) {
        const int s = (kt - kb) % TSTAGES;
        const uint32_t ph = (uint32_t)((kt - kb) / TSTAGES) & 1u;
        mb_wait(&empty[s], ph ^ 1u);
        uint8_t* st = sm + s * STAGE_BYTES;
        mb_expect(&full[s], STAGE_BYTES);
        const int k0 = kt * KE;
        tma2d(st, &tXh, &full[s], k0, m0);
        tma2d(st + A_BYTES, &tXl, &full[s], k0, m0);
        if (MC) {
          const int hr = TBN / 2;
          tma_load_2d_mc(st + 2 * A_BYTES + crank * (B_BYTES / 2), &tWh, &full[s], k0, n0 + (int)crank * hr, 3);
          tma_load_2d_mc(st + 2 * A_BYTES + B_BYTES + crank * (B_BYTES / 2), &tWl, &full[s], k0, n0 + (int)crank * hr,
                         3);
        } else {
          tma2d(st + 2 * A_BYTES, &tWh, &full[s], k0, n0);
          tma2d(st + 2 * A_BYTES + B_BYTES, &tWl, &full[s], k0, n0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      for (int kt = kb; kt < ke; ++kt) {
        const int s = (kt - kb) % TSTAGES;
        const uint32_t ph = (uint32_t)((kt - kb) / TSTAGES) & 1u;
        mb_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t st = su32(sm + s * STAGE_BYTES);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ko = ks * 32;   // 8 tf32 / 16 f16 = 32 bytes along the 64-byte swizzled row
          const uint64_t dxh = desc_sw64(st + ko);
          const uint64_t dxl = desc_sw64(st + A_BYTES + ko);
          const uint64_t dwh = desc_sw64(st + 2 * A_BYTES + ko);
          const uint64_t dwl = desc_sw64(st + 2 * A_BYTES + B_BYTES + ko);
          if (F16) {
            mma_f16(tmem, dxh, dwh, kIdesc, (kt != kb || ks) ? 1u : 0u);
            mma_f16(tmem, dxh, dwl, kIdesc, 1u);
            mma_f16(tmem, dxl, dwh, kIdesc, 1u);
          } else {
            mma_tf32(tmem, dxh, dwh, kIdesc, (kt != kb || ks) ? 1u : 0u);
            mma_tf32(tmem, dxh, dwl, kIdesc, 1u);
            mma_tf32(tmem, dxl, dwh, kIdesc, 1u);
          }
        }
        if (MC)   // slot reusable when both CTAs' MMAs retired
          asm volatile(
              "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                  su32(&empty[s])),
              "h"((uint16_t)3)
              : "memory");
        else
          mma_commit(&empty[s]);    // slot reusable when these MMAs retire
      }
      mma_commit(done);             // accumulator complete
    }
    __syncwarp();
  }

  // ---------------- epilogue: all 4 warps, warp w owns TMEM lanes 32w..32w+31 (rows)
  mb_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int row = warp * 32 + lane;
  const int m = m0 + row;
  const bool mok = m < a.M;
  const float* crow = a.C ? a.C + (int64_t)m * a.ldc : nullptr;
  float* drow = a.D ? a.D + (int64_t)m * a.ldd : nullptr;
#pragma unroll 1
  for (int c = 0; c < TBN / 32; ++c) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * 32);
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
          "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
          "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int nb = n0 + c * 32;
    if (F16 && mok) {
      const float xs = a.xinv[m];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int nn = min(nb + j, a.N - 1);
        v[j] = __float_as_uint(__uint_as_float(v[j]) * (xs * __ldg(a.winv + nn)));
      }
    }
    if (mok) tc_store_chunk(a, v, m, nb, crow, drow);
    __syncwarp();
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  if (MC) cluster_sync_all();                  // no CTA leaves while its peer may still signal it
  else __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(TBN));
  }
}

// ---- tf32 hi/lo split: hi = cvt.rna.tf32(x), lo = cvt.rna.tf32(x - hi) -------------
__global__ void split_tf32_kernel(int64_t count, const float* __restrict__ x, float* __restrict__ hi,
                                  float* __restrict__ lo) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const float v = x[i];
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(v));
  const float hf = __uint_as_float(h);
  uint32_t l;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(l) : "f"(v - hf));
  hi[i] = hf;
  lo[i] = __uint_as_float(l);
}

// ---- per-row scaled f16 hi/lo split (one CTA per row) -------------------------------
__global__ void __launch_bounds__(256) split_f16_rows_kernel(int K, const float* __restrict__ x,
                                                             __half* __restrict__ hi, __half* __restrict__ lo,
                                                             float* __restrict__ xinv) {
  __shared__ float red[8];
  const int m = blockIdx.x;
  const float* row = x + (int64_t)m * K;
  float mx = 0.f;
  for (int k = threadIdx.x; k < K; k += 256) mx = fmaxf(mx, fabsf(row[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, red[w]);
  // S = 2^e with S max <= 2^14 (hi never overflows f16), exact power of two
  int e = 0;
  if (mx > 0.f) { frexpf(16384.f / mx, &e); e -= 1; }
  e = max(-100, min(100, e));
  const float S = ldexpf(1.f, e);
  if (threadIdx.x == 0) xinv[m] = ldexpf(1.f, -e);
  for (int k = threadIdx.x; k < K; k += 256) {
    const float v = row[k] * S;
    const __half h = __float2half_rn(v);
    hi[(int64_t)m * K + k] = h;
    lo[(int64_t)m * K + k] = __float2half_rn(v - __half2float(h));
  }
}

}  // namespace

int tc_gemm_block_m() { return TBM; }

void tc_gemm_f16(const CUtensorMap* xh, const CUtensorMap* xl, const CUtensorMap* wh, const CUtensorMap* wl,
                 const TcGemmArgs& a, cudaStream_t s, int bn) {
  dim3 grid(ceil_div(a.N, bn), ceil_div(a.M, TBM));
  if (bn == 256 && a.wh_mc && grid.y % 2 == 0) {
    NMG_SMEM_OPTIN((tc_gemm_kernel<256, true, true>), TcCfg<256>::SMEM);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(TNT);
    cfg.dynamicSmemBytes = TcCfg<256>::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 2;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, tc_gemm_kernel<256, true, true>, *xh, *xl, *a.wh_mc, *a.wl_mc, a);
  } else if (bn == 256) {
    NMG_SMEM_OPTIN((tc_gemm_kernel<256, true>), TcCfg<256>::SMEM);
    tc_gemm_kernel<256, true><<<grid, TNT, TcCfg<256>::SMEM, s>>>(*xh, *xl, *wh, *wl, a);
  } else {
    NMG_SMEM_OPTIN((tc_gemm_kernel<64, true>), TcCfg<64>::SMEM);
    tc_gemm_kernel<64, true><<<grid, TNT, TcCfg<64>::SMEM, s>>>(*xh, *xl, *wh, *wl, a);
  }
}

void split_f16_rows(int rows, int K, const float* x, uint16_t* hi, uint16_t* lo, float* xinv, cudaStream_t s) {
  split_f16_rows_kernel<<<rows, 256, 0, s>>>(K, x, reinterpret_cast<__half*>(hi), reinterpret_cast<__half*>(lo),
                                             xinv);
}

void tc_gemm(const CUtensorMap* xh, const CUtensorMap* xl, const CUtensorMap* wh, const CUtensorMap* wl,
             const TcGemmArgs& a, cudaStream_t s, int bn) {
  dim3 grid(ceil_div(a.N, bn), ceil_div(a.M, TBM));
  if (bn == 256) {
    NMG_SMEM_OPTIN(tc_gemm_kernel<256>, TcCfg<256>::SMEM);
    tc_gemm_kernel<256><<<grid, TNT, TcCfg<256>::SMEM, s>>>(*xh, *xl, *wh, *wl, a);
  } else {
    NMG_SMEM_OPTIN(tc_gemm_kernel<64>, TcCfg<64>::SMEM);
    tc_gemm_kernel<64><<<grid, TNT, TcCfg<64>::SMEM, s>>>(*xh, *xl, *wh, *wl, a);
  }
}

void split_tf32(int64_t count, const float* x, float* hi, float* lo, cudaStream_t s) {
  split_tf32_kernel<<<(int)ceil_div64(count, 256), 256, 0, s>>>(count, x, hi, lo);
}

}  // namespace nmg
