// fp64-accurate outer residual r = y - X W^T (PAPER.md P:312-313 outer iteration, stop rule
// P:479) emulated with EXACT integer products on the tcgen05 INT8 tensor cores (Ozaki-style
// digit splitting):
//   x_mk = 2^{ex_m} sum_{i=1..S} X_i[m][k] 2^{-7 i},   W_nk = 2^{ew_n} sum_{j=1..S} W_j[n][k] 2^{-7 j}
// with int8 digits |X_i|, |W_j| <= 127 (truncation of the scaled mantissa, so every digit and
// the remainder 2^{-7 S} are exact), and
//   (X W^T)_mn = 2^{ex_m + ew_n} sum_{d=2}^{S+1} 2^{-7 d} sum_{i+j=d} (X_i W_j^T)_mn
// (pairs with i + j > S + 1 contribute below the digit truncation and are dropped).  Each
// X_i W_j^T is an exact int32 GEMM (K 127^2 (S) < 2^31); the diagonals d are accumulated in
// separate TMEM int32 accumulators and combined in fp64 in the epilogue, fused with y - (.),
// the fp32 copy for the inner cycle and the per-row ||r||^2 partials.
// S = 7 digits: 49 bits per operand relative to the row maximum.
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace nmg {
namespace {

constexpr int OS = 7;                       // digits per operand (diagonals d = 2 .. OS + 1)
// Tile / pipeline shape (compile-time knobs for A/B builds, tools/ab_ozaki.sh).  Measured at
// tensor-pipe 31-34 % active (ncu r02, cfg 3); neither 32-wide K blocks in 4 stages of 42 KB
// (SWIZZLE_32B digit maps: cfg 1 gemm64 0.423 vs 0.430 ms, cfg 3 32.7 vs 32.2 ms) nor 32-wide
// N tiles with two CTAs per SM (epilogue of one under the MMAs of the other: cfg 1 0.68 ms,
// cfg 3 32.9 ms) moved it, so the kernel keeps 64 x 64 tiles in two 84 KB stages.
#ifndef NMG_OZ_BK
#define NMG_OZ_BK 64
#endif
#ifndef NMG_OZ_NST
#define NMG_OZ_NST 2
#endif
#ifndef NMG_OZ_BN
#define NMG_OZ_BN 64
#endif
constexpr int OBM = 128, OBN = NMG_OZ_BN, OBK = NMG_OZ_BK, ONSTAGE = NMG_OZ_NST, ONT = 128;
constexpr int OTCOLS = OBN == 32 ? 256 : 512;
constexpr int XS_BYTES = OS * OBM * OBK;    // 28 KB (OBK 32)
constexpr int WS_BYTES = OS * OBN * OBK;    // 14 KB
constexpr int OSTAGE = XS_BYTES + WS_BYTES;
constexpr int OZ_SMEM = ONSTAGE * OSTAGE + 256 + 1024;

// multicast to the CTAs of `mask` (same smem offsets, complete_tx on each CTA's barrier)
NMG_D void tma3d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, "
      "%4, %5}], [%2], %6;\n" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
NMG_D void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
NMG_D uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
NMG_D uint32_t idesc_i8(int nd) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)((OBN * nd) >> 3) << 17) | ((uint32_t)(OBM >> 4) << 24);
}
NMG_D void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// CTA pairs along N share the X digit tile: each CTA loads half of its rows and multicasts
// it to both (halving the L2 -> SM traffic of X, which every N tile re-reads); a stage is
// refilled only after the MMAs of BOTH CTAs released it (commit multicast, count 2).
// GEN: the slab mode's general output mapping and W row offset (else the whole-image mapping)
template <bool GEN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(ONT, OBN == 32 ? 2 : 1)
    ozaki_resid_kernel(const __grid_constant__ CUtensorMap mX, const __grid_constant__ CUtensorMap mW,
                       OzakiArgs a) {
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t* sm = smraw + ((1024u - (su32(smraw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + ONSTAGE * OSTAGE);
  uint64_t* empty = full + ONSTAGE;
  uint64_t* done = empty + ONSTAGE;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int m0 = blockIdx.y * OBM, n0 = blockIdx.x * OBN;
  // K blocks [kb, ke): the union of the two W tiles of the CTA pair (both CTAs run the same
  // blocks: they share the multicast X stages).  Outside it every digit of both W tiles is zero,
  // so the skipped int32 products are exact zeros and the accumulators are bitwise unchanged.
  int kb = 0, ke = a.K / OBK;
  if (a.krange) {
    const int t0 = ((GEN ? a.wrow0 : 0) + (int)(blockIdx.x & ~1u) * OBN) / OBN;
    const int2 r0 = __ldg(&a.krange[t0]), r1 = __ldg(&a.krange[t0 + 1]);
    kb = min(r0.x, r1.x);
    ke = max(r0.y, r1.y);
  }

  const uint32_t crank = cluster_rank();
  if (tid == 0) {
    for (int s = 0; s < ONSTAGE; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 2); }
    mb_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)), "n"(OTCOLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  cluster_sync();                                 // both CTAs' barriers exist before any multicast
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0) {   // TMA producer: all S digit planes of X and W for one 64-wide K block
      for (int kt = kb; kt < ke; ++kt) {
        const int s = (kt - kb) % ONSTAGE;
        mb_wait(&empty[s], ((uint32_t)((kt - kb) / ONSTAGE) & 1u) ^ 1u);
        uint8_t* st = sm + s * OSTAGE;
        mb_expect(&full[s], OSTAGE);                 // own W + both halves of X
#pragma unroll
        for (int d = 0; d < OS; ++d)                 // rows [64 r, 64 r + 64) of every X digit plane
          tma3d_mc(st + d * OBM * OBK + crank * 64 * OBK, &mX, &full[s], kt * OBK, m0 + (int)crank * 64, d, 3);
        tma3d(st + XS_BYTES, &mW, &full[s], kt * OBK, (GEN ? a.wrow0 : 0) + n0, 0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {   // MMA issuer: 28 digit-pair products (10 MMAs) per 32-wide K step
      for (int kt = kb; kt < ke; ++kt) {
        const int s = (kt - kb) % ONSTAGE;
        mb_wait(&full[s], (uint32_t)((kt - kb) / ONSTAGE) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t xs = su32(sm + s * OSTAGE), ws = xs + XS_BYTES;
#pragma unroll
        for (int ks = 0; ks < OBK / 32; ++ks) {
#pragma unroll
          for (int i = 1; i <= OS; ++i) {
            // X_i times up to four consecutive W digits stacked along N (their smem planes are
            // contiguous rows): one MMA with N = 64 nd writes the consecutive diagonal
            // accumulators d = i + j - 2 .., so the X_i tile is read once per four digits
#pragma unroll
            for (int j0 = 1; j0 <= OS + 1 - i; j0 += 4) {
              const int nd = (OS + 2 - i - j0) < 4 ? (OS + 2 - i - j0) : 4;
              const int d = i + j0 - 2;                      // first accumulator 0 .. OS - 1
              const uint64_t da = OBK == 32 ? desc_sw32(xs + (i - 1) * OBM * OBK) : desc_sw64(xs + (i - 1) * OBM * OBK + ks * 32);
              const uint64_t db = OBK == 32 ? desc_sw32(ws + (j0 - 1) * OBN * OBK) : desc_sw64(ws + (j0 - 1) * OBN * OBK + ks * 32);
              // the first products into the diagonals come from i = 1 at kt = kb, ks = 0
              mma_i8(tmem + (uint32_t)(d * OBN), da, db, idesc_i8(nd), (kt == kb && ks == 0 && i == 1) ? 0u : 1u);
            }
          }
        }
        // the stage is free when both CTAs' MMAs have read it
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                su32(&empty[s])),
            "h"((uint16_t)3)
            : "memory");
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(su32(done))
                   : "memory");
    }
    __syncwarp();
  }
  // ---------------- epilogue: warp w owns rows 32 w .. 32 w + 31 (TMEM lanes)
  if (a.tblock && (a.Y || a.ax)) {
    // 2D pass 2: pull the tile's y and x columns into L2 while the MMAs run (the epilogue
    // reads them column by column; a warp's 32 rows of one column are 256 contiguous bytes)
    const int R = GEN ? a.tb_R : a.tblock;                  // 32-bit divisions
    const int64_t S = GEN ? a.tb_S : a.tblock;
    const int64_t img = GEN ? a.tb_img : (int64_t)a.tblock * a.tblock;
    const int mw = m0 + warp * 32;
    if (mw < a.M && (lane & 15) == 0) {
      const int bw = mw / R;
      const int64_t base = (int64_t)bw * img + (mw - bw * R) + (lane >> 4) * 16;
      for (int c = 0; c < OBN; ++c) {
        const int64_t off = base + (int64_t)(n0 + c) * S;
        if (a.Y) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a.Y + off));
        if (a.ax) asm volatile("prefetch.global.L2 [%0];\n" ::"l"(a.ax + off));
      }
    }
  }
  mb_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int m = m0 + warp * 32 + lane;
  double acc[OBN];
#pragma unroll
  for (int c = 0; c < OBN; ++c) acc[c] = 0.0;
#pragma unroll
  for (int d = OS - 1; d >= 0; --d) {          // smallest terms first
    const double sc = ldexp(1.0, -7 * (d + 2));
#pragma unroll
    for (int half = 0; half < OBN / 32; ++half) {
      uint32_t v[32];
      const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(d * OBN + half * 32);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
            "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
            "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int j = 0; j < 32; ++j) acc[half * 32 + j] = fma((double)(int)v[j], sc, acc[half * 32 + j]);
    }
  }
  double sq = 0.0;
  if (m < a.M && a.tblock) {
    // 2D Kronecker passes: transposed store within tb x tb blocks (consecutive rows m of a
    // warp write consecutive addresses); pass 1 stores +X W^T, pass 2 y - X W^T - alpha x
    const int exm = a.ex[m];
    // block mapping: output (m, col) at (m / R) img + col S + m % R (R = S = tb, img = tb^2 by
    // default; the slab mode passes its own); r32 may live in a halo'd slab (r32_img, r32_off)
    const int R = GEN ? a.tb_R : a.tblock;                  // 32-bit divisions
    const int64_t S = GEN ? a.tb_S : a.tblock;
    const int64_t img = GEN ? a.tb_img : (int64_t)a.tblock * a.tblock;
    const int bi = m / R;
    const int64_t base = (int64_t)bi * img + (m - bi * R);
    const int64_t d32 = (GEN && a.r32_img) ? bi * (a.r32_img - img) + a.r32_off : 0;   // r32 offset - output offset
    // batches of 8 columns: all loads of a batch issue before any store (the stores could
    // alias y / x as far as the compiler knows, which would serialise load latencies)
#pragma unroll
    for (int c0 = 0; c0 < OBN; c0 += 8) {
      double yv[8], xv[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int64_t off = base + (int64_t)(n0 + c0 + j) * S;
        yv[j] = (!a.plus && a.Y) ? __ldg(a.Y + off) : 0.0;
        xv[j] = a.ax ? __ldg(a.ax + off) : 0.0;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int c = c0 + j;
        const int64_t off = base + (int64_t)(n0 + c) * S;
        const double p = ldexp(acc[c], exm + a.ew[(GEN ? a.wrow0 : 0) + n0 + c]);
        double v = a.plus ? p : yv[j] - p;
        if (a.ax) v = fma(-a.alpha, xv[j], v);
        if (a.r32) a.r32[off + d32] = (float)v;
        if (a.r64) a.r64[off] = v;
        sq += v * v;
      }
    }
    if (a.part) a.part[(int64_t)m * gridDim.x + blockIdx.x] = sq;
  } else if (m < a.M) {
    const int exm = a.ex[m];
    const double* yr = a.Y + (int64_t)m * a.ldy + n0;
    float* r32 = a.r32 ? a.r32 + (int64_t)m * a.ldr32 + n0 : nullptr;
    double* r64 = a.r64 ? a.r64 + (int64_t)m * a.ldr64 + n0 : nullptr;
#pragma unroll
    for (int c = 0; c < OBN; ++c) {
      const double v = yr[c] - ldexp(acc[c], exm + a.ew[n0 + c]);
      if (r32) r32[c] = (float)v;
      if (r64) r64[c] = v;
      sq += v * v;
    }
    if (a.part) a.part[(int64_t)m * gridDim.x + blockIdx.x] = sq;
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  cluster_sync();                                 // no CTA leaves while its peer may still signal it
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(OTCOLS));
}

// digits of the rows of X (fp64 [M][K]): ex[m] with max_k |x_mk| < 2^{ex[m]}, then S truncation
// digits of x * 2^{-ex}; one CTA per row.  Layout of `dig`: [S][M][K] int8.
__global__ void __launch_bounds__(256) ozaki_split_rows_kernel(int M, int K, const double* __restrict__ X, int64_t ldx,
                                                               int8_t* __restrict__ dig, int64_t plane,
                                                               int* __restrict__ ex) {
  __shared__ double red[32];
  const int m = blockIdx.x;
  const double* xr = X + (int64_t)m * ldx;
  double mx = 0.0;
  for (int k = threadIdx.x; k < K; k += blockDim.x) mx = fmax(mx, fabs(xr[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t = fmax(t, __shfl_xor_sync(0xffffffffu, t, o));
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  mx = red[0];
  int e = 0;
  if (mx > 0.0) { frexp(mx, &e); }             // mx in [2^{e-1}, 2^e)
  if (threadIdx.x == 0) ex[m] = e;
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    double r = ldexp(xr[k], -e);               // |r| < 1
#pragma unroll
    for (int i = 0; i < OS; ++i) {
      r *= 128.0;
      const double dgt = trunc(r);             // |dgt| <= 127
      r -= dgt;
      dig[(int64_t)i * plane + (int64_t)m * K + k] = (int8_t)(int)dgt;
    }
  }
}

// same digits, one warp per row (short rows, K < 2048): 8 rows per CTA
__global__ void __launch_bounds__(256) ozaki_split_rows_warp_kernel(int M, int K, const double* __restrict__ X,
                                                                    int64_t ldx, int8_t* __restrict__ dig,
                                                                    int64_t plane, int* __restrict__ ex) {
  const int m = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (m >= M) return;
  const double* xr = X + (int64_t)m * ldx;
  double mx = 0.0;
  for (int k = lane; k < K; k += 32) mx = fmax(mx, fabs(xr[k]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.0) { frexp(mx, &e); }
  if (lane == 0) ex[m] = e;
  for (int k = 2 * lane; k < K; k += 64) {      // two digits per byte pair store
    double r0 = ldexp(xr[k], -e), r1 = ldexp(xr[k + 1], -e);
#pragma unroll
    for (int i = 0; i < OS; ++i) {
      r0 *= 128.0;
      r1 *= 128.0;
      const double d0 = trunc(r0), d1 = trunc(r1);
      r0 -= d0;
      r1 -= d1;
      const uint32_t pk = ((uint32_t)(uint8_t)(int8_t)(int)d0) | ((uint32_t)(uint8_t)(int8_t)(int)d1 << 8);
      *reinterpret_cast<uint16_t*>(dig + (int64_t)i * plane + (int64_t)m * K + k) = (uint16_t)pk;
    }
  }
}

}  // namespace

int ozaki_bk() { return OBK; }
int ozaki_bn() { return OBN; }
int ozaki_digits() { return OS; }

void ozaki_split_rows(int M, int K, const double* X, int64_t ldx, int8_t* dig, int64_t plane, int* ex,
                      cudaStream_t s) {
  if (K < 2048 && K % 2 == 0) ozaki_split_rows_warp_kernel<<<ceil_div(M, 8), 256, 0, s>>>(M, K, X, ldx, dig, plane, ex);
  else ozaki_split_rows_kernel<<<M, 256, 0, s>>>(M, K, X, ldx, dig, plane, ex);
}

void ozaki_resid(const CUtensorMap* mx, const CUtensorMap* mw, const OzakiArgs& a, cudaStream_t s) {
  const bool gen = a.tb_R || a.tb_S || a.tb_img || a.r32_img || a.wrow0;
  dim3 grid(a.N / OBN, ceil_div(a.M, OBM));
  if (gen) {
    NMG_SMEM_OPTIN(ozaki_resid_kernel<true>, OZ_SMEM);
    OzakiArgs g = a;   // the general mapping needs every field set
    if (!g.tb_R) g.tb_R = g.tblock;
    if (!g.tb_S) g.tb_S = g.tblock;
    if (!g.tb_img) g.tb_img = (int64_t)g.tblock * g.tblock;
    ozaki_resid_kernel<true><<<grid, ONT, OZ_SMEM, s>>>(*mx, *mw, g);
  } else {
    NMG_SMEM_OPTIN(ozaki_resid_kernel<false>, OZ_SMEM);
    ozaki_resid_kernel<false><<<grid, ONT, OZ_SMEM, s>>>(*mx, *mw, a);
  }
}

}  // namespace nmg
