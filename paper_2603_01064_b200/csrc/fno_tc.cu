// FNO W-convolution on the 5th-gen tensor cores (tcgen05, kind::tf32, 3xTF32), the dense
// contraction of the paper's FNO smoother (Appendix A P:651-657:
// f(Z) = sigma(K(Z) + W * Z + B), W a ks (x ks) convolution over c = 64 channels):
//   Z1[b][o][p] = GELU( Z1[b][o][p] + B[o] + sum_{c, t} W[o][c][t] Z0[b][c][p + t - ks/2] )
// with Z1 holding the spectral branch K(Z) on entry.  Implicit GEMM, no im2col buffer:
//   M = 128 output points of one RHS (1D: consecutive positions; 2D: a bx x by pixel box),
//   N = 64 output channels, K = (tap, input channel) in blocks of 16 channels of one tap.
// The layer input is kept channels-last as a tf32 hi/lo pair X = Xh + Xl [b][N_l][c] (written by
// fno_lift_cl / the previous layer's epilogue), so the K block of tap t is the box
// {16 channels, 128 points shifted by t - ks/2} of a rank-3 (1D) / rank-4 (2D) tensor map: the
// TMA unit applies the shift and zero-fills the points outside the image (the "same" padding).
// W is stored [o][tap][c] (tf32 hi/lo, split at load).  X W^T ~= Xh Wh^T + Xh Wl^T + Xl Wh^T
// accumulates in one 128 x 64 fp32 TMEM tile (as tc_gemm_kernel / kron_tc_kernel).
//
// Kernel anatomy (one output tile per CTA, 128 threads, 4-stage 24 KB ring: two CTAs per SM so
// one CTA's epilogue overlaps the other's main loop):
//   warp 0 / lane 0 : TMA producer (cp.async.bulk.tensor 3D/4D for X, 2D for W, SWIZZLE_64B)
//   warp 1 / lane 0 : MMA issuer (tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 64, K = 8)
//   warp 2          : TMEM allocator (64 fp32 columns)
//   all 4 warps     : epilogue (tcgen05.ld -> + K(Z) + bias -> GELU -> Z1 [b][o][p], and the
//                     next layer's channels-last tf32 hi/lo input)
#include <cuda.h>

#include "common.cuh"
#include "kernels.h"
#include "tcgen05.cuh"

namespace nmg {
namespace {

#ifndef NMG_FNO_ST1D
#define NMG_FNO_ST1D 2   // 50 KB: four CTAs per SM (the short 1D K loop is epilogue-latency-bound: 157.6 -> 144.5 ms
                         // per cfg 1 FNO step against 4 stages / two CTAs; 3 stages 147.5)
#endif
#ifndef NMG_FNO_RA
#define NMG_FNO_RA 2     // row-halo kernel rings: 2 input-row stages + 4 W stages = 70 KB, three CTAs per SM
#endif                   // (cfg 2 FNO step 439.8 -> 427.7 ms against 3 + 6 stages / two CTAs)
#ifndef NMG_FNO_RW
#define NMG_FNO_RW 4
#endif
constexpr int FM = 128, FN = 64, FK = 16, FT = 128;
// TMA ring depth of the box kernel (24 KB stages): 1D / 2D
template <int DIM> struct FnoRing { static constexpr int ST = DIM == 1 ? NMG_FNO_ST1D : 4; };
constexpr int FA_BYTES = FM * FK * 4;                         // 8 KB
constexpr int FB_BYTES = FN * FK * 4;                         // 4 KB
constexpr int FSTAGE = 2 * FA_BYTES + 2 * FB_BYTES;           // 24 KB
template <int DIM> constexpr int fno_box_smem() { return FnoRing<DIM>::ST * FSTAGE + 1024 /*barriers*/ + 1024 /*align slack*/; }
// D f32, A/B tf32 K-major, M = 128, N = 64
constexpr uint32_t FIDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(FN >> 3) << 17) |
                            ((uint32_t)(FM >> 4) << 24);

NMG_D float gelu_tc(float z) { return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f)); }

NMG_D void tma4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];\n" ::"r"(su32(dst)),
      "l"(m), "r"(su32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

NMG_D void split_tf32_dev(float v, float& hi, float& lo) {
  uint32_t h, l;
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(h) : "f"(v));
  hi = __uint_as_float(h);
  asm("cvt.rna.tf32.f32 %0, %1;\n" : "=r"(l) : "f"(v - hi));
  lo = __uint_as_float(l);
}

// epilogue of one 128-point tile: warp w owns TMEM lanes 32w .. 32w + 31 (output points); point p
// of RHS b: Z1 <- GELU(Z1 + bias + acc) for every output channel, and the next layer's
// channels-last tf32 hi/lo input
NMG_D void fno_tile_epilogue(const FnoConvArgs& a, uint32_t tmem, int warp, int b, int64_t p, int64_t N) {
  float* z = a.Z1 + (int64_t)b * a.c * N + p;
  float* xh = a.Xh_out ? a.Xh_out + ((int64_t)b * N + p) * a.c : nullptr;
  float* xl = a.Xl_out ? a.Xl_out + ((int64_t)b * N + p) * a.c : nullptr;
#pragma unroll 1
  for (int cc = 0; cc < FN / 32; ++cc) {
    if (cc * 32 >= a.c) break;                       // warp-uniform
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(cc * 32);
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
    for (int j0 = 0; j0 < 32; j0 += 16) {
      if (cc * 32 + j0 >= a.c) break;                // c is a multiple of 16
      float zin[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) zin[j] = z[(int64_t)(cc * 32 + j0 + j) * N];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int o = cc * 32 + j0 + j;
        zin[j] = gelu_tc(zin[j] + __ldg(a.bias + o) + __uint_as_float(v[j0 + j]));
        z[(int64_t)o * N] = zin[j];
      }
      if (xh) {
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          float4 hv, lv;
          split_tf32_dev(zin[j], hv.x, lv.x);
          split_tf32_dev(zin[j + 1], hv.y, lv.y);
          split_tf32_dev(zin[j + 2], hv.z, lv.z);
          split_tf32_dev(zin[j + 3], hv.w, lv.w);
          *reinterpret_cast<float4*>(xh + cc * 32 + j0 + j) = hv;
          *reinterpret_cast<float4*>(xl + cc * 32 + j0 + j) = lv;
        }
      }
    }
    __syncwarp();
  }
}

template <int DIM>
__global__ void __launch_bounds__(FT)
    fno_conv_tc_kernel(const __grid_constant__ CUtensorMap tXh, const __grid_constant__ CUtensorMap tXl,
                       const __grid_constant__ CUtensorMap tWh, const __grid_constant__ CUtensorMap tWl,
                       FnoConvArgs a) {
  constexpr int FST = FnoRing<DIM>::ST;
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + FST * FSTAGE);
  uint64_t* empty = full + FST;
  uint64_t* done = empty + FST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // output tile: RHS b, points x0 .. (1D) or the box [y0, y0 + by) x [x0, x0 + bx) (2D)
  int b, x0, y0 = 0;
  if (DIM == 1) {
    const int tpi = a.n / FM;
    b = blockIdx.x / tpi;
    x0 = (blockIdx.x - b * tpi) * FM;
  } else {
    const int tx = a.n >> a.lbx, ty = a.n / (FM >> a.lbx);
    b = blockIdx.x / (tx * ty);
    const int r = blockIdx.x - b * tx * ty;
    const int iy = r / tx;
    y0 = iy * (FM >> a.lbx);
    x0 = (r - iy * tx) << a.lbx;
  }
  const int hk = a.ks / 2, cbn = a.c / FK;
  const int ktot = (DIM == 1 ? a.ks : a.ks * a.ks) * cbn;

  if (tid == 0) {
    for (int s = 0; s < FST; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 1); }
    mb_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(FN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer
      for (int kt = 0; kt < ktot; ++kt) {
        const int s = kt % FST;
        const uint32_t ph = (uint32_t)(kt / FST) & 1u;
        mb_wait(&empty[s], ph ^ 1u);
        uint8_t* st = sm + s * FSTAGE;
        mb_expect(&full[s], FSTAGE);
        const int tap = kt / cbn, c0 = (kt - tap * cbn) * FK;
        if (DIM == 1) {
          tma3d(st, &tXh, &full[s], c0, x0 + tap - hk, b);
          tma3d(st + FA_BYTES, &tXl, &full[s], c0, x0 + tap - hk, b);
        } else {
          const int t2 = tap / a.ks, t1 = tap - t2 * a.ks;
          tma4d(st, &tXh, &full[s], c0, x0 + t1 - hk, y0 + t2 - hk, b);
          tma4d(st + FA_BYTES, &tXl, &full[s], c0, x0 + t1 - hk, y0 + t2 - hk, b);
        }
        tma2d(st + 2 * FA_BYTES, &tWh, &full[s], kt * FK, 0);
        tma2d(st + 2 * FA_BYTES + FB_BYTES, &tWl, &full[s], kt * FK, 0);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      for (int kt = 0; kt < ktot; ++kt) {
        const int s = kt % FST;
        const uint32_t ph = (uint32_t)(kt / FST) & 1u;
        mb_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t st = su32(sm + s * FSTAGE);
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const uint32_t ko = ks * 32;   // 8 tf32 = 32 bytes along the 64-byte swizzled row
          const uint64_t dxh = desc_sw64(st + ko);
          const uint64_t dxl = desc_sw64(st + FA_BYTES + ko);
          const uint64_t dwh = desc_sw64(st + 2 * FA_BYTES + ko);
          const uint64_t dwl = desc_sw64(st + 2 * FA_BYTES + FB_BYTES + ko);
          mma_tf32(tmem, dxh, dwh, FIDESC, (kt || ks) ? 1u : 0u);
          mma_tf32(tmem, dxh, dwl, FIDESC, 1u);
          mma_tf32(tmem, dxl, dwh, FIDESC, 1u);
        }
        mma_commit(&empty[s]);      // slot reusable when these MMAs retire
      }
      mma_commit(done);             // accumulator complete
    }
    __syncwarp();
  }

  // ---------------- epilogue: warp w owns TMEM lanes 32w .. 32w + 31 (output points)
  mb_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int row = warp * 32 + lane;
  const int64_t N = DIM == 1 ? (int64_t)a.n : (int64_t)a.n * a.n;
  const int64_t p = DIM == 1 ? (int64_t)(x0 + row)
                             : (int64_t)(y0 + (row >> a.lbx)) * a.n + x0 + (row & ((1 << a.lbx) - 1));
  fno_tile_epilogue(a, tmem, warp, b, p, N);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(FN));
  }
}

// ---- 2D, n >= 128: row-halo variant.  The tile is 128 pixels of ONE image row; per (t2, block of
// 16 input channels) the input row y + t2 - ks/2 is loaded ONCE with its x halo (128 + ks - 1
// pixels) through a rank-5 map {4 ch, x, c/4, y, rhs} with box {4, 128 + ks - 1, 4, 1, 1}, which
// lands as the canonical no-swizzle K-major tile [4 chunks][pixels][4 tf32] (16-byte rows,
// chunks LBO = 16 (128 + ks - 1) bytes apart); the x tap t1 is a 16 t1-byte shift of the A
// descriptor's start address.  The layer input is read from L2 ks times instead of ks^2 times
// (the box variant above is L2 -> SM bound at ~195 TFLOP/s); W streams through its own ring.
constexpr int RA_ST = NMG_FNO_RA, RW_ST = NMG_FNO_RW;
constexpr int RA_MAX = 2 * 64 * (FM + 6);                      // hi + lo, ks <= 7: 17,152 B
constexpr int RA_STAGE = (RA_MAX + 1023) / 1024 * 1024;           // the W ring behind it stays 1 KB-aligned (SWIZZLE_64B)
constexpr int RW_STAGE = 2 * FB_BYTES;                          // 8 KB
constexpr int RSMEM = RA_ST * RA_STAGE + RW_ST * RW_STAGE + 1024 /*barriers*/ + 1024 /*align slack*/;

NMG_D void tma5d_ns(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3, int c4) {
  tma5d(dst, m, bar, c0, c1, c2, c3, c4);
}

__global__ void __launch_bounds__(FT)
    fno_conv_rows_kernel(const __grid_constant__ CUtensorMap tXh, const __grid_constant__ CUtensorMap tXl,
                         const __grid_constant__ CUtensorMap tWh, const __grid_constant__ CUtensorMap tWl,
                         FnoConvArgs a) {
  extern __shared__ uint8_t smraw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~uintptr_t(1023));
  uint8_t* smW = sm + RA_ST * RA_STAGE;
  uint64_t* afull = reinterpret_cast<uint64_t*>(smW + RW_ST * RW_STAGE);
  uint64_t* aempty = afull + RA_ST;
  uint64_t* wfull = aempty + RA_ST;
  uint64_t* wempty = wfull + RW_ST;
  uint64_t* done = wempty + RW_ST;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tx = a.n / FM;
  const int b = blockIdx.x / (tx * a.n);
  const int r = blockIdx.x - b * tx * a.n;
  const int y = r / tx, x0 = (r - y * tx) * FM;
  const int ks = a.ks, hk = ks / 2, cbn = a.c / FK;
  const int AW = FM + ks - 1;
  const uint32_t lbo = (uint32_t)AW * 16u, a_plane = (uint32_t)AW * 64u;   // hi plane bytes (4 chunks)
  const int nas = ks * cbn;                                      // A stages: (t2, cb)

  if (tid == 0) {
    for (int s = 0; s < RA_ST; ++s) { mb_init(&afull[s], 1); mb_init(&aempty[s], 1); }
    for (int s = 0; s < RW_ST; ++s) { mb_init(&wfull[s], 1); mb_init(&wempty[s], 1); }
    mb_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tmem_slot)),
                 "r"(FN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer (A ring and W ring, in consumption order)
      int wi = 0;
      for (int as = 0; as < nas; ++as) {
        const int t2 = as / cbn, cb = as - t2 * cbn;
        const int sa = as % RA_ST;
        mb_wait(&aempty[sa], ((uint32_t)(as / RA_ST) & 1u) ^ 1u);
        uint8_t* st = sm + sa * RA_STAGE;
        mb_expect(&afull[sa], 2 * a_plane);
        tma5d_ns(st, &tXh, &afull[sa], 0, x0 - hk, cb * 4, y + t2 - hk, b);
        tma5d_ns(st + a_plane, &tXl, &afull[sa], 0, x0 - hk, cb * 4, y + t2 - hk, b);
        for (int t1 = 0; t1 < ks; ++t1, ++wi) {
          const int sw = wi % RW_ST;
          mb_wait(&wempty[sw], ((uint32_t)(wi / RW_ST) & 1u) ^ 1u);
          uint8_t* wt = smW + sw * RW_STAGE;
          mb_expect(&wfull[sw], RW_STAGE);
          const int k0 = ((t2 * ks + t1) * cbn + cb) * FK;
          tma2d(wt, &tWh, &wfull[sw], k0, 0);
          tma2d(wt + FB_BYTES, &tWl, &wfull[sw], k0, 0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      int wi = 0;
      for (int as = 0; as < nas; ++as) {
        const int sa = as % RA_ST;
        mb_wait(&afull[sa], (uint32_t)(as / RA_ST) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t ah = su32(sm + sa * RA_STAGE), al = ah + a_plane;
        for (int t1 = 0; t1 < ks; ++t1, ++wi) {
          const int sw = wi % RW_ST;
          mb_wait(&wfull[sw], (uint32_t)(wi / RW_ST) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
          const uint32_t wt = su32(smW + sw * RW_STAGE);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {      // K = 8 tf32 = chunks 2 kk, 2 kk + 1
            const uint64_t dxh = desc_ns(ah + (uint32_t)t1 * 16u + (uint32_t)kk * 2u * lbo, lbo);
            const uint64_t dxl = desc_ns(al + (uint32_t)t1 * 16u + (uint32_t)kk * 2u * lbo, lbo);
            const uint64_t dwh = desc_sw64(wt + kk * 32);
            const uint64_t dwl = desc_sw64(wt + FB_BYTES + kk * 32);
            mma_tf32(tmem, dxh, dwh, FIDESC, (wi || kk) ? 1u : 0u);
            mma_tf32(tmem, dxh, dwl, FIDESC, 1u);
            mma_tf32(tmem, dxl, dwh, FIDESC, 1u);
          }
          mma_commit(&wempty[sw]);
        }
        mma_commit(&aempty[sa]);
      }
      mma_commit(done);
    }
    __syncwarp();
  }

  mb_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int64_t N = (int64_t)a.n * a.n;
  fno_tile_epilogue(a, tmem, warp, b, (int64_t)y * a.n + x0 + warp * 32 + lane, N);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 2) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(FN));
  }
}

// X[b][p][ch] = tf32 hi/lo of lift(u)[ch] -- the same expression as fno_lift_kernel (bitwise the
// Z0 it writes), channels-last for the first layer's implicit-GEMM loads
__global__ void fno_lift_cl_kernel(int nrhs, int c, int64_t N, const float* __restrict__ in,
                                   const double* __restrict__ norms, const float* __restrict__ lw,
                                   const float* __restrict__ lb, float* __restrict__ Xh, float* __restrict__ Xl) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nrhs * c * N) return;
  const int ch = (int)(i % c);
  const int64_t bp = i / c;
  const int b = (int)(bp / N);
  const double s = norms ? norms[b] : 1.0;
  const float u = s != 0.0 ? (float)((double)in[bp] / s) : 0.f;
  float hi, lo;
  split_tf32_dev(fmaf(__ldg(lw + ch), u, __ldg(lb + ch)), hi, lo);
  Xh[i] = hi;
  Xl[i] = lo;
}

}  // namespace

bool fno_tc_ok(int dim, int n, int c) {
  if (c < 16 || c > FN || c % FK) return false;
  if (n & (n - 1)) return false;
  return dim == 1 ? n >= FM : n >= 16;
}

bool fno_tc_rows(int dim, int n, int ks) { return dim == 2 && n >= FM && ks <= 7; }

void fno_tc_box(int n, int* bx, int* by) {
  *bx = n < FM ? n : FM;
  *by = FM / *bx;
}

void fno_lift_cl(int nrhs, int c, int64_t N, const float* in, const double* norms, const float* lw, const float* lb,
                 float* Xh, float* Xl, cudaStream_t s) {
  fno_lift_cl_kernel<<<(unsigned)ceil_div64((int64_t)nrhs * c * N, 256), 256, 0, s>>>(nrhs, c, N, in, norms, lw, lb,
                                                                                     Xh, Xl);
}

void fno_conv_tc(const CUtensorMap* xh, const CUtensorMap* xl, const CUtensorMap* wh, const CUtensorMap* wl,
                 const FnoConvArgs& a, cudaStream_t s) {
  if (a.dim == 1) {
    NMG_SMEM_OPTIN(fno_conv_tc_kernel<1>, fno_box_smem<1>());
    const int64_t tiles = (int64_t)a.nrhs * (a.n / FM);
    fno_conv_tc_kernel<1><<<(unsigned)tiles, FT, fno_box_smem<1>(), s>>>(*xh, *xl, *wh, *wl, a);
  } else if (a.rows) {
    NMG_SMEM_OPTIN(fno_conv_rows_kernel, RSMEM);
    const int64_t tiles = (int64_t)a.nrhs * a.n * (a.n / FM);
    fno_conv_rows_kernel<<<(unsigned)tiles, FT, RSMEM, s>>>(*xh, *xl, *wh, *wl, a);
  } else {
    NMG_SMEM_OPTIN(fno_conv_tc_kernel<2>, fno_box_smem<2>());
    const int bx = 1 << a.lbx, by = FM / bx;
    const int64_t tiles = (int64_t)a.nrhs * (a.n / bx) * (a.n / by);
    fno_conv_tc_kernel<2><<<(unsigned)tiles, FT, fno_box_smem<2>(), s>>>(*xh, *xl, *wh, *wl, a);
  }
}

}  // namespace nmg
