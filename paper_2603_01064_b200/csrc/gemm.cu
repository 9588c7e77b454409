// Operator-apply GEMMs.
//  * gemm_f32: register-tiled SIMT fp32 GEMM (128x128x8 tiles), residual epilogue.
//    Inner-cycle operator apply r = y - A x (Alg 3) in fp32.
//  * gemm_f64: DMMA (mma.sync m8n8k4 f64) GEMM for the fp64 outer residual
//    r = y - A x^tau (PAPER.md:312-313 outer iteration, stop rule P:479), with the
//    per-row ||r||^2 partials fused into the epilogue (deterministic order).
#include "common.cuh"
#include "kernels.h"

namespace nmg {

// =============================================================================
// fp32 SIMT GEMM
// =============================================================================
namespace {
constexpr int BM = 128, BN = 128, BK = 8, NT = 256;

template <bool WK>
__global__ void __launch_bounds__(NT) sgemm_kernel(Gemm32Args a) {
  __shared__ __align__(16) float As[2][BK][BM + 4];
  __shared__ __align__(16) float Bs[2][BK][BN + 4];
  const int tid = threadIdx.x;
  const int bz = blockIdx.z;
  const float* X = a.X + bz * a.sx;
  const float* W = a.W + bz * a.sw;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int M = a.M, N = a.N, K = a.K;

  // global->smem mapping: A tile (BM x BK): row tid/2, k (tid&1)*4 .. +3
  const int ar = tid >> 1, ak = (tid & 1) * 4;
  // W K-major: same mapping on rows of W (n); N-major: k = tid/32, n = (tid&31)*4
  const int br = WK ? (tid >> 1) : (tid >> 5);
  const int bc = WK ? ((tid & 1) * 4) : ((tid & 31) * 4);

  float ra[4], rb[4];
  auto load_tiles = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int m = m0 + ar, k = k0 + ak + i;
      ra[i] = (m < M && k < K) ? __ldg(X + (int64_t)m * a.ldx + k) : 0.f;
    }
    if (WK) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int n = n0 + br, k = k0 + bc + i;
        rb[i] = (n < N && k < K) ? __ldg(W + (int64_t)n * a.ldw + k) : 0.f;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        int k = k0 + br, n = n0 + bc + i;
        rb[i] = (n < N && k < K) ? __ldg(W + (int64_t)k * a.ldw + n) : 0.f;
      }
    }
  };
  auto store_tiles = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) As[buf][ak + i][ar] = ra[i];
    if (WK) {
#pragma unroll
      for (int i = 0; i < 4; ++i) Bs[buf][bc + i][br] = rb[i];
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i) Bs[buf][br][bc + i] = rb[i];
    }
  };

  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  const int ty = tid >> 4, tx = tid & 15;
  load_tiles(0);
  store_tiles(0);
  __syncthreads();
  int buf = 0;
  for (int k0 = 0; k0 < K; k0 += BK) {
    const bool more = (k0 + BK) < K;
    if (more) load_tiles(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[8], bv[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][kk][64 + tx * 4]);
      av[0] = a0.x; av[1] = a0.y; av[2] = a0.z; av[3] = a0.w;
      av[4] = a1.x; av[5] = a1.y; av[6] = a1.z; av[7] = a1.w;
      bv[0] = b0.x; bv[1] = b0.y; bv[2] = b0.z; bv[3] = b0.w;
      bv[4] = b1.x; bv[5] = b1.y; bv[6] = b1.z; bv[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (more) {
      store_tiles(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  const float* C = a.C ? a.C + bz * a.sc : nullptr;
  float* D = a.D + bz * a.sd;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int m = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (m >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int n = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (n >= N) continue;
      float v = a.negate ? -acc[i][j] : acc[i][j];
      if (a.tblock) {
        const int64_t tb = a.tblock;
        const int64_t off = (m / tb) * tb * tb + (int64_t)n * tb + (m % tb);
        if (C) v = C[off] + v;
        D[off] = v;
      } else {
        if (C) v = C[(int64_t)m * a.ldc + n] + v;
        D[(int64_t)m * a.ldd + n] = v;
      }
    }
  }
}
}  // namespace

void gemm_f32(const Gemm32Args& a, cudaStream_t s) {
  dim3 grid(ceil_div(a.N, BN), ceil_div(a.M, BM), a.batch);
  if (a.w_kmajor)
    sgemm_kernel<true><<<grid, NT, 0, s>>>(a);
  else
    sgemm_kernel<false><<<grid, NT, 0, s>>>(a);
}

// =============================================================================
// fp64 DMMA GEMM with residual + norm-partial epilogue
// =============================================================================
namespace {
constexpr int DBM = 64, DBN = 64, DBK = 16, DNT = 128, DSTAGES = 3, DPAD = 4;
constexpr int DLDS = DBK + DPAD;   // smem row stride in doubles (conflict-free frags)

NMG_D void cp_async16(void* smem, const void* gmem, bool pred) {
  const unsigned saddr = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr), "l"(gmem), "r"(sz));
}
NMG_D void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
NMG_D void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

NMG_D void dmma_8x8x4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(DNT) dgemm_resid_kernel(Gemm64Args a) {
  extern __shared__ __align__(16) double dsm[];
  double* As = dsm;                                   // [STAGES][DBM][DLDS]
  double* Bs = dsm + DSTAGES * DBM * DLDS;            // [STAGES][DBN][DLDS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;           // 2x2 warps, 32x32 each
  const int g = lane >> 2, t = lane & 3;
  const int m0 = blockIdx.y * DBM, n0 = blockIdx.x * DBN;
  const int M = a.M, N = a.N, K = a.K;
  const int KT = ceil_div(K, DBK);
  const bool k_vec_ok = (K % 2 == 0);

  auto load_stage = [&](int st, int kt) {
    const int k0 = kt * DBK;
    double* as = As + st * DBM * DLDS;
    double* bs = Bs + st * DBN * DLDS;
    // 64 rows x 16 doubles = 512 double2 per operand; 128 threads x 4
#pragma unroll
    for (int it = 0; it < 4; ++it) {
      const int idx = tid + it * DNT;
      const int r = idx >> 3, c2 = (idx & 7) * 2;
      {
        const int m = m0 + r, k = k0 + c2;
        const bool ok = (m < M) && (k < K);
        if (k_vec_ok) {
          cp_async16(as + r * DLDS + c2, a.X + (int64_t)(ok ? m : 0) * a.ldx + (ok ? k : 0), ok);
        } else {
          as[r * DLDS + c2] = (m < M && k < K) ? a.X[(int64_t)m * a.ldx + k] : 0.0;
          as[r * DLDS + c2 + 1] = (m < M && k + 1 < K) ? a.X[(int64_t)m * a.ldx + k + 1] : 0.0;
        }
      }
      {
        const int n = n0 + r, k = k0 + c2;
        const bool ok = (n < N) && (k < K);
        if (k_vec_ok) {
          cp_async16(bs + r * DLDS + c2, a.W + (int64_t)(ok ? n : 0) * a.ldw + (ok ? k : 0), ok);
        } else {
          bs[r * DLDS + c2] = (n < N && k < K) ? a.W[(int64_t)n * a.ldw + k] : 0.0;
          bs[r * DLDS + c2 + 1] = (n < N && k + 1 < K) ? a.W[(int64_t)n * a.ldw + k + 1] : 0.0;
        }
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < DSTAGES - 1; ++st) {
    if (st < KT) load_stage(st, st);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<DSTAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + DSTAGES - 1;
      if (nk < KT) load_stage(nk % DSTAGES, nk);
      cp_async_commit();
    }
    const double* as = As + (kt % DSTAGES) * DBM * DLDS;
    const double* bs = Bs + (kt % DSTAGES) * DBN * DLDS;
#pragma unroll
    for (int kk = 0; kk < DBK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = as[(wm * 32 + i * 8 + g) * DLDS + kk + t];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = bs[(wn * 32 + j * 8 + g) * DLDS + kk + t];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // epilogue: r = y -/+ acc; r32/r64 stores; per-row sum of squares in fixed order
  double* red = dsm;   // reuse: [2][DBM]
  double rowsq[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + wm * 32 + i * 8 + g;
    double sq = 0.0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = n0 + wn * 32 + j * 8 + t * 2 + e;
        if (m < M && n < N) {
          double v = a.negate ? -acc[i][j][e] : acc[i][j][e];
          if (a.tblock) {
            const int64_t tb = a.tblock;
            const int64_t R = a.tb_R ? a.tb_R : tb, S = a.tb_S ? a.tb_S : tb;
            const int64_t img = a.tb_img ? a.tb_img : tb * tb;
            const int64_t bi = m / R, rr = m - bi * R;
            const int64_t off = bi * img + (int64_t)n * S + rr;
            if (a.Y) v = a.Y[off] + v;
            if (a.ax) v = fma(-a.alpha, a.ax[off], v);
            if (a.r32) a.r32[a.r32_img ? bi * a.r32_img + a.r32_off + (int64_t)n * S + rr : off] = (float)v;
            if (a.r64) a.r64[off] = v;
          } else {
            if (a.Y) v = a.Y[(int64_t)m * a.ldy + n] + v;
            if (a.ax) v = fma(-a.alpha, a.ax[(int64_t)m * a.ldy + n], v);
            if (a.r32) a.r32[(int64_t)m * a.ldr32 + n] = (float)v;
            if (a.r64) a.r64[(int64_t)m * a.ldr64 + n] = v;
          }
          sq += v * v;
        }
      }
    }
    sq += __shfl_xor_sync(0xffffffffu, sq, 1);
    sq += __shfl_xor_sync(0xffffffffu, sq, 2);
    rowsq[i] = sq;
  }
  if (a.part) {
    if (t == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) red[wn * DBM + wm * 32 + i * 8 + g] = rowsq[i];
    }
    __syncthreads();
    if (tid < DBM) {
      const int m = m0 + tid;
      if (m < M) a.part[(int64_t)m * gridDim.x + blockIdx.x] = red[tid] + red[DBM + tid];
    }
  }
}
}  // namespace

int gemm_f64_ntiles(int N) { return ceil_div(N, DBN); }

void gemm_f64(const Gemm64Args& a, cudaStream_t s) {
  const size_t smem = (size_t)DSTAGES * (DBM + DBN) * DLDS * sizeof(double);
  NMG_SMEM_OPTIN(dgemm_resid_kernel, smem);
  dim3 grid(ceil_div(a.N, DBN), ceil_div(a.M, DBM));
  dgemm_resid_kernel<<<grid, DNT, smem, s>>>(a);
}

}  // namespace nmg
