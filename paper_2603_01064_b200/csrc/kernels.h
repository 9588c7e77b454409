// Host-side launchers of the nmg device kernels (all enqueue on `s`).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace nmg {

// ---- GEMMs -----------------------------------------------------------------
// Operand conventions: X is [M][K] row-major (K contiguous, leading dim ldx).
// W is either K-major ([N][K], ldw) or N-major ([K][N], ldw).
// D[m][n] = (C ? C[m][n] : 0) - sign * sum_k X[m][k] W(n,k)     (sign = +1: residual form)
// Batched over blockIdx.z with element strides sx/sw/sc/sd.
struct Gemm32Args {
  int M, N, K, batch;
  const float* X; int64_t ldx, sx;
  const float* W; int64_t ldw, sw; bool w_kmajor;
  const float* C; int64_t ldc, sc;       // may be null (then D = acc)
  float* D; int64_t ldd, sd;
  bool negate;                            // D = C - acc (true) or C + acc (false)
  int tblock = 0;                         // >0: row m, col j stored at (m/tb)*tb*ldd + j*tb + m%tb
                                          //     (C read at the same place); batch must be 1
};
void gemm_f32(const Gemm32Args& a, cudaStream_t s);

// fp64 residual GEMM (DMMA): R = Y - X W^T-ish with the same conventions (W K-major,
// batch 1).  Writes r32 (fp32, ldr32) and optionally r64; writes per-row sums of r^2
// for each 64-wide column tile into part[m * n_tiles + tile] (fp64), deterministic.
struct Gemm64Args {
  int M, N, K;
  const double* X; int64_t ldx;
  const double* W; int64_t ldw;          // [N][K] row-major
  const double* Y; int64_t ldy;          // may be null (then R = -acc... used for apply)
  float* r32; int64_t ldr32;             // may be null
  double* r64; int64_t ldr64;            // may be null
  double* part;                           // may be null; [M][ceil(N/64)]
  bool negate;                            // R = Y - acc (true) / Y + acc
  int tblock = 0;                         // >0: transposed store within tb x tb blocks (see Gemm32Args);
                                          //     Y, ax, r32, r64 all use that mapping with ld = tb
  const double* ax = nullptr;             // optional: R -= alpha * ax (same location as R)
  double alpha = 0.0;
  // generalised block mapping (slab mode; 0 = tblock defaults): output (m, n) at
  // (m / tb_R) tb_img + n tb_S + m % tb_R; r32 (when r32_img != 0) at
  // (m / tb_R) r32_img + r32_off + n tb_S + m % tb_R (a halo'd fp32 slab)
  int tb_R = 0, tb_S = 0;
  int64_t tb_img = 0, r32_img = 0, r32_off = 0;
};
int gemm_f64_ntiles(int N);
void gemm_f64(const Gemm64Args& a, cudaStream_t s);

// fp64-accurate residual via exact int8 digit products on tcgen05 (ozaki.cu)
struct OzakiArgs {
  int M, N, K;                           // N % 64 == 0, K % 64 == 0
  const double* Y; int64_t ldy;
  float* r32; int64_t ldr32;             // may be null
  double* r64; int64_t ldr64;            // may be null
  double* part;                          // may be null; [M][N/64]
  const int* ex;                         // [M] row exponents of X
  const int* ew;                         // [N] row exponents of W
  // 2D Kronecker passes: tblock > 0 = transposed store within tblock x tblock blocks (Y, ax,
  // r32, r64 all at that location); plus: store +X W^T (pass 1) instead of Y - X W^T;
  // ax: optional -alpha ax term (pass 2)
  int tblock = 0;
  bool plus = false;
  const double* ax = nullptr;
  double alpha = 0.0;
  // slab mode: generalised block mapping (as Gemm64Args: (m / tb_R) tb_img + col tb_S + m % tb_R,
  // r32 at (m / tb_R) r32_img + r32_off + ...) and the first W row (rows wrow0 .. wrow0 + N)
  int tb_R = 0, tb_S = 0;
  int64_t tb_img = 0, r32_img = 0, r32_off = 0;
  int wrow0 = 0;
  // per ozaki_bn()-row tile of W (absolute W rows): the K blocks [x, y) (units of ozaki_bk())
  // outside which every digit of the tile is zero; null = all K blocks
  const int2* krange = nullptr;
};
int ozaki_digits();
int ozaki_bk();   // K block of the digit tensor maps (box K; 32: SWIZZLE_32B, 64: SWIZZLE_64B)
int ozaki_bn();   // N tile (box rows of the W digit maps; the ||r||^2 partials per row are N / ozaki_bn())
// digit planes [S][plane / K rows][K]: plane = (rows allocated per plane) * K
void ozaki_split_rows(int M, int K, const double* X, int64_t ldx, int8_t* dig, int64_t plane, int* ex,
                      cudaStream_t s);
void ozaki_resid(const CUtensorMap* mx, const CUtensorMap* mw, const OzakiArgs& a, cudaStream_t s);

// tcgen05 3xTF32 GEMM: D = C -/+ X W^T with X = Xh + Xl ([M][K], tensor maps with box
// {16, 128}) and W = Wh + Wl ([N][K], box {16, 256}), SWIZZLE_64B, fp32 row-major C/D.
struct TcGemmArgs {
  int M, N, K;
  const float* C; int64_t ldc;           // may be null
  float* D; int64_t ldd;                 // fp32 output (ignored when Dh is set)
  bool negate;
  int tblock = 0;                        // >0: transposed store within tblock x tblock blocks
  float* Dh = nullptr; float* Dl = nullptr;   // optional tf32 hi/lo split output (no C)
  // FP16x3 variant only: X row m was split as x S_m, W row n as w T_n; xinv[m] = 1 / S_m,
  // winv[n] = 1 / T_n (powers of two, so acc xinv winv is exact)
  const float* xinv = nullptr;
  const float* winv = nullptr;
  // FP16x3, 256-wide tiles: W maps with box rows 128 (host pointers) -> CTA pairs along M
  // multicast the W tile (cluster 1 x 2), when the number of M tiles is even
  const CUtensorMap* wh_mc = nullptr;
  const CUtensorMap* wl_mc = nullptr;
  // optional, per 64-row tile of W: the K elements [x, y) (multiples of 32) outside which the
  // tile's hi and lo planes are all zero (those K blocks are skipped; null = all of K)
  const int2* krange = nullptr;
};
// 2D Kronecker apply passes on tcgen05 (kron_tc.cu).  A = fp32 [M][n] rows (TMA map, box
// {16, 128}, SWIZZLE_64B), W = tf32 hi/lo [n][n] (box {16, kron_tile_n(n)}).
enum { KRON_T = 0, KRON_RESID = 1 };
struct KronArgs {
  int M, n;                    // M = nrhs * n rows
  int mode;                    // KRON_T: D = blockT(A W^T); KRON_RESID: D = Cin -/+ (blockT(A W^T) + alpha S(X))
  float* D;                    // output [nrhs][n][n]
  const float* X = nullptr;    // KRON_RESID: image for the mass stencil S = Q X Q^T
  const float* Cin = nullptr;  // KRON_RESID: may be null (0), may alias D
  const float* Q = nullptr;    // [n][n], half-bandwidth hb
  int hb = 0;
  float alpha = 0.f;
  bool negate = false;
  // slab-sharded mode (0 = whole image): each image is stored as R rows (global rows r0 ..
  // r0 + R - 1) plus H halo rows above and below; img = per-image stride of X / Cin / D.
  // Pass 1 reads all R + 2H stored rows (M = nrhs (R + 2H)) and writes T[b][i1][R] for its
  // slab only; pass 2 (A = the gathered T, M = nrhs n) computes the slab's R output rows
  // (W rows r0 .. r0 + R - 1, W map box rows kron_tile_n(R)).
  int R = 0, H = 0, r0 = 0;
  int64_t img = 0;
  // optional, per 64-row tile of W (absolute rows): the K elements [x, y) (multiples of 16)
  // outside which the tile's tf32 hi and lo values are all zero (skipped; null = all of K)
  const int2* krange = nullptr;
};
int kron_tile_n(int n);
bool kron_supported(int n, int hb);
void kron_tc(const CUtensorMap* A, const CUtensorMap* Wh, const CUtensorMap* Wl, const KronArgs& a, int sms,
             cudaStream_t s);
// bn = 256 or 64 (tile width; W maps must use box rows = bn)
void tc_gemm(const CUtensorMap* xh, const CUtensorMap* xl, const CUtensorMap* wh, const CUtensorMap* wl,
             const TcGemmArgs& a, cudaStream_t s, int bn);
// same with f16 hi/lo operands (kind::f16, tensor maps with f16 elements, box {32, rows}):
// twice the tensor rate of 3xTF32, same fp32-accurate result (2^-22 per product)
void tc_gemm_f16(const CUtensorMap* xh, const CUtensorMap* xl, const CUtensorMap* wh, const CUtensorMap* wl,
                 const TcGemmArgs& a, cudaStream_t s, int bn);
// per-row power-of-two scaled f16 hi/lo split: S = 2^floor(log2(2^14 / max_k |x[m][k]|))
void split_f16_rows(int rows, int K, const float* x, uint16_t* hi, uint16_t* lo, float* xinv, cudaStream_t s);
int tc_gemm_block_m();
// tile width heuristic: 256 when that already fills the GPU, else 64
inline int tc_pick_bn(int M, int N, int num_sms) {
  const int t256 = ((M + 127) / 128) * ((N + 255) / 256);
  return (N >= 256 && t256 >= (num_sms * 4) / 5) ? 256 : 64;
}
void split_tf32(int64_t count, const float* x, float* hi, float* lo, cudaStream_t s);

// ---- 1D smoother: norm -> CNN (3 layers, C=16, k=5) -> F' -> update ----------
// 1D smoother weights by value (smooth1d_f16 reads them as constant-bank operands):
// w0 [16][5], b0 [16] (pre-multiplied by in_scale), b1 [16], w2 [16][5], b2 (state_dict order)
struct Smooth1dW {
  float w0[80], b0[16], b1[16], w2[80], b2;
};
struct Smooth1dArgs {
  int n, nrhs;
  const float* b; int64_t ldb;     // input rows
  float* x; int64_t ldx;           // output rows
  const float* params;             // 1473 floats, state_dict order
  const float2* twiddle; int tw_n; // exp(-2 pi i k / tw_n), k < tw_n/2
  bool normalize;                  // h = s N(b/s) (true) or h = N(b) (debug)
  bool filter;                     // apply F'_l
  bool accumulate;                 // x += (true) or x = (false)
  float* xh = nullptr;             // optional: tf32 hi/lo split of the updated x (for the GEMM)
  float* xl = nullptr;
  // smooth1d_f16 only: layer-2 weights (f16 hi/lo, stacked per tap [5][2][32][8], scaled by T),
  // a1 scale S (a1 is split as a1 S) and 1 / (S T)
  const uint16_t* wb = nullptr;
  float in_scale = 1.f, d_scale = 1.f;
  uint16_t* x16h = nullptr;        // optional (filter path): per-row scaled f16 hi/lo split of the
  uint16_t* x16l = nullptr;        // updated x and 1 / scale, as split_f16_rows
  float* xinv = nullptr;
  Smooth1dW w{};                   // smooth1d_f16 only
};
void smooth1d(const Smooth1dArgs& a, cudaStream_t s);
// same step with the 16 -> 16 layer on tcgen05 (FP16x3, n % 128 == 0), smooth1d_f16.cu
void smooth1d_f16(const Smooth1dArgs& a, cudaStream_t s);
size_t smooth1d_smem(int n);

// ---- 1D transfers (reading R4) ------------------------------------------------
void restrict1d(int nrhs, int n_f, const float* f, int64_t ldf, float* c, int64_t ldc, cudaStream_t s);
void prolong_add1d(int nrhs, int n_c, const float* c, int64_t ldc, float* f, int64_t ldf, cudaStream_t s);

// ---- 1D filter only (debug op) ------------------------------------------------
void filter1d(int n, int nrhs, const float* in, float* out, const float2* tw, int tw_n, cudaStream_t s);

// ---- coarse solve: Cholesky factor applied by forward/back substitution ---------
// same result with the explicit fp64 inverse A_L^{-1} (symmetric [nc][nc], nc <= 256)
void coarse_inv_apply(int nc, int nrhs, const double* Ainv, const float* y, int64_t ldy, float* x, int64_t ldx,
                      cudaStream_t s, float* xh = nullptr, float* xl = nullptr);
void coarse_chol_solve(int nc, int nrhs, const double* Lrow, const double* Lcol,
                       const float* y, int64_t ldy, float* x, int64_t ldx, cudaStream_t s,
                       float* xh = nullptr, float* xl = nullptr);

// ---- outer (fp64) helpers --------------------------------------------------------
void row_norms_f64(int nrhs, int N, const double* y, int64_t ldy, double* out, double* work /*[nrhs][64]*/,
                   cudaStream_t s);
void relres_finalize(int nrhs, int ntiles, const double* part, const double* ynorm, double* relres,
                     double tol, uint8_t* active, cudaStream_t s, int rows_per_rhs = 1);
void update_x(int nrhs, int N, double* x, int64_t ldx, const float* d, int64_t ldd,
              const uint8_t* active, cudaStream_t s);
void f64_to_f32(int64_t count, const double* in, float* out, cudaStream_t s);
void f32_to_f64(int64_t count, const float* in, double* out, cudaStream_t s);
// rows of N doubles: dst[i] = src[map[i]] (gather) or dst[map[i]] = src[i] (scatter)
void permute_rows(int rows, int64_t N, const double* src, double* dst, const int32_t* map, bool scatter,
                  cudaStream_t s);

// ---- 2D level operations (level2d.cu) -------------------------------------------
struct Cnn2dArgs {
  int n, nrhs, C;
  const float* b;          // input [nrhs][n][n]
  const double* norms;     // per-RHS ||b|| (null: h = N(b), debug)
  const float* params;     // device layout: w0, b0, w1 [c][t2][t1][o], b1, w2 [c][t2][t1][o], b2, w3, b3
  float2* Z;               // if set: write (h, 0) for the filter passes
  float* x;                // else: x = h / x += h
  bool accumulate;
};
void cnn2d(const Cnn2dArgs& a, cudaStream_t s);
int cnn2d_smem(int C);
void restrict2d(int nrhs, int n_f, const float* f, float* c, cudaStream_t s);
void prolong_add2d(int nrhs, int n_c, const float* c, float* f, cudaStream_t s);
void qstencil(int nrhs, int n, int hb, float alpha, const float* Q, const float* X, const float* C, float* D,
              cudaStream_t s);
void norms_f32(int nrhs, int64_t N, const float* x, double* part, int chunks, double* out, cudaStream_t s);
// level filter hat F'_l on the per-RHS layout written by zput (common.cuh): Z_b = [n/2][n] complex.
// norms (may be null): per-RHS ||b||; the writers store N(u) and x gets ||b|| F'(N(u))
void filter2d(int nrhs, int n, float2* Z, const float2* tw, int tw_n, float* x, bool accumulate, cudaStream_t s,
              const double* norms, bool rows_done = false);
// strip_combine fused with filter2d's forward row FFTs: Z_b (b = zb0 ..) of the chunk's RHS hold
// the row-transformed N(u) (0 where ||b|| = 0)
void combine_rows_fft(int n, int nrhs, const float* q, const float4* qe, const double* norms, float2* Z, int zb0,
                      const float2* tw, int tw_n, cudaStream_t s);
// per-RHS sum of squares (no sqrt) of N values at x + b img + off
void sumsq_f32(int nrhs, int64_t N, const float* x, int64_t img, int64_t off, double* part, int chunks, double* out,
               cudaStream_t s);
// slab-sharded level filter (level2d.cu; steps in the comment there): Zs [nrhs][R/2][n];
// all-to-all chunks of filter2d_slab_chunk(n, W) complex slots per (RHS, local complex row)
int filter2d_slab_chunk(int n, int W);
void filter2d_slab_rows(int n, int nrhs, int R, float2* Zs, const float2* tw, int tw_n, cudaStream_t s);
void filter2d_slab_pack(int n, int nrhs, int R, int W, float2* Zs, float2* buf, bool unpack, cudaStream_t s);
void filter2d_slab_cols(int n, int nrhs, int R, int W, int rank, float2* buf, const float2* tw, int tw_n,
                        cudaStream_t s);
void filter2d_slab_inverse(int n, int nrhs, int R, float2* Zs, const float2* tw, int tw_n, float* x, int64_t ximg,
                           int64_t xoff, bool accumulate, const double* norms, cudaStream_t s);
void real_to_complex(int nrhs, int n, const float* x, float2* Z, cudaStream_t s);

// ---- 2D CNN, FP16x3 tcgen05 column-strip kernels (conv_strip.cu), n % 128 == 0, C = 32/48 --
// Layers 1+2 (strip_l12): b -> a2 (scaled f16 hi/lo, [b][y][x][C]); layers 3+4 (strip_l34,
// a2 through the 5D tensor maps) -> Q (float4 [b][y][x]: per-t1 partial sums of layer 4);
// strip_combine: h = s (b3 + Q0(x-1) + Q1(x) + Q2(x+1)) -> Z or x.
struct StripArgs {
  int n, nrhs, C, ysplit;
  const float* b;             // l12: input [nrhs][n][n]
  const double* norms;        // l12: per-RHS ||b|| (null: 1)
  const float* w_in;          // l12: w0 [C][9] followed by b0 [C]
  const float* w_out;         // l34: w3 [C][9]
  const uint16_t* wh;         // hidden-layer weights x T, f16 hi/lo, canonical [3C/8][3C][8]
  const uint16_t* wl;
  const float* bias;          // hidden-layer bias [C]
  float in_scale;             // l12: S1 (a1 is split as a1 S1)
  float out_scale;            // l12: S2 (a2 is stored as a2 S2)
  float d_scale;              // 1 / (S T) of this layer
  uint16_t* out_h;            // l12: a2 hi/lo
  uint16_t* out_l;
  float* q;                   // l34: the CNN output h without its strip-edge terms, [nrhs][h][n]
  float4* qe;                 // l34: strip-edge records [nrhs][h][n / 128] (see strip_combine)
  const float* b3;            // l34: last-layer bias (1 value)
  const uint16_t* w4;         // l34: layer-4 weights x T4, f16 hi then lo, [C/8][16][8] (row t2*3+t1)
  float a3_scale;             // l34: S3 (a3 is split as a3 S3)
  float d4_scale;             // l34: 1 / (S3 T4)
  int h = 0;                  // stored rows per image (0: n); slab mode: R + 2 halo rows (the
                              // halo rows' outputs are discarded)
  int ylo = 0, yhi = 0;       // image rows [ylo, yhi) (yhi 0: h); rows outside are the zero
                              // padding of every layer (slabs at the image's top / bottom edge)
};
int strip_ysplit(int n, int nrhs, int num_sms, int hg = 0);
void strip_l12(const StripArgs& a, int num_sms, cudaStream_t s);
void strip_l34(const CUtensorMap* mh, const CUtensorMap* ml, const StripArgs& a, int num_sms, cudaStream_t s);
void strip_combine(int n, int nrhs, const float* q, const float4* qe, const double* norms, float2* Z, int zb0,
                   float* x, bool accumulate, cudaStream_t s, int hg = 0, int hh = 0);


// ---- FNO smoother (fno.cu; Appendix A, Table 6) -------------------------------
struct FnoLayer {
  const float2* R;            // spectral weights [modes][c_in][c_out] complex
  const float* W;             // W convolution [c_out][c_in][ks](x ks)
  const float* B;             // bias [c]
  // tensor-core W-convolution (fno_tc.cu): W as [o][tap][c] tf32 hi/lo, box {16, 64}
  const CUtensorMap* tWh = nullptr;
  const CUtensorMap* tWl = nullptr;
};
// W-convolution + bias + GELU on tcgen05 (3xTF32 implicit GEMM, fno_tc.cu)
struct FnoConvArgs {
  int dim, n, c, ks, nrhs;
  int lbx;                    // 2D: log2 of the output box width bx (box bx x 128 / bx pixels)
  bool rows;                  // 2D, n >= 128: row-halo variant (rank-5 no-swizzle input maps, x taps as
                              // descriptor shifts)
  const float* bias;          // [c]
  float* Z1;                  // [nrhs][c][N]: the spectral branch on entry, the layer output on exit
  float* Xh_out; float* Xl_out;   // next layer's channels-last tf32 hi/lo input [nrhs][N][c] (null: last layer)
};
bool fno_tc_ok(int dim, int n, int c);
bool fno_tc_rows(int dim, int n, int ks);
void fno_tc_box(int n, int* bx, int* by);
void fno_lift_cl(int nrhs, int c, int64_t N, const float* in, const double* norms, const float* lw, const float* lb,
                 float* Xh, float* Xl, cudaStream_t s);
void fno_conv_tc(const CUtensorMap* xh, const CUtensorMap* xl, const CUtensorMap* wh, const CUtensorMap* wl,
                 const FnoConvArgs& a, cudaStream_t s);
struct FnoArgs {
  int dim, n, nrhs, c, L, k, ks;
  const float* in;            // b [nrhs][N]
  const double* norms;        // ||b|| per RHS (null: 1, the debug CNN op)
  const float* lift_w;        // [c]
  const float* lift_b;        // [c]
  const float* proj_w;        // [c]
  float proj_b;
  FnoLayer layer[8];
  float* Z0; float* Z1;       // activations [nrhs][c][N]
  float2* T;                  // 2D: [nrhs][c][n][k]
  float2* Zh; float2* Yh;     // [nrhs][modes][c]
  const float2* tw; int tw_n;
  // output: 1D x (+)= ||b|| F'(h) (filter) or ||b|| h; 2D: Zf (level-filter input, zput) when set,
  // else x (+)= ||b|| h
  float* x; bool accumulate, filter;
  float2* Zf = nullptr; int zb0 = 0;
  // tensor-core W-convolution: channels-last tf32 hi/lo layer inputs (ping-pong pairs) and their
  // tensor maps; null tX: the fp32 SIMT convolution kernels
  const CUtensorMap* tXh[2] = {nullptr, nullptr};
  const CUtensorMap* tXl[2] = {nullptr, nullptr};
  float* Xh[2] = {nullptr, nullptr};
  float* Xl[2] = {nullptr, nullptr};
  bool tc_rows = false;       // the X maps are the row-halo variant's rank-5 maps
};
void fno_forward(const FnoArgs& a, cudaStream_t s);
int fno_launches(int dim, int L, bool tc);
size_t fno_conv_smem(int dim, int c, int ks);

// ---- NMG_PREC_FP64: the whole cycle of one RHS per CTA in one launch (cycle64.cu; 1D, n <= 1024)
struct Cycle64Args {
  int n, L, nrhs, nu1, nu2;
  bool filter;
  const double* A[8];         // fp64 Galerkin operators of the smoothed levels 0 .. L-2 (A[0] = G + alpha I)
  const double* Ainv;         // fp64 (A^(L))^{-1}
  const float* W[8];          // CNN parameters per smoothed level (state_dict order)
  const double* y;            // [nrhs][n]
  double* x;                  // [nrhs][n], in/out
  double* relres;             // [nrhs] or null
  double tol;
  const uint8_t* active_in;   // null: every RHS cycles
  uint8_t* active_out;        // null or [nrhs]: relres > tol
  bool do_cycle;              // run the cycle (else only the relative residual)
  bool relres_after;          // relres of the output x (nmg_solve) instead of the input x (nmg_vcycle)
  // coarse sub-cycle of the mixed path: x_l0 = NMGF(0, y_l0) with fp32 y / x ([nrhs][n]); the
  // levels of this call are the hierarchy's l0 .. L-1 (n, L, A, W, Ainv of that sub-hierarchy)
  const float* yf = nullptr;
  float* xf = nullptr;
};
size_t cycle64_smem(int n, int L);
void cycle64(const Cycle64Args& a, cudaStream_t s);

// ---- slab-sharded single-system mode (slab.cu): slabs of R rows + H halo rows per image --
void restrict_slab(int nrhs, int n_c, int Rc, int r0c, const float* f, int64_t fimg, int64_t foff, float* c,
                   int64_t cimg, int64_t coff, cudaStream_t s);
void prolong_slab(int nrhs, int n_c, int Rf, int r0f, const float* c, int64_t cimg, int64_t coff, float* f,
                  int64_t fimg, int64_t foff, cudaStream_t s);
void halo_pack(int nrhs, int n, int R, int H, const float* x, float* send, cudaStream_t s);
void halo_unpack(int nrhs, int n, int R, int H, int rank, int W, const float* recv, float* x, cudaStream_t s);
void update_slab(int nrhs, int64_t N, double* x, const float* d, int64_t img, int64_t off, const uint8_t* active,
                 cudaStream_t s);
void part_sums(int nrhs, int64_t cnt, const double* part, double* out, cudaStream_t s);
void relres_sums(int nrhs, const double* rsq, const double* ysq, double* relres, double tol, uint8_t* active,
                 cudaStream_t s);
void sqrt_inplace(int n, double* v, cudaStream_t s);
void sumsq_f64(int nrhs, int64_t N, const double* y, double* part /*[nrhs][64]*/, double* out, cudaStream_t s);

}  // namespace nmg
