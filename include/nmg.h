/*
 * nmg.h -- C ABI of the B200-native batched neural-multigrid solve
 *          (arxiv 2603.01064, "A level-wise training scheme for learning
 *          neural multigrid smoothers with application to integral equations").
 *
 * What the library computes (PAPER.md = P):
 *   Solve A x = y for many right-hand sides y,
 *   A = G + alpha I with G a structured smooth-kernel operator (P:51, P:473,
 *   P:569), by repeated NMGF cycles x^tau = NMGF(x^{tau-1}, y), x^0 = 0
 *   (Alg 3 "NMGF1d" P:315-339; Alg 4 "NMGF2d" P:373-401) until the
 *   relative residual ||y - A x||_2 / ||y||_2 <= tol (1e-6).
 *   Each level l < L: b = y_l - A^(l) x*, h = N_theta_l(b/||b||)||b||,
 *   x = x* + F'_l(h) (level filter P:305), y_{l+1} = I_l^{l+1}(y_l - A^(l) x)
 *   (P:331), recurse from 0 on the Galerkin operator, prolongate,
 *   then nu2 post-smoothing steps (reading R9).  Level L: exact solve.
 *
 * Conventions (all functions):
 *   - Level numbers are 1-based as in the paper: level 1 is the finest grid,
 *     level L = desc.levels the coarsest (exact solve).
 *   - Vector layout is RHS-major, contiguous: 1D [nrhs][n_l]; 2D [nrhs][n_l][n_l]
 *     with each RHS a column-major n_l x n_l matrix (element (i1,i2) at
 *     i1 + n_l*i2, the Vec convention of P:363).
 *   - Pointers documented "device" must be cudaMalloc'd memory on desc.device;
 *     "host" pointers are ordinary host memory (pinned preferred for *_host).
 *   - Ownership: the caller owns every buffer it passes; the library deep-copies
 *     operator factors and weights at create/load time and owns all device
 *     workspaces.  nmg_vcycle / nmg_solve never allocate.
 *   - Streams: device-pointer calls enqueue on the caller's stream and return
 *     without synchronising, except nmg_solve, which synchronises once per cycle
 *     and returns when done.
 *   - Errors: no function throws or aborts across the ABI.  Every call returns
 *     an nmg_status; nmg_last_error() gives a thread-local message.  After
 *     NMG_ERR_CUDA the handle is poisoned and must be destroyed.
 *   - Threading: a handle is used by one host thread / stream at a time.
 *   - There is no CPU fallback: without a visible sm_100 device,
 *     nmg_create_hierarchy fails with NMG_ERR_CUDA.
 */
#ifndef NMG_H
#define NMG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct nmg_hierarchy nmg_hierarchy;   /* opaque, library-owned device state */

typedef enum {
  NMG_OK = 0,
  NMG_ERR_INVALID_ARG = 1,  /* null pointer, n not a power of two, n_L < 2, alpha <= 0,
                               nrhs > max_rhs, level out of range                         */
  NMG_ERR_SHAPE = 2,        /* weight count inconsistent with the architecture            */
  NMG_ERR_NOT_SPD = 3,      /* Cholesky pivot <= 0 at the coarsest level (index in msg)   */
  NMG_ERR_NO_WEIGHTS = 4,   /* a cycle was requested while a level 1..L-1 has no smoother */
  NMG_ERR_NONFINITE = 5,    /* NaN/Inf residual; report->fail_cycle / fail_rhs are set    */
  NMG_ERR_CUDA = 6,         /* CUDA runtime / launch failure, or no sm_100 device         */
  NMG_ERR_OOM = 7,          /* device allocation failed                                   */
  NMG_ERR_UNSUPPORTED = 8,  /* architecture / mode not implemented                        */
  NMG_ERR_DIVERGED = 9,     /* opt-in (desc.divergence_check): an active RHS's relres stayed
                               above 10x its initial relres for 5 consecutive cycles
                               (SPEC.md:545 rule); report->fail_cycle / fail_rhs are set     */
  NMG_ERR_NCCL = 10         /* collective failure (NCCL call or asynchronous communicator
                               error, or an emulated peer rank that failed / timed out)      */
} nmg_status;

/* Precision of the cycle (reading R14). */
enum {
  NMG_PREC_MIXED = 0,   /* fp64 outer residual, convergence test and update around an inner
                           NMGF cycle in fp32-accurate split arithmetic on the tensor cores
                           (correction form x + NMGF(0, y - A x), pin P11) -- default       */
  NMG_PREC_FP64 = 1     /* every step of the cycle in fp64 except the CNN's own arithmetic
                           (fp32 weights and activations, BASELINE configs[0]); 1D only,
                           n <= 1024 (one fused kernel per cycle, one CTA per RHS)        */
};

/* Kernel-selection knobs (all 0 = the default production path).  They exist for A/B timing
 * and for the parity tests of the alternative kernels; none changes what is computed beyond
 * floating-point rounding order. */
typedef struct {
  int32_t lanes;          /* RHS lanes: 0 = auto (1D: up to 4 lanes of >= 256 RHS; 2D: 2 lanes
                             while max_rhs*n^2 <= 2^26), 1 = off, K >= 2 = K lanes           */
  int32_t no_graphs;      /* 1: launch every kernel eagerly instead of replaying the cycle's
                             captured CUDA graph                                             */
  int32_t coarse_subst;   /* 1: coarsest solve by forward/back substitution with the Cholesky
                             factor instead of the explicit fp64 inverse A_L^{-1}            */
  int32_t fp64_dmma;      /* 1: fp64 outer residual on DMMA instead of Ozaki int8 digits      */
  int32_t simt_gemm;      /* 1: inner operator applies on the SIMT fp32 GEMM (no tcgen05)     */
  int32_t ffma_cnn;       /* 1: CNN smoother on the FFMA kernels (no tcgen05)                 */
  int32_t no_kron;        /* 1 (2D): Kronecker pair as two plain GEMMs + a stencil pass       */
  int32_t host_chunks;    /* nmg_vcycles_host: 0 = pipelined per RHS lane (default when the
                             handle has lanes), else that many RHS chunks (1..16)            */
  int32_t fused_coarse;   /* N > 0 (1D): the levels with n_l <= N run as ONE fused fp64 sub-cycle
                             kernel per RHS (cycle64) instead of per-level launches (opt-in:
                             slower than the batched kernels for n_l >= 256)                  */
  int32_t no_compaction;  /* 1: nmg_solve keeps cycling the whole batch (converged RHS masked)
                             instead of gathering the active RHS into a smaller batch; 2:
                             gather whenever one RHS converged (parity tests)               */
  int32_t dense_k;        /* 1: the operator contractions run every K block, including the blocks
                             whose split operator digits are all zero (the Gaussian operators'
                             far-off-diagonal blocks; skipping them is exact) */
  int32_t no_balance;     /* 1: load the CNN weights as given instead of lifting hidden channels
                             whose activation bound lies > 2^4 below their layer's largest by a
                             power of two (an exactly equivalent network, see nmg_api.cu)    */
  int32_t simt_fno;       /* 1: FNO W-convolution on the fp32 SIMT kernels instead of the tcgen05
                             3xTF32 implicit GEMM (fno_tc.cu); 2: tcgen05, box variant only (no
                             row-halo kernel for 2D n >= 128)                                  */
} nmg_tuning;

/* Problem descriptor (SPEC ProblemSpec analogue). */
typedef struct {
  int32_t dim;          /* 1 or 2                                                          */
  int32_t n;            /* finest points per axis, power of two, n >> (levels-1) >= 2      */
  int32_t levels;       /* L >= 1; levels 1..L-1 carry a smoother, level L is exact        */
  double  alpha;        /* A = G + alpha I, alpha > 0 (Tikhonov weight)         */
  int32_t nu1, nu2;     /* pre/post smoothing steps per level (paper nu2 = 0, P:233;
                           BASELINE nu1 = nu2 = 1)                                         */
  int32_t level_filter; /* 1: Alg 3/4 with F'_l; 0: Alg 2          */
  int32_t max_rhs;      /* workspace sizing: largest nrhs ever passed                      */
  int32_t device;       /* CUDA ordinal                                                    */
  int32_t precision;    /* NMG_PREC_MIXED (0, default) or NMG_PREC_FP64                    */
  int32_t divergence_check; /* 1: nmg_solve returns NMG_ERR_DIVERGED per SPEC.md:545      */
  const nmg_tuning *tuning; /* host, may be NULL (defaults); copied at create              */
} nmg_problem_desc;

/* CNN smoother architecture (reading R7): n_layers convolutions 1 -> C -> ... -> C -> 1,
 * kernel ksize (per axis), stride 1, zero "same" padding, bias, ReLU between layers,
 * none after the last.  Supported: 1D (3, 16, 5); 2D (4, 32, 3) and (4, 48, 3). */
typedef struct {
  int32_t n_layers, channels, ksize;
} nmg_cnn_arch;

/* FNO smoother architecture (the paper's own smoother: PAPER.md section 3.1 P:208-216,
 * Appendix A; per-grid values in Table 6): lift 1 -> width (pointwise),
 * n_layers Fourier layers GELU(DFT^{-1}(R (.) DFT(Z)) + W * Z + B) with R a complex width x width
 * mixing of the `modes` lowest frequencies per axis (2D: i1-modes 0..modes-1 x i2-modes
 * 0..modes-1 and n-modes..n-1) and W a ksize (x ksize) convolution with zero "same" padding,
 * then proj width -> 1 (pointwise).  Constraints: width <= 64, 1 <= n_layers <= 8, ksize odd
 * <= 7, modes a power of two <= n_l / 4. */
typedef struct {
  int32_t width, n_layers, modes, ksize;
} nmg_fno_arch;

/* Solve report (SPEC SolveReport analogue), caller-allocated HOST memory. */
typedef struct {
  int32_t *cycles;       /* [nrhs] cycles applied to each RHS                              */
  uint8_t *converged;    /* [nrhs] 1 if relres <= tol was reached                          */
  double  *history;      /* [nrhs][max_cycles+1] relres after each cycle (index 0 = x0),
                            NaN after the RHS froze; may be NULL                            */
  double   wall_seconds; /* written: elapsed device time of the cycle loop                 */
  int32_t  total_cycles; /* written: cycles executed for the batch                         */
  int32_t  fail_cycle;   /* written on NMG_ERR_NONFINITE, else -1                          */
  int32_t  fail_rhs;     /* written on NMG_ERR_NONFINITE, else -1                          */
} nmg_report;

/* Build the level hierarchy (host fp64 Galerkin chain A^(l+1) = I_l^{l+1} A^(l) I_{l+1}^l,
 * P:160; coarsest Cholesky; device uploads).  Every device workspace the cycle entries use
 * is allocated here (sized by max_rhs), including the staging of nmg_vcycles_host.
 *   factors (host, read-only, copied):
 *     dim 1: G, n*n doubles row-major, symmetric                 (A = G + alpha I)
 *     dim 2: B then C, each n*n doubles row-major, symmetric:
 *            G = B (x) C, i.e. G Vec(X) = Vec(C X B^T)
 *   out: receives the handle.  Errors: INVALID_ARG, NOT_SPD, CUDA, OOM. */
nmg_status nmg_create_hierarchy(const nmg_problem_desc *desc, const double *factors,
                                nmg_hierarchy **out);

/* Load the smoother theta_l of level `level` (1..L-1), fp32 parameters in PyTorch
 * state_dict order (w0, b0, w1, b1, ...; conv weights [out][in][k] / [out][in][k2][k1]).
 * params: host, n_params floats, copied.  Loading a level twice replaces it; the cycle graphs
 * captured before the reload are discarded (the call synchronises the device first).
 * Errors: INVALID_ARG, SHAPE, UNSUPPORTED, CUDA. */
nmg_status nmg_load_smoother_weights(nmg_hierarchy *h, int32_t level, const nmg_cnn_arch *arch,
                                     const float *params, size_t n_params);

/* Load an FNO smoother theta_l for level `level` (1..L-1) instead of a CNN; params: host fp32,
 * copied, in the order lift.w [c][1], lift.b [c]; per Fourier layer: R as (re, im) pairs
 * [modes][c_in][c_out][2] (1D) or [2 modes][modes][c_in][c_out][2] (2D; i2-mode rows 0..modes-1
 * then n-modes..n-1), W [c_out][c_in][ksize](x ksize), B [c]; proj.w [1][c], proj.b [1].
 * Allocates the level's FNO workspaces (sized by max_rhs, RHS-chunked); replaces whatever
 * smoother the level had; drops captured cycle graphs.  Errors: INVALID_ARG, SHAPE,
 * UNSUPPORTED, OOM, CUDA. */
nmg_status nmg_load_fno_weights(nmg_hierarchy *h, int32_t level, const nmg_fno_arch *arch,
                                const float *params, size_t n_params);

/* One cycle x <- NMGF(x, y) for nrhs right-hand sides (one tau step), computed in
 * correction form x + NMGF(0, y - A x) (pin P11): fp64 outer residual, fp32-accurate
 * inner cycle, fp64 update.  y, x: device fp64 [nrhs][N]; x in/out.  Asynchronous. */
nmg_status nmg_vcycle(nmg_hierarchy *h, int32_t nrhs, const double *y, double *x, void *stream);

/* Outer iteration from the x passed in (x0 = 0 for the paper's solve) until every
 * RHS has relres <= tol or max_cycles; converged RHS are frozen.  y, x: device
 * fp64 [nrhs][N]; rep: host (may be NULL).  Synchronises once per cycle (and polls the
 * communicator's asynchronous error state on a slab handle).  Once the converged RHS are at
 * least 1/8 of the cycling batch (and 2^22 values), the still-active ones are gathered into the
 * handle's staging buffers and cycle as a smaller batch (their arithmetic does not depend on the
 * batch; nmg_tuning.no_compaction = 1 keeps the whole batch); x holds every RHS's final iterate
 * when the call returns (not while it runs).
 * Errors: NONFINITE / DIVERGED (rep->fail_*), NO_WEIGHTS, CUDA, NCCL. */
nmg_status nmg_solve(nmg_hierarchy *h, int32_t nrhs, const double *y, double *x, double tol,
                     int32_t max_cycles, nmg_report *rep, void *stream);

/* Same as nmg_vcycle repeated `cycles` times, but y and x are HOST buffers: the call
 * copies y and x host->device, runs the cycles and copies x back (end-to-end path).
 * relres (host, may be NULL) receives [nrhs] fp64 relative residuals of the input x
 * measured before the last cycle.  The copies are pipelined with the cycles (per RHS lane
 * on a handle with lanes, else per RHS chunk).  Synchronous. */
nmg_status nmg_vcycles_host(nmg_hierarchy *h, int32_t nrhs, const double *y_host, double *x_host,
                            int32_t cycles, double *relres_host, void *stream);

/* fp64 residual r = y - A x at level 1 and relres = ||r||/||y|| per RHS.
 * y, x: device fp64 [nrhs][N]; r: device fp64 [nrhs][N] or NULL; relres: device fp64
 * [nrhs] or NULL.  Asynchronous. */
nmg_status nmg_residual(nmg_hierarchy *h, int32_t nrhs, const double *y, const double *x,
                        double *r, double *relres, void *stream);

/* Diagnostic single-operator entry for parity tests (fp32 device buffers unless noted).
 * level is 1-based.  op:
 *   NMG_OP_APPLY     out = A^(l) in                          in/out [nrhs][N_l]
 *   NMG_OP_RESIDUAL  out = out - A^(l) in  (out holds y_l)    in/out [nrhs][N_l]
 *   NMG_OP_RESTRICT  out = I_l^{l+1} in                       in [nrhs][N_l], out [nrhs][N_{l+1}]
 *   NMG_OP_PROLONG   out = out + I_{l+1}^l in                 in [nrhs][N_{l+1}], out [nrhs][N_l]
 *   NMG_OP_FILTER    out = F'_l(in)                           in/out [nrhs][N_l]
 *   NMG_OP_CNN       out = N_theta_l(in)                      in/out [nrhs][N_l]
 *   NMG_OP_SMOOTH    out = out + F'_l(||in|| N(in/||in||))    in = b, out = x  [nrhs][N_l]
 *   NMG_OP_COARSE    out = (A^(L))^{-1} in  (level must be L)  in/out [nrhs][N_L]
 *   NMG_OP_CYCLE0    out = NMGF(0, in) at level l (fp32)       in/out [nrhs][N_l]
 * Asynchronous. */
enum {
  NMG_OP_APPLY = 0, NMG_OP_RESIDUAL = 1, NMG_OP_RESTRICT = 2, NMG_OP_PROLONG = 3,
  NMG_OP_FILTER = 4, NMG_OP_CNN = 5, NMG_OP_SMOOTH = 6, NMG_OP_COARSE = 7, NMG_OP_CYCLE0 = 8
};
nmg_status nmg_debug_level_op(nmg_hierarchy *h, int32_t level, int32_t op, int32_t nrhs,
                              const void *in, void *out, void *stream);

/* Per-kernel-class device timing for roofline reports: while enabled, the library
 * records a CUDA event pair on the launching stream around every kernel it enqueues
 * and accumulates the elapsed time per class.  nmg_profile(h, 1) clears and starts,
 * nmg_profile(h, 0) stops.  nmg_profile_query synchronises on the recorded events and
 * returns the total device milliseconds and launch count of class `kclass`. */
enum {
  NMG_K_GEMM64 = 0,    /* fp64 outer residual GEMM (+ norm partials)           */
  NMG_K_GEMM32 = 1,    /* fp32-accurate inner operator applies                  */
  NMG_K_SMOOTH = 2,    /* 1D: fused norm + CNN + level filter + update; 2D: CNN  */
  NMG_K_TRANSFER = 3,  /* restriction / prolongation                            */
  NMG_K_COARSE = 4,    /* coarsest Cholesky solve                               */
  NMG_K_MISC = 5,      /* relres, update, norms, conversions                    */
  NMG_K_FILTER = 6,    /* 2D: smoother norms, strip combine + level-filter FFTs */
  NMG_K_COUNT = 7
};
nmg_status nmg_profile(nmg_hierarchy *h, int32_t enable);
nmg_status nmg_profile_query(nmg_hierarchy *h, int32_t kclass, double *total_ms, int64_t *launches);

/* ---------------------------------------------------------------------------------------
 * Slab-sharded single-system mode (BASELINE config 4: one 2D operator
 * row-sharded over W ranks).  Each rank owns the rows i2 in [rank R, rank R + R), R = n / W,
 * of every right-hand side, i.e. the columns i2 of the column-major n x n matrix X.
 * Per cycle and level: the Kronecker apply A_l X = C_l X B_l^T + alpha Q_l X Q_l^T
 * computes T = C_l X[:, slab] locally, all-gathers T and finishes its own slab of rows of
 * T B_l^T (one all-gather of the intermediate per apply, also for the fp64 outer residual);
 * the CNN smoother runs on the slab plus 4 halo rows per side (its receptive field); the level
 * filter F'_l transforms rows locally and columns after an all-to-all
 * transpose; norms ||b_l|| and ||y - A x|| are summed over the ranks; levels whose
 * slab would be thinner than 32 rows (or n_l < 128) run replicated on every rank after one
 * all-gather of the restricted right-hand side.  2D only; strip-kernel CNN (C = 32 / 48).
 * --------------------------------------------------------------------------------------- */
typedef struct nmg_comm nmg_comm;   /* opaque communicator (one per rank)                     */
#define NMG_COMM_ID_BYTES 128
/* NCCL unique id for nmg_comm_create_nccl (call on rank 0, broadcast the 128 bytes). */
nmg_status nmg_comm_nccl_unique_id(void *out_id);
/* One rank of a W-rank NCCL communicator (one process per GPU; libnccl.so.2 is dlopen'ed).
 * Errors: INVALID_ARG, UNSUPPORTED (no libnccl), CUDA (NCCL failure). */
nmg_status nmg_comm_create_nccl(int32_t world, int32_t rank, const void *id, int32_t device,
                                nmg_comm **out);
/* W emulated ranks in ONE process on one device: out[0..world-1] receive one communicator
 * per rank.  Each rank must be driven by its own host thread (its own stream); ranks meet at
 * host barriers and exchange data with stream-ordered device copies (no device-side waits).
 * Used by the tests to run the multi-rank path on a single GPU. */
nmg_status nmg_comm_create_emulated(int32_t world, nmg_comm **out);
/* Destroy a communicator (after every hierarchy that uses it). */
void nmg_comm_destroy(nmg_comm *c);
/* Build this rank's part of a slab-sharded hierarchy (desc.dim must be 2; n / world must be
 * a multiple of 32 and >= 32; the caller keeps `comm` alive).  Afterwards nmg_vcycle,
 * nmg_solve and nmg_residual take this rank's slab: y, x device fp64 [nrhs][R][n] holding
 * rows i2 = rank R .. rank R + R - 1 of each RHS (same row-major [i2][i1] order); every rank
 * must make the same calls with the same nrhs (collectives).  Relative residuals, norms and
 * convergence decisions are global and identical on every rank.  nmg_vcycles_host and
 * nmg_debug_level_op return NMG_ERR_UNSUPPORTED on a slab handle.
 * Errors: as nmg_create_hierarchy, plus UNSUPPORTED for 1D / shapes the slab mode lacks. */
nmg_status nmg_create_hierarchy_slab(const nmg_problem_desc *desc, const double *factors,
                                     nmg_comm *comm, nmg_hierarchy **out);
/* Number of the library's own kernel launches enqueued since the handle was created
 * (bench evidence, "gpu_launches"). */
int64_t nmg_launch_count(const nmg_hierarchy *h);

void nmg_destroy_hierarchy(nmg_hierarchy *h);

/* Thread-local message for the last non-OK status on this thread ("" if none). */
const char *nmg_last_error(void);

/* Library version string. */
const char *nmg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* NMG_H */
