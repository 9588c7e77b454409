// Slab-sharded single-system mode: the i2 axis of every 2D image
// (rows of the row-major [i2][i1] array = columns of the column-major matrix X) is
// split into W contiguous slabs of R = n_l / W rows, one per rank.  A slab is stored with H
// halo rows above and below, [b][R + 2H][n] (halo rows of the global image borders are 0).
// These kernels are the slab versions of the transfer, halo and reduction steps; the index
// maps of the transfers are those of reading R4 (restriction / prolongation in level2d.cu),
// written with GLOBAL row indices so that the result is bitwise the unsharded one.
#include <algorithm>

#include "common.cuh"
#include "kernels.h"

namespace nmg {
namespace {

inline int nblk(int64_t n, int t) { return (int)ceil_div64(n, t); }

NMG_D float r1d(float fm, float f0, float f1, float fp) {
  return __fmul_rn(__fadd_rn(__fadd_rn(fm, fp), __fmul_rn(3.0f, __fadd_rn(f0, f1))), 0.125f);
}
NMG_D float p1d(float cj, float ck) { return __fadd_rn(__fmul_rn(0.75f, cj), __fmul_rn(0.25f, ck)); }

// coarse rows [r0c, r0c + Rc) of R (rows) R (cols) f; f: halo'd fine slab (global row g at
// f + b fimg + foff + g nf); c: row j2 - r0c of image b at c + b cimg + coff
__global__ void restrict_slab_kernel(int nrhs, int n_c, int Rc, int r0c, const float* __restrict__ f, int64_t fimg,
                                     int64_t foff, float* __restrict__ c, int64_t cimg, int64_t coff) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)Rc * n_c;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int rem = (int)(idx - b * per);
  const int jl = rem / n_c, j1 = rem - jl * n_c;
  const int j2 = r0c + jl;
  const int n_f = 2 * n_c;
  const float* F = f + (int64_t)b * fimg + foff;
  const int c1[4] = {max(2 * j1 - 1, 0), 2 * j1, 2 * j1 + 1, min(2 * j1 + 2, n_f - 1)};
  const int c2[4] = {max(2 * j2 - 1, 0), 2 * j2, 2 * j2 + 1, min(2 * j2 + 2, n_f - 1)};
  float r[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const float* row = F + (int64_t)c2[a] * n_f;
    r[a] = r1d(row[c1[0]], row[c1[1]], row[c1[2]], row[c1[3]]);
  }
  c[(int64_t)b * cimg + coff + (int64_t)jl * n_c + j1] = r1d(r[0], r[1], r[2], r[3]);
}

// fine rows [r0f, r0f + Rf) += P c; c: global row g at c + b cimg + coff + g n_c
// (a halo'd coarse slab or the full replicated coarse image); f: row i2 - r0f at f + b fimg + foff
__global__ void prolong_slab_kernel(int nrhs, int n_c, int Rf, int r0f, const float* __restrict__ c, int64_t cimg,
                                    int64_t coff, float* __restrict__ f, int64_t fimg, int64_t foff) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int n_f = 2 * n_c;
  const int64_t per = (int64_t)Rf * n_f;
  if (idx >= nrhs * per) return;
  const int b = (int)(idx / per);
  const int rem = (int)(idx - b * per);
  const int il = rem / n_f, i1 = rem - il * n_f;
  const int i2 = r0f + il;
  const int j1 = i1 >> 1, k1 = min(max((i1 & 1) ? j1 + 1 : j1 - 1, 0), n_c - 1);
  const int j2 = i2 >> 1, k2 = min(max((i2 & 1) ? j2 + 1 : j2 - 1, 0), n_c - 1);
  const float* C = c + (int64_t)b * cimg + coff;
  const float vj = p1d(C[(int64_t)j2 * n_c + j1], C[(int64_t)j2 * n_c + k1]);
  const float vk = p1d(C[(int64_t)k2 * n_c + j1], C[(int64_t)k2 * n_c + k1]);
  float* o = f + (int64_t)b * fimg + foff + (int64_t)il * n_f + i1;
  *o = __fadd_rn(*o, p1d(vj, vk));
}

// send [2][b][H][n]: the slab's first H and last H rows
__global__ void halo_pack_kernel(int nrhs, int n, int R, int H, const float* __restrict__ x, float* __restrict__ send) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)H * n;
  if (i >= 2 * nrhs * per) return;
  const int side = (int)(i / (nrhs * per));
  const int64_t rem = i - side * nrhs * per;
  const int b = (int)(rem / per);
  const int64_t k = rem - b * per;
  const int64_t img = (int64_t)(R + 2 * H) * n;
  send[i] = x[b * img + (int64_t)(side == 0 ? H : R) * n + k];
}
// recv [W][2][b][H][n]: top halo <- rank - 1's last rows, bottom <- rank + 1's first rows (0 at the borders)
__global__ void halo_unpack_kernel(int nrhs, int n, int R, int H, int rank, int W, const float* __restrict__ recv,
                                   float* __restrict__ x) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)H * n;
  if (i >= 2 * nrhs * per) return;
  const int side = (int)(i / (nrhs * per));     // 0: top halo, 1: bottom halo
  const int64_t rem = i - side * nrhs * per;
  const int b = (int)(rem / per);
  const int64_t k = rem - b * per;
  const int64_t img = (int64_t)(R + 2 * H) * n;
  const int peer = side == 0 ? rank - 1 : rank + 1;
  float v = 0.f;
  if (peer >= 0 && peer < W) v = recv[((int64_t)peer * 2 + (side == 0 ? 1 : 0)) * nrhs * per + rem];
  x[b * img + (int64_t)(side == 0 ? 0 : R + H) * n + k] = v;
}

// x[b][j] += d[b img + off + j] (fp64 outer update of the slab), masked by the active flags
__global__ void update_slab_kernel(int nrhs, int64_t N, double* __restrict__ x, const float* __restrict__ d,
                                   int64_t img, int64_t off, const uint8_t* __restrict__ active) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nrhs * N) return;
  const int b = (int)(i / N);
  if (active && !active[b]) return;
  x[i] += (double)d[b * img + off + (i - (int64_t)b * N)];
}

// per-RHS fixed-order sums of cnt consecutive partials (one block per RHS)
__global__ void __launch_bounds__(256) part_sums_kernel(int64_t cnt, const double* __restrict__ part,
                                                        double* __restrict__ out) {
  __shared__ double red[32];
  const int b = blockIdx.x;
  double s = 0.0;
  for (int64_t t = threadIdx.x; t < cnt; t += blockDim.x) s += part[(int64_t)b * cnt + t];
  s = block_sum_f64(s, red);
  if (threadIdx.x == 0) out[b] = s;
}

__global__ void relres_sums_kernel(int nrhs, const double* __restrict__ rsq, const double* __restrict__ ysq,
                                   double* __restrict__ relres, double tol, uint8_t* __restrict__ active) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nrhs) return;
  const double yn = sqrt(ysq[b]), s = rsq[b];
  const double rr = (yn > 0.0) ? sqrt(s) / yn : (yn == 0.0 && s == 0.0 ? 0.0 : sqrt(s) / yn);
  relres[b] = rr;
  if (active) active[b] = (rr > tol || rr != rr) ? 1 : 0;
}

__global__ void sqrt_kernel(int n, double* v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = sqrt(v[i]);
}

__global__ void __launch_bounds__(256) sumsq_f64_kernel(int64_t N, int chunks, const double* __restrict__ y,
                                                        double* __restrict__ part) {
  __shared__ double red[32];
  const int b = blockIdx.y, ch = blockIdx.x;
  const int64_t len = ceil_div64(N, chunks);
  const int64_t lo = ch * len, hi = min(N, lo + len);
  const double* r = y + (int64_t)b * N;
  double s = 0.0;
  for (int64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) s += r[j] * r[j];
  s = block_sum_f64(s, red);
  if (threadIdx.x == 0) part[(int64_t)b * chunks + ch] = s;
}

}  // namespace

void restrict_slab(int nrhs, int n_c, int Rc, int r0c, const float* f, int64_t fimg, int64_t foff, float* c,
                   int64_t cimg, int64_t coff, cudaStream_t s) {
  restrict_slab_kernel<<<nblk((int64_t)nrhs * Rc * n_c, 256), 256, 0, s>>>(nrhs, n_c, Rc, r0c, f, fimg, foff, c, cimg,
                                                                          coff);
}
void prolong_slab(int nrhs, int n_c, int Rf, int r0f, const float* c, int64_t cimg, int64_t coff, float* f,
                  int64_t fimg, int64_t foff, cudaStream_t s) {
  prolong_slab_kernel<<<nblk((int64_t)nrhs * Rf * 2 * n_c, 256), 256, 0, s>>>(nrhs, n_c, Rf, r0f, c, cimg, coff, f,
                                                                              fimg, foff);
}
void halo_pack(int nrhs, int n, int R, int H, const float* x, float* send, cudaStream_t s) {
  halo_pack_kernel<<<nblk((int64_t)2 * nrhs * H * n, 256), 256, 0, s>>>(nrhs, n, R, H, x, send);
}
void halo_unpack(int nrhs, int n, int R, int H, int rank, int W, const float* recv, float* x, cudaStream_t s) {
  halo_unpack_kernel<<<nblk((int64_t)2 * nrhs * H * n, 256), 256, 0, s>>>(nrhs, n, R, H, rank, W, recv, x);
}
void update_slab(int nrhs, int64_t N, double* x, const float* d, int64_t img, int64_t off, const uint8_t* active,
                 cudaStream_t s) {
  update_slab_kernel<<<nblk((int64_t)nrhs * N, 256), 256, 0, s>>>(nrhs, N, x, d, img, off, active);
}
void part_sums(int nrhs, int64_t cnt, const double* part, double* out, cudaStream_t s) {
  part_sums_kernel<<<nrhs, 256, 0, s>>>(cnt, part, out);
}
void relres_sums(int nrhs, const double* rsq, const double* ysq, double* relres, double tol, uint8_t* active,
                 cudaStream_t s) {
  relres_sums_kernel<<<nblk(nrhs, 128), 128, 0, s>>>(nrhs, rsq, ysq, relres, tol, active);
}
void sqrt_inplace(int n, double* v, cudaStream_t s) { sqrt_kernel<<<nblk(n, 128), 128, 0, s>>>(n, v); }
void sumsq_f64(int nrhs, int64_t N, const double* y, double* part, double* out, cudaStream_t s) {
  const int chunks = (int)std::min<int64_t>(64, std::max<int64_t>(1, N / 8192));
  sumsq_f64_kernel<<<dim3(chunks, nrhs), 256, 0, s>>>(N, chunks, y, part);
  part_sums_kernel<<<nrhs, 64, 0, s>>>(chunks, part, out);
}

}  // namespace nmg
