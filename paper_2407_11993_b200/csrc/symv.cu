// y = alpha * A x + beta * y for symmetric A reading ONLY the lower triangle
// (each off-diagonal 64x64 tile is read once and used twice: A_ij x_j -> y_i and
// A_ij^T x_i -> y_j). HBM-bound: n^2/2 * 8 bytes per call. Deterministic: the
// transposed contributions go to a per-tile workspace reduced in fixed order
// (no floating-point atomics).
//
// Used by the Householder tridiagonalisation (the memory-bound half of sytrd)
// and by the Cholesky theta-method's per-step R * I product
// (reference: td1_step_kernel's dense loop, _kernels.py:198-207).
#include "common.cuh"
#include "ctx.h"
#include "linalg.h"

namespace em {

constexpr int SV = 64;       // tile
constexpr int SVCH = 16;     // tiles per CTA chunk along a block row
constexpr int SVT = 256;     // threads

size_t symv_work_size(int64_t n) {
  int64_t nb = (n + SV - 1) / SV;
  int64_t nch = (nb + SVCH - 1) / SVCH;
  return (size_t)(nb * nb * SV + nb * nch * SV);
}

// grid: (chunk, block-row i). Chunk c covers tiles j in [c*SVCH, min(i, c*SVCH+SVCH-1)].
__global__ void __launch_bounds__(SVT) symv_tiles_kernel(int64_t n, const double* __restrict__ A,
                                                         int64_t lda, const double* __restrict__ x,
                                                         double* __restrict__ wcol,
                                                         double* __restrict__ wrow, int64_t nb,
                                                         int64_t nch) {
  __shared__ double S[SV][SV + 1];
  __shared__ double xi[SV], xj[SV];
  __shared__ double red[4][SV];
  const int64_t i = blockIdx.y, ch = blockIdx.x;
  const int64_t j_begin = ch * SVCH;
  if (j_begin > i) return;
  const int64_t j_end = imin64(i, j_begin + SVCH - 1);  // inclusive
  const int tid = threadIdx.x, tx = tid & 63, ty = tid >> 6;
  const int64_t r0 = i * SV;
  if (tid < SV) xi[tid] = (r0 + tid < n) ? x[r0 + tid] : 0.0;
  double rowacc = 0.0;
  for (int64_t j = j_begin; j <= j_end; ++j) {
    const int64_t c0 = j * SV;
    __syncthreads();
    if (tid < SV) xj[tid] = (c0 + tid < n) ? x[c0 + tid] : 0.0;
    double a[16];
    const int64_t r = r0 + tx;
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      const int64_t c = c0 + ty * 16 + cc;
      a[cc] = (r < n && c < n) ? A[r + c * lda] : 0.0;
    }
    if (j == i) {
      // diagonal tile: symmetrise from the lower triangle in shared memory
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) S[tx][ty * 16 + cc] = a[cc];
      __syncthreads();
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        const int c = ty * 16 + cc;
        const double v = (tx >= c) ? S[tx][c] : S[c][tx];
        rowacc = fma(v, xj[c], rowacc);
      }
    } else {
      __syncthreads();  // xj visible
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) {
        rowacc = fma(a[cc], xj[ty * 16 + cc], rowacc);
        S[tx][ty * 16 + cc] = a[cc];
      }
      __syncthreads();
      // column products: thread (cx = tx, row group ty)
      double cs = 0.0;
#pragma unroll
      for (int rr = 0; rr < 16; ++rr) cs = fma(S[ty * 16 + rr][tx], xi[ty * 16 + rr], cs);
      red[ty][tx] = cs;
      __syncthreads();
      if (tid < SV)
        wcol[(i * nb + j) * SV + tid] = red[0][tid] + red[1][tid] + red[2][tid] + red[3][tid];
    }
  }
  __syncthreads();
  red[ty][tx] = rowacc;
  __syncthreads();
  if (tid < SV) wrow[(i * nch + ch) * SV + tid] = red[0][tid] + red[1][tid] + red[2][tid] + red[3][tid];
}

__global__ void symv_reduce_kernel(int64_t n, double alpha, double beta, double* __restrict__ y,
                                   const double* __restrict__ wcol,
                                   const double* __restrict__ wrow, int64_t nb, int64_t nch) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const int64_t j = idx / SV;
  const int t = (int)(idx % SV);
  double s = 0.0;
  const int64_t nchj = j / SVCH + 1;  // chunks present in block row j
  for (int64_t c = 0; c < nchj; ++c) s += wrow[(j * nch + c) * SV + t];
  for (int64_t i = j + 1; i < nb; ++i) s += wcol[(i * nb + j) * SV + t];
  y[idx] = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * y[idx]);
}

void symv_lower(cudaStream_t st, int64_t n, double alpha, const double* A, int64_t lda,
                const double* x, double beta, double* y, double* work) {
  if (n <= 0) return;
  const int64_t nb = (n + SV - 1) / SV;
  const int64_t nch = (nb + SVCH - 1) / SVCH;
  double* wcol = work;
  double* wrow = work + nb * nb * SV;
  dim3 grid((unsigned)nch, (unsigned)nb);
  symv_tiles_kernel<<<grid, SVT, 0, st>>>(n, A, lda, x, wcol, wrow, nb, nch);
  EM_LAUNCHED();
  symv_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, alpha, beta, y, wcol, wrow,
                                                                  nb, nch);
  EM_LAUNCHED();
}

}  // namespace em
