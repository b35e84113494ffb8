// y = alpha * A x + beta * y for symmetric A reading ONLY the lower triangle
// (each off-diagonal 64x64 tile is read once and used twice: A_ij x_j -> y_i and
// A_ij^T x_i -> y_j). HBM-bound: n^2/2 * 8 bytes per call. Deterministic: the
// transposed contributions go to a per-tile workspace reduced in fixed order
// (no floating-point atomics).
//
// Tile mapping: warp w owns columns 8w..8w+7 of a tile, lane l rows l and l+32
// (every load instruction reads 256 contiguous bytes). The next tile is
// prefetched into registers while the current one is consumed; column sums
// are reduced with a 9-shuffle butterfly, so a tile needs no shared memory and
// no barrier.
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

template <bool FULL>
EM_DEVINL void load_tile(double (&a)[2][8], const double* __restrict__ A, int64_t lda, int64_t n,
                         int64_t r0, int64_t c0, int lane, int w) {
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) {
    const int64_t c = c0 + 8 * w + cc;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t r = r0 + lane + 32 * h;
      if (FULL)
        a[h][cc] = A[r + c * lda];
      else
        a[h][cc] = (r < n && c < n) ? A[r + c * lda] : 0.0;
    }
  }
}

// grid: (chunk, block-row i). Chunk ch covers tiles j in [ch*SVCH, min(i, ch*SVCH+SVCH-1)].
__global__ void __launch_bounds__(SVT) symv_tiles_kernel(int64_t n, const double* __restrict__ A,
                                                         int64_t lda, const double* __restrict__ x,
                                                         double* __restrict__ wcol,
                                                         double* __restrict__ wrow, int64_t nb,
                                                         int64_t nch) {
  __shared__ double red[8][SV];
  const int64_t i = blockIdx.y, ch = blockIdx.x;
  const int64_t j_begin = ch * SVCH;
  if (j_begin > i) return;
  const int64_t j_end = imin64(i, j_begin + SVCH - 1);  // inclusive
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t r0 = i * SV;
  const bool row_full = r0 + SV <= n;
  const double xi0 = (r0 + lane < n) ? x[r0 + lane] : 0.0;
  const double xi1 = (r0 + lane + 32 < n) ? x[r0 + lane + 32] : 0.0;
  double row0 = 0.0, row1 = 0.0;
  double nxt[2][8];
  if (row_full && j_begin * SV + SV <= n)
    load_tile<true>(nxt, A, lda, n, r0, j_begin * SV, lane, w);
  else
    load_tile<false>(nxt, A, lda, n, r0, j_begin * SV, lane, w);
  for (int64_t j = j_begin; j <= j_end; ++j) {
    double a[2][8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      a[0][cc] = nxt[0][cc];
      a[1][cc] = nxt[1][cc];
    }
    const int64_t c0 = j * SV;
    if (j < j_end) {
      const int64_t c1 = c0 + SV;
      if (row_full && c1 + SV <= n)
        load_tile<true>(nxt, A, lda, n, r0, c1, lane, w);
      else
        load_tile<false>(nxt, A, lda, n, r0, c1, lane, w);
    }
    double xj[8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int64_t c = c0 + 8 * w + cc;
      xj[cc] = (c < n) ? __ldg(x + c) : 0.0;
    }
    double col[8];
    if (j != i) {
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        row0 = fma(a[0][cc], xj[cc], row0);
        row1 = fma(a[1][cc], xj[cc], row1);
        col[cc] = fma(a[0][cc], xi0, a[1][cc] * xi1);
      }
    } else {
      // diagonal tile: lower triangle only (r >= c for rows, r > c for the transpose)
#pragma unroll
      for (int cc = 0; cc < 8; ++cc) {
        const int c = 8 * w + cc;
        const double l0 = (lane >= c) ? a[0][cc] : 0.0;
        const double l1 = (lane + 32 >= c) ? a[1][cc] : 0.0;
        row0 = fma(l0, xj[cc], row0);
        row1 = fma(l1, xj[cc], row1);
        const double s0 = (lane > c) ? a[0][cc] : 0.0;
        const double s1 = (lane + 32 > c) ? a[1][cc] : 0.0;
        col[cc] = fma(s0, xi0, s1 * xi1);
      }
    }
    // butterfly: reduce 8 column partials over the 32 lanes
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {  // offset 16: lanes < 16 keep cols 0..3, others 4..7
      const bool hi = lane & 16;
      const double send = hi ? col[cc] : col[cc + 4];
      const double keep = hi ? col[cc + 4] : col[cc];
      col[cc] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {  // offset 8
      const bool hi = lane & 8;
      const double send = hi ? col[cc] : col[cc + 2];
      const double keep = hi ? col[cc + 2] : col[cc];
      col[cc] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    {  // offset 4
      const bool hi = lane & 4;
      const double send = hi ? col[0] : col[1];
      const double keep = hi ? col[1] : col[0];
      col[0] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    col[0] += __shfl_xor_sync(0xffffffffu, col[0], 2);
    col[0] += __shfl_xor_sync(0xffffffffu, col[0], 1);
    if ((lane & 3) == 0) {
      // column index held by this lane group: bit4 -> +4, bit3 -> +2, bit2 -> +1
      const int cc = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
      wcol[(i * nb + j) * SV + 8 * w + cc] = col[0];
    }
  }
  red[w][lane] = row0;
  red[w][lane + 32] = row1;
  __syncthreads();
  if (tid < SV) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += red[k][tid];
    wrow[(i * nch + ch) * SV + tid] = s;
  }
}

// y block j: sum of the row-strip partials of block row j and of the transposed
// tile partials of block column j (tiles (i, j), i >= j). One CTA per block; the
// column sum is split over 4 interleaved i-slices (fixed order) for memory-level
// parallelism, then combined in shared memory.
__global__ void __launch_bounds__(256) symv_reduce_kernel(int64_t n, double alpha, double beta,
                                                          double* __restrict__ y,
                                                          const double* __restrict__ wcol,
                                                          const double* __restrict__ wrow,
                                                          int64_t nb, int64_t nch) {
  __shared__ double red[4][SV];
  const int64_t j = blockIdx.x;
  const int t = threadIdx.x & (SV - 1), g = threadIdx.x >> 6;
  double s0 = 0.0, s1 = 0.0;
  int64_t i = j + g;
  for (; i + 4 < nb; i += 8) {
    s0 += wcol[(i * nb + j) * SV + t];
    s1 += wcol[((i + 4) * nb + j) * SV + t];
  }
  if (i < nb) s0 += wcol[(i * nb + j) * SV + t];
  double s = s0 + s1;
  if (g == 0) {
    const int64_t nchj = j / SVCH + 1;  // chunks present in block row j
    for (int64_t c = 0; c < nchj; ++c) s += wrow[(j * nch + c) * SV + t];
  }
  red[g][t] = s;
  __syncthreads();
  if (threadIdx.x < SV) {
    const int64_t idx = j * SV + t;
    if (idx < n) {
      const double v = (red[0][t] + red[1][t]) + (red[2][t] + red[3][t]);
      y[idx] = (beta == 0.0) ? alpha * v : fma(alpha, v, beta * y[idx]);
    }
  }
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
  symv_reduce_kernel<<<(unsigned)nb, 256, 0, st>>>(n, alpha, beta, y, wcol, wrow, nb, nch);
  EM_LAUNCHED();
}

}  // namespace em
