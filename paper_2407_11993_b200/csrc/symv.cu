// y = alpha * A x + beta * y for symmetric A reading ONLY the lower triangle
// (each off-diagonal 64x64 tile is read once and used twice). HBM-bound:
// n^2/2 * 8 bytes per call; deterministic (fixed-order reduction, no atomics).
// Tile bodies in symv_tile.cuh.
//
// Used by the Cholesky theta-method's per-step R * I product
// (reference: td1_step_kernel's dense loop, _kernels.py:198-207) and exposed as
// em_symv_lower; the tridiagonalisation runs the same tiles inside its fused
// persistent kernel (sytrd_fused.cu).
#include "common.cuh"
#include "ctx.h"
#include "linalg.h"
#include "symv_tile.cuh"

namespace em {

size_t symv_work_size(int64_t n) { return (size_t)symv_work_doubles(n); }

// grid: (chunk, block-row i)
__global__ void __launch_bounds__(256) symv_tiles_kernel(int64_t n, const double* __restrict__ A,
                                                         int64_t lda, const double* __restrict__ x,
                                                         double* __restrict__ wcol,
                                                         double* __restrict__ wrow, int64_t nb,
                                                         int64_t nch) {
  __shared__ double red[8][SV];
  const int64_t i = blockIdx.y, ch = blockIdx.x;
  if (ch * SVCH > i) return;
  symv_strip(n, A, lda, x, wcol, wrow, nb, nch, i, ch, red);
}

__global__ void __launch_bounds__(256) symv_reduce_kernel(int64_t n, double alpha, double beta,
                                                          double* __restrict__ y,
                                                          const double* __restrict__ wcol,
                                                          const double* __restrict__ wrow,
                                                          int64_t nb, int64_t nch) {
  __shared__ double red4[4][SV];
  const int64_t j = blockIdx.x;
  const double v = symv_reduce_block(wcol, wrow, nb, nch, j, red4);
  if (threadIdx.x < SV) {
    const int64_t idx = j * SV + threadIdx.x;
    if (idx < n) y[idx] = (beta == 0.0) ? alpha * v : fma(alpha, v, beta * y[idx]);
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
  symv_tiles_kernel<<<grid, 256, 0, st>>>(n, A, lda, x, wcol, wrow, nb, nch);
  EM_LAUNCHED();
  symv_reduce_kernel<<<(unsigned)nb, 256, 0, st>>>(n, alpha, beta, y, wcol, wrow, nb, nch);
  EM_LAUNCHED();
}

}  // namespace em
