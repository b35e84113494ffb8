// Tile bodies of the lower-triangle symv (y = A x, A symmetric, only the lower
// triangle read): the register-prefetch kernels of symv.cu and the tile body of the
// TMA kernel (symv_tma.cu).
//
// Tile mapping: warp w owns columns 8w..8w+7 of a 64x64 tile, lane l rows l and
// l+32 (every load instruction reads 256 contiguous bytes). The next tile is
// prefetched into registers while the current one is consumed; column sums are
// reduced with a 9-shuffle butterfly, so a tile needs no shared memory and no
// barrier. Off-diagonal tile (i, j) contributes A_ij x_j to y_i (row partials,
// summed per strip) and A_ij^T x_i to y_j (one 64-vector per tile in wcol); the
// reduction sums them in a fixed order (deterministic, no atomics).
#pragma once
#include "common.cuh"

namespace em {

constexpr int SV = 64;     // tile
constexpr int SVCH = 16;   // tiles per strip chunk

__host__ __device__ __forceinline__ int64_t symv_work_doubles(int64_t n) {
  const int64_t nb = (n + SV - 1) / SV;
  const int64_t nch = (nb + SVCH - 1) / SVCH;
  return nb * nb * SV + nb * nch * SV;
}

template <bool FULL>
EM_DEVINL void symv_load_tile(double (&a)[2][8], const double* A, int64_t lda,
                              int64_t n, int64_t r0, int64_t c0, int lane, int w) {
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

// x as the tiles see it: xs * x[r], except x[0] = 1 when unit0 (a Householder vector
// whose first entry is implicit, dlarfg convention).
EM_DEVINL double symv_xval(const double* x, int64_t r, int64_t n, double xs, bool unit0) {
  if (r >= n) return 0.0;
  if (unit0 && r == 0) return 1.0;
  return xs * __ldcg(x + r);
}

// One 64x64 tile already in registers: row partials += A_ij x_j, column sums
// A_ij^T x_i written to wdst[0..64). diag: tile on the diagonal (lower part only).
EM_DEVINL void symv_tile_body(const double (&a)[2][8], int64_t n, const double* x, int64_t c0,
                              bool diag, double xi0, double xi1, double& row0, double& row1,
                              double* wdst, int lane, int w, double xs = 1.0,
                              bool unit0 = false) {
  double xj[8];
#pragma unroll
  for (int cc = 0; cc < 8; ++cc) xj[cc] = symv_xval(x, c0 + 8 * w + cc, n, xs, unit0);
  double col[8];
  if (!diag) {
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
    const int cc = ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
    wdst[8 * w + cc] = col[0];
  }
}

// Strip chunk `ch` of block row i (tiles j in [ch*SVCH, min(i, ch*SVCH+SVCH-1)]);
// 256 threads. red: shared [8][SV].
EM_DEVINL void symv_strip(int64_t n, const double* A, int64_t lda,
                          const double* x, double* wcol,
                          double* wrow, int64_t nb, int64_t nch, int64_t i,
                          int64_t ch, double (*red)[SV]) {
  const int64_t j_begin = ch * SVCH;
  const int64_t j_end = imin64(i, j_begin + SVCH - 1);  // inclusive
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t r0 = i * SV;
  const bool row_full = r0 + SV <= n;
  const double xi0 = (r0 + lane < n) ? __ldcg(x + r0 + lane) : 0.0;
  const double xi1 = (r0 + lane + 32 < n) ? __ldcg(x + r0 + lane + 32) : 0.0;
  double row0 = 0.0, row1 = 0.0;
  double nxt[2][8];
  if (row_full && j_begin * SV + SV <= n)
    symv_load_tile<true>(nxt, A, lda, n, r0, j_begin * SV, lane, w);
  else
    symv_load_tile<false>(nxt, A, lda, n, r0, j_begin * SV, lane, w);
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
        symv_load_tile<true>(nxt, A, lda, n, r0, c1, lane, w);
      else
        symv_load_tile<false>(nxt, A, lda, n, r0, c1, lane, w);
    }
    symv_tile_body(a, n, x, c0, j == i, xi0, xi1, row0, row1, wcol + (i * nb + j) * SV, lane, w);
  }
  __syncthreads();  // red may still be read by a previous strip's reduction
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

// Sum for block j: row-strip partials of block row j + transposed partials of
// tiles (i, j), i >= j. 256 threads; red4: shared [4][SV]. Returns the value for
// row j*SV + threadIdx.x in threads < SV (0 elsewhere).
EM_DEVINL double symv_reduce_block(const double* wcol,
                                   const double* wrow, int64_t nb, int64_t nch,
                                   int64_t j, double (*red4)[SV]) {
  const int t = threadIdx.x & (SV - 1), g = threadIdx.x >> 6;
  double s0 = 0.0, s1 = 0.0;
  int64_t i = j + g;
  for (; i + 4 < nb; i += 8) {
    s0 += __ldcg(wcol + (i * nb + j) * SV + t);
    s1 += __ldcg(wcol + ((i + 4) * nb + j) * SV + t);
  }
  if (i < nb) s0 += __ldcg(wcol + (i * nb + j) * SV + t);
  double s = s0 + s1;
  if (g == 0) {
    const int64_t nchj = j / SVCH + 1;  // chunks present in block row j
    for (int64_t c = 0; c < nchj; ++c) s += __ldcg(wrow + (j * nch + c) * SV + t);
  }
  __syncthreads();
  red4[g][t] = s;
  __syncthreads();
  double v = 0.0;
  if (threadIdx.x < SV) v = (red4[0][t] + red4[1][t]) + (red4[2][t] + red4[3][t]);
  return v;
}

}  // namespace em
