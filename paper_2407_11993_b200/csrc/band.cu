// Banded Cholesky of the resistance matrix and the banded triangular solves built on it.
//
// The reference factors R_i as a dense SymMatrix (cholesky_kernel, _kernels.py:18-36) and
// then runs dense triangular solves for the two-sided reduction and the back-transform
// (modal.py:63-73, _kernels.py:56-79). R_i of a voxel plate is a 7-point stencil: in the
// reference's own unknown ordering its lower bandwidth is b = ny*nz, and a Cholesky factor
// of a banded SPD matrix has no fill outside the band (every such entry is an exact zero
// in floating point too). SURVEY §8(d) counts these stages by the band: potrf N b^2,
// two-sided reduction 4 N^2 b, back-transform 2 N^2 b instead of N^3/3, N^3, N^3.
//
// Storage: the factor by 128-wide block columns, panel j = rows [128 j, 128 j + ldp) of
// block column j (ldp = 128 (kb + 1), kb = ceil(b / 128) blocks below the diagonal block),
// column-major with ld = ldp, plus the inverse of every 128 x 128 diagonal block (the
// dense potrf's leaf kernel factors and inverts each diagonal block in shared memory).
// Every product is a DMMA GEMM: per block column one leaf, one panel GEMM and kb
// trailing GEMMs; per block row of a solve two GEMMs with the whole right-hand side.
//
// The two-sided reduction is the reference's own sequence, B = G^-1 (G^-1 L)^T,
// (B + B^T) / 2, with an in-place transpose between the two banded forward solves.
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

__global__ void potf2_inv_kernel(double* A, int64_t lda, int64_t k0, int bs, double* Dinv,
                                 int64_t* info);  // potrf.cu
constexpr int BNB = 128;  // == the dense potrf leaf (PNB)
constexpr int BLD = BNB + 1;

// lower bandwidth: max over columns j of (last row i with A[i, j] != 0) - j
__global__ void band_width_kernel(int64_t n, const double* __restrict__ A, int64_t lda,
                                  unsigned long long* __restrict__ out) {
  const int64_t j = blockIdx.x;
  const double* col = A + j * lda;
  int64_t last = j;
  for (int64_t i = j + threadIdx.x; i < n; i += blockDim.x)
    if (col[i] != 0.0) last = i;
  for (int o = 16; o > 0; o >>= 1) {
    const int64_t x = __shfl_xor_sync(0xffffffffu, last, o);
    last = x > last ? x : last;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)(last - j));
}

int64_t band_lower_width(cudaStream_t st, int64_t n, const double* A, int64_t lda) {
  if (n <= 1) return 0;
  DArr<unsigned long long> d(1, st);
  EM_CK(cudaMemsetAsync(d.p, 0, sizeof(unsigned long long), st));
  band_width_kernel<<<(unsigned)n, 256, 0, st>>>(n, A, lda, d.p);
  EM_LAUNCHED();
  unsigned long long h = 0;
  EM_CK(cudaMemcpyAsync(&h, d.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  return (int64_t)h;
}

// panel j <- rows [128 j, 128 j + ldp) x cols [128 j, 128 j + 128) of A's lower triangle
// (band >= 0: A is LAPACK lower band storage, A[(i - j) + j lda] = a_ij for i - j <= band)
__global__ void band_extract_panels_kernel(int64_t n, const double* __restrict__ A, int64_t lda,
                                           int64_t ldp, int64_t nblk, double* __restrict__ P,
                                           int64_t band) {
  const int64_t per = ldp * BNB;
  const int64_t total = per * nblk;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = t / per, rem = t % per;
    const int64_t c = rem / ldp, r = rem % ldp;
    const int64_t gc = j * BNB + c, gr = j * BNB + r;
    if (band >= 0)
      P[t] = (gr < n && gc < n && gr >= gc && gr - gc <= band) ? A[(gr - gc) + gc * lda] : 0.0;
    else
      P[t] = (gr < n && gc < n && gr >= gc) ? A[gr + gc * lda] : 0.0;
  }
}

int64_t band_potrf(cudaStream_t st, int64_t n, const double* A, int64_t lda, int64_t bw,
                   BandChol& f, bool band_storage) {
  f.n = n;
  f.kb = (int)((bw + BNB - 1) / BNB);
  f.ldp = (int64_t)BNB * (f.kb + 1);
  f.nblk = (n + BNB - 1) / BNB;
  f.P.alloc((size_t)f.ldp * BNB * f.nblk, st);
  f.Dinv.alloc((size_t)BNB * BNB * f.nblk, st);
  {
    const int64_t total = f.ldp * BNB * f.nblk;
    const int blocks = (int)imin64((total + 255) / 256, 32 * num_sms());
    band_extract_panels_kernel<<<blocks, 256, 0, st>>>(n, A, lda, f.ldp, f.nblk, f.P.p,
                                                        band_storage ? bw : -1);
    EM_LAUNCHED();
  }
  DArr<int64_t> info(1, st);
  const int64_t minus1 = -1;
  EM_CK(cudaMemcpyAsync(info.p, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  const size_t smem = ((size_t)BNB * BLD + BNB) * sizeof(double);
  EM_CK(cudaFuncSetAttribute(potf2_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem));
  DBuf T((size_t)f.ldp * BNB, st);
  for (int64_t j = 0; j < f.nblk; ++j) {
    double* Pj = f.panel(j);
    double* Dj = f.Dinv.p + j * BNB * BNB;
    const int cj = (int)imin64(BNB, n - j * BNB);
    potf2_inv_kernel<<<1, 256, smem, st>>>(Pj, f.ldp, j * BNB, cj, Dj, info.p);
    EM_LAUNCHED();
    const int64_t rb = f.rows_below(j);
    if (rb <= 0) continue;
    // L_below = A_below G_jj^-T
    EM_CK(gemm(st, false, true, rb, cj, cj, 1.0, Pj + BNB, f.ldp, Dj, BNB, 0.0, T.p, rb));
    copy_matrix(st, false, rb, cj, T.p, rb, Pj + BNB, f.ldp);
    // trailing band: block column j+k, its rows up to the end of panel j's band
    for (int k = 1; k <= f.kb; ++k) {
      if ((j + k) * BNB >= n) break;
      const int64_t ck = imin64(BNB, n - (j + k) * BNB);
      const int64_t rk = BNB + rb - (int64_t)k * BNB;
      if (rk <= 0) break;
      EM_CK(gemm(st, false, true, rk, ck, BNB, -1.0, Pj + (int64_t)k * BNB, f.ldp,
                 Pj + (int64_t)k * BNB, f.ldp, 1.0, f.panel(j + k), f.ldp));
    }
  }
  int64_t h = -1;
  EM_CK(cudaMemcpyAsync(&h, info.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  return h;
}

// Gershgorin interval of a symmetric matrix in lower band storage (one warp per row):
// out[0] = min_i (a_ii - sum_j |a_ij|), out[1] = max_i (a_ii + sum_j |a_ij|); *neg = 1 if
// some lower end is not positive (atomics on ordered bit patterns of non-negative doubles)
__global__ void band_gershgorin_kernel(int64_t n, const double* __restrict__ B, int64_t ldb,
                                       int64_t bw, unsigned long long* out_lo,
                                       unsigned long long* out_hi, int* neg) {
  const int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t q = 1 + lane; q <= bw; q += 32) {
    if (i - q >= 0) s += fabs(B[q + (i - q) * ldb]);  // a_{i, i-q}
    if (i + q < n) s += fabs(B[q + i * ldb]);         // a_{i+q, i}
  }
  s = warp_sum(s);
  if (lane == 0) {
    const double d = B[i * ldb];
    const double lo = d - s, hi = d + s;
    if (!(lo > 0.0)) atomicExch(neg, 1);
    else atomicMin(out_lo, (unsigned long long)__double_as_longlong(lo));
    atomicMax(out_hi, (unsigned long long)__double_as_longlong(fmax(hi, 0.0)));
  }
}

// C (n x m) <- G^-1 C (trans = false, forward) or G^-T C (trans = true, backward)
void band_solve(cudaStream_t st, const BandChol& f, bool trans, int64_t m, double* C,
                int64_t ldc) {
  const int64_t n = f.n;
  if (n <= 0 || m <= 0) return;
  DBuf T((size_t)BNB * m, st);
  for (int64_t s = 0; s < f.nblk; ++s) {
    const int64_t j = trans ? f.nblk - 1 - s : s;
    const double* Pj = f.panel(j);
    const double* Dj = f.Dinv.p + j * BNB * BNB;
    const int64_t cj = imin64(BNB, n - j * BNB);
    const int64_t rb = f.rows_below(j);
    double* Cj = C + j * BNB;
    if (trans && rb > 0)  // C_j -= L_below^T C_below
      EM_CK(gemm(st, true, false, cj, m, rb, -1.0, Pj + BNB, f.ldp, Cj + BNB, ldc, 1.0, Cj, ldc));
    EM_CK(gemm(st, trans, false, cj, m, cj, 1.0, Dj, BNB, Cj, ldc, 0.0, T.p, BNB));
    copy_matrix(st, false, cj, m, T.p, BNB, Cj, ldc);
    if (!trans && rb > 0)  // C_below -= L_below C_j
      EM_CK(gemm(st, false, false, rb, m, cj, -1.0, Pj + BNB, f.ldp, Cj, ldc, 1.0, Cj + BNB, ldc));
  }
}

// In-place square transpose (op = 0) or symmetrisation A <- (A + A^T) / 2 (op = 1), by
// 32 x 32 tile pairs staged in shared memory.
__global__ void tile_pair_kernel(int64_t n, double* A, int64_t lda, int op) {
  const int64_t bi = blockIdx.y, bj = blockIdx.x;
  if (bi > bj) return;
  __shared__ double s1[32][33], s2[32][33];
  const int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  const int64_t r0 = bi * 32, c0 = bj * 32;
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + tx, c = c0 + k;  // tile (bi, bj): element (r, c), column c
    s1[k][tx] = (r < n && c < n) ? A[r + c * lda] : 0.0;
    const int64_t r2 = c0 + tx, c2 = r0 + k;  // tile (bj, bi)
    s2[k][tx] = (r2 < n && c2 < n) ? A[r2 + c2 * lda] : 0.0;
  }
  __syncthreads();
  // element (r0+a, c0+b) = s1[b][a]; element (c0+a, r0+b) = s2[b][a]
  for (int k = ty; k < 32; k += 8) {
    const int64_t r = r0 + tx, c = c0 + k;
    const int64_t r2 = c0 + tx, c2 = r0 + k;
    if (op == 0) {
      if (r < n && c < n) A[r + c * lda] = s2[tx][k];
      if (r2 < n && c2 < n) A[r2 + c2 * lda] = s1[tx][k];
    } else {
      if (r < n && c < n) A[r + c * lda] = 0.5 * (s1[k][tx] + s2[tx][k]);
      if (r2 < n && c2 < n) A[r2 + c2 * lda] = 0.5 * (s2[k][tx] + s1[tx][k]);
    }
  }
}

static void tile_pairs(cudaStream_t st, int64_t n, double* A, int64_t lda, int op) {
  const int64_t t = (n + 31) / 32;
  dim3 grid((unsigned)t, (unsigned)t);
  tile_pair_kernel<<<grid, dim3(32, 8), 0, st>>>(n, A, lda, op);
  EM_LAUNCHED();
}

// B <- G^-1 B G^-T for symmetric B (full storage in and out), the reference's sequence
// X = G^-1 L, B = G^-1 X^T, B <- (B + B^T)/2 (modal.py:63-68) with banded solves.
void band_sygst(cudaStream_t st, const BandChol& f, double* B, int64_t ldb) {
  band_solve(st, f, false, f.n, B, ldb);
  tile_pairs(st, f.n, B, ldb, 0);
  band_solve(st, f, false, f.n, B, ldb);
  tile_pairs(st, f.n, B, ldb, 1);
}

}  // namespace em
