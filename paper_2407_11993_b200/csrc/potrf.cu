// Cholesky (potrf) and triangular solves (trsm) in FP64, recursive so that
// almost all flops land in large-K DMMA GEMMs.
//
// Reference: cholesky_kernel (_kernels.py:18-36) is an unblocked Crout loop that
// returns the first index whose pivot s = a_jj - sum_k c_jk^2 is not > 0;
// tri_lower_solve_mat / tri_lower_t_solve_mat (_kernels.py:56-79) are column-wise
// substitutions.
//
//   potrf(A) = [ potrf(A11);  A21 <- A21 L11^-T;  A22 -= A21 A21^T;  potrf(A22) ]
//   leaves: 128x128 diagonal blocks factored AND inverted in shared memory by one
//   CTA (the inverse feeds every trsm leaf as a GEMM); the failing pivot is
//   reported with the reference's global index.
//   trsm: the same split; B2 -= L21 X1 is one GEMM with K = n/2, n/4, ...
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

constexpr int PNB = 128;       // leaf block
constexpr int PLD = PNB + 1;   // smem leading dimension

// In-place inversion of the lower-triangular n x n matrix in shared memory
// (column-major, leading dimension ld). Column j (from the right):
// a_jj <- 1/a_jj;  A[j+1:, j] <- -a_jj * Ainv[j+1:, j+1:] * A[j+1:, j].
EM_DEVINL void smem_trtri_lower(double* A, int n, int ld, double* tmp) {
  for (int j = n - 1; j >= 0; --j) {
    __syncthreads();
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) tmp[i] = A[i + j * ld];
    __syncthreads();
    const double ajj = 1.0 / A[j + j * ld];
    for (int i = j + 1 + threadIdx.x; i < n; i += blockDim.x) {
      double s = 0.0;
      for (int k = j + 1; k <= i; ++k) s = fma(A[i + k * ld], tmp[k], s);
      A[i + j * ld] = -ajj * s;
    }
    __syncthreads();
    if (threadIdx.x == 0) A[j + j * ld] = ajj;
  }
  __syncthreads();
}

// Factor the diagonal block A[0:bs, 0:bs] (bs <= PNB; global offset k0 for the
// pivot index), write the factor back (upper part zeroed) and its inverse to
// Dinv (PNB x PNB, ld PNB).
//
// Blocked in shared memory with 32 x 32 blocks so that only the 32-wide diagonal
// factorisations are sequential (one warp each, no block barriers):
//   for each block column kb: warp 0 factors and inverts L_kk; the panel below is
//   L_ik = A_ik L_kk^-T (a product with the inverse); the trailing lower part gets
//   A -= P P^T.  Then the off-diagonal blocks of the inverse follow block-diagonal by
//   block-diagonal: Linv_ij = -Linv_ii sum_{k=j}^{i-1} L_ik Linv_kj.
// Storage: L in the lower triangle of S (with its diagonal), Linv's strictly lower
// entries transposed into the upper triangle (Linv[r][c] at S[c + r*PLD]), Linv's
// diagonal in dinv[]. A failing pivot (s <= 0 or NaN, the reference's test) aborts
// with the global index of the first failing column.
constexpr int PB = 32;  // inner block

EM_DEVINL double linv_at(const double* S, const double* dinv, int r, int c) {
  return r == c ? dinv[r] : (r > c ? S[c + r * PLD] : 0.0);
}

__global__ void __launch_bounds__(256, 1) potf2_inv_kernel(double* A, int64_t lda, int64_t k0, int bs,
                                                        double* Dinv, int64_t* info) {
  extern __shared__ double sm[];
  double* S = sm;                // PNB x PLD
  double* dinv = S + PNB * PLD;  // PNB
  __shared__ int fail;
  if (*info >= 0) return;  // an earlier block already failed
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) fail = -1;
  for (int i = tid; i < PNB * PNB; i += blockDim.x) {
    const int r = i % PNB, c = i / PNB;
    double v;
    if (r < bs && c < bs)
      v = (r >= c) ? A[r + c * lda] : 0.0;
    else
      v = (r == c) ? 1.0 : 0.0;  // identity padding for a partial block
    S[r + c * PLD] = v;
  }
  __syncthreads();
  for (int kb = 0; kb < PNB / PB; ++kb) {
    const int o = kb * PB;
    if (warp == 0) {
      // unblocked Cholesky of the 32 x 32 diagonal block in registers: lane l holds row
      // o + l (a[k], k <= l) and gets the column-j entries of the other rows by shuffle
      double a[PB];
#pragma unroll
      for (int k = 0; k < PB; ++k) a[k] = (k <= lane) ? S[(o + lane) + (o + k) * PLD] : 0.0;
      int f = -1;
#pragma unroll
      for (int j = 0; j < PB; ++j) {
        const double sj = __shfl_sync(0xffffffffu, a[j], j);  // the pivot, in every lane
        if (!(sj > 0.0) && f < 0) f = o + j;  // (the rest of the block is then unused)
        const double d = sqrt(sj);
        const double lj = a[j] * (1.0 / d);
        if (lane == j) a[j] = d;
        if (lane > j) a[j] = lj;
#pragma unroll
        for (int k = 0; k < PB; ++k) {  // (constant trip count: a[] stays in registers)
          if (k > j) {
            const double lk = __shfl_sync(0xffffffffu, lj, k);
            if (lane >= k) a[k] = fma(-lj, lk, a[k]);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < PB; ++k)
        if (k <= lane) S[(o + lane) + (o + k) * PLD] = a[k];
      __syncwarp();
      if (f >= 0) {
        if (lane == 0) fail = f;
      } else {
        // inverse of the block, column c = lane kept in registers:
        // X[r][c] = -(sum_{k=c}^{r-1} L_rk X[k][c]) / L_rr
        const int c = lane;
        const double dc = 1.0 / S[(o + c) + (o + c) * PLD];
        dinv[o + c] = dc;
        __syncwarp();
        double x[PB];
#pragma unroll
        for (int r = 0; r < PB; ++r) x[r] = (r == c) ? dc : 0.0;
#pragma unroll
        for (int r = 1; r < PB; ++r) {
          double a0 = 0.0, a1 = 0.0;
#pragma unroll
          for (int k = 0; k < r; ++k) {
            const double l = S[(o + r) + (o + k) * PLD];
            if (k & 1)
              a1 = fma(l, x[k], a1);
            else
              a0 = fma(l, x[k], a0);
          }
          if (r > c) x[r] = -(a0 + a1) * dinv[o + r];
        }
#pragma unroll
        for (int r = 0; r < PB; ++r)
          if (r > c) S[(o + c) + (o + r) * PLD] = x[r];
      }
    }
    __syncthreads();
    if (fail >= 0) break;
    const int mp = PNB - o - PB;  // rows below the diagonal block
    if (mp <= 0) break;
    // panel: L[o+PB+i][o+c] = sum_{k<=c} A[o+PB+i][o+k] Linv_kk[c][k], 4 x 4 per thread
    {
      const int nbr = mp / 4, nbt = nbr * (PB / 4);
      double acc[4][4];
      const bool act = tid < nbt;
      const int bi = tid % (nbr > 0 ? nbr : 1), bc = tid / (nbr > 0 ? nbr : 1);
      const int r0 = o + PB + 4 * bi, c0 = 4 * bc;
      if (act) {
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
        // k < c0: Linv_kk[c][k] is a strictly-lower entry (packed upper storage); the
        // last four k (the 4 x 4 diagonal piece) go through linv_at
        for (int k = 0; k < c0 + 4; ++k) {
          double a[4], b[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) a[x] = S[(r0 + x) + (o + k) * PLD];
          if (k < c0) {
#pragma unroll
            for (int y = 0; y < 4; ++y) b[y] = S[(o + k) + (o + c0 + y) * PLD];
          } else {
#pragma unroll
            for (int y = 0; y < 4; ++y) b[y] = linv_at(S, dinv, o + c0 + y, o + k);
          }
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
        }
      }
      __syncthreads();
      if (act) {
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) S[(r0 + x) + (o + c0 + y) * PLD] = acc[x][y];
      }
      __syncthreads();
    }
    // trailing: A[r][q] -= sum_k P[r][k] P[q][k], r >= q >= o + PB, in 4 x 4 blocks
    {
      const int nb4 = mp / 4;
      const int nblk = nb4 * (nb4 + 1) / 2;
      for (int b = tid; b < nblk; b += 256) {
        // block (bi, bj), bi >= bj, from the linear index
        int bi = (int)((sqrtf(8.0f * b + 1.0f) - 1.0f) * 0.5f);
        while (bi * (bi + 1) / 2 > b) --bi;
        while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
        const int bj = b - bi * (bi + 1) / 2;
        const int r0 = o + PB + 4 * bi, q0 = o + PB + 4 * bj;
        double acc[4][4];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
        for (int k = 0; k < PB; ++k) {
          double pr[4], pq[4];
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            pr[x] = S[(r0 + x) + (o + k) * PLD];
            pq[x] = S[(q0 + x) + (o + k) * PLD];
          }
#pragma unroll
          for (int x = 0; x < 4; ++x)
#pragma unroll
            for (int y = 0; y < 4; ++y) acc[x][y] = fma(pr[x], pq[y], acc[x][y]);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y)
            if (r0 + x >= q0 + y) S[(r0 + x) + (q0 + y) * PLD] -= acc[x][y];
      }
      __syncthreads();
    }
  }
  __syncthreads();
  if (fail >= 0) {
    if (tid == 0) *info = k0 + fail;
    return;
  }
  // off-diagonal blocks of the inverse, by block distance d = i - j; each thread owns a
  // 4 x 4 piece of one block (rows a0.. of block i, columns b0.. of block j)
  for (int d = 1; d < PNB / PB; ++d) {
    const int nblk = PNB / PB - d;
    const int per = (PB / 4) * (PB / 4);  // 64 pieces per block
    const bool act = tid < nblk * per;
    const int blk = tid / per, pc = tid % per;
    const int j = blk, i = j + d;
    const int r0 = i * PB + 4 * (pc % (PB / 4)), c0 = j * PB + 4 * (pc / (PB / 4));
    double acc[4][4];
    // W = sum_{k=j}^{i-1} L_ik Linv_kj  (Linv[kk][c] = 0 for kk < c)
    if (act) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
      for (int kk = c0; kk < i * PB; ++kk) {
        double a[4], b[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) a[x] = S[(r0 + x) + kk * PLD];
        if (kk >= c0 + 4) {  // strictly below the 4 x 4 diagonal piece: packed storage
#pragma unroll
          for (int y = 0; y < 4; ++y) b[y] = S[(c0 + y) + kk * PLD];
        } else {
#pragma unroll
          for (int y = 0; y < 4; ++y) b[y] = linv_at(S, dinv, kk, c0 + y);
        }
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
      }
    }
    __syncthreads();
    if (act) {  // W[r][c] into the (still empty) packed slot of Linv_ij
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) S[(c0 + y) + (r0 + x) * PLD] = acc[x][y];
    }
    __syncthreads();
    // Linv_ij = -Linv_ii W
    if (act) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = 0.0;
      for (int kk = i * PB; kk < r0 + 4; ++kk) {
        double a[4], b[4];
        if (kk < r0) {  // strictly lower entries of Linv_ii: packed storage
#pragma unroll
          for (int x = 0; x < 4; ++x) a[x] = S[kk + (r0 + x) * PLD];
        } else {
#pragma unroll
          for (int x = 0; x < 4; ++x) a[x] = linv_at(S, dinv, r0 + x, kk);
        }
#pragma unroll
        for (int y = 0; y < 4; ++y) b[y] = S[(c0 + y) + kk * PLD];  // W[kk][c]
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) acc[x][y] = fma(a[x], b[y], acc[x][y]);
      }
    }
    __syncthreads();
    if (act) {
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) S[(c0 + y) + (r0 + x) * PLD] = -acc[x][y];
    }
    __syncthreads();
  }
  for (int i = tid; i < bs * bs; i += blockDim.x) {
    const int r = i % bs, c = i / bs;
    A[r + c * lda] = (r >= c) ? S[r + c * PLD] : 0.0;
  }
  for (int i = tid; i < PNB * PNB; i += blockDim.x) {
    const int r = i % PNB, c = i / PNB;
    Dinv[r + c * PNB] = linv_at(S, dinv, r, c);
  }
}

// Inverses of all NB x NB diagonal blocks of a lower-triangular factor.
template <int NB>
__global__ void __launch_bounds__(256) trtri_blocks_kernel(int64_t n, const double* C,
                                                          int64_t ldc, double* Dinv) {
  extern __shared__ double sm[];
  constexpr int LD = NB + 1;
  double* S = sm;
  double* tmp = S + NB * LD;
  const int64_t k0 = blockIdx.x * (int64_t)NB;
  const int bs = (int)imin64(NB, n - k0);
  for (int i = threadIdx.x; i < NB * NB; i += blockDim.x) {
    int r = i % NB, c = i / NB;
    double v;
    if (r < bs && c < bs)
      v = (r >= c) ? C[(k0 + r) + (k0 + c) * ldc] : 0.0;
    else
      v = (r == c) ? 1.0 : 0.0;
    S[r + c * LD] = v;
  }
  __syncthreads();
  smem_trtri_lower(S, NB, LD, tmp);
  double* D = Dinv + blockIdx.x * (int64_t)NB * NB;
  for (int i = threadIdx.x; i < NB * NB; i += blockDim.x) {
    int r = i % NB, c = i / NB;
    D[r + c * NB] = S[r + c * LD];
  }
}

void trtri_blocks(cudaStream_t st, int nb, int64_t n, const double* C, int64_t ldc, double* Dinv) {
  int64_t nblk = (n + nb - 1) / nb;
  if (nblk <= 0) return;
  if (nb == 64) {
    size_t smem = (64 * 65 + 64) * sizeof(double);
    trtri_blocks_kernel<64><<<(unsigned)nblk, 256, smem, st>>>(n, C, ldc, Dinv);
  } else if (nb == 128) {
    size_t smem = (128 * 129 + 128) * sizeof(double);
    EM_CK(cudaFuncSetAttribute(trtri_blocks_kernel<128>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    trtri_blocks_kernel<128><<<(unsigned)nblk, 256, smem, st>>>(n, C, ldc, Dinv);
  } else {
    throw ArgError{"trtri_blocks: nb must be 64 or 128"};
  }
  EM_LAUNCHED();
}

// split point: a multiple of PNB near the middle
static int64_t split_point(int64_t n) {
  const int64_t nbk = (n + PNB - 1) / PNB;
  return imax64(1, nbk / 2) * PNB;
}

// ---- trsm (left): B <- C^-1 B or C^-T B; Dinv holds inverses of C's PNB diagonal
// blocks, block index offset by blk0 (block of C[0,0]); T is PNB x m workspace.
static void trsm_left_rec(cudaStream_t st, bool trans, int64_t n, int64_t m, const double* C,
                          int64_t ldc, double* B, int64_t ldb, const double* Dinv, int64_t blk0,
                          double* T) {
  if (n <= 0 || m <= 0) return;
  if (n <= PNB) {
    const double* D = Dinv + blk0 * PNB * PNB;
    EM_CK(gemm(st, trans, false, n, m, n, 1.0, D, PNB, B, ldb, 0.0, T, PNB));
    copy_matrix(st, false, n, m, T, PNB, B, ldb);
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  const double* C21 = C + n1;                 // n2 x n1
  const double* C22 = C + n1 + n1 * ldc;
  if (!trans) {
    trsm_left_rec(st, false, n1, m, C, ldc, B, ldb, Dinv, blk0, T);
    EM_CK(gemm(st, false, false, n2, m, n1, -1.0, C21, ldc, B, ldb, 1.0, B + n1, ldb));
    trsm_left_rec(st, false, n2, m, C22, ldc, B + n1, ldb, Dinv, blk0 + n1 / PNB, T);
  } else {
    // C^T = [C11^T C21^T; 0 C22^T]
    trsm_left_rec(st, true, n2, m, C22, ldc, B + n1, ldb, Dinv, blk0 + n1 / PNB, T);
    EM_CK(gemm(st, true, false, n1, m, n2, -1.0, C21, ldc, B + n1, ldb, 1.0, B, ldb));
    trsm_left_rec(st, true, n1, m, C, ldc, B, ldb, Dinv, blk0, T);
  }
}

// ---- trsm (right, transposed): B (m x n) <- B C^-T; T is m x PNB workspace.
static void trsm_right_t_rec(cudaStream_t st, int64_t m, int64_t n, const double* C, int64_t ldc,
                             double* B, int64_t ldb, const double* Dinv, int64_t blk0, double* T,
                             int64_t ldt) {
  if (n <= 0 || m <= 0) return;
  if (n <= PNB) {
    const double* D = Dinv + blk0 * PNB * PNB;
    EM_CK(gemm(st, false, true, m, n, n, 1.0, B, ldb, D, PNB, 0.0, T, ldt));
    copy_matrix(st, false, m, n, T, ldt, B, ldb);
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  const double* C21 = C + n1;
  const double* C22 = C + n1 + n1 * ldc;
  // X C^T = B:  X1 = B1 C11^-T;  B2 -= X1 C21^T;  X2 = B2 C22^-T
  trsm_right_t_rec(st, m, n1, C, ldc, B, ldb, Dinv, blk0, T, ldt);
  EM_CK(gemm(st, false, true, m, n2, n1, -1.0, B, ldb, C21, ldc, 1.0, B + n1 * ldb, ldb));
  trsm_right_t_rec(st, m, n2, C22, ldc, B + n1 * ldb, ldb, Dinv, blk0 + n1 / PNB, T, ldt);
}

// ---- sygst: A <- G^-1 A G^-T (A symmetric, full storage in, lower triangle valid out)
// Recursive two-sided reduction (the ReLAPACK/LAPACK itype-1 scheme, n^3 flops instead
// of the 2 n^3 of two full triangular solves):
//   A11 <- G11^-1 A11 G11^-T                      (recursion)
//   A21 <- A21 G11^-T;  A21 -= 1/2 G21 A11
//   A22 -= A21 G21^T + G21 A21^T                  (two lower GEMMs, then mirrored)
//   A21 -= 1/2 G21 A11;  A21 <- G22^-1 A21
//   A22 <- G22^-1 A22 G22^-T                      (recursion)
// Leaves (n <= 128): A <- D A D^T with the diagonal-block inverse D of potrf.
static void sygst_rec(cudaStream_t st, int64_t n, double* A, int64_t lda, const double* G,
                      int64_t ldg, const double* Dinv, int64_t blk0, double* T, int64_t ldt) {
  if (n <= 0) return;
  if (n <= PNB) {
    const double* D = Dinv + blk0 * PNB * PNB;
    EM_CK(gemm(st, false, false, n, n, n, 1.0, D, PNB, A, lda, 0.0, T, ldt));
    EM_CK(gemm(st, false, true, n, n, n, 1.0, T, ldt, D, PNB, 0.0, A, lda));
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  double* A21 = A + n1;
  double* A22 = A + n1 + n1 * lda;
  const double* G21 = G + n1;
  const double* G22 = G + n1 + n1 * ldg;
  sygst_rec(st, n1, A, lda, G, ldg, Dinv, blk0, T, ldt);
  mirror_lower(st, n1, A, lda);  // A11 is used as a full symmetric matrix below
  trsm_right_t_rec(st, n2, n1, G, ldg, A21, lda, Dinv, blk0, T, ldt);
  EM_CK(gemm(st, false, false, n2, n1, n1, -0.5, G21, ldg, A, lda, 1.0, A21, lda));
  EM_CK(gemm(st, false, true, n2, n2, n1, -1.0, A21, lda, G21, ldg, 1.0, A22, lda, true, 0));
  EM_CK(gemm(st, false, true, n2, n2, n1, -1.0, G21, ldg, A21, lda, 1.0, A22, lda, true, 0));
  mirror_lower(st, n2, A22, lda);
  EM_CK(gemm(st, false, false, n2, n1, n1, -0.5, G21, ldg, A, lda, 1.0, A21, lda));
  trsm_left_rec(st, false, n2, n1, G22, ldg, A21, lda, Dinv, blk0 + n1 / PNB, T);
  sygst_rec(st, n2, A22, lda, G22, ldg, Dinv, blk0 + n1 / PNB, T, ldt);
}

void sygst_lower(cudaStream_t st, int64_t n, double* A, int64_t lda, const double* G, int64_t ldg,
                 const double* Dinv) {
  if (n <= 0) return;
  // T: PNB x n for the left-trsm leaves, n x PNB for the right ones and the sygst leaves
  DBuf T((size_t)n * PNB, st);
  sygst_rec(st, n, A, lda, G, ldg, Dinv, 0, T.p, n);
}

// ---- potrf --------------------------------------------------------------------------
static void potrf_rec(cudaStream_t st, int64_t n, double* A, int64_t lda, int64_t k0,
                      double* Dinv, int64_t* info, double* T, int64_t ldt, size_t smem) {
  if (n <= PNB) {
    potf2_inv_kernel<<<1, 256, smem, st>>>(A, lda, k0, (int)n, Dinv + (k0 / PNB) * PNB * PNB,
                                           info);
    EM_LAUNCHED();
    return;
  }
  const int64_t n1 = split_point(n), n2 = n - n1;
  double* A21 = A + n1;
  double* A22 = A + n1 + n1 * lda;
  potrf_rec(st, n1, A, lda, k0, Dinv, info, T, ldt, smem);
  trsm_right_t_rec(st, n2, n1, A, lda, A21, lda, Dinv, k0 / PNB, T, ldt);
  EM_CK(gemm(st, false, true, n2, n2, n1, -1.0, A21, lda, A21, lda, 1.0, A22, lda, true, 0));
  potrf_rec(st, n2, A22, lda, k0 + n1, Dinv, info, T, ldt, smem);
}

// Lower Cholesky in place. Returns the failing pivot (-1 = success); syncs the stream.
// If Dinv_out is given (>= ceil(n/128) * 128^2 doubles) it receives the inverses of
// the 128 x 128 diagonal blocks of the factor.
int64_t potrf(cudaStream_t st, int64_t n, double* A, int64_t lda, double* Dinv_out) {
  if (n <= 0) return -1;
  DArr<int64_t> info(1, st);
  const int64_t minus1 = -1;
  EM_CK(cudaMemcpyAsync(info.p, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  const int64_t nblk = (n + PNB - 1) / PNB;
  DBuf Dloc;
  double* Dinv = Dinv_out;
  if (!Dinv) {
    Dloc.alloc((size_t)nblk * PNB * PNB, st);
    Dinv = Dloc.p;
  }
  DBuf T((size_t)n * PNB, st);
  const size_t smem = ((size_t)PNB * PLD + PNB) * sizeof(double);
  EM_CK(cudaFuncSetAttribute(potf2_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem));
  potrf_rec(st, n, A, lda, 0, Dinv, info.p, T.p, n, smem);
  zero_upper(st, n, A, lda);  // the reference's factor is exactly lower
  int64_t h = -1;
  EM_CK(cudaMemcpyAsync(&h, info.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  return h;
}

int64_t potrf(cudaStream_t st, int64_t n, double* A, int64_t lda) {
  return potrf(st, n, A, lda, nullptr);
}

// B <- C^-1 B (trans = false) or C^-T B (trans = true); C lower n x n, B n x m.
void trsm_lower(cudaStream_t st, bool trans, int64_t n, int64_t m, const double* C, int64_t ldc,
                double* B, int64_t ldb, const double* Dinv_in) {
  if (n <= 0 || m <= 0) return;
  const int64_t nblk = (n + PNB - 1) / PNB;
  DBuf Dloc;
  const double* Dinv = Dinv_in;
  if (!Dinv) {
    Dloc.alloc((size_t)nblk * PNB * PNB, st);
    trtri_blocks(st, PNB, n, C, ldc, Dloc.p);
    Dinv = Dloc.p;
  }
  DBuf T((size_t)PNB * m, st);
  trsm_left_rec(st, trans, n, m, C, ldc, B, ldb, Dinv, 0, T.p);
}

void trsm_lower(cudaStream_t st, bool trans, int64_t n, int64_t m, const double* C, int64_t ldc,
                double* B, int64_t ldb) {
  trsm_lower(st, trans, n, m, C, ldc, B, ldb, nullptr);
}

}  // namespace em
