// Blocked Cholesky (potrf) and triangular solves (trsm) in FP64.
//
// Reference: cholesky_kernel (_kernels.py:18-36) is an unblocked Crout loop that
// returns the first index whose pivot s = a_jj - sum_k c_jk^2 is not > 0;
// tri_lower_solve_mat / tri_lower_t_solve_mat (_kernels.py:56-79) are column-wise
// substitutions. Here: right-looking blocked potrf with a 128x128 diagonal block
// factored and inverted in shared memory (one CTA), the panel solved as a GEMM
// against the inverted block and the trailing update done by the lower-triangle
// DMMA GEMM; trsm likewise uses inverted diagonal blocks + DMMA GEMM updates.
// The failing pivot is reported with the reference's index semantics.
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

constexpr int PNB = 128;       // potrf / trsm block
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

// Factor the diagonal block A[k0:k0+bs, k0:k0+bs] (bs <= PNB), write the factor
// back (upper part zeroed) and its inverse to Dinv (PNB x PNB, ld PNB).
__global__ void __launch_bounds__(256) potf2_inv_kernel(double* A, int64_t lda, int64_t k0, int bs,
                                                        double* Dinv, int64_t* info) {
  extern __shared__ double sm[];
  double* S = sm;             // PNB x PLD
  double* tmp = S + PNB * PLD;  // PNB
  __shared__ int fail;
  if (*info >= 0) return;  // an earlier block already failed
  if (threadIdx.x == 0) fail = -1;
  for (int i = threadIdx.x; i < PNB * PNB; i += blockDim.x) {
    int r = i % PNB, c = i / PNB;
    double v;
    if (r < bs && c < bs)
      v = (r >= c) ? A[(k0 + r) + (k0 + c) * lda] : 0.0;
    else
      v = (r == c) ? 1.0 : 0.0;  // identity padding for a partial last block
    S[r + c * PLD] = v;
  }
  __syncthreads();
  for (int j = 0; j < bs; ++j) {
    const double s = S[j + j * PLD];
    if (!(s > 0.0)) {  // same test as the reference (NaN fails too)
      if (threadIdx.x == 0) fail = j;
      break;  // uniform: every thread read the same s
    }
    const double d = sqrt(s);
    __syncthreads();
    if (threadIdx.x == 0) S[j + j * PLD] = d;
    for (int i = j + 1 + threadIdx.x; i < bs; i += blockDim.x) S[i + j * PLD] /= d;
    __syncthreads();
    // trailing update of the lower triangle: S[i][k] -= S[i][j] S[k][j], j < k <= i
    const int m = bs - j - 1;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      const int i = j + 1 + idx % m, k = j + 1 + idx / m;
      if (k <= i) S[i + k * PLD] = fma(-S[i + j * PLD], S[k + j * PLD], S[i + k * PLD]);
    }
    __syncthreads();
  }
  __syncthreads();
  if (fail >= 0) {
    if (threadIdx.x == 0) *info = k0 + fail;
    return;
  }
  for (int i = threadIdx.x; i < bs * bs; i += blockDim.x) {
    int r = i % bs, c = i / bs;
    A[(k0 + r) + (k0 + c) * lda] = (r >= c) ? S[r + c * PLD] : 0.0;
  }
  smem_trtri_lower(S, PNB, PLD, tmp);
  for (int i = threadIdx.x; i < PNB * PNB; i += blockDim.x) {
    int r = i % PNB, c = i / PNB;
    Dinv[r + c * PNB] = S[r + c * PLD];
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

// Lower Cholesky in place. Returns the failing pivot (-1 = success); syncs the stream.
int64_t potrf(cudaStream_t st, int64_t n, double* A, int64_t lda) {
  if (n <= 0) return -1;
  DArr<int64_t> info(1, st);
  const int64_t minus1 = -1;
  EM_CK(cudaMemcpyAsync(info.p, &minus1, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  DBuf Dinv((size_t)PNB * PNB, st);
  DBuf P((size_t)n * PNB, st);
  const size_t smem = ((size_t)PNB * PLD + PNB) * sizeof(double);
  EM_CK(cudaFuncSetAttribute(potf2_inv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem));
  for (int64_t k0 = 0; k0 < n; k0 += PNB) {
    const int bs = (int)imin64(PNB, n - k0);
    potf2_inv_kernel<<<1, 256, smem, st>>>(A, lda, k0, bs, Dinv.p, info.p);
    EM_LAUNCHED();
    const int64_t m = n - k0 - bs;
    if (m <= 0) break;
    double* A21 = A + (k0 + bs) + k0 * lda;
    double* A22 = A + (k0 + bs) + (k0 + bs) * lda;
    // P = A21 * inv(L11)^T
    EM_CK(gemm(st, false, true, m, bs, bs, 1.0, A21, lda, Dinv.p, PNB, 0.0, P.p, n));
    // A22 -= P P^T (lower triangle)
    EM_CK(gemm(st, false, true, m, m, bs, -1.0, P.p, n, P.p, n, 1.0, A22, lda, true, 0));
    copy_matrix(st, false, m, bs, P.p, n, A21, lda);
  }
  // zero the strict upper triangle (the reference's factor is exactly lower)
  zero_upper(st, n, A, lda);
  int64_t h = -1;
  EM_CK(cudaMemcpyAsync(&h, info.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  return h;
}

// B <- C^-1 B (trans = false) or C^-T B (trans = true); C lower n x n, B n x m.
void trsm_lower(cudaStream_t st, bool trans, int64_t n, int64_t m, const double* C, int64_t ldc,
                double* B, int64_t ldb) {
  if (n <= 0 || m <= 0) return;
  const int64_t nblk = (n + PNB - 1) / PNB;
  DBuf Dinv((size_t)nblk * PNB * PNB, st);
  trtri_blocks(st, PNB, n, C, ldc, Dinv.p);
  DBuf T((size_t)PNB * m, st);
  if (!trans) {
    for (int64_t kb = 0; kb < nblk; ++kb) {
      const int64_t k0 = kb * PNB;
      const int bs = (int)imin64(PNB, n - k0);
      const double* Dk = Dinv.p + kb * PNB * PNB;
      EM_CK(gemm(st, false, false, bs, m, bs, 1.0, Dk, PNB, B + k0, ldb, 0.0, T.p, PNB));
      const int64_t rest = n - k0 - bs;
      if (rest > 0)
        EM_CK(gemm(st, false, false, rest, m, bs, -1.0, C + (k0 + bs) + k0 * ldc, ldc, T.p, PNB,
                   1.0, B + k0 + bs, ldb));
      copy_matrix(st, false, bs, m, T.p, PNB, B + k0, ldb);
    }
  } else {
    for (int64_t kb = nblk - 1; kb >= 0; --kb) {
      const int64_t k0 = kb * PNB;
      const int bs = (int)imin64(PNB, n - k0);
      const double* Dk = Dinv.p + kb * PNB * PNB;
      EM_CK(gemm(st, true, false, bs, m, bs, 1.0, Dk, PNB, B + k0, ldb, 0.0, T.p, PNB));
      if (k0 > 0)
        EM_CK(gemm(st, true, false, k0, m, bs, -1.0, C + k0, ldc, T.p, PNB, 1.0, B, ldb));
      copy_matrix(st, false, bs, m, T.p, PNB, B + k0, ldb);
    }
  }
}

}  // namespace em
