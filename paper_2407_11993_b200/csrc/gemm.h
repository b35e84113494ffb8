#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace em {

struct GemmArgs {
  int64_t m, n, k;
  const double* A;
  int64_t lda;
  const double* B;
  int64_t ldb;
  double* C;
  int64_t ldc;
  double alpha, beta;
  int64_t diag_off;  // lower mode: element (r, c) is written iff r + diag_off >= c
};

// C(m x n) = alpha * op(A) * op(B) + beta * C; column-major; op = transpose when ta/tb.
// lower: only the lower triangle (r + diag_off >= c) of C is computed/written.
cudaError_t gemm(cudaStream_t st, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                 int64_t ldc, bool lower = false, int64_t diag_off = 0);

// C = alpha * A * B + beta * C with A (m x k) LOWER triangular: only A(r, c) with c <= r
// is read (the stored upper part is ignored) and k-tiles past each row tile are skipped,
// i.e. half the flops of a square product (TRMM-like).
cudaError_t gemm_lower_a(cudaStream_t st, int64_t m, int64_t n, int64_t k, double alpha,
                         const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                         double* C, int64_t ldc);

// Many independent problems in one launch (device-resident argument array).
cudaError_t gemm_grouped(cudaStream_t st, bool ta, bool tb, const GemmArgs* d_probs, int nprob,
                         int max_tiles);

// TMA-fed persistent kernel for large aligned products (gemm_tma.cu); returns
// cudaErrorNotSupported when the product does not qualify (gemm() then takes the cp.async path).
cudaError_t gemm_tma(cudaStream_t st, bool ta, bool tb, const GemmArgs& p, bool lower);
// C (m x n) = A B for a symmetric A read from its lower triangle and the SYMM_BAND diagonals
// above it (gemm_tma.cu); cudaErrorNotSupported when TMA cannot address the operands.
constexpr int SYMM_BAND = 127;
// Column ownership of a distributed band reduction: g ranks, this one r; 64-column blocks
// dealt round-robin, block index = org + column / 64 (org: the operand's first column / 64).
struct GemmOwn {
  int g = 1, r = 0;
  int64_t org = 0;
};
// own.g > 1: only the k-tiles read from owned columns are added (this rank's partial).
cudaError_t gemm_symm_lower_tma(cudaStream_t st, int64_t m, int64_t n, const double* A,
                                int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc,
                                const GemmOwn& own = GemmOwn{});
// The LOWER product of gemm() on the column tiles this rank owns only.
cudaError_t gemm_lower_owned_tma(cudaStream_t st, bool ta, bool tb, const GemmArgs& p,
                                 const GemmOwn& own);
// 2-D TMA tensor map (a CUtensorMap at `map`) over a column-major operand; false when TMA
// cannot address it (base not 16-byte aligned, odd leading dimension, extents past int32).
bool tma_map_2d(void* map, const double* base, int64_t inner, int64_t outer, int64_t ld,
                int box_inner, int box_outer);
// C = alpha * sum_z W_z + beta * C over `splits` m x n partials (fixed order).
void splitk_reduce(cudaStream_t st, int64_t m, int64_t n, int splits, const double* ws,
                   double alpha, double beta, double* C, int64_t ldc, int lower, int64_t diag_off);

cudaError_t scale_matrix(cudaStream_t st, int64_t m, int64_t n, double beta, double* C, int64_t ldc,
                         bool lower, int64_t diag_off);

}  // namespace em
