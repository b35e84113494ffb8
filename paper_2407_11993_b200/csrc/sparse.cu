// Sparse-aware product R V for the post-eigensolve quantities r_n = diag(V^T R V)
// and V^T R (modal.py:80-81). The reference stores R dense (linalg.SymMatrix) and
// multiplies densely; the synthetic plates' R is a 7-point stencil, so when R has
// few nonzeros a CSR copy is built on the device (two passes over the dense
// matrix) and R V becomes an HBM-bound SpMM instead of a 2 N^3 GEMM. The sum
// over each row's nonzeros runs in increasing column order, i.e. the same terms
// in the same order the dense product accumulates (zeros contribute exactly 0).
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "linalg.h"

namespace em {

// nnz per row of a symmetric matrix given by its LOWER triangle (column-major; the upper
// triangle is never read: SymMatrix semantics, E/linalg.py:24-59). Row i = the strided
// entries A[i + k lda] for k < i, then the contiguous column segment A[k + i lda], k >= i.
// One warp per row.
__global__ void csr_count_kernel(int64_t n, const double* __restrict__ A, int64_t lda,
                                 int64_t* __restrict__ cnt) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  int64_t c = 0;
  for (int64_t k = lane; k < row; k += 32) c += (A[row + k * lda] != 0.0);
  const double* col = A + row * lda;
  for (int64_t k = row + lane; k < n; k += 32) c += (col[k] != 0.0);
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[row] = c;
}

// fill: one warp per row, ballot-compacted in increasing column order
__global__ void csr_fill_kernel(int64_t n, const double* __restrict__ A, int64_t lda,
                                const int64_t* __restrict__ rowptr, int* __restrict__ colidx,
                                double* __restrict__ val) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* col = A + row * lda;
  int64_t pos = rowptr[row];
  for (int64_t k0 = 0; k0 < n; k0 += 32) {
    const int64_t k = k0 + lane;
    const double v = k >= n ? 0.0 : (k < row ? A[row + k * lda] : col[k]);
    const unsigned mask = __ballot_sync(0xffffffffu, v != 0.0);
    if (v != 0.0) {
      const int off = __popc(mask & ((1u << lane) - 1u));
      colidx[pos + off] = (int)k;
      val[pos + off] = v;
    }
    pos += __popc(mask);
  }
}

// C (n x m) = A_csr (n x n) * B (n x m); thread per (row, column)
__global__ void csr_spmm_kernel(int64_t n, int64_t m, const int64_t* __restrict__ rowptr,
                                const int* __restrict__ colidx, const double* __restrict__ val,
                                const double* __restrict__ B, int64_t ldb, double* __restrict__ C,
                                int64_t ldc) {
  const int64_t total = n * m;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t % n, j = t / n;
    const double* b = B + j * ldb;
    double s = 0.0;
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s = fma(val[p], b[colidx[p]], s);
    C[i + j * ldc] = s;
  }
}

// writes the CSR entries back into full storage (both triangles: the restored matrix is
// exactly symmetric)
__global__ void csr_scatter_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                   const int* __restrict__ colidx, const double* __restrict__ val,
                                   double* __restrict__ A, int64_t lda) {
  const int64_t row = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  double* col = A + row * lda;  // symmetric: column `row` == row `row`
  for (int64_t p = rowptr[row] + lane; p < rowptr[row + 1]; p += 32) col[colidx[p]] = val[p];
}

// Device CSR copy of a symmetric A (its lower triangle) when it has at most max_fill * n^2
// nonzeros; returns false (and builds nothing) when A is too dense.
// band storage -> CSR, one thread per row, columns ascending (pass 0 counts, 1 fills)
__global__ void csr_band_kernel(int64_t n, const double* __restrict__ Rb, int64_t ldrb,
                                int64_t bw, int pass, int64_t* __restrict__ cnt,
                                const int64_t* __restrict__ rowptr, int* __restrict__ col,
                                double* __restrict__ val) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c = 0, o = pass ? rowptr[i] : 0;
  const int64_t j0 = i - bw < 0 ? 0 : i - bw, j1 = i + bw >= n ? n - 1 : i + bw;
  for (int64_t j = j0; j <= j1; ++j) {
    const double v = j <= i ? Rb[(i - j) + j * ldrb] : Rb[(j - i) + i * ldrb];
    if (v == 0.0) continue;
    if (pass) {
      col[o + c] = (int)j;
      val[o + c] = v;
    }
    ++c;
  }
  if (!pass) cnt[i] = c;
}

void csr_from_band(cudaStream_t st, int64_t n, const double* Rb, int64_t ldrb, int64_t bw,
                   Csr& out) {
  DArr<int64_t> cnt(n + 1, st);
  const unsigned g = (unsigned)((n + 255) / 256);
  csr_band_kernel<<<g, 256, 0, st>>>(n, Rb, ldrb, bw, 0, cnt.p, nullptr, nullptr, nullptr);
  EM_LAUNCHED();
  std::vector<int64_t> h(n + 1, 0);
  EM_CK(cudaMemcpyAsync(h.data() + 1, cnt.p, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) h[i + 1] += h[i];
  EM_CK(cudaMemcpyAsync(cnt.p, h.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  out.n = n;
  out.nnz = h[n];
  out.rowptr = std::move(cnt);
  out.colidx.alloc(imax64(out.nnz, 1), st);
  out.val.alloc(imax64(out.nnz, 1), st);
  csr_band_kernel<<<g, 256, 0, st>>>(n, Rb, ldrb, bw, 1, nullptr, out.rowptr.p, out.colidx.p,
                                     out.val.p);
  EM_LAUNCHED();
  EM_CK(cudaStreamSynchronize(st));  // host vector h lifetime
}

bool csr_from_dense(cudaStream_t st, int64_t n, const double* A, int64_t lda, double max_fill,
                    Csr& out) {
  if (n <= 0) return false;
  DArr<int64_t> cnt(n + 1, st);
  csr_count_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(n, A, lda, cnt.p);
  EM_LAUNCHED();
  std::vector<int64_t> h(n + 1, 0);
  EM_CK(cudaMemcpyAsync(h.data() + 1, cnt.p, n * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  for (int64_t i = 0; i < n; ++i) h[i + 1] += h[i];
  const int64_t nnz = h[n];
  if ((double)nnz > max_fill * (double)n * (double)n) return false;
  EM_CK(cudaMemcpyAsync(cnt.p, h.data(), (n + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  out.n = n;
  out.nnz = nnz;
  out.rowptr = std::move(cnt);
  out.colidx.alloc(imax64(nnz, 1), st);
  out.val.alloc(imax64(nnz, 1), st);
  csr_fill_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(n, A, lda, out.rowptr.p,
                                                          out.colidx.p, out.val.p);
  EM_LAUNCHED();
  EM_CK(cudaStreamSynchronize(st));  // host vector h lifetime
  return true;
}

// C (n x m) = A_csr B
void csr_mm(cudaStream_t st, const Csr& a, int64_t m, const double* B, int64_t ldb, double* C,
            int64_t ldc) {
  const int64_t total = a.n * m;
  if (total <= 0) return;
  const int blocks = (int)imin64((total + 255) / 256, 32 * num_sms());
  csr_spmm_kernel<<<blocks, 256, 0, st>>>(a.n, m, a.rowptr.p, a.colidx.p, a.val.p, B, ldb, C,
                                          ldc);
  EM_LAUNCHED();
}

// y = alpha A x + beta y, one thread per row; each row's nonzeros summed in increasing
// column order (the reference's dense loop order with its exact-zero terms skipped)
__global__ void csr_spmv_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                const int* __restrict__ colidx, const double* __restrict__ val,
                                double alpha, const double* __restrict__ x, double beta,
                                double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s += val[p] * x[colidx[p]];
  y[i] = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * y[i]);
}

void csr_spmv(cudaStream_t st, const Csr& a, double alpha, const double* x, double beta,
              double* y) {
  if (a.n <= 0) return;
  csr_spmv_kernel<<<(unsigned)((a.n + 255) / 256), 256, 0, st>>>(a.n, a.rowptr.p, a.colidx.p,
                                                                  a.val.p, alpha, x, beta, y);
  EM_LAUNCHED();
}

// A (n x n, full storage) <- the matrix held in CSR (every other entry zero).
void csr_to_dense(cudaStream_t st, const Csr& a, double* A, int64_t lda) {
  if (lda == a.n) {
    EM_CK(cudaMemsetAsync(A, 0, (size_t)a.n * a.n * sizeof(double), st));
  } else {
    EM_CK(cudaMemset2DAsync(A, lda * sizeof(double), 0, a.n * sizeof(double), a.n, st));
  }
  csr_scatter_kernel<<<(unsigned)((a.n + 7) / 8), 256, 0, st>>>(a.n, a.rowptr.p, a.colidx.p,
                                                                a.val.p, A, lda);
  EM_LAUNCHED();
}

// out[j] = v_j^T A v_j for the columns of V (r_n = diag(V^T R V), modal.py:80) without an
// N x N product buffer: block j forms (A v_j)_i row by row from the CSR copy (L2-resident)
// and reduces v_ij (A v_j)_i in a fixed order. V is read once: HBM-bound.
__global__ void csr_quadform_kernel(int64_t n, const int64_t* __restrict__ rowptr,
                                    const int* __restrict__ colidx, const double* __restrict__ val,
                                    const double* __restrict__ V, int64_t ldv,
                                    double* __restrict__ out) {
  __shared__ double red[32];
  const double* v = V + blockIdx.x * ldv;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    double t = 0.0;
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) t = fma(val[p], v[colidx[p]], t);
    s = fma(v[i], t, s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[blockIdx.x] = t;
  }
}

void csr_quadform(cudaStream_t st, const Csr& a, int64_t m, const double* V, int64_t ldv,
                  double* out) {
  if (a.n <= 0 || m <= 0) return;
  csr_quadform_kernel<<<(unsigned)m, 256, 0, st>>>(a.n, a.rowptr.p, a.colidx.p, a.val.p, V, ldv,
                                                   out);
  EM_LAUNCHED();
}

// C = A B using CSR when A (symmetric, n x n) has at most max_fill * n^2 nonzeros.
// Returns false (and does nothing) when A is too dense.
bool sym_sparse_mm(cudaStream_t st, int64_t n, const double* A, int64_t lda, int64_t m,
                   const double* B, int64_t ldb, double* C, int64_t ldc, double max_fill) {
  if (n <= 0 || m <= 0) return true;
  Csr a;
  if (!csr_from_dense(st, n, A, lda, max_fill, a)) return false;
  csr_mm(st, a, m, B, ldb, C, ldc);
  EM_CK(cudaStreamSynchronize(st));  // device temporaries lifetime
  return true;
}

}  // namespace em
