// Internal dense FP64 linear-algebra entry points (device pointers, column-major).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "ctx.h"

struct em_td2_plan;
struct em_td1_plan;

namespace em {

// potrf.cu
int64_t potrf(cudaStream_t st, int64_t n, double* A, int64_t lda);  // -1 ok, else pivot
// also returns the inverses of the 128x128 diagonal blocks (ceil(n/128) * 128^2 doubles)
int64_t potrf(cudaStream_t st, int64_t n, double* A, int64_t lda, double* Dinv_out);
void trsm_lower(cudaStream_t st, bool trans, int64_t n, int64_t m, const double* C, int64_t ldc,
                double* B, int64_t ldb);
void trsm_lower(cudaStream_t st, bool trans, int64_t n, int64_t m, const double* C, int64_t ldc,
                double* B, int64_t ldb, const double* Dinv);
constexpr int kTrsmBlock = 128;
void trtri_blocks(cudaStream_t st, int nb, int64_t n, const double* C, int64_t ldc, double* Dinv);
// A <- G^-1 A G^-T for symmetric A (full storage in; the lower triangle is valid on exit),
// G lower with its 128-block diagonal inverses Dinv (from potrf). n^3 flops.
void sygst_lower(cudaStream_t st, int64_t n, double* A, int64_t lda, const double* G, int64_t ldg,
                 const double* Dinv);

// sparse.cu: device CSR of a symmetric matrix stored dense
struct Csr {
  int64_t n = 0, nnz = 0;
  DArr<int64_t> rowptr;
  DArr<int> colidx;
  DBuf val;
};
bool csr_from_dense(cudaStream_t st, int64_t n, const double* A, int64_t lda, double max_fill,
                    Csr& out);
void csr_mm(cudaStream_t st, const Csr& a, int64_t m, const double* B, int64_t ldb, double* C,
            int64_t ldc);
void csr_to_dense(cudaStream_t st, const Csr& a, double* A, int64_t lda);
// CSR of a symmetric matrix given in lower band storage (Rb[(i - j) + j ldrb], i - j <= bw)
void csr_from_band(cudaStream_t st, int64_t n, const double* Rb, int64_t ldrb, int64_t bw,
                   Csr& out);
// out[j] = V[:, j]^T A V[:, j], j < m (no product buffer)
void csr_quadform(cudaStream_t st, const Csr& a, int64_t m, const double* V, int64_t ldv,
                  double* out);
void csr_spmv(cudaStream_t st, const Csr& a, double alpha, const double* x, double beta,
              double* y);
// band.cu: banded Cholesky (128-wide block columns, kb blocks below the diagonal)
struct BandChol {
  int64_t n = 0, ldp = 0, nblk = 0;
  int kb = 0;
  DBuf P, Dinv;
  double* panel(int64_t j) const { return P.p + j * ldp * 128; }
  int64_t rows_below(int64_t j) const {
    const int64_t r0 = (j + 1) * 128;
    return r0 >= n ? 0 : (n - r0 < (int64_t)kb * 128 ? n - r0 : (int64_t)kb * 128);
  }
};
int64_t band_lower_width(cudaStream_t st, int64_t n, const double* A, int64_t lda);
// (band_storage: A is LAPACK lower band storage of bandwidth bw, ld lda >= bw + 1)
int64_t band_potrf(cudaStream_t st, int64_t n, const double* A, int64_t lda, int64_t bw,
                   BandChol& f, bool band_storage = false);
__global__ void band_gershgorin_kernel(int64_t n, const double* __restrict__ B, int64_t ldb,
                                       int64_t bw, unsigned long long* out_lo,
                                       unsigned long long* out_hi, int* neg);
void band_solve(cudaStream_t st, const BandChol& f, bool trans, int64_t m, double* C,
                int64_t ldc);
void band_sygst(cudaStream_t st, const BandChol& f, double* B, int64_t ldb);
// C = A B through a device CSR copy of the symmetric A when nnz <= max_fill n^2
bool sym_sparse_mm(cudaStream_t st, int64_t n, const double* A, int64_t lda, int64_t m,
                   const double* B, int64_t ldb, double* C, int64_t ldc, double max_fill);

// symv.cu: y = alpha*A*x + beta*y using only the lower triangle of A (n x n)
void symv_lower(cudaStream_t st, int64_t n, double alpha, const double* A, int64_t lda,
                const double* x, double beta, double* y, double* work);
size_t symv_work_size(int64_t n);
// Tridiagonalisation column (sytrd.cu): x is the raw column; the symv CTAs run dlarfg
// themselves from the sum-of-squares partials and use v = [1, scale * x[1:]].
struct SymvLarfg {
  const double* part = nullptr;  // partials of ||x[1:]||^2
  int64_t nparts = 0;
  const double* alpha = nullptr;  // x[0]
  double* tau = nullptr;          // outputs, written by CTA 0
  double* e = nullptr;
  double* scale = nullptr;
  double* vav = nullptr;  // optional: per-CTA partials of v^T A v (symv_tma only)
};
// latrd panel products t = [W_p^T v | A_p^T v] (2 x 64) from per-CTA partials over rows
// >= c+2 of the raw column (times scale) plus row c+1 (v = 1 there).
struct LatrdT {
  int i = 0;  // panel columns so far (0: nothing to do)
  int64_t G = 0;
  const double* dpart = nullptr;  // [G][128]
  const double* wr1 = nullptr;    // W row c+1 (stride ldw)
  int64_t ldw = 0;
  const double* ar1 = nullptr;    // A row c+1 from column i0 (stride lda)
  int64_t lda = 0;
  const double* scale = nullptr;
  double* t = nullptr;  // [128]
};
void symv_lower_latrd(cudaStream_t st, int64_t n, const double* A, int64_t lda, const double* x,
                      double* y, double* work, const SymvLarfg& lf, const LatrdT& lt);
// symv_tma.cu: TMA-fed variant. A tensor map spans a whole (rows x cols, ld) matrix; the
// symv runs on the n x n block at coordinates (off, off). symv_map_make returns false
// when TMA cannot address the matrix (base not 16-byte aligned or ld odd).
struct alignas(64) SymvMap {
  unsigned char opaque[2][128];  // CUtensorMaps: box 128 rows (even offsets), 130 rows (odd)
};
bool symv_map_make(SymvMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld);
size_t symv_tma_work_size(int64_t n);
void symv_tma(cudaStream_t st, const SymvMap& m, int64_t off, int64_t n, double alpha,
              const double* x, double beta, double* y, double* work, const SymvLarfg* lf,
              const LatrdT* lt, bool pdl);
// number of CTAs (= quadratic-form partials written to SymvLarfg::vav) for order n
int64_t symv_tma_ctas(int64_t n);
// ... for the block at (off, off) (symv_tma aligns its tiles to 32-row boundaries)
int64_t symv_tma_ctas(int64_t n, int64_t off);

// sytrd.cu: Householder tridiagonalisation (lower). On exit d (n), e (n-1), tau (n-1);
// reflectors stored below the subdiagonal of A (LAPACK dsytrd convention).
void sytrd_lower(cudaStream_t st, int64_t n, double* A, int64_t lda, double* d, double* e,
                 double* tau);
// ormtr: Z <- Q Z with Q = H(0) ... H(n-2) from sytrd_lower (Z n x m)
void ormtr_lower(cudaStream_t st, int64_t n, int64_t m, const double* A, int64_t lda,
                 const double* tau, double* Z, int64_t ldz);
// Z <- H(0) ... H(nref-1) Z, reflector c's vector starts at row c + off of column c of A
// (trans: Z <- (H(0) ... H(nref-1))^T Z)
void ormqr_lower_off(cudaStream_t st, int64_t n, int64_t nref, int64_t off, int64_t m,
                     const double* A, int64_t lda, const double* tau, double* Z, int64_t ldz,
                     bool trans = false);

// sytrd2.cu: two-stage tridiagonalisation (dense -> band b -> tridiagonal) with the
// eigenvector back-transforms: syev_two_stage computes ascending w and Z for A (destroyed)
// (only columns [c0, c0 + nc) of the ascending eigenvector matrix are back-transformed:
// the column-sharded form of parallel.py; nc < 0 = all)
// Yt (optional, n x ky): the "implicit eigenvector" mode — Yt <- (Q U)^T Yt (Q the
// tridiagonalisation's orthogonal factor, U the tridiagonal eigenvectors), neither Q U nor
// U formed (Z unused, may be null); A's storage is reused for the stage-2 reflectors
void syev_two_stage(cudaStream_t st, int64_t n, double* A, int64_t lda, double* w, double* Z,
                    int64_t ldz, int64_t c0 = 0, int64_t nc = -1, double* Yt = nullptr,
                    int64_t ldy = 0, int64_t ky = 0);
// stage pieces (exposed for tests): A -> band AB (ldab = 2b+1, band rows 0..b filled)
void sy2sb(cudaStream_t st, int64_t n, double* A, int64_t lda, double* tau1, double* AB,
           int64_t ldab);
constexpr int kBand = 64;

// stedc.cu: tridiagonal eigensolver (divide and conquer). Eigenvalues ascending in d,
// eigenvectors in Z (n x n, ld ldz). e is destroyed.
// c0, nc: only eigenvector columns [c0, c0 + nc) are needed (nc < 0: all); the others are
// left undefined (the root merge forms just that range)
void stedc(cudaStream_t st, int64_t n, double* d, double* e, double* Z, int64_t ldz,
           int64_t c0 = 0, int64_t nc = -1);
// Eigenvalues ascending in d and Y (n x k) <- U^T Y, U never formed (O(n k) memory)
void stedc_apply(cudaStream_t st, int64_t n, double* d, double* e, double* Y, int64_t ldy,
                 int64_t k);

// syev.cu: symmetric eigendecomposition, eigenvalues ASCENDING; A destroyed.
void syev_ascending(cudaStream_t st, int64_t n, double* A, int64_t lda, double* w, double* Z,
                    int64_t ldz, int64_t c0 = 0, int64_t nc = -1, double* Yt = nullptr,
                    int64_t ldy = 0, int64_t ky = 0);

// td1.cu / td2.cu
void td2_plan_init(em_td2_plan* P, const double* l_n, const double* r_n, const double* P_r,
                   const double* P_l, const double* P_m);
void td2_plan_init_exact(em_td2_plan* P, const double* l_n, const double* r_n, const double* P_r,
                         const double* P_l, const double* P_m);
bool td2_is_exact(const em_td2_plan* P);
void td2_set_observables(em_td2_plan* P, int n_obs, const double* CV, int64_t ldcv,
                         const double* D, int64_t ldd);
void td2_run(em_td2_plan* P, int64_t T, const double* drive, double* q, double* Y,
             int64_t stride, double* Qcap);
void td2_step(em_td2_plan* P, double* q, const double* u_dev);
void td2_run_sweep(em_td2_plan* P, int64_t T, const double* drive, double* Q, double* Y,
                   int64_t stride);

int64_t td1_plan_init(em_td1_plan* P, const double* L, int64_t ldl, const double* R, int64_t ldr,
                      const double* r_d, const double* l_d, const double* m0,
                      const double* Rb = nullptr, int64_t ldrb = 0, int64_t bw = 0,
                      bool in_place = false);
void td1_set_observables(em_td1_plan* P, int n_obs, const double* C, int64_t ldc,
                         const double* D, int64_t ldd);
void td1_run(em_td1_plan* P, int64_t T, const double* drive, double* I, double* Y,
             int64_t stride, double* Icap);
void td1_step(em_td1_plan* P, double* I, const double* u_dev);

// q2reg.cu: Z <- Q2 Z (stage-2 reflectors V2 with task offsets toff, T factors T2)
void q2_apply_reg(cudaStream_t st, int64_t n, int64_t ncols, int64_t ngroups, const double* V2,
                  const int64_t* toff, const double* T2, double* Z, int64_t ldz);

// observers.cu: Biot-Savart probe transfer T (np x 3 x nb) of straight branch segments
// A -> B (nb x 3 row-major); returns -1 or the first probe-on-branch pair p*nb + j
int64_t field_transfer(cudaStream_t st, int64_t nb, const double* A, const double* B,
                       const double* radius, int64_t np, const double* P, double* T);

}  // namespace em
