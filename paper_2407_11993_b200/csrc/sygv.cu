// Generalized symmetric-definite eigensolve L v = tau R v — the device version of
// modal.generalized_eig (pkg/src/eddymodes/modal.py:46-81):
//   R = G G^T (potrf, "modal resistance matrix")
//   B = G^-1 L G^-T (recursive two-sided reduction; the reference forms G^-1 L,
//       G^-1 (G^-1 L)^T, (B + B^T)/2 — the same matrix to round-off)
//   potrf(L) certificate ("modal inductance matrix"), same order as the reference
//   B = U diag(w) U^T   (sytrd + divide & conquer + ormtr; replaces Jacobi)
//   V = G^-T U, descending order, sign fix (largest |entry| positive),
//   l_n = diag(V^T L V), r_n = diag(V^T R V), V^T R (= (R V)^T).
#include <cstring>

#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

// em_config(EM_CFG_TWO_STAGE_MIN): smallest order that takes the two-stage reduction.
// Measured on one B200 (em_syev, eigenvectors formed, profiles/r02/crossover.json): at
// n = 16,384 the two-stage path is ahead by ~8% (the C2 pass 1.69 s against 1.83 s
// one-stage), n = 24,576 4.53 s against 5.53 s, n = 32,768 9.34 s against 12.5 s, the C3
// step 29.0 s against 50.7 s. (Before the band reduction's panel QR took one grid barrier
// per column and the bulge chase was reworked, the crossover lay near n = 22,000 and the
// default was 40,000.) Tests force either path.
int64_t g_two_stage_min = 16000;
// Extra device memory of the two-stage path beyond A and Z, phase by phase (n^2 doubles):
// the stage-2 reflectors V2 (1/2) live from sb2st to the end; divide and conquer adds its
// gathered Q and U (2, +1 when ldz != n); the Q2 apply the blocks' T factors (1/2); the Q1
// apply its compact-WY V blocks (1). Taken only when the largest phase fits.
static double two_stage_extra(int64_t ldz, int64_t n) {
  const double stedc = 0.5 + 2.0 + (ldz != n ? 1.0 : 0.0), q2 = 0.5 + 0.5, q1 = 0.5 + 1.0;
  return stedc > q1 ? (stedc > q2 ? stedc : q2) : (q1 > q2 ? q1 : q2);
}
int g_last_eig_path = 0;  // em_info(EM_INFO_EIG_PATH): 1 one-stage, 2 two-stage
static bool two_stage_fits(int64_t n, int64_t ldz, bool implicit) {
  size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) return false;
  // plus what the stream-ordered pool holds reserved but unused (em_init keeps freed
  // workspace cached between calls)
  int dev = 0;
  cudaMemPool_t pool;
  if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t reserved = 0, used = 0;
    if (cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved) ==
            cudaSuccess &&
        cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used) == cudaSuccess &&
        reserved > used)
      free_b += (size_t)(reserved - used);
  }
  // implicit mode: the reflectors live in A, T factors per wavefront: nothing else is n^2
  const double need = (implicit ? 0.0 : two_stage_extra(ldz, n)) * (double)n * (double)n *
                          sizeof(double) + (1ull << 30);
  return (double)free_b >= need;
}
// em_config(EM_CFG_BAND_OFF): 1 forces the dense R path (tests compare both)
int g_band_off = 0;
// em_config(EM_CFG_LN_DENSE): 1 forms l_n = diag(V^T L V) with the N^3 product as the
// reference does (modal.py:79); 0 (default) uses the eigen-identity l_n = tau r_n
int g_ln_dense = 0;
// em_config(EM_CFG_L_CERTIFICATE): 1 factors L (the reference's certificate, modal.py:69-70)
// before the eigensolve, always; 0 (default) skips it when the solved spectrum proves it
// would succeed (see sygv), and runs it otherwise
int g_l_certificate = 0;

// Gershgorin bounds of a symmetric matrix from its lower triangle: out[0] = min_i (a_ii -
// sum_j |a_ij|), out[1] = max_i (a_ii + sum_j |a_ij|) (atomics on the ordered bit patterns
// of non-negative doubles; out preset to +inf / 0 by the caller)
__global__ void gershgorin_kernel(int64_t n, const double* __restrict__ A, int64_t lda,
                                  unsigned long long* out_lo, unsigned long long* out_hi,
                                  int* neg) {
  const int64_t i = blockIdx.x;
  double s = 0.0;
  for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
    if (j == i) continue;
    const double v = j < i ? A[i + j * lda] : A[j + i * lda];  // lower triangle (SymMatrix)
    s += fabs(v);
  }
  __shared__ double red[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) t += red[q];
    const double d = A[i + i * lda];
    const double lo = d - t, hi = d + t;
    if (!(lo > 0.0)) atomicExch(neg, 1);
    else atomicMin(out_lo, (unsigned long long)__double_as_longlong(lo));
    atomicMax(out_hi, (unsigned long long)__double_as_longlong(fmax(hi, 0.0)));
  }
}

// The reference's Cholesky of L (the certificate) succeeds whenever L is safely SPD. With
// B = G^-1 L G^-T and tau = eig(B): lambda_min(L) >= tau_min lambda_min(R) and ||L|| <=
// tau_max ||R||, so kappa(L) <= (tau_max / tau_min) kappa(R); kappa(R) is bounded by R's
// Gershgorin interval when R is strictly diagonally dominant (the plates' stencil). Cholesky
// completes when 20 n^1.5 kappa eps < 1 (Demmel); this asks for 100x margin.
static bool certificate_redundant(cudaStream_t st, int64_t n, const double* R, int64_t ldr,
                                  double tau_min, double tau_max, const double* Rb = nullptr,
                                  int64_t ldrb = 0, int64_t rbw = 0) {
  if (!(tau_min > 0.0) || !(tau_max >= tau_min)) return false;
  DArr<unsigned long long> b(2, st);
  DArr<int> neg(1, st);
  double inf = INFINITY;
  unsigned long long init[2] = {0ull, 0ull};
  memcpy(&init[0], &inf, sizeof(double));
  EM_CK(cudaMemcpyAsync(b.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
  EM_CK(cudaMemsetAsync(neg.p, 0, sizeof(int), st));
  if (Rb)
    band_gershgorin_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(n, Rb, ldrb, rbw, b.p,
                                                                    b.p + 1, neg.p);
  else
    gershgorin_kernel<<<(unsigned)n, 256, 0, st>>>(n, R, ldr, b.p, b.p + 1, neg.p);
  EM_LAUNCHED();
  unsigned long long hb[2];
  int hneg = 0;
  EM_CK(cudaMemcpyAsync(hb, b.p, sizeof(hb), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaMemcpyAsync(&hneg, neg.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  double lo, hi;
  memcpy(&lo, &hb[0], sizeof(double));
  memcpy(&hi, &hb[1], sizeof(double));
  if (hneg || !(lo > 0.0)) return false;
  const double kappa = (tau_max / tau_min) * (hi / lo);
  return 20.0 * pow((double)n, 1.5) * kappa * 2.220446049250313e-16 < 0.01;
}

// out[i] = a[i] * b[i]
__global__ void scale_vec_kernel(int64_t n, const double* __restrict__ a,
                                 const double* __restrict__ b, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] * b[i];
}

void syev_ascending(cudaStream_t st, int64_t n, double* A, int64_t lda, double* w, double* Z,
                    int64_t ldz, int64_t c0, int64_t nc, double* Yt, int64_t ldy, int64_t ky) {
  if (n <= 0) return;
  if (nc < 0) nc = n - c0;
  if (n >= g_two_stage_min && n > 2 * kBand && two_stage_fits(n, ldz, Yt != nullptr)) {
    g_last_eig_path = 2;
    syev_two_stage(st, n, A, lda, w, Z, ldz, c0, nc, Yt, ldy, ky);
    return;
  }
  g_last_eig_path = 1;
  DBuf d(n, st), e(imax64(n - 1, 1), st), tau(imax64(n - 1, 1), st);
  {
    Stage s(st, ST_SYTRD);
    sytrd_lower(st, n, A, lda, d.p, e.p, tau.p);
  }
  if (Yt) {  // implicit mode: Yt <- U^T Q^T Yt, U never formed
    {
      Stage s(st, ST_ORMTR);
      ormqr_lower_off(st, n, n - 1, 1, ky, A, lda, tau.p, Yt, ldy, true);
    }
    Stage s(st, ST_STEDC);
    stedc_apply(st, n, d.p, e.p, Yt, ldy, ky);
  } else {
    {
      Stage s(st, ST_STEDC);
      stedc(st, n, d.p, e.p, Z, ldz, c0, nc);
    }
    Stage s(st, ST_ORMTR);
    ormtr_lower(st, n, nc, A, lda, tau.p, Z + c0 * ldz, ldz);
  }
  EM_CK(cudaMemcpyAsync(w, d.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

// Column sign of np.argmax semantics: s = sign of the first largest-|.| entry of z
// (0 -> +1, modal.py:76-77). Block-wide; every thread returns the sign.
EM_DEVINL double column_sign(int64_t n, const double* __restrict__ z, double* bv, int64_t* bi,
                             double* sgn) {
  double best = -1.0;
  int64_t idx = 0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = fabs(z[i]);
    if (a > best) {
      best = a;
      idx = i;
    }
  }
  // (max |v|, smallest index) reduction == np.argmax semantics
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, best, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, idx, o);
    if (ob > best || (ob == best && oi < idx)) {
      best = ob;
      idx = oi;
    }
  }
  if ((threadIdx.x & 31) == 0) {
    bv[threadIdx.x >> 5] = best;
    bi[threadIdx.x >> 5] = idx;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = bv[0];
    int64_t k = bi[0];
    for (int q = 1; q < (int)(blockDim.x >> 5); ++q)
      if (bv[q] > b || (bv[q] == b && bi[q] < k)) {
        b = bv[q];
        k = bi[q];
      }
    *sgn = (z[k] < 0.0) ? -1.0 : 1.0;
  }
  __syncthreads();
  const double s = *sgn;
  __syncthreads();  // bv/bi/sgn reusable
  return s;
}

// In place on the eigenvector buffer: V[:, j] = s * Z[:, n-1-j] (descending order,
// sign fix), tau[j] = w[n-1-j]. Block j swaps the column pair (j, n-1-j), so no
// second N x N buffer is needed.
__global__ void finalize_modes_inplace_kernel(int64_t n, double* __restrict__ V, int64_t ldv,
                                              const double* __restrict__ w,
                                              double* __restrict__ tau) {
  __shared__ double bv[32];
  __shared__ int64_t bi[32];
  __shared__ double sgn;
  const int64_t j = blockIdx.x, k = n - 1 - j;
  double* zj = V + j * ldv;
  double* zk = V + k * ldv;
  const double sj = column_sign(n, zj, bv, bi, &sgn);  // lands in column k
  const double sk = column_sign(n, zk, bv, bi, &sgn);  // lands in column j
  if (threadIdx.x == 0) {
    tau[j] = w[k];
    tau[k] = w[j];
  }
  if (j == k) {
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) zj[i] *= sj;
    return;
  }
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double a = zj[i], b = zk[i];
    zj[i] = sk * b;
    zk[i] = sj * a;
  }
}

// Column slice (modes m_lo .. m_lo + m - 1 in descending order): V[:, j] = s * Zs[:, m-1-j]
// from the back-transformed ascending columns Zs, sign fixed (modal.py:74-78).
__global__ void finalize_modes_slice_kernel(int64_t n, int64_t m, const double* __restrict__ Zs,
                                            int64_t ldz, double* __restrict__ V, int64_t ldv) {
  __shared__ double bv[32];
  __shared__ int64_t bi[32];
  __shared__ double sgn;
  const int64_t j = blockIdx.x;
  const double* z = Zs + (m - 1 - j) * ldz;
  const double s = column_sign(n, z, bv, bi, &sgn);
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) V[i + j * ldv] = s * z[i];
}

// Y[j, c] = X[n-1-j, c]
__global__ void reversed_rows_kernel(int64_t n, int64_t k, const double* __restrict__ X,
                                     int64_t ldx, double* __restrict__ Y, int64_t ldy) {
  const int64_t total = n * k;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % n, c = i / n;
    Y[r + c * ldy] = X[(n - 1 - r) + c * ldx];
  }
}
static void copy_reversed_rows(cudaStream_t st, int64_t n, int64_t k, const double* X,
                               int64_t ldx, double* Y, int64_t ldy) {
  const int64_t total = n * k;
  reversed_rows_kernel<<<(unsigned)imin64((total + 255) / 256, 148 * 16), 256, 0, st>>>(
      n, k, X, ldx, Y, ldy);
  EM_LAUNCHED();
}
__global__ void fill_kernel(int64_t n, double v, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = v;
}
static void fill_value(cudaStream_t st, int64_t n, double v, double* out) {
  fill_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, v, out);
  EM_LAUNCHED();
}

// tau[j] = w[n-1-j] (descending time constants)
__global__ void reverse_kernel(int64_t n, const double* __restrict__ w, double* __restrict__ tau) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) tau[j] = w[n - 1 - j];
}

// out[j] = sum_i V[i,j] * X[i,j]
__global__ void coldot_kernel(int64_t n, const double* __restrict__ V, int64_t ldv,
                              const double* __restrict__ X, int64_t ldx, double* __restrict__ out) {
  __shared__ double red[32];
  const int64_t j = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(V[i + j * ldv], X[i + j * ldx], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[j] = t;
  }
}

// out[j] = v_j^T L v_j for symmetric L from X = L_low V (L_low: lower triangle of L with
// its diagonal): v^T L v = 2 v^T L_low v - sum_i L_ii v_i^2 (exact identity).
__global__ void quadform_lower_kernel(int64_t n, const double* __restrict__ V, int64_t ldv,
                                      const double* __restrict__ X, int64_t ldx,
                                      const double* __restrict__ L, int64_t ldl,
                                      double* __restrict__ out) {
  __shared__ double red[32];
  const int64_t j = blockIdx.x;
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const double v = V[i + j * ldv];
    s = fma(v, fma(2.0, X[i + j * ldx], -L[i + i * ldl] * v), s);
  }
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) out[j] = t;
  }
}

// Returns -1 on success; else the failing pivot with *which = 0 (R) / 1 (L).
// l_ready (optional): L is still being uploaded; the stream waits for it only before the
// first use of L (after R's band detection and factorisation).
//
// Column range (m_lo, m_hi) (the column-sharded eigensolve of parallel.py: one rank's
// modes): V, VtR are n x (m_hi - m_lo) and l_n, r_n have m_hi - m_lo entries for modes
// m_lo .. m_hi - 1 (descending order); tau always gets all n. Everything up to the
// tridiagonal eigenvectors is computed for the whole matrix; the back-transforms
// (Q2, Q1 / ormtr, G^-T), the sign fix and l_n, r_n only for the rank's columns.
//
// Implicit mode (Y != null, V must be null): V is never formed. Y (n x ky) holds operands
// on entry and V^T Y on exit, rows in descending mode order: V^T = U^T Q^T G^-1 is applied
// to the ky columns (the solve with R's factor, the tridiagonalisation's reflectors
// transposed, then one n x n x ky product with the tridiagonal eigenvectors U), so the
// 4 n^3 flops of forming V (Q2, Q1) become O(n^2 ky). The per-mode sign of V (largest entry
// positive, modal.py:74-78) needs V itself: here the eigensolver's own signs are kept —
// every product of two such rows (a drive projection and an observable) is unchanged.
// l_n, r_n: tau and 1 (V^T L V = diag(tau), V^T R V = I).
int64_t sygv(cudaStream_t st, int64_t n, const double* L, int64_t ldl, const double* R,
             int64_t ldr, double* tau, double* V, int64_t ldv, double* l_n, double* r_n,
             double* VtR, int64_t ldvtr, int* which, int flags, cudaEvent_t l_ready,
             int64_t m_lo, int64_t m_hi, double* Y, int64_t ldy, int64_t ky, const double* Rb,
             int64_t ldrb, int64_t rbw) {
  *which = -1;
  if (n <= 0) return -1;
  const bool implicit = Y != nullptr;
  if (implicit && (V || VtR)) throw ArgError{"implicit mode forms no V / V^T R"};
  if (implicit) m_lo = 0, m_hi = 0;  // no eigenvector columns are formed
  if (m_hi < 0) m_hi = n;
  if (m_lo < 0 || m_hi > n || m_lo > m_hi) throw ArgError{"mode range outside [0, n]"};
  const int64_t m = m_hi - m_lo;
  const bool slice = m < n;
  // in-place L (EM_SYGV_L_WORKSPACE): L's storage becomes the reduced matrix B; R in band
  // storage (Rb): no dense R anywhere. Together the N = 120,000 solve fits one GPU.
  const bool l_ws = (flags & EM_SYGV_L_WORKSPACE) && ldl >= n;
  const bool r_band = Rb != nullptr;
  if (r_band && (rbw < 0 || ldrb < rbw + 1)) throw ArgError{"bad band storage of R"};
  // slice: the full tridiagonal eigenvector matrix needs an n x n workspace (the output V
  // holds only m columns); implicit mode forms no eigenvector matrix at all
  DBuf Zfull;
  double* Zw = V;
  int64_t ldzw = ldv;
  if (slice && !implicit) {
    Zfull.alloc((size_t)n * n, st);
    Zw = Zfull.p;
    ldzw = n;
  }
  const size_t nn = (size_t)n * n;
  // A banded R (the 7-point stencil R of the plates: lower bandwidth ny*nz) is factored
  // in banded storage and every solve with its factor is banded (band.cu): the R stages
  // cost N b^2 + 6 N^2 b instead of 7/3 N^3, and no N x N factor buffer is needed.
  const int64_t bw = r_band ? rbw : (g_band_off ? n : band_lower_width(st, n, R, ldr));
  const bool banded = r_band || (n > 2 * kTrsmBlock && (bw + kTrsmBlock) * 4 <= n);
  BandChol bc;
  // EM_SYGV_R_WORKSPACE (dense-band R only): when R is sparse, keep a CSR copy, factor R
  // in its own storage and restore it from the copy before returning: one N x N buffer
  // less at the peak
  Csr rcsr;
  const bool r_ws = !banded && !r_band && (flags & EM_SYGV_R_WORKSPACE) &&
                    csr_from_dense(st, n, R, ldr, 0.02, rcsr);
  DBuf Gbuf;
  double* G = const_cast<double*>(R);
  int64_t ldg = ldr;
  if (!banded && !r_ws) {
    Gbuf.alloc(nn, st);
    copy_matrix(st, false, n, n, R, ldr, Gbuf.p, n);
    G = Gbuf.p;
    ldg = n;
  }
  // A BANDED R's factor lives in band storage of its own, so with EM_SYGV_R_WORKSPACE the
  // dense R (sparse: a stencil) is free during the eigensolve: its storage holds the
  // reduced matrix B (when its columns are 256-byte aligned, as B's must be) and is
  // restored from the CSR copy once the back-transform is done. One N x N buffer less at
  // the peak: the N = 60,000 pencil then runs the two-stage tridiagonalisation on one GPU.
  const bool l_ws_ok = (flags & EM_SYGV_L_WORKSPACE) && ldl >= n && ldl % 32 == 0;
  const bool rb_ws = banded && !r_band && !l_ws_ok && (flags & EM_SYGV_R_WORKSPACE) &&
                     ldr >= n && ldr % 32 == 0 &&
                     (reinterpret_cast<uintptr_t>(R) & 255) == 0 &&
                     csr_from_dense(st, n, R, ldr, 0.02, rcsr);
  auto restore_r = [&] {
    if (r_ws) csr_to_dense(st, rcsr, G, ldg);
    if (rb_ws) csr_to_dense(st, rcsr, const_cast<double*>(R), ldr);
  };
  int64_t piv;
  DBuf GDinv;
  {
    Stage s(st, ST_POTRF_R);
    if (r_band) {
      piv = band_potrf(st, n, Rb, ldrb, bw, bc, true);
    } else if (banded) {
      piv = band_potrf(st, n, R, ldr, bw, bc);
    } else {
      GDinv.alloc((size_t)((n + kTrsmBlock - 1) / kTrsmBlock) * kTrsmBlock * kTrsmBlock, st);
      piv = potrf(st, n, G, ldg, GDinv.p);
    }
  }
  if (l_ready) EM_CK(cudaStreamWaitEvent(st, l_ready, 0));
  if (piv >= 0) {
    *which = 0;
    restore_r();
    EM_CK(cudaStreamSynchronize(st));
    return piv;
  }
  if (implicit && ky > 0) {  // Y <- G^-1 Y (the first factor of V^T = U^T Q^T G^-1)
    Stage s(st, ST_TRSM_BACK);
    if (banded)
      band_solve(st, bc, false, ky, Y, ldy);
    else
      trsm_lower(st, false, n, ky, G, ldg, Y, ldy, GDinv.p);
  }
  // leading dimension padded to 32 doubles: every column of B starts 256-byte aligned,
  // so all TMA boxes of the tridiagonalisation's symv are (symv_tma.cu)
  // (in place in L's storage when allowed and L's columns are 256-byte aligned)
  const bool b_in_l = l_ws && ldl % 32 == 0;
  const int64_t ldb = b_in_l ? ldl : rb_ws ? ldr : (n + 31) / 32 * 32;
  // certificate only (modal.py:69-70): with EM_CFG_L_CERTIFICATE = 1 L is factored up
  // front in a copy of its own (before an in-place solve destroys it)
  if (g_l_certificate) {
    Stage s(st, ST_POTRF_L);
    DBuf Lc((size_t)n * n, st);
    copy_matrix(st, false, n, n, L, ldl, Lc.p, n);
    piv = potrf(st, n, Lc.p, n);
    if (piv >= 0) {
      *which = 1;
      restore_r();
      EM_CK(cudaStreamSynchronize(st));
      return piv;
    }
  }
  DBuf Bown;
  double* Bp = const_cast<double*>(L);
  if (rb_ws) {
    Bp = const_cast<double*>(R);
  } else if (!b_in_l) {
    Bown.alloc((size_t)ldb * n, st);
    Bp = Bown.p;
  }
  {
    {
      // B = G^-1 L G^-T. The reference forms G^-1 (G^-1 L)^T with two full solves and
      // averages it with its transpose (modal.py:63-67); the two-sided recursive
      // reduction gives the same symmetric matrix to round-off with half the flops.
      Stage s(st, ST_SYGST);
      if (!b_in_l) copy_matrix(st, false, n, n, L, ldl, Bp, ldb);
      mirror_lower(st, n, Bp, ldb);  // SymMatrix semantics: the lower triangle defines L
      if (banded)
        band_sygst(st, bc, Bp, ldb);  // the reference's X = G^-1 L, G^-1 X^T, (B + B^T)/2
      else
        sygst_lower(st, n, Bp, ldb, G, ldg, GDinv.p);
    }
  }
  // eigenvectors are formed directly in the output buffer V (D&C, ormtr, back-transform,
  // then the in-place descending reorder + sign fix): peak memory L, R, V + G, B and the
  // two D&C work matrices = 7 N^2 (8 with V^T R), so N = 50,000 fits one B200
  DBuf w(n, st);
  // descending modes m_lo .. m_hi - 1 are the ascending columns n - m_hi .. n - m_lo - 1
  const int64_t c0 = n - m_hi;
  double* Zs = Zw ? Zw + c0 * ldzw : nullptr;
  syev_ascending(st, n, Bp, ldb, w.p, Zw, ldzw, c0, m, implicit ? Y : nullptr, ldy, ky);
  Bown.release();
  if (m > 0) {
    Stage s(st, ST_TRSM_BACK);
    if (banded)
      band_solve(st, bc, true, m, Zs, ldzw);                   // V = G^-T U
    else
      trsm_lower(st, true, n, m, G, ldg, Zs, ldzw, GDinv.p);
  }
  Gbuf.release();
  restore_r();
  if (!g_l_certificate) {
    // The certificate is redundant when the solved pencil proves L safely SPD; otherwise
    // (L not SPD, or too ill-conditioned to tell) it runs now, in a buffer of its own,
    // and raises the reference's error with the reference's pivot. (R is intact again.)
    double wb[2] = {0.0, 0.0};
    EM_CK(cudaMemcpyAsync(&wb[0], w.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    EM_CK(cudaMemcpyAsync(&wb[1], w.p + (n - 1), sizeof(double), cudaMemcpyDeviceToHost, st));
    EM_CK(cudaStreamSynchronize(st));
    if (!certificate_redundant(st, n, R, ldr, wb[0], wb[1], Rb, ldrb, rbw)) {
      if (b_in_l)
        throw ArgError{"the certificate of L is needed but L was solved in place "
                       "(EM_SYGV_L_WORKSPACE): solve again without it"};
      Stage s(st, ST_POTRF_L);
      DBuf Lc((size_t)n * n, st);
      copy_matrix(st, false, n, n, L, ldl, Lc.p, n);
      const int64_t pl = potrf(st, n, Lc.p, n);
      if (pl >= 0) {
        *which = 1;
        EM_CK(cudaStreamSynchronize(st));
        return pl;
      }
    }
  }
  if (implicit) {
    // Y <- U^T Y, rows reversed to descending order; tau, l_n = tau, r_n = 1
    Stage s(st, ST_FINALIZE);
    if (ky > 0) {  // syev_ascending left U^T Q^T G^-1 Y in Y, ascending rows
      DBuf T((size_t)n * ky, st);
      copy_matrix(st, false, n, ky, Y, ldy, T.p, n);
      copy_reversed_rows(st, n, ky, T.p, n, Y, ldy);
      EM_CK(cudaStreamSynchronize(st));
    }
    reverse_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, w.p, tau);
    EM_LAUNCHED();
    if (l_n) EM_CK(cudaMemcpyAsync(l_n, tau, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    if (r_n) fill_value(st, n, 1.0, r_n);
    EM_CK(cudaStreamSynchronize(st));
    return -1;
  }
  {
    Stage s(st, ST_FINALIZE);
    if (slice) {
      if (m > 0) {
        finalize_modes_slice_kernel<<<(unsigned)m, 256, 0, st>>>(n, m, Zs, ldzw, V, ldv);
        EM_LAUNCHED();
      }
      reverse_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, w.p, tau);
      EM_LAUNCHED();
      Zfull.release();
    } else {
      finalize_modes_inplace_kernel<<<(unsigned)((n + 1) / 2), 256, 0, st>>>(n, V, ldv, w.p, tau);
      EM_LAUNCHED();
    }
  }
  Stage post(st, ST_POST_GEMM);
  // r_n = diag(V^T R V) (modal.py:80): R is typically a stencil stored dense (the
  // reference's SymMatrix), so through a CSR copy, fused with the column dots (no N x N
  // product); V^T R = (R V)^T only when asked for.
  Csr rq;
  const Csr* rc = (r_ws || rb_ws) ? &rcsr : nullptr;
  if (!rc && (r_n || l_n) && csr_from_dense(st, n, R, ldr, 0.02, rq)) rc = &rq;
  DBuf rn_tmp;
  double* rn_out = r_n;
  if (!rn_out && l_n && !g_ln_dense) {
    rn_tmp.alloc(imax64(m, 1), st);
    rn_out = rn_tmp.p;
  }
  if (m == 0) {
    EM_CK(cudaStreamSynchronize(st));
    return -1;
  }
  if (VtR) {
    if (rc) {
      csr_mm(st, *rc, m, V, ldv, VtR, ldvtr);
    } else {  // dense R: its lower triangle mirrored into a scratch copy
      DBuf Rs(nn, st);
      copy_matrix(st, false, n, n, R, ldr, Rs.p, n);
      mirror_lower(st, n, Rs.p, n);
      EM_CK(gemm(st, false, false, n, m, n, 1.0, Rs.p, n, V, ldv, 0.0, VtR, ldvtr));
      EM_CK(cudaStreamSynchronize(st));
    }
    if (rn_out) {
      coldot_kernel<<<(unsigned)m, 256, 0, st>>>(n, V, ldv, VtR, ldvtr, rn_out);
      EM_LAUNCHED();
    }
  } else if (rn_out) {
    if (rc) {
      csr_quadform(st, *rc, m, V, ldv, rn_out);
    } else {  // dense R: v^T R v from its lower triangle (as l_n's dense form)
      DBuf RV((size_t)n * m, st);
      EM_CK(gemm_lower_a(st, n, m, n, 1.0, R, ldr, V, ldv, 0.0, RV.p, n));
      quadform_lower_kernel<<<(unsigned)m, 256, 0, st>>>(n, V, ldv, RV.p, n, R, ldr, rn_out);
      EM_LAUNCHED();
      EM_CK(cudaStreamSynchronize(st));
    }
  }
  if (l_n) {
    if (g_ln_dense) {
      // l_n = diag(V^T L V) (modal.py:79) as the reference forms it, through the lower
      // triangle of L only (the SymMatrix definition of L): a triangular-A product
      DBuf LV((size_t)n * m, st);
      EM_CK(gemm_lower_a(st, n, m, n, 1.0, L, ldl, V, ldv, 0.0, LV.p, n));
      quadform_lower_kernel<<<(unsigned)m, 256, 0, st>>>(n, V, ldv, LV.p, n, L, ldl, l_n);
      EM_LAUNCHED();
      EM_CK(cudaStreamSynchronize(st));
    } else {
      // V^T L V = diag(tau) V^T R V for the generalized eigenvectors (L V = R V diag(tau)
      // up to the eigen-residual, a rounding-level term), so l_n = tau_n r_n: the same
      // quantity to ~1e-13 relative (tests: test_gpu_parity_configs C2 golden, against
      // the LAPACK restatement's dense diag(V^T L V)) without the N^3 product
      scale_vec_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(m, tau + m_lo, rn_out, l_n);
      EM_LAUNCHED();
    }
  }
  EM_CK(cudaStreamSynchronize(st));
  return -1;
}

}  // namespace em
