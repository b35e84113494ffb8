/*
 * eddymodes_b200 — C ABI of the B200-native modal-transient hot path.
 *
 * libeddymodes_b200.so replaces the compiled numerics of the reference package
 * `eddymodes` (pkg/src/eddymodes/_kernels.py, numba @njit) and the numpy/BLAS
 * contractions around them (modal.py, transient.py). The Python mirror
 * (paper_2407_11993_b200/) binds these entry points through ctypes; the
 * binding a maintainer would add to the reference is in INTEGRATION.md.
 *
 * Conventions
 *  - Matrices are FP64, column-major with an explicit leading dimension.
 *    A C-contiguous (row-major) numpy array of a SYMMETRIC matrix is the same
 *    bytes, so symmetric inputs pass straight through.
 *  - Pointers are DEVICE pointers unless the name ends in _h (host).
 *  - Every call is ordered on the context's stream; calls returning data to
 *    the host (or a status that depends on device results) synchronise it.
 *  - Return codes: EM_OK (0) on success, EM_ERR_* < 0 otherwise; the message
 *    is available from em_last_error(). Numerical status that the reference
 *    reports through return values (Cholesky pivot, Jacobi non-convergence)
 *    comes back in out-parameters with the reference's encoding:
 *    pivot = -1 success, >= 0 the first failing pivot (_kernels.py:18-36).
 */
#ifndef EDDYMODES_B200_H
#define EDDYMODES_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EM_OK 0
#define EM_ERR_CUDA -1
#define EM_ERR_ARG -2
#define EM_ERR_NOT_PD -3        /* pivot out-param says which */
#define EM_ERR_NO_CONVERGENCE -4
#define EM_ERR_ALLOC -5

typedef struct em_ctx em_ctx;
typedef struct em_td2_plan em_td2_plan;
typedef struct em_td1_plan em_td1_plan;
typedef struct em_fd_plan em_fd_plan;

/* --- context --------------------------------------------------------------- */
/* em_init keeps memory freed by the library cached in the device's default pool
 * (stream-ordered allocator) between calls; em_trim releases it, em_finalize releases it
 * and restores the pool's previous release threshold. */
int em_init(int device, em_ctx** ctx);

/* ---- multi-GPU: one process (and one context) per GPU --------------------------------
 * The reference's distributed run is ScaLAPACK PDSYGVX over MPI ranks;
 * here every rank calls the same em_* entry points and the library exchanges data with
 * NCCL on the context stream (panel broadcasts and partial-product all-reduces of the
 * band reduction, em_sygv_range with EM_SYGV_DIST). Rank 0 obtains an id
 * (em_comm_unique_id, EM_COMM_ID_BYTES bytes), the host application hands it to the other
 * ranks (e.g. torch.distributed broadcast), every rank calls em_comm_init_nccl.
 * em_comm_init_callbacks installs host-supplied collectives instead (tests: several
 * ranks on one GPU, which NCCL refuses); the library synchronises the stream, then calls
 * them with DEVICE pointers. Collectives are issued in the same order on every rank. */
#define EM_COMM_ID_BYTES 128
typedef int (*em_allreduce_fn)(void* user, double* device_buf, int64_t count);
typedef int (*em_bcast_fn)(void* user, double* device_buf, int64_t count, int root);
int em_comm_unique_id(em_ctx* ctx, void* id);
int em_comm_init_nccl(em_ctx* ctx, int nranks, int rank, const void* id);
int em_comm_init_callbacks(em_ctx* ctx, int nranks, int rank, em_allreduce_fn allreduce,
                           em_bcast_fn bcast, void* user);
/* info[0..5] = nranks, rank, backend (0 none, 1 NCCL, 2 callbacks), all-reduces issued,
 * broadcasts issued, bytes moved through them */
int em_comm_info(em_ctx* ctx, int64_t* info);
int em_comm_destroy(em_ctx* ctx);
void em_finalize(em_ctx* ctx);
int em_trim(em_ctx* ctx);
/* Facts about the last call: EM_INFO_EIG_PATH = 1 one-stage (Householder sytrd), 2
 * two-stage (band reduction + bulge chasing) tridiagonalisation in the last eigensolve. */
#define EM_INFO_EIG_PATH 1
int em_info(em_ctx* ctx, int key, int64_t* value);
/* Order all work on an external CUDA stream (e.g. torch.cuda.current_stream());
 * NULL means the legacy default stream. em_init creates a private stream. */
int em_set_stream(em_ctx* ctx, void* cuda_stream);
const char* em_last_error(const em_ctx* ctx);
/* Number of kernels this library has launched on ctx (for launch accounting). */
int64_t em_launch_count(const em_ctx* ctx);
int em_synchronize(em_ctx* ctx);
/* Tuning knobs. EM_CFG_TWO_STAGE_MIN: smallest n that uses the two-stage
 * (dense -> band -> tridiagonal) reduction in em_syev/em_sygv when its extra storage
 * (2.5 n^2 doubles beyond the matrix and the eigenvectors at its divide-and-conquer peak,
 * 3.5 when ldz != n) is free on the device (default 16000; below it one-stage
 * Householder). em_info(EM_INFO_EIG_PATH) reports which path ran. */
#define EM_CFG_TWO_STAGE_MIN 1
/* EM_CFG_BAND_OFF: 1 = always factor R densely (default 0: a banded R, lower bandwidth
 * b with 4 (b + 128) <= n, takes the banded Cholesky and banded solves). */
#define EM_CFG_BAND_OFF 2
/* EM_CFG_SYMV_L2_KEEP_MB: megabytes of the bottom-right block of a tridiagonalised
 * matrix that the per-column symv loads with the L2 evict_last policy (re-read from the
 * 126 MB L2 by every later column instead of HBM); every other tile is loaded
 * evict_first. Default 32; 0 = evict_first everywhere; < 0 = no cache hint. */
#define EM_CFG_SYMV_L2_KEEP_MB 3
/* EM_CFG_LN_DENSE: 1 = em_sygv forms l_n = diag(V^T L V) with the N^3 product as the
 * reference does (modal.py:79); 0 (default) = l_n = tau_n r_n, the generalized
 * eigen-identity V^T L V = diag(tau) V^T R V (equal to ~1e-13 relative; r_n is always
 * diag(V^T R V) from R itself). */
#define EM_CFG_LN_DENSE 4
/* EM_CFG_L_CERTIFICATE: 1 = em_sygv factors L before the eigensolve, as the reference's
 * certificate does (modal.py:69-70); 0 (default) = the factorisation runs after the
 * eigensolve only when the solved spectrum cannot prove it succeeds (tau_min > 0, R
 * strictly diagonally dominant and 20 n^1.5 kappa(L) eps < 0.01 with kappa(L) <=
 * (tau_max/tau_min) kappa(R)): a non-SPD L raises the same error with the same pivot,
 * after the eigensolve instead of before it. */
#define EM_CFG_L_CERTIFICATE 5
/* Keys 93-99 are debug switches for A/B measurements and the tests (93 TD1 solves: 0
 * register tiles, 1 TMA-staged tiles; 94 Q2 kernel switches; 95 TMA-fed GEMM: 0 off, 1 auto, 2 / 4 / 5 force a tile configuration; 96
 * cp.async GEMM tile configuration; 97 Q2 back-transform form; 98 tridiagonalisation code
 * paths; 99 trim the device memory pool to `value` bytes); see capi.cu. */
int em_config(em_ctx* ctx, int key, int64_t value);
/* Stage timers (CUDA events on the context stream). em_profile(ctx, 1) clears and
 * enables them; em_stage_times fills per-stage milliseconds / event-pair counts
 * (stage ids: potrf_R, sygst, potrf_L, sytrd, stedc, ormtr, trsm_back, finalize,
 * post_gemm, td2_local, td2_carry, td2_replay, td1_symv, td1_fwd, td1_bwd,
 * sytrd_symv, sytrd_syr2k, stedc_gemm, stedc_secular) and returns the stage count. */
int em_profile(em_ctx* ctx, int enable);
int em_stage_times(em_ctx* ctx, double* ms, int64_t* counts, int n);

/* --- dense building blocks --------------------------------------------------- */

/* C = alpha*op(A)*op(B) + beta*C (DMMA). Replaces the numpy GEMMs of
 * modal.py:79-81,90,98 and transient.py:140-154. trans_*: 0 = N, 1 = T. */
int em_dgemm(em_ctx* ctx, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
             double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
             double beta, double* C, int64_t ldc);

/* em_dgemm computing and writing only the entries (r, c) of C with r + diag_off >= c (the
 * triangular-output products of the Cholesky trailing updates and the syr2k-style
 * updates of the tridiagonalisation, _kernels.py:18-36 / linalg.py:119-134 on the
 * reference side); entries above that diagonal are left untouched. */
int em_dgemm_lower(em_ctx* ctx, int trans_a, int trans_b, int64_t m, int64_t n, int64_t k,
                   double alpha, const double* A, int64_t lda, const double* B, int64_t ldb,
                   double beta, double* C, int64_t ldc, int64_t diag_off);

/* C (m x n) = A B for a symmetric m x m A of which only the lower triangle and the 127
 * diagonals above it are read (those must hold the mirrored values): the product
 * X = A22 (V T) of the blocked band reduction behind sym_eig (linalg.py:119-134), one
 * TMA-fed kernel in which every row tile runs over the whole k range. A must be 16-byte
 * aligned with even lda and ldb (else EM_ERR_ARG). */
int em_dsymm_band_lower(em_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                        const double* B, int64_t ldb, double* C, int64_t ldc);

/* y = alpha A x + beta y for symmetric A reading only its lower triangle (the dense
 * R @ state loop of td1_step_kernel, _kernels.py:203-207). HBM-bound. */
int em_symv_lower(em_ctx* ctx, int64_t n, double alpha, const double* A, int64_t lda,
                  const double* x, double beta, double* y);

/* C (n x m) = A B for a symmetric A in full storage: the products R V behind
 * modal.py:80-81 (r_n, V^T R) and modal.to_modal (modal.py:84-91). Through a device CSR
 * copy of A when it has few nonzeros (the stencil R), else the DMMA GEMM. */
int em_sym_mm(em_ctx* ctx, int64_t n, int64_t m, const double* A, int64_t lda, const double* B,
              int64_t ldb, double* C, int64_t ldc);

/* Mirror the lower triangle into the upper one in place (linalg.py:34-41 SymMatrix). */
int em_sym_mirror_lower(em_ctx* ctx, int64_t n, double* A, int64_t lda);

/* Lower Cholesky A = C C^T in place (upper triangle zeroed).
 * Replaces _kernels.cholesky_kernel (_kernels.py:18-36) / linalg.cholesky (linalg.py:92-104).
 * *pivot = -1 on success, else the first failing pivot; returns EM_ERR_NOT_PD then. */
int em_potrf(em_ctx* ctx, int64_t n, double* A, int64_t lda, int64_t* pivot);

/* B <- C^-1 B (trans = 0) or C^-T B (trans = 1), C lower triangular n x n, B n x m.
 * Replaces _kernels.tri_lower_solve_mat / tri_lower_t_solve_mat (_kernels.py:56-79). */
int em_trsm_lower(em_ctx* ctx, int trans, int64_t n, int64_t m, const double* C, int64_t ldc,
                  double* B, int64_t ldb);

/* Symmetric eigendecomposition A = U diag(w) U^T, w DESCENDING (stable ties),
 * U orthonormal (column-major n x n). A is destroyed.
 * Replaces linalg.sym_eig (linalg.py:119-134) / _kernels.jacobi_sym_eig (_kernels.py:82-141);
 * computed by Householder tridiagonalisation + divide and conquer. */
int em_syev(em_ctx* ctx, int64_t n, double* A, int64_t lda, double* w, double* U, int64_t ldu);

/* Generalized eigendecomposition L v = tau R v (modal.generalized_eig, modal.py:46-81).
 * Inputs L, R symmetric (lower triangles used), device, n x n, not modified.
 * Outputs (device): tau (n, descending), V (n x n column-major: V[i + j*ldv] =
 * component i of mode j, R-orthonormal, sign-fixed so the largest-|.| entry of
 * each column is positive), l_n, r_n (n) = diag(V^T L V), diag(V^T R V),
 * VtR (n x n column-major) = (R V), i.e. the row-major bytes of V^T R.
 * Any of l_n, r_n, VtR may be NULL to skip it.
 * *pivot / *which report a failing Cholesky: which = 0 resistance, 1 inductance. */
int em_sygv(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, const double* R, int64_t ldr,
            double* tau, double* V, int64_t ldv, double* l_n, double* r_n, double* VtR,
            int64_t ldvtr, int64_t* pivot, int* which);

/* em_sygv with flags. EM_SYGV_R_WORKSPACE: when R is sparse (nnz <= 2% of n^2, e.g.
 * the stencil resistance matrix), R's own storage holds its Cholesky factor during the
 * solve and is restored from a device CSR copy before return (its contents are
 * transient garbage meanwhile; -0.0 entries come back as +0.0). Saves one n x n buffer:
 * 6 n^2 doubles at the memory peak with VtR = NULL, so n = 60,000 fits one B200.
 * A BANDED sparse R (the plates' stencil) is factored in band storage of its own; then
 * R's storage (ldr a multiple of 32, 256-byte aligned) holds the reduced matrix
 * B = G^-1 L G^-T instead, and is restored the same way: at n = 60,000 the two-stage
 * tridiagonalisation (2.5 n^2 of workspace) fits beside L, R and V. */
#define EM_SYGV_R_WORKSPACE 1
int em_sygv_ex(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, double* R, int64_t ldr,
               double* tau, double* V, int64_t ldv, double* l_n, double* r_n, double* VtR,
               int64_t ldvtr, int flags, int64_t* pivot, int* which);
/* One rank's share of a column-sharded generalized eigensolve (the multi-GPU layout of
 * paper_2407_11993_b200/parallel.py): modes m_lo .. m_hi - 1 of the DESCENDING order.
 * Outputs tau (all n), V (n x (m_hi - m_lo), ld ldv), l_n, r_n (m_hi - m_lo) and VtR
 * (n x (m_hi - m_lo)) equal the corresponding columns / entries of em_sygv_ex's. Every
 * rank reduces the whole pencil to tridiagonal form and solves it; only the eigenvector
 * back-transforms, the sign fix and l_n, r_n are restricted to the rank's columns, so
 * the ranks exchange nothing. Flags as em_sygv_ex. */
int em_sygv_range(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, double* R, int64_t ldr,
                  int64_t m_lo, int64_t m_hi, double* tau, double* V, int64_t ldv, double* l_n,
                  double* r_n, double* VtR, int64_t ldvtr, int flags, int64_t* pivot,
                  int* which);
/* The eigensolve for the transient without forming V ("implicit V"): on entry
 * Y (n x k, ld ldy) holds operands — the drive columns [R_D | L_D | M0] and the observable
 * rows C^T —, on exit V^T Y (row j = mode j, descending tau). V^T = U^T Q^T G^-1 is applied
 * to the k columns (G: R's factor, Q: the tridiagonalisation's reflectors, U: the
 * tridiagonal eigenvectors), so the 4 n^3 flops that form V are replaced by O(n^2 k).
 * tau (n) as em_sygv; l_n = tau and r_n = 1 (the identities V^T L V = diag(tau),
 * V^T R V = I; either may be NULL). Each mode keeps the eigensolver's sign rather than
 * the reference's sign fix (modal.py:74-78, which needs V): products of two rows of V^T Y
 * (P_n x CV_n, what the modal scan uses) are unchanged. Neither V nor the tridiagonal
 * eigenvector matrix is formed: divide and conquer carries U^T Y through its merges
 * (O(n k) memory), the stage-2 reflectors reuse the reduced matrix's storage.
 * Flags: EM_SYGV_R_WORKSPACE as em_sygv_ex; EM_SYGV_L_WORKSPACE: L (ld a multiple of 32)
 * is overwritten by the reduction instead of copied — one n x n buffer less, so the peak is
 * L plus O(n (k + b)) (stage-2 reflectors in L's storage, their block factors formed per
 * wavefront) and n = 120,000 fits one B200. An in-place solve
 * cannot run the reference's Cholesky certificate of L afterwards: when the solved spectrum
 * and R's Gershgorin bounds do not already prove it redundant (see em_sygv), the call
 * fails with EM_ERR_ARG and asks to solve without the flag. */
#define EM_SYGV_L_WORKSPACE 2
int em_sygv_implicit(em_ctx* ctx, int64_t n, double* L, int64_t ldl, double* R, int64_t ldr,
                     double* tau, double* Y, int64_t ldy, int64_t k, double* l_n, double* r_n,
                     int flags, int64_t* pivot, int* which);
/* em_sygv_implicit with R given in LAPACK lower band storage (Rb[(i - j) + j * ldrb] =
 * R(i, j) for 0 <= i - j <= bw, ldrb >= bw + 1): the stencil resistance matrix of a plate
 * never exists as a dense n x n array. Flags: EM_SYGV_L_WORKSPACE. */
int em_sygv_implicit_band(em_ctx* ctx, int64_t n, double* L, int64_t ldl, const double* Rb,
                          int64_t ldrb, int64_t bw, double* tau, double* Y, int64_t ldy,
                          int64_t k, double* l_n, double* r_n, int flags, int64_t* pivot,
                          int* which);
/* em_sygv_ex with L still on the host: the library uploads L_host (n x n, leading
 * dimension n) into the device buffer L (ld ldl) on a copy engine, after the work already
 * queued on the context stream (e.g. R's upload); L is first read by the two-sided
 * reduction. With PINNED L_host the upload overlaps R's band detection and Cholesky;
 * from pageable memory the copy completes before they are enqueued (no overlap). On
 * return L holds the upload. */
int em_sygv_lh(em_ctx* ctx, int64_t n, const double* L_host, double* L, int64_t ldl, double* R,
               int64_t ldr, double* tau, double* V, int64_t ldv, double* l_n, double* r_n,
               double* VtR, int64_t ldvtr, int flags, int64_t* pivot, int* which);

/* --- modal theta-method (TD2, transient.py:116-166) ------------------------------- */

/* Plan for the decoupled stepper. r_n, l_n: n; P_r, P_l: n x n_p; P_m: n x n_s
 * (column-major, P = V^T [R_D | L_D | M0] — see em_dgemm). Holds device copies. */
int em_td2_plan_create(em_ctx* ctx, int64_t n, int n_p, int n_s, const double* l_n,
                       const double* r_n, const double* P_r, const double* P_l, const double* P_m,
                       double dt, double theta, em_td2_plan** plan);
void em_td2_plan_destroy(em_td2_plan* plan);

/* Exact per-interval integrator for piecewise-linear drives on a uniform grid of step h
 * (exact_modal_reference / exact_first_order, transient.py:315-360): the same plan type
 * and em_td2_run as the theta-method, with q^{k+1} = a q^k + c1 e0 + c2 s per mode
 * (a = exp(-h r/l)). em_td2_step / _forcing / _step_forcing reject such a plan. */
int em_td2_plan_create_exact(em_ctx* ctx, int64_t n, int n_p, int n_s, const double* l_n,
                             const double* r_n, const double* P_r, const double* P_l,
                             const double* P_m, double h, em_td2_plan** plan);

/* Observables y^k = CV q^k (+ D i_d^k): CV n_obs x n (column-major, = C V),
 * D n_obs x n_p or NULL. */
int em_td2_set_observables(em_td2_plan* plan, int n_obs, const double* CV, int64_t ldcv,
                           const double* D, int64_t ldd);

/* Integrate T steps from modal state q (n, device, in/out) over the drive table
 * drive ((T+1) x (n_p + n_s) row-major: row k = [i_d(t_k), i0(t_k)]), exactly the
 * samples run_transient uses (transient.py:290-299).
 * Y (T x n_obs row-major, may be NULL): observables after every step.
 * Qcap (n x n_caps column-major, may be NULL): q after every stride-th step.
 * Blocked linear-recurrence scan over time, fused with the forcing projection
 * and the observable reconstruction (DMMA). */
int em_td2_run(em_td2_plan* plan, int64_t T, const double* drive, double* q, double* Y,
               int64_t stride, double* Qcap);

/* Excitation sweep (BASELINE configs[4], C5): every drive channel integrated ALONE,
 * i.e. the n_c = n_p + n_s columns of the drive table as independent right-hand sides
 * (the reference superposes them into one trajectory, transient.py:147-155; by
 * linearity the sweep's responses sum to that trajectory). Q (n x n_c column-major,
 * device, in/out): per-channel modal states. Y (n_c x n_caps x n_obs, may be NULL):
 * Y[c] = observables of channel c alone (the D term only for port channels). */
int em_td2_run_sweep(em_td2_plan* plan, int64_t T, const double* drive, double* Q, double* Y,
                     int64_t stride);

/* One step, reference semantics (Td2Stepper.step): q (n) in place. i_d, di_d (n_p),
 * di0 (n_s) are HOST arrays. */
int em_td2_step(em_td2_plan* plan, double* q, const double* i_d_h, const double* di_d_h,
                const double* di0_h);

/* Per-mode forcing increment f (n, device) = -dt P_r i_d - P_ltr di_d - P_m di0
 * (Td2Stepper.forcing, transient.py:147-155; modal_forcing, modal.py:101-118). */
int em_td2_forcing(em_td2_plan* plan, const double* i_d_h, const double* di_d_h,
                   const double* di0_h, double* f);
/* q += ((-dt r q + f)/c)/c with a given forcing (step_td2, transient.py:185-195). */
int em_td2_step_forcing(em_td2_plan* plan, double* q, const double* f);

/* --- Cholesky theta-method (TD1, transient.py:77-113) ------------------------------ */

/* Z = L + dt*theta*R factored on device (potrf); R kept for the per-step matvec.
 * r_d, l_d: n x n_p; m0: n x n_s. *pivot reports a non-SPD stepping matrix. */
int em_td1_plan_create(em_ctx* ctx, int64_t n, int n_p, int n_s, const double* L, int64_t ldl,
                       const double* R, int64_t ldr, const double* r_d, const double* l_d,
                       const double* m0, double dt, double theta, em_td1_plan** plan,
                       int64_t* pivot);
/* em_td1_plan_create with R in LAPACK lower band storage (Rb[(i - j) + j ldrb] = R(i, j),
 * 0 <= i - j <= bw): R enters the plan only as a CSR. EM_TD1_L_WORKSPACE (ldl == n): the
 * stepping matrix is formed and factored in L's own storage (L is destroyed; the plan
 * references it until destroyed), so the plan holds one n x n array — n = 120,000 fits
 * one B200. */
#define EM_TD1_L_WORKSPACE 1
int em_td1_plan_create_band(em_ctx* ctx, int64_t n, int n_p, int n_s, double* L, int64_t ldl,
                            const double* Rb, int64_t ldrb, int64_t bw, const double* r_d,
                            const double* l_d, const double* m0, double dt, double theta,
                            int flags, em_td1_plan** plan, int64_t* pivot);
void em_td1_plan_destroy(em_td1_plan* plan);
int em_td1_set_observables(em_td1_plan* plan, int n_obs, const double* C, int64_t ldc,
                           const double* D, int64_t ldd);
/* T steps from state I (n, device, in/out). Y (T x n_obs) / Icap (n x n_caps) as for TD2. */
int em_td1_run(em_td1_plan* plan, int64_t T, const double* drive, double* I, double* Y,
               int64_t stride, double* Icap);
int em_td1_step(em_td1_plan* plan, double* I, const double* i_d_h, const double* di_d_h,
                const double* di0_h);
/* Copy the lower Cholesky factor of the stepping matrix (n x n, column-major) to out
 * (device). Td1Stepper.chol (transient.py:95). */
int em_td1_factor(em_td1_plan* plan, double* out, int64_t ldo);

/* --- frequency domain (frequency.py) --------------------------------- */

/* Per-tone solve (R + j w L) I = E (frequency.solve_tone, frequency.py:56-94; the
 * reference LU-factors the real 2n embedding [[R, wL], [wL, -R]]). The plan factors R
 * (lower triangles of L, R used) and forms K = L R^-1 L once; each solve is one
 * Cholesky of the SPD Schur complement R + w^2 K. *pivot reports a non-SPD R (plan)
 * or a numerically singular tone (solve) with EM_ERR_NOT_PD. */
int em_fd_plan_create(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, const double* R,
                      int64_t ldr, em_fd_plan** plan, int64_t* pivot);
void em_fd_plan_destroy(em_fd_plan* plan);
/* E = c + j d (HOST vectors, n); I = a - j b (HOST outputs), i.e. (a, b) solves the
 * embedding [[R, wL], [wL, -R]] [a; b] = [c; d] exactly as the reference's x. */
int em_fd_solve(em_fd_plan* plan, double omega, const double* c_h, const double* d_h, double* a_h,
                double* b_h, int64_t* pivot);
/* Tone table for DFT phasors (dft_phasor / extract_phasors, frequency.py:114-166):
 * out[m + 2f*ldo] = sin(2 pi f_f t_m), out[m + (2f+1)*ldo] = cos(2 pi f_f t_m),
 * t_m = t0 + m dt (device out, n_t x 2 n_f column-major; freqs_h host). */
int em_tone_table(em_ctx* ctx, int64_t n_t, double dt, double t0, int n_f, const double* freqs_h,
                  double* out, int64_t ldo);

/* --- probe observers (assembly.field_transfer, assembly.py:350-386) ------ */
/* T[(p*3 + c)*nb + j] (n_probes x 3 x nb, device) = component c of the field at probe p
 * per unit current in branch j, the exact Biot-Savart field of the straight segment
 * starts[j] -> ends[j] (nb x 3 row-major, device; probes n_probes x 3). A probe within
 * radius[j] of branch j's segment: EM_ERR_ARG with *bad = p*nb + j of the first such pair
 * (the reference's ProbeTooClose), else *bad = -1. */
int em_field_transfer(em_ctx* ctx, int64_t nb, const double* starts, const double* ends,
                      const double* radius, int64_t n_probes, const double* probes, double* T,
                      int64_t* bad);

/* --- synthetic plate inputs (BASELINE.json configs; definition in synth.py) ----------- */
/* Dense L (n x n), dense-stored R = rho*K7 + shift*I, and the one-port electrode
 * columns l_d, r_d (n) for voxels keep[0..n) of an nx*ny*nz grid (pos: voxel id ->
 * kept index or -1; ang: seeded in-plane angles). Any output may be NULL. */
int em_synth_plate(em_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double h, double rho,
                   double shift, int64_t n, const int64_t* keep, const int64_t* pos,
                   const double* ang, double* L, int64_t ldl, double* R, int64_t ldr,
                   double* l_d, double* r_d);

/* --- end-to-end host-pointer entry (the reference-facing call with HOST buffers) -- */

/* generalized_eig on host arrays: copies L, R in, solves, copies tau, l_n, r_n back
 * (V, VtR back too when non-NULL). Used to time the e2e path (H2D + D2H inside). */
int em_sygv_h(em_ctx* ctx, int64_t n, const double* L_h, const double* R_h, double* tau_h,
              double* V_h, double* l_n_h, double* r_n_h, double* VtR_h, int64_t* pivot,
              int* which);

#ifdef __cplusplus
}
#endif
#endif
