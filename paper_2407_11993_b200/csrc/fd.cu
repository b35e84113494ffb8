// Frequency-domain companions of the modal path:
//
// * per-tone solve (R + j w L) I = E (frequency.solve_tone, E/frequency.py:56-94).
//   The reference factors the real 2n embedding [[R, wL], [wL, -R]] by pivoted LU
//   (16/3 n^3 flop per tone, E/_kernels.py:144-193). With R SPD the embedding has the
//   SPD Schur complement S(w) = R + w^2 L R^-1 L, and K = L R^-1 L = M^T M (M = G^-1 L,
//   R = G G^T) does not depend on w. So a plan factors R and forms K once (potrf +
//   trsm + lower GEMM, DMMA), and each tone is one Cholesky of S plus triangular
//   solves: for E = c + j d and I = a - j b,
//     b = S^-1 (w L R^-1 c - d),  a = R^-1 (c - w L b),
//   followed by two steps of iterative refinement on the embedding's residual (the
//   Schur complement squares the conditioning when w L >> R), which brings the
//   result to the reference's accuracy.
// * the tone table for DFT phasors (frequency.dft_phasor / extract_phasors,
//   E/frequency.py:114-166): [sin(w t_m), cos(w t_m)] per tone with t_m = t0 + m dt,
//   so the phasors of every observable record are one DMMA GEMM.
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

struct em_fd_plan {
  em_ctx* ctx = nullptr;
  int64_t n = 0;
  em::DBuf L, R, G, GDinv, K, S, SDinv, work, v1, v2;
};

namespace em {

__global__ void fd_schur_kernel(int64_t n, double w2, const double* __restrict__ R,
                                const double* __restrict__ K, double* __restrict__ S) {
  const int64_t total = n * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % n, c = i / n;
    S[i] = (r >= c) ? fma(w2, K[i], R[i]) : 0.0;
  }
}

// out = alpha * x + beta * y (n); out may alias x or y (element-wise)
__global__ void fd_axpby_kernel(int64_t n, double alpha, const double* x, double beta,
                                const double* y, double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = fma(alpha, x[i], beta * y[i]);
}

__global__ void tone_table_kernel(int64_t n_t, double dt, double t0, int n_f,
                                  const double* __restrict__ freqs, double* __restrict__ out,
                                  int64_t ldo) {
  const int f = blockIdx.y;
  const double w = 2.0 * 3.141592653589793 * freqs[f];
  for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n_t;
       m += (int64_t)gridDim.x * blockDim.x) {
    const double t = t0 + dt * (double)m;  // the reference's t = t0 + dt * arange(n)
    double s, c;
    sincos(w * t, &s, &c);
    out[m + (int64_t)(2 * f) * ldo] = s;
    out[m + (int64_t)(2 * f + 1) * ldo] = c;
  }
}

}  // namespace em

using namespace em;

namespace {
template <typename F>
int fd_guarded(em_ctx* ctx, F&& f) {
  try {
    if (ctx) cudaSetDevice(ctx->device);
    return f();
  } catch (const CudaError& e) {
    if (ctx) ctx->err = std::string(cudaGetErrorString(e.code)) + " in " + e.where;
    return EM_ERR_CUDA;
  } catch (const ArgError& e) {
    if (ctx) ctx->err = e.what;
    return EM_ERR_ARG;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed";
    return EM_ERR_ALLOC;
  }
}

// x <- A^-1 x for the SPD matrix with lower factor C (n x n) and block inverses Dinv
void spd_solve(cudaStream_t st, int64_t n, const double* C, const double* Dinv, double* x) {
  trsm_lower(st, false, n, 1, C, n, x, n, Dinv);
  trsm_lower(st, true, n, 1, C, n, x, n, Dinv);
}
}  // namespace

extern "C" {

int em_fd_plan_create(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, const double* R,
                      int64_t ldr, em_fd_plan** plan, int64_t* pivot) {
  return fd_guarded(ctx, [&] {
    if (!plan || n < 0) throw ArgError{"bad fd plan arguments"};
    cudaStream_t st = ctx->stream;
    auto* P = new em_fd_plan();
    P->ctx = ctx;
    P->n = n;
    const size_t nn = (size_t)n * n;
    const int64_t nblk = (n + kTrsmBlock - 1) / kTrsmBlock;
    try {
      P->L.alloc(nn, st);
      P->R.alloc(nn, st);
      P->G.alloc(nn, st);
      P->K.alloc(nn, st);
      P->S.alloc(nn, st);
      P->GDinv.alloc((size_t)imax64(nblk, 1) * kTrsmBlock * kTrsmBlock, st);
      P->SDinv.alloc((size_t)imax64(nblk, 1) * kTrsmBlock * kTrsmBlock, st);
      P->work.alloc(symv_work_size(n), st);
      P->v1.alloc(imax64(n, 1), st);
      P->v2.alloc(imax64(n, 1), st);
      // SymMatrix semantics: the lower triangles define L and R
      copy_matrix(st, false, n, n, L, ldl, P->L.p, n);
      copy_matrix(st, false, n, n, R, ldr, P->R.p, n);
      mirror_lower(st, n, P->L.p, n);
      mirror_lower(st, n, P->R.p, n);
      copy_matrix(st, false, n, n, P->R.p, n, P->G.p, n);
      const int64_t piv = potrf(st, n, P->G.p, n, P->GDinv.p);
      if (pivot) *pivot = piv;
      if (piv >= 0) {
        delete P;
        return EM_ERR_NOT_PD;
      }
      // K = M^T M, M = G^-1 L (lower triangle of K is enough for S)
      DBuf M(nn, st);
      copy_matrix(st, false, n, n, P->L.p, n, M.p, n);
      trsm_lower(st, false, n, n, P->G.p, n, M.p, n, P->GDinv.p);
      EM_CK(gemm(st, true, false, n, n, n, 1.0, M.p, n, M.p, n, 0.0, P->K.p, n, true, 0));
      EM_CK(cudaStreamSynchronize(st));
    } catch (...) {
      delete P;
      throw;
    }
    *plan = P;
    return EM_OK;
  });
}

void em_fd_plan_destroy(em_fd_plan* plan) {
  if (!plan) return;
  cudaSetDevice(plan->ctx->device);
  cudaStreamSynchronize(plan->ctx->stream);
  delete plan;
}

int em_fd_solve(em_fd_plan* P, double omega, const double* c_h, const double* d_h, double* a_h,
                double* b_h, int64_t* pivot) {
  em_ctx* ctx = P ? P->ctx : nullptr;
  return fd_guarded(ctx, [&] {
    if (!P || !(omega >= 0.0)) throw ArgError{"bad fd solve arguments"};
    cudaStream_t st = ctx->stream;
    const int64_t n = P->n;
    if (n == 0) return EM_OK;
    DBuf c(n, st), d(n, st), b(n, st);
    EM_CK(cudaMemcpyAsync(c.p, c_h, n * 8, cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(d.p, d_h, n * 8, cudaMemcpyHostToDevice, st));
    const unsigned g = (unsigned)imin64((n * n + 255) / 256, 148 * 16);
    fd_schur_kernel<<<g, 256, 0, st>>>(n, omega * omega, P->R.p, P->K.p, P->S.p);
    EM_LAUNCHED();
    const int64_t piv = potrf(st, n, P->S.p, n, P->SDinv.p);
    if (pivot) *pivot = piv;
    if (piv >= 0) return EM_ERR_NOT_PD;
    const unsigned gv = (unsigned)((n + 255) / 256);
    // one Schur solve: (ca, cb) = rhs -> (xa, xb) with [[R, wL], [wL, -R]] [xa; xb] = rhs
    auto schur = [&](const double* rc, const double* rd, double* xa, double* xb) {
      // v1 = R^-1 c;  xb = S^-1 (w L v1 - d)
      EM_CK(cudaMemcpyAsync(P->v1.p, rc, n * 8, cudaMemcpyDeviceToDevice, st));
      spd_solve(st, n, P->G.p, P->GDinv.p, P->v1.p);
      symv_lower(st, n, omega, P->L.p, n, P->v1.p, 0.0, P->v2.p, P->work.p);
      fd_axpby_kernel<<<gv, 256, 0, st>>>(n, 1.0, P->v2.p, -1.0, rd, xb);
      EM_LAUNCHED();
      spd_solve(st, n, P->S.p, P->SDinv.p, xb);
      // xa = R^-1 (c - w L xb)
      symv_lower(st, n, omega, P->L.p, n, xb, 0.0, P->v2.p, P->work.p);
      fd_axpby_kernel<<<gv, 256, 0, st>>>(n, 1.0, rc, -1.0, P->v2.p, xa);
      EM_LAUNCHED();
      spd_solve(st, n, P->G.p, P->GDinv.p, xa);
    };
    DBuf a(n, st), ra(n, st), rb(n, st), da(n, st), db(n, st);
    schur(c.p, d.p, a.p, b.p);
    // The Schur complement squares the conditioning when w L >> R; two steps of
    // iterative refinement on the embedding's residual (r = rhs - [[R, wL], [wL, -R]] x,
    // four symv) bring the solution to the accuracy of a direct solve of the embedding.
    for (int it = 0; it < 2; ++it) {
      symv_lower(st, n, 1.0, P->R.p, n, a.p, 0.0, ra.p, P->work.p);     // R a
      symv_lower(st, n, omega, P->L.p, n, b.p, 1.0, ra.p, P->work.p);   // + w L b
      symv_lower(st, n, omega, P->L.p, n, a.p, 0.0, rb.p, P->work.p);   // w L a
      symv_lower(st, n, -1.0, P->R.p, n, b.p, 1.0, rb.p, P->work.p);    // - R b
      fd_axpby_kernel<<<gv, 256, 0, st>>>(n, 1.0, c.p, -1.0, ra.p, ra.p);
      EM_LAUNCHED();
      fd_axpby_kernel<<<gv, 256, 0, st>>>(n, 1.0, d.p, -1.0, rb.p, rb.p);
      EM_LAUNCHED();
      schur(ra.p, rb.p, da.p, db.p);
      fd_axpby_kernel<<<gv, 256, 0, st>>>(n, 1.0, a.p, 1.0, da.p, a.p);
      EM_LAUNCHED();
      fd_axpby_kernel<<<gv, 256, 0, st>>>(n, 1.0, b.p, 1.0, db.p, b.p);
      EM_LAUNCHED();
    }
    EM_CK(cudaMemcpyAsync(P->v1.p, a.p, n * 8, cudaMemcpyDeviceToDevice, st));
    EM_CK(cudaMemcpyAsync(a_h, P->v1.p, n * 8, cudaMemcpyDeviceToHost, st));
    EM_CK(cudaMemcpyAsync(b_h, b.p, n * 8, cudaMemcpyDeviceToHost, st));
    EM_CK(cudaStreamSynchronize(st));
    return EM_OK;
  });
}

int em_tone_table(em_ctx* ctx, int64_t n_t, double dt, double t0, int n_f, const double* freqs_h,
                  double* out, int64_t ldo) {
  return fd_guarded(ctx, [&] {
    if (n_t < 0 || n_f < 0 || ldo < n_t) throw ArgError{"bad tone table arguments"};
    if (n_t == 0 || n_f == 0) return EM_OK;
    cudaStream_t st = ctx->stream;
    DBuf f(n_f, st);
    EM_CK(cudaMemcpyAsync(f.p, freqs_h, n_f * 8, cudaMemcpyHostToDevice, st));
    dim3 grid((unsigned)imin64((n_t + 255) / 256, 1024), (unsigned)n_f);
    tone_table_kernel<<<grid, 256, 0, st>>>(n_t, dt, t0, n_f, f.p, out, ldo);
    EM_LAUNCHED();
    EM_CK(cudaStreamSynchronize(st));  // f lifetime
    return EM_OK;
  });
}

}  // extern "C"
