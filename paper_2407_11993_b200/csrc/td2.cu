// Modal theta-method (TD2) on B200: forcing projection + per-mode linear
// recurrence + observable reconstruction.
//
// Reference: Td2Stepper (pkg/src/eddymodes/transient.py:116-166) advances every
// mode by q += ((-dt*r*q + f)/c)/c with c = sqrt(l + dt*theta*r)
// (_kernels.py:213-222) and f = -dt*P_r i_D - P_ltr dI_D - P_m dI_0
// (transient.py:147-155); run_transient (transient.py:248-312) reconstructs the
// observables from V q after every captured step.
//
// Here the recurrence is written q^{k+1} = (1 - eps) q^k + g^k with
// eps = dt*r/den, g^k = W u^k, W = (1/den)[-dt P_r | -P_ltr | -P_m] and
// u^k = [i_D^k, dI_D^k, dI_0^k]; it is linear, hence associative over time, and
// is evaluated as a BLOCKED SCAN: time is cut into blocks of TB steps,
//   pass 1 (td2_local_scan)   end state of every (mode, block) from zero,
//   pass 2 (td2_carry)        block-start states S_b by a short sequential carry,
//   pass 3 (td2_replay)       each CTA replays its block from S_b, keeps the
//                             (modes x TB) trajectory tile in shared memory and
//                             multiplies it by the C V tile on DMMA tensor cores,
// so the O(N T) trajectory never touches HBM and time is a parallel axis.
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"
#include "plans.h"

#include <vector>

struct em_td2_plan {
  em_ctx* ctx = nullptr;
  int64_t n = 0;
  int n_p = 0, n_s = 0, n_u = 0;
  double dt = 0, theta = 0;
  em::DBuf eps, binv, W;       // recurrence form
  em::DBuf rn, cn, Pr, Pltr, Pm;  // reference single-step form
  int n_obs = 0, n_obs_pad = 0;
  em::DBuf CV, D;
  bool exact = false;  // exponential-integrator recurrence (no single-step form)
};

namespace em {

constexpr int TB = 64;        // time steps per block
constexpr int MC = 64;        // modes per chunk in the replay kernel (70 KB of shared
                              // memory per CTA: three CTAs per SM overlap one CTA's
                              // recurrence and loads with the others' DMMA)
constexpr int RT = 256;       // threads per CTA
constexpr int QS = MC + 4;    // Qs row stride (≡ 4 mod 16 doubles: conflict-free B fragments)

__global__ void td2_coeffs_kernel(int64_t n, int n_p, int n_s, double dt, double theta,
                                  const double* __restrict__ l_n, const double* __restrict__ r_n,
                                  const double* __restrict__ P_r, const double* __restrict__ P_l,
                                  const double* __restrict__ P_m, double* eps, double* binv,
                                  double* W, double* rn, double* cn, double* Pr, double* Pltr,
                                  double* Pm) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double den = l_n[i] + dt * theta * r_n[i];
  const double b = 1.0 / den;
  eps[i] = dt * r_n[i] * b;
  binv[i] = b;
  rn[i] = r_n[i];
  cn[i] = sqrt(den);
  for (int p = 0; p < n_p; ++p) {
    const double pr = P_r[i + p * n], pl = P_l[i + p * n];
    const double pltr = pl + dt * theta * pr;
    Pr[i + p * n] = pr;
    Pltr[i + p * n] = pltr;
    W[i + (int64_t)p * n] = -dt * pr * b;
    W[i + (int64_t)(n_p + p) * n] = -pltr * b;
  }
  for (int s = 0; s < n_s; ++s) {
    const double pm = P_m[i + s * n];
    Pm[i + s * n] = pm;
    W[i + (int64_t)(2 * n_p + s) * n] = -pm * b;
  }
}

// Exact per-interval integrator for piecewise-linear drives (exact_modal_reference /
// exact_first_order, E/transient.py:315-360) as the same recurrence
// q^{k+1} = (1 - eps) q^k + W u^k:  with tau = l/r, a = exp(-h/tau),
//   eps = -expm1(-h/tau),  q^{k+1} = a q^k + c1 e0 + c2 s,
//   c1 = (1 - a)/r,  c2 = (h - (1 - a) tau)/r,
//   e0 = -P_r i_d^k - P_l di_d/h - P_m di0/h,  s = -P_r di_d/h  (u = [i_d^k, di_d, di0]).
__global__ void td2_exact_coeffs_kernel(int64_t n, int n_p, int n_s, double h,
                                        const double* __restrict__ l_n,
                                        const double* __restrict__ r_n,
                                        const double* __restrict__ P_r,
                                        const double* __restrict__ P_l,
                                        const double* __restrict__ P_m, double* eps, double* W) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double r = r_n[i], tau = l_n[i] / r;
  const double oma = -expm1(-h / tau);  // 1 - a
  eps[i] = oma;
  const double c1 = oma / r, c2 = (h - oma * tau) / r;
  for (int p = 0; p < n_p; ++p) {
    const double pr = P_r[i + p * n], pl = P_l[i + p * n];
    W[i + (int64_t)p * n] = -c1 * pr;
    W[i + (int64_t)(n_p + p) * n] = -(c1 * pl + c2 * pr) / h;
  }
  for (int s = 0; s < n_s; ++s) W[i + (int64_t)(2 * n_p + s) * n] = -c1 * P_m[i + s * n] / h;
}

// u^k rows from the drive table (row k = [i_d(t_k) | i0(t_k)]).
__global__ void td2_inputs_kernel(int64_t T, int n_p, int n_s, const double* __restrict__ drive,
                                  double* __restrict__ U) {
  const int n_c = n_p + n_s, n_u = 2 * n_p + n_s;
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= T) return;
  const double* d0 = drive + k * n_c;
  const double* d1 = d0 + n_c;
  double* u = U + k * n_u;
  for (int p = 0; p < n_p; ++p) {
    u[p] = d0[p];
    u[n_p + p] = d1[p] - d0[p];
  }
  for (int s = 0; s < n_s; ++s) u[2 * n_p + s] = d1[n_p + s] - d0[n_p + s];
}

// Stage the TB x n_u input rows of block b into shared memory (zero past T).
EM_DEVINL void stage_inputs(double* Us, const double* __restrict__ U, int64_t T, int n_u,
                            int64_t b) {
  for (int i = threadIdx.x; i < TB * n_u; i += blockDim.x) {
    int64_t k = b * TB + i / n_u;
    Us[i] = (k < T) ? U[b * TB * n_u + i] : 0.0;
  }
}

template <int NU>
EM_DEVINL double forcing(const double* w, const double* urow, int n_u) {
  double g = 0.0;
  if (NU > 0) {
#pragma unroll
    for (int j = 0; j < NU; ++j) g = fma(w[j], urow[j], g);
  } else {
    for (int j = 0; j < n_u; ++j) g = fma(w[j], urow[j], g);
  }
  return g;
}

constexpr int NU_MAX_REG = 8;

// pass 1: E[b][m] = state after block b starting from 0
template <int NU>
__global__ void __launch_bounds__(RT) td2_local_scan(int64_t n, int64_t T, int n_u,
                                                     const double* __restrict__ eps,
                                                     const double* __restrict__ W,
                                                     const double* __restrict__ U,
                                                     double* __restrict__ E) {
  extern __shared__ double Us[];
  const int64_t b = blockIdx.x;
  stage_inputs(Us, U, T, n_u, b);
  __syncthreads();
  const int len = (int)imin64(TB, T - b * TB);
  for (int64_t m = threadIdx.x + blockIdx.y * (int64_t)RT; m < n; m += (int64_t)RT * gridDim.y) {
    double w[NU > 0 ? NU : NU_MAX_REG];
    const int nu_loc = NU > 0 ? NU : n_u;
    for (int j = 0; j < nu_loc && j < NU_MAX_REG; ++j) w[j] = W[m + j * n];
    const double e = eps[m];
    double s = 0.0;
    if (NU > 0) {
      for (int k = 0; k < len; ++k) s = fma(-e, s, s) + forcing<NU>(w, Us + k * n_u, n_u);
    } else {
      for (int k = 0; k < len; ++k) {
        double g = 0.0;
        for (int j = 0; j < n_u; ++j) g = fma(W[m + j * n], Us[k * n_u + j], g);
        s = fma(-e, s, s) + g;
      }
    }
    E[b * n + m] = s;
  }
}

// (1 - eps)^len, accurate for eps near 0 (eps = dt*r/den ~ 1e-8..1e-5 here)
EM_DEVINL double decay_pow(double e, int len) {
  if (e < 0.5 && e > -0.5) return exp((double)len * log1p(-e));
  double a = 1.0 - e, r = 1.0;
  int k = len;
  while (k) {
    if (k & 1) r *= a;
    a *= a;
    k >>= 1;
  }
  return r;
}

// pass 2: S[b][m] = state at the start of block b; q <- final state
__global__ void td2_carry(int64_t n, int64_t T, int64_t nb, const double* __restrict__ eps,
                          const double* __restrict__ E, double* __restrict__ S,
                          double* __restrict__ q) {
  int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (m >= n) return;
  const double e = eps[m];
  const double a_full = decay_pow(e, TB);
  double s = q[m];
  for (int64_t b = 0; b < nb; ++b) {
    S[b * n + m] = s;
    const int len = (int)imin64(TB, T - b * TB);
    const double a = (len == TB) ? a_full : decay_pow(e, len);
    s = fma(a, s, E[b * n + m]);
  }
  q[m] = s;
}

// pass 3: replay each block from S_b; Y_tile(n_obs x TB) += CV_chunk * Q_tile on DMMA.
// grid (nb, nsplit); split sp handles modes [sp*mps, (sp+1)*mps).
template <int NU, int MT>
__global__ void __launch_bounds__(RT) td2_replay(
    int64_t n, int64_t T, int n_u, int n_obs, int cvs, int64_t mps, const double* __restrict__ eps,
    const double* __restrict__ W, const double* __restrict__ U, const double* __restrict__ S,
    const double* __restrict__ CV, int ldcv, int64_t stride, double* __restrict__ Yout,
    int64_t ldy_split, double* __restrict__ Qcap, int64_t n_caps) {
  extern __shared__ __align__(16) double sm[];
  double* Qs = sm;                  // [TB][QS]
  double* Cs = Qs + TB * QS;        // [MC][cvs]
  double* Us = Cs + MC * cvs;       // [TB][n_u]
  const int64_t b = blockIdx.x;
  const int64_t m_begin = blockIdx.y * mps;
  const int64_t m_end = imin64(n, m_begin + mps);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;
  stage_inputs(Us, U, T, n_u, b);
  const int len = (int)imin64(TB, T - b * TB);

  // warp tile: WM x 4 warps over (observables x time); each warp MTW m-tiles x NTW
  // n-tiles of 8 x 8 (MT >= 2: half the observables x 16 steps, fewer shared-memory
  // fragment loads per DMMA than all observables x 8 steps)
  constexpr int WM = MT >= 2 ? 2 : 1;
  constexpr int MTW = MT / WM;
  constexpr int NTW = (TB / 8) / (8 / WM);
  const int wm = warp / (8 / WM), wn = warp % (8 / WM);
  double acc[MTW][NTW][2];
#pragma unroll
  for (int i = 0; i < MTW; ++i)
#pragma unroll
    for (int jn = 0; jn < NTW; ++jn) acc[i][jn][0] = acc[i][jn][1] = 0.0;

  // Recurrence split over the whole CTA: thread (mode mm = tid % MC, quarter qq = tid / MC)
  // scans its NQ = TB / 4 steps from zero (local values l_k, end value L_qq), the quarter
  // start states follow from S_{q+1} = a^NQ S_q + L_q (a = 1 - eps), and every value is
  // fixed up as s_k = l_k + a^(k - k_q + 1) S_q: a sequential chain of NQ + 3 + NQ steps
  // on all eight warps instead of TB steps on two.
  static_assert(RT == 4 * MC, "four threads per mode");
  constexpr int NQ = TB / 4;
  __shared__ double Lend[4][MC];
  const int mm = tid % MC, qq = tid / MC;
  for (int64_t c0 = m_begin; c0 < m_end; c0 += MC) {
    __syncthreads();  // previous chunk's fragments consumed (and Us staged on entry)
    // CV chunk -> Cs[mode][o]: asynchronous copies (no registers, overlap the scan)
    {
      const int nw = RT >> 5;
      for (int r = warp; r < MC; r += nw) {
        const int64_t m = c0 + r;
        const bool live = m < m_end;
        for (int o = lane; o < cvs; o += 32) {
          double* dst = Cs + r * cvs + o;
          const bool ok = o < n_obs && live;
          cp_async8(dst, ok ? CV + o + m * (int64_t)ldcv : CV, ok);  // zero fill otherwise
        }
      }
      cp_async_commit();
    }
    const int64_t m = c0 + mm;
    const bool live = m < m_end;
    const double e = live ? eps[m] : 0.0;
    const double s0 = live ? S[b * n + m] : 0.0;
    double w[NU > 0 ? NU : 1];
    if (NU > 0) {
#pragma unroll
      for (int j = 0; j < (NU > 0 ? NU : 1); ++j) w[j] = live ? W[m + j * n] : 0.0;
    }
    const int k0 = qq * NQ;
    double l = 0.0;
#pragma unroll 4
    for (int kk = 0; kk < NQ; ++kk) {
      const int k = k0 + kk;
      double gk;
      if (NU > 0) {
        gk = forcing<NU>(w, Us + k * n_u, n_u);
      } else {
        gk = 0.0;
        if (live)
          for (int j = 0; j < n_u; ++j) gk = fma(W[m + j * n], Us[k * n_u + j], gk);
      }
      l = fma(-e, l, l) + gk;
      Qs[k * QS + mm] = l;
    }
    Lend[qq][mm] = l;
    __syncthreads();
    const double a = 1.0 - e;
    const double aq = decay_pow(e, NQ);
    double sq = s0;
    for (int q = 0; q < qq; ++q) sq = fma(aq, sq, Lend[q][mm]);
    double pw = a;
#pragma unroll 4
    for (int kk = 0; kk < NQ; ++kk) {
      const int k = k0 + kk;
      double v = fma(pw, sq, Qs[k * QS + mm]);
      pw *= a;
      if (k >= len) v = 0.0;
      Qs[k * QS + mm] = v;
      const int64_t kg = b * TB + k;
      if (Qcap && live && k < len && ((kg + 1) % stride) == 0)
        Qcap[m + ((kg + 1) / stride - 1) * n] = v;
    }
    cp_async_wait<0>();
    __syncthreads();
    // DMMA: warp (wm, wn) owns m-tiles [wm MTW, (wm+1) MTW) and time columns
    // [8 NTW wn, 8 NTW (wn+1))
#pragma unroll 4
    for (int kb = 0; kb < MC; kb += 4) {
      double bf[NTW];
#pragma unroll
      for (int jn = 0; jn < NTW; ++jn) bf[jn] = Qs[((wn * NTW + jn) * 8 + g) * QS + kb + t];
#pragma unroll
      for (int mt = 0; mt < MTW; ++mt) {
        const double af = Cs[(kb + t) * cvs + (wm * MTW + mt) * 8 + g];
#pragma unroll
        for (int jn = 0; jn < NTW; ++jn) dmma884(acc[mt][jn][0], acc[mt][jn][1], af, bf[jn]);
      }
    }
  }
  // epilogue: rows o = (wm MTW + mt) 8 + g, time k = b TB + (wn NTW + jn) 8 + 2t + e
#pragma unroll
  for (int mt = 0; mt < MTW; ++mt) {
    const int o = (wm * MTW + mt) * 8 + g;
    if (o >= n_obs) continue;
#pragma unroll
    for (int jn = 0; jn < NTW; ++jn)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t kg = b * TB + (wn * NTW + jn) * 8 + 2 * t + e;
        if (kg >= T || ((kg + 1) % stride) != 0) continue;
        const int64_t cap = (kg + 1) / stride - 1;
        Yout[blockIdx.y * ldy_split + cap * n_obs + o] = acc[mt][jn][e];
      }
  }
}

// Y[c][o] = sum_sp Ypart[sp][c][o] + sum_p D[o,p] i_d(t_{k+1}),  k = (c+1)*stride - 1
__global__ void td2_reduce_kernel(int64_t n_caps, int n_obs, int nsplit, int64_t ldy_split,
                                  const double* __restrict__ Ypart, int n_p, int n_c,
                                  const double* __restrict__ D, int ldd,
                                  const double* __restrict__ drive, int64_t stride,
                                  double* __restrict__ Y) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_caps * n_obs) return;
  const int64_t c = i / n_obs;
  const int o = (int)(i % n_obs);
  double v = 0.0;
  for (int sp = 0; sp < nsplit; ++sp) v += Ypart[sp * ldy_split + i];
  if (D) {
    const int64_t k1 = (c + 1) * stride;  // t_{k+1}
    for (int p = 0; p < n_p; ++p) v = fma(D[o + p * ldd], drive[k1 * n_c + p], v);
  }
  Y[i] = v;
}

// Single step with the reference's update form (Td2Stepper.step).
__global__ void td2_step_kernel(int64_t n, int n_p, int n_s, double dt,
                                const double* __restrict__ Pr, const double* __restrict__ Pltr,
                                const double* __restrict__ Pm, const double* __restrict__ rn,
                                const double* __restrict__ cn, const double* __restrict__ u,
                                double* __restrict__ q) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double f = 0.0;
  for (int p = 0; p < n_p; ++p) f -= dt * (Pr[i + p * n] * u[p]);
  for (int p = 0; p < n_p; ++p) f -= Pltr[i + p * n] * u[n_p + p];
  for (int s = 0; s < n_s; ++s) f -= Pm[i + s * n] * u[2 * n_p + s];
  const double s = rn[i] * q[i];
  const double num = -dt * s + f;
  q[i] += (num / cn[i]) / cn[i];
}

template <int NU, int MT>
static void launch_replay(cudaStream_t st, dim3 grid, size_t smem, int64_t n, int64_t T, int n_u,
                          int n_obs, int cvs, int64_t mps, const double* eps, const double* W,
                          const double* U, const double* S, const double* CV, int ldcv,
                          int64_t stride, double* Y, int64_t ldys, double* Qcap,
                          int64_t n_caps) {
  auto k = td2_replay<NU, MT>;
  EM_CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  k<<<grid, RT, smem, st>>>(n, T, n_u, n_obs, cvs, mps, eps, W, U, S, CV, ldcv, stride, Y, ldys,
                            Qcap, n_caps);
  EM_LAUNCHED();
}

template <int NU>
static void dispatch_mt(int mt, cudaStream_t st, dim3 grid, size_t smem, int64_t n, int64_t T,
                        int n_u, int n_obs, int cvs, int64_t mps, const double* eps,
                        const double* W, const double* U, const double* S, const double* CV,
                        int ldcv, int64_t stride, double* Y, int64_t ldys, double* Qcap,
                        int64_t n_caps) {
#define EM_MT(V)                                                                              \
  if (mt <= V) {                                                                              \
    launch_replay<NU, V>(st, grid, smem, n, T, n_u, n_obs, cvs, mps, eps, W, U, S, CV, ldcv, \
                         stride, Y, ldys, Qcap, n_caps);                                      \
    return;                                                                                   \
  }
  EM_MT(1) EM_MT(2) EM_MT(4) EM_MT(8) EM_MT(16)
#undef EM_MT
  throw ArgError{"n_obs > 128 is not supported by the fused reconstruction"};
}

template <int NU>
static void local_scan(cudaStream_t st, int64_t nb, int64_t n, int64_t T, int n_u,
                       const double* eps, const double* W, const double* U, double* E) {
  size_t smem = (size_t)TB * n_u * sizeof(double);
  int ysplit = (int)imax64(1, imin64((2 * num_sms() + nb - 1) / nb, (n + RT - 1) / RT));
  dim3 grid((unsigned)nb, (unsigned)ysplit);
  td2_local_scan<NU><<<grid, RT, smem, st>>>(n, T, n_u, eps, W, U, E);
  EM_LAUNCHED();
}

// One blocked-scan run over prepared inputs: U (T x n_u, row k = u^k), W (n x n_u),
// q (n, in/out); observables Y (n_caps x n_obs) with the direct term
// sum_p D[o, p] * dtab[k1 * dld + p] for p < n_pd (D n_obs x n_pd, ld = n_obs).
static void td2_core(em_td2_plan* P, int64_t T, int n_u, const double* Wp, const double* Up,
                     double* q, double* Y, int64_t stride, double* Qcap, const double* Dp,
                     int n_pd, const double* dtab, int dld) {
  cudaStream_t st = P->ctx->stream;
  const int64_t n = P->n;
  const int64_t nb = (T + TB - 1) / TB;
  const int64_t n_caps = T / stride;
  DBuf U0;
  if (n_u == 0) {
    U0.alloc((size_t)T, st);
    EM_CK(cudaMemsetAsync(U0.p, 0, (size_t)T * sizeof(double), st));
    Up = U0.p;
  }
  const int nu_eff = imax64(n_u, 1);
  const double* W = n_u > 0 ? Wp : nullptr;
  DBuf Wz;
  if (n_u == 0) {  // no drive: a zero input column keeps the kernels uniform
    Wz.alloc(n, st);
    EM_CK(cudaMemsetAsync(Wz.p, 0, n * sizeof(double), st));
    W = Wz.p;
  }
  DBuf E((size_t)nb * n, st), S((size_t)nb * n, st);
  stage_begin(st, ST_TD2_LOCAL);
  switch (nu_eff) {
    case 1: local_scan<1>(st, nb, n, T, nu_eff, P->eps.p, W, Up, E.p); break;
    case 2: local_scan<2>(st, nb, n, T, nu_eff, P->eps.p, W, Up, E.p); break;
    case 3: local_scan<3>(st, nb, n, T, nu_eff, P->eps.p, W, Up, E.p); break;
    case 4: local_scan<4>(st, nb, n, T, nu_eff, P->eps.p, W, Up, E.p); break;
    default: local_scan<0>(st, nb, n, T, nu_eff, P->eps.p, W, Up, E.p); break;
  }
  stage_end(st, ST_TD2_LOCAL);
  stage_begin(st, ST_TD2_CARRY);
  td2_carry<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, T, nb, P->eps.p, E.p, S.p, q);
  EM_LAUNCHED();
  stage_end(st, ST_TD2_CARRY);

  if (!Y && !Qcap) return;
  // observables (or a dummy single row when only states are captured)
  const int n_obs = (Y && P->n_obs > 0) ? P->n_obs : 1;
  const int n_obs_pad = (n_obs + 7) / 8 * 8;
  const int cvs = n_obs_pad + ((4 - n_obs_pad % 16) + 16) % 16;
  DBuf cvz;
  const double* CV = P->CV.p;
  int ldcv = P->n_obs_pad;
  if (!(Y && P->n_obs > 0)) {
    cvz.alloc(n, st);
    EM_CK(cudaMemsetAsync(cvz.p, 0, n * sizeof(double), st));
    CV = cvz.p;
    ldcv = 1;
  }
  const int64_t nchunks = (n + MC - 1) / MC;
  // mode splits: about 8 waves of 3 CTAs per SM (wave quantisation below ~12%); each
  // split adds one n_caps x n_obs partial to the final reduction
  int nsplit = (int)imax64(1, imin64((24 * num_sms() + nb - 1) / nb, nchunks));
  const int64_t mps = ((nchunks + nsplit - 1) / nsplit) * MC;
  nsplit = (int)((n + mps - 1) / mps);
  const int64_t ldys = imax64(n_caps, 1) * n_obs;
  DBuf Ypart((size_t)nsplit * ldys, st);
  size_t smem = ((size_t)TB * QS + (size_t)MC * cvs + (size_t)TB * nu_eff) * sizeof(double);
  dim3 grid((unsigned)nb, (unsigned)nsplit);
  const int mt = n_obs_pad / 8;
  Stage replay_stage(st, ST_TD2_REPLAY);
  switch (nu_eff) {
    case 1: dispatch_mt<1>(mt, st, grid, smem, n, T, nu_eff, n_obs, cvs, mps, P->eps.p, W, Up, S.p, CV, ldcv, stride, Ypart.p, ldys, Qcap, n_caps); break;
    case 2: dispatch_mt<2>(mt, st, grid, smem, n, T, nu_eff, n_obs, cvs, mps, P->eps.p, W, Up, S.p, CV, ldcv, stride, Ypart.p, ldys, Qcap, n_caps); break;
    case 3: dispatch_mt<3>(mt, st, grid, smem, n, T, nu_eff, n_obs, cvs, mps, P->eps.p, W, Up, S.p, CV, ldcv, stride, Ypart.p, ldys, Qcap, n_caps); break;
    case 4: dispatch_mt<4>(mt, st, grid, smem, n, T, nu_eff, n_obs, cvs, mps, P->eps.p, W, Up, S.p, CV, ldcv, stride, Ypart.p, ldys, Qcap, n_caps); break;
    default: dispatch_mt<0>(mt, st, grid, smem, n, T, nu_eff, n_obs, cvs, mps, P->eps.p, W, Up, S.p, CV, ldcv, stride, Ypart.p, ldys, Qcap, n_caps); break;
  }
  if (Y && P->n_obs > 0 && n_caps > 0) {
    int64_t tot = n_caps * n_obs;
    td2_reduce_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(
        n_caps, n_obs, nsplit, ldys, Ypart.p, n_pd, dld, Dp, P->n_obs, dtab, stride, Y);
    EM_LAUNCHED();
  }
}


void td2_run(em_td2_plan* P, int64_t T, const double* drive, double* q, double* Y,
             int64_t stride, double* Qcap) {
  cudaStream_t st = P->ctx->stream;
  const int n_u = P->n_u, n_c = P->n_p + P->n_s;
  if (T <= 0 || P->n <= 0) return;
  if (stride < 1) throw ArgError{"capture stride must be >= 1"};
  DBuf U((size_t)T * imax64(n_u, 1), st);
  if (n_u > 0) {
    td2_inputs_kernel<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(T, P->n_p, P->n_s, drive, U.p);
    EM_LAUNCHED();
  }
  td2_core(P, T, n_u, P->W.p, n_u > 0 ? U.p : nullptr, q, Y, stride, Qcap,
           P->D.n ? P->D.p : nullptr, P->n_p, drive, n_c);
}

// Inputs of one drive channel alone: a port p gives u^k = [i_d,p(t_k), di_d,p], a source
// s gives [di_0,s, 0] (the second weight column is zero).
__global__ void td2_channel_inputs_kernel(int64_t T, int n_c, int col, bool port,
                                          const double* __restrict__ drive,
                                          double* __restrict__ U) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= T) return;
  const double d0 = drive[k * n_c + col], d1 = drive[(k + 1) * n_c + col];
  U[2 * k] = port ? d0 : d1 - d0;
  U[2 * k + 1] = port ? d1 - d0 : 0.0;
}

void td2_run_sweep(em_td2_plan* P, int64_t T, const double* drive, double* Q, double* Y,
                   int64_t stride) {
  cudaStream_t st = P->ctx->stream;
  const int64_t n = P->n;
  const int n_p = P->n_p, n_c = P->n_p + P->n_s;
  if (T <= 0 || n <= 0 || n_c == 0) return;
  if (stride < 1) throw ArgError{"capture stride must be >= 1"};
  const int64_t n_caps = T / stride;
  const int n_obs = (Y && P->n_obs > 0) ? P->n_obs : 0;
  DBuf U((size_t)T * 2, st), Wc((size_t)n * 2, st);
  for (int c = 0; c < n_c; ++c) {
    const bool port = c < n_p;
    // weight columns of this channel (W = [P_r-part | P_ltr-part | P_m-part] / den)
    if (port) {
      EM_CK(cudaMemcpyAsync(Wc.p, P->W.p + (size_t)c * n, n * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
      EM_CK(cudaMemcpyAsync(Wc.p + n, P->W.p + (size_t)(n_p + c) * n, n * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
    } else {
      EM_CK(cudaMemcpyAsync(Wc.p, P->W.p + (size_t)(2 * n_p + (c - n_p)) * n,
                            n * sizeof(double), cudaMemcpyDeviceToDevice, st));
      EM_CK(cudaMemsetAsync(Wc.p + n, 0, n * sizeof(double), st));
    }
    td2_channel_inputs_kernel<<<(unsigned)((T + 255) / 256), 256, 0, st>>>(T, n_c, c, port,
                                                                         drive, U.p);
    EM_LAUNCHED();
    const double* Dc = (port && P->D.n) ? P->D.p + (size_t)c * P->n_obs : nullptr;
    td2_core(P, T, 2, Wc.p, U.p, Q + (size_t)c * n, n_obs ? Y + (size_t)c * n_caps * n_obs : nullptr,
             stride, nullptr, Dc, Dc ? 1 : 0, drive + c, n_c);
  }
}

void td2_plan_init(em_td2_plan* P, const double* l_n, const double* r_n, const double* P_r,
                   const double* P_l, const double* P_m) {
  cudaStream_t st = P->ctx->stream;
  const int64_t n = P->n;
  P->eps.alloc(n, st);
  P->binv.alloc(n, st);
  P->rn.alloc(n, st);
  P->cn.alloc(n, st);
  P->W.alloc((size_t)n * imax64(P->n_u, 1), st);
  P->Pr.alloc((size_t)n * imax64(P->n_p, 1), st);
  P->Pltr.alloc((size_t)n * imax64(P->n_p, 1), st);
  P->Pm.alloc((size_t)n * imax64(P->n_s, 1), st);
  td2_coeffs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      n, P->n_p, P->n_s, P->dt, P->theta, l_n, r_n, P_r, P_l, P_m, P->eps.p, P->binv.p, P->W.p,
      P->rn.p, P->cn.p, P->Pr.p, P->Pltr.p, P->Pm.p);
  EM_LAUNCHED();
}

void td2_plan_init_exact(em_td2_plan* P, const double* l_n, const double* r_n, const double* P_r,
                         const double* P_l, const double* P_m) {
  cudaStream_t st = P->ctx->stream;
  const int64_t n = P->n;
  P->exact = true;
  P->eps.alloc(n, st);
  P->W.alloc((size_t)n * imax64(P->n_u, 1), st);
  td2_exact_coeffs_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      n, P->n_p, P->n_s, P->dt, l_n, r_n, P_r, P_l, P_m, P->eps.p, P->W.p);
  EM_LAUNCHED();
}

bool td2_is_exact(const em_td2_plan* P) { return P->exact; }

void td2_set_observables(em_td2_plan* P, int n_obs, const double* CV, int64_t ldcv,
                         const double* D, int64_t ldd) {
  cudaStream_t st = P->ctx->stream;
  P->n_obs = n_obs;
  P->n_obs_pad = n_obs;  // CV stored densely with ld = n_obs
  P->CV.alloc((size_t)n_obs * P->n, st);
  copy_matrix(st, false, n_obs, P->n, CV, ldcv, P->CV.p, n_obs);
  if (D && P->n_p > 0) {
    P->D.alloc((size_t)n_obs * P->n_p, st);
    copy_matrix(st, false, n_obs, P->n_p, D, ldd, P->D.p, n_obs);
  } else {
    P->D.release();
  }
}

void td2_step(em_td2_plan* P, double* q, const double* u_dev) {
  cudaStream_t st = P->ctx->stream;
  td2_step_kernel<<<(unsigned)((P->n + 255) / 256), 256, 0, st>>>(
      P->n, P->n_p, P->n_s, P->dt, P->Pr.p, P->Pltr.p, P->Pm.p, P->rn.p, P->cn.p, u_dev, q);
  EM_LAUNCHED();
}

}  // namespace em

namespace em {

em_td2_plan* td2_new(em_ctx* ctx, int64_t n, int n_p, int n_s, double dt, double theta) {
  auto* P = new em_td2_plan();
  P->ctx = ctx;
  P->n = n;
  P->n_p = n_p;
  P->n_s = n_s;
  P->n_u = 2 * n_p + n_s;
  P->dt = dt;
  P->theta = theta;
  return P;
}
void td2_delete(em_td2_plan* p) {
  if (!p) return;
  cudaSetDevice(p->ctx->device);
  cudaStreamSynchronize(p->ctx->stream);
  delete p;
}
em_ctx* td2_ctx(em_td2_plan* p) { return p ? p->ctx : nullptr; }

// f = -dt P_r i_d - P_ltr di_d - P_m di0 (Td2Stepper.forcing, transient.py:147-155)
__global__ void td2_forcing_kernel(int64_t n, int n_p, int n_s, double dt,
                                   const double* __restrict__ Pr, const double* __restrict__ Pltr,
                                   const double* __restrict__ Pm, const double* __restrict__ u,
                                   double* __restrict__ f) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = 0.0;
  if (n_p) {
    double s = 0.0;
    for (int p = 0; p < n_p; ++p) s += Pr[i + p * n] * u[p];
    v -= dt * s;
    s = 0.0;
    for (int p = 0; p < n_p; ++p) s += Pltr[i + p * n] * u[n_p + p];
    v -= s;
  }
  if (n_s) {
    double s = 0.0;
    for (int k = 0; k < n_s; ++k) s += Pm[i + k * n] * u[2 * n_p + k];
    v -= s;
  }
  f[i] = v;
}

// q += ((-dt r q + f)/c)/c  (td2_step_kernel, _kernels.py:213-222)
__global__ void td2_step_forcing_kernel(int64_t n, double dt, const double* __restrict__ rn,
                                        const double* __restrict__ cn,
                                        const double* __restrict__ f, double* __restrict__ q) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = rn[i] * q[i];
  const double num = -dt * s + f[i];
  q[i] += (num / cn[i]) / cn[i];
}

static void upload_u(em_td2_plan* P, DBuf& du, const double* i_d, const double* di_d,
                     const double* di0) {
  std::vector<double> u((size_t)imax64(P->n_u, 1), 0.0);
  for (int p = 0; p < P->n_p; ++p) {
    u[p] = i_d[p];
    u[P->n_p + p] = di_d[p];
  }
  for (int s = 0; s < P->n_s; ++s) u[2 * P->n_p + s] = di0[s];
  du.alloc(u.size(), P->ctx->stream);
  EM_CK(cudaMemcpyAsync(du.p, u.data(), u.size() * sizeof(double), cudaMemcpyHostToDevice,
                        P->ctx->stream));
  EM_CK(cudaStreamSynchronize(P->ctx->stream));  // u is a host temporary
}

void td2_forcing_host(em_td2_plan* P, const double* i_d, const double* di_d, const double* di0,
                      double* f) {
  DBuf du;
  upload_u(P, du, i_d, di_d, di0);
  td2_forcing_kernel<<<(unsigned)((P->n + 255) / 256), 256, 0, P->ctx->stream>>>(
      P->n, P->n_p, P->n_s, P->dt, P->Pr.p, P->Pltr.p, P->Pm.p, du.p, f);
  EM_LAUNCHED();
  EM_CK(cudaStreamSynchronize(P->ctx->stream));
}

void td2_step_forcing(em_td2_plan* P, double* q, const double* f) {
  td2_step_forcing_kernel<<<(unsigned)((P->n + 255) / 256), 256, 0, P->ctx->stream>>>(
      P->n, P->dt, P->rn.p, P->cn.p, f, q);
  EM_LAUNCHED();
}

void td2_step_host(em_td2_plan* P, double* q, const double* i_d, const double* di_d,
                   const double* di0) {
  cudaStream_t st = P->ctx->stream;
  std::vector<double> u((size_t)imax64(P->n_u, 1), 0.0);
  for (int p = 0; p < P->n_p; ++p) {
    u[p] = i_d[p];
    u[P->n_p + p] = di_d[p];
  }
  for (int s = 0; s < P->n_s; ++s) u[2 * P->n_p + s] = di0[s];
  DBuf du(u.size(), st);
  EM_CK(cudaMemcpyAsync(du.p, u.data(), u.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  td2_step(P, q, du.p);
  EM_CK(cudaStreamSynchronize(st));
}

}  // namespace em
