/*
 * CPU ORACLE — test infrastructure only, never the product path.
 *
 * Plain-C restatement of the reference's compiled numerics
 * (pkg/src/eddymodes/_kernels.py, numba @njit, fastmath off). Sequential
 * scalar loops over C-contiguous row-major float64 arrays, in the same
 * operation order as the reference so that results agree bit for bit when
 * compiled with strict IEEE semantics (-O2 -ffp-contract=off, no fast-math).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.
 */
#include <math.h>
#include <stdint.h>

#define A_(i, j) a[(int64_t)(i) * n + (j)]
#define C_(i, j) c[(int64_t)(i) * n + (j)]

/* _kernels.py:18-36  cholesky_kernel: lower Cholesky-Crout; -1 on success,
 * else the first index whose pivot is not > 0. */
int64_t orc_cholesky(const double* a, double* c, int64_t n) {
  for (int64_t j = 0; j < n; ++j) {
    double s = A_(j, j);
    for (int64_t k = 0; k < j; ++k) s -= C_(j, k) * C_(j, k);
    if (!(s > 0.0)) return j;
    double cjj = sqrt(s);
    C_(j, j) = cjj;
    for (int64_t i = j + 1; i < n; ++i) {
      double t = A_(i, j);
      for (int64_t k = 0; k < j; ++k) t -= C_(i, k) * C_(j, k);
      C_(i, j) = t / cjj;
    }
  }
  return -1;
}

/* _kernels.py:39-53  tri_solve_vec: (C C^T) x = b, forward then backward. */
void orc_tri_solve_vec(const double* c, const double* b, double* y, double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double s = b[i];
    for (int64_t k = 0; k < i; ++k) s -= C_(i, k) * y[k];
    y[i] = s / C_(i, i);
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int64_t k = i + 1; k < n; ++k) s -= C_(k, i) * x[k];
    x[i] = s / C_(i, i);
  }
}

/* _kernels.py:56-66  tri_lower_solve_mat: b <- C^-1 b (b is n x m row-major). */
void orc_tri_lower_solve_mat(const double* c, double* b, int64_t n, int64_t m) {
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = 0; i < n; ++i) {
      double s = b[i * m + j];
      for (int64_t k = 0; k < i; ++k) s -= C_(i, k) * b[k * m + j];
      b[i * m + j] = s / C_(i, i);
    }
}

/* _kernels.py:69-79  tri_lower_t_solve_mat: b <- C^-T b. */
void orc_tri_lower_t_solve_mat(const double* c, double* b, int64_t n, int64_t m) {
  for (int64_t j = 0; j < m; ++j)
    for (int64_t i = n - 1; i >= 0; --i) {
      double s = b[i * m + j];
      for (int64_t k = i + 1; k < n; ++k) s -= C_(k, i) * b[k * m + j];
      b[i * m + j] = s / C_(i, i);
    }
}

/* _kernels.py:82-141  jacobi_sym_eig: cyclic Jacobi; returns sweeps or -1. */
int64_t orc_jacobi(double* a, double* v, int64_t n, int64_t max_sweeps, double tol_rel) {
  double fro = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) fro += A_(i, j) * A_(i, j);
  fro = sqrt(fro);
  if (fro == 0.0) return 0;
  double thresh = tol_rel * fro;
  for (int64_t sweep = 0; sweep < max_sweeps; ++sweep) {
    double off = 0.0;
    for (int64_t i = 0; i < n; ++i)
      for (int64_t j = i + 1; j < n; ++j) off += A_(i, j) * A_(i, j);
    if (sqrt(2.0 * off) <= thresh) return sweep;
    for (int64_t p = 0; p < n - 1; ++p)
      for (int64_t q = p + 1; q < n; ++q) {
        double apq = A_(p, q);
        if (apq == 0.0) continue;
        double tau = (A_(q, q) - A_(p, p)) / (2.0 * apq);
        double t;
        if (tau >= 0.0)
          t = 1.0 / (tau + sqrt(1.0 + tau * tau));
        else
          t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
        double cth = 1.0 / sqrt(1.0 + t * t);
        double sth = t * cth;
        for (int64_t k = 0; k < n; ++k) {
          double akp = A_(k, p), akq = A_(k, q);
          A_(k, p) = cth * akp - sth * akq;
          A_(k, q) = sth * akp + cth * akq;
        }
        for (int64_t k = 0; k < n; ++k) {
          double apk = A_(p, k), aqk = A_(q, k);
          A_(p, k) = cth * apk - sth * aqk;
          A_(q, k) = sth * apk + cth * aqk;
        }
        A_(p, q) = 0.0;
        A_(q, p) = 0.0;
        for (int64_t k = 0; k < n; ++k) {
          double vkp = v[k * n + p], vkq = v[k * n + q];
          v[k * n + p] = cth * vkp - sth * vkq;
          v[k * n + q] = sth * vkp + cth * vkq;
        }
      }
  }
  double off = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = i + 1; j < n; ++j) off += A_(i, j) * A_(i, j);
  if (sqrt(2.0 * off) <= thresh) return max_sweeps;
  return -1;
}

/* Timing sample of jacobi_sym_eig: the first `count` rotations of sweep 1 in the
 * reference's cyclic order (same loop body as orc_jacobi). Used only by bench.py's
 * CPU baseline to measure the per-rotation cost at large n, where a full solve
 * would take days; returns the number of rotations performed. */
int64_t orc_jacobi_rotations(double* a, double* v, int64_t n, int64_t count) {
  int64_t done = 0;
  for (int64_t p = 0; p < n - 1 && done < count; ++p)
    for (int64_t q = p + 1; q < n && done < count; ++q) {
      double apq = A_(p, q);
      ++done;
      if (apq == 0.0) continue;
      double tau = (A_(q, q) - A_(p, p)) / (2.0 * apq);
      double t;
      if (tau >= 0.0)
        t = 1.0 / (tau + sqrt(1.0 + tau * tau));
      else
        t = -1.0 / (-tau + sqrt(1.0 + tau * tau));
      double cth = 1.0 / sqrt(1.0 + t * t);
      double sth = t * cth;
      for (int64_t k = 0; k < n; ++k) {
        double akp = A_(k, p), akq = A_(k, q);
        A_(k, p) = cth * akp - sth * akq;
        A_(k, q) = sth * akp + cth * akq;
      }
      for (int64_t k = 0; k < n; ++k) {
        double apk = A_(p, k), aqk = A_(q, k);
        A_(p, k) = cth * apk - sth * aqk;
        A_(q, k) = sth * apk + cth * aqk;
      }
      A_(p, q) = 0.0;
      A_(q, p) = 0.0;
      for (int64_t k = 0; k < n; ++k) {
        double vkp = v[k * n + p], vkq = v[k * n + q];
        v[k * n + p] = cth * vkp - sth * vkq;
        v[k * n + q] = sth * vkp + cth * vkq;
      }
    }
  return done;
}

/* _kernels.py:198-210  td1_step_kernel. b, y, x are scratch of length n. */
void orc_td1_step(const double* c, const double* r, double* state, double dt, const double* extra,
                  double* b, double* y, double* x, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s += r[i * n + k] * state[k];
    b[i] = -dt * s + extra[i];
  }
  orc_tri_solve_vec(c, b, y, x, n);
  for (int64_t i = 0; i < n; ++i) state[i] += x[i];
}

/* _kernels.py:213-222  td2_step_kernel. */
void orc_td2_step(double* state, const double* r_n, const double* c_n, double dt,
                  const double* forcing, int64_t n) {
  for (int64_t i = 0; i < n; ++i) {
    double s = r_n[i] * state[i];
    double num = -dt * s + forcing[i];
    state[i] += (num / c_n[i]) / c_n[i];
  }
}

/* _kernels.py:144-170  lu_factor_kernel: in-place LU with partial pivoting (row swaps
 * recorded in piv); -1 on success, else the column with an exactly zero pivot. */
int64_t orc_lu_factor(double* a, int64_t* piv, int64_t n) {
  for (int64_t k = 0; k < n; ++k) {
    double pmax = fabs(A_(k, k));
    int64_t prow = k;
    for (int64_t i = k + 1; i < n; ++i) {
      const double v = fabs(A_(i, k));
      if (v > pmax) {
        pmax = v;
        prow = i;
      }
    }
    if (pmax == 0.0) return k;
    piv[k] = prow;
    if (prow != k)
      for (int64_t j = 0; j < n; ++j) {
        const double tmp = A_(k, j);
        A_(k, j) = A_(prow, j);
        A_(prow, j) = tmp;
      }
    const double akk = A_(k, k);
    for (int64_t i = k + 1; i < n; ++i) {
      const double lik = A_(i, k) / akk;
      A_(i, k) = lik;
      for (int64_t j = k + 1; j < n; ++j) A_(i, j) -= lik * A_(k, j);
    }
  }
  return -1;
}

/* _kernels.py:173-193  lu_solve_kernel: all row swaps first, then the two sweeps. */
void orc_lu_solve(const double* a, const int64_t* piv, double* b, int64_t n) {
  for (int64_t k = 0; k < n; ++k) {
    const int64_t p = piv[k];
    if (p != k) {
      const double tmp = b[k];
      b[k] = b[p];
      b[p] = tmp;
    }
  }
  for (int64_t k = 0; k < n; ++k)
    for (int64_t i = k + 1; i < n; ++i) b[i] -= A_(i, k) * b[k];
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int64_t k = i + 1; k < n; ++k) s -= A_(i, k) * b[k];
    b[i] = s / A_(i, i);
  }
}

/* run_transient's td2 loop (transient.py:293-306) over Td2Stepper.forcing
 * (transient.py:147-155) and td2_step_kernel (_kernels.py:213-222), driven by a sample
 * table tab ((steps+1) x (n_p+n_s), row k = [i_d(t_k) | i0(t_k)]). p_r, p_ltr: n x n_p,
 * p_m: n x n_s row-major (= V^T R_D, V^T L_D + dt theta V^T R_D, V^T M0). Observables
 * obs[cap][o] = (C V q)_o with cv (n_obs x n row-major) after every stride-th step;
 * q (n) in/out; f is scratch of length n. The forcing is accumulated in the reference's
 * order: f = 0; f -= dt (P_r i_d); f -= P_ltr di_d; f -= P_m di0 (numpy matvec sums in
 * channel order, exact for one channel). */
void orc_td2_run(double* q, const double* r_n, const double* c_n, double dt, const double* p_r,
                 const double* p_ltr, const double* p_m, int64_t n, int64_t n_p, int64_t n_s,
                 const double* tab, int64_t steps, const double* cv, int64_t n_obs,
                 int64_t stride, double* obs, double* f) {
  const int64_t nc = n_p + n_s;
  int64_t cap = 0;
  for (int64_t k = 0; k < steps; ++k) {
    const double* t0 = tab + k * nc;
    const double* t1 = t0 + nc;
    for (int64_t i = 0; i < n; ++i) {
      double fi = 0.0;
      if (n_p) {
        double s = 0.0;
        for (int64_t p = 0; p < n_p; ++p) s += p_r[i * n_p + p] * t0[p];
        fi -= dt * s;
        s = 0.0;
        for (int64_t p = 0; p < n_p; ++p) s += p_ltr[i * n_p + p] * (t1[p] - t0[p]);
        fi -= s;
      }
      if (n_s) {
        double s = 0.0;
        for (int64_t j = 0; j < n_s; ++j) s += p_m[i * n_s + j] * (t1[n_p + j] - t0[n_p + j]);
        fi -= s;
      }
      f[i] = fi;
    }
    orc_td2_step(q, r_n, c_n, dt, f, n);
    if ((k + 1) % stride == 0) {
      if (obs)
        for (int64_t o = 0; o < n_obs; ++o) {
          double s = 0.0;
          for (int64_t i = 0; i < n; ++i) s += cv[o * n + i] * q[i];
          obs[cap * n_obs + o] = s;
        }
      ++cap;
    }
  }
}
