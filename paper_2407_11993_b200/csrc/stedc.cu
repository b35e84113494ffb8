// Symmetric tridiagonal eigensolver: Cuppen divide and conquer with
// Gu-Eisenstat eigenvectors, batched level by level on the GPU.
//
//   leaves (<= 64)   implicit-shift QL, one CTA per leaf, one thread per row
//   merge            z = [last row of Q1, sign(b) first row of Q2]/sqrt(2), rho = 2|b|;
//                    deflation (small z, close poles + Givens), secular equation
//                    per root (one thread each, two-pole rational iteration with a
//                    bisection safeguard, roots stored as pole + offset for
//                    full relative accuracy), z-hat recomputed from the roots
//                    (Gu-Eisenstat) so the vectors are orthogonal, and
//                    Q_new = [Q1 0; 0 Q2] U on the DMMA grouped GEMM.
// This is the eigensolver stage that replaces the reference's cyclic Jacobi
// (_kernels.py:82-141, linalg.py:119-134).
#include <algorithm>
#include <vector>

#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

constexpr int LEAF = 64;

// ---- leaves ---------------------------------------------------------------------

// One CTA (LEAF threads) per leaf. Every thread runs the same scalar QL iteration
// on private copies of d/e and applies each rotation to its own row of Z.
__global__ void __launch_bounds__(LEAF) dc_leaf_kernel(const int64_t* __restrict__ loff,
                                                       const int* __restrict__ lsz,
                                                       const double* __restrict__ d0,
                                                       const double* __restrict__ e0, double* lam,
                                                       double* Q, int64_t ldq) {
  const int64_t off = loff[blockIdx.x];
  const int n = lsz[blockIdx.x];
  const int row = threadIdx.x;
  double d[LEAF], e[LEAF], z[LEAF];
  for (int i = 0; i < n; ++i) {
    d[i] = d0[off + i];
    e[i] = (i < n - 1) ? e0[off + i] : 0.0;
    z[i] = (i == row) ? 1.0 : 0.0;
  }
  const double eps = 2.220446049250313e-16;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (++iter > 60) break;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool underflow = false;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            underflow = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          if (row < n) {
            f = z[i + 1];
            z[i + 1] = s * z[i] + c * f;
            z[i] = c * z[i] - s * f;
          }
        }
        if (underflow && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  // ascending selection sort (identical in every thread), permuting this row
  for (int i = 0; i < n - 1; ++i) {
    int k = i;
    double p = d[i];
    for (int j = i + 1; j < n; ++j)
      if (d[j] < p) {
        k = j;
        p = d[j];
      }
    if (k != i) {
      d[k] = d[i];
      d[i] = p;
      const double t = z[i];
      z[i] = z[k];
      z[k] = t;
    }
  }
  if (row < n) {
    for (int j = 0; j < n; ++j) Q[(off + row) + (off + j) * ldq] = z[j];
    if (row == 0)
      for (int j = 0; j < n; ++j) lam[off + j] = d[j];
  }
}

// ---- merge: deflation -----------------------------------------------------------

struct MergeInfo {  // per merge, written by dc_deflate
  int K, c1, c2, c3, nrot;
};

// Workspace arrays indexed by the block offset (disjoint ranges per merge):
//   dlam, wz: non-deflated poles/weights (ascending), K entries
//   src:      block-local source column of each non-deflated entry
//   pos:      type-grouped position of each non-deflated entry
//   dval/dcol: deflated values (ascending) / block-local columns
//   rot_a/rot_b/rot_c/rot_s: Givens rotations in application order
struct DcWork {
  double *dlam, *wz, *dval, *rot_c, *rot_s, *mu, *zhat, *lamn, *sortd, *sortz;
  int *src, *pos, *dcol, *rot_a, *rot_b, *org, *typ, *perm;
};

__global__ void dc_deflate_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn1,
                                  const int* __restrict__ mn, const double* __restrict__ ebeta,
                                  const double* __restrict__ lam, const double* __restrict__ Q,
                                  int64_t ldq, DcWork w, double* rho_out, MergeInfo* info,
                                  const double* __restrict__ xf = nullptr,
                                  const double* __restrict__ xl = nullptr) {
  const int64_t off = moff[blockIdx.x];
  const int n1 = mn1[blockIdx.x], n = mn[blockIdx.x];
  const double beta = ebeta[blockIdx.x];
  double* z = w.sortz + off;   // scratch (block-local index)
  double* D = w.sortd + off;
  int* perm = w.perm + off;
  const double isq2 = 0.70710678118654752440;
  // z in block-local column order
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double v;
    if (xf)  // implicit form: the children's last / first eigenvector rows are X columns
      v = j < n1 ? xl[off + j] : xf[off + j];
    else if (j < n1)
      v = Q[(off + n1 - 1) + (off + j) * ldq];
    else
      v = Q[(off + n1) + (off + j) * ldq];
    if (j >= n1 && beta < 0.0) v = -v;
    w.zhat[off + j] = v * isq2;  // zhat used as scratch for raw z here
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  const double rho = 2.0 * fabs(beta);
  rho_out[blockIdx.x] = rho;
  const double* zr = w.zhat + off;
  // merge the two ascending halves
  {
    int a = 0, b = n1, k = 0;
    while (a < n1 || b < n) {
      int take;
      if (a >= n1)
        take = b++;
      else if (b >= n)
        take = a++;
      else if (lam[off + b] < lam[off + a])
        take = b++;
      else
        take = a++;
      perm[k] = take;
      D[k] = lam[off + take];
      z[k] = zr[take];
      ++k;
    }
  }
  double dmax = 0.0, zmax = 0.0;
  for (int k = 0; k < n; ++k) {
    dmax = fmax(dmax, fabs(D[k]));
    zmax = fmax(zmax, fabs(z[k]));
  }
  const double eps = 1.1102230246251565e-16;  // LAPACK dlamch('E') (half ulp)
  const double tol = 8.0 * eps * fmax(dmax, zmax);
  int K = 0, nd = 0, nrot = 0;
  int* typ = w.typ + off;  // per sorted entry: 1 top, 2 mixed, 3 bottom
  for (int k = 0; k < n; ++k) typ[k] = perm[k] < n1 ? 1 : 3;
  auto push_defl = [&](double val, int col) {
    // insertion keeps the deflated list ascending
    int p = nd++;
    while (p > 0 && w.dval[off + p - 1] > val) {
      w.dval[off + p] = w.dval[off + p - 1];
      w.dcol[off + p] = w.dcol[off + p - 1];
      --p;
    }
    w.dval[off + p] = val;
    w.dcol[off + p] = col;
  };
  if (rho * zmax <= tol) {
    for (int k = 0; k < n; ++k) push_defl(D[k], perm[k]);
  } else {
    int pj = -1;
    for (int k = 0; k < n; ++k) {
      if (rho * fabs(z[k]) <= tol) {
        push_defl(D[k], perm[k]);
        continue;
      }
      if (pj < 0) {
        pj = k;
        continue;
      }
      double s = z[pj], c = z[k];
      const double tau = hypot(c, s);
      const double t = D[k] - D[pj];
      c /= tau;
      s = -s / tau;
      if (fabs(t * c * s) <= tol) {
        z[k] = tau;
        z[pj] = 0.0;
        if (typ[k] != typ[pj]) typ[k] = 2;
        w.rot_a[off + nrot] = perm[pj];
        w.rot_b[off + nrot] = perm[k];
        w.rot_c[off + nrot] = c;
        w.rot_s[off + nrot] = s;
        ++nrot;
        const double tp = D[pj] * c * c + D[k] * s * s;
        D[k] = D[pj] * s * s + D[k] * c * c;
        D[pj] = tp;
        push_defl(tp, perm[pj]);
        pj = k;
      } else {
        w.dlam[off + K] = D[pj];
        w.wz[off + K] = z[pj];
        w.src[off + K] = perm[pj];
        w.org[off + K] = typ[pj];  // temporarily the type
        ++K;
        pj = k;
      }
    }
    if (pj >= 0) {
      w.dlam[off + K] = D[pj];
      w.wz[off + K] = z[pj];
      w.src[off + K] = perm[pj];
      w.org[off + K] = typ[pj];
      ++K;
    }
  }
  // type-grouped positions (1, then 2, then 3; stable)
  int c1 = 0, c2 = 0, c3 = 0;
  for (int k = 0; k < K; ++k) {
    const int t = w.org[off + k];
    c1 += t == 1;
    c2 += t == 2;
    c3 += t == 3;
  }
  int p1 = 0, p2 = c1, p3 = c1 + c2;
  for (int k = 0; k < K; ++k) {
    const int t = w.org[off + k];
    w.pos[off + k] = t == 1 ? p1++ : (t == 2 ? p2++ : p3++);
  }
  info[blockIdx.x] = MergeInfo{K, c1, c2, c3, nrot};
}

// ---- merge: rotations, secular equation, z-hat, U ---------------------------------

// Apply the deflation rotations to the block columns (every row of the block).
__global__ void dc_rotate_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn,
                                 const MergeInfo* __restrict__ info, DcWork w, double* Q,
                                 int64_t ldq) {
  const int mi = blockIdx.y;
  const int64_t off = moff[mi];
  const int n = mn[mi];
  const int nrot = info[mi].nrot;
  if (nrot == 0) return;
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    double* row = Q + (off + r);
    for (int q = 0; q < nrot; ++q) {
      const int a = w.rot_a[off + q], b = w.rot_b[off + q];
      const double c = w.rot_c[off + q], s = w.rot_s[off + q];
      const double x = row[(off + a) * ldq], y = row[(off + b) * ldq];
      row[(off + a) * ldq] = c * x + s * y;
      row[(off + b) * ldq] = c * y - s * x;
    }
  }
}

// Secular equation 1 + rho sum_j z_j^2/(d_j - lambda) = 0, root i (0-based) of K.
// Returns the origin pole index and mu with lambda = d[org] + mu.
EM_DEVINL void secular_root(int K, const double* __restrict__ d, const double* __restrict__ z,
                            double rho, int i, int& org, double& mu) {
  const double eps = 2.220446049250313e-16;
  double lo, hi;
  if (i < K - 1) {
    const double gap = d[i + 1] - d[i];
    const double mid = 0.5 * gap;
    double f = 1.0;
    for (int j = 0; j < K; ++j) f += rho * z[j] * z[j] / ((d[j] - d[i]) - mid);
    if (f >= 0.0) {
      org = i;
      lo = 0.0;
      hi = mid;
    } else {
      org = i + 1;
      lo = -mid;
      hi = 0.0;
    }
  } else {
    double zz = 0.0;
    for (int j = 0; j < K; ++j) zz += z[j] * z[j];
    org = K - 1;
    lo = 0.0;
    hi = rho * zz;
  }
  const double dorg = d[org];
  // initial guess: bracket midpoint
  double m = 0.5 * (lo + hi);
  if (m == 0.0) m = (org == i) ? hi * 0.5 : lo * 0.5;
  for (int it = 0; it < 200; ++it) {
    double f = 1.0, dpsi = 0.0, dphi = 0.0, eabs = 0.0;
    for (int j = 0; j < K; ++j) {
      const double del = (d[j] - dorg) - m;
      const double t = z[j] / del;
      const double term = rho * z[j] * t;
      f += term;
      eabs += fabs(term);
      const double der = rho * t * t;
      if (j <= i)
        dpsi += der;
      else
        dphi += der;
    }
    if (f == 0.0) break;
    if (f < 0.0)
      lo = m;
    else
      hi = m;
    if (fabs(f) <= eps * (8.0 * eabs + 2.0)) break;
    if (hi - lo <= 4.0 * eps * fmax(fabs(lo), fabs(hi))) break;
    // two-pole rational model through the neighbouring poles
    const double dL = (d[i] - dorg) - m;
    double mn;
    if (i < K - 1) {
      const double dR = (d[i + 1] - dorg) - m;
      const double sL = dL * dL * dpsi, sR = dR * dR * dphi;
      const double c = f - sL / dL - sR / dR;
      const double a2 = c, a1 = -(c * (dL + dR) + sL + sR), a0 = c * dL * dR + sL * dR + sR * dL;
      double eta;
      if (fabs(a2) <= 1e-300 * (fabs(a1) + fabs(a0))) {
        eta = -a0 / a1;
      } else {
        const double disc = fmax(a1 * a1 - 4.0 * a2 * a0, 0.0);
        const double q = -0.5 * (a1 + copysign(sqrt(disc), a1));
        const double e1 = q / a2, e2 = (q != 0.0) ? a0 / q : e1;
        eta = (e1 > dL && e1 < dR) ? e1 : e2;
      }
      mn = m + eta;
    } else {
      const double sL = dL * dL * dpsi;
      const double c = f - sL / dL;
      mn = (c > 0.0) ? m + (dL + sL / c) : 0.5 * (lo + hi);
    }
    if (!(mn > lo && mn < hi)) mn = 0.5 * (lo + hi);
    if (mn == m) break;
    m = mn;
  }
  mu = m;
}

__global__ void dc_secular_kernel(const int64_t* __restrict__ moff,
                                  const MergeInfo* __restrict__ info,
                                  const double* __restrict__ rho, DcWork w) {
  const int mi = blockIdx.y;
  const int64_t off = moff[mi];
  const int K = info[mi].K;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  int org;
  double mu;
  secular_root(K, w.dlam + off, w.wz + off, rho[mi], i, org, mu);
  w.org[off + i] = org;
  w.mu[off + i] = mu;
  w.lamn[off + i] = w.dlam[off + org] + mu;
}

// zhat_i = sign(z_i) sqrt(-W_i), W_i = (d_i - l_i) prod_{j!=i} (d_i - l_j)/(d_i - d_j)
__global__ void dc_zhat_kernel(const int64_t* __restrict__ moff, const MergeInfo* __restrict__ info,
                               DcWork w) {
  const int mi = blockIdx.y;
  const int64_t off = moff[mi];
  const int K = info[mi].K;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= K) return;
  const double* d = w.dlam + off;
  const double di = d[i];
  double W = (di - d[w.org[off + i]]) - w.mu[off + i];
  for (int j = 0; j < K; ++j) {
    if (j == i) continue;
    const double dij = (di - d[w.org[off + j]]) - w.mu[off + j];
    W *= dij / (di - d[j]);
  }
  w.zhat[off + i] = copysign(sqrt(fmax(-W, 0.0)), w.wz[off + i]);
}

// U(:, j) = (zhat_i / (d_i - l_j))_i normalised, written at type-grouped row positions.
// One warp per column.
__global__ void dc_umat_kernel(const int64_t* __restrict__ moff, const MergeInfo* __restrict__ info,
                               DcWork w, double* U, int64_t ldu) {
  const int mi = blockIdx.y;
  const int64_t off = moff[mi];
  const int K = info[mi].K;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= K) return;
  const double* d = w.dlam + off;
  const double dorg = d[w.org[off + j]], mu = w.mu[off + j];
  double ss = 0.0;
  for (int i = lane; i < K; i += 32) {
    const double v = w.zhat[off + i] / ((d[i] - dorg) - mu);
    ss = fma(v, v, ss);
  }
  ss = warp_sum(ss);
  const double inv = 1.0 / sqrt(ss);
  double* col = U + off + (off + j) * ldu;
  for (int i = lane; i < K; i += 32) {
    const double v = w.zhat[off + i] / ((d[i] - dorg) - mu);
    col[w.pos[off + i]] = v * inv;
  }
}

// Q2(:, pos(i)) = Q(:, src(i)) over the block rows
__global__ void dc_gather_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn,
                                 const MergeInfo* __restrict__ info, DcWork w,
                                 const double* __restrict__ Q, double* __restrict__ Q2,
                                 int64_t ldq) {
  const int mi = blockIdx.z;
  const int64_t off = moff[mi];
  const int n = mn[mi];
  const int K = info[mi].K;
  // non-deflated columns to their type-grouped GEMM positions 0..K-1, deflated ones
  // (in ascending-value order) behind them at K..n-1, so that Q is free for the GEMM
  // output afterwards
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    int64_t sc, dc;
    if (i < K) {
      sc = off + w.src[off + i];
      dc = off + w.pos[off + i];
    } else {
      sc = off + w.dcol[off + (i - K)];
      dc = off + i;
    }
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
      Q2[(off + r) + dc * ldq] = Q[(off + r) + sc * ldq];
  }
}

// Deflated columns K..n-1 back next to the GEMM output (same block-local columns).
__global__ void dc_copy_deflated_kernel(const int64_t* __restrict__ moff,
                                        const int* __restrict__ mn,
                                        const MergeInfo* __restrict__ info,
                                        const double* __restrict__ Q2, double* __restrict__ Q,
                                        int64_t ldq) {
  const int mi = blockIdx.z;
  const int64_t off = moff[mi];
  const int n = mn[mi];
  const int K = info[mi].K;
  for (int i = K + blockIdx.y; i < n; i += gridDim.y) {
    const int64_t c = off + i;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
      Q[(off + r) + c * ldq] = Q2[(off + r) + c * ldq];
  }
}

// Final ordering: merge new eigenvalues (ascending) with the deflated ones.
__global__ void dc_order_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn,
                                const MergeInfo* __restrict__ info, DcWork w, double* lam_out) {
  const int mi = blockIdx.x;
  const int64_t off = moff[mi];
  const int n = mn[mi];
  const int K = info[mi].K;
  if (threadIdx.x != 0) return;
  int a = 0, b = 0;
  for (int t = 0; t < n; ++t) {
    const bool take_new = (b >= n - K) || (a < K && w.lamn[off + a] <= w.dval[off + b]);
    if (take_new) {
      lam_out[off + t] = w.lamn[off + a];
      w.perm[off + t] = a;  // >= 0: new column a
      ++a;
    } else {
      lam_out[off + t] = w.dval[off + b];
      w.perm[off + t] = -1 - b;  // < 0: deflated entry b (column K + b after the gather)
      ++b;
    }
  }
}

// Qout column t <- Q column p (new eigenvector p) or K + b (deflated entry b).
__global__ void dc_place_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn,
                                const MergeInfo* __restrict__ info, DcWork w,
                                const double* __restrict__ Q, double* __restrict__ Qout,
                                int64_t ldq, int t0, int t1) {
  const int mi = blockIdx.z;
  const int64_t off = moff[mi];
  const int n = mn[mi];
  const int K = info[mi].K;
  if (t1 > n) t1 = n;
  for (int t = t0 + blockIdx.y; t < t1; t += gridDim.y) {
    const int p = w.perm[off + t];
    const double* src = Q + (off + ((p >= 0) ? p : K + (-1 - p))) * ldq;
    double* dst = Qout + (off + t) * ldq;
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
      dst[off + r] = src[off + r];
  }
}

__global__ void dc_tear_kernel(int nsplit, const int64_t* __restrict__ sp, double* d,
                               const double* __restrict__ e, double* beta) {
  int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nsplit) return;
  const int64_t s = sp[k];
  const double b = e[s - 1];
  beta[k] = b;
  d[s - 1] -= fabs(b);
  d[s] -= fabs(b);
}

__global__ void scale_vec_kernel(int64_t n, double* x, const double* __restrict__ factor,
                                 int invert) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double f = *factor;
  if (f == 0.0) return;
  x[i] = invert ? x[i] / f : x[i] * f;
}

__global__ void absmax_kernel(int64_t n, const double* d, const double* e, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    m = fmax(m, fabs(d[i]));
    if (i < n - 1) m = fmax(m, fabs(e[i]));
  }
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double r = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) r = fmax(r, red[k]);
    *out = r;
  }
}

// ---- implicit form: U^T Y without U --------------------------------------------------
//
// stedc_apply keeps, per tree node, X = U_node^T [Y_node | e_first | e_last] (n x (k + 2),
// column-major, ld n): the operand rows in the node's eigenbasis plus the node's first and
// last eigenvector rows, which are all a merge needs (z = [last row of U_1, first row of
// U_2]). A merge is U = [U_1 0; 0 U_2] G P U~ (deflation rotations G, permutation P,
// Cauchy-like secular eigenvectors U~), so X_new = U~^T P^T G^T [X_1; X_2]: rotations act
// on rows of X, and U~ (zhat_i / (d_i - lambda_j), normalised) is generated tile by tile
// inside the product and never stored. Memory O(n k) instead of the 3 n^2 of stedc.

// One CTA per leaf: the QL iteration as dc_leaf_kernel, then X = Q_leaf^T [Y | e_0 | e_last].
__global__ void __launch_bounds__(LEAF) dc_leaf_apply_kernel(
    const int64_t* __restrict__ loff, const int* __restrict__ lsz, const double* __restrict__ d0,
    const double* __restrict__ e0, double* lam, const double* __restrict__ Y, int64_t ldy, int k,
    double* __restrict__ X, int64_t ldx) {
  __shared__ double Qs[LEAF][LEAF + 1];
  __shared__ double ys[LEAF];
  const int64_t off = loff[blockIdx.x];
  const int n = lsz[blockIdx.x];
  const int row = threadIdx.x;
  double d[LEAF], e[LEAF], z[LEAF];
  for (int i = 0; i < n; ++i) {
    d[i] = d0[off + i];
    e[i] = (i < n - 1) ? e0[off + i] : 0.0;
    z[i] = (i == row) ? 1.0 : 0.0;
  }
  const double eps = 2.220446049250313e-16;
  for (int l = 0; l < n; ++l) {
    int iter = 0;
    int m;
    do {
      for (m = l; m < n - 1; ++m) {
        const double dd = fabs(d[m]) + fabs(d[m + 1]);
        if (fabs(e[m]) <= eps * dd) break;
      }
      if (m != l) {
        if (++iter > 60) break;
        double g = (d[l + 1] - d[l]) / (2.0 * e[l]);
        double r = hypot(g, 1.0);
        g = d[m] - d[l] + e[l] / (g + copysign(r, g));
        double s = 1.0, c = 1.0, p = 0.0;
        int i;
        bool underflow = false;
        for (i = m - 1; i >= l; --i) {
          double f = s * e[i];
          const double b = c * e[i];
          r = hypot(f, g);
          e[i + 1] = r;
          if (r == 0.0) {
            d[i + 1] -= p;
            e[m] = 0.0;
            underflow = true;
            break;
          }
          s = f / r;
          c = g / r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          f = z[i + 1];
          z[i + 1] = s * z[i] + c * f;
          z[i] = c * z[i] - s * f;
        }
        if (underflow && i >= l) continue;
        d[l] -= p;
        e[l] = g;
        e[m] = 0.0;
      }
    } while (m != l);
  }
  for (int i = 0; i < n - 1; ++i) {
    int kk = i;
    double p = d[i];
    for (int j = i + 1; j < n; ++j)
      if (d[j] < p) {
        kk = j;
        p = d[j];
      }
    if (kk != i) {
      d[kk] = d[i];
      d[i] = p;
      const double t = z[i];
      z[i] = z[kk];
      z[kk] = t;
    }
  }
  if (row < n)
    for (int j = 0; j < n; ++j) Qs[row][j] = z[j];
  if (row == 0)
    for (int j = 0; j < n; ++j) lam[off + j] = d[j];
  __syncthreads();
  for (int c = 0; c < k; ++c) {
    if (row < n) ys[row] = Y[(off + row) + c * ldy];
    __syncthreads();
    if (row < n) {
      double acc = 0.0;
      for (int r = 0; r < n; ++r) acc = fma(Qs[r][row], ys[r], acc);
      X[(off + row) + c * ldx] = acc;
    }
    __syncthreads();
  }
  if (row < n) {
    X[(off + row) + (int64_t)k * ldx] = Qs[0][row];
    X[(off + row) + (int64_t)(k + 1) * ldx] = Qs[n - 1][row];
  }
}

// Per merge, one thread per X column: keep only the left child's rows of the first-row
// column and the right child's rows of the last-row column, then the deflation rotations.
__global__ void dc_xrot_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn1,
                               const int* __restrict__ mn, const MergeInfo* __restrict__ info,
                               DcWork w, double* X, int64_t ldx, int ncol) {
  const int mi = blockIdx.y;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncol) return;
  const int64_t off = moff[mi];
  const int n1 = mn1[mi], n = mn[mi];
  double* col = X + off + (int64_t)c * ldx;
  if (c == ncol - 2)
    for (int r = n1; r < n; ++r) col[r] = 0.0;
  else if (c == ncol - 1)
    for (int r = 0; r < n1; ++r) col[r] = 0.0;
  const int nrot = info[mi].nrot;
  for (int q = 0; q < nrot; ++q) {
    const int a = w.rot_a[off + q], b = w.rot_b[off + q];
    const double cs = w.rot_c[off + q], sn = w.rot_s[off + q];
    const double x = col[a], y = col[b];
    col[a] = cs * x + sn * y;
    col[b] = cs * y - sn * x;
  }
}

// 1 / ||(zhat_i / (d_i - lambda_j))_i|| per secular root j (into w.sortd), one warp each
__global__ void dc_unorm_kernel(const int64_t* __restrict__ moff,
                                const MergeInfo* __restrict__ info, DcWork w) {
  const int mi = blockIdx.y;
  const int64_t off = moff[mi];
  const int K = info[mi].K;
  const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= K) return;
  const double* d = w.dlam + off;
  const double dorg = d[w.org[off + j]], mu = w.mu[off + j];
  double ss = 0.0;
  for (int i = lane; i < K; i += 32) {
    const double v = w.zhat[off + i] / ((d[i] - dorg) - mu);
    ss = fma(v, v, ss);
  }
  ss = warp_sum(ss);
  if (lane == 0) w.sortd[off + j] = 1.0 / sqrt(ss);
}

// Xg rows 0..K-1 <- X rows src(i) (non-deflated, secular order), K..n-1 <- deflated rows
__global__ void dc_xgather_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn,
                                  const MergeInfo* __restrict__ info, DcWork w,
                                  const double* __restrict__ X, double* __restrict__ Xg,
                                  int64_t ldx, int ncol) {
  const int mi = blockIdx.z;
  const int64_t off = moff[mi];
  const int n = mn[mi], K = info[mi].K;
  for (int c = blockIdx.y; c < ncol; c += gridDim.y)
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
      const int s = i < K ? w.src[off + i] : w.dcol[off + (i - K)];
      Xg[(off + i) + (int64_t)c * ldx] = X[(off + s) + (int64_t)c * ldx];
    }
}

// Xn(j, :) = sum_i U~(i, j) Xg(i, :) for the K secular roots; U~ generated per 16 x 64 tile.
constexpr int XA_J = 64, XA_C = 64, XA_I = 16;
__global__ void __launch_bounds__(256) dc_xapply_kernel(const int64_t* __restrict__ moff,
                                                        const MergeInfo* __restrict__ info,
                                                        DcWork w, const double* __restrict__ Xg,
                                                        double* __restrict__ Xn, int64_t ldx,
                                                        int ncol) {
  __shared__ double Vs[XA_I][XA_J + 2];
  __shared__ double Xs[XA_I][XA_C + 2];
  const int mi = blockIdx.z;
  const int64_t off = moff[mi];
  const int K = info[mi].K;
  const int j0 = blockIdx.x * XA_J, c0 = blockIdx.y * XA_C;
  if (j0 >= K || c0 >= ncol) return;
  const int tid = threadIdx.x;
  const int tj = tid >> 4, tc = tid & 15;
  const double* d = w.dlam + off;
  double acc[4][4] = {};
  for (int i0 = 0; i0 < K; i0 += XA_I) {
    for (int t = tid; t < XA_I * XA_J; t += 256) {
      const int ii = t / XA_J, jj = t % XA_J;
      const int i = i0 + ii, j = j0 + jj;
      double v = 0.0;
      if (i < K && j < K)
        v = w.zhat[off + i] / ((d[i] - d[w.org[off + j]]) - w.mu[off + j]) * w.sortd[off + j];
      Vs[ii][jj] = v;
    }
    for (int t = tid; t < XA_I * XA_C; t += 256) {
      const int cc = t / XA_I, ii = t % XA_I;
      const int i = i0 + ii, c = c0 + cc;
      Xs[ii][cc] = (i < K && c < ncol) ? Xg[(off + i) + (int64_t)c * ldx] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int ii = 0; ii < XA_I; ++ii) {
      double a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = Vs[ii][tj * 4 + q];
        b[q] = Xs[ii][tc * 4 + q];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(a[p], b[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int j = j0 + tj * 4 + p;
    if (j >= K) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int c = c0 + tc * 4 + q;
      if (c < ncol) Xn[(off + j) + (int64_t)c * ldx] = acc[p][q];
    }
  }
}

// X row t <- Xn row p (new root p) or Xg row K + b (deflated entry b), in final order
__global__ void dc_xplace_kernel(const int64_t* __restrict__ moff, const int* __restrict__ mn,
                                 const MergeInfo* __restrict__ info, DcWork w,
                                 const double* __restrict__ Xn, const double* __restrict__ Xg,
                                 double* __restrict__ X, int64_t ldx, int ncol) {
  const int mi = blockIdx.z;
  const int64_t off = moff[mi];
  const int n = mn[mi], K = info[mi].K;
  for (int c = blockIdx.y; c < ncol; c += gridDim.y)
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
      const int p = w.perm[off + t];
      X[(off + t) + (int64_t)c * ldx] = p >= 0 ? Xn[(off + p) + (int64_t)c * ldx]
                                               : Xg[(off + K + (-1 - p)) + (int64_t)c * ldx];
    }
}

// ---- driver -----------------------------------------------------------------------

struct Node {
  int64_t off;
  int64_t n;
};

// c0, nc: the caller needs eigenvector columns [c0, c0 + nc) only (ascending order; nc < 0:
// all). The root merge — 3/4 of the merge flops — then forms only those columns (a
// contiguous range of the non-deflated eigenvectors, because both the secular roots and
// the deflated values are sorted); the other columns of Z are left undefined.
void stedc(cudaStream_t st, int64_t n, double* d, double* e, double* Z, int64_t ldz, int64_t c0,
           int64_t nc) {
  if (n <= 0) return;
  if (nc < 0 || c0 < 0 || c0 + nc > n) {
    c0 = 0;
    nc = n;
  }
  // tree: levels[0] = root ... levels[L] = leaves
  std::vector<std::vector<Node>> levels;
  levels.push_back({Node{0, n}});
  while (true) {
    const auto& cur = levels.back();
    bool split = false;
    for (auto& nd : cur)
      if (nd.n > LEAF) split = true;
    if (!split) break;
    std::vector<Node> nxt;
    for (auto& nd : cur) {
      if (nd.n > LEAF) {
        const int64_t n1 = nd.n / 2;
        nxt.push_back({nd.off, n1});
        nxt.push_back({nd.off + n1, nd.n - n1});
      } else {
        nxt.push_back(nd);  // carried unchanged to the next level
      }
    }
    levels.push_back(nxt);
  }
  // scale to unit max-norm
  DBuf scal(1, st);
  absmax_kernel<<<1, 1024, 0, st>>>(n, d, e, scal.p);
  EM_LAUNCHED();
  scale_vec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, d, scal.p, 1);
  EM_LAUNCHED();
  if (n > 1) {
    scale_vec_kernel<<<(unsigned)((n - 1 + 255) / 256), 256, 0, st>>>(n - 1, e, scal.p, 1);
    EM_LAUNCHED();
  }
  // split points (every internal node) and tearing
  std::vector<int64_t> splits;
  for (size_t L = 0; L + 1 < levels.size(); ++L)
    for (auto& nd : levels[L])
      if (nd.n > LEAF) splits.push_back(nd.off + nd.n / 2);
  std::sort(splits.begin(), splits.end());
  const int nsplit = (int)splits.size();
  DArr<int64_t> dsplit(imax64(nsplit, 1), st);
  DBuf betas(imax64(nsplit, 1), st);
  if (nsplit) {
    EM_CK(cudaMemcpyAsync(dsplit.p, splits.data(), nsplit * sizeof(int64_t),
                          cudaMemcpyHostToDevice, st));
    dc_tear_kernel<<<(nsplit + 127) / 128, 128, 0, st>>>(nsplit, dsplit.p, d, e, betas.p);
    EM_LAUNCHED();
  }
  // buffers (all eigenvector buffers use ld = n)
  DBuf lam(n, st), lam2(n, st);
  DBuf Qb((size_t)n * n, st), Qz, Ub;
  double* B0 = Z;
  if (ldz != n) {
    Qz.alloc((size_t)n * n, st);
    B0 = Qz.p;
  }
  // off-diagonal child regions must read as zero before their merge
  EM_CK(cudaMemsetAsync(B0, 0, (size_t)n * n * sizeof(double), st));
  double* Qcur = B0;
  // leaves
  {
    const auto& leaves = levels.back();
    std::vector<int64_t> lo;
    std::vector<int> ls;
    for (auto& nd : leaves) {
      lo.push_back(nd.off);
      ls.push_back((int)nd.n);
    }
    DArr<int64_t> dlo(lo.size(), st);
    DArr<int> dls(ls.size(), st);
    EM_CK(cudaMemcpyAsync(dlo.p, lo.data(), lo.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(dls.p, ls.data(), ls.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    dc_leaf_kernel<<<(unsigned)leaves.size(), LEAF, 0, st>>>(dlo.p, dls.p, d, e, lam.p, Qcur, n);
    EM_LAUNCHED();
    EM_CK(cudaStreamSynchronize(st));  // dlo/dls lifetime
  }
  if (levels.size() > 1) {
    EM_CK(cudaMemsetAsync(Qb.p, 0, (size_t)n * n * sizeof(double), st));
    Ub.alloc((size_t)n * n, st);
  }
  // workspace
  DBuf wd((size_t)n * 10, st);
  DArr<int> wi((size_t)n * 8, st);
  DcWork w;
  w.dlam = wd.p;
  w.wz = wd.p + n;
  w.dval = wd.p + 2 * n;
  w.rot_c = wd.p + 3 * n;
  w.rot_s = wd.p + 4 * n;
  w.mu = wd.p + 5 * n;
  w.zhat = wd.p + 6 * n;
  w.lamn = wd.p + 7 * n;
  w.sortd = wd.p + 8 * n;
  w.sortz = wd.p + 9 * n;
  w.src = wi.p;
  w.pos = wi.p + n;
  w.dcol = wi.p + 2 * n;
  w.rot_a = wi.p + 3 * n;
  w.rot_b = wi.p + 4 * n;
  w.org = wi.p + 5 * n;
  w.typ = wi.p + 6 * n;
  w.perm = wi.p + 7 * n;

  double* lam_cur = lam.p;
  double* lam_nxt = lam2.p;
  double* Qalt = Qb.p;
  const int64_t ldcur = n;
  for (int L = (int)levels.size() - 2; L >= 0; --L) {
    // merges at this level: nodes with n > LEAF (their children are at L+1)
    std::vector<int64_t> mo;
    std::vector<int> m1, mnn;
    std::vector<double> dummy;
    std::vector<int> beta_idx;
    for (auto& nd : levels[L]) {
      if (nd.n <= LEAF) continue;
      mo.push_back(nd.off);
      m1.push_back((int)(nd.n / 2));
      mnn.push_back((int)nd.n);
      const int64_t s = nd.off + nd.n / 2;
      beta_idx.push_back((int)(std::lower_bound(splits.begin(), splits.end(), s) - splits.begin()));
    }
    const int nm = (int)mo.size();
    if (nm == 0) continue;
    DArr<int64_t> dmo(nm, st);
    DArr<int> dm1(nm, st), dmn(nm, st), dbi(nm, st);
    DBuf mbeta(nm, st), mrho(nm, st);
    DArr<MergeInfo> minfo(nm, st);
    EM_CK(cudaMemcpyAsync(dmo.p, mo.data(), nm * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(dm1.p, m1.data(), nm * sizeof(int), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(dmn.p, mnn.data(), nm * sizeof(int), cudaMemcpyHostToDevice, st));
    // betas in merge order
    std::vector<double> hb(nsplit);
    EM_CK(cudaMemcpyAsync(hb.data(), betas.p, nsplit * sizeof(double), cudaMemcpyDeviceToHost, st));
    EM_CK(cudaStreamSynchronize(st));
    std::vector<double> mb(nm);
    for (int k = 0; k < nm; ++k) mb[k] = hb[beta_idx[k]];
    EM_CK(cudaMemcpyAsync(mbeta.p, mb.data(), nm * sizeof(double), cudaMemcpyHostToDevice, st));

    // if Qcur has ld != n (it is Z), all kernels take ldq explicitly
    dc_deflate_kernel<<<nm, 128, 0, st>>>(dmo.p, dm1.p, dmn.p, mbeta.p, lam_cur, Qcur, ldcur, w,
                                          mrho.p, minfo.p);
    EM_LAUNCHED();
    std::vector<MergeInfo> hi(nm);
    EM_CK(cudaMemcpyAsync(hi.data(), minfo.p, nm * sizeof(MergeInfo), cudaMemcpyDeviceToHost, st));
    EM_CK(cudaStreamSynchronize(st));
    int maxn = 0, maxK = 0;
    for (int k = 0; k < nm; ++k) {
      maxn = std::max(maxn, mnn[k]);
      maxK = std::max(maxK, hi[k].K);
    }
    {
      dim3 g((unsigned)std::max(1, std::min((maxn + 255) / 256, 64)), (unsigned)nm);
      dc_rotate_kernel<<<g, 256, 0, st>>>(dmo.p, dmn.p, minfo.p, w, Qcur, ldcur);
      EM_LAUNCHED();
    }
    if (maxK > 0) {
      dim3 g1((unsigned)((maxK + 127) / 128), (unsigned)nm);
      stage_begin(st, ST_STEDC_SECULAR);
      dc_secular_kernel<<<g1, 128, 0, st>>>(dmo.p, minfo.p, mrho.p, w);
      EM_LAUNCHED();
      stage_end(st, ST_STEDC_SECULAR);
      dc_zhat_kernel<<<g1, 128, 0, st>>>(dmo.p, minfo.p, w);
      EM_LAUNCHED();
      dim3 g2((unsigned)((maxK + 7) / 8), (unsigned)nm);
      dc_umat_kernel<<<g2, 256, 0, st>>>(dmo.p, minfo.p, w, Ub.p, n);
      EM_LAUNCHED();
    }
    {
      dim3 g3((unsigned)std::max(1, std::min((maxn + 255) / 256, 8)), (unsigned)std::min(maxn, 65535), (unsigned)nm);
      dc_gather_kernel<<<g3, 256, 0, st>>>(dmo.p, dmn.p, minfo.p, w, Qcur, Qalt, n);
      EM_LAUNCHED();
    }
    // the final order of the merged spectrum depends on the eigenvalues only
    dc_order_kernel<<<nm, 32, 0, st>>>(dmo.p, dmn.p, minfo.p, w, lam_nxt);
    EM_LAUNCHED();
    // root merge with a column range: the new eigenvectors landing in [c0, c0 + nc)
    const bool root_range = L == 0 && nm == 1 && mnn[0] == n && nc < n;
    int a_lo = 0, a_hi = nm == 1 ? hi[0].K : 0;
    if (root_range) {
      std::vector<int> hp((size_t)std::max<int64_t>(nc, 1));
      EM_CK(cudaMemcpyAsync(hp.data(), w.perm + c0, nc * sizeof(int), cudaMemcpyDeviceToHost, st));
      EM_CK(cudaStreamSynchronize(st));
      a_lo = hi[0].K;
      a_hi = 0;
      for (int64_t t = 0; t < nc; ++t)
        if (hp[t] >= 0) {
          a_lo = std::min(a_lo, hp[t]);
          a_hi = std::max(a_hi, hp[t] + 1);
        }
      if (a_hi < a_lo) a_lo = a_hi = 0;  // only deflated columns in the range
    }
    // grouped GEMMs: top rows use type 1+2 columns, bottom rows type 2+3
    std::vector<GemmArgs> probs;
    int max_tiles = 1;
    for (int k = 0; k < nm; ++k) {
      const int K = hi[k].K, c1 = hi[k].c1, c2 = hi[k].c2;
      if (K == 0) continue;
      const int64_t off = mo[k];
      const int64_t n1 = m1[k], n2 = mnn[k] - n1;
      GemmArgs top{n1, K, c1 + c2, Qalt + off + off * n, n, Ub.p + off + off * n, n,
                   Qcur + off + off * n, n, 1.0, 0.0, 0};
      GemmArgs bot{n2, K, K - c1, Qalt + (off + n1) + (off + c1) * n, n,
                   Ub.p + (off + c1) + off * n, n, Qcur + (off + n1) + off * n, n, 1.0, 0.0, 0};
      if (root_range) {  // columns a_lo .. a_hi - 1 of the product only
        for (GemmArgs* g : {&top, &bot}) {
          g->n = a_hi - a_lo;
          g->B += (int64_t)a_lo * g->ldb;
          g->C += (int64_t)a_lo * g->ldc;
        }
        if (a_hi <= a_lo) continue;
      }
      probs.push_back(top);
      probs.push_back(bot);
      max_tiles = std::max<int>(max_tiles, (int)(((n1 + 127) / 128) * ((K + 127) / 128)));
      max_tiles = std::max<int>(max_tiles, (int)(((n2 + 127) / 128) * ((K + 127) / 128)));
    }
    if (getenv("EM_DEBUG_STEDC")) {
      double fl = 0.0;
      for (auto& q : probs) fl += 2.0 * q.m * q.n * q.k;
      int maxK = 0;
      for (int k = 0; k < nm; ++k) maxK = std::max(maxK, hi[k].K);
      fprintf(stderr, "stedc level %d: merges %d maxn %d maxK %d gemm_gflop %.1f\n", L, nm, maxn,
              maxK, fl * 1e-9);
    }
    if (!probs.empty()) {
      DArr<GemmArgs> dp(probs.size(), st);
      EM_CK(cudaMemcpyAsync(dp.p, probs.data(), probs.size() * sizeof(GemmArgs),
                            cudaMemcpyHostToDevice, st));
      const int grid_x = std::min(max_tiles, 4 * num_sms());
      Stage sg(st, ST_STEDC_GEMM);
      if (nm <= 8 && maxn >= 4096) {
        // the few large merges at the top of the tree: one product each (TMA-fed kernel)
        for (const GemmArgs& g : probs)
          EM_CK(gemm(st, false, false, g.m, g.n, g.k, g.alpha, g.A, g.lda, g.B, g.ldb, g.beta,
                     g.C, g.ldc));
      } else {
        EM_CK(gemm_grouped(st, false, false, dp.p, (int)probs.size(), grid_x));
      }
      EM_CK(cudaStreamSynchronize(st));  // dp lifetime
    }
    {
      dim3 g((unsigned)std::max(1, std::min((maxn + 255) / 256, 8)), (unsigned)std::min(maxn, 65535), (unsigned)nm);
      // deflated columns next to the GEMM output in Qcur, then everything placed in
      // final order into Qalt (free after the GEMM) and the roles swapped
      dc_copy_deflated_kernel<<<g, 256, 0, st>>>(dmo.p, dmn.p, minfo.p, Qalt, Qcur, n);
      EM_LAUNCHED();
      dc_place_kernel<<<g, 256, 0, st>>>(dmo.p, dmn.p, minfo.p, w, Qcur, Qalt, n,
                                         root_range ? (int)c0 : 0,
                                         root_range ? (int)(c0 + nc) : maxn);
      EM_LAUNCHED();
    }
    // blocks not merged at this level (leaf-sized nodes carried up) keep their data:
    // copy them into Qalt / lam_nxt as well
    for (auto& nd : levels[L]) {
      if (nd.n > LEAF) continue;
      copy_matrix(st, false, nd.n, nd.n, Qcur + nd.off + nd.off * ldcur, ldcur,
                  Qalt + nd.off + nd.off * n, n);
      EM_CK(cudaMemcpyAsync(lam_nxt + nd.off, lam_cur + nd.off, nd.n * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
    }
    EM_CK(cudaStreamSynchronize(st));  // small per-level arrays go out of scope
    std::swap(Qcur, Qalt);
    std::swap(lam_cur, lam_nxt);
  }
  // result: lam_cur (scaled), Qcur
  if (Qcur != Z) copy_matrix(st, false, n, nc, Qcur + c0 * n, n, Z + c0 * ldz, ldz);
  EM_CK(cudaMemcpyAsync(d, lam_cur, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  scale_vec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, d, scal.p, 0);
  EM_LAUNCHED();
  EM_CK(cudaStreamSynchronize(st));
}

}  // namespace em

namespace em {

// Eigenvalues of the symmetric tridiagonal (d, e) ascending in d, and Y (n x k) <- U^T Y
// for its eigenvector matrix U, without forming U (the implicit form above).
void stedc_apply(cudaStream_t st, int64_t n, double* d, double* e, double* Y, int64_t ldy,
                 int64_t k) {
  if (n <= 0) return;
  std::vector<std::vector<Node>> levels;
  levels.push_back({Node{0, n}});
  while (true) {
    bool split = false;
    for (auto& nd : levels.back())
      if (nd.n > LEAF) split = true;
    if (!split) break;
    std::vector<Node> nxt;
    for (auto& nd : levels.back()) {
      if (nd.n > LEAF) {
        const int64_t n1 = nd.n / 2;
        nxt.push_back({nd.off, n1});
        nxt.push_back({nd.off + n1, nd.n - n1});
      } else {
        nxt.push_back(nd);
      }
    }
    levels.push_back(nxt);
  }
  DBuf scal(1, st);
  absmax_kernel<<<1, 1024, 0, st>>>(n, d, e, scal.p);
  EM_LAUNCHED();
  scale_vec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, d, scal.p, 1);
  EM_LAUNCHED();
  if (n > 1) {
    scale_vec_kernel<<<(unsigned)((n - 1 + 255) / 256), 256, 0, st>>>(n - 1, e, scal.p, 1);
    EM_LAUNCHED();
  }
  std::vector<int64_t> splits;
  for (size_t L = 0; L + 1 < levels.size(); ++L)
    for (auto& nd : levels[L])
      if (nd.n > LEAF) splits.push_back(nd.off + nd.n / 2);
  std::sort(splits.begin(), splits.end());
  const int nsplit = (int)splits.size();
  DArr<int64_t> dsplit(imax64(nsplit, 1), st);
  DBuf betas(imax64(nsplit, 1), st);
  std::vector<double> hb(imax64(nsplit, 1));
  if (nsplit) {
    EM_CK(cudaMemcpyAsync(dsplit.p, splits.data(), nsplit * sizeof(int64_t),
                          cudaMemcpyHostToDevice, st));
    dc_tear_kernel<<<(nsplit + 127) / 128, 128, 0, st>>>(nsplit, dsplit.p, d, e, betas.p);
    EM_LAUNCHED();
    EM_CK(cudaMemcpyAsync(hb.data(), betas.p, nsplit * sizeof(double), cudaMemcpyDeviceToHost,
                          st));
  }
  const int ncol = (int)k + 2;
  const int64_t ldx = n;
  DBuf lam(n, st), lam2(n, st), X((size_t)n * ncol, st), Xg((size_t)n * ncol, st),
      Xn((size_t)n * ncol, st);
  {
    const auto& leaves = levels.back();
    std::vector<int64_t> lo;
    std::vector<int> ls;
    for (auto& nd : leaves) {
      lo.push_back(nd.off);
      ls.push_back((int)nd.n);
    }
    DArr<int64_t> dlo(lo.size(), st);
    DArr<int> dls(ls.size(), st);
    EM_CK(cudaMemcpyAsync(dlo.p, lo.data(), lo.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(dls.p, ls.data(), ls.size() * sizeof(int), cudaMemcpyHostToDevice, st));
    dc_leaf_apply_kernel<<<(unsigned)leaves.size(), LEAF, 0, st>>>(dlo.p, dls.p, d, e, lam.p, Y,
                                                                   ldy, (int)k, X.p, ldx);
    EM_LAUNCHED();
    EM_CK(cudaStreamSynchronize(st));
  }
  DBuf wd((size_t)n * 10, st);
  DArr<int> wi((size_t)n * 8, st);
  DcWork w;
  w.dlam = wd.p;
  w.wz = wd.p + n;
  w.dval = wd.p + 2 * n;
  w.rot_c = wd.p + 3 * n;
  w.rot_s = wd.p + 4 * n;
  w.mu = wd.p + 5 * n;
  w.zhat = wd.p + 6 * n;
  w.lamn = wd.p + 7 * n;
  w.sortd = wd.p + 8 * n;
  w.sortz = wd.p + 9 * n;
  w.src = wi.p;
  w.pos = wi.p + n;
  w.dcol = wi.p + 2 * n;
  w.rot_a = wi.p + 3 * n;
  w.rot_b = wi.p + 4 * n;
  w.org = wi.p + 5 * n;
  w.typ = wi.p + 6 * n;
  w.perm = wi.p + 7 * n;
  double* lam_cur = lam.p;
  double* lam_nxt = lam2.p;
  const double* xf = X.p + (int64_t)k * ldx;
  const double* xl = X.p + (int64_t)(k + 1) * ldx;
  for (int L = (int)levels.size() - 2; L >= 0; --L) {
    std::vector<int64_t> mo;
    std::vector<int> m1, mnn;
    std::vector<double> mb;
    for (auto& nd : levels[L]) {
      if (nd.n <= LEAF) continue;
      mo.push_back(nd.off);
      m1.push_back((int)(nd.n / 2));
      mnn.push_back((int)nd.n);
      const int64_t s = nd.off + nd.n / 2;
      mb.push_back(hb[std::lower_bound(splits.begin(), splits.end(), s) - splits.begin()]);
    }
    const int nm = (int)mo.size();
    if (nm == 0) continue;
    DArr<int64_t> dmo(nm, st);
    DArr<int> dm1(nm, st), dmn(nm, st);
    DBuf mbeta(nm, st), mrho(nm, st);
    DArr<MergeInfo> minfo(nm, st);
    EM_CK(cudaMemcpyAsync(dmo.p, mo.data(), nm * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(dm1.p, m1.data(), nm * sizeof(int), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(dmn.p, mnn.data(), nm * sizeof(int), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(mbeta.p, mb.data(), nm * sizeof(double), cudaMemcpyHostToDevice, st));
    dc_deflate_kernel<<<nm, 128, 0, st>>>(dmo.p, dm1.p, dmn.p, mbeta.p, lam_cur, nullptr, 0, w,
                                          mrho.p, minfo.p, xf, xl);
    EM_LAUNCHED();
    std::vector<MergeInfo> hi(nm);
    EM_CK(cudaMemcpyAsync(hi.data(), minfo.p, nm * sizeof(MergeInfo), cudaMemcpyDeviceToHost, st));
    EM_CK(cudaStreamSynchronize(st));
    int maxn = 0, maxK = 0;
    for (int q = 0; q < nm; ++q) {
      maxn = std::max(maxn, mnn[q]);
      maxK = std::max(maxK, hi[q].K);
    }
    dc_xrot_kernel<<<dim3((unsigned)((ncol + 127) / 128), (unsigned)nm), 128, 0, st>>>(
        dmo.p, dm1.p, dmn.p, minfo.p, w, X.p, ldx, ncol);
    EM_LAUNCHED();
    const unsigned gy = (unsigned)std::min(ncol, 65535);
    dc_xgather_kernel<<<dim3((unsigned)std::max(1, std::min((maxn + 255) / 256, 64)), gy,
                             (unsigned)nm), 256, 0, st>>>(dmo.p, dmn.p, minfo.p, w, X.p, Xg.p,
                                                          ldx, ncol);
    EM_LAUNCHED();
    if (maxK > 0) {
      dim3 g1((unsigned)((maxK + 127) / 128), (unsigned)nm);
      stage_begin(st, ST_STEDC_SECULAR);
      dc_secular_kernel<<<g1, 128, 0, st>>>(dmo.p, minfo.p, mrho.p, w);
      EM_LAUNCHED();
      stage_end(st, ST_STEDC_SECULAR);
      dc_zhat_kernel<<<g1, 128, 0, st>>>(dmo.p, minfo.p, w);
      EM_LAUNCHED();
      dc_unorm_kernel<<<dim3((unsigned)((maxK + 7) / 8), (unsigned)nm), 256, 0, st>>>(dmo.p,
                                                                                    minfo.p, w);
      EM_LAUNCHED();
      Stage sg(st, ST_STEDC_GEMM);
      dc_xapply_kernel<<<dim3((unsigned)((maxK + XA_J - 1) / XA_J),
                              (unsigned)((ncol + XA_C - 1) / XA_C), (unsigned)nm), 256, 0, st>>>(
          dmo.p, minfo.p, w, Xg.p, Xn.p, ldx, ncol);
      EM_LAUNCHED();
    }
    dc_order_kernel<<<nm, 32, 0, st>>>(dmo.p, dmn.p, minfo.p, w, lam_nxt);
    EM_LAUNCHED();
    dc_xplace_kernel<<<dim3((unsigned)std::max(1, std::min((maxn + 255) / 256, 64)), gy,
                            (unsigned)nm), 256, 0, st>>>(dmo.p, dmn.p, minfo.p, w, Xn.p, Xg.p,
                                                         X.p, ldx, ncol);
    EM_LAUNCHED();
    for (auto& nd : levels[L]) {  // leaf-sized nodes carried up keep their rows of X
      if (nd.n > LEAF) continue;
      EM_CK(cudaMemcpyAsync(lam_nxt + nd.off, lam_cur + nd.off, nd.n * sizeof(double),
                            cudaMemcpyDeviceToDevice, st));
    }
    EM_CK(cudaStreamSynchronize(st));
    std::swap(lam_cur, lam_nxt);
  }
  copy_matrix(st, false, n, k, X.p, ldx, Y, ldy);
  EM_CK(cudaMemcpyAsync(d, lam_cur, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
  scale_vec_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, d, scal.p, 0);
  EM_LAUNCHED();
  EM_CK(cudaStreamSynchronize(st));
}

}  // namespace em
