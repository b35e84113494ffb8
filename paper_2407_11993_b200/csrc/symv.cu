// y = alpha * A x + beta * y for symmetric A reading ONLY the lower triangle
// (each off-diagonal 64x64 tile is read once and used twice). HBM-bound:
// n^2/2 * 8 bytes per call; deterministic (fixed-order reduction, no atomics).
// Tile bodies in symv_tile.cuh.
//
// Used by the Cholesky theta-method's per-step R * I product
// (reference: td1_step_kernel's dense loop, _kernels.py:198-207) and exposed as
// em_symv_lower. This register-prefetch kernel is the fallback when TMA cannot address
// the matrix (symv_tma.cu).
#include <algorithm>

#include "common.cuh"
#include "ctx.h"
#include "linalg.h"
#include "symv_tile.cuh"

namespace em {

// Persistent schedule: the nb(nb+1)/2 lower tiles in strip-major order (strip i,
// tiles j = 0..i) are cut into P equal contiguous ranges, one per CTA, so every CTA
// streams the same number of bytes (no tail wave) and keeps one tile of prefetch in
// flight across strip boundaries. A strip split between CTAs leaves one row partial
// per piece: slot p - pfirst(i) of strip i, pfirst(i) = off(i) / len.
struct SymvSched {
  int64_t nb, T, P, len;
};

static SymvSched symv_sched(int64_t n) {
  SymvSched s;
  s.nb = (n + SV - 1) / SV;
  s.T = s.nb * (s.nb + 1) / 2;
  s.P = imax64(1, imin64(s.T, 2 * (int64_t)num_sms()));
  s.len = (s.T + s.P - 1) / s.P;
  s.P = (s.T + s.len - 1) / s.len;  // drop empty ranges
  return s;
}

size_t symv_work_size(int64_t n) {
  const int64_t nb = (n + SV - 1) / SV;
  // wcol: nb*nb tiles; wrow: nb strips x (nb + 2) piece slots. Covers symv_work_doubles
  // and the TMA variant's layout too.
  return std::max((size_t)(nb * nb * SV + nb * (nb + 2) * SV), symv_tma_work_size(n));
}

__device__ __forceinline__ int64_t strip_of(int64_t t) {
  // largest i with i(i+1)/2 <= t
  int64_t i = (int64_t)((sqrt(8.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (i * (i + 1) / 2 > t) --i;
  while ((i + 1) * (i + 2) / 2 <= t) ++i;
  return i;
}

template <bool LARFG>
__global__ void __launch_bounds__(256, 2) symv_persist_kernel(int64_t n, const double* __restrict__ A,
                                                              int64_t lda,
                                                              const double* __restrict__ x,
                                                              double* __restrict__ wcol,
                                                              double* __restrict__ wrow, int64_t nb,
                                                              int64_t T, int64_t len,
                                                              SymvLarfg lf) {
  __shared__ double red[8][SV];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t p = blockIdx.x;
  const int64_t t0 = p * len, t1 = imin64(T, t0 + len);
  if (t0 >= t1) return;
  int64_t i = strip_of(t0), j = t0 - i * (i + 1) / 2;
  double nxt[2][8];
  auto load = [&](int64_t ii, int64_t jj) {
    const int64_t r0 = ii * SV, c0 = jj * SV;
    if (r0 + SV <= n && c0 + SV <= n)
      symv_load_tile<true>(nxt, A, lda, n, r0, c0, lane, w);
    else
      symv_load_tile<false>(nxt, A, lda, n, r0, c0, lane, w);
  };
  load(i, j);  // A is not written by the launch this one may overlap
  pdl_wait();
  pdl_trigger();
  // dlarfg of the raw column x (while the first tile is in flight): every CTA forms
  // beta, tau and the scale from the sum-of-squares partials; CTA 0 publishes them.
  double xs = 1.0;
  if (LARFG) {
    double ss = 0.0;
    for (int64_t q = tid; q < lf.nparts; q += 256) ss += __ldcg(lf.part + q);
    ss = warp_sum(ss);
    if (lane == 0) red[0][w] = ss;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tot += red[0][k];
    const double alpha = __ldcg(lf.alpha);
    const double xnorm = sqrt(tot);
    double beta = alpha, tau = 0.0, scale = 0.0;
    if (xnorm != 0.0) {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (p == 0 && tid == 0) {
      *lf.tau = tau;
      *lf.e = beta;
      *lf.scale = scale;
    }
    xs = scale;
    __syncthreads();
  }
  double xi0 = 0.0, xi1 = 0.0, row0 = 0.0, row1 = 0.0;
  bool fresh = true;
  for (int64_t t = t0; t < t1; ++t) {
    double a[2][8];
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      a[0][cc] = nxt[0][cc];
      a[1][cc] = nxt[1][cc];
    }
    const int64_t in = (j < i) ? i : i + 1, jn = (j < i) ? j + 1 : 0;
    if (t + 1 < t1) load(in, jn);
    const int64_t r0 = i * SV;
    if (fresh) {
      xi0 = symv_xval(x, r0 + lane, n, xs, LARFG);
      xi1 = symv_xval(x, r0 + lane + 32, n, xs, LARFG);
      row0 = row1 = 0.0;
      fresh = false;
    }
    symv_tile_body(a, n, x, j * SV, j == i, xi0, xi1, row0, row1, wcol + (i * nb + j) * SV, lane,
                   w, xs, LARFG);
    if (j == i || t + 1 == t1) {  // end of this CTA's piece of strip i
      __syncthreads();
      red[w][lane] = row0;
      red[w][lane + 32] = row1;
      __syncthreads();
      if (tid < SV) {
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k) s += red[k][tid];
        const int64_t slot = p - (i * (i + 1) / 2) / len;
        wrow[(i * (nb + 2) + slot) * SV + tid] = s;
      }
      fresh = true;
    }
    i = in;
    j = jn;
  }
}

// y_j = sum_{i >= j} wcol(i, j) + the row partials of strip j; fixed order.
// 512 threads: 8 groups of 64 rows, 4 independent loads in flight per thread.
// CTAs nb .. nb+7 (only when lt.i > 0): the latrd panel products t (see LatrdT).
__global__ void __launch_bounds__(512) symv_reduce2_kernel(int64_t n, double alpha, double beta,
                                                           double* __restrict__ y,
                                                           const double* __restrict__ wcol,
                                                           const double* __restrict__ wrow,
                                                           int64_t nb, int64_t len, LatrdT lt) {
  __shared__ double red8[32][SV + 1];
  const int64_t j = blockIdx.x;
  pdl_wait();
  pdl_trigger();
  if (j >= nb) {
    // t[col], col < 64: W_p^T v (k = col), col >= 64: A_p^T v (k = col - 64);
    // = scale * (partials over rows >= c+2) + row c+1 (where v = 1)
    const int q = (int)(j - nb);
    const int cl = threadIdx.x & 15, grp = threadIdx.x >> 4;  // 32 groups
    const int col = q * 16 + cl, k = col & 63;
    double s = 0.0;
    if (k < lt.i)
      for (int64_t g = grp; g < lt.G; g += 32) s += __ldcg(lt.dpart + g * 128 + col);
    red8[grp][cl] = s;
    __syncthreads();
    if (threadIdx.x < 16 && k < lt.i) {
      double tot = 0.0;
      for (int g2 = 0; g2 < 32; ++g2) tot += red8[g2][cl];
      const double r1 = (col < 64) ? __ldcg(lt.wr1 + k * lt.ldw) : __ldcg(lt.ar1 + k * lt.lda);
      lt.t[col] = fma(__ldcg(lt.scale), tot, r1);
    }
    return;
  }
  const int t = threadIdx.x & (SV - 1), g = threadIdx.x >> 6;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t i = j + g;
  for (; i + 24 < nb; i += 32) {
    s0 += __ldcg(wcol + (i * nb + j) * SV + t);
    s1 += __ldcg(wcol + ((i + 8) * nb + j) * SV + t);
    s2 += __ldcg(wcol + ((i + 16) * nb + j) * SV + t);
    s3 += __ldcg(wcol + ((i + 24) * nb + j) * SV + t);
  }
  for (; i < nb; i += 8) s0 += __ldcg(wcol + (i * nb + j) * SV + t);
  const int64_t off = j * (j + 1) / 2;
  const int64_t npc = (off + j) / len - off / len + 1;
  for (int64_t q = g; q < npc; q += 8) s1 += __ldcg(wrow + (j * (nb + 2) + q) * SV + t);
  red8[g][t] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (threadIdx.x < SV) {
    const double v = ((red8[0][t] + red8[1][t]) + (red8[2][t] + red8[3][t])) +
                     ((red8[4][t] + red8[5][t]) + (red8[6][t] + red8[7][t]));
    const int64_t idx = j * SV + t;
    if (idx < n) y[idx] = (beta == 0.0) ? alpha * v : fma(alpha, v, beta * y[idx]);
  }
}

void symv_lower(cudaStream_t st, int64_t n, double alpha, const double* A, int64_t lda,
                const double* x, double beta, double* y, double* work) {
  if (n <= 0) return;
  SymvMap m;
  if (symv_map_make(&m, A, n, n, lda)) {
    symv_tma(st, m, 0, n, alpha, x, beta, y, work, nullptr, nullptr, false);
    return;
  }
  const SymvSched s = symv_sched(n);
  double* wcol = work;
  double* wrow = work + s.nb * s.nb * SV;
  symv_persist_kernel<false><<<(unsigned)s.P, 256, 0, st>>>(n, A, lda, x, wcol, wrow, s.nb, s.T,
                                                            s.len, SymvLarfg{});
  EM_LAUNCHED();
  symv_reduce2_kernel<<<(unsigned)s.nb, 512, 0, st>>>(n, alpha, beta, y, wcol, wrow, s.nb, s.len,
                                                      LatrdT{});
  EM_LAUNCHED();
}

void symv_lower_latrd(cudaStream_t st, int64_t n, const double* A, int64_t lda, const double* x,
                      double* y, double* work, const SymvLarfg& lf, const LatrdT& lt) {
  const SymvSched s = symv_sched(n);
  double* wcol = work;
  double* wrow = work + s.nb * s.nb * SV;
  launch_pdl(symv_persist_kernel<true>, dim3((unsigned)s.P), dim3(256), 0, st, n, A, lda, x,
             wcol, wrow, s.nb, s.T, s.len, lf);
  const unsigned extra = lt.i > 0 ? 8u : 0u;
  launch_pdl(symv_reduce2_kernel, dim3((unsigned)s.nb + extra), dim3(512), 0, st, n, 1.0, 0.0, y,
             (const double*)wcol, (const double*)wrow, s.nb, s.len, lt);
}

}  // namespace em
