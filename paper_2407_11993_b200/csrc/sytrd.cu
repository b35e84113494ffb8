// Householder tridiagonalisation (lower, blocked: latrd panels + syr2k) and the
// blocked back-transform Z <- Q Z (ormtr). Together with stedc.cu this replaces
// the reference's cyclic Jacobi eigensolver (_kernels.py:82-141), which is
// O(sweeps N^3) sequential; the result (eigenvalues, invariant subspaces) is
// the same to round-off.
//
// Per panel column the memory-bound part is one lower-triangle symv over the
// trailing matrix (symv.cu); the rank-2k trailing update and the
// back-transform run on the DMMA GEMM. A panel column is four launches:
// latrd_col_kernel (finish the previous W column, update this column, partials of
// its norm and of the panel products), the symv with dlarfg folded into its
// prologue, the symv reduction (+ panel products t), latrd_w_kernel.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

constexpr int TRD_NB = 64;   // panel width
constexpr int RT = 256;

EM_DEVINL double block_sum(double v, double* red) {
  v = warp_sum(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  return t;  // valid in thread 0
}

constexpr int CRW = 64;                 // rows per CTA in the column kernels
constexpr int CTPR = RT / CRW;          // 4 threads per row
constexpr int CKQ = TRD_NB / CTPR;      // panel columns per thread (16)

// Column kernel for panel column c (i = c - i0 earlier panel columns), LAPACK dlatrd:
//  (1) finish W[:, i-1]: w += alpha v, alpha = -tau/2 (w.v), from wtmp (tau (y - ...))
//      and the w.v partials of the previous latrd_w_kernel (every CTA reduces them);
//  (2) A[c:n, c] -= A[c:n, i0:c] W[c, 0:i]^T + W[c:n, 0:i] A[c, i0:c]^T;
//  (3) per-CTA partials over rows >= c+2 of ||x||^2 (dlarfg) and of W_p^T x, A_p^T x
//      (the dlatrd panel products, completed in symv_reduce2_kernel), x = the updated
//      column; alpha_buf = A[c+1, c], d[c] = A[c, c].
// upd = 0: only (1), after the last column of a panel.
// FUSEW (TMA path): the previous column's w is formed here instead of in a separate
// kernel: wtmp holds y = A22 v (the symv reduction), tvec the panel products t, and
// w^T v = tau (v^T A22 v - 2 t1^T t2) comes from the symv's quadratic-form partials
// (vav, nvav), so alpha needs no reduction over w:
//   v = [1, scale x_raw] (written back into A[c:, c-1]),  w = tau (y - A_p t1 - W_p t2),
//   W[:, i-1] = w + alpha v,  alpha = -tau^2/2 (v^T A22 v - 2 t1^T t2).
struct ColW {
  const double* tvec = nullptr;   // t of column c-1 (2 x 64)
  const double* vav = nullptr;    // symv quadratic-form partials of column c-1
  int64_t nvav = 0;
  const double* scale = nullptr;  // dlarfg scale of column c-1
};

template <bool FUSEW>
__global__ void __launch_bounds__(RT) latrd_col_kernel(
    int64_t n, double* A, int64_t lda, int64_t i0, int64_t c, int i, int upd, double* W,
    int64_t ldw, const double* wtmp, const double* part_wv, int64_t n_wv, const double* tau,
    double* part_norm, double* dpart, double* alpha_buf, double* d, ColW cw) {
  __shared__ double wr[TRD_NB], ar[TRD_NB], red[RT / 32];
  __shared__ double pred[RT / 32][2 * TRD_NB];
  __shared__ double t1s[TRD_NB], t2s[TRD_NB];
  __shared__ double s_alpha, s_wc;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = tid & (CTPR - 1);
  const int64_t r = c + blockIdx.x * (int64_t)CRW + tid / CTPR;
  const bool valid = r < n;
  // before the dependency wait: panel columns k < i-1 (finished two launches ago or
  // earlier) and the raw columns c-1 (FUSEW) and c (only this kernel writes them)
  double av[CKQ], wv[CKQ];
  double acol = 0.0, xprev = 0.0;
  if (upd || FUSEW) {
    for (int k = tid; k < i - 1; k += RT) {
      wr[k] = W[(c - i0) + k * ldw];
      ar[k] = A[c + (i0 + k) * lda];
    }
#pragma unroll
    for (int q = 0; q < CKQ; ++q) {
      const int k = sub + CTPR * q;
      const bool ok = valid && k < i - 1;
      av[q] = ok ? A[r + (i0 + k) * lda] : 0.0;
      wv[q] = ok ? W[(r - i0) + k * ldw] : 0.0;
    }
    if (valid && upd) acol = A[r + c * lda];
    if (FUSEW && i > 0 && valid) xprev = A[r + (c - 1) * lda];
  }
  double tprev = 0.0, scprev = 0.0, vavsum = 0.0;
  if (FUSEW && i > 0) {  // from the symv two launches back
    tprev = tau[c - 1];
    scprev = *cw.scale;
    double sv = 0.0;
    for (int64_t q = tid; q < cw.nvav; q += RT) sv += cw.vav[q];
    vavsum = block_sum(sv, red);  // thread 0
  }
  pdl_wait();
  pdl_trigger();
  double alpha_p = 0.0, wlast = 0.0, vlast = 0.0;
  if (!FUSEW) {
    if (i > 0) {
      double s = 0.0;
      for (int64_t q = tid; q < n_wv; q += RT) s += __ldcg(part_wv + q);
      const double t = block_sum(s, red);
      if (tid == 0) s_alpha = -0.5 * __ldcg(tau + c - 1) * t;
      __syncthreads();
      alpha_p = s_alpha;
    }
    // column i-1 of W: w + alpha v (v_{c-1} = A[:, c-1], written by the previous launch)
    if (i > 0 && valid) {
      vlast = __ldcg(A + r + (c - 1) * lda);
      wlast = fma(alpha_p, vlast, __ldcg(wtmp + r));
    }
  } else if (i > 0) {
    // everything from the previous launch in one round of loads: t, y at this row and
    // (warp 0) y at row c
    const double yr = valid ? __ldcg(wtmp + r) : 0.0;
    const double yc = (warp == 0) ? __ldcg(wtmp + c) : 0.0;
    for (int k = tid; k < i - 1; k += RT) {
      t1s[k] = __ldcg(cw.tvec + k);
      t2s[k] = __ldcg(cw.tvec + TRD_NB + k);
    }
    __syncthreads();
    if (warp == 0) {  // alpha and w[c] (row c: v = 1), computed by every CTA
      double tt = 0.0, dc = 0.0;
      for (int k = lane; k < i - 1; k += 32) {
        tt = fma(t1s[k], t2s[k], tt);
        dc = fma(ar[k], t1s[k], fma(wr[k], t2s[k], dc));
      }
      tt = warp_sum(tt);
      dc = warp_sum(dc);
      if (lane == 0) {
        s_alpha = -0.5 * tprev * tprev * (vavsum - 2.0 * tt);
        s_wc = tprev * (yc - dc);
      }
    }
    double sdot = 0.0;
#pragma unroll
    for (int q = 0; q < CKQ; ++q) {
      const int k = sub + CTPR * q;
      if (k < i - 1) sdot = fma(av[q], t1s[k], fma(wv[q], t2s[k], sdot));
    }
    sdot += __shfl_xor_sync(0xffffffffu, sdot, 1);
    sdot += __shfl_xor_sync(0xffffffffu, sdot, 2);
    __syncthreads();
    alpha_p = s_alpha;
    if (valid) {
      vlast = (r == c) ? 1.0 : scprev * xprev;
      wlast = fma(alpha_p, vlast, tprev * (yr - sdot));
      if (sub == 0) A[r + (c - 1) * lda] = vlast;
    }
  }
  if (!upd) {
    if (valid && sub == 0) W[(r - i0) + (int64_t)(i - 1) * ldw] = wlast;
    return;
  }
  if (i > 0 && tid == 0) {
    if (FUSEW) {
      wr[i - 1] = fma(alpha_p, 1.0, s_wc);
      ar[i - 1] = 1.0;
    } else {
      const double vc = __ldcg(A + c + (c - 1) * lda);
      wr[i - 1] = fma(alpha_p, vc, __ldcg(wtmp + c));
      ar[i - 1] = vc;
    }
  }
  __syncthreads();
  if (i > 0 && valid && sub == ((i - 1) & (CTPR - 1))) {
    W[(r - i0) + (int64_t)(i - 1) * ldw] = wlast;
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < CKQ; ++q) {
    const int k = sub + CTPR * q;
    if (k == i - 1) {
      av[q] = vlast;
      wv[q] = wlast;
    }
    if (k < i) s = fma(av[q], wr[k], fma(wv[q], ar[k], s));
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  double x = 0.0;
  if (valid) {
    x = acol - s;
    if (sub == 0) {
      if (i > 0) A[r + c * lda] = x;
      if (r == c) d[c] = x;
      if (r == c + 1) *alpha_buf = x;
    }
  }
  const bool tail = valid && r >= c + 2;
  const double ss = (tail && sub == 0) ? x * x : 0.0;
  if (i > 0) {
    const double xt = tail ? x : 0.0;
#pragma unroll
    for (int q = 0; q < CKQ; ++q) {
      double pw = wv[q] * xt, pa = av[q] * xt;
#pragma unroll
      for (int off = 4; off < 32; off <<= 1) {
        pw += __shfl_xor_sync(0xffffffffu, pw, off);
        pa += __shfl_xor_sync(0xffffffffu, pa, off);
      }
      if (lane < CTPR) {
        pred[warp][lane + CTPR * q] = pw;
        pred[warp][TRD_NB + lane + CTPR * q] = pa;
      }
    }
    __syncthreads();
    if (tid < 2 * TRD_NB) {
      double v = 0.0;
      if ((tid & (TRD_NB - 1)) < i)
#pragma unroll
        for (int w8 = 0; w8 < RT / 32; ++w8) v += pred[w8][tid];
      dpart[blockIdx.x * (int64_t)(2 * TRD_NB) + tid] = v;
    }
  }
  const double tn = block_sum(ss, red);
  if (tid == 0) part_norm[blockIdx.x] = tn;
}

// w = tau (y - A_p t1 - W_p t2) on rows >= c+1 (y in wtmp, overwritten with w);
// v = [1, scale x[1:]] written back into A[c+1:, c]; per-CTA partials of w.v.
__global__ void __launch_bounds__(RT) latrd_w_kernel(int64_t n, double* A, int64_t lda,
                                                     int64_t i0, int64_t c, int i,
                                                     const double* W, int64_t ldw, double* wtmp,
                                                     const double* tvec, const double* tau,
                                                     const double* scale, double* part_wv) {
  __shared__ double t1[TRD_NB], t2[TRD_NB], red[RT / 32];
  const int tid = threadIdx.x;
  const int sub = tid & (CTPR - 1);
  const int64_t r = c + 1 + blockIdx.x * (int64_t)CRW + tid / CTPR;
  const bool valid = r < n;
  // before the dependency wait: the panel (complete), tau/scale (from the symv, two
  // launches back) and the raw column
  double av[CKQ], wv[CKQ];
#pragma unroll
  for (int q = 0; q < CKQ; ++q) {
    const int k = sub + CTPR * q;
    const bool ok = valid && k < i;
    av[q] = ok ? A[r + (i0 + k) * lda] : 0.0;
    wv[q] = ok ? W[(r - i0) + k * ldw] : 0.0;
  }
  const double tc = tau[c], sc = *scale;
  const double xr = valid ? A[r + c * lda] : 0.0;
  pdl_wait();
  pdl_trigger();
  for (int k = tid; k < i; k += RT) {
    t1[k] = __ldcg(tvec + k);
    t2[k] = __ldcg(tvec + TRD_NB + k);
  }
  __syncthreads();
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < CKQ; ++q) {
    const int k = sub + CTPR * q;
    if (k < i) s = fma(av[q], t1[k], fma(wv[q], t2[k], s));
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  double dd = 0.0;
  if (valid && sub == 0) {
    const double v = (r == c + 1) ? 1.0 : sc * xr;
    A[r + c * lda] = v;
    const double x = tc * (__ldcg(wtmp + r) - s);
    wtmp[r] = x;
    dd = x * v;
  }
  const double t = block_sum(dd, red);
  if (tid == 0) part_wv[blockIdx.x] = t;
}

__global__ void set_diag_kernel(int64_t n, const double* A, int64_t lda, int64_t c, double* d) {
  if (threadIdx.x == 0 && blockIdx.x == 0) d[c] = A[c + c * lda];
}

// restore A[c+1, c] = e[c] for the panel columns
__global__ void restore_sub_kernel(int64_t n, double* A, int64_t lda, int64_t i0, int w,
                                   const double* e) {
  int k = threadIdx.x;
  if (k < w) {
    int64_t c = i0 + k;
    if (c + 1 < n) A[(c + 1) + c * lda] = e[c];
  }
}

// em_config debug key 98 (tests): bit0 no TMA symv, bit1 no PDL, bit2 no graph,
// bit3 the 4-launch column chain.
int g_sytrd_dbg = 0;

void sytrd_lower(cudaStream_t st, int64_t n, double* A, int64_t lda, double* d, double* e,
                 double* tau) {
  if (n <= 0) return;
  if (n == 1) {
    set_diag_kernel<<<1, 32, 0, st>>>(n, A, lda, 0, d);
    EM_LAUNCHED();
    return;
  }
  DBuf W((size_t)n * TRD_NB, st);
  DBuf XW((size_t)n * 2 * TRD_NB, st), YW((size_t)n * 2 * TRD_NB, st);
  const int64_t gmax = (n + CRW - 1) / CRW;
  DBuf part_norm(gmax, st), part_wv(gmax, st), dpart((size_t)gmax * 2 * TRD_NB, st);
  DBuf wtmp(n, st), tvec(2 * TRD_NB, st), slots(2, st);  // slots: alpha, scale
  DBuf swork(symv_work_size(n), st);
  SymvMap tmap;  // the whole matrix; each column's trailing block by coordinates
  const bool tma_ok = !(g_sytrd_dbg & 1) && symv_map_make(&tmap, A, n, n, lda);
  // TMA path: 3 launches per column (the w kernel folded into the next column kernel)
  const bool fusew = tma_ok && !(g_sytrd_dbg & 8);
  DBuf vav(imax64(symv_tma_ctas(n), 1), st);
  double* alpha_buf = slots.p;
  double* scale_buf = slots.p + 1;
  // Each panel's ~260 dependent launches (4 per column) are captured once into a CUDA
  // graph and replayed (cudaGraphExecUpdate reuses the executable across panels).
  const bool use_graph = !(g_sytrd_dbg & 4);
  cudaGraphExec_t exec = nullptr;
  // capture on a private stream (the context stream may be the legacy default stream,
  // which cannot be captured); the graph itself is launched on st
  cudaStream_t sc = st;
  if (use_graph) EM_CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  // debug (EM_SYTRD_PANEL_TIMES set): per-panel chain times printed to stderr
  const bool ptimes = getenv("EM_SYTRD_PANEL_TIMES") != nullptr;
  std::vector<cudaEvent_t> pev;
  for (int64_t i0 = 0; i0 < n; i0 += TRD_NB) {
    const int w = (int)imin64(TRD_NB, n - i0);
    if (use_graph) EM_CK(cudaStreamBeginCapture(sc, cudaStreamCaptureModeThreadLocal));
    int64_t gw_prev = 0, nvav_prev = 0;
    bool last = false;
    auto col_launch = [&](int64_t c, int i, int upd) {
      const int64_t G = (n - c + CRW - 1) / CRW;
      ColW cw;
      if (fusew) {
        cw.tvec = tvec.p;
        cw.vav = vav.p;
        cw.nvav = nvav_prev;
        cw.scale = scale_buf;
        launch_pdl(latrd_col_kernel<true>, dim3((unsigned)G), dim3(RT), 0, sc, n, A, lda, i0, c,
                   i, upd, W.p, (int64_t)n, (const double*)wtmp.p, (const double*)part_wv.p,
                   gw_prev, (const double*)tau, part_norm.p, dpart.p, alpha_buf, d, cw);
      } else {
        launch_pdl(latrd_col_kernel<false>, dim3((unsigned)G), dim3(RT), 0, sc, n, A, lda, i0,
                   c, i, upd, W.p, (int64_t)n, (const double*)wtmp.p, (const double*)part_wv.p,
                   gw_prev, (const double*)tau, part_norm.p, dpart.p, alpha_buf, d, cw);
      }
    };
    for (int i = 0; i < w; ++i) {
      const int64_t c = i0 + i;
      const int64_t G = (n - c + CRW - 1) / CRW;
      col_launch(c, i, 1);
      if (c == n - 1) {
        last = true;
        break;
      }
      const int64_t m = n - c - 1;
      SymvLarfg lf;
      lf.part = part_norm.p;
      lf.nparts = G;
      lf.alpha = alpha_buf;
      lf.tau = tau + c;
      lf.e = e + c;
      lf.scale = scale_buf;
      if (fusew) lf.vav = vav.p;
      LatrdT lt;
      lt.i = i;
      lt.G = G;
      lt.dpart = dpart.p;
      lt.wr1 = W.p + (c + 1 - i0);
      lt.ldw = n;
      lt.ar1 = A + (c + 1) + i0 * lda;
      lt.lda = lda;
      lt.scale = scale_buf;
      lt.t = tvec.p;
      // wtmp[c+1:] = A22 v with dlarfg folded into the symv and the panel products t
      if (tma_ok)
        symv_tma(sc, tmap, c + 1, m, 1.0, A + (c + 1) + c * lda, 0.0, wtmp.p + (c + 1), swork.p,
                 &lf, &lt, !(g_sytrd_dbg & 2));
      else
        symv_lower_latrd(sc, m, A + (c + 1) + (c + 1) * lda, lda, A + (c + 1) + c * lda,
                         wtmp.p + (c + 1), swork.p, lf, lt);
      const int64_t gw = (m + CRW - 1) / CRW;
      if (!fusew)
        launch_pdl(latrd_w_kernel, dim3((unsigned)gw), dim3(RT), 0, sc, n, A, lda, i0, c, i,
                   (const double*)W.p, (int64_t)n, wtmp.p, (const double*)tvec.p,
                   (const double*)tau, (const double*)scale_buf, part_wv.p);
      gw_prev = gw;
      nvav_prev = fusew ? symv_tma_ctas(m, c + 1) : 0;
    }
    if (!last) col_launch(i0 + w, w, 0);  // finish W[:, w-1] for the trailing update
    if (use_graph) {
      cudaGraph_t g = nullptr;
      EM_CK(cudaStreamEndCapture(sc, &g));
      bool ok = false;
      if (exec) {
        cudaGraphExecUpdateResultInfo info;
        ok = cudaGraphExecUpdate(exec, g, &info) == cudaSuccess;
        if (!ok) {
          cudaGetLastError();
          cudaGraphExecDestroy(exec);
          exec = nullptr;
        }
      }
      if (!ok) EM_CK(cudaGraphInstantiate(&exec, g, 0));
      if (ptimes) {
        pev.resize(pev.size() + 2);
        cudaEventCreate(&pev[pev.size() - 2]);
        cudaEventCreate(&pev.back());
        cudaEventRecord(pev[pev.size() - 2], st);
      }
      EM_CK(cudaGraphLaunch(exec, st));
      if (ptimes) cudaEventRecord(pev.back(), st);
      cudaGraphDestroy(g);
    }
    const int64_t t0 = i0 + w;
    const int64_t mt = n - t0;
    if (mt > 0) {
      Stage s(st, ST_SYTRD_SYR2K);
      // A22 -= V W^T + W V^T as one K = 2w lower GEMM: [V | W] [W | V]^T
      copy_matrix(st, false, mt, w, A + t0 + i0 * lda, lda, XW.p, n);
      copy_matrix(st, false, mt, w, W.p + (t0 - i0), n, XW.p + (int64_t)w * n, n);
      copy_matrix(st, false, mt, w, W.p + (t0 - i0), n, YW.p, n);
      copy_matrix(st, false, mt, w, A + t0 + i0 * lda, lda, YW.p + (int64_t)w * n, n);
      EM_CK(gemm(st, false, true, mt, mt, 2 * w, -1.0, XW.p, n, YW.p, n, 1.0,
                 A + t0 + t0 * lda, lda, true, 0));
    }
    restore_sub_kernel<<<1, TRD_NB, 0, st>>>(n, A, lda, i0, w, e);
    EM_LAUNCHED();
  }
  if (exec) {
    EM_CK(cudaStreamSynchronize(st));
    cudaGraphExecDestroy(exec);
  }
  for (size_t k = 0; k + 1 < pev.size(); k += 2) {
    float t = 0.f;
    cudaEventElapsedTime(&t, pev[k], pev[k + 1]);
    fprintf(stderr, "sytrd_panel %zu m %lld ms %.4f\n", k / 2,
            (long long)(n - (int64_t)(k / 2) * TRD_NB), t);
    cudaEventDestroy(pev[k]);
    cudaEventDestroy(pev[k + 1]);
  }
  if (use_graph) cudaStreamDestroy(sc);
}

// ---- ormtr ----------------------------------------------------------------------

// Explicit V block for reflectors i0..i0+w-1 whose vectors start `off` rows below
// their column (off = 1 for sytrd, = band width for sy2sb); rows i0+off .. n-1:
// V[r, k] = 0 (r < k), 1 (r == k), A[i0+off+r, i0+k] (r > k).
__global__ void build_v_kernel(int64_t n, const double* A, int64_t lda, int64_t i0, int w,
                               int64_t off, double* V, int64_t ldv) {
  const int64_t m = n - i0 - off;
  const int k = blockIdx.y;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x) {
    double v;
    if (r < k)
      v = 0.0;
    else if (r == k)
      v = 1.0;
    else
      v = A[(i0 + off + r) + (i0 + k) * lda];
    V[r + k * ldv] = v;
  }
}

// Wide-block larft: T (w x w upper, ld ldt, global memory) from G = V^T V, w <= 256.
__global__ void larft_wide_kernel(int w, const double* __restrict__ G, int64_t ldg,
                                  const double* __restrict__ tau, int64_t c0, double* T,
                                  int64_t ldt) {
  __shared__ double gk[256];
  const int tid = threadIdx.x;
  for (int i = tid; i < w * w; i += blockDim.x) T[(i % w) + (i / w) * ldt] = 0.0;
  __syncthreads();
  for (int k = 0; k < w; ++k) {
    const double tk = tau[c0 + k];
    if (tid < k) gk[tid] = G[tid + k * ldg];
    __syncthreads();
    if (tid < k) {
      double s = 0.0;
      for (int j = tid; j < k; ++j) s = fma(T[tid + j * ldt], gk[j], s);
      T[tid + k * ldt] = -tk * s;
    }
    if (tid == 0) T[k + k * ldt] = tk;
    __syncthreads();
  }
}

// larft for the diagonal 128-blocks of T (w x w, ld ldt): CTA `half` builds the block of
// reflectors [half*w1, half*w1 + 128) (w1 = 128 unless w < 128) from the matching diagonal
// block of G = V^T V in shared memory; also zeroes the blocks of T left of it.
EM_DEVINL void larft_smem_body(int half, int w, int w1, const double* __restrict__ G,
                               int64_t ldg, const double* __restrict__ tau, int64_t c0,
                               double* T, int64_t ldt, double* Ts, double* gk) {
  constexpr int LD = 129;
  const int off = half * w1;
  const int bw = w - off < w1 ? w - off : w1;
  const int tid = threadIdx.x;
  for (int i = tid; i < 128 * LD; i += blockDim.x) Ts[i] = 0.0;
  __syncthreads();
  for (int k = 0; k < bw; ++k) {
    const double tk = tau[c0 + off + k];
    if (tid < k) gk[tid] = G[(off + tid) + (off + k) * ldg];
    __syncthreads();
    if (tid < k) {
      double s = 0.0;
      for (int j = tid; j < k; ++j) s = fma(Ts[tid + j * LD], gk[j], s);
      Ts[tid + k * LD] = -tk * s;
    }
    if (tid == 0) Ts[k + k * LD] = tk;
    __syncthreads();
  }
  for (int i = tid; i < bw * bw; i += blockDim.x) {
    const int r = i % bw, c = i / bw;
    T[(off + r) + (off + c) * ldt] = Ts[r + c * LD];
  }
  // strictly-lower block row: rows [off, off + bw) x columns [0, off)
  for (int i = tid; i < bw * off; i += blockDim.x) T[(off + i % bw) + (i / bw) * ldt] = 0.0;
}

__global__ void __launch_bounds__(128) larft_smem_kernel(int w, int w1,
                                                         const double* __restrict__ G,
                                                         int64_t ldg,
                                                         const double* __restrict__ tau,
                                                         int64_t c0, double* T, int64_t ldt) {
  extern __shared__ double Ts[];  // 128 x 129
  __shared__ double gk[128];
  larft_smem_body(blockIdx.x, w, w1, G, ldg, tau, c0, T, ldt, Ts, gk);
}

// every ORM_NB-reflector block of ormqr at once: block p = blockIdx.y (G, T with
// stride nb^2, ld = its width), 128-reflector sub-block = blockIdx.x
__global__ void __launch_bounds__(128) larft_batched_kernel(int64_t nref, int nb,
                                                            const double* __restrict__ G,
                                                            const double* __restrict__ tau,
                                                            double* T, int64_t p0) {
  extern __shared__ double Ts[];
  __shared__ double gk[128];
  const int64_t p = blockIdx.y;  // block p0 + p, stored at index p
  const int64_t c0 = (p0 + p) * nb;
  const int w = (int)imin64(nb, nref - c0);
  const int w1 = w < 128 ? w : 128;
  if ((int)blockIdx.x * w1 >= w) return;
  const size_t str = (size_t)nb * nb;
  larft_smem_body(blockIdx.x, w, w1, G + p * str, w, tau, c0, T + p * str, w, Ts, gk);
}

// Z <- Q Z, Q = H(0)...H(n-2), in blocks of ORM_NB reflectors (compact WY,
// three DMMA GEMMs per block; a wide block keeps the rank-w updates of Z
// compute-bound instead of re-streaming Z once per 64 reflectors: the accumulating
// rank-256 update ran at 32 TF/s, a rank-512 one runs at 34, tools/gemm_probe.py).
constexpr int ORM_NB = 512;

void ormtr_lower(cudaStream_t st, int64_t n, int64_t m, const double* A, int64_t lda,
                 const double* tau, double* Z, int64_t ldz) {
  ormqr_lower_off(st, n, n - 1, 1, m, A, lda, tau, Z, ldz);  // reflectors H(0..n-2)
}

// Z <- H(0) ... H(nref-1) Z for reflectors stored below the `off`-th subdiagonal of A.
// The V blocks and their T factors do not depend on Z: all of them are built first
// (one launch each for V, the grouped G = V^T V, the larft halves of every block in
// one grid, the grouped T12 joins), so only the three Z GEMMs per block are sequential.
void ormqr_lower_off(cudaStream_t st, int64_t n, int64_t nref, int64_t off, int64_t m,
                     const double* A, int64_t lda, const double* tau, double* Z, int64_t ldz,
                     bool trans) {
  if (nref <= 0 || m <= 0) return;
  const int64_t npan = (nref + ORM_NB - 1) / ORM_NB;
  const size_t vstride = (size_t)n * ORM_NB, tstride = (size_t)ORM_NB * ORM_NB;
  // the V blocks are built a chunk of panels at a time (about 2 GiB), so the workspace
  // stays O(n) columns instead of the n x nref of all blocks at once (N = 120,000 fits)
  const int64_t chunk =
      imax64(1, imin64(npan, (int64_t)((2ull << 30) / (vstride * sizeof(double)))));
  const int64_t nch = (npan + chunk - 1) / chunk;
  DBuf V(vstride * chunk, st), G(tstride * chunk, st), T(tstride * chunk, st),
      T1G(tstride * chunk, st);
  DBuf W1((size_t)ORM_NB * m, st), W2((size_t)ORM_NB * m, st);
  EM_CK(cudaFuncSetAttribute(larft_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(128 * 129 * sizeof(double))));
  EM_CK(cudaFuncSetAttribute(larft_batched_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(128 * 129 * sizeof(double))));
  // Q Z: blocks last to first with T; Q^T Z: first to last with T^T
  for (int64_t cs = 0; cs < nch; ++cs) {
    const int64_t ci = trans ? cs : nch - 1 - cs;
    const int64_t p0 = ci * chunk, p1 = imin64(npan, p0 + chunk), np = p1 - p0;
    // T of a block from its 128-reflector diagonal blocks (larft) joined pairwise, then the
    // pairs joined: T_ab = -T_a G_ab T_b (two grouped products per level)
    std::vector<GemmArgs> gg, jx[2], jt[2];
    int max_g = 1, max_j[2] = {1, 1};
    for (int64_t p = p0; p < p1; ++p) {
      const int64_t i0 = p * ORM_NB;
      const int w = (int)imin64(ORM_NB, nref - i0);
      const int64_t mr = n - i0 - off;
      double* Vp = V.p + (p - p0) * vstride;
      dim3 grid((unsigned)imax64(1, imin64((mr + 255) / 256, 64)), (unsigned)w);
      build_v_kernel<<<grid, 256, 0, st>>>(n, A, lda, i0, w, off, Vp, n);
      EM_LAUNCHED();
      double* Gp = G.p + (p - p0) * tstride;
      gg.push_back(GemmArgs{w, w, mr, Vp, n, Vp, n, Gp, w, 1.0, 0.0, 0});
      max_g = (int)imax64(max_g, ((w + 127) / 128) * ((w + 63) / 64));
      double* Tp = T.p + (p - p0) * tstride;
      double* Xp = T1G.p + (p - p0) * tstride;
      auto join = [&](int lvl, int a0, int na, int b0, int nb2, double* X) {
        if (nb2 <= 0) return;
        jx[lvl].push_back(GemmArgs{na, nb2, na, Tp + a0 + (int64_t)a0 * w, w,
                                   Gp + a0 + (int64_t)b0 * w, w, X, na, 1.0, 0.0, 0});
        jt[lvl].push_back(GemmArgs{na, nb2, nb2, X, na, Tp + b0 + (int64_t)b0 * w, w,
                                   Tp + a0 + (int64_t)b0 * w, w, -1.0, 0.0, 0});
        max_j[lvl] = (int)imax64(max_j[lvl], ((na + 127) / 128) * ((nb2 + 63) / 64));
      };
      join(0, 0, 128, 128, (int)imin64(128, w - 128), Xp);
      join(0, 256, 128, 384, (int)imin64(128, w - 384), Xp + 128 * 128);
      join(1, 0, 256, 256, w - 256, Xp + 2 * 128 * 128);
    }
    DArr<GemmArgs> dgg(gg.size(), st);
    EM_CK(cudaMemcpyAsync(dgg.p, gg.data(), gg.size() * sizeof(GemmArgs),
                          cudaMemcpyHostToDevice, st));
    EM_CK(gemm_grouped(st, true, false, dgg.p, (int)gg.size(), max_g));
    larft_batched_kernel<<<dim3(ORM_NB / 128, (unsigned)np), 128,
                           (size_t)128 * 129 * sizeof(double), st>>>(nref, ORM_NB, G.p, tau, T.p,
                                                                     p0);
    EM_LAUNCHED();
    DArr<GemmArgs> djx[2], djt[2];
    for (int lvl = 0; lvl < 2; ++lvl) {
      if (jx[lvl].empty()) continue;
      djx[lvl].alloc(jx[lvl].size(), st);
      djt[lvl].alloc(jt[lvl].size(), st);
      EM_CK(cudaMemcpyAsync(djx[lvl].p, jx[lvl].data(), jx[lvl].size() * sizeof(GemmArgs),
                            cudaMemcpyHostToDevice, st));
      EM_CK(cudaMemcpyAsync(djt[lvl].p, jt[lvl].data(), jt[lvl].size() * sizeof(GemmArgs),
                            cudaMemcpyHostToDevice, st));
      EM_CK(gemm_grouped(st, false, false, djx[lvl].p, (int)jx[lvl].size(), max_j[lvl]));
      EM_CK(gemm_grouped(st, false, false, djt[lvl].p, (int)jt[lvl].size(), max_j[lvl]));
    }
    for (int64_t s = 0; s < np; ++s) {
      const int64_t p = trans ? p0 + s : p1 - 1 - s;
      const int64_t i0 = p * ORM_NB;
      const int w = (int)imin64(ORM_NB, nref - i0);
      const int64_t mr = n - i0 - off;
      const double* Vp = V.p + (p - p0) * vstride;
      const double* Tp = T.p + (p - p0) * tstride;
      double* Zs = Z + (i0 + off);
      EM_CK(gemm(st, true, false, w, m, mr, 1.0, Vp, n, Zs, ldz, 0.0, W1.p, w));
      EM_CK(gemm(st, trans, false, w, m, w, 1.0, Tp, w, W1.p, w, 0.0, W2.p, w));
      EM_CK(gemm(st, false, false, mr, m, w, -1.0, Vp, n, W2.p, w, 1.0, Zs, ldz));
    }
    EM_CK(cudaStreamSynchronize(st));  // host argument arrays, V/G/T reuse by the next chunk
  }
}

}  // namespace em
