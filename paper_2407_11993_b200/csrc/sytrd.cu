// Householder tridiagonalisation (lower, blocked: latrd panels + syr2k) and the
// blocked back-transform Z <- Q Z (ormtr). Together with stedc.cu this replaces
// the reference's cyclic Jacobi eigensolver (_kernels.py:82-141), which is
// O(sweeps N^3) sequential; the result (eigenvalues, invariant subspaces) is
// the same to round-off.
//
// Per panel column the memory-bound part is one lower-triangle symv over the
// trailing matrix (symv.cu); the rank-2k trailing update and the
// back-transform run on the DMMA GEMM. The per-column panel work (latrd) uses
// 8 threads per row so that a 16k-row column update keeps ~130k threads busy.
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

constexpr int TRD_NB = 64;   // panel width
constexpr int RT = 256;
constexpr int TPR = 8;                 // threads per row in the panel kernels
constexpr int ROWS_PER_CTA = RT / TPR;  // 32

EM_DEVINL double group_sum8(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

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

// A[c:n, c] -= A[c:n, i0:c] W[c, 0:i]^T + W[c:n, 0:i] A[c, i0:c]^T, then per-CTA
// partial sums of squares of the updated A[c+2:n, c] (the dlarfg norm).
__global__ void __launch_bounds__(RT) latrd_colupd_kernel(int64_t n, double* A, int64_t lda,
                                                          int64_t i0, int64_t c,
                                                          const double* __restrict__ W,
                                                          int64_t ldw, double* part,
                                                          double* alpha_buf) {
  const int i = (int)(c - i0);
  __shared__ double wr[TRD_NB], ar[TRD_NB], red[RT / 32];
  for (int k = threadIdx.x; k < i; k += blockDim.x) {
    wr[k] = W[(c - i0) + k * ldw];  // W row c (W rows are indexed from i0)
    ar[k] = A[c + (i0 + k) * lda];  // A row c
  }
  __syncthreads();
  const int sub = threadIdx.x & (TPR - 1);
  const int64_t r = c + blockIdx.x * (int64_t)ROWS_PER_CTA + threadIdx.x / TPR;
  double ss = 0.0;
  if (r < n) {
    double s = 0.0;
    for (int k = sub; k < i; k += TPR) {
      s = fma(A[r + (i0 + k) * lda], wr[k], s);
      s = fma(W[(r - i0) + k * ldw], ar[k], s);
    }
    s = group_sum8(s);
    if (sub == 0) {
      const double v = A[r + c * lda] - s;
      if (i > 0) A[r + c * lda] = v;
      if (r >= c + 2) ss = v * v;
      if (r == c + 1) *alpha_buf = v;  // dlarfg's alpha, read by larfg_kernel
    }
  } else {
    group_sum8(0.0);
  }
  const double t = block_sum(ss, red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// dlarfg on x = A[c+1:n, c] with ||x[1:]||^2 = sum(part): beta, tau; v = [1, x[1:]/(alpha-beta)];
// e[c] = beta; d[c] = A[c,c]. Every CTA reduces the partials itself and scales its slice.
__global__ void __launch_bounds__(RT) larfg_kernel(int64_t n, double* A, int64_t lda, int64_t c,
                                                   const double* __restrict__ part, int nparts,
                                                   const double* __restrict__ alpha_buf,
                                                   double* d, double* e, double* tau) {
  __shared__ double red[RT / 32];
  __shared__ double sc;
  double s = 0.0;
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) s += part[p];
  const double tot = block_sum(s, red);
  const double alpha = *alpha_buf;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    d[c] = A[c + c * lda];
    A[(c + 1) + c * lda] = 1.0;  // v[0]; alpha itself is read from alpha_buf
  }
  if (threadIdx.x == 0) {
    const double xnorm = sqrt(tot);
    double scale = 0.0;
    if (xnorm == 0.0) {
      if (blockIdx.x == 0) {
        tau[c] = 0.0;
        e[c] = alpha;
      }
    } else {
      const double beta = -copysign(hypot(alpha, xnorm), alpha);
      scale = 1.0 / (alpha - beta);
      if (blockIdx.x == 0) {
        tau[c] = (beta - alpha) / beta;
        e[c] = beta;
      }
    }
    sc = scale;
  }
  __syncthreads();
  const double f = sc;
  if (f != 0.0)
    for (int64_t r = c + 2 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x)
      A[r + c * lda] *= f;
  // every CTA has read alpha above; make sure all CTAs did before CTA 0 overwrites it
}

__global__ void larfg_finish_kernel(double* A, int64_t lda, int64_t c, double* d) {
  if (threadIdx.x == 0) {
    d[c] = A[c + c * lda];
    A[(c + 1) + c * lda] = 1.0;
  }
}

// Partial dots: tmp[which][k] partials over row chunks of  W[c+1:, k].v (which 0)
// and A[c+1:, i0+k].v (which 1). grid (chunks, ceil(2i/8)); warp per column.
constexpr int DOT_ROWS = 2048;
__global__ void __launch_bounds__(RT) latrd_dots_kernel(int64_t n, const double* A, int64_t lda,
                                                        int64_t i0, int64_t c, const double* W,
                                                        int64_t ldw, double* dpart, int nchunk) {
  const int i = (int)(c - i0);
  const int col = blockIdx.y * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (col >= 2 * i) return;
  const int which = col / i, k = col % i;
  const int64_t rb = c + 1 + blockIdx.x * (int64_t)DOT_ROWS;
  const int64_t re = imin64(n, rb + DOT_ROWS);
  const double* v = A + c * lda;
  const double* colp = which == 0 ? W + k * ldw - i0 : A + (i0 + k) * lda;
  double s = 0.0;
  for (int64_t r = rb + lane; r < re; r += 32) s = fma(colp[r], v[r], s);
  s = warp_sum(s);
  if (lane == 0) dpart[(which * TRD_NB + k) * nchunk + blockIdx.x] = s;
}

// w = tau*(w - A_p t1 - W_p t2), t1/t2 summed from the chunk partials; per-CTA
// partial dot of w and v.
__global__ void __launch_bounds__(RT) latrd_wcol_kernel(int64_t n, const double* A, int64_t lda,
                                                        int64_t i0, int64_t c, double* W,
                                                        int64_t ldw, const double* dpart,
                                                        int nchunk, const double* tau,
                                                        double* part) {
  const int i = (int)(c - i0);
  __shared__ double t1[TRD_NB], t2[TRD_NB], red[RT / 32];
  for (int q = threadIdx.x; q < 2 * i; q += blockDim.x) {
    const int which = q / i, k = q % i;
    double s = 0.0;
    for (int ch = 0; ch < nchunk; ++ch) s += dpart[(which * TRD_NB + k) * nchunk + ch];
    if (which == 0)
      t1[k] = s;
    else
      t2[k] = s;
  }
  __syncthreads();
  const double tc = tau[c];
  const double* v = A + c * lda;
  double* w = W + i * ldw;
  const int sub = threadIdx.x & (TPR - 1);
  const int64_t r = c + 1 + blockIdx.x * (int64_t)ROWS_PER_CTA + threadIdx.x / TPR;
  double dd = 0.0;
  if (r < n) {
    double s = 0.0;
    for (int k = sub; k < i; k += TPR) {
      s = fma(A[r + (i0 + k) * lda], t1[k], s);
      s = fma(W[(r - i0) + k * ldw], t2[k], s);
    }
    s = group_sum8(s);
    if (sub == 0) {
      const double x = tc * (w[r - i0] - s);
      w[r - i0] = x;
      dd = x * v[r];
    }
  } else {
    group_sum8(0.0);
  }
  const double t = block_sum(dd, red);
  if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// w += alpha v,  alpha = -tau/2 * (w.v)
__global__ void latrd_wfix_kernel(int64_t n, const double* A, int64_t lda, int64_t i0, int64_t c,
                                  double* W, int64_t ldw, const double* tau, const double* part,
                                  int nparts) {
  __shared__ double red[RT / 32];
  double s = 0.0;
  for (int p = threadIdx.x; p < nparts; p += blockDim.x) s += part[p];
  __shared__ double alpha;
  const double tot = block_sum(s, red);
  if (threadIdx.x == 0) alpha = -0.5 * tau[c] * tot;
  __syncthreads();
  const int i = (int)(c - i0);
  const double* v = A + c * lda;
  double* w = W + i * ldw;
  const double a = alpha;
  for (int64_t r = c + 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
       r += (int64_t)gridDim.x * blockDim.x)
    w[r - i0] = fma(a, v[r], w[r - i0]);
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

// em_config(EM_CFG_SYTRD_FUSED). The fused cooperative panel kernel (sytrd_fused.cu) is
// experimental: slower than the graph path at N = 16k and not yet race-free; off.
bool g_sytrd_fused = false;

void sytrd_lower(cudaStream_t st, int64_t n, double* A, int64_t lda, double* d, double* e,
                 double* tau) {
  if (n <= 0) return;
  if (g_sytrd_fused && n > 1) {
    sytrd_lower_fused(st, n, A, lda, d, e, tau);
    return;
  }
  if (n == 1) {
    set_diag_kernel<<<1, 32, 0, st>>>(n, A, lda, 0, d);
    EM_LAUNCHED();
    return;
  }
  DBuf W((size_t)n * TRD_NB, st);
  DBuf XW((size_t)n * 2 * TRD_NB, st), YW((size_t)n * 2 * TRD_NB, st);
  const int max_rows_ctas = (int)((n + ROWS_PER_CTA - 1) / ROWS_PER_CTA);
  DBuf part(imax64(max_rows_ctas, 1), st);
  const int max_chunks = (int)((n + DOT_ROWS - 1) / DOT_ROWS);
  DBuf dpart((size_t)2 * TRD_NB * max_chunks, st);
  DBuf swork(symv_work_size(n), st);
  DBuf abuf(1, st);
  // Each panel's ~450 dependent small launches are captured once into a CUDA graph
  // and replayed (cudaGraphExecUpdate reuses the executable across panels), which
  // removes most of the per-launch gap that dominates the short columns.
  const bool use_graph = true;
  cudaGraphExec_t exec = nullptr;
  // capture on a private stream (the context stream may be the legacy default stream,
  // which cannot be captured); the graph itself is launched on st
  cudaStream_t sc = st;
  if (use_graph) EM_CK(cudaStreamCreateWithFlags(&sc, cudaStreamNonBlocking));
  for (int64_t i0 = 0; i0 < n; i0 += TRD_NB) {
    const int w = (int)imin64(TRD_NB, n - i0);
    if (use_graph) EM_CK(cudaStreamBeginCapture(sc, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < w; ++i) {
      const int64_t c = i0 + i;
      const int gcol = (int)((n - c + ROWS_PER_CTA - 1) / ROWS_PER_CTA);
      latrd_colupd_kernel<<<gcol, RT, 0, sc>>>(n, A, lda, i0, c, W.p, n, part.p, abuf.p);
      EM_LAUNCHED();
      if (c == n - 1) {
        set_diag_kernel<<<1, 32, 0, sc>>>(n, A, lda, c, d);
        EM_LAUNCHED();
        break;
      }
      const int64_t m = n - c - 1;
      const int gsc = (int)imax64(1, imin64((m + RT - 1) / RT, 2 * num_sms()));
      larfg_kernel<<<gsc, RT, 0, sc>>>(n, A, lda, c, part.p, gcol, abuf.p, d, e, tau);
      EM_LAUNCHED();
      // W[c+1:, i] = A22 v  (A22 = trailing lower triangle)
      symv_lower(sc, m, 1.0, A + (c + 1) + (c + 1) * lda, lda, A + (c + 1) + c * lda, 0.0,
                 W.p + (c + 1 - i0) + (int64_t)i * n, swork.p);
      const int nchunk = (int)((m + DOT_ROWS - 1) / DOT_ROWS);
      if (i > 0) {
        dim3 gd((unsigned)nchunk, (unsigned)((2 * i + 7) / 8));
        latrd_dots_kernel<<<gd, RT, 0, sc>>>(n, A, lda, i0, c, W.p, n, dpart.p, nchunk);
        EM_LAUNCHED();
      }
      const int gw = (int)((m + ROWS_PER_CTA - 1) / ROWS_PER_CTA);
      latrd_wcol_kernel<<<gw, RT, 0, sc>>>(n, A, lda, i0, c, W.p, n, dpart.p, nchunk, tau,
                                           part.p);
      EM_LAUNCHED();
      const int gf = (int)imax64(1, imin64((m + RT - 1) / RT, 2 * num_sms()));
      latrd_wfix_kernel<<<gf, RT, 0, sc>>>(n, A, lda, i0, c, W.p, n, tau, part.p, gw);
      EM_LAUNCHED();
    }
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
      EM_CK(cudaGraphLaunch(exec, st));
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

// larft for the diagonal 128-blocks of T (w x w, ld ldt): CTA b builds the block of
// reflectors [b*w1, ...) from the matching diagonal block of G = V^T V in shared
// memory; also zeroes the strictly-lower blocks of T.
__global__ void __launch_bounds__(128) larft_smem_kernel(int w, int w1,
                                                         const double* __restrict__ G,
                                                         int64_t ldg,
                                                         const double* __restrict__ tau,
                                                         int64_t c0, double* T, int64_t ldt) {
  extern __shared__ double Ts[];  // 128 x 129
  __shared__ double gk[128];
  constexpr int LD = 129;
  const int off = blockIdx.x * w1;
  const int bw = blockIdx.x == 0 ? w1 : w - w1;
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
  if (blockIdx.x == 1)  // strictly-lower off-diagonal block
    for (int i = tid; i < bw * w1; i += blockDim.x) T[(w1 + i % bw) + (i / bw) * ldt] = 0.0;
}

// Z <- Q Z, Q = H(0)...H(n-2), in blocks of ORM_NB reflectors (compact WY,
// three DMMA GEMMs per block; a wide block keeps the rank-w updates of Z
// compute-bound instead of re-streaming Z once per 64 reflectors).
constexpr int ORM_NB = 256;

void ormtr_lower(cudaStream_t st, int64_t n, int64_t m, const double* A, int64_t lda,
                 const double* tau, double* Z, int64_t ldz) {
  ormqr_lower_off(st, n, n - 1, 1, m, A, lda, tau, Z, ldz);  // reflectors H(0..n-2)
}

// Z <- H(0) ... H(nref-1) Z for reflectors stored below the `off`-th subdiagonal of A.
void ormqr_lower_off(cudaStream_t st, int64_t n, int64_t nref, int64_t off, int64_t m,
                     const double* A, int64_t lda, const double* tau, double* Z, int64_t ldz) {
  if (nref <= 0 || m <= 0) return;
  DBuf V((size_t)n * ORM_NB, st), G((size_t)ORM_NB * ORM_NB, st), T((size_t)ORM_NB * ORM_NB, st);
  DBuf W1((size_t)ORM_NB * m, st), W2((size_t)ORM_NB * m, st);
  const int64_t npan = (nref + ORM_NB - 1) / ORM_NB;
  EM_CK(cudaFuncSetAttribute(larft_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(128 * 129 * sizeof(double))));
  for (int64_t p = npan - 1; p >= 0; --p) {
    const int64_t i0 = p * ORM_NB;
    const int w = (int)imin64(ORM_NB, nref - i0);
    const int64_t mr = n - i0 - off;  // rows of V
    dim3 grid((unsigned)imax64(1, imin64((mr + 255) / 256, 64)), (unsigned)w);
    build_v_kernel<<<grid, 256, 0, st>>>(n, A, lda, i0, w, off, V.p, n);
    EM_LAUNCHED();
    EM_CK(gemm(st, true, false, w, w, mr, 1.0, V.p, n, V.p, n, 0.0, G.p, w));
    // T from two 128-halves built in shared memory, joined by T12 = -T1 G12 T2
    const int w1 = imin64(w, 128), w2 = w - w1;
    larft_smem_kernel<<<w2 > 0 ? 2 : 1, 128, (size_t)128 * 129 * sizeof(double), st>>>(
        w, w1, G.p, w, tau, i0, T.p, w);
    EM_LAUNCHED();
    if (w2 > 0) {
      EM_CK(gemm(st, false, false, w1, w2, w1, 1.0, T.p, w, G.p + (int64_t)w1 * w, w, 0.0,
                 W1.p, w1));
      EM_CK(gemm(st, false, false, w1, w2, w2, -1.0, W1.p, w1, T.p + w1 + (int64_t)w1 * w, w,
                 0.0, T.p + (int64_t)w1 * w, w));
    }
    double* Zs = Z + (i0 + off);
    EM_CK(gemm(st, true, false, w, m, mr, 1.0, V.p, n, Zs, ldz, 0.0, W1.p, w));
    EM_CK(gemm(st, false, false, w, m, w, 1.0, T.p, w, W1.p, w, 0.0, W2.p, w));
    EM_CK(gemm(st, false, false, mr, m, w, -1.0, V.p, n, W2.p, w, 1.0, Zs, ldz));
  }
}

}  // namespace em
