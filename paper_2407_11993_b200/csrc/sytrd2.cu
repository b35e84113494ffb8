// Two-stage tridiagonalisation for the symmetric eigensolve (north-star (a)):
//
//   stage 1 (sy2sb)  dense -> band of width b = 64: per 64-column panel a
//                    Householder QR (one cooperative kernel: the panel lives in
//                    shared memory across all SMs, two grid barriers per column),
//                    then the two-sided update A22 <- Q^T A22 Q as DMMA GEMMs
//                    (X = A22 V T, W = X - V T^T V^T X / 2, A22 -= V W^T + W V^T).
//                    No matrix-vector product over the trailing matrix: the
//                    memory-bound symv of one-stage sytrd disappears.
//   stage 2 (sb2st)  band -> tridiagonal by bulge chasing: one persistent kernel,
//                    sweep s owned by CTA s mod P, task k of sweep s waits until
//                    sweep s-1 finished task k+2 (release/acquire progress flags);
//                    the band (2b+1 diagonals, bulge room) stays L2-resident.
//   back-transform   Z <- Q2 Z: stage-2 reflectors of b consecutive sweeps and the
//                    same block position form one compact-WY block (V: 2b-1 x b
//                    parallelogram, T precomputed per block); blocks are applied per
//                    sweep group (last group first) in ascending position order,
//                    which respects every non-commuting pair. A persistent kernel
//                    gives each CTA a column slab of Z and runs the whole sequence
//                    on DMMA in shared memory. Then Z <- Q1 Z (compact WY, GEMM).
//
// Replaces the reference's cyclic Jacobi (_kernels.py:82-141) for large n.
#include <algorithm>
#include <queue>
#include <vector>

#include "common.cuh"
#include "comm.h"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

namespace em {

constexpr int B2 = kBand;  // 64

// ---- grid-wide barrier (all CTAs co-resident: cooperative launch) ----------------
struct GridBar {
  unsigned int count;
  unsigned int gen;
};

EM_DEVINL void grid_sync(GridBar* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* vgen = &bar->gen;
    const unsigned int g = *vgen;
    __threadfence();
    if (atomicAdd(&bar->count, 1u) == nblocks - 1) {
      bar->count = 0;
      __threadfence();
      atomicAdd(&bar->gen, 1u);
    } else {
      while (*vgen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

EM_DEVINL double block_reduce_sum(double v, double* red) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : 0.0;
    t = warp_sum(t);
  }
  return t;  // valid in thread 0
}

// ---- stage 1: cooperative panel QR ----------------------------------------------
struct QRArgs {
  int64_t m;      // panel rows
  int nbw;        // panel columns (<= 64)
  int p;          // reflectors = min(m, nbw)
  double* P;      // panel (m x nbw, ld ldp), in place: R above, V below the diagonal
  int64_t ldp;
  double* tau;    // p
  double* part;   // 2 x (G*64 + 64) scratch (double-buffered by the column's parity)
  GridBar* bar;
  int R;          // rows per CTA
};

// GM: the panel is worked on in place in global memory (L2-resident) instead of shared
// memory — for panels taller than the CTAs' shared memory holds (m > ~59,000 rows).
//
// ONE grid barrier per column: from the unscaled column x = P[j+1:, j] every CTA publishes
// its partial sum of squares and its partial products d_c = x^T P[j+1:, c] (c > j), the
// owner of row j that row; behind the barrier every CTA forms beta, tau, scale and
// w_c = v^T P[:, c] = P[j, c] + scale d_c itself (v = scale x below the unit entry) and
// updates its own rows. (Two barriers per column — the norm, then the products with the
// scaled v — and a single thread summing the G partials cost 1.7 ms per panel at C3, 1.3 s
// of the band reduction on its critical path.) The partials are double-buffered by the
// column's parity: a CTA writing column j + 1's has passed barrier j, which every CTA
// reaches only after reading column j - 1's.
template <bool GM>
__global__ void __launch_bounds__(256) qr_panel_kernel(QRArgs a) {
  extern __shared__ double Ssm[];  // column-major [nbw][R]
  __shared__ double wsh[B2];
  __shared__ double rowsh[B2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned G = gridDim.x;
  const int64_t r0 = blockIdx.x * (int64_t)a.R;
  const int nr = (int)imax64(0, imin64(a.R, a.m - r0));
  double* S = GM ? a.P + r0 : Ssm;
  const int64_t ls = GM ? a.ldp : a.R;
  if (!GM) {
    for (int idx = tid; idx < nr * a.nbw; idx += blockDim.x) {
      const int lr = idx % nr, c = idx / nr;
      S[c * ls + lr] = a.P[(r0 + lr) + c * a.ldp];
    }
  }
  __syncthreads();
  const int chunk = (int)((G + 3) / 4);
  for (int j = 0; j < a.p; ++j) {
    double* Sj = S + j * ls;
    double* dotpart = a.part + (size_t)(j & 1) * ((size_t)G * B2 + B2);
    double* rowj = dotpart + (size_t)G * B2;
    // (a) partials over the own rows below row j: slot j = sum of squares, slot c = x^T P[:, c]
    for (int c = j + warp; c < a.nbw; c += 8) {
      const double* Sc = S + c * ls;
      double s = 0.0;
      for (int lr = lane; lr < nr; lr += 32)
        if (r0 + lr > j) s = fma(Sj[lr], Sc[lr], s);
      s = warp_sum(s);
      if (lane == 0) dotpart[(size_t)blockIdx.x * B2 + c] = s;
    }
    if (j >= r0 && j < r0 + nr)
      for (int c = j + tid; c < a.nbw; c += blockDim.x) rowj[c] = S[c * ls + (j - r0)];
    grid_sync(a.bar, G);
    // (b) totals in a fixed order: 4 threads per column, a contiguous quarter of the CTAs each
    {
      const int c = tid >> 2, q = tid & 3;
      double s = 0.0;
      if (c >= j && c < a.nbw) {
        // every load of the thread's quarter in flight at once (one L2 round trip for up to
        // 160 CTAs), summed in a fixed order
        const int b0 = q * chunk, b1 = (int)imin64(b0 + chunk, G);
        for (int bb = b0; bb < b1; bb += 40) {
          double t[40];
#pragma unroll
          for (int u = 0; u < 40; ++u)
            t[u] = bb + u < b1 ? __ldcg(dotpart + (size_t)(bb + u) * B2 + c) : 0.0;
#pragma unroll
          for (int u = 0; u < 40; ++u) s += t[u];
        }
      }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (q == 0 && c < a.nbw) {
        wsh[c] = s;
        rowsh[c] = c >= j ? __ldcg(rowj + c) : 0.0;
      }
    }
    __syncthreads();
    // (c) beta, tau, scale: identical in every thread of every CTA
    const double alpha = rowsh[j], xnorm = sqrt(wsh[j]);
    double beta = alpha, tau = 0.0, scale = 0.0;
    if (xnorm != 0.0) {
      beta = -copysign(hypot(alpha, xnorm), alpha);
      tau = (beta - alpha) / beta;
      scale = 1.0 / (alpha - beta);
    }
    if (blockIdx.x == 0 && tid == 0) a.tau[j] = tau;
    // (d) apply H_j to the remaining columns of the own rows: w_c = P[j, c] + scale d_c
    if (tau != 0.0) {
      // 64 row lanes x 4 column groups (no index divisions)
      const int lr0 = tid & 63;
      for (int c = j + 1 + (tid >> 6); c < a.nbw; c += 4) {
        const double twc = -tau * fma(scale, wsh[c], rowsh[c]);
        double* Sc = S + c * ls;
        for (int lr = lr0; lr < nr; lr += 64) {
          const int64_t r = r0 + lr;
          if (r >= j) Sc[lr] = fma(twc, (r == j) ? 1.0 : Sj[lr] * scale, Sc[lr]);
        }
      }
    }
    __syncthreads();
    for (int lr = tid; lr < nr; lr += blockDim.x) {
      const int64_t r = r0 + lr;
      if (r > j && scale != 0.0) Sj[lr] *= scale;
      else if (r == j) Sj[lr] = beta;
    }
    // (column j is not read again; the next column's wsh / rowsh writes come behind its
    // grid barrier)
  }
  __syncthreads();
  if (!GM) {
    for (int idx = tid; idx < nr * a.nbw; idx += blockDim.x) {
      const int lr = idx % nr, c = idx / nr;
      a.P[(r0 + lr) + c * a.ldp] = S[c * ls + lr];
    }
  }
}

__global__ void band_extract_kernel(int64_t n, int b, const double* __restrict__ A, int64_t lda,
                                    double* __restrict__ AB, int64_t ldab) {
  const int64_t c = blockIdx.x;
  for (int d = threadIdx.x; d < ldab; d += blockDim.x) {
    const int64_t r = c + d;
    AB[d + c * ldab] = (d <= b && r < n) ? A[r + c * lda] : 0.0;
  }
}

// larft (forward, columnwise) for w <= 128 reflectors from G = V^T V (sytrd.cu)
__global__ void __launch_bounds__(128) larft_smem_kernel(int w, int w1,
                                                         const double* __restrict__ G,
                                                         int64_t ldg,
                                                         const double* __restrict__ tau,
                                                         int64_t c0, double* T, int64_t ldt);
__global__ void build_v_kernel(int64_t n, const double* A, int64_t lda, int64_t i0, int w,
                               int64_t off, double* V, int64_t ldv);

int g_qr_gm = 0;  // em_config debug key 92: 1 = the panel QR always in its global-memory form

static void coop_launch(const void* fn, unsigned grid, unsigned block, void** args, size_t smem,
                        cudaStream_t st) {
  EM_CK(cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(block), args, smem, st));
  count_launch();
}

void sy2sb(cudaStream_t st, int64_t n, double* A, int64_t lda, double* tau1, double* AB,
           int64_t ldab) {
  const int b = B2;
  constexpr int64_t SB = 2048;  // column block of the symmetric product (band above: SB - 1)
  // The symmetric product as ONE TMA-fed kernel (every row tile runs over the whole k
  // range, reading left of its diagonal block as stored and below it transposed) when TMA
  // can address A: then only SYMM_BAND diagonals above the diagonal are kept current.
  extern int64_t g_gemm_tma;
  const bool symm_tma = g_gemm_tma != 0 && (lda & 1) == 0 && (n & 1) == 0 &&
                        (reinterpret_cast<uintptr_t>(A) & 15) == 0 && n >= 1024;
  const int64_t band_up = symm_tma ? SYMM_BAND : SB - 1;
  // Distributed reduction (a communicator with G > 1 ranks on the calling context, every
  // rank holding the same A on entry): the columns of the trailing matrix are owned in
  // 64-column blocks dealt round-robin (global block c / 64 -> rank (c / 64) mod G). Per
  // panel the owner of its columns factors it and broadcasts the finished columns; every
  // rank forms V, T, V T itself, adds up the k-tiles of X = A22 (V T) that read its own
  // columns, the partials are all-reduced, and the rank-2b update touches only owned column
  // tiles. Each finished column block is thus valid on every rank (band extraction and the
  // Q1 back-transform read them), everything right of the current panel only on its owner.
  em_ctx* cctx = g_cur_ctx;
  const int G = (symm_tma && cctx && cctx->stream == st) ? comm_size(cctx) : 1;
  const int rk = G > 1 ? comm_rank(cctx) : 0;
  DBuf PB(G > 1 ? (size_t)n * b + b : 0, st);  // a panel's columns (with its diagonal block) + tau
  const int sms = num_sms();
  DBuf VW((size_t)n * 2 * b, st), WV((size_t)n * 2 * b, st), VT((size_t)n * b, st);
  DBuf Gm((size_t)b * b, st), T((size_t)b * b, st), Y((size_t)b * b, st), M((size_t)b * b, st);
  DBuf part(2 * ((size_t)sms * b + b) + 8, st);
  DArr<GridBar> bar(1, st);
  EM_CK(cudaMemsetAsync(bar.p, 0, sizeof(GridBar), st));
  EM_CK(cudaFuncSetAttribute(qr_panel_kernel<false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  EM_CK(cudaFuncSetAttribute(larft_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(128 * 129 * sizeof(double))));
  for (int64_t k0 = 0; k0 + b < n; k0 += b) {
    const int64_t m = n - k0 - b;
    const int p = (int)imin64(b, m);
    double* P = A + (k0 + b) + k0 * lda;
    double* A22 = A + (k0 + b) + (k0 + b) * lda;
    const int owner = G > 1 ? (int)((k0 / b) % G) : 0;
    GemmOwn own;
    own.g = G;
    own.r = rk;
    own.org = (k0 + b) / 64;
    // panel QR
    if (rk == owner) {
      const int64_t gmax = imax64(1, imin64(sms, (m + 15) / 16));
      const int R = (int)(((m + gmax - 1) / gmax + 7) / 8 * 8);
      const unsigned G = (unsigned)((m + R - 1) / R);
      QRArgs qa{m, b, p, P, lda, tau1 + k0, part.p, bar.p, R};
      void* args[] = {&qa};
      Stage sq(st, ST_SY2SB_QR);
      const bool gm = g_qr_gm || (size_t)R * b * sizeof(double) > 200 * 1024;
      if (gm)
        coop_launch((const void*)qr_panel_kernel<true>, G, 256, args, 0, st);
      else
        coop_launch((const void*)qr_panel_kernel<false>, G, 256, args,
                    (size_t)R * b * sizeof(double), st);
    }
    if (G > 1) {  // columns k0 .. k0 + b - 1 from their diagonal block down, and the panel's tau
      const int64_t rows = n - k0;
      if (rk == owner) {
        copy_matrix(st, false, rows, b, A + k0 + k0 * lda, lda, PB.p, rows);
        EM_CK(cudaMemcpyAsync(PB.p + rows * b, tau1 + k0, b * sizeof(double),
                              cudaMemcpyDeviceToDevice, st));
      }
      comm_bcast(cctx, PB.p, rows * b + b, owner);
      if (rk != owner) {
        copy_matrix(st, false, rows, b, PB.p, rows, A + k0 + k0 * lda, lda);
        EM_CK(cudaMemcpyAsync(tau1 + k0, PB.p + rows * b, b * sizeof(double),
                              cudaMemcpyDeviceToDevice, st));
      }
    }
    // V (m x p) into VW[:, 0:p]; T from G = V^T V
    double* V = VW.p;
    double* X = VW.p + (size_t)p * n;
    dim3 gv((unsigned)imax64(1, imin64((m + 255) / 256, 64)), (unsigned)p);
    build_v_kernel<<<gv, 256, 0, st>>>(n, A, lda, k0, p, b, V, n);
    EM_LAUNCHED();
    EM_CK(gemm(st, true, false, p, p, m, 1.0, V, n, V, n, 0.0, Gm.p, p));
    larft_smem_kernel<<<1, 128, (size_t)128 * 129 * sizeof(double), st>>>(p, p, Gm.p, p, tau1,
                                                                          k0, T.p, p);
    EM_LAUNCHED();
    // X = A22 (V T);  M = T^T (V^T X);  W = X - V M / 2
    EM_CK(gemm(st, false, false, m, p, p, 1.0, V, n, T.p, p, 0.0, VT.p, n));
    // X = A22 VT from the lower triangle plus the band of width SB above the diagonal
    // (column blocks J: X[J:] += A22[J:, J] VT[J], X[J] += A22[J+SB:, J]^T VT[J+SB:])
    bool symm_done = false;
    if (symm_tma) {
      const cudaError_t e = gemm_symm_lower_tma(st, m, p, A22, lda, VT.p, n, X, n, own);
      if (e != cudaSuccess) EM_CK(e);  // operands were checked above: no fallback mid-way
      symm_done = true;
      if (G > 1) {  // partial products -> X (rows below m zeroed: the block is sent whole)
        if (m < n)
          EM_CK(cudaMemset2DAsync(X + m, n * sizeof(double), 0, (n - m) * sizeof(double), p, st));
        comm_allreduce_sum(cctx, X, n * (int64_t)p);
      }
    }
    for (int64_t j = 0; j < m && !symm_done; j += SB) {
      const int64_t w = imin64(SB, m - j);
      EM_CK(gemm(st, false, false, m - j, p, w, 1.0, A22 + j + j * lda, lda, VT.p + j, n,
                 j == 0 ? 0.0 : 1.0, X + j, n));
      if (j + w < m)
        EM_CK(gemm(st, true, false, w, p, m - j - w, 1.0, A22 + (j + w) + j * lda, lda,
                   VT.p + j + w, n, 1.0, X + j, n));
    }
    EM_CK(gemm(st, true, false, p, p, m, 1.0, V, n, X, n, 0.0, Y.p, p));
    EM_CK(gemm(st, true, false, p, p, p, 1.0, T.p, p, Y.p, p, 0.0, M.p, p));
    EM_CK(gemm(st, false, false, m, p, p, -0.5, V, n, M.p, p, 1.0, X, n));
    // A22 -= [V W] [W V]^T on the lower triangle and the band c - r < SB above it (what
    // the next panel's blocked product reads; 1.5x fewer flops than both triangles)
    copy_matrix(st, false, m, p, X, n, WV.p, n);
    copy_matrix(st, false, m, p, V, n, WV.p + (size_t)p * n, n);
    if (G > 1) {
      GemmArgs ua{m, m, 2 * p, VW.p, n, WV.p, n, A22, lda, -1.0, 1.0, band_up};
      EM_CK(gemm_lower_owned_tma(st, false, true, ua, own));
    } else {
      EM_CK(gemm(st, false, true, m, m, 2 * p, -1.0, VW.p, n, WV.p, n, 1.0, A22, lda, true,
                 band_up));
    }
  }
  if (G > 1) {  // the columns right of the last panel: valid on their owner only
    const int64_t kl = ((n - 1) / b) * b;  // = last k0 + b (or 0 when there was no panel)
    const int owner = (int)((kl / b) % G);
    const int64_t rows = n - kl;
    if (rk == owner) copy_matrix(st, false, rows, rows, A + kl + kl * lda, lda, PB.p, rows);
    comm_bcast(cctx, PB.p, rows * rows, owner);
    if (rk != owner) copy_matrix(st, false, rows, rows, PB.p, rows, A + kl + kl * lda, lda);
  }
  band_extract_kernel<<<(unsigned)n, 128, 0, st>>>(n, b, A, lda, AB, ldab);
  EM_LAUNCHED();
}

// ---- stage 2: bulge chasing ------------------------------------------------------
struct SbArgs {
  int64_t n;
  double* AB;
  int64_t ldab;       // 2b + 1
  double* V2;         // per task: b entries
  double* TAU2;       // per task
  const int64_t* toff;
  int* prog;          // tasks completed per sweep
  int64_t nsweeps;
};

EM_DEVINL int ld_acquire_int(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
EM_DEVINL void st_release_int(int* p, int v) {
  asm volatile("st.release.gpu.global.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

__host__ __device__ __forceinline__ int64_t ntasks(int64_t n, int64_t s) {
  return (n - 1 - s + B2 - 1) / B2;
}

constexpr int SBLD = B2 + 1;

// dlarfg on x[0..L) (L <= 64) in shared memory, every thread computing the scalars itself:
// returns tau, sets beta, writes v (v[0] = 1, zero from L on). x is left untouched. One
// barrier inside (the two warp sums of squares) and one at the end (v visible). beta =
// -sign(alpha) sqrt(alpha^2 + |x[1:]|^2) from the sum of squares directly.
EM_DEVINL double larfg64(const double* x, int L, double* v, double* red, double& beta) {
  const int tid = threadIdx.x;
  if (tid < B2) {
    const double xv = (tid >= 1 && tid < L) ? x[tid] : 0.0;
    const double ss = warp_sum(xv * xv);
    if ((tid & 31) == 0) red[tid >> 5] = ss;
  }
  __syncthreads();
  const double ss = red[0] + red[1];
  const double alpha = x[0];
  double tau = 0.0, scale = 0.0;
  beta = alpha;
  if (ss != 0.0) {
    beta = -copysign(sqrt(fma(alpha, alpha, ss)), alpha);
    tau = (beta - alpha) / beta;
    scale = 1.0 / (alpha - beta);
  }
  if (tid < B2) v[tid] = tid == 0 ? 1.0 : (tid < L ? x[tid] * scale : 0.0);
  __syncthreads();
  return tau;
}

// One task = one 64 x 64 off-diagonal block E (right application of the sweep's previous
// reflector, new reflector from its first column, left application) and the diagonal block
// D (two-sided). Thread (i = tid & 63, jg = tid >> 6) owns the elements (i, jg + 4 u),
// u < 16, of both blocks IN REGISTERS from the loads to the final stores (band storage:
// element (i, j) sits at base + j (ldab - 1), one add per element); shared memory holds the
// copies the matrix-vector products read. The scalars (beta, tau, the rank-2 coefficient)
// are computed redundantly by every thread or warp instead of by one thread behind two
// barriers: 9 barriers per task instead of 17 (the chase is bound by the task latency: a
// sweep follows its predecessor by two tasks).
__global__ void __launch_bounds__(256, 2) sb2st_kernel(SbArgs a) {
  extern __shared__ double sm[];
  double* E = sm;                 // E[i*SBLD + j]: row i of block k, column j of block k-1
  double* D = E + B2 * SBLD;      // full symmetric copy of the diagonal block
  __shared__ double v[B2], vn[B2], w[B2], w2[B2], xcol[B2], red[2];
  const int tid = threadIdx.x;
  const int q = tid & 3, row = tid >> 2;  // 4 threads per row (or column) in the matvecs
  const int ti = tid & (B2 - 1), jg = tid >> 6;  // owner of elements (ti, jg + 4 u)
  const int64_t n = a.n, ldab = a.ldab, st1 = a.ldab - 1;
  double* AB = a.AB;
  for (int64_t s = blockIdx.x; s < a.nsweeps; s += gridDim.x) {
    const int64_t K = ntasks(n, s);
    const int64_t Kp = s > 0 ? ntasks(n, s - 1) : 0;
    double tp = 0.0;  // tau of the sweep's previous reflector
    for (int64_t k = 0; k < K; ++k) {
      if (s > 0 && tid == 0) {
        // Task (s, k) touches rows a0 .. a0 + 63 = s + 1 + 64 k .. s + 64 (k + 1) only (its
        // E and D blocks); task (s - 1, k') rows s + 64 k' .. s + 64 k' + 63: k' <= k + 1
        // overlap, k' = k + 2 starts one row below. A lag of two tasks, not three: the
        // critical path of the chase is (lag x n) task latencies.
        const int need = (int)imin64(k + 2, Kp);
        // acquire by thread 0, made CTA-wide by the barrier below; the band is read with
        // L2-only loads (__ldcg), so no L1 invalidation is needed
        while (ld_acquire_int(a.prog + (s - 1)) < need) __nanosleep(32);
      }
      __syncthreads();
      const int64_t a0 = s + 1 + k * B2;
      const int64_t ap = a0 - B2;
      const int L = (int)imin64(B2, n - a0);
      // Every load of the task is issued before the first value is used: one L2 round trip
      // per task (the loads were 40% of a task's non-waiting stall samples,
      // profiles/r02/ncu_sb2st.json). D from its lower triangle only (mirrored into shared
      // memory); the diagonal block [a0, a0+L) is not touched by the off-diagonal work.
      double* dbase = AB + ti + a0 * ldab;       // (ti, j) at dbase + j (ldab - 1), j <= ti
      double* ebase = AB + (B2 + ti) + ap * ldab;  // (ti, j) at ebase + j (ldab - 1)
      double dreg[16], ereg[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int j = jg + 4 * u;
        dreg[u] = (j <= ti && ti < L) ? __ldcg(dbase + j * st1) : 0.0;
      }
      if (k > 0) {
#pragma unroll
        for (int u = 0; u < 16; ++u) ereg[u] = ti < L ? __ldcg(ebase + (jg + 4 * u) * st1) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int j = jg + 4 * u;
        if (j <= ti) {
          D[ti * SBLD + j] = dreg[u];
          D[j * SBLD + ti] = dreg[u];
        }
      }
      double tau, beta;
      if (k == 0) {
        // type 1: reflector from column s, rows a0 .. a0+L-1 (band offsets 1..L)
        if (tid < B2) xcol[tid] = (tid < L) ? __ldcg(AB + (1 + tid) + s * ldab) : 0.0;
        __syncthreads();
        tau = larfg64(xcol, L, vn, red, beta);
        if (tid < L) AB[(1 + tid) + s * ldab] = (tid == 0) ? beta : 0.0;
      } else {
        // type 2 on E = A[a0.., ap..] (element (i, j) at band offset 64 + i - j)
#pragma unroll
        for (int u = 0; u < 16; ++u) E[ti * SBLD + jg + 4 * u] = ereg[u];
        __syncthreads();
        {  // w = E v (right application of the previous reflector)
          double s2 = 0.0;
          for (int j = q; j < B2; j += 4) s2 = fma(E[row * SBLD + j], v[j], s2);
          s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
          s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
          if (q == 0) w[row] = s2;
        }
        __syncthreads();
        {  // E -= tp w v^T in the owner's registers and the shared copy; its first column
          const double twi = -tp * w[ti];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int j = jg + 4 * u;
            ereg[u] = fma(twi, v[j], ereg[u]);
            E[ti * SBLD + j] = ereg[u];
          }
          if (jg == 0) xcol[ti] = ereg[0];  // (rows from L on are zero)
        }
        __syncthreads();
        tau = larfg64(xcol, L, vn, red, beta);
        {  // u_j = sum_i vn_i E_ij, j >= 1 (left application of the new reflector)
          const int j = row;
          double s2 = 0.0;
          if (j >= 1)
            for (int i = q; i < L; i += 4) s2 = fma(vn[i], E[i * SBLD + j], s2);
          s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
          s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
          if (q == 0) w[j] = s2;
        }
        __syncthreads();
        if (ti < L) {
          const double tvi = -tau * vn[ti];
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int j = jg + 4 * u;
            const double val = (j == 0) ? ((ti == 0) ? beta : 0.0) : fma(tvi, w[j], ereg[u]);
            ebase[j * st1] = val;
          }
        }
      }
      // type 3 (and 1): D <- H D H on the diagonal block [a0, a0+L) (w2: the E stores above
      // may still be reading w)
      {
        double s2 = 0.0;
        for (int j = q; j < B2; j += 4) s2 = fma(D[row * SBLD + j], vn[j], s2);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 1);
        s2 += __shfl_xor_sync(0xffffffffu, s2, 2);
        if (q == 0) w2[row] = tau * s2;
      }
      __syncthreads();
      {
        // alpha = -tau/2 (w2 . vn), by every warp; w' = w2 + alpha vn formed where needed
        const int lane = tid & 31;
        double t2 = fma(w2[lane], vn[lane], w2[lane + 32] * vn[lane + 32]);
        t2 = warp_sum(t2);
        const double alpha = -0.5 * tau * t2;
        if (ti < L) {
          const double vi = vn[ti], wi = fma(alpha, vi, w2[ti]);
#pragma unroll
          for (int u = 0; u < 16; ++u) {
            const int j = jg + 4 * u;
            if (j <= ti) {
              const double vj = vn[j], wj = fma(alpha, vj, w2[j]);
              dbase[j * st1] = dreg[u] - vi * wj - wi * vj;
            }
          }
        }
      }
      // record the reflector; it becomes the "previous" one for the next task
      const int64_t t = a.toff[s] + k;
      if (tid < B2) {
        a.V2[t * B2 + tid] = vn[tid];
        v[tid] = vn[tid];
      }
      if (tid == 0) a.TAU2[t] = tau;
      tp = tau;
      // bar.sync orders every thread's band stores before thread 0's gpu-scope release
      // (cumulativity), as in the TD1 solves
      __syncthreads();
      if (tid == 0) st_release_int(a.prog + s, (int)(k + 1));
    }
  }
}

__global__ void tridiag_extract_kernel(int64_t n, const double* __restrict__ AB, int64_t ldab,
                                       double* d, double* e) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  d[i] = AB[i * ldab];
  if (i + 1 < n) e[i] = AB[1 + i * ldab];
}

// ---- Q2 back-transform -------------------------------------------------------------
// Block (g, k): reflectors of sweeps s = g*b + t (t < b, k < ntasks(s)), rows
// R0 + t .. R0 + t + L - 1 with R0 = g*b + 1 + k*b. V is (2b-1) x b, T is b x b.

constexpr int VR = 2 * B2;  // padded parallelogram rows (128)

struct Q2Block {
  int64_t g, k;  // group and position
};

// T for every block: V from the reflector store, G = V^T V, forward larft.
__global__ void __launch_bounds__(256) q2_tfactor_kernel(int64_t n, const Q2Block* __restrict__ blocks,
                                                         const double* __restrict__ V2,
                                                         const double* __restrict__ TAU2,
                                                         const int64_t* __restrict__ toff,
                                                         double* __restrict__ T2) {
  extern __shared__ double sm[];
  double* Vs = sm;              // [VR][B2]
  double* Ts = Vs + VR * B2;    // [B2][B2+1]
  double* Gs = Ts + B2 * (B2 + 1);  // [B2][B2+1]
  __shared__ double taus[B2];
  const Q2Block blk = blocks[blockIdx.x];
  const int tid = threadIdx.x;
  for (int i = tid; i < VR * B2; i += blockDim.x) Vs[i] = 0.0;
  __syncthreads();
  for (int idx = tid; idx < B2 * B2; idx += blockDim.x) {
    const int t = idx / B2, i = idx % B2;
    const int64_t s = blk.g * B2 + t;
    double tv = 0.0;
    if (s < n - 1 && blk.k < ntasks(n, s)) {
      const int64_t task = toff[s] + blk.k;
      Vs[(t + i) * B2 + t] = V2[task * B2 + i];
      tv = TAU2[task];
    }
    if (i == 0) taus[t] = tv;
  }
  __syncthreads();
  for (int idx = tid; idx < B2 * B2; idx += blockDim.x) {
    const int i = idx / B2, j = idx % B2;
    if (i < j) {
      double s2 = 0.0;
      for (int r = j; r < i + B2; ++r) s2 = fma(Vs[r * B2 + i], Vs[r * B2 + j], s2);
      Gs[i * (B2 + 1) + j] = s2;
    }
  }
  for (int i = tid; i < B2 * (B2 + 1); i += blockDim.x) Ts[i] = 0.0;
  __syncthreads();
  for (int k = 0; k < B2; ++k) {
    const double tk = taus[k];
    if (tid < k) {
      double s2 = 0.0;
      for (int j = tid; j < k; ++j) s2 = fma(Ts[tid * (B2 + 1) + j], Gs[j * (B2 + 1) + k], s2);
      Ts[tid * (B2 + 1) + k] = -tk * s2;
    }
    if (tid == 0) Ts[k * (B2 + 1) + k] = tk;
    __syncthreads();
  }
  double* Tout = T2 + blockIdx.x * (size_t)B2 * B2;
  for (int idx = tid; idx < B2 * B2; idx += blockDim.x) {
    const int i = idx / B2, j = idx % B2;
    Tout[idx] = Ts[i * (B2 + 1) + j];  // row-major i, j
  }
}

// Explicit V (VR x b, column-major, ld VR) of a list of blocks for one wavefront, and
// VT = V T (the block's T folded into the update: Z -= (V T) (V^T Z), one GEMM fewer).
// T2 holds each block's T row-major (T upper triangular).
// trans: VT = V T^T instead (the block's H^T = I - V T^T V^T, for Q2^T)
__global__ void __launch_bounds__(256) q2_buildv_kernel(int64_t n, const Q2Block* __restrict__ blocks,
                                                        const int64_t* __restrict__ ids,
                                                        const double* __restrict__ V2,
                                                        const int64_t* __restrict__ toff,
                                                        const double* __restrict__ T2,
                                                        double* __restrict__ Vout,
                                                        double* __restrict__ VTout, int trans,
                                                        int t_by_slot) {
  extern __shared__ double Vs[];  // VR x B2 (64 KB), column-major like Vout
  const Q2Block blk = blocks[ids[blockIdx.x]];
  double* V = Vout + blockIdx.x * (size_t)VR * B2;
  double* VT = VTout + blockIdx.x * (size_t)VR * B2;
  // T2 indexed by block id, or (t_by_slot) a per-launch buffer indexed by launch slot
  const double* T = T2 + (t_by_slot ? (int64_t)blockIdx.x : ids[blockIdx.x]) * (size_t)B2 * B2;
  const int64_t R0 = blk.g * B2 + 1 + blk.k * B2;
  for (int idx = threadIdx.x; idx < VR * B2; idx += blockDim.x) {
    const int r = idx % VR, t = idx / VR;  // row r of column t
    const int64_t s = blk.g * B2 + t;
    const int i = r - t;
    double val = 0.0;
    if (i >= 0 && i < B2 && R0 + r < n && s < n - 1 && blk.k < ntasks(n, s))
      val = V2[(toff[s] + blk.k) * B2 + i];
    V[idx] = val;
    Vs[idx] = val;
  }
  __syncthreads();
  // VT[r, j] = sum_{i <= j} V[r, i] T[i, j]; V[r, i] = 0 unless i <= r <= i + 63
  // (trans: sum_{i >= j} V[r, i] T[j, i])
  for (int idx = threadIdx.x; idx < VR * B2; idx += blockDim.x) {
    const int r = idx % VR, j = idx / VR;
    const int lo = r - (B2 - 1) > 0 ? r - (B2 - 1) : 0;
    const int hi = r < B2 - 1 ? r : B2 - 1;
    double acc = 0.0;
    if (!trans) {
      for (int i = lo; i <= (hi < j ? hi : j); ++i)
        acc = fma(Vs[i * VR + r], __ldg(T + i * B2 + j), acc);
    } else {
      for (int i = (lo > j ? lo : j); i <= hi; ++i)
        acc = fma(Vs[i * VR + r], __ldg(T + j * B2 + i), acc);
    }
    VT[idx] = acc;
  }
}

// ---- Q2 back-transform, column-strip form ----------------------------------------------
// The columns of Z transform independently, so one CTA owns a strip of WC columns and
// applies every block of a sweep group in order (positions ascending) with no
// inter-CTA synchronisation. Block k of group g touches rows W0 + 1 .. W0 + 127,
// W0 = 64 (g + k): consecutive blocks overlap by 64 rows, so the strip's rows live in
// a ring of three 64-row halves in shared memory (two for the window, one being
// prefetched), each half read from and written to HBM once per group instead of the
// three passes of the grouped-GEMM form. Per block, on DMMA:
//   W  = V^T Zwin      (64 x WC, k = 128; the parallelogram's zero k-range skipped)
//   Zwin -= (V T) W    (128 x WC, k = 64; VT rows r only need j >= r - 64)
// with V in compact form (64 reflectors x 64 entries) and VT = V T built per group
// (row-major, window coordinates). Loads of the next block's V, VT and Z half are
// issued while the current block computes (cp.async groups).
constexpr int Q2_LDC = 3 * 64 + 4;  // Z ring, column-major [col][3 halves]: = 4 mod 16
constexpr int Q2_LDV = 85;          // compact reflectors [t][8 + i], zero pads: LDV - 1 = 4 mod 16
constexpr int Q2_LDT = 68;          // VT row-major [r][j]: = 4 mod 16
int g_q2_mode = 0;  // debug key 97: 0 register-resident (q2reg.cu), 1 the wavefront grouped-GEMM
                    // form, 2 the shared-memory column strips

// VT (128 x 64 row-major, window row r = global row 64 (g + k) + r) of every block of
// group g; T2g = the group's T factors (row-major 64 x 64, upper).
__global__ void __launch_bounds__(256) q2_vt_kernel(int64_t n, int64_t g,
                                                    const double* __restrict__ V2,
                                                    const int64_t* __restrict__ toff,
                                                    const double* __restrict__ T2g,
                                                    double* __restrict__ VT) {
  __shared__ double Vs[B2 * (B2 + 1)];  // [t][i]
  const int64_t k = blockIdx.x;
  const double* T = T2g + k * B2 * B2;
  const int64_t W0 = B2 * (g + k);
  for (int e = threadIdx.x; e < B2 * B2; e += blockDim.x) {
    const int t = e >> 6, i = e & 63;
    const int64_t s = g * B2 + t;
    double v = 0.0;
    if (s < n - 1 && k < ntasks(n, s) && W0 + 1 + t + i < n) v = V2[(toff[s] + k) * B2 + i];
    Vs[t * (B2 + 1) + i] = v;
  }
  __syncthreads();
  double* out = VT + k * (int64_t)VR * B2;
  for (int e = threadIdx.x; e < VR * B2; e += blockDim.x) {
    const int r = e >> 6, j = e & 63;
    const int i0 = r - B2 > 0 ? r - B2 : 0;
    const int i1 = r - 1 < j ? r - 1 : j;
    double acc = 0.0;
    for (int i = i0; i <= i1; ++i) acc = fma(Vs[i * (B2 + 1) + (r - 1 - i)], __ldg(T + i * B2 + j), acc);
    out[e] = acc;
  }
}

template <int NJ>
struct Q2Strip {
  static constexpr int WC = 8 * NJ;
  static constexpr int LDW = (WC + 11) / 16 * 16 + 4;  // W row-major [j][c]: = 4 mod 16
  static constexpr int OFF_W = WC * Q2_LDC;
  static constexpr int OFF_V = OFF_W + B2 * LDW;
  static constexpr int OFF_T = OFF_V + B2 * Q2_LDV;
  static constexpr size_t SMEM = (size_t)(OFF_T + VR * Q2_LDT) * sizeof(double);
};

// rows 64 hg .. 64 hg + 63 of the strip's columns into ring slot hg % 3
template <int NJ>
EM_DEVINL void q2_load_half(double* Zw, const double* Z, int64_t ldz, int64_t n, int64_t ncols,
                            int64_t c0, int64_t hg) {
  const int slot = (int)(hg % 3);
  for (int e = threadIdx.x; e < 64 * Q2Strip<NJ>::WC; e += blockDim.x) {
    const int i = e & 63, c = e >> 6;
    const int64_t row = 64 * hg + i, col = c0 + c;
    const bool v = row < n && col < ncols;
    cp_async8(Zw + c * Q2_LDC + slot * 64 + i, v ? Z + row + col * ldz : Z, v);
  }
}

// W rows t = 8 W + gq of block k: W[t][c] = sum_r V[r][t] Zwin[r][c] over the 18 k-steps
// r = 8 W + 4 s + tq (V[r][t] = v_t[r - 1 - t], zero outside [t + 1, t + 64]: the padded
// compact row makes that a plain load). Even and odd steps accumulate separately (two
// DMMA chains per tile); every address is a per-thread base plus an immediate.
template <int NJ, int W>  // NJ: column fragments of this warp
EM_DEVINL void q2_step_a(const double* zlo, const double* zhi, const double* vrow, double* wrow) {
  double acc[2][NJ][2];
#pragma unroll
  for (int p = 0; p < 2; ++p)
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj) acc[p][jj][0] = acc[p][jj][1] = 0.0;
#pragma unroll
  for (int s = 0; s < 18; ++s) {
    const int r = 8 * W + 4 * s;  // + tq (in the bases)
    const double a = vrow[4 * s];
    const double* zc = (r < 64 ? zlo : zhi) + r;
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
      dmma884(acc[s & 1][jj][0], acc[s & 1][jj][1], a, zc[8 * jj * Q2_LDC]);
  }
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    wrow[8 * jj] = acc[0][jj][0] + acc[1][jj][0];
    wrow[8 * jj + 1] = acc[0][jj][1] + acc[1][jj][1];
  }
}

// Zwin -= VT W for row fragments W (top half; the result goes to HBM through zg) and
// 15 - W (bottom half; back to the ring). VT[r][j] = 0 for j < r - 64, so the bottom
// fragment joins at step s1 = 14 - 2 W; both share the W fragments.
template <int NJ, int LDW, int W>  // NJ: column fragments of this warp
EM_DEVINL void q2_step_c(double* z0, double* z1, const double* arow0, const double* arow1,
                         const double* bcol, double* zg, int64_t ldz, int64_t cl) {
  constexpr int s1 = 14 - 2 * W;
  double c0a[NJ][2], c1a[NJ][2];
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    c0a[jj][0] = z0[8 * jj * Q2_LDC];
    c0a[jj][1] = z0[(8 * jj + 1) * Q2_LDC];
    c1a[jj][0] = z1[8 * jj * Q2_LDC];
    c1a[jj][1] = z1[(8 * jj + 1) * Q2_LDC];
  }
#pragma unroll
  for (int s = 0; s < 16; ++s) {
    const double x0 = -arow0[4 * s];
    if (s < s1) {
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj)
        dmma884(c0a[jj][0], c0a[jj][1], x0, bcol[4 * s * LDW + 8 * jj]);
    } else {
      const double x1 = -arow1[4 * s];
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        const double b = bcol[4 * s * LDW + 8 * jj];
        dmma884(c0a[jj][0], c0a[jj][1], x0, b);
        dmma884(c1a[jj][0], c1a[jj][1], x1, b);
      }
    }
  }
#pragma unroll
  for (int jj = 0; jj < NJ; ++jj) {
    if (zg) {
      if (8 * jj < cl) zg[8 * jj * ldz] = c0a[jj][0];
      if (8 * jj + 1 < cl) zg[(8 * jj + 1) * ldz] = c0a[jj][1];
    }
    z1[8 * jj * Q2_LDC] = c1a[jj][0];
    z1[(8 * jj + 1) * Q2_LDC] = c1a[jj][1];
  }
}

template <int NJ>
EM_DEVINL void q2_strip_body(int64_t n, int64_t ncols, int64_t g, int64_t K,
                             const double* __restrict__ V2, const int64_t* __restrict__ toff,
                             const double* __restrict__ VT, double* __restrict__ Z, int64_t ldz,
                             int64_t c0, double* sm) {
  using S = Q2Strip<NJ>;
  double* Zw = sm;
  double* Ws = sm + S::OFF_W;
  double* Vc = sm + S::OFF_V;
  double* VTs = sm + S::OFF_T;
  __shared__ int64_t s_toff[B2];  // task offset of each sweep of the group
  __shared__ int64_t s_nt[B2];    // its task count (0: no such sweep)
  // 16 warps: warp & 7 picks the row fragments, warp >> 3 the half of the column
  // fragments (NH of them) the warp works on
  static_assert(NJ % 2 == 0, "two column halves");
  constexpr int NH = NJ / 2;
  // Row roles are paired so that each scheduler (warps w, w + 4, w + 8, w + 12) gets
  // roles r and 7 - r: step C costs 18 + 2 r k-step units for role r, so every scheduler
  // carries the same 100 units.
  const int tid = threadIdx.x, lane = tid & 31, gq = lane >> 2, tq = lane & 3;
  const int warp = ((tid >> 7) & 1) ? 7 - ((tid >> 5) & 3) : ((tid >> 5) & 3);
  const int jb = 8 * NH * (tid >> 8);  // first column of the warp's half
  if (tid < B2) {
    const int64_t s = g * B2 + tid;
    s_toff[tid] = s < n - 1 ? toff[s] : 0;
    s_nt[tid] = s < n - 1 ? ntasks(n, s) : 0;
  }
  for (int e = tid; e < B2 * Q2_LDV; e += blockDim.x) Vc[e] = 0.0;  // the pads stay zero
  __syncthreads();

  auto load_v = [&](int64_t k) {
    if (k >= K) return;
    const int64_t W0 = B2 * (g + k);
    for (int e = tid; e < B2 * B2; e += blockDim.x) {
      const int t = e >> 6, i = e & 63;
      const bool v = k < s_nt[t] && W0 + 1 + t + i < n;
      cp_async8(Vc + t * Q2_LDV + 8 + i, v ? V2 + (s_toff[t] + k) * B2 + i : V2, v);
    }
  };
  auto load_vt = [&](int64_t k) {
    const double* src = VT + k * (int64_t)VR * B2;
    for (int e = tid; e < VR * B2 / 2; e += blockDim.x) {
      const int r = e >> 5, j = (e & 31) * 2;
      cp_async16(VTs + r * Q2_LDT + j, src + r * B2 + j, 16);
    }
  };

  // prologue: halves g, g + 1 and V(0)
  q2_load_half<NJ>(Zw, Z, ldz, n, ncols, c0, g);
  q2_load_half<NJ>(Zw, Z, ldz, n, ncols, c0, g + 1);
  load_v(0);
  cp_async_commit();

  for (int64_t k = 0; k < K; ++k) {
    // halves g + k, g + k + 1 and V(k) landed; every warp is past block k - 1
    cp_async_wait<0>();
    __syncthreads();
    if (k + 2 <= K) q2_load_half<NJ>(Zw, Z, ldz, n, ncols, c0, g + k + 2);
    load_vt(k);
    cp_async_commit();
    const int hb = (int)((g + k) % 3);  // ring slot of the window's top half
    const int base_lo = hb * 64, base_hi = ((hb + 1) % 3) * 64 - 64;
    auto prow = [&](int r) { return (r < 64 ? base_lo : base_hi) + r; };

    // W = V^T Zwin (the warp's rows t = 8 warp + gq), see q2_step_a
    {
      const double* zlo = Zw + (jb + gq) * Q2_LDC + base_lo + tq;
      const double* zhi = Zw + (jb + gq) * Q2_LDC + base_hi + tq;
      const double* vrow = Vc + (8 * warp + gq) * Q2_LDV + 8 + tq - gq - 1;
      double* wrow = Ws + (8 * warp + gq) * S::LDW + jb + 2 * tq;
      switch (warp) {
        case 0: q2_step_a<NH, 0>(zlo, zhi, vrow, wrow); break;
        case 1: q2_step_a<NH, 1>(zlo, zhi, vrow, wrow); break;
        case 2: q2_step_a<NH, 2>(zlo, zhi, vrow, wrow); break;
        case 3: q2_step_a<NH, 3>(zlo, zhi, vrow, wrow); break;
        case 4: q2_step_a<NH, 4>(zlo, zhi, vrow, wrow); break;
        case 5: q2_step_a<NH, 5>(zlo, zhi, vrow, wrow); break;
        case 6: q2_step_a<NH, 6>(zlo, zhi, vrow, wrow); break;
        default: q2_step_a<NH, 7>(zlo, zhi, vrow, wrow); break;
      }
    }
    cp_async_wait<0>();  // VT(k) (and half k + 2)
    __syncthreads();     // Ws complete; Vc free
    load_v(k + 1);
    cp_async_commit();

    // Zwin -= VT W for row fragments a0 = warp (top half: written straight to HBM) and
    // a1 = 15 - warp (bottom half: back to the ring), see q2_step_c
    {
      const int pr0 = base_lo + 8 * warp + gq, pr1 = base_hi + 8 * (15 - warp) + gq;
      double* z0 = Zw + (jb + 2 * tq) * Q2_LDC + pr0;
      double* z1 = Zw + (jb + 2 * tq) * Q2_LDC + pr1;
      const double* arow0 = VTs + (8 * warp + gq) * Q2_LDT + tq;
      const double* arow1 = VTs + (8 * (15 - warp) + gq) * Q2_LDT + tq;
      const double* bcol = Ws + tq * S::LDW + jb + gq;
      const int64_t row0 = B2 * (g + k) + 8 * warp + gq;
      double* zg = row0 < n ? Z + row0 + (c0 + jb + 2 * tq) * ldz : nullptr;
      const int64_t cl = ncols - c0 - jb - 2 * tq;  // columns left from this thread's first
      switch (warp) {
        case 0: q2_step_c<NH, S::LDW, 0>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
        case 1: q2_step_c<NH, S::LDW, 1>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
        case 2: q2_step_c<NH, S::LDW, 2>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
        case 3: q2_step_c<NH, S::LDW, 3>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
        case 4: q2_step_c<NH, S::LDW, 4>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
        case 5: q2_step_c<NH, S::LDW, 5>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
        case 6: q2_step_c<NH, S::LDW, 6>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
        default: q2_step_c<NH, S::LDW, 7>(z0, z1, arow0, arow1, bcol, zg, ldz, cl); break;
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  {  // the last window's bottom half
    const int64_t hg = g + K;
    const int slot = (int)(hg % 3);
    for (int e = tid; e < 64 * S::WC; e += blockDim.x) {
      const int i = e & 63, c = e >> 6;
      const int64_t row = 64 * hg + i, col = c0 + c;
      if (row < n && col < ncols) Z[row + col * ldz] = Zw[c * Q2_LDC + slot * 64 + i];
    }
  }
}
// Strips [0, n6) are 48 columns wide, the rest 32: CTAs are dispatched in index order,
// so the narrow strips fill the last wave behind the wide ones.
__global__ void __launch_bounds__(512, 1) q2_strip_kernel(int64_t n, int64_t ncols, int64_t g,
                                                          int64_t K, const double* __restrict__ V2,
                                                          const int64_t* __restrict__ toff,
                                                          const double* __restrict__ VT,
                                                          double* __restrict__ Z, int64_t ldz,
                                                          int64_t n6) {
  extern __shared__ double sm[];
  const int64_t b = blockIdx.x;
  if (b < n6)
    q2_strip_body<6>(n, ncols, g, K, V2, toff, VT, Z, ldz, 48 * b, sm);
  else
    q2_strip_body<4>(n, ncols, g, K, V2, toff, VT, Z, ldz, 48 * n6 + 32 * (b - n6), sm);
}

// Makespan (in column-fragment units, ~1.5 units of per-block overhead per strip) of n6
// wide and n4 narrow strips dispatched in order onto `sms` SMs, one CTA per SM.
static double q2_makespan(int64_t n6, int64_t n4, int64_t sms) {
  std::priority_queue<double, std::vector<double>, std::greater<double>> q;
  for (int64_t i = 0; i < sms; ++i) q.push(0.0);
  double end = 0.0;
  for (int64_t i = 0; i < n6 + n4; ++i) {
    const double t = q.top() + (i < n6 ? 7.5 : 5.5);
    q.pop();
    q.push(t);
    end = t > end ? t : end;
  }
  return end;
}

// Z <- Q2 Z over all sweep groups (last group first). T2 holds the blocks' T factors in
// the order groups descending, positions ascending.
static void q2_apply_strips(cudaStream_t st, int64_t n, int64_t ncols, int64_t ngroups,
                            const double* V2, const int64_t* toff, const double* T2, double* Z,
                            int64_t ldz) {
  if (ncols <= 0) return;
  const int64_t sms = num_sms();
  const int64_t max6 = (ncols + 47) / 48;
  int64_t n6 = max6, n4 = 0;
  double best = q2_makespan(max6, 0, sms);
  const int64_t step = imax64(1, max6 / 256);
  for (int64_t a = 0; a < max6; a += step) {
    const int64_t b = (ncols - 48 * a + 31) / 32;
    const double t = q2_makespan(a, b, sms);
    if (t < best) best = t, n6 = a, n4 = b;
  }
  EM_CK(cudaFuncSetAttribute(q2_strip_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)Q2Strip<6>::SMEM));
  const int64_t kmax = ntasks(n, 0);
  DBuf VTg((size_t)imax64(kmax, 1) * VR * B2, st);
  int64_t off = 0;
  for (int64_t g = ngroups - 1; g >= 0; --g) {
    const int64_t K = ntasks(n, g * B2);
    if (K <= 0) continue;
    q2_vt_kernel<<<(unsigned)K, 256, 0, st>>>(n, g, V2, toff, T2 + off * B2 * B2, VTg.p);
    EM_LAUNCHED();
    q2_strip_kernel<<<(unsigned)(n6 + n4), 512, Q2Strip<6>::SMEM, st>>>(
        n, ncols, g, K, V2, toff, VTg.p, Z, ldz, n6);
    EM_LAUNCHED();
    off += K;
  }
}

// Z (n x ncols) <- Q2 Z (trans: Q2^T Z) as wavefronts of grouped DMMA GEMMs: block (g, k)
// belongs to wavefront w = k + 2 (G-1-g); blocks of one wavefront touch disjoint rows and
// every block a block depends on sits on an earlier wavefront (Q2^T: later, and the
// wavefronts run in reverse). Per block W = V^T Z, Z -= (V T) W (V T^T for Q2^T).
// T2 == nullptr: the blocks' T factors are formed per wavefront (from V2, TAU2) into a
// QCH-block buffer instead of all at once (n^2 / 2 doubles less: the N = 120,000 solve).
static void q2_apply_waves(cudaStream_t st, int64_t n, int64_t ncols, int64_t ngroups,
                           const std::vector<Q2Block>& blocks, const Q2Block* dblk,
                           const double* V2, const int64_t* dtoff, const double* T2, double* Z,
                           int64_t ldz, bool trans, const double* TAU2 = nullptr) {
  const int b = B2;
  const int64_t nblk = (int64_t)blocks.size();
  if (nblk == 0 || ncols <= 0) return;
  EM_CK(cudaFuncSetAttribute(q2_buildv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(VR * B2 * sizeof(double))));
  // blocks per grouped launch: a block is one CTA of the V / T kernels and a few tiles of
  // the grouped products, so a skinny operand (implicit mode: the drive and observable
  // columns) takes up to 512 blocks per launch — whole wavefronts, more CTAs than SMs —
  // while wide operands keep the per-launch workspace (QCH x 64 x ncols) small
  const int QCH = ncols <= 2048 ? 512 : 64;
  std::vector<std::vector<int64_t>> waves;
  {
    std::vector<std::vector<int64_t>> byw;
    for (int64_t i = 0; i < nblk; ++i) {
      const int64_t wv = blocks[i].k + 2 * (ngroups - 1 - blocks[i].g);
      if ((int64_t)byw.size() <= wv) byw.resize(wv + 1);
      byw[wv].push_back(i);
    }
    if (trans) std::reverse(byw.begin(), byw.end());
    for (auto& wl : byw)
      for (size_t c = 0; c < wl.size(); c += QCH)
        waves.emplace_back(wl.begin() + c, wl.begin() + std::min(wl.size(), c + QCH));
  }
  std::vector<int64_t> ids;
  std::vector<Q2Block> wblk;  // the blocks in launch order (per-wavefront T factors)
  std::vector<GemmArgs> args;
  std::vector<int64_t> wstart;
  const bool t_waves = T2 == nullptr;
  DBuf Vb((size_t)QCH * VR * B2, st), VTb((size_t)QCH * VR * B2, st),
      W1((size_t)QCH * B2 * ncols, st), Tw;
  if (t_waves) Tw.alloc((size_t)QCH * B2 * B2, st);
  for (auto& wl : waves) {
    wstart.push_back((int64_t)ids.size());
    for (size_t j = 0; j < wl.size(); ++j) {
      const Q2Block& bk = blocks[wl[j]];
      const int64_t R0 = bk.g * b + 1 + bk.k * b;
      const int64_t nrow = imin64(VR - 1, n - R0);
      double* Vj = Vb.p + j * (size_t)VR * B2;
      double* VTj = VTb.p + j * (size_t)VR * B2;
      double* W1j = W1.p + j * (size_t)B2 * ncols;
      ids.push_back(wl[j]);
      wblk.push_back(bk);
      args.push_back(GemmArgs{B2, ncols, nrow, Vj, VR, Z + R0, ldz, W1j, B2, 1.0, 0.0, 0});
      args.push_back(GemmArgs{nrow, ncols, B2, VTj, VR, W1j, B2, Z + R0, ldz, -1.0, 1.0, 0});
    }
  }
  wstart.push_back((int64_t)ids.size());
  DArr<int64_t> dids(ids.size(), st);
  DArr<GemmArgs> dargs(args.size(), st);
  EM_CK(cudaMemcpyAsync(dids.p, ids.data(), ids.size() * sizeof(int64_t), cudaMemcpyHostToDevice,
                        st));
  // phase-major argument arrays: [phase][problem]
  std::vector<GemmArgs> ph(args.size());
  const size_t np = ids.size();
  for (size_t i = 0; i < np; ++i)
    for (int q = 0; q < 2; ++q) ph[q * np + i] = args[2 * i + q];
  EM_CK(cudaMemcpyAsync(dargs.p, ph.data(), ph.size() * sizeof(GemmArgs), cudaMemcpyHostToDevice,
                        st));
  const int tiles_n = (int)((ncols + 127) / 128);
  DArr<Q2Block> dwblk(t_waves ? wblk.size() : 1, st);
  const size_t smt = ((size_t)VR * B2 + 2 * (size_t)B2 * (B2 + 1)) * sizeof(double);
  if (t_waves) {
    EM_CK(cudaMemcpyAsync(dwblk.p, wblk.data(), wblk.size() * sizeof(Q2Block),
                          cudaMemcpyHostToDevice, st));
    EM_CK(cudaFuncSetAttribute(q2_tfactor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smt));
  }
  for (size_t wi = 0; wi + 1 < wstart.size(); ++wi) {
    const int64_t o = wstart[wi], cnt = wstart[wi + 1] - wstart[wi];
    if (t_waves) {
      q2_tfactor_kernel<<<(unsigned)cnt, 256, smt, st>>>(n, dwblk.p + o, V2, TAU2, dtoff, Tw.p);
      EM_LAUNCHED();
    }
    q2_buildv_kernel<<<(unsigned)cnt, 256, (size_t)VR * B2 * sizeof(double), st>>>(
        n, dblk, dids.p + o, V2, dtoff, t_waves ? Tw.p : T2, Vb.p, VTb.p, trans ? 1 : 0,
        t_waves ? 1 : 0);
    EM_LAUNCHED();
    EM_CK(gemm_grouped(st, true, false, dargs.p + o, (int)cnt, tiles_n));
    EM_CK(gemm_grouped(st, false, false, dargs.p + np + o, (int)cnt, tiles_n));
  }
  EM_CK(cudaStreamSynchronize(st));  // host argument arrays / device lists lifetime
}

// ---- driver -------------------------------------------------------------------------
void syev_two_stage(cudaStream_t st, int64_t n, double* A, int64_t lda, double* w, double* Z,
                    int64_t ldz, int64_t c0, int64_t nc, double* Yt, int64_t ldy, int64_t ky) {
  if (nc < 0) nc = n - c0;
  double* Zc = Z ? Z + c0 * ldz : nullptr;  // the back-transformed columns
  const int b = B2;
  const int64_t ldab = 2 * b + 1;
  DBuf tau1(n, st), AB((size_t)ldab * n, st);
  {
    Stage s(st, ST_SYTRD);
    mirror_lower(st, n, A, lda);  // stage 1 reads the lower triangle and a band above it
    Stage s1(st, ST_SY2SB);
    sy2sb(st, n, A, lda, tau1.p, AB.p, ldab);
  }
  if (Yt && n > b) {  // implicit mode: Q^T = Q2^T Q1^T, so Q1^T first; A is free after it
    Stage sq1(st, ST_Q1);
    ormqr_lower_off(st, n, n - b, b, ky, A, lda, tau1.p, Yt, ldy, true);
  }
  // stage 2
  const int64_t nsw = n - 1;
  std::vector<int64_t> toff(nsw + 1, 0);
  for (int64_t s = 0; s < nsw; ++s) toff[s + 1] = toff[s] + ntasks(n, s);
  const int64_t ntask = toff[nsw];
  DArr<int64_t> dtoff(nsw + 1, st);
  EM_CK(cudaMemcpyAsync(dtoff.p, toff.data(), (nsw + 1) * sizeof(int64_t), cudaMemcpyHostToDevice,
                        st));
  // the stage-2 reflectors: in implicit mode in A's storage (no longer needed once Q1^T is
  // applied), so the N = 120,000 eigensolve holds A plus the Q2 T factors only
  const size_t v2n = (size_t)imax64(ntask, 1) * b;
  DBuf V2own;
  double* V2 = A;
  if (!(Yt && lda >= n && v2n <= (size_t)lda * n)) {
    V2own.alloc(v2n, st);
    V2 = V2own.p;
  }
  DBuf TAU2(imax64(ntask, 1), st);
  DArr<int> prog(imax64(nsw, 1), st);
  EM_CK(cudaMemsetAsync(prog.p, 0, imax64(nsw, 1) * sizeof(int), st));
  DBuf d(n, st), e(imax64(n - 1, 1), st);
  {
    Stage s(st, ST_SYTRD);
    const size_t smem = (size_t)2 * B2 * SBLD * sizeof(double);
    EM_CK(cudaFuncSetAttribute(sb2st_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)smem));
    int per_sm = 1;
    EM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sb2st_kernel, 256, smem));
    const unsigned grid = (unsigned)imax64(1, imin64(nsw, (int64_t)num_sms() * imax64(per_sm, 1)));
    SbArgs sa{n, AB.p, ldab, V2, TAU2.p, dtoff.p, prog.p, nsw};
    void* args[] = {&sa};
    Stage s2(st, ST_SB2ST);
    if (nsw > 0) coop_launch((const void*)sb2st_kernel, grid, 256, args, smem, st);
    tridiag_extract_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, AB.p, ldab, d.p, e.p);
    EM_LAUNCHED();
  }
  AB.release();
  if (!Yt) {
    Stage s(st, ST_STEDC);
    stedc(st, n, d.p, e.p, Z, ldz, c0, nc);
  }
  {
    Stage s(st, ST_ORMTR);
    // Q2: blocks (g, k) = reflectors of sweeps g*b .. g*b+b-1 at position k. The order
    // "groups last to first, positions ascending" is satisfied by applying wavefronts
    // w = k + 2 (G-1-g) in increasing w: blocks of one wavefront touch disjoint rows and
    // every block they depend on sits on an earlier wavefront. Each wavefront is two
    // grouped DMMA GEMMs over all columns of Z (W = V^T Z, Z -= (V T) W).
    std::vector<Q2Block> blocks;
    const int64_t ngroups = (nsw + b - 1) / b;
    for (int64_t g = ngroups - 1; g >= 0; --g) {
      const int64_t K = ntasks(n, g * b);
      for (int64_t k = 0; k < K; ++k) blocks.push_back(Q2Block{g, k});
    }
    const int64_t nblk = (int64_t)blocks.size();
    if (nblk > 0) {
      Stage sq(st, ST_Q2);
      DArr<Q2Block> dblk(nblk, st);
      EM_CK(cudaMemcpyAsync(dblk.p, blocks.data(), nblk * sizeof(Q2Block), cudaMemcpyHostToDevice,
                            st));
      DBuf T2;
      if (!Yt) {
        T2.alloc((size_t)nblk * b * b, st);
        const size_t smt = ((size_t)VR * B2 + 2 * (size_t)B2 * (B2 + 1)) * sizeof(double);
        EM_CK(cudaFuncSetAttribute(q2_tfactor_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smt));
        q2_tfactor_kernel<<<(unsigned)nblk, 256, smt, st>>>(n, dblk.p, V2, TAU2.p, dtoff.p,
                                                            T2.p);
        EM_LAUNCHED();
      }
      if (Yt) {
        // implicit mode: Yt <- Q2^T (Q1^T Yt) (Q1^T applied above), T factors per wavefront
        q2_apply_waves(st, n, ky, ngroups, blocks, dblk.p, V2, dtoff.p, nullptr, Yt, ldy, true,
                       TAU2.p);
      } else if (g_q2_mode == 0) {
        q2_apply_reg(st, n, nc, ngroups, V2, dtoff.p, T2.p, Zc, ldz);
        EM_CK(cudaStreamSynchronize(st));  // dblk lifetime
      } else if (g_q2_mode == 2) {
        q2_apply_strips(st, n, nc, ngroups, V2, dtoff.p, T2.p, Zc, ldz);
        EM_CK(cudaStreamSynchronize(st));  // dblk lifetime
      } else {
        q2_apply_waves(st, n, nc, ngroups, blocks, dblk.p, V2, dtoff.p, T2.p, Zc, ldz, false);
      }
    }
    // Q1 (stage-1 reflectors, vectors start b rows below their column)
    if (!Yt) {
      Stage sq1(st, ST_Q1);
      if (n > b) ormqr_lower_off(st, n, n - b, b, nc, A, lda, tau1.p, Zc, ldz);
    }
  }
  if (Yt) {  // Yt <- U^T Yt without forming U
    Stage s(st, ST_STEDC);
    stedc_apply(st, n, d.p, e.p, Yt, ldy, ky);
  }
  EM_CK(cudaMemcpyAsync(w, d.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
}

}  // namespace em
