// One persistent cooperative kernel per 64-column panel of the one-stage
// Householder tridiagonalisation (latrd): per column
//   A  column update A[c:, c] -= A_p W[c, :]^T + W_p A[c, i0:c]^T (+ the deferred
//      w += alpha v fix of the previous column), partial norms   | grid barrier
//   B  dlarfg (every CTA forms beta/tau/scale), scale v           | grid barrier
//   C  symv tiles of the trailing matrix (HBM-bound, symv_tile.cuh) and the panel
//      dot products W_p^T v, A_p^T v                              | grid barrier
//   D  symv reduction + w = tau (A22 v - A_p t1 - W_p t2), partial w.v
//                                                                 | grid barrier
// replacing ~7 dependent launches per column by 4 grid barriers; the
// trailing-matrix product is the same tile code as em_symv_lower.
// Every read of data another CTA may have written inside this kernel (the panel
// columns, W, the partial sums) goes through L2 (__ldcg): an SM may still hold
// those lines in L1 from an earlier column's trailing-matrix tiles.
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"
#include "symv_tile.cuh"

namespace em {

namespace {

struct Bar {
  unsigned int count;
  unsigned int gen;
};

EM_DEVINL void bar_sync(Bar* bar, unsigned nblocks) {
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
      while (*vgen == g) __nanosleep(20);
    }
    __threadfence();  // also invalidates this SM's L1 (CCTL.IVALL)
  }
  __syncthreads();
}

constexpr int FT = 256;           // threads
constexpr int FNB = 64;           // panel width
constexpr int RB = 32;            // rows per row block (8 threads per row)


EM_DEVINL double bsum(double v, double* red8) {
  v = warp_sum(v);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red8[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int k = 0; k < FT / 32; ++k) t += red8[k];
  return t;  // every thread
}

EM_DEVINL double gsum8(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 4);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v;
}

struct LatrdArgs {
  int64_t n;
  double* A;
  int64_t lda;
  int64_t i0;
  int w;
  double* W;  // rows indexed from i0, ld ldw
  int64_t ldw;
  double *d, *e, *tau;
  double* part;   // [G]
  double* part2;  // [G]
  double* dpart;  // [2*64][nchunk]
  double* wcol;
  double* wrow;
  double* abuf;
  Bar* bar;
  int dotr;  // rows per dot chunk
};

}  // namespace

__global__ void __launch_bounds__(FT, 2) latrd_fused_kernel(LatrdArgs a) {
  __shared__ double red8[FT / 32];
  __shared__ double red[8][SV];
  __shared__ double red4[4][SV];
  __shared__ double wr[FNB], ar[FNB], t1[FNB], t2[FNB], ysh[SV];
  __shared__ double bc[4];
  const unsigned G = gridDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int sub = tid & 7, rl = tid >> 3;  // 8 threads per row, 32 rows per row block
  const int64_t n = a.n, lda = a.lda, i0 = a.i0, ldw = a.ldw;
  double* A = a.A;
  double* W = a.W;
  bool have_prev = false;  // column i-1 produced a W column awaiting its alpha fix
  for (int i = 0; i < a.w; ++i) {
    const int64_t c = i0 + i;
    // ---------------- phase A ----------------
    double alpha_prev = 0.0;
    if (have_prev) {
      double s = 0.0;
      for (unsigned b = tid; b < G; b += FT) s += __ldcg(a.part2 + b);
      s = bsum(s, red8);
      alpha_prev = -0.5 * __ldcg(a.tau + c - 1) * s;
    }
    for (int k = tid; k < i; k += FT) {
      double wv = __ldcg(W + (c - i0) + k * ldw);
      if (have_prev && k == i - 1) wv += alpha_prev;  // v_{c-1}[c] = 1
      wr[k] = wv;
      ar[k] = __ldcg(A + c + (i0 + k) * lda);
    }
    __syncthreads();
    double ss = 0.0;
    for (int64_t rb = (c / RB) + ((blockIdx.x + G - (unsigned)((c / RB) % G)) % G);
         rb * RB < n; rb += G) {
      const int64_t r = rb * RB + rl;
      double s = 0.0;
      if (r >= c && r < n) {
        for (int k = sub; k < i; k += 8) {
          double wk = __ldcg(W + (r - i0) + k * ldw);
          if (have_prev && k == i - 1) {
            wk = fma(alpha_prev, __ldcg(A + r + (c - 1) * lda), wk);  // deferred w += alpha v fix
            W[(r - i0) + k * ldw] = wk;
          }
          s = fma(__ldcg(A + r + (i0 + k) * lda), wr[k], s);
          s = fma(wk, ar[k], s);
        }
      }
      s = gsum8(s);
      if (sub == 0 && r >= c && r < n) {
        const double v = __ldcg(A + r + c * lda) - s;
        if (i > 0) A[r + c * lda] = v;
        if (r >= c + 2) ss = fma(v, v, ss);
        if (r == c + 1) *a.abuf = v;
      }
    }
    ss = bsum(ss, red8);
    if (tid == 0) a.part[blockIdx.x] = ss;
    bar_sync(a.bar, G);
    if (c == n - 1) {  // last column: no reflector
      if (blockIdx.x == 0 && tid == 0) a.d[c] = __ldcg(A + c + c * lda);
      have_prev = false;
      break;
    }
    // ---------------- phase B ----------------
    {
      double s = 0.0;
      for (unsigned b = tid; b < G; b += FT) s += __ldcg(a.part + b);
      s = bsum(s, red8);
      if (tid == 0) {
        const double alpha = *(volatile double*)a.abuf;
        const double xnorm = sqrt(s);
        double beta, tau, scale;
        if (xnorm == 0.0) {
          beta = alpha;
          tau = 0.0;
          scale = 0.0;
        } else {
          beta = -copysign(hypot(alpha, xnorm), alpha);
          tau = (beta - alpha) / beta;
          scale = 1.0 / (alpha - beta);
        }
        bc[0] = beta;
        bc[1] = tau;
        bc[2] = scale;
        if (blockIdx.x == 0) {
          a.d[c] = __ldcg(A + c + c * lda);
          a.e[c] = beta;
          a.tau[c] = tau;
          A[(c + 1) + c * lda] = 1.0;
        }
      }
      __syncthreads();
      const double scale = bc[2];
      if (scale != 0.0)
        for (int64_t r = c + 2 + (int64_t)blockIdx.x * FT + tid; r < n; r += (int64_t)G * FT)
          A[r + c * lda] = __ldcg(A + r + c * lda) * scale;
    }
    bar_sync(a.bar, G);
    const double tauc = bc[1];
    // ---------------- phase C: symv tiles + panel dots ----------------
    const int64_t m = n - c - 1;
    const double* A22 = A + (c + 1) + (c + 1) * lda;
    const double* v = A + (c + 1) + c * lda;  // v[0] = 1
    const int64_t nbm = (m + SV - 1) / SV;
    const int64_t nch = (nbm + SVCH - 1) / SVCH;
    {
      int64_t u = 0;
      for (int64_t I = 0; I < nbm; ++I) {
        const int64_t chs = I / SVCH + 1;
        // units of this row: u .. u+chs-1
        int64_t first = u + ((blockIdx.x + G - (unsigned)(u % G)) % G);
        for (int64_t uu = first; uu < u + chs; uu += G)
          symv_strip(m, A22, lda, v, a.wcol, a.wrow, nbm, nch, I, uu - u, red);
        u += chs;
      }
    }
    const int DOTR = a.dotr;
    const int nchunk = (int)((m + DOTR - 1) / DOTR);
    if (i > 0) {
      const int ngrp = (2 * i + 7) / 8;
      const int64_t units = (int64_t)ngrp * nchunk;
      for (int64_t uu = blockIdx.x; uu < units; uu += G) {
        const int grp = (int)(uu / nchunk), ch = (int)(uu % nchunk);
        const int col = grp * 8 + warp;
        if (col < 2 * i) {
          const int which = col / i, k = col % i;
          const int64_t rbeg = c + 1 + (int64_t)ch * DOTR;
          const int64_t rend = imin64(n, rbeg + DOTR);
          const double* colp = which == 0 ? W + k * ldw - i0 : A + (i0 + k) * lda;
          const double* vv = A + c * lda;
          double s = 0.0;
          for (int64_t r = rbeg + lane; r < rend; r += 32) s = fma(__ldcg(colp + r), __ldcg(vv + r), s);
          s = warp_sum(s);
          if (lane == 0) a.dpart[(which * FNB + k) * nchunk + ch] = s;
        }
      }
    }
    bar_sync(a.bar, G);
    // ---------------- phase D: reduce + W column ----------------
    for (int q = tid; q < 2 * i; q += FT) {
      const int which = q / i, k = q % i;
      double s = 0.0;
      for (int ch = 0; ch < nchunk; ++ch) s += __ldcg(a.dpart + (which * FNB + k) * nchunk + ch);
      if (which == 0)
        t1[k] = s;
      else
        t2[k] = s;
    }
    double dd = 0.0;
    for (int64_t J = blockIdx.x; J < nbm; J += G) {
      const double y = symv_reduce_block(a.wcol, a.wrow, nbm, nch, J, red4);
      if (tid < SV) ysh[tid] = y;
      __syncthreads();
      // 4 threads per row: row t = tid >> 2 of the block
      const int t = tid >> 2, qq = tid & 3;
      const int64_t r = c + 1 + J * SV + t;
      double s = 0.0;
      if (r < n)
        for (int k = qq; k < i; k += 4) {
          s = fma(__ldcg(A + r + (i0 + k) * lda), t1[k], s);
          s = fma(__ldcg(W + (r - i0) + k * ldw), t2[k], s);
        }
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      if (qq == 0 && r < n) {
        const double x = tauc * (ysh[t] - s);
        W[(r - i0) + i * ldw] = x;
        dd = fma(x, __ldcg(A + r + c * lda), dd);
      }
      __syncthreads();
    }
    dd = bsum(dd, red8);
    if (tid == 0) a.part2[blockIdx.x] = dd;
    have_prev = true;
    bar_sync(a.bar, G);
  }
  // final deferred fix of the panel's last W column
  if (have_prev) {
    const int64_t c = i0 + a.w - 1;
    double s = 0.0;
    for (unsigned b = tid; b < G; b += FT) s += __ldcg(a.part2 + b);
    s = bsum(s, red8);
    const double alpha = -0.5 * __ldcg(a.tau + c) * s;
    for (int64_t r = c + 1 + (int64_t)blockIdx.x * FT + tid; r < n; r += (int64_t)G * FT)
      W[(r - i0) + (a.w - 1) * ldw] =
          fma(alpha, __ldcg(A + r + c * lda), __ldcg(W + (r - i0) + (a.w - 1) * ldw));
  }
}

// restore A[c+1, c] = e[c] for the panel columns
__global__ void restore_sub_kernel2(int64_t n, double* A, int64_t lda, int64_t i0, int w,
                                    const double* e) {
  const int k = threadIdx.x;
  if (k < w) {
    const int64_t c = i0 + k;
    if (c + 1 < n) A[(c + 1) + c * lda] = e[c];
  }
}

int g_latrd_dotr = 2048;

void sytrd_lower_fused(cudaStream_t st, int64_t n, double* A, int64_t lda, double* d, double* e,
                       double* tau) {
  int per_sm = 0;
  EM_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, latrd_fused_kernel, FT, 0));
  const unsigned G = (unsigned)imax64(1, (int64_t)num_sms() * imax64(per_sm, 1));
  DBuf W((size_t)n * FNB, st);
  DBuf XW((size_t)n * 2 * FNB, st), YW((size_t)n * 2 * FNB, st);
  DBuf part(G, st), part2(G, st), abuf(1, st);
  const int DOTR = g_latrd_dotr;
  DBuf dpart((size_t)2 * FNB * ((n + DOTR - 1) / DOTR + 1), st);
  DBuf swork(symv_work_doubles(n), st);
  DArr<Bar> bar(1, st);
  EM_CK(cudaMemsetAsync(bar.p, 0, sizeof(Bar), st));
  const int64_t nb = (n + SV - 1) / SV;
  for (int64_t i0 = 0; i0 < n; i0 += FNB) {
    const int w = (int)imin64(FNB, n - i0);
    LatrdArgs la{n, A, lda, i0, w, W.p, n, d, e, tau, part.p, part2.p, dpart.p, swork.p,
                 swork.p + nb * nb * SV, abuf.p, bar.p, DOTR};
    void* args[] = {&la};
    EM_CK(cudaLaunchCooperativeKernel((const void*)latrd_fused_kernel, dim3(G), dim3(FT), args,
                                      0, st));
    count_launch();
    const int64_t t0 = i0 + w;
    const int64_t mt = n - t0;
    if (mt > 0) {
      Stage s(st, ST_SYTRD_SYR2K);
      copy_matrix(st, false, mt, w, A + t0 + i0 * lda, lda, XW.p, n);
      copy_matrix(st, false, mt, w, W.p + (t0 - i0), n, XW.p + (int64_t)w * n, n);
      copy_matrix(st, false, mt, w, W.p + (t0 - i0), n, YW.p, n);
      copy_matrix(st, false, mt, w, A + t0 + i0 * lda, lda, YW.p + (int64_t)w * n, n);
      EM_CK(gemm(st, false, true, mt, mt, 2 * w, -1.0, XW.p, n, YW.p, n, 1.0,
                 A + t0 + t0 * lda, lda, true, 0));
    }
    restore_sub_kernel2<<<1, FNB, 0, st>>>(n, A, lda, i0, w, e);
    EM_LAUNCHED();
  }
}

}  // namespace em
