// TMA-fed lower-triangle symv (the HBM-bound product of every tridiagonalisation
// column and of the Cholesky theta-method step). Same contract as symv.cu: y = alpha
// A x + beta y reading only the lower triangle, deterministic fixed-order reduction.
//
// B200 mapping
//  - one persistent CTA per SM (512 threads); the strips of 128 rows are cut into
//    tiles of 128 x 64 (64 KB) and the nbs(nbs+1)-ish tiles of the lower triangle are
//    split into equal contiguous ranges, one per CTA (no tail wave);
//  - tiles arrive by cp.async.bulk.tensor (one instruction per tile, issued by one
//    thread) into a 3-stage shared-memory ring with full/empty mbarriers, so two tiles
//    (128 KB) are in flight per SM while the third is consumed. tools/bw_probe.cu
//    measures this access pattern at 6.6 TB/s with that much in flight (5.7 with one
//    tile), against 7.2 TB/s for a flat read;
//  - each element is used twice from shared memory: row sums A_ij x_j accumulate in
//    registers across the strip, column sums A_ij^T x_i are reduced across the warp once
//    per tile (128 rows) and written to wcol; a second kernel sums the partials.
// The tensor map spans the whole matrix, so a trailing submatrix (sytrd) is addressed
// by coordinates and the out-of-range part of the last strip is zero-filled by TMA.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "ctx.h"
#include "linalg.h"
#include "symv_tile.cuh"
#include "symv_tma.cuh"

namespace em {

static_assert(sizeof(SymvMap) == 2 * sizeof(CUtensorMap), "SymvMap holds two CUtensorMaps");
extern int g_symv_align_off;

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

bool symv_map_make(SymvMap* m, const double* base, int64_t rows, int64_t cols, int64_t ld) {
  if (rows <= 0 || cols <= 0) return false;
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 8) & 15)) return false;
  if (rows > INT32_MAX || cols > INT32_MAX) return false;
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)rows, (cuuint64_t)cols};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t es[2] = {1, 1};
  for (int sh = 0; sh < 2; ++sh) {
    cuuint32_t box[2] = {(cuuint32_t)(sh ? BR : HR), WC};
    const CUresult r = fn(reinterpret_cast<CUtensorMap*>(m->opaque[sh]),
                          CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                          strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return false;
  }
  return true;
}

// ---- schedule ----------------------------------------------------------------------
// strip i (rows 128i..) has tiles j = 0 .. min(2i+2, ncj)-1 (64-column tiles up to the
// diagonal); off(i) = i(i+1) for every strip (only the last one can be clipped).
struct TmaSched {
  int64_t nbs, ncj, T, P, len, slots;
};

static TmaSched tma_sched(int64_t n) {
  TmaSched s;
  s.nbs = (n + HR - 1) / HR;
  s.ncj = (n + WC - 1) / WC;
  s.T = s.nbs * (s.nbs - 1) + imin64(2 * s.nbs, s.ncj);
  s.P = imax64(1, imin64(s.T, (int64_t)num_sms()));
  s.len = (s.T + s.P - 1) / s.P;
  s.P = (s.T + s.len - 1) / s.len;
  s.slots = 2 * s.nbs + 2;
  return s;
}

int64_t symv_tma_ctas(int64_t n) { return tma_sched(n).P; }
int64_t symv_tma_ctas(int64_t n, int64_t off) {
  return tma_sched(n + (g_symv_align_off ? 0 : off % 32)).P;
}
int g_symv_align_off = 0;  // em_config debug key 98 bit 4: no 32-row alignment shift
int64_t g_symv_keep_mb = 32;  // EM_CFG_SYMV_L2_KEEP_MB (A/B at N = 16k: 0 -> 32 MB saves ~10 ms)

size_t symv_tma_work_size(int64_t n) {
  const TmaSched s = tma_sched(n);
  return (size_t)(s.nbs * s.ncj * WC + s.nbs * s.slots * HR);
}

// ---- kernel ----------------------------------------------------------------------------
template <bool LARFG, int SH>
__global__ void __launch_bounds__(TT, 1) symv_tma_kernel(const __grid_constant__ CUtensorMap map,
                                                         int64_t off, int64_t n, int64_t d,
                                                         const double* __restrict__ x,
                                                         double* __restrict__ wcol,
                                                         double* __restrict__ wrow, int64_t nbs,
                                                         int64_t ncj, int64_t T, int64_t len,
                                                         int64_t slots, int64_t keep_c0,
                                                         SymvLarfg lf) {
  extern __shared__ __align__(128) double ring[];
  __shared__ uint64_t full[NST], empty[NST];
  __shared__ double red[TT / 32][HR];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int64_t p = blockIdx.x;
  const int64_t t0 = p * len, t1 = imin64(T, t0 + len);
  if (t0 >= t1) {  // not launched by symv_tma (P is trimmed to the last non-empty range)
    if (LARFG && lf.vav != nullptr && tid == 0) lf.vav[p] = 0.0;
    return;
  }
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const TmaRing R{ring, full, empty};
  TmaPolicy pol;
  pol.keep = pol_evict_last();
  pol.stream = keep_c0 == INT64_MIN ? pol_evict_normal() : pol_evict_first();
  if (keep_c0 == INT64_MIN) pol.keep = pol.stream;  // no hints at all
  pol.keep_c0 = keep_c0;
  int64_t pi = tstrip_of(t0, nbs), pj = t0 - pi * (pi + 1);  // producer cursor (thread 0)
  // prologue: the first NST-1 tiles (A is not written by the launch this one may overlap)
  if (tid == 0)
    for (int s = 0; s < NST - 1 && t0 + s < t1; ++s)
      symv_tma_issue<SH>(&map, R, (uint32_t)s, off, pi, pj, ncj, pol);
  pdl_wait();
  pdl_trigger();
  // dlarfg of the raw column x (while the first tiles are in flight); CTA 0 publishes
  double xs = 1.0;
  if (LARFG) {
    double ss = 0.0;
    for (int64_t q = tid; q < lf.nparts; q += TT) ss += __ldcg(lf.part + q);
    ss = warp_sum(ss);
    if (lane == 0) red[0][w] = ss;
    __syncthreads();
    double tot = 0.0;
#pragma unroll
    for (int k = 0; k < TT / 32; ++k) tot += red[0][k];
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
    __syncthreads();  // red is reused by the tile loop
  }
  const bool want_vav = LARFG && lf.vav != nullptr;
  double vav = symv_tma_loop<LARFG, SH>(&map, R, 0u, off, n, d, x, xs, wcol, wrow, nbs, ncj, len,
                                        slots, p, t0, t1, pi, pj, pol, want_vav, red);
  if (want_vav) {
    __syncthreads();
    double sv = warp_sum(vav);
    if (lane == 0) red[0][w] = sv;
    __syncthreads();
    if (tid == 0) {
      double tot = 0.0;
      for (int k2 = 0; k2 < TT / 32; ++k2) tot += red[0][k2];
      lf.vav[p] = tot;
    }
  }
}

// y_b (64 rows) = sum_{i >= b/2} wcol(i, b) + the row partials of strip b/2 (half b%2).
// CTAs ncj .. ncj+7 (only when lt.i > 0): the latrd panel products t (linalg.h LatrdT).
__global__ void __launch_bounds__(512) symv_tma_reduce_kernel(int64_t n, double alpha, double beta,
                                                              double* __restrict__ y,
                                                              const double* __restrict__ wcol,
                                                              const double* __restrict__ wrow,
                                                              int64_t nbs, int64_t ncj, int64_t len,
                                                              int64_t slots, int64_t d, LatrdT lt) {
  __shared__ double red8[32][WC + 1];
  const int64_t b = blockIdx.x;
  pdl_wait();
  pdl_trigger();
  if (b >= ncj) {
    const int q = (int)(b - ncj);
    const int cl = threadIdx.x & 15, grp = threadIdx.x >> 4;
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
  const int t = threadIdx.x & (WC - 1), g = threadIdx.x >> 6;
  double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
  int64_t i = b / 2 + g;
  for (; i + 24 < nbs; i += 32) {
    s0 += __ldcg(wcol + (i * ncj + b) * WC + t);
    s1 += __ldcg(wcol + ((i + 8) * ncj + b) * WC + t);
    s2 += __ldcg(wcol + ((i + 16) * ncj + b) * WC + t);
    s3 += __ldcg(wcol + ((i + 24) * ncj + b) * WC + t);
  }
  for (; i < nbs; i += 8) s0 += __ldcg(wcol + (i * ncj + b) * WC + t);
  const int64_t sb = b / 2, o = sb * (sb + 1), tiles = imin64(2 * sb + 2, ncj);
  const int64_t npc = (o + tiles - 1) / len - o / len + 1;
  for (int64_t q = g; q < npc; q += 8) s1 += __ldcg(wrow + (sb * slots + q) * HR + (b & 1) * 64 + t);
  red8[g][t] = (s0 + s1) + (s2 + s3);
  __syncthreads();
  if (threadIdx.x < WC) {
    const double v = ((red8[0][t] + red8[1][t]) + (red8[2][t] + red8[3][t])) +
                     ((red8[4][t] + red8[5][t]) + (red8[6][t] + red8[7][t]));
    const int64_t idx = b * WC + t - d;
    if (idx >= 0 && idx < n) y[idx] = (beta == 0.0) ? alpha * v : fma(alpha, v, beta * y[idx]);
  }
}

template <bool LARFG, int SH>
static void symv_tma_launch(cudaStream_t st, bool pdl, const TmaSched& s, const CUtensorMap& map,
                            int64_t off, int64_t n, int64_t d, const double* x, double* wcol,
                            double* wrow, int64_t keep_c0, const SymvLarfg& lf) {
  static bool attr = false;
  if (!attr) {
    EM_CK(cudaFuncSetAttribute(symv_tma_kernel<LARFG, SH>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)RING_BYTES));
    attr = true;
  }
  if (pdl) {
    launch_pdl(symv_tma_kernel<LARFG, SH>, dim3((unsigned)s.P), dim3(TT), RING_BYTES, st, map, off,
               n, d, x, wcol, wrow, s.nbs, s.ncj, s.T, s.len, s.slots, keep_c0, lf);
  } else {
    symv_tma_kernel<LARFG, SH><<<(unsigned)s.P, TT, RING_BYTES, st>>>(
        map, off, n, d, x, wcol, wrow, s.nbs, s.ncj, s.T, s.len, s.slots, keep_c0, lf);
    EM_LAUNCHED();
  }
}

void symv_tma(cudaStream_t st, const SymvMap& m, int64_t off, int64_t n, double alpha,
              const double* x, double beta, double* y, double* work, const SymvLarfg* lf,
              const LatrdT* lt, bool pdl) {
  if (n <= 0) return;
  // The tiles start on a 32-row boundary: the block at (off, off) is extended by d = off
  // mod 32 leading rows and columns whose x entries are zero (their products vanish and
  // their y rows are dropped). With a 256-byte aligned base and ld every TMA box then
  // starts 256-byte aligned: 5.9 TB/s instead of 5.0 for 16..64-byte aligned boxes
  // (tools/prof_kernels.py symvoff), and no odd-row box is needed.
  const int64_t d = g_symv_align_off ? 0 : off % 32;
  const int64_t offa = off - d, na = n + d;
  const TmaSched s = tma_sched(na);
  double* wcol = work;
  double* wrow = work + s.nbs * s.ncj * WC;
  const SymvLarfg lfv = lf ? *lf : SymvLarfg{};
  const LatrdT ltv = lt ? *lt : LatrdT{};
  const CUtensorMap& map0 = reinterpret_cast<const CUtensorMap&>(m.opaque[0]);
  const CUtensorMap& map1 = reinterpret_cast<const CUtensorMap&>(m.opaque[1]);
  // L2 retention: the last `keep` columns of the block (their lower part is ~4 keep^2
  // bytes) stay in L2 between launches; 0 = stream everything
  const int64_t keep = (int64_t)sqrt((double)g_symv_keep_mb * 1e6 / 4.0);
  const int64_t keep_c0 = g_symv_keep_mb > 0    ? off + n - keep
                          : g_symv_keep_mb == 0 ? INT64_MAX   // evict_first everywhere
                                                : INT64_MIN;  // < 0: no hint (evict_normal)
  if (offa & 1) {  // only without the alignment shift: a 130-row box from the row before
    if (lf)
      symv_tma_launch<true, 1>(st, pdl, s, map1, offa, n, d, x, wcol, wrow, keep_c0, lfv);
    else
      symv_tma_launch<false, 1>(st, pdl, s, map1, offa, n, d, x, wcol, wrow, keep_c0, lfv);
  } else {
    if (lf)
      symv_tma_launch<true, 0>(st, pdl, s, map0, offa, n, d, x, wcol, wrow, keep_c0, lfv);
    else
      symv_tma_launch<false, 0>(st, pdl, s, map0, offa, n, d, x, wcol, wrow, keep_c0, lfv);
  }
  const unsigned extra = ltv.i > 0 ? 8u : 0u;
  if (pdl) {
    launch_pdl(symv_tma_reduce_kernel, dim3((unsigned)s.ncj + extra), dim3(512), 0, st, n, alpha,
               beta, y, (const double*)wcol, (const double*)wrow, s.nbs, s.ncj, s.len, s.slots,
               d, ltv);
  } else {
    symv_tma_reduce_kernel<<<(unsigned)s.ncj + extra, 512, 0, st>>>(
        n, alpha, beta, y, wcol, wrow, s.nbs, s.ncj, s.len, s.slots, d, ltv);
    EM_LAUNCHED();
  }
}

}  // namespace em
