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

namespace em {

static_assert(sizeof(SymvMap) == 2 * sizeof(CUtensorMap), "SymvMap holds two CUtensorMaps");
extern int g_symv_align_off;

constexpr int HR = 128;                 // tile rows (strip height)
constexpr int WC = 64;                  // tile columns
constexpr int BR = HR + 2;              // box rows for an odd offset: TMA needs a 16-byte
                                        // aligned row start, so it loads from one row earlier
constexpr int NST = 3;                  // ring stages
constexpr int TT = 512;                 // threads per CTA (16 warps x 4 columns)
// box rows / shared column stride / bytes per tile for row offset parity SH
template <int SH>
constexpr int box_rows() { return SH ? BR : HR; }
template <int SH>
constexpr unsigned tile_bytes() { return box_rows<SH>() * WC * sizeof(double); }
constexpr size_t RING_BYTES = (size_t)NST * BR * WC * sizeof(double);

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

__device__ __forceinline__ int64_t tstrip_of(int64_t t, int64_t nbs) {
  int64_t i = (int64_t)((sqrt(4.0 * (double)t + 1.0) - 1.0) * 0.5);
  while (i > 0 && i * (i + 1) > t) --i;
  while ((i + 1) * (i + 2) <= t) ++i;
  return imin64(i, nbs - 1);
}

// ---- mbarrier / TMA ------------------------------------------------------------------
EM_DEVINL void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
EM_DEVINL void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
EM_DEVINL void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
EM_DEVINL void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
EM_DEVINL void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar,
                           uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
// L2 policies: the bottom-right block of the matrix (read by every column's symv of a
// tridiagonalisation) is loaded evict_last, everything else evict_first, so the part of
// the trailing matrix that fits in the 126 MB L2 is re-read from L2, not HBM.
EM_DEVINL uint64_t pol_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
EM_DEVINL uint64_t pol_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}
EM_DEVINL uint64_t pol_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// x of the block extended by d leading rows/columns (see symv_tma): xd = x - d, na = n + d;
// zero for r < d (only reachable in the first strip / first column block: callers take
// this path there and xfast elsewhere), v = [1, xs x] starts at r = d.
EM_DEVINL double xshift(const double* xd, int64_t r, int64_t d, int64_t na, double xs,
                        bool unit0) {
  if (r < d || r >= na) return 0.0;
  if (unit0 && r == d) return 1.0;
  return xs * __ldcg(xd + r);
}
EM_DEVINL double xfast(const double* xd, int64_t r, int64_t na, double xs) {
  return r < na ? xs * __ldcg(xd + r) : 0.0;
}

// ---- kernel ----------------------------------------------------------------------------
// SH = off & 1. Thread rows within the tile (h, q in {0, 1}): SH = 0: 64h + 2 lane + q
// (128-bit shared loads); SH = 1: 64h + 32q + lane (the tile sits one row into the
// box, so 64-bit loads with consecutive lanes on consecutive rows).
template <int SH>
EM_DEVINL int trow(int h, int q, int lane) {
  return SH ? 64 * h + 32 * q + lane : 64 * h + 2 * lane + q;
}

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
  const double* xd = x - d;
  const int64_t na = n + d;
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
  auto tiles_in = [&](int64_t ii) { return imin64(2 * ii + 2, ncj); };
  int64_t i = tstrip_of(t0, nbs), j = t0 - i * (i + 1);
  int64_t pi = i, pj = j;  // producer cursor (thread 0)
  const uint64_t pkeep = pol_evict_last();
  const uint64_t pstream = keep_c0 == INT64_MIN ? pol_evict_normal() : pol_evict_first();
  auto pol_of = [&](int64_t cj) {
    return keep_c0 != INT64_MIN && off + WC * cj >= keep_c0 ? pkeep : pstream;
  };
  // prologue: the first NST-1 tiles (A is not written by the launch this one may overlap)
  if (tid == 0) {
    for (int s = 0; s < NST - 1; ++s) {
      if (t0 + s < t1) {
        mbar_expect_tx(&full[s], tile_bytes<SH>());
        tma_load_2d(ring + (size_t)s * BR * WC, &map, (int)(off + HR * pi - SH),
                    (int)(off + WC * pj), &full[s], pol_of(pj));
      }
      if (pj + 1 < tiles_in(pi)) ++pj; else { ++pi; pj = 0; }
    }
  }
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
  }
  // v^T A v partial of this CTA (x = v): sum x_c colsum_c over tiles + x_r rowsum_r
  double vav = 0.0;
  const bool want_vav = LARFG && lf.vav != nullptr;
  // thread rows 64h + 2*lane + q (h, q in {0,1}); columns 4w + cc
  double xi[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double row[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  bool fresh = true;
  for (int64_t t = t0; t < t1; ++t) {
    const int k = (int)(t - t0);
    const int s = k % NST;
    // producer: tile k+NST-1 into the stage released by tile k-1
    if (tid == 0 && t + NST - 1 < t1) {
      const int kp = k + NST - 1, ps = kp % NST;
      if (kp >= NST) mbar_wait(&empty[ps], (unsigned)((kp / NST - 1) & 1));
      mbar_expect_tx(&full[ps], tile_bytes<SH>());
      tma_load_2d(ring + (size_t)ps * BR * WC, &map, (int)(off + HR * pi - SH),
                  (int)(off + WC * pj), &full[ps], pol_of(pj));
      if (pj + 1 < tiles_in(pi)) ++pj; else { ++pi; pj = 0; }
    }
    const int64_t r0 = i * HR, c0 = j * WC;
    if (fresh) {
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          xi[h][q] = (i == 0) ? xshift(xd, r0 + trow<SH>(h, q, lane), d, na, xs, LARFG)
                              : xfast(xd, r0 + trow<SH>(h, q, lane), na, xs);
          row[h][q] = 0.0;
        }
      fresh = false;
    }
    double xj[4];
    if (j == 0) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) xj[cc] = xshift(xd, c0 + 4 * w + cc, d, na, xs, LARFG);
    } else {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) xj[cc] = xfast(xd, c0 + 4 * w + cc, na, xs);
    }
    mbar_wait(&full[s], (unsigned)((k / NST) & 1));
    const double* S = ring + (size_t)s * BR * WC + SH;
    double col[4];
    // v[h][q]: element (trow(h, q), 4w + cc) of the tile
    auto ld2 = [&](int cc, int h, double& v0, double& v1) {
      const double* Sc = S + (4 * w + cc) * box_rows<SH>();
      if (SH == 0) {
        const double2 v = *reinterpret_cast<const double2*>(Sc + 64 * h + 2 * lane);
        v0 = v.x;
        v1 = v.y;
      } else {
        v0 = Sc[64 * h + lane];
        v1 = Sc[64 * h + 32 + lane];
      }
    };
    if (j < 2 * i) {
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        double cs = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double v0, v1;
          ld2(cc, h, v0, v1);
          row[h][0] = fma(v0, xj[cc], row[h][0]);
          row[h][1] = fma(v1, xj[cc], row[h][1]);
          cs = fma(v0, xi[h][0], fma(v1, xi[h][1], cs));
        }
        col[cc] = cs;
      }
    } else {
      // diagonal tiles j = 2i, 2i+1: element (r, c) is lower when r >= c + 64 (j - 2i)
      const int dsh = 64 * (int)(j - 2 * i);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int c = 4 * w + cc + dsh;
        double cs = 0.0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double v0, v1;
          ld2(cc, h, v0, v1);
          const int ra = trow<SH>(h, 0, lane), rb = trow<SH>(h, 1, lane);
          const double l0 = (ra >= c) ? v0 : 0.0, l1 = (rb >= c) ? v1 : 0.0;
          const double s0 = (ra > c) ? v0 : 0.0, s1 = (rb > c) ? v1 : 0.0;
          row[h][0] = fma(l0, xj[cc], row[h][0]);
          row[h][1] = fma(l1, xj[cc], row[h][1]);
          cs = fma(s0, xi[h][0], fma(s1, xi[h][1], cs));
        }
        col[cc] = cs;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with the stage
    {  // column sums over the 32 lanes: 4 values, 6 shuffles
      const bool h16 = lane & 16, h8 = lane & 8;
      const double a0 = h16 ? col[2] : col[0], a1 = h16 ? col[3] : col[1];
      const double b0 = h16 ? col[0] : col[2], b1 = h16 ? col[1] : col[3];
      const double c0v = a0 + __shfl_xor_sync(0xffffffffu, b0, 16);
      const double c1v = a1 + __shfl_xor_sync(0xffffffffu, b1, 16);
      double v = (h8 ? c1v : c0v) + __shfl_xor_sync(0xffffffffu, h8 ? c0v : c1v, 8);
      v += __shfl_xor_sync(0xffffffffu, v, 4);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      if ((lane & 7) == 0) {
        const int cc = (h16 ? 2 : 0) + (h8 ? 1 : 0);
        wcol[(i * ncj + j) * WC + 4 * w + cc] = v;
        // (selects, not xj[cc]: a runtime index would put xj in local memory)
        if (want_vav) vav = fma(v, h16 ? (h8 ? xj[3] : xj[2]) : (h8 ? xj[1] : xj[0]), vav);
      }
    }
    if (j + 1 == tiles_in(i) || t + 1 == t1) {  // end of this CTA's piece of strip i
      __syncthreads();
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        red[w][trow<SH>(h, 0, lane)] = row[h][0];
        red[w][trow<SH>(h, 1, lane)] = row[h][1];
      }
      __syncthreads();
      if (tid < HR) {
        double sum = 0.0;
#pragma unroll
        for (int k2 = 0; k2 < TT / 32; ++k2) sum += red[k2][tid];
        const int64_t slot = p - (i * (i + 1)) / len;
        wrow[(i * slots + slot) * HR + tid] = sum;
        if (want_vav) vav = fma(sum, xshift(xd, r0 + tid, d, na, xs, LARFG), vav);
      }
      fresh = true;
    }
    if (j + 1 < tiles_in(i)) ++j; else { ++i; j = 0; }
  }
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
