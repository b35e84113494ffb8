// Device side of the TMA-fed lower-triangle symv (symv_tma.cu), shared with the
// persistent tridiagonalisation panel kernel (sytrd_panel.cu): constants, mbarrier/TMA
// helpers, the tile schedule and the tile loop of one CTA.
#pragma once
#include <cudaTypedefs.h>

#include "common.cuh"

namespace em {

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

// SH = off & 1. Thread rows within the tile (h, q in {0, 1}): SH = 0: 64h + 2 lane + q
// (128-bit shared loads); SH = 1: 64h + 32q + lane (the tile sits one row into the
// box, so 64-bit loads with consecutive lanes on consecutive rows).
template <int SH>
EM_DEVINL int trow(int h, int q, int lane) {
  return SH ? 64 * h + 32 * q + lane : 64 * h + 2 * lane + q;
}

// ---- one CTA's share of a symv: tiles [t0, t1) of the lower triangle (strip-major) ----
// The mbarrier ring (NST stages of BR x WC doubles, full/empty barriers) may be reused
// across calls: kb counts the tiles this CTA consumed before (stage = (kb + k) % NST and
// the phase parities follow from it). Thread 0 is the producer.
struct TmaRing {
  double* ring;
  uint64_t* full;
  uint64_t* empty;
};
struct TmaPolicy {
  uint64_t keep, stream;
  int64_t keep_c0;  // tiles from this absolute column on use `keep`
  EM_DEVINL uint64_t of(int64_t col) const { return col >= keep_c0 ? keep : stream; }
};

// issue tile number g (global count) at producer cursor (pi, pj) and advance the cursor
template <int SH>
EM_DEVINL void symv_tma_issue(const CUtensorMap* map, const TmaRing& R, uint32_t g, int64_t off,
                              int64_t& pi, int64_t& pj, int64_t ncj, const TmaPolicy& pol) {
  const int ps = (int)(g % NST);
  if (g >= (uint32_t)NST) mbar_wait(&R.empty[ps], (unsigned)((g / NST - 1) & 1));
  mbar_expect_tx(&R.full[ps], tile_bytes<SH>());
  tma_load_2d(R.ring + (size_t)ps * BR * WC, map, (int)(off + HR * pi - SH), (int)(off + WC * pj),
              &R.full[ps], pol.of(off + WC * pj));
  if (pj + 1 < imin64(2 * pi + 2, ncj)) ++pj; else { ++pi; pj = 0; }
}

// Consume tiles [t0, t1) (the first min(NST - 1, t1 - t0) already issued by the caller,
// the producer cursor (pi, pj) just past them). Column sums of every tile go to wcol,
// row sums of this CTA's piece of each strip to wrow (slot p - off(i)/len). Returns this
// thread's part of v^T A v (want_vav). x is scaled by xs; LARFG: x[d] is taken as 1.
template <bool LARFG, int SH>
EM_DEVINL double symv_tma_loop(const CUtensorMap* map, const TmaRing& R, uint32_t kb, int64_t off,
                               int64_t n, int64_t d, const double* __restrict__ x, double xs,
                               double* __restrict__ wcol, double* __restrict__ wrow, int64_t nbs,
                               int64_t ncj, int64_t len, int64_t slots, int64_t p, int64_t t0,
                               int64_t t1, int64_t& pi, int64_t& pj, const TmaPolicy& pol,
                               bool want_vav, double (*red)[HR]) {
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const double* xd = x - d;
  const int64_t na = n + d;
  auto tiles_in = [&](int64_t ii) { return imin64(2 * ii + 2, ncj); };
  int64_t i = tstrip_of(t0, nbs), j = t0 - i * (i + 1);
  double vav = 0.0;
  // thread rows 64h + 2*lane + q (h, q in {0,1}); columns 4w + cc
  double xi[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  double row[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  bool fresh = true;
  for (int64_t t = t0; t < t1; ++t) {
    const uint32_t k = kb + (uint32_t)(t - t0);
    const int s = (int)(k % NST);
    // producer: tile k+NST-1 into the stage released by tile k-1
    if (tid == 0 && t + NST - 1 < t1) symv_tma_issue<SH>(map, R, k + NST - 1, off, pi, pj, ncj, pol);
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
    mbar_wait(&R.full[s], (unsigned)((k / NST) & 1));
    const double* S = R.ring + (size_t)s * BR * WC + SH;
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
    // this warp is done with the stage; the release is data-dependent on the column sums
    // (into which every value loaded from the stage went), so it cannot be scheduled ahead
    // of the loads' completion (never_set, common.cuh; the hazard is described in gemm_tma.cu)
    const unsigned never =
        never_set(col[0]) | never_set(col[1]) | never_set(col[2]) | never_set(col[3]);
    __syncwarp();
    if (lane == 0)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&R.empty[s]) +
                                                                      never)
                   : "memory");
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
  return vav;
}

}  // namespace em
