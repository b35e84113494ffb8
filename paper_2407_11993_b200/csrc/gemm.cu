// FP64 DMMA GEMM for sm_100a: C = alpha * op(A) * op(B) + beta * C, column-major.
//
// This is the dense-contraction workhorse of the eigensolve (potrf trailing
// updates, trsm, sygst, sytrd syr2k, D&C merges, Householder back-transform)
// and of the stepping setup (drive projections V^T[R_D L_D M0], C V).
// The reference does these through numpy/OpenBLAS (pkg/src/eddymodes/modal.py:79-81,
// transient.py:140-154) or scalar numba loops (_kernels.py:56-79).
//
// Warp tile 32x32 = 4x4 DMMA.8x8x4 fragments, k tile 16, 3-4-stage cp.async pipeline,
// padded shared-memory layouts chosen so every 8-byte fragment load is bank-conflict
// free (row strides = 4 mod 16 doubles). Two CTA configurations (GCfg below): 64x64
// tiles with 4 warps and 4 CTAs per SM (the default), 128x64 with 8 warps and 2 CTAs.
#include "common.cuh"
#include "gemm.h"
#include "ctx.h"

namespace em {

// tile configuration (em_config debug key 96): 0 = CfgT3 for transposed A, else CfgT;
// 2 = CfgT, 3 = CfgS, 4 = CfgT3, 5 = paired-fragment tiles (gemm_tile_pf) (A/B). In the C2
// step CfgT everywhere beats the shape rule "CfgS for long k" that the isolated probes
// suggested (2113 -> 2103 ms: ormtr 326 -> 322, l_n product 160 -> 154)
int64_t g_gemm_cfg = 0;

constexpr int GBK = 16, GTHREADS = 256;
constexpr int SPAD_K = GBK + 4;  // 20 ≡ 4 (mod 16)

// CTA tile BM x BN, warp tile (8 TM) x (8 TN) DMMA 8x8 fragments, MINB CTAs per SM.
template <int BM, int BN, int TM, int TN, int MINB>
struct GCfg {
  static constexpr int M = BM, N = BN, WTM = TM, WTN = TN, MINB_ = MINB;
  static constexpr int WGM = BM / (8 * TM);  // warps along m
  static constexpr int WGN = BN / (8 * TN);  // warps along n
  static constexpr int SPM = BM + 4, SPN = BN + 4;  // ≡ 4 (mod 16): conflict-free fragments
  static constexpr int THREADS = WGM * WGN * 32;
};
// 128x64 tiles, 32x32 warp tiles, two CTAs per SM (the epilogue of one overlaps the
// other's main loop): the previous default, kept for A/B (debug key 96 = 3).
using CfgS = GCfg<128, 64, 4, 4, 2>;
// 64x64 tiles, 4 warps of 32x32, four CTAs per SM (barriers over 4 warps, three other
// CTAs to cover each one's prologue and epilogue): short K (tools/gemm_probe.py, beta = 1:
// K = 128 23.8 -> 27.6 TF/s, K = 256 27.4 -> 29.8, K = 512 29.7 -> 31.0; long K with
// few output tiles measured better on CfgS in isolation, not inside the eigensolve).
// Measured and dropped: 128x128 tiles with 32x64 warp tiles, one CTA per SM (30.4 vs
// 31.8 TF/s at 8192^3), and 64x128 tiles with 4 warps of 32x64, two CTAs per SM (no
// better anywhere): every configuration plateaus at ~32 TF/s on large squares
// (cuBLAS: 36).
using CfgT = GCfg<64, 64, 4, 4, 4>;
using CfgT3 = GCfg<64, 64, 4, 4, 3>;  // three CTAs per SM (up to 168 registers)
constexpr int GBM = 128;  // m tile of both configurations (split-K / grouped bookkeeping)

// Strides of the "paired fragment" tiles (PF, 16-byte operands): every thread loads the
// fragments of two consecutive k-steps (k-contiguous tiles) or of two 8-row fragments
// (m/n-contiguous tiles) with ONE 16-byte shared load. The k order inside a 8-deep k pair
// is permuted to k = 8q + 2t + e (k-step 2q + e, lane t) on both operands, and the rows /
// columns of a fragment pair are interleaved (fragment 2p + e, lane g: row 16p + 2g + e).
// Bank-conflict free for these strides: 24 doubles for k-contiguous tiles, 66 for m/n.
constexpr int PF_K = 24;

template <int TA, class C, int PF = 0>
struct ATile {
  static constexpr int SK = PF ? PF_K : SPAD_K, SM = PF ? C::M + 2 : C::SPM;
  static constexpr int size = TA ? C::M * SK : GBK * SM;
  EM_DEVINL static int idx(int m, int k) { return TA ? m * SK + k : k * SM + m; }
};
template <int TB, class C, int PF = 0>
struct BTile {
  static constexpr int SK = PF ? PF_K : SPAD_K, SN = PF ? C::N + 2 : C::SPN;
  static constexpr int size = TB ? GBK * SN : C::N * SK;
  EM_DEVINL static int idx(int k, int n) { return TB ? k * SN + n : n * SK + k; }
};

// Pipeline depth: 4 stages when all MINB CTAs still fit in shared memory, else 3.
template <int TA, int TB, class C, int PF = 0>
constexpr int gstages() {
  constexpr int per = (ATile<TA, C, PF>::size + BTile<TB, C, PF>::size) * 8;
  return C::MINB_ >= 3 ? (per * 4 * C::MINB_ <= 220 * 1024 ? 4 : 3)
                       : (per * 4 * C::MINB_ <= 226 * 1024 ? 4 : 3);
}

// Load a LONG x GBK slab of op(X) (the "long" extent is LONG, the k extent GBK).
// TRANS == 0: X stored long-contiguous (X[l + k*ld]); TRANS == 1: k-contiguous (X[k + l*ld]).
// AL: X is lower triangular (element (l, k) used only when k <= l; the stored upper
// part is ignored) — VEC == 1 only.
template <int TRANS, int VEC, int LONG, int AL = 0, int NT = GTHREADS, int PF = 0>
EM_DEVINL void load_slab(double* s, const double* __restrict__ X, int64_t ld, int64_t l0,
                         int64_t k0, int64_t L, int64_t K, int tid) {
  static_assert(!AL || (VEC == 1 && TRANS == 0), "lower-A loads are 8-byte, long-contiguous");
  constexpr int SPL = PF ? LONG + 2 : LONG + 4;
  constexpr int SKK = PF ? PF_K : SPAD_K;
  if (!TRANS) {
    // contiguous along l; smem [k][l] stride SPL
    constexpr int CH = LONG * GBK / VEC;
#pragma unroll
    for (int c = tid; c < CH; c += NT) {
      int kk = c / (LONG / VEC);
      int l = (c % (LONG / VEC)) * VEC;
      int64_t gl = l0 + l, gk = k0 + kk;
      double* dst = s + kk * SPL + l;
      if (VEC == 2) {
        int nv = (gk < K) ? (int)imin64(imax64(L - gl, 0), 2) : 0;
        const double* src = nv ? X + gl + gk * ld : X;
        cp_async16(dst, src, nv * 8);
      } else {
        bool v = (gk < K) && (gl < L) && (!AL || gk <= gl);
        cp_async8(dst, v ? X + gl + gk * ld : X, v);
      }
    }
  } else {
    // contiguous along k; smem [l][k] stride SPAD_K
    constexpr int CH = LONG * GBK / VEC;
#pragma unroll
    for (int c = tid; c < CH; c += NT) {
      int l = c / (GBK / VEC);
      int kk = (c % (GBK / VEC)) * VEC;
      int64_t gl = l0 + l, gk = k0 + kk;
      double* dst = s + l * SKK + kk;
      if (VEC == 2) {
        int nv = (gl < L) ? (int)imin64(imax64(K - gk, 0), 2) : 0;
        const double* src = nv ? X + gk + gl * ld : X;
        cp_async16(dst, src, nv * 8);
      } else {
        bool v = (gk < K) && (gl < L);
        cp_async8(dst, v ? X + gk + gl * ld : X, v);
      }
    }
  }
}

// One CTA tile of the product. Shared by the plain and grouped kernels.
// AL: A (TA == 0) is lower triangular: k-tiles past the tile's last row are skipped.
template <int TA, int TB, int LOWER, int VEC, int AL = 0, class C = CfgS>
EM_DEVINL void gemm_tile(const GemmArgs& p, int64_t m0, int64_t n0, double* smem) {
  constexpr int WGM = C::WGM, WTM = C::WTM, WTN = C::WTN, GBN = C::N;
  using AT = ATile<TA, C>;
  using BT = BTile<TB, C>;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WGM, wn = warp / WGM;  // warp grid WGM x WGN

  constexpr int ASZ = AT::size, BSZ = BT::size;
  constexpr int GSTAGES = gstages<TA, TB, C>();
  double* As = smem;
  double* Bs = smem + GSTAGES * ASZ;

  double acc[WTM][WTN][2];
#pragma unroll
  for (int i = 0; i < WTM; ++i)
#pragma unroll
    for (int j = 0; j < WTN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int64_t nk = AL ? imin64((p.k + GBK - 1) / GBK, (m0 + C::M + GBK - 1) / GBK)
                        : (p.k + GBK - 1) / GBK;
  // prologue
#pragma unroll
  for (int s = 0; s < GSTAGES - 1; ++s) {
    if (s < nk) {
      load_slab<TA, VEC, C::M, AL, C::THREADS>(As + s * ASZ, p.A, p.lda, m0, s * GBK, p.m, p.k, tid);
      load_slab<!TB, VEC, GBN, 0, C::THREADS>(Bs + s * BSZ, p.B, p.ldb, n0, s * GBK, p.n, p.k, tid);
    }
    cp_async_commit();
  }

  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    // issue the load for kt + STAGES - 1 (its buffer was consumed at kt - 1)
    {
      int64_t kn = kt + GSTAGES - 1;
      int sb = (int)(kn % GSTAGES);
      if (kn < nk) {
        load_slab<TA, VEC, C::M, AL, C::THREADS>(As + sb * ASZ, p.A, p.lda, m0, kn * GBK, p.m, p.k, tid);
        load_slab<!TB, VEC, GBN, 0, C::THREADS>(Bs + sb * BSZ, p.B, p.ldb, n0, kn * GBK, p.n, p.k, tid);
      }
      cp_async_commit();
    }
    const double* as = As + (kt % GSTAGES) * ASZ;
    const double* bs = Bs + (kt % GSTAGES) * BSZ;
    // fragments double-buffered in registers: the loads for k-step ks+1 are issued
    // before the 32 DMMAs of k-step ks
    double af[2][WTM], bf[2][WTN];
#pragma unroll
    for (int i = 0; i < WTM; ++i) af[0][i] = as[AT::idx(wm * 8 * WTM + i * 8 + g, t)];
#pragma unroll
    for (int j = 0; j < WTN; ++j) bf[0][j] = bs[BT::idx(t, wn * 8 * WTN + j * 8 + g)];
#pragma unroll
    for (int ks = 0; ks < GBK / 4; ++ks) {
      const int cur = ks & 1, nx = cur ^ 1;
      if (ks + 1 < GBK / 4) {
        const int kk = (ks + 1) * 4 + t;
#pragma unroll
        for (int i = 0; i < WTM; ++i) af[nx][i] = as[AT::idx(wm * 8 * WTM + i * 8 + g, kk)];
#pragma unroll
        for (int j = 0; j < WTN; ++j) bf[nx][j] = bs[BT::idx(kk, wn * 8 * WTN + j * 8 + g)];
      }
#pragma unroll
      for (int i = 0; i < WTM; ++i)
#pragma unroll
        for (int j = 0; j < WTN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
    }
  }
  cp_async_wait<0>();

  // epilogue: C = alpha acc + beta C. The C loads of two 8-row fragment groups are
  // issued together before any of their stores (16 loads in flight per thread), so a
  // beta != 0 update (trsm, syr2k, potrf, ormtr) is not a chain of dependent round trips.
  double* __restrict__ Cr = p.C;
  const bool has_beta = p.beta != 0.0;
  constexpr int EB = WTN > 4 ? 1 : 2;  // fragment rows per C-load batch (registers)
#pragma unroll
  for (int i2 = 0; i2 < WTM; i2 += EB) {
    double cv[EB][WTN][2];
    bool ok[EB][WTN][2];
#pragma unroll
    for (int ii = 0; ii < EB; ++ii) {
      const int64_t row = m0 + wm * 8 * WTM + (i2 + ii) * 8 + g;
#pragma unroll
      for (int j = 0; j < WTN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = n0 + wn * 8 * WTN + j * 8 + 2 * t + e;
          ok[ii][j][e] = row < p.m && col < p.n && !(LOWER && row + p.diag_off < col);
          cv[ii][j][e] = (has_beta && ok[ii][j][e]) ? Cr[row + col * p.ldc] : 0.0;
        }
    }
#pragma unroll
    for (int ii = 0; ii < EB; ++ii) {
      const int64_t row = m0 + wm * 8 * WTM + (i2 + ii) * 8 + g;
#pragma unroll
      for (int j = 0; j < WTN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if (!ok[ii][j][e]) continue;
          const int64_t col = n0 + wn * 8 * WTN + j * 8 + 2 * t + e;
          const double v = p.alpha * acc[i2 + ii][j][e];
          Cr[row + col * p.ldc] = has_beta ? fma(p.beta, cv[ii][j][e], v) : v;
        }
    }
  }
}

// gemm_tile with paired fragments (16-byte operands only): half the shared-memory load
// instructions of gemm_tile for the same bytes (see PF_K above).
template <int TA, int TB, int LOWER, class C>
EM_DEVINL void gemm_tile_pf(const GemmArgs& p, int64_t m0, int64_t n0, double* smem) {
  constexpr int WGM = C::WGM, WTM = C::WTM, WTN = C::WTN, GBN = C::N;
  static_assert(WTM % 2 == 0 && WTN % 2 == 0, "fragment pairs");
  using AT = ATile<TA, C, 1>;
  using BT = BTile<TB, C, 1>;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % WGM, wn = warp / WGM;
  constexpr int ASZ = AT::size, BSZ = BT::size;
  constexpr int GSTAGES = gstages<TA, TB, C, 1>();
  double* As = smem;
  double* Bs = smem + GSTAGES * ASZ;
  double acc[WTM][WTN][2];
#pragma unroll
  for (int i = 0; i < WTM; ++i)
#pragma unroll
    for (int j = 0; j < WTN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int64_t nk = (p.k + GBK - 1) / GBK;
#pragma unroll
  for (int s2 = 0; s2 < GSTAGES - 1; ++s2) {
    if (s2 < nk) {
      load_slab<TA, 2, C::M, 0, C::THREADS, 1>(As + s2 * ASZ, p.A, p.lda, m0, s2 * GBK, p.m, p.k, tid);
      load_slab<!TB, 2, GBN, 0, C::THREADS, 1>(Bs + s2 * BSZ, p.B, p.ldb, n0, s2 * GBK, p.n, p.k, tid);
    }
    cp_async_commit();
  }
  const int mb = wm * 8 * WTM, nb = wn * 8 * WTN;
  for (int64_t kt = 0; kt < nk; ++kt) {
    cp_async_wait<GSTAGES - 2>();
    __syncthreads();
    {
      const int64_t kn = kt + GSTAGES - 1;
      const int sb = (int)(kn % GSTAGES);
      if (kn < nk) {
        load_slab<TA, 2, C::M, 0, C::THREADS, 1>(As + sb * ASZ, p.A, p.lda, m0, kn * GBK, p.m, p.k, tid);
        load_slab<!TB, 2, GBN, 0, C::THREADS, 1>(Bs + sb * BSZ, p.B, p.ldb, n0, kn * GBK, p.n, p.k, tid);
      }
      cp_async_commit();
    }
    const double* as = As + (kt % GSTAGES) * ASZ;
    const double* bs = Bs + (kt % GSTAGES) * BSZ;
#pragma unroll
    for (int q = 0; q < GBK / 8; ++q) {
      double af[2][WTM], bf[2][WTN];
      if (TA == 0) {  // [k][m]: one load = rows 16p + 2g, +1 of one k-step
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int pp = 0; pp < WTM / 2; ++pp) {
            const double2 v = *reinterpret_cast<const double2*>(
                as + AT::idx(mb + 16 * pp + 2 * g, 8 * q + 2 * t + e));
            af[e][2 * pp] = v.x;
            af[e][2 * pp + 1] = v.y;
          }
      } else {  // [m][k]: one load = k-steps 2q, 2q+1 of one fragment
#pragma unroll
        for (int i = 0; i < WTM; ++i) {
          const double2 v =
              *reinterpret_cast<const double2*>(as + AT::idx(mb + 8 * i + g, 8 * q + 2 * t));
          af[0][i] = v.x;
          af[1][i] = v.y;
        }
      }
      if (TB == 0) {  // [n][k]
#pragma unroll
        for (int j = 0; j < WTN; ++j) {
          const double2 v =
              *reinterpret_cast<const double2*>(bs + BT::idx(8 * q + 2 * t, nb + 8 * j + g));
          bf[0][j] = v.x;
          bf[1][j] = v.y;
        }
      } else {  // [k][n]: one load = columns 16p + 2g, +1 of one k-step
#pragma unroll
        for (int e = 0; e < 2; ++e)
#pragma unroll
          for (int pp = 0; pp < WTN / 2; ++pp) {
            const double2 v = *reinterpret_cast<const double2*>(
                bs + BT::idx(8 * q + 2 * t + e, nb + 16 * pp + 2 * g));
            bf[e][2 * pp] = v.x;
            bf[e][2 * pp + 1] = v.y;
          }
      }
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int i = 0; i < WTM; ++i)
#pragma unroll
          for (int j = 0; j < WTN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[e][i], bf[e][j]);
    }
  }
  cp_async_wait<0>();
  // epilogue (rows / columns of the interleaved fragment pairs)
  double* __restrict__ Cr = p.C;
  const bool has_beta = p.beta != 0.0;
#pragma unroll
  for (int i = 0; i < WTM; ++i) {
    const int64_t row = m0 + mb + (TA == 0 ? 16 * (i >> 1) + 2 * g + (i & 1) : 8 * i + g);
    double cv[WTN][2];
    bool ok[WTN][2];
#pragma unroll
    for (int j = 0; j < WTN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int64_t col =
            n0 + nb + (TB == 1 ? 16 * (j >> 1) + 2 * (2 * t + e) + (j & 1) : 8 * j + 2 * t + e);
        ok[j][e] = row < p.m && col < p.n && !(LOWER && row + p.diag_off < col);
        cv[j][e] = (has_beta && ok[j][e]) ? Cr[row + col * p.ldc] : 0.0;
      }
#pragma unroll
    for (int j = 0; j < WTN; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if (!ok[j][e]) continue;
        const int64_t col =
            n0 + nb + (TB == 1 ? 16 * (j >> 1) + 2 * (2 * t + e) + (j & 1) : 8 * j + 2 * t + e);
        const double v = p.alpha * acc[i][j][e];
        Cr[row + col * p.ldc] = has_beta ? fma(p.beta, cv[j][e], v) : v;
      }
  }
}

template <int TA, int TB, int LOWER, int VEC, int AL = 0, class C = CfgS>
__global__ void __launch_bounds__(C::THREADS, C::MINB_) gemm_kernel(GemmArgs p, double* ws, int64_t kc) {
  constexpr int GBN = C::N;
  extern __shared__ __align__(16) double smem[];
  if (ws) {
    // split-K: slice z of the k range into its own m x n partial (alpha = 1, beta = 0)
    const int64_t z = blockIdx.z;
    const int64_t k0 = z * kc;
    const int64_t kk = imin64(kc, p.k - k0);
    p.A += TA ? k0 : k0 * p.lda;
    p.B += TB ? k0 * p.ldb : k0;
    p.k = kk;
    p.C = ws + z * p.m * p.n;
    p.ldc = p.m;
    p.alpha = 1.0;
    p.beta = 0.0;
  }
  // grouped-M swizzle for L2 reuse: walk 8 m-tiles per n-tile column group
  const int64_t tiles_m = (p.m + C::M - 1) / C::M;
  const int64_t tiles_n = (p.n + GBN - 1) / GBN;
  const int64_t bid = blockIdx.x;
  constexpr int GROUP = 8;
  const int64_t per_group = GROUP * tiles_n;
  const int64_t grp = bid / per_group;
  const int64_t first_m = grp * GROUP;
  const int64_t gsz = imin64(tiles_m - first_m, GROUP);
  const int64_t tm = first_m + (bid % per_group) % gsz;
  const int64_t tn = (bid % per_group) / gsz;
  const int64_t m0 = tm * C::M, n0 = tn * GBN;
  if (LOWER && m0 + C::M - 1 + p.diag_off < n0) return;  // tile strictly above the diagonal
  if constexpr (VEC == 3)
    gemm_tile_pf<TA, TB, LOWER, C>(p, m0, n0, smem);
  else
    gemm_tile<TA, TB, LOWER, VEC, AL, C>(p, m0, n0, smem);
}

// Grouped launch: blockIdx.y selects a problem; problems carry their own sizes/pointers.
template <int TA, int TB, class C>
__global__ void __launch_bounds__(C::THREADS, C::MINB_) gemm_grouped_kernel(
    const GemmArgs* __restrict__ ps, int nprob) {
  extern __shared__ __align__(16) double smem[];
  GemmArgs p = ps[blockIdx.y];
  if (p.m <= 0 || p.n <= 0) return;
  const int64_t tiles_m = (p.m + C::M - 1) / C::M;
  const int64_t tiles_n = (p.n + C::N - 1) / C::N;
  // 16-byte copies when this problem's operands allow them (problem-uniform branch)
  const bool vec = ((reinterpret_cast<uintptr_t>(p.A) | reinterpret_cast<uintptr_t>(p.B)) & 15) == 0 &&
                   ((p.lda | p.ldb) & 1) == 0;
  for (int64_t b = blockIdx.x; b < tiles_m * tiles_n; b += gridDim.x) {
    const int64_t tm = b % tiles_m, tn = b / tiles_m;
    // (k <= 0: C = beta C through the tile with zero accumulators)
    if (vec)
      gemm_tile<TA, TB, 0, 2, 0, C>(p, tm * C::M, tn * C::N, smem);
    else
      gemm_tile<TA, TB, 0, 1, 0, C>(p, tm * C::M, tn * C::N, smem);
    __syncthreads();
  }
}

template <int TA, int TB, class C = CfgS, int PF = 0>
static size_t smem_bytes_t() {
  return (size_t)(ATile<TA, C, PF>::size + BTile<TB, C, PF>::size) * gstages<TA, TB, C, PF>() *
         sizeof(double);
}

// C = alpha * sum_z W_z + beta * C  (split-K reduction, fixed order)
__global__ void splitk_reduce_kernel(int64_t m, int64_t n, int splits, const double* __restrict__ ws,
                                     double alpha, double beta, double* C, int64_t ldc, int lower,
                                     int64_t diag_off) {
  const int64_t total = m * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % m, c = i / m;
    if (lower && r + diag_off < c) continue;
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += ws[z * total + i];
    double* cp = C + r + c * ldc;
    *cp = (beta == 0.0) ? alpha * s : fma(alpha, s, beta * *cp);
  }
}

void splitk_reduce(cudaStream_t st, int64_t m, int64_t n, int splits, const double* ws,
                   double alpha, double beta, double* C, int64_t ldc, int lower, int64_t diag_off) {
  const int64_t total = m * n;
  const int blocks = (int)imin64((total + 255) / 256, 8 * (int64_t)num_sms());
  splitk_reduce_kernel<<<blocks, 256, 0, st>>>(m, n, splits, ws, alpha, beta, C, ldc, lower,
                                               diag_off);
  count_launch();
}

template <int TA, int TB, int LOWER, int VEC, class C>
static cudaError_t launch_t(const GemmArgs& p, cudaStream_t st) {
  auto k = gemm_kernel<TA, TB, LOWER, VEC, 0, C>;
  size_t sm = smem_bytes_t<TA, TB, C, VEC == 3 ? 1 : 0>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  const int64_t tiles = ((p.m + C::M - 1) / C::M) * ((p.n + C::N - 1) / C::N);
  const int sms = num_sms() * (C::MINB_ >= 3 ? C::MINB_ : 1);  // CfgT: CTA slots per SM
  // few output tiles and a long k loop: split k so every SM has work
  // pick the split count with the best wave quantisation (each slice >= 512 deep)
  int64_t splits = 1;
  if (tiles < 4 * sms && p.k >= 2 * 512) {
    auto eff = [&](int64_t s) {
      const int64_t ctas = tiles * s;
      return (double)ctas / (double)(((ctas + sms - 1) / sms) * sms);
    };
    double best = eff(1);
    for (int64_t s = 2; s <= 16 && p.k / s >= 512; ++s) {
      const double e = eff(s);
      if (e > best + 0.03) {
        best = e;
        splits = s;
      }
    }
  }
  if (splits <= 1) {
    k<<<(unsigned)tiles, C::THREADS, sm, st>>>(p, nullptr, 0);
    count_launch();
    return cudaGetLastError();
  }
  int64_t kc = (p.k + splits - 1) / splits;
  kc = (kc + GBK - 1) / GBK * GBK;  // whole k-tiles per split (alignment of the slices)
  splits = (p.k + kc - 1) / kc;
  double* ws = nullptr;
  cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws),
                                  (size_t)splits * p.m * p.n * sizeof(double), st);
  if (e != cudaSuccess) return e;
  dim3 grid((unsigned)tiles, 1, (unsigned)splits);
  k<<<grid, C::THREADS, sm, st>>>(p, ws, kc);
  count_launch();
  splitk_reduce(st, p.m, p.n, (int)splits, ws, p.alpha, p.beta, p.C, p.ldc, LOWER, p.diag_off);
  cudaFreeAsync(ws, st);
  return cudaGetLastError();
}

template <int TA, int TB, int LOWER>
static cudaError_t launch_v(const GemmArgs& p, cudaStream_t st) {
  auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  bool vec = al(p.A) && al(p.B) && (p.lda % 2 == 0) && (p.ldb % 2 == 0);
  // 16-byte chunks also need the tile starts to be even along the contiguous dim;
  // tiles start at multiples of 128 (long dims) and 16 (k), so base alignment suffices.
  // transposed A: three CTAs per SM (more registers) measured faster (V^T Z at K = 16k:
  // 29.6 -> 31.6 TF/s, rank-256 A^T B 28.1 -> 30.3); non-transposed A: four
  if (g_gemm_cfg == 5 && vec)  // paired-fragment tiles
    return TA ? launch_t<TA, TB, LOWER, 3, CfgT3>(p, st) : launch_t<TA, TB, LOWER, 3, CfgT>(p, st);
  if (g_gemm_cfg == 4 || (g_gemm_cfg == 0 && TA))
    return vec ? launch_t<TA, TB, LOWER, 2, CfgT3>(p, st) : launch_t<TA, TB, LOWER, 1, CfgT3>(p, st);
  if (g_gemm_cfg != 3)
    return vec ? launch_t<TA, TB, LOWER, 2, CfgT>(p, st) : launch_t<TA, TB, LOWER, 1, CfgT>(p, st);
  return vec ? launch_t<TA, TB, LOWER, 2, CfgS>(p, st) : launch_t<TA, TB, LOWER, 1, CfgS>(p, st);
}

cudaError_t gemm(cudaStream_t st, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
                 const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
                 int64_t ldc, bool lower, int64_t diag_off) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  GemmArgs p{m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, diag_off};
  if (k <= 0) {
    // pure scaling: C = beta*C
    return scale_matrix(st, m, n, beta, C, ldc, lower, diag_off);
  }
  {  // large aligned products: the TMA-fed persistent kernel (gemm_tma.cu)
    const cudaError_t e = gemm_tma(st, ta, tb, p, lower);
    if (e != cudaErrorNotSupported) return e;
  }
  int code = (ta ? 4 : 0) | (tb ? 2 : 0) | (lower ? 1 : 0);
  switch (code) {
    case 0: return launch_v<0, 0, 0>(p, st);
    case 1: return launch_v<0, 0, 1>(p, st);
    case 2: return launch_v<0, 1, 0>(p, st);
    case 3: return launch_v<0, 1, 1>(p, st);
    case 4: return launch_v<1, 0, 0>(p, st);
    case 5: return launch_v<1, 0, 1>(p, st);
    case 6: return launch_v<1, 1, 0>(p, st);
    default: return launch_v<1, 1, 1>(p, st);
  }
}

template <class C>
static cudaError_t launch_lower_a(const GemmArgs& p, cudaStream_t st) {
  auto kern = gemm_kernel<0, 0, 0, 1, 1, C>;
  const size_t sm = smem_bytes_t<0, 0, C>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  const int64_t tiles = ((p.m + C::M - 1) / C::M) * ((p.n + C::N - 1) / C::N);
  kern<<<(unsigned)tiles, C::THREADS, sm, st>>>(p, nullptr, 0);
  count_launch();
  return cudaGetLastError();
}

cudaError_t gemm_lower_a(cudaStream_t st, int64_t m, int64_t n, int64_t k, double alpha,
                         const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                         double* C, int64_t ldc) {
  if (m <= 0 || n <= 0) return cudaSuccess;
  if (k <= 0) return scale_matrix(st, m, n, beta, C, ldc, false, 0);
  GemmArgs p{m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, 0};
  if (g_gemm_cfg == 4) return launch_lower_a<CfgT3>(p, st);
  if (g_gemm_cfg != 3) return launch_lower_a<CfgT>(p, st);
  return launch_lower_a<CfgS>(p, st);
}

// max_tiles counts 128x64 tiles (the callers' bookkeeping); the 64x64 configuration
// (default, debug key 96 != 3) launches four CTAs per counted tile
template <int TA, int TB, class C>
static cudaError_t grouped_c(const GemmArgs* d_probs, int nprob, int max_tiles, cudaStream_t st) {
  auto k = gemm_grouped_kernel<TA, TB, C>;
  size_t sm = smem_bytes_t<TA, TB, C>();
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured = true;
  }
  const int per = (GBM / C::M) * (CfgS::N / C::N);
  dim3 grid((unsigned)max(1, max_tiles * per), (unsigned)nprob);
  k<<<grid, C::THREADS, sm, st>>>(d_probs, nprob);
  count_launch();
  return cudaGetLastError();
}
template <int TA, int TB>
static cudaError_t grouped_t(const GemmArgs* d_probs, int nprob, int max_tiles, cudaStream_t st) {
  if (g_gemm_cfg == 3) return grouped_c<TA, TB, CfgS>(d_probs, nprob, max_tiles, st);
  return grouped_c<TA, TB, CfgT>(d_probs, nprob, max_tiles, st);
}

cudaError_t gemm_grouped(cudaStream_t st, bool ta, bool tb, const GemmArgs* d_probs, int nprob,
                         int max_tiles) {
  if (nprob <= 0) return cudaSuccess;
  if (!ta && !tb) return grouped_t<0, 0>(d_probs, nprob, max_tiles, st);
  if (!ta && tb) return grouped_t<0, 1>(d_probs, nprob, max_tiles, st);
  if (ta && !tb) return grouped_t<1, 0>(d_probs, nprob, max_tiles, st);
  return grouped_t<1, 1>(d_probs, nprob, max_tiles, st);
}

__global__ void scale_kernel(int64_t m, int64_t n, double beta, double* C, int64_t ldc, int lower,
                             int64_t diag_off) {
  int64_t total = m * n;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i % m, c = i / m;
    if (lower && r + diag_off < c) continue;
    double* p = C + r + c * ldc;
    *p = beta == 0.0 ? 0.0 : beta * *p;
  }
}

cudaError_t scale_matrix(cudaStream_t st, int64_t m, int64_t n, double beta, double* C, int64_t ldc,
                         bool lower, int64_t diag_off) {
  if (m <= 0 || n <= 0 || beta == 1.0) return cudaSuccess;
  int64_t total = m * n;
  int blocks = (int)imin64((total + 255) / 256, 148 * 16);
  scale_kernel<<<blocks, 256, 0, st>>>(m, n, beta, C, ldc, lower ? 1 : 0, diag_off);
  count_launch();
  return cudaGetLastError();
}

}  // namespace em
