// TMA-fed, warp-specialised, persistent FP64 DMMA GEMM for sm_100a (large products).
//
// C = alpha * op(A) * op(B) + beta * C, column-major, as gemm.cu (whose cp.async kernels
// stay for small, unaligned, grouped and triangular-A products). The reference does these
// contractions through numpy/OpenBLAS (pkg/src/eddymodes/modal.py:64-81,
// transient.py:140-154).
//
// One producer warp per CTA issues `cp.async.bulk.tensor.2d` for the A and B slabs of
// every k-tile (16 deep) into a ring of shared-memory stages guarded by full/empty
// mbarriers; the consumer warps only wait on a stage's barrier, load DMMA fragments and
// issue `mma.sync.m8n8k4.f64`, then one lane releases the stage. No CTA-wide barrier and no
// per-thread address arithmetic in the main loop (the cp.async kernel spends ~5 non-DMMA
// instructions per DMMA and reaches 86% DMMA-pipe activity, profiles/r01_ncu_gemm_full.json).
// The TMA boxes include the 4-double padding of the conflict-free fragment layouts
// (row strides 132 / 68 / 20 doubles, all = 4 mod 16), so the boxes land in exactly the
// layout the fragments are read from; rows or k past the operand are zero-filled by the
// TMA unit, so edge tiles need no predicates on the load side.
// Tiles are claimed from a global counter (persistent CTAs, self-resetting), in an order
// that keeps 16 tile rows x a run of tile columns in flight (L2 reuse); with LOWER only
// tiles touching the lower triangle are computed. Few-tile / long-k products are split
// along k into workspace partials (fixed-order reduction, as the cp.async path).
#include <cudaTypedefs.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "symv_tma.cuh"

namespace em {

int64_t g_gemm_tma = 1;  // em_config debug key 95: 0 = off, 1 = auto, 2 / 4 / 5 = force TC2 / TC3 / TC4

namespace {

constexpr int TBK = 16;        // k depth of one stage
constexpr int TPK = TBK + 4;   // k-contiguous row stride (20 = 4 mod 16)

// CTA tile BM x BN, consumer warp tile (8 TM) x (8 TN), MINB CTAs per SM, NST stages.
// PW producer warps lead the CTA (one lane of the first issues the TMA copies). With PW = 4
// the producers are a whole warpgroup and `setmaxnreg` moves registers from it to the
// consumer warpgroups (RP / RC registers per thread after the split; 0 = leave as launched).
template <int BM_, int BN_, int TM_, int TN_, int MINB_, int NST_, int PW_, int RC_, int RP_>
struct TCfg {
  static constexpr int BM = BM_, BN = BN_, TM = TM_, TN = TN_, MINB = MINB_, NST = NST_;
  static constexpr int PW = PW_, RC = RC_, RP = RP_;
  static constexpr int WGM = BM / (8 * TM), WGN = BN / (8 * TN);
  static constexpr int NCW = WGM * WGN;        // consumer warps
  static constexpr int THREADS = (NCW + PW) * 32;
  static constexpr int SPM = BM + 4, SPN = BN + 4;
  static_assert(RC == 0 || (PW == 4 && NCW % 4 == 0), "setmaxnreg works on whole warpgroups");
};

template <int R>
EM_DEVINL void reg_dec() {
  if constexpr (R > 0) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(R));
}
template <int R>
EM_DEVINL void reg_inc() {
  if constexpr (R > 0) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(R));
}

template <int TA, class C>
struct TATile {
  static constexpr int size = TA ? C::BM * TPK : TBK * C::SPM;
  __host__ __device__ static constexpr int idx(int m, int k) { return TA ? m * TPK + k : k * C::SPM + m; }
};
template <int TB, class C>
struct TBTile {
  static constexpr int size = TB ? TBK * C::SPN : C::BN * TPK;
  __host__ __device__ static constexpr int idx(int k, int n) { return TB ? k * C::SPN + n : n * TPK + k; }
};

// Ring depth: C::NST stages, fewer when MINB CTAs of that depth do not fit in shared memory.
template <int TA, int TB, class C>
constexpr int tma_stages() {
  constexpr int per = (TATile<TA, C>::size + TBTile<TB, C>::size) * 8;
  constexpr int budget = 227 * 1024 / C::MINB - 1024 - 256;
  return budget / per < C::NST ? budget / per : C::NST;
}

struct TmaGemmParams {
  GemmArgs p;
  double* ws;          // split-k partials (nullptr: direct)
  int64_t kc;          // k per split (multiple of TBK)
  int splits;
  int64_t tiles_m, tiles_n;
  unsigned long long* ctr;  // [0] next unit, [1] CTAs done
  int prefetch_c;           // beta != 0 and C admits a tensor map: L2-prefetch each C tile
  // Column ownership of a distributed band reduction (own_g ranks, this one own_r; 64-column
  // blocks dealt round-robin, block index = own_org + column / 64): a LOWER product
  // updates only the owned column tiles (BN = 64); a SYMM product adds up only the k-tiles
  // read from owned columns (stored reads: the k-tile's block; transposed reads: the row
  // tile's block, BM = 64), i.e. this rank's partial of the product. own_g = 1: everything.
  int own_g, own_r;
  int64_t own_org;
  int sh_a, sh_b;           // operand starts 8 bytes past a 16-byte boundary: the map's base is
                            // the aligned address below it (TMA box starts must be 16-byte
                            // aligned), so the tile sits one element into its box — inside
                            // the 4 padding elements — and the fragment offsets move up by 1
};

constexpr int TGROUP = 16;  // tile rows walked per tile-column run

template <class C, int LOWER>
EM_DEVINL bool unit_decode(const TmaGemmParams& q, int64_t u, int64_t& m0, int64_t& n0, int& z) {
  const int64_t tiles = q.tiles_m * q.tiles_n;
  z = (int)(u / tiles);
  const int64_t b = u % tiles;
  const int64_t per_group = TGROUP * q.tiles_n;
  const int64_t grp = b / per_group;
  const int64_t first_m = grp * TGROUP;
  const int64_t gsz = imin64(q.tiles_m - first_m, TGROUP);
  const int64_t tm = first_m + (b % per_group) % gsz;
  const int64_t tn = (b % per_group) / gsz;
  m0 = tm * C::BM;
  n0 = tn * C::BN;
  if (LOWER && q.own_g > 1 && (q.own_org + n0 / 64) % q.own_g != q.own_r) return false;
  return !(LOWER && m0 + C::BM - 1 + q.p.diag_off < n0);
}

// SYMM with column ownership: does this rank add k-tile kk of row tile m0?
template <class C>
EM_DEVINL bool ktile_owned(const TmaGemmParams& q, int64_t m0, int64_t kk) {
  if (q.own_g <= 1) return true;
  const int64_t col = kk >= m0 + C::BM ? m0 : kk;  // transposed reads come from columns m0..
  return (q.own_org + col / 64) % q.own_g == q.own_r;
}

// One k-tile of the warp tile: fragments of a TA_/TB_-layout stage (pointers at this lane's
// k-step-0 fragments), double-buffered in registers.
template <int TA_, int TB_, class C>
EM_DEVINL void ktile_mma(double (&acc)[C::TM][C::TN][2], const double* as, const double* bs) {
  using AT = TATile<TA_, C>;
  using BT = TBTile<TB_, C>;
  constexpr int WTM = C::TM, WTN = C::TN;
  constexpr int A_I = AT::idx(8, 0) - AT::idx(0, 0);   // next 8-row fragment
  constexpr int A_K = AT::idx(0, 4) - AT::idx(0, 0);   // next k-step
  constexpr int B_J = BT::idx(0, 8) - BT::idx(0, 0);
  constexpr int B_K = BT::idx(4, 0) - BT::idx(0, 0);
  double af[2][WTM], bf[2][WTN];
#pragma unroll
  for (int i = 0; i < WTM; ++i) af[0][i] = as[i * A_I];
#pragma unroll
  for (int j = 0; j < WTN; ++j) bf[0][j] = bs[j * B_J];
#pragma unroll
  for (int ks = 0; ks < TBK / 4; ++ks) {
    const int cur = ks & 1, nx = cur ^ 1;
    if (ks + 1 < TBK / 4) {
#pragma unroll
      for (int i = 0; i < WTM; ++i) af[nx][i] = as[i * A_I + (ks + 1) * A_K];
#pragma unroll
      for (int j = 0; j < WTN; ++j) bf[nx][j] = bs[j * B_J + (ks + 1) * B_K];
    }
#pragma unroll
    for (int i = 0; i < WTM; ++i)
#pragma unroll
      for (int j = 0; j < WTN; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[cur][i], bf[cur][j]);
  }
}

// SYMM: C = A B for a symmetric A given by its lower triangle plus the BM - 1 diagonals above
// it (TA is ignored, A is m x m = k x k): the k-tiles of a row tile left of and on its
// diagonal block are read as stored (A[m0.., kk..], m-contiguous boxes of mapA), those
// below it through the transpose (A[kk.., m0..]^T, k-contiguous boxes of mapC, which no
// beta = 0 product needs for C) — every row tile runs over the whole k range.
template <int TA, int TB, int LOWER, class C, int SYMM = 0>
__global__ void __launch_bounds__(C::THREADS, C::MINB)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap mapA,
                    const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapC, const TmaGemmParams q) {
  using AT = TATile<SYMM ? 0 : TA, C>;
  using ATT = TATile<1, C>;  // SYMM: the transposed reads
  using BT = TBTile<TB, C>;
  constexpr int ASZ = SYMM ? (ATT::size > AT::size ? ATT::size : AT::size) : AT::size;
  constexpr int BSZ = BT::size, NST = tma_stages<(SYMM ? 1 : TA), TB, C>();
  constexpr unsigned STAGE_BYTES = (AT::size + BSZ) * sizeof(double);
  constexpr unsigned STAGE_BYTES_T = (ATT::size + BSZ) * sizeof(double);
  extern __shared__ __align__(128) double smem[];
  double* As = smem;
  double* Bs = smem + NST * ASZ;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + NST * (ASZ + BSZ));
  uint64_t* empty = full + NST;
  uint64_t* tq_full = empty + NST;   // [2]
  uint64_t* tq_empty = tq_full + 2;  // [2]
  long long* tq_val = reinterpret_cast<long long*>(tq_empty + 2);  // [2]

  const int tid = threadIdx.x;
  const int warp_all = tid >> 5, lane = tid & 31;
  if (tid == 0) {
#pragma unroll
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C::NCW);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tq_full[s], 1);
      mbar_init(&tq_empty[s], C::NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int64_t total = q.tiles_m * q.tiles_n * q.splits;

  if (warp_all < C::PW) {
    // ---------------- producer ----------------
    reg_dec<C::RP>();
    if (tid != 0) return;
    const uint64_t pol = pol_evict_normal();
    unsigned it = 0, tq = 0;
    for (;;) {
      int64_t u, m0 = 0, n0 = 0;
      int z = 0;
      do {
        u = (int64_t)atomicAdd(q.ctr, 1ull);
      } while (u < total && !unit_decode<C, LOWER>(q, u, m0, n0, z));
      mbar_wait(&tq_empty[tq & 1], ((tq >> 1) & 1) ^ 1);
      tq_val[tq & 1] = u < total ? (long long)u : -1ll;
      mbar_arrive(&tq_full[tq & 1]);
      ++tq;
      if (u >= total) break;
      // the epilogue's reads of C (beta != 0) are dependent round trips: fetch the tile into
      // L2 now, a whole main loop ahead
      if (!SYMM && q.prefetch_c)
        asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];\n" ::"l"(
                         &mapC),
                     "r"((int)m0), "r"((int)n0)
                     : "memory");
      const int64_t k0 = (int64_t)z * q.kc;
      const int64_t kl = imin64(q.kc, q.p.k - k0);
      const int nk = (int)((kl + TBK - 1) / TBK);
      for (int kt = 0; kt < nk; ++kt) {
        const int kk = (int)(k0 + (int64_t)kt * TBK);
        if (SYMM && !ktile_owned<C>(q, m0, kk)) continue;
        const int s = it % NST;
        mbar_wait(&empty[s], ((it / NST) & 1) ^ 1);
        ++it;
        if (SYMM && kk >= m0 + C::BM) {
          mbar_expect_tx(&full[s], STAGE_BYTES_T);
          tma_load_2d(As + s * ASZ, &mapC, kk, (int)m0, &full[s], pol);
        } else {
          mbar_expect_tx(&full[s], STAGE_BYTES);
          tma_load_2d(As + s * ASZ, &mapA, (SYMM || !TA) ? (int)m0 : kk,
                      (SYMM || !TA) ? kk : (int)m0, &full[s], pol);
        }
        tma_load_2d(Bs + s * BSZ, &mapB, TB ? (int)n0 : kk, TB ? kk : (int)n0, &full[s], pol);
      }
    }
    // the last CTA to finish claiming resets the counters for the next launch
    const unsigned long long done = atomicAdd(q.ctr + 1, 1ull);
    if (done == gridDim.x - 1) {
      q.ctr[0] = 0ull;
      q.ctr[1] = 0ull;
      __threadfence();
    }
    return;
  }

  // ---------------- consumers ----------------
  reg_inc<C::RC>();
  const int warp = warp_all - C::PW;
  constexpr int WTM = C::TM, WTN = C::TN;
  const int g = lane >> 2, t = lane & 3;
  const int wm = warp % C::WGM, wn = warp / C::WGM;
  const int mb = wm * 8 * WTM, nb = wn * 8 * WTN;
  // fragment offsets of this lane for k-step 0 (constant over the kernel)
  const int a_off = AT::idx(mb + g, t) + q.sh_a;
  const int a_off_t = ATT::idx(mb + g, t);
  const int b_off = BT::idx(t, nb + g) + q.sh_b;
  unsigned it = 0, tq = 0;
  for (;;) {
    mbar_wait(&tq_full[tq & 1], (tq >> 1) & 1);
    const long long u = tq_val[tq & 1];
    __syncwarp();
    if (lane == 0) mbar_arrive(&tq_empty[tq & 1]);
    ++tq;
    if (u < 0) break;
    int64_t m0, n0;
    int z;
    unit_decode<C, LOWER>(q, u, m0, n0, z);
    const int64_t k0 = (int64_t)z * q.kc;
    const int64_t kl = imin64(q.kc, q.p.k - k0);
    const int nk = (int)((kl + TBK - 1) / TBK);

    double acc[WTM][WTN][2];
#pragma unroll
    for (int i = 0; i < WTM; ++i)
#pragma unroll
      for (int j = 0; j < WTN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    int done = 0;  // k-tiles of this unit consumed so far
    for (int kt = 0; kt < nk; ++kt) {
      const int64_t kk = k0 + (int64_t)kt * TBK;
      if (SYMM && !ktile_owned<C>(q, m0, kk)) continue;
      const int s = it % NST;
      mbar_wait(&full[s], (it / NST) & 1);
      ++it;
      const double* bs = Bs + s * BSZ + b_off;
      if (SYMM && kk >= m0 + C::BM)
        ktile_mma<1, TB, C>(acc, As + s * ASZ + a_off_t, bs);
      else
        ktile_mma<(SYMM ? 0 : TA), TB, C>(acc, As + s * ASZ + a_off, bs);
      // Release the PREVIOUS stage: every DMMA that consumed its fragments has been issued
      // by now (they precede this k-tile's barrier wait), so its shared-memory reads are
      // done. Releasing a stage right after its own last fragment load is not safe: ptxas
      // places the arrive directly behind the last LDS, ahead of the DMMAs that consume it,
      // and an LDS queued behind the epilogue's global loads/stores of the other warps can
      // be overtaken by the arrive and then by the producer's next TMA write into the stage
      // (seen as wrong 16 x 64 blocks with beta != 0, tools/dbg_gemm_tma.py).
      __syncwarp();
      if (done > 0 && lane == 0) mbar_arrive(&empty[(it + NST - 2) % NST]);
      ++done;
    }

    if (done > 0) {
      // The tile's last stage is released before the epilogue (so the producer refills the
      // whole ring under it). The barrier address carries a data dependency on every
      // accumulator, so the arrive cannot issue before the final DMMAs have delivered, i.e.
      // before their fragment loads are done (the added term is always zero: never_set in
      // common.cuh).
      unsigned never = 0u;
#pragma unroll
      for (int i = 0; i < WTM; ++i)
#pragma unroll
        for (int j = 0; j < WTN; ++j) never |= never_set(acc[i][j][0]);
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(
                         smem_u32(&empty[(it + NST - 1) % NST]) + never)
                     : "memory");
    }
    // epilogue: C = alpha acc + beta C (split-k: the partial of slice z, alpha 1, beta 0)
    double* __restrict__ Cr = q.ws ? q.ws + (int64_t)z * q.p.m * q.p.n : q.p.C;
    const int64_t ldc = q.ws ? q.p.m : q.p.ldc;
    const double alpha = q.ws ? 1.0 : q.p.alpha;
    const double beta = q.ws ? 0.0 : q.p.beta;
    const bool has_beta = beta != 0.0;
    // Interior tiles (no edge, not cut by the LOWER diagonal) take a path without
    // per-element predicates or address arithmetic, software-pipelined over the fragment
    // rows: the C loads of row i + 1 are in flight while row i is combined and stored (the
    // general path below spilled registers and waited on every load round trip:
    // profiles/r02/ncu_gemm_tma.json, K = 128, beta = 1).
    const bool interior = m0 + C::BM <= q.p.m && n0 + C::BN <= q.p.n &&
                          (!LOWER || q.ws != nullptr || m0 + q.p.diag_off >= n0 + C::BN - 1);
    if (interior) {
      double* cp = Cr + (m0 + mb + g) + (n0 + nb + 2 * t) * ldc;
      double cv[2][WTN][2];
      if (has_beta) {
#pragma unroll
        for (int j = 0; j < WTN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) cv[0][j][e] = cp[(8 * j + e) * ldc];
      }
#pragma unroll
      for (int i = 0; i < WTM; ++i) {
        if (has_beta && i + 1 < WTM) {
#pragma unroll
          for (int j = 0; j < WTN; ++j)
#pragma unroll
            for (int e = 0; e < 2; ++e) cv[(i + 1) & 1][j][e] = cp[8 * (i + 1) + (8 * j + e) * ldc];
        }
#pragma unroll
        for (int j = 0; j < WTN; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const double v = alpha * acc[i][j][e];
            cp[8 * i + (8 * j + e) * ldc] = has_beta ? fma(beta, cv[i & 1][j][e], v) : v;
          }
      }
      continue;
    }
#pragma unroll
    for (int i2 = 0; i2 < WTM; ++i2) {
      const int64_t row = m0 + mb + i2 * 8 + g;
#pragma unroll
      for (int j = 0; j < WTN; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t col = n0 + nb + j * 8 + 2 * t + e;
          const bool ok = row < q.p.m && col < q.p.n &&
                          !(LOWER && !q.ws && row + q.p.diag_off < col);
          if (!ok) continue;
          const double v = alpha * acc[i2][j][e];
          double* cpe = Cr + row + col * ldc;
          *cpe = has_beta ? fma(beta, *cpe, v) : v;
        }
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) ==
            cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    else
      cudaGetLastError();
  }
  return fn;
}

// 2-D map over a column-major operand: `inner` contiguous elements, `outer` columns of
// stride ld; box = (box_inner, box_outer).
bool make_map(CUtensorMap* m, const double* base, int64_t inner, int64_t outer, int64_t ld,
              int box_inner, int box_outer) {
  auto fn = tma_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
            es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// claim counters: a ring, so that products in flight on different streams do not share one
constexpr int NCTR = 64;
std::atomic<unsigned> g_tma_launch_no{0};
constexpr int kMaxDev = 64;
int cur_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev >= 0 && dev < kMaxDev ? dev : 0;
}
unsigned long long* claim_counters() {  // one ring per device
  static unsigned long long* d[kMaxDev] = {};
  const int dev = cur_device();
  if (!d[dev]) {
    if (cudaMalloc(reinterpret_cast<void**>(&d[dev]), NCTR * 2 * sizeof(unsigned long long)) !=
        cudaSuccess) {
      cudaGetLastError();
      return nullptr;
    }
    cudaMemset(d[dev], 0, NCTR * 2 * sizeof(unsigned long long));
  }
  return d[dev];
}

template <int TA, int TB, class C>
constexpr size_t tma_smem_bytes() {  // (SYMM launches pass TA = 1: the larger A stage)
  return (size_t)(TATile<TA, C>::size + TBTile<TB, C>::size) * tma_stages<TA, TB, C>() *
             sizeof(double) +
         (2 * tma_stages<TA, TB, C>() + 4) * sizeof(uint64_t) + 2 * sizeof(long long);
}

template <int TA, int TB, int LOWER, class C, int SYMM = 0>
cudaError_t launch_tma(const GemmArgs& p, cudaStream_t st, const GemmOwn& own = GemmOwn{}) {
  static_assert(!SYMM || C::BM == 128 || C::BM == 64, "symmetric band: BM - 1 diagonals");
  if (own.g > 1 && ((LOWER && C::BN != 64) || (SYMM && C::BM != 64) || (!LOWER && !SYMM)))
    return cudaErrorInvalidValue;
  unsigned long long* ctrs = claim_counters();
  if (!ctrs) return cudaErrorMemoryAllocation;
  CUtensorMap mapA, mapB;
  const int sh_a = (reinterpret_cast<uintptr_t>(p.A) & 15) ? 1 : 0;
  const int sh_b = (reinterpret_cast<uintptr_t>(p.B) & 15) ? 1 : 0;
  if (SYMM && sh_a) return cudaErrorNotSupported;
  const bool okA = (TA && !SYMM) ? make_map(&mapA, p.A - sh_a, p.k + sh_a, p.m, p.lda, TPK, C::BM)
                      : make_map(&mapA, p.A - sh_a, p.m + sh_a, p.k, p.lda, C::SPM, TBK);
  const bool okB = TB ? make_map(&mapB, p.B - sh_b, p.n + sh_b, p.k, p.ldb, C::SPN, TBK)
                      : make_map(&mapB, p.B - sh_b, p.k + sh_b, p.n, p.ldb, TPK, C::BN);
  if (!okA || !okB) return cudaErrorNotSupported;
  CUtensorMap mapC = mapA;  // placeholder when C is not prefetched
  if (SYMM && !make_map(&mapC, p.A, p.k, p.m, p.lda, TPK, C::BM)) return cudaErrorNotSupported;
  const bool okC = !SYMM && p.beta != 0.0 && (reinterpret_cast<uintptr_t>(p.C) & 15) == 0 &&
                   (p.ldc & 1) == 0 && p.ldc * 8 < (1ll << 40) &&
                   make_map(&mapC, p.C, p.m, p.n, p.ldc, C::BM, C::BN);
  auto kern = gemm_tma_kernel<TA, TB, LOWER, C, SYMM>;
  constexpr size_t sm = tma_smem_bytes<(SYMM ? 1 : TA), TB, C>();
  static bool configured[kMaxDev] = {};  // the attribute is per device
  if (!configured[cur_device()]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    configured[cur_device()] = true;
  }
  TmaGemmParams q;
  q.p = p;
  q.tiles_m = (p.m + C::BM - 1) / C::BM;
  q.tiles_n = (p.n + C::BN - 1) / C::BN;
  const int64_t tiles = q.tiles_m * q.tiles_n;
  const int slots = num_sms() * C::MINB;
  // few output tiles and a long k: split k (each slice >= 512 deep) for wave quantisation
  int64_t splits = 1;
  if (!LOWER && tiles < 6 * slots && p.k >= 2 * 512) {
    auto eff = [&](int64_t s) {
      const int64_t ctas = tiles * s;
      return (double)ctas / (double)(((ctas + slots - 1) / slots) * slots);
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
  int64_t kc = p.k;
  double* ws = nullptr;
  if (splits > 1) {
    kc = (p.k + splits - 1) / splits;
    kc = (kc + TBK - 1) / TBK * TBK;
    splits = (p.k + kc - 1) / kc;
  }
  if (splits > 1) {
    cudaError_t e = cudaMallocAsync(reinterpret_cast<void**>(&ws),
                                    (size_t)splits * p.m * p.n * sizeof(double), st);
    if (e != cudaSuccess) return e;
  } else {
    splits = 1;
    kc = (p.k + TBK - 1) / TBK * TBK;
  }
  q.ws = ws;
  q.kc = kc;
  q.splits = (int)splits;
  q.prefetch_c = (okC && !ws) ? 1 : 0;
  q.sh_a = sh_a;
  q.sh_b = sh_b;
  q.own_g = own.g;
  q.own_r = own.r;
  q.own_org = own.org;
  q.ctr = ctrs + 2 * (g_tma_launch_no.fetch_add(1, std::memory_order_relaxed) % NCTR);
  const int grid = (int)imin64((int64_t)slots, tiles * splits);
  kern<<<grid, C::THREADS, sm, st>>>(mapA, mapB, mapC, q);
  count_launch();
  if (ws) {
    splitk_reduce(st, p.m, p.n, (int)splits, ws, p.alpha, p.beta, p.C, p.ldc, LOWER, p.diag_off);
    cudaFreeAsync(ws, st);
  }
  return cudaGetLastError();
}

// Register budgets (64K per SM, allocated per 4 warps): a producer warpgroup gives its
// registers to the consumers with setmaxnreg, so 32 x 64 warp tiles (128 accumulator
// registers) run without spills.
// 128 x 64 tiles, 4 consumer warps of 32 x 64, two CTAs per SM (launched at 128, then 216/40)
using TC2 = TCfg<128, 64, 4, 8, 2, 4, 4, 216, 40>;
// 128 x 128 tiles, 8 consumer warps of 32 x 64, one CTA per SM (launched at 168, then 232/40)
using TC3 = TCfg<128, 128, 4, 8, 1, 5, 4, 232, 40>;
// 64 x 64 tiles, 4 consumer warps of 32 x 32 and one producer warp, two CTAs per SM: the
// row tile of a symmetric band product whose columns are owned in 64-column blocks
using TC6 = TCfg<64, 64, 4, 4, 2, 5, 1, 0, 0>;
// 128 x 96 tiles, 12 consumer warps of 32 x 32 and one producer warp, one CTA per SM (128)
using TC4 = TCfg<128, 96, 4, 4, 1, 6, 1, 0, 0>;

template <int TA, int TB, int LOWER>
cudaError_t launch_cfg(const GemmArgs& p, cudaStream_t st, int cfg) {
  // measured (tools/gemm_probe.py, profiles/r02/gemm_tma): TC3 >= TC2 > TC4 on every shape
  switch (cfg) {
    case 2: return launch_tma<TA, TB, LOWER, TC2>(p, st);
    case 5: return launch_tma<TA, TB, LOWER, TC4>(p, st);
    default: return launch_tma<TA, TB, LOWER, TC3>(p, st);
  }
}

}  // namespace

// Returns cudaErrorNotSupported when the product does not qualify (the caller falls back
// to the cp.async kernels): the leading dimensions must be even (TMA strides),
// extents must fit TMA's 32-bit coordinates, and the product must be large enough to fill
// the persistent grid.
cudaError_t gemm_tma(cudaStream_t st, bool ta, bool tb, const GemmArgs& p, bool lower) {
  if (g_gemm_tma == 0) return cudaErrorNotSupported;
  if ((p.lda & 1) || (p.ldb & 1)) return cudaErrorNotSupported;  // TMA strides: 16-byte units
  if (p.m > INT32_MAX || p.n > INT32_MAX || p.k > INT32_MAX) return cudaErrorNotSupported;
  if (p.lda * 8 >= (1ll << 40) || p.ldb * 8 >= (1ll << 40)) return cudaErrorNotSupported;
  if (g_gemm_tma == 1) {
    // auto: at least ~two waves of 128 x 64 tiles over a k of 64 or more
    const int64_t tiles = ((p.m + 127) / 128) * ((p.n + 63) / 64);
    if (p.k < 64 || tiles * imin64(p.k, 1024) < (int64_t)num_sms() * 2 * 1024)
      return cudaErrorNotSupported;
  }
  static const bool log_calls = getenv("EM_GEMM_TMA_LOG") != nullptr;
  if (log_calls)
    fprintf(stderr, "gemm_tma ta=%d tb=%d lower=%d m=%lld n=%lld k=%lld lda=%lld ldb=%lld ldc=%lld "
            "doff=%lld alpha=%g beta=%g A=%p B=%p C=%p\n", (int)ta, (int)tb, (int)lower,
            (long long)p.m, (long long)p.n, (long long)p.k, (long long)p.lda, (long long)p.ldb,
            (long long)p.ldc, (long long)p.diag_off, p.alpha, p.beta, (const void*)p.A,
            (const void*)p.B, (const void*)p.C);
  int cfg = (int)g_gemm_tma;
  // auto: 128-column tiles unless they would pad n by more than 5% (n = 64 panels of the
  // band reduction: half of every 128 x 128 tile would be zero work)
  if (cfg == 1) {
    const int64_t n128 = (p.n + 127) / 128 * 128, n64 = (p.n + 63) / 64 * 64;
    cfg = (n128 - n64) * 20 > n128 ? 2 : 4;
  }
  const int code = (ta ? 4 : 0) | (tb ? 2 : 0) | (lower ? 1 : 0);
  switch (code) {
    case 0: return launch_cfg<0, 0, 0>(p, st, cfg);
    case 1: return launch_cfg<0, 0, 1>(p, st, cfg);
    case 2: return launch_cfg<0, 1, 0>(p, st, cfg);
    case 3: return launch_cfg<0, 1, 1>(p, st, cfg);
    case 4: return launch_cfg<1, 0, 0>(p, st, cfg);
    case 5: return launch_cfg<1, 0, 1>(p, st, cfg);
    case 6: return launch_cfg<1, 1, 0>(p, st, cfg);
    default: return launch_cfg<1, 1, 1>(p, st, cfg);
  }
}

// 2-D tensor map over a column-major operand (shared with td1.cu): `map` points at a
// CUtensorMap; inner = contiguous extent, outer = columns of stride ld doubles.
bool tma_map_2d(void* map, const double* base, int64_t inner, int64_t outer, int64_t ld,
                int box_inner, int box_outer) {
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (ld & 1) || inner <= 0 || outer <= 0 ||
      inner > INT32_MAX || outer > INT32_MAX || ld * 8 >= (1ll << 40))
    return false;
  return make_map(static_cast<CUtensorMap*>(map), base, inner, outer, ld, box_inner, box_outer);
}

// C (m x n) = A B for a symmetric m x m A of which only the lower triangle and the 127
// diagonals above it are read (B is m x n, column-major; the product X = A22 (V T) of the
// band reduction, n = 64). cudaErrorNotSupported when TMA cannot address the operands.
cudaError_t gemm_symm_lower_tma(cudaStream_t st, int64_t m, int64_t n, const double* A,
                                int64_t lda, const double* B, int64_t ldb, double* C,
                                int64_t ldc, const GemmOwn& own) {
  if (g_gemm_tma == 0 || m <= 0 || n <= 0) return cudaErrorNotSupported;
  if ((lda & 1) || (ldb & 1) || (reinterpret_cast<uintptr_t>(A) & 15)) return cudaErrorNotSupported;
  if (m > INT32_MAX || n > INT32_MAX || lda * 8 >= (1ll << 40) || ldb * 8 >= (1ll << 40))
    return cudaErrorNotSupported;
  GemmArgs p{m, n, m, A, lda, B, ldb, C, ldc, 1.0, 0.0, 0};
  static_assert(TC2::BM == 128 && TC3::BM == 128, "the band above the diagonal is BM - 1 wide");
  if (own.g > 1) return launch_tma<0, 0, 0, TC6, 1>(p, st, own);  // (64-row tiles)
  if (n <= 64) return launch_tma<0, 0, 0, TC2, 1>(p, st);
  return launch_tma<0, 0, 0, TC3, 1>(p, st);
}

// The LOWER product of gemm() restricted to the column tiles this rank owns (64-column
// blocks, see TmaGemmParams): the trailing update of a distributed band reduction.
cudaError_t gemm_lower_owned_tma(cudaStream_t st, bool ta, bool tb, const GemmArgs& p,
                                 const GemmOwn& own) {
  if ((p.lda & 1) || (p.ldb & 1)) return cudaErrorNotSupported;
  if (p.m > INT32_MAX || p.n > INT32_MAX || p.k > INT32_MAX) return cudaErrorNotSupported;
  if (!ta && tb) return launch_tma<0, 1, 1, TC2>(p, st, own);
  if (!ta && !tb) return launch_tma<0, 0, 1, TC2>(p, st, own);
  if (ta && !tb) return launch_tma<1, 0, 1, TC2>(p, st, own);
  return launch_tma<1, 1, 1, TC2>(p, st, own);
}

}  // namespace em
