// Cholesky-factor theta-method (TD1) on B200 — the comparator of the paper.
//
// Reference: Td1Stepper (pkg/src/eddymodes/transient.py:77-113) factors
// Z = L_i + dt*theta*R_i once (cholesky, "stepping matrix") and every step runs
// td1_step_kernel (_kernels.py:198-210): b = -dt R I + drive_rhs (modal.py:121-131),
// forward then backward substitution with the factor (tri_solve_vec,
// _kernels.py:39-53), I += x.
//
// GPU form per step: one kernel forms b = E u^k - dt*R*I (CSR SpMV of the stencil R, or
// the lower-triangle symv) and resets the solution vectors to a sentinel, then two
// PERSISTENT triangular-solve kernels. Block rows of 64 are claimed in order from an
// atomic counter; a CTA streams the off-diagonal tiles of its block row (the next tile is
// in flight while the current one waits), reduces with warp shuffles / shared memory and
// applies the pre-inverted 64x64 diagonal block. The products with the two neighbouring
// blocks' solutions are folded into precomputed 64x64 matrices (E_r = D_r C_{r,r-1},
// E2_r = D_r C_{r,r-2}; F_r, F2_r for the backward solve), so a block's own reduction
// finishes two chain steps ahead and its chain step is one product. There are no ready
// flags: a solution entry is published by storing it over the sentinel (a NaN payload no
// arithmetic produces; 64-bit stores are single-copy atomic), and a consumer polls the
// entries it needs directly, so each link of the dependency chain is one L2 round trip
// instead of flag acquire + data load + fenced release. Each solve reads the factor once.
#include "common.cuh"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"
#include "plans.h"
#include "symv_tma.cuh"

#include <vector>

struct em_td1_plan {
  em_ctx* ctx = nullptr;
  int64_t n = 0;
  int n_p = 0, n_s = 0, n_u = 0;
  double dt = 0, theta = 0;
  em::DBuf C, R, Dinv, DinvT, Ef, Fb, Ef2, Fb2, E, work, b, y, x;
  double* Cp = nullptr;  // the factor: C.p, or the caller's L storage (in-place plan)
  int64_t ldc = 0;
  em::Csr Rs;          // R as CSR when it is sparse (the stencil): R I is an SpMV
  bool r_sparse = false;
  em::DArr<unsigned int>* counters = nullptr;
  alignas(64) unsigned char cmap[128] = {};  // CUtensorMap over the factor (TMA-staged solves)
  bool tma_ok = false;
  int n_obs = 0;
  em::DBuf Cobs, D;
  ~em_td1_plan() { delete counters; }
};

namespace em {

constexpr int TS = 64;  // triangular-solve block
int64_t g_td1_staged = 1;  // em_config debug key 93: 0 = register-tile solves, 1 = TMA-staged

__global__ void td1_z_kernel(int64_t n, const double* __restrict__ L, int64_t ldl,
                             const double* __restrict__ R, int64_t ldr, double dt_theta,
                             double* __restrict__ Z, double* __restrict__ Rc) {
  for (int64_t c = blockIdx.y; c < n; c += gridDim.y)
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n;
         r += (int64_t)gridDim.x * blockDim.x) {
      // symmetric inputs: use the lower triangle (SymMatrix semantics, linalg.py:40-41)
      const int64_t rr = r >= c ? r : c, cc = r >= c ? c : r;
      const double l = L[rr + cc * ldl], rv = R[rr + cc * ldr];
      Z[r + c * n] = l + dt_theta * rv;
      Rc[r + c * n] = rv;
    }
}

// DinvT_b = Dinv_b^T for every TS x TS diagonal inverse (backward solve reads it coalesced)
__global__ void transpose_blocks_kernel(const double* __restrict__ Din, double* __restrict__ Dout) {
  __shared__ double t[TS][TS + 1];
  const double* src = Din + (int64_t)blockIdx.x * TS * TS;
  double* dst = Dout + (int64_t)blockIdx.x * TS * TS;
  for (int e = threadIdx.x; e < TS * TS; e += blockDim.x) t[e % TS][e / TS] = src[e];
  __syncthreads();
  for (int e = threadIdx.x; e < TS * TS; e += blockDim.x) dst[e] = t[e / TS][e % TS];
}

// E = [-dt R_D | -(L_D + dt theta R_D) | -M0]  (drive_rhs, modal.py:121-131)
__global__ void td1_e_kernel(int64_t n, int n_p, int n_s, double dt, double theta,
                             const double* __restrict__ r_d, const double* __restrict__ l_d,
                             const double* __restrict__ m0, double* __restrict__ E) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (int p = 0; p < n_p; ++p) {
    const double rd = r_d[i + p * n], ld = l_d[i + p * n];
    E[i + p * n] = -dt * rd;
    E[i + (int64_t)(n_p + p) * n] = -(ld + dt * theta * rd);
  }
  for (int s = 0; s < n_s; ++s) E[i + (int64_t)(2 * n_p + s) * n] = -m0[i + s * n];
}

// Published solution entries replace this NaN payload (arithmetic only ever produces the
// canonical NaN 0x7ff8000000000000).
constexpr unsigned long long kSentinel = 0x7ff4dead00c0ffeeull;

EM_DEVINL double ld_poll(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];\n" : "=d"(v) : "l"(p) : "memory");
  return v;
}
EM_DEVINL void st_pub(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}
EM_DEVINL bool is_sentinel(double v) {
  return (unsigned long long)__double_as_longlong(v) == kSentinel;
}
// the 16 entries p[0..15] once all are published
EM_DEVINL void poll16(const double* p, double (&v)[16]) {
#pragma unroll
  for (int cc = 0; cc < 16; ++cc) v[cc] = ld_poll(p + cc);
  while (true) {
    bool ready = true;
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) ready &= !is_sentinel(v[cc]);
    if (ready) break;
#pragma unroll
    for (int cc = 0; cc < 16; ++cc)
      if (is_sentinel(v[cc])) v[cc] = ld_poll(p + cc);
  }
}

// ---- TMA-staged tile stream (STG = 1) -----------------------------------------------------
// The factor tiles of a block row do not depend on the solution, only their USE does: a
// producer warp streams the row's 64 x 64 tiles with cp.async.bulk.tensor into a ring of
// TD1_NST shared-memory stages (192 KB in flight per SM, against two register tiles = 64 KB
// in the register form, whose 214 registers allow one CTA per SM), the 8 consumer warps
// wait on a stage, take their solution entry and accumulate from shared memory. The
// producer also claims the block rows (in order) and hands them to the consumers through a
// two-slot queue; consumer-wide barriers are the named barrier 1 (256 threads).
constexpr int TD1_NST = 6;
constexpr int TD1_TILE = TS * TS;  // doubles
constexpr size_t TD1_SMEM = (size_t)TD1_NST * TD1_TILE * sizeof(double) + 128;

struct Td1Ring {
  double* tiles;
  uint64_t* full;      // [TD1_NST]
  uint64_t* empty;     // [TD1_NST]
  uint64_t* tq_full;   // [2]
  uint64_t* tq_empty;  // [2]
  long long* tq_val;   // [2]
};

template <int STG>
EM_DEVINL void csync() {
  if constexpr (STG)
    asm volatile("bar.sync 1, 256;\n" ::: "memory");
  else
    __syncthreads();
}

EM_DEVINL Td1Ring td1_ring_init(double* dyn, uint64_t* bars) {
  Td1Ring R{dyn, bars, bars + TD1_NST, bars + 2 * TD1_NST, bars + 2 * TD1_NST + 2,
            reinterpret_cast<long long*>(bars + 2 * TD1_NST + 4)};
  if (threadIdx.x == 0) {
    for (int s = 0; s < TD1_NST; ++s) {
      mbar_init(&R.full[s], 1);
      mbar_init(&R.empty[s], 8);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&R.tq_full[s], 1);
      mbar_init(&R.tq_empty[s], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  return R;
}

// Producer (one lane): claims block rows from `counter` (forward: ascending, backward:
// descending) and streams tiles (j, r) of each row — forward j = 0 .. r-3, backward
// j = nblk-1 .. r+3 — as boxes {64 rows at 64 j, 64 columns at 64 r} of the factor.
template <int BWD>
EM_DEVINL void td1_producer(const CUtensorMap* map, const Td1Ring& R, int64_t nblk,
                            unsigned int* counter) {
  const uint64_t pol = pol_evict_first();
  unsigned it = 0, tq = 0;
  for (;;) {
    const int64_t c = (int64_t)atomicAdd(counter, 1u);
    const int64_t r = BWD ? nblk - 1 - c : c;
    const bool done = BWD ? r < 0 : r >= nblk;
    mbar_wait(&R.tq_empty[tq & 1], ((tq >> 1) & 1) ^ 1);
    R.tq_val[tq & 1] = done ? -1ll : (long long)r;
    mbar_arrive(&R.tq_full[tq & 1]);
    ++tq;
    if (done) return;
    const int64_t j0 = BWD ? nblk - 1 : 0, cnt = BWD ? nblk - 3 - r : r - 2;
    for (int64_t q = 0; q < cnt; ++q, ++it) {
      const int64_t j = BWD ? j0 - q : j0 + q;
      const int s = it % TD1_NST;
      mbar_wait(&R.empty[s], ((it / TD1_NST) & 1) ^ 1);
      mbar_expect_tx(&R.full[s], TD1_TILE * sizeof(double));
      tma_load_2d(R.tiles + s * TD1_TILE, map, (int)(j * TS), (int)(r * TS), &R.full[s], pol);
    }
  }
}

// Consumers: next block row from the queue (-1: none left).
EM_DEVINL int64_t td1_next_row(const Td1Ring& R, unsigned& tq, int lane) {
  mbar_wait(&R.tq_full[tq & 1], (tq >> 1) & 1);
  const long long r = R.tq_val[tq & 1];
  __syncwarp();
  if (lane == 0) mbar_arrive(&R.tq_empty[tq & 1]);
  ++tq;
  return (int64_t)r;
}

// Consumers: acc[cc] += tile[ty*16 + cc][tx] * v for the cnt tiles of a row; the solution
// entry of tile q is sol[(BWD ? j0 - q : j0 + q) * TS + tx], polled past the sentinel.
// A stage is released one tile late (after the next stage's wait: every FMA that read it
// has issued, so its shared-memory loads are done — see gemm_tma.cu), the row's last stage
// behind a data dependency on the accumulators.
template <int BWD>
EM_DEVINL void td1_stream(const Td1Ring& R, unsigned& it, int64_t j0, int64_t cnt,
                          const double* sol, int tx, int ty, int lane, double (&acc)[16]) {
  if (cnt <= 0) return;
  double vnext = ld_poll(sol + j0 * TS + tx);
  for (int64_t q = 0; q < cnt; ++q) {
    const int64_t j = BWD ? j0 - q : j0 + q;
    const int s = it % TD1_NST;
    mbar_wait(&R.full[s], (it / TD1_NST) & 1);
    ++it;
    double v = vnext;
    if (q + 1 < cnt) vnext = ld_poll(sol + (BWD ? j - 1 : j + 1) * TS + tx);
    const double* t = R.tiles + s * TD1_TILE + (ty * 16) * TS + tx;
    double a[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) a[cc] = t[cc * TS];
    while (is_sentinel(v)) v = ld_poll(sol + j * TS + tx);
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) acc[cc] = fma(a[cc], v, acc[cc]);
    __syncwarp();
    if (q > 0 && lane == 0) mbar_arrive(&R.empty[(it + TD1_NST - 2) % TD1_NST]);
  }
  unsigned never = 0u;
#pragma unroll
  for (int cc = 0; cc < 16; ++cc) never |= never_set(acc[cc]);
  __syncwarp();
  if (lane == 0)
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(
                     smem_u32(&R.empty[(it + TD1_NST - 1) % TD1_NST]) + never)
                 : "memory");
}

// Forward solve C y = b, C lower (col-major, ld ldc; its upper triangle holds the
// mirror C^T, so a block row of C is read as a block column). Block rows claimed in order.
// y_r = D_r (b_r - sum_{j < r-2} C_rj y_j) - E2_r y_{r-2} - E_r y_{r-1} with
// E_r = D_r C_{r,r-1}, E2_r = D_r C_{r,r-2} precomputed: the tile stream and the D_r
// product wait only on blocks up to r-3, so they finish two steps ahead of the chain,
// whose step per block is: see y_{r-1}, one product, publish y_r. y must hold the
// sentinel on entry (td1_pre_kernel).
template <int STG>
__global__ void __launch_bounds__(STG ? 288 : 256) trsv_fwd_kernel(
    const __grid_constant__ CUtensorMap cmap, int64_t n, const double* __restrict__ C,
    int64_t ldc, const double* __restrict__ Dinv, const double* __restrict__ Ef,
    const double* __restrict__ Ef2, const double* __restrict__ b, double* __restrict__ y,
    unsigned int* counter) {
  extern __shared__ __align__(128) double dyn[];
  __shared__ uint64_t bars[2 * TD1_NST + 6];
  __shared__ int64_t rblk;
  __shared__ double red[4][TS];
  __shared__ double red8[8][16];
  __shared__ double part[TS];
  const int tid = threadIdx.x, tx = tid & 63, ty = (tid >> 6) & 3, lane = tid & 31, warp = tid >> 5;
  const int64_t nblk = (n + TS - 1) / TS;
  Td1Ring R{};
  unsigned it = 0, tq = 0;
  if constexpr (STG) {
    R = td1_ring_init(dyn, bars);
    if (warp == 8) {
      if (lane == 0) td1_producer<0>(&cmap, R, nblk, counter);
      return;
    }
  }
  while (true) {
    int64_t r;
    if constexpr (STG) {
      csync<STG>();  // the previous row's readers of the reduction buffers are done
      r = td1_next_row(R, tq, lane);
      if (r < 0) break;
    } else {
      __syncthreads();
      if (tid == 0) rblk = atomicAdd(counter, 1u);
      __syncthreads();
      r = rblk;
      if (r >= nblk) break;
    }
    const int64_t r0 = r * TS;
    const double bb = (tid < TS && r0 + tid < n) ? b[r0 + tid] : 0.0;
    // tiles j <= r - 3, read from the mirrored upper triangle (Cm[j0 + b, r0 + a] =
    // C[r0 + a, j0 + b]): thread (tx, ty) holds C_rj[ty*16 + cc][tx] for the 16 rows
    // cc, coalesced along tx, and needs the single entry y_j[tx]; tile j+1 is loaded
    // before waiting for block j
    double acc[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) acc[cc] = 0.0;
    if constexpr (STG) {
      td1_stream<0>(R, it, 0, r - 2, y, tx, ty, lane, acc);
    } else {
      const int64_t c0 = r0 + ty * 16;
      double a[16];
      if (r > 2) {
  #pragma unroll
        for (int cc = 0; cc < 16; ++cc) a[cc] = (c0 + cc < n) ? C[tx + (c0 + cc) * ldc] : 0.0;
      }
      // the solution entry of the NEXT tile is requested together with that tile's data
      // (blocks far behind the chain are published long ago: their poll is a plain L2 load
      // whose latency used to be exposed once per tile — 64% of the stall samples at
      // N = 40,000, profiles/r02/ncu_trsv_fwd_40k.json); a sentinel is re-polled when due
      double ynext = r > 2 ? ld_poll(y + tx) : 0.0;
      for (int64_t j = 0; j + 2 < r; ++j) {
        double an[16];
        double yv = ynext;
        if (j + 3 < r) {
          const int64_t rn = (j + 1) * TS + tx;
  #pragma unroll
          for (int cc = 0; cc < 16; ++cc) an[cc] = (c0 + cc < n) ? C[rn + (c0 + cc) * ldc] : 0.0;
          ynext = ld_poll(y + rn);
        }
        while (is_sentinel(yv)) yv = ld_poll(y + j * TS + tx);
  #pragma unroll
        for (int cc = 0; cc < 16; ++cc) acc[cc] = fma(a[cc], yv, acc[cc]);
  #pragma unroll
        for (int cc = 0; cc < 16; ++cc) a[cc] = an[cc];
      }
    }
    // reduce acc[cc] over the 64 columns (tx): warp shuffle, then the two warps per ty
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) acc[cc] = warp_sum(acc[cc]);
    if (lane == 0) {
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) red8[warp][cc] = acc[cc];
    }
    csync<STG>();
    if (tid < TS) {
      const int gq = tid >> 4, cc = tid & 15;  // row tid = gq*16 + cc (warps 2gq, 2gq+1)
      part[tid] = bb - (red8[2 * gq][cc] + red8[2 * gq + 1][cc]);
    }
    csync<STG>();
    // p_r = D_r part (off the chain)
    const double* D = Dinv + r * TS * TS;
    double s = 0.0;
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) s = fma(D[tx + (ty * 16 + cc) * TS], part[ty * 16 + cc], s);
    red[ty][tx] = s;
    csync<STG>();
    double pr = 0.0;
    if (tid < TS) pr = red[0][tid] + red[1][tid] + red[2][tid] + red[3][tid];
    // the chain operands (loaded while y_{r-2}, y_{r-1} are still on their way)
    const double* Er = Ef + r * TS * TS;
    const double* Er2 = Ef2 + r * TS * TS;
    double ev[16], e2v[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      ev[cc] = r > 0 ? Er[tx + (ty * 16 + cc) * TS] : 0.0;
      e2v[cc] = r > 1 ? Er2[tx + (ty * 16 + cc) * TS] : 0.0;
    }
    // E2_r y_{r-2} (one step ahead of the chain), then the chain: E_r y_{r-1}
    double se = 0.0;
    if (r > 1) {
      double yv[16];
      poll16(y + (r - 2) * TS + ty * 16, yv);
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) se = fma(e2v[cc], yv[cc], se);
    }
    if (r > 0) {
      double yv[16];
      poll16(y + (r - 1) * TS + ty * 16, yv);
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) se = fma(ev[cc], yv[cc], se);
    }
    csync<STG>();  // red: the p_r readers are done
    red[ty][tx] = se;
    csync<STG>();
    if (tid < TS) {
      // rows past n (last block) publish 0 so the pollers of a full 16-entry group finish
      const double v = r0 + tid < n
                           ? pr - ((red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]))
                           : 0.0;
      st_pub(y + r0 + tid, v);
    }
  }
}

// Backward solve C^T x = y; then I += x (and capture). Block rows claimed from the bottom.
// x_r = DT_r (y_r - sum_{j > r+2} C_jr^T x_j) - F2_r x_{r+2} - F_r x_{r+1},
// F_r = DT_r C_{r+1,r}^T, F2_r = DT_r C_{r+2,r}^T precomputed (DT_r = D_r^T): one 64 x 64
// product on the dependency chain. x must hold the sentinel on entry.
template <int STG>
__global__ void __launch_bounds__(STG ? 288 : 256) trsv_bwd_kernel(
    const __grid_constant__ CUtensorMap cmap, int64_t n, const double* __restrict__ C,
    int64_t ldc, const double* __restrict__ Dinv, const double* __restrict__ Fb,
    const double* __restrict__ Fb2, const double* __restrict__ y, double* __restrict__ x,
    double* __restrict__ I, double* __restrict__ Icap, unsigned int* counter) {
  extern __shared__ __align__(128) double dyn[];
  __shared__ uint64_t bars[2 * TD1_NST + 6];
  __shared__ int64_t rblk;
  __shared__ double red[8][TS];
  __shared__ double part[TS];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tx = tid & 63, ty = (tid >> 6) & 3;
  const int64_t nblk = (n + TS - 1) / TS;
  Td1Ring R{};
  unsigned it = 0, tq = 0;
  if constexpr (STG) {
    R = td1_ring_init(dyn, bars);
    if (warp == 8) {
      if (lane == 0) td1_producer<1>(&cmap, R, nblk, counter);
      return;
    }
  }
  while (true) {
    int64_t r;
    if constexpr (STG) {
      csync<STG>();  // the previous row's readers of the reduction buffers are done
      r = td1_next_row(R, tq, lane);
      if (r < 0) break;
    } else {
      __syncthreads();
      if (tid == 0) rblk = nblk - 1 - (int64_t)atomicAdd(counter, 1u);
      __syncthreads();
      r = rblk;
      if (r < 0) break;
    }
    const int64_t r0 = r * TS;
    double acc[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) acc[cc] = 0.0;
    // tiles (j, r), j = nblk-1 .. r+3; tile j-1 is prefetched before waiting for block j
    const int64_t c0 = r0 + ty * 16;
    const double yr = (tid < TS && r0 + tid < n) ? y[r0 + tid] : 0.0;
    if constexpr (STG) {
      td1_stream<1>(R, it, nblk - 1, nblk - 3 - r, x, tx, ty, lane, acc);
    } else {
      double a[16];
      if (nblk - 3 > r) {
        const int64_t rowj = (nblk - 1) * TS + tx;
  #pragma unroll
        for (int cc = 0; cc < 16; ++cc) a[cc] = (rowj < n) ? C[rowj + (c0 + cc) * ldc] : 0.0;
      }
      // (the next tile's solution entry travels with its data, as in the forward solve)
      double xnext = nblk - 3 > r ? ld_poll(x + (nblk - 1) * TS + tx) : 0.0;
      for (int64_t j = nblk - 1; j > r + 2; --j) {
        double an[16];
        double xv = xnext;  // rows past n are published as 0
        if (j - 1 > r + 2) {
          const int64_t rown = (j - 1) * TS + tx;
  #pragma unroll
          for (int cc = 0; cc < 16; ++cc) an[cc] = (rown < n) ? C[rown + (c0 + cc) * ldc] : 0.0;
          xnext = ld_poll(x + rown);
        }
        const int64_t rowj = j * TS + tx;
        while (is_sentinel(xv)) xv = ld_poll(x + rowj);
  #pragma unroll
        for (int cc = 0; cc < 16; ++cc) acc[cc] = fma(a[cc], xv, acc[cc]);
  #pragma unroll
        for (int cc = 0; cc < 16; ++cc) a[cc] = an[cc];
      }
    }
    const bool has_next = r + 1 < nblk, has_next2 = r + 2 < nblk;
    // reduce acc[cc] over the 64 rows (tx): warp shuffle, then the two warps per ty
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) acc[cc] = warp_sum(acc[cc]);
    if (lane == 0) {
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) red[warp][cc] = acc[cc];
    }
    csync<STG>();
    if (tid < TS) {
      const int g = tid >> 4, cc = tid & 15;  // column tid = g*16 + cc belongs to ty = g (warps 2g, 2g+1)
      const double sumc = red[2 * g][cc] + red[2 * g + 1][cc];
      part[tid] = yr - sumc;
    }
    csync<STG>();
    // p_r = DT_r part with the pre-transposed block (coalesced), off the chain
    const double* D = Dinv + r * TS * TS;
    double s = 0.0;
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) s = fma(D[tx + (ty * 16 + cc) * TS], part[ty * 16 + cc], s);
    red[ty][tx] = s;
    csync<STG>();
    double pr = 0.0;
    if (tid < TS) pr = red[0][tid] + red[1][tid] + red[2][tid] + red[3][tid];
    const double* Fr = Fb + r * TS * TS;
    const double* Fr2 = Fb2 + r * TS * TS;
    double fv[16], f2v[16];
#pragma unroll
    for (int cc = 0; cc < 16; ++cc) {
      fv[cc] = has_next ? Fr[tx + (ty * 16 + cc) * TS] : 0.0;
      f2v[cc] = has_next2 ? Fr2[tx + (ty * 16 + cc) * TS] : 0.0;
    }
    // F2_r x_{r+2}, then the chain: F_r x_{r+1}
    double sf = 0.0;
    if (has_next2) {
      double xv2[16];
      poll16(x + (r + 2) * TS + ty * 16, xv2);
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) sf = fma(f2v[cc], xv2[cc], sf);
    }
    if (has_next) {
      double xv2[16];
      poll16(x + (r + 1) * TS + ty * 16, xv2);
#pragma unroll
      for (int cc = 0; cc < 16; ++cc) sf = fma(fv[cc], xv2[cc], sf);
    }
    csync<STG>();  // red: the p_r readers are done
    red[ty][tx] = sf;
    csync<STG>();
    if (tid < TS) {
      if (r0 + tid < n) {
        const double xv = pr - ((red[0][tid] + red[1][tid]) + (red[2][tid] + red[3][tid]));
        st_pub(x + r0 + tid, xv);
        const double iv = I[r0 + tid] + xv;
        I[r0 + tid] = iv;
        if (Icap) Icap[r0 + tid] = iv;
      } else {
        st_pub(x + r0 + tid, 0.0);
      }
    }
  }
}

// b = E u - dt R I (u = [i_d^k, di_d^k, di0^k] from drive rows k, k+1, or u_dev when drive
// is null); y, x <- sentinel for the step's two solves; the solves' row counters <- 0.
__global__ void td1_pre_kernel(int64_t n, int64_t npad, int n_p, int n_s, int n_u,
                               const double* __restrict__ E, const double* __restrict__ drive,
                               int64_t k, const double* __restrict__ u_dev,
                               const int64_t* __restrict__ rowptr, const int* __restrict__ colidx,
                               const double* __restrict__ val, double dt,
                               const double* __restrict__ I, double* __restrict__ b,
                               double* __restrict__ y, double* __restrict__ x,
                               unsigned int* counters) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i == 0) counters[0] = counters[1] = 0u;
  if (i < npad) {
    y[i] = __longlong_as_double((long long)kSentinel);
    x[i] = __longlong_as_double((long long)kSentinel);
  }
  if (i >= n) return;
  double v = 0.0;
  if (drive) {
    const int n_c = n_p + n_s;
    const double* d0 = drive + k * n_c;
    const double* d1 = d0 + n_c;
    for (int p = 0; p < n_p; ++p) {
      v = fma(E[i + p * n], d0[p], v);
      v = fma(E[i + (int64_t)(n_p + p) * n], d1[p] - d0[p], v);
    }
    for (int s = 0; s < n_s; ++s)
      v = fma(E[i + (int64_t)(2 * n_p + s) * n], d1[n_p + s] - d0[n_p + s], v);
  } else {
    for (int j = 0; j < n_u; ++j) v = fma(E[i + (int64_t)j * n], u_dev[j], v);
  }
  if (rowptr) {  // b -= dt R I, R's nonzeros in increasing column order
    double s = 0.0;
    for (int64_t p = rowptr[i]; p < rowptr[i + 1]; ++p) s += val[p] * I[colidx[p]];
    v = fma(-dt, s, v);
  }
  b[i] = v;
}

// Z += dt theta R on the lower band of Z (R in lower band storage)
__global__ void td1_z_band_kernel(int64_t n, const double* __restrict__ Rb, int64_t ldrb,
                                  int64_t bw, double dt_theta, double* __restrict__ Z,
                                  int64_t ldz) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y)
    for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q <= bw && j + q < n;
         q += (int64_t)gridDim.x * blockDim.x)
      Z[(j + q) + j * ldz] += dt_theta * Rb[q + j * ldrb];
}

// Rb (band storage) given: Z = L + dt theta R is formed in L's own storage when in_place
// (ldl == n; the caller's L is the factor afterwards), R enters only as its CSR.
int64_t td1_plan_init(em_td1_plan* P, const double* L, int64_t ldl, const double* R, int64_t ldr,
                      const double* r_d, const double* l_d, const double* m0, const double* Rb,
                      int64_t ldrb, int64_t bw, bool in_place) {
  cudaStream_t st = P->ctx->stream;
  const int64_t n = P->n;
  if (Rb) {
    if (in_place) {
      if (ldl < n) throw ArgError{"in-place TD1 plan needs ldl >= n"};
      P->Cp = const_cast<double*>(L);
      P->ldc = ldl;
    } else {
      P->C.alloc((size_t)n * n, st);
      P->Cp = P->C.p;
      P->ldc = n;
      copy_matrix(st, false, n, n, L, ldl, P->Cp, n);
    }
    dim3 grid((unsigned)((bw + 256) / 256), (unsigned)imin64(n, 65535));
    td1_z_band_kernel<<<grid, 256, 0, st>>>(n, Rb, ldrb, bw, P->dt * P->theta, P->Cp, P->ldc);
    EM_LAUNCHED();
    // Z symmetric in both triangles, as the dense plan forms it (the lower one defines L)
    mirror_lower(st, n, P->Cp, P->ldc);
    P->r_sparse = true;
    csr_from_band(st, n, Rb, ldrb, bw, P->Rs);
  } else {
    P->C.alloc((size_t)n * n, st);
    P->Cp = P->C.p;
    P->ldc = n;
    P->R.alloc((size_t)n * n, st);
    dim3 grid((unsigned)imin64((n + 255) / 256, 64), (unsigned)imin64(n, 65535));
    td1_z_kernel<<<grid, 256, 0, st>>>(n, L, ldl, R, ldr, P->dt * P->theta, P->Cp, P->R.p);
    EM_LAUNCHED();
  }
  const int64_t ldc = P->ldc;
  const int64_t piv = potrf(st, n, P->Cp, ldc);
  if (piv >= 0) return piv;
  // the forward solve reads block rows of C as block columns of C^T: keep the mirror in
  // the (zeroed) upper triangle
  mirror_lower(st, n, P->Cp, ldc);
  // the stencil R: keep only its CSR (7 nonzeros per row) for the per-step R I
  if (!Rb) {
    P->r_sparse = csr_from_dense(st, n, P->R.p, n, 0.02, P->Rs);
    if (P->r_sparse) P->R.release();
  }
  const int64_t nblk = (n + TS - 1) / TS;
  P->Dinv.alloc((size_t)nblk * TS * TS, st);
  trtri_blocks(st, TS, n, P->Cp, ldc, P->Dinv.p);
  P->DinvT.alloc((size_t)nblk * TS * TS, st);
  transpose_blocks_kernel<<<(unsigned)nblk, 256, 0, st>>>(P->Dinv.p, P->DinvT.p);
  EM_LAUNCHED();
  // the chain products: Ef_r = D_r C_{r,r-1} (forward), Fb_r = D_r^T C_{r+1,r}^T (backward)
  // and E2_r = D_r C_{r,r-2}, F2_r = D_r^T C_{r+2,r}^T (one step further)
  P->Ef.alloc((size_t)nblk * TS * TS, st);
  P->Fb.alloc((size_t)nblk * TS * TS, st);
  P->Ef2.alloc((size_t)nblk * TS * TS, st);
  P->Fb2.alloc((size_t)nblk * TS * TS, st);
  for (DBuf* m : {&P->Ef, &P->Fb, &P->Ef2, &P->Fb2})
    EM_CK(cudaMemsetAsync(m->p, 0, (size_t)nblk * TS * TS * sizeof(double), st));
  if (nblk > 1) {
    std::vector<GemmArgs> pf, pb;
    for (int64_t r = 1; r < nblk; ++r) {
      const int64_t r0 = r * TS, bs = imin64(TS, n - r0);
      pf.push_back(GemmArgs{bs, TS, bs, P->Dinv.p + r * TS * TS, TS, P->Cp + r0 + (r0 - TS) * ldc, ldc,
                            P->Ef.p + r * TS * TS, TS, 1.0, 0.0, 0});
      const int64_t q = r - 1;  // Fb_q with block q + 1 = r below it
      pb.push_back(GemmArgs{TS, bs, TS, P->DinvT.p + q * TS * TS, TS, P->Cp + r0 + q * TS * ldc, ldc,
                            P->Fb.p + q * TS * TS, TS, 1.0, 0.0, 0});
      if (r >= 2) {
        pf.push_back(GemmArgs{bs, TS, bs, P->Dinv.p + r * TS * TS, TS,
                              P->Cp + r0 + (r0 - 2 * TS) * ldc, ldc, P->Ef2.p + r * TS * TS, TS, 1.0,
                              0.0, 0});
        const int64_t q2 = r - 2;  // Fb2_q2 with block q2 + 2 = r below it
        pb.push_back(GemmArgs{TS, bs, TS, P->DinvT.p + q2 * TS * TS, TS,
                              P->Cp + r0 + q2 * TS * ldc, ldc, P->Fb2.p + q2 * TS * TS, TS, 1.0,
                              0.0, 0});
      }
    }
    DArr<GemmArgs> df(pf.size(), st), db(pb.size(), st);
    EM_CK(cudaMemcpyAsync(df.p, pf.data(), pf.size() * sizeof(GemmArgs), cudaMemcpyHostToDevice, st));
    EM_CK(cudaMemcpyAsync(db.p, pb.data(), pb.size() * sizeof(GemmArgs), cudaMemcpyHostToDevice, st));
    EM_CK(gemm_grouped(st, false, false, df.p, (int)pf.size(), 1));
    EM_CK(gemm_grouped(st, false, true, db.p, (int)pb.size(), 1));
    EM_CK(cudaStreamSynchronize(st));  // host argument arrays
  }
  P->E.alloc((size_t)n * imax64(P->n_u, 1), st);
  if (P->n_u > 0) {
    td1_e_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(n, P->n_p, P->n_s, P->dt, P->theta,
                                                             r_d, l_d, m0, P->E.p);
    EM_LAUNCHED();
  }
  P->work.alloc(symv_work_size(n), st);
  P->b.alloc(n, st);
  P->y.alloc((size_t)nblk * TS, st);  // padded to whole blocks: pollers read full groups
  P->x.alloc((size_t)nblk * TS, st);
  P->counters = new DArr<unsigned int>(2, st);
  // tiles of the factor (with its mirror in the upper triangle) as TMA boxes of 64 x 64
  P->tma_ok = tma_map_2d(P->cmap, P->Cp, n, n, P->ldc, TS, TS);
  return -1;
}

void td1_set_observables(em_td1_plan* P, int n_obs, const double* C, int64_t ldc, const double* D,
                         int64_t ldd) {
  cudaStream_t st = P->ctx->stream;
  P->n_obs = n_obs;
  P->Cobs.alloc((size_t)n_obs * P->n, st);
  copy_matrix(st, false, n_obs, P->n, C, ldc, P->Cobs.p, n_obs);
  if (D && P->n_p > 0) {
    P->D.alloc((size_t)n_obs * P->n_p, st);
    copy_matrix(st, false, n_obs, P->n_p, D, ldd, P->D.p, n_obs);
  } else {
    P->D.release();
  }
}

// one step: b = E u - dt R I, forward and backward solve, I += x; Icap column or null.
// drive (row k) or u_dev gives u.
static void td1_solve_step(em_td1_plan* P, double* I, double* Icap_col, const double* drive,
                           int64_t k, const double* u_dev) {
  cudaStream_t st = P->ctx->stream;
  const int64_t n = P->n;
  const int64_t nblk = (n + TS - 1) / TS;
  {
    Stage s(st, ST_TD1_SYMV);
    const bool fused_r = P->r_sparse;
    td1_pre_kernel<<<(unsigned)((nblk * TS + 255) / 256), 256, 0, st>>>(
        n, nblk * TS, P->n_p, P->n_s, P->n_u, P->E.p, P->n_u > 0 ? drive : nullptr, k,
        P->n_u > 0 ? u_dev : nullptr, fused_r ? P->Rs.rowptr.p : nullptr,
        fused_r ? P->Rs.colidx.p : nullptr, fused_r ? P->Rs.val.p : nullptr, P->dt, I, P->b.p,
        P->y.p, P->x.p, P->counters->p);
    EM_LAUNCHED();
    if (!fused_r) symv_lower(st, n, -P->dt, P->R.p, n, I, 1.0, P->b.p, P->work.p);
  }
  const int grid = (int)imin64(nblk, 2 * num_sms());
  const CUtensorMap& cmap = *reinterpret_cast<const CUtensorMap*>(P->cmap);
  const bool staged = P->tma_ok && g_td1_staged != 0;
  if (staged) {
    static bool configured[64] = {};  // the attribute is per device
    const int dev = P->ctx->device >= 0 && P->ctx->device < 64 ? P->ctx->device : 0;
    if (!configured[dev]) {
      EM_CK(cudaFuncSetAttribute(trsv_fwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)TD1_SMEM));
      EM_CK(cudaFuncSetAttribute(trsv_bwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)TD1_SMEM));
      configured[dev] = true;
    }
  }
  const int grid_s = (int)imin64(nblk, (int64_t)num_sms());
  {
    Stage s(st, ST_TD1_FWD);
    if (staged)
      trsv_fwd_kernel<1><<<grid_s, 288, TD1_SMEM, st>>>(cmap, n, P->Cp, P->ldc, P->Dinv.p,
                                                        P->Ef.p, P->Ef2.p, P->b.p, P->y.p,
                                                        P->counters->p);
    else
      trsv_fwd_kernel<0><<<grid, 256, 0, st>>>(cmap, n, P->Cp, P->ldc, P->Dinv.p, P->Ef.p,
                                               P->Ef2.p, P->b.p, P->y.p, P->counters->p);
    EM_LAUNCHED();
  }
  {
    Stage s(st, ST_TD1_BWD);
    if (staged)
      trsv_bwd_kernel<1><<<grid_s, 288, TD1_SMEM, st>>>(cmap, n, P->Cp, P->ldc, P->DinvT.p,
                                                        P->Fb.p, P->Fb2.p, P->y.p, P->x.p, I,
                                                        Icap_col, P->counters->p + 1);
    else
      trsv_bwd_kernel<0><<<grid, 256, 0, st>>>(cmap, n, P->Cp, P->ldc, P->DinvT.p, P->Fb.p,
                                               P->Fb2.p, P->y.p, P->x.p, I, Icap_col,
                                               P->counters->p + 1);
    EM_LAUNCHED();
  }
}

void td1_step(em_td1_plan* P, double* I, const double* u_dev) {
  td1_solve_step(P, I, nullptr, nullptr, 0, u_dev);
}

void td1_run(em_td1_plan* P, int64_t T, const double* drive, double* I, double* Y, int64_t stride,
             double* Icap) {
  cudaStream_t st = P->ctx->stream;
  const int64_t n = P->n;
  if (stride < 1) throw ArgError{"capture stride must be >= 1"};
  const int64_t n_caps = T / stride;
  const bool want_y = Y && P->n_obs > 0 && n_caps > 0;
  // observables are formed in chunks: capture states, then one DMMA GEMM per chunk
  const int64_t chunk = Icap ? n_caps : imin64(n_caps, 512);
  DBuf tmpcap;
  if (!Icap && want_y) tmpcap.alloc((size_t)n * imax64(chunk, 1), st);
  int64_t cap = 0, chunk_start = 0;
  auto flush = [&](int64_t upto) {
    if (!want_y || upto <= chunk_start) return;
    const int64_t cnt = upto - chunk_start;
    const double* src = Icap ? Icap + chunk_start * n : tmpcap.p;
    // Y rows [chunk_start, upto): Y^T (n_obs x cnt, col-major == row-major Y) = Cobs * I
    EM_CK(gemm(st, false, false, P->n_obs, cnt, n, 1.0, P->Cobs.p, P->n_obs, src, n, 0.0,
               Y + chunk_start * P->n_obs, P->n_obs));
    chunk_start = upto;
  };
  for (int64_t k = 0; k < T; ++k) {
    double* col = nullptr;
    const bool is_cap = ((k + 1) % stride) == 0;
    if (is_cap && (Icap || want_y)) {
      col = Icap ? Icap + cap * n : tmpcap.p + (cap - chunk_start) * n;
    }
    td1_solve_step(P, I, col, drive, k, nullptr);
    if (is_cap) {
      ++cap;
      if (!Icap && want_y && cap - chunk_start == chunk) flush(cap);
    }
  }
  flush(cap);
  if (want_y && P->D.n) {
    // Y += D i_d(t_{k+1}) at each capture: small GEMM-free loop on host-less path
    // (drive rows (c+1)*stride): gather rows then GEMM would be overkill; use gemm on a
    // strided view: drive row stride = (n_p+n_s)*stride.
    const int n_c = P->n_p + P->n_s;
    EM_CK(gemm(st, false, false, P->n_obs, n_caps, P->n_p, 1.0, P->D.p, P->n_obs,
               drive + (int64_t)stride * n_c, (int64_t)stride * n_c, 1.0, Y, P->n_obs));
  }
}

}  // namespace em

namespace em {

em_td1_plan* td1_new(em_ctx* ctx, int64_t n, int n_p, int n_s, double dt, double theta) {
  auto* P = new em_td1_plan();
  P->ctx = ctx;
  P->n = n;
  P->n_p = n_p;
  P->n_s = n_s;
  P->n_u = 2 * n_p + n_s;
  P->dt = dt;
  P->theta = theta;
  return P;
}
void td1_delete(em_td1_plan* p) {
  if (!p) return;
  cudaSetDevice(p->ctx->device);
  cudaStreamSynchronize(p->ctx->stream);
  delete p;
}
em_ctx* td1_ctx(em_td1_plan* p) { return p ? p->ctx : nullptr; }
void td1_copy_factor(em_td1_plan* P, double* out, int64_t ldo) {
  copy_matrix(P->ctx->stream, false, P->n, P->n, P->Cp, P->ldc, out, ldo);
  zero_upper(P->ctx->stream, P->n, out, ldo);  // the plan keeps C^T there
  EM_CK(cudaStreamSynchronize(P->ctx->stream));
}

void td1_step_host(em_td1_plan* P, double* I, const double* i_d, const double* di_d,
                   const double* di0) {
  cudaStream_t st = P->ctx->stream;
  std::vector<double> u((size_t)imax64(P->n_u, 1), 0.0);
  for (int p = 0; p < P->n_p; ++p) {
    u[p] = i_d[p];
    u[P->n_p + p] = di_d[p];
  }
  for (int s = 0; s < P->n_s; ++s) u[2 * P->n_p + s] = di0[s];
  DBuf du(u.size(), st);
  EM_CK(cudaMemcpyAsync(du.p, u.data(), u.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  td1_step(P, I, du.p);
  EM_CK(cudaStreamSynchronize(st));
}

}  // namespace em
