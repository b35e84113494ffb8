// Q2 back-transform of the two-stage tridiagonalisation, register-resident form:
// Z <- Q2 Z with Q2 the product of the bulge-chasing reflectors (sytrd2.cu, stage 2).
//
// Reflectors of 64 consecutive sweeps at one position form a block (g, k): V is a
// 128 x 64 parallelogram in window rows r = 1..127 of rows W0 = 64 (g + k) onward
// (V[r][j] = v_j[r - 1 - j]), T its 64 x 64 compact-WY factor, VT = V T. A group's
// blocks are applied in ascending k; groups last to first.
//
// The columns of Z transform independently. One CTA owns a strip of 8 NW columns and
// each consumer warp owns 8 of them for the whole group: it keeps the 128-row window
// of its columns TRANSPOSED in registers, as the accumulator fragments of
// m8n8k4 DMMA (thread (g, t) holds Z[8R + 2t + e][col g], e = 0, 1). With the k index
// of each product permuted to the rows a thread already holds (k-step (R, e) covers rows
// 8R + 2t + e), those fragments are ALSO the A operand:
//   W^T (8 x 64)  = Zwin^T V         A = the Z registers, B = V from shared memory
//   Zwin^T       -= W^T (V T)^T      A = the W^T accumulators (same permutation over j),
//                                    B = -(V T) from shared memory
// so Z and W never touch shared memory and the warps need no barrier between the two
// products (W is warp-private). Shared memory holds only the block's operands, packed
// by q2r_pack_kernel in fragment order (one 16-byte load = the B fragments of two
// consecutive k-steps, conflict-free) and streamed in by a producer warp with bulk
// copies on a two-stage mbarrier ring. The window slides 64 rows
// per block: the bottom half becomes the top half (register roles swap, loop unrolled by
// two), the next 64 rows are prefetched into a warp-private staging buffer with cp.async
// and the finished top half is stored straight from the registers.
//
// Per block and 8 columns: 144 DMMA for W (the parallelogram's zero row tiles skipped)
// + 200 for the update (zero tiles of VT skipped); 2 x 64 x 64 x 2 useful flops per
// column: 1.34x the useful count.
#include <vector>

#include "common.cuh"
#include "ctx.h"
#include "linalg.h"
#include "symv_tma.cuh"

namespace em {

int g_q2r_dbg = 0;  // debug key 94: bit0 VT(k) waits for C(k-1); bit1 uniform strips;
                    // bit2 synchronous Z staging loads; bit3 fences before the empty arrivals;
                    // bit4 seven consumer warps (8 warps per CTA, 255 registers); bit5 eight
                    // consumer warps instead of twelve; bit6 twelve even for few columns

namespace {
constexpr int QB = 64;                  // sweeps per group, reflector length
constexpr int VP = 8 * 9 * 64;          // packed V: 8 column tiles J x 9 row tiles (R = J..J+8)
constexpr int VTP = 100 * 64;           // packed -VT: the 100 nonzero 8 x 8 tiles (R, J >= R - 8)
constexpr int ZLD = 64;                 // staging column stride (no padding: 12 warps' buffers
                                        // fit beside the rings); 16-byte slots XOR-swizzled
                                        // by the column's parity for conflict-free reads
// element (column c, row i) of a staging buffer
__host__ __device__ __forceinline__ int zidx(int c, int i) {
  return c * ZLD + ((((i >> 1) ^ ((c & 1) << 2)) << 1) | (i & 1));
}

__host__ __device__ __forceinline__ int64_t tasks(int64_t n, int64_t s) {
  return (n - 1 - s + QB - 1) / QB;
}
// -VT row tile R holds column tiles J = vt_j0(R) .. 7 (VT[r][j] = 0 for j < r - 64), stored
// from tile vt_t0(R) on
__host__ __device__ constexpr int vt_j0(int R) { return R < 9 ? 0 : R - 8; }
__host__ __device__ constexpr int vt_t0(int R) {
  return R < 9 ? 8 * R : 72 + (R - 9) * 7 - (R - 9) * (R - 10) / 2;
}

template <int NW>
struct Q2R {
  static constexpr int WC = 8 * NW;
  static constexpr int OFF_VT = 2 * VP;          // V ring: 2 stages, VT ring: 2 stages
  static constexpr int OFF_Z = OFF_VT + 2 * VTP;
  static constexpr int OFF_BAR = OFF_Z + NW * 8 * ZLD;
  static constexpr size_t SMEM = (size_t)OFF_BAR * sizeof(double) + 8 * sizeof(uint64_t);
};

EM_DEVINL void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// plain loads and a non-volatile DMMA: the compiler may schedule fragment loads ahead of
// the products (the mbarrier waits carry "memory" clobbers, so no load crosses them)
EM_DEVINL double2 lds128(const double* p) { return *reinterpret_cast<const double2*>(p); }
EM_DEVINL void mma(double& c0, double& c1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}
}  // namespace

// Packed operands of every block k of group g (T2g: the group's T factors, row-major).
//   Vp[k][(J*9 + dR)*64 + lane*2 + e]   = V[8(J + dR) + 2t + e][8J + g]
//   VTp[k][(vt_t0(R) + J - vt_j0(R))*64 + lane*2 + e] = -VT[8R + g][8J + 2t + e]
// with lane = 4g + t; V is zero outside the parallelogram and beyond row n.
__global__ void __launch_bounds__(256) q2r_pack_kernel(int64_t n, int64_t g,
                                                       const double* __restrict__ V2,
                                                       const int64_t* __restrict__ toff,
                                                       const double* __restrict__ T2g,
                                                       double* __restrict__ Vp,
                                                       double* __restrict__ VTp) {
  extern __shared__ double psm[];
  double* Vs = psm;                  // [j][i] = v_j[i]
  double* Ts = psm + QB * (QB + 1);  // [i][j]
  const int64_t k = blockIdx.x;
  const int64_t W0 = QB * (g + k);
  const int tid = threadIdx.x;
  for (int e = tid; e < QB * QB; e += blockDim.x) {
    const int j = e >> 6, i = e & 63;
    const int64_t s = g * QB + j;
    double v = 0.0;
    if (s < n - 1 && k < tasks(n, s) && W0 + 1 + j + i < n) v = V2[(toff[s] + k) * QB + i];
    Vs[j * (QB + 1) + i] = v;
    Ts[(e >> 6) * (QB + 1) + (e & 63)] = T2g[k * QB * QB + e];
  }
  __syncthreads();
  auto vval = [&](int r, int j) -> double {
    const int i = r - 1 - j;
    return (i >= 0 && i < QB) ? Vs[j * (QB + 1) + i] : 0.0;
  };
  double* vp = Vp + k * (int64_t)VP;
  for (int e = tid; e < VP; e += blockDim.x) {
    const int tile = e >> 6, w = e & 63, lane = w >> 1, ee = w & 1;
    const int J = tile / 9, R = J + tile % 9;
    vp[e] = vval(8 * R + 2 * (lane & 3) + ee, 8 * J + (lane >> 2));
  }
  double* vtp = VTp + k * (int64_t)VTP;
  for (int e = tid; e < VTP; e += blockDim.x) {
    const int tile = e >> 6, w = e & 63, lane = w >> 1, ee = w & 1;
    int R = 0;
    while (R < 15 && vt_t0(R + 1) <= tile) ++R;
    const int J = vt_j0(R) + tile - vt_t0(R);
    const int r = 8 * R + (lane >> 2), j = 8 * J + 2 * (lane & 3) + ee;
    const int i0 = r - QB > 0 ? r - QB : 0;
    const int i1 = r - 1 < j ? r - 1 : j;
    double acc = 0.0;
    for (int i = i0; i <= i1; ++i) acc = fma(vval(r, i), Ts[i * (QB + 1) + j], acc);
    vtp[e] = -acc;
  }
}

namespace {
template <int NW>
struct Q2RWarp {
  const double* Vs;   // V ring base (2 stages)
  const double* VTs;  // VT ring base (2 stages)
  double* zst;        // this warp's staging buffer [8 cols][ZLD]
  double* Z;
  int64_t ldz, n, ncols, col, c0w;
  int lane, gq, tq, dbg;

  // rows 64 h .. 64 h + 63 of the warp's 8 columns into the staging buffer. L2-only
  // copies (.cg): Z rows this SM stored earlier (the previous group's launch, or lines that
  // straddle two halves when a column does not start 128-byte aligned) must not be served
  // from a stale L1 line. 16-byte copies of row pairs when ldz is even, else synchronous
  // 8-byte loads.
  EM_DEVINL void load_half(int64_t h) const {
    if ((ldz & 1) == 0 && !(dbg & 4)) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int e = q * 32 + lane, c = e >> 5, i = 2 * (e & 31);
        const int64_t row = 64 * h + i, cg = c0w + c;
        const int bytes = (cg < ncols && row < n) ? (row + 1 < n ? 16 : 8) : 0;
        cp_async16(zst + zidx(c, i), bytes ? Z + row + cg * ldz : Z, bytes);
      }
    } else {
#pragma unroll
      for (int q = 0; q < 16; ++q) {
        const int e = q * 32 + lane, c = e >> 6, i = e & 63;
        const int64_t row = 64 * h + i, cg = c0w + c;
        const bool ok = row < n && cg < ncols;
        // (8-byte cp.async exists only as .ca: synchronous L2 loads instead)
        zst[zidx(c, i)] = ok ? __ldcg(Z + row + cg * ldz) : 0.0;
      }
    }
    cp_async_commit();
  }
  EM_DEVINL void read_half(double (&z)[8][2]) const {
    cp_async_wait<0>();
    __syncwarp();
#pragma unroll
    for (int R = 0; R < 8; ++R) {
      const double2 v = lds128(zst + zidx(gq, 8 * R + 2 * tq));
      z[R][0] = v.x;
      z[R][1] = v.y;
    }
    __syncwarp();
  }
  EM_DEVINL void store_half(const double (&z)[8][2], int64_t h) const {
    if (col >= ncols) return;
#pragma unroll
    for (int R = 0; R < 8; ++R) {
      const int64_t row = 64 * h + 8 * R + 2 * tq;
      if (row < n) Z[row + col * ldz] = z[R][0];
      if (row + 1 < n) Z[row + 1 + col * ldz] = z[R][1];
    }
  }
  // W^T = Zwin^T V (k-step (R, e) = rows 8R + 2t + e; R = J .. J + 8 carry V's nonzeros).
  // Per dR the 8 fragment pairs are loaded first and the e = 0 products of all J issued
  // before the e = 1 ones: a DMMA never waits on the one issued just before it.
  EM_DEVINL void step_a(const double (&zt)[8][2], const double (&zb)[8][2], const double* vs,
                        double (&w)[8][2]) const {
#pragma unroll
    for (int J = 0; J < 8; ++J) w[J][0] = w[J][1] = 0.0;
    // fragment pairs double-buffered: the loads of dR + 1 are in flight under dR's products
    double2 b[2][8];
#pragma unroll
    for (int J = 0; J < 8; ++J) b[0][J] = lds128(vs + (J * 9) * 64 + 2 * lane);
#pragma unroll
    for (int dR = 0; dR < 9; ++dR) {
      const int cur = dR & 1;
      if (dR + 1 < 9) {
#pragma unroll
        for (int J = 0; J < 8; ++J) b[cur ^ 1][J] = lds128(vs + (J * 9 + dR + 1) * 64 + 2 * lane);
      }
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int J = 0; J < 8; ++J) {
          const int R = J + dR;
          const double a = R < 8 ? zt[R & 7][e] : zb[R & 7][e];
          mma(w[J][0], w[J][1], a, e ? b[cur][J].y : b[cur][J].x);
        }
    }
  }
  // Zwin^T += W^T (-(V T))^T (k-step (J, e) = reflectors 8J + 2t + e); VT[r][j] = 0 for
  // j < r - 64: row tiles R >= 9 start at J = R - 8. Row tiles in groups of 8, the e = 0
  // products of a group before its e = 1 ones.
  EM_DEVINL void step_c(double (&zt)[8][2], double (&zb)[8][2], const double* vts,
                        const double (&w)[8][2]) const {
    // 16 (J, h) half-steps, fragment pairs double-buffered across them
    double2 b[2][8];
    auto load = [&](int step, double2(&bb)[8]) {
      const int J = step >> 1, h = step & 1;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int R = 8 * h + q;
        if (J >= vt_j0(R)) bb[q] = lds128(vts + (vt_t0(R) + J - vt_j0(R)) * 64 + 2 * lane);
      }
    };
    load(0, b[0]);
#pragma unroll
    for (int step = 0; step < 16; ++step) {
      const int J = step >> 1, h = step & 1, cur = step & 1;
      if (step + 1 < 16) load(step + 1, b[cur ^ 1]);
#pragma unroll
      for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int R = 8 * h + q;
          if (J < vt_j0(R)) continue;
          double(&c)[2] = h == 0 ? zt[q] : zb[q];
          mma(c[0], c[1], w[J][e], e ? b[cur][q].y : b[cur][q].x);
        }
    }
  }
};
}  // namespace

// One launch per group g (K blocks): CTA = strip of 8 NW columns, NW consumer warps + one
// producer warp (bulk copies of the packed V / VT of each block).
//
// Strips: CTAs [0, nfull) take 8 NW columns each (a whole number of waves when nfull is a
// multiple of the SM count); the ntail CTAs after them share the remaining `rem` 8-column
// units as evenly as possible (fewer active warps each), so the last wave is short
// instead of partly empty.
// With NW a multiple of 4 the producer is a whole warpgroup (one active lane) that hands
// its registers to the consumer warpgroups (setmaxnreg): the consumers run at RC registers
// (no spills, V / VT fragments of the next step prefetched) instead of 168.
template <int NW>
struct Q2RRegs {
  static constexpr bool kSplit = NW % 4 == 0;
  static constexpr int PW = kSplit ? 4 : 1;
  static constexpr int RP = 40;
  static constexpr int RC = kSplit ? ((65536 - 128 * RP) / (NW * 32)) / 8 * 8 > 232
                                         ? 232
                                         : ((65536 - 128 * RP) / (NW * 32)) / 8 * 8
                                   : 0;
};

template <int NW>
__global__ void __launch_bounds__((NW + Q2RRegs<NW>::PW) * 32, 1) q2r_kernel(int64_t n, int64_t ncols,
                                                               int64_t g, int64_t K,
                                                               const double* __restrict__ Vp,
                                                               const double* __restrict__ VTp,
                                                               double* __restrict__ Z,
                                                               int64_t ldz, int64_t nfull,
                                                               int64_t ntail, int64_t rem,
                                                               int dbg) {
  using S = Q2R<NW>;
  extern __shared__ __align__(128) double sm[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + S::OFF_BAR);
  uint64_t* full_v = bars;        // [2]
  uint64_t* empty_v = bars + 2;   // [2]
  uint64_t* full_vt = bars + 4;   // [2]
  uint64_t* empty_vt = bars + 6;  // [2]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int64_t c0 = (int64_t)blockIdx.x * S::WC;
  int nact = NW;
  if ((int64_t)blockIdx.x >= nfull) {
    const int64_t i = blockIdx.x - nfull, base = rem / ntail, extra = rem % ntail;
    nact = (int)(base + (i < extra ? 1 : 0));
    c0 = nfull * S::WC + 8 * (i * base + (i < extra ? i : extra));
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&full_v[s], 1);
      mbar_init(&empty_v[s], nact);
      mbar_init(&full_vt[s], 1);
      mbar_init(&empty_vt[s], nact);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  if (warp >= NW) {  // producer
    if constexpr (Q2RRegs<NW>::kSplit)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(Q2RRegs<NW>::RP));
    if (warp == NW && lane == 0) {
      for (int64_t k = 0; k < K; ++k) {
        const int s = (int)(k & 1);
        const unsigned par = (unsigned)(((k >> 1) - 1) & 1);
        if (k >= 2) mbar_wait(&empty_v[s], par);
        mbar_expect_tx(&full_v[s], VP * sizeof(double));
        bulk_g2s(sm + s * VP, Vp + k * (int64_t)VP, VP * sizeof(double), &full_v[s]);
        if (k >= 2) mbar_wait(&empty_vt[s], par);
        if ((dbg & 1) && k >= 1) mbar_wait(&empty_vt[s ^ 1], (unsigned)(((k - 1) >> 1) & 1));
        mbar_expect_tx(&full_vt[s], VTP * sizeof(double));
        bulk_g2s(sm + S::OFF_VT + s * VTP, VTp + k * (int64_t)VTP, VTP * sizeof(double),
                 &full_vt[s]);
      }
    }
    return;
  }
  if constexpr (Q2RRegs<NW>::kSplit)
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(Q2RRegs<NW>::RC));
  if (warp >= nact) return;

  Q2RWarp<NW> W;
  W.Vs = sm;
  W.VTs = sm + S::OFF_VT;
  W.zst = sm + S::OFF_Z + warp * 8 * ZLD;
  W.Z = Z;
  W.ldz = ldz;
  W.n = n;
  W.ncols = ncols;
  W.lane = lane;
  W.dbg = dbg;
  W.gq = lane >> 2;
  W.tq = lane & 3;
  W.c0w = c0 + 8 * warp;
  W.col = W.c0w + W.gq;

  double za[8][2], zb[8][2], w[8][2];
  W.load_half(g);
  W.read_half(za);
  W.load_half(g + 1);

  auto block = [&](double(&zt)[8][2], double(&zbt)[8][2], int64_t k) {
    W.read_half(zbt);  // half g + k + 1
    const int s = (int)(k & 1);
    mbar_wait(&full_v[s], (unsigned)((k >> 1) & 1));
    // Stage releases come one phase late, behind the NEXT barrier wait: every DMMA that
    // read the stage precedes that wait in program order, and a DMMA issues only once its
    // fragment loads have delivered, so the stage's shared-memory reads are done. (Released
    // right after its last use, ptxas schedules the arrive directly behind the last LDS,
    // ahead of the consuming DMMAs, and a load delayed behind other warps' global traffic
    // can be overtaken by the producer's next bulk copy: seen in gemm_tma.cu. A release
    // made data-dependent on the accumulators is safe too but stalls the warp: +4%.)
    __syncwarp();
    if (k > 0 && lane == 0) mbar_arrive(&empty_vt[s ^ 1]);  // VT(k-1): step C of block k-1
    W.step_a(zt, zbt, W.Vs + s * VP, w);
    // The staging buffer is refilled only after every value read from it went into a
    // product: the asm below consumes the W accumulators (so every step-A DMMA, and with it
    // every staging load feeding one, is issued before it), and the cp.async writes
    // follow it. An async copy issued right after the loads raced with them.
#pragma unroll
    for (int J = 0; J < 8; ++J) asm volatile("" : "+d"(w[J][0]), "+d"(w[J][1]));
    if (k + 2 <= K) W.load_half(g + k + 2);
    if (dbg & 8) {
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __threadfence_block();
    }
    mbar_wait(&full_vt[s], (unsigned)((k >> 1) & 1));
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_v[s]);  // V(k): step A above
    W.step_c(zt, zbt, W.VTs + s * VTP, w);
    W.store_half(zt, g + k);  // final for this group
  };
  int64_t k = 0;
  for (; k + 1 < K; k += 2) {
    block(za, zb, k);
    block(zb, za, k + 1);
  }
  if (k < K) {
    block(za, zb, k);
    W.store_half(zb, g + K);
  } else {
    W.store_half(za, g + K);
  }
}

// Z (n x ncols, ld ldz) <- Q2 Z for all groups (last first); T2: every block's T factor,
// groups descending and positions ascending (q2_tfactor_kernel's order).
// NW consumer warps + 1 producer per CTA. The register file is split between the four
// SM sub-partitions, so 9 warps (NW = 8: 3 on one sub-partition) allow 168 registers per
// thread (a few spills) while 8 warps (NW = 7) allow 255 (no spills, one consumer fewer).
template <int NW>
static void q2_apply_nw(cudaStream_t st, int64_t n, int64_t ncols, int64_t ngroups,
                        const double* V2, const int64_t* toff, const double* T2, double* Z,
                        int64_t ldz) {
  using S = Q2R<NW>;
  EM_CK(cudaFuncSetAttribute(q2r_kernel<NW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)S::SMEM));
  constexpr size_t kPackSmem = 2 * QB * (QB + 1) * sizeof(double);
  EM_CK(cudaFuncSetAttribute(q2r_pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)kPackSmem));
  const int64_t kmax = imax64(tasks(n, 0), 1);
  DBuf Vp((size_t)kmax * VP, st), VTp((size_t)kmax * VTP, st);
  const int64_t sms = num_sms();
  const int64_t units = (ncols + 7) / 8;
  int64_t nfull = units / NW / sms * sms;
  if (g_q2r_dbg & 2) nfull = (units + NW - 1) / NW;
  const int64_t rem = imax64(units - nfull * NW, 0);
  const int64_t ntail = imin64(rem, sms);
  int64_t off = 0;
  for (int64_t g = ngroups - 1; g >= 0; --g) {
    const int64_t K = tasks(n, g * QB);
    if (K <= 0) continue;
    q2r_pack_kernel<<<(unsigned)K, 256, kPackSmem, st>>>(n, g, V2, toff, T2 + off * QB * QB,
                                                         Vp.p, VTp.p);
    EM_LAUNCHED();
    q2r_kernel<NW><<<(unsigned)(nfull + ntail), (NW + Q2RRegs<NW>::PW) * 32, S::SMEM, st>>>(
        n, ncols, g, K, Vp.p, VTp.p, Z, ldz, nfull, imax64(ntail, 1), rem, g_q2r_dbg);
    EM_LAUNCHED();
    off += K;
  }
}

void q2_apply_reg(cudaStream_t st, int64_t n, int64_t ncols, int64_t ngroups, const double* V2,
                  const int64_t* toff, const double* T2, double* Z, int64_t ldz) {
  if (ncols <= 0 || n <= 1) return;
  // 12 consumer warps per CTA run the tensor pipe fuller (C3: 11.05 s against 11.31 s with
  // 8), but with fewer than two full waves of 96-column strips the short last wave costs
  // more than that (n = 16,384: 505 ms against 450 ms): 8 warps there
  const bool few = (ncols + 7) / 8 < 2 * 12 * (int64_t)num_sms();
  if (g_q2r_dbg & 16)
    q2_apply_nw<7>(st, n, ncols, ngroups, V2, toff, T2, Z, ldz);
  else if ((g_q2r_dbg & 32) || (few && !(g_q2r_dbg & 64)))
    q2_apply_nw<8>(st, n, ncols, ngroups, V2, toff, T2, Z, ldz);
  else
    q2_apply_nw<12>(st, n, ncols, ngroups, V2, toff, T2, Z, ldz);
}

}  // namespace em
