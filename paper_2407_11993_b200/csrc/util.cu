// Memory-bound helpers: symmetric mirroring, (transposed) copies, symmetrisation.
// All tile through shared memory so both the read and the write are coalesced.
#include "common.cuh"
#include "ctx.h"
#include "plans.h"

namespace em {

std::atomic<int64_t> g_launches{0};

int num_sms() {
  static int cached = 0;
  if (!cached) {
    int d = 0;
    cudaGetDevice(&d);
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, d);
    if (cached <= 0) cached = 148;
  }
  return cached;
}

constexpr int TT = 32;  // transpose tile

// A(r, c) for r < c  <-  A(c, r)   (upper := mirror of lower)
__global__ void mirror_lower_kernel(int64_t n, double* A, int64_t lda) {
  __shared__ double t[TT][TT + 1];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;  // tile (row block bi, col block bj), bj <= bi
  if (bj > bi) return;
  const int64_t r0 = bi * TT, c0 = bj * TT;  // source tile in the lower triangle
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < n && c < n) t[k][threadIdx.x] = A[r + c * lda];
  }
  __syncthreads();
  // write transposed: dest (row c, col r) for r > c
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t dr = c0 + threadIdx.x, dc = r0 + k;  // dest row in [c0..), dest col in [r0..)
    if (dr < n && dc < n && dr < dc) A[dr + dc * lda] = t[threadIdx.x][k];
  }
}

void mirror_lower(cudaStream_t st, int64_t n, double* A, int64_t lda) {
  if (n <= 1) return;
  int64_t nt = (n + TT - 1) / TT;
  dim3 grid((unsigned)nt, (unsigned)nt), block(TT, 8);
  mirror_lower_kernel<<<grid, block, 0, st>>>(n, A, lda);
  EM_LAUNCHED();
}

__global__ void copy_kernel(int64_t m, int64_t n, const double* __restrict__ A, int64_t lda,
                            double* __restrict__ B, int64_t ldb) {
  int64_t r = blockIdx.x * (int64_t)TT + threadIdx.x;
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t c = blockIdx.y * (int64_t)TT + k;
    if (r < m && c < n) B[r + c * ldb] = A[r + c * lda];
  }
}

// B(m x n) = A^T where A is n x m
__global__ void transpose_kernel(int64_t m, int64_t n, const double* __restrict__ A, int64_t lda,
                                 double* __restrict__ B, int64_t ldb) {
  __shared__ double t[TT][TT + 1];
  const int64_t r0 = blockIdx.x * (int64_t)TT, c0 = blockIdx.y * (int64_t)TT;  // B tile origin
  // read A(c, r) for r in [r0, r0+TT), c in [c0, c0+TT): A rows = c (contiguous), cols = r
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t ar = c0 + threadIdx.x, ac = r0 + k;
    if (ar < n && ac < m) t[k][threadIdx.x] = A[ar + ac * lda];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t br = r0 + threadIdx.x, bc = c0 + k;
    if (br < m && bc < n) B[br + bc * ldb] = t[threadIdx.x][k];
  }
}

void copy_matrix(cudaStream_t st, bool trans, int64_t m, int64_t n, const double* A, int64_t lda,
                 double* B, int64_t ldb) {
  if (m <= 0 || n <= 0) return;
  dim3 grid((unsigned)((m + TT - 1) / TT), (unsigned)((n + TT - 1) / TT)), block(TT, 8);
  if (trans)
    transpose_kernel<<<grid, block, 0, st>>>(m, n, A, lda, B, ldb);
  else
    copy_kernel<<<grid, block, 0, st>>>(m, n, A, lda, B, ldb);
  EM_LAUNCHED();
}

// C = alpha*A + beta*A^T   (C may alias A only if it is done tile-pair-wise: here C != A)
__global__ void add_transpose_kernel(int64_t n, double alpha, const double* __restrict__ A,
                                     int64_t lda, double beta, double* __restrict__ C,
                                     int64_t ldc) {
  __shared__ double t[TT][TT + 1];
  const int64_t r0 = blockIdx.x * (int64_t)TT, c0 = blockIdx.y * (int64_t)TT;
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t ar = c0 + threadIdx.x, ac = r0 + k;  // A^T tile
    if (ar < n && ac < n) t[k][threadIdx.x] = A[ar + ac * lda];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t r = r0 + threadIdx.x, c = c0 + k;
    if (r < n && c < n) C[r + c * ldc] = alpha * A[r + c * lda] + beta * t[threadIdx.x][k];
  }
}

void add_transpose(cudaStream_t st, int64_t n, double alpha, const double* A, int64_t lda,
                   double beta, double* C, int64_t ldc) {
  if (n <= 0) return;
  dim3 grid((unsigned)((n + TT - 1) / TT), (unsigned)((n + TT - 1) / TT)), block(TT, 8);
  add_transpose_kernel<<<grid, block, 0, st>>>(n, alpha, A, lda, beta, C, ldc);
  EM_LAUNCHED();
}

__global__ void zero_upper_kernel(int64_t n, double* A, int64_t lda) {
  int64_t r = blockIdx.x * (int64_t)TT + threadIdx.x;
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t c = blockIdx.y * (int64_t)TT + k;
    if (r < n && c < n && r < c) A[r + c * lda] = 0.0;
  }
}

void zero_upper(cudaStream_t st, int64_t n, double* A, int64_t lda) {
  if (n <= 1) return;
  dim3 grid((unsigned)((n + TT - 1) / TT), (unsigned)((n + TT - 1) / TT)), block(TT, 8);
  zero_upper_kernel<<<grid, block, 0, st>>>(n, A, lda);
  EM_LAUNCHED();
}

__global__ void set_identity_kernel(int64_t n, double* A, int64_t lda) {
  int64_t r = blockIdx.x * (int64_t)TT + threadIdx.x;
  for (int k = threadIdx.y; k < TT; k += blockDim.y) {
    int64_t c = blockIdx.y * (int64_t)TT + k;
    if (r < n && c < n) A[r + c * lda] = (r == c) ? 1.0 : 0.0;
  }
}

void set_identity(cudaStream_t st, int64_t n, double* A, int64_t lda) {
  if (n <= 0) return;
  dim3 grid((unsigned)((n + TT - 1) / TT), (unsigned)((n + TT - 1) / TT)), block(TT, 8);
  set_identity_kernel<<<grid, block, 0, st>>>(n, A, lda);
  EM_LAUNCHED();
}

__global__ void reverse_columns_kernel(int64_t m, int64_t n, const double* __restrict__ A,
                                       int64_t lda, const double* __restrict__ w_in,
                                       double* __restrict__ B, int64_t ldb, double* w_out) {
  const int64_t j = blockIdx.y;
  const int64_t src = n - 1 - j;
  if (blockIdx.x == 0 && threadIdx.x == 0 && w_in) w_out[j] = w_in[src];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < m;
       r += (int64_t)gridDim.x * blockDim.x)
    B[r + j * ldb] = A[r + src * lda];
}

void reverse_columns(cudaStream_t st, int64_t m, int64_t n, const double* A, int64_t lda,
                     const double* w_in, double* B, int64_t ldb, double* w_out) {
  if (m <= 0 || n <= 0) return;
  dim3 grid((unsigned)imax64(1, imin64((m + 255) / 256, 32)), (unsigned)n);
  reverse_columns_kernel<<<grid, 256, 0, st>>>(m, n, A, lda, w_in, B, ldb, w_out);
  EM_LAUNCHED();
}

}  // namespace em

// ---- stage timers -----------------------------------------------------------------
namespace em {

namespace {
struct StageRec {
  int id;
  cudaEvent_t a, b;
};
bool g_stage_on = false;
std::vector<StageRec> g_recs;
std::vector<int> g_open[ST_COUNT];
}  // namespace

bool stages_enabled() { return g_stage_on; }

int g_stage_level = 0;  // 1: top-level stages, 2: also per-call inner stages

// stages recorded many times per call (per column, merge or panel): level 2 only; the
// two-stage pieces (one event pair per eigensolve each) are top-level
static bool inner_stage(int id) {
  return id == ST_SYTRD_SYMV || id == ST_SYTRD_SYR2K || id == ST_STEDC_GEMM ||
         id == ST_STEDC_SECULAR || id == ST_SY2SB_QR;
}

void stage_begin(cudaStream_t st, int id) {
  if (!g_stage_on || (inner_stage(id) && g_stage_level < 2)) return;
  StageRec r{id, nullptr, nullptr};
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  cudaEventRecord(r.a, st);
  g_open[id].push_back((int)g_recs.size());
  g_recs.push_back(r);
}

void stage_end(cudaStream_t st, int id) {
  if (!g_stage_on || g_open[id].empty()) return;
  const int k = g_open[id].back();
  g_open[id].pop_back();
  cudaEventRecord(g_recs[k].b, st);
}

void stages_level(int level) { g_stage_level = level; }

void stages_reset(bool on) {
  for (auto& r : g_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_recs.clear();
  for (auto& o : g_open) o.clear();
  g_stage_on = on;
}

int stages_read(double* ms, int64_t* counts, int n) {
  for (int i = 0; i < n; ++i) {
    ms[i] = 0.0;
    if (counts) counts[i] = 0;
  }
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess && r.id < n) {
      ms[r.id] += t;
      if (counts) counts[r.id] += 1;
    }
  }
  return ST_COUNT;
}

}  // namespace em
