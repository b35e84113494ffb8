// Internal runtime: context, error capture, stream-ordered device workspace,
// launch accounting. Everything here is plumbing for the C ABI in capi.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <utility>
#include <vector>

#include "../../include/eddymodes_b200.h"

struct em_comm;
struct em_ctx {
  em_comm* comm = nullptr;          // inter-GPU communicator (em_comm_init_*), else single GPU
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::string err;
  int sms = 148;
  bool pool_set = false;            // em_init raised the default pool's release threshold
  uint64_t saved_threshold = 0;     // ... from this value (restored by em_finalize)
};

namespace em {

extern std::atomic<int64_t> g_launches;
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Throws on CUDA error; caught at the C ABI boundary and turned into EM_ERR_CUDA.
struct CudaError {
  cudaError_t code;
  std::string where;
};
struct ArgError {
  std::string what;
};

#define EM_CK(x)                                                                      \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess) throw ::em::CudaError{e_, std::string(#x) + " @" __FILE__}; \
  } while (0)
#define EM_LAUNCHED()                      \
  do {                                     \
    ::em::count_launch();                  \
    EM_CK(cudaGetLastError());             \
  } while (0)

// Launch with programmatic stream serialization: the kernel may start while its
// predecessor drains; it must call pdl_wait() (common.cuh) before touching the
// predecessor's outputs.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  EM_CK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
  count_launch();
}

// Stream-ordered device buffer (cudaMallocAsync pool).
struct DBuf {
  double* p = nullptr;
  size_t n = 0;
  cudaStream_t st = nullptr;
  DBuf() = default;
  DBuf(size_t count, cudaStream_t s) { alloc(count, s); }
  void alloc(size_t count, cudaStream_t s) {
    release();
    st = s;
    n = count;
    if (count) EM_CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(double), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
    n = 0;
  }
  ~DBuf() { release(); }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), n(o.n), st(o.st) { o.p = nullptr; o.n = 0; }
};

template <typename T>
struct DArr {
  T* p = nullptr;
  cudaStream_t st = nullptr;
  DArr() = default;
  DArr(size_t count, cudaStream_t s) { alloc(count, s); }
  void alloc(size_t count, cudaStream_t s) {
    release();
    st = s;
    if (count) EM_CK(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), s));
  }
  void release() {
    if (p) cudaFreeAsync(p, st);
    p = nullptr;
  }
  ~DArr() { release(); }
  DArr(const DArr&) = delete;
  DArr& operator=(const DArr&) = delete;
  DArr(DArr&& o) noexcept : p(o.p), st(o.st) { o.p = nullptr; }
  DArr& operator=(DArr&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p;
      st = o.st;
      o.p = nullptr;
    }
    return *this;
  }
};

// --- stage timers (CUDA events on the launching stream; profiling mode only) ---
enum StageId {
  ST_POTRF_R = 0, ST_SYGST, ST_POTRF_L, ST_SYTRD, ST_STEDC, ST_ORMTR, ST_TRSM_BACK,
  ST_FINALIZE, ST_POST_GEMM, ST_TD2_LOCAL, ST_TD2_CARRY, ST_TD2_REPLAY, ST_TD1_SYMV,
  ST_TD1_FWD, ST_TD1_BWD, ST_SYTRD_SYMV, ST_SYTRD_SYR2K, ST_STEDC_GEMM, ST_STEDC_SECULAR,
  ST_SY2SB, ST_SB2ST, ST_Q2, ST_Q1, ST_SY2SB_QR,
  ST_COUNT
};
void stage_begin(cudaStream_t st, int id);
void stage_end(cudaStream_t st, int id);
bool stages_enabled();
struct Stage {
  cudaStream_t st;
  int id;
  Stage(cudaStream_t s, int i) : st(s), id(i) { stage_begin(st, id); }
  ~Stage() { stage_end(st, id); }
};

// --- small utility kernels (util.cu) ---------------------------------------
void mirror_lower(cudaStream_t st, int64_t n, double* A, int64_t lda);
// B = op(A) (m x n result), op = transpose when trans
void copy_matrix(cudaStream_t st, bool trans, int64_t m, int64_t n, const double* A, int64_t lda,
                 double* B, int64_t ldb);
// C = alpha*A + beta*B^T (square n) — used for symmetrisation (A + A^T)/2
void add_transpose(cudaStream_t st, int64_t n, double alpha, const double* A, int64_t lda,
                   double beta, double* C, int64_t ldc);
void zero_upper(cudaStream_t st, int64_t n, double* A, int64_t lda);
void set_identity(cudaStream_t st, int64_t n, double* A, int64_t lda);
int num_sms();

}  // namespace em
