// extern "C" boundary of libeddymodes_b200.so (see include/eddymodes_b200.h).
// Every entry catches internal exceptions and maps them to EM_ERR_* codes with
// a message retrievable through em_last_error().
#include <stdio.h>

#include <string>

#include "common.cuh"
#include "comm.h"
#include "ctx.h"
#include "gemm.h"
#include "linalg.h"

struct em_td2_plan;
struct em_td1_plan;

namespace em {
extern int64_t g_two_stage_min;
extern int g_qr_gm;
extern int g_sytrd_dbg;
extern int g_band_off;
extern int g_ln_dense;
extern int g_l_certificate;
extern int g_q2r_dbg;
extern int g_last_eig_path;
extern int g_q2_mode;
extern int g_symv_align_off;
extern int64_t g_symv_keep_mb;
extern int64_t g_gemm_cfg;
extern int64_t g_gemm_tma;
extern int64_t g_td1_staged;
void stages_reset(bool on);
void stages_level(int level);
int stages_read(double* ms, int64_t* counts, int n);
int64_t sygv(cudaStream_t st, int64_t n, const double* L, int64_t ldl, const double* R,
             int64_t ldr, double* tau, double* V, int64_t ldv, double* l_n, double* r_n,
             double* VtR, int64_t ldvtr, int* which, int flags,
             cudaEvent_t l_ready = nullptr, int64_t m_lo = 0, int64_t m_hi = -1,
             double* Y = nullptr, int64_t ldy = 0, int64_t ky = 0, const double* Rb = nullptr,
             int64_t ldrb = 0, int64_t rbw = -1);
}

// full definitions live in td1.cu / td2.cu; re-declare the layout-independent API here
#include "plans.h"

namespace {

template <typename F>
int guarded(em_ctx* ctx, F&& f) {
  try {
    if (ctx) cudaSetDevice(ctx->device);
    em::g_cur_ctx = ctx;  // the context whose communicator the distributed stages use
    return f();
  } catch (const em::CudaError& e) {
    if (ctx) ctx->err = std::string(cudaGetErrorString(e.code)) + " in " + e.where;
    return EM_ERR_CUDA;
  } catch (const em::ArgError& e) {
    if (ctx) ctx->err = e.what;
    return EM_ERR_ARG;
  } catch (const std::bad_alloc&) {
    if (ctx) ctx->err = "host allocation failed";
    return EM_ERR_ALLOC;
  }
}

}  // namespace

extern "C" {

int em_init(int device, em_ctx** out) {
  if (!out) return EM_ERR_ARG;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    *out = nullptr;
    return EM_ERR_CUDA;
  }
  if (device < 0 || device >= count) return EM_ERR_ARG;
  auto* ctx = new em_ctx();
  ctx->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return EM_ERR_CUDA;
  }
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return EM_ERR_CUDA;
  }
  ctx->own_stream = true;
  ctx->sms = em::num_sms();
  // keep freed pool memory cached between calls (stream-ordered allocator); the previous
  // threshold comes back and the cache is released in em_finalize (em_trim releases it
  // on demand)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess &&
      cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &ctx->saved_threshold) ==
          cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    ctx->pool_set =
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr) == cudaSuccess;
  }
  *out = ctx;
  return EM_OK;
}

int em_comm_unique_id(em_ctx* ctx, void* id) {
  if (!ctx || !id) return EM_ERR_ARG;
  return guarded(ctx, [&] {
    em::comm_unique_id(id);
    return EM_OK;
  });
}

int em_comm_init_nccl(em_ctx* ctx, int nranks, int rank, const void* id) {
  if (!ctx || !id) return EM_ERR_ARG;
  return guarded(ctx, [&] {
    EM_CK(cudaSetDevice(ctx->device));
    em::comm_init_nccl(ctx, nranks, rank, id);
    return EM_OK;
  });
}

int em_comm_init_callbacks(em_ctx* ctx, int nranks, int rank, em_allreduce_fn allreduce,
                           em_bcast_fn bcast, void* user) {
  if (!ctx) return EM_ERR_ARG;
  return guarded(ctx, [&] {
    em::comm_init_callbacks(ctx, nranks, rank, allreduce, bcast, user);
    return EM_OK;
  });
}

int em_comm_info(em_ctx* ctx, int64_t* info) {
  if (!ctx || !info) return EM_ERR_ARG;
  const em_comm* c = ctx->comm;
  info[0] = c ? c->nranks : 1;
  info[1] = c ? c->rank : 0;
  info[2] = c ? c->backend : 0;
  info[3] = c ? c->n_allreduce : 0;
  info[4] = c ? c->n_bcast : 0;
  info[5] = c ? c->bytes : 0;
  return EM_OK;
}

int em_comm_destroy(em_ctx* ctx) {
  if (!ctx) return EM_ERR_ARG;
  return guarded(ctx, [&] {
    em::comm_destroy(ctx);
    return EM_OK;
  });
}

void em_finalize(em_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  em::comm_destroy(ctx);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  cudaMemPool_t pool;
  if (ctx->pool_set && cudaDeviceGetDefaultMemPool(&pool, ctx->device) == cudaSuccess) {
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &ctx->saved_threshold);
    cudaMemPoolTrimTo(pool, 0);
  }
  delete ctx;
}

int em_trim(em_ctx* ctx) {
  if (!ctx) return EM_ERR_ARG;
  return guarded(ctx, [&] {
    EM_CK(cudaStreamSynchronize(ctx->stream));
    cudaMemPool_t pool;
    EM_CK(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
    EM_CK(cudaMemPoolTrimTo(pool, 0));
    return EM_OK;
  });
}

int em_info(em_ctx* ctx, int key, int64_t* value) {
  if (!ctx || !value) return EM_ERR_ARG;
  if (key == EM_INFO_EIG_PATH) {
    *value = em::g_last_eig_path;
    return EM_OK;
  }
  return EM_ERR_ARG;
}

int em_set_stream(em_ctx* ctx, void* s) {
  if (!ctx) return EM_ERR_ARG;
  return guarded(ctx, [&] {
    if (ctx->own_stream && ctx->stream) {
      EM_CK(cudaStreamSynchronize(ctx->stream));
      EM_CK(cudaStreamDestroy(ctx->stream));
    }
    // used as given: NULL is the legacy default stream (torch's default stream)
    ctx->stream = reinterpret_cast<cudaStream_t>(s);
    ctx->own_stream = false;
    return EM_OK;
  });
}

const char* em_last_error(const em_ctx* ctx) { return ctx ? ctx->err.c_str() : "no context"; }

int64_t em_launch_count(const em_ctx*) { return em::g_launches.load(); }

int em_profile(em_ctx* ctx, int enable) {
  return guarded(ctx, [&] {
    EM_CK(cudaStreamSynchronize(ctx->stream));
    em::stages_reset(enable != 0);
    em::stages_level(enable);
    return EM_OK;
  });
}

int em_stage_times(em_ctx* ctx, double* ms, int64_t* counts, int n) {
  return guarded(ctx, [&] {
    EM_CK(cudaStreamSynchronize(ctx->stream));
    return em::stages_read(ms, counts, n);
  });
}

int em_config(em_ctx* ctx, int key, int64_t value) {
  return guarded(ctx, [&] {
    if (key == EM_CFG_TWO_STAGE_MIN) {
      em::g_two_stage_min = value;
      return EM_OK;
    }
    if (key == EM_CFG_BAND_OFF) {
      em::g_band_off = value ? 1 : 0;
      return EM_OK;
    }
    if (key == EM_CFG_L_CERTIFICATE) {
      em::g_l_certificate = value ? 1 : 0;
      return EM_OK;
    }
    if (key == EM_CFG_LN_DENSE) {
      em::g_ln_dense = value ? 1 : 0;
      return EM_OK;
    }
    if (key == EM_CFG_SYMV_L2_KEEP_MB) {
      em::g_symv_keep_mb = value;
      return EM_OK;
    }
    if (key == 95) {  // debug: TMA-fed GEMM (0 off, 1 auto, 2 / 4 / 5 force a tile configuration)
      em::g_gemm_tma = value;
      return EM_OK;
    }
    if (key == 96) {  // debug: GEMM tiles (0 default, 2 64x64 x4, 3 128x64, 4 64x64 x3)
      em::g_gemm_cfg = value;
      return EM_OK;
    }
    if (key == 99) {  // debug: release the device pool's cached memory down to `value` bytes
      EM_CK(cudaStreamSynchronize(ctx->stream));
      cudaMemPool_t pool;
      EM_CK(cudaDeviceGetDefaultMemPool(&pool, ctx->device));
      EM_CK(cudaMemPoolTrimTo(pool, (size_t)value));
      return EM_OK;
    }
    if (key == 92) {  // debug: the band reduction's panel QR in global memory (tall-panel form)
      em::g_qr_gm = value ? 1 : 0;
      return EM_OK;
    }
    if (key == 93) {  // debug: TD1 solves (0 register tiles, 1 TMA-staged tiles)
      em::g_td1_staged = value;
      return EM_OK;
    }
    if (key == 94) {  // debug: register-resident Q2 switches (q2reg.cu)
      em::g_q2r_dbg = (int)value;
      return EM_OK;
    }
    if (key == 97) {  // debug: Q2 back-transform (0 register-resident, 1 wavefront GEMMs, 2 strips)
      em::g_q2_mode = (int)value;
      return EM_OK;
    }
    if (key == 98) {  // debug: sytrd switches (bit0 no TMA symv, bit1 no PDL, bit2 no graph,
                      // bit3 the 4-launch column chain)
      em::g_sytrd_dbg = (int)value;
      em::g_symv_align_off = (value & 16) ? 1 : 0;
      return EM_OK;
    }
    throw em::ArgError{"unknown em_config key"};
  });
}

int em_synchronize(em_ctx* ctx) {
  return guarded(ctx, [&] {
    EM_CK(cudaStreamSynchronize(ctx->stream));
    return EM_OK;
  });
}

int em_dgemm(em_ctx* ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
             const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
             int64_t ldc) {
  return guarded(ctx, [&] {
    EM_CK(em::gemm(ctx->stream, ta != 0, tb != 0, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc));
    return EM_OK;
  });
}

int em_dgemm_lower(em_ctx* ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
                   const double* A, int64_t lda, const double* B, int64_t ldb, double beta,
                   double* C, int64_t ldc, int64_t diag_off) {
  return guarded(ctx, [&] {
    EM_CK(em::gemm(ctx->stream, ta != 0, tb != 0, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc,
                   true, diag_off));
    return EM_OK;
  });
}

int em_dsymm_band_lower(em_ctx* ctx, int64_t m, int64_t n, const double* A, int64_t lda,
                        const double* B, int64_t ldb, double* C, int64_t ldc) {
  return guarded(ctx, [&] {
    const cudaError_t e = em::gemm_symm_lower_tma(ctx->stream, m, n, A, lda, B, ldb, C, ldc);
    if (e == cudaErrorNotSupported)
      throw em::ArgError{"em_dsymm_band_lower: A must be 16-byte aligned with even lda, ldb"};
    EM_CK(e);
    return EM_OK;
  });
}

int em_symv_lower(em_ctx* ctx, int64_t n, double alpha, const double* A, int64_t lda,
                  const double* x, double beta, double* y) {
  return guarded(ctx, [&] {
    em::DBuf work(em::symv_work_size(n), ctx->stream);
    em::symv_lower(ctx->stream, n, alpha, A, lda, x, beta, y, work.p);
    return EM_OK;
  });
}

int em_sym_mm(em_ctx* ctx, int64_t n, int64_t m, const double* A, int64_t lda, const double* B,
              int64_t ldb, double* C, int64_t ldc) {
  return guarded(ctx, [&] {
    if (n < 0 || m < 0) throw em::ArgError{"bad em_sym_mm sizes"};
    if (!em::sym_sparse_mm(ctx->stream, n, A, lda, m, B, ldb, C, ldc, 0.02))
      EM_CK(em::gemm(ctx->stream, false, false, n, m, n, 1.0, A, lda, B, ldb, 0.0, C, ldc));
    return EM_OK;
  });
}

int em_sym_mirror_lower(em_ctx* ctx, int64_t n, double* A, int64_t lda) {
  return guarded(ctx, [&] {
    em::mirror_lower(ctx->stream, n, A, lda);
    return EM_OK;
  });
}

int em_potrf(em_ctx* ctx, int64_t n, double* A, int64_t lda, int64_t* pivot) {
  return guarded(ctx, [&] {
    const int64_t p = em::potrf(ctx->stream, n, A, lda);
    if (pivot) *pivot = p;
    return p >= 0 ? EM_ERR_NOT_PD : EM_OK;
  });
}

int em_trsm_lower(em_ctx* ctx, int trans, int64_t n, int64_t m, const double* C, int64_t ldc,
                  double* B, int64_t ldb) {
  return guarded(ctx, [&] {
    em::trsm_lower(ctx->stream, trans != 0, n, m, C, ldc, B, ldb);
    return EM_OK;
  });
}

int em_syev(em_ctx* ctx, int64_t n, double* A, int64_t lda, double* w, double* U, int64_t ldu) {
  return guarded(ctx, [&] {
    cudaStream_t st = ctx->stream;
    em::DBuf wa(n, st), Za((size_t)n * n, st);
    em::syev_ascending(st, n, A, lda, wa.p, Za.p, n);
    // descending order (linalg.py:132-134): reverse
    em::reverse_columns(st, n, n, Za.p, n, wa.p, U, ldu, w);
    EM_CK(cudaStreamSynchronize(st));
    return EM_OK;
  });
}

int em_sygv_ex(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, double* R, int64_t ldr,
               double* tau, double* V, int64_t ldv, double* l_n, double* r_n, double* VtR,
               int64_t ldvtr, int flags, int64_t* pivot, int* which) {
  return guarded(ctx, [&] {
    if (flags & ~EM_SYGV_R_WORKSPACE) throw em::ArgError{"unknown em_sygv_ex flags"};
    int wh = -1;
    const int64_t p = em::sygv(ctx->stream, n, L, ldl, R, ldr, tau, V, ldv, l_n, r_n, VtR, ldvtr,
                               &wh, flags);
    if (pivot) *pivot = p;
    if (which) *which = wh;
    return p >= 0 ? EM_ERR_NOT_PD : EM_OK;
  });
}

int em_sygv_range(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, double* R, int64_t ldr,
                  int64_t m_lo, int64_t m_hi, double* tau, double* V, int64_t ldv, double* l_n,
                  double* r_n, double* VtR, int64_t ldvtr, int flags, int64_t* pivot,
                  int* which) {
  return guarded(ctx, [&] {
    if (flags & ~EM_SYGV_R_WORKSPACE) throw em::ArgError{"unknown em_sygv_range flags"};
    if (m_lo < 0 || m_hi > n || m_lo > m_hi) throw em::ArgError{"em_sygv_range: bad mode range"};
    int wh = -1;
    const int64_t p = em::sygv(ctx->stream, n, L, ldl, R, ldr, tau, V, ldv, l_n, r_n, VtR, ldvtr,
                               &wh, flags, nullptr, m_lo, m_hi);
    if (pivot) *pivot = p;
    if (which) *which = wh;
    return p >= 0 ? EM_ERR_NOT_PD : EM_OK;
  });
}

int em_sygv_implicit(em_ctx* ctx, int64_t n, double* L, int64_t ldl, double* R, int64_t ldr,
                     double* tau, double* Y, int64_t ldy, int64_t k, double* l_n, double* r_n,
                     int flags, int64_t* pivot, int* which) {
  return guarded(ctx, [&] {
    if (flags & ~(EM_SYGV_R_WORKSPACE | EM_SYGV_L_WORKSPACE))
      throw em::ArgError{"unknown em_sygv_implicit flags"};
    if (k < 0 || (k > 0 && (!Y || ldy < n))) throw em::ArgError{"em_sygv_implicit: bad Y"};
    int wh = -1;
    double dummy = 0.0;
    const int64_t p = em::sygv(ctx->stream, n, L, ldl, R, ldr, tau, nullptr, n, l_n, r_n,
                               nullptr, n, &wh, flags, nullptr, 0, -1, k > 0 ? Y : &dummy,
                               ldy, k);
    if (pivot) *pivot = p;
    if (which) *which = wh;
    return p >= 0 ? EM_ERR_NOT_PD : EM_OK;
  });
}

int em_sygv_implicit_band(em_ctx* ctx, int64_t n, double* L, int64_t ldl, const double* Rb,
                          int64_t ldrb, int64_t bw, double* tau, double* Y, int64_t ldy,
                          int64_t k, double* l_n, double* r_n, int flags, int64_t* pivot,
                          int* which) {
  return guarded(ctx, [&] {
    if (flags & ~EM_SYGV_L_WORKSPACE) throw em::ArgError{"unknown em_sygv_implicit_band flags"};
    if (!Rb || bw < 0 || ldrb < bw + 1) throw em::ArgError{"em_sygv_implicit_band: bad band"};
    if (k < 0 || (k > 0 && (!Y || ldy < n))) throw em::ArgError{"em_sygv_implicit_band: bad Y"};
    int wh = -1;
    double dummy = 0.0;
    const int64_t p = em::sygv(ctx->stream, n, L, ldl, nullptr, n, tau, nullptr, n, l_n, r_n,
                               nullptr, n, &wh, flags, nullptr, 0, -1, k > 0 ? Y : &dummy,
                               ldy, k, Rb, ldrb, bw);
    if (pivot) *pivot = p;
    if (which) *which = wh;
    return p >= 0 ? EM_ERR_NOT_PD : EM_OK;
  });
}

int em_sygv_lh(em_ctx* ctx, int64_t n, const double* L_host, double* L, int64_t ldl, double* R,
               int64_t ldr, double* tau, double* V, int64_t ldv, double* l_n, double* r_n,
               double* VtR, int64_t ldvtr, int flags, int64_t* pivot, int* which) {
  return guarded(ctx, [&] {
    if (flags & ~EM_SYGV_R_WORKSPACE) throw em::ArgError{"unknown em_sygv_lh flags"};
    if (!L_host || !L) throw em::ArgError{"em_sygv_lh: L_host and L are required"};
    cudaStream_t st = ctx->stream;
    // the copy engine takes L after everything already queued on the stream (R's upload)
    cudaStream_t cs = nullptr;
    cudaEvent_t queued = nullptr, l_ready = nullptr;
    EM_CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    EM_CK(cudaEventCreateWithFlags(&queued, cudaEventDisableTiming));
    EM_CK(cudaEventCreateWithFlags(&l_ready, cudaEventDisableTiming));
    struct Cleanup {
      cudaStream_t cs;
      cudaEvent_t a, b;
      ~Cleanup() {
        cudaStreamSynchronize(cs);
        cudaEventDestroy(a);
        cudaEventDestroy(b);
        cudaStreamDestroy(cs);
      }
    } cleanup{cs, queued, l_ready};
    EM_CK(cudaEventRecord(queued, st));
    EM_CK(cudaStreamWaitEvent(cs, queued, 0));
    EM_CK(cudaMemcpy2DAsync(L, (size_t)ldl * 8, L_host, (size_t)n * 8, (size_t)n * 8, (size_t)n,
                            cudaMemcpyHostToDevice, cs));
    EM_CK(cudaEventRecord(l_ready, cs));
    int wh = -1;
    const int64_t p = em::sygv(st, n, L, ldl, R, ldr, tau, V, ldv, l_n, r_n, VtR, ldvtr, &wh,
                               flags, l_ready);
    EM_CK(cudaStreamWaitEvent(st, l_ready, 0));  // (an early R failure returns before L is used)
    if (pivot) *pivot = p;
    if (which) *which = wh;
    return p >= 0 ? EM_ERR_NOT_PD : EM_OK;
  });
}

int em_sygv(em_ctx* ctx, int64_t n, const double* L, int64_t ldl, const double* R, int64_t ldr,
            double* tau, double* V, int64_t ldv, double* l_n, double* r_n, double* VtR,
            int64_t ldvtr, int64_t* pivot, int* which) {
  return em_sygv_ex(ctx, n, L, ldl, const_cast<double*>(R), ldr, tau, V, ldv, l_n, r_n, VtR,
                    ldvtr, 0, pivot, which);
}

int em_sygv_h(em_ctx* ctx, int64_t n, const double* L_h, const double* R_h, double* tau_h,
              double* V_h, double* l_n_h, double* r_n_h, double* VtR_h, int64_t* pivot,
              int* which) {
  return guarded(ctx, [&] {
    cudaStream_t st = ctx->stream;
    const size_t nn = (size_t)n * n;
    em::DBuf L(nn, st), R(nn, st), V(nn, st), t(n, st), ln(n, st), rn(n, st), VtR;
    if (VtR_h) VtR.alloc(nn, st);
    EM_CK(cudaMemcpyAsync(R.p, R_h, nn * 8, cudaMemcpyHostToDevice, st));
    int wh = -1;
    // L is uploaded by em_sygv_lh on a copy engine while R is factored; R is this call's
    // own upload: use it as the factor workspace when it is sparse
    int64_t p = -1;
    const int rc = em_sygv_lh(ctx, n, L_h, L.p, n, R.p, n, t.p, V.p, n, ln.p, rn.p,
                              VtR_h ? VtR.p : nullptr, n, EM_SYGV_R_WORKSPACE, &p, &wh);
    if (rc != EM_OK && rc != EM_ERR_NOT_PD) return rc;  // (ctx->err already set)
    if (pivot) *pivot = p;
    if (which) *which = wh;
    if (p >= 0) return EM_ERR_NOT_PD;
    EM_CK(cudaMemcpyAsync(tau_h, t.p, n * 8, cudaMemcpyDeviceToHost, st));
    if (l_n_h) EM_CK(cudaMemcpyAsync(l_n_h, ln.p, n * 8, cudaMemcpyDeviceToHost, st));
    if (r_n_h) EM_CK(cudaMemcpyAsync(r_n_h, rn.p, n * 8, cudaMemcpyDeviceToHost, st));
    if (V_h) EM_CK(cudaMemcpyAsync(V_h, V.p, nn * 8, cudaMemcpyDeviceToHost, st));
    if (VtR_h) EM_CK(cudaMemcpyAsync(VtR_h, VtR.p, nn * 8, cudaMemcpyDeviceToHost, st));
    EM_CK(cudaStreamSynchronize(st));
    return EM_OK;
  });
}

// ---- TD2 ----------------------------------------------------------------------------

int em_td2_plan_create(em_ctx* ctx, int64_t n, int n_p, int n_s, const double* l_n,
                       const double* r_n, const double* P_r, const double* P_l, const double* P_m,
                       double dt, double theta, em_td2_plan** plan) {
  return guarded(ctx, [&] {
    if (!plan || n < 0 || n_p < 0 || n_s < 0) throw em::ArgError{"bad td2 plan arguments"};
    auto* P = em::td2_new(ctx, n, n_p, n_s, dt, theta);
    try {
      em::td2_plan_init(P, l_n, r_n, P_r, P_l, P_m);
      EM_CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      em::td2_delete(P);
      throw;
    }
    *plan = P;
    return EM_OK;
  });
}

int em_td2_plan_create_exact(em_ctx* ctx, int64_t n, int n_p, int n_s, const double* l_n,
                             const double* r_n, const double* P_r, const double* P_l,
                             const double* P_m, double h, em_td2_plan** plan) {
  return guarded(ctx, [&] {
    if (!plan || n < 0 || n_p < 0 || n_s < 0 || !(h > 0.0))
      throw em::ArgError{"bad exact-integrator plan arguments"};
    auto* P = em::td2_new(ctx, n, n_p, n_s, h, 1.0);
    try {
      em::td2_plan_init_exact(P, l_n, r_n, P_r, P_l, P_m);
      EM_CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      em::td2_delete(P);
      throw;
    }
    *plan = P;
    return EM_OK;
  });
}

void em_td2_plan_destroy(em_td2_plan* plan) { em::td2_delete(plan); }

int em_td2_set_observables(em_td2_plan* plan, int n_obs, const double* CV, int64_t ldcv,
                           const double* D, int64_t ldd) {
  em_ctx* ctx = em::td2_ctx(plan);
  return guarded(ctx, [&] {
    em::td2_set_observables(plan, n_obs, CV, ldcv, D, ldd);
    return EM_OK;
  });
}

int em_td2_run(em_td2_plan* plan, int64_t T, const double* drive, double* q, double* Y,
               int64_t stride, double* Qcap) {
  em_ctx* ctx = em::td2_ctx(plan);
  return guarded(ctx, [&] {
    em::td2_run(plan, T, drive, q, Y, stride, Qcap);
    return EM_OK;
  });
}

int em_td2_run_sweep(em_td2_plan* plan, int64_t T, const double* drive, double* Q, double* Y,
                     int64_t stride) {
  em_ctx* ctx = em::td2_ctx(plan);
  return guarded(ctx, [&] {
    em::td2_run_sweep(plan, T, drive, Q, Y, stride);
    return EM_OK;
  });
}

int em_td2_step(em_td2_plan* plan, double* q, const double* i_d_h, const double* di_d_h,
                const double* di0_h) {
  em_ctx* ctx = em::td2_ctx(plan);
  return guarded(ctx, [&] {
    if (em::td2_is_exact(plan)) throw em::ArgError{"per-step calls need a theta-method plan"};
    em::td2_step_host(plan, q, i_d_h, di_d_h, di0_h);
    return EM_OK;
  });
}

int em_td2_forcing(em_td2_plan* plan, const double* i_d_h, const double* di_d_h,
                   const double* di0_h, double* f) {
  em_ctx* ctx = em::td2_ctx(plan);
  return guarded(ctx, [&] {
    if (em::td2_is_exact(plan)) throw em::ArgError{"per-step calls need a theta-method plan"};
    em::td2_forcing_host(plan, i_d_h, di_d_h, di0_h, f);
    return EM_OK;
  });
}

int em_td2_step_forcing(em_td2_plan* plan, double* q, const double* f) {
  em_ctx* ctx = em::td2_ctx(plan);
  return guarded(ctx, [&] {
    if (em::td2_is_exact(plan)) throw em::ArgError{"per-step calls need a theta-method plan"};
    em::td2_step_forcing(plan, q, f);
    EM_CK(cudaStreamSynchronize(ctx->stream));
    return EM_OK;
  });
}

// ---- TD1 ----------------------------------------------------------------------------

int em_td1_plan_create(em_ctx* ctx, int64_t n, int n_p, int n_s, const double* L, int64_t ldl,
                       const double* R, int64_t ldr, const double* r_d, const double* l_d,
                       const double* m0, double dt, double theta, em_td1_plan** plan,
                       int64_t* pivot) {
  return guarded(ctx, [&] {
    if (!plan || n < 0 || n_p < 0 || n_s < 0) throw em::ArgError{"bad td1 plan arguments"};
    auto* P = em::td1_new(ctx, n, n_p, n_s, dt, theta);
    int64_t piv = -1;
    try {
      piv = em::td1_plan_init(P, L, ldl, R, ldr, r_d, l_d, m0);
      EM_CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      em::td1_delete(P);
      throw;
    }
    if (pivot) *pivot = piv;
    if (piv >= 0) {
      em::td1_delete(P);
      *plan = nullptr;
      return EM_ERR_NOT_PD;
    }
    *plan = P;
    return EM_OK;
  });
}

int em_td1_plan_create_band(em_ctx* ctx, int64_t n, int n_p, int n_s, double* L, int64_t ldl,
                            const double* Rb, int64_t ldrb, int64_t bw, const double* r_d,
                            const double* l_d, const double* m0, double dt, double theta,
                            int flags, em_td1_plan** plan, int64_t* pivot) {
  return guarded(ctx, [&] {
    if (!plan || n < 0 || n_p < 0 || n_s < 0) throw em::ArgError{"bad td1 plan arguments"};
    if (!Rb || bw < 0 || ldrb < bw + 1) throw em::ArgError{"em_td1_plan_create_band: bad band"};
    if (flags & ~EM_TD1_L_WORKSPACE) throw em::ArgError{"unknown em_td1_plan_create_band flags"};
    auto* P = em::td1_new(ctx, n, n_p, n_s, dt, theta);
    int64_t piv = -1;
    try {
      piv = em::td1_plan_init(P, L, ldl, nullptr, 0, r_d, l_d, m0, Rb, ldrb, bw,
                              (flags & EM_TD1_L_WORKSPACE) != 0);
      EM_CK(cudaStreamSynchronize(ctx->stream));
    } catch (...) {
      em::td1_delete(P);
      throw;
    }
    if (pivot) *pivot = piv;
    if (piv >= 0) {
      em::td1_delete(P);
      *plan = nullptr;
      return EM_ERR_NOT_PD;
    }
    *plan = P;
    return EM_OK;
  });
}

void em_td1_plan_destroy(em_td1_plan* plan) { em::td1_delete(plan); }

int em_td1_set_observables(em_td1_plan* plan, int n_obs, const double* C, int64_t ldc,
                           const double* D, int64_t ldd) {
  em_ctx* ctx = em::td1_ctx(plan);
  return guarded(ctx, [&] {
    em::td1_set_observables(plan, n_obs, C, ldc, D, ldd);
    return EM_OK;
  });
}

int em_td1_run(em_td1_plan* plan, int64_t T, const double* drive, double* I, double* Y,
               int64_t stride, double* Icap) {
  em_ctx* ctx = em::td1_ctx(plan);
  return guarded(ctx, [&] {
    em::td1_run(plan, T, drive, I, Y, stride, Icap);
    return EM_OK;
  });
}

int em_td1_step(em_td1_plan* plan, double* I, const double* i_d_h, const double* di_d_h,
                const double* di0_h) {
  em_ctx* ctx = em::td1_ctx(plan);
  return guarded(ctx, [&] {
    em::td1_step_host(plan, I, i_d_h, di_d_h, di0_h);
    return EM_OK;
  });
}

int em_td1_factor(em_td1_plan* plan, double* out, int64_t ldo) {
  em_ctx* ctx = em::td1_ctx(plan);
  return guarded(ctx, [&] {
    em::td1_copy_factor(plan, out, ldo);
    return EM_OK;
  });
}

}  // extern "C"

int em_field_transfer(em_ctx* ctx, int64_t nb, const double* starts, const double* ends,
                      const double* radius, int64_t np, const double* probes, double* T,
                      int64_t* bad) {
  return guarded(ctx, [&] {
    if (nb < 0 || np < 0) throw em::ArgError{"em_field_transfer: negative size"};
    const int64_t b = em::field_transfer(ctx->stream, nb, starts, ends, radius, np, probes, T);
    if (bad) *bad = b;
    return b >= 0 ? EM_ERR_ARG : EM_OK;
  });
}

