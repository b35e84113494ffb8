// Plan lifetime helpers shared by the C ABI (definitions in td1.cu / td2.cu).
#pragma once
#include <stdint.h>

#include "ctx.h"

namespace em {
em_td2_plan* td2_new(em_ctx* ctx, int64_t n, int n_p, int n_s, double dt, double theta);
void td2_delete(em_td2_plan* p);
em_ctx* td2_ctx(em_td2_plan* p);
void td2_step_host(em_td2_plan* p, double* q, const double* i_d, const double* di_d,
                   const double* di0);

void td2_forcing_host(em_td2_plan* p, const double* i_d, const double* di_d, const double* di0,
                      double* f);
void td2_step_forcing(em_td2_plan* p, double* q, const double* f);

em_td1_plan* td1_new(em_ctx* ctx, int64_t n, int n_p, int n_s, double dt, double theta);
void td1_delete(em_td1_plan* p);
em_ctx* td1_ctx(em_td1_plan* p);
void td1_copy_factor(em_td1_plan* p, double* out, int64_t ldo);
void td1_step_host(em_td1_plan* p, double* I, const double* i_d, const double* di_d,
                   const double* di0);

// out columns j = in column (n-1-j), w_out[j] = w_in[n-1-j]
void reverse_columns(cudaStream_t st, int64_t m, int64_t n, const double* A, int64_t lda,
                     const double* w_in, double* B, int64_t ldb, double* w_out);
}  // namespace em
