/* C caller of the drop-in boundary (include/eddymodes_b200.h): no Python, no torch.
 * Builds a small SPD pencil, solves L v = tau R v on the device, runs the modal
 * theta-method for a ramp drive, and prints the results for tests/test_cabi_c.py. */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "eddymodes_b200.h"

#define CK(x)                                                                 \
  do {                                                                        \
    int rc_ = (x);                                                            \
    if (rc_ != EM_OK) {                                                       \
      fprintf(stderr, "%s failed: %d %s\n", #x, rc_, em_last_error(ctx));     \
      return 1;                                                               \
    }                                                                         \
  } while (0)

int main(void) {
  const int64_t n = 40;
  double *L = malloc(n * n * 8), *R = malloc(n * n * 8);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const double d = fabs((double)(i - j));
      L[i + j * n] = 1.0 / (1.0 + d) + (i == j ? 1.0 : 0.0);   /* SPD (diag dominant) */
      R[i + j * n] = (i == j) ? 2.0 + 0.01 * i : (d == 1.0 ? -0.5 : 0.0);
    }
  em_ctx* ctx = NULL;
  if (em_init(0, &ctx) != EM_OK) {
    fprintf(stderr, "no device\n");
    return 2;
  }
  double *tau = malloc(n * 8), *V = malloc(n * n * 8), *ln = malloc(n * 8), *rn = malloc(n * 8);
  int64_t piv = -1;
  int which = -1;
  CK(em_sygv_h(ctx, n, L, R, tau, V, ln, rn, NULL, &piv, &which));
  /* residual of the first and last mode: || L v - tau R v || */
  double res = 0.0;
  for (int64_t k = 0; k < n; k += n - 1)
    for (int64_t i = 0; i < n; ++i) {
      double lv = 0.0, rv = 0.0;
      for (int64_t j = 0; j < n; ++j) {
        lv += L[i + j * n] * V[j + k * n];
        rv += R[i + j * n] * V[j + k * n];
      }
      res = fmax(res, fabs(lv - tau[k] * rv));
    }
  /* TD2 run from rest: one port, ramp drive, observable = mode coordinates of mode 0 */
  const int64_t T = 200;
  double *dl = NULL, *dr = NULL, *dpr = NULL, *dpl = NULL, *dpm = NULL, *dcv = NULL, *ddrive = NULL,
         *dq = NULL, *dy = NULL;
  cudaMalloc((void**)&dl, n * 8);
  cudaMalloc((void**)&dr, n * 8);
  cudaMalloc((void**)&dpr, n * 8);
  cudaMalloc((void**)&dpl, n * 8);
  cudaMalloc((void**)&dpm, 8);
  cudaMalloc((void**)&dcv, n * 8);
  cudaMalloc((void**)&ddrive, (T + 1) * 8);
  cudaMalloc((void**)&dq, n * 8);
  cudaMalloc((void**)&dy, T * 8);
  double *pr = malloc(n * 8), *cv = calloc(n, 8), *drive = malloc((T + 1) * 8), *y = malloc(T * 8);
  for (int64_t i = 0; i < n; ++i) pr[i] = V[i + 0 * n];  /* P = V^T e_0 */
  cv[0] = 1.0;
  for (int64_t k = 0; k <= T; ++k) drive[k] = fmin(1.0, k / 50.0);
  cudaMemcpy(dl, ln, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dr, rn, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dpr, pr, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dpl, pr, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dcv, cv, n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(ddrive, drive, (T + 1) * 8, cudaMemcpyHostToDevice);
  cudaMemset(dq, 0, n * 8);
  em_td2_plan* plan = NULL;
  CK(em_td2_plan_create(ctx, n, 1, 0, dl, dr, dpr, dpl, dpm, 1e-3, 0.5, &plan));
  CK(em_td2_set_observables(plan, 1, dcv, 1, NULL, 0));
  CK(em_td2_run(plan, T, ddrive, dq, dy, 1, NULL));
  CK(em_synchronize(ctx));
  cudaMemcpy(y, dy, T * 8, cudaMemcpyDeviceToHost);
  /* scalar reference of mode 0 (transient.py:299-308 / _kernels.py:213-222) */
  const double dt = 1e-3, th = 0.5, den = ln[0] + dt * th * rn[0], c = sqrt(den);
  double q = 0.0, err = 0.0;
  for (int64_t k = 0; k < T; ++k) {
    const double id = drive[k], did = drive[k + 1] - drive[k];
    const double f = -dt * pr[0] * id - (pr[0] + dt * th * pr[0]) * did;
    q += ((-dt * rn[0] * q + f) / c) / c;
    err = fmax(err, fabs(q - y[k]) / (fabs(q) + 1e-300));
  }
  /* the two "ranks" of a column-sharded solve (em_sygv_range): modes [0, h) and [h, n)
   * must equal the corresponding columns of the full solve */
  const int64_t h = 17;
  double *dL = NULL, *dR = NULL, *dtau = NULL, *dV = NULL, *dln = NULL, *drn = NULL;
  cudaMalloc((void**)&dL, n * n * 8);
  cudaMalloc((void**)&dR, n * n * 8);
  cudaMalloc((void**)&dtau, n * 8);
  cudaMalloc((void**)&dV, n * n * 8);
  cudaMalloc((void**)&dln, n * 8);
  cudaMalloc((void**)&drn, n * 8);
  cudaMemcpy(dL, L, n * n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dR, R, n * n * 8, cudaMemcpyHostToDevice);
  double shard_err = 0.0, *Vs = malloc(n * n * 8), *lns = malloc(n * 8);
  for (int r = 0; r < 2; ++r) {
    const int64_t lo = r ? h : 0, hi = r ? n : h;
    CK(em_sygv_range(ctx, n, dL, n, dR, n, lo, hi, dtau, dV, n, dln, drn, NULL, n, 0, &piv,
                     &which));
    cudaMemcpy(Vs, dV, n * (hi - lo) * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(lns, dln, (hi - lo) * 8, cudaMemcpyDeviceToHost);
    for (int64_t j = lo; j < hi; ++j) {
      shard_err = fmax(shard_err, fabs(lns[j - lo] - ln[j]) / ln[j]);
      for (int64_t i = 0; i < n; ++i)
        shard_err = fmax(shard_err, fabs(Vs[i + (j - lo) * n] - V[i + j * n]));
    }
  }
  int64_t path = 0;
  CK(em_info(ctx, EM_INFO_EIG_PATH, &path));
  CK(em_trim(ctx));
  printf("n %lld tau0 %.17g taulast %.17g res %.3e td2_relerr %.3e launches %lld "
         "shard_err %.3e path %lld\n",
         (long long)n, tau[0], tau[n - 1], res, err, (long long)em_launch_count(ctx), shard_err,
         (long long)path);
  em_td2_plan_destroy(plan);
  em_finalize(ctx);
  return 0;
}
