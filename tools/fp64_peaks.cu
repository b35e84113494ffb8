// Measurement tool (not product code): FP64 peaks on the B200 box.
//  1. DMMA.8x8x4 issue-rate peak, 2. DFMA peak, 3. cuBLAS DGEMM (comparator only),
//  4. the in-tree DMMA GEMM at the same sizes + correctness against cuBLAS.
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <math.h>
#include <vector>
#include "../paper_2407_11993_b200/csrc/common.cuh"
#include "../paper_2407_11993_b200/csrc/gemm.h"

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

int em_num_sms() { int d, n; cudaGetDevice(&d); cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d); return n; }

__global__ void dmma_peak(double* out, int iters) {
  double c[8][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) em::dmma884(c[i][0], c[i][1], a, b);
  }
  double s = 0; for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}
__global__ void dfma_peak(double* out, int iters) {
  double c[16];
  double a = threadIdx.x * 1e-3, b = 1.0 - blockIdx.x * 1e-9;
  for (int i = 0; i < 16; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0; for (int i = 0; i < 16; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

__global__ void fill(double* p, size_t n, unsigned seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned x = (unsigned)(i * 2654435761u) ^ seed; x ^= x >> 13; x *= 0x5bd1e995; x ^= x >> 15;
    p[i] = (x & 0xffffff) / 16777216.0 - 0.5;
  }
}

int main(int argc, char** argv) {
  int sms = em_num_sms();
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int iters = 20000;
  for (int w : {4, 8, 16}) {
    dmma_peak<<<sms * 2, 32 * w>>>(d, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dmma_peak<<<sms * 2, 32 * w>>>(d, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * 8.0 * iters * (sms * 2.0 * w);
    printf("{\"probe\":\"dmma884_peak\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", w, fl / ms / 1e9);
  }
  for (int w : {8, 16}) {
    dfma_peak<<<sms * 2, 32 * w>>>(d, 100); CK(cudaDeviceSynchronize());
    cudaEventRecord(e0); dfma_peak<<<sms * 2, 32 * w>>>(d, iters); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 16 * iters * 32.0 * w * sms * 2;
    printf("{\"probe\":\"dfma_peak\",\"warps_per_cta\":%d,\"tflops\":%.2f}\n", w, fl / ms / 1e9);
  }

  cublasHandle_t h; cublasCreate(&h);
  for (int n : {2048, 4096, 8192, 16384}) {
    size_t nn = (size_t)n * n;
    double *A, *B, *C, *C2;
    CK(cudaMalloc(&A, nn * 8)); CK(cudaMalloc(&B, nn * 8)); CK(cudaMalloc(&C, nn * 8)); CK(cudaMalloc(&C2, nn * 8));
    fill<<<1024, 256>>>(A, nn, 1); fill<<<1024, 256>>>(B, nn, 2);
    double one = 1, zero = 0;
    int reps = n >= 16384 ? 2 : 5;
    for (int variant = 0; variant < 2; ++variant) {
      for (int r = 0; r < 2; ++r) {
        if (variant == 0) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
        else em::gemm(0, false, false, n, n, n, 1.0, A, n, B, n, 0.0, C2, n);
      }
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      for (int r = 0; r < reps; ++r) {
        if (variant == 0) cublasDgemm(h, CUBLAS_OP_N, CUBLAS_OP_N, n, n, n, &one, A, n, B, n, &zero, C, n);
        else em::gemm(0, false, false, n, n, n, 1.0, A, n, B, n, 0.0, C2, n);
      }
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"probe\":\"%s\",\"n\":%d,\"tflops\":%.2f}\n", variant == 0 ? "cublas_dgemm_nn" : "em_dgemm_nn", n,
             2.0 * n * (double)n * n * reps / ms / 1e9);
    }
    if (n <= 4096) {
      std::vector<double> h1(nn), h2(nn);
      cudaMemcpy(h1.data(), C, nn * 8, cudaMemcpyDeviceToHost); cudaMemcpy(h2.data(), C2, nn * 8, cudaMemcpyDeviceToHost);
      double md = 0, mx = 0; for (size_t i = 0; i < nn; ++i) { md = fmax(md, fabs(h1[i] - h2[i])); mx = fmax(mx, fabs(h1[i])); }
      printf("{\"check\":\"nn\",\"n\":%d,\"max_abs_diff\":%.3e,\"max_abs\":%.3e}\n", n, md, mx);
    }
    cudaFree(A); cudaFree(B); cudaFree(C); cudaFree(C2);
  }
  // odd shapes / transposes / lower mode vs cuBLAS
  {
    int m = 1000, n = 777, k = 333, ld = 1001;
    size_t sz = (size_t)ld * 1001;
    double *A, *B, *C, *C2;
    CK(cudaMalloc(&A, sz * 8)); CK(cudaMalloc(&B, sz * 8)); CK(cudaMalloc(&C, sz * 8)); CK(cudaMalloc(&C2, sz * 8));
    fill<<<512, 256>>>(A, sz, 3); fill<<<512, 256>>>(B, sz, 4); fill<<<512, 256>>>(C, sz, 5);
    for (int ta = 0; ta < 2; ++ta) for (int tb = 0; tb < 2; ++tb) for (int off = 0; off < 2; ++off) {
      fill<<<512, 256>>>(C, sz, 5); fill<<<512, 256>>>(C2, sz, 5);
      double al = 0.75, be = -0.5;
      const double* Ao = A + off; const double* Bo = B + off;  // odd offsets → 8-byte path
      cublasDgemm(h, ta ? CUBLAS_OP_T : CUBLAS_OP_N, tb ? CUBLAS_OP_T : CUBLAS_OP_N, m, n, k, &al, Ao, ld, Bo, ld, &be, C, ld);
      em::gemm(0, ta, tb, m, n, k, al, Ao, ld, Bo, ld, be, C2, ld);
      CK(cudaDeviceSynchronize());
      std::vector<double> h1(sz), h2(sz);
      cudaMemcpy(h1.data(), C, sz * 8, cudaMemcpyDeviceToHost); cudaMemcpy(h2.data(), C2, sz * 8, cudaMemcpyDeviceToHost);
      double md = 0; for (size_t i = 0; i < sz; ++i) md = fmax(md, fabs(h1[i] - h2[i]));
      printf("{\"check\":\"ta%d_tb%d_off%d\",\"max_abs_diff\":%.3e}\n", ta, tb, off, md);
    }
  }
  printf("{\"done\":1}\n");
  return 0;
}
