// Measurement tool (not product code): DMMA.8x8x4 throughput as a function of the number
// of independent accumulator chains per warp and warps per SM sub-partition (one CTA per
// SM) — how much instruction-level parallelism a warp needs to keep the FP64 tensor pipe
// busy. Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/dmma_latency.cu
#include <cuda_runtime.h>
#include <stdio.h>
#include "../paper_2407_11993_b200/csrc/common.cuh"

int em_num_sms() { int d, n; cudaGetDevice(&d); cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d); return n; }

template <int NACC>
__global__ void chains(double* out, int iters) {
  double c[NACC][2];
  double a = threadIdx.x * 1e-3, b = 1.0 + blockIdx.x * 1e-6;
#pragma unroll
  for (int i = 0; i < NACC; ++i) c[i][0] = c[i][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16 / NACC; ++r)
#pragma unroll
      for (int i = 0; i < NACC; ++i) em::dmma884(c[i][0], c[i][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NACC; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int NACC>
void run(double* d, int sms) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4000;
  for (int w : {4, 8, 12, 16}) {
    chains<NACC><<<sms, 32 * w>>>(d, 10); cudaDeviceSynchronize();
    cudaEventRecord(e0); chains<NACC><<<sms, 32 * w>>>(d, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 512.0 * 16 * iters * (double)sms * w;
    printf("{\"probe\":\"dmma_chains\",\"acc_per_warp\":%d,\"warps_per_smsp\":%d,\"tflops\":%.2f}\n", NACC, w / 4, fl / ms / 1e9);
  }
}

int main() {
  const int sms = em_num_sms();
  double* d; cudaMalloc(&d, 8);
  run<1>(d, sms); run<2>(d, sms); run<4>(d, sms); run<8>(d, sms); run<16>(d, sms);
  return 0;
}
