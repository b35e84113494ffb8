// Read-bandwidth ceiling probe for the symv (measurement tool, not product).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bw_probe tools/bw_probe.cu
// (a) flat streaming read of 1 GiB (16-byte loads, 8 in flight per thread)
// (b) 64x64-tile strip read of the lower triangle of a 16384^2 column-major matrix
//     (the symv access pattern: 512-byte column segments, stride lda)
#include <cstdio>
#include <cuda_runtime.h>

__global__ void flat_read(const double2* __restrict__ p, size_t n2, double* out) {
  double s = 0.0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 7 * stride < n2; i += 8 * stride) {
    double2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = p[i + k * stride];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
  }
  for (; i < n2; i += stride) s += p[i].x + p[i].y;
  if (s == 12345.678) *out = s;
}

// tiles of the lower triangle, strip-major, equal ranges per CTA; D tiles of prefetch
template <int D>
__global__ void __launch_bounds__(256) tile_read(const double* __restrict__ A, long lda, long nb,
                                                 long T, long len, double* out) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const long t0 = blockIdx.x * len, t1 = min(T, t0 + len);
  double s = 0.0;
  for (long t = t0; t < t1; t += D) {
    double a[D][16];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      long tt = t + d;
      if (tt >= t1) tt = t1 - 1;
      long i = (long)((sqrt(8.0 * (double)tt + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > tt) --i;
      while ((i + 1) * (i + 2) / 2 <= tt) ++i;
      const long j = tt - i * (i + 1) / 2;
#pragma unroll
      for (int cc = 0; cc < 8; ++cc)
#pragma unroll
        for (int h = 0; h < 2; ++h) a[d][cc * 2 + h] = A[(i * 64 + lane + 32 * h) + (j * 64 + 8 * w + cc) * lda];
    }
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int k = 0; k < 16; ++k) s += a[d][k];
  }
  if (s == 12345.678) *out = s;
}

int main() {
  const long n = 16384;
  double* A;
  double* out;
  cudaMalloc(&A, n * n * sizeof(double));
  cudaMalloc(&out, sizeof(double));
  cudaMemset(A, 0, n * n * sizeof(double));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    for (int per : {2, 4, 8}) {
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) flat_read<<<sms * per, 256>>>((const double2*)A, n * n / 2, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"probe\": \"flat_read\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", per,
             10.0 * n * n * 8 / (ms * 1e-3) / 1e9);
    }
    const long nb = n / 64, T = nb * (nb + 1) / 2;
    for (int per : {1, 2}) {
      const long P = sms * per, len = (T + P - 1) / P;
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) tile_read<1><<<P, 256>>>(A, n, nb, T, len, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"probe\": \"tile_read_D1\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", per,
             10.0 * T * 64 * 64 * 8 / (ms * 1e-3) / 1e9);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) tile_read<2><<<P, 256>>>(A, n, nb, T, len, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"probe\": \"tile_read_D2\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", per,
             10.0 * T * 64 * 64 * 8 / (ms * 1e-3) / 1e9);
      cudaEventRecord(e0);
      for (int r = 0; r < 10; ++r) tile_read<4><<<P, 256>>>(A, n, nb, T, len, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("{\"probe\": \"tile_read_D4\", \"ctas_per_sm\": %d, \"GBps\": %.1f}\n", per,
             10.0 * T * 64 * 64 * 8 / (ms * 1e-3) / 1e9);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
