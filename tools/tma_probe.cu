// TMA box-shape probe for the symv (measurement tool, not product): one persistent CTA per
// SM streams an equal share of the 64 KB boxes covering the lower triangle of a 16384^2
// column-major FP64 matrix through a 3-stage mbarrier ring (the symv_tma.cu pattern; 16
// warps read every element once from shared memory). Box shapes: rows x cols = 128x64
// (the symv's), 256x32, 64x128 (64 KB) and 128x32, 256x16 (32 KB).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o tools/tma_probe \
//        tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

constexpr int NST = 3, TT = 512;

__device__ __forceinline__ unsigned su32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mb_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void mb_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, unsigned ph) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra W_%=;\n}\n" ::"r"(su32(b)),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void tma2d(void* dst, const CUtensorMap* m, int c0, int c1, uint64_t* b) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(dst)),
      "l"(m), "r"(c0), "r"(c1), "r"(su32(b))
      : "memory");
}

__global__ void __launch_bounds__(TT, 1) probe(const __grid_constant__ CUtensorMap map,
                                               const int2* __restrict__ tiles, long T, long len,
                                               int R, int C, double* out) {
  extern __shared__ __align__(128) double ring[];
  __shared__ uint64_t full[NST], empty[NST];
  const int tid = threadIdx.x;
  const long t0 = blockIdx.x * len, t1 = min(T, t0 + len);
  if (t0 >= t1) return;
  if (tid == 0) {
    for (int s = 0; s < NST; ++s) {
      mb_init(&full[s], 1);
      mb_init(&empty[s], TT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const unsigned bytes = (unsigned)(R * C * 8);
  const int elems = R * C;
  if (tid == 0)
    for (int s = 0; s < NST - 1 && t0 + s < t1; ++s) {
      mb_tx(&full[s], bytes);
      const int2 rc = tiles[t0 + s];
      tma2d(ring + (size_t)s * elems, &map, rc.x * R, rc.y * C, &full[s]);
    }
  double acc = 0.0;
  for (long t = t0; t < t1; ++t) {
    const long k = t - t0;
    const int s = (int)(k % NST);
    if (tid == 0 && t + NST - 1 < t1) {
      const long kp = k + NST - 1;
      const int ps = (int)(kp % NST);
      if (kp >= NST) mb_wait(&empty[ps], (unsigned)((kp / NST - 1) & 1));
      mb_tx(&full[ps], bytes);
      const int2 rc = tiles[t + NST - 1];
      tma2d(ring + (size_t)ps * elems, &map, rc.x * R, rc.y * C, &full[ps]);
    }
    mb_wait(&full[s], (unsigned)((k / NST) & 1));
    const double2* S = reinterpret_cast<const double2*>(ring + (size_t)s * elems);
    for (int i = tid; i < elems / 2; i += TT) {
      const double2 v = S[i];
      acc += v.x + v.y;
    }
    __syncwarp();
    if ((tid & 31) == 0) mb_arrive(&empty[s]);
  }
  if (acc == 12345.678) *out = acc;
}

int main() {
  const long n = 16384;
  double* A;
  cudaMalloc(&A, n * n * 8);
  cudaMemset(A, 0, n * n * 8);
  double* out;
  cudaMalloc(&out, 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  const int shapes[][2] = {{128, 64}, {256, 32}, {64, 128}, {128, 32}, {256, 16}};
  for (auto& sh : shapes) {
    const int R = sh[0], C = sh[1];
    // boxes covering the lower triangle: row block i has column blocks j with j*C < (i+1)*R
    std::vector<int2> tl;
    for (int i = 0; i < n / R; ++i)
      for (int j = 0; j * C < (i + 1) * R && j < n / C; ++j) tl.push_back(make_int2(i, j));
    int2* dt;
    cudaMalloc(&dt, tl.size() * sizeof(int2));
    cudaMemcpy(dt, tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)n};
    cuuint64_t strides[1] = {(cuuint64_t)n * 8};
    cuuint32_t box[2] = {(cuuint32_t)R, (cuuint32_t)C};
    cuuint32_t es[2] = {1, 1};
    if (R > 256 || C > 256) {  // TMA box dimensions are limited to 256
      printf("{\"box\": \"%dx%d\", \"skipped\": \"box dimension > 256\"}\n", R, C);
      continue;
    }
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("{\"box\": \"%dx%d\", \"error\": %d}\n", R, C, (int)r);
      continue;
    }
    const long T = (long)tl.size();
    const long len = (T + sms - 1) / sms;
    const size_t smem = (size_t)NST * R * C * 8;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    probe<<<sms, TT, smem>>>(map, dt, T, len, R, C, out);
    cudaEventRecord(e0);
    const int reps = 10;
    for (int k = 0; k < reps; ++k) probe<<<sms, TT, smem>>>(map, dt, T, len, R, C, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double byts = (double)T * R * C * 8;
    printf("{\"box\": \"%dx%d\", \"tiles\": %ld, \"GBps\": %.1f, \"err\": \"%s\"}\n", R, C, T,
           byts / (ms / reps * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    cudaFree(dt);
  }
  return 0;
}
