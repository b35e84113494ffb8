// Shared device helpers for the eddymodes B200 kernels (sm_100a, FP64).
//
// FP64 tensor math on sm_100a is warp-level DMMA: tcgen05 has no f64 kind, so
// every dense contraction below issues `mma.sync.aligned.m8n8k4 ... f64`
// (SASS DMMA.8x8x4) on shared-memory tiles staged with cp.async.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define EM_DEVINL __device__ __forceinline__

namespace em {

// D(8x8) += A(8x4, row) * B(4x8, col), FP64.
// Fragment ownership (lane l, g = l>>2, t = l&3):
//   A: A[g][t]     B: B[t][g]     C: C[g][2t], C[g][2t+1]
EM_DEVINL void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

EM_DEVINL uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// cp.async with zero fill when `valid` is false (src-size 0).
EM_DEVINL void cp_async8(void* smem, const void* gmem, bool valid) {
  uint32_t s = smem_u32(smem);
  int n = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
EM_DEVINL void cp_async16(void* smem, const void* gmem, int valid_bytes) {
  uint32_t s = smem_u32(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem),
               "r"(valid_bytes));
}
EM_DEVINL void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
EM_DEVINL void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }

// Programmatic dependent launch (kernels launched with launch_pdl): code before
// pdl_wait() may only read data written before the PREVIOUS kernel started (the
// predecessor of the predecessor has completed once this grid is running, because
// every kernel in such a chain calls pdl_wait() before pdl_trigger()). No-ops for a
// normal launch.
EM_DEVINL void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
EM_DEVINL void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// 0 for every double an arithmetic instruction can produce (results are never signalling
// NaNs: high word 0x7ff00001 has the quiet bit clear), but data-dependent on x: OR-ing it
// over a set of accumulators and adding the result to an address makes the instruction
// using that address wait for all of them (used to order mbarrier releases and async
// copies behind the DMMAs that consumed a shared-memory stage).
EM_DEVINL unsigned never_set(double x) {
  return __double2hiint(x) == 0x7ff00001 ? 8u : 0u;
}

EM_DEVINL double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace em

// Number of SMs on the current device (cached per process).
int em_num_sms();
