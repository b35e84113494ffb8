// Probe observers: the Biot-Savart transfer from branch currents to the
// magnetic field at probe points — the reference's assembly.field_transfer
// (pkg/src/eddymodes/assembly.py:350-386), exact for finite straight segments — as one
// elementwise kernel over (probe, branch) pairs. run_transient's probe fields
// (transient.py:266-273, 302-305) then become observables of the modal scan.
#include "common.cuh"
#include "ctx.h"
#include "linalg.h"

namespace em {

// T[(p*3 + c)*nb + j] = B_c at probe p per unit current in branch j; *bad = the smallest
// p*nb + j with the probe within branch j's wire radius of its segment (else untouched)
__global__ void field_transfer_kernel(int64_t nb, const double* __restrict__ A,
                                      const double* __restrict__ B,
                                      const double* __restrict__ radius, int64_t np,
                                      const double* __restrict__ P, double* __restrict__ T,
                                      unsigned long long* bad) {
  const int64_t total = np * nb;
  const double mu0 = 4e-7 * 3.141592653589793;
  const double k = mu0 / (4.0 * 3.141592653589793);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = i / nb, j = i % nb;
    const double ax = A[3 * j], ay = A[3 * j + 1], az = A[3 * j + 2];
    const double ux = B[3 * j] - ax, uy = B[3 * j + 1] - ay, uz = B[3 * j + 2] - az;
    const double lu = sqrt(ux * ux + uy * uy + uz * uz);
    const double tx = ux / lu, ty = uy / lu, tz = uz / lu;
    const double px = P[3 * p], py = P[3 * p + 1], pz = P[3 * p + 2];
    const double r1x = px - ax, r1y = py - ay, r1z = pz - az;
    const double r2x = px - B[3 * j], r2y = py - B[3 * j + 1], r2z = pz - B[3 * j + 2];
    const double n1 = sqrt(r1x * r1x + r1y * r1y + r1z * r1z);
    const double n2 = sqrt(r2x * r2x + r2y * r2y + r2z * r2z);
    const double cx = ty * r1z - tz * r1y, cy = tz * r1x - tx * r1z, cz = tx * r1y - ty * r1x;
    const double d2 = cx * cx + cy * cy + cz * cz;
    const double t1 = tx * r1x + ty * r1y + tz * r1z;
    const double t2 = tx * r2x + ty * r2y + tz * r2z;
    const double dseg = t1 < 0.0 ? n1 : (t2 > 0.0 ? n2 : sqrt(fmax(d2, 0.0)));
    if (dseg <= radius[j]) atomicMin(bad, (unsigned long long)i);
    double coef = k * (t1 / n1 - t2 / n2) / d2;
    if (d2 < 1e-14 * lu * lu) coef = 0.0;  // on the axis outside the segment: exactly zero
    T[(p * 3 + 0) * nb + j] = coef * cx;
    T[(p * 3 + 1) * nb + j] = coef * cy;
    T[(p * 3 + 2) * nb + j] = coef * cz;
  }
}

// Returns -1, or the first too-close pair p*nb + j.
int64_t field_transfer(cudaStream_t st, int64_t nb, const double* A, const double* B,
                       const double* radius, int64_t np, const double* P, double* T) {
  if (nb <= 0 || np <= 0) return -1;
  DArr<unsigned long long> bad(1, st);
  EM_CK(cudaMemsetAsync(bad.p, 0xff, sizeof(unsigned long long), st));
  const int64_t total = np * nb;
  const unsigned grid = (unsigned)imin64((total + 255) / 256, 148 * 32);
  field_transfer_kernel<<<grid, 256, 0, st>>>(nb, A, B, radius, np, P, T, bad.p);
  EM_LAUNCHED();
  unsigned long long h = ~0ull;
  EM_CK(cudaMemcpyAsync(&h, bad.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  EM_CK(cudaStreamSynchronize(st));
  return h == ~0ull ? -1 : (int64_t)h;
}

}  // namespace em
