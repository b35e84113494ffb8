// Device generator for the synthetic plates of BASELINE.json (see synth.py for
// the definition): dense L_ij = 1e-7 (a_i.a_j)/(|x_i-x_j| + h/2),
// dense-stored R = rho*K7 + 1e-3*I, and the electrode-path port columns
// L_D[i] = 1e-7 (a_i.x) sum_j s/(r_ij + h/2), R_D = (rho K7)((a.x) o s).
// Elementwise / HBM-bound; used so the N >= 16k configurations do not spend
// minutes in host numpy before the benchmark starts.
#include "common.cuh"
#include "ctx.h"

namespace em {

struct PlateGeom {
  int64_t nx, ny, nz;
  double h, rho, shift;
};

EM_DEVINL void voxel_xyz(const PlateGeom& g, int64_t vid, double& x, double& y, double& z,
                         int64_t& ix, int64_t& iy, int64_t& iz) {
  iz = vid % g.nz;
  iy = (vid / g.nz) % g.ny;
  ix = vid / (g.nz * g.ny);
  x = (ix + 0.5) * g.h;
  y = (iy + 0.5) * g.h;
  z = (iz + 0.5) * g.h;
}

__global__ void synth_lr_kernel(PlateGeom g, int64_t n, const int64_t* __restrict__ keep,
                                const double* __restrict__ ang, double* __restrict__ L,
                                int64_t ldl, double* __restrict__ R, int64_t ldr) {
  for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {  // column
  int64_t jx, jy, jz;
  double xj, yj, zj;
  voxel_xyz(g, keep[j], xj, yj, zj, jx, jy, jz);
  double sj, cj;
  sincos(ang[j], &sj, &cj);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t ix, iy, iz;
    double xi, yi, zi;
    voxel_xyz(g, keep[i], xi, yi, zi, ix, iy, iz);
    double si, ci;
    sincos(ang[i], &si, &ci);
    const double dx = xi - xj, dy = yi - yj, dz = zi - zj;
    const double d = sqrt(dx * dx + dy * dy + dz * dz);
    const double dot = ci * cj + si * sj;
    if (L) L[i + j * ldl] = 1e-7 * dot / (d + 0.5 * g.h);
    if (R) {
      double r = 0.0;
      if (i == j) {
        r = g.rho * 6.0 + g.shift;
      } else {
        const int64_t m = llabs(ix - jx) + llabs(iy - jy) + llabs(iz - jz);
        if (m == 1) r = -g.rho;
      }
      R[i + j * ldr] = r;
    }
  }
  }
}

// one warp per row i: l_d[i] = 1e-7 (a_i.x) sum_j s/(r_ij + h/2); r_d from the 7-point stencil
__global__ void synth_port_kernel(PlateGeom g, int64_t n, const int64_t* __restrict__ keep,
                                  const double* __restrict__ ang, const int64_t* __restrict__ pos,
                                  double s, double* __restrict__ l_d, double* __restrict__ r_d) {
  const int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  int64_t ix, iy, iz;
  double xi, yi, zi;
  voxel_xyz(g, keep[i], xi, yi, zi, ix, iy, iz);
  double acc = 0.0;
  for (int64_t j = lane; j < n; j += 32) {
    int64_t jx, jy, jz;
    double xj, yj, zj;
    voxel_xyz(g, keep[j], xj, yj, zj, jx, jy, jz);
    const double dx = xi - xj, dy = yi - yj, dz = zi - zj;
    acc += s / (sqrt(dx * dx + dy * dy + dz * dz) + 0.5 * g.h);
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    const double axi = cos(ang[i]);
    l_d[i] = 1e-7 * axi * acc;
    // (rho K7)(a.x o s): 6 rho a_i.x s - rho sum_{face neighbours} a_j.x s
    double r = 6.0 * g.rho * axi * s;
    const int64_t d3[6][3] = {{1, 0, 0}, {-1, 0, 0}, {0, 1, 0}, {0, -1, 0}, {0, 0, 1}, {0, 0, -1}};
    for (int k = 0; k < 6; ++k) {
      const int64_t jx = ix + d3[k][0], jy = iy + d3[k][1], jz = iz + d3[k][2];
      if (jx < 0 || jy < 0 || jz < 0 || jx >= g.nx || jy >= g.ny || jz >= g.nz) continue;
      const int64_t p = pos[(jx * g.ny + jy) * g.nz + jz];
      if (p < 0) continue;
      r -= g.rho * cos(ang[p]) * s;
    }
    r_d[i] = r;
  }
}

}  // namespace em

extern "C" int em_synth_plate(em_ctx* ctx, int64_t nx, int64_t ny, int64_t nz, double h,
                              double rho, double shift, int64_t n, const int64_t* keep,
                              const int64_t* pos, const double* ang, double* L, int64_t ldl,
                              double* R, int64_t ldr, double* l_d, double* r_d) {
  try {
    cudaSetDevice(ctx->device);
    em::PlateGeom g{nx, ny, nz, h, rho, shift};
    cudaStream_t st = ctx->stream;
    if (L || R) {
      dim3 grid((unsigned)em::imax64(1, em::imin64((n + 255) / 256, 32)),
                (unsigned)em::imin64(n, 65535));
      em::synth_lr_kernel<<<grid, 256, 0, st>>>(g, n, keep, ang, L, ldl, R, ldr);
      EM_LAUNCHED();
    }
    if (l_d && r_d) {
      const double s = 1.0 / (double)(ny * nz);
      em::synth_port_kernel<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(g, n, keep, ang, pos, s, l_d,
                                                                     r_d);
      EM_LAUNCHED();
    }
    EM_CK(cudaStreamSynchronize(st));
    return EM_OK;
  } catch (const em::CudaError& e) {
    ctx->err = std::string(cudaGetErrorString(e.code)) + " in " + e.where;
    return EM_ERR_CUDA;
  }
}
