// K5/K6/K10 — velocity Verlet halves (driver.py:74-93), the displacement
// guard (neighbor.py:197-206, driver.py:115-125) fused into the drift, and the
// kinetic-energy / momentum reduction for thermo output.
//
// Element-wise and HBM-bound: each thread streams one atom's SoA components;
// products and sums use explicit round-to-nearest ops so the update is
// bitwise the reference's `v += (0.5 dt / m) F; x += dt v`.
#include "tmd_common.cuh"

namespace tmd {

__global__ void __launch_bounds__(256) k_kick_drift(double* __restrict__ pos, double* __restrict__ vel,
                                                    const double* __restrict__ frc, int64_t ld,
                                                    int64_t ld_f, int32_t n, double c, double dt,
                                                    const double* __restrict__ xref, int64_t ld_ref,
                                                    double* dispmax2) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  double d2 = 0.0;
  if (i < n) {
    double p[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      double v = add_rn(vel[q * ld + i], mul_rn(c, frc[q * ld_f + i]));
      vel[q * ld + i] = v;
      p[q] = add_rn(pos[q * ld + i], mul_rn(dt, v));
      pos[q * ld + i] = p[q];
    }
    if (xref)
      d2 = norm2_seq(sub_rn(p[0], xref[i]), sub_rn(p[1], xref[ld_ref + i]),
                     sub_rn(p[2], xref[2 * ld_ref + i]));
  }
  if (xref) {
    double m = warp_max(d2);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(dispmax2, m);
  }
}

__global__ void __launch_bounds__(256) k_kick(double* __restrict__ vel, const double* __restrict__ frc,
                                              int64_t ld, int64_t ld_f, int32_t n, double c) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
#pragma unroll
  for (int q = 0; q < 3; ++q) vel[q * ld + i] = add_rn(vel[q * ld + i], mul_rn(c, frc[q * ld_f + i]));
}

__global__ void __launch_bounds__(256) k_kinetic(const double* __restrict__ vel, int64_t ld, int32_t n,
                                                 double* partials, unsigned int* counter,
                                                 double* out, double mass) {
  double red[4] = {0.0, 0.0, 0.0, 0.0};
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double vx = vel[i], vy = vel[ld + i], vz = vel[2 * ld + i];
    red[0] += vx * vx + vy * vy + vz * vz;
    red[1] += vx;
    red[2] += vy;
    red[3] += vz;
  }
  __shared__ double sm[4 * 32];
  block_sum<4>(red, sm);
  double v[4] = {0.5 * mass * red[0], mass * red[1], mass * red[2], mass * red[3]};
  grid_sum_finish<4>(v, partials, counter, out, false);
}

}  // namespace tmd

using namespace tmd;

extern "C" int tmd_kick_drift(double* d_pos, double* d_vel, const double* d_frc, int64_t ld,
                              int64_t ld_f, int32_t n, double c, double dt, const double* d_xref,
                              int64_t ld_ref, double* d_dispmax2, void* stream) {
  if (n <= 0) return TMD_OK;
  k_kick_drift<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d_pos, d_vel, d_frc, ld, ld_f, n, c,
                                                                dt, d_xref, ld_ref, d_dispmax2);
  TMD_LAUNCH_CHECK("kick_drift");
  return TMD_OK;
}


extern "C" int tmd_kick(double* d_vel, const double* d_frc, int64_t ld, int64_t ld_f, int32_t n,
                        double c, void* stream) {
  if (n <= 0) return TMD_OK;
  k_kick<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d_vel, d_frc, ld, ld_f, n, c);
  TMD_LAUNCH_CHECK("kick");
  return TMD_OK;
}

extern "C" int tmd_kinetic(const double* d_vel, int64_t ld, int32_t n, double mass, double* d_out,
                           void* stream) {
  cudaStream_t s = as_stream(stream);
  if (n <= 0) {
    TMD_CUDA_TRY(cudaMemsetAsync(d_out, 0, 4 * sizeof(double), s), "kinetic");
    return TMD_OK;
  }
  int g = grid_for(n, 256);
  if (g > 2 * sm_count()) g = 2 * sm_count();
  ReduceScratch rs{};
  if (reduce_scratch(&rs, g, 4, s) != TMD_OK) return TMD_ERR_CUDA;
  k_kinetic<<<g, 256, 0, s>>>(d_vel, ld, n, rs.partials, rs.counter, d_out, mass);
  TMD_LAUNCH_CHECK("kinetic");
  return TMD_OK;
}

extern "C" int tmd_zero_rows(double* d, int64_t ld, int32_t rows, int64_t start, int64_t count, void* stream) {
  if (count <= 0) return TMD_OK;
  if (!d || rows < 1 || start < 0 || start + count > ld) return TMD_ERR_ARG;
  for (int32_t q = 0; q < rows; ++q)
    TMD_CUDA_TRY(cudaMemsetAsync(d + q * ld + start, 0, sizeof(double) * (size_t)count, as_stream(stream)),
                 "zero_rows");
  return TMD_OK;
}
