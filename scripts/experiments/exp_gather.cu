// Micro-experiment: LJ force loop over the production (tiered, quad) lists with
// (a) SoA positions, three 64-bit gathers per candidate (current kernel), vs
// (b) AoS4 positions (x, y, z, pad), one 256-bit gather per candidate.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

template <bool AOS>
__global__ void __launch_bounds__(128) k_lj(const double* __restrict__ pos, int64_t ld,
                                            const int32_t* __restrict__ nbr, int64_t ld_nbr,
                                            const int32_t* __restrict__ cnts, int32_t n, double rc2,
                                            double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double xi, yi, zi, wi;
  if (AOS) ld256(pos + 4 * (int64_t)i, xi, yi, zi, wi);
  else { xi = pos[i]; yi = pos[ld + i]; zi = pos[2 * ld + i]; }
  const int32_t cnt = cnts[i];
  const int4* row = reinterpret_cast<const int4*>(nbr) + i;
  const int32_t nq = (cnt + 3) >> 2;
  const int4 self4 = make_int4(i, i, i, i);
  int4 a = nq > 0 ? __ldcs(row) : self4;
  int4 b = nq > 1 ? __ldcs(row + ld_nbr) : self4;
  double fx = 0, fy = 0, fz = 0;
  for (int32_t q = 0; q < nq; ++q) {
    const int4 c = (q + 2 < nq) ? __ldcs(row + (int64_t)(q + 2) * ld_nbr) : self4;
    const int32_t jj[4] = {a.x, a.y, a.z, a.w};
    double xj[4], yj[4], zj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (AOS) {
        double w;
        ld256(pos + 4 * (int64_t)jj[u], xj[u], yj[u], zj[u], w);
      } else {
        xj[u] = __ldg(pos + jj[u]);
        yj[u] = __ldg(pos + ld + jj[u]);
        zj[u] = __ldg(pos + 2 * ld + jj[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double dx = xi - xj[u], dy = yi - yj[u], dz = zi - zj[u];
      const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
      if (4 * q + u < cnt && rsq < rc2) {
        const double sr2 = rcp_fast(rsq);
        const double sr6 = sr2 * sr2 * sr2;
        const double f = 48.0 * sr6 * (sr6 - 0.5) * sr2;
        fx = fma(f, dx, fx); fy = fma(f, dy, fy); fz = fma(f, dz, fz);
      }
    }
    a = b;
    b = c;
  }
  out[i] = fx; out[ld + i] = fy; out[2 * ld + i] = fz;
}

__global__ void k_to_aos(const double* __restrict__ pos, int64_t ld, int32_t n, double* __restrict__ aos) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  aos[4 * (int64_t)i] = pos[i]; aos[4 * (int64_t)i + 1] = pos[ld + i]; aos[4 * (int64_t)i + 2] = pos[2 * ld + i];
  aos[4 * (int64_t)i + 3] = 0.0;
}

extern "C" int exp_to_aos(const double* pos, int64_t ld, int32_t n, double* aos, void* s) {
  k_to_aos<<<(n + 255) / 256, 256, 0, (cudaStream_t)s>>>(pos, ld, n, aos);
  return (int)cudaGetLastError();
}

extern "C" int exp_lj(int aos, const double* pos, int64_t ld, const int32_t* nbr, int64_t ld_nbr,
                      const int32_t* cnts, int32_t n, double rc2, double* out, void* s) {
  if (aos) k_lj<true><<<(n + 127) / 128, 128, 0, (cudaStream_t)s>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out);
  else k_lj<false><<<(n + 127) / 128, 128, 0, (cudaStream_t)s>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out);
  return (int)cudaGetLastError();
}
