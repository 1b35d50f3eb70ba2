// Force-loop variants on the production (tiered, quad-interleaved) lists.
// V0 = the current tmd_step_lj loop body; later variants trim the FP64 chain
// or change occupancy / unrolling.  Forces only (no integration epilogue).
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double rcp2(double x) {  // seed + 2 Newton steps
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rcp1(double x) {  // seed + 1 Newton step with a cubic correction
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);  // r (1 + e + e^2)
}

template <int V>
__device__ __forceinline__ void pair(double dx, double dy, double dz, bool ok, double rc2, double& fx, double& fy,
                                     double& fz) {
  const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
  if (ok && rsq < rc2) {
    if (V == 0) {
      const double sr2 = rcp2(rsq);
      const double sr6 = sr2 * sr2 * sr2 * 1.0;
      const double f = 48.0 * sr6 * (sr6 - 0.5) * sr2;
      fx = fma(f, dx, fx); fy = fma(f, dy, fy); fz = fma(f, dz, fz);
    } else {
      const double sr2 = rcp1(rsq);
      const double sr6 = sr2 * sr2 * sr2;
      const double f = fma(48.0, sr6, -24.0) * (sr6 * sr2);
      fx = fma(f, dx, fx); fy = fma(f, dy, fy); fz = fma(f, dz, fz);
    }
  }
}

template <int V, int QPI>
__device__ __forceinline__ void body(const double* __restrict__ pos, int64_t ld, const int32_t* __restrict__ nbr,
                                     int64_t ld_nbr, const int32_t* __restrict__ cnts, int32_t n, double rc2,
                                     double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int32_t cnt = cnts[i];
  const int4* row = reinterpret_cast<const int4*>(nbr) + i;
  const int32_t nq = (cnt + 3) >> 2;
  const int4 self4 = make_int4(i, i, i, i);
  double fx = 0, fy = 0, fz = 0;
  if (QPI == 1) {
    int4 a = nq > 0 ? __ldcs(row) : self4;
    int4 b = nq > 1 ? __ldcs(row + ld_nbr) : self4;
    for (int32_t q = 0; q < nq; ++q) {
      const int4 c = (q + 2 < nq) ? __ldcs(row + (int64_t)(q + 2) * ld_nbr) : self4;
      const int32_t jj[4] = {a.x, a.y, a.z, a.w};
      double xj[4], yj[4], zj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        xj[u] = __ldg(pos + jj[u]); yj[u] = __ldg(pos + ld + jj[u]); zj[u] = __ldg(pos + 2 * ld + jj[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) pair<V>(xi - xj[u], yi - yj[u], zi - zj[u], 4 * q + u < cnt, rc2, fx, fy, fz);
      a = b;
      b = c;
    }
  } else {  // two quads per iteration, one quad of lookahead
    int4 a = nq > 0 ? __ldcs(row) : self4;
    int4 b = nq > 1 ? __ldcs(row + ld_nbr) : self4;
    for (int32_t q = 0; q < nq; q += 2) {
      const int4 c = (q + 2 < nq) ? __ldcs(row + (int64_t)(q + 2) * ld_nbr) : self4;
      const int4 d = (q + 3 < nq) ? __ldcs(row + (int64_t)(q + 3) * ld_nbr) : self4;
      const int32_t jj[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      double xj[8], yj[8], zj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xj[u] = __ldg(pos + jj[u]); yj[u] = __ldg(pos + ld + jj[u]); zj[u] = __ldg(pos + 2 * ld + jj[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) pair<V>(xi - xj[u], yi - yj[u], zi - zj[u], 4 * q + u < cnt, rc2, fx, fy, fz);
      a = c;
      b = d;
    }
  }
  out[i] = fx; out[ld + i] = fy; out[2 * ld + i] = fz;
}

// V5: x,y gathered as one 16-byte load from an interleaved (x, y) copy, z from SoA
__global__ void __launch_bounds__(128, 8) k_xy(const double* __restrict__ pos, const double2* __restrict__ xy,
                                              int64_t ld, const int32_t* __restrict__ nbr, int64_t ld_nbr,
                                              const int32_t* __restrict__ cnts, int32_t n, double rc2,
                                              double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int32_t cnt = cnts[i];
  const int4* row = reinterpret_cast<const int4*>(nbr) + i;
  const int32_t nq = (cnt + 3) >> 2;
  const int4 self4 = make_int4(i, i, i, i);
  double fx = 0, fy = 0, fz = 0;
  int4 a = nq > 0 ? __ldcs(row) : self4;
  int4 b = nq > 1 ? __ldcs(row + ld_nbr) : self4;
  for (int32_t q = 0; q < nq; ++q) {
    const int4 c = (q + 2 < nq) ? __ldcs(row + (int64_t)(q + 2) * ld_nbr) : self4;
    const int32_t jj[4] = {a.x, a.y, a.z, a.w};
    double2 pj[4];
    double zj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      pj[u] = __ldg(xy + jj[u]);
      zj[u] = __ldg(pos + 2 * ld + jj[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) pair<0>(xi - pj[u].x, yi - pj[u].y, zi - zj[u], 4 * q + u < cnt, rc2, fx, fy, fz);
    a = b;
    b = c;
  }
  out[i] = fx; out[ld + i] = fy; out[2 * ld + i] = fz;
}

template <int V, int QPI>
__global__ void __launch_bounds__(128) k_plain(const double* __restrict__ pos, int64_t ld, const int32_t* __restrict__ nbr,
                                               int64_t ld_nbr, const int32_t* __restrict__ cnts, int32_t n,
                                               double rc2, double* __restrict__ out) {
  body<V, QPI>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out);
}

template <int V, int QPI>
__global__ void __launch_bounds__(128, 8) k_occ(const double* __restrict__ pos, int64_t ld, const int32_t* __restrict__ nbr,
                                                int64_t ld_nbr, const int32_t* __restrict__ cnts, int32_t n,
                                                double rc2, double* __restrict__ out) {
  body<V, QPI>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out);
}

extern "C" int exp_force(int variant, const double* pos, int64_t ld, const int32_t* nbr, int64_t ld_nbr,
                         const int32_t* cnts, int32_t n, double rc2, double* out, void* s, const double* aux) {
  const dim3 g((n + 127) / 128), b(128);
  cudaStream_t st = (cudaStream_t)s;
  switch (variant) {
    case 0: k_plain<0, 1><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 1: k_plain<1, 1><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 2: k_occ<1, 1><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 3: k_plain<1, 2><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 4: k_occ<1, 2><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 5: k_xy<<<g, b, 0, st>>>(pos, reinterpret_cast<const double2*>(aux), ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 6: k_occ<0, 1><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}
