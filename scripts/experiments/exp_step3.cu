// FP64-trimmed variants of the production force loop (front segment only):
//   V0  production arithmetic (rcp seed + 2 Newton, sr6 then f = 48 sr6 (sr6 - 0.5) sr2)
//   V1  rcp seed + 1 Newton with cubic correction, f = (A t - B) t sr2 with t = sr2^3
//   V2  V1 at 10 blocks/SM (48 registers)
//   V3  V1, two quads (8 candidates) per iteration
//   V4  V1 at 6 blocks/SM
// plus a reciprocal accuracy probe.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ double rcp2(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double rcp1c(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

template <int V>
__device__ __forceinline__ void pair(double dx, double dy, double dz, bool ok, double rc2, double& fx, double& fy,
                                     double& fz) {
  const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
  const bool in = ok && rsq < rc2;
  const double rs = in ? rsq : 1.0;
  double f;
  if (V == 0) {
    const double sr2 = rcp2(rs);
    const double sr6 = sr2 * sr2 * sr2 * 1.0;
    f = 48.0 * sr6 * (sr6 - 0.5) * sr2;
  } else {
    const double sr2 = rcp1c(rs);
    const double t = sr2 * sr2 * sr2;
    f = fma(48.0, t, -24.0) * (t * sr2);
  }
  f = in ? f : 0.0;
  fx = fma(f, dx, fx);
  fy = fma(f, dy, fy);
  fz = fma(f, dz, fz);
}

template <int V, int QPI>
__device__ __forceinline__ void atom(int32_t i, const double* __restrict__ pos, int64_t ld,
                                     const int32_t* __restrict__ nbr, int64_t ld_nbr,
                                     const int32_t* __restrict__ cnts, double rc2, double* __restrict__ out) {
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const double* __restrict__ py = pos + ld;
  const double* __restrict__ pz = pos + 2 * ld;
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
        xj[u] = __ldg(pos + jj[u]);
        yj[u] = __ldg(py + jj[u]);
        zj[u] = __ldg(pz + jj[u]);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) pair<V>(xi - xj[u], yi - yj[u], zi - zj[u], 4 * q + u < cnt, rc2, fx, fy, fz);
      a = b;
      b = c;
    }
  } else {
    int4 a = nq > 0 ? __ldcs(row) : self4;
    int4 b = nq > 1 ? __ldcs(row + ld_nbr) : self4;
    for (int32_t q = 0; q < nq; q += 2) {
      const int4 c = (q + 2 < nq) ? __ldcs(row + (int64_t)(q + 2) * ld_nbr) : self4;
      const int4 d = (q + 3 < nq) ? __ldcs(row + (int64_t)(q + 3) * ld_nbr) : self4;
      const int32_t jj[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      double xj[8], yj[8], zj[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        xj[u] = __ldg(pos + jj[u]);
        yj[u] = __ldg(py + jj[u]);
        zj[u] = __ldg(pz + jj[u]);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) pair<V>(xi - xj[u], yi - yj[u], zi - zj[u], 4 * q + u < cnt, rc2, fx, fy, fz);
      a = c;
      b = d;
    }
  }
  out[i] = fx;
  out[ld + i] = fy;
  out[2 * ld + i] = fz;
}

template <int V, int QPI, int MINB, int BS = 128>
__global__ void __launch_bounds__(BS, MINB) k_var(const double* __restrict__ pos, int64_t ld,
                                                  const int32_t* __restrict__ nbr, int64_t ld_nbr,
                                                  const int32_t* __restrict__ cnts, int32_t n, double rc2,
                                                  double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atom<V, QPI>(i, pos, ld, nbr, ld_nbr, cnts, rc2, out);
}

__global__ void k_rcp_probe(const double* x, int n, double* err) {
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double a = x[t];
  const double exact = 1.0 / a;
  err[2 * t] = fabs(rcp1c(a) - exact) / exact;
  err[2 * t + 1] = fabs(rcp2(a) - exact) / exact;
}

}  // namespace

extern "C" int exp_step3(int variant, const double* pos, int64_t ld, const int32_t* nbr, int64_t ld_nbr,
                         const int32_t* cnts, int32_t n, double rc2, double* out, void* s) {
  cudaStream_t st = (cudaStream_t)s;
  const dim3 g((n + 127) / 128), b(128);
  const dim3 g64((n + 63) / 64), b64(64), g256((n + 255) / 256), b256(256);
  switch (variant) {
    case 0: k_var<0, 1, 8><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 1: k_var<1, 1, 8><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 2: k_var<1, 1, 6><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 3: k_var<1, 1, 5><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 4: k_var<1, 1, 4><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 5: k_var<1, 2, 5><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 6: k_var<1, 2, 4><<<g, b, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 7: k_var<1, 1, 12, 64><<<g64, b64, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 8: k_var<1, 1, 3, 256><<<g256, b256, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 9: k_var<1, 1, 10, 64><<<g64, b64, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}

extern "C" int exp_rcp_probe(const double* x, int n, double* err, void* s) {
  k_rcp_probe<<<(n + 255) / 256, 256, 0, (cudaStream_t)s>>>(x, n, err);
  return (int)cudaGetLastError();
}
