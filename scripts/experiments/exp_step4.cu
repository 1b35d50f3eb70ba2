// Block-size / cache-policy variants of the FP64-trimmed force loop
// (front segments, forces only); see exp_step3.cu for the arithmetic.
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

__device__ __forceinline__ double rcp1c(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

template <int L>
__device__ __forceinline__ int4 ld_list(const int4* p) {
  if (L == 0) return __ldcs(p);
  int4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

template <int PL>
__device__ __forceinline__ double ld_pos(const double* p) {
  if (PL == 0) return __ldg(p);
  double v;
  asm volatile("ld.global.nc.L1::evict_last.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}

__device__ __forceinline__ void pair(double dx, double dy, double dz, bool ok, double rc2, double& fx, double& fy,
                                     double& fz) {
  const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
  const bool in = ok && rsq < rc2;
  const double rs = in ? rsq : 1.0;
  const double sr2 = rcp1c(rs);
  const double t = sr2 * sr2 * sr2;
  double f = fma(48.0, t, -24.0) * (t * sr2);
  f = in ? f : 0.0;
  fx = fma(f, dx, fx);
  fy = fma(f, dy, fy);
  fz = fma(f, dz, fz);
}

template <int L, int PL>
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
  int4 a = nq > 0 ? ld_list<L>(row) : self4;
  int4 b = nq > 1 ? ld_list<L>(row + ld_nbr) : self4;
  for (int32_t q = 0; q < nq; ++q) {
    const int4 c = (q + 2 < nq) ? ld_list<L>(row + (int64_t)(q + 2) * ld_nbr) : self4;
    const int32_t jj[4] = {a.x, a.y, a.z, a.w};
    double xj[4], yj[4], zj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      xj[u] = ld_pos<PL>(pos + jj[u]);
      yj[u] = ld_pos<PL>(py + jj[u]);
      zj[u] = ld_pos<PL>(pz + jj[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) pair(xi - xj[u], yi - yj[u], zi - zj[u], 4 * q + u < cnt, rc2, fx, fy, fz);
    a = b;
    b = c;
  }
  out[i] = fx;
  out[ld + i] = fy;
  out[2 * ld + i] = fz;
}

template <int BS, int MINB, int L, int PL>
__global__ void __launch_bounds__(BS, MINB) k_var(const double* __restrict__ pos, int64_t ld,
                                                  const int32_t* __restrict__ nbr, int64_t ld_nbr,
                                                  const int32_t* __restrict__ cnts, int32_t n, double rc2,
                                                  double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atom<L, PL>(i, pos, ld, nbr, ld_nbr, cnts, rc2, out);
}

template <int BS, int MINB, int L, int PL>
int launch(const double* pos, int64_t ld, const int32_t* nbr, int64_t ld_nbr, const int32_t* cnts, int32_t n,
           double rc2, double* out, cudaStream_t st, int carve) {
  if (carve >= 0) cudaFuncSetAttribute(k_var<BS, MINB, L, PL>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
  k_var<BS, MINB, L, PL><<<(n + BS - 1) / BS, BS, 0, st>>>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out);
  return 0;
}

}  // namespace

extern "C" int exp_step4(int variant, const double* pos, int64_t ld, const int32_t* nbr, int64_t ld_nbr,
                         const int32_t* cnts, int32_t n, double rc2, double* out, void* s) {
  cudaStream_t st = (cudaStream_t)s;
  switch (variant) {
    case 0: launch<256, 3, 0, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 1: launch<384, 2, 0, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 2: launch<512, 2, 0, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 3: launch<512, 1, 0, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 4: launch<1024, 1, 0, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 5: launch<256, 3, 1, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 6: launch<256, 3, 0, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, 0); break;
    case 7: launch<512, 2, 1, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 8: launch<256, 3, 1, 1>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    case 9: launch<256, 2, 0, 0>(pos, ld, nbr, ld_nbr, cnts, n, rc2, out, st, -1); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}
