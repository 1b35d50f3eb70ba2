// Block-staged force loop on the REAL production lists (front segments):
// each 256-atom block copies the positions of the union of its atoms'
// neighbours (a sorted list of atom indices, prepared on the host side) into
// shared memory, then every thread walks its row of uint16 staging indices
// (octets: slot k of atom i at idx[(k / 8) * n + i].k%8).  Rows come either
// in list order or reordered so that slot k of lane l hits fp64 bank pair
// class (k + l) mod 16 where possible.  Compare with exp_step4 (L1 gathers).
#include <cuda_runtime.h>
#include <stdint.h>

namespace {

constexpr int kB = 256;

__device__ __forceinline__ double rcp1c(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

__global__ void __launch_bounds__(kB, 3) k_staged(const double* __restrict__ pos, int64_t ld,
                                                 const int32_t* __restrict__ uniq, const int32_t* __restrict__ ustart,
                                                 const uint4* __restrict__ idx, const int32_t* __restrict__ cnt,
                                                 int32_t n, double rc2, double* __restrict__ out, int max_stage) {
  extern __shared__ double st[];
  double* sx = st;
  double* sy = st + max_stage;
  double* sz = st + 2 * max_stage;
  const int b = blockIdx.x;
  const int32_t u0 = ustart[b], u1 = ustart[b + 1];
  for (int32_t s = u0 + threadIdx.x; s < u1; s += kB) {
    const int32_t j = __ldg(uniq + s);
    sx[s - u0] = __ldg(pos + j);
    sy[s - u0] = __ldg(pos + ld + j);
    sz[s - u0] = __ldg(pos + 2 * ld + j);
  }
  __syncthreads();
  const int32_t i = b * kB + threadIdx.x;
  if (i >= n) return;
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int32_t c = cnt[i];
  const int32_t no = (c + 7) >> 3;
  double fx = 0, fy = 0, fz = 0;
  uint4 a = no > 0 ? __ldcs(idx + i) : make_uint4(0, 0, 0, 0);
  for (int32_t q = 0; q < no; ++q) {
    const uint4 nx = (q + 1 < no) ? __ldcs(idx + (int64_t)(q + 1) * n + i) : a;
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      double xj[4], yj[4], zj[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t s = (w[2 * h + (u >> 1)] >> (16 * (u & 1))) & 0xFFFFu;
        xj[u] = sx[s];
        yj[u] = sy[s];
        zj[u] = sz[s];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t slot = 8 * q + 4 * h + u;
        const double dx = xi - xj[u], dy = yi - yj[u], dz = zi - zj[u];
        const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
        const bool in = slot < c && rsq < rc2;
        const double sr2 = rcp1c(in ? rsq : 1.0);
        const double t = sr2 * sr2 * sr2;
        const double f = in ? fma(48.0, t, -24.0) * (t * sr2) : 0.0;
        fx = fma(f, dx, fx);
        fy = fma(f, dy, fy);
        fz = fma(f, dz, fz);
      }
    }
    a = nx;
  }
  out[i] = fx;
  out[ld + i] = fy;
  out[2 * ld + i] = fz;
}

}  // namespace

extern "C" int exp_staged(const double* pos, int64_t ld, const int32_t* uniq, const int32_t* ustart, const void* idx,
                          const int32_t* cnt, int32_t n, double rc2, double* out, int max_stage, void* s) {
  const size_t smem = sizeof(double) * 3 * (size_t)max_stage;
  cudaFuncSetAttribute(k_staged, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  if (smem > 200 * 1024) return -2;
  k_staged<<<(n + kB - 1) / kB, kB, smem, (cudaStream_t)s>>>(pos, ld, uniq, ustart,
                                                              reinterpret_cast<const uint4*>(idx), cnt, n, rc2, out,
                                                              max_stage);
  return (int)cudaGetLastError();
}
