// Experiment: two atoms per thread over merged neighbour rows.  Thread p owns
// atoms (2p, 2p+1) (brick-adjacent) and walks the union of their rows: each
// x_j is gathered once and used for both atoms (masked when j is not within
// rc of one of them).  Baseline: one atom per thread over its own row.  Both
// rows are slot-major int32 (slot k of row p at rows[k * ld + p]), LJ with the
// production arithmetic, forces only.
#include <cuda_runtime.h>
#include <stdint.h>

__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

extern "C" __global__ void __launch_bounds__(256, 4)
k_single(const double* __restrict__ pos, int64_t ld, int32_t n, const int32_t* __restrict__ rows, int64_t ldr,
         const int32_t* __restrict__ cnt, double rc2, double A, double B, double* __restrict__ f) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  double fx = 0, fy = 0, fz = 0;
  const int32_t c = cnt[i];
#pragma unroll 4
  for (int32_t k = 0; k < c; ++k) {
    const int32_t j = __ldg(rows + (int64_t)k * ldr + i);
    const double dx = xi - __ldg(pos + j), dy = yi - __ldg(pos + ld + j), dz = zi - __ldg(pos + 2 * ld + j);
    const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
    const bool in = rsq < rc2;
    const double sr2 = rcp_fast(in ? rsq : 1.0);
    const double t = sr2 * sr2 * sr2;
    const double ff = in ? fma(A, t, -B) * (t * sr2) : 0.0;
    fx = fma(ff, dx, fx);
    fy = fma(ff, dy, fy);
    fz = fma(ff, dz, fz);
  }
  f[i] = fx;
  f[ld + i] = fy;
  f[2 * ld + i] = fz;
}

extern "C" __global__ void __launch_bounds__(256, 3)
k_pair(const double* __restrict__ pos, int64_t ld, int32_t n, const int32_t* __restrict__ rows, int64_t ldr,
       const int32_t* __restrict__ cnt, double rc2, double A, double B, double* __restrict__ f) {
  const int32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t i0 = 2 * p, i1 = 2 * p + 1;
  if (i0 >= n) return;
  const bool has1 = i1 < n;
  const double x0 = pos[i0], y0 = pos[ld + i0], z0 = pos[2 * ld + i0];
  const double x1 = has1 ? pos[i1] : 0.0, y1 = has1 ? pos[ld + i1] : 0.0, z1 = has1 ? pos[2 * ld + i1] : 0.0;
  double fx0 = 0, fy0 = 0, fz0 = 0, fx1 = 0, fy1 = 0, fz1 = 0;
  const int32_t c = cnt[p];
#pragma unroll 2
  for (int32_t k = 0; k < c; ++k) {
    const int32_t j = __ldg(rows + (int64_t)k * ldr + p);
    const double xj = __ldg(pos + j), yj = __ldg(pos + ld + j), zj = __ldg(pos + 2 * ld + j);
    {
      const double dx = x0 - xj, dy = y0 - yj, dz = z0 - zj;
      const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
      const bool in = rsq < rc2 && j != i0;
      const double sr2 = rcp_fast(in ? rsq : 1.0);
      const double t = sr2 * sr2 * sr2;
      const double ff = in ? fma(A, t, -B) * (t * sr2) : 0.0;
      fx0 = fma(ff, dx, fx0);
      fy0 = fma(ff, dy, fy0);
      fz0 = fma(ff, dz, fz0);
    }
    {
      const double dx = x1 - xj, dy = y1 - yj, dz = z1 - zj;
      const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
      const bool in = has1 && rsq < rc2 && j != i1;
      const double sr2 = rcp_fast(in ? rsq : 1.0);
      const double t = sr2 * sr2 * sr2;
      const double ff = in ? fma(A, t, -B) * (t * sr2) : 0.0;
      fx1 = fma(ff, dx, fx1);
      fy1 = fma(ff, dy, fy1);
      fz1 = fma(ff, dz, fz1);
    }
  }
  f[i0] = fx0;
  f[ld + i0] = fy0;
  f[2 * ld + i0] = fz0;
  if (has1) {
    f[i1] = fx1;
    f[ld + i1] = fy1;
    f[2 * ld + i1] = fz1;
  }
}

extern "C" int run_single(const double* pos, int64_t ld, int32_t n, const int32_t* rows, int64_t ldr,
                          const int32_t* cnt, double rc2, double A, double B, double* f, void* s) {
  k_single<<<(n + 255) / 256, 256, 0, (cudaStream_t)s>>>(pos, ld, n, rows, ldr, cnt, rc2, A, B, f);
  return (int)cudaGetLastError();
}

extern "C" int run_pair(const double* pos, int64_t ld, int32_t n, const int32_t* rows, int64_t ldr,
                        const int32_t* cnt, double rc2, double A, double B, double* f, void* s) {
  const int32_t np = (n + 1) / 2;
  k_pair<<<(np + 255) / 256, 256, 0, (cudaStream_t)s>>>(pos, ld, n, rows, ldr, cnt, rc2, A, B, f);
  return (int)cudaGetLastError();
}
