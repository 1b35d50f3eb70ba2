// Force-loop layout experiments on the production (split, quad-interleaved)
// lists, front segment only, forces only (no epilogue):
//   V0  SoA gathers, thread per atom (the production loop)
//   V1  AoS4 (x, y, z, pad) 32-byte gathers (LDG.256), thread per atom
//   V2  AoS4 as two 16-byte gathers, thread per atom
//   V3  V1 + SM-local persistent sweep (each SM walks a contiguous atom range)
//   V4  V0 + SM-local persistent sweep
//   V5  4 lanes per atom, AoS4 LDG.256
//   V6  4 lanes per atom, SoA
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

__device__ __forceinline__ void ld256(const double* p, double& a, double& b, double& c) {
  double d;
  asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

__device__ __forceinline__ void pair(double dx, double dy, double dz, bool ok, double rc2, double& fx, double& fy,
                                     double& fz) {
  const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
  const bool in = ok && rsq < rc2;
  const double rs = in ? rsq : 1.0;
  const double sr2 = rcp2(rs);
  const double sr6 = sr2 * sr2 * sr2;
  const double f = in ? 48.0 * sr6 * (sr6 - 0.5) * sr2 : 0.0;
  fx = fma(f, dx, fx);
  fy = fma(f, dy, fy);
  fz = fma(f, dz, fz);
}

// gather modes: 0 SoA, 1 AoS4 256-bit, 2 AoS4 2x128-bit
template <int G>
__device__ __forceinline__ void gather(const double* __restrict__ pos, int64_t ld, const double* __restrict__ aos,
                                       int32_t j, double& x, double& y, double& z) {
  if (G == 0) {
    x = __ldg(pos + j);
    y = __ldg(pos + ld + j);
    z = __ldg(pos + 2 * ld + j);
  } else if (G == 1) {
    ld256(aos + 4 * (int64_t)j, x, y, z);
  } else {
    const double2 a = __ldg(reinterpret_cast<const double2*>(aos) + 2 * (int64_t)j);
    const double2 b = __ldg(reinterpret_cast<const double2*>(aos) + 2 * (int64_t)j + 1);
    x = a.x;
    y = a.y;
    z = b.x;
  }
}

template <int G>
__device__ __forceinline__ void atom(int32_t i, const double* __restrict__ pos, int64_t ld,
                                     const double* __restrict__ aos, const int32_t* __restrict__ nbr, int64_t ld_nbr,
                                     const int32_t* __restrict__ cnts, double rc2, double* __restrict__ out) {
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
    double xj[4], yj[4], zj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) gather<G>(pos, ld, aos, jj[u], xj[u], yj[u], zj[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) pair(xi - xj[u], yi - yj[u], zi - zj[u], 4 * q + u < cnt, rc2, fx, fy, fz);
    a = b;
    b = c;
  }
  out[i] = fx;
  out[ld + i] = fy;
  out[2 * ld + i] = fz;
}

template <int G>
__global__ void __launch_bounds__(128, 8) k_thread(const double* __restrict__ pos, int64_t ld,
                                                  const double* __restrict__ aos, const int32_t* __restrict__ nbr,
                                                  int64_t ld_nbr, const int32_t* __restrict__ cnts, int32_t n,
                                                  double rc2, double* __restrict__ out) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) atom<G>(i, pos, ld, aos, nbr, ld_nbr, cnts, rc2, out);
}

// ---- SM-local persistent sweep -------------------------------------------------
// region r = [n r / R, n (r + 1) / R) of the atom order, R = number of SMs present;
// CTAs on SM s take tiles of region rank(s) in order (per-region atomic counter),
// then steal tiles from regions that still have work.
__device__ __forceinline__ int smid() {
  int s;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  return s;
}

template <int G>
__global__ void __launch_bounds__(128, 8) k_sweep(const double* __restrict__ pos, int64_t ld,
                                                 const double* __restrict__ aos, const int32_t* __restrict__ nbr,
                                                 int64_t ld_nbr, const int32_t* __restrict__ cnts, int32_t n,
                                                 double rc2, double* __restrict__ out,
                                                 const int16_t* __restrict__ sm_rank, int32_t R,
                                                 unsigned int* __restrict__ ctr) {
  __shared__ int s_t;
  const int my = sm_rank[smid()];
  auto region_lo = [&](int r) { return (int32_t)((int64_t)n * r / R); };
  auto ntiles = [&](int r) { return (region_lo(r + 1) - region_lo(r) + 127) >> 7; };
  for (int pass = 0; pass < R; ++pass) {
    const int r = (my + pass) % R;
    if (pass > 0) {  // cheap skip of exhausted regions
      if (*((volatile unsigned int*)ctr + r) >= (unsigned)ntiles(r)) continue;
    }
    const int nt = ntiles(r);
    const int32_t lo = region_lo(r), hi = region_lo(r + 1);
    while (true) {
      if (threadIdx.x == 0) s_t = atomicAdd(ctr + r, 1u);
      __syncthreads();
      const int t = s_t;
      __syncthreads();
      if (t >= nt) break;
      const int32_t i = lo + t * 128 + threadIdx.x;
      if (i < hi) atom<G>(i, pos, ld, aos, nbr, ld_nbr, cnts, rc2, out);
    }
  }
}

// ---- T lanes per atom ------------------------------------------------------------
template <int G>
__global__ void __launch_bounds__(128, 8) k_coop4(const double* __restrict__ pos, int64_t ld,
                                                 const double* __restrict__ aos, const int32_t* __restrict__ nbr,
                                                 int64_t ld_nbr, const int32_t* __restrict__ cnts, int32_t n,
                                                 double rc2, double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int sub = lane & 3;
  const int32_t i = blockIdx.x * 32 + (threadIdx.x >> 2);
  const bool live = i < n;
  const int32_t ii = live ? i : 0;
  const double xi = pos[ii], yi = pos[ld + ii], zi = pos[2 * ld + ii];
  const int32_t cnt = live ? cnts[ii] : 0;
  const int32_t nq = (cnt + 3) >> 2;
  const int32_t* col = nbr + 4 * (int64_t)ii + sub;
  const int64_t qs = 4 * ld_nbr;
  double fx = 0, fy = 0, fz = 0;
  // 4 quads per iteration: each lane has 4 gathers in flight
  int32_t q = 0;
  for (; q + 4 <= nq; q += 4) {
    int32_t jj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) jj[u] = __ldcs(col + (q + u) * qs);
    double xj[4], yj[4], zj[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) gather<G>(pos, ld, aos, jj[u], xj[u], yj[u], zj[u]);
#pragma unroll
    for (int u = 0; u < 4; ++u) pair(xi - xj[u], yi - yj[u], zi - zj[u], 4 * (q + u) + sub < cnt, rc2, fx, fy, fz);
  }
  for (; q < nq; ++q) {
    const int32_t j = __ldcs(col + q * qs);
    double xj, yj, zj;
    gather<G>(pos, ld, aos, j, xj, yj, zj);
    pair(xi - xj, yi - yj, zi - zj, 4 * q + sub < cnt, rc2, fx, fy, fz);
  }
#pragma unroll
  for (int m = 1; m < 4; m <<= 1) {
    fx += __shfl_xor_sync(0xffffffffu, fx, m);
    fy += __shfl_xor_sync(0xffffffffu, fy, m);
    fz += __shfl_xor_sync(0xffffffffu, fz, m);
  }
  if (live && sub == 0) {
    out[i] = fx;
    out[ld + i] = fy;
    out[2 * ld + i] = fz;
  }
}

}  // namespace

extern "C" int exp_step2(int variant, const double* pos, int64_t ld, const double* aos, const int32_t* nbr,
                         int64_t ld_nbr, const int32_t* cnts, int32_t n, double rc2, double* out,
                         const int16_t* sm_rank, int32_t R, unsigned int* ctr, void* s) {
  cudaStream_t st = (cudaStream_t)s;
  const dim3 g((n + 127) / 128), b(128);
  switch (variant) {
    case 0: k_thread<0><<<g, b, 0, st>>>(pos, ld, aos, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 1: k_thread<1><<<g, b, 0, st>>>(pos, ld, aos, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 2: k_thread<2><<<g, b, 0, st>>>(pos, ld, aos, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 3:
    case 4: {
      cudaMemsetAsync(ctr, 0, sizeof(unsigned int) * R, st);
      const dim3 gp(8 * R);
      if (variant == 3)
        k_sweep<1><<<gp, b, 0, st>>>(pos, ld, aos, nbr, ld_nbr, cnts, n, rc2, out, sm_rank, R, ctr);
      else
        k_sweep<0><<<gp, b, 0, st>>>(pos, ld, aos, nbr, ld_nbr, cnts, n, rc2, out, sm_rank, R, ctr);
      break;
    }
    case 5: k_coop4<1><<<dim3((n + 31) / 32), b, 0, st>>>(pos, ld, aos, nbr, ld_nbr, cnts, n, rc2, out); break;
    case 6: k_coop4<0><<<dim3((n + 31) / 32), b, 0, st>>>(pos, ld, aos, nbr, ld_nbr, cnts, n, rc2, out); break;
    default: return -1;
  }
  return (int)cudaGetLastError();
}

// SM ids present: one block per SM-slot records its %smid
__global__ void k_smids(int* out) {
  if (threadIdx.x == 0) out[blockIdx.x] = smid();
}
extern "C" int exp_smids(int* out, int nblocks, void* s) {
  k_smids<<<nblocks, 32, 0, (cudaStream_t)s>>>(out);
  return (int)cudaGetLastError();
}
