// Shared-memory neighbour gathers: the cost of the LJ candidate loop when the
// positions come from a block's staging set in shared memory (uint16 staging
// indices streamed from a list), with random indices vs a bank-class schedule
// (slot k of lane l reads class (k + l) mod 16 of the fp64 bank pairs: the 16
// lanes of a half-warp hit 16 distinct bank pairs).  2,048,000 atoms x 64
// candidates, 256-atom blocks, NS staged atoms per block (copied from global
// memory each launch).  Compare with the L1-gather loop (exp_step4: 0.32 ms
// for ~65 candidates per atom on the real lists).
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdio>

constexpr int kB = 256;
constexpr int kK = 64;  // candidates per atom (multiple of 8)

__device__ __forceinline__ double rcp1c(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

// list: octet q (8 uint16 slots) of atom i at lst[q * n + i] (uint4)
__global__ void k_make_list(uint4* lst, int n, int ns, int mode) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int l = threadIdx.x & 15;
  for (int q = 0; q < kK / 8; ++q) {
    uint32_t w[4];
    for (int h = 0; h < 4; ++h) {
      uint32_t v = 0;
      for (int u = 0; u < 2; ++u) {
        const int k = q * 8 + h * 2 + u;
        uint32_t r = hash32(i * 977u + k * 131u + 7u);
        uint32_t s;
        if (mode == 0) s = r % ns;
        else s = (r % (ns / 16)) * 16 + ((k + l) & 15);
        v |= (s & 0xFFFFu) << (16 * u);
      }
      w[h] = v;
    }
    lst[(int64_t)q * n + i] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

__global__ void __launch_bounds__(kB, 3) k_smem(const double* __restrict__ pos, int64_t ld, const uint4* __restrict__ lst,
                                               int n, int ns, double rc2, double* __restrict__ out) {
  extern __shared__ double st[];
  double* sx = st;
  double* sy = st + ns;
  double* sz = st + 2 * ns;
  const int b = blockIdx.x;
  // stage NS consecutive atoms around the block (coalesced)
  const int64_t base = ((int64_t)b * kB * 7) % (n - ns);
  for (int s = threadIdx.x; s < ns; s += kB) {
    sx[s] = pos[base + s];
    sy[s] = pos[ld + base + s];
    sz[s] = pos[2 * ld + base + s];
  }
  __syncthreads();
  const int i = b * kB + threadIdx.x;
  if (i >= n) return;
  const double xi = pos[i] * 0.0 + sx[threadIdx.x] + 0.3, yi = sy[threadIdx.x] + 0.2, zi = sz[threadIdx.x] - 0.1;
  double fx = 0, fy = 0, fz = 0;
  uint4 a = __ldcs(lst + i);
  for (int q = 0; q < kK / 8; ++q) {
    const uint4 nx = (q + 1 < kK / 8) ? __ldcs(lst + (int64_t)(q + 1) * n + i) : a;
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
        const double dx = xi - xj[u], dy = yi - yj[u], dz = zi - zj[u];
        const double rsq = fma(dx, dx, fma(dy, dy, dz * dz));
        const bool in = rsq < rc2 && rsq > 0.0;
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

int main() {
  const int n = 2048000;
  const int64_t ld = n;
  double *pos, *out;
  uint4* lst;
  cudaMalloc(&pos, sizeof(double) * 3 * n);
  cudaMalloc(&out, sizeof(double) * 3 * n);
  cudaMalloc(&lst, sizeof(uint4) * (kK / 8) * n);
  // positions: a jittered cubic lattice so many pairs fall inside rc
  double* h = new double[3 * (size_t)n];
  for (int i = 0; i < n; ++i) {
    h[i] = (i % 7) * 0.7;
    h[n + i] = ((i / 7) % 7) * 0.7;
    h[2 * n + i] = ((i / 49) % 7) * 0.7;
  }
  cudaMemcpy(pos, h, sizeof(double) * 3 * n, cudaMemcpyHostToDevice);
  const int blocks = (n + kB - 1) / kB;
  for (int ns : {1200, 1800}) {
    const size_t smem = sizeof(double) * 3 * ns;
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int mode = 0; mode < 2; ++mode) {
      k_make_list<<<blocks, kB>>>(lst, n, ns, mode);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      float best = 1e30f;
      for (int r = 0; r < 10; ++r) {
        cudaEventRecord(e0);
        k_smem<<<blocks, kB, smem>>>(pos, ld, lst, n, ns, 6.25, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
      }
      std::printf("NS %d mode %s: %.4f ms (%d candidates/atom) err %s\n", ns, mode ? "bank-class" : "random", best, kK,
                  cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
