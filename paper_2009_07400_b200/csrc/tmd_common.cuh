// Shared helpers for the tinyMD B200 kernels (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tinymd_b200.h"

namespace tmd {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// error plumbing
// ---------------------------------------------------------------------------
void set_last_error(const char* where, cudaError_t e);
void count_launch();

// every kernel launch in the library is followed by this check, which also
// counts it (tmd_launch_count: evidence of how many device kernels ran)
#define TMD_LAUNCH_CHECK(where)                              \
  do {                                                       \
    ::tmd::count_launch();                                   \
    cudaError_t _e = cudaGetLastError();                     \
    if (_e != cudaSuccess) {                                 \
      ::tmd::set_last_error(where, _e);                      \
      return TMD_ERR_CUDA;                                   \
    }                                                        \
  } while (0)

#define TMD_CUDA_TRY(call, where)                            \
  do {                                                       \
    cudaError_t _e = (call);                                 \
    if (_e != cudaSuccess) {                                 \
      ::tmd::set_last_error(where, _e);                      \
      return TMD_ERR_CUDA;                                   \
    }                                                        \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(int64_t n, int block) {
  int64_t g = (n + block - 1) / block;
  return g < 1 ? 1 : (int)g;
}

int sm_count();

// ---------------------------------------------------------------------------
// device status word (see include/tinymd_b200.h)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void raise_status(int64_t* st, int code, unsigned long long key) {
  atomicMax(reinterpret_cast<unsigned long long*>(st), (unsigned long long)code);
  atomicMin(reinterpret_cast<unsigned long long*>(st + 1), key);
}

__device__ __forceinline__ void need_capacity(int64_t* st, int need) {
  atomicMax(reinterpret_cast<unsigned long long*>(st), (unsigned long long)TMD_CAPACITY);
  atomicMax(reinterpret_cast<unsigned long long*>(st + 2), (unsigned long long)need);
}

// Non-negative doubles order like their bit patterns: max via integer atomics.
__device__ __forceinline__ void atomic_max_nonneg(double* p, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(p), (unsigned long long)__double_as_longlong(v));
}

// ---------------------------------------------------------------------------
// reference-order arithmetic: explicit round-to-nearest ops so nvcc cannot
// contract into FMA (numpy evaluates every product and sum separately)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// numpy einsum('ijk,ijk->ij') order on a 3-vector: (x*x + z*z) + y*y
__device__ __forceinline__ double rsq_ref(double dx, double dy, double dz) {
  return add_rn(add_rn(mul_rn(dx, dx), mul_rn(dz, dz)), mul_rn(dy, dy));
}

// numpy (d*d).sum(axis=1) on an (n, 3) array: (x*x + y*y) + z*z
__device__ __forceinline__ double norm2_seq(double dx, double dy, double dz) {
  return add_rn(add_rn(mul_rn(dx, dx), mul_rn(dy, dy)), mul_rn(dz, dz));
}

// quad-interleaved neighbor-major list layout: slot k of local i
__device__ __forceinline__ int64_t slot_index(int32_t k, int32_t i, int64_t ld_nbr) {
  return (((int64_t)(k >> 2)) * ld_nbr + i) * 4 + (k & 3);
}

// ---------------------------------------------------------------------------
// warp / block reductions (deterministic: fixed tree)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Sum NV values over the block; result valid in thread 0.  smem >= NV * 32 doubles.
template <int NV>
__device__ __forceinline__ void block_sum(double (&v)[NV], double* smem) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int q = 0; q < NV; ++q) v[q] = warp_sum(v[q]);
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) smem[q * 32 + wid] = v[q];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      double t = lane < nw ? smem[q * 32 + lane] : 0.0;
      v[q] = warp_sum(t);
    }
  }
  __syncthreads();
}

// Deterministic grid reduction: every block writes NV partials, the last block
// to finish sums them in block order and writes d_out[q] (+= if accumulate).
// Needs a zero-initialised counter; it is reset by the last block.
template <int NV>
__device__ void grid_sum_finish(const double (&v)[NV], double* partials, unsigned int* counter,
                                double* d_out, bool accumulate) {
  __shared__ bool is_last;
  __shared__ double red[NV * 32];
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) partials[(size_t)q * gridDim.x + blockIdx.x] = v[q];
    __threadfence();
    unsigned int done = atomicAdd(counter, 1u);
    is_last = (done == gridDim.x - 1);
  }
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  // each thread sums blocks tid, tid + B, tid + 2B, ... in that order; the
  // loads of four strides and all NV values are issued together (L2 reads:
  // the partials were written by other blocks), a chain of dependent volatile
  // loads took tens of microseconds at 8000 blocks
  double acc[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) acc[q] = 0.0;
  const unsigned int B = blockDim.x, G = gridDim.x;
  for (unsigned int b0 = threadIdx.x; b0 < G; b0 += 4 * B) {
    double v[4][NV];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned int b = b0 + u * B;
#pragma unroll
      for (int q = 0; q < NV; ++q) v[u][q] = b < G ? __ldcg(partials + (size_t)q * G + b) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int q = 0; q < NV; ++q)
        if (b0 + u * B < G) acc[q] += v[u][q];
    }
  }
  block_sum<NV>(acc, red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NV; ++q) d_out[q] = accumulate ? d_out[q] + acc[q] : acc[q];
    *counter = 0u;
  }
}

// ---------------------------------------------------------------------------
// Ghost refresh fused into a drift (replaces synchronize, comm.py:469-498):
// every ghost copy is listed under the local atom it mirrors (root) with its
// destination rank, slot and accumulated periodic shift; the atom's thread
// writes x_new + shift into the destination rank's position buffer -- its
// own, or a peer GPU's through CUDA IPC over NVLink.  No fence: the caller
// orders the peers' reads after this kernel (stream order, then a barrier).
// ---------------------------------------------------------------------------
constexpr int kMaxPeers = 8;
struct Exports {
  const int32_t* start;  // (n_local + 1) CSR over locals; null = no fused refresh
  const int32_t* rank;   // destination rank of entry e
  const int32_t* slot;   // destination ghost slot
  const double* sh;      // (3, n_ex) shifts
  int64_t n_ex;
  double* base[kMaxPeers];  // destination rank's position buffer
  int64_t ld[kMaxPeers];
  // border gate: only atoms whose build-time position lies within r of a slab
  // face (x_d > thr_hi[d] or x_d < thr_lo[d]) can have copies (the borders'
  // own selection tests); gate = 0 reads every atom's table entry
  int gate;
  double thr_hi[3], thr_lo[3];
};

__device__ __forceinline__ void write_exports_ungated(const Exports& ex, int32_t i, double x, double y, double z) {
  const int32_t e1 = ex.start[i + 1];
  for (int32_t q = ex.start[i]; q < e1; ++q) {
    const int r = ex.rank[q];
    const int32_t g = ex.slot[q];
    double* __restrict__ dst = ex.base[r];
    const int64_t L = ex.ld[r];
    dst[g] = add_rn(x, ex.sh[q]);
    dst[L + g] = add_rn(y, ex.sh[ex.n_ex + q]);
    dst[2 * L + g] = add_rn(z, ex.sh[2 * ex.n_ex + q]);
  }
}

// (xr, yr, zr) = the atom's build-time position (the border gate)
__device__ __forceinline__ void write_exports_at(const Exports& ex, int32_t i, double x, double y, double z, double xr,
                                                 double yr, double zr) {
  if (!ex.start) return;
  if (ex.gate) {
    const bool border = xr > ex.thr_hi[0] || xr < ex.thr_lo[0] || yr > ex.thr_hi[1] || yr < ex.thr_lo[1] ||
                        zr > ex.thr_hi[2] || zr < ex.thr_lo[2];
    if (!border) return;
  }
  write_exports_ungated(ex, i, x, y, z);
}

// Host side: the Exports argument block from the C-ABI arguments.
inline int make_exports(const int32_t* d_ex_start, const int32_t* d_ex_rank, const int32_t* d_ex_slot,
                        const double* d_ex_sh, int64_t n_ex, int32_t n_peers, double* const* h_peer_base,
                        const int64_t* h_peer_ld, const double* h_ex_border, const double* d_xref, Exports* ex) {
  *ex = Exports{};
  if (!d_ex_start) return TMD_OK;
  if (n_peers < 1 || n_peers > kMaxPeers || !h_peer_base || !h_peer_ld) return TMD_ERR_ARG;
  ex->start = d_ex_start;
  ex->rank = d_ex_rank;
  ex->slot = d_ex_slot;
  ex->sh = d_ex_sh;
  ex->n_ex = n_ex;
  if (h_ex_border) {
    if (!d_xref) return TMD_ERR_ARG;
    ex->gate = 1;
    for (int d = 0; d < 3; ++d) {
      ex->thr_hi[d] = h_ex_border[d];
      ex->thr_lo[d] = h_ex_border[3 + d];
    }
  }
  for (int q = 0; q < n_peers; ++q) {
    ex->base[q] = h_peer_base[q];
    ex->ld[q] = h_peer_ld[q];
  }
  return TMD_OK;
}

// Scratch for grid reductions: partial buffer sized for max_blocks * nv and a
// counter; lives for the process (per device).
struct ReduceScratch {
  double* partials;
  unsigned int* counter;
  int max_blocks;
};
int reduce_scratch(ReduceScratch* rs, int blocks, int nv, cudaStream_t stream);

// ---------------------------------------------------------------------------
// exclusive scan of int32 (used by binning and halo compaction)
// ---------------------------------------------------------------------------
// out[i] = sum_{k<i} in[k] for i in [0, n]; out has n + 1 entries.
int scan_exclusive(const int32_t* d_in, int32_t* d_out, int64_t n, cudaStream_t s);
void keep_pool_memory();

}  // namespace tmd
