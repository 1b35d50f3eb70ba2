// SFC keys and per-block weights for the space-filling-curve load balancer
// (balance.py; SPEC.md:517-625 -- the reference ships no balance module, its
// comm.py:277-332 block_neighborhood_pattern consumes one).
//
// Integer work on the particles: each particle's cell at the forest's maximum
// depth D (2^D cells per axis over the global box), its Morton or Hilbert key
// (3D bits), and the count of particles per leaf block (leaves are contiguous
// key ranges of either curve, sorted by first key).
#include "tmd_common.cuh"

namespace tmd {

// x in the least significant position of each bit triad
__host__ __device__ inline uint64_t morton3(uint32_t x, uint32_t y, uint32_t z, int depth) {
  uint64_t k = 0;
  for (int b = 0; b < depth; ++b) {
    k |= (uint64_t)((x >> b) & 1u) << (3 * b);
    k |= (uint64_t)((y >> b) & 1u) << (3 * b + 1);
    k |= (uint64_t)((z >> b) & 1u) << (3 * b + 2);
  }
  return k;
}

// 3-D Hilbert index by Skilling's transpose construction ("Programming the
// Hilbert curve", AIP Conf. Proc. 707, 2004): axes -> transposed index, then
// the transpose's bits interleaved most significant first (x in the highest
// position of each triad).
__host__ __device__ inline uint64_t hilbert3(uint32_t x0, uint32_t y0, uint32_t z0, int depth) {
  uint32_t X[3] = {x0, y0, z0};
  const uint32_t M = 1u << (depth - 1);
  // inverse undo excess work
  for (uint32_t Q = M; Q > 1; Q >>= 1) {
    const uint32_t P = Q - 1;
    for (int i = 0; i < 3; ++i) {
      if (X[i] & Q) {
        X[0] ^= P;
      } else {
        const uint32_t t = (X[0] ^ X[i]) & P;
        X[0] ^= t;
        X[i] ^= t;
      }
    }
  }
  // Gray encode
  for (int i = 1; i < 3; ++i) X[i] ^= X[i - 1];
  uint32_t t = 0;
  for (uint32_t Q = M; Q > 1; Q >>= 1)
    if (X[2] & Q) t ^= Q - 1;
  for (int i = 0; i < 3; ++i) X[i] ^= t;
  uint64_t k = 0;
  for (int b = depth - 1; b >= 0; --b)
    for (int i = 0; i < 3; ++i) k = (k << 1) | ((X[i] >> b) & 1u);
  return k;
}

__global__ void k_sfc_keys(const double* __restrict__ pos, int64_t ld, int32_t n, double lo0, double lo1, double lo2,
                           double w0, double w1, double w2, int depth, int curve, uint64_t* __restrict__ keys) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t top = (1 << depth) - 1;
  int32_t c[3];
  const double lo[3] = {lo0, lo1, lo2}, w[3] = {w0, w1, w2};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const int32_t v = (int32_t)floor((pos[d * ld + i] - lo[d]) / w[d]);
    c[d] = v < 0 ? 0 : (v > top ? top : v);
  }
  keys[i] = curve == 0 ? morton3(c[0], c[1], c[2], depth) : hilbert3(c[0], c[1], c[2], depth);
}

// counts[b] += particles whose key lies in leaf b's range [start[b], start[b+1])
__global__ void k_leaf_counts(const uint64_t* __restrict__ keys, int32_t n, const uint64_t* __restrict__ start,
                              int32_t n_leaves, int32_t* __restrict__ counts) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t k = keys[i];
  int32_t lo = 0, hi = n_leaves - 1;  // last leaf with start <= k
  while (lo < hi) {
    const int32_t mid = (lo + hi + 1) >> 1;
    if (start[mid] <= k) lo = mid; else hi = mid - 1;
  }
  atomicAdd(counts + lo, 1);
}

}  // namespace tmd

using namespace tmd;

extern "C" int tmd_sfc_keys(const double* d_pos, int64_t ld, int32_t n, const double* h_lo, const double* h_width,
                            int32_t depth, int32_t curve, uint64_t* d_keys, void* stream) {
  if (n <= 0) return TMD_OK;
  if (!h_lo || !h_width || depth < 1 || depth > 21 || (curve != 0 && curve != 1)) return TMD_ERR_ARG;
  k_sfc_keys<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d_pos, ld, n, h_lo[0], h_lo[1], h_lo[2], h_width[0],
                                                              h_width[1], h_width[2], depth, curve, d_keys);
  TMD_LAUNCH_CHECK("sfc_keys");
  return TMD_OK;
}

extern "C" int tmd_leaf_counts(const uint64_t* d_keys, int32_t n, const uint64_t* d_leaf_start, int32_t n_leaves,
                               int32_t* d_counts, void* stream) {
  if (n_leaves < 1 || !d_leaf_start || !d_counts) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  TMD_CUDA_TRY(cudaMemsetAsync(d_counts, 0, sizeof(int32_t) * (size_t)n_leaves, s), "leaf_counts");
  if (n <= 0) return TMD_OK;
  k_leaf_counts<<<grid_for(n, 256), 256, 0, s>>>(d_keys, n, d_leaf_start, n_leaves, d_counts);
  TMD_LAUNCH_CHECK("leaf_counts");
  return TMD_OK;
}

// host entry points of the same key functions (tests, forest bookkeeping)
extern "C" uint64_t tmd_morton_key(uint32_t x, uint32_t y, uint32_t z, int32_t depth) { return morton3(x, y, z, depth); }
extern "C" uint64_t tmd_hilbert_key(uint32_t x, uint32_t y, uint32_t z, int32_t depth) {
  return hilbert3(x, y, z, depth);
}
