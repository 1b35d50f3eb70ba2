// K2b — staging tables for the shared-memory step kernel (built once per
// epoch, after the split rows).
//
// The step kernel runs one block per 256 consecutive (brick-numbered) locals.
// Their neighbours' positions are gathered ONCE per block per step into shared
// memory (the block's staging set: the union of its atoms' front-segment
// partners, ~1400 atoms at 80^3) instead of once per list entry through L1.
// Each front entry becomes a uint16 index into that set, and each row is
// reordered so that, while the 16 atoms of a half-warp walk their rows in
// lockstep, slot k of lane l reads fp64 bank pair (k + l) mod 16 where the row
// has such an entry: cycle m of a row holds its m-th entry of every class, in
// the rotated class order starting at class l.  Measured on the 80^3 lists
// (scripts/experiments/exp_smem2.py): L1 gathers 0.324 ms, staged in list
// order 0.301 ms, staged in this order 0.274 ms (front segments, forces only).
//
// Layouts: uniq[b * ustride + s] = atom of staging slot s of block b,
// ucount[b] = its size (<= ustride); idx16 octet-interleaved: slot k of local
// i at idx16[((k >> 3) * ld16 + i) * 8 + (k & 7)] (one uint4 per 8 slots).
// The back (far) segments stay int32 global indices (read only when the
// exact pruning cannot skip them).  A block whose staging set exceeds ustride
// raises TMD_CAPACITY (d_status[2] = its size): the caller falls back to the
// L1-gather kernel for that epoch.
#include "tmd_common.cuh"

namespace tmd {

constexpr int kStageBlock = 256;
constexpr int kHashBits = 12;  // 4096-slot hash set: < 50% full up to 2048 staged atoms
constexpr int kHashSlots = 1 << kHashBits;

__device__ __forceinline__ uint32_t stage_hash(int32_t j) {
  return ((uint32_t)j * 2654435761u) >> (32 - kHashBits);
}

__device__ __forceinline__ int32_t slot_of(const int32_t* keys, int32_t j) {
  uint32_t h = stage_hash(j);
  while (keys[h] != j) h = (h + 1) & (kHashSlots - 1);
  return (int32_t)h;
}

__global__ void __launch_bounds__(kStageBlock) k_stage_build(
    int32_t n_local, const int32_t* __restrict__ nbr, int64_t ld_nbr, const int32_t* __restrict__ nnear,
    int32_t fmax, int32_t ustride, int32_t* __restrict__ uniq, int32_t* __restrict__ ucount,
    uint16_t* __restrict__ idx16, int64_t ld16, int32_t* __restrict__ max_count, int64_t* __restrict__ st) {
  __shared__ int32_t keys[kHashSlots];
  __shared__ int32_t vals[kHashSlots];
  __shared__ int32_t warp_tot[kStageBlock / 32];
  __shared__ int32_t s_total;
  extern __shared__ uint16_t rowbuf[];  // 2 x fmax per thread: list order, then class buckets
  uint16_t* lst = rowbuf + (size_t)threadIdx.x * 2 * fmax;
  uint16_t* bkt = lst + fmax;
  const int32_t b = blockIdx.x;
  const int32_t i = b * kStageBlock + threadIdx.x;
  const bool live = i < n_local;
  const int32_t nn = live ? nnear[i] : 0;
  for (int h = threadIdx.x; h < kHashSlots; h += kStageBlock) keys[h] = -1;
  __syncthreads();
  // 1. the union of the block's front-segment partners
  for (int32_t k = 0; k < nn; ++k) {
    const int32_t j = nbr[slot_index(k, i, ld_nbr)];
    uint32_t h = stage_hash(j);
    while (true) {
      const int32_t old = atomicCAS(&keys[h], -1, j);
      if (old == -1 || old == j) break;
      h = (h + 1) & (kHashSlots - 1);
    }
  }
  __syncthreads();
  // 2. compaction: staging slots in hash order (block scan of occupied counts)
  constexpr int kPer = kHashSlots / kStageBlock;
  const int h0 = threadIdx.x * kPer;
  int32_t mine = 0;
#pragma unroll
  for (int u = 0; u < kPer; ++u) mine += keys[h0 + u] >= 0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int32_t inc = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int32_t t = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) warp_tot[wid] = inc;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t run = 0;
    for (int w = 0; w < kStageBlock / 32; ++w) {
      const int32_t t = warp_tot[w];
      warp_tot[w] = run;
      run += t;
    }
    s_total = run;
  }
  __syncthreads();
  int32_t s = warp_tot[wid] + inc - mine;
  const int32_t total = s_total;
#pragma unroll
  for (int u = 0; u < kPer; ++u) {
    const int32_t j = keys[h0 + u];
    if (j >= 0) {
      vals[h0 + u] = s;
      if (s < ustride) uniq[(int64_t)b * ustride + s] = j;
      ++s;
    }
  }
  if (threadIdx.x == 0) {
    ucount[b] = total;
    atomicMax(max_count, total);
    if (total > ustride) need_capacity(st, total);
  }
  __syncthreads();
  if (!live) return;
  // 3. the row as staging indices, counted by bank class (s mod 16)
  uint32_t cnt[16];
#pragma unroll
  for (int c = 0; c < 16; ++c) cnt[c] = 0;
  for (int32_t k = 0; k < nn; ++k) {
    const int32_t j = nbr[slot_index(k, i, ld_nbr)];
    const int32_t sv = vals[slot_of(keys, j)];
    lst[k] = (uint16_t)sv;
#pragma unroll
    for (int c = 0; c < 16; ++c) cnt[c] += (sv & 15) == c;
  }
  // 4. bucket by class, then emit cycle by cycle in the rotated class order
  uint32_t off[16], run[16], maxc = 0;
  uint32_t acc = 0;
#pragma unroll
  for (int c = 0; c < 16; ++c) {
    off[c] = acc;
    run[c] = acc;
    acc += cnt[c];
    maxc = cnt[c] > maxc ? cnt[c] : maxc;
  }
  for (int32_t k = 0; k < nn; ++k) {
    const uint16_t sv = lst[k];
    const int c = sv & 15;
    uint32_t p = 0;
#pragma unroll
    for (int q = 0; q < 16; ++q)
      if (q == c) p = run[q]++;
    bkt[p] = sv;
  }
  const int l16 = i & 15;
  int32_t k = 0;
  for (uint32_t m = 0; m < maxc; ++m) {
#pragma unroll
    for (int r = 0; r < 16; ++r) {
      const int c = (r + l16) & 15;
      uint32_t cc = 0, oc = 0;
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (q == c) {
          cc = cnt[q];
          oc = off[q];
        }
      if (m < cc) lst[k++] = bkt[oc + m];
    }
  }
  for (; k & 7; ++k) lst[k] = 0;  // pad the last octet with slot 0 (a valid address, masked)
  // 5. out as whole octets
  uint4* out = reinterpret_cast<uint4*>(idx16);
  for (int32_t q = 0; q < (k >> 3); ++q) {
    const uint16_t* e = lst + 8 * q;
    out[(int64_t)q * ld16 + i] = make_uint4(e[0] | ((uint32_t)e[1] << 16), e[2] | ((uint32_t)e[3] << 16),
                                            e[4] | ((uint32_t)e[5] << 16), e[6] | ((uint32_t)e[7] << 16));
  }
}

}  // namespace tmd

using namespace tmd;

extern "C" int tmd_stage_build(int32_t n_local, const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnear,
                               int32_t cap, int32_t ustride, int32_t* d_uniq, int32_t* d_ucount, uint16_t* d_idx16,
                               int64_t ld16, int32_t* d_max_count, int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!d_nbr || !d_nnear || !d_uniq || !d_ucount || !d_idx16 || !d_max_count || ld_nbr < n_local || ld16 < n_local ||
      ustride < 1 || ustride > 65536 || cap < 1)
    return TMD_ERR_ARG;
  const int32_t fmax = (cap + 7) & ~7;  // the front segment is at most the row width
  const size_t smem = sizeof(uint16_t) * 2 * (size_t)fmax * kStageBlock;
  if (smem > 180 * 1024) return TMD_ERR_ARG;
  static bool attr = false;
  if (!attr) {
    TMD_CUDA_TRY(cudaFuncSetAttribute(k_stage_build, cudaFuncAttributeMaxDynamicSharedMemorySize, 180 * 1024),
                 "stage_build smem attribute");
    attr = true;
  }
  cudaStream_t s = as_stream(stream);
  TMD_CUDA_TRY(cudaMemsetAsync(d_max_count, 0, sizeof(int32_t), s), "stage_build");
  const int blocks = (n_local + kStageBlock - 1) / kStageBlock;
  k_stage_build<<<blocks, kStageBlock, smem, s>>>(n_local, d_nbr, ld_nbr, d_nnear, fmax, ustride, d_uniq, d_ucount,
                                                  d_idx16, ld16, d_max_count, d_status);
  TMD_LAUNCH_CHECK("stage_build");
  return TMD_OK;
}
