// K2 — Verlet-list build over the 27-cell stencil (reference: _fill_lists /
// build_neighbor_lists, neighbor.py:92-194) and K6 — displacement since the
// last rebuild (max_displacement_since_rebuild, neighbor.py:197-206).
//
// List layout (both builders): "quad-interleaved neighbor-major".  Slot k of
// local i lives at nbr[((k >> 2) * ld_nbr + i) * 4 + (k & 3)]: the four slots
// 4q..4q+3 of an atom are one 16-byte int4, and the int4s of 32 consecutive
// atoms are one contiguous 512-byte run, so a warp fetches four candidates per
// atom with one fully coalesced vector load.  Unused slots of the last quad
// hold i itself (a valid address, masked by the count).
//
// The 27-cell stencil is walked as 9 contiguous runs of the cell table: for a
// fixed (dx, dy), the cells dz = -1, 0, +1 have consecutive ids, so their atoms
// are one range of cell_atoms (ascending inside each cell) — exactly the
// reference's candidate order (neighbor.py:30-33, 81-86, 127-131).
//
//  * reference order (tmd_build_lists): rows identical slot for slot to the
//    reference; the rsq predicate is evaluated in the reference's operation
//    order, so membership is bit-exact.
//  * tiered order (tmd_build_lists_tiered, production): same membership,
//    rows bucketed by distance tier R_t = rc + m_t (m_t <= skin) and the
//    cumulative count per tier stored in tcnt[t * ld_nbr + i].  A force pass
//    whose atoms moved at most d since the build only needs the prefix of
//    tier t with m_t >= 2 d: every pair beyond it is farther than rc.
#include "tmd_common.cuh"

namespace tmd {

struct Stencil {
  int g0, g1, g2;
};

// Visit the candidates of local i in the reference's order; f(j, rsq) per candidate
// (rsq already in reference order), j != i for full lists, half rule applied.
// Candidate positions come from cell_pos (positions in cell order, written
// by tmd_cell_positions), so a run is a contiguous stream with no dependent
// index -> position load; the index is read only to test/record j.
template <typename F>
__device__ __forceinline__ void for_candidates(const double* __restrict__ pos, int64_t ld, int32_t i,
                                               int32_t n_local, int half, const int32_t* __restrict__ cell_of,
                                               const int32_t* __restrict__ cell_start,
                                               const int32_t* __restrict__ cell_atoms,
                                               const double* __restrict__ cp, int64_t ld_cp, Stencil g,
                                               F&& f) {
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int cid = cell_of[i];
  const int c2 = cid % g.g2, c1 = (cid / g.g2) % g.g1, c0 = cid / (g.g1 * g.g2);
  const int zlo = c2 > 0 ? c2 - 1 : 0, zhi = c2 + 1 < g.g2 ? c2 + 1 : g.g2 - 1;
  for (int a = c0 - 1; a <= c0 + 1; ++a) {
    if (a < 0 || a >= g.g0) continue;
    for (int b = c1 - 1; b <= c1 + 1; ++b) {
      if (b < 0 || b >= g.g1) continue;
      const int base = (a * g.g1 + b) * g.g2;
      const int32_t e = __ldg(cell_start + base + zhi + 1);
      int32_t k = __ldg(cell_start + base + zlo);
#pragma unroll 4
      for (; k < e; ++k) {
        const int32_t j = __ldg(cell_atoms + k);
        const double dx = sub_rn(xi, __ldg(cp + k));
        const double dy = sub_rn(yi, __ldg(cp + ld_cp + k));
        const double dz = sub_rn(zi, __ldg(cp + 2 * ld_cp + k));
        if (half ? !(j >= n_local || j > i) : (j == i)) continue;
        f(j, rsq_ref(dx, dy, dz));
      }
    }
  }
}

struct Cells {
  const int32_t* cell_of;
  const int32_t* cell_start;
  const int32_t* cell_atoms;
  const double* cp;  // positions in cell order
  int64_t ld_cp;
  Stencil g;
};

// Rows are written as whole int4 quads: four accepted candidates are packed
// in registers and stored together, so every 16-byte quad (and every 32-byte
// sector) is written once and completely.  Scattered 4-byte stores left
// sectors partially written long enough to be evicted from L2 once the list
// outgrew it, turning the list write into DRAM read-modify-write traffic.
struct QuadWriter {
  int4* out;  // quad q of atom i at out[q * ld + i]
  int64_t ld;
  int32_t i;
  int32_t a0, a1, a2, a3;
  __device__ __forceinline__ void put(int32_t o, int32_t j) {
    const int r = o & 3;
    a0 = r == 0 ? j : a0;
    a1 = r == 1 ? j : a1;
    a2 = r == 2 ? j : a2;
    a3 = r == 3 ? j : a3;
    if (r == 3) out[(int64_t)(o >> 2) * ld + i] = make_int4(a0, a1, a2, a3);
  }
  // pad the last partial quad with the atom itself (a valid, masked address)
  __device__ __forceinline__ void finish(int32_t o) {
    if (o & 3) {
      for (int32_t k = o; k & 3; ++k) put(k, i);
    }
  }
};

__global__ void __launch_bounds__(128) k_build_lists(
    const double* __restrict__ pos, int64_t ld, int32_t n_local, Cells C, double rsq_max, int half,
    int32_t cap, int32_t* __restrict__ nbr, int64_t ld_nbr, int32_t* __restrict__ nnbr,
    int64_t* __restrict__ st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  QuadWriter w{reinterpret_cast<int4*>(nbr), ld_nbr, i, i, i, i, i};
  int32_t cnt = 0;
  for_candidates(pos, ld, i, n_local, half, C.cell_of, C.cell_start, C.cell_atoms, C.cp, C.ld_cp, C.g,
                 [&](int32_t j, double rsq) {
                   if (rsq < rsq_max) {
                     if (cnt < cap) w.put(cnt, j);
                     ++cnt;
                   }
                 });
  nnbr[i] = cnt;
  if (cnt > cap) {
    need_capacity(st, cnt);
    return;
  }
  w.finish(cnt);
}

constexpr int kMaxTiers = 8;
constexpr int kTierShift = 28;  // rows staged as j | tier << 28 (n_total < 2^28)

struct Tiers {
  double r2[kMaxTiers];  // ascending squared tier radii, padded with the list radius^2
  int nt;
};

// Single pass: the accepted candidates of a row are staged in shared memory
// (slot k of thread t at sm[k * blockDim + t], bank-conflict free) with their
// tier, then emitted tier by tier as whole quads; cumulative tier counts go to
// tcnt[t * ld_nbr + i].
__global__ void k_build_tiered(const double* __restrict__ pos, int64_t ld, int32_t n_local, Cells C, Tiers T,
                               int32_t cap, int32_t* __restrict__ nbr, int64_t ld_nbr,
                               int32_t* __restrict__ tcnt, int32_t* __restrict__ nnbr,
                               int64_t* __restrict__ st) {
  extern __shared__ int32_t stage[];
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  const int B = blockDim.x, tid = threadIdx.x;
  double r2[kMaxTiers];
  int32_t tc[kMaxTiers];
#pragma unroll
  for (int q = 0; q < kMaxTiers; ++q) {
    r2[q] = T.r2[q];
    tc[q] = 0;
  }
  const double rsq_max = r2[kMaxTiers - 1];
  int32_t cnt = 0;
  for_candidates(pos, ld, i, n_local, 0, C.cell_of, C.cell_start, C.cell_atoms, C.cp, C.ld_cp, C.g,
                 [&](int32_t j, double rsq) {
                   if (rsq < rsq_max) {
                     int t = 0;
#pragma unroll
                     for (int q = 0; q < kMaxTiers - 1; ++q) t += (rsq < r2[q]) ? 0 : 1;
#pragma unroll
                     for (int q = 0; q < kMaxTiers; ++q) tc[q] += (q == t) ? 1 : 0;
                     if (cnt < cap) stage[cnt * B + tid] = j | (t << kTierShift);
                     ++cnt;
                   }
                 });
  nnbr[i] = cnt;
  if (cnt > cap) {
    need_capacity(st, cnt);
    return;
  }
  int32_t run = 0;
#pragma unroll
  for (int q = 0; q < kMaxTiers; ++q) {
    run += tc[q];
    if (q < T.nt) tcnt[(int64_t)q * ld_nbr + i] = run;
  }
  QuadWriter w{reinterpret_cast<int4*>(nbr), ld_nbr, i, i, i, i, i};
  int32_t o = 0;
#pragma unroll
  for (int q = 0; q < kMaxTiers; ++q) {
    int32_t left = tc[q];
    for (int32_t k = 0; left > 0 && k < cnt; ++k) {
      const int32_t v = stage[k * B + tid];
      if ((v >> kTierShift) == q) {
        w.put(o++, v & ((1 << kTierShift) - 1));
        --left;
      }
    }
  }
  w.finish(o);
}

__global__ void k_max_disp2(const double* __restrict__ pos, int64_t ld, const double* __restrict__ ref,
                            int64_t ld_ref, int32_t n, double* __restrict__ out) {
  double m = 0.0;
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double dx = sub_rn(pos[i], ref[i]);
    double dy = sub_rn(pos[ld + i], ref[ld_ref + i]);
    double dz = sub_rn(pos[2 * ld + i], ref[2 * ld_ref + i]);
    m = fmax(m, norm2_seq(dx, dy, dz));
  }
  m = warp_max(m);
  if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

}  // namespace tmd

using namespace tmd;

static Cells make_cells(const int32_t* cell_of, const int32_t* cell_start, const int32_t* cell_atoms,
                        const double* cell_pos, int64_t ld_cp, const int32_t* h_dims) {
  Cells C;
  C.cell_of = cell_of;
  C.cell_start = cell_start;
  C.cell_atoms = cell_atoms;
  C.cp = cell_pos;
  C.ld_cp = ld_cp;
  C.g = Stencil{h_dims[0] + 2, h_dims[1] + 2, h_dims[2] + 2};
  return C;
}

static bool make_tiers(const double* h_tier_r2, int32_t n_tiers, Tiers* T) {
  if (!h_tier_r2 || n_tiers < 1 || n_tiers > kMaxTiers) return false;
  for (int q = 0; q < kMaxTiers; ++q) T->r2[q] = h_tier_r2[q < n_tiers ? q : n_tiers - 1];
  T->nt = n_tiers;
  return true;
}

extern "C" int tmd_build_lists(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_cell_of,
                               const int32_t* d_cell_start, const int32_t* d_cell_atoms,
                               const double* d_cell_pos, int64_t ld_cp, const int32_t* h_dims,
                               double rsq_max, int32_t half, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                               int32_t* d_nnbr, int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!h_dims || !d_cell_pos || cap < 0 || ld_nbr < n_local) return TMD_ERR_ARG;
  const int B = 128;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims);
  k_build_lists<<<grid_for(n_local, B), B, 0, as_stream(stream)>>>(d_pos, ld, n_local, C, rsq_max, half,
                                                                   cap, d_nbr, ld_nbr, d_nnbr, d_status);
  TMD_LAUNCH_CHECK("build_lists");
  return TMD_OK;
}

extern "C" int tmd_build_lists_tiered(const double* d_pos, int64_t ld, int32_t n_local,
                                      const int32_t* d_cell_of, const int32_t* d_cell_start,
                                      const int32_t* d_cell_atoms, const double* d_cell_pos,
                                      int64_t ld_cp, const int32_t* h_dims, const double* h_tier_r2,
                                      int32_t n_tiers, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                                      int32_t* d_tcnt, int32_t* d_nnbr, int64_t* d_status,
                                      void* stream) {
  if (n_local <= 0) return TMD_OK;
  Tiers T;
  if (!h_dims || !d_cell_pos || !make_tiers(h_tier_r2, n_tiers, &T) || cap < 0 || ld_nbr < n_local ||
      ld_cp >= (1ll << kTierShift))
    return TMD_ERR_ARG;
  // block size from the staging budget: cap ints per thread
  int B = 128;
  while (B > 32 && (size_t)cap * B * 4 > 96 * 1024) B >>= 1;
  const size_t smem = (size_t)(cap > 0 ? cap : 1) * B * 4;
  if (smem > 200 * 1024) return TMD_ERR_ARG;
  TMD_CUDA_TRY(cudaFuncSetAttribute(k_build_tiered, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "build_lists_tiered smem");
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims);
  k_build_tiered<<<grid_for(n_local, B), B, smem, as_stream(stream)>>>(d_pos, ld, n_local, C, T, cap, d_nbr,
                                                                      ld_nbr, d_tcnt, d_nnbr, d_status);
  TMD_LAUNCH_CHECK("build_lists_tiered");
  return TMD_OK;
}

extern "C" int tmd_max_disp2(const double* d_pos, int64_t ld, const double* d_xref, int64_t ld_ref,
                             int32_t n, double* d_dispmax2, void* stream) {
  if (n <= 0) return TMD_OK;
  const int B = 256;
  int g = grid_for(n, B);
  if (g > 4 * sm_count()) g = 4 * sm_count();
  k_max_disp2<<<g, B, 0, as_stream(stream)>>>(d_pos, ld, d_xref, ld_ref, n, d_dispmax2);
  TMD_LAUNCH_CHECK("max_disp2");
  return TMD_OK;
}
