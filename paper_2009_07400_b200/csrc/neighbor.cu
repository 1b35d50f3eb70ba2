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

__global__ void __launch_bounds__(128) k_build_lists(
    const double* __restrict__ pos, int64_t ld, int32_t n_local, Cells C, double rsq_max, int half,
    int32_t cap, int32_t* __restrict__ nbr, int64_t ld_nbr, int32_t* __restrict__ nnbr,
    int64_t* __restrict__ st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  int32_t cnt = 0;
  for_candidates(pos, ld, i, n_local, half, C.cell_of, C.cell_start, C.cell_atoms, C.cp, C.ld_cp, C.g,
                 [&](int32_t j, double rsq) {
                   if (rsq < rsq_max) {
                     if (cnt < cap) nbr[slot_index(cnt, i, ld_nbr)] = j;
                     ++cnt;
                   }
                 });
  nnbr[i] = cnt;
  if (cnt > cap) {
    need_capacity(st, cnt);
    return;
  }
  for (int32_t k = cnt; k & 3; ++k) nbr[slot_index(k, i, ld_nbr)] = i;  // pad the quad
}

constexpr int kMaxTiers = 8;

struct Tiers {
  double r2[kMaxTiers];  // ascending squared tier radii, padded with the list radius^2
  int nt;
};

// pass 1: cumulative count per tier (tcnt) and total (nnbr); pass 2: bucketed write.
template <bool WRITE>
__global__ void __launch_bounds__(128) k_build_tiered(
    const double* __restrict__ pos, int64_t ld, int32_t n_local, Cells C, Tiers T, int32_t cap,
    int32_t* __restrict__ nbr, int64_t ld_nbr, int32_t* __restrict__ tcnt, int32_t* __restrict__ nnbr,
    int64_t* __restrict__ st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  // tier radii in registers (the kernel-parameter copy is not addressable)
  double r2[kMaxTiers];
  int32_t c[kMaxTiers];
#pragma unroll
  for (int q = 0; q < kMaxTiers; ++q) {
    r2[q] = T.r2[q];
    c[q] = 0;
  }
  const double rsq_max = r2[kMaxTiers - 1];
  if (WRITE) {
    // write cursors: tier t starts after all nearer tiers
#pragma unroll
    for (int q = 1; q < kMaxTiers; ++q)
      if (q < T.nt) c[q] = tcnt[(int64_t)(q - 1) * ld_nbr + i];
  }
  for_candidates(pos, ld, i, n_local, 0, C.cell_of, C.cell_start, C.cell_atoms, C.cp, C.ld_cp, C.g,
                 [&](int32_t j, double rsq) {
                   if (rsq < rsq_max) {
#pragma unroll
                     for (int q = 0; q < kMaxTiers; ++q) {
                       // the first tier whose radius holds rsq (padding tiers repeat the last)
                       const bool here = rsq < r2[q] && (q == 0 || !(rsq < r2[q > 0 ? q - 1 : 0]));
                       if (here) {
                         if (WRITE) nbr[slot_index(c[q], i, ld_nbr)] = j;
                         ++c[q];
                       }
                     }
                   }
                 });
  if (!WRITE) {
    int32_t run = 0;
#pragma unroll
    for (int q = 0; q < kMaxTiers; ++q) {
      run += c[q];
      if (q < T.nt) tcnt[(int64_t)q * ld_nbr + i] = run;
    }
    nnbr[i] = run;
    if (run > cap) need_capacity(st, run);
  } else {
    const int32_t cnt = nnbr[i];
    for (int32_t k = cnt; k & 3; ++k) nbr[slot_index(k, i, ld_nbr)] = i;  // pad the quad
  }
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
  if (!h_dims || !d_cell_pos || !make_tiers(h_tier_r2, n_tiers, &T) || cap < 0 || ld_nbr < n_local)
    return TMD_ERR_ARG;
  const int B = 128;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims);
  k_build_tiered<false><<<grid_for(n_local, B), B, 0, as_stream(stream)>>>(d_pos, ld, n_local, C, T, cap,
                                                                          d_nbr, ld_nbr, d_tcnt, d_nnbr,
                                                                          d_status);
  TMD_LAUNCH_CHECK("build_lists_tiered count");
  return TMD_OK;
}

extern "C" int tmd_build_lists_tiered_fill(const double* d_pos, int64_t ld, int32_t n_local,
                                           const int32_t* d_cell_of, const int32_t* d_cell_start,
                                           const int32_t* d_cell_atoms, const double* d_cell_pos,
                                           int64_t ld_cp, const int32_t* h_dims, const double* h_tier_r2,
                                           int32_t n_tiers, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                                           const int32_t* d_tcnt, const int32_t* d_nnbr, void* stream) {
  if (n_local <= 0) return TMD_OK;
  Tiers T;
  if (!h_dims || !d_cell_pos || !make_tiers(h_tier_r2, n_tiers, &T) || ld_nbr < n_local) return TMD_ERR_ARG;
  const int B = 128;
  Cells C = make_cells(d_cell_of, d_cell_start, d_cell_atoms, d_cell_pos, ld_cp, h_dims);
  k_build_tiered<true><<<grid_for(n_local, B), B, 0, as_stream(stream)>>>(
      d_pos, ld, n_local, C, T, cap, d_nbr, ld_nbr, const_cast<int32_t*>(d_tcnt),
      const_cast<int32_t*>(d_nnbr), nullptr);
  TMD_LAUNCH_CHECK("build_lists_tiered fill");
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
