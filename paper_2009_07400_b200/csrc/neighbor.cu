// K2 — Verlet-list build over the 27-cell stencil (reference: _fill_lists /
// build_neighbor_lists, neighbor.py:92-194) and K6 — displacement since the
// last rebuild (max_displacement_since_rebuild, neighbor.py:197-206).
//
// One thread per local atom walks the stencil in the reference's order (dx
// slowest, dz fastest; ascending atom index inside a cell), so rows come out
// slot-for-slot identical to the reference; the rsq predicate is evaluated
// in the reference's operation order, so membership is bit-exact.  Rows are
// stored neighbor-major (slot k of atom i at nbr[k * ld_nbr + i]): a warp's
// 32 consecutive atoms write and later read one 128-byte line per slot.
#include "tmd_common.cuh"

namespace tmd {

__global__ void __launch_bounds__(128) k_build_lists(
    const double* __restrict__ pos, int64_t ld, int32_t n_local, const int32_t* __restrict__ cell_of,
    const int32_t* __restrict__ cell_start, const int32_t* __restrict__ cell_atoms, int g0, int g1,
    int g2, double rsq_max, int half, int32_t cap, int32_t* __restrict__ nbr, int64_t ld_nbr,
    int32_t* __restrict__ nnbr, int64_t* __restrict__ st) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_local) return;
  const double xi = pos[i], yi = pos[ld + i], zi = pos[2 * ld + i];
  const int cid = cell_of[i];
  const int c2 = cid % g2, c1 = (cid / g2) % g1, c0 = cid / (g1 * g2);
  int32_t cnt = 0;
  for (int a = c0 - 1; a <= c0 + 1; ++a) {
    if (a < 0 || a >= g0) continue;
    for (int b = c1 - 1; b <= c1 + 1; ++b) {
      if (b < 0 || b >= g1) continue;
      for (int c = c2 - 1; c <= c2 + 1; ++c) {
        if (c < 0 || c >= g2) continue;
        const int cell = (a * g1 + b) * g2 + c;
        const int32_t e = cell_start[cell + 1];
        for (int32_t k = cell_start[cell]; k < e; ++k) {
          const int32_t j = cell_atoms[k];
          if (half ? !(j >= n_local || j > i) : (j == i)) continue;
          const double dx = sub_rn(xi, pos[j]);
          const double dy = sub_rn(yi, pos[ld + j]);
          const double dz = sub_rn(zi, pos[2 * ld + j]);
          if (rsq_ref(dx, dy, dz) < rsq_max) {
            if (cnt < cap) nbr[(int64_t)cnt * ld_nbr + i] = j;
            ++cnt;
          }
        }
      }
    }
  }
  nnbr[i] = cnt;
  if (cnt > cap) need_capacity(st, cnt);
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

extern "C" int tmd_build_lists(const double* d_pos, int64_t ld, int32_t n_local,
                               const int32_t* d_cell_of, const int32_t* d_cell_start,
                               const int32_t* d_cell_atoms, const int32_t* h_dims, double rsq_max,
                               int32_t half, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                               int32_t* d_nnbr, int64_t* d_status, void* stream) {
  if (n_local <= 0) return TMD_OK;
  if (!h_dims || cap < 0 || ld_nbr < n_local) return TMD_ERR_ARG;
  const int B = 128;
  k_build_lists<<<grid_for(n_local, B), B, 0, as_stream(stream)>>>(
      d_pos, ld, n_local, d_cell_of, d_cell_start, d_cell_atoms, h_dims[0] + 2, h_dims[1] + 2,
      h_dims[2] + 2, rsq_max, half, cap, d_nbr, ld_nbr, d_nnbr, d_status);
  TMD_LAUNCH_CHECK("build_lists");
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
