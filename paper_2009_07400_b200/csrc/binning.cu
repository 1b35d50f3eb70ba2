// K1 — cell binning as a counting sort (reference: build_cell_grid, neighbor.py:58-89).
//
//   pass 1  cell id per atom (IEEE floor((p - lo) / r)), shell check, histogram
//   pass 2  exclusive scan of the histogram -> cell_start
//   pass 3  scatter atoms into their cell's segment (atomic slot)
//   pass 4  sort every segment ascending, which reproduces the reference's
//           stable argsort order inside a cell
#include "tmd_common.cuh"

namespace tmd {

struct Grid3 {
  int g0, g1, g2;  // dims including the ghost shell (interior + 2 * shell)
  int shell;       // shell layers: 1 for the reference grid (cell = r), 2 for the r/2 grid
};

__global__ void k_cell_ids(const double* __restrict__ pos, int64_t ld, int32_t n, double lo0,
                           double lo1, double lo2, double r, int d0, int d1, int d2, Grid3 g,
                           int32_t* __restrict__ cell_of, int32_t* __restrict__ count,
                           int64_t* __restrict__ st, const int32_t* __restrict__ d_add) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (d_add) n += *d_add;  // device-side count (n = n0 + *d_add; grid sized for the maximum)
  if (i >= n) return;
  // neighbor.py:67: floor((pos - lo) / r), IEEE division
  double c0 = floor(div_rn(sub_rn(pos[i], lo0), r));
  double c1 = floor(div_rn(sub_rn(pos[ld + i], lo1), r));
  double c2 = floor(div_rn(sub_rn(pos[2 * ld + i], lo2), r));
  // neighbor.py:68-75: beyond the ghost shell (NaN counts as outside)
  const double lo_c = -(double)g.shell;
  bool ok = (c0 >= lo_c && c0 <= (double)(d0 + g.shell - 1)) && (c1 >= lo_c && c1 <= (double)(d1 + g.shell - 1)) &&
            (c2 >= lo_c && c2 <= (double)(d2 + g.shell - 1));
  if (!ok) {
    raise_status(st, TMD_PROTOCOL, (unsigned long long)i);
    cell_of[i] = -1;
    return;
  }
  int cid = (((int)c0 + g.shell) * g.g1 + ((int)c1 + g.shell)) * g.g2 + ((int)c2 + g.shell);
  cell_of[i] = cid;
  atomicAdd(&count[cid], 1);
}

__global__ void k_scatter_cells(const int32_t* __restrict__ cell_of, int32_t n,
                                const int32_t* __restrict__ start, int32_t* __restrict__ fill,
                                int32_t* __restrict__ atoms, const int32_t* __restrict__ d_add) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (d_add) n += *d_add;
  if (i >= n) return;
  int cid = cell_of[i];
  if (cid < 0) return;
  int slot = atomicAdd(&fill[cid], 1);
  atoms[start[cid] + slot] = i;
}

// One thread per cell; segments are short (tens of atoms), insertion sort.
__global__ void k_sort_cells(const int32_t* __restrict__ start, int32_t n_cells,
                             int32_t* __restrict__ atoms) {
  int32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n_cells) return;
  int32_t b = start[c], e = start[c + 1];
  for (int32_t k = b + 1; k < e; ++k) {
    int32_t v = atoms[k];
    int32_t q = k - 1;
    while (q >= b && atoms[q] > v) {
      atoms[q + 1] = atoms[q];
      --q;
    }
    atoms[q + 1] = v;
  }
}

// Positions in cell order (cell_pos[c * ld_cp + k] = pos[c][cell_atoms[k]]):
// the list builders then stream a stencil run's candidate positions
// contiguously instead of chasing cell_atoms[k] -> pos[j] per candidate.
__global__ void k_cell_positions(const double* __restrict__ pos, int64_t ld,
                                 const int32_t* __restrict__ atoms, int32_t n,
                                 double* __restrict__ cell_pos, int64_t ld_cp, float* __restrict__ cell_pos_f,
                                 const int32_t* __restrict__ d_add) {
  int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (d_add) n += *d_add;
  if (k >= n) return;
  const int32_t j = atoms[k];
  // an atom rejected by the shell check leaves its slot unset: never chase it
  // (the rejection is already in the status word)
  const bool ok = (uint32_t)j < (uint32_t)n;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const double v = ok ? pos[q * ld + j] : 0.0;
    cell_pos[q * ld_cp + k] = v;
    if (cell_pos_f) cell_pos_f[q * ld_cp + k] = __double2float_rn(v);
  }
}

// dst[c][t] = src[c][perm[t]] for c < ncomp (cell-order permutation of the locals)
__global__ void k_permute_rows(const double* __restrict__ src, int64_t ld_src, const int32_t* __restrict__ perm,
                               int32_t n, double* __restrict__ dst, int64_t ld_dst, int ncomp) {
  int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int32_t j = perm[t];
  const bool ok = (uint32_t)j < (uint32_t)n;  // see k_cell_positions
  for (int q = 0; q < ncomp; ++q) dst[q * ld_dst + t] = ok ? src[q * ld_src + j] : 0.0;
}

// Brick-major order of the locals for the shared-memory step kernel: cells of
// edge w (the production r/2 grid) grouped into bricks of 4 x 4 x 4 cells;
// key = brick * 64 + cell-in-brick (z fastest).  Same cell formula as
// k_cell_ids, clamped to the interior (a local can only round onto the
// upper face of the slab, and the list builder checks every candidate
// against its brick's staging range).
__global__ void k_brick_keys(const double* __restrict__ pos, int64_t ld, int32_t n, double lo0, double lo1,
                             double lo2, double w, int d0, int d1, int d2, int nb1, int nb2, int sx, int sy, int sz,
                             int32_t* __restrict__ key, int32_t* __restrict__ count) {
  int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double c0 = floor(div_rn(sub_rn(pos[i], lo0), w));
  const double c1 = floor(div_rn(sub_rn(pos[ld + i], lo1), w));
  const double c2 = floor(div_rn(sub_rn(pos[2 * ld + i], lo2), w));
  const int x = min(max((int)fmax(c0, 0.0), 0), d0 - 1);
  const int y = min(max((int)fmax(c1, 0.0), 0), d1 - 1);
  const int z = min(max((int)fmax(c2, 0.0), 0), d2 - 1);
  // brick of 2^sx x 2^sy x 2^sz cells, cells z-fastest inside
  const int b = ((x >> sx) * nb1 + (y >> sy)) * nb2 + (z >> sz);
  const int k = (b << (sx + sy + sz)) + ((((x & ((1 << sx) - 1)) << sy) + (y & ((1 << sy) - 1))) << sz) +
                (z & ((1 << sz) - 1));
  key[i] = k;
  atomicAdd(&count[k], 1);
}

// inv[perm[k]] = k; out[t] = inv[idx[t]]
__global__ void k_invert(const int32_t* __restrict__ perm, int32_t n, int32_t* __restrict__ inv) {
  const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) inv[perm[k]] = k;
}

__global__ void k_gather_i32(const int32_t* __restrict__ src, const int32_t* __restrict__ idx, int32_t n,
                             int32_t* __restrict__ out) {
  const int32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) out[t] = src[idx[t]];
}

}  // namespace tmd

using namespace tmd;

extern "C" int tmd_brick_sort(const double* d_pos, int64_t ld, int32_t n_local, const double* h_lo, double w,
                              const int32_t* h_dims, const int32_t* h_shape, int32_t* d_key, int32_t* d_key_start,
                              int32_t* d_perm, void* stream) {
  if (w <= 0 || n_local < 0 || !h_lo || !h_dims) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  const int sx = h_shape ? h_shape[0] : 2, sy = h_shape ? h_shape[1] : 2, sz = h_shape ? h_shape[2] : 2;
  if (sx < 0 || sy < 0 || sz < 0 || sx + sy + sz > 12) return TMD_ERR_ARG;
  const int nb0 = (h_dims[0] + (1 << sx) - 1) >> sx, nb1 = (h_dims[1] + (1 << sy) - 1) >> sy,
            nb2 = (h_dims[2] + (1 << sz) - 1) >> sz;
  const int64_t n_keys = ((int64_t)nb0 * nb1 * nb2) << (sx + sy + sz);
  keep_pool_memory();
  int32_t* counts = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (size_t)(2 * n_keys + 1), s), "brick alloc");
  int32_t* fill = counts + n_keys;
  TMD_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)(2 * n_keys + 1), s), "brick memset");
  const int B = 256;
  if (n_local > 0) {
    k_brick_keys<<<grid_for(n_local, B), B, 0, s>>>(d_pos, ld, n_local, h_lo[0], h_lo[1], h_lo[2], w, h_dims[0],
                                                    h_dims[1], h_dims[2], nb1, nb2, sx, sy, sz, d_key, counts);
    TMD_LAUNCH_CHECK("brick keys");
  }
  int rc = scan_exclusive(counts, d_key_start, n_keys, s);
  if (rc != TMD_OK) return rc;
  if (n_local > 0) {
    k_scatter_cells<<<grid_for(n_local, B), B, 0, s>>>(d_key, n_local, d_key_start, fill, d_perm, nullptr);
    TMD_LAUNCH_CHECK("brick scatter");
    k_sort_cells<<<grid_for(n_keys, B), B, 0, s>>>(d_key_start, (int32_t)n_keys, d_perm);
    TMD_LAUNCH_CHECK("brick sort");
  }
  TMD_CUDA_TRY(cudaFreeAsync(counts, s), "brick free");
  return TMD_OK;
}

extern "C" int tmd_permute_rows(const double* d_src, int64_t ld_src, const int32_t* d_perm, int32_t n,
                                double* d_dst, int64_t ld_dst, int32_t ncomp, void* stream) {
  if (n <= 0) return TMD_OK;
  k_permute_rows<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(d_src, ld_src, d_perm, n, d_dst, ld_dst,
                                                                  ncomp);
  TMD_LAUNCH_CHECK("permute_rows");
  return TMD_OK;
}

extern "C" int tmd_compose_inverse(const int32_t* d_perm, const int32_t* d_idx, int32_t n, int32_t* d_out,
                                   void* stream) {
  if (n <= 0) return TMD_OK;
  cudaStream_t s = as_stream(stream);
  keep_pool_memory();
  int32_t* inv = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&inv), sizeof(int32_t) * (size_t)n, s), "compose_inverse");
  k_invert<<<grid_for(n, 256), 256, 0, s>>>(d_perm, n, inv);
  TMD_LAUNCH_CHECK("compose_inverse");
  k_gather_i32<<<grid_for(n, 256), 256, 0, s>>>(inv, d_idx, n, d_out);
  TMD_LAUNCH_CHECK("compose_inverse");
  TMD_CUDA_TRY(cudaFreeAsync(inv, s), "compose_inverse");
  return TMD_OK;
}

extern "C" int tmd_cell_positions(const double* d_pos, int64_t ld, const int32_t* d_cell_atoms,
                                  int32_t n_total, double* d_cell_pos, int64_t ld_cp, void* stream) {
  return tmd_cell_positions_dev(d_pos, ld, d_cell_atoms, n_total, n_total, nullptr, d_cell_pos, ld_cp, nullptr,
                                stream);
}

extern "C" int tmd_cell_positions_dev(const double* d_pos, int64_t ld, const int32_t* d_cell_atoms, int32_t n0,
                                      int32_t n_max, const int32_t* d_add, double* d_cell_pos, int64_t ld_cp,
                                      float* d_cell_pos_f, void* stream) {
  if (n_max <= 0) return TMD_OK;
  k_cell_positions<<<grid_for(n_max, 256), 256, 0, as_stream(stream)>>>(d_pos, ld, d_cell_atoms, n0, d_cell_pos,
                                                                        ld_cp, d_cell_pos_f, d_add);
  TMD_LAUNCH_CHECK("cell_positions");
  return TMD_OK;
}

extern "C" int tmd_bin_cells_ex(const double* d_pos, int64_t ld, int32_t n_total, const double* h_lo,
                                double r, const int32_t* h_dims, int32_t shell, int32_t* d_cell_of,
                                int32_t* d_cell_start, int32_t* d_cell_atoms, int64_t* d_status,
                                void* stream) {
  return tmd_bin_cells_dev(d_pos, ld, n_total, n_total, nullptr, h_lo, r, h_dims, shell, d_cell_of, d_cell_start,
                           d_cell_atoms, d_status, stream);
}

extern "C" int tmd_bin_cells_dev(const double* d_pos, int64_t ld, int32_t n0, int32_t n_max, const int32_t* d_add,
                                 const double* h_lo, double r, const int32_t* h_dims, int32_t shell,
                                 int32_t* d_cell_of, int32_t* d_cell_start, int32_t* d_cell_atoms,
                                 int64_t* d_status, void* stream) {
  if (r <= 0 || n0 < 0 || n_max < n0 || !h_lo || !h_dims || shell < 1) return TMD_ERR_ARG;
  cudaStream_t s = as_stream(stream);
  Grid3 g{h_dims[0] + 2 * shell, h_dims[1] + 2 * shell, h_dims[2] + 2 * shell, shell};
  int64_t n_cells = (int64_t)g.g0 * g.g1 * g.g2;
  keep_pool_memory();
  int32_t* counts = nullptr;
  TMD_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (size_t)(2 * n_cells + 1), s), "bin alloc");
  int32_t* fill = counts + n_cells;
  TMD_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)(2 * n_cells + 1), s), "bin memset");
  const int B = 256;
  if (n_max > 0) {
    k_cell_ids<<<grid_for(n_max, B), B, 0, s>>>(d_pos, ld, n0, h_lo[0], h_lo[1], h_lo[2], r, h_dims[0], h_dims[1],
                                                h_dims[2], g, d_cell_of, counts, d_status, d_add);
    TMD_LAUNCH_CHECK("bin_cells ids");
  }
  int rc = scan_exclusive(counts, d_cell_start, n_cells, s);
  if (rc != TMD_OK) return rc;
  if (n_max > 0) {
    k_scatter_cells<<<grid_for(n_max, B), B, 0, s>>>(d_cell_of, n0, d_cell_start, fill, d_cell_atoms, d_add);
    TMD_LAUNCH_CHECK("bin_cells scatter");
    k_sort_cells<<<grid_for(n_cells, B), B, 0, s>>>(d_cell_start, (int32_t)n_cells, d_cell_atoms);
    TMD_LAUNCH_CHECK("bin_cells sort");
  }
  TMD_CUDA_TRY(cudaFreeAsync(counts, s), "bin free");
  return TMD_OK;
}

extern "C" int tmd_bin_cells(const double* d_pos, int64_t ld, int32_t n_total, const double* h_lo, double r,
                             const int32_t* h_dims, int32_t* d_cell_of, int32_t* d_cell_start,
                             int32_t* d_cell_atoms, int64_t* d_status, void* stream) {
  return tmd_bin_cells_ex(d_pos, ld, n_total, h_lo, r, h_dims, 1, d_cell_of, d_cell_start, d_cell_atoms,
                          d_status, stream);
}

// The production epoch's renumbering in one call (driver.Simulation._sort_locals):
// bin the locals at the r / shell grid, brick-sort them, compose the builder's
// thread -> atom map (cell order, in the new numbering) and permute x and v
// into the output buffers.
extern "C" int tmd_sort_locals(const double* d_pos, const double* d_vel, int64_t ld, int32_t n, const double* h_lo,
                               double edge, const int32_t* h_dims, int32_t shell, const int32_t* h_shape,
                               int32_t* d_cell_of, int32_t* d_cell_start, int32_t* d_cell_atoms, int32_t* d_key,
                               int32_t* d_key_start, int32_t* d_perm, int32_t* d_order, double* d_pos_out,
                               double* d_vel_out, int64_t* d_status, void* stream) {
  if (n <= 0) return TMD_OK;
  if (!d_pos || !d_vel || !d_pos_out || !d_vel_out || !d_order) return TMD_ERR_ARG;
  int rc = tmd_bin_cells_ex(d_pos, ld, n, h_lo, edge, h_dims, shell, d_cell_of, d_cell_start, d_cell_atoms, d_status,
                            stream);
  if (rc != TMD_OK) return rc;
  rc = tmd_brick_sort(d_pos, ld, n, h_lo, edge, h_dims, h_shape, d_key, d_key_start, d_perm, stream);
  if (rc != TMD_OK) return rc;
  rc = tmd_compose_inverse(d_perm, d_cell_atoms, n, d_order, stream);
  if (rc != TMD_OK) return rc;
  rc = tmd_permute_rows(d_pos, ld, d_perm, n, d_pos_out, ld, 3, stream);
  if (rc != TMD_OK) return rc;
  return tmd_permute_rows(d_vel, ld, d_perm, n, d_vel_out, ld, 3, stream);
}
