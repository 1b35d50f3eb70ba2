// The production P = 1 epoch in one host call (driver.Simulation._rebuild_p1):
// the reference's _reneighbor (driver.py:102-112) -- exchange (periodic wrap,
// comm.py:340-400 with every peer being this rank), borders (comm.py:434-466),
// build_cell_grid (neighbor.py:58-89), build_neighbor_lists
// (neighbor.py:153-194) -- plus the production renumbering and the export
// table of the fused ghost refresh.  Every size that depends on the data (the
// ghost count) stays on the device; the host reads [status words, margin,
// ghost count] once afterwards.  The sequence and the arguments are exactly
// those of the Python device-count epoch, so both give the same state bit for
// bit (tests/test_gpu_parity.py).
#include "tmd_common.cuh"

namespace tmd {
// exchange at P = 1 in one pass: every dimension wrapped in place (the three
// self rounds of comm.py:340-400, tmd_wrap_self), then the half-open
// ownership check (tmd_check_owned) on the wrapped position
struct WrapAll {
  double hi[3], lo[3], sp[3], sm[3], slo[3], shi[3];
};

__global__ void k_wrap_all_check(double* __restrict__ pos, int64_t ld, int32_t n, WrapAll w, int64_t* st) {
  const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool in = true;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double x = pos[d * ld + i];
    if (x >= w.hi[d]) {
      x = add_rn(x, w.sp[d]);
      pos[d * ld + i] = x;
    } else if (x < w.lo[d]) {
      x = add_rn(x, w.sm[d]);
      pos[d * ld + i] = x;
    }
    in = in && x >= w.slo[d] && x < w.shi[d];
  }
  if (!in) raise_status(st, TMD_PROTOCOL, (unsigned long long)i);
}
}  // namespace tmd

#define TMD_TRY(call)                  \
  do {                                 \
    const int _rc = (call);            \
    if (_rc != TMD_OK) return _rc;     \
  } while (0)

extern "C" int tmd_epoch_p1(const TmdEpochP1* e, void* stream) {
  if (!e || e->n <= 0 || !e->pos || !e->pos_alt || !e->vel || !e->vel_alt || !e->status || !e->list_status)
    return TMD_ERR_ARG;
  const int32_t n = (int32_t)e->n;
  const int32_t room = (int32_t)e->room;
  const int64_t ld = e->ld;
  TMD_TRY(tmd_status_reset(e->status, stream));
  // exchange at P = 1: wrap every dimension in place, then the ownership check
  {
    tmd::WrapAll w;
    for (int d = 0; d < 3; ++d) {
      w.hi[d] = e->wrap_hi[d];
      w.lo[d] = e->wrap_lo[d];
      w.sp[d] = e->wrap_s_plus[d];
      w.sm[d] = e->wrap_s_minus[d];
      w.slo[d] = e->slab_lo[d];
      w.shi[d] = e->slab_hi[d];
    }
    tmd::k_wrap_all_check<<<tmd::grid_for(n, 256), 256, 0, tmd::as_stream(stream)>>>(e->pos, ld, n, w, e->status);
    TMD_LAUNCH_CHECK("epoch wrap");
  }
  // renumbering: x, v permuted into the alternate buffers (the caller swaps)
  const int32_t sdims[3] = {(int32_t)e->sort_dims[0], (int32_t)e->sort_dims[1], (int32_t)e->sort_dims[2]};
  const int32_t shape[3] = {(int32_t)e->sort_shape[0], (int32_t)e->sort_shape[1], (int32_t)e->sort_shape[2]};
  TMD_TRY(tmd_sort_locals(e->pos, e->vel, ld, n, e->sort_lo, e->sort_edge, sdims, (int32_t)e->sort_shell, shape,
                          e->sort_cell_of, e->sort_cell_start, e->sort_cell_atoms, e->sort_key, e->sort_key_start,
                          e->sort_perm, e->order, e->pos_alt, e->vel_alt, e->status, stream));
  double* P = e->pos_alt;
  double* V = e->vel_alt;
  // borders: copies into the reserved ghost slots, count at off[n] on the device
  TMD_TRY(tmd_borders_count(P, ld, n, e->thr_hi, e->thr_lo, e->off, stream));
  TMD_TRY(tmd_borders_fill_capped(P, ld, n, e->thr_hi, e->thr_lo, e->s_hi, e->s_lo, nullptr, e->off, P + n, ld, V + n,
                                  e->root, e->sh, e->ld_sh, nullptr, room, stream));
  const int32_t* d_k = e->off + n;
  if (e->sd && room > 0) {  // ghost velocities are 0 in both buffers (particles.py:148)
    for (double* v : {V, e->vel})
      TMD_CUDA_TRY(cudaMemset2DAsync(v + n, sizeof(double) * ld, 0, sizeof(double) * room, 3, tmd::as_stream(stream)),
                   "epoch zero ghost velocities");
  }
  // the production grid over locals + ghosts
  const int32_t bdims[3] = {(int32_t)e->bin_dims[0], (int32_t)e->bin_dims[1], (int32_t)e->bin_dims[2]};
  TMD_TRY(tmd_bin_cells_dev(P, ld, n, n + room, d_k, e->bin_lo, e->bin_edge, bdims, (int32_t)e->bin_shell,
                            e->cell_of, e->cell_start, e->cell_atoms, e->status, stream));
  TMD_TRY(tmd_cell_positions_dev(P, ld, e->cell_atoms, n, n + room, d_k, e->cell_pos, e->ld_cp, e->cell_pos_f,
                                   stream));
  // the near/far split from the epoch's guard maxima
  if (e->margin_out)
    TMD_TRY(tmd_split_margin(e->dispmax2, (int32_t)e->margin_i0, (int32_t)e->margin_i1, e->margin_floor,
                             e->margin_factor, e->margin_cap, e->cutoff, e->margin_out, stream));
  // split rows
  TMD_TRY(tmd_status_reset(e->list_status, stream));
  TMD_TRY(tmd_build_lists_split(P, ld, n, e->cell_of, e->cell_start, e->cell_atoms, e->cell_pos, e->ld_cp,
                                e->cell_pos_f, e->f32_eps, bdims,
                                (int32_t)e->bin_shell, e->near_rsq, e->margin_out, e->rsq_max, (int32_t)e->cap,
                                e->nbr, e->ld_nbr, e->nnear, e->counts, e->order, e->list_status, stream));
  TMD_TRY(tmd_copy_rows(P, ld, e->xref, e->ld_ref, 3, n, stream));
  // export table: ghost slot n + t mirrors root[t] with shift sh[:, t]
  return tmd_exports_build_dev(n, room, d_k, e->root, e->ex_zeros, e->ex_slots, e->sh, e->ld_sh, e->ex_start,
                               e->ex_rank, e->ex_slot, e->ex_sh, e->ld_o, e->status, stream);
}
