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
  for (int d = 0; d < 3; ++d)
    TMD_TRY(tmd_wrap_self(e->pos, ld, n, d, e->wrap_hi[d], e->wrap_lo[d], e->wrap_s_plus[d], e->wrap_s_minus[d],
                          stream));
  TMD_TRY(tmd_check_owned(e->pos, ld, n, e->slab_lo, e->slab_hi, e->status, stream));
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
    TMD_TRY(tmd_zero_rows(V, ld, 3, n, room, stream));
    TMD_TRY(tmd_zero_rows(e->vel, ld, 3, n, room, stream));
  }
  // the production grid over locals + ghosts
  const int32_t bdims[3] = {(int32_t)e->bin_dims[0], (int32_t)e->bin_dims[1], (int32_t)e->bin_dims[2]};
  TMD_TRY(tmd_bin_cells_dev(P, ld, n, n + room, d_k, e->bin_lo, e->bin_edge, bdims, (int32_t)e->bin_shell,
                            e->cell_of, e->cell_start, e->cell_atoms, e->status, stream));
  TMD_TRY(tmd_cell_positions_dev(P, ld, e->cell_atoms, n, n + room, d_k, e->cell_pos, e->ld_cp, stream));
  // the near/far split from the epoch's guard maxima
  if (e->margin_out)
    TMD_TRY(tmd_split_margin(e->dispmax2, (int32_t)e->margin_i0, (int32_t)e->margin_i1, e->margin_floor,
                             e->margin_factor, e->margin_cap, e->cutoff, e->margin_out, stream));
  // split rows
  TMD_TRY(tmd_status_reset(e->list_status, stream));
  TMD_TRY(tmd_build_lists_split(P, ld, n, e->cell_of, e->cell_start, e->cell_atoms, e->cell_pos, e->ld_cp, bdims,
                                (int32_t)e->bin_shell, e->near_rsq, e->margin_out, e->rsq_max, (int32_t)e->cap,
                                e->nbr, e->ld_nbr, e->nnear, e->counts, e->order, e->list_status, stream));
  TMD_TRY(tmd_copy_rows(P, ld, e->xref, e->ld_ref, 3, n, stream));
  // export table: ghost slot n + t mirrors root[t] with shift sh[:, t]
  return tmd_exports_build_dev(n, room, d_k, e->root, e->ex_zeros, e->ex_slots, e->sh, e->ld_sh, e->ex_start,
                               e->ex_rank, e->ex_slot, e->ex_sh, e->ld_o, e->status, stream);
}
