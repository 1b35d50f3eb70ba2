/*
 * tinymd_b200.h — C ABI of the B200 pairwise-interaction timestep library
 * (libtinymd_b200.so, built from the CUDA sources in paper_2009_07400_b200/csrc/ for sm_100a).
 *
 * The reference (nanopair, pure Python/numpy) has no FFI; these entry points are
 * what its step loop's operator calls become when bound through ctypes
 * (INTEGRATION.md shows the binding).  Each function names the reference
 * interface it replaces.
 *
 * Conventions
 *  - Every pointer named d_* is DEVICE memory owned by the caller (torch
 *    tensors in the Python host layer); h_* pointers are host memory read
 *    during the call only.  The library never frees or retains caller memory.
 *  - Per-atom vectors are SoA fp64 with a leading dimension: component c of
 *    atom i lives at d_pos[c * ld + i].  Locals occupy [0, n_local), ghosts
 *    [n_local, n_total) — the reference's ParticleStore layout
 *    (particles.py:1-6, 30-158).
 *  - Neighbor lists are int32, quad-interleaved neighbor-major: slot k of
 *    local i is at d_nbr[((k >> 2) * ld_nbr + i) * 4 + (k & 3)] — the
 *    reference's neighbor-major (column_major) list layout
 *    (neighbor.py:153-194, layout.py) with four slots packed per int4.  The
 *    buffer holds ceil(cap / 4) * ld_nbr int4; unused slots of an atom's last
 *    quad hold the atom itself.
 *  - All calls are asynchronous on `stream` (a cudaStream_t); they return
 *    TMD_OK or TMD_ERR_CUDA for launch failures (message: tmd_last_error()).
 *    Data-dependent failures are written to the caller's device status word
 *    d_status (int64[TMD_STATUS_WORDS]), reset with tmd_status_reset:
 *      d_status[0]  error code (atomicMax; TMD_* below)
 *      d_status[1]  smallest offending key (atomicMin): atom index, or
 *                   (local << 32 | slot) for TMD_SINGULARITY
 *      d_status[2]  required list capacity (atomicMax) for TMD_CAPACITY
 *  - Not re-entrant per stream; one host thread per device.
 */
#ifndef TINYMD_B200_H
#define TINYMD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TMD_OK 0
#define TMD_CAPACITY 1    /* list row overflow: rerun with cap >= d_status[2] (neighbor.py:176-181) */
#define TMD_PROTOCOL 2    /* atom beyond ghost shell / outside ownership (neighbor.py:68-75, comm.py:394-400) */
#define TMD_SINGULARITY 3 /* rsq == 0 inside the cutoff (potential.py:174-178) */
#define TMD_GUARD 4       /* displacement >= buffer / 2 (driver.py:115-125) */
#define TMD_ERR_CUDA 5
#define TMD_ERR_ARG 6

#define TMD_STATUS_WORDS 4

/* force-kernel flags */
#define TMD_F_ENERGY 1u   /* also reduce PE and virial into d_thermo[0..1] */
#define TMD_F_EXACT 2u    /* reference operation order, bitwise equal forces */
#define TMD_F_STORE_FORCES 4u /* tmd_step_lj: also store F into d_frc (the fused path never reads it) */
#define TMD_F_NO_PRUNE 8u     /* tmd_step_lj: scan both segments of every split row (tests) */
#define TMD_F_SKIP_FORCES 16u /* tmd_step_*: no force pass; the NEXT phase kicks with d_frc (stored by the
                                 previous launch, TMD_F_STORE_FORCES): splits a step so its state can be read */

/* selection predicates for halo compaction (comm.py:242-256) */
#define TMD_SEL_GE 0 /* x_d >= thr  (exchange, + face) */
#define TMD_SEL_LT 1 /* x_d <  thr  (exchange, - face; border, - face) */
#define TMD_SEL_GT 2 /* x_d >  thr  (border, + face) */
#define TMD_SEL_IN 3 /* thr <= x_d < thr2 (exchange survivors) */

int tmd_version(void);
const char* tmd_last_error(void);
/* number of kernels this library has launched in the process */
int64_t tmd_launch_count(void);
int tmd_device_info(int* sm_count, int* cc_major, int* cc_minor, int64_t* l2_bytes);

/* Reset d_status to "no error". */
int tmd_status_reset(int64_t* d_status, void* stream);

/* ---- cell binning: build_cell_grid (neighbor.py:58-89) --------------------
 * Counting sort of [0, n_total) into cells of edge r over the rank box
 * (origin h_lo) plus one ghost shell; h_dims = interior cells per axis
 * (max(1, ceil(ext / r - 1e-12)), computed by the caller as the reference
 * does).  cell id = ((cx+1) * gy + cy+1) * gz + cz+1 with g = dims + 2 and
 * c = floor((p - lo) / r) in IEEE division.  Outputs: d_cell_of[n_total],
 * d_cell_start[n_cells + 1] (exclusive prefix of counts), d_cell_atoms[n_total]
 * (atoms grouped by cell, ascending index inside a cell = the reference's
 * stable argsort).  An atom outside the shell sets TMD_PROTOCOL. */
int tmd_bin_cells(const double* d_pos, int64_t ld, int32_t n_total, const double* h_lo, double r,
                  const int32_t* h_dims, int32_t* d_cell_of, int32_t* d_cell_start,
                  int32_t* d_cell_atoms, int64_t* d_status, void* stream);
/* Same with cell edge `r` and `shell` ghost layers (coordinates -shell ..
 * dims + shell - 1 accepted); tmd_bin_cells is shell = 1. */
int tmd_bin_cells_ex(const double* d_pos, int64_t ld, int32_t n_total, const double* h_lo, double r,
                     const int32_t* h_dims, int32_t shell, int32_t* d_cell_of, int32_t* d_cell_start,
                     int32_t* d_cell_atoms, int64_t* d_status, void* stream);

/* Positions in cell order: d_cell_pos[c * ld_cp + k] = pos[c][d_cell_atoms[k]]
 * (input of the list builders: candidate positions are then streamed). */
int tmd_cell_positions(const double* d_pos, int64_t ld, const int32_t* d_cell_atoms, int32_t n_total,
                       double* d_cell_pos, int64_t ld_cp, void* stream);

/* Device-count variants (the P = 1 epoch without a host sync on the ghost
 * count): the atom count is n0 + *d_add (d_add on the device, NULL = n0),
 * at most n_max; grids are sized for n_max and threads past the count exit. */
int tmd_bin_cells_dev(const double* d_pos, int64_t ld, int32_t n0, int32_t n_max, const int32_t* d_add,
                      const double* h_lo, double r, const int32_t* h_dims, int32_t shell, int32_t* d_cell_of,
                      int32_t* d_cell_start, int32_t* d_cell_atoms, int64_t* d_status, void* stream);
/* d_cell_pos_f (optional, float, same ld_cp): the positions rounded to
 * float as well -- the split builder's candidate pre-filter. */
int tmd_cell_positions_dev(const double* d_pos, int64_t ld, const int32_t* d_cell_atoms, int32_t n0, int32_t n_max,
                           const int32_t* d_add, double* d_cell_pos, int64_t ld_cp, float* d_cell_pos_f,
                           void* stream);

/* dst[c][t] = src[c][perm[t]], c < ncomp: reorders the locals into cell order
 * at a rebuild (production path; the store order is free there, results are
 * compared as sorted sets). */
int tmd_permute_rows(const double* d_src, int64_t ld_src, const int32_t* d_perm, int32_t n, double* d_dst,
                     int64_t ld_dst, int32_t ncomp, void* stream);

/* ---- Verlet lists: build_neighbor_lists (neighbor.py:92-194) --------------
 * Row of local i = atoms j of the 27 stencil cells (dx slowest, dz fastest;
 * ascending index inside a cell) with rsq < rsq_max, rsq evaluated in the
 * reference's order (dx*dx + dz*dz) + dy*dy; full lists drop j == i, half
 * lists keep j >= n_local || j > i.  d_nnbr gets the true count; a row longer
 * than cap sets TMD_CAPACITY with the needed length in d_status[2]. */
int tmd_build_lists(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_cell_of,
                    const int32_t* d_cell_start, const int32_t* d_cell_atoms, const double* d_cell_pos,
                    int64_t ld_cp, const int32_t* h_dims, double rsq_max, int32_t half, int32_t cap,
                    int32_t* d_nbr, int64_t ld_nbr, int32_t* d_nnbr, int64_t* d_status, void* stream);

/* Production variant ("split rows"): same membership; the grid may have cells
 * of edge r / shell with `shell` ghost layers (stencil (2 shell + 1)^3 cells —
 * the production path bins at r / 2, ~256 instead of ~443 candidates per
 * atom).  Pairs with rsq < near_rsq fill the row from the front (slots
 * [0, d_nnear[i])), the others from the back (slots [cap4 - far, cap4),
 * cap4 = round_up(cap, 4), far = d_nnbr[i] - d_nnear[i]); order inside a
 * segment is stencil order.  TMD_CAPACITY reports round4(near) + round4(far)
 * when it exceeds cap4.  One pass; the partial quads at the two segment
 * ends are padded with the atom itself.  d_order (n_local,
 * optional): builder thread t builds the row of local d_order[t] -- the
 * locals in cell order, so warps walk coherent stencil runs even when the
 * rows (the atoms) are numbered in another order (brick-major).  d_near_rsq
 * (optional): near_rsq read from device memory instead (tmd_split_margin).
 * d_cell_pos_f (optional; tmd_cell_positions_dev): float copies of the
 * candidate positions.  A candidate whose float squared distance is farther
 * than f32_eps from both thresholds is decided on it; the rest (and a NaN)
 * are recomputed in double with the reference's rounding, so the rows are
 * the same as without the copies.  f32_eps must bound the float error:
 * tinymd_f32_eps() in neighbor.py. */
int tmd_build_lists_split(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_cell_of,
                          const int32_t* d_cell_start, const int32_t* d_cell_atoms, const double* d_cell_pos,
                          int64_t ld_cp, const float* d_cell_pos_f, double f32_eps, const int32_t* h_dims,
                          int32_t shell, double near_rsq,
                          const double* d_near_rsq, double rsq_max, int32_t cap, int32_t* d_nbr, int64_t ld_nbr,
                          int32_t* d_nnear, int32_t* d_nnbr, const int32_t* d_order, int64_t* d_status,
                          void* stream);

/* The near/far split for the next build from the guard maxima d_dispmax2[i0,
 * i1) of the epoch's steps: margin = min(max(floor_margin, factor *
 * sqrt(max)), cap); d_out[0] = (cutoff + margin)^2 (pass as d_near_rsq),
 * d_out[1] = margin.  The epoch can then enqueue the build before reading the
 * maxima back. */
int tmd_split_margin(const double* d_dispmax2, int32_t i0, int32_t i1, double floor_margin, double factor,
                     double cap, double cutoff, double* d_out, void* stream);

/* ---- the production P = 1 epoch in one call --------------------------------
 * Periodic wrap of every dimension and the ownership check (exchange,
 * comm.py:340-400), the brick-major renumbering into pos_alt / vel_alt
 * (tmd_sort_locals; the caller swaps the buffers afterwards), the borders into
 * the `room` reserved ghost slots (tmd_borders_count / _fill_capped; copy
 * count at off[n] on the device), ghost velocities zeroed (Spring-Dashpot),
 * the production grid and cell positions (tmd_bin_cells_dev /
 * _cell_positions_dev), the split margin (tmd_split_margin, when margin_out is
 * set), the split rows (tmd_build_lists_split; list status reset first),
 * x_ref, and the export table (tmd_exports_build_dev).  The same sequence and
 * arguments as the Python device-count epoch.  All integer fields int64. */
typedef struct {
  double *pos, *pos_alt, *vel, *vel_alt;
  int64_t ld, n, room, sd;
  double wrap_hi[3], wrap_lo[3], wrap_s_plus[3], wrap_s_minus[3], slab_lo[3], slab_hi[3];
  double sort_lo[3], sort_edge;
  int64_t sort_dims[3], sort_shell, sort_shape[3];
  int32_t *sort_cell_of, *sort_cell_start, *sort_cell_atoms, *sort_key, *sort_key_start, *sort_perm, *order;
  double thr_hi[3], thr_lo[3], s_hi[3], s_lo[3];
  int32_t *off, *root;
  double* sh;
  int64_t ld_sh;
  double bin_lo[3], bin_edge;
  int64_t bin_dims[3], bin_shell;
  int32_t *cell_of, *cell_start, *cell_atoms;
  double* cell_pos;
  int64_t ld_cp;
  float* cell_pos_f; /* optional float copies (tmd_build_lists_split's pre-filter) */
  double f32_eps;
  double* dispmax2;
  int64_t margin_i0, margin_i1;
  double margin_floor, margin_factor, margin_cap, cutoff;
  double* margin_out;
  int32_t* nbr;
  int64_t ld_nbr;
  int32_t *nnear, *counts;
  int64_t cap;
  double near_rsq, rsq_max;
  double* xref;
  int64_t ld_ref;
  int32_t *ex_start, *ex_rank, *ex_slot;
  double* ex_sh;
  int32_t *ex_zeros, *ex_slots;
  int64_t ld_o;
  int64_t *status, *list_status;
} TmdEpochP1;
int tmd_epoch_p1(const TmdEpochP1* epoch, void* stream);

/* ---- batched step loop ---------------------------------------------------
 * The launches of steps k0 .. k1-1 of a production run between two epochs
 * (what driver.Simulation.advance issues), one host call per batch.  Per step
 * k: positions come from pos_a when (k - k0) is even, else pos_b (and go to
 * the other); SD velocities alternate the same way (LJ: vel_a in place);
 * phases = FINAL | NEXT except NEXT off at k_last; TMD_F_ENERGY when k %
 * thermo_every == 0 or k == k_last; TMD_F_STORE_FORCES when store_every or k
 * == k_last; prune/guard maxima dispmax2[k] / dispmax2[k + 1]; thermo row
 * thermo + k * thermo_stride; guard limit 0 at k0 when rebuild_at_k0; the
 * export table (ex_*) written when step k + 1 exists and is not a rebuild
 * step ((k + 1) % reneigh != 0), with peer buffers peer_base0 / peer_base1 by
 * parity (k - epoch_step) & 1; at size > 1, tmd_peer_sync after every step
 * but k_last (epochs barrier_epoch0 + 1, ...).  law: 0 LJ (p0..p2 = rc2, eps,
 * sigma^6), 1 SD (stiffness, damping, diameter).  All integer fields int64. */
typedef struct {
  int64_t law;
  double *pos_a, *pos_b, *vel_a, *vel_b;
  int64_t ld, n_local;
  const int32_t* nbr;
  int64_t ld_nbr;
  const int32_t *nnbr, *nnear;
  int64_t cap;
  double near_margin;
  double* dispmax2;
  const int32_t *ex_start, *ex_rank, *ex_slot;
  const double* ex_sh;
  int64_t n_ex, n_peers;
  const uint64_t *peer_base0, *peer_base1;
  const int64_t* peer_ld;
  const double* ex_border;
  double p0, p1, p2, half_dt_over_m, dt;
  double* frc;
  int64_t ld_f;
  const double* xref;
  int64_t ld_ref;
  double* thermo;
  int64_t thermo_stride;
  int64_t* status;
  double guard_lim2;
  int64_t k_last, epoch_step, reneigh, thermo_every, store_every, rebuild_at_k0;
  int64_t barrier_epoch0, rank, size;
  const uint64_t* mailboxes;
  double barrier_timeout_s;
  int64_t time_launches; /* record CUDA events around each step launch */
} TmdStepRun;
int tmd_run_steps(const TmdStepRun* run, int32_t k0, int32_t k1, void* stream);
/* Per-launch milliseconds of the timed launches on `stream` since the last
 * call (after the caller synchronised it; h_ms = NULL just resets); returns
 * how many were written (<= n). */
int tmd_run_launch_times(void* stream, float* h_ms, int32_t n);

/* ---- forces: compute_forces (potential.py:134-213), full lists ------------
 * LJ (potential.py:30-57): F_i = sum_j 48 eps sr6 (sr6 - 1/2) sr2 delta_ij over
 * list entries with rsq < rc2.  Writes d_frc[c * ld_f + i] for locals.  With
 * TMD_F_ENERGY: d_thermo[0] = 1/2 sum PE pairs, d_thermo[1] = virial
 * W = 1/2 sum delta.F (deterministic tree reduction). */
int tmd_force_lj(const double* d_pos, int64_t ld, int32_t n_local, const int32_t* d_nbr,
                 int64_t ld_nbr, const int32_t* d_nnbr, int32_t cap, double rc2, double eps,
                 double sigma6, uint32_t flags, double* d_frc, int64_t ld_f, double* d_thermo,
                 int64_t* d_status, void* stream);

/* Spring-Dashpot (potential.py:60-97): K overlap n - gamma (n.(vi - vj)) n while
 * overlapping (rsq < diam^2 and diam - sqrt(rsq) > 0).  Needs velocities of
 * locals and ghosts (ghost v = 0, particles.py:148). */
int tmd_force_sd(const double* d_pos, const double* d_vel, int64_t ld, int32_t n_local,
                 const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr, int32_t cap,
                 double stiffness, double damping, double diameter, uint32_t flags, double* d_frc,
                 int64_t ld_f, double* d_thermo, int64_t* d_status, void* stream);

/* Half-list force evaluation with reaction scatter (potential.py:187-191,
 * 205-209).  Reactions use fp64 atomics (summation order differs from the
 * reference; results within 1e-10). */
int tmd_force_half(const double* d_pos, const double* d_vel, int64_t ld, int32_t n_local,
                   const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr, int32_t law,
                   double p0, double p1, double p2, uint32_t flags, double* d_frc, int64_t ld_f,
                   double* d_thermo, int64_t* d_status, void* stream);

/* ---- fused timestep kernel (the production path) ---------------------------
 * One launch = compute_forces (LJ, full list) of step k, then in its
 * epilogue (phases & TMD_PHASE_FINAL) final_integrate of step k
 * (driver.py:86-93), optional thermo (PE, W, KE, momentum -> d_thermo[0..5];
 * KE/momentum after the kick) and (phases & TMD_PHASE_NEXT) initial_integrate
 * of step k+1 (driver.py:74-83) plus the displacement of every local against
 * d_xref (the guard, neighbor.py:197-206): d_dispmax2 gets the max squared
 * displacement (atomicMax on the bit pattern).  The drifted local positions
 * go to d_pos_out (same ld, a different buffer than d_pos: other blocks are
 * still gathering neighbour positions from d_pos).  Forces are stored into
 * d_frc only with TMD_F_STORE_FORCES (the step loop never reads them back;
 * the last step of a run stores them for the caller).
 * Replaces, per step: compute_forces (potential.py:134-213), final_integrate
 * and initial_integrate (driver.py:74-93), the guard (driver.py:115-125) and
 * synchronize (comm.py:469-498) of the reference's rank_program loop. */
#define TMD_PHASE_FINAL 1
#define TMD_PHASE_NEXT 2
int tmd_step_lj(const double* d_pos, double* d_pos_out, double* d_vel, int64_t ld, int32_t n_local,
                const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr, const int32_t* d_nnear,
                int32_t cap, double near_margin, const double* d_prune_disp2, const int32_t* d_ex_start,
                const int32_t* d_ex_rank, const int32_t* d_ex_slot, const double* d_ex_sh, int64_t n_ex,
                int32_t n_peers, double* const* h_peer_base, const int64_t* h_peer_ld, const double* h_ex_border,
                double rc2, double eps, double sigma6, double half_dt_over_m, double dt, int32_t phases,
                uint32_t flags,
                double* d_frc, int64_t ld_f, const double* d_xref, int64_t ld_ref, double* d_dispmax2,
                double* d_thermo, int64_t* d_status, double guard_lim2, void* stream);
/* Spring-Dashpot production step (potential.py:60-97, driver.py:74-93): as
 * tmd_step_lj with the contact law (K = stiffness, gamma = damping, d =
 * diameter; cutoff d); the dashpot reads neighbours' velocities, so the
 * kicked velocities go to d_vel_out (a different buffer than d_vel when an
 * integration phase is set; ghost velocities are 0 in both). */
int tmd_step_sd(const double* d_pos, double* d_pos_out, const double* d_vel, double* d_vel_out, int64_t ld,
                int32_t n_local, const int32_t* d_nbr, int64_t ld_nbr, const int32_t* d_nnbr, const int32_t* d_nnear,
                int32_t cap, double near_margin, const double* d_prune_disp2, const int32_t* d_ex_start,
                const int32_t* d_ex_rank, const int32_t* d_ex_slot, const double* d_ex_sh, int64_t n_ex,
                int32_t n_peers, double* const* h_peer_base, const int64_t* h_peer_ld, const double* h_ex_border,
                double stiffness, double damping, double diameter, double half_dt_over_m, double dt,
                int32_t phases, uint32_t flags, double* d_frc, int64_t ld_f, const double* d_xref, int64_t ld_ref,
                double* d_dispmax2, double* d_thermo, int64_t* d_status, double guard_lim2, void* stream);
/* Fail fast (both step kernels): when d_status already holds an error, or
 * guard_lim2 > 0 and *d_prune_disp2 >= guard_lim2 (the current positions
 * moved half the skin since the build: the reference's GuardViolation,
 * driver.py:115-125, raised before the step's forces), the launch advances no
 * atom and sets TMD_GUARD for the guard case: the state stays at the failing
 * step until the host reads the status.
 * Exact pruning in tmd_step_lj / tmd_step_sd: with split rows (d_nnear != NULL) and
 * d_prune_disp2 = the max squared displacement d^2 of any atom (locals and
 * ghosts) since the lists were built, atom i's back segment is skipped while
 * d_i + d <= near_margin - 1e-9 (d_i = |x_i - d_xref_i|, near_margin =
 * sqrt(near_rsq) - rc): every back-segment pair is then farther than rc.
 * d_xref is required with split rows.  TMD_F_NO_PRUNE scans every segment.
 * Fused ghost refresh (synchronize, comm.py:469-498): with d_ex_start != NULL
 * (export table from tmd_exports_build) the NEXT phase also writes
 * x_new + shift into every ghost slot mirroring the atom, in the destination
 * rank's next position buffer h_peer_base[rank] (leading dimension
 * h_peer_ld[rank]); peers' buffers are CUDA-IPC mappings over NVLink.
 * h_ex_border (6 doubles: hi - r per dim, then lo + r; NULL = off) skips the
 * table for atoms whose build-time position (d_xref) is not within r of a
 * face.  The kernel issues no fence: the caller orders the peers' reads
 * after this kernel (stream order, then an inter-rank collective). */

/* Export table for the fused ghost refresh: entries (root local index, dest
 * rank, dest slot, shift (3, ld_sh)) grouped by root: d_start[n_local + 1]
 * (CSR), d_o_rank / d_o_slot / d_o_sh (3, n_ex) in grouped order. */
int tmd_exports_build(int32_t n_local, int32_t n_ex, const int32_t* d_root, const int32_t* d_rank,
                      const int32_t* d_slot, const double* d_sh, int64_t ld_sh, int32_t* d_start,
                      int32_t* d_o_rank, int32_t* d_o_slot, double* d_o_sh, int64_t* d_status,
                      void* stream);
/* The same with the entry count on the device (*d_n_ex <= n_ex_max) and the
 * output shift table's leading dimension ld_o (>= n_ex_max; pass it as the
 * step kernels' n_ex). */
int tmd_exports_build_dev(int32_t n_local, int32_t n_ex_max, const int32_t* d_n_ex, const int32_t* d_root,
                          const int32_t* d_rank, const int32_t* d_slot, const double* d_sh, int64_t ld_sh,
                          int32_t* d_start, int32_t* d_o_rank, int32_t* d_o_slot, double* d_o_sh, int64_t ld_o,
                          int64_t* d_status, void* stream);

/* Provenance of one stencil entry's border copies (define_borders,
 * comm.py:434-466): for t < k, p = d_idx[t] is a local (-> rank me, root p)
 * or an earlier ghost (-> its provenance from d_p_* at p - n_local, leading
 * dimension ld_p); the shift on `dim` becomes d_sh[t].  Written to d_o_*
 * (rank, root, shift (3, ld_o)) at [0, k). */
int tmd_ghost_provenance(int32_t n_local, int32_t me, int32_t k, const int32_t* d_idx, int32_t dim,
                         const double* d_sh, const int32_t* d_p_rank, const int32_t* d_p_root,
                         const double* d_p_sh, int64_t ld_p, int32_t* d_o_rank, int32_t* d_o_root,
                         double* d_o_sh, int64_t ld_o, void* stream);

/* define_borders in one pass when every stencil entry is self (P = 1):
 * round d copies atoms with x_d > thr_hi[d] (= hi_d - r; shift s_hi[d] = -L_d)
 * and x_d < thr_lo[d] (= lo_d + r; shift s_lo[d] = +L_d); atom i's ghosts
 * are the product of its per-dimension options minus the identity -- the
 * same copies as the three rounds (comm.py:434-466), grouped by local.
 * tmd_borders_count writes the exclusive scan of per-local copy counts to
 * d_off[0 .. n_local] (total at d_off[n_local]); tmd_borders_fill writes the
 * copies to slots n_local + g (v = 0) with provenance root d_root[g] and
 * recorded shifts d_sh (3, ld_sh). */
int tmd_borders_count(const double* d_pos, int64_t ld, int32_t n_local, const double* h_thr_hi,
                      const double* h_thr_lo, int32_t* d_off, void* stream);
int tmd_borders_fill(const double* d_pos, int64_t ld, int32_t n_local, const double* h_thr_hi,
                     const double* h_thr_lo, const double* h_s_hi, const double* h_s_lo, const int32_t* h_grid,
                     const int32_t* d_off, double* d_out_pos, int64_t ld_out, double* d_out_vel, int32_t* d_root,
                     double* d_sh, int64_t ld_sh, int32_t* d_dest, void* stream);
/* (fill, continued) copies go to d_out_pos (3, ld_out) at [0, total) (and v = 0 to
 * d_out_vel if given); with h_grid = {coords[3], grid[3]} (NULL: one rank) and
 * d_dest, each copy's destination rank (option "> thr_hi" = the + neighbour).
 * At P > 1 the shifts s_hi / s_lo are the global-edge shifts of this rank
 * (0 away from the edge) -- the multi-hop chains of the three rounds
 * collapse into one direct copy to the rank that would end up holding it. */
/* tmd_borders_fill writing only copies g < max_out (the caller's room in its
 * ghost region; it compares d_off[n_local] with max_out afterwards). */
int tmd_borders_fill_capped(const double* d_pos, int64_t ld, int32_t n_local, const double* h_thr_hi,
                            const double* h_thr_lo, const double* h_s_hi, const double* h_s_lo,
                            const int32_t* h_grid, const int32_t* d_off, double* d_out_pos, int64_t ld_out,
                            double* d_out_vel, int32_t* d_root, double* d_sh, int64_t ld_sh, int32_t* d_dest,
                            int64_t max_out, void* stream);

/* Direct exchange for the production path (comm.py:340-400 in one pass):
 * self dimensions (grid 1) wrap in place; in a remote dimension x >= hi goes
 * to the + neighbour, x < lo to the - neighbour, with the global-edge shift
 * applied in place.  d_dest[i] = destination rank or -1; stable index lists
 * of staying / leaving locals and their counts (d_counts[0..1]).  d_scratch:
 * 4 n + 2 int32 of caller scratch (NULL: stream-ordered allocation). */
int tmd_exchange_classify(double* d_pos, int64_t ld, int32_t n, const double* h_lo, const double* h_hi,
                          const double* h_s_hi, const double* h_s_lo, const int32_t* h_grid, int32_t* d_dest,
                          int32_t* d_keep_idx, int32_t* d_leave_idx, int32_t* d_counts, int32_t* d_scratch,
                          void* stream);

/* Step barrier + max over NVLink peer memory (the fused refresh's ordering
 * point): publishes *d_value with `epoch` (>= 1, increasing, the same on
 * every rank) into every rank's mailbox h_mailbox[r] (tmd_mailbox_words()
 * int64 each, zero-initialised, CUDA-IPC mapped), waits for all n_peers
 * ranks, then *d_value = the maximum.  A rank missing for timeout_s
 * seconds (device globaltimer) sets TMD_PROTOCOL in d_status instead of
 * hanging; the host passes a generous bound (Simulation(peer_timeout_s=120))
 * so host pauses between steps (trajectory dumps, GC) are tolerated. */
int tmd_mailbox_words(void);
int tmd_peer_sync(int64_t epoch, int32_t me, int32_t n_peers, int64_t* const* h_mailbox, double* d_value,
                  double timeout_s, int64_t* d_status, void* stream);

/* Small all-gather over the same mailboxes (the P > 1 epoch's count
 * exchanges, replacing an NCCL all-gather plus its host round trip): every
 * rank publishes d_in[0 .. w) (w <= tmd_peer_gather_words()) with call
 * number `epoch` (>= 1, increasing, the same on every rank, independent of
 * the barrier's), and d_out (n_peers, w) receives every rank's values.
 * Timeout as tmd_peer_sync. */
int tmd_peer_gather_words(void);
int tmd_peer_allgather(int64_t epoch, int32_t me, int32_t n_peers, int64_t* const* h_mailbox, const int64_t* d_in,
                       int32_t w, int64_t* d_out, double timeout_s, int64_t* d_status, void* stream);

/* CUDA IPC of a device pointer that may lie inside a larger cudaMalloc block:
 * handle (tmd_ipc_handle_size() bytes) + byte offset; tmd_ipc_open maps a
 * peer's block into this process (peer access enabled lazily) and returns the
 * pointer and the mapped base (for tmd_ipc_close). */
int tmd_ipc_handle_size(void);
int tmd_ipc_handle(const void* d_ptr, void* handle_out, int64_t* offset_out);
int tmd_ipc_open(const void* handle, int64_t offset, void** d_ptr_out, void** d_base_out);
int tmd_ipc_close(void* d_base);

/* d_out[t] = inverse(d_perm)[d_idx[t]] for t < n (d_perm a permutation of
 * [0, n), d_idx values in [0, n)): the list builder's cell-order walk in the
 * brick-major numbering. */
int tmd_compose_inverse(const int32_t* d_perm, const int32_t* d_idx, int32_t n, int32_t* d_out, void* stream);

/* Host-side plumbing: tmd_check_pack writes [d_status[0], d_vals[0 .. n)] as
 * doubles to d_out (one read-back of an epoch's status and guard maxima);
 * tmd_copy_rows copies `count` entries of `rows` rows between (rows, ld)
 * blocks (a device copy, e.g. the x_ref snapshot of neighbor.py:192). */
int tmd_check_pack(const int64_t* d_status, const double* d_vals, int32_t n, double* d_out, void* stream);
/* Allocate `stream`'s reduction scratch ahead of a run (a device allocation
 * orders every stream of the context; with in-process ranks whose barrier
 * kernels wait for each other it must not land mid-run). */
int tmd_prepare_stream(void* stream);
int tmd_copy_rows(const double* d_src, int64_t ld_src, double* d_dst, int64_t ld_dst, int32_t rows, int64_t count,
                  void* stream);

/* ---- space-filling-curve balancing (balance.py) ----------
 * tmd_sfc_keys: key of every particle's cell at depth D (2^D cells of width
 * h_width per axis from h_lo, clamped): curve 0 Morton (x least significant
 * in each bit triad), 1 Hilbert (Skilling's transpose construction).
 * tmd_leaf_counts: d_counts[b] = particles with d_leaf_start[b] <= key <
 * d_leaf_start[b + 1] (leaves sorted by first key; every octree leaf is a
 * contiguous key range of either curve).  tmd_morton_key / tmd_hilbert_key:
 * the same keys on the host. */
int tmd_sfc_keys(const double* d_pos, int64_t ld, int32_t n, const double* h_lo, const double* h_width, int32_t depth,
                 int32_t curve, uint64_t* d_keys, void* stream);
int tmd_leaf_counts(const uint64_t* d_keys, int32_t n, const uint64_t* d_leaf_start, int32_t n_leaves,
                    int32_t* d_counts, void* stream);
uint64_t tmd_morton_key(uint32_t x, uint32_t y, uint32_t z, int32_t depth);
uint64_t tmd_hilbert_key(uint32_t x, uint32_t y, uint32_t z, int32_t depth);

/* ---- direct-protocol bookkeeping (P > 1 production path) ------------------
 * tmd_group_by_rank: stable grouping of m records by d_rank[t] in [0, n_ranks)
 * (n_ranks <= 8; records with another rank, e.g. -1, drop out):
 * d_out_ids[pos] = d_ids[t] (t if d_ids is NULL),
 * d_out_rank[pos] = the rank (optional), d_counts[r] = group sizes -- the
 * order the all-to-all sends them in (comm.py:340-466 send order per peer).
 * tmd_pack_rows / tmd_unpack_rows: records as contiguous rows of width 3
 * (x) or 6 (x, v) for the all-to-all, and received rows into the store at
 * slot `at` (width 3: ghosts, v = 0, particles.py:148).
 * tmd_border_slots: d_slot[t] = h_base[d_rank[t]] + t (a grouped border
 * copy's slot on its receiver).  tmd_gather_i32: d_out[t] = d_src[d_idx[t]]. */
int tmd_group_by_rank(const int32_t* d_rank, const int32_t* d_ids, int32_t m, int32_t n_ranks, int32_t* d_out_ids,
                      int32_t* d_out_rank, int32_t* d_counts, void* stream);
int tmd_pack_rows(const double* d_pos, const double* d_vel, int64_t ld, const int32_t* d_idx, int32_t k,
                  int32_t width, double* d_rows, void* stream);
int tmd_unpack_rows(const double* d_rows, int32_t k, int32_t width, double* d_pos, double* d_vel, int64_t ld,
                    int32_t at, void* stream);
int tmd_border_slots(const int32_t* d_rank, int32_t m, int32_t n_ranks, const int64_t* h_base, int32_t* d_slot,
                     void* stream);
int tmd_gather_i32(const int32_t* d_src, const int32_t* d_idx, int32_t n, int32_t* d_out, void* stream);

/* ---- atom numbering of the production path ------------------------------
 * Bricks of 2^sx x 2^sy x 2^sz cells of the r/2 grid (edge w, interior dims
 * h_dims); brick b = (bx * nb1 + by) * nb2 + bz.  tmd_brick_sort: stable
 * counting sort of the locals by key = brick * 2^(sx+sy+sz) + cell-in-brick
 * (h_shape = {sx, sy, sz}, NULL = {2, 2, 2}): d_perm (n_local) = the locals in
 * brick-major order, d_key_start (n_keys + 1) the key offsets, d_key
 * (n_local scratch).  Same cell formula as tmd_bin_cells_ex, clamped to the
 * interior.  A warp's 32 consecutive atoms then form a compact block, so the
 * neighbour gathers of tmd_step_lj share cache lines. */
int tmd_brick_sort(const double* d_pos, int64_t ld, int32_t n_local, const double* h_lo, double w,
                   const int32_t* h_dims, const int32_t* h_shape, int32_t* d_key, int32_t* d_key_start,
                   int32_t* d_perm, void* stream);

/* The production epoch's renumbering in one call: tmd_bin_cells_ex of the n
 * locals at cell edge `edge` (shell layers `shell`; scratch d_cell_of (n),
 * d_cell_start (cells + 1), d_cell_atoms (n)), tmd_brick_sort (scratch d_key
 * (n), d_key_start, d_perm (n)), d_order = the builder's thread -> atom map
 * (cell order, new numbering; tmd_compose_inverse), and x, v permuted into
 * d_pos_out / d_vel_out (leading dimension ld). */
int tmd_sort_locals(const double* d_pos, const double* d_vel, int64_t ld, int32_t n, const double* h_lo, double edge,
                    const int32_t* h_dims, int32_t shell, const int32_t* h_shape, int32_t* d_cell_of,
                    int32_t* d_cell_start, int32_t* d_cell_atoms, int32_t* d_key, int32_t* d_key_start,
                    int32_t* d_perm, int32_t* d_order, double* d_pos_out, double* d_vel_out, int64_t* d_status,
                    void* stream);

/* ---- integrators (driver.py:74-93) -----------------------------------------
 * kick_drift: v += c F; x += dt v on locals (c = 0.5 dt / m); if d_xref, also
 * max |x - xref|^2 into d_dispmax2.  kick: v += c F. */
int tmd_kick_drift(double* d_pos, double* d_vel, const double* d_frc, int64_t ld, int64_t ld_f,
                   int32_t n, double c, double dt, const double* d_xref, int64_t ld_ref,
                   double* d_dispmax2, void* stream);
int tmd_kick(double* d_vel, const double* d_frc, int64_t ld, int64_t ld_f, int32_t n, double c,
             void* stream);
/* Zero `count` entries starting at `start` in each of `rows` rows of a
 * (rows, ld) fp64 block (ghost velocities, particles.py:148). */
int tmd_zero_rows(double* d, int64_t ld, int32_t rows, int64_t start, int64_t count, void* stream);

/* max |x - xref|^2 over locals (neighbor.py:197-206) into d_dispmax2 (atomicMax). */
int tmd_max_disp2(const double* d_pos, int64_t ld, const double* d_xref, int64_t ld_ref,
                  int32_t n, double* d_dispmax2, void* stream);

/* KE = 1/2 m sum v^2 and momentum m sum v over locals -> d_out[0..3]. */
int tmd_kinetic(const double* d_vel, int64_t ld, int32_t n, double mass, double* d_out,
                void* stream);

/* ---- halo protocol building blocks (comm.py:340-498) ----------------------
 * select: order-preserving indices i in [0, n) with pred(d_coord[i], thr);
 * count to d_count (device int32). */
int tmd_select(const double* d_coord, int32_t n, int32_t kind, double thr, double thr2,
               int32_t* d_idx, int32_t* d_count, void* stream);

/* Both entries of a stencil round in one pass: order-preserving index lists for
 * pred_a and pred_b over [0, n), counts to d_counts[0..1] (device int32). */
int tmd_select_pair(const double* d_coord, int32_t n, int32_t kind_a, double thr_a, int32_t kind_b,
                    double thr_b, int32_t* d_idx_a, int32_t* d_idx_b, int32_t* d_counts, void* stream);

/* Self-peer border emission (comm.py:448-451): ghost g0 + t = pos[idx[t]] + shift
 * (h_shift, 3 doubles), ghost velocity 0 (particles.py:148), and the plan's
 * recorded shift along dim d_sh[t] = (x + shift_dim) - x (comm.py:449). */
int tmd_emit_ghosts(double* d_pos, double* d_vel, int64_t ld, const int32_t* d_idx, int32_t k,
                    const double* h_shift, int32_t dim, int32_t g0, double* d_sh, void* stream);

/* emitted[c][t] = pos[c][idx[t]] + shift[c]  (comm.py:248/256, 483) with
 * optional per-entry shift along dim (d_shift_d != NULL: shift[dim] is
 * replaced by d_shift_d[t], the plan's recorded emitted - pos). */
int tmd_gather_shift(const double* d_pos, int64_t ld, const int32_t* d_idx, int32_t k,
                     const double* h_shift, int32_t dim, const double* d_shift_d, double* d_out,
                     int64_t ld_out, void* stream);

/* d_sh[t] = (pos[dim][idx[t]] + s) - pos[dim][idx[t]]  (comm.py:449) */
int tmd_plan_shift(const double* d_pos, int64_t ld, const int32_t* d_idx, int32_t k, int32_t dim,
                   double s, double* d_sh, void* stream);

/* In-place periodic wrap for a dimension whose +/- peers are this rank
 * (comm.py:367-370): x_d >= hi -> x_d + s_plus, else x_d < lo -> x_d + s_minus. */
int tmd_wrap_self(double* d_pos, int64_t ld, int32_t n, int32_t dim, double hi, double lo,
                  double s_plus, double s_minus, void* stream);

/* Half-open ownership check (comm.py:394-400): TMD_PROTOCOL if a local is
 * outside [lo, hi). */
int tmd_check_owned(const double* d_pos, int64_t ld, int32_t n, const double* h_lo,
                    const double* h_hi, int64_t* d_status, void* stream);

/* Flattened self-ghost sync (P = 1 fast path of synchronize, comm.py:469-498):
 * x[c][g0 + t] = x[c][src[t]] + sh[c * k + t]. */
int tmd_sync_flat(double* d_pos, int64_t ld, int32_t g0, int32_t k, const int32_t* d_src,
                  const double* d_sh, void* stream);

/* Build the flattened plan for ghosts [g0, g0+k) created from d_idx with
 * per-ghost shift d_sh along dim: src/sh of parents that are ghosts are
 * inherited. */
int tmd_flatten_round(int32_t n_local, int32_t g0, int32_t k, const int32_t* d_idx, int32_t dim,
                      const double* d_sh, int32_t* d_src, double* d_flat_sh, int64_t k_total,
                      void* stream);

/* ---- pair laws on arrays (LennardJones/SpringDashpot.pair_force/energy,
 * potential.py:46-57, 80-97): out (n x 3, row-major) for delta (n x 3, row-major). */
int tmd_pair_force(int32_t law, const double* d_delta, const double* d_rsq, const double* d_vi,
                   const double* d_vj, int32_t n, double p0, double p1, double p2, double* d_out,
                   void* stream);
int tmd_pair_energy(int32_t law, const double* d_rsq, int32_t n, double p0, double p1, double p2,
                    double* d_out, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* TINYMD_B200_H */
