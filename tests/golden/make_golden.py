"""Generate the golden fixtures in this directory by running the REFERENCE itself.

Run here (the container that has /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py          # 8^3 / P-rank / SD fixtures
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py --lj32   # 32^3 x 100 steps (lj32_p1.npz)

It imports ``nanopair`` from /root/reference/pkg/src, builds six-stencil
worlds (comm.py:171-274) with ``grid_box = slab`` and one MailboxTransport
(comm.py:83-104), advances every rank's ``rank_program`` generator
(driver.py:128-177) in lockstep — the harness the reference leaves to its
user (driver.py:134-139) — and records what the oracle and the GPU build are
checked against.  Per-step PE comes from the step's own force call
(``accumulate_energy=True``, full mode, potential.py:192-195); the virial
W = 1/2 sum delta.F_ij is evaluated from the same lists with the reference's
own ``law.pair_force``; KE = 1/2 m sum v^2 after the closing half-kick.

The reference cannot travel to the GPU box, so only these .npz files do.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.dirname(os.path.abspath(__file__))


def _import_reference():
    sys.dont_write_bytecode = True
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import nanopair.backend as backend
    import nanopair.comm as comm
    import nanopair.core as core
    import nanopair.driver as driver
    import nanopair.layout as layout
    import nanopair.neighbor as neighbor
    import nanopair.particles as particles
    import nanopair.potential as potential

    return dict(backend=backend, comm=comm, core=core, driver=driver, layout=layout,
                neighbor=neighbor, particles=particles, potential=potential)


def _virial(store, lists, law):
    """W = 1/2 sum_i sum_{j in list(i), rsq < rc^2} delta_ij . F_ij (full lists)."""
    n = store.n_local
    if n == 0:
        return 0.0
    pos = store.all_positions()
    vel = store.all_velocities()
    mat = lists.as_matrix()
    cap = mat.shape[1]
    valid = np.arange(cap)[None, :] < lists.counts[:, None]
    j = np.where(valid, mat, 0)
    delta = pos[:n, None, :] - pos[j]
    rsq = np.einsum("ijk,ijk->ij", delta, delta)
    within = valid & (rsq < law.cutoff_rsq)
    safe = np.where(within, rsq, 1.0)
    if law.needs_velocities:
        f = law.pair_force(delta, safe, vel[:n, None, :], vel[j])
    else:
        f = law.pair_force(delta, safe)
    f = np.where(within[..., None], f, 0.0)
    return 0.5 * float((f * delta).sum())


def reference_run(cfg, nranks, steps=None, capture=None, threads=1):
    """Lockstep run of the reference; returns thermo rows and the final rank stores.

    ``threads`` > 1 runs the force phase on the reference's ThreadBackend
    (backend.py:31-40), whose results are identical to the serial backend's."""
    R = _import_reference()
    comm, driver, particles, layout, potential = (R["comm"], R["driver"], R["particles"],
                                                  R["layout"], R["potential"])
    if steps is not None:
        cfg = cfg.with_overrides(steps=steps)
    cfg.validate()
    gbox = cfg.domain()
    r = cfg.interaction_radius()
    grid = comm.factor_rank_grid(nranks)
    transport = comm.MailboxTransport(nranks)
    full = particles.create_lattice(cfg, gbox)
    pos0, vel0 = full.local_positions(), full.local_velocities()
    stores, gens = [], []
    for rk in range(nranks):
        slab = comm.slab_bounds(gbox, grid, comm.rank_grid_coords(rk, grid))
        dom = comm.RankDomain(rk, [slab], r, grid_box=slab)
        pat = comm.six_stencil_pattern(grid, rk, gbox, r)
        world = comm.RankWorld(nranks, rk, transport, gbox, dom, pat)
        inside = slab.contains(pos0)
        st = particles.ParticleStore(layout.row_major_layout(), max(int(inside.sum()), 1))
        st.append_locals(pos0[inside], vel0[inside])
        stores.append(st)
        be = R["backend"].ThreadBackend(threads) if threads > 1 else R["backend"].SerialBackend()
        gens.append(driver.rank_program(cfg, world, st, backend=be))

    # hook the step's own force call to also return PE and W (forces are unchanged)
    per_call = {}
    orig = potential.compute_forces

    def hooked(store, lists, law, half=None, backend=None, accumulate_energy=False):
        e = orig(store, lists, law, half=half, backend=backend, accumulate_energy=True)
        per_call[id(store)] = (e, _virial(store, lists, law))
        return None

    driver.compute_forces = hooked
    rows, reports = [], [None] * nranks
    vol = gbox.volume()
    try:
        while True:
            marks = []
            for k, g in enumerate(gens):
                if reports[k] is not None:
                    continue
                try:
                    marks.append(next(g))
                except StopIteration as stop:
                    reports[k] = stop.value
            if all(rep is not None for rep in reports):
                break
            if marks and all(isinstance(m, tuple) and m[0] == "step" for m in marks):
                step = marks[0][1]
                pe = sum(per_call[id(s)][0] for s in stores)
                w = sum(per_call[id(s)][1] for s in stores)
                ke = 0.0
                mom = np.zeros(3)
                for s in stores:
                    v = s.local_velocities()
                    ke += 0.5 * cfg.mass * float(np.sum(v * v))
                    mom += cfg.mass * v.sum(axis=0)
                press = (2.0 * ke + w) / (3.0 * vol)
                rows.append([step, pe, ke, w, press, mom[0], mom[1], mom[2]])
                if capture is not None:
                    capture(step, gens, stores)
    finally:
        driver.compute_forces = orig
    return np.array(rows), stores, reports


def sorted_state(stores):
    s = np.vstack([np.hstack([st.local_positions(), st.local_velocities()]) for st in stores])
    return s[np.lexsort((s[:, 2], s[:, 1], s[:, 0]))]


def lj32_run():
    """BASELINE configs[1] (32^3 = 131,072 atoms, P = 1) for 100 steps: thermo every
    step and the sorted final state (about 2 minutes on 8 threads)."""
    R = _import_reference()
    lj32 = R["core"].SimConfig(unit_cells=(32, 32, 32), steps=100)
    rows, stores, reports = reference_run(lj32, 1, threads=os.cpu_count() or 1)
    st = sorted_state(stores)
    np.savez_compressed(os.path.join(OUT, "lj32_p1.npz"), thermo=rows, final_state=st,
                        momentum_initial=reports[0].momentum_initial,
                        momentum_final=reports[0].momentum_final,
                        max_disp_seen=reports[0].max_displacement_seen)
    print("lj32_p1", rows[-1])


def main():
    if "--lj32" in sys.argv:
        lj32_run()
        return
    R = _import_reference()
    core = R["core"]
    lj8 = core.SimConfig(unit_cells=(8, 8, 8), steps=100)

    # ---- LJ 8^3, P = 1: thermo, final state, step-0 and step-100 op snapshots
    snaps = {}

    def cap(step, gens, stores):
        if step in (0, 100):
            st = gens[0].gi_frame.f_locals["state"]
            store = stores[0]
            snaps[step] = dict(
                pos=store.all_positions(),
                vel=store.all_velocities(),
                n_local=store.n_local,
                coords=st.grid.coords.copy(),
                counts=st.grid.counts.copy(),
                occupants=st.grid.occupants.copy(),
                dims=st.grid.dims.copy(),
                mat=st.lists.as_matrix().copy(),
                lcounts=st.lists.counts.copy(),
                forces=store.local_forces(),
            )

    rows, stores, reports = reference_run(lj8, 1, capture=cap)
    s0, s100 = snaps[0], snaps[100]
    np.savez_compressed(
        os.path.join(OUT, "lj8_p1.npz"),
        thermo=rows,
        final_state=sorted_state(stores),
        momentum_initial=reports[0].momentum_initial,
        momentum_final=reports[0].momentum_final,
        max_disp_seen=reports[0].max_displacement_seen,
        s0_pos=s0["pos"], s0_nlocal=s0["n_local"], s0_coords=s0["coords"].astype(np.int16),
        s0_counts=s0["counts"].astype(np.int16), s0_occupants=s0["occupants"],
        s0_dims=s0["dims"], s0_mat=s0["mat"], s0_lcounts=s0["lcounts"], s0_forces=s0["forces"],
        s100_pos=s100["pos"], s100_vel=s100["vel"], s100_nlocal=s100["n_local"],
        s100_coords=s100["coords"].astype(np.int16), s100_mat=s100["mat"],
        s100_lcounts=s100["lcounts"], s100_forces=s100["forces"],
    )
    print("lj8_p1", rows[-1])

    # half lists + half-mode forces on the step-100 state (potential.py:187-191)
    neighbor, potential, particles, layout = R["neighbor"], R["potential"], R["particles"], R["layout"]
    st = particles.ParticleStore(layout.row_major_layout(), s100["pos"].shape[0])
    n = s100["n_local"]
    st.append_locals(s100["pos"][:n], s100["vel"][:n])
    st.append_ghosts(s100["pos"][n:], peer=0)
    box = lj8.domain()
    grid = neighbor.build_cell_grid(st, box, lj8.interaction_radius())
    hl = neighbor.build_neighbor_lists(st, grid, lj8.interaction_radius(), half=True)
    e_half = potential.compute_forces(st, hl, potential.law_from_config(lj8), accumulate_energy=True)
    np.savez_compressed(
        os.path.join(OUT, "lj8_half_s100.npz"),
        mat=hl.as_matrix(), counts=hl.counts, forces=st.local_forces(), energy=e_half,
    )

    # ---- LJ 8^3 at P = 2, 4, 8: thermo + sorted final state
    for p in (2, 4, 8):
        rows_p, stores_p, _ = reference_run(lj8, p)
        np.savez_compressed(
            os.path.join(OUT, f"lj8_p{p}.npz"),
            thermo=rows_p, final_state=sorted_state(stores_p),
            n_local=np.array([s.n_local for s in stores_p]),
            n_ghost=np.array([s.n_ghost for s in stores_p]),
        )
        print(f"lj8_p{p}", rows_p[-1])

    # ---- Spring-Dashpot DEM, 8^3 fcc, d = 1.2 (12 contacts), damping on (ghost v = 0)
    sd8 = core.SimConfig(unit_cells=(8, 8, 8), steps=100, potential_kind="sd", diameter=1.2,
                         cutoff=1.2, stiffness=100.0, damping=0.5)
    for p in (1, 8):
        rows_p, stores_p, _ = reference_run(sd8, p)
        np.savez_compressed(
            os.path.join(OUT, f"sd8_p{p}.npz"),
            thermo=rows_p, final_state=sorted_state(stores_p),
        )
        print(f"sd8_p{p}", rows_p[-1])

    # ---- 32^3 step 0 only: ghost count, PE/atom, list statistics at P = 1
    lj32 = core.SimConfig(unit_cells=(32, 32, 32), steps=0)
    stat = {}

    def cap32(step, gens, stores):
        stt = gens[0].gi_frame.f_locals["state"]
        stat.update(n_ghost=stores[0].n_ghost, lcounts=np.bincount(stt.lists.counts),
                    cap=stt.lists.as_matrix().shape[1], max_occ=stt.grid.occupants.shape[1])

    rows32, _, _ = reference_run(lj32, 1, capture=cap32)
    np.savez_compressed(os.path.join(OUT, "lj32_step0.npz"), thermo=rows32, **stat)
    print("lj32 step0", rows32[0], stat["n_ghost"])


if __name__ == "__main__":
    main()
