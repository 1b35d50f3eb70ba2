"""GPU parity: the CUDA path through the C ABI against the oracle and the golden
fixtures made by the reference itself.

Bars (BASELINE.json north_star): cells and neighbor sets bit-exact; per-atom
forces within 1e-10 scale-relative (|dF| <= 1e-10 * max(|F|, sum_j |F_ij|),
the scale idea of the reference's test_potential.py:48-66); thermo energy and
pressure within 1e-8 (relative) over 100 steps.  The exact-order kernels are
held to bitwise equality.
"""

import numpy as np
import pytest

import oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07400_b200")
from paper_2009_07400_b200 import (AABB, LennardJones, ParticleStore, ProtocolError, SimConfig,  # noqa: E402
                                   SingularityError, SpringDashpot, Vec3, build_cell_grid,
                                   build_neighbor_lists, compute_forces, lj_force,
                                   spring_dashpot_force)

LJ8 = SimConfig(unit_cells=(8, 8, 8), steps=100)
SD8 = SimConfig(unit_cells=(8, 8, 8), steps=100, potential_kind="sd", diameter=1.2, cutoff=1.2,
                stiffness=100.0, damping=0.5)
FORCE_TOL = 1e-10
THERMO_TOL = 1e-8


def make_store(pos, n_ghost=0, vel=None):
    pos = np.asarray(pos, dtype=np.float64)
    n_local = len(pos) - n_ghost
    st = ParticleStore(max(len(pos), 1))
    v = np.zeros((n_local, 3)) if vel is None else np.asarray(vel)[:n_local]
    st.append_locals(pos[:n_local], v)
    if n_ghost:
        st.append_ghosts(pos[n_local:], peer=0)
    return st


def force_scale(pos, n_local, mat, counts, rc2):
    """sum_j |F_ij| per atom (the magnitude the summed force cancels from)."""
    cap = mat.shape[1]
    valid = np.arange(cap)[None, :] < counts[:, None]
    j = np.where(valid, mat, 0)
    d = pos[:n_local, None, :] - pos[j]
    rsq = O.rsq_ref_order(d)
    inside = valid & (rsq < rc2)
    f = O.lj_pair_force(d, np.where(inside, rsq, 1.0), 1.0, 1.0)
    return np.where(inside[..., None], np.abs(f), 0.0).sum(axis=1)


def assert_forces_close(got, want, scale):
    bound = FORCE_TOL * np.maximum(np.abs(want), scale)
    assert np.all(np.abs(got - want) <= bound), np.max(np.abs(got - want) / np.maximum(bound, 1e-300))


# --------------------------------------------------------------------------
# pair laws (test_potential.py:28-131)
# --------------------------------------------------------------------------

def test_lj_unit_separation_exact():
    f = lj_force(Vec3(1.0, 0.0, 0.0), 1.0, epsilon=1.0, sigma=1.0)
    assert (f.x, f.y, f.z) == (24.0, 0.0, 0.0)


def test_lj_matches_oracle_bitwise_and_eq2_within_4ulp():
    rng = np.random.default_rng(42)
    n = 10_000
    r = rng.uniform(0.8, 2.5, size=n)
    u = rng.normal(size=(n, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    d = u * r[:, None]
    rsq = (d * d).sum(axis=1)
    got = LennardJones(1.0, 1.0).pair_force(d, rsq)
    assert np.array_equal(got, O.lj_pair_force(d, rsq, 1.0, 1.0))
    s6 = (1.0 / rsq) ** 3
    want = (24.0 * s6 * (2.0 * s6 - 1.0) / rsq)[:, None] * d
    mag = (48.0 * s6 * (s6 + 0.5) / rsq)[:, None] * np.abs(d)
    scale = np.maximum(np.maximum(np.abs(got), np.abs(want)), mag)
    assert np.all(np.abs(got - want) <= 4 * np.spacing(scale))
    e = LennardJones(1.3, 0.9).pair_energy(rsq)
    np.testing.assert_allclose(e, O.lj_pair_energy(rsq, 1.3, 0.9), rtol=1e-15)


def test_sd_worked_examples():
    f = spring_dashpot_force(Vec3(0.8, 0, 0), 0.64, Vec3(0, 0, 0), Vec3(0, 0, 0), 100.0, 0.0, 1.0)
    assert f.x == pytest.approx(20.0, abs=1e-12) and (f.y, f.z) == (0.0, 0.0)
    f = spring_dashpot_force(Vec3(0.8, 0, 0), 0.64, Vec3(-1, 0, 0), Vec3(1, 0, 0), 0.0, 3.0, 1.0)
    assert f.x == pytest.approx(6.0, abs=1e-12)
    f = spring_dashpot_force(Vec3(1.2, 0, 0), 1.44, Vec3(1, 0, 0), Vec3(-1, 0, 0), 100.0, 5.0, 1.0)
    assert (f.x, f.y, f.z) == (0.0, 0.0, 0.0)
    with pytest.raises(SingularityError):
        spring_dashpot_force(Vec3(0, 0, 0), 0.0, Vec3(0, 0, 0), Vec3(0, 0, 0), 1.0, 1.0, 1.0)


def test_sd_matches_oracle_bitwise_and_antisymmetric():
    rng = np.random.default_rng(7)
    n = 10_000
    d = rng.normal(size=(n, 3))
    d *= rng.uniform(0.3, 1.2, size=n)[:, None] / np.linalg.norm(d, axis=1)[:, None]
    rsq = (d * d).sum(axis=1)
    vi, vj = rng.normal(size=(2, n, 3))
    law = SpringDashpot(80.0, 2.5, 1.0)
    fwd = law.pair_force(d, rsq, vi, vj)
    assert np.array_equal(fwd, O.sd_pair_force(d, rsq, vi, vj, 80.0, 2.5, 1.0))
    assert np.array_equal(fwd, -law.pair_force(-d, rsq, vj, vi))


# --------------------------------------------------------------------------
# binning and lists (test_neighbor.py)
# --------------------------------------------------------------------------

def test_binning_known_answers_and_shell():
    g = build_cell_grid(make_store([[5.7, 0.1, 0.2]]), AABB.cube(0.0, 8.4), 2.8)
    assert tuple(g.coords[0] - 1) == (2, 0, 0)
    g = build_cell_grid(make_store([[2.8, 0.0, 0.0]]), AABB.cube(0.0, 8.4), 2.8)
    assert g.coords[0][0] - 1 == 1
    build_cell_grid(make_store([[5.0, 5, 5], [-2.4, 5, 5]], n_ghost=1), AABB.cube(0.0, 10.0), 2.5)
    with pytest.raises(ProtocolError):
        build_cell_grid(make_store([[5.0, 5, 5], [-2.6, 5, 5]], n_ghost=1), AABB.cube(0.0, 10.0), 2.5)


def test_every_particle_binned_once_matches_oracle():
    rng = np.random.default_rng(8)
    pos = rng.uniform(0, 10, size=(400, 3))
    st = make_store(pos, n_ghost=50)
    g = build_cell_grid(st, AABB.cube(0.0, 10.0), 2.5)
    ob = O.bin_cells(pos, 350, np.zeros(3), np.full(3, 10.0), 2.5)
    assert np.array_equal(g.coords, ob.coords)
    assert np.array_equal(g.occupants, ob.occupants())
    assert int(g.counts.sum()) == 400


@pytest.mark.parametrize("half", [False, True])
def test_random_cloud_lists_equal_oracle_and_brute_force(half):
    rng = np.random.default_rng(21)
    pos = rng.uniform(0, 9, size=(300, 3))
    st = make_store(pos)
    g = build_cell_grid(st, AABB.cube(0.0, 9.0), 2.1)
    lists = build_neighbor_lists(st, g, 2.1, half=half)
    ob = O.bin_cells(pos, 300, np.zeros(3), np.full(3, 9.0), 2.1)
    ot = O.build_lists(pos, 300, ob, 2.1, half=half)
    assert np.array_equal(lists.as_matrix(), ot.mat)
    assert np.array_equal(lists.counts, ot.counts)


def test_capacity_regrow():
    rng = np.random.default_rng(5)
    pos = 5.0 + rng.uniform(-0.1, 0.1, size=(60, 3))
    st = make_store(pos)
    g = build_cell_grid(st, AABB.cube(0.0, 10.0), 2.5)
    lists = build_neighbor_lists(st, g, 2.5, half=False, initial_capacity=4)
    assert lists.counts.tolist() == [59] * 60 and lists.cap == 64


@pytest.mark.parametrize("step", [0, 100])
def test_golden_cells_and_lists_bitwise(golden, step):
    g = golden("lj8_p1")
    p = f"s{step}_"
    pos, n = g[p + "pos"], int(g[p + "nlocal"])
    st = make_store(pos, n_ghost=pos.shape[0] - n)
    box = LJ8.domain()
    grid = build_cell_grid(st, box, LJ8.interaction_radius())
    assert np.array_equal(grid.coords, g[p + "coords"].astype(np.int64))
    if step == 0:
        assert np.array_equal(grid.occupants, g["s0_occupants"])
    lists = build_neighbor_lists(st, grid, LJ8.interaction_radius(), half=False)
    assert np.array_equal(lists.as_matrix(), g[p + "mat"])
    assert np.array_equal(lists.counts, g[p + "lcounts"])


# --------------------------------------------------------------------------
# forces (potential.py:134-213)
# --------------------------------------------------------------------------

@pytest.mark.parametrize("step", [0, 100])
def test_golden_forces_exact_bitwise_fast_within_tol(golden, step):
    g = golden("lj8_p1")
    p = f"s{step}_"
    pos, n = g[p + "pos"], int(g[p + "nlocal"])
    st = make_store(pos, n_ghost=pos.shape[0] - n)
    grid = build_cell_grid(st, LJ8.domain(), 2.8)
    lists = build_neighbor_lists(st, grid, 2.8, half=False)
    law = LennardJones()
    compute_forces(st, lists, law, exact=True)
    assert np.array_equal(st.local_forces(), g[p + "forces"])
    e, w = compute_forces(st, lists, law, exact=False, return_virial=True)
    scale = force_scale(pos, n, g[p + "mat"], g[p + "lcounts"], 6.25)
    assert_forces_close(st.local_forces(), g[p + "forces"], scale)
    table = O.NeighborTable(False, 2.8, g[p + "mat"], g[p + "lcounts"], pos[:n], n)
    _, e_o, w_o = O.evaluate_forces(pos, None, n, table, O.Law.from_cfg(LJ8), energy=True)
    assert abs(e - e_o) <= 1e-12 * abs(e_o) and abs(w - w_o) <= 1e-12 * abs(w_o)


def test_half_lists_and_forces_against_golden(golden):
    g, h = golden("lj8_p1"), golden("lj8_half_s100")
    pos, n = g["s100_pos"], int(g["s100_nlocal"])
    st = make_store(pos, n_ghost=pos.shape[0] - n)
    grid = build_cell_grid(st, LJ8.domain(), 2.8)
    lists = build_neighbor_lists(st, grid, 2.8, half=True)
    assert np.array_equal(lists.as_matrix(), h["mat"])
    e = compute_forces(st, lists, LennardJones(), accumulate_energy=True)
    assert np.max(np.abs(st.local_forces() - h["forces"])) < 1e-10
    assert abs(e - float(h["energy"])) < 1e-9 * abs(float(h["energy"]))


def test_sd_forces_bitwise_against_oracle():
    rng = np.random.default_rng(3)
    pos = rng.uniform(0, 6, size=(500, 3))
    vel = rng.normal(size=(500, 3))
    st = make_store(pos, vel=vel)
    grid = build_cell_grid(st, AABB.cube(0.0, 6.0), 1.5)
    lists = build_neighbor_lists(st, grid, 1.5, half=False)
    law = SpringDashpot(100.0, 0.5, 1.2)
    e = compute_forces(st, lists, law, accumulate_energy=True)
    ob = O.bin_cells(pos, 500, np.zeros(3), np.full(3, 6.0), 1.5)
    ot = O.build_lists(pos, 500, ob, 1.5)
    F, e_o, _ = O.evaluate_forces(pos, vel, 500, ot, O.Law("sd", k=100.0, gamma=0.5, diam=1.2), energy=True)
    assert np.array_equal(st.local_forces(), F)
    assert abs(e - e_o) <= 1e-12 * abs(e_o)


def test_singular_pair_identified():
    st = make_store([[4.0, 4.0, 4.0], [4.0, 4.0, 4.0]])
    grid = build_cell_grid(st, AABB.cube(0, 9), 2.8)
    lists = build_neighbor_lists(st, grid, 2.8, half=False)
    for exact in (True, False):
        with pytest.raises(SingularityError):
            compute_forces(st, lists, LennardJones(), exact=exact)


def test_translation_invariance_exact():
    rng = np.random.default_rng(11)
    pos = (rng.integers(0, 2**22, size=(64, 3)) * 2.0**-20) + 1.0
    outs = []
    for delta in (np.zeros(3), np.array([1.0, 2.0, 0.5])):
        st = make_store(pos + delta)
        grid = build_cell_grid(st, AABB.from_arrays(delta - 16.0, delta + 16.0), 2.8)
        lists = build_neighbor_lists(st, grid, 2.8, half=False)
        compute_forces(st, lists, LennardJones())
        outs.append(st.local_forces())
    np.testing.assert_array_equal(outs[0], outs[1])


# --------------------------------------------------------------------------
# whole runs (driver.py:128-177)
# --------------------------------------------------------------------------

def _thermo_close(got, want, tol=THERMO_TOL):
    # columns: step, PE, KE, W, P
    assert np.array_equal(got[:, 0], want[:, 0])
    for c in (1, 2, 3, 4):
        np.testing.assert_allclose(got[:, c], want[:, c], rtol=tol, atol=0)


def _sorted_state(sim):
    s = sim.store.local_state()
    return s[np.lexsort((s[:, 2], s[:, 1], s[:, 0]))]


def test_lj8_exact_run_bitwise_trajectory(golden):
    g = golden("lj8_p1")
    sim = P.Simulation(LJ8, mode="exact")
    rep = sim.run()
    assert np.array_equal(_sorted_state(sim), g["final_state"])
    _thermo_close(rep.thermo, g["thermo"], 1e-12)
    assert rep.ranks[0].max_displacement_seen == pytest.approx(float(g["max_disp_seen"]), rel=1e-12)


def test_lj8_fast_run_within_tolerance(golden):
    g = golden("lj8_p1")
    sim = P.Simulation(LJ8, mode="fast")
    rep = sim.run()
    _thermo_close(rep.thermo, g["thermo"])
    np.testing.assert_allclose(_sorted_state(sim), g["final_state"], rtol=0, atol=1e-9)
    drift = np.abs(rep.ranks[0].momentum_final - rep.ranks[0].momentum_initial)
    assert np.all(drift <= 1e-9)


def test_sd8_run_bitwise(golden):
    g = golden("sd8_p1")
    sim = P.Simulation(SD8, mode="exact")
    rep = sim.run()
    assert np.array_equal(_sorted_state(sim), g["final_state"])
    _thermo_close(rep.thermo, g["thermo"], 1e-12)


def test_sd8_production_run_within_tolerance(golden):
    """Spring-Dashpot production path (tmd_step_sd: fused contact forces with
    rsqrt arithmetic, pruned split rows, integration, ghost refresh) against
    the reference's own run: thermo within 1e-8, final state within 1e-9."""
    g = golden("sd8_p1")
    sim = P.Simulation(SD8, mode="fast")
    rep = sim.run()
    assert sim.fused and sim.sd and sim.lists.order == "split"
    _thermo_close(rep.thermo, g["thermo"])
    np.testing.assert_allclose(_sorted_state(sim), g["final_state"], rtol=0, atol=1e-9)


def test_sd_step_kernel_per_atom_against_exact():
    """tmd_step_sd's forces (pruning on and off) per atom against the exact
    Spring-Dashpot kernel on reference-order lists of the same state (mid-epoch,
    damped, moving spheres), within 1e-10 scale-relative (potential.py:80-93)."""
    cfg = SimConfig(unit_cells=(10, 10, 10), steps=30, potential_kind="sd", diameter=1.2, cutoff=1.2,
                    stiffness=100.0, damping=0.5, velocity_scale=2.0)
    sim = P.Simulation(cfg, mode="fast")
    gen = sim.iter_steps()
    for _ in range(28):
        next(gen)
    s = sim.store
    n = s.n_local
    pos_all = s.all_positions()
    vel_all = np.vstack([s.local_state()[:, 3:6], np.zeros((s.n_ghost, 3))])
    st = make_store(pos_all, n_ghost=pos_all.shape[0] - n, vel=vel_all)
    r = cfg.interaction_radius()
    grid = build_cell_grid(st, cfg.domain(), r)
    lists = build_neighbor_lists(st, grid, r, half=False)
    law = SpringDashpot(cfg.stiffness, cfg.damping, cfg.diameter)
    compute_forces(st, lists, law, exact=True)
    want = st.local_forces()
    mat, cnt = lists.as_matrix(), lists.counts
    valid = np.arange(mat.shape[1])[None, :] < cnt[:, None]
    j = np.where(valid, mat, 0)
    d = pos_all[:n, None, :] - pos_all[j]
    rsq = O.rsq_ref_order(d)
    inside = valid & (rsq < cfg.diameter ** 2)
    f = O.sd_pair_force(d, np.where(inside, rsq, 1.0), vel_all[:n, None, :], vel_all[j], 100.0, 0.5, 1.2)
    scale = np.where(inside[..., None], np.abs(f), 0.0).sum(axis=1)
    assert np.count_nonzero(np.abs(want).sum(axis=1)) > n // 2  # contacts exist
    for prune in (True, False):
        assert_forces_close(sim.production_forces(prune=prune), want, scale)


def test_guard_violation_raised():
    hot = SimConfig(unit_cells=(6, 6, 6), steps=30, velocity_scale=40.0, reneigh_interval=50)
    with pytest.raises(P.GuardViolation):
        P.Simulation(hot).run()


def _violating_step(exc) -> int:
    return int(str(exc.value).split(":")[0].split()[1])


def test_guard_fail_fast_same_step_and_state_as_reference():
    """driver.py:115-125: the reference raises GuardViolation at the first step
    whose positions moved half the skin, before that step's forces.  The
    production path reports the same step; with check_every_step (the
    rank_program default) it raises there, and without it the step kernels
    freeze on the device at that step, so both leave the same state."""
    hot = SimConfig(unit_cells=(6, 6, 6), steps=30, velocity_scale=12.0, reneigh_interval=50)
    with pytest.raises(O.OracleGuardViolation) as ref:
        O.run(hot, 1)
    k_ref = int(str(ref.value).split("step ")[1].split(":")[0])
    strict = P.Simulation(hot, check_every_step=True)
    with pytest.raises(P.GuardViolation) as e1:
        strict.run()
    lazy = P.Simulation(hot)
    with pytest.raises(P.GuardViolation) as e2:
        lazy.run()
    assert _violating_step(e1) == _violating_step(e2) == k_ref
    assert np.array_equal(_sorted_state(strict), _sorted_state(lazy))


@pytest.mark.parametrize("cfg", [LJ8, SD8], ids=["lj", "sd"])
def test_exact_yields_state_of_step_k(cfg):
    """rank_program semantics (driver.py:128-177): at ("step", k) the store
    holds step k's state.  With exact_yields the fused step is split (forces +
    closing kick, yield, next kick + drift with the stored forces): the
    trajectory is bitwise that of the unsplit run, and the yielded states match
    the oracle's step-k states within the parity tolerance."""
    seen = {}
    O.run(cfg, 1, on_step=lambda k, w: seen.__setitem__(k, w.ranks[0].pos[:w.ranks[0].n_local].copy())
          if k in (0, 37, 100) else None)
    split = P.Simulation(cfg, mode="fast", exact_yields=True)
    got = {}
    for _, k in split.iter_steps():
        if k in (0, 37, 100):
            st = split.store.local_positions()
            got[k] = st[np.lexsort((st[:, 2], st[:, 1], st[:, 0]))]
    rs = split.finish()
    plain = P.Simulation(cfg, mode="fast")
    rp = plain.run()
    assert np.array_equal(rs.thermo, rp.thermo)
    assert np.array_equal(_sorted_state(split), _sorted_state(plain))
    for k, want in seen.items():
        want = want[np.lexsort((want[:, 2], want[:, 1], want[:, 0]))]
        np.testing.assert_allclose(got[k], want, rtol=0, atol=1e-9)


def test_singular_pair_in_a_run_raises():
    """potential.py:174-178 on the production path: a coincident pair within
    the cutoff raises SingularityError (the step kernels freeze after it)."""
    cfg = SimConfig(unit_cells=(5, 5, 5), steps=10)
    pos, vel = O.initial_state(cfg)
    pos = np.vstack([pos, pos[:1]])
    vel = np.vstack([vel, vel[:1]])
    for strict in (False, True):
        sim = P.Simulation(cfg, store=ParticleStore.from_host(pos, vel), check_every_step=strict)
        with pytest.raises(SingularityError):
            sim.run()


def test_lj32_step0_golden(golden):
    g = golden("lj32_step0")
    cfg = SimConfig(unit_cells=(32, 32, 32), steps=0)
    sim = P.Simulation(cfg)
    rep = sim.run()
    assert sim.store.n_ghost == 47883
    np.testing.assert_allclose(rep.thermo[0, 1:3], g["thermo"][0, 1:3], rtol=1e-12)
    assert abs(rep.thermo[0, 1] / 131072 - (-6.773368053252959)) < 1e-12


# --------------------------------------------------------------------------
# production (split) lists and pruning
# --------------------------------------------------------------------------

@pytest.mark.parametrize("shell", [1, 2])
@pytest.mark.parametrize("step", [0, 100])
def test_split_lists_same_sets_and_segments_sound(golden, step, shell):
    """Production lists (r/2 grid, 5^3 stencil, near/far split rows): same sets as the reference."""
    g = golden("lj8_p1")
    p = f"s{step}_"
    pos, n = g[p + "pos"], int(g[p + "nlocal"])
    st = make_store(pos, n_ghost=pos.shape[0] - n)
    grid = build_cell_grid(st, LJ8.domain(), 2.8, shell=shell)
    lists = build_neighbor_lists(st, grid, 2.8, half=False, order="split", cutoff=2.5)
    mat, cnt = lists.as_matrix(), lists.counts
    assert np.array_equal(cnt, g[p + "lcounts"])
    want = g[p + "mat"]
    for i in range(n):
        assert sorted(mat[i, :cnt[i]]) == sorted(want[i, :cnt[i]])
    # near entries inside cutoff + margin, far entries outside it
    nn = lists.nnear[:n].cpu().numpy()
    near_r2 = (2.5 + lists.near_margin) ** 2
    d = pos[:n, None, :] - pos[np.where(mat >= 0, mat, 0)]
    rsq = O.rsq_ref_order(d)
    slot = np.arange(mat.shape[1])[None, :]
    assert np.all(rsq[slot < nn[:, None]] < near_r2)
    assert np.all(rsq[(slot >= nn[:, None]) & (slot < cnt[:, None])] >= near_r2)


@pytest.mark.parametrize("kind", ["threshold-lattice", "hot", "far-from-origin"])
def test_split_float_prefilter_rows_bitwise(kind):
    """The split builder's float pre-filter (cell_pos_f, decided only when the
    float rsq is more than tinymd_f32_eps from both thresholds) gives the same
    rows, near counts and totals, bit for bit, as the double-only walk -- on a
    simple-cubic lattice of spacing r/2 (pairs exactly at the list radius and
    near it), on a hot random state and far from the origin."""
    rng = np.random.default_rng(7)
    r, cut = 2.8, 2.5
    if kind == "threshold-lattice":
        side = 24
        g = np.arange(side) * (r / 2)
        pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3) + 0.05
        box = AABB.cube(0.0, side * r / 2 + 0.1)
    else:
        side = 20
        g = np.arange(side) * 1.5
        pos = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
        pos = pos + rng.normal(0.0, 0.15, pos.shape) + 0.5
        off = 1000.0 if kind == "far-from-origin" else 0.0
        pos = pos + off
        box = AABB.cube(off, off + side * 1.5 + 1.0)
    rows = []
    for use_f32 in (True, False):
        st = make_store(pos)
        grid = build_cell_grid(st, box, r, shell=2)
        assert grid.cell_pos_f is not None
        if not use_f32:
            grid.cell_pos_f = None
        lists = build_neighbor_lists(st, grid, r, half=False, order="split", cutoff=cut, margin=0.12)
        rows.append((lists.as_matrix(), lists.counts.copy(), lists.nnear[:st.n_local].cpu().numpy()))
    for a, b in zip(rows[0], rows[1]):
        assert np.array_equal(a, b)
    assert rows[0][1].sum() > 0


def test_fused_pruned_path_matches_exact_every_step():
    """Fast path (cell-sorted atoms, split lists, pruning by displacement) vs the exact path.

    Hot atoms move far within an epoch, so every pruning tier is exercised; a
    pair wrongly pruned would shift PE by ~1e-6 relative, far above 1e-10.
    """
    cfg = SimConfig(unit_cells=(6, 6, 6), steps=40, reneigh_interval=10, velocity_scale=2.2)
    fast = P.Simulation(cfg, mode="fast").run()
    exact_sim = P.Simulation(cfg, mode="exact")
    exact = exact_sim.run()
    np.testing.assert_allclose(fast.thermo[:, 1:5], exact.thermo[:, 1:5], rtol=1e-10, atol=0)
    assert fast.ranks[0].max_displacement_seen > 0.05  # the upper tiers were in use


@pytest.mark.parametrize("cells,reneigh", [(8, 20), (6, 7)])
def test_fused_ghost_refresh_equals_three_round_sync(cells, reneigh):
    """The step kernel's own ghost writes (export table) vs the reference's
    synchronize rounds: same trajectory bit for bit (x_root + s == hop sums)."""
    cfg = SimConfig(unit_cells=(cells,) * 3, steps=45, reneigh_interval=reneigh)
    a = P.Simulation(cfg, mode="fast", fused_refresh=True)
    ra = a.run()
    assert a.exports is not None and a.exports.n_entries == a.store.n_ghost <= a.exports.n_ex
    b = P.Simulation(cfg, mode="fast", fused_refresh=False)
    rb = b.run()
    assert b.exports is None
    assert np.array_equal(ra.thermo, rb.thermo)
    assert np.array_equal(_sorted_state(a), _sorted_state(b))
    # ghosts of the final state mirror their roots exactly
    s = a.store
    if a.rebuild_steps[a.steps]:
        return
    pos = s.pos[:, : s.n_total].cpu().numpy()
    root = a.plan.prov_root.cpu().numpy()
    sh = a.plan.prov_sh.cpu().numpy()
    assert np.array_equal(pos[:, s.n_local:], pos[:, root] + sh)


@pytest.mark.parametrize("step", [0, 100])
def test_direct_borders_same_ghosts_as_three_rounds(golden, step):
    """One-pass periodic borders (P = 1 production path) vs the reference's
    three self rounds: identical ghost coordinates (as a multiset, bitwise),
    and each ghost equals its root plus its recorded shift."""
    g = golden("lj8_p1")
    p = f"s{step}_"
    n = int(g[p + "nlocal"])
    pos = g[p + "pos"][:n]
    decomp = P.Decomposition(LJ8.domain(), 1, 0, LJ8.interaction_radius())
    plans = {}
    for direct in (False, True):
        st = make_store(pos)
        plans[direct] = (P.Halo(decomp).define_borders(st, provenance=True, direct=direct), st)
    (pa, sa), (pb, sb) = plans[False], plans[True]
    assert pb.rounds == [] and pb.n_ghost == pa.n_ghost == sa.n_ghost
    ga = sa.all_positions()[n:]
    gb = sb.all_positions()[n:]
    assert np.array_equal(ga[np.lexsort(ga.T[::-1])], gb[np.lexsort(gb.T[::-1])])
    for plan, st in plans.values():
        allp = st.all_positions()
        root = plan.prov_root.cpu().numpy()
        sh = plan.prov_sh.cpu().numpy().T
        assert np.array_equal(allp[n:], allp[root] + sh)
        assert np.all(plan.prov_rank.cpu().numpy() == 0)


def test_integration_stub_layout_bitwise(golden):
    """INTEGRATION.md's ctypes stub: a plain (n, cap) list matrix converted to
    the quad-interleaved layout and passed to tmd_force_lj gives the same
    forces as compute_forces (exact mode), bit for bit."""
    import ctypes as C

    import torch

    from paper_2009_07400_b200 import _native as N

    g = golden("lj8_p1")
    pos = g["s0_pos"]
    n = int(g["s0_nlocal"])
    st = make_store(pos, n_ghost=pos.shape[0] - n)
    grid = build_cell_grid(st, LJ8.domain(), 2.8)
    lists = build_neighbor_lists(st, grid, 2.8, half=False)
    law = LennardJones()
    compute_forces(st, lists, law, exact=True)
    want = st.local_forces()
    lib = C.CDLL(N.LIB_PATH)
    mat = lists.as_matrix()
    q = (mat.shape[1] + 3) // 4
    quad = np.zeros((n, 4 * q), dtype=np.int32)
    quad[:, :mat.shape[1]] = np.where(mat >= 0, mat, 0)
    nbr = torch.from_numpy(np.ascontiguousarray(quad.reshape(n, q, 4).transpose(1, 0, 2))).cuda()
    n_tot = pos.shape[0]
    p = torch.from_numpy(np.ascontiguousarray(pos.T)).cuda()
    cnt = torch.from_numpy(lists.counts.astype(np.int32)).cuda()
    frc = torch.empty((3, n), dtype=torch.float64, device="cuda")
    thermo = torch.zeros(2, dtype=torch.float64, device="cuda")
    status = torch.zeros(4, dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    v, i32, i64, u32, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_double
    lib.tmd_force_lj.argtypes = [v, i64, i32, v, i64, v, i32, f64, f64, f64, u32, v, i64, v, v, v]
    lib.tmd_status_reset.argtypes = [v, v]
    lib.tmd_status_reset(status.data_ptr(), s)
    rc = lib.tmd_force_lj(p.data_ptr(), n_tot, n, nbr.data_ptr(), n, cnt.data_ptr(), 4 * q, law.cutoff_rsq,
                          law.epsilon, law.sigma ** 6, N.F_EXACT, frc.data_ptr(), n, thermo.data_ptr(),
                          status.data_ptr(), s)
    assert rc == 0 and int(status[0].item()) == 0
    assert np.array_equal(frc.t().cpu().numpy(), want)


# --------------------------------------------------------------------------
# the production step kernel itself (tmd_step_lj), per atom
# --------------------------------------------------------------------------

def _exact_forces_on(pos_all, n, cfg):
    """Reference-order lists + the exact kernel on the same positions (bitwise
    the reference's compute_forces): per-atom forces and the force scale."""
    st = make_store(pos_all, n_ghost=pos_all.shape[0] - n)
    r = cfg.interaction_radius()
    grid = build_cell_grid(st, cfg.domain(), r)
    lists = build_neighbor_lists(st, grid, r, half=False)
    compute_forces(st, lists, LennardJones(cfg.epsilon, cfg.sigma), exact=True)
    mat, cnt = lists.as_matrix(), lists.counts
    return st.local_forces(), force_scale(pos_all, n, mat, cnt, cfg.cutoff ** 2)


def _by_position(pos, arr):
    order = np.lexsort((pos[:, 2], pos[:, 1], pos[:, 0]))
    return arr[order]


@pytest.mark.parametrize("prune", [True, False])
def test_step_kernel_per_atom_golden_s100(golden, prune):
    """tmd_step_lj (production: brick-numbered atoms, split rows, pruning on
    and forced off, no integration phase) on the reference's step-100 state:
    per-atom forces within 1e-10 scale-relative of the reference's own
    step-100 forces (potential.py:134-213)."""
    g = golden("lj8_p1")
    n = int(g["s100_nlocal"])
    pos, vel = g["s100_pos"][:n], g["s100_vel"][:n]
    sim = P.Simulation(LJ8, store=ParticleStore.from_host(pos, vel), mode="fast")
    sim.rebuild()
    got = sim.production_forces(prune=prune)
    mine = sim.store.local_positions()
    assert sim.lists.order == "split" and int(sim.lists.nnear[:n].sum()) < int(sim.lists.d_counts[:n].sum())
    scale = force_scale(g["s100_pos"], n, g["s100_mat"], g["s100_lcounts"], 6.25)
    want = _by_position(pos, g["s100_forces"])
    assert np.array_equal(_by_position(mine, mine), _by_position(pos, pos))
    assert_forces_close(_by_position(mine, got), want, _by_position(pos, scale))


def test_step_kernel_per_atom_hot_state_pruned_and_unpruned():
    """A 10^3 system stopped mid-epoch (atoms moved since the build, so the
    per-atom pruning skips some back segments and must scan others): the
    production kernel with pruning on and off against the exact kernel on
    reference-order lists of the same positions, per atom within 1e-10."""
    cfg = SimConfig(unit_cells=(10, 10, 10), steps=40)
    sim = P.Simulation(cfg, mode="fast")
    gen = sim.iter_steps()
    for _ in range(36):  # setup + 35 steps: 15 steps into the second epoch
        next(gen)
    s = sim.store
    n = s.n_local
    moved = float(np.sqrt(sim.dispmax2[36].item()))  # x(36): step 35's kernel drifted the atoms
    assert 0.0 < moved < 0.5 * cfg.verlet_buffer
    want, scale = _exact_forces_on(s.all_positions(), n, cfg)
    for prune in (True, False):
        assert_forces_close(sim.production_forces(prune=prune), want, scale)


def test_lj32_production_run_against_reference_golden(golden):
    """BASELINE configs[1] (32^3 = 131,072 atoms) for 100 steps on the
    production path against the reference's own run: thermo within 1e-8 at
    every step, sorted final state within 1e-9, momentum drift <= 1e-9."""
    g = golden("lj32_p1")
    cfg = SimConfig(unit_cells=(32, 32, 32), steps=100)
    sim = P.Simulation(cfg, mode="fast")
    rep = sim.run()
    _thermo_close(rep.thermo, g["thermo"])
    np.testing.assert_allclose(_sorted_state(sim), g["final_state"], rtol=0, atol=1e-9)
    assert np.all(np.abs(rep.thermo[-1, 5:8] - rep.thermo[0, 5:8]) <= 1e-9)


def test_lj80_production_vs_exact_100_steps():
    """The benchmarked configuration (80^3 = 2,048,000 atoms): the production
    path against the GPU exact mode (bitwise the reference's arithmetic) over
    100 steps -- thermo within 1e-10, final state within 1e-9 -- and the
    step-0 PE per atom of the perfect lattice."""
    cfg = SimConfig(unit_cells=(80, 80, 80), steps=100)
    fast = P.Simulation(cfg, mode="fast")
    rf = fast.run()
    assert abs(rf.thermo[0, 1] / 2_048_000 - (-6.773368053252959)) < 1e-12
    sf = _sorted_state(fast)
    del fast
    exact = P.Simulation(cfg, mode="exact")
    re_ = exact.run()
    np.testing.assert_allclose(rf.thermo[:, 1:5], re_.thermo[:, 1:5], rtol=1e-10, atol=0)
    np.testing.assert_allclose(sf, _sorted_state(exact), rtol=0, atol=1e-9)


@pytest.mark.parametrize("cells,extra", [((4, 4, 4), {}), ((10, 17, 6), {}),
                                         ((12, 7, 9), {"velocity_scale": 3.0, "reneigh_interval": 10}),
                                         ((9, 13, 11), {"potential_kind": "sd", "diameter": 1.2, "cutoff": 1.2,
                                                        "stiffness": 100.0, "damping": 0.0})],
                         ids=["lj4", "lj-noncubic", "lj-hot", "sd-noncubic-undamped"])
def test_production_vs_exact_odd_boxes(cells, extra):
    """Small and non-cubic boxes (uneven brick and cell counts per axis, a hot
    start, an undamped DEM): the production path (renumbering, split rows,
    device-count epoch, batched steps) against the GPU exact mode over 60
    steps (3 or 6 rebuilds)."""
    cfg = SimConfig(unit_cells=cells, steps=60, **extra)
    fast = P.Simulation(cfg, mode="fast")
    rf = fast.run()
    exact = P.Simulation(cfg, mode="exact")
    re_ = exact.run()
    np.testing.assert_allclose(rf.thermo[:, 1:5], re_.thermo[:, 1:5], rtol=THERMO_TOL, atol=1e-9)
    np.testing.assert_allclose(_sorted_state(fast), _sorted_state(exact), rtol=0, atol=1e-9)


def test_multi_gpu_parity_torchrun():
    """2 ranks over NCCL + NVLink (scripts/mgpu_check.py): exact mode bitwise
    the reference's own 2-rank run, the production path (direct protocol,
    owner-written ghosts, mailbox barrier) within 1e-13.  Needs >= 2 GPUs."""
    import json
    import os
    import subprocess
    import sys

    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--nproc-per-node", "2",
                          os.path.join(root, "scripts", "mgpu_check.py")], capture_output=True, text=True,
                         timeout=600, cwd=root)
    checks = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert out.returncode == 0, out.stderr[-2000:]
    assert len(checks) == 6 and all(c["pass"] for c in checks), checks


@pytest.mark.parametrize("m,n_ranks", [(1, 2), (1000, 3), (4096, 8), (4097, 2), (250_000, 8)])
def test_group_by_rank_stable_multi_block(m, n_ranks):
    """tmd_group_by_rank (the direct protocol's per-peer send lists): a stable
    grouping by destination rank, equal to numpy's stable argsort, across the
    multi-block passes (4096 records per block)."""
    import torch

    from paper_2009_07400_b200.halo_ops import DeviceHaloOps

    rng = np.random.default_rng(m + n_ranks)
    rank = rng.integers(-1, n_ranks, m).astype(np.int32)  # -1: the record drops out
    if m > 10_000:
        rank[: m // 3] = n_ranks - 1  # a long run of one rank across blocks
    ids = rng.integers(0, 1 << 30, m).astype(np.int32)
    dev = torch.device("cuda", 0)
    got_ids, got_rank, counts = DeviceHaloOps().group_by_rank(torch.from_numpy(rank).to(dev),
                                                              torch.from_numpy(ids).to(dev), n_ranks)
    keep = np.nonzero(rank >= 0)[0]
    order = keep[np.argsort(rank[keep], kind="stable")]
    k = order.size
    assert np.array_equal(got_ids.cpu().numpy()[:k], ids[order])
    assert np.array_equal(got_rank.cpu().numpy()[:k], rank[order])
    assert np.array_equal(counts.cpu().numpy(), np.bincount(rank[keep], minlength=n_ranks))


@pytest.mark.parametrize("cfg", [LJ8, SD8], ids=["lj", "sd"])
def test_device_count_epoch_matches_synchronous_epoch(cfg, monkeypatch):
    """The P = 1 epoch with the ghost count kept on the device (one host sync),
    issued by one library call (tmd_epoch_p1) or from Python, runs the same
    trajectory, bit for bit, as the synchronous epoch; an epoch whose ghosts
    exceed the reserved room falls back to the synchronous one."""
    a = P.Simulation(cfg)  # the native epoch (tmd_epoch_p1)
    ra = a.run()
    monkeypatch.setenv("TMD_EPOCH_SYNC", "1")
    b = P.Simulation(cfg)
    rb = b.run()
    monkeypatch.delenv("TMD_EPOCH_SYNC")
    assert np.array_equal(ra.thermo, rb.thermo)
    assert np.array_equal(_sorted_state(a), _sorted_state(b))
    monkeypatch.setenv("TMD_EPOCH_NATIVE", "0")  # the same epoch driven from Python
    d = P.Simulation(cfg)
    rd = d.run()
    monkeypatch.delenv("TMD_EPOCH_NATIVE")
    assert np.array_equal(ra.thermo, rd.thermo)
    assert np.array_equal(_sorted_state(a), _sorted_state(d))
    # room too small at every epoch after setup: each falls back and grows the store
    c = P.Simulation(cfg)
    calls = []
    monkeypatch.setattr(c, "_ghost_room", lambda: calls.append(1) or 16)
    rc = c.run()
    assert len(calls) == cfg.steps // cfg.reneigh_interval + 1  # the setup epoch too
    assert np.array_equal(ra.thermo, rc.thermo)
    assert np.array_equal(_sorted_state(a), _sorted_state(c))


@pytest.mark.parametrize("cfg", [LJ8, SD8, SimConfig(unit_cells=(6, 6, 6), steps=45, reneigh_interval=7)], ids=["lj", "sd", "odd-epochs"])
def test_batched_step_loop_matches_per_step_loop(cfg, monkeypatch):
    """Simulation.run drives the steps between epochs with one tmd_run_steps
    call per epoch; the per-step Python loop (iter_steps) is the same
    trajectory bit for bit (thermo rows, final state, forces)."""
    a = P.Simulation(cfg)
    ra = a.run()
    assert a._batched
    monkeypatch.setenv("TMD_BATCH", "0")
    b = P.Simulation(cfg)
    rb = b.run()
    assert not b._batched
    assert np.array_equal(ra.thermo, rb.thermo)
    assert np.array_equal(_sorted_state(a), _sorted_state(b))
    fa = a.store.local_forces()[np.lexsort(a.store.local_positions().T[::-1])]
    fb = b.store.local_forces()[np.lexsort(b.store.local_positions().T[::-1])]
    assert np.array_equal(fa, fb)


def test_batched_advance_in_pieces_and_launch_times():
    """advance(n) in uneven pieces (crossing epochs) equals one run; the
    per-launch device times come back for every timed launch."""
    cfg = SimConfig(unit_cells=(6, 6, 6), steps=50, reneigh_interval=7)
    a = P.Simulation(cfg)
    ra = a.run()
    b = P.Simulation(cfg)
    b.event_pairs = []
    b.start()
    b.launch_times()
    for n in (3, 4, 1, 13, 100):
        b.advance(n)
    rb = b.finish()
    assert np.array_equal(ra.thermo, rb.thermo)
    assert len(b.launch_times()) == 50  # steps 1 .. 50, one launch each
    c = P.Simulation(cfg)
    c.event_pairs = []
    c.start()
    c.launch_times()
    c.advance(20)
    t = c.launch_times()
    assert len(t) == 20 and all(x > 0 for x in t)
    c.advance(100)
