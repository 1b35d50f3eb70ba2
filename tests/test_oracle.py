"""Pin the CPU oracle to the reference: golden fixtures (made by running the
reference itself, tests/golden/make_golden.py) must be reproduced bit for bit.

CPU only; these run in the driver's ``-m "not gpu"`` pass.
"""

import os

import numpy as np
import pytest

import oracle as O
from paper_2009_07400_b200.core import SimConfig

LJ8 = SimConfig(unit_cells=(8, 8, 8), steps=100)
SD8 = SimConfig(unit_cells=(8, 8, 8), steps=100, potential_kind="sd", diameter=1.2,
                cutoff=1.2, stiffness=100.0, damping=0.5)


def test_einsum_order_matches_this_numpy():
    # the bit-exact predicates rely on this order
    rng = np.random.default_rng(0)
    d = rng.normal(size=(2048, 64, 3)) * 2.0
    assert np.array_equal(O.rsq_ref_order(d), np.einsum("ijk,ijk->ij", d, d))
    u, v = rng.normal(size=(2, 4096, 16, 3))
    assert np.array_equal(O.dot3_ref_order(u, v), np.einsum("...k,...k->...", u, v))


def test_lattice_counts_and_velocities():
    # test_particles.py:16-24
    assert O.lattice_positions(SimConfig(unit_cells=(32, 32, 32))).shape == (131072, 3)
    assert O.lattice_positions(SimConfig(unit_cells=(96, 96, 96))).shape == (3538944, 3)
    pos, vel = O.initial_state(LJ8)
    assert np.all(np.abs(vel.sum(axis=0)) < 1e-12)


def test_lj_known_answers():
    # test_potential.py:28-30, 48-66
    f = O.lj_pair_force(np.array([1.0, 0.0, 0.0]), np.float64(1.0), 1.0, 1.0)
    assert tuple(f) == (24.0, 0.0, 0.0)
    rng = np.random.default_rng(42)
    r = rng.uniform(0.8, 2.5, size=10_000)
    u = rng.normal(size=(10_000, 3))
    u /= np.linalg.norm(u, axis=1)[:, None]
    d = u * r[:, None]
    rsq = (d * d).sum(axis=1)
    got = O.lj_pair_force(d, rsq, 1.0, 1.0)
    s6 = (1.0 / rsq) ** 3
    want = (24.0 * s6 * (2.0 * s6 - 1.0) / rsq)[:, None] * d
    mag = (48.0 * s6 * (s6 + 0.5) / rsq)[:, None] * np.abs(d)
    scale = np.maximum(np.maximum(np.abs(got), np.abs(want)), mag)
    assert np.all(np.abs(got - want) <= 4 * np.spacing(scale))


def test_sd_known_answers():
    # test_potential.py:83-111
    z = np.zeros(3)
    f = O.sd_pair_force(np.array([0.8, 0.0, 0.0]), np.float64(0.64), z, z, 100.0, 0.0, 1.0)
    assert f[0] == pytest.approx(20.0, abs=1e-12) and f[1] == 0.0 and f[2] == 0.0
    f = O.sd_pair_force(np.array([0.8, 0, 0]), np.float64(0.64), np.array([-1.0, 0, 0]),
                        np.array([1.0, 0, 0]), 0.0, 3.0, 1.0)
    assert f[0] == pytest.approx(6.0, abs=1e-12)
    f = O.sd_pair_force(np.array([1.2, 0, 0]), np.float64(1.44), np.array([1.0, 0, 0]),
                        np.array([-1.0, 0, 0]), 100.0, 5.0, 1.0)
    assert tuple(f) == (0.0, 0.0, 0.0)


def test_binning_known_answers():
    # test_neighbor.py:37-47, 59-65
    b = O.bin_cells(np.array([[5.7, 0.1, 0.2]]), 1, np.zeros(3), np.full(3, 8.4), 2.8)
    assert tuple(b.coords[0] - 1) == (2, 0, 0)
    b = O.bin_cells(np.array([[2.8, 0.0, 0.0]]), 1, np.zeros(3), np.full(3, 8.4), 2.8)
    assert b.coords[0][0] - 1 == 1
    O.bin_cells(np.array([[5.0, 5, 5], [-2.4, 5, 5]]), 1, np.zeros(3), np.full(3, 10.0), 2.5)
    with pytest.raises(O.OracleProtocolError):
        O.bin_cells(np.array([[5.0, 5, 5], [-2.6, 5, 5]]), 1, np.zeros(3), np.full(3, 10.0), 2.5)


@pytest.mark.parametrize("half", [False, True])
def test_lists_match_brute_force(half):
    # test_neighbor.py:87-104
    rng = np.random.default_rng(21)
    pos = rng.uniform(0, 9, size=(300, 3))
    b = O.bin_cells(pos, 300, np.zeros(3), np.full(3, 9.0), 2.1)
    t = O.build_lists(pos, 300, b, 2.1, half=half)
    got = {(min(i, j), max(i, j)) for i, j in t.pairs()}
    want = set()
    for i in range(300):
        dd = pos[i] - pos
        rsq = (dd * dd).sum(axis=1)
        want |= {(i, j) for j in range(i + 1, 300) if rsq[j] < 2.1 * 2.1}
    assert got == want
    assert len(t.pairs()) == (len(want) if half else 2 * len(want))


def test_capacity_regrow():
    # test_neighbor.py:149-157
    rng = np.random.default_rng(5)
    pos = 5.0 + rng.uniform(-0.1, 0.1, size=(60, 3))
    b = O.bin_cells(pos, 60, np.zeros(3), np.full(3, 10.0), 2.5)
    t = O.build_lists(pos, 60, b, 2.5, cap=4)
    assert t.counts.tolist() == [59] * 60 and t.cap == 64


@pytest.fixture(scope="module")
def lj8_run():
    snaps = {}

    def grab(step, world):
        if step in (0, 100):
            R = world.ranks[0]
            snaps[step] = dict(pos=R.pos.copy(), bins=R.bins, table=R.table,
                               F=R.frc[:R.n_local].copy())

    run = O.run(LJ8, 1, on_step=grab)
    return run, snaps


def test_lj8_p1_thermo_and_state_bitwise(lj8_run, golden):
    run, _ = lj8_run
    g = golden("lj8_p1")
    # PE, KE, momentum bitwise; the virial (our extension) to 1e-12
    assert np.array_equal(run.thermo[:, [0, 1, 2, 5, 6, 7]], g["thermo"][:, [0, 1, 2, 5, 6, 7]])
    np.testing.assert_allclose(run.thermo[:, 3:5], g["thermo"][:, 3:5], rtol=1e-12)
    assert np.array_equal(run.global_state(), g["final_state"])
    assert np.array_equal(run.momentum_final, g["momentum_final"])
    assert run.thermo[0, 1] / 2048 == -6.773368053252959
    assert run.world.ranks[0].max_disp_seen == float(g["max_disp_seen"])


@pytest.mark.parametrize("step", [0, 100])
def test_lj8_p1_cells_lists_forces_bitwise(lj8_run, golden, step):
    _, snaps = lj8_run
    g = golden("lj8_p1")
    s = snaps[step]
    p = f"s{step}_"
    assert np.array_equal(s["pos"], g[p + "pos"])
    assert np.array_equal(s["bins"].coords, g[p + "coords"].astype(np.int64))
    assert np.array_equal(s["table"].mat, g[p + "mat"])
    assert np.array_equal(s["table"].counts, g[p + "lcounts"])
    assert np.array_equal(s["F"], g[p + "forces"])
    if step == 0:
        assert np.array_equal(s["bins"].occupants(), g["s0_occupants"])
        assert np.array_equal(s["bins"].counts, g["s0_counts"].astype(np.int64))
        assert s["pos"].shape[0] - 2048 == 4035
        assert set(np.unique(s["table"].counts)) == {78}


def test_half_mode_bitwise(golden):
    g, h = golden("lj8_p1"), golden("lj8_half_s100")
    pos, n = g["s100_pos"], int(g["s100_nlocal"])
    lo, hi = O.domain_bounds(LJ8)
    b = O.bin_cells(pos, n, lo, hi, 2.8)
    t = O.build_lists(pos, n, b, 2.8, half=True)
    assert np.array_equal(t.mat, h["mat"]) and np.array_equal(t.counts, h["counts"])
    F, e, _ = O.evaluate_forces(pos, g["s100_vel"], n, t, O.Law.from_cfg(LJ8), energy=True)
    assert np.array_equal(F, h["forces"]) and e == float(h["energy"])
    # half == full within 1e-10 (test_potential.py:178-188)
    assert np.max(np.abs(F - g["s100_forces"])) < 1e-10


@pytest.mark.parametrize("p", [2, 4, 8])
def test_lj8_multirank_bitwise(golden, p):
    g = golden(f"lj8_p{p}")
    run = O.run(LJ8, p)
    assert np.array_equal(run.thermo[:, [0, 1, 2]], g["thermo"][:, [0, 1, 2]])
    np.testing.assert_allclose(run.thermo[:, 3:5], g["thermo"][:, 3:5], rtol=1e-12)
    assert np.array_equal(run.global_state(), g["final_state"])
    assert [R.n_local for R in run.world.ranks] == g["n_local"].tolist()
    assert [R.n_ghost for R in run.world.ranks] == g["n_ghost"].tolist()
    # cross-P: within the north-star tolerance of the P = 1 run
    g1 = golden("lj8_p1")
    np.testing.assert_allclose(run.global_state(), g1["final_state"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("p", [1, 8])
def test_sd8_bitwise(golden, p):
    g = golden(f"sd8_p{p}")
    run = O.run(SD8, p)
    assert np.array_equal(run.thermo[:, [0, 1, 2]], g["thermo"][:, [0, 1, 2]])
    np.testing.assert_allclose(run.thermo[:, 3:5], g["thermo"][:, 3:5], rtol=1e-12)
    assert np.array_equal(run.global_state(), g["final_state"])


@pytest.mark.slow
def test_lj32_step0(golden):
    g = golden("lj32_step0")
    cfg = SimConfig(unit_cells=(32, 32, 32), steps=0)
    seen = {}
    run = O.run(cfg, 1, on_step=lambda s, w: seen.update(ng=w.ranks[0].n_ghost,
                                                          cnt=np.bincount(w.ranks[0].table.counts),
                                                          cap=w.ranks[0].table.cap))
    assert np.array_equal(run.thermo[:, [0, 1, 2]], g["thermo"][:, [0, 1, 2]])
    assert seen["ng"] == int(g["n_ghost"]) == 47883
    assert np.array_equal(seen["cnt"], g["lcounts"]) and seen["cap"] == int(g["cap"])


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference not mounted")
def test_oracle_vs_live_reference_small():
    """Where the reference is importable (this container), compare live on a 5^3 run."""
    import sys

    sys.path.insert(0, os.path.join(os.path.dirname(__file__), "golden"))
    from make_golden import _import_reference, reference_run, sorted_state

    cfg = SimConfig(unit_cells=(5, 5, 5), steps=25, reneigh_interval=5)
    rcfg = _import_reference()["core"].SimConfig(unit_cells=(5, 5, 5), steps=25, reneigh_interval=5)
    rows, stores, _ = reference_run(rcfg, 2)
    run = O.run(cfg, 2)
    assert np.array_equal(run.thermo[:, :3], rows[:, :3])
    assert np.array_equal(run.global_state(), sorted_state(stores))


@pytest.mark.slow
def test_lj32_first_steps_thermo_bitwise(golden):
    """BASELINE configs[1] (32^3): the oracle's thermo rows over steps 0..20
    (one in-loop rebuild) equal the reference's 100-step run bit for bit."""
    g = golden("lj32_p1")
    cfg = SimConfig(unit_cells=(32, 32, 32), steps=20)
    run = O.run(cfg, 1, threads=os.cpu_count() or 1)
    assert np.array_equal(run.thermo[:, [0, 1, 2]], g["thermo"][:21, [0, 1, 2]])
    np.testing.assert_allclose(run.thermo[:, 3:5], g["thermo"][:21, 3:5], rtol=1e-12)
    assert np.array_equal(run.thermo[:, 5:8], g["thermo"][:21, 5:8])
