"""P > 1 device path on ONE GPU: P in-process ranks (paper_2009_07400_b200.loopback),
each with its own thread and CUDA stream, against the reference's own P-rank
runs (golden lj8_p{2,4,8}, sd8_p8 from tests/golden/make_golden.py).

The real multi-rank kernels run here: tmd_exchange_classify, tmd_borders_count
/ tmd_borders_fill with destination ranks, tmd_exports_build, the step
kernel's ghost writes into a peer's next position buffer, and the per-step
mailbox barrier tmd_peer_sync.  Only the transport differs from torchrun
(device copies + a host barrier instead of NCCL; device pointers instead of
CUDA-IPC mappings).  Reference: comm.py:340-498, driver.py:128-177.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2009_07400_b200")
from paper_2009_07400_b200 import SimConfig, run_loopback  # noqa: E402

LJ8 = SimConfig(unit_cells=(8, 8, 8), steps=100)
SD8 = SimConfig(unit_cells=(8, 8, 8), steps=100, potential_kind="sd", diameter=1.2, cutoff=1.2,
                stiffness=100.0, damping=0.5)
THERMO_TOL = 1e-8


def _global_state(sims):
    s = np.vstack([sim.store.local_state() for sim in sims])
    return s[np.lexsort((s[:, 2], s[:, 1], s[:, 0]))]


def _thermo_close(got, want, tol):
    assert np.array_equal(got[:, 0], want[:, 0])
    for c in (1, 2, 3, 4):
        np.testing.assert_allclose(got[:, c], want[:, c], rtol=tol, atol=0)


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_lj8_exact_loopback_bitwise(golden, nranks):
    """Reference protocol (three NCCL-style rounds, exact kernels): bitwise the
    reference's own P-rank trajectory."""
    g = golden(f"lj8_p{nranks}")
    reps, sims = run_loopback(LJ8, nranks, mode="exact", peer_timeout_s=30.0)
    assert np.array_equal(_global_state(sims), g["final_state"])
    _thermo_close(reps[0].thermo, g["thermo"], 1e-12)


@pytest.mark.parametrize("nranks", [2, 4, 8])
def test_lj8_production_loopback_within_tolerance(golden, nranks):
    """Production protocol: direct exchange/borders, export tables, ghost writes
    into peers' buffers by the step kernel, mailbox barrier each step."""
    g = golden(f"lj8_p{nranks}")
    reps, sims = run_loopback(LJ8, nranks, mode="fast", peer_timeout_s=30.0)
    assert all(s.exports is not None and s.exports.mailbox is not None for s in sims)
    assert sum(s.store.n_local for s in sims) == 2048
    _thermo_close(reps[0].thermo, g["thermo"], THERMO_TOL)
    np.testing.assert_allclose(_global_state(sims), g["final_state"], rtol=0, atol=1e-9)
    drift = np.abs(reps[0].ranks[0].momentum_final - reps[0].ranks[0].momentum_initial)
    assert np.all(drift <= 1e-9)


def test_sd8_p8_loopback(golden):
    """Spring-Dashpot at P = 8: exact protocol bitwise the reference; the
    production direct path (drift writes the ghost copies) within 1e-12 of it
    (damped DEM gives ghosts v = 0, so only the same P is comparable)."""
    g = golden("sd8_p8")
    reps, sims = run_loopback(SD8, 8, mode="exact", peer_timeout_s=30.0)
    assert np.array_equal(_global_state(sims), g["final_state"])
    _thermo_close(reps[0].thermo, g["thermo"], 1e-12)
    reps_f, sims_f = run_loopback(SD8, 8, mode="fast", peer_timeout_s=30.0)
    assert all(s.sd_direct for s in sims_f)
    _thermo_close(reps_f[0].thermo, g["thermo"], 1e-10)
    np.testing.assert_allclose(_global_state(sims_f), g["final_state"], rtol=0, atol=1e-12)


def test_capacity_growth_mid_run_remaps_peers():
    """A rank whose store grows inside the borders (locals + arriving ghosts >
    capacity) moves its position buffers; every peer must re-map them at that
    epoch.  A tight initial capacity forces growths after the
    first epoch; the run must equal the default-capacity run bit for bit."""
    cfg = SimConfig(unit_cells=(8, 8, 8), steps=60, velocity_scale=2.0, reneigh_interval=10)
    ref_reps, ref_sims = run_loopback(cfg, 2, mode="fast", peer_timeout_s=30.0)
    # capacity: just above the locals, so the first borders grow the store, and
    # every later epoch whose ghost count exceeds the grown capacity grows again
    reps, sims = run_loopback(cfg, 2, mode="fast", peer_timeout_s=30.0, capacity=1100)
    growths = sims[0].capacity_growths
    assert any(epoch > 1 for epoch, _ in growths), growths
    assert np.array_equal(reps[0].thermo, ref_reps[0].thermo)
    assert np.array_equal(_global_state(sims), _global_state(ref_sims))
