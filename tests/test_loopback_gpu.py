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

import os

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
    # global momentum (thermo columns px, py, pz are summed over ranks)
    drift = np.abs(reps[0].thermo[-1, 5:8] - reps[0].thermo[0, 5:8])
    assert np.all(drift <= 1e-9)


def test_sd8_p8_loopback(golden):
    """Spring-Dashpot at P = 8: exact protocol bitwise the reference; the
    production path (tmd_step_sd: fused contact forces + integration + ghost
    writes into peers' buffers) within tolerance of it (damped DEM gives
    ghosts v = 0, so only the same P is comparable)."""
    g = golden("sd8_p8")
    reps, sims = run_loopback(SD8, 8, mode="exact", peer_timeout_s=30.0)
    assert np.array_equal(_global_state(sims), g["final_state"])
    _thermo_close(reps[0].thermo, g["thermo"], 1e-12)
    reps_f, sims_f = run_loopback(SD8, 8, mode="fast", peer_timeout_s=30.0)
    assert all(s.fused and s.sd and s.exports is not None for s in sims_f)
    _thermo_close(reps_f[0].thermo, g["thermo"], THERMO_TOL)
    np.testing.assert_allclose(_global_state(sims_f), g["final_state"], rtol=0, atol=1e-9)


def test_capacity_growth_mid_run_remaps_peers(monkeypatch):
    """A rank whose store grows inside the borders (locals + arriving ghosts >
    capacity) moves its position buffers after its buffer flags were
    gathered; every peer must re-map them at that epoch.  Rank 1's
    capacity is made to look too small at two later epochs (its store then
    really reallocates); the run must equal an undisturbed run bit for bit."""
    from paper_2009_07400_b200.comm import Halo
    from paper_2009_07400_b200.store import ParticleStore

    cfg = SimConfig(unit_cells=(8, 8, 8), steps=60, reneigh_interval=10)
    ref_reps, ref_sims = run_loopback(cfg, 2, mode="fast", peer_timeout_s=30.0)
    real_cap = ParticleStore.capacity
    monkeypatch.setattr(ParticleStore, "capacity",
                        property(lambda self: real_cap.fget(self) - getattr(self, "_hide", 0)))
    real_borders = Halo.define_borders_direct
    calls, moved = {0: 0, 1: 0}, []

    def borders(self, store, extra=(), **kw):
        rank = self.decomp.rank
        calls[rank] += 1
        if rank == 1 and calls[rank] in (3, 5):
            store._hide = real_cap.fget(store) - store.n_local - 1  # capacity looks like n_local + 1
            before = store.pos.data_ptr()
            try:
                return real_borders(self, store, extra, **kw)
            finally:
                store._hide = 0
                moved.append(store.pos.data_ptr() != before)
        return real_borders(self, store, extra, **kw)

    monkeypatch.setattr(Halo, "define_borders_direct", borders)
    reps, sims = run_loopback(cfg, 2, mode="fast", peer_timeout_s=30.0)
    assert moved == [True, True]
    assert [e for e, _ in sims[0].capacity_growths if e > 0] == [2, 4]
    assert np.array_equal(reps[0].thermo, ref_reps[0].thermo)
    assert np.array_equal(_global_state(sims), _global_state(ref_sims))


@pytest.mark.parametrize("cfg", [LJ8, SD8], ids=["lj", "sd"])
def test_batched_loop_with_peer_barrier_bitwise(cfg, monkeypatch):
    """P > 1: the batched step loop (tmd_run_steps issuing the step launches
    and the mailbox barriers) is the same trajectory bit for bit as the
    per-step Python loop."""
    reps_a, sims_a = run_loopback(cfg, 4, mode="fast", peer_timeout_s=30.0)
    assert all(s._batched for s in sims_a)
    monkeypatch.setenv("TMD_BATCH", "0")
    reps_b, sims_b = run_loopback(cfg, 4, mode="fast", peer_timeout_s=30.0)
    assert not any(s._batched for s in sims_b)
    assert np.array_equal(reps_a[0].thermo, reps_b[0].thermo)
    assert np.array_equal(_global_state(sims_a), _global_state(sims_b))


@pytest.mark.skipif(os.environ.get("TMD_TEST_INPROCESS_MAILBOX") != "1",
                    reason="in-process ranks use the transport gather: P spinning gather kernels of one process "
                           "can starve each other (1 timeout in 3 suite runs, gpurun_out/r8q); the mailbox "
                           "gathers are covered across processes by test_multi_gpu_parity_torchrun (mailbox gathers are the multi-process default)")
def test_mailbox_count_gather_equals_transport_gather(monkeypatch):
    """The epoch's count all-gathers over the NVLink mailboxes
    (tmd_peer_allgather, every epoch after the first) give the same run, bit
    for bit, as the transport's all-gather (in-process ranks, forced; opt-in:
    TMD_TEST_INPROCESS_MAILBOX=1)."""
    cfg = SimConfig(unit_cells=(8, 8, 8), steps=60, reneigh_interval=10)
    monkeypatch.setenv("TMD_MAIL_GATHER", "force")  # in-process ranks use the transport by default
    reps_a, sims_a = run_loopback(cfg, 4, mode="fast", peer_timeout_s=30.0)
    assert all(getattr(s.exports, "gather_epoch", 0) >= 2 * 5 for s in sims_a)  # two per epoch after the first
    monkeypatch.setenv("TMD_MAIL_GATHER", "0")
    reps_b, sims_b = run_loopback(cfg, 4, mode="fast", peer_timeout_s=30.0)
    assert all(getattr(s.exports, "gather_epoch", 0) == 0 for s in sims_b)
    assert np.array_equal(reps_a[0].thermo, reps_b[0].thermo)
    assert np.array_equal(_global_state(sims_a), _global_state(sims_b))
