"""World-size 2 and 4 runs of the host-side halo protocol over gloo on CPU.

Each process plays one rank of the six-stencil decomposition with the real
``Halo`` (comm.py) and ``DistTransport`` over gloo, and the CPU test double
for the device primitives.  After exchange, border definition and three
synchronisations of a jittered lattice, every rank's store (locals then
ghosts, in order) must equal the oracle's lockstep run of the reference
protocol bit for bit (comm.py:340-498).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

CELLS = (6, 5, 6)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _state(seed=3):
    import oracle as O
    from paper_2009_07400_b200.core import SimConfig

    cfg = SimConfig(unit_cells=CELLS)
    pos, vel = O.initial_state(cfg)
    rng = np.random.default_rng(seed)
    lo, hi = O.domain_bounds(cfg)
    # jitter, some atoms pushed just outside the box so exchange has leavers
    pos = pos + rng.uniform(-0.12, 0.12, size=pos.shape)
    return cfg, pos, vel


def _moves(seed, n):
    return np.random.default_rng(seed).uniform(-0.05, 0.05, size=(n, 3))


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_07400_b200.comm import DistTransport

        reference_protocol_rank(rank, world, DistTransport(), out_dir)
    finally:
        dist.destroy_process_group()


def reference_protocol_rank(rank, world, transport, out_dir):
    """One rank of the reference (three-round) protocol over `transport`."""
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from halo_fakes import CpuHaloOps
    from paper_2009_07400_b200.comm import Decomposition, Halo
    from paper_2009_07400_b200.store import ParticleStore

    cfg, pos, vel = _state()
    decomp = Decomposition(cfg.domain(), world, rank, cfg.interaction_radius())
    # initial ownership from the un-jittered slab test, as the oracle World does
    inside = np.all((pos >= decomp.slab.lo) & (pos < decomp.slab.hi), axis=1)
    store = ParticleStore(64, device="cpu")
    store.append_locals(pos[inside], vel[inside])
    halo = Halo(decomp, transport, ops=CpuHaloOps())
    # move every local a little so the first exchange has leavers
    mv = _moves(rank + 11, store.n_local)
    store.pos[:, :store.n_local] += torch.from_numpy(mv.T.copy())
    halo.exchange(store)
    plan = halo.define_borders(store)
    snaps = [store.pos[:, :store.n_total].t().numpy().copy()]
    for k in range(3):
        shake = _moves(100 * k + rank, store.n_local) * 0.2
        store.pos[:, :store.n_local] += torch.from_numpy(shake.T.copy())
        halo.synchronize(store, plan)
        snaps.append(store.pos[:, :store.n_total].t().numpy().copy())
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), *snaps, n_local=store.n_local,
             n_ghost=store.n_ghost, vel=store.vel[:, :store.n_local].t().numpy())


def _oracle_replay(world):
    import oracle as O

    cfg, pos, vel = _state()
    W = O.World(cfg, world, pos, vel)
    for R in W.ranks:
        R.pos[:R.n_local] += _moves(R.rank + 11, R.n_local)
    W.exchange()
    W.define_borders()
    snaps = {R.rank: [R.pos.copy()] for R in W.ranks}
    for k in range(3):
        for R in W.ranks:
            R.pos[:R.n_local] += _moves(100 * k + R.rank, R.n_local) * 0.2
        W.synchronize()
        for R in W.ranks:
            snaps[R.rank].append(R.pos.copy())
    return W, snaps


@pytest.mark.parametrize("world", [2, 4])
def test_halo_protocol_gloo_matches_oracle(world, tmp_path):
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    check_reference_protocol(world, tmp_path)


def check_reference_protocol(world, tmp_path):
    W, snaps = _oracle_replay(world)
    total = 0
    for R in W.ranks:
        got = np.load(tmp_path / f"rank{R.rank}.npz")
        assert int(got["n_local"]) == R.n_local and int(got["n_ghost"]) == R.n_ghost
        for k in range(4):
            assert np.array_equal(got[f"arr_{k}"], snaps[R.rank][k]), (R.rank, k)
        assert np.array_equal(got["vel"], R.vel[:R.n_local])
        total += R.n_local
    cfg, pos, _ = _state()
    lo, hi = cfg.domain().lo, cfg.domain().hi
    assert total == int(np.all((pos >= lo) & (pos < hi), axis=1).sum())  # exchange conserves atoms


def _direct_worker(rank, world, port, out_dir):
    """The production (direct) protocol on one rank: exchange_direct +
    define_borders_direct, then the export records applied by hand."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2009_07400_b200.comm import DistTransport

        direct_protocol_rank(rank, world, DistTransport(), out_dir)
    finally:
        dist.destroy_process_group()


def direct_protocol_rank(rank, world, transport, out_dir):
    """One rank of the direct (production) protocol over `transport`."""
    import sys

    sys.path.insert(0, os.path.dirname(__file__))
    from halo_fakes import CpuHaloOps
    from paper_2009_07400_b200.comm import Decomposition, Halo
    from paper_2009_07400_b200.store import ParticleStore

    cfg, pos, vel = _state()
    decomp = Decomposition(cfg.domain(), world, rank, cfg.interaction_radius())
    inside = np.all((pos >= decomp.slab.lo) & (pos < decomp.slab.hi), axis=1)
    store = ParticleStore(64, device="cpu")
    store.append_locals(pos[inside], vel[inside])
    halo = Halo(decomp, transport, ops=CpuHaloOps())
    mv = _moves(rank + 11, store.n_local)
    store.pos[:, :store.n_local] += torch.from_numpy(mv.T.copy())
    halo.exchange_direct(store)
    plan, (root, dst, slot, sh) = halo.define_borders_direct(store)
    assert plan.direct and plan.n_ghost == store.n_ghost
    np.savez(os.path.join(out_dir, f"direct{rank}.npz"), pos=store.pos[:, :store.n_total].t().numpy(),
             vel=store.vel[:, :store.n_local].t().numpy(), n_local=store.n_local, n_ghost=store.n_ghost,
             root=root.numpy(), dst=dst.numpy(), slot=slot.numpy(), sh=sh.t().numpy())


def _rows(a):
    return a[np.lexsort(a.T[::-1])]


@pytest.mark.parametrize("world", [2, 4, 8])
def test_direct_protocol_gloo_same_atoms_ghosts_and_export_slots(world, tmp_path):
    """Direct exchange/borders (one all-to-all each) vs the reference rounds:
    every rank owns the same atoms with the same coordinates and holds the
    same ghost set (bitwise, as multisets), and every export record (root,
    destination rank, slot, shift) addresses exactly the ghost it mirrors:
    pos_owner[root] + shift == pos_dest[slot] bit for bit."""
    port = _free_port()
    mp.start_processes(_direct_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True,
                       start_method="spawn")
    check_direct_protocol(world, tmp_path)


def check_direct_protocol(world, tmp_path):
    W, snaps = _oracle_replay(world)
    got = [np.load(tmp_path / f"direct{r}.npz") for r in range(world)]
    n_ex = 0
    for R in W.ranks:
        g = got[R.rank]
        nl, ng = int(g["n_local"]), int(g["n_ghost"])
        assert nl == R.n_local and ng == R.n_ghost
        want = snaps[R.rank][0]
        assert np.array_equal(_rows(g["pos"][:nl]), _rows(want[:R.n_local]))
        assert np.array_equal(_rows(g["pos"][nl:]), _rows(want[R.n_local:R.n_local + R.n_ghost]))
        n_ex += g["root"].size
    for q in range(world):
        g = got[q]
        for e in range(g["root"].size):
            d = got[int(g["dst"][e])]
            assert int(g["slot"][e]) >= int(d["n_local"])
            assert np.array_equal(g["pos"][int(g["root"][e])] + g["sh"][e], d["pos"][int(g["slot"][e])])
    assert n_ex == sum(int(g["n_ghost"]) for g in got)  # every ghost has exactly one writer
