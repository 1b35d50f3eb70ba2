"""Velocity-Verlet step loop, thermo output and the run() entry point.

Reference: driver.py:27-177 (``initial_integrate``, ``final_integrate``,
``rank_program``, ``RankReport``, ``PhaseTimers``); the reference has no
``run()`` or thermo (SPEC.md:390-399, 627-689 describe them), so those follow
the spec and the north star: ``run(cfg) -> Report`` with one thermo row
(step, PE, KE, W, pressure, momentum) per output step.

Step order is the reference's: initial_integrate -> (epoch ? exchange +
borders + re-bin + rebuild : ghost sync) -> guard -> forces ->
final_integrate.  Two device paths:

* ``mode="fast"`` (LJ, full lists; the production path): one fused kernel
  per step computes the forces of step k, applies the closing half-kick,
  reduces thermo when due, and applies the next step's half-kick + drift and
  the displacement guard in its epilogue (tmd_step_lj).  With the P = 1
  flattened ghost refresh a non-epoch step is two launches.
* ``mode="exact"``: separate kernels in the reference's exact operation
  order; trajectories are bitwise equal to the reference.

Spring-Dashpot and half lists always take the separate-kernel path.
Nothing synchronises with the host between epochs: the guard maxima, thermo
rows and status words stay on the device and are checked at every epoch and
at the end of the run (a violation is reported with its step number).
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from contextlib import contextmanager
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .comm import BorderPlan, Decomposition, DistTransport, Halo, SingleRankTransport
from .core import SimConfig
from .errors import GuardViolation
from .exports import GhostExports
from .lattice import lattice_positions, lattice_velocities
from .neighbor import (BrickIndex, DeviceStatus, _stream, build_cell_grid, build_neighbor_lists, near_margin,
                       tinymd_f32_eps)
from .potential import _singular_detail, launch_forces, law_from_config
from .store import ParticleStore, device_of

__all__ = ["PhaseTimers", "RankReport", "Report", "Simulation", "initial_integrate", "final_integrate",
           "rank_program", "run", "THERMO_COLUMNS"]

_T_IMPORT = time.perf_counter()  # process-relative clock for epoch diagnostics
# near/far split of the production rows: margin = max(floor, factor * largest
# guard displacement of the previous epoch), capped at skin / 2
_MARGIN_FLOOR, _MARGIN_FACTOR = 0.05, 2.2

THERMO_COLUMNS = ("step", "pe", "ke", "virial", "pressure", "px", "py", "pz")


@dataclass
class PhaseTimers:
    """driver.py:30-46 (wall clock; with Simulation(profile=True) phases are device-synchronised)."""

    force: float = 0.0
    neigh: float = 0.0
    comm: float = 0.0
    other: float = 0.0

    @contextmanager
    def track(self, phase: str, sync: bool = False):
        if sync:
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        try:
            yield
        finally:
            if sync:
                torch.cuda.synchronize()
            setattr(self, phase, getattr(self, phase) + time.perf_counter() - t0)

    def total(self) -> float:
        return self.force + self.neigh + self.comm + self.other


@dataclass
class RankReport:
    """driver.py:63-71."""

    rank: int
    n_local: int
    momentum_initial: np.ndarray
    momentum_final: np.ndarray
    timers: PhaseTimers
    max_displacement_seen: float
    steps: int


@dataclass
class Report:
    thermo: np.ndarray  # rows: THERMO_COLUMNS
    ranks: list
    n_atoms: int
    steps: int
    wall_s: float  # steps 1..K (setup excluded), device-synchronised
    rebuilds: int = 0

    @property
    def atom_steps_per_s(self) -> float:
        return self.n_atoms * self.steps / self.wall_s if self.wall_s > 0 else float("nan")

    def thermo_table(self) -> str:
        head = " ".join(f"{c:>16s}" for c in THERMO_COLUMNS)
        rows = [" ".join(f"{v:16.9g}" for v in row) for row in self.thermo]
        return "\n".join([head, *rows])


# ---------------------------------------------------------------------------
# op-level integrators (driver.py:74-93)
# ---------------------------------------------------------------------------

def initial_integrate(store: ParticleStore, dt: float, mass: float) -> None:
    """Half-kick then drift on the locals: v += dt/2 F/m, x += dt v."""
    if store.n_local == 0 or dt == 0.0:
        return
    N.call("tmd_kick_drift", store.pos.data_ptr(), store.vel.data_ptr(), store.frc.data_ptr(), store.ld,
           store.ld, store.n_local, 0.5 * dt / mass, float(dt), 0, 0, 0, _stream())


def final_integrate(store: ParticleStore, dt: float, mass: float) -> None:
    """Closing half-kick: v += dt/2 F/m."""
    if store.n_local == 0 or dt == 0.0:
        return
    N.call("tmd_kick", store.vel.data_ptr(), store.frc.data_ptr(), store.ld, store.ld, store.n_local,
           0.5 * dt / mass, _stream())


def _kinetic(store: ParticleStore, mass: float, out: torch.Tensor) -> None:
    N.call("tmd_kinetic", store.vel.data_ptr(), store.ld, store.n_local, float(mass), out.data_ptr(),
           _stream())


def momentum(store: ParticleStore, mass: float) -> np.ndarray:
    out = torch.zeros(4, dtype=torch.float64, device=store.device)
    _kinetic(store, mass, out)
    return out.cpu().numpy()[1:4].copy()


# ---------------------------------------------------------------------------
# the per-rank simulation
# ---------------------------------------------------------------------------

def local_store_for(cfg: SimConfig, decomp: Decomposition, device=None) -> ParticleStore:
    """This rank's locals: the create_lattice arrays filtered by its slab, in lattice order."""
    box = cfg.domain()
    pos = lattice_positions(cfg, box)
    vel = lattice_velocities(cfg, pos.shape[0])
    if decomp.size > 1:
        mine = decomp.owns(pos)
        pos, vel = pos[mine], vel[mine]
    return ParticleStore.from_host(pos, vel, device=device)


class Simulation:
    """One rank's device-resident run (the reference's rank_program state, driver.py:49-60)."""

    def __init__(self, cfg: SimConfig, store: ParticleStore | None = None, decomp: Decomposition | None = None,
                 transport=None, mode: str = "fast", thermo_every: int = 1, device=None, profile=False,
                 fused_refresh: bool = True, peer_timeout_s: float = 120.0, capacity: int | None = None,
                 peer_barrier: bool = True, store_forces: str = "final", check_every_step: bool = False,
                 exact_yields=False, rank_grid=None):
        self.cfg = cfg.validate()
        # P > 1: a rank not reaching the per-step NVLink barrier within this many
        # seconds fails the run (ProtocolError) instead of hanging its peers
        self.peer_timeout_s = float(peer_timeout_s)
        # the fused step kernel stores F only when asked: "final" (the last step,
        # so store.frc holds the final forces as in the reference) or "every"
        if store_forces not in ("final", "every"):
            raise ValueError("store_forces must be 'final' or 'every'")
        self.store_forces = store_forces
        # check_every_step: read the status word and the guard maximum before every
        # step's force launch and raise at the failing step, as the reference does
        # (one small device->host read per step).  Off: the step kernels freeze
        # at the failing step on the device and the host raises at the next epoch
        # or at the end of the run, reporting the step.
        self.check_every_step = bool(check_every_step)
        # exact_yields: at the yield of ("step", k) the store holds the reference's
        # state of step k (x(k), v(k) after the closing kick).  The fused kernel
        # otherwise already drifted to x(k + 1); a yield step is then split into
        # forces + closing kick, the yield, and the next kick + drift + ghost
        # refresh (TMD_F_SKIP_FORCES).  True: every step; an int k: every k-th step.
        self.exact_yields = exact_yields
        if mode not in ("fast", "exact"):
            raise ValueError("mode must be 'fast' or 'exact'")
        self.mode = mode
        self.law = law_from_config(cfg)
        self.r = cfg.interaction_radius()
        self.half = bool(cfg.half_neighbor)
        self.transport = transport or SingleRankTransport()
        if decomp is None:
            decomp = Decomposition(cfg.domain(), self.transport.size, self.transport.rank, self.r, grid=rank_grid)
        self.decomp = decomp
        self.device = device_of(device)
        self.store = store if store is not None else local_store_for(cfg, decomp, self.device)
        if capacity is not None:
            # explicit store capacity (locals + ghosts); growth later is handled
            # (peers re-map the moved buffers at that epoch) but costs a handle exchange
            self.store.ensure_capacity(int(capacity))
        elif mode == "fast":
            # reserve locals + ghost shell (+10%) once: a reallocation later would
            # move the buffers peers write into (new IPC mappings mid-run)
            ext = decomp.slab.extent()
            r = self.r
            shell = float(np.prod(ext + 2.0 * r) / max(float(np.prod(ext)), 1e-300))
            self.store.ensure_capacity(int(1.1 * self.store.n_local * shell) + 1024)
        self.capacity_growths = []  # (epoch index, ranks) of epochs where a rank's store grew in the borders
        self.halo = Halo(decomp, self.transport)
        if self.transport.size > 1 and hasattr(self.transport, "warm_up") and self.device.type == "cuda":
            self.transport.warm_up(self.device)
        self.grid_box = decomp.slab  # static cell grid over the slab
        self.thermo_every = max(int(thermo_every), 1)
        self.profile = profile
        self.timers = PhaseTimers()
        self.status = DeviceStatus(self.device)
        # production path: one fused step kernel per step (tmd_step_lj / tmd_step_sd)
        self.fused = (mode == "fast" and not self.half)
        self.sd = cfg.potential_kind == "sd"
        # fused ghost refresh (exports.py): the step kernel writes the ghost copies
        # itself, locally and into peers' buffers over NVLink; fused_refresh=False
        # keeps the reference's three-round synchronize instead
        self.use_exports = self.fused and bool(fused_refresh) and self.transport.size <= 8
        # brick-major numbering of the locals (neighbor.BrickIndex): a warp's 32
        # atoms form a compact block, so its neighbour gathers share cache lines
        self.bricks = None
        self.build_order = self._order = None  # list builder's thread -> atom map (cell order)
        # per-step ordering at P > 1: NVLink mailbox barrier (tmd_peer_sync);
        # peer_barrier=False uses an NCCL all-reduce instead
        self._peer_barrier = bool(peer_barrier)
        self.exports = None
        if self.use_exports and self.transport.size == 1:
            # P = 1: the export table's object exists before the setup epoch, so
            # that epoch takes the single-sync path too (rebuild -> _rebuild_p1)
            self.exports = GhostExports(self.transport, self.device, self.status, decomp=self.decomp,
                                        peer_timeout_s=self.peer_timeout_s)
        self.epoch_step = 0
        # near/far split of the production rows for the next build: 2.2x the largest
        # displacement of the previous epoch (capped at skin / 2; None = skin / 2).
        # A step whose atoms moved farther just scans the far segment too.
        self.next_margin = None
        self.grid = self.lists = self.plan = None
        self.rebuilds = 0
        self.event_pairs = None  # list -> (start, end) CUDA events around every force launch
        self.launch_trace = None  # list -> (step, host ms inside the tmd_step_lj call)
        self.epoch_wall = []  # (step, host ms of the check + rebuild at that step)
        if self.device.type == "cuda":
            # host-pinned check buffers and the stream's reduction scratch now: a
            # page-locked or device allocation orders every stream of the context,
            # which in-process ranks (loopback.py) must not see mid-run while a
            # peer's barrier kernel waits for this rank
            N.call("tmd_prepare_stream", _stream())
            self._alloc_check_buffers(cfg.steps + 2)
            # the P = 1 epoch's read-back: [list status, epoch status, margin, ghost count]
            self._epoch_words = torch.empty(2 * N.STATUS_WORDS + 2, dtype=torch.int64, pin_memory=True)

    # -- epochs ---------------------------------------------------------------
    def rebuild(self) -> None:
        """driver.py:102-112: exchange, borders, re-bin, rebuild lists."""
        self._epoch_single_call = False
        if self.use_exports and self.transport.size == 1 and self.exports is not None and \
                os.environ.get("TMD_EPOCH_SYNC", "0") != "1":
            native = os.environ.get("TMD_EPOCH_NATIVE", "1") != "0" and self.device.type == "cuda"
            if (self._rebuild_p1_native() if native else self._rebuild_p1()):
                return
        self._rebuild()

    def _rebuild_p1(self) -> bool:
        """The production epoch at P = 1 with one host synchronisation.

        The ghost count stays on the device until the end: the borders write
        their copies into the store's reserved ghost region (``room`` slots),
        and binning, cell positions and the export table take the count from
        device memory.  Everything is enqueued while the GPU still runs the
        previous epoch's steps; the host then reads [list status, epoch status,
        ghost count] once.  A ghost count above the room (the reserve is 10%
        over the shell estimate) falls back to the synchronous epoch, after
        growing the store.  Returns False when it fell back."""
        mark = self._tracer()
        s = self.store
        self.status.reset()
        self.halo.exchange(s, status=self.status)  # P = 1: wraps in place, ownership check on the device
        mark("exchange")
        with self.timers.track("neigh", self.profile):
            self._sort_locals()
        mark("sort")
        n = s.n_local
        room = self._ghost_room()
        dc = self.decomp
        root, sh, off = self.halo.ops.borders_direct_dev(s, dc.slab, dc.spacing, dc.global_box.extent(), room)
        d_k = off.data_ptr() + 4 * n
        mark("borders")
        if self.sd:
            # ghost velocities are 0 (particles.py:148) in both velocity buffers
            for v in (s.vel, s.vel_alt):
                if v is not None and v.shape == s.pos.shape and room > 0:
                    N.call("tmd_zero_rows", v.data_ptr(), s.ld, 3, n, room, _stream())
        with self.timers.track("neigh", self.profile):
            self.grid = build_cell_grid(s, self.grid_box, self.r, status=self.status, shell=2, check=False,
                                        reuse=self.grid, count=(n, n + room, d_k))
            mark("bin")
            if getattr(self, "list_status", None) is None:
                self.list_status = DeviceStatus(self.device)
            if getattr(self, "_margin_dev", None) is None:
                self._margin_dev = torch.zeros(2, dtype=torch.float64, device=self.device)
            # the near/far split from this epoch's guard maxima, computed on the
            # device (the host reads them only at the end); _check_finish derives
            # the same value on the host
            d_near = None
            pend = getattr(self, "_check_pending", None)
            if pend is not None:
                i0, i1 = self.epoch_step + 1, min(pend[0] + 2, self.dispmax2.numel())
                if i1 > i0:
                    cut = self.cfg.cutoff
                    N.call("tmd_split_margin", self.dispmax2.data_ptr(), i0, i1, _MARGIN_FLOOR, _MARGIN_FACTOR,
                           near_margin(cut, self.r), cut, self._margin_dev.data_ptr(), _stream())
                    d_near = self._margin_dev
            lists = build_neighbor_lists(s, self.grid, self.r, False, status=self.list_status, order="split",
                                         cutoff=self.cfg.cutoff, reuse=self.lists, margin=self.next_margin,
                                         build_order=self.build_order, also=self.status,
                                         also_context=f"rank {dc.rank}: epoch (exchange ownership / ghost shell)",
                                         defer=True, d_near=d_near)
            mark("lists")
        with self.timers.track("comm", self.profile):
            self.exports.build_dev(s, root, sh, d_k, room)
        mark("exports")
        # the previous epoch's deferred check first (it waits for the previous
        # steps only), then the one read-back of this epoch
        self._check_finish()
        words = torch.cat([self.list_status.t, self.status.t, self._margin_dev.view(torch.int64)[1:2],
                           off[n:n + 1].to(torch.int64)]).cpu().numpy()
        k = int(words[-1])
        if k > room:
            # not enough reserved ghost slots: grow and redo the epoch synchronously
            # (the locals are already exchanged and sorted; exchange is idempotent)
            s.ensure_capacity(n + int(1.1 * k) + 1024)
            self.lists = lists
            return False
        s.n_ghost = k
        s.set_ghost_segments([0], [k])
        self.exports.n_entries = k
        self.grid.n_total = n + k
        self.plan = BorderPlan(n_local=n, n_ghost=k, flat_src=root[:k], flat_sh=sh[:, :k])
        self.plan.prov_rank = None
        self.plan.prov_root, self.plan.prov_sh = root[:k], sh[:, :k]
        if d_near is not None:
            lists.near_margin = float(words[-2:-1].view(np.float64)[0])
        self.lists = lists.finish(words[:-2])
        mark("lists_status")
        self.rebuilds += 1
        return True

    def _rebuild_p1_native(self) -> bool:
        """_rebuild_p1 with every kernel of the epoch issued by one library call
        (tmd_epoch_p1): the host prepares the persistent buffers, the library
        enqueues wrap, renumbering, borders, binning, split margin, list build,
        x_ref and the export table, and the host reads the device back once.
        The same kernels with the same arguments as _rebuild_p1 (bitwise the
        same state; tests/test_gpu_parity.py).  Returns False when it fell back
        to the synchronous epoch (more ghosts than reserved slots)."""
        mark = self._tracer()
        s, dc = self.store, self.decomp
        n = s.n_local
        room = self._ghost_room()
        if n <= 0 or room <= 0:
            return self._rebuild_p1()
        s.clear_ghosts()
        dev = self.device
        e = N.EpochP1()
        for name in ("pos", "vel"):
            cur, alt = getattr(s, name), getattr(s, name + "_alt")
            if alt is None or alt.shape != cur.shape:
                setattr(s, name + "_alt", torch.empty_like(cur))
        e.pos, e.pos_alt, e.vel, e.vel_alt = (s.pos.data_ptr(), s.pos_alt.data_ptr(), s.vel.data_ptr(),
                                              s.vel_alt.data_ptr())
        e.ld, e.n, e.room, e.sd = s.ld, n, room, int(self.sd)
        # exchange at P = 1 (Halo.exchange: every round is a self round)
        for entries in dc.rounds:
            d = entries[0].dim
            plus, minus = entries
            e.wrap_hi[d], e.wrap_lo[d] = float(plus.face), float(minus.face)
            e.wrap_s_plus[d], e.wrap_s_minus[d] = float(plus.shift[d]), float(minus.shift[d])
        for d in range(3):
            e.slab_lo[d], e.slab_hi[d] = float(dc.slab.lo[d]), float(dc.slab.hi[d])
        # renumbering (as _sort_locals)
        edge = self.r / 2
        sdims = np.maximum(1, np.ceil(self.grid_box.extent() / edge - 1e-12).astype(np.int64))
        if self.bricks is None or not np.array_equal(self.bricks.dims, sdims):
            self.bricks = BrickIndex(sdims, s.device)
        shape = BrickIndex.SHAPE
        n_cells = int(np.prod(sdims + 4)) + 1
        n_keys = (int(np.prod([(int(dd) + (1 << k) - 1) >> k for dd, k in zip(sdims, shape)])) << sum(shape)) + 1
        need = 6 * n + n_cells + n_keys
        buf = getattr(self, "_sort_buf", None)
        if buf is None or buf.numel() < need:
            buf = self._sort_buf = torch.empty(int(need * 1.05) + 4096, dtype=torch.int32, device=dev)
        if self._order is None or self._order.numel() < n:
            self._order = torch.empty(int(n * 1.05) + 1024, dtype=torch.int32, device=dev)
        parts, o = [], 0
        for size in (n, n_cells, n, n, n_keys, n):
            parts.append(buf[o:o + size].data_ptr())
            o += size
        for d in range(3):
            e.sort_lo[d] = float(self.grid_box.lo[d])
            e.sort_dims[d], e.sort_shape[d] = int(sdims[d]), int(shape[d])
        e.sort_edge, e.sort_shell = float(edge), 2
        (e.sort_cell_of, e.sort_cell_start, e.sort_cell_atoms, e.sort_key, e.sort_key_start,
         e.sort_perm) = parts
        e.order = self._order.data_ptr()
        # borders into the reserved ghost slots (the renumbered store: pos_alt becomes pos)
        r, ext = dc.spacing, dc.global_box.extent()
        root, sh, off = self.halo.ops.borders_direct_dev(s, dc.slab, r, ext, room, launch=False)
        for d in range(3):
            e.thr_hi[d], e.thr_lo[d] = float(dc.slab.hi[d]) - r, float(dc.slab.lo[d]) + r
            e.s_hi[d], e.s_lo[d] = -float(ext[d]), float(ext[d])
        e.off, e.root, e.sh, e.ld_sh = off.data_ptr(), root.data_ptr(), sh.data_ptr(), sh.stride(0)
        d_k = off.data_ptr() + 4 * n
        # the production grid
        self.grid = build_cell_grid(s, self.grid_box, self.r, shell=2, check=False, reuse=self.grid,
                                    count=(n, n + room, d_k), launch=False)
        g = self.grid
        for d in range(3):
            e.bin_lo[d], e.bin_dims[d] = float(g.origin[d]), int(g.dims[d])
        e.bin_edge, e.bin_shell = float(g.cell_size), int(g.shell)
        e.cell_of, e.cell_start, e.cell_atoms = g.cell_of.data_ptr(), g.cell_start.data_ptr(), g.cell_atoms.data_ptr()
        e.cell_pos, e.ld_cp = g.cell_pos.data_ptr(), g.cell_pos.stride(0)
        e.cell_pos_f = g.cell_pos_f.data_ptr() if g.cell_pos_f is not None else 0
        # split margin from the epoch's guard maxima (device)
        if getattr(self, "list_status", None) is None:
            self.list_status = DeviceStatus(dev)
        if getattr(self, "_margin_dev", None) is None:
            self._margin_dev = torch.zeros(2, dtype=torch.float64, device=dev)
        d_near = None
        pend = getattr(self, "_check_pending", None)
        if pend is not None:
            i0, i1 = self.epoch_step + 1, min(pend[0] + 2, self.dispmax2.numel())
            if i1 > i0:
                cut = self.cfg.cutoff
                e.dispmax2, e.margin_i0, e.margin_i1 = self.dispmax2.data_ptr(), i0, i1
                e.margin_floor, e.margin_factor = _MARGIN_FLOOR, _MARGIN_FACTOR
                e.margin_cap, e.cutoff = near_margin(cut, self.r), cut
                e.margin_out = self._margin_dev.data_ptr()
                d_near = self._margin_dev
        lists = build_neighbor_lists(s, g, self.r, False, status=self.list_status, order="split",
                                     cutoff=self.cfg.cutoff, reuse=self.lists, margin=self.next_margin,
                                     build_order=self._order[:n], also=self.status,
                                     also_context=f"rank {dc.rank}: epoch (exchange ownership / ghost shell)",
                                     defer=True, d_near=d_near, launch=False)
        e.nbr, e.ld_nbr = lists.nbr.data_ptr(), lists.ld_nbr
        e.nnear, e.counts, e.cap = lists.nnear.data_ptr(), lists.d_counts.data_ptr(), lists.cap
        e.near_rsq, e.rsq_max = lists.near_rsq, lists.rsq_max
        e.f32_eps = tinymd_f32_eps(g, lists.rsq_max) if g.cell_pos_f is not None else 0.0
        e.xref, e.ld_ref = lists.ref_positions_dev.data_ptr(), lists.ref_positions_dev.stride(0)
        # export table buffers
        zeros, slots = self.exports.build_dev(s, root, sh, d_k, room, launch=False)
        ex = self.exports
        e.ex_start, e.ex_rank, e.ex_slot, e.ex_sh = (ex.start.data_ptr(), ex.rank.data_ptr(), ex.slot.data_ptr(),
                                                     ex.sh.data_ptr())
        e.ex_zeros, e.ex_slots, e.ld_o = zeros.data_ptr(), slots.data_ptr(), ex.n_ex
        e.status, e.list_status = self.status.ptr, self.list_status.ptr
        mark("prepare")
        N.call("tmd_epoch_p1", C.byref(e), _stream())
        # the renumbered x, v are in the alternate buffers
        s.pos, s.pos_alt = s.pos_alt, s.pos
        s.vel, s.vel_alt = s.vel_alt, s.vel
        self.build_order = self._order[:n]
        self.exports._peer_buffers(s)
        mark("enqueue")
        if getattr(self, "_pre_read", None) is not None:
            self._pre_read()
        # the read-back is enqueued right behind the epoch (into pinned memory),
        # before the host waits for the previous epoch's check
        words_dev = torch.cat([self.list_status.t, self.status.t, self._margin_dev.view(torch.int64)[1:2],
                               off[n:n + 1].to(torch.int64)])
        if getattr(self, "_epoch_words", None) is None or self._epoch_words.numel() != words_dev.numel():
            self._epoch_words = torch.empty(words_dev.numel(), dtype=torch.int64, pin_memory=True)
        self._epoch_words.copy_(words_dev, non_blocking=True)
        done = torch.cuda.Event()
        done.record()
        self._check_finish()
        done.synchronize()
        words = self._epoch_words.numpy().copy()
        k = int(words[-1])
        if k > room:
            s.ensure_capacity(n + int(1.1 * k) + 1024)
            self.lists = lists
            return False
        s.n_ghost = k
        s.set_ghost_segments([0], [k])
        self.exports.n_entries = k
        g.n_total = n + k
        self.plan = BorderPlan(n_local=n, n_ghost=k, flat_src=root[:k], flat_sh=sh[:, :k])
        self.plan.prov_rank = None
        self.plan.prov_root, self.plan.prov_sh = root[:k], sh[:, :k]
        if d_near is not None:
            lists.near_margin = float(words[-2:-1].view(np.float64)[0])
        self.lists = lists.finish(words[:-2])
        mark("lists_status")
        self.rebuilds += 1
        self._epoch_single_call = True
        return True

    def _ghost_room(self) -> int:
        """Reserved ghost slots of the store (the device-count epoch writes at most this many)."""
        return self.store.capacity - self.store.n_local

    def _rebuild(self) -> None:
        # device-side checks of this epoch (ownership after exchange, binning shells)
        # accumulate in the status word and are read back once, before the lists
        mark = self._tracer()
        self.status.reset()
        # production path at P > 1: one all-to-all each for migration and borders,
        # ghosts refreshed by the owners' step kernels (exports.py)
        direct = self.use_exports and self.transport.size > 1
        records = None
        # the direct protocol's count all-gathers go through the NVLink mailboxes
        # once they are mapped (every epoch after the first)
        # (multi-process runs only: in-process ranks share one CUDA context, where an
        # allocation by one rank would wait for a peer's spinning gather kernel)
        mg = os.environ.get("TMD_MAIL_GATHER", "1")
        self.halo.small_gather = (self.exports.allgather if direct and self.exports is not None
                                  and self.exports.ready() and mg != "0"
                                  and (mg == "force" or not getattr(self.transport, "same_process", False))
                                  else None)
        with self.timers.track("comm", self.profile):
            if direct:
                self.halo.exchange_direct(self.store, status=self.status)
            else:
                self.halo.exchange(self.store, status=self.status)
        mark("exchange")
        if self.fused:
            with self.timers.track("neigh", self.profile):
                self._sort_locals()
            mark("sort")
        with self.timers.track("comm", self.profile):
            if direct:
                if self.exports is None:
                    self.exports = GhostExports(self.transport, self.device, self.status, decomp=self.decomp,
                                                peer_timeout_s=self.peer_timeout_s)
                self.plan, records = self.halo.define_borders_direct(
                    self.store, extra=self.exports.buffer_flags(self.store), lazy=True)
            else:
                self.plan = self.halo.define_borders(self.store, provenance=self.use_exports, direct=self.fused)
        mark("borders")
        # the previous epoch's deferred check (iter_steps): its read-back landed
        # with the borders' count read (raised before the lists are built)
        self._check_finish()
        if self.fused and self.sd:
            # ghost velocities are 0 (particles.py:148) in both velocity buffers
            self._zero_ghost_velocities(self.store.vel)
            if self.store.vel_alt is not None and self.store.vel_alt.shape == self.store.vel.shape:
                self._zero_ghost_velocities(self.store.vel_alt)
        with self.timers.track("neigh", self.profile):
            # production path: r/2 cells, 5^3 stencil; exact path: the reference grid
            self.grid = build_cell_grid(self.store, self.grid_box, self.r, status=self.status,
                                        shell=2 if self.fused else 1, check=False, reuse=self.grid)
            if not self.fused:
                N.raise_for_status(self.status.read(), context=f"rank {self.decomp.rank}: epoch "
                                   "(exchange ownership / ghost shell)")
            mark("bin")
            if self.fused:
                # the lists get their own status word: the epoch's (exchange ownership,
                # ghost shell) is read once, after the build, with no extra sync
                if getattr(self, "list_status", None) is None:
                    self.list_status = DeviceStatus(self.device)
                # deferred: the export tables below are enqueued while the build runs;
                # the build's status (and the epoch's) is read once, at the end
                self.lists = build_neighbor_lists(self.store, self.grid, self.r, False,
                                                  status=self.list_status,
                                                  order="split",
                                                  cutoff=self.cfg.cutoff, reuse=self.lists,
                                                  margin=self.next_margin, build_order=self.build_order,
                                                  also=self.status, also_context=f"rank {self.decomp.rank}: epoch "
                                                  "(exchange ownership / ghost shell)", defer=True)
            else:
                self.lists = build_neighbor_lists(self.store, self.grid, self.r, self.half, status=self.status)
            s = self.store
            # ghost positions at build time: ghost displacement bounds the pruning at P > 1
            self.xref_ghost = (s.pos[:, s.n_local:s.n_total].clone()
                               if self.transport.size > 1 and not self.use_exports else None)
        mark("lists")
        if self.use_exports:
            with self.timers.track("comm", self.profile):
                if self.exports is None:
                    self.exports = GhostExports(self.transport, self.device, self.status, decomp=self.decomp,
                                                peer_timeout_s=self.peer_timeout_s)
                if records is not None:
                    flags = self.halo.gathered_extra
                    # a capacity growth inside define_borders_direct moved that rank's
                    # buffers after its flags were gathered: force the handle exchange
                    flags[:, 0] |= self.halo.gathered_grew.astype(flags.dtype)
                    if self.halo.gathered_grew.any():
                        self.capacity_growths.append(
                            (self.rebuilds, [int(q) for q in np.nonzero(self.halo.gathered_grew)[0]]))
                    self.exports.build_direct(self.store, records() if callable(records) else records,
                                              flags=flags)
                else:
                    self.exports.build(self.store, self.plan)
            mark("exports")
        if self.fused:
            self.lists.finish()
            mark("lists_status")
        self.rebuilds += 1

    def _tracer(self):
        """TMD_TRACE_REBUILD=1: device-synchronised per-phase times of each rebuild
        appended to self.rebuild_trace (diagnostics; adds host syncs); =2: host
        clock per phase without extra synchronisation."""
        mode = os.environ.get("TMD_TRACE_REBUILD", "0")
        if mode not in ("1", "2", "3"):
            return lambda name: None
        sync = mode == "1"  # "2": host clock only, no extra synchronisation; "3": + CUDA events
        if mode == "3":
            if not hasattr(self, "rebuild_events"):
                self.rebuild_events = []
            evs = [("start", torch.cuda.Event(enable_timing=True))]
            evs[0][1].record()
            self.rebuild_events.append(evs)
        if sync:
            torch.cuda.synchronize(self.device)
        rec = {}
        t = [time.perf_counter()]
        if not hasattr(self, "rebuild_trace"):
            self.rebuild_trace = []
        self.rebuild_trace.append(rec)

        def mark(name):
            if sync:
                torch.cuda.synchronize(self.device)
            if mode == "3":
                ev = torch.cuda.Event(enable_timing=True)
                ev.record()
                evs.append((name, ev))
                if name == "exports":
                    rec["mem_alloc_mb"] = torch.cuda.memory_allocated(self.device) / 2**20
                    rec["mem_reserved_mb"] = torch.cuda.memory_reserved(self.device) / 2**20
            now = time.perf_counter()
            rec[name] = (now - t[0]) * 1e3
            t[0] = now

        return mark

    def _sort_locals(self) -> None:
        """Renumber the locals brick-major (production path).

        Atoms of one brick of r/2 cells become contiguous, so a warp's 32 atoms
        are spatial neighbours and the x_j gathers of a warp fall on a few
        cache lines.  The list builder walks the atoms in cell order through a
        thread -> atom map (``build_order``), keeping its warps on coherent
        stencil runs.  Ghosts are empty here (right after exchange); the
        borders and the lists are then built on the sorted store.
        """
        s = self.store
        n = s.n_local
        if n == 0:
            return
        edge = self.r / 2
        dims = np.maximum(1, np.ceil(self.grid_box.extent() / edge - 1e-12).astype(np.int64))
        if (self.bricks is None or not np.array_equal(self.bricks.dims, dims)
                or getattr(self, "_sort_h", None) is None):
            self.bricks = BrickIndex(dims, s.device)
            self._sort_h = (N.host_f64(self.grid_box.lo), N.host_i32(dims), N.host_i32(BrickIndex.SHAPE))
        h_lo, h_dims, h_shape = self._sort_h
        shape = BrickIndex.SHAPE
        n_cells = int(np.prod(dims + 4)) + 1
        n_keys = (int(np.prod([(int(d) + (1 << e) - 1) >> e for d, e in zip(dims, shape)])) << sum(shape)) + 1
        # persistent scratch (5% headroom): n_local drifts with migration and a
        # fresh allocation of these sizes can stall an epoch
        need = 6 * n + n_cells + n_keys
        buf = getattr(self, "_sort_buf", None)
        if buf is None or buf.numel() < need:
            buf = self._sort_buf = torch.empty(int(need * 1.05) + 4096, dtype=torch.int32, device=s.device)
        if self._order is None or self._order.numel() < n:
            self._order = torch.empty(int(n * 1.05) + 1024, dtype=torch.int32, device=s.device)
        parts, o = [], 0
        for size in (n, n_cells, n, n, n_keys, n):  # cell_of, cell_start, cell_atoms, key, key_start, perm
            parts.append(buf[o:o + size])
            o += size
        outs = []
        for name in ("pos", "vel"):
            cur, alt = getattr(s, name), getattr(s, name + "_alt")
            if alt is None or alt.shape != cur.shape:
                alt = torch.empty_like(cur)
            outs.append(alt)
        N.call("tmd_sort_locals", s.pos.data_ptr(), s.vel.data_ptr(), s.ld, n, N.hp(h_lo), float(edge), N.hp(h_dims),
               2, N.hp(h_shape), *(t.data_ptr() for t in parts), self._order.data_ptr(), outs[0].data_ptr(),
               outs[1].data_ptr(), self.status.ptr, _stream())
        self.build_order = self._order[:n]
        for name, alt in zip(("pos", "vel"), outs):
            cur = getattr(s, name)
            setattr(s, name, alt)
            setattr(s, name + "_alt", cur)

    def _energy_due(self, step: int, last: int) -> bool:
        return step % self.thermo_every == 0 or step == last

    # -- one force evaluation (+ fused integration) ---------------------------
    def _fused(self, step, phases, energy, refresh=False, extra_flags=0):
        """One tmd_step_lj / tmd_step_sd launch; `refresh`: the NEXT phase also writes the ghost copies."""
        s, L = self.store, self.lists
        # element pointers by offset (a torch slice per argument costs microseconds per step)
        d0 = self.dispmax2.data_ptr()
        disp = d0 + 8 * (step + 1) if phases & 2 else d0
        nxt = None
        if phases & 2:
            if s.pos_alt is None or s.pos_alt.shape != s.pos.shape:
                s.pos_alt = torch.empty_like(s.pos)
            nxt = s.pos_alt
        ev = self._event_begin()
        t_launch = time.perf_counter() if self.launch_trace is not None else 0.0
        rows = (L.nbr.data_ptr(), L.ld_nbr, L.d_counts.data_ptr(), L.nnear.data_ptr(), L.cap, float(L.near_margin),
                d0 + 8 * step, *self._export_args(nxt, refresh, step),
                *self._law_args(), 0.5 * self.cfg.dt / self.cfg.mass,
                float(self.cfg.dt), phases, self._step_flags(step, energy) | extra_flags, s.frc.data_ptr(), s.ld,
                L.ref_positions_dev.data_ptr(), L.ref_positions_dev.stride(0), disp,
                self.thermo.data_ptr() + 8 * self.thermo.shape[1] * step, self.status.ptr, self._guard_lim2(step),
                _stream())
        out = nxt.data_ptr() if nxt is not None else 0
        if self.sd:
            # the dashpot reads v_j: kicked velocities go to the other buffer
            if s.vel_alt is None or s.vel_alt.shape != s.vel.shape:
                s.vel_alt = torch.zeros_like(s.vel)
                self._zero_ghost_velocities(s.vel_alt)
            N.call("tmd_step_sd", s.pos.data_ptr(), out, s.vel.data_ptr(), s.vel_alt.data_ptr(), s.ld, s.n_local,
                   *rows)
            s.vel, s.vel_alt = s.vel_alt, s.vel
        else:
            N.call("tmd_step_lj", s.pos.data_ptr(), out, s.vel.data_ptr(), s.ld, s.n_local, *rows)
        if self.launch_trace is not None:
            self.launch_trace.append((step, (time.perf_counter() - t_launch) * 1e3))
        self._event_end(ev)
        if nxt is not None:
            s.swap_positions()

    def _law_args(self):
        law = self.law
        if self.sd:
            return float(law.stiffness), float(law.damping), float(law.diameter)
        return float(law.cutoff_rsq), float(law.epsilon), float(law.sigma6)

    def _zero_ghost_velocities(self, vel: torch.Tensor) -> None:
        """Ghost velocities are 0 (particles.py:148) in both velocity buffers."""
        s = self.store
        if s.n_ghost:
            N.call("tmd_zero_rows", vel.data_ptr(), s.ld, 3, s.n_local, s.n_ghost, _stream())

    def _guard_lim2(self, step: int) -> float:
        """The step kernel's fail-fast guard: (buffer / 2)^2, or 0 on a rebuild step
        (the reference skips the guard right after reneighboring)."""
        if self.rebuild_steps[step]:
            return 0.0
        return (0.5 * self.cfg.verlet_buffer) ** 2

    def _split_due(self, step: int, K: int) -> bool:
        ey = self.exact_yields
        if not self.fused or ey is False or ey is None or step >= K:
            return False
        return True if ey is True else step % int(ey) == 0

    def _step_flags(self, step: int, energy: bool) -> int:
        flags = N.F_ENERGY if energy else 0
        if self.store_forces == "every" or step == getattr(self, "steps", -1):
            flags |= N.F_STORE_FORCES
        return flags

    def production_forces(self, prune: bool = True) -> np.ndarray:
        """Forces on the locals from the production step kernel itself (tmd_step_lj /
        tmd_step_sd with no integration phase), at the current positions on the current
        lists; ``prune=False`` scans both segments of every split row.  For
        parity tests (P = 1: the pruning bound uses the locals' displacement)."""
        if not self.fused or self.lists is None:
            raise ValueError("production_forces needs the fused path after setup")
        s, L = self.store, self.lists
        d2 = torch.zeros(1, dtype=torch.float64, device=self.device)
        ref = L.ref_positions_dev
        N.call("tmd_max_disp2", s.pos.data_ptr(), s.ld, ref.data_ptr(), ref.stride(0), s.n_local, d2.data_ptr(),
               _stream())
        thermo = torch.zeros(6, dtype=torch.float64, device=self.device)
        flags = N.F_STORE_FORCES | (0 if prune else N.F_NO_PRUNE)
        rows = (L.nbr.data_ptr(), L.ld_nbr, L.d_counts.data_ptr(), L.nnear.data_ptr(), L.cap, float(L.near_margin),
                d2.data_ptr(), 0, 0, 0, 0, 0, 0, 0, 0, 0, *self._law_args(), 0.0, 0.0, 0, flags, s.frc.data_ptr(),
                s.ld, ref.data_ptr(), ref.stride(0), d2.data_ptr(), thermo.data_ptr(), self.status.ptr, 0.0, _stream())
        if self.sd:  # no integration phase: velocities are rewritten unchanged
            N.call("tmd_step_sd", s.pos.data_ptr(), 0, s.vel.data_ptr(), s.vel.data_ptr(), s.ld, s.n_local, *rows)
        else:
            N.call("tmd_step_lj", s.pos.data_ptr(), 0, s.vel.data_ptr(), s.ld, s.n_local, *rows)
        N.raise_for_status(self.status.read(), context="production_forces")
        return s.local_forces()

    def _export_args(self, nxt, refresh, step):
        """tmd_step_lj's fused ghost-refresh arguments (none: refresh by synchronize)."""
        if self.exports is None or nxt is None or not refresh:
            return (0, 0, 0, 0, 0, 0, 0, 0, 0)
        # every fused step since the epoch began swapped the buffers once
        return self.exports.args((step - self.epoch_step) & 1)

    def _event_begin(self):
        if self.event_pairs is None:
            return None
        a = torch.cuda.Event(enable_timing=True)
        a.record()
        return a

    def _event_end(self, a):
        if a is not None:
            b = torch.cuda.Event(enable_timing=True)
            b.record()
            self.event_pairs.append((a, b))

    def _separate_force(self, step, energy):
        ev = self._event_begin()
        launch_forces(self.store, self.lists, self.law, self.half, energy, self.mode == "exact",
                      self.thermo[step], self.status)
        self._event_end(ev)

    # -- driving ----------------------------------------------------------------
    def iter_steps(self, steps: int | None = None):
        """Generator: yields ("step", k) after step k (k = 0 after setup), like rank_program."""
        cfg = self.cfg
        K = cfg.steps if steps is None else int(steps)
        self.steps = K
        dev = self.device
        self.thermo = torch.zeros((K + 1, 6), dtype=torch.float64, device=dev)
        self.dispmax2 = torch.zeros(K + 2, dtype=torch.float64, device=dev)
        self.rebuild_steps = np.zeros(K + 2, dtype=bool)
        s = self.store
        self.p0 = momentum(s, cfg.mass)
        self.status.reset()
        c = 0.5 * cfg.dt / cfg.mass
        # setup: epoch + first force call (driver.py:146-148)
        self.rebuild()
        self.rebuild_steps[0] = True
        self.epoch_step = 0
        split = self._split_due(0, K)
        if self.fused:
            with self.timers.track("force", self.profile):
                if split:
                    self._fused(0, 0, True, extra_flags=N.F_STORE_FORCES)
                else:
                    self._fused(0, 2 if K > 0 else 0, True, refresh=self._refresh_due(0, K))
                    self._step_barrier(0, K)
        else:
            with self.timers.track("force", self.profile):
                self._separate_force(0, True)
            _kinetic(s, cfg.mass, self.thermo[0, 2:6])
        self._check(0)
        yield ("step", 0)
        if split:
            self._finish_split(0, K)
        torch.cuda.current_stream(dev).synchronize()  # this rank's stream only (loopback ranks share a device)
        self.t_start = time.perf_counter()
        for step in range(1, K + 1):
            energy = self._energy_due(step, K)
            if not self.fused:
                with self.timers.track("other", self.profile):
                    ref = self.lists.ref_positions_dev
                    N.call("tmd_kick_drift", s.pos.data_ptr(), s.vel.data_ptr(), s.frc.data_ptr(), s.ld,
                           s.ld, s.n_local, c, float(cfg.dt), ref.data_ptr(), ref.stride(0),
                           self.dispmax2[step:step + 1].data_ptr(), _stream())
            if step % cfg.reneigh_interval == 0:
                t_epoch = time.perf_counter()
                if self.check_every_step or not self.fused:
                    self._check(step - 1)
                else:
                    # read back with the epoch's first host sync (rebuild raises there)
                    self._check_begin(step - 1)
                self.rebuild()
                self.epoch_wall.append((step, (time.perf_counter() - t_epoch) * 1e3, t_epoch - _T_IMPORT))
                self.rebuild_steps[step] = True
                self.epoch_step = step
                # fresh lists: nothing has moved since the build
                N.call("tmd_zero_rows", self.dispmax2.data_ptr(), self.dispmax2.numel(), 1, step, 1, _stream())
            elif self.exports is not None:
                pass  # ghosts were written by the previous step's kernel
            else:
                with self.timers.track("comm", self.profile):
                    self.halo.synchronize(s, self.plan)
                    if self.fused and self.xref_ghost is not None and s.n_ghost:
                        # remote ghosts: their displacement also bounds the list pruning
                        N.call("tmd_max_disp2", s.pos[:, s.n_local:].data_ptr(), s.ld,
                               self.xref_ghost.data_ptr(), self.xref_ghost.stride(0), s.n_ghost,
                               self.dispmax2[step:step + 1].data_ptr(), _stream())
            if self.check_every_step and step % cfg.reneigh_interval != 0:
                self._check(step - 1)  # status + guard of the positions this step's forces would use
            split = self._split_due(step, K)
            with self.timers.track("force", self.profile):
                if self.fused and split:
                    self._fused(step, 1, energy, extra_flags=N.F_STORE_FORCES)
                elif self.fused:
                    self._fused(step, 1 | (2 if step < K else 0), energy, refresh=self._refresh_due(step, K))
                    self._step_barrier(step, K)
                else:
                    self._separate_force(step, energy)
            if not self.fused:
                with self.timers.track("other", self.profile):
                    N.call("tmd_kick", s.vel.data_ptr(), s.frc.data_ptr(), s.ld, s.ld, s.n_local, c, _stream())
                    if energy:
                        _kinetic(s, cfg.mass, self.thermo[step, 2:6])
            yield ("step", step)
            if split:
                self._finish_split(step, K)
        torch.cuda.current_stream(dev).synchronize()  # this rank's stream only (loopback ranks share a device)
        self.wall = time.perf_counter() - self.t_start
        self._check(K)

    def _finish_split(self, step: int, K: int) -> None:
        """Second half of a split step: next kick + drift + ghost refresh with the
        stored forces (no force pass)."""
        with self.timers.track("force", self.profile):
            self._fused(step, 2, False, refresh=self._refresh_due(step, K), extra_flags=N.F_SKIP_FORCES)
            self._step_barrier(step, K)

    def _refresh_due(self, step: int, K: int) -> bool:
        """Fused refresh after step `step`: the next step exists and is not a rebuild."""
        return self.exports is not None and step < K and (step + 1) % self.cfg.reneigh_interval != 0

    def _step_barrier(self, step: int, K: int) -> None:
        """P > 1 with the fused refresh: all-reduce (max) of the step's guard
        displacement.  It also orders the ranks' kernels (exports.py)."""
        if self.exports is not None and self.transport.size > 1 and step < K:
            with self.timers.track("comm", self.profile):
                if self._peer_barrier:
                    self.exports.barrier(self.dispmax2[step + 1:step + 2])
                else:
                    self.transport.allreduce_(self.dispmax2[step + 1:step + 2], "max")

    def _check(self, upto: int) -> None:
        """Collective check of the device status word and the guard maxima up to step `upto`."""
        self._check_begin(upto)
        self._check_finish()

    def _check_begin(self, upto: int) -> None:
        """Enqueue the check's read-back (asynchronous): [status code, guard maxima
        of steps 0 .. upto + 1] (max over ranks at P > 1) and the status words,
        into pinned host buffers.  ``_check_finish`` waits and raises."""
        n2 = min(upto + 2, self.dispmax2.numel())
        cap = self.dispmax2.numel() + 1
        if getattr(self, "_check_buf", None) is None or self._check_buf.numel() < cap:
            self._alloc_check_buffers(cap)
        t = self._check_buf[:n2 + 1]
        N.call("tmd_check_pack", self.status.ptr, self.dispmax2.data_ptr(), n2, t.data_ptr(), _stream())
        if self.transport.size > 1:
            self.transport.allreduce_(t, "max")
        self._check_host[:n2 + 1].copy_(t, non_blocking=True)
        self._check_words.copy_(self.status.t, non_blocking=True)
        ev = torch.cuda.Event() if self.device.type == "cuda" else None
        if ev is not None:
            ev.record()
        self._check_pending = (upto, n2, ev)

    def _alloc_check_buffers(self, cap: int) -> None:
        cap = max(int(cap), 64)
        pin = self.device.type == "cuda"
        self._check_buf = torch.empty(cap, dtype=torch.float64, device=self.device)
        self._check_host = torch.empty(cap, dtype=torch.float64, pin_memory=pin)
        self._check_words = torch.empty(N.STATUS_WORDS, dtype=torch.int64, pin_memory=pin)

    def _check_finish(self) -> None:
        pending = getattr(self, "_check_pending", None)
        if pending is None:
            return
        self._check_pending = None
        upto, n2, ev = pending
        if ev is not None:
            ev.synchronize()
        h = self._check_host[:n2 + 1].numpy().copy()
        words = self._check_words.numpy().copy()
        code = max(int(words[0]), int(h[0]))
        d2 = h[1:upto + 2]
        # the epoch's moves: guard maxima of steps epoch_step + 1 .. upto + 1 (the
        # positions the coming rebuild sees); per-step global maxima at P > 1
        moved = h[1 + self.epoch_step + 1: 1 + upto + 2]
        if moved.size and self.transport.size > 1 and not self._peer_barrier:
            moved = None
        if moved is not None and moved.size:
            self.next_margin = max(_MARGIN_FLOOR, _MARGIN_FACTOR * float(np.sqrt(moved.max())))
        # the guard first: a violating step freezes the step kernels (TMD_GUARD), and
        # its step number comes from the per-step maxima
        limit = 0.5 * self.cfg.verlet_buffer
        checked = ~self.rebuild_steps[: upto + 1]
        disp = np.sqrt(d2)
        bad = np.nonzero(checked & (disp >= limit))[0]
        if bad.size:
            k = int(bad[0])
            raise GuardViolation(
                f"step {k}: particles moved {disp[k]:.4g} since the last rebuild, which exceeds half "
                f"the Verlet buffer ({self.cfg.verlet_buffer}); increase the buffer or lower "
                f"reneigh_interval ({self.cfg.reneigh_interval})")
        if code != N.OK:
            if int(words[0]) != N.OK:
                N.raise_for_status(words, context=f"rank {self.decomp.rank} (at or before step {upto + 1})",
                                   describe=_singular_detail(self.lists) if self.lists else None)
            raise N.ProtocolError(f"rank {self.decomp.rank}: a peer rank failed (code {code})")

    def finish(self) -> Report:
        cfg, K = self.cfg, self.steps
        th = self.thermo.clone()
        if self.transport.size > 1:
            self.transport.allreduce_(th, "sum")
        th = th.cpu().numpy()
        if self.fused:
            # the fused step kernel reduces 0.5 sum v^2 and sum v (unit mass); the
            # separate path's tmd_kinetic already includes the mass (driver.py:96-99)
            th[:, 2:6] *= cfg.mass
        vol = cfg.domain().volume()
        rows = []
        for k in range(K + 1):
            if not (k == 0 or self._energy_due(k, K)):
                continue
            pe, w, ke, px, py, pz = th[k]
            rows.append([k, pe, ke, w, (2.0 * ke + w) / (3.0 * vol), px, py, pz])
        d2 = self.dispmax2[: K + 1].cpu().numpy()
        seen = float(np.sqrt(d2[~self.rebuild_steps[: K + 1]].max())) if (~self.rebuild_steps[: K + 1]).any() else 0.0
        rep = RankReport(self.decomp.rank, self.store.n_local, self.p0, momentum(self.store, cfg.mass),
                         self.timers, seen, K)
        reports = [rep]
        n_atoms = self.store.n_local
        if self.transport.size > 1:
            t = torch.tensor([float(n_atoms), self.wall], dtype=torch.float64, device=self.device)
            self.transport.allreduce_(t[0:1], "sum")
            self.transport.allreduce_(t[1:2], "max")
            n_atoms, wall = int(t[0].item()), float(t[1].item())
        else:
            wall = self.wall
        return Report(np.array(rows), reports, n_atoms, K, wall, self.rebuilds)

    def run(self, steps: int | None = None) -> Report:
        self.start(steps)
        self.advance(self.steps)
        return self.finish()

    # -- batched driving (the production loop) ----------------------------------
    def batchable(self) -> bool:
        """Whether advance() batches: the fused path with the kernel-side ghost
        refresh and no per-step host work (no per-step checks, split yields,
        launch tracing or phase timers; at P > 1 the NVLink barrier)."""
        ey = self.exact_yields
        return (self.fused and not self.check_every_step and (ey is False or ey is None) and not self.profile
                and self.launch_trace is None and self.exports is not None
                and (self.transport.size == 1 or self._peer_barrier)
                and os.environ.get("TMD_BATCH", "1") != "0")

    def start(self, steps: int | None = None) -> None:
        """Setup epoch and step 0 (iter_steps up to its first yield); then
        advance(n) runs the following steps with one library call per epoch."""
        self._gen = self.iter_steps(steps)
        next(self._gen)
        self._next_step = 1
        self._finished = False
        # decided once the setup epoch exists (the export table, the transport)
        self._batched = self.batchable()
        if self._batched:
            torch.cuda.current_stream(self.device).synchronize()
            self.t_start = time.perf_counter()

    def advance(self, n: int) -> None:
        """Run the next n steps (at most through step K): per epoch the rebuild
        as in iter_steps, then the epoch's steps in one tmd_run_steps call."""
        K = self.steps
        k, end = self._next_step, min(K + 1, self._next_step + max(int(n), 0))
        if getattr(self, "_finished", False):
            return
        if not self._batched:
            for _ in range(end - k):
                next(self._gen)
            self._next_step = end
            if end == K + 1:
                for _ in self._gen:  # the generator's epilogue (wall clock, final check)
                    pass
                self._finished = True
            return
        R = self.cfg.reneigh_interval
        while k < end:
            rebuilt = k % R == 0
            stop = min(end, (k // R + 1) * R)
            prepared = None
            if rebuilt:
                t_epoch = time.perf_counter()
                self._check_begin(k - 1)
                # the single-sync epochs call this right before their read-back: the
                # guard slot is zeroed and the batch's arguments are filled while the
                # GPU still works on the epoch
                hook = {"k": k, "run": None}

                def pre_read(hook=hook, k=k, stop=stop):
                    N.call("tmd_zero_rows", self.dispmax2.data_ptr(), self.dispmax2.numel(), 1, k, 1, _stream())
                    hook["run"] = self._batch_args(k, stop, True, epoch_step=k)

                self._pre_read = pre_read
                try:
                    self.rebuild()
                finally:
                    self._pre_read = None
                self.epoch_wall.append((k, (time.perf_counter() - t_epoch) * 1e3, t_epoch - _T_IMPORT))
                self.rebuild_steps[k] = True
                self.epoch_step = k
                # (an epoch that fell back to the synchronous path rebuilt everything)
                prepared = hook["run"] if self._epoch_single_call else None
                if hook["run"] is None:
                    N.call("tmd_zero_rows", self.dispmax2.data_ptr(), self.dispmax2.numel(), 1, k, 1, _stream())
            self._launch_batch(k, stop, rebuilt, prepared)
            k = stop
        self._next_step = end
        if end == K + 1:
            # the generator's epilogue: wall clock, final check
            torch.cuda.current_stream(self.device).synchronize()
            self.wall = time.perf_counter() - self.t_start
            self._check(K)
            self._gen = None
            self._finished = True

    def _launch_batch(self, k0: int, k1: int, rebuilt: bool, prepared=None) -> None:
        s, L, ex, K = self.store, self.lists, self.exports, self.steps
        if prepared is not None and prepared.pos_a == s.pos.data_ptr() and prepared.vel_a == s.vel.data_ptr():
            r = prepared
            # filled before the epoch's read-back: the list fields come from the
            # lists finished since (rows possibly rebuilt wider, the split margin
            # read back)
            r.nbr, r.ld_nbr, r.nnbr, r.nnear = L.nbr.data_ptr(), L.ld_nbr, L.d_counts.data_ptr(), L.nnear.data_ptr()
            r.cap, r.near_margin = L.cap, float(L.near_margin)
            r.xref, r.ld_ref = L.ref_positions_dev.data_ptr(), L.ref_positions_dev.stride(0)
        else:
            r = self._batch_args(k0, k1, rebuilt, epoch_step=self.epoch_step)
        N.call("tmd_run_steps", C.byref(r), k0, k1, _stream())
        # host bookkeeping of the buffer roles and barrier epochs
        n_next = min(k1, K) - k0  # launches with the NEXT phase (all but step K)
        if n_next & 1:
            s.swap_positions()
        if self.sd and (k1 - k0) & 1:
            s.vel, s.vel_alt = s.vel_alt, s.vel
        if ex is not None and self.transport.size > 1:
            ex.epoch += n_next

    def _batch_args(self, k0: int, k1: int, rebuilt: bool, epoch_step: int):
        """TmdStepRun of the steps k0 .. k1-1 (tmd_run_steps)."""
        s, L, ex, cfg = self.store, self.lists, self.exports, self.cfg
        K = self.steps
        if s.pos_alt is None or s.pos_alt.shape != s.pos.shape:
            s.pos_alt = torch.empty_like(s.pos)
        if self.sd and (s.vel_alt is None or s.vel_alt.shape != s.vel.shape):
            s.vel_alt = torch.zeros_like(s.vel)
            self._zero_ghost_velocities(s.vel_alt)
        r = N.StepRun()
        r.law = 1 if self.sd else 0
        r.pos_a, r.pos_b = s.pos.data_ptr(), s.pos_alt.data_ptr()
        r.vel_a = s.vel.data_ptr()
        r.vel_b = s.vel_alt.data_ptr() if self.sd else 0
        r.ld, r.n_local = s.ld, s.n_local
        r.nbr, r.ld_nbr, r.nnbr, r.nnear = L.nbr.data_ptr(), L.ld_nbr, L.d_counts.data_ptr(), L.nnear.data_ptr()
        r.cap, r.near_margin = L.cap, float(L.near_margin)
        r.dispmax2 = self.dispmax2.data_ptr()
        if ex is not None:
            r.ex_start, r.ex_rank, r.ex_slot, r.ex_sh = (ex.start.data_ptr(), ex.rank.data_ptr(),
                                                         ex.slot.data_ptr(), ex.sh.data_ptr())
            r.n_ex, r.n_peers = ex.n_ex, self.transport.size
            r.peer_base0, r.peer_base1, r.peer_ld = N.hp(ex.base[0]), N.hp(ex.base[1]), N.hp(ex.ld)
            r.ex_border = N.hp(ex.border) if ex.border is not None else 0
            r.mailboxes = N.hp(ex.mail_ptrs)
            r.barrier_epoch0 = ex.epoch
        r.p0, r.p1, r.p2 = self._law_args()
        r.half_dt_over_m, r.dt = 0.5 * cfg.dt / cfg.mass, float(cfg.dt)
        r.frc, r.ld_f = s.frc.data_ptr(), s.ld
        r.xref, r.ld_ref = L.ref_positions_dev.data_ptr(), L.ref_positions_dev.stride(0)
        r.thermo, r.thermo_stride = self.thermo.data_ptr(), self.thermo.shape[1]
        r.status, r.guard_lim2 = self.status.ptr, (0.5 * cfg.verlet_buffer) ** 2
        r.k_last, r.epoch_step, r.reneigh = K, epoch_step, cfg.reneigh_interval
        r.thermo_every, r.store_every, r.rebuild_at_k0 = self.thermo_every, int(self.store_forces == "every"), int(
            rebuilt)
        r.rank, r.size, r.barrier_timeout_s = self.transport.rank, self.transport.size, self.peer_timeout_s
        r.time_launches = int(self.event_pairs is not None)
        return r

    def launch_times(self) -> list:
        """Device milliseconds of every step launch timed since the last call
        (batched path with ``event_pairs`` set; CUDA events on the stream)."""
        torch.cuda.current_stream(self.device).synchronize()
        out = []
        if self.event_pairs is not None:
            out = [a.elapsed_time(b) for a, b in self.event_pairs]
            self.event_pairs.clear()
        buf = np.zeros(1 << 16, dtype=np.float32)
        m = N.lib.tmd_run_launch_times(_stream(), N.hp(buf), buf.size)
        return out + [float(x) for x in buf[:max(m, 0)]]


def rank_program(cfg: SimConfig, world=None, store: ParticleStore | None = None, backend=None, **kw):
    """Generator with the reference's shape (driver.py:128-177): yields ("step", k), returns a RankReport.

    ``world`` may be a ``Decomposition`` (or None for this process's rank in
    torch.distributed / a single rank); ``backend`` is accepted and ignored.
    """
    transport = kw.pop("transport", None)
    if transport is None and torch.distributed.is_available() and torch.distributed.is_initialized():
        transport = DistTransport()
    # the reference raises at the failing step and never yields a violating state
    kw.setdefault("check_every_step", True)
    kw.setdefault("store_forces", "every")  # callers inspect store forces at the yields
    kw.setdefault("exact_yields", True)  # and the state of step k at ("step", k)
    sim = Simulation(cfg, store=store, decomp=world, transport=transport, **kw)
    yield from sim.iter_steps()
    return sim.finish().ranks[0]


def run(cfg: SimConfig, steps: int | None = None, mode: str = "fast", thermo_every: int = 1,
        device=None, transport=None, profile: bool = False) -> Report:
    """Run cfg on this process's GPU(s): one rank per process, NCCL between ranks.

    Single process -> P = 1.  Under torchrun (torch.distributed initialised
    with the NCCL backend) every process is one rank of the six-stencil
    decomposition.
    """
    if transport is None and torch.distributed.is_available() and torch.distributed.is_initialized():
        transport = DistTransport()
    sim = Simulation(cfg, transport=transport, mode=mode, thermo_every=thermo_every, device=device,
                     profile=profile)
    return sim.run(steps)
