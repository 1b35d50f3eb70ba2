"""3-D domain decomposition and the halo protocol on device buffers.

Reference: comm.py:171-498.  Same decomposition (``factor_rank_grid``, rank
numbering, ``slab_bounds`` expression, six-stencil rounds x -> y -> z with a
(+, -) entry pair per round) and the same three phases:

  exchange        comm.py:340-400  migrate leavers, wrap at the periodic face
  define_borders  comm.py:434-466  ship border copies, record the plan
  synchronize     comm.py:469-498  replay the plan every step

Data movement is done by libtinymd_b200.so kernels (order-preserving select,
gather + periodic shift, in-place self wrap, flattened self-ghost refresh);
rank-to-rank traffic is NCCL point-to-point through ``torch.distributed``
(one process per GPU; counts first, then payloads, the reference's mailbox
FIFO order per peer).  The store order produced is exactly the reference's:
survivors keep their order, arrivals are appended per entry, ghosts are
appended round by round and entry by entry.

``HaloOps`` is the device-primitive layer; the gloo CPU tests substitute a
test double for it (tests/halo_fakes.py) to exercise the host-side protocol
with world_size > 1 on CPU.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .core import AABB
from .errors import ProtocolError

__all__ = ["factor_rank_grid", "rank_grid_index", "rank_grid_coords", "slab_bounds", "Face",
           "Decomposition", "SingleRankTransport", "DistTransport", "BorderPlan", "Halo"]


# ---------------------------------------------------------------------------
# decomposition (comm.py:171-274)
# ---------------------------------------------------------------------------

def factor_rank_grid(p: int) -> tuple:
    """Near-cubic factorisation, largest primes onto the smallest axis (comm.py:171-186)."""
    if p <= 0:
        raise ValueError("rank count must be positive")
    primes, rest, q = [], p, 2
    while rest > 1:
        while rest % q == 0:
            primes.append(q)
            rest //= q
        q += 1
    dims = [1, 1, 1]
    for f in sorted(primes, reverse=True):
        dims[int(np.argmin(dims))] *= f
    return tuple(sorted(dims, reverse=True))


def rank_grid_index(coords, grid) -> int:
    """rank = (cz * gy + cy) * gx + cx (comm.py:189-192)."""
    return (coords[2] * grid[1] + coords[1]) * grid[0] + coords[0]


def rank_grid_coords(rank: int, grid) -> tuple:
    return rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1])


def slab_bounds(global_box: AABB, grid, coords) -> AABB:
    """lo + ext * (c / g) .. lo + ext * ((c + 1) / g), bit-identical on both sides of a face."""
    lo, ext = global_box.lo, global_box.extent()
    g = np.asarray(grid, dtype=np.float64)
    c = np.asarray(coords, dtype=np.float64)
    return AABB.from_arrays(lo + ext * (c / g), lo + ext * ((c + 1.0) / g))


@dataclass
class Face:
    """One stencil entry: traffic through the +/- face of dimension `dim`."""

    dim: int
    sign: int
    send_to: int
    recv_from: int
    face: float
    shift: np.ndarray  # (3,) periodic shift applied on the way out

    @property
    def tag(self) -> int:
        return 0 if self.sign > 0 else 1


class Decomposition:
    """This rank's place in the six-stencil rank grid (comm.py:210-274)."""

    def __init__(self, global_box: AABB, size: int = 1, rank: int = 0, spacing: float = 0.0, grid=None):
        self.global_box = global_box
        self.size = size
        self.rank = rank
        if grid is None:
            grid = factor_rank_grid(size)
        grid = tuple(int(g) for g in grid)
        if len(grid) != 3 or min(grid) < 1 or int(np.prod(grid)) != size:
            raise ValueError(f"rank grid {grid} does not hold {size} ranks")
        self.grid = grid
        self.coords = rank_grid_coords(rank, self.grid)
        self.slab = slab_bounds(global_box, self.grid, self.coords)
        self.spacing = float(spacing)
        ext = global_box.extent()
        self.rounds: list[list[Face]] = []
        for dim in range(3):
            pair = []
            for sign in (+1, -1):
                to = list(self.coords)
                to[dim] = (self.coords[dim] + sign) % self.grid[dim]
                frm = list(self.coords)
                frm[dim] = (self.coords[dim] - sign) % self.grid[dim]
                edge = (self.coords[dim] == self.grid[dim] - 1) if sign > 0 else (self.coords[dim] == 0)
                shift = np.zeros(3)
                if edge:
                    shift[dim] = -ext[dim] if sign > 0 else ext[dim]
                face = self.slab.hi[dim] if sign > 0 else self.slab.lo[dim]
                pair.append(Face(dim, sign, rank_grid_index(to, self.grid),
                                 rank_grid_index(frm, self.grid), float(face), shift))
            self.rounds.append(pair)

    def is_self(self, dim: int) -> bool:
        return self.grid[dim] == 1

    @property
    def all_self(self) -> bool:
        return self.size == 1

    def owns(self, points) -> np.ndarray:
        return self.slab.contains(points)


# ---------------------------------------------------------------------------
# transports
# ---------------------------------------------------------------------------

_ZERO3 = np.zeros(3)


class _Ticks:
    """TMD_TRACE_REBUILD=3: host times of a protocol call's sub-steps, appended
    to owner.ticks (diagnostics)."""

    def __init__(self, owner, name):
        import os
        import time

        self.on = os.environ.get("TMD_TRACE_REBUILD") == "3"
        if not self.on:
            return
        self.time = time.perf_counter
        self.t = self.time()
        self.rec = {"call": name}
        if not hasattr(owner, "ticks"):
            owner.ticks = []
        owner.ticks.append(self.rec)

    def __call__(self, label):
        if self.on:
            now = self.time()
            self.rec[label] = round((now - self.t) * 1e3, 2)
            self.t = now


class SingleRankTransport:
    """P = 1: every peer is this rank; nothing travels."""

    rank, size = 0, 1

    def sendrecv(self, sends, recvs):
        if sends or recvs:
            raise ProtocolError("single-rank transport asked to move data")

    def allreduce_(self, t: torch.Tensor, op="sum"):
        return t

    def barrier(self):
        pass

    def alltoall(self, payload: torch.Tensor, send_counts):
        """Rows of `payload` grouped by destination rank -> (received rows, per-source counts)."""
        return payload, list(send_counts)

    def alltoall_v(self, payload: torch.Tensor, send_counts, recv_counts):
        return payload

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        """(P, *t.shape) stack of every rank's t."""
        return t[None]

    def all_gather_object(self, obj):
        return [obj]


class DistTransport:
    """Point-to-point over torch.distributed (NCCL on GPUs, gloo in CPU tests).

    Each round posts every send and receive of the round in one
    ``batch_isend_irecv`` group, tagged by stencil entry, so messages between
    the same two ranks are matched in entry order (the reference's per-pair
    FIFO, comm.py:83-104).
    """

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)

    def sendrecv(self, sends, recvs):
        ops = []
        for peer, tag, t in sends:
            if t.numel():
                ops.append(self.dist.P2POp(self.dist.isend, t, peer, self.group, tag))
        for peer, tag, t in recvs:
            if t.numel():
                ops.append(self.dist.P2POp(self.dist.irecv, t, peer, self.group, tag))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce_(self, t: torch.Tensor, op="sum"):
        red = self.dist.ReduceOp.SUM if op == "sum" else self.dist.ReduceOp.MAX
        self.dist.all_reduce(t, op=red, group=self.group)
        return t

    def barrier(self):
        self.dist.barrier(group=self.group)

    def alltoall(self, payload: torch.Tensor, send_counts):
        dist, dev = self.dist, payload.device
        sc = torch.tensor([int(c) for c in send_counts], dtype=torch.int64, device=dev)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = [int(c) for c in rc.cpu().tolist()]
        out = torch.empty((sum(recv_counts),) + tuple(payload.shape[1:]), dtype=payload.dtype, device=dev)
        dist.all_to_all_single(out, payload.contiguous(), recv_counts, [int(c) for c in send_counts],
                               group=self.group)
        return out, recv_counts

    def warm_up(self, device) -> None:
        """Establish every pairwise connection once (NCCL creates them lazily on
        first use; a rare first message, e.g. the first diagonal migration,
        would otherwise pay the set-up inside a step)."""
        if getattr(self, "_warm", False):
            return
        # small and large messages: NCCL adds P2P channels the first time a message
        # passes its size thresholds (the migration payload grows as a run warms up)
        for per_peer in (1, 1 << 18):
            buf = torch.ones((self.size * per_peer, 1), dtype=torch.float64, device=device)
            self.alltoall_v(buf, [per_peer] * self.size, [per_peer] * self.size)
        one = torch.ones(1, dtype=torch.float64, device=device)
        self.allgather(one)
        self.allreduce_(one, "max")
        torch.cuda.synchronize(device)
        self._warm = True

    def alltoall_v(self, payload: torch.Tensor, send_counts, recv_counts):
        out = torch.empty((int(sum(recv_counts)),) + tuple(payload.shape[1:]), dtype=payload.dtype,
                          device=payload.device)
        self.dist.all_to_all_single(out, payload.contiguous(), [int(c) for c in recv_counts],
                                    [int(c) for c in send_counts], group=self.group)
        return out

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        flat = t.contiguous().reshape(-1)
        out = torch.empty(self.size * flat.numel(), dtype=t.dtype, device=t.device)
        self.dist.all_gather_into_tensor(out, flat, group=self.group)  # concatenated (gloo and NCCL)
        return out.view((self.size,) + tuple(t.shape))

    def all_gather_object(self, obj):
        out = [None] * self.size
        self.dist.all_gather_object(out, obj, group=self.group)
        return out


# ---------------------------------------------------------------------------
# the plan (comm.py:403-431)
# ---------------------------------------------------------------------------

@dataclass
class PlanSend:
    peer: int
    tag: int
    dim: int
    idx: torch.Tensor  # int32 source slots (locals or earlier ghosts)
    sh: torch.Tensor  # fp64 recorded shift along dim: (x + s) - x (comm.py:449)
    ghost_start: int = -1  # self entries deliver in place


@dataclass
class PlanRecv:
    peer: int
    tag: int
    ghost_start: int
    count: int


@dataclass
class BorderPlan:
    rounds: list = field(default_factory=list)  # [(sends, recvs)] per dimension
    n_local: int = 0
    n_ghost: int = 0
    flat_src: torch.Tensor | None = None  # P = 1 fast path: root local of every ghost
    flat_sh: torch.Tensor | None = None  # (3, n_ghost) accumulated shifts
    # define_borders(provenance=True): owner rank, owner's local index and the
    # accumulated shift of every ghost (the fused refresh's export requests)
    prov_rank: torch.Tensor | None = None
    prov_root: torch.Tensor | None = None
    prov_sh: torch.Tensor | None = None
    # define_borders_direct: no rounds; ghosts are refreshed by their owners'
    # step kernels only (exports), so synchronize() refuses this plan
    direct: bool = False


class _Provenance:
    """Growing device arrays of ghost provenance, indexed by ghost ordinal."""

    def __init__(self, device, cap):
        cap = max(int(cap), 1)
        self.rank = torch.empty(cap, dtype=torch.int32, device=device)
        self.root = torch.empty(cap, dtype=torch.int32, device=device)
        self.sh = torch.zeros((3, cap), dtype=torch.float64, device=device)

    def ensure(self, n):
        cap = self.rank.numel()
        if n <= cap:
            return
        new = max(n, 2 * cap)
        for name in ("rank", "root"):
            t = getattr(self, name)
            u = torch.empty(new, dtype=t.dtype, device=t.device)
            u[:cap] = t
            setattr(self, name, u)
        u = torch.zeros((3, new), dtype=torch.float64, device=self.sh.device)
        u[:, :cap] = self.sh
        self.sh = u


# ---------------------------------------------------------------------------
# the protocol
# ---------------------------------------------------------------------------

class Halo:
    """Exchange / borders / sync of one rank, on device buffers."""

    def __init__(self, decomp: Decomposition, transport=None, ops=None):
        self.decomp = decomp
        self.transport = transport or SingleRankTransport()
        if ops is None:
            from .halo_ops import DeviceHaloOps

            ops = DeviceHaloOps()
        self.ops = ops
        self.small_gather = None
        if self.transport.size > 1 and torch.cuda.is_available():
            # the borders' count message (a page-locked allocation mid-run would order
            # every stream of the context; see Simulation.__init__)
            self._meta_pin = torch.empty(16, dtype=torch.int64, pin_memory=True)

    # comm.py:340-400
    def exchange(self, store, status=None) -> None:
        """Migrate leavers; with ``status`` the final ownership check is written to that
        device status word (TMD_PROTOCOL) instead of being read back here."""
        store.clear_ghosts()
        ops, tr = self.ops, self.transport
        for entries in self.decomp.rounds:
            d = entries[0].dim
            n = store.n_local
            if self.decomp.is_self(d):
                plus, minus = entries
                ops.wrap_self(store, d, plus.face, minus.face, plus.shift[d], minus.shift[d])
                continue
            plus, minus = entries
            picked = ops.select_pair(store.pos[d], n, (ops.GE, plus.face), (ops.LT, minus.face))
            outgoing = [(e, ops.pack_pos_vel(store, idx, e.shift)) for e, idx in zip(entries, picked)]
            keep = ops.select(store.pos[d], n, ops.IN, entries[1].face, entries[0].face)
            ops.compact_locals(store, keep)
            counts = self._exchange_counts([(e.send_to, e.tag, p.shape[1]) for e, p in outgoing],
                                           [(e.recv_from, e.tag) for e in entries])
            inbox = [(e.recv_from, e.tag, ops.empty((6, c), store)) for e, c in zip(entries, counts)]
            tr.sendrecv([(e.send_to, e.tag, p) for e, p in outgoing], inbox)
            for _, _, data in inbox:
                if data.shape[1]:
                    store.append_locals(data[0:3].t(), data[3:6].t())
        if status is not None and hasattr(ops, "check_owned_deferred"):
            ops.check_owned_deferred(store, self.decomp.slab, status)
        elif ops.any_outside(store, self.decomp.slab):
            raise ProtocolError(
                f"rank {self.decomp.rank}: after exchange a local particle is outside the ownership region")

    def _exchange_counts(self, sends, recvs):
        tr = self.transport
        dev = self.ops.count_device()
        out = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in recvs]
        tr.sendrecv([(p, tag, torch.full((1,), int(k), dtype=torch.int64, device=dev)) for p, tag, k in sends],
                    [(p, tag, t) for (p, tag), t in zip(recvs, out)])
        return [int(t.item()) for t in out]

    # comm.py:434-466
    def define_borders(self, store, provenance: bool = False, direct: bool = False) -> BorderPlan:
        """With ``provenance`` the plan also records every ghost's owner (rank,
        local index, accumulated shift) and remote border packets carry it.

        ``direct`` (P = 1 only): one pass instead of three rounds -- the same
        ghost set with the same coordinates, grouped by local atom instead of
        the reference's round order (the production path; exact mode keeps
        the rounds so its lists follow the reference's order)."""
        if store.n_ghost:
            raise ProtocolError("define_borders must start with an empty ghost region")
        if direct and self.decomp.all_self and hasattr(self.ops, "borders_direct"):
            root, sh = self.ops.borders_direct(store, self.decomp.slab, self.decomp.spacing,
                                               self.decomp.global_box.extent())
            plan = BorderPlan(n_local=store.n_local, n_ghost=store.n_ghost, flat_src=root, flat_sh=sh)
            plan.prov_rank = torch.zeros(root.numel(), dtype=torch.int32, device=root.device)
            plan.prov_root, plan.prov_sh = root, sh
            return plan
        ops, tr, r = self.ops, self.transport, self.decomp.spacing
        me, nl = self.decomp.rank, store.n_local
        prov = _Provenance(store.device, store.n_local // 4) if provenance else None
        plan = BorderPlan()
        for entries in self.decomp.rounds:
            d = entries[0].dim
            n0 = store.n_total
            sends, recvs, outgoing = [], [], []
            plus, minus = entries
            # both faces tested against the round-start snapshot [0, n0) (comm.py:446-448)
            picked = ops.select_pair(store.pos[d], n0, (ops.GT, plus.face - r), (ops.LT, minus.face + r))
            for e, idx in zip(entries, picked):
                if e.send_to == self.decomp.rank:
                    start, sh = ops.emit_ghosts(store, idx, e.shift, d, peer=e.send_to)
                    sends.append(PlanSend(e.send_to, e.tag, d, idx, sh, start))
                    if prov is not None:
                        g0, k = start - nl, idx.numel()
                        prov.ensure(g0 + k)
                        ops.provenance(nl, me, idx, d, sh, prov, prov.rank[g0:], prov.root[g0:],
                                       prov.sh[:, g0:], prov.sh.stride(0))
                else:
                    sh = ops.plan_shift(store, idx, d, e.shift[d])
                    if prov is not None:
                        outgoing.append((e, ops.pack_pos_prov(store, idx, e.shift, nl, me, d, sh, prov)))
                    else:
                        outgoing.append((e, ops.pack_pos(store, idx, e.shift)))
                    sends.append(PlanSend(e.send_to, e.tag, d, idx, sh))
            if outgoing:
                rows = 8 if prov is not None else 3
                counts = self._exchange_counts([(e.send_to, e.tag, p.shape[1]) for e, p in outgoing],
                                               [(e.recv_from, e.tag) for e in entries])
                inbox = [(e.recv_from, e.tag, ops.empty((rows, c), store)) for e, c in zip(entries, counts)]
                tr.sendrecv([(e.send_to, e.tag, p) for e, p in outgoing], inbox)
                for (peer, tag, data) in inbox:
                    start = store.append_ghosts(data[0:3].t(), peer=peer)
                    recvs.append(PlanRecv(peer, tag, start, data.shape[1]))
                    if prov is not None and data.shape[1]:
                        g0, k = start - nl, data.shape[1]
                        prov.ensure(g0 + k)
                        prov.rank[g0:g0 + k] = data[3].to(torch.int32)
                        prov.root[g0:g0 + k] = data[4].to(torch.int32)
                        prov.sh[:, g0:g0 + k] = data[5:8]
            plan.rounds.append((sends, recvs))
        plan.n_local, plan.n_ghost = store.n_local, store.n_ghost
        if prov is not None:
            ng = plan.n_ghost
            prov.ensure(ng)
            plan.prov_rank, plan.prov_root, plan.prov_sh = prov.rank[:ng], prov.root[:ng], prov.sh[:, :ng]
        if self.decomp.all_self:
            plan.flat_src, plan.flat_sh = ops.flatten_plan(store, plan)
        return plan

    # -- direct protocol (production path at P > 1) -----------------------------
    def _edge_shifts(self):
        dc = self.decomp
        ext = dc.global_box.extent()
        s_hi = [-float(ext[d]) if dc.coords[d] == dc.grid[d] - 1 else 0.0 for d in range(3)]
        s_lo = [float(ext[d]) if dc.coords[d] == 0 else 0.0 for d in range(3)]
        return N.host_f64(s_hi), N.host_f64(s_lo), N.host_i32(list(dc.coords) + list(dc.grid))

    def _allgather(self, t: torch.Tensor) -> torch.Tensor:
        """The direct protocol's count all-gathers: over the NVLink mailboxes once
        the driver has mapped them (``self.small_gather``, GhostExports.allgather),
        else through the transport (NCCL)."""
        g = getattr(self, "small_gather", None)
        if g is not None and t.numel() <= N.lib.tmd_peer_gather_words():
            return g(t)
        return self.transport.allgather(t)

    def exchange_direct(self, store, status=None) -> None:
        """comm.py:340-400 in one all-to-all: every leaver goes straight to the
        rank that the three rounds would deliver it to (the guard bounds a move
        to one slab), with the same wrap shifts.  Survivors keep their order;
        arrivals are appended by source rank (the production path re-sorts the
        locals by cell right after)."""
        store.clear_ghosts()
        tr, dc, dev = self.transport, self.decomp, store.device
        P, me, n = tr.size, dc.rank, store.n_local
        tick = _Ticks(self, "exchange_direct")
        s_hi, s_lo, geom = self._edge_shifts()
        # classification and grouping stay on the device: the leavers' counts per
        # destination and this rank's (kept, leaving) totals travel in one
        # all-gather, the exchange's only host read
        dest, keep, leave, cnt = self.ops.exchange_classify_dev(store, dc.slab, s_hi, s_lo, geom)
        tick("classify")
        ids, _, per = self.ops.group_by_rank(dest[:n], None, P)  # stayers (dest -1) drop out
        meta = self._allgather(torch.cat([per.to(torch.int64), cnt.to(torch.int64)])).cpu().numpy()
        C = meta[:, :P]  # C[src, dst]
        nk, nl = int(meta[me, P]), int(meta[me, P + 1])
        tick("allgather")
        # leavers grouped by destination, packed as (x, v) rows
        payload = self.ops.pack_rows(store.pos, store.vel, store.ld, ids[:nl], 6)
        tick("pack")
        if nk != n:
            if hasattr(self.ops, "compact_locals_swap"):
                self.ops.compact_locals_swap(store, keep[:nk])
            else:
                self.ops.compact_locals(store, keep[:nk])
        tick("compact")
        got = tr.alltoall_v(payload, C[me], C[:, me])
        tick("alltoall")
        R = int(got.shape[0])
        if R:
            store.ensure_capacity(nk + R)
            self.ops.unpack_rows(store, got, nk)
            store.n_local = nk + R
        tick("append")
        if status is not None and hasattr(self.ops, "check_owned_deferred"):
            self.ops.check_owned_deferred(store, dc.slab, status)
        elif self.ops.any_outside(store, dc.slab):
            raise ProtocolError(f"rank {me}: after exchange a local particle is outside the ownership region")

    def define_borders_direct(self, store, extra=(), lazy=False):
        """comm.py:434-466 in one all-to-all: every copy the three rounds would
        create (including the corner chains) is sent straight to the rank that
        holds it, with the same coordinates and recorded shifts.  Returns the
        plan and the export records (root, rank, slot, shift (3, M)) for the
        fused refresh: the sender knows each copy's slot on its receiver from
        the all-gathered count matrix (receivers append by source rank).
        ``extra``: small ints every rank contributes to the same all-gather
        (left in ``self.gathered_extra``).  ``lazy``: return the records as a
        callable (the driver computes them after launching the list build)."""
        if store.n_ghost:
            raise ProtocolError("define_borders must start with an empty ghost region")
        tr, dc, dev = self.transport, self.decomp, store.device
        P, me, n, r = tr.size, dc.rank, store.n_local, dc.spacing
        tick = _Ticks(self, "borders_direct")
        s_hi, s_lo, geom = self._edge_shifts()
        thr_hi = N.host_f64([float(h) - r for h in dc.slab.hi])
        thr_lo = N.host_f64([float(lo) + r for lo in dc.slab.lo])
        M, rec, root, sh, dest = self.ops.borders_records(store, thr_hi, thr_lo, s_hi, s_lo, geom)
        tick("records")
        # copies grouped by destination on the device (records in group order)
        perm, rank_sorted, per = self.ops.group_by_rank(dest[:M], None, P)
        tick("group")
        ex = [int(v) for v in extra]
        # [per-destination counts (device), n_local, capacity, extra] in one all-gather
        host = np.array([n, store.capacity] + ex, dtype=np.int64)
        if dev.type == "cuda":
            pin = getattr(self, "_meta_pin", None)
            if pin is None or pin.numel() < host.size:
                pin = self._meta_pin = torch.empty(max(host.size, 16), dtype=torch.int64, pin_memory=True)
            pin.numpy()[:host.size] = host
            tail = pin[:host.size].to(dev, non_blocking=True)
        else:
            tail = torch.from_numpy(host)
        meta = self._allgather(torch.cat([per.to(torch.int64), tail])).cpu().numpy()
        tick("allgather")
        C, nl_all, cap_all = meta[:, :P], meta[:, P], meta[:, P + 1]
        self.gathered_extra = meta[:, P + 2:].copy()  # every rank's `extra` (e.g. buffer flags)
        # a rank whose locals + arriving ghosts exceed its capacity reallocates its
        # buffers below (ensure_capacity); every rank sees that from the same
        # all-gather, so buffer flags gathered before the growth are corrected here
        self.gathered_grew = (nl_all + C.sum(axis=0)) > cap_all
        payload = self.ops.pack_rows(rec, None, rec.stride(0), perm, 3)
        tick("pack")
        got = tr.alltoall_v(payload, C[me], C[:, me])
        tick("alltoall")
        R = int(got.shape[0])
        store.ensure_capacity(n + R)
        if R:
            self.ops.unpack_rows(store, got, n)
        store.n_ghost = R
        store.set_ghost_segments(np.arange(P), C[:, me])
        tick("append")
        # slot of my t-th copy to q: receiver's n_local + copies from lower ranks + rank within my packet
        base = nl_all + np.array([C[:me, q].sum() for q in range(P)], dtype=np.int64)
        start = np.concatenate([[0], np.cumsum(C[me])[:-1]])

        def records():
            slot = self.ops.border_slots(rank_sorted, base - start)
            return self.ops.gather_i32(root, perm), rank_sorted, slot, self.ops.gather_cols(sh, perm)

        plan = BorderPlan(n_local=n, n_ghost=R, direct=True)
        if lazy:
            return plan, records
        return plan, records()

    # comm.py:469-498
    def synchronize(self, store, plan: BorderPlan) -> None:
        if plan.direct:
            raise ProtocolError("a direct border plan is refreshed by the fused step kernel, not synchronize()")
        if store.n_local != plan.n_local or store.n_ghost != plan.n_ghost:
            raise ProtocolError(
                f"rank {self.decomp.rank}: store ({store.n_local} locals, {store.n_ghost} ghosts) "
                f"does not match the border plan ({plan.n_local}, {plan.n_ghost})")
        ops = self.ops
        if plan.flat_src is not None:
            ops.sync_flat(store, plan)
            return
        for sends, recvs in plan.rounds:
            outgoing = []
            for s in sends:
                if s.ghost_start >= 0:
                    ops.gather_into_ghosts(store, s)
                else:
                    outgoing.append((s.peer, s.tag, ops.pack_sync(store, s)))
            if outgoing or recvs:
                inbox = [(rv.peer, rv.tag, ops.empty((3, rv.count), store)) for rv in recvs]
                self.transport.sendrecv(outgoing, inbox)
                for rv, (_, _, data) in zip(recvs, inbox):
                    if data.shape[1] != rv.count:
                        raise ProtocolError("sync payload does not match the plan")
                    store.pos[:, rv.ghost_start:rv.ghost_start + rv.count] = data
