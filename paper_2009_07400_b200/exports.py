"""Fused ghost refresh: export tables and peer position buffers.

The reference refreshes ghosts once per step with the synchronize phase
(comm.py:469-498): three rounds of pack -> send -> unpack along x, y, z.  On
B200 the owner of each mirrored atom writes the copies itself, in the same
kernel that drifts it (tmd_step_lj's NEXT phase): ``x_new + s`` goes straight
into every ghost slot that mirrors the atom -- in this rank's next position
buffer, or in a peer's next buffer mapped over NVLink by CUDA IPC.

A ghost's provenance (owner rank, owner's local index, accumulated shift s,
recorded by ``Halo.define_borders(provenance=True)``) becomes an export
request sent to the owner (one all-to-all per epoch); the owner groups the
requests by local index (tmd_exports_build).  Because each hop of the
reference's chain moves one coordinate once, ``x_root + s`` equals the
hop-by-hop sum bit for bit.

Ordering across ranks: every fused step is followed by an all-reduce (max)
of the step's guard displacement.  It completes only after every rank's
kernel of that step, so (a) ghost slots written by peers are complete before
the next kernel reads them, and (b) no rank writes a buffer a peer is still
reading.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _native as N
from .errors import ProtocolError
from .neighbor import _stream

KMAX_PEERS = 8  # force.cu kMaxPeers


def _handle_of(t: torch.Tensor):
    size = N.lib.tmd_ipc_handle_size()
    buf = (C.c_char * size)()
    off = C.c_int64(0)
    N.call("tmd_ipc_handle", t.data_ptr(), C.addressof(buf), C.addressof(off))
    return bytes(buf), int(off.value)


class PeerMaps:
    """CUDA-IPC mappings of peers' position blocks, opened once per block."""

    def __init__(self):
        self.bases = {}  # handle bytes -> mapped base pointer

    def open(self, handle: bytes, offset: int) -> int:
        base = self.bases.get(handle)
        if base is None:
            buf = C.create_string_buffer(handle, len(handle))
            ptr, b = C.c_void_p(0), C.c_void_p(0)
            N.call("tmd_ipc_open", C.addressof(buf), 0, C.addressof(ptr), C.addressof(b))
            base = int(b.value)
            self.bases[handle] = base
        return base + int(offset)

    def close(self):
        for base in self.bases.values():
            try:
                N.lib.tmd_ipc_close(C.c_void_p(base))
            except Exception:  # noqa: BLE001 - best effort at teardown
                pass
        self.bases.clear()


# one mapping per peer block for the whole process: a block the caching
# allocator hands to the next Simulation keeps its handle and its mapping
_PROCESS_MAPS = PeerMaps()


class GhostExports:
    """Export table of one epoch plus the per-step peer buffer pointers."""

    def __init__(self, transport, device, status, peer_maps: PeerMaps | None = None, decomp=None,
                 peer_timeout_s: float = 120.0):
        if transport.size > KMAX_PEERS:
            raise ValueError(f"the fused ghost refresh supports up to {KMAX_PEERS} ranks")
        self.tr = transport
        self.device = device
        self.status = status
        self.maps = peer_maps if peer_maps is not None else _PROCESS_MAPS
        self.n_ex = 0  # entries; also the leading dimension of the shift table
        self.n_entries = 0
        self.start = self.rank = self.slot = self.sh = None
        self.base = [np.zeros(KMAX_PEERS, dtype=np.uint64) for _ in range(2)]
        self.ld = np.zeros(KMAX_PEERS, dtype=np.int64)
        # per-step barrier mailboxes (tmd_peer_sync), one per rank, IPC-mapped
        self.mailbox = None
        self.mail_ptrs = np.zeros(KMAX_PEERS, dtype=np.uint64)
        self.epoch = 0
        self.peer_timeout_s = float(peer_timeout_s)
        if transport.size > 1:
            self.mailbox = torch.zeros(N.lib.tmd_mailbox_words(), dtype=torch.int64, device=device)
        # the borders' selection thresholds: only atoms built inside them have copies
        self.border = None
        if decomp is not None:
            r = decomp.spacing
            self.border = N.host_f64([float(h) - r for h in decomp.slab.hi] + [float(lo) + r for lo in decomp.slab.lo])

    # -- per epoch -------------------------------------------------------------
    def build(self, store, plan) -> None:
        """Export table from the plan's provenance; peer buffers of this epoch."""
        if plan.prov_rank is None:
            raise ProtocolError("fused ghost refresh needs a border plan with provenance")
        tr, dev = self.tr, self.device
        nl, ng = plan.n_local, plan.n_ghost
        slot = torch.arange(nl, nl + ng, dtype=torch.int32, device=dev)
        if tr.size == 1:
            root, src, sh = plan.prov_root, torch.zeros(ng, dtype=torch.int32, device=dev), plan.prov_sh
            n_ex = ng
        else:
            owner = plan.prov_rank.to(torch.int64)
            order = torch.argsort(owner, stable=True)
            counts = torch.bincount(owner, minlength=tr.size).cpu().tolist()
            req = torch.stack([plan.prov_root.to(torch.float64), slot.to(torch.float64), plan.prov_sh[0],
                               plan.prov_sh[1], plan.prov_sh[2]], dim=1)[order]
            got, rc = tr.alltoall(req, counts)
            n_ex = got.shape[0]
            src = torch.repeat_interleave(torch.arange(tr.size, dtype=torch.int32, device=dev),
                                          torch.tensor(rc, dtype=torch.int64, device=dev))
            root = got[:, 0].to(torch.int32)
            slot = got[:, 1].to(torch.int32)
            sh = got[:, 2:5].t().contiguous()
        self._table(nl, n_ex, root, src, slot, sh)
        self._peer_buffers(store)

    def build_dev(self, store, root, sh, d_count: int, room: int, launch: bool = True):
        """P = 1 export table from borders_direct_dev's buffers, the copy count
        on the device (at address d_count, at most ``room``): entry e is ghost
        slot n_local + e, mirroring local root[e] with shift sh[:, e].  The
        shift table's leading dimension is ``room`` (n_ex)."""
        dev = self.device
        nl = store.n_local
        m = max(room, 1)
        if getattr(self, "_dev_bufs", None) is None or self._dev_bufs[0].numel() < m + 1 or \
                self._dev_bufs[2].numel() < nl + 1:
            big = int(max(m, nl) * 1.05) + 1024
            self._dev_bufs = (torch.zeros(big, dtype=torch.int32, device=dev),  # source rank: 0
                              torch.empty(big, dtype=torch.int32, device=dev),  # receiver slots
                              torch.empty(big, dtype=torch.int32, device=dev))  # CSR start
        zeros, slots, start = self._dev_bufs
        if getattr(self, "_dev_slots_for", None) != (nl, m, slots.data_ptr()):
            # entry e's receiver slot is n_local + e (n_local is fixed at P = 1)
            torch.arange(nl, nl + m, dtype=torch.int32, device=dev, out=slots[:m])
            self._dev_slots_for = (nl, m, slots.data_ptr())
        self.n_ex = m  # the shift table's leading dimension
        self.n_entries = None  # on the device until the epoch's read-back (driver sets it)
        self.start = start[: nl + 1]
        if self.rank is None or self.rank.numel() < m or self.sh is None or self.sh.stride(0) != m:
            self.rank = torch.empty(m, dtype=torch.int32, device=dev)
            self.slot = torch.empty(m, dtype=torch.int32, device=dev)
            self.sh = torch.empty((3, m), dtype=torch.float64, device=dev)
        if not launch:  # buffers only (tmd_epoch_p1 builds the table); the caller maps the peers
            return zeros, slots
        N.call("tmd_exports_build_dev", nl, room, d_count, root.data_ptr(), zeros.data_ptr(), slots.data_ptr(),
               sh.data_ptr(), sh.stride(0), self.start.data_ptr(), self.rank.data_ptr(), self.slot.data_ptr(),
               self.sh.data_ptr(), m, self.status.ptr, _stream())
        self._peer_buffers(store)

    def build_direct(self, store, records, flags=None) -> None:
        """Export table from the sender-side records of Halo.define_borders_direct;
        ``flags``: every rank's buffer_flags(), already all-gathered with the
        border counts (saves the separate all-gather)."""
        root, rank, slot, sh = records
        self._table(store.n_local, int(root.numel()), root, rank, slot, sh)
        self._peer_buffers(store, flags)

    def buffer_flags(self, store):
        """(reallocated, roles swapped) of this rank's position buffers since the
        last epoch -- what _peer_buffers all-gathers."""
        if store.pos_alt is None or store.pos_alt.shape != store.pos.shape:
            store.pos_alt = torch.empty_like(store.pos)
        alt, cur, ld = store.pos_alt.data_ptr(), store.pos.data_ptr(), int(store.ld)
        prev = getattr(self, "_mine", None)
        if prev is not None and {prev[0], prev[1]} == {alt, cur} and prev[2] == ld:
            return (0, 1 if prev[0] != alt else 0)
        return (1, 0)

    def _table(self, nl, n_ex, root, src, slot, sh) -> None:
        dev = self.device
        self.n_ex = self.n_entries = n_ex
        self.start = torch.empty(nl + 1, dtype=torch.int32, device=dev)
        self.rank = torch.empty(max(n_ex, 1), dtype=torch.int32, device=dev)
        self.slot = torch.empty(max(n_ex, 1), dtype=torch.int32, device=dev)
        self.sh = torch.empty((3, max(n_ex, 1)), dtype=torch.float64, device=dev)
        ld_sh = sh.stride(0) if n_ex else 1
        N.call("tmd_exports_build", nl, n_ex, root.data_ptr() if n_ex else 0, src.data_ptr() if n_ex else 0,
               slot.data_ptr() if n_ex else 0, sh.data_ptr() if n_ex else 0, ld_sh, self.start.data_ptr(),
               self.rank.data_ptr(), self.slot.data_ptr(), self.sh.data_ptr(), self.status.ptr, _stream())
        if self.sh.stride(0) != max(n_ex, 1):
            raise ProtocolError("export shift table must be (3, n_ex)")

    def _peer_buffers(self, store, gathered=None) -> None:
        """Both position buffers of every rank; parity 0 = the current `pos_alt` is next.

        IPC handles travel only when some rank's buffers were reallocated; an
        epoch that merely swapped roles (the cell sort swaps, every step swaps)
        costs one small all-gather of (reallocated, swapped) flags."""
        if store.pos_alt is None or store.pos_alt.shape != store.pos.shape:
            store.pos_alt = torch.empty_like(store.pos)
        me = self.tr.rank
        alt, cur, ld = store.pos_alt.data_ptr(), store.pos.data_ptr(), int(store.ld)
        if self.tr.size == 1:
            self.base[0][0], self.base[1][0], self.ld[0] = alt, cur, ld
            return
        if gathered is not None:
            allf = np.asarray(gathered)
        else:
            flags = self.buffer_flags(store)
            allf = self.tr.allgather(torch.tensor(flags, dtype=torch.int64, device=self.device)).cpu().numpy()
        self._mine = (alt, cur, ld)
        if not allf[:, 0].any():
            for r in range(self.tr.size):
                if allf[r, 1]:
                    self.base[0][r], self.base[1][r] = self.base[1][r], self.base[0][r]
            return
        if getattr(self.tr, "same_process", False):
            # in-process ranks (loopback.py): peers' buffers are plain device pointers
            allp = self.tr.all_gather_object((alt, cur, ld, self.mailbox.data_ptr()))
            for r, (p_alt, p_cur, ld_r, p_mail) in enumerate(allp):
                self.base[0][r], self.base[1][r], self.ld[r], self.mail_ptrs[r] = p_alt, p_cur, ld_r, p_mail
            return
        allb = self.tr.all_gather_object((_handle_of(store.pos_alt), _handle_of(store.pos), ld,
                                          _handle_of(self.mailbox)))
        for r, (h_alt, h_cur, ld_r, h_mail) in enumerate(allb):
            if r == me:
                self.base[0][r], self.base[1][r] = alt, cur
                self.mail_ptrs[r] = self.mailbox.data_ptr()
            else:
                self.base[0][r] = self.maps.open(*h_alt)
                self.base[1][r] = self.maps.open(*h_cur)
                self.mail_ptrs[r] = self.maps.open(*h_mail)
            self.ld[r] = ld_r
        # nobody writes into a peer's buffers while that peer is still mapping
        # (a write racing the peer's own IPC mapping work stalled for ~0.5 s)
        self.tr.barrier()

    def ready(self) -> bool:
        """Peers' mailboxes are mapped (after the first epoch's export table)."""
        return self.mailbox is not None and bool(self.mail_ptrs[: self.tr.size].all())

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        """(P, w) stack of every rank's int64 vector t (w <= tmd_peer_gather_words)
        through the NVLink mailboxes, on the stream (tmd_peer_allgather)."""
        w = int(t.numel())
        out = torch.empty((self.tr.size, max(w, 1)), dtype=torch.int64, device=self.device)
        self.gather_epoch = getattr(self, "gather_epoch", 0) + 1
        src = t.to(torch.int64).contiguous()
        N.call("tmd_peer_allgather", self.gather_epoch, self.tr.rank, self.tr.size, N.hp(self.mail_ptrs),
               src.data_ptr(), w, out.data_ptr(), self.peer_timeout_s, self.status.ptr, _stream())
        return out[:, :w]

    def barrier(self, value: torch.Tensor) -> None:
        """Step barrier over NVLink + in-place max of a one-element fp64 tensor."""
        self.epoch += 1
        N.call("tmd_peer_sync", self.epoch, self.tr.rank, self.tr.size, N.hp(self.mail_ptrs), value.data_ptr(),
               self.peer_timeout_s, self.status.ptr, _stream())

    # -- per step ---------------------------------------------------------------
    def args(self, parity: int):
        """tmd_step_lj's export arguments; `parity` = buffer swaps since the epoch began, mod 2."""
        base = self.base[parity & 1]
        return (self.start.data_ptr(), self.rank.data_ptr(), self.slot.data_ptr(), self.sh.data_ptr(), self.n_ex,
                self.tr.size, N.hp(base), N.hp(self.ld), N.hp(self.border) if self.border is not None else 0)
