"""Device primitives of the halo protocol (libtinymd_b200.so halo kernels).

Each method is one or two kernel launches on the current stream; the only
host synchronisations are the selection counts, which the protocol needs to
size NCCL messages and store regions (the reference's counts travel in its
wire header, comm.py:63-80).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .errors import ProtocolError
from .neighbor import DeviceStatus, _stream

_ZERO3 = np.zeros(3)


class DeviceHaloOps:
    GE, LT, GT, IN = N.SEL_GE, N.SEL_LT, N.SEL_GT, N.SEL_IN

    def __init__(self):
        self._count = None

    def count_device(self):
        return torch.device("cuda", torch.cuda.current_device())

    def empty(self, shape, store):
        return torch.empty(shape, dtype=torch.float64, device=store.device)

    def select(self, row: torch.Tensor, n: int, kind: int, thr: float, thr2: float = 0.0) -> torch.Tensor:
        dev = row.device
        if self._count is None or self._count.device != dev:
            self._count = torch.zeros(1, dtype=torch.int32, device=dev)
        idx = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        N.call("tmd_select", row.data_ptr(), n, kind, float(thr), float(thr2), idx.data_ptr(),
               self._count.data_ptr(), _stream())
        k = int(self._count.item())
        return idx[:k]

    def select_pair(self, row: torch.Tensor, n: int, a, b):
        """Both entries of a round in one pass, one count readback: (idx_a, idx_b)."""
        dev = row.device
        if getattr(self, "_counts2", None) is None or self._counts2.device != dev:
            self._counts2 = torch.zeros(2, dtype=torch.int32, device=dev)
        ia = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        ib = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        N.call("tmd_select_pair", row.data_ptr(), n, a[0], float(a[1]), b[0], float(b[1]), ia.data_ptr(),
               ib.data_ptr(), self._counts2.data_ptr(), _stream())
        ka, kb = (int(v) for v in self._counts2.cpu().tolist())
        return ia[:ka], ib[:kb]

    def emit_ghosts(self, store, idx, shift, dim, peer=0):
        """Self-peer border copies appended as ghosts; returns (first slot, recorded shifts)."""
        k = idx.numel()
        start = store.n_total
        store.ensure_capacity(start + k)
        sh = torch.empty(max(k, 1), dtype=torch.float64, device=store.device)
        h = N.host_f64(shift)
        N.call("tmd_emit_ghosts", store.pos.data_ptr(), store.vel.data_ptr(), store.ld, idx.data_ptr(), k,
               N.hp(h), dim, start, sh.data_ptr(), _stream())
        store.n_ghost += k
        store.ghost_peer = np.concatenate([store.ghost_peer, np.full(k, peer, dtype=np.int32)])
        store.ghost_ordinal = np.concatenate([store.ghost_ordinal, np.arange(k, dtype=np.int32)])
        return start, sh[:k]

    def _gather(self, src: torch.Tensor, ld: int, idx: torch.Tensor, shift, dim=0, sh=None, out=None,
                ld_out=None):
        k = idx.numel()
        if out is None:
            out = torch.empty((3, max(k, 1)), dtype=torch.float64, device=src.device)
            ld_out = out.stride(0)
        h = N.host_f64(shift)
        N.call("tmd_gather_shift", src.data_ptr(), ld, idx.data_ptr(), k, N.hp(h), dim,
               sh.data_ptr() if sh is not None else 0, out.data_ptr(), ld_out, _stream())
        return out[:, :k]

    def pack_pos(self, store, idx, shift):
        return self._gather(store.pos, store.ld, idx, shift).contiguous()

    def provenance(self, n_local, me, idx, dim, sh, prov, o_rank, o_root, o_sh, ld_o):
        """Provenance of one entry's copies (tmd_ghost_provenance) into the o_* views."""
        k = idx.numel()
        N.call("tmd_ghost_provenance", n_local, me, k, idx.data_ptr(), dim, sh.data_ptr(), prov.rank.data_ptr(),
               prov.root.data_ptr(), prov.sh.data_ptr(), prov.sh.stride(0), o_rank.data_ptr(), o_root.data_ptr(),
               o_sh.data_ptr(), ld_o, _stream())

    def pack_pos_prov(self, store, idx, shift, n_local, me, dim, sh, prov):
        """Border packet with provenance rows: (x, y, z, rank, root, s0, s1, s2) per copy."""
        k = idx.numel()
        out = torch.empty((8, max(k, 1)), dtype=torch.float64, device=store.device)
        self._gather(store.pos, store.ld, idx, shift, out=out, ld_out=out.stride(0))
        ids = torch.empty((2, max(k, 1)), dtype=torch.int32, device=store.device)
        self.provenance(n_local, me, idx, dim, sh, prov, ids[0], ids[1], out[5:], out.stride(0))
        out[3:5] = ids.to(torch.float64)
        return out[:, :k].contiguous()

    def borders_direct(self, store, slab, r, ext):
        """All-self borders in one pass (tmd_borders_count / _fill): returns (root, sh)."""
        n = store.n_local
        thr_hi = N.host_f64([float(h) - r for h in slab.hi])
        thr_lo = N.host_f64([float(lo) + r for lo in slab.lo])
        s_hi, s_lo = N.host_f64([-float(e) for e in ext]), N.host_f64([float(e) for e in ext])
        off = torch.empty(n + 1, dtype=torch.int32, device=store.device)
        N.call("tmd_borders_count", store.pos.data_ptr(), store.ld, n, N.hp(thr_hi), N.hp(thr_lo), off.data_ptr(),
               _stream())
        k = int(off[n].item())
        store.ensure_capacity(n + k)
        root = torch.empty(max(k, 1), dtype=torch.int32, device=store.device)
        sh = torch.empty((3, max(k, 1)), dtype=torch.float64, device=store.device)
        es = 8  # element size: the ghost region starts n_local columns into each row
        N.call("tmd_borders_fill", store.pos.data_ptr(), store.ld, n, N.hp(thr_hi), N.hp(thr_lo), N.hp(s_hi),
               N.hp(s_lo), 0, off.data_ptr(), store.pos.data_ptr() + es * n, store.ld,
               store.vel.data_ptr() + es * n, root.data_ptr(), sh.data_ptr(), sh.stride(0), 0, _stream())
        store.n_ghost = k
        store.set_ghost_segments([0], [k])
        return root[:k], sh[:, :k]

    def borders_direct_dev(self, store, slab, r, ext, room: int, launch: bool = True):
        """borders_direct without the count read-back: copies are written into
        the ghost region up to ``room`` slots; returns (root (room), sh (3, room),
        off) with the copy count at off[n_local] on the device.  The caller
        compares it with ``room`` once it reads it, and only then sets the
        store's ghost count."""
        n, dev = store.n_local, store.device
        thr_hi = N.host_f64([float(h) - r for h in slab.hi])
        thr_lo = N.host_f64([float(lo) + r for lo in slab.lo])
        s_hi, s_lo = N.host_f64([-float(e) for e in ext]), N.host_f64([float(e) for e in ext])
        buf = getattr(self, "_bdev", None)
        need = (n + 1) + room
        if buf is None or buf[0].numel() < need or buf[1].shape[1] < max(room, 1) or buf[0].device != dev:
            cap = int(need * 1.05) + 1024
            buf = self._bdev = (torch.empty(cap, dtype=torch.int32, device=dev),
                                torch.empty((3, int(max(room, 1) * 1.05) + 1024), dtype=torch.float64, device=dev))
        off = buf[0][: n + 1]
        root = buf[0][n + 1: n + 1 + room]
        sh = buf[1]
        if not launch:  # the buffers only (tmd_epoch_p1 fills them)
            return root, sh, off
        N.call("tmd_borders_count", store.pos.data_ptr(), store.ld, n, N.hp(thr_hi), N.hp(thr_lo), off.data_ptr(),
               _stream())
        es = 8  # element size: the ghost region starts n_local columns into each row
        N.call("tmd_borders_fill_capped", store.pos.data_ptr(), store.ld, n, N.hp(thr_hi), N.hp(thr_lo), N.hp(s_hi),
               N.hp(s_lo), 0, off.data_ptr(), store.pos.data_ptr() + es * n, store.ld,
               store.vel.data_ptr() + es * n, root.data_ptr(), sh.data_ptr(), sh.stride(0), 0, room, _stream())
        return root, sh, off

    def exchange_classify_dev(self, store, slab, s_hi, s_lo, geom):
        """Direct exchange classification (tmd_exchange_classify): wraps self
        dimensions and applies edge shifts in place; returns (dest, keep, leave,
        counts) with counts = [n_keep, n_leave] on the device."""
        n, dev = store.n_local, store.device
        lo, hi = N.host_f64(slab.lo), N.host_f64(slab.hi)
        # persistent buffers (7 n + 4 int32, 5% headroom): no allocation per epoch
        need = 7 * max(n, 1) + 4
        buf = getattr(self, "_xbuf", None)
        if buf is None or buf.numel() < need or buf.device != dev:
            buf = self._xbuf = torch.empty(int(need * 1.05) + 1024, dtype=torch.int32, device=dev)
        m = max(n, 1)
        dest, keep, leave = buf[:m], buf[m:2 * m], buf[2 * m:3 * m]
        cnt = buf[3 * m:3 * m + 2]
        scratch = buf[3 * m + 2:]
        N.call("tmd_exchange_classify", store.pos.data_ptr(), store.ld, n, N.hp(lo), N.hp(hi), N.hp(s_hi),
               N.hp(s_lo), N.hp(geom), dest.data_ptr(), keep.data_ptr(), leave.data_ptr(), cnt.data_ptr(),
               scratch.data_ptr(), _stream())
        return dest, keep, leave, cnt

    def exchange_classify(self, store, slab, s_hi, s_lo, geom):
        """exchange_classify_dev with the counts read back: (dest, keep, leave, n_keep, n_leave)."""
        dest, keep, leave, cnt = self.exchange_classify_dev(store, slab, s_hi, s_lo, geom)
        nk, nl = (int(v) for v in cnt.cpu().tolist())
        return dest, keep, leave, nk, nl

    def borders_records(self, store, thr_hi, thr_lo, s_hi, s_lo, geom):
        """Every border copy of every local (tmd_borders_count / _fill): returns
        (M, positions (3, M), root (M), recorded shifts (3, M), destination rank (M))."""
        n, dev = store.n_local, store.device
        off = torch.empty(n + 1, dtype=torch.int32, device=dev)
        N.call("tmd_borders_count", store.pos.data_ptr(), store.ld, n, N.hp(thr_hi), N.hp(thr_lo), off.data_ptr(),
               _stream())
        M = int(off[n].item())
        rec = torch.empty((3, max(M, 1)), dtype=torch.float64, device=dev)
        sh = torch.empty((3, max(M, 1)), dtype=torch.float64, device=dev)
        root = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        dest = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
        N.call("tmd_borders_fill", store.pos.data_ptr(), store.ld, n, N.hp(thr_hi), N.hp(thr_lo), N.hp(s_hi),
               N.hp(s_lo), N.hp(geom), off.data_ptr(), rec.data_ptr(), rec.stride(0), 0, root.data_ptr(),
               sh.data_ptr(), sh.stride(0), dest.data_ptr(), _stream())
        return M, rec[:, :M], root[:M], sh[:, :M], dest[:M]

    # -- direct-protocol bookkeeping (library kernels; no host sorts) ---------
    def group_by_rank(self, rank: torch.Tensor, ids, P: int):
        """Stable grouping of records by destination rank (tmd_group_by_rank):
        (ids in group order, their ranks, per-rank counts as a device tensor).
        Records with a rank outside [0, P) (e.g. -1: stays) drop out."""
        m = int(rank.numel())
        dev = rank.device
        out_ids = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        out_rank = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        counts = torch.empty(P, dtype=torch.int32, device=dev)
        N.call("tmd_group_by_rank", rank.data_ptr() if m else 0, ids.data_ptr() if ids is not None and m else 0, m, P,
               out_ids.data_ptr(), out_rank.data_ptr(), counts.data_ptr(), _stream())
        return out_ids[:m], out_rank[:m], counts

    def gather_i32(self, src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
        k = int(idx.numel())
        out = torch.empty(max(k, 1), dtype=torch.int32, device=idx.device)
        N.call("tmd_gather_i32", src.data_ptr(), idx.data_ptr(), k, out.data_ptr(), _stream())
        return out[:k]

    def pack_rows(self, pos: torch.Tensor, vel, ld: int, idx: torch.Tensor, width: int) -> torch.Tensor:
        """(k, width) rows (x[, v]) of records idx from SoA blocks with leading dimension ld."""
        k = int(idx.numel())
        rows = torch.empty((max(k, 1), width), dtype=torch.float64, device=idx.device)
        N.call("tmd_pack_rows", pos.data_ptr(), vel.data_ptr() if vel is not None else 0, ld, idx.data_ptr(), k,
               width, rows.data_ptr(), _stream())
        return rows[:k]

    def unpack_rows(self, store, rows: torch.Tensor, at: int) -> None:
        """Received rows into the store at slots [at, at + k) (width 3: ghosts, v = 0)."""
        k, width = int(rows.shape[0]), int(rows.shape[1])
        N.call("tmd_unpack_rows", rows.data_ptr(), k, width, store.pos.data_ptr(), store.vel.data_ptr(), store.ld,
               int(at), _stream())

    def gather_cols(self, src: torch.Tensor, idx: torch.Tensor) -> torch.Tensor:
        """(3, k) columns idx of a (3, ld) block."""
        return self._gather(src, src.stride(0), idx, _ZERO3)

    def border_slots(self, rank: torch.Tensor, base) -> torch.Tensor:
        m = int(rank.numel())
        slot = torch.empty(max(m, 1), dtype=torch.int32, device=rank.device)
        h = np.ascontiguousarray(np.asarray(base, dtype=np.int64))
        N.call("tmd_border_slots", rank.data_ptr(), m, int(h.size), N.hp(h), slot.data_ptr(), _stream())
        return slot[:m]

    def pack_pos_vel(self, store, idx, shift):
        k = idx.numel()
        out = torch.empty((6, max(k, 1)), dtype=torch.float64, device=store.device)
        self._gather(store.pos, store.ld, idx, shift, out=out, ld_out=out.stride(0))
        self._gather(store.vel, store.ld, idx, _ZERO3, out=out[3:], ld_out=out.stride(0))
        return out[:, :k].contiguous()

    def compact_locals_swap(self, store, keep_idx):
        """Production path: gather the kept locals' x and v into the store's
        alternate buffers and swap them in -- no allocation (forces are
        recomputed after every epoch, so F is not carried)."""
        k = keep_idx.numel()
        if k == store.n_local:
            return
        for name in ("pos", "vel"):
            cur, alt = getattr(store, name), getattr(store, name + "_alt")
            if alt is None or alt.shape != cur.shape:
                alt = torch.empty_like(cur)
            self._gather(cur, store.ld, keep_idx, _ZERO3, out=alt, ld_out=alt.stride(0))
            setattr(store, name, alt)
            setattr(store, name + "_alt", cur)
        store.n_local = k

    def compact_locals(self, store, keep_idx):
        """Order-preserving compaction of the locals to keep_idx (particles.py:117-132)."""
        k = keep_idx.numel()
        if k == store.n_local:
            return
        for name in ("pos", "vel", "frc"):
            t = getattr(store, name)
            tmp = self._gather(t, store.ld, keep_idx, _ZERO3).clone()
            t[:, :k] = tmp
        store.n_local = k

    def wrap_self(self, store, d, hi, lo, s_plus, s_minus):
        N.call("tmd_wrap_self", store.pos.data_ptr(), store.ld, store.n_local, d, float(hi), float(lo),
               float(s_plus), float(s_minus), _stream())

    def check_owned_deferred(self, store, slab, status) -> None:
        """Ownership check into a caller's status word (read later with the epoch's other checks)."""
        lo, hi = N.host_f64(slab.lo), N.host_f64(slab.hi)
        N.call("tmd_check_owned", store.pos.data_ptr(), store.ld, store.n_local, N.hp(lo), N.hp(hi),
               status.ptr, _stream())

    def any_outside(self, store, slab) -> bool:
        if getattr(self, "_status", None) is None or self._status.t.device != store.device:
            self._status = DeviceStatus(store.device)
        st = self._status
        st.reset()
        lo, hi = N.host_f64(slab.lo), N.host_f64(slab.hi)
        N.call("tmd_check_owned", store.pos.data_ptr(), store.ld, store.n_local, N.hp(lo), N.hp(hi),
               st.ptr, _stream())
        return N.decode_status(st.read())[0] != N.OK

    def plan_shift(self, store, idx, d, s):
        k = idx.numel()
        sh = torch.empty(max(k, 1), dtype=torch.float64, device=store.device)
        N.call("tmd_plan_shift", store.pos.data_ptr(), store.ld, idx.data_ptr(), k, d, float(s),
               sh.data_ptr(), _stream())
        return sh[:k]

    def append_ghosts_shifted(self, store, idx, shift, peer=0) -> int:
        k = idx.numel()
        start = store.n_total
        store.ensure_capacity(start + k)
        if k:
            self._gather(store.pos, store.ld, idx, shift, out=store.pos[:, start:], ld_out=store.ld)
            store.vel[:, start:start + k] = 0.0
            store.frc[:, start:start + k] = 0.0
        store.n_ghost += k
        store.ghost_peer = np.concatenate([store.ghost_peer, np.full(k, peer, dtype=np.int32)])
        store.ghost_ordinal = np.concatenate([store.ghost_ordinal, np.arange(k, dtype=np.int32)])
        return start

    def gather_into_ghosts(self, store, s):
        self._gather(store.pos, store.ld, s.idx, _ZERO3, dim=s.dim, sh=s.sh,
                     out=store.pos[:, s.ghost_start:], ld_out=store.ld)

    def pack_sync(self, store, s):
        return self._gather(store.pos, store.ld, s.idx, _ZERO3, dim=s.dim, sh=s.sh).contiguous()

    def flatten_plan(self, store, plan):
        """Root local + summed shift of every ghost when all entries are self (P = 1)."""
        ng, nl = store.n_ghost, store.n_local
        src = torch.empty(max(ng, 1), dtype=torch.int32, device=store.device)
        fsh = torch.zeros((3, max(ng, 1)), dtype=torch.float64, device=store.device)
        for sends, recvs in plan.rounds:
            if recvs:
                raise ProtocolError("flattened sync needs an all-self plan")
            for s in sends:
                k = s.idx.numel()
                N.call("tmd_flatten_round", nl, s.ghost_start, k, s.idx.data_ptr(), s.dim,
                       s.sh.data_ptr(), src.data_ptr(), fsh.data_ptr(), fsh.stride(0), _stream())
        return src, fsh

    def sync_flat(self, store, plan):
        ng = plan.n_ghost
        N.call("tmd_sync_flat", store.pos.data_ptr(), store.ld, store.n_local, ng,
               plan.flat_src.data_ptr(), plan.flat_sh.data_ptr(), _stream())
