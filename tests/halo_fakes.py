"""Test double for the device halo primitives (paper_2009_07400_b200.halo_ops).

CPU torch-tensor implementations of the same methods, so the host-side halo
protocol (rounds, entry order, counts-then-payload messaging, plan
bookkeeping) can be exercised with world_size > 1 over gloo on a machine
without a GPU.  Test infrastructure only; the product never imports it.
"""

from __future__ import annotations

import numpy as np
import torch


class CpuHaloOps:
    GE, LT, GT, IN = 0, 1, 2, 3

    def count_device(self):
        return torch.device("cpu")

    def empty(self, shape, store):
        return torch.empty(shape, dtype=torch.float64)

    def select(self, row, n, kind, thr, thr2=0.0):
        x = row[:n]
        m = {0: x >= thr, 1: x < thr, 2: x > thr, 3: (x >= thr) & (x < thr2)}[kind]
        return torch.nonzero(m).flatten().to(torch.int32)

    def select_pair(self, row, n, a, b):
        return self.select(row, n, a[0], a[1]), self.select(row, n, b[0], b[1])

    def emit_ghosts(self, store, idx, shift, dim, peer=0):
        sh = self.plan_shift(store, idx, dim, shift[dim])
        return self.append_ghosts_shifted(store, idx, shift, peer), sh

    def _gather(self, t, idx, shift):
        s = torch.as_tensor(np.asarray(shift, dtype=np.float64))[:, None]
        return t[:, idx.long()] + s

    def pack_pos(self, store, idx, shift):
        return self._gather(store.pos, idx, shift).contiguous()

    def pack_pos_vel(self, store, idx, shift):
        return torch.cat([self._gather(store.pos, idx, shift), store.vel[:, idx.long()]]).contiguous()

    def compact_locals(self, store, keep_idx):
        k = keep_idx.numel()
        for t in (store.pos, store.vel, store.frc):
            t[:, :k] = t[:, keep_idx.long()].clone()
        store.n_local = k

    def wrap_self(self, store, d, hi, lo, sp, sm):
        x = store.pos[d, :store.n_local]
        up, down = x >= hi, x < lo
        x[up] = x[up] + sp
        x[down & ~up] = x[down & ~up] + sm

    def any_outside(self, store, slab):
        p = store.pos[:, :store.n_local].t().numpy()
        return bool((~slab.contains(p)).any()) if p.shape[0] else False

    def plan_shift(self, store, idx, d, s):
        x = store.pos[d, idx.long()]
        return (x + s) - x

    def append_ghosts_shifted(self, store, idx, shift, peer=0):
        return store.append_ghosts(self._gather(store.pos, idx, shift).t(), peer=peer)

    def _sync_data(self, store, s):
        shift = torch.zeros((3, s.idx.numel()), dtype=torch.float64)
        shift[s.dim] = s.sh
        return store.pos[:, s.idx.long()] + shift

    def gather_into_ghosts(self, store, s):
        k = s.idx.numel()
        store.pos[:, s.ghost_start:s.ghost_start + k] = self._sync_data(store, s)

    def pack_sync(self, store, s):
        return self._sync_data(store, s).contiguous()

    def flatten_plan(self, store, plan):
        return None, None

    def sync_flat(self, store, plan):
        raise AssertionError("not used with flat_src None")

    # -- direct protocol (production path at P > 1), same semantics as
    #    tmd_exchange_classify / tmd_borders_count / tmd_borders_fill
    @staticmethod
    def _rank(geom, o):
        c, g = geom[:3], geom[3:]
        x, y, z = ((int(c[d]) + o[d]) % int(g[d]) for d in range(3))
        return (z * int(g[1]) + y) * int(g[0]) + x

    # direct-protocol bookkeeping (the device library's grouping/packing)
    def group_by_rank(self, rank, ids, P):
        """Records with rank < 0 drop out (as in tmd_group_by_rank)."""
        r = rank.to(torch.int64)
        sel = torch.nonzero(r >= 0).flatten()
        order = sel[torch.sort(r[sel], stable=True).indices]
        out_ids = (ids[order] if ids is not None else order).to(torch.int32)
        return out_ids, rank[order].to(torch.int32), torch.bincount(r[sel], minlength=P).to(torch.int32)

    def exchange_classify_dev(self, store, slab, s_hi, s_lo, geom):
        dest, keep, leave, nk, nl = self.exchange_classify(store, slab, s_hi, s_lo, geom)
        return dest, keep, leave, torch.tensor([nk, nl], dtype=torch.int32)

    def gather_i32(self, src, idx):
        return src[idx.long()].to(torch.int32)

    def pack_rows(self, pos, vel, ld, idx, width):
        j = idx.long()
        parts = [pos[:3, j]] + ([vel[:3, j]] if width == 6 else [])
        return torch.cat(parts).t().contiguous()

    def unpack_rows(self, store, rows, at):
        k = rows.shape[0]
        store.pos[:, at:at + k] = rows[:, 0:3].t()
        store.vel[:, at:at + k] = rows[:, 3:6].t() if rows.shape[1] == 6 else 0.0

    def gather_cols(self, src, idx):
        return src[:3, idx.long()].clone()

    def border_slots(self, rank, base):
        b = torch.as_tensor(np.asarray(base, dtype=np.int64))
        return (b[rank.long()] + torch.arange(rank.numel(), dtype=torch.int64)).to(torch.int32)

    def exchange_classify(self, store, slab, s_hi, s_lo, geom):
        n = store.n_local
        dest = torch.full((max(n, 1),), -1, dtype=torch.int32)
        for i in range(n):
            o, moved = [0, 0, 0], False
            for d in range(3):
                x = float(store.pos[d, i])
                if x >= slab.hi[d]:
                    store.pos[d, i] = x + s_hi[d]
                    if geom[3 + d] > 1:
                        o[d], moved = 1, True
                elif x < slab.lo[d]:
                    store.pos[d, i] = x + s_lo[d]
                    if geom[3 + d] > 1:
                        o[d], moved = -1, True
            if moved:
                dest[i] = self._rank(geom, o)
        d = dest[:n]
        keep = torch.nonzero(d < 0).flatten().to(torch.int32)
        leave = torch.nonzero(d >= 0).flatten().to(torch.int32)
        return dest, keep, leave, int(keep.numel()), int(leave.numel())

    def borders_records(self, store, thr_hi, thr_lo, s_hi, s_lo, geom):
        recs, roots, shs, dests = [], [], [], []
        for i in range(store.n_local):
            x = [float(store.pos[d, i]) for d in range(3)]
            opts = []
            for d in range(3):
                o = [(0.0, 0)]
                if x[d] > thr_hi[d]:
                    o.append((s_hi[d], 1))
                if x[d] < thr_lo[d]:
                    o.append((s_lo[d], -1))
                opts.append(o)
            for a, oa in enumerate(opts[0]):
                for b, ob in enumerate(opts[1]):
                    for c, oc in enumerate(opts[2]):
                        if a == b == c == 0:
                            continue
                        sel = (a, b, c)
                        e, r = [], []
                        for d, (s, _) in enumerate((oa, ob, oc)):
                            if sel[d]:
                                v = np.float64(x[d]) + np.float64(s)
                                e.append(v)
                                r.append(v - np.float64(x[d]))
                            else:
                                e.append(x[d])
                                r.append(0.0)
                        recs.append(e)
                        shs.append(r)
                        roots.append(i)
                        dests.append(self._rank(geom, (oa[1], ob[1], oc[1])))
        M = len(roots)
        rec = torch.tensor(np.asarray(recs, dtype=np.float64).reshape(M, 3).T.copy())
        sh = torch.tensor(np.asarray(shs, dtype=np.float64).reshape(M, 3).T.copy())
        return (M, rec, torch.tensor(roots, dtype=torch.int32), sh, torch.tensor(dests, dtype=torch.int32))

