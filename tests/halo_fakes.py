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
