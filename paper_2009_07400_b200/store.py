"""Device-resident particle store (reference: ParticleStore, particles.py:30-158).

Three SoA fp64 blocks of shape (3, capacity) in HBM — positions, velocities,
forces — with locals in [0, n_local) and ghosts in [n_local, n_total), the
reference's contiguous local/ghost regions.  Capacity grows as the reference
does (x1.5 + 8, particles.py:27, 52-58).  Accessors that return numpy arrays
(``local_positions()`` etc.) copy device -> host; the step loop never calls
them.

torch supplies the allocations only; every kernel that touches the data is
in libtinymd_b200.so.
"""

from __future__ import annotations

import numpy as np
import torch

_GROWTH = 1.5

__all__ = ["ParticleStore", "device_of"]


def device_of(device=None) -> torch.device:
    if device is None:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2009_07400_b200 needs a CUDA device (B200); there is no CPU path")
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def _to_soa(a, device) -> torch.Tensor:
    """(k, 3) host or device array -> (3, k) fp64 device tensor."""
    if isinstance(a, torch.Tensor):
        t = a.to(device=device, dtype=torch.float64)
        return t.t().contiguous() if t.dim() == 2 and t.shape[-1] == 3 else t
    arr = np.ascontiguousarray(np.atleast_2d(np.asarray(a, dtype=np.float64)).T)
    return torch.from_numpy(arr).to(device)


class ParticleStore:
    """Positions, velocities and forces of one rank, SoA fp64 on the GPU."""

    def __init__(self, capacity: int = 1, device=None, layout=None):
        self.device = device_of(device)
        self.layout = layout  # accepted for API compatibility (layout.py); ignored
        cap = max(int(capacity), 1)
        self.pos = torch.zeros((3, cap), dtype=torch.float64, device=self.device)
        self.vel = torch.zeros((3, cap), dtype=torch.float64, device=self.device)
        self.frc = torch.zeros((3, cap), dtype=torch.float64, device=self.device)
        self.pos_alt = None  # second position buffer for the fused step kernel
        self.vel_alt = None  # scratch for the cell-order permutation
        self.n_local = 0
        self.n_ghost = 0
        self._ghost_peer = np.empty(0, dtype=np.int32)
        self._ghost_ordinal = np.empty(0, dtype=np.int32)
        self._ghost_segments = None

    # -- geometry of the buffers ---------------------------------------------
    # ghost bookkeeping of the reference (particles.py:141-155): source peer and
    # ordinal in that peer's message per ghost; the direct protocol records it
    # as (peer, count) segments and materialises the arrays only when read
    @property
    def ghost_peer(self) -> np.ndarray:
        self._materialise_ghosts()
        return self._ghost_peer

    @ghost_peer.setter
    def ghost_peer(self, v) -> None:
        self._ghost_segments = None
        self._ghost_peer = v

    @property
    def ghost_ordinal(self) -> np.ndarray:
        self._materialise_ghosts()
        return self._ghost_ordinal

    @ghost_ordinal.setter
    def ghost_ordinal(self, v) -> None:
        self._ghost_segments = None
        self._ghost_ordinal = v

    def set_ghost_segments(self, peers, counts) -> None:
        self._ghost_segments = (np.asarray(peers, dtype=np.int32), np.asarray(counts, dtype=np.int64))

    def _materialise_ghosts(self) -> None:
        if self._ghost_segments is None:
            return
        peers, counts = self._ghost_segments
        self._ghost_segments = None
        self._ghost_peer = np.repeat(peers, counts).astype(np.int32)
        self._ghost_ordinal = (np.concatenate([np.arange(c, dtype=np.int32) for c in counts])
                               if counts.sum() else np.empty(0, dtype=np.int32))

    @property
    def capacity(self) -> int:
        return self.pos.shape[1]

    @property
    def ld(self) -> int:
        return self.pos.stride(0)

    @property
    def n_total(self) -> int:
        return self.n_local + self.n_ghost

    def ensure_capacity(self, needed: int) -> None:
        if needed <= self.capacity:
            return
        new_cap = max(int(needed), int(self.capacity * _GROWTH) + 8)
        n = self.n_total
        for name in ("pos", "vel", "frc"):
            old = getattr(self, name)
            new = torch.zeros((3, new_cap), dtype=torch.float64, device=self.device)
            new[:, :n] = old[:, :n]
            setattr(self, name, new)
        self.pos_alt = None
        self.vel_alt = None

    def swap_positions(self) -> None:
        """Make the freshly drifted buffer current (ghost slots are refilled by the next sync)."""
        self.pos, self.pos_alt = self.pos_alt, self.pos

    # -- host views (D2H copies) ---------------------------------------------
    def _rows(self, t, start, count) -> np.ndarray:
        return t[:, start:start + count].t().contiguous().cpu().numpy()

    def local_positions(self) -> np.ndarray:
        return self._rows(self.pos, 0, self.n_local)

    def all_positions(self) -> np.ndarray:
        return self._rows(self.pos, 0, self.n_total)

    def local_velocities(self) -> np.ndarray:
        return self._rows(self.vel, 0, self.n_local)

    def all_velocities(self) -> np.ndarray:
        return self._rows(self.vel, 0, self.n_total)

    def local_forces(self) -> np.ndarray:
        return self._rows(self.frc, 0, self.n_local)

    def local_state(self, out=None) -> np.ndarray:
        """(n_local, 6) positions then velocities: one device-side transpose, one D2H.

        ``out``: a caller-owned (n_local, 6) float64 C-contiguous array or host
        tensor (a pinned tensor makes the copy one DMA); default: a pinned
        buffer from torch's host caching allocator."""
        k = self.n_local
        # (k, 6) rows assembled in a persistent device buffer (no allocation per call)
        stage = getattr(self, "_state_stage", None)
        if stage is None or stage.shape[0] < k or stage.device != self.device:
            stage = self._state_stage = torch.empty((int(k * 1.05) + 1024, 6), dtype=torch.float64,
                                                    device=self.device)
        dev = stage[:k]
        dev[:, 0:3] = self.pos[:, :k].t()
        dev[:, 3:6] = self.vel[:, :k].t()
        if out is None:
            host = torch.empty((k, 6), dtype=torch.float64, pin_memory=True)
            host.copy_(dev)
            return host.numpy()
        if isinstance(out, torch.Tensor):  # e.g. a pinned host tensor: one DMA
            if tuple(out.shape) != (k, 6) or out.dtype != torch.float64 or out.device.type != "cpu":
                raise ValueError(f"out must be a float64 host tensor of shape ({k}, 6)")
            out.copy_(dev, non_blocking=True)
            torch.cuda.current_stream(dev.device).synchronize()
            return out.numpy()
        if out.shape != (k, 6) or out.dtype != np.float64 or not out.flags["C_CONTIGUOUS"]:
            raise ValueError(f"out must be a C-contiguous float64 array of shape ({k}, 6)")
        torch.from_numpy(out).copy_(dev)
        return out

    @classmethod
    def from_host(cls, pos, vel, capacity: int | None = None, device=None) -> "ParticleStore":
        """A store whose locals are host (k, 3) arrays: two H2D copies straight from
        the caller's arrays (the driver stages pageable memory itself, faster than
        interleaving into a pinned buffer on the host), SoA transpose on device."""
        pos = np.ascontiguousarray(pos, dtype=np.float64)
        vel = np.ascontiguousarray(vel, dtype=np.float64)
        k = pos.shape[0]
        st = cls(capacity or max(2 * k, 16), device=device)
        if k:
            st.pos[:, :k] = torch.from_numpy(pos).to(st.device).t()
            st.vel[:, :k] = torch.from_numpy(vel).to(st.device).t()
        st.n_local = k
        return st

    # -- editing (particles.py:83-158) ----------------------------------------
    def append_locals(self, pos, vel) -> None:
        p = _to_soa(pos, self.device)
        v = _to_soa(vel, self.device)
        k = p.shape[1]
        if k == 0:
            return
        self.ensure_capacity(self.n_total + k)
        nl, ng = self.n_local, self.n_ghost
        if ng:
            # slide the ghost block right so it stays contiguous after the locals
            for t in (self.pos, self.vel, self.frc):
                t[:, nl + k:nl + k + ng] = t[:, nl:nl + ng].clone()
        self.pos[:, nl:nl + k] = p
        self.vel[:, nl:nl + k] = v
        self.frc[:, nl:nl + k] = 0.0
        self.n_local += k

    def compact_locals(self, keep) -> None:
        """Drop locals where keep is False, survivors keep their order (particles.py:117-132)."""
        if self.n_ghost:
            raise RuntimeError("compact_locals requires an empty ghost region")
        keep = torch.as_tensor(np.asarray(keep, dtype=bool), device=self.device)
        if keep.shape != (self.n_local,):
            raise ValueError("keep mask must cover exactly the local region")
        idx = torch.nonzero(keep).flatten()
        k = idx.numel()
        for t in (self.pos, self.vel, self.frc):
            t[:, :k] = t[:, idx]
        self.n_local = k

    def clear_ghosts(self) -> None:
        self.n_ghost = 0
        self.ghost_peer = np.empty(0, dtype=np.int32)
        self.ghost_ordinal = np.empty(0, dtype=np.int32)

    def append_ghosts(self, pos, peer: int = 0) -> int:
        """Append ghost copies (v = F = 0, particles.py:141-155); returns the first slot."""
        p = _to_soa(pos, self.device)
        k = p.shape[1]
        start = self.n_total
        self.ensure_capacity(start + k)
        self.pos[:, start:start + k] = p
        self.vel[:, start:start + k] = 0.0
        self.frc[:, start:start + k] = 0.0
        self.ghost_peer = np.concatenate([self.ghost_peer, np.full(k, peer, dtype=np.int32)])
        self.ghost_ordinal = np.concatenate([self.ghost_ordinal, np.arange(k, dtype=np.int32)])
        self.n_ghost += k
        return start

    def set_ghost_positions(self, start: int, pos) -> None:
        p = _to_soa(pos, self.device)
        self.pos[:, start:start + p.shape[1]] = p
