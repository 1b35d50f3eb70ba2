"""Space-filling-curve load balancing (the paper's §5 / §6.3).

The reference ships no ``balance`` module; its
``block_neighborhood_pattern`` (comm.py:277-332) consumes one.  This module
is that balancer, with the particle-side work on the device:

* ``sfc_keys`` -- every particle's Morton or Hilbert key at the forest's
  maximum depth (tmd_sfc_keys: integer bit work per particle);
* ``BlockForest`` -- an octree of blocks over the global box, refined where a
  block's weight exceeds ``refine_threshold`` and merged where a complete
  octet weighs less than ``merge_threshold``; per-block weights are counts of
  local (computational) and ghost (communication) particles per leaf
  (tmd_leaf_counts: leaves are contiguous key ranges of either curve);
* ``partition`` -- the leaves in curve order, split greedily into P
  contiguous segments of cumulative weight ~W / P;
* ``block_neighbors`` -- the neighbour table of comm.py:277-332: ranks owning
  a block within ``spacing`` (max-norm, periodic images) of an owned block;
* ``migrate`` -- particles regrouped by the owner of their block (the global
  multiset is preserved).

The production decomposition of the GPU path is the reference's six-stencil
slab grid (comm.py:171-274); the balancer computes a partition and moves
particles between ranks but the step kernels still run on slabs (a
block-list ownership test in the exchange/borders kernels is not built).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from .neighbor import _stream

__all__ = ["MORTON", "HILBERT", "morton_key", "hilbert_key", "sfc_keys", "Block", "BlockForest", "partition",
           "block_neighbors", "migrate", "rank_weights"]

MORTON, HILBERT = 0, 1
_CURVES = {"morton": MORTON, "hilbert": HILBERT}

N.lib.tmd_morton_key.restype = C.c_uint64
N.lib.tmd_morton_key.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int32]
N.lib.tmd_hilbert_key.restype = C.c_uint64
N.lib.tmd_hilbert_key.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_int32]


def _curve(curve) -> int:
    return _CURVES[curve] if isinstance(curve, str) else int(curve)


def morton_key(ix: int, iy: int, iz: int, depth: int) -> int:
    """Bit-interleaved key, x in the least significant position of each triad."""
    return int(N.lib.tmd_morton_key(ix, iy, iz, depth))


def hilbert_key(ix: int, iy: int, iz: int, depth: int) -> int:
    """3-D Hilbert index (Skilling's transpose construction)."""
    return int(N.lib.tmd_hilbert_key(ix, iy, iz, depth))


def key_of(cell, depth: int, curve) -> int:
    return (morton_key if _curve(curve) == MORTON else hilbert_key)(int(cell[0]), int(cell[1]), int(cell[2]), depth)


def sfc_keys(pos: torch.Tensor, ld: int, n: int, lo, hi, depth: int, curve) -> torch.Tensor:
    """uint64 (as int64) keys of n particles of a (3, ld) SoA block at the given depth."""
    width = (np.asarray(hi, dtype=np.float64) - np.asarray(lo, dtype=np.float64)) / float(1 << depth)
    keys = torch.empty(max(n, 1), dtype=torch.int64, device=pos.device)
    N.call("tmd_sfc_keys", pos.data_ptr(), ld, n, N.hp(N.host_f64(lo)), N.hp(N.host_f64(width)), depth,
           _curve(curve), keys.data_ptr(), _stream())
    return keys[:n]


@dataclass
class Block:
    level: int
    cell: tuple  # block coordinates at its level
    key: int = 0  # first key of its range at the forest's max depth
    comp: int = 0  # computational weight: local particles inside
    comm: int = 0  # communication weight: ghosts inside
    owner: int = 0

    @property
    def weight(self) -> int:
        return self.comp + self.comm


@dataclass
class BlockForest:
    """Octree leaves over the global box [lo, hi)."""

    lo: np.ndarray
    hi: np.ndarray
    max_depth: int = 6
    refine_threshold: int = 800
    merge_threshold: int = 100
    curve: str = "hilbert"
    leaves: list = field(default_factory=list)

    def __post_init__(self):
        self.lo = np.asarray(self.lo, dtype=np.float64)
        self.hi = np.asarray(self.hi, dtype=np.float64)
        if not self.merge_threshold < self.refine_threshold:
            raise ValueError("merge_threshold must be below refine_threshold")
        if not self.leaves:
            self.leaves = [Block(0, (0, 0, 0))]
        self._order()

    # -- geometry ----------------------------------------------------------------
    def aabb(self, b: Block):
        w = (self.hi - self.lo) / float(1 << b.level)
        lo = self.lo + w * np.asarray(b.cell, dtype=np.float64)
        return lo, lo + w

    def _order(self):
        D = self.max_depth
        for b in self.leaves:
            s = D - b.level
            b.key = key_of([c << s for c in b.cell], D, self.curve) >> (3 * s) << (3 * s)
        self.leaves.sort(key=lambda b: b.key)

    # -- weights ---------------------------------------------------
    def compute_weights(self, pos: torch.Tensor, ld: int, n_local: int, n_total: int | None = None) -> None:
        """Local / ghost particle counts per leaf, on the device."""
        n_total = n_local if n_total is None else n_total
        dev = pos.device
        starts = torch.tensor([b.key for b in self.leaves], dtype=torch.int64, device=dev)
        counts = torch.empty((2, len(self.leaves)), dtype=torch.int32, device=dev)
        for row, (a, z) in enumerate(((0, n_local), (n_local, n_total))):
            keys = sfc_keys(pos[:, a:], ld, z - a, self.lo, self.hi, self.max_depth, self.curve)
            N.call("tmd_leaf_counts", keys.data_ptr(), z - a, starts.data_ptr(), len(self.leaves),
                   counts[row].data_ptr(), _stream())
        c = counts.cpu().numpy()
        for b, comp, comm in zip(self.leaves, c[0], c[1]):
            b.comp, b.comm = int(comp), int(comm)

    # -- refine / merge ------------------------------------------
    def refine_and_merge(self, pos: torch.Tensor, ld: int, n_local: int, n_total: int | None = None,
                         max_rounds: int = 32) -> int:
        """Split heavy leaves into octants, collapse light complete octets, to a
        fixed point; returns the number of rounds that changed the forest."""
        changed = 0
        for _ in range(max_rounds):
            self.compute_weights(pos, ld, n_local, n_total)
            new, did = [], False
            for b in self.leaves:
                if b.weight > self.refine_threshold and b.level < self.max_depth:
                    did = True
                    for o in range(8):
                        c = tuple(2 * b.cell[d] + ((o >> d) & 1) for d in range(3))
                        new.append(Block(b.level + 1, c))
                else:
                    new.append(b)
            if not did:
                # merge complete octets whose total weight stays below the threshold
                groups = {}
                for b in new:
                    if b.level > 0:
                        groups.setdefault((b.level - 1, tuple(c >> 1 for c in b.cell)), []).append(b)
                merged = set()
                for (lvl, parent), kids in groups.items():
                    if len(kids) == 8 and all(k.level == lvl + 1 for k in kids) and \
                            sum(k.weight for k in kids) < self.merge_threshold:
                        merged.add((lvl, parent))
                if merged:
                    did = True
                    keep = [b for b in new if not (b.level > 0 and
                                                    (b.level - 1, tuple(c >> 1 for c in b.cell)) in merged)]
                    new = keep + [Block(lvl, parent) for lvl, parent in merged]
            self.leaves = new
            self._order()
            if not did:
                break
            changed += 1
        self.compute_weights(pos, ld, n_local, n_total)
        return changed


def partition(forest: BlockForest, P: int) -> np.ndarray:
    """Greedy prefix split of the curve-ordered leaves into P contiguous
    segments targeting ceil(W / P) each; sets owners and
    returns them."""
    w = np.array([b.weight for b in forest.leaves], dtype=np.float64)
    total = float(w.sum())
    owners = np.zeros(len(w), dtype=np.int64)
    if P > 1 and total > 0:
        # leaf t goes to the segment holding the midpoint of its weight interval
        mid = np.cumsum(w) - 0.5 * w
        quota = np.ceil(total / P)
        owners = np.minimum((mid // quota).astype(np.int64), P - 1)
        # keep segments contiguous and monotone (zero-weight leaves follow their left neighbour)
        owners = np.maximum.accumulate(owners)
    for b, o in zip(forest.leaves, owners):
        b.owner = int(o)
    return owners


def rank_weights(forest: BlockForest, P: int) -> np.ndarray:
    out = np.zeros(P, dtype=np.int64)
    for b in forest.leaves:
        out[b.owner] += b.weight
    return out


def _linf_gap(lo_a, hi_a, lo_b, hi_b) -> float:
    """Max-norm distance between two boxes (0 when they touch or overlap)."""
    return float(np.max(np.maximum(0.0, np.maximum(lo_b - hi_a, lo_a - hi_b))))


def block_neighbors(forest: BlockForest, rank: int, spacing: float) -> list:
    """comm.py:277-332: every rank owning a block within `spacing` (max-norm,
    periodic images of the global box) of a block owned by `rank`, with the
    blocks that qualify; a rank may neighbour itself across the boundary."""
    ext = forest.hi - forest.lo
    steps = np.array([-1.0, 0.0, 1.0])
    offsets = np.stack(np.meshgrid(steps, steps, steps, indexing="ij"), axis=-1).reshape(-1, 3) * ext
    mine = [forest.aabb(b) for b in forest.leaves if b.owner == rank]
    table = {}
    for b in forest.leaves:
        blo, bhi = forest.aabb(b)
        for off in offsets:
            if b.owner == rank and not np.any(off):
                continue
            if any(_linf_gap(mlo, mhi, blo + off, bhi + off) <= spacing for mlo, mhi in mine):
                table.setdefault(b.owner, []).append(b)
                break
    return sorted(table.items())


def migrate(forest: BlockForest, pos: np.ndarray, vel: np.ndarray, P: int):
    """Particles grouped by the owner of their leaf: a list
    of (pos, vel) per rank, each in the original relative order."""
    dev = torch.device("cuda", torch.cuda.current_device())
    p = torch.from_numpy(np.ascontiguousarray(np.asarray(pos, dtype=np.float64).T)).to(dev)
    keys = sfc_keys(p, p.stride(0), p.shape[1], forest.lo, forest.hi, forest.max_depth, forest.curve)
    starts = np.array([b.key for b in forest.leaves], dtype=np.int64)
    leaf = np.searchsorted(starts, keys.cpu().numpy(), side="right") - 1
    owner = np.array([b.owner for b in forest.leaves], dtype=np.int64)[leaf]
    return [(pos[owner == r], vel[owner == r]) for r in range(P)]
