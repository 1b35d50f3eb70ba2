"""Space-filling-curve balancing (paper_2009_07400_b200/balance.py): SPEC.md
acceptance criteria 7 (curve keys) and 8 (the half-diagonal DEM imbalance of
the paper's §6.3), the partition examples of SPEC.md:568-576 and the
block-neighbourhood table of comm.py:277-332."""

import itertools

import numpy as np
import pytest

from paper_2009_07400_b200 import balance as B


def _interleave(x, y, z, depth):
    k = 0
    for b in range(depth):
        k |= ((x >> b) & 1) << (3 * b) | ((y >> b) & 1) << (3 * b + 1) | ((z >> b) & 1) << (3 * b + 2)
    return k


def test_morton_keys_equal_bit_interleave_oracle():
    assert B.morton_key(0, 0, 0, 4) == 0
    assert (B.morton_key(1, 0, 0, 1), B.morton_key(0, 1, 0, 1), B.morton_key(0, 0, 1, 1)) == (1, 2, 4)
    keys = []
    for x, y, z in itertools.product(range(16), repeat=3):
        k = B.morton_key(x, y, z, 4)
        assert k == _interleave(x, y, z, 4)
        keys.append(k)
    assert sorted(keys) == list(range(4096))


def test_hilbert_bijective_face_adjacent_and_nested():
    for depth in (1, 2, 3, 4):
        side = 1 << depth
        cell_of = {}
        for c in itertools.product(range(side), repeat=3):
            cell_of[B.hilbert_key(*c, depth)] = c
        assert sorted(cell_of) == list(range(side ** 3))
        assert cell_of[0] == (0, 0, 0)
        for k in range(side ** 3 - 1):
            a, b = np.array(cell_of[k]), np.array(cell_of[k + 1])
            assert np.abs(a - b).sum() == 1, (depth, k)
    # every octree cube at level l is one contiguous key range (the forest relies on it)
    D = 4
    for lvl in (1, 2, 3):
        s = D - lvl
        for c in itertools.product(range(16), repeat=3):
            parent = tuple(v >> s for v in c)
            first = B.hilbert_key(*[v << s for v in parent], D) >> (3 * s)
            assert B.hilbert_key(*c, D) >> (3 * s) == first


class _Leaves:
    def __init__(self, w):
        self.leaves = [B.Block(1, (0, 0, 0), key=i, comp=int(v)) for i, v in enumerate(w)]


def _best_contiguous(w, P):
    best = float("inf")
    for cuts in itertools.combinations(range(1, len(w)), P - 1):
        b = [0, *cuts, len(w)]
        best = min(best, max(sum(w[b[i]:b[i + 1]]) for i in range(P)))
    return best


def test_partition_examples():
    f = _Leaves([5, 5, 5, 5])
    assert list(B.partition(f, 2)) == [0, 0, 1, 1]
    w = [8, 0, 0, 0, 8, 0, 0, 8]
    f = _Leaves(w)
    owners = B.partition(f, 3)
    seg = np.bincount(owners, weights=w, minlength=3)
    assert seg.max() <= 2 * np.mean(seg) and seg.max() <= _best_contiguous(w, 3)
    assert np.all(np.diff(owners) >= 0)  # contiguous along the curve
    assert list(B.partition(_Leaves(w), 1)) == [0] * 8
    # scale invariance
    g = _Leaves([3 * v for v in w])
    assert list(B.partition(g, 3)) == list(owners)


@pytest.mark.gpu
@pytest.mark.parametrize("curve", ["morton", "hilbert"])
def test_half_diagonal_dem_balance(curve):
    """SPEC.md acceptance 8: the diagonal half-filled DEM domain at P = 8 --
    slab decomposition max/mean rank weight >= 1.9, after balancing <= 1.3;
    migration preserves the particle multiset; device keys equal host keys."""
    import torch

    from paper_2009_07400_b200 import Decomposition, SimConfig, lattice_positions, lattice_velocities

    cfg = SimConfig(unit_cells=(24, 24, 24), potential_kind="sd", fill="half-diagonal", stiffness=0.0,
                    damping=0.0, diameter=1.2, cutoff=1.2)
    box = cfg.domain()
    pos = lattice_positions(cfg, box)
    vel = lattice_velocities(cfg, pos.shape[0])
    P = 8
    slab = np.array([int(Decomposition(box, P, r, cfg.interaction_radius()).owns(pos).sum()) for r in range(P)])
    assert slab.sum() == pos.shape[0] and slab.max() / slab.mean() >= 1.9
    forest = B.BlockForest(box.lo, box.hi, max_depth=6, refine_threshold=800, merge_threshold=100, curve=curve)
    dev = torch.device("cuda")
    p = torch.from_numpy(np.ascontiguousarray(pos.T)).to(dev)
    forest.refine_and_merge(p, p.stride(0), pos.shape[0])
    assert sum(b.weight for b in forest.leaves) == pos.shape[0]
    assert max(b.level for b in forest.leaves) >= 2
    B.partition(forest, P)
    w = B.rank_weights(forest, P)
    assert w.sum() == pos.shape[0] and w.max() / w.mean() <= 1.3, w
    parts = B.migrate(forest, pos, vel, P)
    assert [len(a) for a, _ in parts] == list(w)
    got = np.vstack([np.hstack([a, v]) for a, v in parts])
    want = np.hstack([pos, vel])
    assert np.array_equal(got[np.lexsort(got.T[::-1])], want[np.lexsort(want.T[::-1])])
    keys = B.sfc_keys(p, p.stride(0), 64, box.lo, box.hi, 6, curve).cpu().numpy()
    width = (box.hi - box.lo) / 64.0
    cells = np.clip(np.floor((pos[:64] - box.lo) / width).astype(np.int64), 0, 63)
    assert list(keys) == [B.key_of(c, 6, curve) for c in cells]
    # every rank's neighbour table holds only ranks owning blocks near its own
    for r in range(P):
        for peer, blocks in B.block_neighbors(forest, r, cfg.interaction_radius()):
            assert all(b.owner == peer for b in blocks)
