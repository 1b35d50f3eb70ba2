"""Cell binning and Verlet lists on the GPU (reference: neighbor.py:38-206).

Same call signatures, return types and errors as the reference:

    build_cell_grid(store, rank_aabb, r)                       -> CellGrid
    build_neighbor_lists(store, grid, r, half, list_layout=None,
                         initial_capacity=None)                -> NeighborLists
    max_displacement_since_rebuild(store, lists)               -> float

The work runs in libtinymd_b200.so (tmd_bin_cells, tmd_build_lists,
tmd_max_disp2).  The host-side views the reference exposes as numpy arrays
(``coords``, ``occupants``, ``counts``, ``as_matrix()``, ``pairs()``) are
materialised lazily by device -> host copies for inspection and tests.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _native as N
from .core import AABB
from .errors import ProtocolError
from .store import ParticleStore

__all__ = ["BrickIndex", "CellGrid", "NeighborLists", "build_cell_grid", "build_neighbor_lists",
           "max_displacement_since_rebuild", "initial_list_capacity"]


def _stream() -> int:
    """The calling thread's current CUDA stream on the current device (raw
    handle; the torch.cuda.current_stream() wrapper costs ~20 us per call)."""
    return torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice())


class DeviceStatus:
    """A device status word (int64[4]) plus helpers to reset and read it."""

    def __init__(self, device):
        self.t = torch.zeros(N.STATUS_WORDS, dtype=torch.int64, device=device)
        self.reset()

    @property
    def ptr(self) -> int:
        return self.t.data_ptr()

    def reset(self) -> None:
        N.call("tmd_status_reset", self.ptr, _stream())

    def read(self) -> np.ndarray:
        return self.t.cpu().numpy()


class CellGrid:
    """Counting-sorted cells over the rank box plus one ghost shell (neighbor.py:38-55).

    Device arrays: ``cell_of`` (n_total), ``cell_start`` (n_cells + 1),
    ``cell_atoms`` (n_total, grouped by cell, ascending inside a cell).
    """

    def __init__(self, origin, cell_size, dims, cell_of, cell_start, cell_atoms, n_total, shell=1):
        self.origin = np.asarray(origin, dtype=np.float64)
        self.cell_size = float(cell_size)
        self.dims = np.asarray(dims, dtype=np.int64)
        self.cell_of = cell_of
        self.cell_start = cell_start
        self.cell_atoms = cell_atoms
        self.n_total = n_total
        self.shell = int(shell)
        self._h_dims = N.host_i32(self.dims)

    @property
    def shell_dims(self) -> np.ndarray:
        return self.dims + 2 * self.shell

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.shell_dims))

    def cell_id(self, coords: np.ndarray) -> np.ndarray:
        gd = self.shell_dims
        return (coords[..., 0] * gd[1] + coords[..., 1]) * gd[2] + coords[..., 2]

    @property
    def coords(self) -> np.ndarray:
        """(n_total, 3) shell-shifted integer coordinates (neighbor.py:76)."""
        cid = self.cell_of[: self.n_total].cpu().numpy().astype(np.int64)
        gd = self.shell_dims
        return np.stack([cid // (gd[1] * gd[2]), (cid // gd[2]) % gd[1], cid % gd[2]], axis=1)

    @property
    def counts(self) -> np.ndarray:
        return np.diff(self.cell_start.cpu().numpy().astype(np.int64))

    @property
    def occupants(self) -> np.ndarray:
        """(n_cells, max_occ) -1 padded table, the reference's layout (neighbor.py:81-86)."""
        start = self.cell_start.cpu().numpy().astype(np.int64)
        atoms = self.cell_atoms[: self.n_total].cpu().numpy()
        counts = np.diff(start)
        width = int(counts.max()) if self.n_total else 1
        table = np.full((counts.size, width), -1, dtype=np.int32)
        cell = np.repeat(np.arange(counts.size), counts)
        table[cell, np.arange(atoms.size) - start[cell]] = atoms
        return table


def _describe_bin_failure(store: ParticleStore, lo, hi):
    def describe(code, key):
        i = int(key)
        kind = "local" if i < store.n_local else "ghost"
        p = store.pos[:, i].cpu().numpy()
        return (f" ({kind} particle {i} at {p} lies more than one cell shell outside the rank box "
                f"{lo}..{hi}; an exchange was probably missed)")

    return describe


def _recycle(old, shape, dtype, dev):
    """A tensor of `shape` in `old`'s storage when it is large enough, else a new
    one with 5% headroom (atom counts drift by a few per epoch; a fresh
    allocation of these sizes stalls the device for milliseconds)."""
    numel = int(np.prod(shape))
    if old is not None and old.dtype == dtype and old.device == dev:
        flat = old.untyped_storage()
        cap = flat.nbytes() // old.element_size()
        if cap >= numel:
            return torch.empty(0, dtype=dtype, device=dev).set_(flat, 0, shape)
    buf = torch.empty(int(numel * 1.05) + 1024, dtype=dtype, device=dev)
    return buf[:numel].view(shape)


def build_cell_grid(store: ParticleStore, rank_aabb: AABB, r: float, status: DeviceStatus | None = None,
                    check: bool = True, shell: int = 1, reuse: "CellGrid | None" = None,
                    positions: bool = True, count: tuple | None = None, launch: bool = True) -> CellGrid:
    """Bin every local and ghost atom into cells of edge r (neighbor.py:58-89).

    ``shell=2`` (production path) bins at edge r / 2 with two ghost layers; the
    list stencil is then 5^3 half-cells (~256 candidates per atom instead of
    ~443 for the reference's 27 cells of edge r).  ``reuse``: a dead grid whose
    device buffers are recycled (the step loop re-bins every epoch).
    ``positions=False`` skips the cell-ordered position copy (only the order
    is needed).  ``count=(n0, n_max, d_add)``: the atom count is n0 + *d_add,
    known only on the device (d_add: a device int32 address; n_max bounds
    it) -- the epoch then needs no host sync here; the caller sets
    ``grid.n_total`` once it has read the count.  ``launch=False``: only the
    buffers (the caller's own kernel sequence fills them: tmd_epoch_p1).
    """
    if r <= 0:
        raise ValueError("interaction radius must be positive")
    lo = rank_aabb.lo
    ext = rank_aabb.extent()
    edge = r / shell
    dims = np.maximum(1, np.ceil(ext / edge - 1e-12).astype(np.int64))
    n = store.n_total if count is None else int(count[1])
    n_cells = int(np.prod(dims + 2 * shell))
    dev = store.device
    i32 = torch.int32
    cell_of = _recycle(reuse.cell_of if reuse else None, (max(n, 1),), i32, dev)
    cell_start = _recycle(reuse.cell_start if reuse else None, (n_cells + 1,), i32, dev)
    cell_atoms = _recycle(reuse.cell_atoms if reuse else None, (max(n, 1),), i32, dev)
    if not launch:
        grid = CellGrid(lo, edge, dims, cell_of, cell_start, cell_atoms, n, shell)
        grid.cell_pos = _recycle(getattr(reuse, "cell_pos", None), (3, max(n, 1)), torch.float64, dev)
        grid.cell_pos_f = _cell_pos_f(grid, reuse)
        return grid
    st = status or DeviceStatus(dev)
    if status is None or check:
        st.reset()
    h_lo = N.host_f64(lo)
    h_dims = N.host_i32(dims)
    if count is None:
        N.call("tmd_bin_cells_ex", store.pos.data_ptr(), store.ld, n, N.hp(h_lo), float(edge), N.hp(h_dims),
               int(shell), cell_of.data_ptr(), cell_start.data_ptr(), cell_atoms.data_ptr(), st.ptr, _stream())
    else:
        N.call("tmd_bin_cells_dev", store.pos.data_ptr(), store.ld, int(count[0]), n, int(count[2]), N.hp(h_lo),
               float(edge), N.hp(h_dims), int(shell), cell_of.data_ptr(), cell_start.data_ptr(),
               cell_atoms.data_ptr(), st.ptr, _stream())
    if check:
        N.raise_for_status(st.read(), context="build_cell_grid",
                           describe=_describe_bin_failure(store, lo, rank_aabb.hi))
    grid = CellGrid(lo, edge, dims, cell_of, cell_start, cell_atoms, n, shell)
    grid.cell_pos = grid.cell_pos_f = None
    if positions:
        # positions in cell order: the list builders stream candidates from here
        grid.cell_pos = _recycle(getattr(reuse, "cell_pos", None), (3, max(n, 1)), torch.float64, dev)
        grid.cell_pos_f = _cell_pos_f(grid, reuse)
        n0, d_add = (n, 0) if count is None else (int(count[0]), int(count[2]))
        N.call("tmd_cell_positions_dev", store.pos.data_ptr(), store.ld, cell_atoms.data_ptr(), n0, n, d_add,
               grid.cell_pos.data_ptr(), grid.cell_pos.stride(0),
               grid.cell_pos_f.data_ptr() if grid.cell_pos_f is not None else 0, _stream())
    return grid


def _cell_pos_f(grid: "CellGrid", reuse) -> "torch.Tensor | None":
    """Float copies of the cell-ordered positions (same leading dimension) for
    the split builder's pre-filter; only the r/2 production grid has them."""
    if grid.shell < 2:
        return None
    old = getattr(reuse, "cell_pos_f", None) if reuse is not None else None
    ld = grid.cell_pos.stride(0)
    if old is not None and old.shape == (3, ld) and old.device == grid.cell_pos.device:
        return old
    return torch.empty((3, ld), dtype=torch.float32, device=grid.cell_pos.device)


def tinymd_f32_eps(grid: "CellGrid", rsq_max: float) -> float:
    """A bound (x2) on |rsq_float - rsq| for a candidate near the list radius:
    coordinates are at most X in magnitude (the grid box plus its shells and
    one more cell), each float coordinate is off by <= 2^-24 X, a float
    difference by <= 2^-23 X + 2^-24 R, and the float squares and sums add
    <= 4 * 2^-24 rsq (R = 1.01 sqrt(rsq_max))."""
    pad = (grid.shell + 1) * grid.cell_size
    lo = np.asarray(grid.origin, dtype=np.float64) - pad
    hi = np.asarray(grid.origin, dtype=np.float64) + np.asarray(grid.dims, dtype=np.float64) * grid.cell_size + pad
    x = float(max(np.abs(lo).max(), np.abs(hi).max()))
    r = 1.01 * math.sqrt(rsq_max)
    ec = 2.0 ** -23 * x + 2.0 ** -24 * r
    return 2.0 * (2.0 * math.sqrt(3.0) * ec * r + 3.0 * ec * ec + 4.0 * 2.0 ** -24 * (rsq_max + 1.0))


class NeighborLists:
    """Per-local candidate lists (neighbor.py:92-113), stored on the device.

    ``nbr`` is an int32 (ceil(cap / 4), ld_nbr, 4) tensor — quad-interleaved
    neighbor-major: slot k of local i is nbr[k // 4, i, k % 4] (see
    include/tinymd_b200.h).  ``cap`` is the logical row width (the
    reference's capacity).  ``order`` is "reference" (rows slot-for-slot the
    reference's) or "split" (the production rows: same sets, pairs with
    r_build < cutoff + near_margin at the front of the row — ``nnear`` of them
    — and the rest at the back, so a step whose atoms moved less than
    near_margin / 2 scans only the front).
    """

    def __init__(self, half, radius, nbr, d_counts, ref_positions, n_local, cap, order="reference",
                 nnear=None, near_margin=None):
        self.half = bool(half)
        self.radius = float(radius)
        self.nbr = nbr
        self.d_counts = d_counts
        self.ref_positions_dev = ref_positions  # (3, n_local) device copy
        self.n_local = int(n_local)
        self.cap = int(cap)
        self.order = order
        self.nnear = nnear
        self.near_margin = near_margin

    @property
    def ld_nbr(self) -> int:
        return self.nbr.shape[1]

    @property
    def cap4(self) -> int:
        """Row width in slots (a multiple of 4)."""
        return self.nbr.shape[2] * self.nbr.shape[0]

    @property
    def counts(self) -> np.ndarray:
        return self.d_counts[: self.n_local].cpu().numpy()

    @property
    def ref_positions(self) -> np.ndarray:
        return self.ref_positions_dev.t().contiguous().cpu().numpy()

    def _slots(self) -> np.ndarray:
        q, ld, w = self.nbr.shape
        return self.nbr.permute(1, 0, 2).reshape(ld, w * q)[: self.n_local].cpu().numpy()

    def slot_atom(self, i: int, k: int) -> int:
        """The atom in slot k of local i's row (for error messages)."""
        return int(self._slots()[i, k])

    def as_matrix(self) -> np.ndarray:
        """(n_local, cap) int32 rows, -1 beyond each count (neighbor.py:330-331).

        Split rows are returned near entries first, then the far entries in
        build order.
        """
        slots = self._slots()
        cnt = self.counts
        n = self.n_local
        width = max(self.cap, int(cnt.max()) if n else 0)
        mat = np.full((n, width), -1, dtype=np.int32)
        if self.order != "split":
            mat[:, : min(width, slots.shape[1])] = slots[:, :width]
            mat[np.arange(width)[None, :] >= cnt[:, None]] = -1
            return mat[:, : self.cap]
        nn = self.nnear[:n].cpu().numpy()
        c4 = slots.shape[1]
        for i in range(n):
            k, f = int(nn[i]), int(cnt[i] - nn[i])
            mat[i, :k] = slots[i, :k]
            mat[i, k:k + f] = slots[i, c4 - f:][::-1]
        return mat

    def pairs(self) -> np.ndarray:
        mat = self.as_matrix()
        valid = np.arange(mat.shape[1])[None, :] < self.counts[:, None]
        ii, slot = np.nonzero(valid)
        return np.column_stack([ii, mat[ii, slot]])


class BrickIndex:
    """Brick-major numbering of the locals (tmd_brick_sort; include/tinymd_b200.h):
    bricks of 2^shape cells of the production r/2 grid, cells z-fastest inside a
    brick.  A warp's 32 consecutive atoms then form a compact block, so the
    neighbour gathers of the step kernel share cache lines."""

    SHAPE = (1, 2, 2)  # log2 brick edges: 2 x 4 x 4 cells (best measured of 1x4x4 ... 8x8x8 at 80^3)

    def __init__(self, dims, device):
        self.dims = np.asarray(dims, dtype=np.int64)
        self.key = None
        self._h_dims = N.host_i32(self.dims)

    def sort(self, store: ParticleStore, lo, edge: float, shape=SHAPE) -> torch.Tensor:
        """Permutation of the locals into brick-major order (device int32)."""
        n = store.n_local
        dev = store.device
        self.key = _recycle(self.key, (max(n, 1),), torch.int32, dev)
        self._perm = perm = _recycle(getattr(self, "_perm", None), (max(n, 1),), torch.int32, dev)
        nk = int(np.prod([(int(d) + (1 << int(e)) - 1) >> int(e) for d, e in zip(self.dims, shape)])) << int(
            sum(int(e) for e in shape))
        ks = _recycle(getattr(self, "_ks", None), (nk + 1,), torch.int32, dev)
        self._ks = ks
        N.call("tmd_brick_sort", store.pos.data_ptr(), store.ld, n, N.hp(N.host_f64(lo)), float(edge),
               N.hp(self._h_dims), N.hp(N.host_i32(shape)), self.key.data_ptr(), ks.data_ptr(), perm.data_ptr(),
               _stream())
        return perm[:n]


def initial_list_capacity(n_local: int, dims, cell_size: float, r: float, half: bool) -> int:
    """neighbor.py:170-174: uniform-cloud estimate with headroom."""
    density = max(n_local, 1) / max(np.prod(dims) * cell_size**3, 1e-30)
    expect = 4.19 * r**3 * density * (0.6 if half else 1.1)
    return max(8, int(expect) + 8)


# largest near/far split margin, as a fraction of the skin: measured on the 80^3
# weak run (bench, 100 steps): 0.3 / 0.4 / 0.5 / 0.65 / 1.0 of the skin ->
# 4.45 / 4.52 / 4.46 / 4.14 / 4.13e9 atom-steps/s (profiles/r2_exp_phases.txt)
NEAR_MARGIN_FRACTION = 0.4


def near_margin(cutoff: float, r: float) -> float:
    """Largest front/back split of the production rows: 0.4 of the skin.

    The front alone is exact while an atom's own displacement plus the
    largest displacement stays below the margin -- early in an epoch; later
    steps scan the back segment too (the guard stops a run at skin / 2).
    """
    return max(NEAR_MARGIN_FRACTION * (r - cutoff), 0.0)


def build_neighbor_lists(store: ParticleStore, grid: CellGrid, r: float, half: bool,
                         list_layout=None, initial_capacity: int | None = None,
                         status: DeviceStatus | None = None, ld_nbr: int | None = None,
                         order: str = "reference", cutoff: float | None = None,
                         reuse: NeighborLists | None = None, margin: float | None = None,
                         build_order: torch.Tensor | None = None,
                         also: DeviceStatus | None = None, also_context: str = "",
                         defer: bool = False, d_near: torch.Tensor | None = None,
                         launch: bool = True) -> NeighborLists:
    """Every local's partners within r (neighbor.py:153-194).

    Capacity starts at the reference's estimate and doubles until the rows fit
    (the reference reruns its pass per doubling; here the first pass reports
    the longest row, so at most one rerun).  ``list_layout`` is accepted for
    compatibility.  ``order="split"`` (full lists only) builds the production
    rows (near pairs, cutoff + near_margin, at the front).  ``reuse``: a
    previous (now dead) NeighborLists whose device buffers are recycled — the
    step loop rebuilds every 20 steps and a 2M-atom list is ~0.7 GB.
    ``also``: another status word read back with the build's (one host sync),
    raised first (context ``also_context``).  ``defer``: launch the build and
    return at once; the caller runs ``lists.finish()`` (status read, capacity
    retry) after enqueueing its next independent work.  ``d_near``: a device
    (near_rsq, margin) pair (tmd_split_margin) that overrides ``margin``; the
    caller sets ``lists.near_margin`` from it once read back.  ``launch=False``
    (with ``defer``): only the buffers and the ``finish`` closure -- the
    caller's own kernel sequence runs the first build (tmd_epoch_p1).
    """
    n_local = store.n_local
    dev = store.device
    production = order == "split"
    cap = initial_capacity if initial_capacity is not None else initial_list_capacity(
        n_local, grid.dims, grid.cell_size, r, half)
    if production and initial_capacity is None:
        # production rows: 30% headroom over the mean instead of the reference's
        # 10%, and never below the width the previous epoch needed -- a thermal
        # density fluctuation then costs neither a second pass nor a doubling
        est = initial_list_capacity(n_local, grid.dims, grid.cell_size, r, half)
        cap = max(int((est - 8) * 1.3 / 1.1) + 8, reuse.cap if reuse is not None else 0)
    st = status or DeviceStatus(dev)
    ld_n = max(int(ld_nbr or n_local), 1)
    if production and ld_nbr is None:
        # rows for 5% more atoms than now, kept across epochs: migration changes
        # n_local by a few atoms per epoch and must not reallocate ~1 GB of list
        old_ld = reuse.ld_nbr if reuse is not None else 0
        ld_n = old_ld if old_ld >= n_local else int(1.05 * n_local) + 64
    i32 = torch.int32
    d_counts = _recycle(reuse.d_counts if reuse else None, (ld_n,), i32, dev)
    split = production
    if split:
        if half:
            raise ValueError("split rows are full lists")
        cut = float(cutoff if cutoff is not None else r)
        margin = near_margin(cut, r) if margin is None else min(float(margin), near_margin(cut, r))
        near_rsq = (cut + margin) * (cut + margin)  # the same rounding as tmd_split_margin
        nnear = _recycle(reuse.nnear if reuse is not None and reuse.nnear is not None else None, (ld_n,), i32, dev)
    elif order != "reference":
        raise ValueError(f"unknown list order {order!r}")
    rsq_max = r * r
    old_nbr = reuse.nbr if reuse else None

    def launch_rows(cap):
        nbr = _recycle(old_nbr, (max((cap + 3) // 4, 1), ld_n, 4), i32, dev)
        st.reset()
        common = (store.pos.data_ptr(), store.ld, n_local, grid.cell_of.data_ptr(),
                  grid.cell_start.data_ptr(), grid.cell_atoms.data_ptr(), grid.cell_pos.data_ptr(),
                  grid.cell_pos.stride(0), N.hp(grid._h_dims))
        if split:
            cpf = getattr(grid, "cell_pos_f", None)
            N.call("tmd_build_lists_split", *common[:8],
                   cpf.data_ptr() if cpf is not None else 0,
                   tinymd_f32_eps(grid, rsq_max) if cpf is not None else 0.0, common[8], grid.shell, float(near_rsq),
                   d_near.data_ptr() if d_near is not None else 0, float(rsq_max), int(cap),
                   nbr.data_ptr(), ld_n, nnear.data_ptr(), d_counts.data_ptr(),
                   build_order.data_ptr() if build_order is not None else 0, st.ptr, _stream())
        else:
            if grid.shell != 1:
                raise ValueError("reference-order lists need the reference grid (cells of edge r)")
            N.call("tmd_build_lists", *common, float(rsq_max), int(bool(half)), int(cap),
                   nbr.data_ptr(), ld_n, d_counts.data_ptr(), st.ptr, _stream())
        return nbr

    first_launch = launch
    launch = launch_rows
    nbr = launch(cap) if first_launch else _recycle(old_nbr, (max((cap + 3) // 4, 1), ld_n, 4), i32, dev)
    # x_ref rows in a (3, ld_n) buffer kept across epochs (a view of it is the
    # lists' ref_positions_dev; its leading dimension is passed to the kernels)
    base = getattr(reuse, "_ref_base", None) if reuse is not None else None
    if base is None or base.shape[1] < ld_n or base.device != dev:
        base = torch.empty((3, ld_n), dtype=torch.float64, device=dev)
    ref = base[:, :n_local]
    if first_launch:
        N.call("tmd_copy_rows", store.pos.data_ptr(), store.ld, ref.data_ptr(), ref.stride(0), 3, n_local,
               _stream())
    if split:
        out = NeighborLists(half, r, nbr, d_counts, ref, n_local, cap, "split", nnear, margin)
    else:
        out = NeighborLists(half, r, nbr, d_counts, ref, n_local, cap)
    out._ref_base = base

    def finish(words=None):
        """Read the build's status (one host sync); rebuild wider rows on overflow.
        ``words``: the first read, already done by the caller (the list status
        words, then ``also``'s)."""
        cap = out.cap
        while True:
            if words is None:
                words = st.read() if also is None else torch.cat([st.t, also.t]).cpu().numpy()
            code, _, need = N.decode_status(words[:N.STATUS_WORDS])
            if code == N.CAPACITY:
                if production:
                    cap = max(cap + 8, (int(need * 1.15) + 15) // 8 * 8)  # grow to the need, not x2
                else:
                    while cap < need:  # the reference's doubling (neighbor.py:176-181)
                        cap *= 2
                out.nbr, out.cap = launch_rows(cap), cap
                words = None
                continue
            if also is not None:
                # the caller's status word (its earlier kernels' checks) rides on the same read
                N.raise_for_status(words[N.STATUS_WORDS:], context=also_context)
            N.raise_for_status(words[:N.STATUS_WORDS], context="build_neighbor_lists")
            return out

    if split:
        out.near_rsq, out.rsq_max = float(near_rsq), float(rsq_max)
    if defer:
        out.finish = finish
        return out
    return finish()


def max_displacement_since_rebuild(store: ParticleStore, lists: NeighborLists) -> float:
    """Largest local move since the lists were built (neighbor.py:197-206)."""
    if lists.n_local == 0:
        return 0.0
    if store.n_local != lists.n_local:
        raise ProtocolError(
            f"store has {store.n_local} locals but lists were built for {lists.n_local}")
    out = torch.zeros(1, dtype=torch.float64, device=store.device)
    ref = lists.ref_positions_dev
    N.call("tmd_max_disp2", store.pos.data_ptr(), store.ld, ref.data_ptr(), ref.stride(0),
           store.n_local, out.data_ptr(), _stream())
    return float(np.sqrt(out.cpu().numpy()[0]))
