"""Numpy restatement of the reference (``nanopair``) hot path — TEST INFRASTRUCTURE ONLY.

This module is the parity *checker* for the B200 build.  It restates, with
plain arrays instead of the reference's store/handle classes, every step of
the reference's pairwise-interaction timestep:

  lattice + seeded velocities   particles.py:186-227, core.py:255-265
  cell binning (counting sort)  neighbor.py:58-89
  Verlet list build             neighbor.py:92-194
  LJ / Spring-Dashpot laws      potential.py:30-105
  force evaluation + energy     potential.py:134-213
  velocity Verlet               driver.py:74-93
  displacement guard            neighbor.py:197-206, driver.py:115-125
  six-stencil decomposition     comm.py:171-274
  exchange / borders / sync     comm.py:340-498 (ranks advanced in lockstep)
  step loop                     driver.py:128-177

plus what the reference does not have: a lockstep multi-rank runner (the
reference ships none, driver.py:134-139) and a thermo extension (PE, KE,
virial W and pressure P = (2 KE + W) / (3 V); the virial/pressure definition
is ours — the reference defines no pressure, so pressure parity is pinned only
against this oracle).

Arithmetic order follows the reference so results are bitwise identical on the
same numpy: in particular ``einsum('ijk,ijk->ij')`` of a 3-vector evaluates as
``(dx*dx + dz*dz) + dy*dy`` on numpy 2.3 (checked by ``tests/test_oracle.py``
against the live einsum) and ``sum(axis=1)`` over list slots is sequential.

Parity pinned against ``tests/golden/*.npz`` (generated from the reference by
``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import math
from collections import deque
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "OracleConfig",
    "OracleProtocolError",
    "OracleSingularityError",
    "OracleGuardViolation",
    "lattice_constant",
    "domain_bounds",
    "lattice_positions",
    "initial_state",
    "rsq_ref_order",
    "dot3_ref_order",
    "CellBins",
    "bin_cells",
    "NeighborTable",
    "build_lists",
    "lj_pair_force",
    "lj_pair_energy",
    "sd_pair_force",
    "sd_pair_energy",
    "Law",
    "evaluate_forces",
    "kick_drift",
    "kick",
    "max_displacement",
    "factor_rank_grid",
    "rank_coords",
    "rank_index",
    "slab_of",
    "stencil_entries",
    "RankState",
    "World",
    "run",
]

CHUNK = 4096  # backend.py:20 / neighbor.py:35


class OracleProtocolError(RuntimeError):
    """errors.py:4-5"""


class OracleSingularityError(ArithmeticError):
    """errors.py:8-9"""


class OracleGuardViolation(RuntimeError):
    """errors.py:12-13"""


def _get(cfg, name, default=None):
    return getattr(cfg, name, default)


@dataclass
class OracleConfig:
    """The reference's ``SimConfig`` fields and defaults (core.py:187-215), as a
    plain record: the oracle and bench.py's CPU arm describe a run without
    importing the product package.  Any object with these attributes works."""

    unit_cells: tuple = (32, 32, 32)
    particles_per_cell: int = 4
    lattice_density: float = 0.8442
    dt: float = 0.005
    steps: int = 100
    cutoff: float = 2.5
    verlet_buffer: float = 0.3
    reneigh_interval: int = 20
    potential_kind: str = "lj"
    epsilon: float = 1.0
    sigma: float = 1.0
    stiffness: float = 100.0
    damping: float = 0.0
    diameter: float = 1.0
    half_neighbor: bool = False
    mass: float = 1.0
    rng_seed: int = 42
    velocity_scale: float = 1.0
    fill: str = "full"

    def n_atoms(self) -> int:
        """particles.py:186-208 (full fill): cells x basis."""
        nx, ny, nz = self.unit_cells
        return nx * ny * nz * self.particles_per_cell


# ---------------------------------------------------------------------------
# lattice  (core.py:255-265, particles.py:19-25, 186-227)
# ---------------------------------------------------------------------------

_BASIS = {
    1: ((0.0, 0.0, 0.0),),
    2: ((0.0, 0.0, 0.0), (0.5, 0.5, 0.5)),
    4: ((0.0, 0.0, 0.0), (0.5, 0.5, 0.0), (0.5, 0.0, 0.5), (0.0, 0.5, 0.5)),
}


def lattice_constant(cfg) -> float:
    """core.py:259-260: a = (ppc / rho)^(1/3)."""
    return (cfg.particles_per_cell / cfg.lattice_density) ** (1.0 / 3.0)


def domain_bounds(cfg):
    """core.py:262-265: the box is [0, n_d * a) per axis."""
    a = lattice_constant(cfg)
    nx, ny, nz = cfg.unit_cells
    return np.zeros(3), np.array([nx * a, ny * a, nz * a], dtype=np.float64)


def lattice_positions(cfg) -> np.ndarray:
    """particles.py:186-208: unit cells x-major, basis innermost, times a, plus lo."""
    a = lattice_constant(cfg)
    nx, ny, nz = cfg.unit_cells
    cells = np.indices((nx, ny, nz)).reshape(3, -1).T.astype(np.float64)
    basis = np.array(_BASIS[cfg.particles_per_cell], dtype=np.float64)
    sites = (cells[:, None, :] + basis[None, :, :]).reshape(-1, 3) * a
    lo, hi = domain_bounds(cfg)
    sites += lo
    if _get(cfg, "fill", "full") == "half-diagonal":
        frac = (sites - lo) / (hi - lo)
        sites = sites[frac[:, 0] + frac[:, 1] < 1.0]
    return sites


def initial_state(cfg):
    """particles.py:211-227: uniform [-0.5, 0.5) * scale from PCG64(seed), mean removed."""
    pos = lattice_positions(cfg)
    n = pos.shape[0]
    gen = np.random.default_rng(cfg.rng_seed)
    vel = (gen.random((n, 3)) - 0.5) * cfg.velocity_scale
    if n > 0 and cfg.velocity_scale > 0:
        vel -= vel.mean(axis=0)
    return pos, vel


# ---------------------------------------------------------------------------
# arithmetic-order helpers (Appendix A-1 of SURVEY.md)
# ---------------------------------------------------------------------------


def rsq_ref_order(d: np.ndarray) -> np.ndarray:
    """The order numpy's einsum('ijk,ijk->ij') uses on this host: (x*x + z*z) + y*y.

    Reference call sites: neighbor.py:135, potential.py:172.
    """
    return (d[..., 0] * d[..., 0] + d[..., 2] * d[..., 2]) + d[..., 1] * d[..., 1]


def dot3_ref_order(u: np.ndarray, v: np.ndarray) -> np.ndarray:
    """einsum('...k,...k->...') order, used by the dashpot term (potential.py:91)."""
    return (u[..., 0] * v[..., 0] + u[..., 2] * v[..., 2]) + u[..., 1] * v[..., 1]


# ---------------------------------------------------------------------------
# cell binning  (neighbor.py:38-89)
# ---------------------------------------------------------------------------


@dataclass
class CellBins:
    lo: np.ndarray
    r: float
    dims: np.ndarray  # interior cells per axis
    coords: np.ndarray  # (n, 3) shell-shifted cell coordinates
    cid: np.ndarray  # (n,) flat cell id, x slowest
    counts: np.ndarray  # (n_cells,)
    start: np.ndarray  # (n_cells,) exclusive prefix sum of counts
    order: np.ndarray  # stable sort of atom indices by cid

    @property
    def shell_dims(self) -> np.ndarray:
        return self.dims + 2

    def occupants(self) -> np.ndarray:
        """The reference's (n_cells, max_occ) -1 padded table (neighbor.py:81-86)."""
        n_cells = self.counts.size
        width = int(self.counts.max()) if self.order.size else 1
        table = np.full((n_cells, width), -1, dtype=np.int32)
        cell_of_sorted = self.cid[self.order]
        rank_in_cell = np.arange(self.order.size) - self.start[cell_of_sorted]
        table[cell_of_sorted, rank_in_cell] = self.order
        return table


def bin_cells(pos: np.ndarray, n_local: int, lo, hi, r: float) -> CellBins:
    """neighbor.py:58-89 — floor((p - lo) / r) with IEEE division, one ghost shell."""
    if r <= 0:
        raise ValueError("interaction radius must be positive")
    lo = np.asarray(lo, dtype=np.float64)
    ext = np.asarray(hi, dtype=np.float64) - lo
    dims = np.maximum(1, np.ceil(ext / r - 1e-12).astype(np.int64))
    c = np.floor((pos - lo) / r).astype(np.int64)
    outside = np.any((c < -1) | (c > dims), axis=1)
    if outside.any():
        i = int(np.argmax(outside))
        kind = "local" if i < n_local else "ghost"
        raise OracleProtocolError(f"{kind} particle {i} beyond the ghost shell")
    s = c + 1
    g = dims + 2
    cid = (s[:, 0] * g[1] + s[:, 1]) * g[2] + s[:, 2]
    n_cells = int(np.prod(g))
    counts = np.bincount(cid, minlength=n_cells)
    start = np.zeros(n_cells, dtype=np.int64)
    np.cumsum(counts[:-1], out=start[1:])
    order = np.argsort(cid, kind="stable")
    return CellBins(lo, r, dims, s, cid, counts, start, order)


# ---------------------------------------------------------------------------
# Verlet lists  (neighbor.py:30-33, 92-194)
# ---------------------------------------------------------------------------

_OFFSETS = np.array(
    [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)], dtype=np.int64
)


@dataclass
class NeighborTable:
    half: bool
    r: float
    mat: np.ndarray  # (n_local, cap) int32, -1 padded
    counts: np.ndarray  # (n_local,) int32
    ref_positions: np.ndarray
    n_local: int

    @property
    def cap(self) -> int:
        return self.mat.shape[1]

    def pairs(self) -> np.ndarray:
        keep = np.arange(self.cap)[None, :] < self.counts[:, None]
        ii, kk = np.nonzero(keep)
        return np.column_stack([ii, self.mat[ii, kk]])


def _initial_cap(n_local, dims, r, half):
    """neighbor.py:170-174."""
    density = max(n_local, 1) / max(np.prod(dims) * r**3, 1e-30)
    expect = 4.19 * r**3 * density * (0.6 if half else 1.1)
    return max(8, int(expect) + 8)


def _candidate_rows(bins: CellBins, occ: np.ndarray, lo_i: int, hi_i: int):
    """Stencil cells x-slowest/z-fastest, occupants ascending: (m, 27 * width)."""
    g = bins.shell_dims
    nb = bins.coords[lo_i:hi_i, None, :] + _OFFSETS[None, :, :]
    cells = (nb[..., 0] * g[1] + nb[..., 1]) * g[2] + nb[..., 2]
    return occ[cells].reshape(hi_i - lo_i, -1)


def build_lists(pos, n_local, bins: CellBins, r, half=False, cap=None) -> NeighborTable:
    """neighbor.py:153-194; a pass that overflows cap reruns with cap doubled."""
    rsq_max = r * r
    if cap is None:
        cap = _initial_cap(n_local, bins.dims, r, half)
    occ = bins.occupants()
    rows_all, cols_all, counts = [], [], np.zeros(n_local, dtype=np.int32)
    for lo_i in range(0, n_local, CHUNK):
        hi_i = min(lo_i + CHUNK, n_local)
        cand = _candidate_rows(bins, occ, lo_i, hi_i)
        present = cand >= 0
        j = np.where(present, cand, 0)
        d = pos[lo_i:hi_i, None, :] - pos[j]
        rsq = rsq_ref_order(d)
        me = np.arange(lo_i, hi_i)[:, None]
        keep = present & (rsq < rsq_max)
        keep &= ((j >= n_local) | (j > me)) if half else (j != me)
        rr, cc = np.nonzero(keep)
        counts[lo_i:hi_i] = np.bincount(rr, minlength=hi_i - lo_i)
        rows_all.append(rr + lo_i)
        cols_all.append(cand[rr, cc])
    need = int(counts.max()) if n_local else 0
    while need > cap:
        cap *= 2
    mat = np.full((n_local, cap), -1, dtype=np.int32)
    if n_local:
        rr = np.concatenate(rows_all)
        jj = np.concatenate(cols_all)
        first = np.zeros(n_local, dtype=np.int64)
        np.cumsum(counts[:-1], out=first[1:])
        mat[rr, np.arange(rr.size) - first[rr]] = jj
    return NeighborTable(half, r, mat, counts, pos[:n_local].copy(), n_local)


# ---------------------------------------------------------------------------
# pair laws  (potential.py:30-105)
# ---------------------------------------------------------------------------


def lj_pair_force(delta, rsq, eps, sigma):
    """potential.py:46-52: f = 48 eps sr6 (sr6 - 1/2) sr2, sr6 = sr2^3 sigma^6."""
    s6 = sigma**6
    sr2 = 1.0 / rsq
    sr6 = sr2 * sr2 * sr2 * s6
    f = 48.0 * sr6 * (sr6 - 0.5) * sr2 * eps
    return f[..., None] * delta


def lj_pair_energy(rsq, eps, sigma):
    """potential.py:54-57: 4 eps (sr6^2 - sr6), unshifted."""
    sr6 = sigma**6 / (rsq * rsq * rsq)
    return 4.0 * eps * (sr6 * sr6 - sr6)


def sd_pair_force(delta, rsq, vi, vj, k, gamma, diam):
    """potential.py:80-93: K overlap n - gamma (n . (vi - vj)) n while overlapping."""
    dist = np.sqrt(rsq)
    overlap = diam - dist
    n = delta / dist[..., None]
    spring = k * overlap[..., None] * n
    if vi is None or vj is None:
        dash = 0.0
    else:
        dash = -gamma * dot3_ref_order(n, vi - vj)[..., None] * n
    return np.where((overlap > 0.0)[..., None], spring + dash, 0.0)


def sd_pair_energy(rsq, k, diam):
    """potential.py:95-97."""
    ov = np.maximum(diam - np.sqrt(rsq), 0.0)
    return 0.5 * k * ov * ov


@dataclass(frozen=True)
class Law:
    kind: str  # "lj" | "sd"
    eps: float = 1.0
    sigma: float = 1.0
    cutoff: float = 2.5
    k: float = 100.0
    gamma: float = 0.0
    diam: float = 1.0

    @classmethod
    def from_cfg(cls, cfg) -> "Law":
        """potential.py:100-105."""
        if cfg.potential_kind == "lj":
            return cls("lj", eps=cfg.epsilon, sigma=cfg.sigma, cutoff=cfg.cutoff)
        if cfg.potential_kind == "sd":
            return cls("sd", k=cfg.stiffness, gamma=cfg.damping, diam=cfg.diameter)
        raise ValueError(cfg.potential_kind)

    @property
    def cutoff_rsq(self) -> float:
        return self.cutoff * self.cutoff if self.kind == "lj" else self.diam * self.diam

    def force(self, delta, rsq, vi=None, vj=None):
        if self.kind == "lj":
            return lj_pair_force(delta, rsq, self.eps, self.sigma)
        return sd_pair_force(delta, rsq, vi, vj, self.k, self.gamma, self.diam)

    def energy(self, rsq):
        if self.kind == "lj":
            return lj_pair_energy(rsq, self.eps, self.sigma)
        return sd_pair_energy(rsq, self.k, self.diam)


# ---------------------------------------------------------------------------
# force evaluation  (potential.py:134-213)
# ---------------------------------------------------------------------------


def evaluate_forces(pos, vel, n_local, table: NeighborTable, law: Law, half=None,
                    energy=False, threads=1):
    """Returns (F (n_local, 3), PE or None, virial W or None).

    Full mode: F_i = sequential sum over list slots of the masked pair force
    (potential.py:185); PE = 1/2 sum of pair energies (potential.py:193-195).
    Half mode adds -F_ij to local partners after the owned sums, chunk by
    chunk (potential.py:187-191, 205-209).  W = 1/2 sum_i sum_j delta.F_ij in
    full mode, sum over stored pairs in half mode (oracle extension).
    """
    if half is None:
        half = table.half
    mat, counts = table.mat, table.counts
    cap = mat.shape[1] if mat.size else 0
    rc2 = law.cutoff_rsq
    slots = np.arange(cap, dtype=np.int32)[None, :]
    needs_v = law.kind == "sd"

    def chunk(lo_i, hi_i):
        rows = mat[lo_i:hi_i]
        valid = slots < counts[lo_i:hi_i, None]
        j = np.where(valid, rows, 0)
        d = pos[lo_i:hi_i, None, :] - pos[j]
        rsq = rsq_ref_order(d)
        inside = valid & (rsq < rc2)
        hit = inside & (rsq == 0.0)
        if hit.any():
            a, b = np.nonzero(hit)
            raise OracleSingularityError(f"coincident pair: local {lo_i + a[0]} and neighbor {rows[a[0], b[0]]}")
        safe = np.where(inside, rsq, 1.0)
        if needs_v:
            f = law.force(d, safe, vel[lo_i:hi_i, None, :], vel[j])
        else:
            f = law.force(d, safe)
        f = np.where(inside[..., None], f, 0.0)
        own = f.sum(axis=1)
        react = None
        if half:
            jj, ff = j[inside], f[inside]
            back = jj < n_local
            react = (jj[back], ff[back])
        e = w = None
        if energy:
            e_sum = np.where(inside, law.energy(safe), 0.0).sum()
            e = e_sum if half else 0.5 * e_sum
            w_sum = (f * d).sum()
            w = w_sum if half else 0.5 * w_sum
        return lo_i, own, react, e, w

    bounds = list(range(0, n_local, CHUNK)) or [0]
    tasks = [(b, min(b + CHUNK, n_local)) for b in bounds]
    if threads > 1 and len(tasks) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            results = [f.result() for f in [pool.submit(chunk, *t) for t in tasks]]
    else:
        results = [chunk(*t) for t in tasks]
    F = np.zeros((n_local, 3))
    es, ws = [], []
    for lo_i, own, _, e, w in results:
        F[lo_i:lo_i + own.shape[0]] = own
        if e is not None:
            es.append(e)
            ws.append(w)
    for _, _, react, _, _ in results:
        if react is not None:
            jj, ff = react
            for c in range(3):
                F[:, c] -= np.bincount(jj, weights=ff[:, c], minlength=n_local)
    if energy:
        return F, float(np.sum(es)), float(np.sum(ws))
    return F, None, None


# ---------------------------------------------------------------------------
# integration and guard  (driver.py:74-93, neighbor.py:197-206)
# ---------------------------------------------------------------------------


def kick_drift(pos, vel, F, n, dt, mass):
    """driver.py:74-83: v += (dt/2 / m) F; x += dt v on locals."""
    if n == 0 or dt == 0.0:
        return
    vel[:n] = vel[:n] + (0.5 * dt / mass) * F[:n]
    pos[:n] = pos[:n] + dt * vel[:n]


def kick(vel, F, n, dt, mass):
    """driver.py:86-93."""
    if n == 0 or dt == 0.0:
        return
    vel[:n] = vel[:n] + (0.5 * dt / mass) * F[:n]


def max_displacement(pos_local, ref_positions) -> float:
    """neighbor.py:197-206."""
    if ref_positions.shape[0] == 0:
        return 0.0
    d = pos_local - ref_positions
    return float(np.sqrt((d * d).sum(axis=1).max()))


# ---------------------------------------------------------------------------
# decomposition  (comm.py:171-274)
# ---------------------------------------------------------------------------


def factor_rank_grid(p: int):
    """comm.py:171-186: prime factors, largest first, onto the smallest axis."""
    if p <= 0:
        raise ValueError("rank count must be positive")
    primes, n, f = [], p, 2
    while n > 1:
        while n % f == 0:
            primes.append(f)
            n //= f
        f += 1
    dims = [1, 1, 1]
    for q in sorted(primes, reverse=True):
        dims[int(np.argmin(dims))] *= q
    return tuple(sorted(dims, reverse=True))


def rank_coords(rank, grid):
    """comm.py:195-197."""
    return rank % grid[0], (rank // grid[0]) % grid[1], rank // (grid[0] * grid[1])


def rank_index(coords, grid):
    """comm.py:189-192."""
    return (coords[2] * grid[1] + coords[1]) * grid[0] + coords[0]


def slab_of(lo, hi, grid, coords):
    """comm.py:200-207 — same fp64 expression on both sides of every face."""
    lo = np.asarray(lo, dtype=np.float64)
    ext = np.asarray(hi, dtype=np.float64) - lo
    g = np.asarray(grid, dtype=np.float64)
    c = np.asarray(coords, dtype=np.float64)
    return lo + ext * (c / g), lo + ext * ((c + 1.0) / g)


@dataclass
class Entry:
    dim: int
    sign: int  # +1 / -1
    send_to: int
    recv_from: int
    face: float
    shift: np.ndarray  # (3,), +-L on the periodic face


def stencil_entries(grid, rank, lo, hi):
    """comm.py:210-274: per dimension one round of (+, -) entries."""
    me = rank_coords(rank, grid)
    s_lo, s_hi = slab_of(lo, hi, grid, me)
    ext = np.asarray(hi, dtype=np.float64) - np.asarray(lo, dtype=np.float64)
    rounds = []
    for d in range(3):
        pair = []
        for sign in (+1, -1):
            to = list(me)
            to[d] = (me[d] + sign) % grid[d]
            frm = list(me)
            frm[d] = (me[d] - sign) % grid[d]
            edge = me[d] == grid[d] - 1 if sign > 0 else me[d] == 0
            shift = np.zeros(3)
            if edge:
                shift[d] = -ext[d] if sign > 0 else ext[d]
            face = s_hi[d] if sign > 0 else s_lo[d]
            pair.append(Entry(d, sign, rank_index(to, grid), rank_index(frm, grid), face, shift))
        rounds.append(pair)
    return rounds, (s_lo, s_hi)


# ---------------------------------------------------------------------------
# per-rank state and the three halo phases  (particles.py:30-158, comm.py:340-498)
# ---------------------------------------------------------------------------


@dataclass
class RankState:
    rank: int
    rounds: list
    slab: tuple
    pos: np.ndarray  # (n_local + n_ghost, 3)
    vel: np.ndarray
    frc: np.ndarray
    n_local: int
    n_ghost: int = 0
    plan: list = field(default_factory=list)  # per round: (sends, recvs)
    table: NeighborTable | None = None
    bins: CellBins | None = None
    since_rebuild: int = 0
    max_disp_seen: float = 0.0

    def clear_ghosts(self):
        """particles.py:136-139."""
        n = self.n_local
        self.pos, self.vel, self.frc = self.pos[:n].copy(), self.vel[:n].copy(), self.frc[:n].copy()
        self.n_ghost = 0

    def add_ghosts(self, p) -> int:
        """particles.py:141-155: ghost v and F start at zero."""
        start = self.pos.shape[0]
        k = p.shape[0]
        self.pos = np.vstack([self.pos, p]) if k else self.pos
        self.vel = np.vstack([self.vel, np.zeros((k, 3))]) if k else self.vel
        self.frc = np.vstack([self.frc, np.zeros((k, 3))]) if k else self.frc
        self.n_ghost += k
        return start

    def add_locals(self, p, v):
        """particles.py:83-98 (ghost region is empty during exchange)."""
        if p.shape[0] == 0:
            return
        assert self.n_ghost == 0
        self.pos = np.vstack([self.pos, p])
        self.vel = np.vstack([self.vel, v])
        self.frc = np.vstack([self.frc, np.zeros_like(p)])
        self.n_local += p.shape[0]

    def owns(self, p):
        """core.py:100-103 half-open membership."""
        lo, hi = self.slab
        return np.all((p >= lo) & (p < hi), axis=1)


class World:
    """All simulated ranks plus one FIFO per (src, dst), as comm.py:83-104."""

    def __init__(self, cfg, nranks: int, positions=None, velocities=None):
        self.cfg = cfg
        self.size = nranks
        self.grid = factor_rank_grid(nranks)
        self.lo, self.hi = domain_bounds(cfg)
        self.r = cfg.cutoff + cfg.verlet_buffer  # core.py:255-257
        if positions is None:
            positions, velocities = initial_state(cfg)
        self.ranks = []
        for rk in range(nranks):
            rounds, slab = stencil_entries(self.grid, rk, self.lo, self.hi)
            inside = np.all((positions >= slab[0]) & (positions < slab[1]), axis=1)
            p = positions[inside].copy()
            v = velocities[inside].copy()
            self.ranks.append(RankState(rk, rounds, slab, p, v, np.zeros_like(p), p.shape[0]))
        self._box: dict[tuple[int, int], deque] = {}

    def _send(self, src, dst, payload):
        self._box.setdefault((src, dst), deque()).append(payload)

    def _recv(self, dst, src):
        q = self._box.get((src, dst))
        if not q:
            raise OracleProtocolError(f"rank {dst} expected a message from {src}")
        return q.popleft()

    # comm.py:340-400
    def exchange(self):
        for R in self.ranks:
            R.clear_ghosts()
        for d in range(3):
            for R in self.ranks:
                snap = R.pos[:R.n_local].copy()
                leaving = np.zeros(R.n_local, dtype=bool)
                for e in R.rounds[d]:
                    sel = snap[:, d] >= e.face if e.sign > 0 else snap[:, d] < e.face
                    idx = np.nonzero(sel)[0]
                    out = snap[idx] + e.shift
                    if e.send_to == R.rank:
                        R.pos[idx] = out
                        continue
                    self._send(R.rank, e.send_to, (out, R.vel[idx].copy()))
                    leaving[idx] = True
                if leaving.any():
                    keep = ~leaving
                    R.pos, R.vel, R.frc = R.pos[keep], R.vel[keep], R.frc[keep]
                    R.n_local = int(keep.sum())
            for R in self.ranks:
                for e in R.rounds[d]:
                    if e.recv_from == R.rank:
                        continue
                    p, v = self._recv(R.rank, e.recv_from)
                    R.add_locals(p, v)
        for R in self.ranks:
            bad = ~R.owns(R.pos[:R.n_local])
            if bad.any():
                raise OracleProtocolError(f"rank {R.rank}: local outside ownership after exchange")

    # comm.py:403-466
    def define_borders(self):
        r = self.r
        for R in self.ranks:
            R.plan = []
        for d in range(3):
            for R in self.ranks:
                snap = R.pos.copy()
                sends = []
                for e in R.rounds[d]:
                    sel = snap[:, d] > e.face - r if e.sign > 0 else snap[:, d] < e.face + r
                    idx = np.nonzero(sel)[0]
                    out = snap[idx] + e.shift
                    shift = out - snap[idx] if idx.size else np.empty((0, 3))
                    if e.send_to == R.rank:
                        start = R.add_ghosts(out)
                        sends.append((R.rank, idx, shift, start))
                    else:
                        self._send(R.rank, e.send_to, out)
                        sends.append((e.send_to, idx, shift, -1))
                R.plan.append((sends, []))
            for R in self.ranks:
                for e in R.rounds[d]:
                    if e.recv_from == R.rank:
                        continue
                    p = self._recv(R.rank, e.recv_from)
                    start = R.add_ghosts(p)
                    R.plan[d][1].append((e.recv_from, start, p.shape[0]))

    # comm.py:469-498
    def synchronize(self):
        for d in range(3):
            for R in self.ranks:
                for peer, idx, shift, start in R.plan[d][0]:
                    data = R.pos[idx] + shift
                    if peer == R.rank:
                        R.pos[start:start + idx.size] = data
                    else:
                        self._send(R.rank, peer, data)
            for R in self.ranks:
                for peer, start, count in R.plan[d][1]:
                    data = self._recv(R.rank, peer)
                    if data.shape[0] != count:
                        raise OracleProtocolError("sync count mismatch")
                    R.pos[start:start + count] = data


# ---------------------------------------------------------------------------
# step loop  (driver.py:102-177) + thermo extension
# ---------------------------------------------------------------------------


@dataclass
class OracleRun:
    thermo: np.ndarray  # rows: step, PE, KE, W, P, Px, Py, Pz
    world: World
    momentum_initial: np.ndarray
    momentum_final: np.ndarray

    def global_state(self):
        """(N, 6) locals of every rank, rows sorted lexicographically by position."""
        parts = [np.hstack([R.pos[:R.n_local], R.vel[:R.n_local]]) for R in self.world.ranks]
        s = np.vstack(parts)
        order = np.lexsort((s[:, 2], s[:, 1], s[:, 0]))
        return s[order]


def _rebuild(world: World, half: bool):
    """driver.py:102-112 with grid_box = the rank slab (static grid)."""
    world.exchange()
    world.define_borders()
    for R in world.ranks:
        R.bins = bin_cells(R.pos, R.n_local, R.slab[0], R.slab[1], world.r)
        R.table = build_lists(R.pos, R.n_local, R.bins, world.r, half)
        R.since_rebuild = 0


def _forces(world: World, law: Law, half: bool, threads: int):
    """Per-rank force call; rank totals combined with Python's (compensated) sum()."""
    es, ws = [], []
    for R in world.ranks:
        F, e, v = evaluate_forces(R.pos, R.vel, R.n_local, R.table, law, half, energy=True,
                                  threads=threads)
        R.frc[:R.n_local] = F
        R.frc[R.n_local:] = 0.0
        es.append(e)
        ws.append(v)
    return sum(es), sum(ws)


def _thermo_row(world: World, step, pe, w, mass):
    ke = 0.0
    mom = np.zeros(3)
    for R in world.ranks:
        v = R.vel[:R.n_local]
        ke += 0.5 * mass * float(np.sum(v * v))
        mom += mass * v.sum(axis=0)
    vol = float(np.prod(world.hi - world.lo))
    press = (2.0 * ke + w) / (3.0 * vol)
    return [step, pe, ke, w, press, mom[0], mom[1], mom[2]]


def run(cfg, nranks: int = 1, steps: int | None = None, threads=1,
        positions=None, velocities=None, on_step=None) -> OracleRun:
    """Lockstep multi-rank run of driver.py:128-177 with a thermo row per step.

    Row k: PE and W from step k's force call, KE from velocities after step
    k's closing half-kick; row 0 comes from the setup force call.  ``threads``
    is a thread count for the force phase or a callable step -> count (the
    results do not depend on it: chunks are combined in fixed order).
    """
    nthreads = threads if callable(threads) else (lambda step, _t=threads: _t)
    steps = cfg.steps if steps is None else steps
    half = bool(_get(cfg, "half_neighbor", False))
    law = Law.from_cfg(cfg)
    world = World(cfg, nranks, positions, velocities)
    mass, dt = cfg.mass, cfg.dt
    p0 = np.zeros(3)
    for R in world.ranks:
        p0 += mass * R.vel[:R.n_local].sum(axis=0) if R.n_local else 0.0
    _rebuild(world, half)
    pe, w = _forces(world, law, half, nthreads(0))
    rows = [_thermo_row(world, 0, pe, w, mass)]
    if on_step:
        on_step(0, world)
    for step in range(1, steps + 1):
        for R in world.ranks:
            kick_drift(R.pos, R.vel, R.frc, R.n_local, dt, mass)
        if step % cfg.reneigh_interval == 0:
            _rebuild(world, half)
        else:
            world.synchronize()
            for R in world.ranks:
                R.since_rebuild += 1
        for R in world.ranks:
            if R.since_rebuild:
                disp = max_displacement(R.pos[:R.n_local], R.table.ref_positions)
                R.max_disp_seen = max(R.max_disp_seen, disp)
                if disp >= 0.5 * cfg.verlet_buffer:
                    raise OracleGuardViolation(f"rank {R.rank} step {step}: moved {disp:.4g}")
        pe, w = _forces(world, law, half, nthreads(step))
        for R in world.ranks:
            kick(R.vel, R.frc, R.n_local, dt, mass)
        rows.append(_thermo_row(world, step, pe, w, mass))
        if on_step:
            on_step(step, world)
    p1 = np.zeros(3)
    for R in world.ranks:
        p1 += mass * R.vel[:R.n_local].sum(axis=0) if R.n_local else 0.0
    return OracleRun(np.array(rows), world, p0, p1)
