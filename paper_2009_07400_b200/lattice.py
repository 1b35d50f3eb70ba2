"""Lattice setup (reference: lattice_positions / create_lattice, particles.py:186-227).

Setup runs once on the host so the initial state is bit-identical to the
reference: the same fcc/bcc/sc sites in the same order and the same numpy
PCG64 velocity stream.  The arrays are then copied into the device store.
"""

from __future__ import annotations

import numpy as np

from .core import AABB, ConfigError, SimConfig
from .store import ParticleStore

__all__ = ["lattice_positions", "lattice_velocities", "create_lattice"]

# unit-cell basis in cell fractions: sc, bcc, fcc (particles.py:19-25)
_BASES = {
    1: np.array([[0.0, 0.0, 0.0]]),
    2: np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.5]]),
    4: np.array([[0.0, 0.0, 0.0], [0.5, 0.5, 0.0], [0.5, 0.0, 0.5], [0.0, 0.5, 0.5]]),
}


def lattice_positions(cfg: SimConfig, domain: AABB) -> np.ndarray:
    """Sites ordered x-major over unit cells, basis innermost (particles.py:186-208)."""
    basis = _BASES.get(cfg.particles_per_cell)
    if basis is None:
        raise ConfigError(
            f"particles_per_cell must be one of {sorted(_BASES)}, got {cfg.particles_per_cell}")
    a = cfg.lattice_constant()
    nx, ny, nz = cfg.unit_cells
    origin = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"),
                      axis=-1).reshape(-1, 3).astype(np.float64)
    sites = (origin[:, None, :] + basis[None, :, :]).reshape(-1, 3) * a
    sites += domain.lo
    if cfg.fill == "half-diagonal":
        frac = (sites - domain.lo) / domain.extent()
        sites = sites[frac[:, 0] + frac[:, 1] < 1.0]
    return sites


def lattice_velocities(cfg: SimConfig, n: int) -> np.ndarray:
    """U[-0.5, 0.5) * velocity_scale from PCG64(rng_seed), net momentum removed."""
    gen = np.random.default_rng(cfg.rng_seed)
    vel = (gen.random((n, 3)) - 0.5) * cfg.velocity_scale
    if n > 0 and cfg.velocity_scale > 0:
        vel -= vel.mean(axis=0)
    return vel


def create_lattice(cfg: SimConfig, domain: AABB, layout=None, device=None) -> ParticleStore:
    """Whole lattice as locals of one device store (particles.py:211-227)."""
    pos = lattice_positions(cfg, domain)
    vel = lattice_velocities(cfg, pos.shape[0])
    store = ParticleStore(max(pos.shape[0], 1), device=device, layout=layout)
    store.append_locals(pos, vel)
    return store
