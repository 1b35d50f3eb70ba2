"""Force laws and the force operator on the GPU (reference: potential.py:20-213).

``LennardJones`` / ``SpringDashpot`` keep the reference's dataclass fields,
``cutoff_rsq``, ``needs_velocities`` and ``pair_force`` / ``pair_energy``
(evaluated by libtinymd_b200.so on device copies of the arrays).
``compute_forces`` has the reference's signature and error behaviour:

    compute_forces(store, lists, law, half=None, backend=None,
                   accumulate_energy=False) -> float | None

Full lists run the no-atomics thread-per-atom kernels (``exact=True``, the
default here, reproduces the reference bit for bit; ``exact=False`` is the
FMA/fast-reciprocal production kernel).  Half lists scatter reactions with
fp64 atomics.  ``backend`` is accepted and ignored: the GPU grid replaces the
reference's chunk backend (backend.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .core import Vec3
from .errors import SingularityError
from .neighbor import DeviceStatus, NeighborLists, _stream
from .store import ParticleStore, device_of

__all__ = ["LennardJones", "SpringDashpot", "law_from_config", "lj_force", "spring_dashpot_force",
           "compute_forces"]

LAW_LJ, LAW_SD = 0, 1


def _dev_rows(a, device) -> torch.Tensor:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return torch.from_numpy(arr).to(device)


def _pair_force(law_id, p, delta, rsq, v_i=None, v_j=None):
    delta = np.asarray(delta, dtype=np.float64)
    rsq = np.asarray(rsq, dtype=np.float64)
    shape = np.broadcast_shapes(delta.shape[:-1], rsq.shape)
    d = np.broadcast_to(delta, shape + (3,)).reshape(-1, 3)
    r = np.broadcast_to(rsq, shape).reshape(-1)
    dev = device_of()
    dd, rr = _dev_rows(d, dev), _dev_rows(r, dev)
    vi = vj = None
    if v_i is not None and v_j is not None:
        vi = _dev_rows(np.broadcast_to(np.asarray(v_i, np.float64), shape + (3,)).reshape(-1, 3), dev)
        vj = _dev_rows(np.broadcast_to(np.asarray(v_j, np.float64), shape + (3,)).reshape(-1, 3), dev)
    out = torch.empty_like(dd)
    N.call("tmd_pair_force", law_id, dd.data_ptr(), rr.data_ptr(), vi.data_ptr() if vi is not None else 0,
           vj.data_ptr() if vj is not None else 0, r.size, p[0], p[1], p[2], out.data_ptr(), _stream())
    return out.cpu().numpy().reshape(shape + (3,))


def _pair_energy(law_id, p, rsq):
    rsq = np.asarray(rsq, dtype=np.float64)
    r = rsq.reshape(-1)
    dev = device_of()
    rr = _dev_rows(r, dev)
    out = torch.empty_like(rr)
    N.call("tmd_pair_energy", law_id, rr.data_ptr(), r.size, p[0], p[1], p[2], out.data_ptr(), _stream())
    return out.cpu().numpy().reshape(rsq.shape)


@dataclass(frozen=True)
class LennardJones:
    """Truncated 12-6 potential, force 48 eps sr6 (sr6 - 1/2) sr2 (potential.py:30-57)."""

    epsilon: float = 1.0
    sigma: float = 1.0
    cutoff: float = 2.5

    needs_velocities = False
    law_id = LAW_LJ

    @property
    def cutoff_rsq(self) -> float:
        return self.cutoff * self.cutoff

    @property
    def sigma6(self) -> float:
        return self.sigma**6

    def params(self):
        return (float(self.epsilon), float(self.sigma6), float(self.cutoff))

    def pair_force(self, delta, rsq, v_i=None, v_j=None) -> np.ndarray:
        return _pair_force(LAW_LJ, self.params(), delta, rsq)

    def pair_energy(self, rsq) -> np.ndarray:
        return _pair_energy(LAW_LJ, self.params(), rsq)


@dataclass(frozen=True)
class SpringDashpot:
    """Linear normal contact K ov n - gamma (n.vrel) n (potential.py:60-97)."""

    stiffness: float = 100.0
    damping: float = 0.0
    diameter: float = 1.0

    needs_velocities = True
    law_id = LAW_SD

    @property
    def cutoff_rsq(self) -> float:
        return self.diameter * self.diameter

    def params(self):
        return (float(self.stiffness), float(self.damping), float(self.diameter))

    def pair_force(self, delta, rsq, v_i=None, v_j=None) -> np.ndarray:
        return _pair_force(LAW_SD, self.params(), delta, rsq, v_i, v_j)

    def pair_energy(self, rsq) -> np.ndarray:
        return _pair_energy(LAW_SD, self.params(), rsq)


def law_from_config(cfg):
    """potential.py:100-105."""
    if cfg.potential_kind == "lj":
        return LennardJones(cfg.epsilon, cfg.sigma, cfg.cutoff)
    if cfg.potential_kind == "sd":
        return SpringDashpot(cfg.stiffness, cfg.damping, cfg.diameter)
    raise ValueError(f"unknown potential {cfg.potential_kind!r}")


def lj_force(delta: Vec3, rsq: float, epsilon: float, sigma: float) -> Vec3:
    """Force on i from one LJ partner (potential.py:108-113)."""
    if rsq == 0.0:
        raise SingularityError("coincident particles in Lennard-Jones force")
    return Vec3.from_array(LennardJones(epsilon, sigma).pair_force(delta.as_array(), np.float64(rsq)))


def spring_dashpot_force(delta: Vec3, rsq: float, v_i: Vec3, v_j: Vec3, stiffness: float,
                         damping: float, diameter: float) -> Vec3:
    """Contact force on sphere i (potential.py:116-131)."""
    if rsq == 0.0:
        raise SingularityError("coincident particles in spring-dashpot force")
    law = SpringDashpot(stiffness, damping, diameter)
    return Vec3.from_array(law.pair_force(delta.as_array(), np.float64(rsq), v_i.as_array(), v_j.as_array()))


def _singular_detail(lists: NeighborLists):
    def describe(code, key):
        if code != N.SINGULARITY:
            return ""
        i, k = key >> 32, key & 0xFFFFFFFF
        return f" and neighbor {lists.slot_atom(i, k)}"

    return describe


def launch_forces(store: ParticleStore, lists: NeighborLists, law, half: bool, energy: bool,
                  exact: bool, thermo: torch.Tensor, status: DeviceStatus) -> None:
    """Enqueue the force kernel for `law` (no host synchronisation)."""
    if lists.order != "reference":
        raise ValueError("compute_forces needs reference-order lists; split rows are consumed by the "
                         "fused step kernel only")
    flags = (N.F_ENERGY if energy else 0) | (N.F_EXACT if exact else 0)
    n = store.n_local
    pos, vel, frc = store.pos, store.vel, store.frc
    if half:
        p = law.params()
        N.call("tmd_force_half", pos.data_ptr(), vel.data_ptr(), store.ld, n, lists.nbr.data_ptr(),
               lists.ld_nbr, lists.d_counts.data_ptr(), law.law_id, p[0], p[1], p[2], flags,
               frc.data_ptr(), store.ld, thermo.data_ptr(), status.ptr, _stream())
    elif law.law_id == LAW_LJ:
        N.call("tmd_force_lj", pos.data_ptr(), store.ld, n, lists.nbr.data_ptr(), lists.ld_nbr,
               lists.d_counts.data_ptr(), lists.cap, float(law.cutoff_rsq), float(law.epsilon),
               float(law.sigma6), flags, frc.data_ptr(), store.ld, thermo.data_ptr(), status.ptr,
               _stream())
    else:
        N.call("tmd_force_sd", pos.data_ptr(), vel.data_ptr(), store.ld, n, lists.nbr.data_ptr(),
               lists.ld_nbr, lists.d_counts.data_ptr(), lists.cap, float(law.stiffness),
               float(law.damping), float(law.diameter), flags, frc.data_ptr(), store.ld,
               thermo.data_ptr(), status.ptr, _stream())


def compute_forces(store: ParticleStore, lists: NeighborLists, law, half: bool | None = None,
                   backend=None, accumulate_energy: bool = False, exact: bool = True,
                   return_virial: bool = False):
    """Evaluate pair forces into store.frc for every local (potential.py:134-213).

    Returns the total pair energy (full lists: 1/2 of the pair sum, half
    lists: the pair sum, as the reference) when ``accumulate_energy``, else
    None; with ``return_virial`` returns (energy, virial W = 1/2 sum delta.F).
    """
    if half is None:
        half = lists.half
    if half and not lists.half:
        raise ValueError("half-mode accumulation needs half-built lists")
    dev = store.device
    thermo = torch.zeros(2, dtype=torch.float64, device=dev)
    st = DeviceStatus(dev)
    energy = accumulate_energy or return_virial
    launch_forces(store, lists, law, half, energy, exact, thermo, st)
    if store.n_ghost:
        store.frc[:, store.n_local:store.n_total] = 0.0
    N.raise_for_status(st.read(), context="compute_forces", describe=_singular_detail(lists))
    if not energy:
        return None
    e, w = (float(x) for x in thermo.cpu().numpy())
    if return_virial:
        return e, w
    return e
