"""tinyMD's pairwise-interaction timestep, B200-native.

A drop-in for the reference ``nanopair`` simulation API (lattice setup,
force-model selection, the per-step operators, ``run(steps)`` with thermo
output) whose every hot operation is a hand-written sm_100a kernel in
``libtinymd_b200.so``, called through a C ABI (include/tinymd_b200.h) with
torch tensors as device buffers and NCCL (torch.distributed) between ranks.

Importing the package loads the CUDA library; if it is missing the import
fails — there is no CPU fallback.
"""

from .core import AABB, SimConfig, Vec3, minimum_image, pbc_correct
from .errors import ConfigError, GuardViolation, NativeError, ProtocolError, SingularityError
from . import _native  # noqa: F401  (loads libtinymd_b200.so eagerly)
from .store import ParticleStore
from .lattice import create_lattice, lattice_positions, lattice_velocities
from .neighbor import (CellGrid, NeighborLists, build_cell_grid, build_neighbor_lists,
                       max_displacement_since_rebuild)
from .potential import (LennardJones, SpringDashpot, compute_forces, law_from_config, lj_force,
                        spring_dashpot_force)
from .comm import (BorderPlan, Decomposition, DistTransport, Halo, factor_rank_grid, rank_grid_coords,
                   rank_grid_index, slab_bounds)
from .driver import (PhaseTimers, RankReport, Report, Simulation, THERMO_COLUMNS, final_integrate,
                     initial_integrate, rank_program, run)
from .loopback import LoopbackTransport, LoopbackWorld, run_loopback

__all__ = [
    "AABB", "SimConfig", "Vec3", "minimum_image", "pbc_correct",
    "ConfigError", "GuardViolation", "NativeError", "ProtocolError", "SingularityError",
    "ParticleStore", "create_lattice", "lattice_positions", "lattice_velocities",
    "CellGrid", "NeighborLists", "build_cell_grid", "build_neighbor_lists",
    "max_displacement_since_rebuild",
    "LennardJones", "SpringDashpot", "compute_forces", "law_from_config", "lj_force",
    "spring_dashpot_force",
    "BorderPlan", "Decomposition", "DistTransport", "Halo", "factor_rank_grid", "rank_grid_coords",
    "rank_grid_index", "slab_bounds",
    "PhaseTimers", "RankReport", "Report", "Simulation", "THERMO_COLUMNS", "final_integrate",
    "initial_integrate", "rank_program", "run",
    "LoopbackTransport", "LoopbackWorld", "run_loopback",
]
