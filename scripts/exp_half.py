"""f2 data point: the half-list force kernel (tmd_force_half: reactions by fp64
atomics, potential.py:187-191) against the full-list kernels on the same 80^3
state -- pairs evaluated once instead of twice, at the cost of scattered
atomic reactions."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402
from paper_2009_07400_b200 import _native as N  # noqa: E402
from paper_2009_07400_b200.neighbor import build_cell_grid, build_neighbor_lists  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=0)
sim = P.Simulation(cfg, mode="exact")
for _ in sim.iter_steps():
    pass
s = sim.store
r = cfg.interaction_radius()
law = P.LennardJones()
st = torch.cuda.current_stream().cuda_stream
grid = build_cell_grid(s, cfg.domain(), r)
res = {}
for half in (False, True):
    L = build_neighbor_lists(s, grid, r, half=half)
    for exact in ((True, False) if not half else (True,)):
        flags = N.F_EXACT if exact else 0
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            if half:
                N.call("tmd_force_half", s.pos.data_ptr(), s.vel.data_ptr(), s.ld, s.n_local, L.nbr.data_ptr(),
                       L.ld_nbr, L.d_counts.data_ptr(), 0, law.epsilon, law.sigma6, cfg.cutoff, flags,
                       s.frc.data_ptr(), s.ld, 0, sim.status.ptr, st)
            else:
                N.call("tmd_force_lj", s.pos.data_ptr(), s.ld, s.n_local, L.nbr.data_ptr(), L.ld_nbr,
                       L.d_counts.data_ptr(), L.cap, law.cutoff_rsq, law.epsilon, law.sigma6, flags,
                       s.frc.data_ptr(), s.ld, 0, sim.status.ptr, st)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        name = ("half" if half else "full") + ("-exact" if exact else "-fast")
        res[name] = {"ms": float(np.median(ts)), "mean_row": float(L.d_counts[: s.n_local].float().mean())}
        print(name, res[name], flush=True)
