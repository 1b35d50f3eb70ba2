"""Host-side cost of a P = 1 production epoch (cProfile around Simulation.rebuild)
on the C5 DEM system and the 80^3 LJ system: where the Python/ctypes time goes."""
import cProfile
import io
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402

for name, cfg in (("c5", P.SimConfig(unit_cells=(40, 40, 40), steps=40, potential_kind="sd", diameter=1.2,
                                     cutoff=1.2, stiffness=100.0, damping=0.5)),
                  ("lj80", P.SimConfig(unit_cells=(80, 80, 80), steps=40))):
    sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
    g = sim.iter_steps()
    for _ in range(25):
        next(g)
    torch.cuda.synchronize()
    walls = []
    pr = cProfile.Profile()
    for _ in range(5):
        t0 = time.perf_counter()
        pr.enable()
        sim.rebuild()
        pr.disable()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
    s = io.StringIO()
    pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
    print(f"== {name}: rebuild wall ms {[round(w, 2) for w in walls]}")
    print(s.getvalue()[:6000])
