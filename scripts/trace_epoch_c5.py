"""Host time per phase of the P = 1 epoch (TMD_TRACE_REBUILD=2: host clock, no
extra syncs) on C5 and 80^3, after warm-up."""
import os
import sys

os.environ["TMD_TRACE_REBUILD"] = "2"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_07400_b200 as P  # noqa: E402

for name, cfg in (("c5", P.SimConfig(unit_cells=(40, 40, 40), steps=120, potential_kind="sd", diameter=1.2,
                                     cutoff=1.2, stiffness=100.0, damping=0.5)),
                  ("lj80", P.SimConfig(unit_cells=(80, 80, 80), steps=120))):
    sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
    sim.start()
    sim.advance(120)
    sim.finish()
    for rec in sim.rebuild_trace[-3:]:
        print(name, " ".join(f"{k} {v:.3f}" for k, v in rec.items()))
    print(name, "epoch host ms", [round(w, 3) for _, w, _ in sim.epoch_wall[-4:]])
