"""bench.py's secondary C5 leg (device_rate) in isolation: first call vs second,
with the epoch host times, to see where a slow first measurement comes from."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2009_07400_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
if len(sys.argv) > 1 and sys.argv[1] == "big":
    cfg = P.SimConfig(unit_cells=(80, 80, 80), steps=105)
    P.Simulation(cfg, mode="fast", thermo_every=105, device=dev).run()
    print("ran the 80^3 run first", flush=True)
cells, _ = bench.workload_cells("c5", 1)
for rep in range(3):
    c5 = P.SimConfig(unit_cells=cells, steps=105, **bench.workload_overrides("c5"))
    t0 = time.perf_counter()
    v, ms, kern, n = bench.device_rate(P, c5, 100, 5, dev)
    print(f"rep {rep}: {v:.3e} atom-steps/s, {ms:.4f} ms/step, kernel {kern:.4f} ms, wall {time.perf_counter() - t0:.2f} s",
          flush=True)
