"""Kernel-level timeline of one production rebuild (torch.profiler / CUPTI).

    python scripts/profile_rebuild.py [cells]
Prints the CUDA kernels and host ops of the rebuild at step 40 with their
device times, and the wall time of the rebuild.
"""

import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    sd = len(sys.argv) > 2 and sys.argv[2] == "sd"
    extra = dict(potential_kind="sd", diameter=1.2, cutoff=1.2, stiffness=100.0, damping=0.5) if sd else {}
    cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=45, **extra)
    sim = P.Simulation(cfg, mode="fast", thermo_every=45)
    gen = sim.iter_steps()
    for _ in range(40):  # through step 39
        next(gen)
    torch.cuda.synchronize()
    for _ in range(3):  # warm rebuilds (outside the capture)
        sim.rebuild()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        t0 = time.perf_counter()
        sim.rebuild()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
    print(f"rebuild wall {wall * 1e3:.2f} ms")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=40, max_name_column_width=60))
    print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=25, max_name_column_width=60))
    os.makedirs("gpurun_out", exist_ok=True)
    prof.export_chrome_trace("gpurun_out/rebuild_trace.json")


if __name__ == "__main__":
    main()
