"""Kernel table of a 40-step window (two epochs) under torch.profiler, plus
the window's wall time without the profiler.

    python scripts/profile_window.py [c5|lj80|c3]
"""
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
if name == "c5":
    cfg = P.SimConfig(unit_cells=(40, 40, 40), steps=200, potential_kind="sd", diameter=1.2, cutoff=1.2,
                      stiffness=100.0, damping=0.5)
elif name == "c3":
    cfg = P.SimConfig(unit_cells=(64, 64, 64), steps=200)
else:
    cfg = P.SimConfig(unit_cells=(80, 80, 80), steps=200)
sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
g = sim.iter_steps()
for _ in range(25):
    next(g)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(40):
    next(g)
torch.cuda.synchronize()
print(f"{name}: 40-step window wall {1e3 * (time.perf_counter() - t0):.2f} ms (no profiler)")
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    for _ in range(40):
        next(g)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=60))
# GPU idle gaps between consecutive device activities (kernels, memcpy, memset)
import json, tempfile  # noqa: E402
path = os.path.join(tempfile.gettempdir(), f"window_{name}.json")
prof.export_chrome_trace(path)
with open(path) as fh:
    ev = json.load(fh)["traceEvents"]
dev = sorted((e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
             if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"))
busy = sum(b - a for a, b, _ in dev)
span = dev[-1][1] - dev[0][0]
gaps = [(dev[i + 1][0] - dev[i][1], dev[i][2][:40], dev[i + 1][2][:40]) for i in range(len(dev) - 1)]
big = sorted(gaps, reverse=True)[:15]
print(f"device span {span / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, idle {(span - busy) / 1e3:.3f} ms "
      f"in {sum(1 for g in gaps if g[0] > 2)} gaps > 2 us")
for g, a, b in big:
    print(f"  gap {g:8.1f} us after {a!r} before {b!r}")
