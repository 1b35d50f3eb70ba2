"""Where the e2e D2H time goes (bench.py's e2e leg, timed in sub-steps)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=100)
pos_h = P.lattice_positions(cfg, cfg.domain())
vel_h = P.lattice_velocities(cfg, pos_h.shape[0])
n = pos_h.shape[0]
in_pos = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
in_vel = torch.empty((n, 3), dtype=torch.float64, pin_memory=True)
in_pos.numpy()[:] = pos_h
in_vel.numpy()[:] = vel_h
out = torch.empty((n + n // 8 + 1024, 6), dtype=torch.float64, pin_memory=True)
out.copy_(torch.zeros(out.shape, dtype=torch.float64, device=dev))
torch.cuda.synchronize()
for rep in range(3):
    t = [time.perf_counter()]
    store = P.ParticleStore.from_host(in_pos.numpy(), in_vel.numpy(), device=dev)
    t.append(time.perf_counter())
    sim = P.Simulation(cfg, store=store, mode="fast", thermo_every=100, device=dev)
    rep2 = sim.run()
    t.append(time.perf_counter())
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    s = sim.store
    k = s.n_local
    stage = torch.empty((int(k * 1.05) + 1024, 6), dtype=torch.float64, device=dev)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = stage[:k]
    d[:, 0:3] = s.pos[:, :k].t()
    d[:, 3:6] = s.vel[:, :k].t()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    out[:k].copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    final = s.local_state(out=out[:k])
    t.append(time.perf_counter())
    print(rep, "from_host, run, sync, stage alloc, transpose, copy, local_state ms:",
          [round((b - a) * 1e3, 2) for a, b in zip(t, t[1:])], flush=True)
    del sim, store, stage, d
