"""Device-synchronised phase breakdown of a run (diagnostics, not a bench number).

    python scripts/profile_phases.py [--cells 32] [--steps 40]
"""

import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2009_07400_b200 as P  # noqa: E402
from paper_2009_07400_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=32)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--mode", default="fast")
    a = ap.parse_args()
    cfg = P.SimConfig(unit_cells=(a.cells,) * 3, steps=a.steps)
    sim = P.Simulation(cfg, mode=a.mode, thermo_every=a.steps, profile=True)
    # time the individual pieces of one epoch
    t0 = time.perf_counter()
    gen = sim.iter_steps()
    next(gen)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    sim.timers = P.PhaseTimers()
    l0 = N.launch_count()
    t0 = time.perf_counter()
    for _ in gen:
        pass
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    tm = sim.timers
    n = sim.store.n_local
    print(f"atoms {n} ghosts {sim.store.n_ghost} steps {a.steps} rebuilds {sim.rebuilds - 1} "
          f"launches {N.launch_count() - l0}")
    print(f"setup {t_setup * 1e3:.1f} ms; steps wall {wall * 1e3:.1f} ms = {wall / a.steps * 1e3:.3f} ms/step")
    print(f"force {tm.force * 1e3:.2f} ms  comm {tm.comm * 1e3:.2f} ms  neigh {tm.neigh * 1e3:.2f} ms  "
          f"other {tm.other * 1e3:.2f} ms")
    # one isolated epoch, split
    s = sim.store
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    sim.halo.exchange(s)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    plan = sim.halo.define_borders(s)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    grid = P.build_cell_grid(s, sim.grid_box, sim.r)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    P.build_neighbor_lists(s, grid, sim.r, False)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"epoch: exchange {1e3 * (t1 - t0):.2f} ms borders {1e3 * (t2 - t1):.2f} ms "
          f"bin {1e3 * (t3 - t2):.2f} ms lists {1e3 * (t4 - t3):.2f} ms")
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.halo.synchronize(s, plan)
        torch.cuda.synchronize()
        print(f"sync {1e6 * (time.perf_counter() - t0):.1f} us", end="; ")
    print()


if __name__ == "__main__":
    main()
