"""Wall vs device time of the epoch (rebuild) and of regular steps, no extra syncs.

    python scripts/profile_epoch.py [--cells 80] [--steps 60]
"""

import argparse
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2009_07400_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=80)
    ap.add_argument("--steps", type=int, default=60)
    a = ap.parse_args()
    cfg = P.SimConfig(unit_cells=(a.cells,) * 3, steps=a.steps)
    sim = P.Simulation(cfg, mode="fast", thermo_every=a.steps)
    orig = sim.rebuild
    rec = []

    def timed_rebuild():
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        orig()
        e1.record()
        t1 = time.perf_counter()
        rec.append((t1 - t0, e0, e1))

    sim.rebuild = timed_rebuild
    step_wall = []
    gen = sim.iter_steps()
    last = time.perf_counter()
    prof = cProfile.Profile()
    for k, _ in enumerate(gen):
        now = time.perf_counter()
        step_wall.append(now - last)
        last = now
        if k == 39:
            prof.enable()
        if k == 40:
            prof.disable()
    torch.cuda.synchronize()
    for wall, e0, e1 in rec:
        print(f"rebuild: host wall {wall * 1e3:7.2f} ms   device span {e0.elapsed_time(e1):7.2f} ms")
    sw = sorted(step_wall[2:])
    print(f"host time per yielded step: median {sw[len(sw) // 2] * 1e3:.3f} ms  max {sw[-1] * 1e3:.2f} ms")
    print(f"run wall (steps 1..K, synced): {sim.wall * 1e3:.1f} ms = {sim.wall / a.steps * 1e3:.3f} ms/step")
    pstats.Stats(prof).sort_stats("cumtime").print_stats(25)


if __name__ == "__main__":
    main()
