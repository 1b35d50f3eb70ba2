"""Phase times of the bench's end-to-end path (1 GPU): host arrays -> store,
Simulation setup epoch, K steps, final-state D2H.  Runs the path 3 times.

    python scripts/e2e_phases.py [cells] [steps]
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=K)
    pos_h = P.lattice_positions(cfg, cfg.domain())
    vel_h = P.lattice_velocities(cfg, pos_h.shape[0])
    P.Simulation(cfg.with_overrides(steps=41), mode="fast", thermo_every=41).run()  # warm-up
    for rep in range(3):
        torch.cuda.synchronize()
        t = [time.perf_counter()]
        store = P.ParticleStore.from_host(pos_h, vel_h)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        sim = P.Simulation(cfg, store=store, mode="fast", thermo_every=K)
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        gen = sim.iter_steps()
        next(gen)  # setup epoch + step-0 force
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        for _ in gen:
            pass
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        rep_ = sim.finish()
        final = sim.store.local_state()
        t.append(time.perf_counter())
        names = ["from_host", "Simulation()", "setup epoch", f"{K} steps", "finish+D2H"]
        print(f"rep {rep}: " + ", ".join(f"{n} {(b - a) * 1e3:.1f} ms" for n, a, b in zip(names, t, t[1:])) +
              f"; total {(t[-1] - t[0]) * 1e3:.1f} ms", flush=True)
        del sim, gen, store, final, rep_


if __name__ == "__main__":
    main()
