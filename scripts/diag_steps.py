"""Per-step fused-kernel time and pruning state of a single-GPU run (diagnostics).

    python scripts/diag_steps.py [cells] [steps]
"""

import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 45
    cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=steps)
    sim = P.Simulation(cfg, mode="fast", thermo_every=steps)
    sim.event_pairs = []
    for _ in sim.iter_steps():
        pass
    torch.cuda.synchronize()
    d2 = sim.dispmax2.cpu().numpy()
    lim = (0.5 * (sim.lists.near_margin - 1e-9)) ** 2
    nn = float(sim.lists.nnear[: sim.lists.n_local].float().mean())
    nt = float(sim.lists.d_counts[: sim.lists.n_local].float().mean())
    print(f"near mean {nn:.2f}  total mean {nt:.2f}  near d^2 limit {lim:.3e}")
    for k, (a, b) in enumerate(sim.event_pairs):
        print(f"step {k:3d} kernel {a.elapsed_time(b):7.3f} ms  d {np.sqrt(d2[k]):.4f}  back {'yes' if d2[k] > lim else 'no'}")


if __name__ == "__main__":
    main()
