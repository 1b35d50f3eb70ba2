"""Per-step diagnostics of the fused kernel under torchrun (kernel time, pruning
displacement, tier prefix length) — for performance debugging only.

    torchrun --standalone --nproc-per-node N scripts/diag_mgpu.py [cells]
"""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    tr = None
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        tr = P.DistTransport()
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    dims = {1: (cells,) * 3, 2: (2 * cells, cells, cells), 4: (2 * cells, 2 * cells, cells),
            8: (2 * cells,) * 3}[world]
    cfg = P.SimConfig(unit_cells=dims, steps=30)
    sim = P.Simulation(cfg, transport=tr, mode="fast", thermo_every=30)
    sim.event_pairs = []
    rows = []
    for step, _ in enumerate(sim.iter_steps()):
        torch.cuda.synchronize()
        L = sim.lists
        d2 = float(sim.dispmax2[step].item()) if step < sim.dispmax2.numel() else 0.0
        tc = L.tcnt[:, : L.n_local].float().mean(dim=1).cpu().numpy()
        rows.append((step, sim.event_pairs[-1][0].elapsed_time(sim.event_pairs[-1][1]), np.sqrt(d2), tc))
    rank = dist.get_rank() if world > 1 else 0
    s = sim.store
    print(f"[rank {rank}] n_local {s.n_local} n_ghost {s.n_ghost} cap {sim.lists.cap} grid dims {sim.grid.dims}"
          f" shell {sim.grid.shell}", flush=True)
    for step, ms, d, tc in rows[:25]:
        print(f"[rank {rank}] step {step:3d} kernel {ms:7.3f} ms  disp {d:.4f}  tier means "
              + " ".join(f"{x:.1f}" for x in tc), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
