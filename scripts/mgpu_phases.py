"""Where a multi-GPU step spends its time (rank 0): per-step wall clock and a
cProfile of the host side, fused NVLink refresh vs three-round NCCL refresh.

    torchrun --standalone --nproc-per-node N scripts/mgpu_phases.py [cells_per_rank] [steps]
"""

import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402
from paper_2009_07400_b200.comm import SingleRankTransport  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    multi = "WORLD_SIZE" in os.environ
    if multi:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        n, rank = dist.get_world_size(), dist.get_rank()
    else:
        n, rank = 1, 0
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    grid = P.factor_rank_grid(n)
    cfg = P.SimConfig(unit_cells=tuple(cells * g for g in grid), steps=steps)
    tr = P.DistTransport() if multi else SingleRankTransport()
    asyn = os.environ.get("ASYNC", "0") == "1"
    for fused in (True, False, True):
        sim = P.Simulation(cfg, transport=tr, mode="fast", thermo_every=steps, fused_refresh=fused)
        prof = cProfile.Profile()
        walls = []
        gen = sim.iter_steps()
        next(gen)
        torch.cuda.synchronize()
        if multi:
            dist.barrier()
        prof.enable()
        last = time.perf_counter()
        sim.event_pairs = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in gen:
            if not asyn:
                torch.cuda.synchronize()
            now = time.perf_counter()
            walls.append(now - last)
            last = now
        e1.record()
        torch.cuda.synchronize()
        prof.disable()
        kern = np.array([a.elapsed_time(b) for a, b in sim.event_pairs])
        if rank == 0:
            print(f"-- device total {e0.elapsed_time(e1):.1f} ms; kernel median {np.median(kern):.3f} "
                  f"max {kern.max():.3f} ms; kernels > 1 ms: {int((kern > 1).sum())}", flush=True)
        sim.finish()
        if rank == 0 and getattr(sim, "rebuild_trace", None):
            for rec in sim.rebuild_trace:
                print("   rebuild", " ".join(f"{k} {v:.2f}" for k, v in rec.items()), flush=True)
        if rank == 0:
            w = np.array(walls) * 1e3
            reb = np.array([k for k in range(1, steps + 1) if sim.rebuild_steps[k]]) - 1
            mask = np.ones(len(w), bool)
            mask[reb] = False
            print(f"== P={n} fused_refresh={fused}: step median {np.median(w[mask]):.3f} ms, "
                  f"rebuild steps {np.round(w[reb], 2).tolist()} ms, total {w.sum():.1f} ms", flush=True)
            st = pstats.Stats(prof)
            st.sort_stats("tottime").print_stats(18)
        del sim
    if multi:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
