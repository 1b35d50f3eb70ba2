"""Kernel-level profile (torch.profiler / CUPTI) of regular steps, any world size.

    [torchrun --nproc-per-node N] python scripts/profile_steps.py [cells_per_rank] [steps]
Rank 0 prints per-kernel device time over `steps` consecutive non-epoch steps
(default 15, steps 22..36) and the device span of that window.
"""

import os
import sys

import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402
from paper_2009_07400_b200.comm import SingleRankTransport  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    multi = "WORLD_SIZE" in os.environ
    if multi:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    tr = P.DistTransport() if multi else SingleRankTransport()
    n, rank = tr.size, tr.rank
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
    grid = P.factor_rank_grid(n)
    cfg = P.SimConfig(unit_cells=tuple(cells * g for g in grid), steps=60)
    sim = P.Simulation(cfg, transport=tr, mode="fast", thermo_every=60)
    gen = sim.iter_steps()
    for _ in range(22):
        next(gen)
    torch.cuda.synchronize()
    if multi:
        dist.barrier()
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            next(gen)
        e1.record()
        torch.cuda.synchronize()
    if rank == 0:
        print(f"P={n}: {steps} steps, device span {e0.elapsed_time(e1):.3f} ms "
              f"({e0.elapsed_time(e1) / steps:.3f} ms/step)")
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
        print(prof.key_averages().table(sort_by="cpu_time_total", row_limit=20, max_name_column_width=70))
        prof.export_chrome_trace(os.path.join("gpurun_out", f"steps_trace_p{n}.json"))
    for _ in gen:
        pass
    if multi:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
