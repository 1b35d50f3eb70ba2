"""Per-step device time of the fused kernel and of the step barrier on every
rank (diagnostics for multi-GPU jitter).

    torchrun --standalone --nproc-per-node N scripts/mgpu_stepdump.py [cells] [steps] [repeats]
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
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, rank = dist.get_world_size(), dist.get_rank()
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    grid = P.factor_rank_grid(n)
    tr = P.DistTransport()
    for rep in range(reps):
        cfg = P.SimConfig(unit_cells=tuple(cells * g for g in grid), steps=steps)
        sim = P.Simulation(cfg, transport=tr, mode="fast", thermo_every=steps)
        sim.event_pairs = []
        sim.launch_trace = []
        marks = []
        gen = sim.iter_steps()
        for k, _ in enumerate(gen):
            e = torch.cuda.Event(enable_timing=True)
            e.record()
            marks.append(e)
        torch.cuda.synchronize()
        kern = np.array([a.elapsed_time(b) for a, b in sim.event_pairs])
        step = np.array([marks[k].elapsed_time(marks[k + 1]) for k in range(len(marks) - 1)])
        slow_k = np.nonzero(kern > 1.0)[0].tolist()
        lt = [(k, round(ms, 1)) for k, ms in sim.launch_trace if ms > 1.0]
        print(f"rep {rep} rank {rank}: slow host launches {lt}", flush=True)
        slow_s = np.nonzero(step > 2.0)[0].tolist()
        print(f"rep {rep} rank {rank}: total {step.sum():.1f} ms, kernel med {np.median(kern):.3f}; "
              f"slow kernels {[(k, round(float(kern[k]), 1)) for k in slow_k]}; "
              f"slow steps {[(k + 1, round(float(step[k]), 1)) for k in slow_s]}", flush=True)
        sim.finish()
        del sim, gen
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
