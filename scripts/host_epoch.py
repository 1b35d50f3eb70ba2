"""Host-side cost of a production epoch at P = 1: cProfile of rebuild() (with
the device time from CUDA events), after warm-up.

    python scripts/host_epoch.py [cells]
"""
import cProfile
import os
import pstats
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402


def main():
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    tr = None
    if "WORLD_SIZE" in os.environ:
        import torch.distributed as dist

        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        tr = P.DistTransport()
    grid = P.factor_rank_grid(tr.size if tr else 1)
    cfg = P.SimConfig(unit_cells=tuple(cells * g for g in grid), steps=200)
    sim = P.Simulation(cfg, mode="fast", thermo_every=200, transport=tr)
    gen = sim.iter_steps()
    for _ in range(90):
        next(gen)
    torch.cuda.synchronize()
    walls = []
    prof = cProfile.Profile()
    for rep in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record()
        if rep >= 2:
            prof.enable()
        sim.rebuild()
        if rep >= 2:
            prof.disable()
        e1.record()
        torch.cuda.synchronize()
        walls.append(((time.perf_counter() - t0) * 1e3, e0.elapsed_time(e1)))
    if tr is None or tr.rank == 0:
        print("rebuild wall/device ms:", [(round(a, 2), round(b, 2)) for a, b in walls])
        st = pstats.Stats(prof)
        st.sort_stats("tottime").print_stats(30)


if __name__ == "__main__":
    main()
