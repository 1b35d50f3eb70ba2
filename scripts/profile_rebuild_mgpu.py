"""One production epoch at P > 1 (torchrun): wall time per phase (host clock,
TMD_TRACE_REBUILD=3: host clock + protocol sub-step ticks, no extra syncs) and rank 0's device kernels
under torch.profiler.

    torchrun --standalone --nproc-per-node N scripts/profile_rebuild_mgpu.py [cells_per_rank]
"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_07400_b200 as P  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, rank = dist.get_world_size(), dist.get_rank()
    cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    grid = P.factor_rank_grid(n)
    cfg = P.SimConfig(unit_cells=tuple(cells * g for g in grid), steps=200)
    sim = P.Simulation(cfg, transport=P.DistTransport(), mode="fast", thermo_every=200)
    gen = sim.iter_steps()
    for _ in range(40):
        next(gen)
    torch.cuda.synchronize()
    os.environ["TMD_TRACE_REBUILD"] = "3"
    walls = []
    for _ in range(4):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.rebuild()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
    if rank == 0:
        print(f"P={n} rebuild wall ms {[round(w, 2) for w in walls]}")
        for rec in sim.rebuild_trace[-3:]:
            print("   phases (host ms)", " ".join(f"{k} {v:.2f}" for k, v in rec.items()))
        for t in getattr(sim.halo, "ticks", [])[-8:]:
            print("   halo ticks", t)
    os.environ["TMD_TRACE_REBUILD"] = "0"
    import cProfile
    import io
    import pstats
    pr = cProfile.Profile()
    for _ in range(3):
        dist.barrier()
        torch.cuda.synchronize()
        pr.enable()
        sim.rebuild()
        pr.disable()
        torch.cuda.synchronize()
    if rank == 0:
        out = io.StringIO()
        pstats.Stats(pr, stream=out).sort_stats("tottime").print_stats(30)
        print(out.getvalue())
    dist.barrier()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        sim.rebuild()
        torch.cuda.synchronize()
    if rank == 0:
        print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
        import json
        import tempfile
        path = os.path.join(tempfile.gettempdir(), "rebuild_mgpu.json")
        prof.export_chrome_trace(path)
        with open(path) as fh:
            ev = json.load(fh)["traceEvents"]
        dev = sorted((e["ts"], e["ts"] + e.get("dur", 0), e["name"]) for e in ev
                     if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset"))
        busy = sum(b - a for a, b, _ in dev)
        span = dev[-1][1] - dev[0][0]
        print(f"device span {span / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, idle {(span - busy) / 1e3:.3f} ms")
        gaps = sorted(((dev[i + 1][0] - dev[i][1], dev[i][2][:40], dev[i + 1][2][:40]) for i in range(len(dev) - 1)),
                      reverse=True)[:12]
        for g, a, b in gaps:
            print(f"  gap {g:8.1f} us after {a!r} before {b!r}")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
