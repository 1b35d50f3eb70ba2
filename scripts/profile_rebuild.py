"""Per-primitive, device-synchronised timing of one rebuild epoch (diagnostics).

    python scripts/profile_rebuild.py [--cells 32]
"""

import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2009_07400_b200 as P  # noqa: E402
from paper_2009_07400_b200 import neighbor as NB  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cells", type=int, default=32)
    a = ap.parse_args()
    cfg = P.SimConfig(unit_cells=(a.cells,) * 3, steps=4)
    sim = P.Simulation(cfg, mode="fast", thermo_every=4)
    sim.run()  # warm everything up (allocator pools, module loads)
    acc = collections.defaultdict(float)
    cnt = collections.Counter()

    def wrap(obj, name):
        fn = getattr(obj, name)

        def timed(*args, **kw):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = fn(*args, **kw)
            torch.cuda.synchronize()
            acc[name] += time.perf_counter() - t0
            cnt[name] += 1
            return out

        setattr(obj, name, timed)

    for name in ("select_pair", "select", "emit_ghosts", "flatten_plan", "wrap_self", "any_outside",
                 "pack_pos_vel", "compact_locals", "plan_shift", "pack_pos"):
        if hasattr(sim.halo.ops, name):
            wrap(sim.halo.ops, name)
    for name in ("exchange", "define_borders"):
        wrap(sim.halo, name)
    for name in ("build_cell_grid", "build_neighbor_lists"):
        wrap(NB, name)
    import paper_2009_07400_b200.driver as D

    D.build_cell_grid = NB.build_cell_grid
    D.build_neighbor_lists = NB.build_neighbor_lists
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sim.rebuild()
        torch.cuda.synchronize()
        acc["rebuild total"] += time.perf_counter() - t0
        cnt["rebuild total"] += 1
    for k in sorted(acc, key=lambda k: -acc[k]):
        print(f"{k:24s} {1e3 * acc[k] / cnt[k]:9.3f} ms/call  x{cnt[k] // 3}")
    # host-side view of one epoch (sync waits show up in .cpu()/.item()/tolist)
    import cProfile
    import pstats

    prof = cProfile.Profile()
    torch.cuda.synchronize()
    prof.enable()
    sim.rebuild()
    torch.cuda.synchronize()
    prof.disable()
    pstats.Stats(prof).sort_stats("tottime").print_stats(18)
    # list builders in isolation
    s = sim.store
    grid = P.build_cell_grid(s, sim.grid_box, sim.r)
    for order in ("reference", "tiered"):
        prev = None
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            prev = P.build_neighbor_lists(s, grid, sim.r, False, order=order, cutoff=cfg.cutoff, reuse=prev)
            torch.cuda.synchronize()
            print(f"lists[{order}] call {rep}: {1e3 * (time.perf_counter() - t0):.3f} ms")
        del prev


if __name__ == "__main__":
    main()
