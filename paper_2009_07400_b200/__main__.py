"""Command line: run a tinyMD system on this node's GPUs, print thermo, dump XYZ.

    python -m paper_2009_07400_b200 --cells 32 32 32 --steps 100 [--thermo-every 10]
        [--potential lj|sd] [--mode fast|exact] [--dump final.xyz] [--json]
    torchrun --nproc-per-node 4 -m paper_2009_07400_b200 --cells 64 64 64 ...

The reference ships no CLI (SPEC.md:627-689 describe one);
this is the thin user-facing wrapper over ``SimConfig`` + ``run`` that a
reference user would otherwise script.  Under torchrun every process is one
rank (NCCL); rank 0 prints and writes.  The XYZ dump holds the final
positions of all atoms (species ``Ar`` for LJ, ``S`` for spheres) in
lexicographic position order, the comparison order of the reference's tests.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np


def _parse(argv):
    ap = argparse.ArgumentParser(prog="python -m paper_2009_07400_b200", description=__doc__.split("\n")[0])
    ap.add_argument("--cells", type=int, nargs=3, default=(32, 32, 32), metavar=("NX", "NY", "NZ"),
                    help="fcc unit cells per dimension (4 atoms each)")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--thermo-every", type=int, default=10)
    ap.add_argument("--potential", choices=("lj", "sd"), default="lj")
    ap.add_argument("--mode", choices=("fast", "exact"), default="fast",
                    help="fast: fused production kernels; exact: bitwise the reference's arithmetic")
    ap.add_argument("--dt", type=float, default=0.005)
    ap.add_argument("--cutoff", type=float, default=None, help="LJ cutoff (default 2.5) / SD diameter")
    ap.add_argument("--skin", type=float, default=0.3)
    ap.add_argument("--reneigh", type=int, default=20)
    ap.add_argument("--stiffness", type=float, default=100.0)
    ap.add_argument("--damping", type=float, default=0.0)
    ap.add_argument("--velocity-scale", type=float, default=1.0)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--dump", default=None, help="write the final state as XYZ (rank 0)")
    ap.add_argument("--json", action="store_true", help="print the report as one JSON object")
    return ap.parse_args(argv)


def config_from_args(a):
    from .core import SimConfig

    kw = dict(unit_cells=tuple(int(c) for c in a.cells), steps=a.steps, dt=a.dt, verlet_buffer=a.skin,
              reneigh_interval=a.reneigh, potential_kind=a.potential, velocity_scale=a.velocity_scale,
              rng_seed=a.seed)
    if a.potential == "lj":
        kw["cutoff"] = 2.5 if a.cutoff is None else a.cutoff
    else:
        d = 1.2 if a.cutoff is None else a.cutoff
        kw.update(diameter=d, cutoff=d, stiffness=a.stiffness, damping=a.damping)
    return SimConfig(**kw).validate()


def write_xyz(path: str, state: np.ndarray, species: str, comment: str) -> None:
    """state: (N, 6) positions then velocities."""
    pos = state[np.lexsort((state[:, 2], state[:, 1], state[:, 0]))][:, :3]
    with open(path, "w") as fh:
        fh.write(f"{pos.shape[0]}\n{comment}\n")
        for x, y, z in pos:
            fh.write(f"{species} {x:.17g} {y:.17g} {z:.17g}\n")


def main(argv=None) -> int:
    a = _parse(sys.argv[1:] if argv is None else argv)
    import torch
    import torch.distributed as dist

    from .comm import DistTransport
    from .driver import Simulation

    multi = "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1
    transport = None
    if multi:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        transport = DistTransport()
    rank = transport.rank if transport else 0
    cfg = config_from_args(a)
    sim = Simulation(cfg, transport=transport, mode=a.mode, thermo_every=a.thermo_every)
    rep = sim.run()
    state = sim.store.local_state()
    if multi:
        parts = [None] * transport.size
        dist.all_gather_object(parts, state)
        state = np.vstack(parts)
    if rank == 0:
        if a.json:
            print(json.dumps({"atoms": rep.n_atoms, "steps": rep.steps, "wall_s": rep.wall_s,
                              "atom_steps_per_s": rep.atom_steps_per_s, "rebuilds": rep.rebuilds,
                              "thermo_columns": ["step", "pe", "ke", "virial", "pressure", "px", "py", "pz"],
                              "thermo": rep.thermo.tolist()}))
        else:
            print(rep.thermo_table())
            print(f"# {rep.n_atoms} atoms, {rep.steps} steps on {transport.size if transport else 1} GPU(s): "
                  f"{rep.wall_s:.3f} s, {rep.atom_steps_per_s:.4g} atom-steps/s, {rep.rebuilds} neighbor builds")
        if a.dump:
            write_xyz(a.dump, state, "Ar" if cfg.potential_kind == "lj" else "S",
                      f"tinyMD {cfg.potential_kind} {cfg.unit_cells} step {cfg.steps}")
    if multi:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
