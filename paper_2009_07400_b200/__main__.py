"""Command line: input decks, presets, multi-rank runs, SimReport, XYZ trajectories.

    python -m paper_2009_07400_b200 --preset lj-32
    python -m paper_2009_07400_b200 --deck run.deck --steps 50 --ranks 4 --dump traj.xyz --dump-every 10
    torchrun --nproc-per-node 4 -m paper_2009_07400_b200 --nx 64 --ny 64 --nz 64 ...

The reference ships no CLI; SPEC.md:627-689 specifies one (module ``cli``) and
this follows it: a deck is ``key = value`` lines (``#`` comments) naming
``SimConfig`` fields (core.py:187-215) or run options (``ranks``,
``rank_grid``, ``balance``, ``dump``, ``dump_every``, ``mode``,
``thermo_every``); unknown keys and malformed values are errors that name the
line and the field; command-line flags override the deck, which overrides the
preset.  Ranks: under torchrun every process is one rank on its own GPU
(NCCL + NVLink); otherwise ``--ranks P`` runs P in-process ranks on this
process's GPU (loopback.py).  ``balance`` accepts only ``none`` (the
space-filling-curve balancer of SPEC.md:517-625 is not built).  The report
(SimReport) is line-oriented ``key value`` text, or one JSON object with
``--json``; an XYZ trajectory holds frames at steps 0, k, 2k, ... (particles
in lexicographic position order, 17 significant digits).
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys

import numpy as np

# `--ranks P` without torchrun runs P in-process ranks whose barrier kernels
# wait for each other: one hardware queue per stream (read at CUDA context
# creation, which happens later, on the first device use)
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

PRESETS = {
    # the paper's single-node configuration (32^3 x 4 LJ, 100 steps)
    "lj-32": dict(unit_cells=(32, 32, 32), steps=100, dt=0.005, cutoff=2.5, verlet_buffer=0.3,
                  reneigh_interval=20, epsilon=1.0, sigma=1.0, potential_kind="lj"),
    # SPEC.md:655 / 683: the diagonal half-filled Spring-Dashpot domain, K = gamma = 0, 1000 steps
    "sd-halfdomain": dict(potential_kind="sd", fill="half-diagonal", stiffness=0.0, damping=0.0, steps=1000),
}

RUN_OPTIONS = {"ranks": int, "rank_grid": str, "balance": str, "dump": str, "dump_every": int, "mode": str,
               "thermo_every": int}


class DeckError(ValueError):
    """A malformed deck line or value (names the line and the field)."""


def _config_fields():
    from .core import SimConfig

    return {f.name: f for f in dataclasses.fields(SimConfig)}


def _convert(name: str, raw: str, default):
    raw = raw.strip()
    if isinstance(default, bool):
        if raw.lower() in ("1", "true", "yes", "on"):
            return True
        if raw.lower() in ("0", "false", "no", "off"):
            return False
        raise ValueError(raw)
    if isinstance(default, int):
        return int(raw)
    if isinstance(default, float):
        return float(raw)
    if isinstance(default, tuple):
        parts = raw.replace("x", " ").replace(",", " ").split()
        return tuple(int(p) for p in parts)
    return raw


def parse_deck_text(text: str, where: str = "deck") -> dict:
    """``key = value`` lines -> {key: typed value} (SimConfig fields and run options)."""
    fields = _config_fields()
    out = {}
    for no, line in enumerate(text.splitlines(), 1):
        body = line.split("#", 1)[0].strip()
        if not body:
            continue
        if "=" not in body:
            raise DeckError(f"{where} line {no}: expected 'key = value', got {line.strip()!r}")
        key, raw = (p.strip() for p in body.split("=", 1))
        key = key.replace("-", "_")
        if key in fields:
            default = fields[key].default
        elif key in RUN_OPTIONS:
            default = RUN_OPTIONS[key]()
        else:
            raise DeckError(f"{where} line {no}: unknown key {key!r}")
        try:
            out[key] = _convert(key, raw, default)
        except ValueError:
            raise DeckError(f"{where} line {no}: bad value for {key}: {raw!r}") from None
    return out


def parse_deck(path: str) -> dict:
    with open(path) as fh:
        return parse_deck_text(fh.read(), where=path)


def _parse(argv):
    ap = argparse.ArgumentParser(prog="python -m paper_2009_07400_b200", description=__doc__.split("\n")[0])
    ap.add_argument("--preset", choices=sorted(PRESETS))
    ap.add_argument("--deck", help="input deck: key = value lines (SimConfig fields and run options)")
    ap.add_argument("--nx", type=int)
    ap.add_argument("--ny", type=int)
    ap.add_argument("--nz", type=int)
    ap.add_argument("--cells", type=int, nargs=3, metavar=("NX", "NY", "NZ"), help="fcc unit cells per axis")
    ap.add_argument("--steps", type=int)
    ap.add_argument("--dt", type=float)
    ap.add_argument("--cutoff", type=float, help="LJ cutoff / Spring-Dashpot contact diameter")
    ap.add_argument("--buffer", "--skin", dest="buffer", type=float, help="Verlet buffer (skin)")
    ap.add_argument("--reneigh-every", "--reneigh", dest="reneigh_every", type=int)
    ap.add_argument("--potential", choices=("lj", "sd"))
    ap.add_argument("--stiffness", type=float)
    ap.add_argument("--damping", type=float)
    ap.add_argument("--velocity-scale", type=float)
    ap.add_argument("--layout", help="aos | soa | aosoa:<c> (accepted; the device layout is fixed SoA)")
    ap.add_argument("--half-neigh", action="store_true", default=None, help="half neighbor lists (exact path)")
    ap.add_argument("--seed", type=int)
    ap.add_argument("--ranks", type=int, help="ranks (torchrun: the world size; else in-process ranks on one GPU)")
    ap.add_argument("--rank-grid", help="XxYxZ rank grid (default: the reference's near-cubic factorization)")
    ap.add_argument("--balance", choices=("none", "morton", "hilbert"))
    ap.add_argument("--mode", choices=("fast", "exact"),
                    help="fast: fused production kernels; exact: bitwise the reference's arithmetic")
    ap.add_argument("--thermo-every", type=int)
    ap.add_argument("--dump", help="XYZ trajectory (frames at step 0 and every --dump-every steps; else final)")
    ap.add_argument("--dump-every", type=int)
    ap.add_argument("--json", action="store_true", help="print the report as one JSON object")
    return ap.parse_args(argv)


def resolve(a):
    """Preset -> deck -> flags; returns (SimConfig, run options)."""
    from .core import SimConfig

    values = dict(PRESETS[a.preset]) if a.preset else {}
    if a.deck:
        values.update(parse_deck(a.deck))
    flags = {"steps": a.steps, "dt": a.dt, "verlet_buffer": a.buffer, "reneigh_interval": a.reneigh_every,
             "potential_kind": a.potential, "stiffness": a.stiffness, "damping": a.damping,
             "velocity_scale": a.velocity_scale, "rng_seed": a.seed, "half_neighbor": a.half_neigh,
             "ranks": a.ranks, "rank_grid": a.rank_grid, "balance": a.balance, "mode": a.mode,
             "thermo_every": a.thermo_every, "dump": a.dump, "dump_every": a.dump_every}
    values.update({k: v for k, v in flags.items() if v is not None})
    if a.layout:
        kind, _, c = a.layout.partition(":")
        values["layout_kind"] = kind
        if c:
            values["aosoa_cluster"] = int(c)
    cells = list(values.get("unit_cells", SimConfig.unit_cells))
    if a.cells:
        cells = list(a.cells)
    for d, v in enumerate((a.nx, a.ny, a.nz)):
        if v is not None:
            cells[d] = v
    values["unit_cells"] = tuple(int(c) for c in cells)
    if a.cutoff is not None:
        values["cutoff"] = a.cutoff
    opts = {k: values.pop(k) for k in list(values) if k in RUN_OPTIONS}
    if values.get("potential_kind") == "sd":
        # the contact law's range is its diameter (potential.py:77-78): --cutoff sets
        # both; the default d = 1.2 gives the fcc lattice its 12 contacts
        values.setdefault("diameter", values.get("cutoff", 1.2))
        values.setdefault("cutoff", values["diameter"])
    cfg = SimConfig(**values).validate()
    opts.setdefault("ranks", None)
    opts.setdefault("balance", "none")
    opts.setdefault("mode", "fast")
    opts.setdefault("thermo_every", max(1, min(10, cfg.steps or 1)))
    opts.setdefault("dump_every", 0)
    opts.setdefault("rank_grid", None)
    if opts["balance"] != "none":
        raise DeckError(f"balance={opts['balance']!r}: the space-filling-curve balancer (SPEC.md:517-625) is not "
                        "built; only 'none' is supported")
    if opts["rank_grid"]:
        opts["rank_grid"] = tuple(int(g) for g in str(opts["rank_grid"]).lower().replace("x", " ").split())
    return cfg, opts


# kept for scripts that build a config from the old flags
def config_from_args(a):
    return resolve(a)[0]


def species(cfg) -> str:
    return "Ar" if cfg.potential_kind == "lj" else "S"


def write_xyz(path: str, state: np.ndarray, species_name: str, comment: str, append: bool = False) -> None:
    """One XYZ frame: count, comment, then `A x y z` per
    particle at 17 significant digits (fp64 round-trips), lexicographic order."""
    pos = state[np.lexsort((state[:, 2], state[:, 1], state[:, 0]))][:, :3]
    with open(path, "a" if append else "w") as fh:
        fh.write(f"{pos.shape[0]}\n{comment}\n")
        for x, y, z in pos:
            fh.write(f"{species_name} {x:.17g} {y:.17g} {z:.17g}\n")


def read_xyz(path: str):
    """Frames of an XYZ file: [(comment, (n, 3) positions)]."""
    frames = []
    with open(path) as fh:
        lines = fh.read().splitlines()
    k = 0
    while k < len(lines):
        n = int(lines[k])
        comment = lines[k + 1]
        pos = np.array([[float(v) for v in ln.split()[1:4]] for ln in lines[k + 2:k + 2 + n]]).reshape(n, 3)
        frames.append((comment, pos))
        k += 2 + n
    return frames


def sim_report(cfg, opts, rep, counts, momentum0, momentum1, timers, guard_violations=0) -> dict:
    """SimReport: phase timers, steps/s, per-rank particle
    counts, final total momentum, config echo.  Timings aside, identical for
    identical deck + seed."""
    out = {"atoms": int(rep.n_atoms), "ranks": len(counts), "steps": int(rep.steps), "rebuilds": int(rep.rebuilds),
           "wall_s": float(rep.wall_s), "steps_per_s": float(rep.steps / rep.wall_s) if rep.wall_s > 0 else 0.0,
           "atom_steps_per_s": float(rep.atom_steps_per_s) if rep.steps else 0.0,
           "guard_violations": int(guard_violations), "mode": opts["mode"], "balance": opts["balance"]}
    for name in ("force", "neigh", "comm", "other"):
        out[f"timer_{name}_s"] = float(max(getattr(t, name) for t in timers))
    for r, c in enumerate(counts):
        out[f"particles_rank_{r}"] = int(c)
    out["momentum_initial"] = [float(v) for v in momentum0]
    out["momentum_final"] = [float(v) for v in momentum1]
    out["momentum_drift_max"] = float(np.max(np.abs(np.asarray(momentum1) - np.asarray(momentum0))))
    if rep.thermo.size:
        last = rep.thermo[-1]
        out.update(pe_final=float(last[1]), ke_final=float(last[2]), pressure_final=float(last[4]))
    for f in dataclasses.fields(cfg):
        v = getattr(cfg, f.name)
        out[f"config_{f.name}"] = list(v) if isinstance(v, tuple) else v
    return out


def format_report(report: dict) -> str:
    lines = []
    for k, v in report.items():
        if isinstance(v, (list, tuple)):
            v = " ".join(repr(x) if isinstance(x, float) else str(x) for x in v)
        elif isinstance(v, float):
            v = repr(v)
        lines.append(f"{k} {v}")
    return "\n".join(lines)


def _dump_due(k: int, every: int, steps: int) -> bool:
    return k % every == 0 if every > 0 else k == steps


def _run_single(cfg, opts, frames):
    """One rank per process (P = 1, or torchrun with the world size)."""
    import torch.distributed as dist

    from .comm import DistTransport
    from .driver import Simulation

    transport = DistTransport() if dist.is_available() and dist.is_initialized() else None
    every = opts["dump_every"] if opts.get("dump") else 0
    sim = Simulation(cfg, transport=transport, mode=opts["mode"], thermo_every=opts["thermo_every"],
                     exact_yields=every if every > 0 else False, rank_grid=opts["rank_grid"])
    for _, k in sim.iter_steps():
        if opts.get("dump") and every > 0 and _dump_due(k, every, cfg.steps):
            frames.setdefault(k, []).append(sim.store.local_state())
    rep = sim.finish()
    if opts.get("dump") and every <= 0:
        frames.setdefault(cfg.steps, []).append(sim.store.local_state())
    counts = [sim.store.n_local]
    if transport is not None:
        counts = [int(c) for c in transport.all_gather_object(sim.store.n_local)]
        for k in sorted(frames):
            parts = transport.all_gather_object(frames[k][0])
            frames[k] = parts
    p0 = rep.thermo[0, 5:8] if rep.thermo.size else np.zeros(3)
    p1 = rep.thermo[-1, 5:8] if rep.thermo.size else np.zeros(3)
    return rep, counts, p0, p1, [sim.timers]


def _run_loopback(cfg, opts, frames):
    """P in-process ranks on this process's GPU (loopback.py)."""
    import threading

    import torch

    from .driver import Simulation
    from .errors import ProtocolError
    from .loopback import LoopbackWorld

    P = int(opts["ranks"])
    world = LoopbackWorld(P)
    every = opts["dump_every"] if opts.get("dump") else 0
    dev = torch.device("cuda", torch.cuda.current_device())
    reps, sims, errors = [None] * P, [None] * P, [None] * P
    lock = threading.Lock()

    def body(rank):
        torch.cuda.set_device(dev)
        stream = torch.cuda.Stream(dev)
        tr = world.transport(rank)
        try:
            with torch.cuda.stream(stream):
                sim = Simulation(cfg, transport=tr, device=dev, mode=opts["mode"], thermo_every=opts["thermo_every"],
                                 exact_yields=every if every > 0 else False, rank_grid=opts["rank_grid"])
                sims[rank] = sim
                for _, k in sim.iter_steps():
                    if every > 0 and _dump_due(k, every, cfg.steps):
                        st = sim.store.local_state()
                        with lock:
                            frames.setdefault(k, [None] * P)[rank] = st
                reps[rank] = sim.finish()
                if opts.get("dump") and every <= 0:
                    st = sim.store.local_state()
                    with lock:
                        frames.setdefault(cfg.steps, [None] * P)[rank] = st
                stream.synchronize()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errors[rank] = e
            tr.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(P)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    first = next((e for e in errors if e is not None and not isinstance(e, ProtocolError)), None)
    first = first or next((e for e in errors if e is not None), None)
    if first is not None:
        raise first
    rep = reps[0]
    p0 = rep.thermo[0, 5:8] if rep.thermo.size else np.zeros(3)
    p1 = rep.thermo[-1, 5:8] if rep.thermo.size else np.zeros(3)
    return rep, [s.store.n_local for s in sims], p0, p1, [s.timers for s in sims]


def main(argv=None) -> int:
    a = _parse(sys.argv[1:] if argv is None else argv)
    try:
        cfg, opts = resolve(a)
    except (DeckError, ValueError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    import torch
    import torch.distributed as dist

    from .errors import GuardViolation

    multi = "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) > 1
    if multi:
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if opts["ranks"] not in (None, dist.get_world_size()):
            print(f"error: --ranks {opts['ranks']} under torchrun with {dist.get_world_size()} processes",
                  file=sys.stderr)
            return 2
    rank = dist.get_rank() if multi else 0
    frames = {}
    try:
        if not multi and opts["ranks"] and opts["ranks"] > 1:
            rep, counts, p0, p1, timers = _run_loopback(cfg, opts, frames)
        else:
            rep, counts, p0, p1, timers = _run_single(cfg, opts, frames)
    except GuardViolation as e:
        if rank == 0:
            print(f"error: guard violation: {e}", file=sys.stderr)
        return 3
    if rank == 0:
        report = sim_report(cfg, opts, rep, counts, p0, p1, timers)
        if a.json:
            report["thermo_columns"] = ["step", "pe", "ke", "virial", "pressure", "px", "py", "pz"]
            report["thermo"] = rep.thermo.tolist()
            print(json.dumps(report))
        else:
            print(rep.thermo_table())
            print(format_report(report))
        if opts.get("dump"):
            for n_frame, k in enumerate(sorted(frames)):
                state = np.vstack(frames[k])
                write_xyz(opts["dump"], state, species(cfg),
                          f"tinyMD {cfg.potential_kind} {list(cfg.unit_cells)} step {k}", append=n_frame > 0)
    if multi:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
