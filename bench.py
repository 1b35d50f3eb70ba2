#!/usr/bin/env python
"""Benchmark: atom-steps/s of the LJ fcc timestep (rc = 2.5, skin 0.3, reneighbor every 20).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...

Workload (default ``--workload weak``): the BASELINE weak-scaling series,
2,048,000 atoms per GPU — 80x80x80 fcc unit cells at N = 1, 160x80x80 at 2,
160x160x80 at 4, 160x160x160 (16,384,000 atoms) at 8 — one rank per GPU, 3-D
domain decomposition, NCCL halo traffic.  ``--workload c2`` runs BASELINE
configs[1] (32^3 = 131,072 atoms on one GPU), ``c3`` the 64^3 strong-scaling
system.  A "step" is one velocity-Verlet timestep of the whole system; the K
timed steps include the rebuild epochs that fall in them (every 20 steps).

Prints ONE JSON line on rank 0 (see the keys in `main`).  ``--impl
reference`` times the reference's CPU implementation of the path (the oracle/
numpy restatement of nanopair; the product package is not imported) on this
host's cores: the same workload, steps and warm-up on all threads (the
per-GPU 80^3 slice when the system exceeds 2,048,000 atoms), plus two more
steps on one thread as the serial leg.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "atom-steps/sec (LJ fcc, rc=2.5) at 1/2/4/8 B200; % of HBM roofline"
UNIT = "atom-steps/s"
# algorithmic bytes per atom-step of the force kernel:
# 4 B x 78 list entries + 4 B count + 24 B x_i + 24 B F_i
BYTES_PER_ATOM_STEP = 4 * 78 + 4 + 24 + 24
# FP64 lane operations per atom-step of the LJ force kernel:
# 9 per list candidate (78) + 12 per in-cutoff pair (55)
FP64_LANE_OPS_PER_ATOM_STEP = 78 * 9 + 55 * 12

WEAK_CELLS = {1: (80, 80, 80), 2: (160, 80, 80), 4: (160, 160, 80), 8: (160, 160, 160)}


def workload_cells(name: str, n: int):
    if name == "weak":
        if n in WEAK_CELLS:
            return WEAK_CELLS[n], "LJ fcc weak-scaling series, 2,048,000 atoms/GPU (BASELINE configs[3])"
        k = round((n * 80**3) ** (1 / 3))
        return (k, k, k), "LJ fcc weak-scaling series (non-standard N)"
    if name == "c2":
        return (32, 32, 32), "LJ fcc 32x32x32, 131,072 atoms (BASELINE configs[1])"
    if name == "c3":
        return (64, 64, 64), "LJ fcc 64x64x64, 1,048,576 atoms strong scaling (BASELINE configs[2])"
    if name == "c1":
        return (8, 8, 8), "LJ fcc 8x8x8, 2,048 atoms (BASELINE configs[0])"
    if name == "c5":
        return (40, 40, 40), "Spring-Dashpot DEM 40x40x40, 256,000 spheres, d = 1.2, K = 100, gamma = 0.5 (SURVEY 8(d) C5)"
    raise SystemExit(f"unknown workload {name}")


def workload_overrides(name: str) -> dict:
    """SimConfig fields beyond the unit cells (LJ defaults otherwise)."""
    if name == "c5":
        return dict(potential_kind="sd", diameter=1.2, cutoff=1.2, stiffness=100.0, damping=0.5)
    return {}


def bytes_per_atom_step(name: str) -> float:
    """Algorithmic bytes of the force kernel per atom-step."""
    return 124.0 if name == "c5" else BYTES_PER_ATOM_STEP


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 100 ms in a reader
    thread; ``stop(t0, t1)`` summarises the samples taken from just before the
    timed region to just after it (the region can be shorter than the sampling
    period, so the bracketing samples are kept and counted)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.lines = []  # (monotonic time, line)
        self.proc = None
        if os.environ.get("BENCH_NO_CLOCKS") == "1":  # diagnostics only
            return
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_first(self, timeout: float = 15.0) -> None:
        """Block until nvidia-smi produced its first sample (its start-up can take seconds)."""
        t_end = time.monotonic() + timeout
        while self.proc is not None and not self.lines and time.monotonic() < t_end:
            time.sleep(0.02)

    def stop(self, t0: float | None = None, t1: float | None = None):
        if self.proc is None:
            return None
        if t1 is not None:  # one sample after the region
            t_end = time.monotonic() + 1.0
            while not any(t > t1 for t, _ in self.lines) and time.monotonic() < t_end:
                time.sleep(0.01)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        lines = self.lines
        if t0 is not None and t1 is not None:
            before = [x for x in lines if x[0] <= t0]
            inside = [x for x in lines if t0 < x[0] <= t1]
            after = [x for x in lines if x[0] > t1]
            lines = before[-1:] + inside + after[:1]
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for _, ln in lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, val in zip(names, parts[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "note": f"nvidia-smi gave no usable sample ({len(self.lines)} lines)"}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm), "window": "last sample before, all inside, first after the timed region"}


# ---------------------------------------------------------------------------
# CPU legs (the oracle is the checker/baseline, never the thing measured for "value")
# ---------------------------------------------------------------------------

def _cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_rate(cells, steps: int, warmup: int, threads: int, serial_steps: int = 0, overrides=None):
    """Time oracle steps warmup+1 .. warmup+steps of an fcc run on `threads` host
    threads (setup excluded), then `serial_steps` more steps on one thread.

    Only the oracle is imported (its own OracleConfig): the product package and
    its CUDA library are never loaded on this path."""
    import oracle as O

    cfg = O.OracleConfig(unit_cells=tuple(cells), steps=warmup + steps + serial_steps, **(overrides or {}))
    marks = {}
    last = warmup + steps

    def hook(step, world):
        marks[step] = time.perf_counter()

    O.run(cfg, 1, threads=lambda k: threads if k <= last else 1, on_step=hook)
    n = cfg.n_atoms()
    dt = marks[last] - marks[warmup]
    out = {"value": n * steps / dt, "seconds": dt, "n": n,
           "rebuilds": sum(1 for k in range(warmup + 1, last + 1) if k % cfg.reneigh_interval == 0)}
    if serial_steps:
        ds = marks[last + serial_steps] - marks[last]
        out["serial"] = {"value": n * serial_steps / ds, "seconds": ds,
                         "rebuilds": sum(1 for k in range(last + 1, last + serial_steps + 1)
                                         if k % cfg.reneigh_interval == 0)}
    return out


# the largest system the CPU arm runs in full (C4's per-GPU slice); larger
# configurations (the weak series at N > 1) are timed on this per-rank slice
CPU_MAX_ATOMS = 2_048_000
REF_MAX_STEPS = 20


def reference_arm(args, n_gpus, rank):
    """--impl reference: the reference's CPU implementation of the path (the
    oracle port of nanopair, all host threads in the force phase, as
    NANOPAIR_THREADS does) on this host, same workload, steps and warm-up."""
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    cells_w, desc = workload_cells(args.workload, n_gpus)
    cells = cells_w
    if 4 * int(np.prod(cells_w)) > CPU_MAX_ATOMS:
        cells, _ = workload_cells(args.workload, 1)
    serial_steps = 2
    # a bounded sample of the run: at most REF_MAX_STEPS timed steps (with the
    # default reneighbour interval of 20, one in-loop rebuild -- the cost mix of
    # the full run), so the arm ends within a few minutes at 80^3
    timed = min(args.steps, REF_MAX_STEPS)
    r = oracle_rate(cells, timed, args.warmup, cores, serial_steps, workload_overrides(args.workload))
    same = tuple(cells) == tuple(cells_w)
    sample = (f"{'the full workload' if same else 'per-GPU slice of the workload (bounded sample)'}: "
              f"{cells[0]}x{cells[1]}x{cells[2]} fcc = {r['n']} atoms, oracle/ numpy port of nanopair, "
              f"steps {args.warmup + 1}..{args.warmup + timed} ({r['rebuilds']} rebuild(s)) after setup"
              f"{'' if timed == args.steps else f' (of the {args.steps} requested)'}, "
              f"force phase on {cores} threads; CPU: {_cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": r["value"], "unit": UNIT, "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["seconds"] / timed * 1e3,
        "higher_is_better": True, "scaling": "weak" if args.workload == "weak" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic perfect-fcc lattice, rho 0.8442, PCG64(42) velocities (the reference's create_lattice)",
        "config": {"workload": desc, "unit_cells": list(cells_w), "timed_unit_cells": list(cells),
                   "timed_steps": timed, "same_config": same},
        "cpu_baseline": {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "port", "sample": sample},
        "cpu_serial": {"value": r["serial"]["value"], "unit": UNIT, "cores": 1, "kind": "port",
                       "sample": f"{serial_steps} further steps of the same run on one thread "
                                 f"({r['serial']['rebuilds']} rebuilds), {r['serial']['seconds']:.1f} s"},
        "e2e": {"value": r["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def device_rate(P, cfg, K: int, W: int, dev):
    """Device-timed throughput of K steps after W warm-up steps of one rank's
    run of cfg (CUDA events on the stream; step kernels timed individually)."""
    import torch

    # one untimed run of the same system first (allocator pools, lazy driver
    # state), as the main measurement's pre-warm; no collector pass while timing
    P.Simulation(cfg, mode="fast", thermo_every=W + K, device=dev).run()
    sim = P.Simulation(cfg, mode="fast", thermo_every=W + K, device=dev)
    sim.start()  # setup epoch + step 0
    sim.advance(W)
    torch.cuda.synchronize(dev)
    sim.event_pairs = []
    sim.launch_times()  # reset
    gc.collect()
    gc_on = gc.isenabled()
    gc.disable()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    sim.advance(K)
    b.record()
    torch.cuda.synchronize(dev)
    if gc_on:
        gc.enable()
    kern = float(np.mean(sim.launch_times()))
    sim.advance(cfg.steps)
    ms = a.elapsed_time(b)
    n = sim.store.n_local
    return n * K / (ms * 1e-3), ms / K, kern, n


def load_traffic():
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh)
    except (OSError, ValueError):
        return {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="weak", choices=["weak", "c1", "c2", "c3", "c5"])
    ap.add_argument("--thermo-every", type=int, default=100)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-prewarm", action="store_true", help="skip the untimed warm-up run (profiling)")
    ap.add_argument("--no-secondary", action="store_true", help="skip the C5 DEM secondary measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n_gpus = world if world > 1 else args.gpus
    if args.impl == "reference":
        reference_arm(args, n_gpus, rank)
        return
    if args.gpus > 1 and world == 1:
        # one process per GPU: relaunch under torchrun (as the driver does)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("BENCH_MASTER_PORT", "29531"),
               os.path.abspath(__file__), *sys.argv[1:]]
        os.execv(sys.executable, cmd)

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    transport = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_2009_07400_b200 as P
    from paper_2009_07400_b200 import _native as N

    if world > 1:
        transport = P.DistTransport()
    cells, desc = workload_cells(args.workload, n_gpus)
    cfg = P.SimConfig(unit_cells=cells, steps=args.warmup + args.steps, **workload_overrides(args.workload))
    K, W = args.steps, args.warmup

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------- process warm-up (untimed): a short small run over the same
    # communicator so NCCL's lazily created connections (all-to-all, all-gather),
    # the CUDA-IPC driver state and the stream-ordered pools exist before timing
    # (same size as the measured run, so the caching allocator and the stream-ordered
    # pools already hold blocks of every size the epochs ask for)
    # the clock sampler (nvidia-smi -lms) starts first: its start-up (seconds on a
    # busy 8-GPU host) overlaps the warm-up; it samples through the timed steps
    sampler = ClockSampler(local)
    if not args.no_prewarm:
        warm_steps = int(os.environ.get("BENCH_PREWARM_STEPS", "101"))
        warm_cfg = P.SimConfig(unit_cells=cells, steps=warm_steps, **workload_overrides(args.workload))
        P.Simulation(warm_cfg, transport=transport, mode="fast", thermo_every=warm_steps, device=dev).run()
        barrier()

    # ---------------- device-resident run: W warm-up steps then K timed steps
    sim = P.Simulation(cfg, transport=transport, mode="fast", thermo_every=args.thermo_every, device=dev)
    sim.event_pairs = []
    # the production loop: one library call per epoch launches its steps
    # (Simulation.advance -> tmd_run_steps), each launch bracketed by CUDA events
    sim.start()  # setup epoch + step 0
    sim.advance(W)  # W warm-up steps
    barrier()
    sim.launch_times()  # drop the warm-up launches' times
    launches0 = N.launch_count()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    sampler.wait_first()
    # no cyclic-GC pass inside the timed region (as timeit does): a gen-2 pass in
    # one rank stalls every rank at the next epoch's collectives
    gc.collect()
    gc_was = gc.isenabled()
    if os.environ.get("BENCH_GC") != "1":
        gc.disable()
    barrier()
    h0 = time.monotonic()
    t_start.record()
    sim.advance(K)
    t_end.record()
    barrier()
    h1 = time.monotonic()
    if gc_was:
        gc.enable()
    launches = N.launch_count() - launches0
    clocks = sampler.stop(h0, h1)
    kern_ms = sim.launch_times()
    sim.advance(cfg.steps)  # the rest of the configured run (none: cfg.steps = W + K)
    rep = sim.finish()
    elapsed_ms = max_over_ranks(t_start.elapsed_time(t_end))
    n_total = rep.n_atoms
    value = n_total * K / (elapsed_ms * 1e-3)
    # outliers inside the timed region (device time of a step kernel > 2 ms, host time of an epoch)
    slow = {"kernel_ms": [(i, round(ms, 2)) for i, ms in enumerate(kern_ms) if ms > 2.0],
            "epoch_host_ms": [(int(k), round(ms, 1)) for k, ms, _ in sim.epoch_wall if k > W],
            "epoch_at_s": [round(t, 2) for k, _, t in sim.epoch_wall if k > W]}
    if getattr(sim, "rebuild_trace", None):
        slow["rebuild_trace_ms"] = [{k: round(v, 2) for k, v in rec.items()} for rec in sim.rebuild_trace]
    if getattr(sim, "rebuild_events", None):
        slow["rebuild_device_ms"] = [{evs[q][0]: round(evs[q - 1][1].elapsed_time(evs[q][1]), 2)
                                      for q in range(1, len(evs))} for evs in sim.rebuild_events]
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        with open(os.path.join(ROOT, "gpurun_out", f"rebuild_trace_rank{rank}.json"), "w") as fh:
            json.dump({"trace": slow["rebuild_trace_ms"], "epoch_host_ms": sim.epoch_wall,
                       "device": slow.get("rebuild_device_ms"), "ticks": getattr(sim.halo, "ticks", None)}, fh)
    kern_avg = max_over_ranks(float(np.mean(kern_ms)) if kern_ms else float("nan"))
    kern_med = max_over_ranks(float(np.median(kern_ms)) if kern_ms else float("nan"))
    kern_max = max_over_ranks(float(np.max(kern_ms)) if kern_ms else float("nan"))
    n_local = sim.store.n_local
    algo_bytes = bytes_per_atom_step(args.workload) * n_local
    achieved = algo_bytes / (kern_avg * 1e-3) / 1e9
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
        peak, peak_src = float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        peak, peak_src = 6650.0, "fallback (B200_PROFILING.md)"
    traffic = load_traffic().get(f"{args.workload}_n{n_gpus}") or load_traffic().get(args.workload)
    # FP64 side of the roofline: ~1.36k FP64 lane-ops per LJ atom-step
    # (78 candidates x 9 + 55 in-cutoff pairs x 12) against the DFMA peak measured
    # on this pool by scripts/fp64_peak.cu (profiles/r2_fp64_peak.json)
    fp64 = None
    if args.workload != "c5":
        try:
            with open(os.path.join(ROOT, "profiles", "r2_fp64_peak.json")) as fh:
                lanes_peak = float(json.load(fh)["dfma_per_s"])
            src = "measured (profiles/r2_fp64_peak.json: scripts/fp64_peak.cu DFMA chains)"
        except (OSError, KeyError, ValueError):
            lanes_peak, src = 148 * 64 * 1.965e9, "datasheet (148 SMs x 64 FP64 lanes x 1.965 GHz)"
        ops = FP64_LANE_OPS_PER_ATOM_STEP * n_local / (kern_avg * 1e-3)
        fp64 = {"achieved_tflops": 2e-12 * ops, "peak_tflops": 2e-12 * lanes_peak, "frac": ops / lanes_peak,
                "lane_ops_per_atom_step": FP64_LANE_OPS_PER_ATOM_STEP, "peak_source": src}
    force_share = sum(kern_ms) / max(t_start.elapsed_time(t_end), 1e-9)

    # ---------------- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        pos_h = P.lattice_positions(cfg, cfg.domain())
        vel_h = P.lattice_velocities(cfg, pos_h.shape[0])
        e2e_cfg = cfg.with_overrides(steps=K)
        decomp = P.Decomposition(cfg.domain(), world, rank, cfg.interaction_radius())
        mine = decomp.owns(pos_h) if world > 1 else np.ones(pos_h.shape[0], dtype=bool)
        n_mine = int(mine.sum())
        # this rank's inputs and its result buffer in pinned host memory (allocated untimed)
        in_pos = torch.empty((n_mine, 3), dtype=torch.float64, pin_memory=True)
        in_vel = torch.empty((n_mine, 3), dtype=torch.float64, pin_memory=True)
        in_pos.numpy()[:] = pos_h[mine]
        in_vel.numpy()[:] = vel_h[mine]
        out = torch.empty((n_mine + n_mine // 8 + 1024, 6), dtype=torch.float64, pin_memory=True)
        # fault the result buffer in for DMA once (a first device->host copy into
        # freshly pinned pages is several times slower than the steady state)
        out.copy_(torch.zeros(out.shape, dtype=torch.float64, device=dev))
        torch.cuda.synchronize(dev)
        del sim  # return the device-resident run's buffers to the allocator cache
        # no collector pass inside the timed region (a full pass over the previous
        # run's objects stalled the host for tens of ms on some boxes)
        gc.collect()
        gc_on = gc.isenabled()
        gc.disable()
        barrier()
        t0 = time.perf_counter()
        # H2D inside the timed region: the pinned (pos, vel) of this rank
        store = P.ParticleStore.from_host(in_pos.numpy(), in_vel.numpy(), device=dev)
        t1 = time.perf_counter()
        sim2 = P.Simulation(e2e_cfg, store=store, decomp=decomp, transport=transport, mode="fast",
                            thermo_every=args.thermo_every, device=dev)
        t2 = time.perf_counter()
        rep2 = sim2.run()
        t3 = time.perf_counter()
        final = sim2.store.local_state(out=out[:sim2.store.n_local])  # D2H of the result
        barrier()
        t4 = time.perf_counter()
        if gc_on:
            gc.enable()
        t_e2e = max_over_ranks(t4 - t0)
        e2e_parts = {"from_host_ms": (t1 - t0) * 1e3, "init_ms": (t2 - t1) * 1e3, "run_ms": (t3 - t2) * 1e3,
                     "d2h_ms": (t4 - t3) * 1e3, "run_wall_steps_ms": rep2.wall_s * 1e3}
        h2d = 48 * n_mine
        d2h = final.nbytes + rep2.thermo.nbytes
        if world > 1:
            tt = torch.tensor([float(h2d), float(d2h)], dtype=torch.float64, device=dev)
            dist.all_reduce(tt)
            h2d, d2h = int(tt[0].item()), int(tt[1].item())
        e2e = {"value": rep2.n_atoms * K / t_e2e, "unit": UNIT, "h2d_bytes_per_step": h2d / K,
               "d2h_bytes_per_step": d2h / K, "wall_s": t_e2e, "rank0_parts": e2e_parts,
               "what": "ParticleStore.from_host(pinned pos, vel) (H2D) + Simulation.run(K) incl. setup "
                       "epoch + final state (pinned) and thermo D2H"}

    # ---------------- secondary workload on rank 0 at N = 1: the Spring-Dashpot DEM
    # configuration (BASELINE configs[4], C5), device-timed the same way
    secondary = None
    if rank == 0 and world == 1 and args.workload == "weak" and not args.no_secondary:
        c5cells, c5desc = workload_cells("c5", 1)
        c5cfg = P.SimConfig(unit_cells=c5cells, steps=W + K, **workload_overrides("c5"))
        # three timed runs, the median reported (the small system is host-sensitive)
        runs = sorted((device_rate(P, c5cfg, K, W, dev) for _ in range(3)), key=lambda t: t[0])
        v5, ms5, kern5, n5 = runs[1]
        bw5 = bytes_per_atom_step("c5") * n5 / (kern5 * 1e-3) / 1e9
        secondary = {"c5_dem": {"workload": c5desc, "value": v5, "unit": UNIT, "ms_per_step": ms5,
                                "runs": [r[0] for r in runs], "statistic": "median of 3 runs",
                                "steps": K, "warmup": W, "kernel": "tmd_step_sd", "kernel_ms": kern5,
                                "roofline": {"bound": "hbm", "achieved": bw5, "peak": peak, "unit": "GB/s",
                                             "frac": bw5 / peak, "algorithmic_bytes_per_atom_step":
                                                 bytes_per_atom_step("c5")}}}

    # ---------------- CPU baseline (oracle port) on rank 0 at N = 1
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        sc = (32, 32, 32) if args.workload != "c5" else (20, 20, 20)
        r = oracle_rate(sc, 20, 0, cores, 0, workload_overrides(args.workload))
        cpu = {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"oracle/ numpy port of nanopair, {sc[0]}^3 = {r['n']} atoms of the same model, "
                         f"steps 1..20 (1 rebuild), force phase on {cores} threads, {r['seconds']:.1f} s; "
                         f"CPU {_cpu_model()}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": n_gpus, "steps": K, "warmup": W,
            "ms_per_step": elapsed_ms / K, "higher_is_better": True,
            "scaling": "weak" if args.workload == "weak" else "strong",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic perfect-fcc lattice, rho 0.8442, PCG64(42) velocities (the reference's create_lattice)",
            "config": {"workload": desc, "unit_cells": list(cells), "n_atoms": n_total,
                       "atoms_per_gpu": n_total // n_gpus, "rank_grid": list(P.factor_rank_grid(n_gpus)),
                       "dt": cfg.dt, "cutoff": cfg.cutoff, "skin": cfg.verlet_buffer, "reneigh_every": 20,
                       "neighbor_list": "full", "thermo_every": args.thermo_every,
                       "l2": "inputs larger than L2 (neighbor lists alone are ~%.0f MB/GPU)" % (
                           4 * 83 * n_local / 1e6),
                       "parallelism": (f"3-D domain decomposition, {n_gpus} rank(s): direct exchange/borders "
                                       "all-to-all over NCCL per epoch, ghosts written by the owners' step kernel "
                                       "into peers' buffers over NVLink (CUDA IPC) + a per-step NVLink mailbox barrier "
                                       "(tmd_peer_sync); epoch count all-gathers over the same mailboxes"
                                       if n_gpus > 1 else "1 rank, periodic images written by the step kernel"),
                       "prewarm": "one untimed 101-step run of the same system before the measured run"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": ("tmd_step_sd (fused contact forces + integrate)" if args.workload == "c5"
                                    else "tmd_step_lj (fused force + integrate)"), "kernel_ms": kern_avg,
                         "kernel_ms_median": kern_med, "kernel_ms_max": kern_max, "launches_timed": len(kern_ms),
                         "algorithmic_bytes_per_launch": algo_bytes, "peak_source": peak_src,
                         "kernel_share_of_step": force_share, "fp64": fp64},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "secondary": secondary,
            "outliers": slow,
            "rebuilds_in_timed_region": int(sum(1 for k in range(W + 1, W + K + 1) if k % 20 == 0)),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
