"""Decompose the production step kernel's time on the 80^3 state at a given
step of an epoch: forces only (phases 0) vs + closing kick (1) vs + next kick,
drift, guard (3), with the exact pruning on and forced off, and the mean
front / full row lengths."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import ctypes as C  # noqa: E402
import subprocess  # noqa: E402

import paper_2009_07400_b200 as P  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "exp_step4.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       "-o", so, os.path.join(here, "exp_step4.cu")])
exp = C.CDLL(so)
from paper_2009_07400_b200 import _native as N  # noqa: E402

cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
for stop in [int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else "61,70,79").split(",")]:
    cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=stop + 5)
    sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
    g = sim.iter_steps()
    for _ in range(stop + 1):
        next(g)
    torch.cuda.synchronize()
    s, L, law = sim.store, sim.lists, sim.law
    n = s.n_local
    st = torch.cuda.current_stream().cuda_stream
    scratch = torch.empty_like(s.pos)
    vel0 = s.vel.clone()
    d2 = torch.zeros(1, dtype=torch.float64, device=s.device)
    ref = L.ref_positions_dev
    N.call("tmd_max_disp2", s.pos.data_ptr(), s.ld, ref.data_ptr(), ref.stride(0), n, d2.data_ptr(), st)
    out2 = torch.zeros(1, dtype=torch.float64, device=s.device)
    thermo = torch.zeros(6, dtype=torch.float64, device=s.device)
    print(f"step {stop}: max disp {float(d2.sqrt()):.4f} margin {L.near_margin:.4f}  mean front "
          f"{float(L.nnear[:n].float().mean()):.1f} mean row {float(L.d_counts[:n].float().mean()):.1f}", flush=True)
    cnt = L.nnear[:n].contiguous()
    outx = torch.zeros((3, s.ld), dtype=torch.float64, device=s.device)
    for v in (0, 5):
        ts = []
        for _ in range(15):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            exp.exp_step4(C.c_int(v), C.c_void_p(s.pos.data_ptr()), C.c_int64(s.ld), C.c_void_p(L.nbr.data_ptr()),
                          C.c_int64(L.ld_nbr), C.c_void_p(cnt.data_ptr()), C.c_int32(n), C.c_double(6.25),
                          C.c_void_p(outx.data_ptr()), C.c_void_p(st))
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        print(f"  exp_step4 variant {v} (front only, forces only): {np.median(ts):.4f} ms", flush=True)
    for phases in (0, 1, 3):
        for flags in (0, N.F_NO_PRUNE):
            ts = []
            for _ in range(15):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record()
                N.call("tmd_step_lj", s.pos.data_ptr(), scratch.data_ptr(), s.vel.data_ptr(), s.ld, n,
                       L.nbr.data_ptr(), L.ld_nbr, L.d_counts.data_ptr(), L.nnear.data_ptr(), L.cap,
                       float(L.near_margin), d2.data_ptr(), 0, 0, 0, 0, 0, 0, 0, 0, 0, float(law.cutoff_rsq),
                       float(law.epsilon), float(law.sigma6), 0.0025, 0.005, phases, flags, s.frc.data_ptr(), s.ld,
                       ref.data_ptr(), ref.stride(0), out2.data_ptr(), thermo.data_ptr(), sim.status.ptr, 0.0, st)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            s.vel.copy_(vel0)
            print(f"  phases {phases} {'no-prune' if flags else 'pruned  '}: {np.median(ts):.4f} ms", flush=True)
    del g, sim
    torch.cuda.empty_cache()
