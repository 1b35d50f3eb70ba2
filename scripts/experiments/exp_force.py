"""Time force-loop variants (exp_force.cu) on the 80^3 production lists; check
they agree with V0 within the parity tolerance."""
import ctypes as C
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_07400_b200 as P  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "exp_force.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                       "-fPIC", "-Xptxas", "-v", "-o", so, os.path.join(here, "exp_force.cu")])
lib = C.CDLL(so)
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=10)
sim = P.Simulation(cfg, mode="fast", thermo_every=10)
g = sim.iter_steps()
for _ in range(6):
    next(g)
s, L = sim.store, sim.lists
n = s.n_local
st = torch.cuda.current_stream().cuda_stream
names = ["V0 current", "V1 1NR+fma f", "V2 V1+occ8", "V3 V1+8/iter", "V4 V3+occ8", "V5 xy16+z8 occ8",
         "V6 V0+occ8"]
# the production fused kernel on the same state: phases 0 (forces only), 1 (+final kick), 3 (+drift, guard)
from paper_2009_07400_b200 import _native as N  # noqa: E402

scratch = torch.empty_like(s.pos)
vel_backup = s.vel.clone()
disp = torch.zeros(2, dtype=torch.float64, device=s.device)
thermo = torch.zeros(6, dtype=torch.float64, device=s.device)
for phases in (0, 1, 3):
    ts = []
    for _ in range(15):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        N.call("tmd_step_lj", s.pos.data_ptr(), scratch.data_ptr(), s.vel.data_ptr(), s.ld, n, L.nbr.data_ptr(),
               L.ld_nbr, L.d_counts.data_ptr(), L.nnear.data_ptr(), L.cap, float(L.near_margin),
               disp[0:1].data_ptr(), 0, 0, 0, 0, 0, 0, 0, 0, 0, 6.25, 1.0, 1.0, 0.0025, 0.005, phases, 0, s.frc.data_ptr(), s.ld,
               L.ref_positions_dev.data_ptr(), L.ref_positions_dev.stride(0), disp[1:2].data_ptr(),
               thermo.data_ptr(), sim.status.ptr, st)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    s.vel.copy_(vel_backup)
    print(f"production tmd_step_lj phases={phases}: {np.median(ts):.3f} ms (prune disp 0 -> tier 0)", flush=True)
# interleaved (x, y) copy of every position (locals and ghosts) for V5
xy = torch.stack([s.pos[0, :s.n_total], s.pos[1, :s.n_total]], dim=1).contiguous()
for tier in (0,):
    cnt = L.nnear.contiguous()  # the near (front) segment only: the exp loop reads one segment
    ref = None
    for v, name in enumerate(names):
        out = torch.zeros((3, s.ld), dtype=torch.float64, device=s.device)
        ts = []
        for _ in range(15):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = lib.exp_force(C.c_int(v), C.c_void_p(s.pos.data_ptr()), C.c_int64(s.ld),
                               C.c_void_p(L.nbr.data_ptr()), C.c_int64(L.ld_nbr), C.c_void_p(cnt.data_ptr()),
                               C.c_int32(n), C.c_double(6.25), C.c_void_p(out.data_ptr()), C.c_void_p(st),
                               C.c_void_p(xy.data_ptr()))
            b.record()
            torch.cuda.synchronize()
            assert rc == 0, rc
            ts.append(a.elapsed_time(b))
        f = out[:, :n]
        if ref is None:
            ref = f.clone()
        err = float((f - ref).abs().max() / ref.abs().max().clamp_min(1.0))
        print(f"tier {tier} prefix {float(cnt[:n].float().mean()):.1f}  {name:16s} {np.median(ts):.3f} ms  "
              f"max rel dF {err:.2e}", flush=True)
