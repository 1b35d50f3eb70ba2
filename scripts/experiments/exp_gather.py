"""Time the SoA vs AoS4 gather variants of the LJ loop on the 80^3 production lists."""
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
so = os.path.join(here, "exp_gather.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                       "-fPIC", "-o", so, os.path.join(here, "exp_gather.cu")])
lib = C.CDLL(so)
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=10)
sim = P.Simulation(cfg, mode="fast", thermo_every=10)
g = sim.iter_steps()
for _ in range(6):
    next(g)
s, L = sim.store, sim.lists
n = s.n_local
cnt = L.tcnt[4].contiguous()  # a mid tier prefix, like a mid-epoch step
out = torch.empty((3, s.ld), dtype=torch.float64, device=s.device)
aos = torch.empty((s.n_total, 4), dtype=torch.float64, device=s.device)
st = torch.cuda.current_stream().cuda_stream
lib.exp_to_aos(C.c_void_p(s.pos.data_ptr()), C.c_int64(s.ld), C.c_int32(s.n_total), C.c_void_p(aos.data_ptr()), C.c_void_p(st))
res = {}
for mode in (0, 1, 0, 1):
    ptr = aos.data_ptr() if mode else s.pos.data_ptr()
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        lib.exp_lj(C.c_int(mode), C.c_void_p(ptr), C.c_int64(s.ld), C.c_void_p(L.nbr.data_ptr()), C.c_int64(L.ld_nbr),
                   C.c_void_p(cnt.data_ptr()), C.c_int32(n), C.c_double(6.25), C.c_void_p(out.data_ptr()), C.c_void_p(st))
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[mode] = np.median(ts)
    f = out[:, :n].clone()
    if mode == 0:
        f0 = f
    else:
        print("max |dF| soa vs aos", float((f - f0).abs().max()))
print(f"n={n} mean prefix={float(cnt[:n].float().mean()):.1f}  SoA {res[0]:.3f} ms   AoS4-256bit {res[1]:.3f} ms")
