"""Block-size / cache-policy variants (exp_step4.cu) on the 80^3 production state."""
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
so = os.path.join(here, "exp_step4.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                       "-fPIC", "-o", so, os.path.join(here, "exp_step4.cu")])
lib = C.CDLL(so)
st = torch.cuda.current_stream().cuda_stream
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
stop = int(sys.argv[2]) if len(sys.argv) > 2 else 70
cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=stop + 5)
sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
g = sim.iter_steps()
for _ in range(stop + 1):
    next(g)
torch.cuda.synchronize()
s, L = sim.store, sim.lists
n = s.n_local
cnt = L.nnear[:n].contiguous()
names = ["256x3", "384x2", "512x2", "512x1", "1024x1", "256x3 list no_alloc", "256x3 carveout L1",
         "512x2 list no_alloc", "256x3 no_alloc+pos evict_last", "256x2"]
ref = None
for v, name in enumerate(names):
    out = torch.zeros((3, s.ld), dtype=torch.float64, device=s.device)
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.exp_step4(C.c_int(v), C.c_void_p(s.pos.data_ptr()), C.c_int64(s.ld), C.c_void_p(L.nbr.data_ptr()),
                           C.c_int64(L.ld_nbr), C.c_void_p(cnt.data_ptr()), C.c_int32(n), C.c_double(6.25),
                           C.c_void_p(out.data_ptr()), C.c_void_p(st))
        b.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        ts.append(a.elapsed_time(b))
    f = out[:, :n]
    if ref is None:
        ref = f.clone()
    err = float((f - ref).abs().max() / ref.abs().max().clamp_min(1.0))
    print(f"{name:26s} median {np.median(ts):.4f} ms  min {np.min(ts):.4f}  max rel dF {err:.2e}", flush=True)
