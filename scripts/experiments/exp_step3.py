"""FP64-trimmed force-loop variants (exp_step3.cu) on the 80^3 production state
(thermalised, mid-epoch, front segments), checked against V0; plus the accuracy
of the one-Newton cubic reciprocal."""
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
so = os.path.join(here, "exp_step3.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                       "-fPIC", "-o", so, os.path.join(here, "exp_step3.cu")])
lib = C.CDLL(so)
st = torch.cuda.current_stream().cuda_stream
# reciprocal accuracy over the LJ range of rsq (and a wide range)
x = torch.cat([torch.empty(1 << 22, dtype=torch.float64, device="cuda").uniform_(0.5, 7.0),
               torch.exp(torch.empty(1 << 20, dtype=torch.float64, device="cuda").uniform_(-300, 300))])
err = torch.empty((x.numel(), 2), dtype=torch.float64, device="cuda")
lib.exp_rcp_probe(C.c_void_p(x.data_ptr()), C.c_int(x.numel()), C.c_void_p(err.data_ptr()), C.c_void_p(st))
torch.cuda.synchronize()
print(f"rcp max rel err: 1 Newton cubic {float(err[:, 0].max()):.3e}  2 Newton {float(err[:, 1].max()):.3e}",
      flush=True)

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
names = ["V0 production arith", "V1 trimmed", "V2 trimmed occ10", "V3 trimmed 8/iter occ6",
         "V4 trimmed occ6", "V5 trimmed occ12"]
ref = None
for v, name in enumerate(names):
    out = torch.zeros((3, s.ld), dtype=torch.float64, device=s.device)
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = lib.exp_step3(C.c_int(v), C.c_void_p(s.pos.data_ptr()), C.c_int64(s.ld), C.c_void_p(L.nbr.data_ptr()),
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
