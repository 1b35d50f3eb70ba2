"""A/B under ncu: the production step kernel (phases 0, forces only) against
the experiment loop exp_step4 variant 0 on the same 80^3 state (step 61).
Run: ncu --profile-from-start off --set full ... python exp_ab.py"""
import ctypes as C
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_07400_b200 as P  # noqa: E402
from paper_2009_07400_b200 import _native as N  # noqa: E402

here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "exp_step4.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(here, "exp_step4.cu")])
exp = C.CDLL(so)
cfg = P.SimConfig(unit_cells=(80, 80, 80), steps=70)
sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
g = sim.iter_steps()
for _ in range(62):
    next(g)
torch.cuda.synchronize()
s, L, law = sim.store, sim.lists, sim.law
n = s.n_local
st = torch.cuda.current_stream().cuda_stream
scratch = torch.empty_like(s.pos)
d2 = torch.zeros(1, dtype=torch.float64, device=s.device)
ref = L.ref_positions_dev
N.call("tmd_max_disp2", s.pos.data_ptr(), s.ld, ref.data_ptr(), ref.stride(0), n, d2.data_ptr(), st)
out2 = torch.zeros(1, dtype=torch.float64, device=s.device)
thermo = torch.zeros(6, dtype=torch.float64, device=s.device)
cnt = L.nnear[:n].contiguous()
outx = torch.zeros((3, s.ld), dtype=torch.float64, device=s.device)
torch.cuda.synchronize()
torch.cuda.profiler.start()
exp.exp_step4(C.c_int(0), C.c_void_p(s.pos.data_ptr()), C.c_int64(s.ld), C.c_void_p(L.nbr.data_ptr()),
              C.c_int64(L.ld_nbr), C.c_void_p(cnt.data_ptr()), C.c_int32(n), C.c_double(6.25),
              C.c_void_p(outx.data_ptr()), C.c_void_p(st))
N.call("tmd_step_lj", s.pos.data_ptr(), scratch.data_ptr(), s.vel.data_ptr(), s.ld, n, L.nbr.data_ptr(), L.ld_nbr,
       L.d_counts.data_ptr(), L.nnear.data_ptr(), L.cap, float(L.near_margin), d2.data_ptr(), 0, 0, 0, 0, 0, 0, 0, 0,
       0, float(law.cutoff_rsq), float(law.epsilon), float(law.sigma6), 0.0025, 0.005, 0, 0, s.frc.data_ptr(), s.ld,
       ref.data_ptr(), ref.stride(0), out2.data_ptr(), thermo.data_ptr(), sim.status.ptr, 0.0, st)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("done")
