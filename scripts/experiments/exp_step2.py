"""Time the force-loop layout variants of exp_step2.cu on the 80^3 production
state (thermalised, mid-epoch), in the production (brick-major) atom order and
in a Morton order of r/2 cells; check every variant against V0."""
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
so = os.path.join(here, "exp_step2.so")
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                       "-fPIC", "-Xptxas", "-v", "-o", so, os.path.join(here, "exp_step2.cu")],
                      stderr=subprocess.DEVNULL)
lib = C.CDLL(so)
cells = int(sys.argv[1]) if len(sys.argv) > 1 else 80
stop = int(sys.argv[2]) if len(sys.argv) > 2 else 70
cfg = P.SimConfig(unit_cells=(cells,) * 3, steps=stop + 5)
sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
g = sim.iter_steps()
for _ in range(stop + 1):
    next(g)
torch.cuda.synchronize()
s, L = sim.store, sim.lists
n, nt = s.n_local, s.n_total
dev = s.device
st = torch.cuda.current_stream().cuda_stream

# SMs present -> dense rank
nsm = torch.cuda.get_device_properties(dev).multi_processor_count
ids = torch.zeros(4096, dtype=torch.int32, device=dev)
lib.exp_smids(C.c_void_p(ids.data_ptr()), C.c_int(4096), C.c_void_p(st))
present = sorted(set(ids.cpu().tolist()))
sm_rank = torch.full((max(present) + 1,), -1, dtype=torch.int16)
for r, sid in enumerate(present):
    sm_rank[sid] = r
sm_rank = sm_rank.to(dev)
R = len(present)
ctr = torch.zeros(R, dtype=torch.int32, device=dev)
print(f"n_local {n} n_total {nt} SMs {nsm} present {R} mean front {float(L.nnear[:n].float().mean()):.1f}",
      flush=True)


def state(order):
    pos = s.pos[:, :nt].contiguous()
    nbr = L.nbr.view(-1, L.ld_nbr, 4)
    cnt = L.nnear[:n].contiguous()
    if order == "morton":
        lo = torch.tensor(sim.grid_box.lo, dtype=torch.float64, device=dev)[:, None]
        c = torch.floor((pos[:, :n] - lo) / 1.4).to(torch.int64).clamp_min(0)
        key = torch.zeros(n, dtype=torch.int64, device=dev)
        for b in range(10):
            for d in range(3):
                key |= ((c[d] >> b) & 1) << (3 * b + (2 - d))
        perm = torch.sort(key, stable=True).indices
        inv = torch.arange(nt, dtype=torch.int64, device=dev)
        inv[perm] = torch.arange(n, dtype=torch.int64, device=dev)
        pos = torch.cat([pos[:, perm], pos[:, n:]], dim=1).contiguous()
        body = nbr[:, :n, :][:, perm, :]
        body = inv[body.long()].to(torch.int32)
        nbr = torch.cat([body, nbr[:, n:, :]], dim=1).contiguous()
        cnt = cnt[perm].contiguous()
    aos = torch.zeros((nt, 4), dtype=torch.float64, device=dev)
    aos[:, :3] = pos.t()
    return pos, nt, aos, nbr.view(-1), cnt


names = ["V0 SoA thread", "V1 AoS256 thread", "V2 AoS2x128 thread", "V3 AoS256 sweep", "V4 SoA sweep",
         "V5 AoS256 4-lane", "V6 SoA 4-lane"]
for order in ("brick", "morton"):
    pos, ld, aos, nbr, cnt = state(order)
    ref = None
    for v, name in enumerate(names):
        out = torch.zeros((3, ld), dtype=torch.float64, device=dev)
        ts = []
        for _ in range(20):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            rc = lib.exp_step2(C.c_int(v), C.c_void_p(pos.data_ptr()), C.c_int64(ld), C.c_void_p(aos.data_ptr()),
                               C.c_void_p(nbr.data_ptr()), C.c_int64(L.ld_nbr), C.c_void_p(cnt.data_ptr()),
                               C.c_int32(n), C.c_double(6.25), C.c_void_p(out.data_ptr()),
                               C.c_void_p(sm_rank.data_ptr()), C.c_int32(R), C.c_void_p(ctr.data_ptr()),
                               C.c_void_p(st))
            b.record()
            torch.cuda.synchronize()
            assert rc == 0, rc
            ts.append(a.elapsed_time(b))
        f = out[:, :n]
        if ref is None:
            ref = f.clone()
        err = float((f - ref).abs().max() / ref.abs().max().clamp_min(1.0))
        print(f"{order:6s} {name:20s} median {np.median(ts):.4f} ms  min {np.min(ts):.4f}  max rel dF {err:.2e}",
              flush=True)
