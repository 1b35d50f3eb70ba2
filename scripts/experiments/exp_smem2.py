"""Block-staged shared-memory force loop on the 80^3 production lists
(exp_smem2.cu): staging sets = union of each 256-atom block's neighbours,
uint16 staging indices in list order vs a bank-class schedule; the L1-gather
loop (exp_step4.cu variant 0) on the same state as the yardstick."""
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
libs = {}
for name in ("exp_smem2", "exp_step4"):
    so = os.path.join(here, name + ".so")
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", "-o", so, os.path.join(here, name + ".cu")])
    libs[name] = C.CDLL(so)
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
B = 256
cnt = L.nnear[:n].contiguous()
Q = L.nbr.shape[0]
rows = L.nbr.permute(1, 0, 2).reshape(L.ld_nbr, Q * 4)[:n]
F = int(cnt.max().item())
F8 = (F + 7) // 8 * 8
mat = rows[:, :F8].to(torch.int64)
slot = torch.arange(F8, device=dev)
valid = slot[None, :] < cnt[:, None].to(torch.int64)
blk = torch.arange(n, device=dev) // B
key = blk[:, None] * nt + mat
uk = torch.unique(key[valid])
nb = (n + B - 1) // B
ustart = torch.searchsorted(uk // nt, torch.arange(nb + 1, device=dev))
uniq = (uk % nt).to(torch.int32).contiguous()
ustart32 = ustart.to(torch.int32).contiguous()
sidx = torch.searchsorted(uk, key) - ustart[blk][:, None]
sidx = torch.where(valid, sidx, torch.zeros_like(sidx))
max_stage = int((ustart[1:] - ustart[:-1]).max().item())
print(f"n {n} front max {F} mean {float(cnt.float().mean()):.1f}  staged per block: max {max_stage} "
      f"mean {float((ustart[1:] - ustart[:-1]).float().mean()):.0f} (256 atoms)", flush=True)

# bank-class schedule: entry of class c = s mod 16 in lane l = i mod 16 gets the key
# (occurrence of its class in the row) * 16 + (c - l) mod 16; masked slots last
lane16 = (torch.arange(n, device=dev) % 16)[:, None]
cls = sidx % 16
rot = (cls - lane16) % 16
rank = torch.empty_like(sidx)
for c0 in range(0, n, 1 << 18):
    c1 = min(n, c0 + (1 << 18))
    oh = torch.nn.functional.one_hot(cls[c0:c1], 16).to(torch.int32) * valid[c0:c1, :, None].to(torch.int32)
    rank[c0:c1] = torch.gather(oh.cumsum(1) - 1, 2, cls[c0:c1, :, None]).squeeze(2).to(torch.int64)
key2 = torch.where(valid, rank * 16 + rot, (1 << 20) + slot[None, :])
perm = torch.argsort(key2, dim=1, stable=True)
sidx_bank = torch.gather(sidx, 1, perm)


def pack(si):
    w = (si[:, 0::2] | (si[:, 1::2] << 16)).to(torch.int32)  # (n, F8/2)
    return w.reshape(n, F8 // 8, 4).permute(1, 0, 2).contiguous()


def conflicts(si):
    """mean bank-pair conflict degree (max lanes per class) per half-warp slot"""
    m = si[: (n // 16) * 16].reshape(-1, 16, F8) % 16
    oh = torch.nn.functional.one_hot(m[:4096], 16).sum(1)  # (halfwarps, F8, 16)
    return float(oh.max(-1).values.float().mean())


pos = s.pos
out = torch.zeros((3, s.ld), dtype=torch.float64, device=dev)


def timeit(fn):
    ts = []
    for _ in range(20):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rc = fn()
        b.record()
        torch.cuda.synchronize()
        assert rc == 0, rc
        ts.append(a.elapsed_time(b))
    return np.median(ts)


t_l1 = timeit(lambda: libs["exp_step4"].exp_step4(C.c_int(0), C.c_void_p(pos.data_ptr()), C.c_int64(s.ld),
                                                  C.c_void_p(L.nbr.data_ptr()), C.c_int64(L.ld_nbr),
                                                  C.c_void_p(cnt.data_ptr()), C.c_int32(n), C.c_double(6.25),
                                                  C.c_void_p(out.data_ptr()), C.c_void_p(st)))
ref = out[:, :n].clone()
print(f"L1 gathers (256x3)          {t_l1:.4f} ms", flush=True)
for name, si in (("staged, list order", sidx), ("staged, bank-class order", sidx_bank)):
    idx = pack(si)
    out.zero_()
    t = timeit(lambda: libs["exp_smem2"].exp_staged(C.c_void_p(pos.data_ptr()), C.c_int64(s.ld),
                                                    C.c_void_p(uniq.data_ptr()),
                                                    C.c_void_p(ustart32.data_ptr()),
                                                    C.c_void_p(idx.data_ptr()), C.c_void_p(cnt.data_ptr()),
                                                    C.c_int32(n), C.c_double(6.25), C.c_void_p(out.data_ptr()),
                                                    C.c_int(max_stage), C.c_void_p(st)))
    err = float((out[:, :n] - ref).abs().max() / ref.abs().max().clamp_min(1.0))
    print(f"{name:27s} {t:.4f} ms  max rel dF {err:.2e}  mean max-lanes-per-bank-class {conflicts(si):.2f}",
          flush=True)
