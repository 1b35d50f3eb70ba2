"""Does the order of entries inside a row matter for the step kernel's
gathers?  On the 80^3 state at step 61 (mid-epoch), time the production step
kernel (forces only, pruning on) on the builder's rows (stencil order) and on
the same rows with the near segment sorted by neighbour index (brick-major
numbering: the k-th neighbours of adjacent lanes then fall in the same
bricks), and check the forces agree within 1e-12 relative."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_2009_07400_b200 as P  # noqa: E402

cfg = P.SimConfig(unit_cells=(80, 80, 80), steps=70)
sim = P.Simulation(cfg, mode="fast", thermo_every=1000)
g = sim.iter_steps()
for _ in range(62):
    next(g)
torch.cuda.synchronize()
L = sim.lists
n = sim.store.n_local


from paper_2009_07400_b200 import _native as N  # noqa: E402
from paper_2009_07400_b200.neighbor import _stream  # noqa: E402


def launch():
    s = sim.store
    d2 = sim._d2
    ref = L.ref_positions_dev
    rows = (L.nbr.data_ptr(), L.ld_nbr, L.d_counts.data_ptr(), L.nnear.data_ptr(), L.cap, float(L.near_margin),
            d2.data_ptr(), 0, 0, 0, 0, 0, 0, 0, 0, 0, *sim._law_args(), 0.0, 0.0, 0, N.F_STORE_FORCES,
            s.frc.data_ptr(), s.ld, ref.data_ptr(), ref.stride(0), d2.data_ptr(), sim._th.data_ptr(),
            sim.status.ptr, 0.0, _stream())
    N.call("tmd_step_lj", s.pos.data_ptr(), 0, s.vel.data_ptr(), s.ld, s.n_local, *rows)


sim._d2 = torch.zeros(1, dtype=torch.float64, device=sim.device)
sim._th = torch.zeros(6, dtype=torch.float64, device=sim.device)
ref0 = L.ref_positions_dev
N.call("tmd_max_disp2", sim.store.pos.data_ptr(), sim.store.ld, ref0.data_ptr(), ref0.stride(0), n,
       sim._d2.data_ptr(), _stream())


def timed(reps=20):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    launch()
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(reps):
        launch()
    ev[1].record()
    torch.cuda.synchronize()
    return ev[0].elapsed_time(ev[1]) / reps, sim.store.local_forces()


t0, f0 = timed()
q, ld, w = L.nbr.shape
rows = L.nbr.permute(1, 0, 2).reshape(ld, q * w)[:n].clone()  # (n, cap4) row-major
nn = L.nnear[:n].long()
col = torch.arange(q * w, device=rows.device)[None, :]
big = torch.iinfo(torch.int32).max
near = torch.where(col < nn[:, None], rows, torch.full_like(rows, big))
srt = torch.sort(near, dim=1).values
rows2 = torch.where(col < nn[:, None], srt, rows)
# pad quads of the near segment keep their values (the kernel masks by count)
L.nbr[:, :n, :] = rows2.reshape(n, q, w).permute(1, 0, 2)
t1, f1 = timed()
scale = np.maximum(np.abs(f0).max(axis=1), 1e-300)
rel = float(np.max(np.abs(f1 - f0).max(axis=1) / scale))
print(f"stencil-order rows {t0:.4f} ms/launch; index-sorted near segments {t1:.4f} ms/launch; max rel dF {rel:.2e}")
