"""The ADVICE r1 capacity-growth scenario with the fix disabled: the peers'
stale mappings of a grown rank's buffers make the run diverge from the
undisturbed one (evidence that test_capacity_growth_mid_run_remaps_peers
exercises the bug).  One GPU, in-process ranks (loopback.py)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07400_b200 import SimConfig, run_loopback  # noqa: E402
from paper_2009_07400_b200.comm import Halo  # noqa: E402
from paper_2009_07400_b200.store import ParticleStore  # noqa: E402

cfg = SimConfig(unit_cells=(8, 8, 8), steps=60, reneigh_interval=10)
ref, _ = run_loopback(cfg, 2, mode="fast", peer_timeout_s=30.0)
real_cap = ParticleStore.capacity
ParticleStore.capacity = property(lambda self: real_cap.fget(self) - getattr(self, "_hide", 0))
real_borders = Halo.define_borders_direct
calls = {0: 0, 1: 0}


def borders(self, store, extra=(), **kw):
    rank = self.decomp.rank
    calls[rank] += 1
    hide = rank == 1 and calls[rank] in (3, 5)
    if hide:
        store._hide = real_cap.fget(store) - store.n_local - 1
    try:
        out = real_borders(self, store, extra, **kw)
    finally:
        store._hide = 0
    self.gathered_grew[:] = False  # the fix disabled: peers keep their stale mappings
    return out


Halo.define_borders_direct = borders
try:
    got, _ = run_loopback(cfg, 2, mode="fast", peer_timeout_s=30.0)
    diff = float(np.max(np.abs(got[0].thermo[:, 1:5] - ref[0].thermo[:, 1:5]) / np.abs(ref[0].thermo[:, 1:5])))
    print({"fix_disabled_max_rel_thermo_diff": diff, "diverged": diff > 1e-12})
except Exception as e:  # noqa: BLE001
    print({"fix_disabled_error": repr(e)[:300]})
