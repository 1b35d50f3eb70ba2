"""The in-process P-rank transport (paper_2009_07400_b200.loopback) on CPU:
the same host-side halo protocols and checks as test_multirank_gloo.py, with
the ranks as threads of one process instead of gloo processes (comm.py:340-498).
The GPU runs of the same transport are in test_loopback_gpu.py."""

import threading

import pytest

import test_multirank_gloo as G
from paper_2009_07400_b200.loopback import LoopbackWorld


def _threads(body, world, out_dir):
    lw = LoopbackWorld(world, timeout=60.0)
    errs = []

    def run(rank):
        try:
            body(rank, world, lw.transport(rank), out_dir)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            lw.transport(rank).abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("world", [2, 4])
def test_reference_protocol_loopback_matches_oracle(world, tmp_path):
    _threads(G.reference_protocol_rank, world, str(tmp_path))
    G.check_reference_protocol(world, tmp_path)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_direct_protocol_loopback_matches_oracle(world, tmp_path):
    _threads(G.direct_protocol_rank, world, str(tmp_path))
    G.check_direct_protocol(world, tmp_path)
