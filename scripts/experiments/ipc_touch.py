"""Cost of the first kernel writes into a freshly CUDA-IPC-mapped peer buffer.

    torchrun --standalone --nproc-per-node 2 scripts/experiments/ipc_touch.py
"""
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2009_07400_b200 as P  # noqa: E402
from paper_2009_07400_b200 import _native as N  # noqa: E402
from paper_2009_07400_b200.exports import PeerMaps, _handle_of  # noqa: E402


def write_peer(ptr, ld, k, src, idx):
    N.call("tmd_gather_shift", src.data_ptr(), src.stride(0), idx.data_ptr(), k, N.hp(np.zeros(3)), 0, 0, ptr, ld,
           torch.cuda.current_stream().cuda_stream)


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank = dist.get_rank()
    ld = 2_600_000
    bufs = [torch.zeros((3, ld), dtype=torch.float64, device="cuda") for _ in range(3)]
    src = torch.randn((3, ld), dtype=torch.float64, device="cuda")
    idx = torch.arange(ld, dtype=torch.int32, device="cuda")
    handles = [_handle_of(b) for b in bufs]
    allh = [None] * 2
    dist.all_gather_object(allh, handles)
    peer = allh[1 - rank]
    maps = PeerMaps()
    for b, (h, off) in enumerate(peer):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ptr = maps.open(h, off)
        t_open = time.perf_counter() - t0
        res = []
        for k in (1000, 100_000, ld, ld):
            dist.barrier()
            torch.cuda.synchronize()
            a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record()
            write_peer(ptr, ld, k, src, idx)
            e.record()
            torch.cuda.synchronize()
            res.append((k, round(a.elapsed_time(e), 3), round((time.perf_counter() - t0) * 1e3, 3)))
        print(f"rank {rank} buffer {b}: open {t_open * 1e3:.2f} ms; writes (k, dev ms, wall ms) {res}", flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
