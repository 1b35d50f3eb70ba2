"""Stress test of tmd_peer_allgather with P in-process ranks (threads + streams)
on one GPU: every call's gathered rows must equal what each rank published.

Finding (profiles/r2_exp_phases.txt): at P = 8 in ONE process some calls time
out -- a rank thread blocked in a call that orders every stream of the shared
context (allocation, pageable copy) waits for a peer's spinning gather kernel,
which waits for that rank.  Hence in-process ranks keep the epoch's count
all-gathers on the host transport; across processes (torchrun) the contexts
are separate and the mailbox gather is the production path."""
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_07400_b200 import _native as N  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
ITERS = int(sys.argv[2]) if len(sys.argv) > 2 else 300
dev = torch.device("cuda", 0)
words = N.lib.tmd_mailbox_words()
boxes = [torch.zeros(words, dtype=torch.int64, device=dev) for _ in range(P)]
ptrs = np.array([b.data_ptr() for b in boxes], dtype=np.uint64)
torch.cuda.synchronize()
errors = []
bar = threading.Barrier(P)


def body(rank):
    torch.cuda.set_device(dev)
    s = torch.cuda.Stream(dev)
    st = torch.zeros(4, dtype=torch.int64, device=dev)
    rng = np.random.default_rng(rank)
    with torch.cuda.stream(s):
        for it in range(1, ITERS + 1):
            w = 6 if it % 2 else 8
            vals = (np.arange(w) + 1000 * rank + 100000 * it).astype(np.int64)
            t = torch.from_numpy(vals).to(dev)
            out = torch.empty((P, w), dtype=torch.int64, device=dev)
            N.call("tmd_peer_allgather", it, rank, P, N.hp(ptrs), t.data_ptr(), w, out.data_ptr(), 10.0,
                   st.data_ptr(), torch._C._cuda_getCurrentRawStream(0))
            if rng.random() < 0.3:
                torch.cuda.current_stream().synchronize()
            got = out.cpu().numpy()
            want = np.stack([(np.arange(w) + 1000 * q + 100000 * it) for q in range(P)])
            if not np.array_equal(got, want):
                bad = [(q, got[q].tolist(), want[q].tolist()) for q in range(P) if not np.array_equal(got[q], want[q])]
                errors.append((rank, it, bad))
                return
        if int(st[0].item()) != 0:
            errors.append((rank, "status", st.cpu().tolist()))


th = [threading.Thread(target=body, args=(r,)) for r in range(P)]
for t in th:
    t.start()
for t in th:
    t.join()
print("P", P, "iters", ITERS, "errors", len(errors), errors[:3])
