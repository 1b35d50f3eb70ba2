"""P ranks of the decomposition inside one process, on one GPU.

Each rank is a host thread with its own CUDA stream and its own
``Simulation``; the transport moves data with device copies and orders the
ranks with a ``threading.Barrier``.  Every device kernel of the multi-rank
production path runs exactly as under torchrun -- exchange classification,
border records, export tables, the step kernel's ghost writes into a peer's
position buffer (a plain device pointer here instead of a CUDA-IPC mapping)
and the per-step mailbox barrier kernel (tmd_peer_sync) -- so a single-GPU box
can check the P > 1 path against the reference's own P-rank runs.

    reports = run_loopback(cfg, P, mode="fast")   # one Report per rank

The ranks' barrier kernels wait for each other on one GPU, so every rank
stream needs its own hardware queue: set CUDA_DEVICE_MAX_CONNECTIONS=32 before
the CUDA context is created (the test suite and the CLI do).  The count
all-gathers of the epoch stay on the transport here (a device or page-locked
allocation by one rank orders every stream of the shared context).

The collectives follow ``DistTransport`` (comm.py); the reference's
equivalent is the in-process ``MailboxTransport`` (comm.py:83-104), which
advances rank generators in lockstep.
"""

from __future__ import annotations

import threading

import torch

from .errors import ProtocolError

__all__ = ["LoopbackWorld", "LoopbackTransport", "run_loopback"]


class LoopbackWorld:
    """Shared rendezvous of P in-process ranks."""

    def __init__(self, size: int, timeout: float = 120.0):
        if size < 1:
            raise ValueError("size must be >= 1")
        self.size = size
        self.timeout = timeout
        self._bar = threading.Barrier(size, timeout=timeout)
        self._slots = [None] * size

    def transport(self, rank: int) -> "LoopbackTransport":
        return LoopbackTransport(self, rank)


class LoopbackTransport:
    """The DistTransport interface over device copies between threads."""

    same_process = True  # peers' buffers are plain device pointers (no CUDA IPC)

    def __init__(self, world: LoopbackWorld, rank: int):
        self.world = world
        self.rank = rank
        self.size = world.size

    # one rendezvous: publish `obj`, see everybody's; the producers' streams are
    # complete before anyone reads, and nobody republishes before all have read
    @staticmethod
    def _sync():
        if torch.cuda.is_available() and torch.cuda.is_initialized():
            torch.cuda.current_stream().synchronize()

    def _exchange(self, obj, consume):
        w = self.world
        self._sync()
        w._slots[self.rank] = obj
        try:
            w._bar.wait()
            out = consume(list(w._slots))
            self._sync()
            w._bar.wait()
        except threading.BrokenBarrierError as e:
            raise ProtocolError(f"loopback rank {self.rank}: a peer rank failed or timed out") from e
        return out

    def barrier(self):
        self._exchange(None, lambda slots: None)

    def abort(self):
        self.world._bar.abort()

    def allreduce_(self, t: torch.Tensor, op="sum"):
        def red(slots):
            stack = torch.stack([s.to(t.device) for s in slots])
            return stack.sum(0) if op == "sum" else stack.max(0).values

        t.copy_(self._exchange(t.clone(), red))
        return t

    def allgather(self, t: torch.Tensor) -> torch.Tensor:
        return self._exchange(t.contiguous().clone(), lambda slots: torch.stack([s.to(t.device) for s in slots]))

    def all_gather_object(self, obj):
        return self._exchange(obj, lambda slots: slots)

    def alltoall_v(self, payload: torch.Tensor, send_counts, recv_counts):
        me = self.rank

        def take(slots):
            parts = []
            for src, (p, sc) in enumerate(slots):
                off = int(sum(sc[:me]))
                parts.append(p[off:off + int(sc[me])])
            out = torch.cat(parts) if parts else payload[:0]
            if out.shape[0] != int(sum(recv_counts)):
                raise ProtocolError("loopback all-to-all: counts disagree")
            return out.clone()

        return self._exchange((payload.contiguous(), [int(c) for c in send_counts]), take)

    def alltoall(self, payload: torch.Tensor, send_counts):
        counts = [int(c) for c in send_counts]
        me = self.rank
        rc = self._exchange(counts, lambda slots: [int(s[me]) for s in slots])
        return self.alltoall_v(payload, counts, rc), rc

    def sendrecv(self, sends, recvs):
        """Tagged point-to-point messages of one round (the reference protocol)."""
        me = self.rank
        mine = {(peer, tag): t.contiguous() for peer, tag, t in sends}

        def deliver(slots):
            for peer, tag, t in recvs:
                src = slots[peer].get((me, tag))
                if src is None or src.shape != t.shape:
                    raise ProtocolError(f"loopback rank {me}: no matching message from {peer} tag {tag}")
                t.copy_(src)

        self._exchange(mine, deliver)

    def warm_up(self, device) -> None:
        pass


def run_loopback(cfg, nranks: int, device=None, steps=None, **sim_kw):
    """Run cfg as `nranks` ranks on one GPU (one thread + stream each); returns
    every rank's Report (thermo summed over ranks, as under torchrun) and the
    Simulations (for state inspection)."""
    from .driver import Simulation

    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    world = LoopbackWorld(nranks)
    reports, sims, errors = [None] * nranks, [None] * nranks, [None] * nranks

    def body(rank):
        torch.cuda.set_device(dev)
        stream = torch.cuda.Stream(dev)
        tr = world.transport(rank)
        try:
            with torch.cuda.stream(stream):
                sim = Simulation(cfg, transport=tr, device=dev, **sim_kw)
                sims[rank] = sim
                reports[rank] = sim.run(steps)
                stream.synchronize()
        except BaseException as e:  # noqa: BLE001 - re-raised on the caller's thread
            errors[rank] = e
            tr.abort()

    threads = [threading.Thread(target=body, args=(r,), name=f"tmd-rank{r}") for r in range(nranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    first = next((e for e in errors if e is not None and not isinstance(e, ProtocolError)), None)
    first = first or next((e for e in errors if e is not None), None)
    if first is not None:
        raise first
    return reports, sims
