"""In-process communicator for running the ranks of a sharded filter as threads on ONE GPU
(TEST INFRASTRUCTURE).  Each rank thread has its own CUDA stream (the library's scratch pool is
per stream); every exchange synchronises the device, then swaps tensors through a barrier.
This exercises the real resample_sharded / migrate_sharded code and kernels on one device; the
multi-process collectives are covered by tests/test_multirank_gloo.py."""
from __future__ import annotations

import threading

import torch


class Hub:
    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world


class LoopbackComm:
    def __init__(self, hub: Hub, rank: int):
        self.hub, self.rank, self.world = hub, rank, hub.world

    def _exchange(self, obj):
        torch.cuda.synchronize()
        self.hub.slots[self.rank] = obj
        self.hub.barrier.wait()
        got = list(self.hub.slots)
        self.hub.barrier.wait()
        return got

    def all_reduce_max(self, t):
        return torch.stack(self._exchange(t)).max(dim=0).values

    def all_gather_cat(self, t):
        return torch.cat(self._exchange(t))

    def reduce_scatter_sum(self, t):
        n = t.shape[0] // self.world
        s = torch.stack(self._exchange(t)).sum(dim=0).to(t.dtype)
        return s[self.rank * n:(self.rank + 1) * n].contiguous()

    def broadcast_(self, t, src: int):
        got = self._exchange(t)
        if self.rank != src:
            t.copy_(got[src])
        return t

    def all_to_all_v(self, t, send_splits, recv_splits):
        got = self._exchange((t, list(send_splits)))
        parts = []
        for q, (tq, sq) in enumerate(got):
            a = sum(sq[:self.rank])
            parts.append(tq[a:a + sq[self.rank]])
        out = torch.cat(parts)
        assert out.shape[0] == sum(recv_splits)
        return out


def run_ranks(world: int, fn):
    """fn(rank, comm) in one thread per rank, each on its own stream; returns the results by rank."""
    hub = Hub(world)
    res, errs = [None] * world, []
    dev = torch.cuda.current_device()

    def body(r):
        try:
            torch.cuda.set_device(dev)
            with torch.cuda.stream(torch.cuda.Stream()):
                res[r] = fn(r, LoopbackComm(hub, r))
                torch.cuda.synchronize()
        except BaseException as e:  # noqa: BLE001 - re-raised below
            errs.append(e)
            hub.barrier.abort()

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]
    return res
