"""Host-resident batches: copy-in, resample, copy-out overlapped across chunks of filters.

Filters are independent (the Philox counter carries the global filter index, NS-6), so a
batch split into chunks of filters gives the same results as one call.  Each chunk's
host->device copy, its `pf_resample_batched` call and the device->host copy of its
permutation run on three CUDA streams ordered by events, so chunk k+1's input copy and chunk
k-1's output copy overlap chunk k's kernel (each copy direction has its own engine).  With
``chain=True`` consecutive calls also overlap each other: a call's input copies wait only for the
previous call's kernel on the same chunk (the device buffer they overwrite), not for the caller's
stream, so the next batch streams in while the previous one streams out and both PCIe
directions stay busy.  Plumbing only: every step of the method runs in libpfresample.
"""
from __future__ import annotations

from . import PfError, pf_resample_batched


class HostPipeline:
    """Reusable device buffers + streams for resampling host-resident log-weights.

    h_logw: pinned float32 [N, P] host tensor; returns into h_perm (pinned int32 [N, P]) the
    canonical permutation (or the ancestors when ``output="ancestors"``); the device state X
    ([N, P, ...], optional) is gathered in place on the device.
    """

    def __init__(self, N: int, P: int, device, chunks: int = 8):
        import torch

        if chunks < 1 or N < 1 or P < 1:
            raise PfError("N, P and chunks must be >= 1")
        self.N, self.P = N, P
        self.dev = torch.device(device)
        self.chunks = min(chunks, N)
        self.bounds = [(N * c // self.chunks, N * (c + 1) // self.chunks) for c in range(self.chunks)]
        self.d_logw = torch.empty((N, P), dtype=torch.float32, device=self.dev)
        self.anc = torch.empty((N, P), dtype=torch.int32, device=self.dev)
        self.off = torch.empty((N, P), dtype=torch.int32, device=self.dev)
        self.perm = torch.empty((N, P), dtype=torch.int32, device=self.dev)
        self.s_in = torch.cuda.Stream(self.dev)
        self.s_run = torch.cuda.Stream(self.dev)
        self.s_out = torch.cuda.Stream(self.dev)
        self._consumed = [None] * self.chunks  # per chunk: the last call's kernel (reads d_logw)

    def run(self, scheme, h_logw, seed: int, h_out, B: int = 0, first_filter: int = 0, state=None,
            output: str = "permutation", stream=None, chain: bool = False):
        """Enqueue the whole batch; the caller's stream (default: current) waits for the last copy.

        The kernels and the output copies follow everything already enqueued on the caller's
        stream (e.g. a propagate step writing ``state``).  The input copies do too, unless
        ``chain``: then h_logw must be complete on the host when run() is called (not produced by
        work pending on the caller's stream), and each chunk's input copy waits only for the
        previous call's kernel on that chunk."""
        import torch

        if not (h_logw.is_pinned() and h_out.is_pinned()):
            raise PfError("h_logw and h_out must be pinned host tensors")
        if tuple(h_logw.shape) != (self.N, self.P) or tuple(h_out.shape) != (self.N, self.P):
            raise PfError("shape mismatch with the pipeline's (N, P)")
        src = {"permutation": self.perm, "ancestors": self.anc, "offspring": self.off}[output]
        caller = stream or torch.cuda.current_stream(self.dev)
        # the streams start after everything already enqueued on the caller's stream
        start = torch.cuda.Event()
        start.record(caller)
        for s in ((self.s_run, self.s_out) if chain else (self.s_in, self.s_run, self.s_out)):
            s.wait_event(start)
        done = None
        for c, (a, b) in enumerate(self.bounds):
            e_in = torch.cuda.Event()
            e_run = torch.cuda.Event()
            with torch.cuda.stream(self.s_in):
                if chain and self._consumed[c] is not None:
                    self.s_in.wait_event(self._consumed[c])
                self.d_logw[a:b].copy_(h_logw[a:b], non_blocking=True)
                e_in.record(self.s_in)
            self.s_run.wait_event(e_in)
            X = state[a:b] if state is not None else None
            pf_resample_batched(scheme, self.d_logw[a:b], seed, B=B, first_filter=first_filter + a,
                                ancestors=self.anc[a:b], offspring_out=self.off[a:b],
                                permuted_out=self.perm[a:b], state=X, stream=self.s_run)
            e_run.record(self.s_run)
            self._consumed[c] = e_run
            self.s_out.wait_event(e_run)
            with torch.cuda.stream(self.s_out):
                h_out[a:b].copy_(src[a:b], non_blocking=True)
            done = torch.cuda.Event()
            done.record(self.s_out)
        caller.wait_event(done)
        return h_out
