"""Giant-filter sharding over GPUs (BASELINE config C5).

One filter of ``P_global`` particles is split into contiguous shards, shard g
(rank g) owning particles ``[p0, p0 + Pl)`` (``shard_range``).  The exchange
steps are the only communication (P:125-128's "collective prefix-sum", split
into a per-GPU scan plus an 8-byte-per-rank exchange):

  prefix-sum schemes:  max  -> all_reduce(MAX) of 1 float (+ bad flag)
                       scan -> all_gather of the 8-byte shard totals
                       search: every rank computes its own slot range from the
                       totals (positions are functions of the slot index) and
                       writes the ancestors of those slots.
  sorted multinomial   (a6, ``flags=PF_SORTED``) additionally all-gathers the
                       8-byte totals of the exponential spacings of each
                       spacing shard; each rank then regenerates
                       only the spacing shards that hold its slots.
  Metropolis:          max  -> all_reduce(MAX); weights -> all_gather of the
                       weight vector; chains for the rank's own slots
                       (no collective inside the resampler).

The arithmetic of every stage is the single-GPU numeric spec evaluated with the
global max and k_fx(P_global), so the result is bit-identical to
``pf_resample_ex`` on the whole filter.  Stages run in libpfresample kernels
(``GpuStages``); the communicator is ``TorchComm`` (torch.distributed, NCCL over
NVLink on the GPU box).  Both are parameters so that the decomposition logic can
be exercised on CPU with gloo (tests/test_multirank_gloo.py).
"""
from __future__ import annotations

import math

SCHEMES = {"multinomial": 1, "stratified": 2, "systematic": 3, "metropolis": 4}
PF_SORTED = 1


def shard_range(P_global: int, world: int, rank: int):
    """Contiguous shards of ceil(P/world) particles (the last may be shorter)."""
    per = -(-P_global // world)
    p0 = min(P_global, rank * per)
    return p0, min(P_global, p0 + per) - p0


class TorchComm:
    """Collectives over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def all_reduce_max(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t

    def all_gather_cat(self, t):
        import torch

        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return torch.cat(out)


class SingleComm:
    """World of one (no communication): the sharded path on a single GPU."""

    rank, world = 0, 1

    def all_reduce_max(self, t):
        return t

    def all_gather_cat(self, t):
        return t


class GpuStages:
    """Shard stages in libpfresample kernels (device tensors)."""

    def __init__(self):
        import paper_1202_6163_b200 as pf

        self.pf = pf

    def max(self, logw):
        return self.pf.pf_shard_max(logw)

    def scan(self, logw, P_global, gmax):
        return self.pf.pf_shard_scan(logw, P_global, gmax)

    def search(self, scheme, Q, p0, P_global, totals, shard, gmax, gbad, seed, filter_index, anc_out):
        return self.pf.pf_shard_search(scheme, Q, p0, P_global, totals, shard, gmax, gbad, seed, filter_index,
                                       anc_out)

    def spacings_total(self, P_global, nshards, shard, seed, filter_index, device):
        return self.pf.pf_shard_spacings_total(P_global, nshards, shard, seed, filter_index, device)

    def search_sorted(self, Q, p0, P_global, totals, etotals, shard, gmax, gbad, seed, filter_index, anc_out):
        return self.pf.pf_shard_search_sorted(Q, p0, P_global, totals, etotals, shard, gmax, gbad, seed,
                                              filter_index, anc_out)

    def weights(self, logw, gmax):
        return self.pf.pf_shard_weights(logw, gmax)

    def metropolis(self, w_full, slot0, nslots, seed, B, filter_index, gmax, gbad):
        return self.pf.pf_metropolis_from_weights(w_full, slot0, nslots, seed, B, filter_index, gmax, gbad)


def resample_sharded(scheme, logw_local, P_global: int, seed: int, B: int = 0, filter_index: int = 0,
                     comm=None, stages=None, assemble: bool = True, flags: int = 0):
    """Resample one filter sharded over the ranks of ``comm``.

    logw_local: this rank's contiguous shard (``shard_range(P_global, world, rank)``).
    Returns (ancestors, info): with ``assemble`` the full int32 [P_global] ancestor
    vector on every rank (all_reduce MAX of per-rank slot writes / all_gather of
    Metropolis chains); otherwise this rank's slots only (Metropolis: slots
    [p0, p0 + Pl); prefix-sum schemes: entries [k_lo, k_hi) of a [P_global] buffer).
    """
    import torch

    comm = comm or TorchComm()
    stages = stages or GpuStages()
    scheme_id = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
    is_sorted = _sorted(scheme_id, flags)
    world, rank = comm.world, comm.rank
    p0, Pl = shard_range(P_global, world, rank)
    if logw_local.shape[0] != Pl:
        raise ValueError(f"rank {rank}: shard has {logw_local.shape[0]} particles, expected {Pl}")
    if Pl < 1:
        raise ValueError("every rank needs at least one particle")
    lmax, bad = stages.max(logw_local)
    gmax = comm.all_reduce_max(lmax.clone())
    gbad = comm.all_reduce_max(bad.clone())
    info = {"p0": p0, "Pl": Pl}
    if scheme_id == 4:
        w = stages.weights(logw_local, gmax)
        per = -(-P_global // world)
        if Pl < per:  # equal-size pieces for the all-gather
            w = torch.cat([w, torch.zeros(per - Pl, dtype=w.dtype, device=w.device)])
        w_full = comm.all_gather_cat(w)[:P_global].contiguous()
        anc_local = stages.metropolis(w_full, p0, Pl, seed, B, filter_index, gmax, gbad)
        info["slot_range"] = (p0, p0 + Pl)
        if not assemble:
            return anc_local, info
        per_anc = anc_local
        if Pl < per:
            per_anc = torch.cat([anc_local, torch.zeros(per - Pl, dtype=anc_local.dtype, device=anc_local.device)])
        return comm.all_gather_cat(per_anc)[:P_global].contiguous(), info
    Q, total, wsum = stages.scan(logw_local, P_global, gmax)
    totals = comm.all_gather_cat(total)
    wsums = comm.all_gather_cat(wsum)
    anc = torch.full((P_global,), -1, dtype=torch.int32, device=logw_local.device)
    if is_sorted:
        etot = stages.spacings_total(P_global, world, rank, seed, filter_index, logw_local.device)
        etotals = comm.all_gather_cat(etot)
        rng = stages.search_sorted(Q, p0, P_global, totals, etotals, rank, gmax, gbad, seed, filter_index, anc)
    else:
        rng = stages.search(scheme_id, Q, p0, P_global, totals, rank, gmax, gbad, seed, filter_index, anc)
    info["slot_range_dev"] = rng
    info["lse"] = (gmax, wsums)  # lse = gmax + ln(sum wsums) (NS-13), left on the device
    if not assemble:
        return anc, info
    return comm.all_reduce_max(anc), info


def _sorted(scheme_id: int, flags: int) -> bool:
    if flags & ~PF_SORTED:
        raise ValueError(f"unsupported flags {flags:#x}")
    if flags & PF_SORTED and scheme_id != 1:
        raise ValueError("PF_SORTED applies to the multinomial scheme only")
    return bool(flags & PF_SORTED)


def resample_sharded_local(scheme, logw_full, nshards: int, seed: int, B: int = 0, filter_index: int = 0,
                           stages=None, flags: int = 0):
    """Fake-shard mode: all shards on one device, exchanges done on the host.
    Exercises exactly the shard kernels and the offset logic of ``resample_sharded``."""
    import torch

    stages = stages or GpuStages()
    scheme_id = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
    is_sorted = _sorted(scheme_id, flags)
    P_global = logw_full.shape[0]
    parts = [shard_range(P_global, nshards, g) for g in range(nshards)]
    pieces = [logw_full[p0:p0 + Pl] for p0, Pl in parts]
    mx = [stages.max(x) for x in pieces]
    gmax = torch.stack([m for m, _ in mx]).max(dim=0).values
    gbad = torch.stack([b for _, b in mx]).max(dim=0).values
    if scheme_id == 4:
        w_full = torch.cat([stages.weights(x, gmax) for x in pieces])
        return torch.cat([stages.metropolis(w_full, p0, Pl, seed, B, filter_index, gmax, gbad) for p0, Pl in parts])
    scans = [stages.scan(x, P_global, gmax) for x in pieces]
    totals = torch.cat([t for _, t, _ in scans])
    anc = torch.full((P_global,), -1, dtype=torch.int32, device=logw_full.device)
    if is_sorted:
        etotals = torch.cat([stages.spacings_total(P_global, nshards, g, seed, filter_index, logw_full.device)
                             for g in range(nshards)])
        for g, ((p0, Pl), (Q, _, _)) in enumerate(zip(parts, scans)):
            stages.search_sorted(Q, p0, P_global, totals, etotals, g, gmax, gbad, seed, filter_index, anc)
        return anc
    for g, ((p0, Pl), (Q, _, _)) in enumerate(zip(parts, scans)):
        stages.search(scheme_id, Q, p0, P_global, totals, g, gmax, gbad, seed, filter_index, anc)
    return anc
