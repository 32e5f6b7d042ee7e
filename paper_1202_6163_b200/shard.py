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
  unsorted multinomial routed (NEXT-4): rank g generates only the positions of its own
                       slot shard, all-gathers the per-owner counts (G x G int64) and sends
                       each position to the shard whose weight range holds it in one
                       variable all_to_all; the owner searches its local Q (work ~ P/G).
  sorted multinomial   (a6, ``flags=PF_SORTED``) additionally all-gathers the
                       8-byte totals of the exponential spacings of each
                       spacing shard; each rank then regenerates
                       only the spacing shards that hold its slots.
  Metropolis:          max  -> all_reduce(MAX); weights -> all_gather of the
                       weight vector; chains for the rank's own slots
                       (no collective inside the resampler).
  migration            (``migrate_sharded``; NEXT-4) the in-place permutation and state
                       gather of the whole filter: offspring of the rank's particles
                       (Metropolis: reduce_scatter of slot histograms), all_gather of the
                       16-byte (extras, free) counts, one variable all_to_all of the
                       extra rows (and their indices); survivors never move.

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


def check_shards(P_global: int, world: int):
    """Every rank must hold at least one particle (the exchange steps assume it).  Evaluated from
    (P_global, world) alone, so every rank reaches the same verdict before any collective: a bad
    configuration raises on all ranks instead of leaving the others waiting in a collective."""
    if world < 1 or P_global < 1:
        raise ValueError(f"P_global={P_global}, world={world}")
    per = -(-P_global // world)
    if (world - 1) * per >= P_global:
        raise ValueError(f"P_global={P_global} over {world} ranks leaves ranks without particles "
                         f"(contiguous shards of {per}); use at most {-(-P_global // per)} ranks or a larger filter")


class TorchComm:
    """Collectives over torch.distributed (NCCL on GPUs, gloo on CPU).

    With ``timing=True`` (CUDA tensors) every collective is bracketed by CUDA events on the
    current stream, so ``collect_times()`` reports each kind's device time as the stream sees it
    (the NCCL kernel plus its wait): {name: (calls, total_ms, bytes)}."""

    def __init__(self, group=None, timing: bool = False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.timing = timing
        self._ev = []

    def _timed(self, name, nbytes, fn):
        if not self.timing:
            return fn()
        import torch

        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        r = fn()
        b.record()
        self._ev.append((name, a, b, nbytes))
        return r

    def collect_times(self):
        import torch

        torch.cuda.synchronize()
        out = {}
        for name, a, b, nb in self._ev:
            c, ms, by = out.get(name, (0, 0.0, 0))
            out[name] = (c + 1, ms + a.elapsed_time(b), by + nb)
        self._ev = []
        return out

    def all_reduce_max(self, t):
        self._timed("all_reduce_max", t.numel() * t.element_size(),
                    lambda: self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group))
        return t

    def all_gather_cat(self, t):
        import torch

        out = [torch.empty_like(t) for _ in range(self.world)]
        self._timed("all_gather", t.numel() * t.element_size() * self.world,
                    lambda: self.dist.all_gather(out, t, group=self.group))
        return torch.cat(out)

    def reduce_scatter_sum(self, t):
        """t: [world * n]; returns this rank's n-slice of the sum over ranks."""
        import torch

        n = t.shape[0] // self.world
        out = torch.empty(n, dtype=t.dtype, device=t.device)
        if self.dist.get_backend(self.group) == "gloo":  # gloo has no reduce_scatter
            self.dist.all_reduce(t, group=self.group)
            out.copy_(t[self.rank * n:(self.rank + 1) * n])
        else:
            self._timed("reduce_scatter", t.numel() * t.element_size(),
                        lambda: self.dist.reduce_scatter_tensor(out, t, group=self.group))
        return out

    def all_to_all_v(self, t, send_splits, recv_splits):
        """Rows t[sum(send_splits[:g]) : ...] go to rank g; returns the rows received, in rank order."""
        import torch

        out = torch.empty((sum(recv_splits),) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        row = math.prod(t.shape[1:]) * t.element_size()
        self._timed("all_to_all", row * (sum(recv_splits) + sum(send_splits)),
                    lambda: self.dist.all_to_all_single(out, t.contiguous(), output_split_sizes=list(recv_splits),
                                                        input_split_sizes=list(send_splits), group=self.group))
        return out

    def broadcast_(self, t, src: int):
        """t (contiguous) from rank ``src`` to every rank, in place."""
        self._timed("broadcast", t.numel() * t.element_size(),
                    lambda: self.dist.broadcast(t, src=self.dist.get_global_rank(self.group, src) if self.group
                                                else src, group=self.group))
        return t


class SingleComm:
    """World of one (no communication): the sharded path on a single GPU."""

    rank, world = 0, 1

    def collect_times(self):
        return {}

    def all_reduce_max(self, t):
        return t

    def all_gather_cat(self, t):
        return t

    def reduce_scatter_sum(self, t):
        return t

    def all_to_all_v(self, t, send_splits, recv_splits):
        return t

    def broadcast_(self, t, src: int):
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

    def route_count(self, totals, shard, P_global, gmax, gbad, seed, filter_index):
        return self.pf.pf_shard_route_count(totals, shard, P_global, gmax, gbad, seed, filter_index)

    def route_pack(self, totals, shard, P_global, gmax, gbad, seed, filter_index, counts, n_send):
        return self.pf.pf_shard_route_pack(totals, shard, P_global, gmax, gbad, seed, filter_index, counts, n_send)

    def route_search(self, Q, p0, P_global, totals, shard, gmax, gbad, rx, rk, anc_out):
        return self.pf.pf_shard_route_search(Q, p0, P_global, totals, shard, gmax, gbad, rx, rk, anc_out)

    def spacings_total(self, P_global, nshards, shard, seed, filter_index, device):
        return self.pf.pf_shard_spacings_total(P_global, nshards, shard, seed, filter_index, device)

    def search_sorted(self, Q, p0, P_global, totals, etotals, shard, gmax, gbad, seed, filter_index, anc_out):
        return self.pf.pf_shard_search_sorted(Q, p0, P_global, totals, etotals, shard, gmax, gbad, seed,
                                              filter_index, anc_out)

    def weights(self, logw, gmax):
        return self.pf.pf_shard_weights(logw, gmax)

    def metropolis(self, w_full, slot0, nslots, seed, B, filter_index, gmax, gbad):
        return self.pf.pf_metropolis_from_weights(w_full, slot0, nslots, seed, B, filter_index, gmax, gbad)

    def offspring(self, anc, win0, Pw, slot_range, gmax, gbad):
        return self.pf.pf_shard_offspring(anc, win0, Pw, slot_range=slot_range, gmax=gmax, gbad=gbad)

    def migration_counts(self, o):
        return self.pf.pf_shard_migration_counts(o)

    def pack(self, X, o, plan, p0, E):
        return self.pf.pf_shard_migrate_pack(X, o, plan, p0, E)

    def unpack(self, X, o, plan, p0, rows, src):
        return self.pf.pf_shard_migrate_unpack(X, o, plan, p0, rows, src)


def resample_sharded(scheme, logw_local, P_global: int, seed: int, B: int = 0, filter_index: int = 0,
                     comm=None, stages=None, assemble: bool = True, flags: int = 0):
    """Resample one filter sharded over the ranks of ``comm``.

    logw_local: this rank's contiguous shard (``shard_range(P_global, world, rank)``).
    Returns (ancestors, info): with ``assemble`` the full int32 [P_global] ancestor
    vector on every rank (each rank's contiguous slot range broadcast from it: P_global x 4
    bytes received per rank; the unsorted multinomial, whose slots scatter over the filter,
    all-reduces the vector; Metropolis all-gathers the chains); otherwise this rank's slots
    only (Metropolis: slots [p0, p0 + Pl); prefix-sum schemes: entries [k_lo, k_hi) of a
    [P_global] buffer).

    Errors never strand the other ranks in a collective: a configuration that leaves a rank
    without particles raises on every rank before any exchange (``check_shards``); a shard of
    the wrong size is replaced by a NaN shard of the right size (so every rank computes the
    NS-1 invalid result through the same exchanges) and then raises on its own rank.
    """
    import torch

    comm = comm or TorchComm()
    stages = stages or GpuStages()
    scheme_id = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
    is_sorted = _sorted(scheme_id, flags)
    world, rank = comm.world, comm.rank
    check_shards(P_global, world)
    p0, Pl = shard_range(P_global, world, rank)
    shape_err = None
    if logw_local.dim() != 1 or logw_local.shape[0] != Pl:
        shape_err = f"rank {rank}: shard has shape {tuple(logw_local.shape)}, expected ({Pl},)"
        logw_local = torch.full((Pl,), float("nan"), dtype=logw_local.dtype, device=logw_local.device)
    lmax, bad = stages.max(logw_local)
    gmax = comm.all_reduce_max(lmax.clone())
    gbad = comm.all_reduce_max(bad.clone())
    info = {"p0": p0, "Pl": Pl, "P_global": P_global, "scheme": scheme_id, "sorted": is_sorted, "gmax": gmax,
            "gbad": gbad}
    if scheme_id == 4:
        w = stages.weights(logw_local, gmax)
        per = -(-P_global // world)
        if Pl < per:  # equal-size pieces for the all-gather
            w = torch.cat([w, torch.zeros(per - Pl, dtype=w.dtype, device=w.device)])
        w_full = comm.all_gather_cat(w)[:P_global].contiguous()
        anc_local = stages.metropolis(w_full, p0, Pl, seed, B, filter_index, gmax, gbad)
        info["slot_range"] = (p0, p0 + Pl)
        if not assemble:
            _raise_if(shape_err)
            return anc_local, info
        per_anc = anc_local
        if Pl < per:
            per_anc = torch.cat([anc_local, torch.zeros(per - Pl, dtype=anc_local.dtype, device=anc_local.device)])
        out = comm.all_gather_cat(per_anc)[:P_global].contiguous()
        _raise_if(shape_err)
        return out, info
    Q, total, wsum = stages.scan(logw_local, P_global, gmax)
    totals = comm.all_gather_cat(total)
    wsums = comm.all_gather_cat(wsum)
    anc = torch.full((P_global,), -1, dtype=torch.int32, device=logw_local.device)
    if is_sorted:
        etot = stages.spacings_total(P_global, world, rank, seed, filter_index, logw_local.device)
        etotals = comm.all_gather_cat(etot)
        rng = stages.search_sorted(Q, p0, P_global, totals, etotals, rank, gmax, gbad, seed, filter_index, anc)
    elif scheme_id == 1:
        rng = _route_multinomial(Q, p0, P_global, totals, world, rank, gmax, gbad, seed, filter_index, anc,
                                 comm, stages)
    else:
        rng = stages.search(scheme_id, Q, p0, P_global, totals, rank, gmax, gbad, seed, filter_index, anc)
    info["slot_range_dev"] = rng
    info["lse"] = (gmax, wsums)  # lse = gmax + ln(sum wsums) (NS-13), left on the device
    if not assemble:
        _raise_if(shape_err)
        return anc, info
    if scheme_id == 1 and not is_sorted:
        # the unsorted multinomial's slots scatter over the whole filter
        out = comm.all_reduce_max(anc)
    else:
        # contiguous slot ranges: each rank's slice broadcast from it (an invalid filter's
        # identity was written over every rank's own particle range)
        rngs = comm.all_gather_cat(rng).cpu().view(-1, 2).tolist()
        invalid = bool(int(gbad.max().item()) != 0 or float(gmax.max().item()) == float("-inf"))
        for g in range(world):
            a, b = shard_range(P_global, world, g) if invalid else rngs[g]
            if invalid:
                b = a + b
            if b > a:
                comm.broadcast_(anc[a:b], g)
        out = anc
    _raise_if(shape_err)
    return out, info


def route_splits(counts_matrix, rank: int):
    """(send_splits, recv_splits) of ``rank`` from the all-gathered G x G matrix of per-owner
    position counts (row g = what rank g's slot shard sends to each owner)."""
    send = [int(v) for v in counts_matrix[rank]]
    recv = [int(row[rank]) for row in counts_matrix]
    return send, recv


def _route_multinomial(Q, p0, P_global, totals, world, rank, gmax, gbad, seed, filter_index, anc, comm, stages):
    """Routed unsorted multinomial (include/pf.h 3a-3c): this rank's slot shard's positions to
    their owners, one variable all_to_all of (x, k); the owners' searches write anc[k].  One host
    read of the G x G counts sizes the exchange.  Returns an empty slot range (slots scatter)."""
    import torch

    cnt = stages.route_count(totals, rank, P_global, gmax, gbad, seed, filter_index)
    M = comm.all_gather_cat(cnt).cpu().view(world, world).tolist()
    send, recv = route_splits(M, rank)
    sx, sk = stages.route_pack(totals, rank, P_global, gmax, gbad, seed, filter_index, cnt, sum(send))
    rx = comm.all_to_all_v(sx, send, recv)
    rk = comm.all_to_all_v(sk, send, recv)
    stages.route_search(Q, p0, P_global, totals, rank, gmax, gbad, rx, rk, anc)
    return torch.zeros(2, dtype=torch.int64, device=anc.device)


def _raise_if(msg):
    if msg:
        raise ValueError(msg)


def _overlap(a0, a1, b0, b1):
    return max(0, min(a1, b1) - max(a0, b0))


def migration_splits(counts, rank: int):
    """Split sizes of the migration all-to-all from the all-gathered (E_g, F_g) of every rank:
    rank r's extras occupy [Epre_r, Epre_r + E_r) of the global extras list (NS-15 order),
    rank g's free slots [Fpre_g, Fpre_g + F_g) of the global free list; extra n goes to free
    slot n.  Returns (send_splits, recv_splits) of ``rank``."""
    E = [int(e) for e, _ in counts]
    F = [int(f) for _, f in counts]
    if sum(E) != sum(F):
        raise RuntimeError(f"migration counts disagree: sum E = {sum(E)}, sum F = {sum(F)}")
    Epre = [sum(E[:g]) for g in range(len(E))]
    Fpre = [sum(F[:g]) for g in range(len(F))]
    send = [_overlap(Epre[rank], Epre[rank] + E[rank], Fpre[g], Fpre[g] + F[g]) for g in range(len(F))]
    recv = [_overlap(Epre[g], Epre[g] + E[g], Fpre[rank], Fpre[rank] + F[rank]) for g in range(len(E))]
    return send, recv


def migrate_sharded(X_local, anc, info, comm=None, stages=None):
    """Cross-GPU particle migration (include/pf.h 4a-4d).

    After ``resample_sharded(..., assemble=False)`` (``anc``, ``info`` as it returned; an
    assembled [P_global] vector works too), applies the whole filter's canonical permutation
    (NS-15) and in-place gather (NS-16) to this rank's state rows ``X_local`` [Pl, ...] (or
    None: indices only).  Returns this rank's slice of the permutation (int32 [Pl]: global
    index of the particle each slot now holds).  Survivors stay; only extra rows travel, in
    one variable all_to_all; the host reads back 16 bytes per rank for the split sizes.
    """
    import torch

    comm = comm or TorchComm()
    stages = stages or GpuStages()
    p0, Pl, P_global = info["p0"], info["Pl"], info["P_global"]
    if X_local is not None and X_local.shape[0] != Pl:
        raise ValueError(f"X_local has {X_local.shape[0]} rows, expected {Pl}")
    if anc.shape[0] == P_global:
        # prefix-sum schemes (or any assembled vector): the rank's particles' ancestors are all here
        # (stratified, systematic, sorted multinomial: within the slot range the search reported)
        rng = info.get("slot_range_dev") if (info["scheme"] in (2, 3) or info["sorted"]) else None
        o = stages.offspring(anc, p0, Pl, rng, info["gmax"], info["gbad"])
    else:
        # Metropolis slots [p0, p0 + Pl): ancestors anywhere -> slot histogram, summed over ranks
        per = -(-P_global // comm.world)
        h = stages.offspring(anc, 0, per * comm.world, None, None, None)
        o = comm.reduce_scatter_sum(h)[:Pl].contiguous()
    cnt, plan = stages.migration_counts(o)
    counts = comm.all_gather_cat(cnt).cpu().view(-1, 2).tolist()
    send, recv = migration_splits(counts, comm.rank)
    rows, src = stages.pack(X_local, o, plan, p0, int(counts[comm.rank][0]))
    rsrc = comm.all_to_all_v(src, send, recv)
    rrows = comm.all_to_all_v(rows, send, recv) if rows is not None else None
    return stages.unpack(X_local, o, plan, p0, rrows, rsrc)


def migrate_sharded_local(X_full, anc_full, nshards: int, stages=None):
    """Fake-shard mode of ``migrate_sharded``: every shard's stages on one device, the
    all-to-all done by slicing.  X_full [P, ...] is updated in place (shard by shard);
    returns the assembled permutation.  Exercises exactly the kernels and split logic."""
    import torch

    stages = stages or GpuStages()
    P = anc_full.shape[0]
    parts = [shard_range(P, nshards, g) for g in range(nshards)]
    Xs = [X_full[p0:p0 + Pl] if X_full is not None else None for p0, Pl in parts]
    os_ = [stages.offspring(anc_full, p0, Pl, None, None, None) for p0, Pl in parts]
    cp = [stages.migration_counts(o) for o in os_]
    counts = [[int(v) for v in c.cpu().tolist()] for c, _ in cp]
    packed = [stages.pack(x, o, cp[g][1], p0, counts[g][0]) for g, (x, o, (p0, _)) in enumerate(zip(Xs, os_, parts))]
    splits = [migration_splits(counts, g) for g in range(nshards)]
    perms = []
    for g, (p0, Pl) in enumerate(parts):
        rows, srcs = [], []
        for h in range(nshards):
            a = sum(splits[h][0][:g])
            n = splits[h][0][g]
            srcs.append(packed[h][1][a:a + n])
            if packed[h][0] is not None:
                rows.append(packed[h][0][a:a + n])
        rsrc = torch.cat(srcs)
        rrows = torch.cat(rows) if rows else None
        perms.append(stages.unpack(Xs[g], os_[g], cp[g][1], p0, rrows, rsrc))
    return torch.cat(perms)


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
    if scheme_id == 1:
        # routed: every slot shard's positions to their owners (the all-to-all by slicing)
        cnts = [stages.route_count(totals, g, P_global, gmax, gbad, seed, filter_index) for g in range(nshards)]
        M = torch.stack(cnts).cpu().tolist()
        packs = [stages.route_pack(totals, g, P_global, gmax, gbad, seed, filter_index, cnts[g], sum(M[g]))
                 for g in range(nshards)]
        for h, ((p0, Pl), (Q, _, _)) in enumerate(zip(parts, scans)):
            xs, ks = [], []
            for g in range(nshards):
                a = sum(M[g][:h])
                xs.append(packs[g][0][a:a + M[g][h]])
                ks.append(packs[g][1][a:a + M[g][h]])
            stages.route_search(Q, p0, P_global, totals, h, gmax, gbad, torch.cat(xs), torch.cat(ks), anc)
        return anc
    for g, ((p0, Pl), (Q, _, _)) in enumerate(zip(parts, scans)):
        stages.search(scheme_id, Q, p0, P_global, totals, g, gmax, gbad, seed, filter_index, anc)
    return anc
