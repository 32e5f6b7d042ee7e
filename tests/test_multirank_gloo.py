"""World-size-2 multi-process tests of the N>1 paths on CPU (gloo, 127.0.0.1).

* Giant filter sharded over ranks (config C5's decomposition):
  paper_1202_6163_b200.shard.resample_sharded with real torch.distributed
  collectives (all_reduce MAX, all_gather of totals / weights) and CPU stand-in
  stages (oracle-based), assembled ancestors == the oracle's single-filter run.
  Includes the sorted multinomial (a6), whose ranks also all-gather the totals of
  their spacing shards.
* Particle migration (migrate_sharded, include/pf.h 4a-4d): after the sharded resampling,
  the ranks' state rows equal the oracle's in-place gather of the whole filter with its
  canonical permutation (one variable all_to_all of the extra rows over gloo).
* Batched filters sharded over ranks (config C3, bench.py): rank g owns filters
  [g N, (g+1) N) with first_filter = g N; the union equals a single-rank batch.
"""
from __future__ import annotations

import json
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir, cases):
    sys.path.insert(0, ROOT)
    import oracle
    import pfinputs
    from paper_1202_6163_b200.shard import TorchComm, migrate_sharded, resample_sharded, shard_range
    from tests._cpu_shard_stages import CpuOracleStages

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm = TorchComm()
    stages = CpuOracleStages()
    for ci, (scheme, P, var, seed, B, kind) in enumerate(cases):
        x = pfinputs.gaussian_logw(P, var, seed=P)
        if kind == "neg_inf_shard":
            p0, Pl = shard_range(P, world, 1)
            x[p0:p0 + Pl] = -np.inf  # rank 1 holds no weight at all
        if kind == "invalid":
            x[3] = np.nan
        p0, Pl = shard_range(P, world, rank)
        flags = 1 if kind == "sorted" else 0
        anc, info = resample_sharded(scheme, torch.from_numpy(x[p0:p0 + Pl].copy()), P, seed, B=B,
                                     filter_index=5, comm=comm, stages=stages, flags=flags)
        if rank == 0:
            np.save(os.path.join(outdir, f"shard_{ci}.npy"), anc.numpy())
        # migration of the state rows (unassembled ancestors; the permuted form of the whole filter)
        anc_u, info_u = resample_sharded(scheme, torch.from_numpy(x[p0:p0 + Pl].copy()), P, seed, B=B,
                                         filter_index=5, comm=comm, stages=stages, flags=flags, assemble=False)
        X = torch.from_numpy(pfinputs.state_matrix(P, 3, seed=ci)[p0:p0 + Pl].copy())
        perm = migrate_sharded(X, anc_u, info_u, comm=comm, stages=stages)
        np.save(os.path.join(outdir, f"mig_{ci}_{rank}.npy"), X.numpy())
        np.save(os.path.join(outdir, f"migp_{ci}_{rank}.npy"), perm.numpy())
    # batched filters: rank g owns filters [g N, (g+1) N)
    N, P = 3, 500
    xs = pfinputs.gaussian_logw(P, 1.0, seed=11, N=N * world)
    mine = xs[rank * N:(rank + 1) * N]
    st, A = oracle.resample_batched("stratified", mine, 99, first_filter=rank * N)
    parts = [torch.zeros((N, P), dtype=torch.int32) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(A))
    if rank == 0:
        np.save(os.path.join(outdir, "batched.npy"), torch.cat(parts).numpy())
    dist.barrier()
    dist.destroy_process_group()


CASES = [
    ("systematic", 1000, 1.0, 7, 0, ""),
    ("stratified", 999, 10.0, 8, 0, ""),
    ("multinomial", 777, 1.0, 9, 0, ""),
    ("metropolis", 1001, 1.0, 10, 12, ""),
    ("systematic", 1024, 1.0, 11, 0, "neg_inf_shard"),
    ("metropolis", 600, 0.1, 12, 7, "neg_inf_shard"),
    ("stratified", 500, 1.0, 13, 0, "invalid"),
    ("metropolis", 500, 1.0, 14, 3, "invalid"),
    ("multinomial", 1000, 1.0, 15, 0, "sorted"),
    ("multinomial", 777, 10.0, 16, 0, "sorted"),
]


def test_two_rank_giant_filter_and_batches(tmp_path):
    import oracle
    import pfinputs
    from paper_1202_6163_b200.shard import shard_range

    oracle.build()
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), CASES), nprocs=world, join=True)
    for ci, (scheme, P, var, seed, B, kind) in enumerate(CASES):
        x = pfinputs.gaussian_logw(P, var, seed=P)
        if kind == "neg_inf_shard":
            p0, Pl = shard_range(P, world, 1)
            x[p0:p0 + Pl] = -np.inf
        if kind == "invalid":
            x[3] = np.nan
        if kind == "sorted":
            _, want = oracle.resample_sorted_multinomial(x, seed, filter_index=5)
        else:
            _, want = oracle.resample(scheme, x, seed, B=B, filter_index=5)
        got = np.load(os.path.join(tmp_path, f"shard_{ci}.npy"))
        assert np.array_equal(got, want), (scheme, P, kind)
        # migration: the ranks' rows = the whole filter's in-place gather with its permutation
        wp = oracle.permute(want)
        wX = oracle.gather_inplace(pfinputs.state_matrix(P, 3, seed=ci), wp)
        gotX = np.concatenate([np.load(os.path.join(tmp_path, f"mig_{ci}_{r}.npy")) for r in range(world)])
        gotp = np.concatenate([np.load(os.path.join(tmp_path, f"migp_{ci}_{r}.npy")) for r in range(world)])
        assert np.array_equal(gotp, wp), (scheme, P, kind)
        assert np.array_equal(gotX, wX), (scheme, P, kind)
    xs = pfinputs.gaussian_logw(500, 1.0, seed=11, N=3 * world)
    _, want = oracle.resample_batched("stratified", xs, 99, first_filter=0)
    assert np.array_equal(np.load(os.path.join(tmp_path, "batched.npy")), want)


def _worker_errors(rank, world, port, outdir):
    sys.path.insert(0, ROOT)
    import pfinputs
    from paper_1202_6163_b200.shard import TorchComm, resample_sharded, shard_range
    from tests._cpu_shard_stages import CpuOracleStages

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    comm, stages = TorchComm(), CpuOracleStages()
    res = {}
    # a wrong-size shard on rank 1: every rank finishes the exchanges (the filter is NS-1 invalid
    # everywhere), rank 1 raises, rank 0 holds the identity
    P = 600
    x = pfinputs.gaussian_logw(P, 1.0, seed=3)
    for scheme in ("systematic", "metropolis"):
        p0, Pl = shard_range(P, world, rank)
        mine = x[p0:p0 + Pl - (5 if rank == 1 else 0)].copy()
        try:
            anc, _ = resample_sharded(scheme, torch.from_numpy(mine), P, 4, B=3, comm=comm, stages=stages)
            res[scheme] = ("ok", anc.numpy().tolist())
        except ValueError as e:
            res[scheme] = ("error", str(e))
    # a configuration that leaves a rank without particles raises on every rank, before any collective
    try:
        resample_sharded("systematic", torch.zeros(1), 1, 4, comm=comm, stages=stages)
        res["empty"] = ("ok", None)
    except ValueError as e:
        res["empty"] = ("error", str(e))
    dist.barrier()  # both ranks are still in step
    np.save(os.path.join(outdir, f"err_{rank}.npy"), np.array([json.dumps(res)]))
    dist.destroy_process_group()


def test_two_rank_errors_do_not_hang(tmp_path):
    world = 2
    mp.spawn(_worker_errors, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    r0 = json.loads(str(np.load(os.path.join(tmp_path, "err_0.npy"))[0]))
    r1 = json.loads(str(np.load(os.path.join(tmp_path, "err_1.npy"))[0]))
    for scheme in ("systematic", "metropolis"):
        assert r1[scheme][0] == "error" and "shape" in r1[scheme][1]
        assert r0[scheme][0] == "ok" and r0[scheme][1] == list(range(600))  # NS-1: identity
    assert r0["empty"][0] == "error" and r1["empty"][0] == "error"
