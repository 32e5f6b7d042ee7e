#!/usr/bin/env python
"""bench.py — particle-filter resampling throughput on B200.

One step = one pass of the whole hot path over a batch of synthetic filters
(BASELINE.json configs[2], "batched PMCMC: 1024 independent filters x 2^16"):
  pf_resample_batched(..., offspring_out, permuted_out, state=X): a1-a5 (max,
      dexp + u64 scan, ancestor search), a8 (offspring), a9 (the canonical
      in-place permutation) and a10 (the in-place gather of a D=16 float32
      state) in the one-launch cluster kernel.
The same step as two calls (resample with permutation, then
pf_gather_state_batched) and the generic chain through pf_permute(ancestors)
(histogram path) are timed as extras.
Metric: resampled particles/s (whole job, all ranks).  Multi-GPU: one process
per GPU (torchrun); rank g owns filters [g*N, (g+1)*N) (global Philox filter
indices), no data-path collective -> weak scaling; --strong splits a fixed N.

--impl reference runs the CPU oracle (oracle/, the reference arm of this tier)
on a bounded sample of the same workload on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "resampled particles/sec vs P and weight variance; % of B200 HBM/L2 roofline"
UNIT = "particles/s"

WORKLOADS = {
    # name: (N filters per GPU, P particles, description)
    "c3": (1024, 1 << 16, "C3 batched PMCMC: 1024 filters x 2^16 particles per GPU"),
    "c2": (1, 1 << 20, "C2 single filter P=2^20"),
    "p24": (1, 1 << 24, "single filter P=2^24"),
    # C5: one giant filter, 2^25 particles per GPU (weak), sharded with NCCL exchanges
    "c5": (1, 1 << 25, "C5 giant filter sharded over GPUs: 2^25 particles per GPU"),
    # C4: bootstrap particle filter step on the 16-dim linear-Gaussian model
    "c4": (1, 1 << 18, "C4 bootstrap PF step, linear-Gaussian model, P=2^18, D=16"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--scheme", default="systematic", choices=["multinomial", "stratified", "systematic", "metropolis"])
    ap.add_argument("--B", type=int, default=32, help="Metropolis steps (Metropolis scheme / extras)")
    ap.add_argument("--var", type=float, default=1.0, help="log-weight variance sigma^2")
    ap.add_argument("--D", type=int, default=16, help="state dimension (float32) for the gather")
    ap.add_argument("--strong", action="store_true", help="split a fixed N over ranks (strong scaling)")
    ap.add_argument("--sorted", action="store_true",
                    help="c5 with --scheme multinomial: the sorted-uniform multinomial (a6, PF_SORTED)")
    ap.add_argument("--migrate", type=int, default=0, metavar="D",
                    help="c5: also migrate D float32 state rows per particle across the shards (NEXT-4)")
    ap.add_argument("--no-extras", action="store_true", help="skip per-scheme / e2e / cpu_baseline extras")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers
def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU is under load."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            parts = [p.strip() for p in l.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nme, v in zip(names, parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(nme)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        top = max(sm)
        loaded = [v for v in sm if v >= 0.5 * top] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- GPU arm
def run_c5(args):
    """Giant filter: P_global = 2^25 x world, contiguous shards, NCCL all_reduce / all_gather
    between the shard stages (paper_1202_6163_b200.shard).  The line carries the dominant
    kernel's roofline (library-stated algorithmic bytes over its live CUDA-event time), the
    per-collective device times of a traced pass, the oracle's single-core rate on a bounded
    sample (cpu_baseline) and an end-to-end rate with the log-weight shard copied in from pinned
    host memory and the rank's ancestors copied out every step (e2e)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1202_6163_b200 as pf
    import pfinputs
    from paper_1202_6163_b200.shard import SingleComm, TorchComm, migrate_sharded, resample_sharded, shard_range

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    comm = TorchComm() if world > 1 else SingleComm()
    _, Pper, desc = WORKLOADS["c5"]
    P_global = Pper * world
    p0, Pl = shard_range(P_global, world, rank)
    logw = pfinputs.gaussian_logw_torch(Pl, args.var, pfinputs.BASE_SEED + rank, 1, dev)[0].contiguous()
    scheme = args.scheme
    B = args.B if scheme == "metropolis" else 0
    seed = pfinputs.seed_for(0)

    flags = 1 if (args.sorted and scheme == "multinomial") else 0

    X = None
    if args.migrate:
        gen = torch.Generator(device=dev).manual_seed(pfinputs.BASE_SEED + rank)
        X = torch.randn((Pl, args.migrate), device=dev, generator=gen)

    def step(lw=logw):
        anc, info = resample_sharded(scheme, lw, P_global, seed, B=B, comm=comm, assemble=False, flags=flags)
        if X is not None:  # cross-GPU particle migration of the state rows (include/pf.h 4a-4d)
            migrate_sharded(X, anc, info, comm=comm)
        return anc, info

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    l0 = pf.pf_launch_count()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize(dev)
    launches = pf.pf_launch_count() - l0
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.barrier()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    clocks = sampler.stop()

    # ---------------- traced pass: per-kernel and per-collective device times (same stream)
    kprof = min(args.steps, 5)
    if world > 1:
        comm.timing = True
    pf.pf_profile_enable(True)
    for _ in range(kprof):
        step()
    kt = pf.pf_profile_collect()
    pf.pf_profile_enable(False)
    coll = comm.collect_times() if world > 1 else {}
    if world > 1:
        comm.timing = False
    hbm, peak_src = peaks()
    kernels = {}
    for name, (cnt, tot, alg_sum, _row) in kt.items():
        ent = {"launches_per_step": cnt / kprof, "avg_ms": tot / max(cnt, 1)}
        if alg_sum > 0:
            ent["alg_bytes"] = int(alg_sum / max(cnt, 1))
            ent["gbs"] = ent["alg_bytes"] / (ent["avg_ms"] / 1e3) / 1e9
            ent["frac_hbm"] = ent["gbs"] / hbm
        kernels[name] = ent
    roofline = None
    stated = {k: v for k, v in kernels.items() if "frac_hbm" in v}
    if stated:
        dom = max(stated, key=lambda k: stated[k]["avg_ms"] * stated[k]["launches_per_step"])
        d = stated[dom]
        step_kernel_ms = sum(v["avg_ms"] * v["launches_per_step"] for v in kernels.values())
        roofline = {"bound": "hbm", "kernel": dom, "achieved": round(d["gbs"], 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(d["frac_hbm"], 4), "traffic": None, "alg_bytes_per_launch": d["alg_bytes"],
                    "avg_ms": round(d["avg_ms"], 5),
                    "share_of_step": round(d["avg_ms"] * d["launches_per_step"] / max(step_kernel_ms, 1e-9), 3),
                    "peak_source": peak_src}
    collectives = {k: {"calls_per_step": c / kprof, "ms_per_step": round(m / kprof, 4),
                       "bytes_per_step": int(b / kprof)} for k, (c, m, b) in coll.items()}

    # ---------------- e2e: pinned host shard in, the rank's ancestor slots out, every step
    host_logw = logw.cpu().pin_memory()
    dev_logw = torch.empty_like(logw)
    out_host = torch.empty(max(Pl, 1), dtype=torch.int32).pin_memory()
    h2d = Pl * 4
    d2h_total = 0

    def e2e_step():
        nonlocal d2h_total
        dev_logw.copy_(host_logw, non_blocking=True)
        anc, info = step(dev_logw)
        if scheme == "metropolis":
            a, b = 0, Pl
        else:
            a, b = (int(v) for v in info["slot_range_dev"].tolist())  # device -> host: the rank's slot range
        n = b - a
        if n > out_host.numel():
            return anc
        out_host[:n].copy_(anc[a:b], non_blocking=True)
        d2h_total += n * 4 + (0 if scheme == "metropolis" else 16)
        return anc

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize(dev)
    d2h_total = 0
    if world > 1:
        dist.barrier()
    f0 = torch.cuda.Event(enable_timing=True)
    f1 = torch.cuda.Event(enable_timing=True)
    f0.record()
    for _ in range(args.steps):
        e2e_step()
    f1.record()
    torch.cuda.synchronize(dev)
    te = torch.tensor([f0.elapsed_time(f1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e = {"value": P_global * args.steps / (float(te.item()) / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
           "d2h_bytes_per_step": int(d2h_total / args.steps),
           "note": "rank's pinned host log-weight shard -> H2D -> sharded resample -> D2H of the rank's "
                   "ancestor slots (slot range read back first)"}

    # ---------------- oracle on one host core over a bounded sample (one 2^22-particle filter)
    cpu = None
    if rank == 0 and not args.no_extras:
        import oracle

        oracle.build()
        Ps = 1 << 22
        xs = pfinputs.gaussian_logw(Ps, args.var, pfinputs.BASE_SEED)
        reps, t0 = 0, time.perf_counter()
        while True:
            if flags:
                oracle.resample_sorted_multinomial(xs, seed)
            else:
                oracle.resample(scheme, xs, seed, B=B)
            reps += 1
            if time.perf_counter() - t0 > 10.0 or reps >= 20:
                break
        el = time.perf_counter() - t0
        cpu = {"value": Ps * reps / el, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"{reps} resampling(s) of one 2^22-particle filter of the same law (sigma^2={args.var}, "
                         f"{scheme}{' sorted a6' if flags else ''}{f', B={B}' if B else ''}) on one host thread"}
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": P_global * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 log-weights / u64 fixed-point scan / int32 indices",
            "data": "synthetic",
            "config": {"workload": desc + f", P_global={P_global}, sigma^2={args.var}, scheme={scheme}"
                                  + (" (sorted-uniform, a6)" if flags else "")
                                  + (f", B={B}" if scheme == "metropolis" else "")
                                  + (f", + migration of D={args.migrate} float32 state rows" if args.migrate else ""),
                       "parallelism": f"particle-sharded x{world}: all_reduce(MAX) + all_gather(totals)"
                                      + (" + all_gather(weights)" if scheme == "metropolis" else "")
                                      + (" + all_gather(spacing totals)" if flags else "")
                                      + (" + all_gather(counts) + all_to_all(extra rows)" if args.migrate else ""),
                       "process_group_ranks": dist.get_world_size() if world > 1 else 1,
                       "l2": "inputs larger than L2 (logw 128 MiB/GPU, Q 256 MiB/GPU)"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "kernels": kernels, "collectives": collectives,
        }))
    if world > 1:
        dist.destroy_process_group()


def run_c4(args):
    """C4: one step = one bootstrap-PF time step (propagate + weight, resample with lse, offspring
    and the canonical permutation, in-place gather of the D=16 state, log-likelihood accumulation);
    K steps captured in a CUDA graph (the filter loop is launch-bound at P = 2^18), replayed once
    untimed (graph upload) and once timed."""
    import torch

    import paper_1202_6163_b200 as pf
    import pfinputs
    from paper_1202_6163_b200.pf_demo import LinearGaussianPF

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _, P, desc = WORKLOADS["c4"]
    ys = pfinputs.lg_observations(args.steps + args.warmup, seed=pfinputs.BASE_SEED + rank)
    f = LinearGaussianPF(P=P, D=args.D, scheme=args.scheme, B=args.B if args.scheme == "metropolis" else 0,
                         seed=pfinputs.seed_for(rank), device=dev)
    s = torch.cuda.Stream(dev)
    sampler = ClockSampler(local)
    sampler.start()
    with torch.cuda.stream(s):
        for t in range(args.warmup):
            f.step(float(ys[t]))
    torch.cuda.synchronize(dev)
    g = torch.cuda.CUDAGraph()
    l0 = pf.pf_launch_count()
    with torch.cuda.graph(g, stream=s):
        for t in range(args.steps):
            f.step(float(ys[args.warmup + t]))
    launches = pf.pf_launch_count() - l0
    g.replay()  # untimed: the first replay uploads the graph
    torch.cuda.synchronize(dev)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        e0.record(s)
        g.replay()
        e1.record(s)
    torch.cuda.synchronize(dev)
    ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": P * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32 state / f32 log-weights / u64 scan / int32 indices",
            "data": "synthetic (observations simulated from the model)",
            "config": {"workload": desc + f", scheme={args.scheme}", "P": P, "D": args.D,
                       "pf_steps_per_s": args.steps / (ms / 1e3), "timing": "K steps captured in one CUDA graph"},
            "roofline": None, "cpu_baseline": None, "e2e": None, "gpu_launches": launches, "clocks": clocks,
        }))


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1202_6163_b200 as pf
    import pfinputs

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    N0, P, desc = WORKLOADS[args.workload]
    if args.strong and world > 1:
        N = N0 // world
        first = rank * N
    else:
        N = N0
        first = rank * N0
    stream = torch.cuda.current_stream(dev)
    scheme = args.scheme
    B = args.B if scheme == "metropolis" else 0
    seed = pfinputs.seed_for(0)

    # inputs resident in HBM before timing (weak scaling: each rank its own filters)
    logw = pfinputs.gaussian_logw_torch(P, args.var, pfinputs.BASE_SEED + first, N, dev)
    X = torch.randn((N, P, args.D), generator=torch.Generator(device=dev).manual_seed(first + 1), device=dev,
                    dtype=torch.float32)
    anc = torch.empty((N, P), dtype=torch.int32, device=dev)
    off = torch.empty((N, P), dtype=torch.int32, device=dev)
    perm = torch.empty((N, P), dtype=torch.int32, device=dev)

    # L2 policy (timing rules): the C3 inputs (logw 256 MiB, state 4 GiB) exceed the 126 MB L2;
    # smaller workloads (C2, P = 2^24) flush L2 before every timed step
    flush_l2 = N * P * 4 < 2 * 126 * (1 << 20)
    l2_scratch = torch.empty(1 << 27, dtype=torch.int32, device=dev) if flush_l2 else None

    def step():
        # a1-a5, a8 (offspring), a9 (canonical permutation) and a10 (in-place state gather) in one
        # call (fused into the cluster kernel for P <= 65536)
        pf.pf_resample_batched(scheme, logw, seed, B=B, first_filter=first, ancestors=anc, offspring_out=off,
                               permuted_out=perm, state=X, stream=stream)

    sampler = ClockSampler(local)
    sampler.start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)

    # ---------------- timed region: exactly K steps
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize(dev)
    l0 = pf.pf_launch_count()
    if flush_l2:
        # inputs smaller than twice L2: flush it before every step (a 512 MiB write) and time the
        # steps one by one with events, so no step reads the previous step's inputs from L2
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
        for k in range(args.steps):
            l2_scratch.fill_(k)
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize(dev)
        ms = sum(a.elapsed_time(b) for a, b in ev)
    else:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms = e0.elapsed_time(e1)
    if world > 1:
        dist.barrier()
    launches = pf.pf_launch_count() - l0
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    units = N * P * world * args.steps
    value = units / (ms_max / 1e3)

    # ---------------- per-kernel live durations (separate traced pass, same stream)
    pf.pf_profile_enable(True)
    kprof_steps = min(args.steps, 5)
    for _ in range(kprof_steps):
        step()
    kt = pf.pf_profile_collect()
    pf.pf_profile_enable(False)
    torch.cuda.synchronize(dev)

    # algorithmic bytes per launch of each kernel of the step, as the library states them for
    # what each launch was asked to read and write (pf_kernel_time.alg_bytes), plus one read and
    # one write per state row the gather moved (pf_kernel_time.row_bytes x moved rows)
    survivors = int((off > 0).sum().item())
    moved = N * P - survivors  # rows the in-place gather rewrites (the free slots)
    hbm, peak_src = peaks()
    kernels = {}
    for name, (cnt, tot, alg_sum, row_sum) in kt.items():
        per = tot / max(cnt, 1)
        ent = {"launches_per_step": cnt / kprof_steps, "avg_ms": per}
        if alg_sum > 0:
            alg_launch = (alg_sum + row_sum * moved) / max(cnt, 1)
            ent["alg_bytes"] = int(alg_launch)
            ent["gbs"] = alg_launch / (per / 1e3) / 1e9
            ent["frac_hbm"] = ent["gbs"] / hbm
        kernels[name] = ent
    # committed ncu evidence (DRAM traffic and warp instructions per launch) for this workload
    evidence = {}
    try:
        with open(os.path.join(ROOT, "profiles", "kernel_evidence.json")) as f:
            evidence = json.load(f).get(f"{args.workload}/{scheme}", {})
    except Exception:
        evidence = {}
    # issue roofline: 148 SMs x 4 schedulers x 1 warp-instruction / cycle at the max SM clock
    sm_count = torch.cuda.get_device_properties(dev).multi_processor_count
    issue_peak = sm_count * 4 * 1.965e9 / 1e9  # G warp-instructions / s
    for name, ent in kernels.items():
        ev = evidence.get(name)
        if ev:
            ent["dram_traffic_bytes_ncu"] = ev["dram_bytes"]
            ent["warp_inst_ncu"] = ev["warp_inst"]
            ent["issue_ginst_s"] = ev["warp_inst"] / (ent["avg_ms"] / 1e3) / 1e9
            ent["frac_issue"] = ent["issue_ginst_s"] / issue_peak
    dom = max(kernels, key=lambda k: kernels[k]["avg_ms"] * kernels[k]["launches_per_step"]) if kernels else None
    step_kernel_ms = sum(v["avg_ms"] * v["launches_per_step"] for v in kernels.values())
    roofline = None
    if dom:
        d = kernels[dom]
        share = round(d["avg_ms"] * d["launches_per_step"] / max(step_kernel_ms, 1e-9), 3)
        if d.get("frac_issue", 0.0) > d.get("frac_hbm", 0.0):
            # the kernel is bound by instruction issue, not by HBM
            roofline = {"bound": "alu", "kernel": dom, "achieved": round(d["issue_ginst_s"], 1), "peak": round(issue_peak, 1),
                        "unit": "G warp-inst/s", "frac": round(d["frac_issue"], 4),
                        "traffic": d.get("dram_traffic_bytes_ncu"),
                        "hbm_frac_of_alg_bytes": round(d.get("frac_hbm", 0.0), 4),
                        "alg_bytes_per_launch": d.get("alg_bytes"), "avg_ms": round(d["avg_ms"], 5),
                        "share_of_step": share,
                        "peak_source": f"{sm_count} SMs x 4 schedulers x 1.965 GHz (sm_max_mhz); HBM peak {peak_src}"}
        else:
            roofline = {"bound": "hbm", "kernel": dom, "achieved": round(d.get("gbs", 0.0), 1), "peak": hbm,
                        "unit": "GB/s", "frac": round(d.get("frac_hbm", 0.0), 4),
                        "traffic": d.get("dram_traffic_bytes_ncu"),
                        "alg_bytes_per_launch": d.get("alg_bytes"), "avg_ms": round(d["avg_ms"], 5),
                        "share_of_step": share, "peak_source": peak_src}

    extras = {}
    e2e = None
    if not args.no_extras:
        # ---------------- per-scheme resample-only throughput (same inputs)
        per_scheme = {}
        for sch in ("systematic", "stratified", "multinomial", "metropolis"):
            b = args.B if sch == "metropolis" else 0
            for _ in range(2):
                pf.pf_resample_batched(sch, logw, seed, B=b, first_filter=first, ancestors=anc, stream=stream)
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            reps = max(3, min(args.steps, 10))
            a0.record(stream)
            for _ in range(reps):
                pf.pf_resample_batched(sch, logw, seed, B=b, first_filter=first, ancestors=anc, stream=stream)
            a1.record(stream)
            torch.cuda.synchronize(dev)
            sms = a0.elapsed_time(a1) / reps
            per_scheme[sch if sch != "metropolis" else f"metropolis_B{b}"] = {
                "ms": round(sms, 4), "particles_per_s": N * P / (sms / 1e3)}
        # a6: sorted-uniform multinomial (PF_SORTED)
        for _ in range(2):
            pf.pf_resample_batched("multinomial", logw, seed, first_filter=first, ancestors=anc, flags=pf.PF_SORTED,
                                   stream=stream)
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        for _ in range(reps):
            pf.pf_resample_batched("multinomial", logw, seed, first_filter=first, ancestors=anc, flags=pf.PF_SORTED,
                                   stream=stream)
        a1.record(stream)
        torch.cuda.synchronize(dev)
        sms = a0.elapsed_time(a1) / reps
        per_scheme["multinomial_sorted_a6"] = {"ms": round(sms, 4), "particles_per_s": N * P / (sms / 1e3)}
        extras["resample_only"] = per_scheme

        # binary64 log-weights (NS-3d): the same weights with an accumulated-log-likelihood offset,
        # resample only and the full step (offspring, permutation, D-dim state gather)
        logw64 = logw.double() - 1e7
        f64 = {}
        for label, kw in (("systematic_resample_only", {}),
                          ("systematic_step", {"offspring_out": off, "permuted_out": perm, "state": X})):
            def call64():
                pf.pf_resample_batched("systematic", logw64, seed, first_filter=first, ancestors=anc, stream=stream,
                                       **kw)
            for _ in range(2):
                call64()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(reps):
                call64()
            a1.record(stream)
            torch.cuda.synchronize(dev)
            sms = a0.elapsed_time(a1) / reps
            f64[label] = {"ms": round(sms, 4), "particles_per_s": N * P / (sms / 1e3)}
        del logw64
        extras["f64_logw"] = f64

        # the paper's pre-sorted weight series (PF_SORT_WEIGHTS, NS-17): sort + resample
        presorted = {}
        for sch in ("multinomial", "stratified", "systematic"):
            def call_sorted():
                pf.pf_resample_batched(sch, logw, seed, first_filter=first, ancestors=anc, flags=pf.PF_SORT_WEIGHTS,
                                       stream=stream)
            call_sorted()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            for _ in range(reps):
                call_sorted()
            a1.record(stream)
            torch.cuda.synchronize(dev)
            sms = a0.elapsed_time(a1) / reps
            presorted[sch] = {"ms": round(sms, 4), "particles_per_s": N * P / (sms / 1e3)}
        extras["resample_presorted_weights"] = presorted

        # C1 (BASELINE configs[0]): single resampling of P = 16, latency per call with the calls
        # captured in a CUDA graph (device time, no host overhead on the timeline)
        from tools.sweep import time_calls

        x16 = pfinputs.gaussian_logw_torch(16, 1.0, pfinputs.BASE_SEED, 1, dev)[0].contiguous()
        a16 = torch.empty(16, dtype=torch.int32, device=dev)
        c1 = {}
        for sch in ("multinomial", "stratified", "systematic", "metropolis"):
            b = 32 if sch == "metropolis" else 0
            c1[sch + ("_B32" if b else "")] = round(
                1e3 * time_calls(lambda: pf.pf_resample_ex(sch, x16, seed, b, ancestors=a16), 50, dev), 2)
        extras["c1_latency_us_per_call_P16"] = c1

        # ---------------- the same step as two calls: resample + permutation, then the gather
        def step_two_calls():
            pf.pf_resample_batched(scheme, logw, seed, B=B, first_filter=first, ancestors=anc, offspring_out=off,
                                   permuted_out=perm, stream=stream)
            pf.pf_gather_state(X, perm, stream=stream)

        step_two_calls()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(max(3, min(args.steps, 10))):
            step_two_calls()
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gms = g0.elapsed_time(g1) / max(3, min(args.steps, 10))
        extras["step_two_calls_resample_then_gather"] = {"ms": round(gms, 4), "particles_per_s": N * P / (gms / 1e3)}

        # ---------------- generic chain: permutation from arbitrary ancestors (histogram path)
        def step_generic():
            pf.pf_resample_batched(scheme, logw, seed, B=B, first_filter=first, ancestors=anc, stream=stream)
            pf.pf_permute(anc, permuted=perm, stream=stream)
            pf.pf_gather_state(X, perm, stream=stream)

        step_generic()
        g0 = torch.cuda.Event(enable_timing=True)
        g1 = torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(max(3, min(args.steps, 10))):
            step_generic()
        g1.record(stream)
        torch.cuda.synchronize(dev)
        gms = g0.elapsed_time(g1) / max(3, min(args.steps, 10))
        extras["step_via_pf_permute_of_ancestors"] = {"ms": round(gms, 4), "particles_per_s": N * P / (gms / 1e3)}

        # ---------------- end to end through the public API with host buffers: the chunked
        # host pipeline (paper_1202_6163_b200.pipeline) overlaps each chunk's H2D copy, kernel
        # and D2H copy of the permutation on three streams
        from paper_1202_6163_b200.pipeline import HostPipeline

        h_logw = logw.cpu().pin_memory()
        h_out = torch.empty((N, P), dtype=torch.int32).pin_memory()
        pipe = HostPipeline(N, P, dev, chunks=8)

        def e2e_step():
            pipe.run(scheme, h_logw, seed, h_out, B=B, first_filter=first, state=X, stream=stream, chain=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        b0 = torch.cuda.Event(enable_timing=True)
        b1 = torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        b1.record(stream)
        torch.cuda.synchronize(dev)
        et = torch.tensor([b0.elapsed_time(b1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": N * P * world * args.steps / (float(et.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": N * P * 4, "d2h_bytes_per_step": N * P * 4,
               "note": "host logw (pinned) -> H2D -> resample/permute/gather -> D2H permuted ancestors, "
                       "8 chunks of filters overlapped on three streams, consecutive steps chained "
                       "(paper_1202_6163_b200.pipeline, chain=True); state X stays resident"}
        # the link's own ceiling: both copy directions at once, same bytes, same pinned buffers
        link = link_rates(dev, h_logw, h_out, pipe.d_logw, pipe.perm)
        e2e["link"] = link
        e2e["frac_of_link"] = round(e2e["value"] / (N * P * world / (max(
            N * P * 4 / (link["both_h2d_gbs"] * 1e9), N * P * 4 / (link["both_d2h_gbs"] * 1e9)))), 3)
    clocks = sampler.stop()

    cpu = None
    if rank == 0 and world == 1 and not args.no_extras:
        cpu = cpu_baseline(args, logw.cpu().numpy(), seed, first, budget_s=12.0)

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if (args.strong and world > 1) else "weak", "vs_baseline": None,
            "dtype": "f32 log-weights / u64 fixed-point scan / int32 indices", "data": "synthetic",
            "config": {"workload": desc + f", sigma^2={args.var}, scheme={scheme}"
                                  + (f", B={B}" if scheme == "metropolis" else "")
                                  + f", in-place gather of a D={args.D} f32 state",
                       "filters_per_gpu": N, "P": P, "var": args.var, "scheme": scheme, "D": args.D,
                       "global_filters": N * world, "parallelism": f"filter-sharded x{world} (no collective)",
                       "process_group_ranks": dist.get_world_size() if world > 1 else 1,
                       "l2": ("L2 flushed (512 MiB write) before every timed step; steps timed one by one"
                              if flush_l2 else "inputs larger than L2 (logw N*P*4 B, state N*P*D*4 B), no flush")},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clocks,
            "kernels": kernels,
            "stage_survivor_fraction": survivors / (N * P),
            "extras": extras,
        }
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------------------- CPU oracle legs
def link_rates(dev, h_in, h_out, d_in, d_out, reps: int = 5):
    """Host<->device copy rates over the e2e step's own pinned buffers (GB/s): H2D alone,
    D2H alone, and each direction while both run at once (two streams)."""
    import torch

    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    out = {}
    for name, h2d, d2h in (("h2d", True, False), ("d2h", False, True), ("both", True, True)):
        cur = torch.cuda.current_stream(dev)
        ev = {}
        for tag, s in (("h2d", s1), ("d2h", s2)):
            ev[tag] = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        torch.cuda.synchronize(dev)
        for s in (s1, s2):
            s.wait_stream(cur)
        for it in range(reps + 1):
            if it == 1:
                if h2d:
                    ev["h2d"][0].record(s1)
                if d2h:
                    ev["d2h"][0].record(s2)
            if h2d:
                with torch.cuda.stream(s1):
                    d_in.copy_(h_in, non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_out.copy_(d_out, non_blocking=True)
        if h2d:
            ev["h2d"][1].record(s1)
        if d2h:
            ev["d2h"][1].record(s2)
        torch.cuda.synchronize(dev)
        for tag, on in (("h2d", h2d), ("d2h", d2h)):
            if on:
                ms = ev[tag][0].elapsed_time(ev[tag][1]) / reps
                key = f"{tag}_gbs" if name != "both" else f"both_{tag}_gbs"
                nbytes = h_in.numel() * h_in.element_size() if tag == "h2d" else d_out.numel() * d_out.element_size()
                out[key] = round(nbytes / (ms / 1e3) / 1e9, 2)
    return out


def _oracle_pass(scheme, logw_np, X_np, seed, first, B, threads):
    """Oracle pipeline (resample -> permute -> in-place gather) over the given filters, one filter
    per task on `threads` host threads (ctypes releases the GIL; each call is single-threaded C)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle

    def one(n):
        _, a = oracle.resample(scheme, logw_np[n], seed, B=B, filter_index=first + n)
        p = oracle.permute(a)
        X_np[n] = oracle.gather_inplace(X_np[n], p)
        return 0

    with ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(one, range(logw_np.shape[0])))


def cpu_baseline(args, logw_np, seed, first, budget_s=12.0, n_sample=None):
    import numpy as np

    import oracle

    oracle.build()
    cores = os.cpu_count() or 1
    scheme = args.scheme
    B = args.B if scheme == "metropolis" else 0
    N, P = logw_np.shape
    n_s = n_sample or min(N, max(cores, 32))
    sample = np.ascontiguousarray(logw_np[:n_s])
    X = np.random.default_rng(0).standard_normal((n_s, P, args.D), dtype=np.float32)
    t0 = time.perf_counter()
    passes = 0
    while True:
        _oracle_pass(scheme, sample, X, seed, first, B, cores)
        passes += 1
        el = time.perf_counter() - t0
        if el >= budget_s or passes >= 50:
            break
    return {"value": n_s * P * passes / el, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{passes} pass(es) over the first {n_s} of {N} filters (P={P}, D={args.D}) of the same "
                      f"workload: oracle resample({scheme}) -> permute -> gather, one filter per thread",
            "cpu_model": _cpu_model()}


def _cpu_model():
    try:
        for l in open("/proc/cpuinfo"):
            if l.startswith("model name"):
                return l.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args):
    import numpy as np

    import oracle
    import pfinputs

    world, rank, _ = dist_env()
    if rank != 0:
        return
    oracle.build()
    N, P, desc = WORKLOADS[args.workload]
    scheme = args.scheme
    B = args.B if scheme == "metropolis" else 0
    seed = pfinputs.seed_for(0)
    cores = os.cpu_count() or 1
    n_s = min(N, cores)  # bounded sample per step
    logw = pfinputs.gaussian_logw(P, args.var, pfinputs.BASE_SEED, N=n_s)
    X = np.random.default_rng(0).standard_normal((n_s, P, args.D), dtype=np.float32)
    for _ in range(args.warmup):
        _oracle_pass(scheme, logw, X, seed, 0, B, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        _oracle_pass(scheme, logw, X, seed, 0, B, cores)
    el = time.perf_counter() - t0
    value = n_s * P * args.steps / el
    out = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el * 1e3 / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32 log-weights / u64 fixed-point scan / int32 indices", "data": "synthetic",
        "config": {"workload": desc + f", sigma^2={args.var}, scheme={scheme}, in-place gather of a D={args.D} "
                              "f32 state", "filters_per_gpu": N, "P": P, "var": args.var, "scheme": scheme,
                   "D": args.D},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                         "sample": f"each step: {n_s} of {N} filters (P={P}) through oracle resample -> permute "
                                   f"-> gather, one filter per host thread", "cpu_model": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(out))


def spawn_ranks(n: int) -> int:
    """`--gpus N` (N > 1) without a torchrun environment: launch N ranks of this same command
    line through torch.distributed.run on 127.0.0.1 (one process per GPU), so that a multi-GPU
    request never silently measures one GPU.  Returns the launcher's exit code."""
    import socket

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    print(f"bench.py: spawning {n} ranks: {' '.join(cmd)}", file=sys.stderr)
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}: refusing to report a mismatched run",
              file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    elif args.workload == "c5":
        run_c5(args)
    elif args.workload == "c4":
        run_c4(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
