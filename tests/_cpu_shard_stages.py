"""CPU stand-ins for the shard stages of paper_1202_6163_b200.shard, built on the
oracle (TEST INFRASTRUCTURE).  They let the multi-rank decomposition logic
(offsets from all-gathered totals, slot ranges, assembly) run under
torch.distributed with gloo on CPU; the GPU kernels of the same stages are
checked against the oracle in tests/test_gpu_parity.py (fake-shard mode)."""
from __future__ import annotations

import numpy as np
import torch

import oracle


class CpuOracleStages:
    def max(self, logw):
        x = logw.numpy()
        bad = bool(np.isnan(x).any() or np.isposinf(x).any())
        ok = x[~np.isnan(x) & ~np.isposinf(x)]
        m = np.float32(ok.max()) if ok.size else np.float32(-np.inf)
        return torch.tensor([m], dtype=torch.float32), torch.tensor([int(bad)], dtype=torch.int32)

    def scan(self, logw, P_global, gmax):
        x = logw.numpy()
        g = float(gmax.item())
        Q = oracle.cumulative_with(x, g, oracle.kfx(P_global))
        w = oracle.weights_with(x, g)
        return (torch.from_numpy(Q.view(np.int64).copy()), torch.tensor([int(Q[-1])], dtype=torch.int64),
                torch.tensor([float(np.sum(w.astype(np.float64)))], dtype=torch.float64))

    def search(self, scheme, Q, p0, P_global, totals, shard, gmax, gbad, seed, filter_index, anc_out):
        Ql = Q.numpy().view(np.uint64)
        Pl = len(Ql)
        if int(gbad.item()) or float(gmax.item()) == -np.inf:
            anc_out[p0:p0 + Pl] = torch.arange(p0, p0 + Pl, dtype=torch.int32)
            return torch.tensor([0, 0], dtype=torch.int64)
        tot = [int(v) for v in totals.numpy().view(np.uint64)]
        off, Qtot, T = sum(tot[:shard]), sum(tot), tot[shard]
        ks = []
        for k in range(P_global):
            x = oracle.position(scheme, P_global, Qtot, seed, filter_index, k)
            if off <= x < off + T:
                anc_out[k] = p0 + int(np.searchsorted(Ql, np.uint64(x - off), side="right"))
                ks.append(k)
        rng = (min(ks), max(ks) + 1) if ks else (0, 0)
        return torch.tensor(rng, dtype=torch.int64)

    # routed unsorted multinomial (include/pf.h 3a-3c): slot shard g = [g ceil(P/G), ...)
    @staticmethod
    def _owner(x, tot):
        c = 0
        for h, t in enumerate(tot):
            if c <= x < c + t:
                return h, c
            c += t
        raise AssertionError("position outside [0, Q)")

    def _slot_positions(self, totals, shard, P_global, gmax, gbad, seed, filter_index):
        if int(gbad.item()) or float(gmax.item()) == -np.inf:
            return []
        tot = [int(v) for v in totals.numpy().view(np.uint64)]
        per = -(-P_global // len(tot))
        k0, k1 = min(P_global, shard * per), min(P_global, (shard + 1) * per)
        out = []
        for k in range(k0, k1):
            x = oracle.position(1, P_global, sum(tot), seed, filter_index, k)
            out.append((self._owner(x, tot)[0], x, k))
        return out

    def route_count(self, totals, shard, P_global, gmax, gbad, seed, filter_index):
        c = np.zeros(totals.shape[0], dtype=np.int64)
        for h, _, _ in self._slot_positions(totals, shard, P_global, gmax, gbad, seed, filter_index):
            c[h] += 1
        return torch.from_numpy(c)

    def route_pack(self, totals, shard, P_global, gmax, gbad, seed, filter_index, counts, n_send):
        pos = sorted(self._slot_positions(totals, shard, P_global, gmax, gbad, seed, filter_index))
        assert len(pos) == n_send
        xs = np.array([x for _, x, _ in pos], dtype=np.uint64).view(np.int64)
        ks = np.array([k for _, _, k in pos], dtype=np.int32)
        return torch.from_numpy(xs), torch.from_numpy(ks)

    def route_search(self, Q, p0, P_global, totals, shard, gmax, gbad, rx, rk, anc_out):
        Ql = Q.numpy().view(np.uint64)
        if int(gbad.item()) or float(gmax.item()) == -np.inf:
            anc_out[p0:p0 + len(Ql)] = torch.arange(p0, p0 + len(Ql), dtype=torch.int32)
            return anc_out
        tot = [int(v) for v in totals.numpy().view(np.uint64)]
        off = sum(tot[:shard])
        for x, k in zip(rx.numpy().view(np.uint64), rk.numpy()):
            anc_out[int(k)] = p0 + int(np.searchsorted(Ql, np.uint64(int(x) - off), side="right"))
        return anc_out

    # a6 sorted multinomial (NS-12): spacing totals per spacing shard, positions
    # x_k = floor(G_k Q / G_P) in exact Python integers from the oracle's G.
    @staticmethod
    def _spacing_range(P_global, nshards, h):
        per = -(-(P_global + 1) // nshards)
        return min(P_global + 1, h * per), min(P_global + 1, (h + 1) * per)

    def spacings_total(self, P_global, nshards, shard, seed, filter_index, device=None):
        G = [int(v) for v in oracle.spacings(P_global, seed, filter_index)]
        k0, k1 = self._spacing_range(P_global, nshards, shard)
        tot = (G[k1 - 1] - (G[k0 - 1] if k0 > 0 else 0)) if k1 > k0 else 0
        return torch.tensor([tot], dtype=torch.int64)

    def search_sorted(self, Q, p0, P_global, totals, etotals, shard, gmax, gbad, seed, filter_index, anc_out):
        Ql = Q.numpy().view(np.uint64)
        Pl = len(Ql)
        if int(gbad.item()) or float(gmax.item()) == -np.inf:
            anc_out[p0:p0 + Pl] = torch.arange(p0, p0 + Pl, dtype=torch.int32)
            return torch.tensor([0, 0], dtype=torch.int64)
        tot = [int(v) for v in totals.numpy().view(np.uint64)]
        off, Qtot, T = sum(tot[:shard]), sum(tot), tot[shard]
        GP = sum(int(v) for v in etotals.numpy().view(np.uint64))
        G = [int(v) for v in oracle.spacings(P_global, seed, filter_index)]
        assert G[P_global] == GP
        ks = []
        for k in range(P_global):
            x = G[k] * Qtot // GP
            if off <= x < off + T:
                anc_out[k] = p0 + int(np.searchsorted(Ql, np.uint64(x - off), side="right"))
                ks.append(k)
        rng = (min(ks), max(ks) + 1) if ks else (0, 0)
        return torch.tensor(rng, dtype=torch.int64)

    def weights(self, logw, gmax):
        return torch.from_numpy(oracle.weights_with(logw.numpy(), float(gmax.item())))

    def metropolis(self, w_full, slot0, nslots, seed, B, filter_index, gmax, gbad):
        if int(gbad.item()) or float(gmax.item()) == -np.inf:
            return torch.arange(slot0, slot0 + nslots, dtype=torch.int32)
        a = oracle.metropolis_chains(w_full.numpy(), slot0, nslots, seed, B, filter_index)
        return torch.from_numpy(a)

    # migration stages (include/pf.h 4a-4d) in plain numpy, for the gloo decomposition tests
    def offspring(self, anc, win0, Pw, slot_range, gmax, gbad):
        if gbad is not None and (int(gbad.item()) or float(gmax.item()) == -np.inf):
            return torch.ones(Pw, dtype=torch.int32)
        a = anc.numpy().astype(np.int64)
        if slot_range is not None:
            lo, hi = (int(v) for v in slot_range.tolist())
            a = a[max(lo, 0):min(hi, len(a))]
        a = a[(a >= win0) & (a < win0 + Pw)] - win0
        return torch.from_numpy(np.bincount(a, minlength=Pw).astype(np.int32))

    def migration_counts(self, o):
        v = o.numpy()
        return torch.tensor([int(np.maximum(v - 1, 0).sum()), int((v == 0).sum())], dtype=torch.int64), None

    def pack(self, X, o, plan, p0, E):
        v = o.numpy()
        idx = np.repeat(np.arange(len(v)), np.maximum(v - 1, 0))
        assert len(idx) == E
        rb = X[0].numel() * X.element_size() if X is not None else 0
        rows = None if X is None else X[torch.from_numpy(idx)].contiguous().view(torch.uint8).reshape(E, rb)
        return rows, torch.from_numpy((p0 + idx).astype(np.int32))

    def unpack(self, X, o, plan, p0, rows, src):
        v = o.numpy()
        free = np.flatnonzero(v == 0)
        perm = (p0 + np.arange(len(v))).astype(np.int32)
        perm[free] = src.numpy()
        if X is not None and len(free):
            X[torch.from_numpy(free)] = rows.view(X.dtype).reshape((len(free),) + tuple(X.shape[1:]))
        return torch.from_numpy(perm)
