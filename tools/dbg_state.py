import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1202_6163_b200 as pf, pfinputs, oracle
dev = torch.device("cuda:0")
for scheme in ("stratified", "systematic"):
    for var in (1.0, 10.0):
        for withperm in (False, True):
            for P in (8192, 8193, 20000, 65536):
                N, D = 4, 16
                x = pfinputs.gaussian_logw(P, var, seed=3, N=N)
                X = np.stack([pfinputs.state_matrix(P, D, seed=n + 50) for n in range(N)])
                gX = torch.from_numpy(X).to(dev)
                perm = torch.empty((N, P), dtype=torch.int32, device=dev) if withperm else None
                a = pf.pf_resample_batched(scheme, torch.from_numpy(x).to(dev), 30, state=gX, permuted_out=perm)
                torch.cuda.synchronize()
                _, want = oracle.resample_batched(scheme, x, 30)
                bad = []
                for n in range(N):
                    wp = oracle.permute(want[n])
                    g = oracle.gather_inplace(X[n], wp)
                    rows = np.nonzero(~np.all(gX[n].cpu().numpy() == g, axis=1))[0]
                    if len(rows):
                        src = [int(np.nonzero(np.all(X[n] == gX[n, r].cpu().numpy(), axis=1))[0][0]) if np.any(np.all(X[n] == gX[n, r].cpu().numpy(), axis=1)) else -1 for r in rows[:5]]
                        bad.append((n, len(rows), rows[:5].tolist(), wp[rows[:5]].tolist(), src))
                print(scheme, var, withperm, P, "anc_ok", np.array_equal(a.cpu().numpy(), want), "bad", bad[:2])
