"""SURVEY §8(f1) sweep: the paper's synthetic families (App. D) at n = 2,500 .. 20,000 on one B200,
all eigenpairs: time, entries/s, clustering rho = largest cluster / n (Table tab:clusteringdouble P:6560-6590),
d_max, phi = fraction of computed representations that pass the growth test, and
the paper's accuracy measures (def:defresortho2) R = max_i ||T z_i - lambda_i z_i||_1 / ||T||_1 and
O = max_{i != j} |z_i^T z_j|, printed as multiples of n eps.  (GPU vs oracle parity of the same families is in
tests/test_gpu_families.py; R and O here are fp64 evaluations on the device, a diagnostic, not a gate.)

    python scripts/family_sweep.py [sizes...] > profiles/r02_family_sweep.txt
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

EPS = 2.0 ** -53
sizes = [int(x) for x in sys.argv[1:]] or [2500, 5000, 10000, 20000]
print("family      n      ms/solve  entries/s   rho*n  rho      d_max  phi    R/(n eps)  O/(n eps)  blocks")
for fam in ["uniform", "geometric", "121", "clement", "wilkinson", "hermite", "legendre", "laguerre"]:
    for n0 in sizes:
        if fam in ("uniform", "geometric") and n0 > 5000:
            continue  # dense similarity + reduction on the host: O(n^3)
        d, e = mi.FAMILIES[fam](n0)
        n = d.size
        dt, et = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
        s = m.Solver()
        W = torch.empty(n, dtype=torch.float64, device="cuda")
        Z = torch.empty((n, n), dtype=torch.float64, device="cuda")
        for _ in range(2):
            s.eig(dt, et, W=W, Z=Z)
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            _, Zc = s.eig(dt, et, W=W, Z=Z)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        st = s.stats()
        # R: 1-norm residuals of all columns (tridiagonal product on the device), O: off-diagonal of Z^T Z
        Zm = Zc  # (n, n), column j = eigenvector j
        TZ = dt[:, None] * Zm
        TZ[1:] += et[:, None] * Zm[:-1]
        TZ[:-1] += et[:, None] * Zm[1:]
        res = (TZ - Zm * W[None, :]).abs().sum(0).max().item()
        tn1 = max(float(np.max(np.abs(d) + np.append(np.abs(e), 0) + np.append(0, np.abs(e)))), 1e-300)
        R = res / tn1
        G = Zm.T @ Zm
        G.fill_diagonal_(0.0)
        O = G.abs().max().item()
        rho_n = max(st["largest_cluster"], 1)
        phi = 1.0 - st["uncertified"] / max(st["n_clusters"], 1)
        print(f"{fam:10s} {n:6d} {ms:10.3f} {n * n / (ms * 1e-3):10.3e} {rho_n:6d} {rho_n / n:8.2e} {st['d_max']:5d} "
              f"{phi:5.2f}  {R / (n * EPS):9.3f}  {O / (n * EPS):9.3f}  {st['nblocks']}", flush=True)
        del Z, Zc, Zm, TZ, G
        s.close()
        torch.cuda.empty_cache()
