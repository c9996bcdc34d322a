"""SURVEY §8(f3) subset-fraction sweep (the paper's Fig. subset: time to compute a fraction of the
eigenpairs): indices 1..k of a configuration for k/n = 1%, 5%, 10%, 25%, 50%, 100%, ms per solve (CUDA events,
median of 3 after 2 warm-ups) and entries/s.

    python scripts/subset_sweep.py C2 C5a > profiles/r02_subset_sweep.txt
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

print("config  n       fraction  k       ms/solve   entries/s   ms of the all-pairs solve")
for name in sys.argv[1:] or ["C2", "C5a"]:
    cfg = mi.CONFIGS[name]
    d, e = cfg.matrix()
    n = cfg.n
    dt, et = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
    s = m.Solver()
    full = None
    for frac in (1.0, 0.5, 0.25, 0.10, 0.05, 0.01):
        k = max(1, int(round(frac * n)))
        W = torch.empty(k, dtype=torch.float64, device="cuda")
        Z = torch.empty((k, n), dtype=torch.float64, device="cuda")
        ts = []
        for r in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            s.eig(dt, et, 1, k, W=W, Z=Z)
            b.record()
            torch.cuda.synchronize()
            if r >= 2:
                ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        full = ms if full is None else full
        print(f"{name:6s} {n:6d}  {frac:7.2f}  {k:6d}  {ms:9.3f}  {k * n / (ms * 1e-3):10.3e}  {ms / full:6.3f}", flush=True)
        del W, Z
        torch.cuda.empty_cache()
    s.close()
