# deferred tail: reproduce the MRRR_SEGYW=8 failure matrix by matrix (run under compute-sanitizer)
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
import mrrr_inputs as mi
import paper_1401_4950_b200 as m
which = sys.argv[1] if len(sys.argv) > 1 else "all"
mats = {"rand": mi.random_tridiag(2000, 17, -1.0), "wilk": mi.wilkinson(200), "glued": mi.glued_wilkinson(6, 40, 1e-10)}
for name, (d, e) in mats.items():
    if which != "all" and name != which:
        continue
    s = m.Solver(keep_diag=True)
    try:
        W, Z = s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
        torch.cuda.synchronize()
        st = s.stats()
        print(name, "ok", {k: st[k] for k in ("d_max", "n_clusters", "largest_cluster", "rqi_handover")}, flush=True)
    except Exception as ex:
        print(name, "FAIL", ex, flush=True)
        break
    s.close()
