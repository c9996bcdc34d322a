"""Developer check of the segmented RQI on small cases: orthogonality / residual vs the oracle, per K."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import mrrr_inputs as mi, oracle
import paper_1401_4950_b200 as m
EPS = 2.0 ** -53
cases = {"glued_3x21": mi.glued_wilkinson(3, 10, 1e-10), "wilk_21": mi.wilkinson(10), "rand_257": mi.random_tridiag(257, 4, -1.0),
         "rand_2000": mi.random_tridiag(2000, 17, -1.0)}
for name, (d, e) in cases.items():
    for k in sys.argv[1:] or ["1", "2", "8"]:
        os.environ["MRRR_RQISEGK"] = k
        s = m.Solver(keep_diag=True)
        W, Z = s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda())
        torch.cuda.synchronize()
        W, Z = W.cpu().numpy(), Z.cpu().numpy()
        st = s.stats()
        r = oracle.mrrr(d, e)
        n = d.size
        G = np.abs(Z.T @ Z - np.eye(n))
        res = oracle.residuals(d, e, W, Z)
        bad = np.nonzero(G.max(0) > 32 * max(n, 32) * EPS)[0]
        dg = s.diag()
        print(f"{name:12s} K={k} ortho {G.max()/(max(n,32)*EPS):.3g} res {res.max()/(max(n,32)*EPS*np.abs(r.W).max()):.3g} "
              f"handover {st['rqi_handover']} iters {st['rqi_iters']} badcols {bad[:8]} depth {dg.depth[bad[:8]]}", flush=True)
        s.close()
