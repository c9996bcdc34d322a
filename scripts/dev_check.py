"""Developer parity sweep: GPU (libmrrr) vs oracle on small/medium cases; prints one line per case."""
import os
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mrrr_inputs as mi  # noqa: E402
import oracle  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

EPS = 2.0 ** -53


def run(name, d, e, il=None, iu=None, side=0, ortho=True):
    n = d.size
    il = 1 if il is None else il
    iu = n if iu is None else iu
    s = m.Solver(keep_diag=True, root_side=side)
    dt = torch.from_numpy(d).cuda()
    et = torch.from_numpy(e if n > 1 else np.zeros(1)).cuda()
    torch.cuda.synchronize()
    t0 = time.time()
    W, Z = s.eig(dt, et, il, iu)
    torch.cuda.synchronize()
    tg = time.time() - t0
    W = W.cpu().numpy()
    Z = Z.cpu().numpy()
    g = s.diag()
    st = s.stats()
    tm = s.times()
    t0 = time.time()
    r = oracle.mrrr(d, e, il, iu, root_side=side)
    to = time.time() - t0
    tn = max(abs(r.W).max(), 1e-300)
    ne = max(n, 32)
    dW = np.max(np.abs(W - r.W)) / (8 * ne * EPS * tn)
    res = oracle.residuals(d, e, W, Z).max() / (ne * EPS * tn)
    orth = oracle.ortho_full(Z) / (ne * EPS) if ortho else -1
    same = lambda a, b: np.array_equal(a, b, equal_nan=True)
    ints = dict(blocks=same(g.block_start, r.block_start), mu=same(g.mu, r.mu), side=same(g.side, r.side),
                rlo=same(g.root_lo, r.root_lo), rhi=same(g.root_hi, r.root_hi), gst=same(g.root_gstart, r.root_gstart),
                gf=same(g.grp_first, r.grp_first), gl=same(g.grp_last, r.grp_last), dep=same(g.depth, r.depth),
                fin=same(g.fin_lo, r.fin_lo) and same(g.fin_hi, r.fin_hi))
    bad = [k for k, v in ints.items() if not v]
    ok = dW <= 1 and res <= 1 and orth <= 1 and not bad
    print(f"{'OK ' if ok else 'BAD'} {name:18s} n={n:6d} k={iu-il+1:6d} dW={dW:.3g} res={res:.3g} orth={orth:.3g} "
          f"intmismatch={bad} gpu={tg*1e3:.1f}ms oracle={to:.2f}s clusters={st['n_clusters']} "
          f"dmax={st['d_max']} unc={st['uncertified']}/{r.stats['uncertified']} rounds={st['rounds']} "
          f"iters={st['rqi_iters']}/{r.stats['rqi_iters']} fb={st['rqi_fallbacks']} t={tm}", flush=True)
    if "rlo" in bad:
        i = np.nonzero(~((g.root_lo == r.root_lo) | (np.isnan(g.root_lo) & np.isnan(r.root_lo))))[0]
        print("   rlo mismatch at", i[:10], g.root_lo[i[:3]], r.root_lo[i[:3]])
    s.close()
    return ok


cases = [
    ("n1", np.array([3.0]), np.zeros(0)),
    ("n2", *mi.random_tridiag(2, 1, -1.0)),
    ("121_10", *mi.one_two_one(10)),
    ("rand_64", *mi.random_tridiag(64, 3, -1.0)),
    ("121_1000", *mi.one_two_one(1000)),
    ("rand_2000", *mi.random_tridiag(2000, 5, -1.0)),
    ("rand_3001_pos", *mi.random_tridiag(3001, 6, 0.0)),
    ("wilk_101", *mi.wilkinson(50)),
    ("wilk_1001", *mi.wilkinson(500)),
    ("glued_8", *mi.glued_wilkinson(8, 100, 1e-10)),
    ("clement_500", *mi.clement(500)),
    ("hermite_500", *mi.hermite(500)),
]
if len(sys.argv) > 1 and sys.argv[1] == "glued":
    cases = [("glued_128_10", *mi.glued_wilkinson(128, 10, 1e-10))]
allok = True
for c in cases:
    try:
        allok &= run(*c)
    except Exception:
        traceback.print_exc()
        allok = False
if len(sys.argv) > 1:
    print("ALL OK" if allok else "SOME FAILED")
    sys.exit(0)
d, e = mi.random_tridiag(3000, 9, -1.0)
for il, iu in [(1, 40), (100, 400), (2901, 3000)]:
    try:
        allok &= run(f"sub_{il}_{iu}", d, e, il, iu)
    except Exception:
        traceback.print_exc()
        allok = False
rng = np.random.default_rng(3)
d = rng.uniform(-1, 1, 40); e = rng.uniform(-1, 1, 39); e[[4, 5, 17, 30]] = 0.0; e[22] = 1e-300
for il, iu in [(1, 40), (3, 9), (40, 40)]:
    try:
        allok &= run(f"split_{il}_{iu}", d, e, il, iu)
    except Exception:
        traceback.print_exc()
        allok = False
print("ALL OK" if allok else "SOME FAILED")
