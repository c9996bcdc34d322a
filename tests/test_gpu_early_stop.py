"""GPU parity of the early classification stop (MRRR_EARLY_STOP, S5'; sec. 3.2.2 remark (3) P:3204-3210,
DESIGN.md A-41) against the oracle run with the same rule: bit-exact block starts, mu, side, every root interval
(stage-1 intervals of the stopped indices, rtol intervals of the others), root group starts, group extents per
depth and final-node intervals; W, residuals and orthogonality within the north_star tolerances; the number of
stopped indices equal on both sides.  C1 and C2 at full size, small cases of every family, subsets with guard
extension, a split matrix, virtual shards and the single/double realisation.
"""
import numpy as np
import pytest

import mrrr_inputs as mi
import oracle
from test_gpu_parity import EPS, SMALL, check_integers, check_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def es_solve(torch, d, e, il=None, iu=None, side=0):
    import paper_1401_4950_b200 as m
    s = m.Solver(keep_diag=True, root_side=side, early_stop=True)
    n = d.size
    W, Z = s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e if n > 1 else np.zeros(1)).cuda(), il, iu)
    torch.cuda.synchronize()
    small = Z.numel() <= (1 << 27)
    return dict(W=W.cpu().numpy(), Z=Z.cpu().numpy() if small else None, Zd=Z, stats=s.stats(), diag=s.diag())


@pytest.mark.parametrize("name", sorted(SMALL))
def test_es_parity_small(torch_cuda, name):
    d, e = SMALL[name]()
    g = es_solve(torch_cuda, d, e)
    r = oracle.mrrr(d, e, early_stop=True)
    assert r.info == 0
    check_integers(g, r)
    tn = max(abs(r.W).max(), 1e-300)
    check_tol(d, e, g["W"], g["Z"], r.W, tn)
    assert oracle.ortho_full(g["Z"]) <= max(d.size, 32) * EPS
    assert g["stats"]["early_stops"] == r.stats["early_stops"]


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_es_parity_full_size(torch_cuda, cfg):
    c = mi.CONFIGS[cfg]
    d, e = c.matrix()
    g = es_solve(torch_cuda, d, e, c.il, c.iu)
    r = oracle.mrrr(d, e, c.il, c.iu, early_stop=True)
    assert r.info == 0
    dg = g["diag"]
    assert np.array_equal(dg.root_lo, r.root_lo, equal_nan=True) and np.array_equal(dg.root_hi, r.root_hi, equal_nan=True)
    assert np.array_equal(dg.root_gstart, r.root_gstart)
    assert g["stats"]["early_stops"] == r.stats["early_stops"] > c.n // 2
    tn = max(abs(r.W).max(), 1e-300)
    assert np.max(np.abs(g["W"] - r.W)) <= 8 * c.n * EPS * tn
    res = oracle.residuals(d, e, g["W"], g["Z"]).max()
    assert res <= c.n * EPS * tn
    Z = g["Z"]
    j = np.arange(c.k - 1)
    assert oracle.ortho_pairs(Z, j, j + 1) <= c.n * EPS
    rng = np.random.default_rng(5)
    pi, pj = rng.integers(0, c.k, 4000), rng.integers(0, c.k, 4000)
    assert oracle.ortho_pairs(Z, pi, pj) <= c.n * EPS
    # the same eigenvalues as the default solve (the early stop changes only where the RQI starts)
    full = oracle.mrrr(d, e, c.il, c.iu, roots_only=True)
    assert np.array_equal(full.root_gstart, r.root_gstart)


@pytest.mark.parametrize("il,iu,side", [(1, 40, 0), (100, 400, 0), (2901, 3000, 0), (1500, 1500, 0), (700, 2100, 1)])
def test_es_parity_subsets(torch_cuda, il, iu, side):
    d, e = mi.random_tridiag(3000, 9, -1.0)
    g = es_solve(torch_cuda, d, e, il, iu, side)
    r = oracle.mrrr(d, e, il, iu, root_side=side, early_stop=True)
    check_integers(g, r)
    check_tol(d, e, g["W"], g["Z"], r.W, max(abs(r.W).max(), 2.0))


def test_es_parity_subset_in_cluster(torch_cuda):
    d, e = mi.wilkinson(300)
    for il, iu in [(600, 601), (2, 2), (300, 450)]:
        g = es_solve(torch_cuda, d, e, il, iu)
        r = oracle.mrrr(d, e, il, iu, early_stop=True)
        check_integers(g, r)
        check_tol(d, e, g["W"], g["Z"], r.W, 301.0)


def test_es_parity_split_matrix(torch_cuda):
    rng = np.random.default_rng(31)
    d = rng.uniform(-1, 1, 2000)
    e = rng.uniform(-1, 1, 1999)
    e[[40, 41, 170, 1200]] = 0.0
    g = es_solve(torch_cuda, d, e)
    r = oracle.mrrr(d, e, early_stop=True)
    assert r.nblocks == 5
    check_integers(g, r)
    check_tol(d, e, g["W"], g["Z"], r.W, max(abs(r.W).max(), 1.0))
    assert g["stats"]["early_stops"] == r.stats["early_stops"] > 0


def test_es_virtual_shards_match_full_solve(torch_cuda):
    # the stop test reads only j-1, j, j+1 (whatever the computed set): every owned column of a shard equals
    # the single-GPU early-stop solve bit for bit, as without the stop
    import paper_1401_4950_b200 as m
    from paper_1401_4950_b200 import dist as pd
    for (d, e), sels in [(mi.random_tridiag(3000, 17, -1.0), [(1, 3000), (1201, 2400)]),
                         (mi.wilkinson(400), [(1, 801), (300, 450)])]:
        dt, et = torch_cuda.from_numpy(d).cuda(), torch_cuda.from_numpy(e).cuda()
        for il, iu in sels:
            g = es_solve(torch_cuda, d, e, il, iu)
            covered = []
            for P in (2, 3):
                for rank in range(P):
                    sl, su = pd.shard_range(il, iu, P, rank)
                    if su < sl:
                        continue
                    s = m.Solver(early_stop=True)
                    jlo, jhi, W, Z = s.eig_shard(dt, et, sl, su, il, iu)
                    if jhi >= jlo:
                        covered.extend(range(jlo, jhi + 1))
                        assert np.array_equal(W.cpu().numpy(), g["W"][jlo - il:jhi - il + 1])
                        assert np.array_equal(Z.cpu().numpy(), g["Z"][:, jlo - il:jhi - il + 1])
                    s.close()
            assert sorted(covered) == sorted(list(range(il, iu + 1)) * 2)


def test_es_single_double(torch_cuda):
    import paper_1401_4950_b200 as m
    d, e = mi.random_tridiag(3000, 44, -1.0)
    d32, e32 = d.astype(np.float32), e.astype(np.float32)
    s = m.Solver(keep_diag=True, early_stop=True)
    W, Z = s.seig(torch_cuda.from_numpy(d32).cuda(), torch_cuda.from_numpy(e32).cuda())
    torch_cuda.cuda.synchronize()
    r = oracle.mrrr(d32.astype(np.float64), e32.astype(np.float64), sd=True, early_stop=True)
    dg = s.diag()
    assert np.array_equal(dg.root_lo, r.root_lo, equal_nan=True) and np.array_equal(dg.root_hi, r.root_hi, equal_nan=True)
    assert np.array_equal(dg.root_gstart, r.root_gstart)
    eps_s = 2.0 ** -24
    assert np.max(np.abs(W.cpu().numpy().astype(np.float64) - r.W)) <= 8 * 3000 * eps_s * 3
