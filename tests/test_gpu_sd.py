"""GPU parity of the single/double realisation (mrrr_seig) against the oracle built
from the same source with -DORACLE_SD (oracle/liboracle_sd.so): binary32 input and output, binary64 inside,
gaptol 1e-5.

The inputs are binary32 values (the synthetic recipes rounded to float32); the oracle receives their exact
binary64 images.  Bit-exact: block starts, mu and side, every root interval, root group starts, group extents
per depth and final-node intervals -- both sides build the child representations with the same binary64
operations (Alg. dstqds P:3324-3351 in the reference order), so unlike the double/dd path (A-33) no rounding
case is allowed.  Toleranced, in eps_s = 2^-24 (the realisation's output precision): |W - W_oracle| <=
8 n eps_s ||T||, max ||T z - lambda z|| <= n eps_s ||T||, max |Z^T Z - I| <= n eps_s (n -> max(n, 32), A-27),
with W and Z the binary32 outputs and the oracle's binary64 results rounded to binary32.
"""
import numpy as np
import pytest

import mrrr_inputs as mi
import oracle

pytestmark = pytest.mark.gpu
EPS_S = 2.0 ** -24


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def f32(d, e):
    return np.asarray(d, np.float32), np.asarray(e, np.float32)


def gpu_seig(torch, d32, e32, il=None, iu=None, side=0):
    import paper_1401_4950_b200 as m
    s = m.Solver(keep_diag=True, root_side=side)
    n = d32.size
    dt = torch.from_numpy(d32).cuda()
    et = torch.from_numpy(e32 if n > 1 else np.zeros(1, np.float32)).cuda()
    W, Z = s.seig(dt, et, il, iu)
    torch.cuda.synchronize()
    assert W.dtype == torch.float32 and Z.dtype == torch.float32
    out = dict(W=W.cpu().numpy(), Z=Z.cpu().numpy(), stats=s.stats(), diag=s.diag())
    s.close()
    return out


def same(a, b):
    return np.array_equal(a, b, equal_nan=True)


def check_integers(g, r):
    dg = g["diag"]
    assert same(dg.block_start, r.block_start)
    assert same(dg.mu, r.mu)
    assert same(dg.side, r.side)
    assert same(dg.root_lo, r.root_lo) and same(dg.root_hi, r.root_hi)
    assert same(dg.root_gstart, r.root_gstart)
    assert same(dg.grp_first, r.grp_first)
    assert same(dg.grp_last, r.grp_last)
    assert same(dg.depth, r.depth)
    mism = ~((dg.fin_lo == r.fin_lo) & (dg.fin_hi == r.fin_hi))
    if np.any(mism):
        print("final-interval mismatches at", np.nonzero(mism)[0][:20])
    assert mism.sum() == 0


def check_tol(d64, e64, g, r, k_ortho=True):
    n = d64.size
    ne = max(n, 32)
    tn = max(oracle.norm1(d64, e64), 1e-300)
    W = g["W"].astype(np.float64)
    Z = g["Z"].astype(np.float64)
    Wref = r.W.astype(np.float32).astype(np.float64)
    assert np.max(np.abs(W - Wref)) <= 8 * ne * EPS_S * tn
    res = oracle.residuals(d64, e64, W, Z).max()
    assert res <= ne * EPS_S * tn, res / (ne * EPS_S * tn)
    if k_ortho:
        assert oracle.ortho_full(Z) <= ne * EPS_S


SMALL = {
    "n1": lambda: (np.array([3.0]), np.zeros(0)),
    "n2": lambda: mi.random_tridiag(2, 1, -1.0),
    "rand_64": lambda: mi.random_tridiag(64, 3, -1.0),
    "rand_257": lambda: mi.random_tridiag(257, 4, -1.0),
    "121_1000": lambda: mi.one_two_one(1000),
    "rand_3001_pos": lambda: mi.random_tridiag(3001, 6, 0.0),
    "rand_3000": lambda: mi.random_tridiag(3000, 9, -1.0),
    "wilk_21": lambda: mi.wilkinson(10),
    "wilk_1001": lambda: mi.wilkinson(500),
    "glued_8x201": lambda: mi.glued_wilkinson(8, 100, 1e-10),
    "clement_500": lambda: mi.clement(500),
    "hermite_400": lambda: mi.hermite(400),
    "legendre_300": lambda: mi.legendre(300),
    "laguerre_300": lambda: mi.laguerre(300),
    "diag_5": lambda: (np.array([3.0, -1.0, 2.0, 2.0, 0.5]), np.zeros(4)),
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_sd_parity_small(torch_cuda, name):
    d32, e32 = f32(*SMALL[name]())
    d64, e64 = d32.astype(np.float64), e32.astype(np.float64)
    g = gpu_seig(torch_cuda, d32, e32)
    r = oracle.mrrr(d64, e64, sd=True)
    assert r.info == 0
    check_integers(g, r)
    check_tol(d64, e64, g, r)
    assert g["stats"]["n_clusters"] == r.stats["n_clusters"]
    assert g["stats"]["uncertified"] == r.stats["uncertified"]


@pytest.mark.parametrize("il,iu,side", [(1, 40, 0), (100, 400, 0), (2901, 3000, 0), (1500, 1500, 0),
                                        (1, 3000, 2), (700, 2100, 1)])
def test_sd_parity_subsets(torch_cuda, il, iu, side):
    d32, e32 = f32(*mi.random_tridiag(3000, 9, -1.0))
    d64, e64 = d32.astype(np.float64), e32.astype(np.float64)
    g = gpu_seig(torch_cuda, d32, e32, il, iu, side)
    r = oracle.mrrr(d64, e64, il, iu, root_side=side, sd=True)
    check_integers(g, r)
    check_tol(d64, e64, g, r)


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_sd_parity_configs(torch_cuda, cfg):
    # the BASELINE configurations C1 (1-2-1, n = 1000) and C2 (random, n = 8192) in binary32, all pairs
    c = mi.CONFIGS[cfg]
    d32, e32 = f32(*c.matrix())
    d64, e64 = d32.astype(np.float64), e32.astype(np.float64)
    g = gpu_seig(torch_cuda, d32, e32)
    r = oracle.mrrr(d64, e64, sd=True)
    check_integers(g, r)
    check_tol(d64, e64, g, r, k_ortho=(c.n <= 2000))
    if c.n > 2000:  # orthogonality on every pair of neighbours plus random pairs (binary128 dots)
        rng = np.random.default_rng(7)
        k = c.n
        pi = np.concatenate([np.arange(k - 1), rng.integers(0, k, 20000)])
        pj = np.concatenate([np.arange(1, k), rng.integers(0, k, 20000)])
        Z = g["Z"].astype(np.float64)
        assert oracle.ortho_pairs(Z, pi, pj) <= k * EPS_S


def test_sd_host_entry(torch_cuda):
    # mrrr_seig_host (host buffers) returns the device entry's results bit for bit
    import paper_1401_4950_b200 as m
    d32, e32 = f32(*mi.random_tridiag(500, 11, -1.0))
    g = gpu_seig(torch_cuda, d32, e32, 20, 300)
    s = m.Solver()
    W, Z = s.eig_host(d32, e32, 20, 300, single=True)
    s.close()
    assert W.dtype == np.float32 and np.array_equal(W, g["W"]) and np.array_equal(Z, g["Z"])


def test_sd_profile_restored(torch_cuda):
    # a single/double solve does not change the handle's double/dd results (profile restored after the call)
    import paper_1401_4950_b200 as m
    d, e = mi.random_tridiag(700, 12, -1.0)
    s = m.Solver()
    dt, et = torch_cuda.from_numpy(d).cuda(), torch_cuda.from_numpy(e).cuda()
    W1, Z1 = s.eig(dt, et)
    W1, Z1 = W1.clone(), Z1.clone()
    s.seig(dt.float(), et.float())
    W2, Z2 = s.eig(dt, et)
    assert torch_cuda.equal(W1, W2) and torch_cuda.equal(Z1, Z2)
    s.close()
