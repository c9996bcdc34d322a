"""GPU numerical-support truncation (S10', Getvec remark (2) P:3459-3463, A-42; on by default,
MRRR_FULL_SUPPORT turns it off).

* Against the GPU's own full-support solve: W, every integer and interval bit-identical; every entry outside a
  column's support exactly zero; every entry inside equal up to the normalisation (the full solve divides by
  the whole recurrence's ||z||, the truncated one by the support's, in dd; root frames take their factors from
  the z recompute window of k_zrc, the same operations from the same exact states as the stored pass).
* Against the oracle run with the same rule (oracle.mrrr(..., support=True)): the support ends.  They are decided
  by fp64 comparisons of z values that the two sides compute at slightly different lambda-hat (RQI results are
  toleranced, not bit-exact) and, on the GPU, from normalised fl64 values; so an end may move by one row where
  the coupling term sits within rounding of gap*eps_x.  Gate: |end_gpu - end_oracle| <= 1 everywhere and
  >= 99% identical.
* The closed form of tests/test_oracle_support.py (graded diagonal, z(j +- k) = delta^k / k!): exact ends.
* The north_star gates (W, residual, orthogonality) on the truncated vectors; the careful sequential z solve
  (fault injection) and the single/double realisation apply the same rule.
"""
import math

import numpy as np
import pytest

import mrrr_inputs as mi
import oracle
from test_gpu_parity import EPS, check_integers, check_tol

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def solve(torch, d, e, full_support=False, single=False, il=None, iu=None):
    import paper_1401_4950_b200 as m
    s = m.Solver(keep_diag=True, full_support=full_support)
    dt = torch.float32 if single else torch.float64
    n = d.size
    dd = torch.from_numpy(np.asarray(d)).to(dt).cuda()
    ee = torch.from_numpy(np.asarray(e) if n > 1 else np.zeros(1)).to(dt).cuda()
    W, Z = (s.seig if single else s.eig)(dd, ee, il, iu)
    torch.cuda.synchronize()
    out = dict(W=W.cpu().numpy(), Z=Z.cpu().numpy(), stats=s.stats(), diag=s.diag())
    s.close()
    return out


def support(Z):
    nz = Z != 0
    first = nz.argmax(axis=0)
    last = Z.shape[0] - 1 - nz[::-1].argmax(axis=0)
    return first, last


def check_vs_full(g, f):
    assert np.array_equal(g["W"], f["W"])
    for fld in ("root_lo", "root_hi", "root_gstart", "grp_first", "grp_last", "fin_lo", "fin_hi", "depth"):
        assert np.array_equal(getattr(g["diag"], fld), getattr(f["diag"], fld), equal_nan=True), fld
    first, last = support(g["Z"])
    rows = np.arange(g["Z"].shape[0])[:, None]
    inside = (rows >= first[None, :]) & (rows <= last[None, :])
    assert np.all(g["Z"][~inside] == 0.0)
    eps = 2.0 ** -24 if g["Z"].dtype == np.float32 else EPS
    assert np.all(np.abs(g["Z"] - f["Z"])[inside] <= 4 * eps * np.abs(f["Z"])[inside] + 4 * eps * eps), \
        np.max(np.abs(g["Z"] - f["Z"])[inside])
    return first, last


def check_ends(g, r, allow=1, frac=0.99):
    fg, lg = support(g["Z"])
    fr, lr = support(r.Z)
    df, dl = np.abs(fg - fr), np.abs(lg - lr)
    bad = np.flatnonzero((df > allow) | (dl > allow))
    if bad.size:
        print("support ends differ at columns", bad[:10], fg[bad[:10]], fr[bad[:10]], lg[bad[:10]], lr[bad[:10]])
    assert bad.size == 0
    same = np.mean((df == 0) & (dl == 0))
    assert same >= frac, same
    return fg, lg


CASES = {
    "rand_3000": lambda: mi.random_tridiag(3000, 9, -1.0),
    "rand_3001_pos": lambda: mi.random_tridiag(3001, 6, 0.0),
    "121_1000": lambda: mi.one_two_one(1000),
    "wilk_1001": lambda: mi.wilkinson(500),
    "glued_8x201": lambda: mi.glued_wilkinson(8, 100, 1e-10),
    "clement_500": lambda: mi.clement(500),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_support_parity(torch_cuda, name):
    d, e = CASES[name]()
    n = d.size
    g = solve(torch_cuda, d, e)
    f = solve(torch_cuda, d, e, full_support=True)
    check_vs_full(g, f)
    r = oracle.mrrr(d, e, support=True)
    assert r.info == 0
    check_integers(g, r)
    check_ends(g, r)
    tn = max(abs(r.W[0]), abs(r.W[-1]))
    check_tol(d, e, g["W"], g["Z"], r.W, tn)
    assert oracle.ortho_full(g["Z"]) <= max(n, 32) * EPS
    if name.startswith("rand"):
        fg, lg = support(g["Z"])
        assert np.median(lg - fg + 1) < 0.25 * n  # localised vectors: most of each column is not computed
    if name == "121_1000":
        fg, lg = support(g["Z"])
        assert np.all(fg == 0) and np.all(lg == n - 1)  # closed form: nothing negligible


@pytest.mark.parametrize("delta", [1e-3, 1e-2, 1e-1])
def test_support_closed_form(torch_cuda, delta):
    n = 64
    d = np.arange(n, dtype=np.float64)
    e = np.full(n - 1, delta)
    cpl = lambda k: delta * (delta ** k / math.factorial(k) + delta ** (k + 1) / math.factorial(k + 1))
    kstar = next(k for k in range(1, 40) if cpl(k) <= EPS)
    g = solve(torch_cuda, d, e)
    fg, lg = support(g["Z"])
    j = np.arange(kstar + 1, n - kstar - 1)
    assert np.all(fg[j] == j - kstar) and np.all(lg[j] == j + kstar)


def test_support_full_size_C2(torch_cuda):
    c = mi.CONFIGS["C2"]
    d, e = c.matrix()
    g = solve(torch_cuda, d, e)
    f = solve(torch_cuda, d, e, full_support=True)
    first, last = check_vs_full(g, f)
    # the oracle with the same rule on a window of columns (its cost is per vector: run on a subset)
    il, iu = 4001, 4096
    r = oracle.mrrr(d, e, il, iu, support=True)
    sub = dict(Z=g["Z"][:, il - 1:iu])
    check_ends(sub, r)
    tn = max(abs(g["W"][0]), abs(g["W"][-1]))
    assert oracle.residuals(d, e, g["W"], g["Z"]).max() <= c.n * EPS * tn
    jj = np.arange(c.k - 1)
    assert oracle.ortho_pairs(g["Z"], jj, jj + 1) <= c.n * EPS
    print("C2 support rows: median", np.median(last - first + 1), "mean", np.mean(last - first + 1))


@pytest.mark.parametrize("fault", [2])
def test_support_careful_path(torch_cuda, fault, monkeypatch):
    # every Getvec through the careful pass: the sequential z solve (zsolve) applies the rule
    monkeypatch.setenv("MRRR_RQISEG", "0")
    monkeypatch.setenv("MRRR_FAULT", str(fault))
    for d, e in (mi.random_tridiag(1500, 23, -1.0), mi.glued_wilkinson(4, 40, 1e-10)):
        g = solve(torch_cuda, d, e)
        f = solve(torch_cuda, d, e, full_support=True)
        check_vs_full(g, f)
        r = oracle.mrrr(d, e, support=True)
        check_ends(g, r)
        tn = max(abs(r.W[0]), abs(r.W[-1]))
        check_tol(d, e, g["W"], g["Z"], r.W, tn)
        assert g["stats"]["careful"] == d.size


def test_support_single_double(torch_cuda):
    d, e = mi.random_tridiag(3000, 9, -1.0)
    d32, e32 = d.astype(np.float32), e.astype(np.float32)
    g = solve(torch_cuda, d32, e32, single=True)
    f = solve(torch_cuda, d32, e32, single=True, full_support=True)
    check_vs_full(g, f)
    r = oracle.mrrr(d32.astype(np.float64), e32.astype(np.float64), sd=True, support=True)
    rz = type("R", (), {})()
    rz.Z = r.Z.astype(np.float32)
    check_ends(g, rz)
    fg, lg = support(g["Z"])
    assert np.median(lg - fg + 1) < 0.1 * d.size  # eps_x = 2^-24: shorter supports than the double/dd solve
    eps_s = 2.0 ** -24
    tn = max(abs(r.W[0]), abs(r.W[-1]))
    res = oracle.residuals(d32.astype(np.float64), e32.astype(np.float64), g["W"].astype(np.float64),
                           g["Z"].astype(np.float64)).max()
    assert res <= d.size * eps_s * tn


@pytest.mark.parametrize("zwin", ["16", "64"])
def test_zwin_reruns(torch_cuda, zwin, monkeypatch):
    # a z recompute window shorter than the supports: those singletons take a stored pass at the accepted lambda
    # (k_zrc_settle hands a stored pass that does not accept to the two-lane kernel); gates unchanged
    monkeypatch.setenv("MRRR_ZWIN", zwin)
    d, e = mi.random_tridiag(3000, 9, -1.0)
    g = solve(torch_cuda, d, e)
    monkeypatch.setenv("MRRR_ZWIN", "0")
    f = solve(torch_cuda, d, e)  # support on, every factor from a stored pass
    assert g["stats"]["zwin_reruns"] > 0
    r = oracle.mrrr(d, e, support=True)
    check_integers(g, r)
    check_ends(g, r)
    tn = max(abs(r.W[0]), abs(r.W[-1]))
    check_tol(d, e, g["W"], g["Z"], r.W, tn)
    assert oracle.ortho_full(g["Z"]) <= d.size * EPS
    assert np.max(np.abs(g["Z"] - f["Z"])) <= 4 * EPS
