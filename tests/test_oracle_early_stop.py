"""Pins of the oracle's early classification stop (S5', MRRR_EARLY_STOP; sec. 3.2.2 remark (3) P:3204-3210,
DESIGN.md A-41).  Every expectation is fixed by mathematics or by the paper's own definitions, not by the
oracle's output: Sturm counts of T in binary128 (the interval of index j holds exactly eigenvalue j), binary128
Jacobi eigenvalues for n <= 128, LAPACK's (an independent library) above (the stopped width against the
true gap), the bisection path (a continued index ends exactly
where the default solve ends; a stopped interval contains the default solve's interval), the monotonicity of
reldist under nested intervals (the cluster boundaries are those of the default solve), and the accuracy
gates of the north_star against Jacobi / binary128 residuals.
"""
import numpy as np
import pytest
import scipy.linalg as sla

import mrrr_inputs as mi
import oracle

EPS = 2.0 ** -53

CASES = {
    "rand_600": lambda: mi.random_tridiag(600, 5, -1.0),
    "rand_pos_500": lambda: mi.random_tridiag(500, 8, 0.0),
    "121_400": lambda: mi.one_two_one(400),
    "wilk_201": lambda: mi.wilkinson(100),
    "glued_4x41": lambda: mi.glued_wilkinson(4, 20, 1e-10),
    "clement_300": lambda: mi.clement(300),
    "laguerre_200": lambda: mi.laguerre(200),
    "uniform_300": lambda: mi.uniform_spectrum(300),
}


def test_stage1_tolerance():
    # rtol_c = max(rtol, 2^-(10 + ceil(log2 n))): dyadic, never finer than the classification rtol
    assert oracle.es_rtol(8192, 1e-12) == 2.0 ** -23
    assert oracle.es_rtol(8193, 1e-12) == 2.0 ** -24
    assert oracle.es_rtol(1000, 1e-12) == 2.0 ** -20
    assert oracle.es_rtol(1, 1e-12) == 2.0 ** -10
    assert oracle.es_rtol(1 << 40, 1e-12) == 1e-12


def test_stop_rule_definition():
    # the rule's three clauses, each decided by a case where only that clause fails
    L, C, R = (0.0, 1.0), (10.0, 10.0 + 2.0 ** -7 * 9.0), (300.0, 301.0)
    assert oracle.es_stop(L, C, R, 1e-10)              # width = 2^-7 * absgap (left gap 9): stops (inclusive)
    C2 = (10.0, 10.0 + 2.0 ** -7 * 9.0 * (1 + 2 ** -40))
    assert not oracle.es_stop(L, C2, R, 1e-10)         # width just above 2^-7 * absgap
    assert oracle.es_stop(L, C, R, 0.85)               # reldist left 9/10.07 = 0.89, right 289.9/301 = 0.96
    assert not oracle.es_stop(L, C, R, 0.9)            # left pair no longer a classification boundary
    assert not oracle.es_stop((0.0, 10.0), C, R, 1e-10)  # touching neighbour: gap 0
    assert not oracle.es_stop(C, C, R, 1e-10)          # shared stage-1 node (two indices, one interval)


@pytest.mark.parametrize("name", sorted(CASES))
def test_early_stop_invariants(name):
    d, e = CASES[name]()
    n = d.size
    full = oracle.mrrr(d, e, roots_only=True)
    es = oracle.mrrr(d, e, roots_only=True, early_stop=True)
    assert full.info == 0 and es.info == 0
    lo, hi, flo, fhi = es.root_lo, es.root_hi, full.root_lo, full.root_hi
    cont = (lo == flo) & (hi == fhi)
    stopped = ~cont
    assert es.stats["early_stops"] == int(stopped.sum()) or es.stats["early_stops"] >= int(stopped.sum())
    # a stopped interval contains the default solve's interval (the same bisection path, cut earlier)
    assert np.all(lo[stopped] <= flo[stopped]) and np.all(fhi[stopped] <= hi[stopped])
    # the block's first and last index never stop
    assert cont[0] and cont[-1]
    # cluster boundaries are those of the default solve (reldist only grows under nested intervals)
    assert np.array_equal(es.root_gstart, full.root_gstart)
    # Sturm counts of T itself (binary128, Alg. negcountT): index j's interval holds exactly eigenvalue j
    mu = es.mu[0]
    for j in np.nonzero(stopped)[0][:64]:
        assert oracle.negcount_t(d, e, lo[j], mu) <= j < oracle.negcount_t(d, e, hi[j], mu)
    # width <= 2^-7 of the true gap (LAPACK eigenvalues, error ~1e-16 ||T||; the stage-1 gap is a lower
    # bound of the true gap)
    lam = sla.eigvalsh_tridiagonal(d, e)
    tn = max(abs(lam[0]), abs(lam[-1]))
    x = lam - mu
    gap = np.minimum(np.r_[np.inf, np.diff(x)], np.r_[np.diff(x), np.inf])
    w = hi - lo
    assert np.all(w[stopped] <= 2.0 ** -7 * gap[stopped] + 1e-14 * tn)
    # every stopped index is a certified singleton: its relative gaps exceed gaptol
    rel = gap / np.maximum(np.abs(x), 1e-300)
    assert np.all(rel[stopped] >= 1e-10)


SMALL = {
    "rand_120": lambda: mi.random_tridiag(120, 5, -1.0),
    "121_100": lambda: mi.one_two_one(100),
    "wilk_41": lambda: mi.wilkinson(20),
    "glued_3x21": lambda: mi.glued_wilkinson(3, 10, 1e-10),
    "clement_90": lambda: mi.clement(90),
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_early_stop_full_solve_vs_jacobi(name):
    d, e = SMALL[name]()
    n = d.size
    r = oracle.mrrr(d, e, early_stop=True)
    assert r.info == 0
    lam, _ = oracle.jacobi(d, e)
    tn = max(abs(lam[0]), abs(lam[-1]))
    assert np.max(np.abs(r.W - lam)) <= 8 * n * EPS * tn
    assert oracle.residuals(d, e, r.W, r.Z).max() <= n * EPS * tn
    assert oracle.ortho_full(r.Z) <= n * EPS
    if name in ("rand_120", "121_100"):
        assert r.stats["early_stops"] > n // 2


@pytest.mark.parametrize("name", ["rand_600", "121_400", "wilk_201"])
def test_early_stop_full_solve_accuracy(name):
    d, e = CASES[name]()
    n = d.size
    r = oracle.mrrr(d, e, early_stop=True)
    assert r.info == 0
    lam = sla.eigvalsh_tridiagonal(d, e)
    tn = max(abs(lam[0]), abs(lam[-1]))
    assert np.max(np.abs(r.W - lam)) <= 8 * n * EPS * tn
    assert oracle.residuals(d, e, r.W, r.Z).max() <= n * EPS * tn
    assert oracle.ortho_full(r.Z) <= n * EPS
    assert r.stats["early_stops"] > 0


def test_early_stop_subsets_and_guards():
    # subsets (guard extension, one index at a time): the same intervals as the all-pairs early-stop solve
    # (the stop test depends only on j-1, j, j+1) and the default solve's computed set
    d, e = mi.random_tridiag(800, 21, -1.0)
    allp = oracle.mrrr(d, e, roots_only=True, early_stop=True)
    for il, iu in [(1, 1), (2, 50), (300, 420), (799, 800)]:
        s = oracle.mrrr(d, e, il, iu, roots_only=True, early_stop=True, root_side=1)
        f = oracle.mrrr(d, e, il, iu, roots_only=True, root_side=1)
        comp = ~np.isnan(s.root_lo)
        assert np.array_equal(comp, ~np.isnan(f.root_lo))
        assert np.array_equal(s.root_lo[comp], allp.root_lo[comp]) and np.array_equal(s.root_hi[comp], allp.root_hi[comp])
    dw, ew = mi.wilkinson(150)
    for il, iu in [(300, 301), (150, 160)]:
        s = oracle.mrrr(dw, ew, il, iu, early_stop=True)
        f = oracle.mrrr(dw, ew, il, iu)
        assert np.array_equal(s.root_gstart, f.root_gstart)
        assert np.max(np.abs(s.W - f.W)) <= 8 * dw.size * EPS * 151


def test_early_stop_multiblock():
    rng = np.random.default_rng(31)
    d = rng.uniform(-1, 1, 300)
    e = rng.uniform(-1, 1, 299)
    e[[40, 41, 170]] = 0.0
    r = oracle.mrrr(d, e, early_stop=True)
    f = oracle.mrrr(d, e)
    assert r.info == 0 and r.nblocks == 4
    assert np.array_equal(r.root_gstart, f.root_gstart)
    lam = sla.eigvalsh_tridiagonal(d, e)
    assert np.max(np.abs(r.W - lam)) <= 8 * 300 * EPS * 3
    assert oracle.residuals(d, e, r.W, r.Z).max() <= 300 * EPS * 3
    assert r.stats["early_stops"] > 0


def test_early_stop_single_double():
    d, e = mi.random_tridiag(400, 44, -1.0)
    d32, e32 = d.astype(np.float32).astype(np.float64), e.astype(np.float32).astype(np.float64)
    r = oracle.mrrr(d32, e32, sd=True, early_stop=True)
    f = oracle.mrrr(d32, e32, sd=True)
    assert r.info == 0
    assert np.array_equal(r.root_gstart, f.root_gstart)
    lam = sla.eigvalsh_tridiagonal(d32, e32)
    eps_s = 2.0 ** -24
    assert np.max(np.abs(r.W - lam)) <= 8 * 400 * eps_s * 3
