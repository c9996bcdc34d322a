"""Pins of the single/double oracle (liboracle_sd.so: oracle/mrrr_oracle.c built with -DORACLE_SD; P:6224-6248,
SURVEY §8(f2)) against what the paper and the mathematics fix: binary128 Jacobi brute force (n <= 64), the 1-2-1
closed form (App. D), Sturm-count invariants, the split rule with eps_x = 2^-24,
the perturbation size xi = eps_x, the residual / orthogonality targets in eps_s = 2^-24, the
published clustering structure of the Wilkinson family, and the fact that the realisation computes in binary64
(its results are not those of the binary128 oracle).  No expected value comes from the oracle or the CUDA path.
"""
import math

import numpy as np
import pytest

import mrrr_inputs as mi
import oracle

EPS_S = 2.0 ** -24


def f32(d, e):
    return np.asarray(d, np.float32).astype(np.float64), np.asarray(e, np.float32).astype(np.float64)


def acc(d, e, r):
    """(max residual / (||T|| n_eff eps_s), max |Z^T Z - I| / (n_eff eps_s)) of the binary32-rounded output"""
    n = d.size
    ne = max(n, 32)
    W = r.W.astype(np.float32).astype(np.float64)
    Z = r.Z.astype(np.float32).astype(np.float64)
    tn = oracle.norm1(d, e)
    return (oracle.residuals(d, e, W, Z).max() / (tn * ne * EPS_S), oracle.ortho_full(Z) / (ne * EPS_S))


FAMS = {
    "rand": lambda n: mi.random_tridiag(n, 5 + n, -1.0),
    "rand_pos": lambda n: mi.random_tridiag(n, 9 + n, 0.0),
    "121": lambda n: mi.one_two_one(n),
    "wilk": lambda n: mi.wilkinson((n - 1) // 2),
    "clement": lambda n: mi.clement(n),
    "laguerre": lambda n: mi.laguerre(n),
}


@pytest.mark.parametrize("fam", sorted(FAMS))
@pytest.mark.parametrize("n", [2, 7, 31, 63])
def test_sd_small_vs_jacobi(fam, n):
    if fam == "wilk" and n % 2 == 0:
        n += 1
    d, e = f32(*FAMS[fam](n))
    r = oracle.mrrr(d, e, sd=True)
    assert r.info == 0
    hi, lo = oracle.jacobi(d, e)
    tn = max(abs(hi[0]), abs(hi[-1]))
    W = r.W.astype(np.float32).astype(np.float64)
    assert np.max(np.abs(W - hi)) <= 8 * max(n, 32) * EPS_S * tn
    res, orth = acc(d, e, r)
    assert res <= 1.0 and orth <= 1.0


@pytest.mark.parametrize("n", [100, 1000])
def test_sd_121_closed_form(n):
    d, e = mi.one_two_one(n)   # binary32-exact data
    r = oracle.mrrr(d, e, sd=True)
    j = np.arange(1, n + 1, dtype=np.longdouble)
    lam = 4 * np.sin(j * np.pi / (2 * (n + 1))) ** 2
    W = r.W.astype(np.float32).astype(np.longdouble)
    assert np.max(np.abs(W - lam)) <= 8 * n * EPS_S * 4
    res, orth = acc(d, e, r)
    assert res <= 1 and orth <= 1


def test_sd_is_binary64_not_binary128():
    # the two realisations share the steps but not the arithmetic: on a random matrix their W differ by far more
    # than binary64 rounding of one result (xi = 2^-25 vs 2^-54 perturbations, binary64 vs binary128 y-data),
    # while both stay within their own accuracy targets
    d, e = f32(*mi.random_tridiag(300, 3, -1.0))
    a = oracle.mrrr(d, e, sd=True)
    b = oracle.mrrr(d, e)
    diff = np.max(np.abs(a.W - b.W))
    assert diff > 1e-12
    assert diff <= 8 * 300 * EPS_S * oracle.norm1(d, e)


def test_sd_perturbation_scale():
    # xi = eps_x: the same counter-based SplitMix64 stream as the double/quadruple realisation,
    # scaled to [-2^-25, 2^-25)
    raw = mi.splitmix64(7, 64)
    for idx in range(64):
        u = float(int(raw[idx]) >> 11) * 2.0 ** -53
        x = oracle.xi(7, idx, sd=True)
        assert x == (u - 0.5) * 2.0 ** -24
        assert -(2.0 ** -25) <= x < 2.0 ** -25


def test_sd_root_is_binary64_perturbed():
    # S3 in binary64: d_y = fl64(d_x + fl64(d_x xi)), and M_x = M_y (no binary64 copy is rounded)
    d, e = f32(*mi.random_tridiag(50, 4, -1.0))
    r = oracle.root_y(d, e, True, 0, sd=True)
    rx = oracle.root_x(d, e, True)
    assert np.all(r["d_lo"] == 0.0) and np.all(r["l_lo"] == 0.0)
    assert np.array_equal(r["dx"], r["d_hi"])
    rel = np.abs(r["d_hi"] - rx["d"]) / np.abs(rx["d"])
    assert np.max(rel) <= 2.0 ** -25 + 2.0 ** -52 and np.max(rel) > 2.0 ** -40   # perturbed by ~eps_x, not eps_y


def test_sd_split_threshold():
    # |beta_i| <= eps_x sqrt(n) ||T||_1 with eps_x = 2^-24: inclusive, one ulp above does not split
    d = np.array([3.0, 1.0, 1.0, 1.0])
    tol = (EPS_S * math.sqrt(4.0)) * 4.0
    e = np.array([1.0, tol, 1.0])
    assert list(oracle.split(d, e, sd=True)) == [0, 2, 4]
    assert list(oracle.split(d, e)) == [0, 4]          # the double realisation's eps_x = 2^-53 keeps it whole
    e[1] = np.nextafter(tol, 1.0)
    assert list(oracle.split(d, e, sd=True)) == [0, 4]
    r = oracle.mrrr(d, np.array([1.0, tol, 1.0]), sd=True)
    assert r.nblocks == 2


@pytest.mark.parametrize("n", [40, 300])
def test_sd_sturm_invariant_root_intervals(n):
    # every computed root interval brackets its index on the representation's own x-count (Alg. Bisection
    # P:3077-3111), and is no wider than rtol = 1e-2 gaptol = 1e-7 relative
    d, e = f32(*mi.random_tridiag(n, 21, -1.0))
    r = oracle.mrrr(d, e, sd=True)
    ry = oracle.root_y(d, e, bool(r.side[0] == 1), 0, sd=True)
    for j in range(1, n + 1):
        lo, hi = r.root_lo[j - 1], r.root_hi[j - 1]
        assert oracle.negcount_x(ry["dx"], ry["dllx"], lo) < j <= oracle.negcount_x(ry["dx"], ry["dllx"], hi)
        assert hi - lo <= max(1e-7 * max(abs(lo), abs(hi)), 2 * 2.2250738585072014e-308)


def test_sd_gaptol_1e5_classification():
    # gaptol 1e-5: root groups split exactly where reldist >= 1e-5 between neighbours' intervals
    d, e = f32(*mi.random_tridiag(400, 8, -1.0))
    r = oracle.mrrr(d, e, sd=True)
    for j in range(2, 401):
        lo1, hi1, lo2, hi2 = r.root_lo[j - 2], r.root_hi[j - 2], r.root_lo[j - 1], r.root_hi[j - 1]
        rel = (lo2 - hi1) / max(abs(lo1), abs(hi1), abs(lo2), abs(hi2))
        assert r.root_gstart[j - 1] == (1 if rel >= 1e-5 else 0)


@pytest.mark.parametrize("m", [10, 100])
def test_sd_wilkinson_pairs(m):
    # Wilkinson pairs are clusters at gaptol 1e-5 as at 1e-10 (rho = 2/n, d_max = 1, phi = 1: Table
    # tab:clusteringdouble P:6580-6581), accuracy in eps_s
    d, e = mi.wilkinson(m)
    r = oracle.mrrr(d, e, sd=True)
    assert r.info == 0
    assert r.stats["largest_cluster"] >= 2 and r.stats["d_max"] >= 1 and r.stats["uncertified"] == 0
    res, orth = acc(d, e, r)
    assert res <= 1 and orth <= 1


def test_sd_glued_clusters_vs_jacobi():
    # glued Wilkinson (n = 63): deep clusters through the binary64 child representations, checked against
    # binary128 Jacobi
    d, e = mi.glued_wilkinson(3, 10, 1e-10)
    r = oracle.mrrr(d, e, sd=True)
    hi, _ = oracle.jacobi(d, e)
    tn = max(abs(hi[0]), abs(hi[-1]))
    assert r.stats["n_clusters"] > 0
    assert np.max(np.abs(r.W.astype(np.float32) - hi)) <= 8 * 63 * EPS_S * tn
    res, orth = acc(d, e, r)
    assert res <= 1 and orth <= 1
