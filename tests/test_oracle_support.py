"""Pins of the oracle's numerical-support truncation (S10', Getvec remark (2) P:3459-3463, A-42).

The rule: going outward from the twist index r (z(r) = 1), the support ends at the first edge i with
|dl(i)| (|z(i)| + |z(i+1)|) <= gap eps_x; the entries past it are zero.  Every expectation below is fixed by
mathematics, not by the oracle's output:
  * a closed form -- on T = diag(0, 1, ..., n-1) + delta (off-diagonal) the eigenvector of lambda ~ j has
    z(j +- k) = delta^k / k! (1 + O(k delta^2)) (first-order perturbation series, row j+k of (T - lambda) z = 0),
    so the support is exactly [j - k*, j + k*] with k* the first k whose coupling term
    delta (delta^k/k! + delta^(k+1)/(k+1)!) is below gap eps_x (cases chosen with a factor >= 2 margin);
  * the 1-2-1 closed form z_j(i) ~ sin(i j pi / (n + 1)): no entry is negligible, so nothing is truncated;
  * the gap theorem: the cut changes the residual by at most gap eps_x, so the truncated vector stays within
    O(eps_x) of the untruncated one, and the north_star gates (residual, orthogonality, binary128) still hold --
    also on Wilkinson / glued-Wilkinson inputs, whose resolved child-level pairs carry mass at both ends of the
    matrix (both ends must survive);
  * W and every integer output are unchanged (the truncation acts after the RQI).
"""
import math

import numpy as np
import pytest

import mrrr_inputs as mi
import oracle

EPS = 2.0 ** -53


def _support(Z):
    """first / last nonzero row of every column (columns are never all zero)"""
    nz = Z != 0
    first = nz.argmax(axis=0)
    last = Z.shape[0] - 1 - nz[::-1].argmax(axis=0)
    return first, last


def _coupling(delta, k):
    return delta * (delta ** k / math.factorial(k) + delta ** (k + 1) / math.factorial(k + 1))


@pytest.mark.parametrize("delta", [1e-3, 1e-2, 1e-1])
def test_support_closed_form_graded_diagonal(delta):
    n = 64
    d = np.arange(n, dtype=np.float64)
    e = np.full(n - 1, delta)
    tau = 1.0 * EPS  # gap ~ 1 (neighbours at distance 1 - O(delta^2))
    kstar = next(k for k in range(1, 40) if _coupling(delta, k) <= tau)
    assert _coupling(delta, kstar) <= tau / 2 and _coupling(delta, kstar - 1) >= 2 * tau  # margin of the case
    res = oracle.mrrr(d, e, support=True)
    full = oracle.mrrr(d, e)
    assert res.info == 0 and np.array_equal(res.W, full.W)
    first, last = _support(res.Z)
    for j in range(kstar + 1, n - kstar - 1):  # interior eigenvectors (lambda_j ~ j, 0-based)
        assert first[j] == j - kstar and last[j] == j + kstar, (j, first[j], last[j], kstar)
        # the entries kept follow the closed form delta^k / k! (relative O(k delta^2))
        z = res.Z[:, j] / res.Z[j, j]
        for k in range(1, kstar + 1):
            want = delta ** k / math.factorial(k)
            assert abs(abs(z[j + k]) / want - 1) <= 4 * k * delta ** 2 + 1e-12
            assert abs(abs(z[j - k]) / want - 1) <= 4 * k * delta ** 2 + 1e-12
    assert res.stats["support_rows"] == int(np.sum(last - first + 1))


def test_support_121_closed_form_full():
    # z_j(i) ~ sin(i j pi / (n+1)): the smallest |entry| is ~ sin(pi/(n+1)) / sqrt(n/2), never negligible
    n = 400
    d, e = mi.one_two_one(n)
    res = oracle.mrrr(d, e, support=True)
    first, last = _support(res.Z)
    assert np.all(first == 0) and np.all(last == n - 1)
    assert res.stats["support_rows"] == n * n


CASES = {
    "rand_800": lambda: mi.random_tridiag(800, 11, -1.0),
    "rand_pos_600": lambda: mi.random_tridiag(600, 12, 0.0),
    "wilk_201": lambda: mi.wilkinson(100),
    "glued_4x41": lambda: mi.glued_wilkinson(4, 20, 1e-10),
    "glued_8x201": lambda: mi.glued_wilkinson(8, 100, 1e-10),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_support_gap_theorem_and_gates(name):
    d, e = CASES[name]()
    n = d.size
    res = oracle.mrrr(d, e, support=True)
    full = oracle.mrrr(d, e)
    assert res.info == 0 and full.info == 0
    assert np.array_equal(res.W, full.W)
    for f in ("root_lo", "root_hi", "root_gstart", "grp_first", "grp_last", "fin_lo", "fin_hi", "depth"):
        assert np.array_equal(getattr(res, f), getattr(full, f), equal_nan=True), f
    # contiguous support: zeros only outside [first, last]
    first, last = _support(res.Z)
    rows = np.arange(n)[:, None]
    inside = (rows >= first[None, :]) & (rows <= last[None, :])
    assert np.all(res.Z[inside] != 0)
    # gap theorem: the cut moves each vector by O(eps_x) (entries kept agree with the full vector to rounding)
    dz = np.abs(res.Z - full.Z).max(axis=0)
    assert dz.max() <= 4 * EPS, dz.max()
    # north_star gates in binary128 on the truncated vectors
    tn = max(abs(res.W[0]), abs(res.W[-1]))
    nn = max(n, 32)
    assert oracle.residuals(d, e, res.W, res.Z).max() <= nn * EPS * tn
    assert oracle.ortho_full(res.Z) <= nn * EPS
    if name.startswith("rand"):
        # localised vectors (1-D random matrices): the support is a small part of the column
        assert np.median(last - first + 1) < 0.5 * n


def test_support_wilkinson_two_ended_vectors_kept():
    # W+_21: the top pairs (splitting 7e-14 and 6e-11) are resolved clusters whose child-level singletons are the
    # symmetric / antisymmetric combinations with mass ~0.38 and ~0.55 at BOTH ends of the matrix; the rule
    # must keep the far end (the pair stays orthogonal).  (For W+_201 the top pairs split below eps ||T||: any
    # basis of the pair is an answer, and the computed one is localised at one end.)
    d, e = mi.wilkinson(10)
    res = oracle.mrrr(d, e, support=True)
    full = oracle.mrrr(d, e)
    n = d.size
    top = np.argsort(res.W)[-4:]
    assert res.stats["d_max"] >= 1  # the pairs went through the cluster path
    for j in top:
        z = res.Z[:, j]
        assert abs(z[0]) > 0.3 and abs(z[-1]) > 0.3, j  # both ends present
        assert np.array_equal(z, full.Z[:, j])
    for a in top:
        for b in top:
            if a < b:
                assert abs(res.Z[:, a] @ res.Z[:, b]) <= 32 * EPS


def test_support_rqi_unit():
    # oracle_rqi with support: same eigenvalue, truncated vector within eps of the full one
    d, e = mi.random_tridiag(500, 3, -1.0)
    full = oracle.mrrr(d, e, roots_only=True)
    mu = full.mu[0]
    # the root representation of T - mu I in x (LDL^T multiplied out in the unit test of the pins file)
    dd = np.empty(d.size)
    ll = np.empty(d.size - 1)
    dd[0] = d[0] - mu
    for i in range(d.size - 1):
        ll[i] = e[i] / dd[i]
        dd[i + 1] = (d[i + 1] - mu) - ll[i] * e[i]
    j = 250
    lo, hi = full.root_lo[j - 1], full.root_hi[j - 1]
    gap = min((lo + (hi - lo) / 2) - full.root_hi[j - 2], full.root_lo[j] - (lo + (hi - lo) / 2))
    a = oracle.rqi(dd, ll, j, lo, hi, gap)
    b = oracle.rqi(dd, ll, j, lo, hi, gap, support=True)
    assert a["W"] == b["W"] and a["iters"] == b["iters"]
    nz = np.flatnonzero(b["z"])
    assert nz.size < d.size and np.all(np.diff(nz) == 1)
    assert np.abs(a["z"] - b["z"]).max() <= 4 * EPS
