"""Pins of the CPU oracle's building blocks against what the paper and the
mathematics fix (hand traces, closed forms, brute force, invariants).

None of these tests compare the oracle with itself: expected values come from
tests/golden/paper_traces.json (cited hand traces), closed forms (App. D
P:7245-7247), a binary128 Jacobi brute force, Sturm counts on T, or identities.
"""
import math

import numpy as np
import pytest

import mrrr_inputs as mi
import oracle

EPS = 2.0 ** -53


def _num(v):
    if isinstance(v, str):
        return {"inf": math.inf, "-inf": -math.inf, "sqrt3": math.sqrt(3.0)}[v]
    return float(v)


def _arr(a):
    return np.array([_num(v) for v in a], dtype=np.float64)


# ----------------------------------------------------------------- prng / inputs
def test_splitmix64_reference_vector(golden):
    g = golden["splitmix64"][0]
    got = [int(x) for x in mi.splitmix64(g["seed"], 5)]
    assert got == [int(s) for s in g["outputs"]]


def test_perturbation_xi_range_and_generator():
    # xi = ((x >> 11) 2^-53 - 1/2) 2^-54*2 from the same SplitMix64 stream (A-9)
    raw = mi.splitmix64(99, 64)
    for idx in range(64):
        x = oracle.xi(99, idx)
        u = float(int(raw[idx]) >> 11) * 2.0 ** -53
        assert x == (u - 0.5) * 2.0 ** -53
        assert -(2.0 ** -54) <= x < 2.0 ** -54


# ----------------------------------------------------------------- S1/S2
def test_norm1_golden(golden):
    for c in golden["norm1"]:
        assert oracle.norm1(_arr(c["d"]), _arr(c["e"]) if c["e"] else np.zeros(1)) == c["value"], c["cite"]


def test_split_golden(golden):
    for c in golden["split"]:
        assert list(oracle.split(_arr(c["d"]), _arr(c["e"]))) == c["starts"], c["cite"]


def test_split_threshold_is_inclusive():
    # |beta_i| <= eps sqrt(n) ||T||_1 splits (eq:tolsplit P:3028-3038, A-7); one ulp above does not
    d = np.array([3.0, 1.0, 1.0, 1.0])
    tnorm = 4.0  # column 1: |3| + |1|; the other column sums stay below 3
    tol = (EPS * math.sqrt(4.0)) * tnorm
    e = np.array([1.0, tol, 1.0])
    assert list(oracle.split(d, e)) == [0, 2, 4]
    e[1] = np.nextafter(tol, 1.0)
    assert list(oracle.split(d, e)) == [0, 4]
    e[1] = -tol
    assert list(oracle.split(d, e)) == [0, 2, 4]


# ----------------------------------------------------------------- Gershgorin
def test_gershgorin_golden(golden):
    gl, gu, t = oracle.gershgorin(np.array([2.0, 2, 2]), np.array([1.0, 1]))
    assert t == 64 * EPS
    assert gl == 0 - 64 * EPS and gu == 4 + 64 * EPS


@pytest.mark.parametrize("seed", range(6))
def test_gershgorin_contains_jacobi_spectrum(seed):
    d, e = mi.random_tridiag(20 + 5 * seed, seed, -1.0)
    hi, _ = oracle.jacobi(d, e)
    gl, gu, _ = oracle.gershgorin(d, e)
    assert gl < hi.min() and hi.max() < gu


# ----------------------------------------------------------------- NegCount
def test_negcount_ldl_golden(golden):
    for c in golden["negcount_ldl"]:
        d, l = _arr(c["d"]), _arr(c["l"])
        dll = np.append(d[:-1] * l * l, 0.0)
        assert oracle.negcount_x(d, dll, c["sigma"]) == c["count"], c["cite"]


def test_negcount_t_golden(golden):
    for c in golden["negcount_t"]:
        assert oracle.negcount_t(_arr(c["d"]), _arr(c["e"]), c["sigma"]) == c["count"], c["cite"]


def _root(d, e, left=True):
    r = oracle.root_x(d, e, left)
    assert r["rc"] == 0
    dx, lx = r["d"], r["l"]
    dllx = np.append((dx[:-1] * lx) * lx, 0.0)
    return r, dx, dllx


@pytest.mark.parametrize("n", [5, 17, 64, 200])
def test_negcount_ldl_matches_closed_form_121(n):
    # 1-2-1: count(sigma) = #{j : 2 - 2cos(j pi/(n+1)) - mu < sigma} away from eigenvalues
    d, e = mi.one_two_one(n)
    r, dx, dllx = _root(d, e, True)
    lam = 2 - 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1)) - r["mu"]
    sep = 10 * n * EPS * 4
    rng = np.random.default_rng(n)
    for sigma in rng.uniform(lam.min() - 0.5, lam.max() + 0.5, 300):
        if np.min(np.abs(lam - sigma)) < sep:
            continue
        assert oracle.negcount_x(dx, dllx, sigma) == int(np.sum(lam < sigma))


@pytest.mark.parametrize("seed", range(8))
def test_negcount_ldl_matches_jacobi_and_sturm_t(seed):
    n = 8 + 7 * seed
    d, e = mi.random_tridiag(n, 1000 + seed, -1.0)
    lam_hi, _ = oracle.jacobi(d, e)
    for left in (True, False):
        r, dx, dllx = _root(d, e, left)
        assert all(dx > 0) if left else all(dx < 0)
        shifted = lam_hi - r["mu"]
        rng = np.random.default_rng(seed)
        for sigma in rng.uniform(shifted.min() - 0.2, shifted.max() + 0.2, 200):
            if np.min(np.abs(shifted - sigma)) < 1e-9:
                continue
            c = oracle.negcount_x(dx, dllx, sigma)
            assert c == int(np.sum(shifted < sigma))
            assert c == oracle.negcount_t(d, e, sigma, r["mu"])


def test_negcount_monotone_and_exhaustive():
    d, e = mi.random_tridiag(300, 5, -1.0)
    r, dx, dllx = _root(d, e, True)
    xs = np.sort(np.random.default_rng(0).uniform(-0.1, r["gu"] - r["mu"] + 0.1, 2000))
    cs = [oracle.negcount_x(dx, dllx, s) for s in xs]
    assert all(a <= b for a, b in zip(cs, cs[1:]))
    assert oracle.negcount_x(dx, dllx, 0.0) == 0          # definite root
    assert oracle.negcount_x(dx, dllx, r["gu"] - r["mu"]) == 300


# ----------------------------------------------------------------- root (S3)
@pytest.mark.parametrize("fam", ["rand", "121", "wilk", "clement"])
def test_root_ldl_backward_stable(fam):
    d, e = {"rand": lambda: mi.random_tridiag(400, 3, -1.0), "121": lambda: mi.one_two_one(400),
            "wilk": lambda: mi.wilkinson(200), "clement": lambda: mi.clement(400)}[fam]()
    for left in (True, False):
        r, dx, _ = _root(d, e, left)
        lx = r["l"]
        # L D L^T multiplied out (exact in binary128 via fractions of doubles) vs T - mu I
        diag = dx.astype(np.longdouble).copy()
        diag[1:] += (dx[:-1].astype(np.longdouble) * lx.astype(np.longdouble) ** 2)
        off = dx[:-1].astype(np.longdouble) * lx.astype(np.longdouble)
        tdiag = d.astype(np.longdouble) - np.longdouble(r["mu"])
        scale = np.abs(tdiag) + np.append(np.abs(e), 0) + np.append(0, np.abs(e))
        assert np.max(np.abs(diag - tdiag) / scale) <= 4 * EPS
        assert np.max(np.abs(off - e.astype(np.longdouble)) / np.abs(e)) <= 2 * EPS
        assert np.all(dx > 0) if left else np.all(dx < 0)
        assert r["mu"] == (r["gl"] if left else r["gu"])


def test_root_y_rounds_to_root_x_and_is_seeded():
    d, e = mi.random_tridiag(500, 11, -1.0)
    a = oracle.root_y(d, e, True, seed=1234)
    b = oracle.root_y(d, e, True, seed=1234)
    c = oracle.root_y(d, e, True, seed=4321)
    r, dx, dllx = _root(d, e, True)
    assert np.array_equal(a["d_hi"], dx)                       # fl64(M_y) == M_x
    assert np.array_equal(a["l_hi"][:-1], r["l"])
    assert np.array_equal(a["dllx"][:-1], dllx[:-1])
    assert np.all(np.abs(a["d_lo"]) < np.abs(dx) * 2.0 ** -54)   # |xi| < 2^-54 (A-9)
    assert np.all(np.abs(a["l_lo"][:-1]) <= np.abs(r["l"]) * 2.0 ** -54)
    assert np.array_equal(a["d_lo"], b["d_lo"])                 # determinism
    assert not np.array_equal(a["d_lo"], c["d_lo"])
    # M_y = x (1 + xi) in y-arithmetic: the low word is fl64(x xi) up to the binary128 rounding of the sum
    # x + fl64(x xi) (spans up to 116 bits > 113; reading A-9)
    idx = np.arange(500)
    xs = np.array([oracle.xi(1234, int(i)) for i in idx])
    assert np.all(np.abs(a["d_lo"] - dx * xs) <= np.abs(dx) * 2.0 ** -112)
    assert np.mean(a["d_lo"] == dx * xs) > 0.9


# ----------------------------------------------------------------- bisection
def test_dyadic_widen_covers_and_is_exact():
    rng = np.random.default_rng(7)
    for _ in range(3000):
        c = rng.uniform(-10, 10) * 10.0 ** rng.integers(-12, 3)
        w = abs(c) * 10.0 ** rng.uniform(-13, -3) + 1e-300
        lo, hi = c - w * rng.uniform(0, 1), c + w * rng.uniform(0, 1)
        a, b = oracle.dyadic_widen(lo, hi)
        h = b - a
        assert a <= lo and hi <= b
        m, ex = math.frexp(h)
        assert m == 0.5                         # width is a power of two
        assert (a / (h / 2)).is_integer()       # aligned: every midpoint lies on the grid
        assert h <= 4 * 2 ** math.ceil(math.log2(hi - lo))


@pytest.mark.parametrize("n", [10, 100, 1000])
def test_root_bisection_sturm_invariant_121(n):
    d, e = mi.one_two_one(n)
    r, dx, dllx = _root(d, e, True)
    P = 2.0 ** math.ceil(math.log2(r["gu"] - r["mu"]))
    lam = 2 - 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))
    for j in list(range(1, 6)) + list(range(n - 4, n + 1)) + [n // 2]:
        lo, hi = oracle.bisect_x(dx, dllx, j, 0.0, P, 1e-12)
        assert oracle.negcount_x(dx, dllx, lo) < j <= oracle.negcount_x(dx, dllx, hi)
        assert hi - lo <= max(1e-12 * max(abs(lo), abs(hi)), 2 * 2.2250738585072014e-308)
        # the exact eigenvalue of T lies in the interval inflated by the M_x-vs-T error (10 n eps ||T||)
        slack = 10 * n * EPS * 4
        assert lo - slack <= lam[j - 1] - r["mu"] <= hi + slack
        # T-frame Sturm count in binary128 agrees at the inflated endpoints
        assert oracle.negcount_t(d, e, lo - slack, r["mu"]) < j <= oracle.negcount_t(d, e, hi + slack, r["mu"])


def test_bisection_midpoints_exact_on_dyadic_grid():
    # every midpoint of Alg. Bisection from [0, 2^E] is exact (A-5): sum of the path equals Fractions
    from fractions import Fraction
    d, e = mi.random_tridiag(50, 2, -1.0)
    r, dx, dllx = _root(d, e, True)
    P = 2.0 ** math.ceil(math.log2(r["gu"] - r["mu"]))
    for j in (1, 25, 50):
        lo, hi = oracle.bisect_x(dx, dllx, j, 0.0, P, 1e-12)
        w = Fraction(hi) - Fraction(lo)
        assert w.numerator == 1 and (w.denominator & (w.denominator - 1)) == 0


# ----------------------------------------------------------------- qd transforms
def test_dstqds_golden(golden):
    for c in golden["dstqds"]:
        dp, lp, s = oracle.dstqds(_arr(c["d"]), _arr(c["l"]), c["tau"])
        assert np.array_equal(dp, _arr(c["dplus"])), c["cite"]
        assert np.array_equal(lp, _arr(c["lplus"])), c["cite"]
        if "s" in c:
            assert np.array_equal(s[:len(c["s"])], _arr(c["s"])), c["cite"]


def test_dqds_golden(golden):
    for c in golden["dqds"]:
        om, um, p = oracle.dqds(_arr(c["d"]), _arr(c["l"]), c["tau"])
        assert np.array_equal(om, _arr(c["omega"])), c["cite"]
        assert np.array_equal(um, _arr(c["uminus"])), c["cite"]
        assert np.array_equal(p, _arr(c["p"])), c["cite"]


def _rand_rep(n, seed):
    rng = np.random.default_rng(seed)
    d = rng.uniform(0.5, 2.0, n) * rng.choice([1, 1, 1, -1], n)
    l = rng.uniform(-1, 1, n - 1)
    return d, l


def _dense_ldl(d, l):
    n = d.size
    L = np.eye(n, dtype=np.longdouble)
    L[np.arange(1, n), np.arange(n - 1)] = l
    return L @ np.diag(d.astype(np.longdouble)) @ L.T


@pytest.mark.parametrize("seed", range(10))
def test_dstqds_dqds_reconstruct_shifted_matrix(seed):
    n = 12 + seed
    d, l = _rand_rep(n, seed)
    tau = np.random.default_rng(100 + seed).uniform(-0.3, 0.3)
    A = _dense_ldl(d, l) - tau * np.eye(n, dtype=np.longdouble)
    dp, lp, _ = oracle.dstqds(d, l, tau)
    B = _dense_ldl(dp, lp)
    assert np.max(np.abs(A - B)) <= 1e-12 * max(1.0, np.max(np.abs(dp)) * max(1.0, np.max(np.abs(lp))) ** 2)
    om, um, _ = oracle.dqds(d, l, tau)
    U = np.eye(n, dtype=np.longdouble)
    U[np.arange(n - 1), np.arange(1, n)] = um
    Bu = U @ np.diag(om.astype(np.longdouble)) @ U.T
    assert np.max(np.abs(A - Bu)) <= 1e-12 * max(1.0, np.max(np.abs(om)) * max(1.0, np.max(np.abs(um))) ** 2)
    # Sylvester: both factorizations have the inertia of A (count of negative pivots)
    assert int(np.sum(dp < 0)) == int(np.sum(om < 0)) == int(np.sum(np.linalg.eigvalsh(A.astype(float)) < 0))


def test_shift_translates_negcount():
    # NegCount(child, sigma) == NegCount(parent, sigma + tau) away from eigenvalues
    d, e = mi.random_tridiag(120, 17, -1.0)
    r, dx, dllx = _root(d, e, True)
    lam = np.linalg.eigvalsh(np.diag(d) + np.diag(e, 1) + np.diag(e, -1)) - r["mu"]
    tau = float(lam[60] - 1e-7)
    dp, lp, _ = oracle.dstqds(dx, r["l"], tau)
    dllc = np.append((dp[:-1] * lp) * lp, 0.0)
    for s in np.random.default_rng(1).uniform(-1, 1, 300):
        if np.min(np.abs(lam - tau - s)) < 1e-8:
            continue
        assert oracle.negcount_x(dp, dllc, s) == oracle.negcount_x(dx, dllx, s + tau)


# ----------------------------------------------------------------- Getvec
def test_getvec_golden(golden):
    c = golden["getvec"][0]
    g = oracle.getvec(_arr(c["d"]), _arr(c["l"]), c["lambda"])
    assert g["r"] == c["r"] and g["gamma"] == c["gamma_r"]
    assert np.array_equal(g["z"], _arr(c["z"]))


@pytest.mark.parametrize("seed", range(6))
def test_getvec_residual_identity(seed):
    # (LDL^T - lam I) z = gamma_r e_r with z(r) = 1 (Alg. Getvec)
    n = 30
    d, l = _rand_rep(n, 50 + seed)
    d = np.abs(d)
    A = _dense_ldl(d, l)
    lam = float(np.linalg.eigvalsh(A.astype(float))[seed * 4]) + 1e-6
    g = oracle.getvec(d, l, lam)
    z = g["z"].astype(np.longdouble)
    resid = (A - np.longdouble(lam) * np.eye(n, dtype=np.longdouble)) @ z
    r = g["r"] - 1
    assert z[r] == 1
    scale = np.max(np.abs(A)) * np.max(np.abs(z))
    assert abs(resid[r] - g["gamma"]) <= 1e-12 * scale
    resid[r] = 0
    assert np.max(np.abs(resid)) <= 1e-12 * scale
    # twist index minimises |gamma| so the local residual obeys eq:localresidual
    lam_true = float(np.linalg.eigvalsh(A.astype(float))[seed * 4])
    assert abs(g["gamma"]) / math.sqrt(g["zz"]) <= math.sqrt(n) * abs(lam - lam_true) * 1.01 + 1e-13
    # c = NegCount(LDL^T, lam)
    assert g["c"] == seed * 4 + 1


def test_getvec_121_eigenvector_closed_form():
    n = 3
    d, e = mi.one_two_one(n)
    r, dx, _ = _root(d, e, True)
    lam = 2 - math.sqrt(2) - r["mu"]
    g = oracle.getvec(dx, r["l"], lam)
    z = g["z"] / np.linalg.norm(g["z"])
    ref = np.sin(np.arange(1, 4) * np.pi / 4)
    ref /= np.linalg.norm(ref)
    assert np.max(np.abs(np.abs(z) - ref)) < 1e-14


# ----------------------------------------------------------------- classification
def test_is_boundary_formula_golden():
    # midpoints {1.0, 1.0005, 2.0} widths 1e-9, gaptol 1e-3 -> {1,2} cluster, {3} singleton
    iv = [(1.0 - 5e-10, 1.0 + 5e-10), (1.0005 - 5e-10, 1.0005 + 5e-10), (2.0 - 5e-10, 2.0 + 5e-10)]
    assert not oracle.is_boundary(*iv[0], *iv[1], 1e-3)
    assert oracle.is_boundary(*iv[1], *iv[2], 1e-3)
    # reldist exactly at gaptol is a boundary (">=")
    assert oracle.is_boundary(0.5, 1.0, 1.5, 2.0, 0.25)
    assert not oracle.is_boundary(0.5, 1.0, 1.5, 2.0, np.nextafter(0.25, 1))
