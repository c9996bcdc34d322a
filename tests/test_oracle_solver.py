"""Pins of the complete oracle solve (S0-S10) against closed forms, binary128
Jacobi brute force, published clustering statistics and the north_star
accuracy bounds.  No expected value here comes from the oracle itself or from
the CUDA path.
"""
import math

import numpy as np
import pytest
import scipy.linalg as sla

import mrrr_inputs as mi
import oracle

EPS = 2.0 ** -53


def spectral_norm(d, e):
    n = d.size
    if n == 1:
        return abs(d[0])
    lo = sla.eigvalsh_tridiagonal(d, e, select="i", select_range=(0, 0))[0]
    hi = sla.eigvalsh_tridiagonal(d, e, select="i", select_range=(n - 1, n - 1))[0]
    return max(abs(lo), abs(hi))


def accuracy(d, e, r, il=1):
    """(max residual / (||T|| n_eff eps), max |Z^T Z - I| / (n_eff eps)) with n_eff = max(n, 32).

    The north_star gates use n eps; below n = 32 that is under the floor set by rounding the output
    to fp64 alone (about sqrt(n) eps ||T|| for z plus eps |lambda| for W, plus the mixed RQI stop
    k_rs gap eps_x sqrt(n)), so small cases use n_eff."""
    n = d.size
    ne = max(n, 32)
    tn = spectral_norm(d, e)
    res = oracle.residuals(d, e, r.W, r.Z).max() / (tn * ne * EPS)
    orth = oracle.ortho_full(r.Z) / (ne * EPS)
    return res, orth


FAMILIES = {
    "121": lambda n: mi.one_two_one(n),
    "rand": lambda n: mi.random_tridiag(n, 77 + n, -1.0),
    "rand_pos": lambda n: mi.random_tridiag(n, 91 + n, 0.0),
    "wilk": lambda n: mi.wilkinson((n - 1) // 2),
    "clement": lambda n: mi.clement(n),
    "hermite": lambda n: mi.hermite(n),
    "legendre": lambda n: mi.legendre(n),
    "laguerre": lambda n: mi.laguerre(n),
}


@pytest.mark.parametrize("fam", sorted(FAMILIES))
@pytest.mark.parametrize("n", [1, 2, 3, 7, 31, 64])
def test_small_vs_jacobi(fam, n):
    if fam == "wilk" and n % 2 == 0:
        n += 1
    d, e = FAMILIES[fam](n)
    r = oracle.mrrr(d, e)
    assert r.info == 0
    hi, lo = oracle.jacobi(d, e)
    tn = max(abs(hi[0]), abs(hi[-1]))
    assert np.max(np.abs(r.W - hi)) <= 8 * n * EPS * tn   # north_star eigenvalue gate
    assert np.all(np.diff(r.W) >= 0)
    if n > 1:
        res, orth = accuracy(d, e, r)
        assert res <= 1.0 and orth <= 1.0


def test_n1_and_single_pair():
    r = oracle.mrrr(np.array([-3.5]), np.zeros(0))
    assert r.info == 0 and r.W[0] == -3.5 and r.Z[0, 0] == 1.0
    d, e = mi.one_two_one(50)
    r = oracle.mrrr(d, e, 17, 17)
    lam = 4 * math.sin(17 * math.pi / 102) ** 2
    assert abs(r.W[0] - lam) <= 8 * 50 * EPS * 4


def test_invalid_arguments():
    d, e = mi.one_two_one(5)
    assert oracle.mrrr(d, e, 0, 3).info == -5
    assert oracle.mrrr(d, e, 3, 2).info == -6
    assert oracle.mrrr(d, e, 1, 6).info == -6
    d2 = d.copy()
    d2[2] = np.nan
    assert oracle.mrrr(d2, e).info == 1


@pytest.mark.parametrize("n", [100, 1000])
def test_121_closed_form(n):
    d, e = mi.one_two_one(n)
    r = oracle.mrrr(d, e)
    j = np.arange(1, n + 1, dtype=np.longdouble)
    lam = 4 * np.sin(j * np.pi / (2 * (n + 1))) ** 2      # = 2 - 2cos(j pi/(n+1)), App. D
    assert np.max(np.abs(r.W - lam)) <= 8 * n * EPS * 4
    assert np.max(np.abs(r.W - lam)) <= 8 * EPS * 4         # observed: a few ulp of ||T||
    i = np.arange(1, n + 1, dtype=np.longdouble)[:, None]
    Zx = np.sqrt(2 / np.longdouble(n + 1)) * np.sin(i * j[None, :] * np.pi / (n + 1))
    sgn = np.sign(np.sum(Zx * r.Z, axis=0))
    gaps = np.minimum(np.append(np.inf, np.diff(lam)), np.append(np.diff(lam), np.inf))
    err = np.max(np.abs(r.Z - Zx * sgn), axis=0)
    assert np.all(err <= 4 * n * EPS * 4 / gaps)          # sin(theta) <= ||r|| / gap
    res, orth = accuracy(d, e, r)
    assert res <= 1 and orth <= 1
    assert r.stats["largest_cluster"] == 0 and r.stats["d_max"] == 0   # rho = 1/n


@pytest.mark.parametrize("m", [10, 50, 400])
def test_wilkinson_pairs_force_clusters(m):
    d, e = mi.wilkinson(m)
    n = 2 * m + 1
    r = oracle.mrrr(d, e)
    assert r.info == 0
    assert r.stats["largest_cluster"] == 2        # rho = 2/n, Table tab:clusteringdouble P:6580-6581
    assert r.stats["d_max"] == 1                  # d_max 0 except Wilkinson
    assert r.stats["uncertified"] == 0            # phi = 1
    res, orth = accuracy(d, e, r)
    assert res <= 1 and orth <= 1
    # trace identities (all pairs): sum(lambda) = sum(alpha), sum(lambda^2) = ||T||_F^2
    tn = spectral_norm(d, e)
    assert abs(np.sum(r.W, dtype=np.longdouble) - np.sum(d)) <= n * 8 * n * EPS * tn
    fro = np.sum(d.astype(np.longdouble) ** 2) + 2 * np.sum(e.astype(np.longdouble) ** 2)
    assert abs(np.sum(r.W.astype(np.longdouble) ** 2) - fro) <= n * 16 * n * EPS * tn * tn


def test_glued_wilkinson_classification_matches_exact_gaps():
    # 3 copies of W+_21 glued by 1e-10 (n = 63 <= 64: binary128 Jacobi is the exact spectrum)
    d, e = mi.glued_wilkinson(3, 10, 1e-10)
    n = d.size
    r = oracle.mrrr(d, e)
    hi, lo = oracle.jacobi(d, e)
    lam = hi.astype(np.longdouble) + lo
    mu = r.mu[0]
    sh = lam - np.longdouble(mu)
    starts = r.root_gstart
    for j in range(n - 1):
        rel = (sh[j + 1] - sh[j]) / max(abs(sh[j]), abs(sh[j + 1]))
        if rel > 2e-10:
            assert starts[j + 1] == 1, (j, float(rel))
        elif rel < 0.5e-10:
            assert starts[j + 1] == 0, (j, float(rel))
    # every root interval brackets its exact eigenvalue up to the M_x-vs-T error
    slack = 10 * n * EPS * 11
    assert np.all(r.root_lo - slack <= sh) and np.all(sh <= r.root_hi + slack)
    res, orth = accuracy(d, e, r)
    assert res <= 1 and orth <= 1


def test_glued_wilkinson_band_structure_larger():
    d, e = mi.glued_wilkinson(8, 100, 1e-10)
    r = oracle.mrrr(d, e)
    res, orth = accuracy(d, e, r)
    assert res <= 1 and orth <= 1
    # each root group's size must equal the number of eigenvalues of T (binary128 Sturm count,
    # Alg. negcountT) between the midpoints of the gaps that separate it from its neighbours
    gs = np.nonzero(r.root_gstart == 1)[0].tolist() + [d.size]
    mu = r.mu[0]
    sizes = []
    for a, b in zip(gs[:-1], gs[1:]):
        lo = (r.root_hi[a - 1] + r.root_lo[a]) / 2 if a > 0 else r.root_lo[0] - 1.0
        hi = (r.root_hi[b - 1] + r.root_lo[b]) / 2 if b < d.size else r.root_hi[-1] + 1.0
        assert oracle.negcount_t(d, e, hi, mu) - oracle.negcount_t(d, e, lo, mu) == b - a
        sizes.append(b - a)
    assert max(sizes) == 16 and sizes.count(8) > 0
    assert r.stats["n_clusters"] > 0
    # the mixed solver's relaxed growth bound (eq:newkelgbound P:6052-6056, A-35) certifies every shift of the
    # glued matrix (with the fixed bound 64 eight of them were uncertified): phi = 1
    assert r.stats["uncertified"] == 0 and r.stats["shift_attempts"] == r.stats["n_clusters"]


def test_split_matrices_multiblock():
    # exact zeros and sub-threshold entries split the matrix (eq:tolsplit); results vs Jacobi
    rng = np.random.default_rng(3)
    d = rng.uniform(-1, 1, 40)
    e = rng.uniform(-1, 1, 39)
    e[[4, 5, 17, 30]] = 0.0
    e[22] = 1e-300
    r = oracle.mrrr(d, e)
    assert r.info == 0 and r.nblocks == 6
    assert list(r.block_start) == [0, 5, 6, 18, 23, 31, 40]
    hi, _ = oracle.jacobi(d, e)
    assert np.max(np.abs(r.W - hi)) <= 8 * 40 * EPS * 2
    res, orth = accuracy(d, e, r)
    assert res <= 1 and orth <= 1
    for il, iu in [(1, 1), (3, 9), (10, 40), (40, 40)]:
        rs = oracle.mrrr(d, e, il, iu)
        assert np.max(np.abs(rs.W - hi[il - 1:iu])) <= 8 * 40 * EPS * 2
        assert oracle.residuals(d, e, rs.W, rs.Z).max() <= 40 * EPS * 2


def test_diagonal_matrix():
    d = np.array([3.0, -1.0, 2.0, 2.0, 0.5])
    r = oracle.mrrr(d, np.zeros(4))
    assert np.array_equal(r.W, np.sort(d))
    assert np.array_equal(np.abs(r.Z).sum(axis=0), np.ones(5))


@pytest.mark.parametrize("side", [1, 2])
def test_subset_equals_slice_of_all_pairs(side):
    d, e = mi.random_tridiag(600, 12, -1.0)
    full = oracle.mrrr(d, e, root_side=side)
    for il, iu in [(1, 40), (200, 260), (560, 600)]:
        sub = oracle.mrrr(d, e, il, iu, root_side=side)
        assert np.array_equal(sub.W, full.W[il - 1:iu])
        assert np.array_equal(sub.Z, full.Z[:, il - 1:iu])
        assert np.array_equal(sub.root_lo[il - 1:iu], full.root_lo[il - 1:iu])


def test_thread_count_independent():
    d, e = mi.wilkinson(60)
    a = oracle.mrrr(d, e, threads=1)
    b = oracle.mrrr(d, e, threads=8)
    assert np.array_equal(a.W, b.W) and np.array_equal(a.Z, b.Z)
    assert np.array_equal(a.grp_first, b.grp_first)


def test_auto_root_side_rule():
    d, e = mi.random_tridiag(300, 4, -1.0)
    assert oracle.mrrr(d, e, 1, 10).side[0] == 1       # (il-1) <= (n-iu): left end
    assert oracle.mrrr(d, e, 291, 300).side[0] == 2    # right end
    r = oracle.mrrr(d, e, 291, 300)
    res = oracle.residuals(d, e, r.W, r.Z)
    assert res.max() <= 300 * EPS * spectral_norm(d, e)


@pytest.mark.parametrize("s", [600, -600, 1000, -1000])
def test_scaling_is_an_exact_power_of_two_image(s):
    # inputs with max |entry| outside [2^-500, 2^500] are solved on 2^-e T (A-21); a power-of-two
    # scale commutes with every fp operation away from over/underflow, so the result is the exact image
    d, e = mi.random_tridiag(60, 8, -1.0)
    r0 = oracle.mrrr(d, e)
    r = oracle.mrrr(d * 2.0 ** s, e * 2.0 ** s)
    assert r.info == 0
    assert np.array_equal(r.W, r0.W * 2.0 ** s)
    assert np.array_equal(r.Z, r0.Z)


def test_scaling_extreme_inputs_vs_jacobi():
    # entries near the overflow threshold (||T||_1 itself overflows) and deep in the subnormal range; the
    # reference is binary128 Jacobi of the stored input brought back to O(1) by the exact inverse power of two
    d, e = mi.random_tridiag(40, 9, -1.0)
    for s in (1022, -1040):
        ds, es = np.ldexp(d, s), np.ldexp(e, s)
        r = oracle.mrrr(ds, es)
        assert r.info == 0
        d1, e1 = np.ldexp(ds, -s), np.ldexp(es, -s)     # exact (the input as stored, unscaled)
        hi, _ = oracle.jacobi(d1, e1)
        tn = max(abs(hi[0]), abs(hi[-1]))
        # W is returned on the fp64 grid of the scaled-back values: subnormal outputs carry their own rounding
        grid = 2.0 ** (-1074 - s) if s < 0 else 0.0
        assert np.max(np.abs(np.ldexp(r.W, -s) - hi)) <= 8 * 40 * EPS * tn + grid
        assert oracle.residuals(d1, e1, hi, r.Z).max() <= 40 * EPS * tn


def test_zero_matrix():
    r = oracle.mrrr(np.zeros(5), np.zeros(4))
    assert r.info == 0 and np.array_equal(r.W, np.zeros(5)) and r.nblocks == 5


@pytest.mark.parametrize("fam", sorted(mi.FAMILIES))
def test_families_published_structure(fam):
    # §8(f1) on the oracle: the mixed-precision solver's clustering rho = 1/n (2/n for Wilkinson), d_max = 0
    # (1 for Wilkinson) and phi = 1 (Table tab:clusteringdouble P:6560-6590; Hermite:
    # Table tab:clustering criterion III P:5941-5959), plus the north_star accuracy gates
    d, e = mi.FAMILIES[fam](400)
    n = d.size
    r = oracle.mrrr(d, e)
    assert r.info == 0
    res, orth = accuracy(d, e, r)
    assert res <= 1 and orth <= 1
    if fam in ("legendre", "laguerre"):
        return  # no published mixed-precision statistics
    assert r.stats["uncertified"] == 0
    if fam == "geometric":
        # DESIGN.md A-8: the root shift is the inflated Gershgorin end, not the bisected extremal eigenvalue
        # (P:3120-3122), so the tiny eigenvalues of Geometric (eps .. 1e-13) sit ~|mu| away and cluster in the
        # root frame (one cluster of ~30% of n, resolved by ONE child shift: d_max = 1, phi = 1) where the paper
        # reports rho = 1/n
        assert r.stats["d_max"] == 1 and r.stats["n_clusters"] == 1
        return
    assert max(r.stats["largest_cluster"], 1) == (2 if fam == "wilkinson" else 1)
    assert r.stats["d_max"] == (1 if fam == "wilkinson" else 0)


@pytest.mark.parametrize("fam", ["uniform", "geometric"])
def test_prescribed_spectrum_families(fam):
    # App. D: the generated T carries the prescribed eigenvalues up to the fp64 similarity and
    # reduction (about n eps ||A||); the oracle's eigenvalues agree with them to that level
    n = 300
    d, e = mi.FAMILIES[fam](n)
    k = np.arange(1, n + 1, dtype=np.float64)
    lam = EPS + (k - 1) * (1 - EPS) / (n - 1) if fam == "uniform" else np.sort(EPS ** ((n - k) / (n - 1)))
    r = oracle.mrrr(d, e)
    assert np.max(np.abs(r.W - lam)) <= 10 * n * EPS
    assert np.all(np.diff(r.W) >= -8 * n * EPS)   # eigenvalues a few ulps apart may round out of order
