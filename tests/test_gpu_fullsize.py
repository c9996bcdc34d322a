"""Full-size GPU parity on the BASELINE configurations C3 (Wilkinson n=16385), C4 (glued Wilkinson n=25728),
C5b (random n=65536, indices 1..6553) and C5a (random n=65536, all pairs), in the launch configuration bench.py
times (VERDICT r1 "missing" 5: every config compared in full, not on windows).

The oracle's full solves take minutes to an hour of CPU time, so they are stored: tests/golden/oracle_<cfg>.npz,
written by scripts/make_oracle_golden.py, which calls only oracle/.  Each file records the SHA-256 of the input
bytes and of oracle/mrrr_oracle.c; both are checked here, so a stale file fails instead of passing.

Bit-exact, with ZERO allowed mismatches (printed if any): block starts, mu and side, every root interval (fp64
bits) and root group start, depth and group extents (cluster boundaries) at every depth.  Final-node intervals of
outputs below the root (child frames) are bit-exact except for an explicit, fixed list of outputs per config where
the dd and binary128 realisations of a child datum round to different fp64 neighbours (KNOWN_CHILD_ROUNDING).  Toleranced (north_star): |W - W_oracle| <= 8 n eps ||T||; residuals and
orthogonality on samples (binary128 re-checks).  Properties at full size: the Sturm-count invariant
NegCount(M_x, lo_j) < j <= NegCount(M_x, hi_j) for every root interval (Alg. negcountLDL on the root
representation, evaluated by the oracle's plain count), ascending W, unit columns.  Singleton vectors agree with
the oracle's (computed live on windows) within the Davis-Kahan bound 2 (rho_gpu + rho_oracle) / gap_j.
"""
import hashlib
import json
import os

import numpy as np
import pytest

import mrrr_inputs as mi
import oracle

pytestmark = pytest.mark.gpu
EPS = 2.0 ** -53
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def load_golden(name):
    z = np.load(os.path.join(ROOT, "tests", "golden", f"oracle_{name}.npz"))
    out = {k: z[k] for k in z.files if k != "meta"}
    out["meta"] = json.loads(str(z["meta"]))
    return out


def input_sha(d, e):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(d, np.float64).tobytes())
    h.update(np.ascontiguousarray(e, np.float64).tobytes())
    return h.hexdigest()


def oracle_sha():
    with open(os.path.join(ROOT, "oracle", "mrrr_oracle.c"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


# outputs whose child-frame interval differs between the dd (GPU) and binary128 (oracle) realisations of the
# y-arithmetic on these inputs (see test_fullsize_parity); measured once, fixed here, never widened silently
KNOWN_CHILD_ROUNDING = {"C3": [9807], "C4": [2209, 2210, 13044, 13098, 13115, 13165, 13169, 13172, 13178, 13232, 13238, 13268,
                                           13433]}


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def _report(name, mask, idx_label="index"):
    if np.any(mask):
        bad = np.nonzero(mask)[0]
        print(f"{name}: {bad.size} mismatches at {idx_label} {bad[:20].tolist()}")
    return int(np.sum(mask))


def _same(a, b):
    return (a == b) | (np.isnan(a) & np.isnan(b))


def _window_vectors(torch, d, e, c, W, Zd, G, tn):
    """Singleton vectors on windows vs a live oracle solve of the same window: Davis-Kahan bound."""
    rng = np.random.default_rng(7)
    width = 6 if c.n > 30000 else 8
    starts = sorted(set([1, c.k - width + 1] + list(rng.integers(1, c.k - width + 2, 3))))
    side = int(G["side"][0])
    Wg = G["W"]
    for a in starts:
        b = a + width - 1
        r = oracle.mrrr(d, e, c.il + a - 1, c.il + b - 1, root_side=side)
        cols = slice(a - 1, b)
        Zw = Zd[:, cols].cpu().numpy()
        rho_g = oracle.residuals(d, e, W[cols], Zw)
        rho_o = oracle.residuals(d, e, r.W, r.Z)
        assert rho_g.max() <= c.n * EPS * tn and rho_o.max() <= c.n * EPS * tn
        for t in range(width):
            j = a - 1 + t
            if r.depth[t] != 0:
                continue  # cluster members: any orthonormal basis of the cluster subspace (parity unpinned)
            gl = Wg[j] - Wg[j - 1] if j > 0 else np.inf
            gr = Wg[j + 1] - Wg[j] if j + 1 < c.k else np.inf
            gap = min(gl, gr)
            zg, zo = Zw[:, t], r.Z[:, t]
            sgn = 1.0 if np.dot(zg, zo) >= 0 else -1.0
            dz = np.max(np.abs(zg - sgn * zo))
            bound = 2 * (rho_g[t] + rho_o[t]) / gap + 8 * np.sqrt(c.n) * EPS
            assert dz <= bound, (j, dz, bound)


@pytest.mark.parametrize("cfg", ["C3", "C4", "C5b", "C5a"])
def test_fullsize_parity(torch_cuda, cfg):
    import paper_1401_4950_b200 as m
    c = mi.CONFIGS[cfg]
    d, e = c.matrix()
    G = load_golden(cfg)
    assert G["meta"]["input_sha256"] == input_sha(d, e), "golden file is for other input bytes"
    assert G["meta"]["oracle_sha256"] == oracle_sha(), "golden file is stale: rerun scripts/make_oracle_golden.py"
    s = m.Solver(keep_diag=True)
    dt, et = torch_cuda.from_numpy(d).cuda(), torch_cuda.from_numpy(e).cuda()
    W, Zd = s.eig(dt, et, c.il, c.iu)
    torch_cuda.cuda.synchronize()
    W = W.cpu().numpy()
    dg = s.diag()
    # ---- integers and fp64 decision path: bit-exact, zero mismatches
    assert np.array_equal(dg.block_start, G["block_start"])
    assert np.array_equal(dg.mu, G["mu"]) and np.array_equal(dg.side, G["side"])
    bad = _report("root_lo", ~_same(dg.root_lo, G["root_lo"])) + _report("root_hi", ~_same(dg.root_hi, G["root_hi"]))
    bad += _report("root_gstart", dg.root_gstart != G["root_gstart"])
    dmax = G["grp_first"].shape[0]
    bad += _report("depth", dg.depth != G["depth"], "output")
    bad += _report("grp_first", np.any(dg.grp_first[:dmax] != G["grp_first"], axis=0), "output")
    bad += _report("grp_last", np.any(dg.grp_last[:dmax] != G["grp_last"], axis=0), "output")
    assert np.all(dg.grp_first[dmax:] == -1)
    below = G["depth"] > 0
    fin = ~((dg.fin_lo == G["fin_lo"]) & (dg.fin_hi == G["fin_hi"])) & below
    _report("final-node (child) intervals", fin, "output")
    assert bad == 0
    # Child-frame intervals come from fl64 of child data computed in y-arithmetic: dd on the GPU, binary128 in
    # the oracle (A-33).  They are bit-identical except where a child datum lies within the two
    # realisations' difference of an fp64 rounding boundary; the outputs where that happens on these inputs are
    # listed here, every other child interval must match bit for bit, and the listed ones must still be
    # equivalent bisection results (same group structure, overlapping or adjacent cells of comparable width).
    # A child eigenvalue is fixed by its representation only to the representation's own y-rounding, about
    # 2^-100 spdiam absolute when the shift could not be certified (C4's uncertified children),
    # so the listed intervals must lie within max(one width, 2^-100 spdiam) of each other.
    known = set(KNOWN_CHILD_ROUNDING.get(cfg, []))
    got = set(np.nonzero(fin)[0].tolist())
    assert got <= known, f"unexpected child-interval mismatches {sorted(got - known)}"
    gl_, gu_, _ = oracle.gershgorin(d, e)
    yround = 2.0 ** -100 * (gu_ - gl_)
    for j in sorted(got):
        a, b, c_, d_ = dg.fin_lo[j], dg.fin_hi[j], G["fin_lo"][j], G["fin_hi"][j]
        wg, wo = b - a, d_ - c_
        print(f"  output {j}: gpu [{a!r}, {b!r}] oracle [{c_!r}, {d_!r}] shift {(a - c_) / wo:+.3g} widths "
              f"= {(a - c_) / yround:+.3g} x 2^-100 spdiam")
        assert max(a, c_) - min(b, d_) <= max(wg, wo, yround) and 0.25 <= wg / wo <= 4.0
    # ---- eigenvalues (north_star gate)
    tn = max(abs(G["W"][0]), abs(G["W"][-1])) if c.k == c.n else float(np.max(np.abs(G["W"])) + 2.0)
    assert np.max(np.abs(W - G["W"])) <= 8 * c.n * EPS * tn
    assert np.all(np.diff(W) >= 0)
    # ---- Sturm-count invariant of every root interval on the root representation M_x (Alg. negcountLDL)
    rx = oracle.root_x(d, e, bool(G["side"][0] == 1))
    assert rx["mu"] == G["mu"][0]
    dx = rx["d"]
    dllx = np.append((dx[:-1] * rx["l"]) * rx["l"], 0.0)
    pos = np.nonzero(~np.isnan(dg.root_lo))[0]
    cl = oracle.negcount_x_many(dx, dllx, dg.root_lo[pos])
    ch = oracle.negcount_x_many(dx, dllx, dg.root_hi[pos])
    j = pos + 1
    assert np.all(cl < j) and np.all(j <= ch)
    # ---- vectors: unit norms, sampled orthogonality and residuals (binary128 re-checks), window vectors
    nrm = (Zd * Zd).sum(0).sqrt().cpu().numpy()
    assert np.max(np.abs(nrm - 1)) <= 4 * np.sqrt(c.n) * EPS
    rng = np.random.default_rng(1)
    S = np.sort(rng.choice(c.k, min(256, c.k), replace=False))
    Gm = Zd[:, S].T @ Zd
    Gm[np.arange(S.size), S] -= 1.0
    big = torch_cuda.nonzero(Gm.abs() > 0.25 * c.n * EPS).cpu().numpy()
    if big.size:
        big = big[:2000]
        cols_needed = np.unique(np.concatenate([S[big[:, 0]], big[:, 1]]))
        Zs = Zd[:, cols_needed].cpu().numpy()
        rel = {cc: i for i, cc in enumerate(cols_needed)}
        pi = np.array([rel[x] for x in S[big[:, 0]]])
        pj = np.array([rel[x] for x in big[:, 1]])
        assert oracle.ortho_pairs(Zs, pi, pj) <= c.n * EPS
    assert float(Gm.abs().max()) <= 1.5 * c.n * EPS
    cols = np.sort(rng.choice(c.k, min(64, c.k), replace=False))
    assert oracle.residuals(d, e, W[cols], Zd[:, cols].cpu().numpy()).max() <= c.n * EPS * tn
    _window_vectors(torch_cuda, d, e, c, W, Zd, G, tn)
    # ---- statistics that the oracle fixes as integers
    st = s.stats()
    assert st["n_clusters"] == G["meta"]["stats"]["n_clusters"]
    assert st["uncertified"] == G["meta"]["stats"]["uncertified"]
    assert st["d_max"] == G["meta"]["stats"]["d_max"]
    s.close()
