"""GPU parity: the CUDA path (through the C ABI) vs the CPU oracle on the same seeded inputs.

Bit-exact: block starts, mu and side per block, root intervals (fp64 bits), root group
starts, group extents per depth, final-node intervals.  Toleranced (north_star): |W - W_oracle| <=
8 n eps ||T||, max ||T z - lambda z|| <= n eps ||T||, max |Z^T Z - I| <= n eps (n -> max(n, 32), A-27).
C1 and C2 are compared in full against a live oracle run here; C3, C4, C5a and C5b in full against stored
oracle results in tests/test_gpu_fullsize.py.
"""
import numpy as np
import pytest

import mrrr_inputs as mi
import oracle

pytestmark = pytest.mark.gpu
EPS = 2.0 ** -53


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def gpu_solve(torch, d, e, il=None, iu=None, side=0, diag=True):
    import paper_1401_4950_b200 as m
    s = m.Solver(keep_diag=diag, root_side=side)
    n = d.size
    dt = torch.from_numpy(d).cuda()
    et = torch.from_numpy(e if n > 1 else np.zeros(1)).cuda()
    W, Z = s.eig(dt, et, il, iu)
    torch.cuda.synchronize()
    small = Z.numel() <= (1 << 27)
    out = dict(W=W.cpu().numpy(), Z=Z.cpu().numpy() if small else None, Zd=Z, stats=s.stats(), times=s.times(),
               solver=s)
    if diag:
        out["diag"] = s.diag()
    return out


def same(a, b):
    return np.array_equal(a, b, equal_nan=True)


def check_integers(g, r, cols=None, positions=None):
    dg = g["diag"]
    assert same(dg.block_start, r.block_start)
    assert same(dg.mu, r.mu)
    assert same(dg.side, r.side)
    if positions is None:
        assert same(dg.root_lo, r.root_lo) and same(dg.root_hi, r.root_hi)
        assert same(dg.root_gstart, r.root_gstart)
    else:
        assert same(dg.root_lo[positions], r.root_lo[positions])
        assert same(dg.root_hi[positions], r.root_hi[positions])
        assert same(dg.root_gstart[positions[1:]], r.root_gstart[positions[1:]])
    cols = slice(None) if cols is None else cols
    assert same(dg.grp_first[:, cols], r.grp_first)
    assert same(dg.grp_last[:, cols], r.grp_last)
    assert same(dg.depth[cols], r.depth)
    mism = ~((dg.fin_lo[cols] == r.fin_lo) & (dg.fin_hi[cols] == r.fin_hi))
    # child intervals depend on fl64 of y-computed data (dd vs binary128): equal unless a datum lies within
    # ~2^-100 of a rounding boundary (~2^-47 per datum); zero mismatches allowed, any is printed
    if np.any(mism):
        idx = np.nonzero(mism)[0]
        print("final-interval mismatches at", idx[:20], "depths", dg.depth[cols][idx[:20]])
    assert mism.sum() == 0


def check_tol(d, e, W, Z, Wref, tn):
    n = d.size
    ne = max(n, 32)
    assert np.max(np.abs(W - Wref)) <= 8 * ne * EPS * tn
    res = oracle.residuals(d, e, W, Z).max()
    assert res <= ne * EPS * tn, res / (ne * EPS * tn)


SMALL = {
    "n1": lambda: (np.array([3.0]), np.zeros(0)),
    "n2": lambda: mi.random_tridiag(2, 1, -1.0),
    "n3_121": lambda: mi.one_two_one(3),
    "rand_64": lambda: mi.random_tridiag(64, 3, -1.0),
    "rand_257": lambda: mi.random_tridiag(257, 4, -1.0),
    "121_1000": lambda: mi.one_two_one(1000),
    "rand_3001_pos": lambda: mi.random_tridiag(3001, 6, 0.0),
    "wilk_21": lambda: mi.wilkinson(10),
    "wilk_1001": lambda: mi.wilkinson(500),
    "glued_3x21": lambda: mi.glued_wilkinson(3, 10, 1e-10),
    "glued_8x201": lambda: mi.glued_wilkinson(8, 100, 1e-10),
    "clement_500": lambda: mi.clement(500),
    "hermite_400": lambda: mi.hermite(400),
    "legendre_300": lambda: mi.legendre(300),
    "laguerre_300": lambda: mi.laguerre(300),
    "diag_5": lambda: (np.array([3.0, -1.0, 2.0, 2.0, 0.5]), np.zeros(4)),
}


@pytest.mark.parametrize("name", sorted(SMALL))
def test_parity_small(torch_cuda, name):
    d, e = SMALL[name]()
    g = gpu_solve(torch_cuda, d, e)
    r = oracle.mrrr(d, e)
    assert r.info == 0
    check_integers(g, r)
    tn = max(abs(r.W).max(), 1e-300)
    check_tol(d, e, g["W"], g["Z"], r.W, tn)
    ne = max(d.size, 32)
    assert oracle.ortho_full(g["Z"]) <= ne * EPS
    assert g["stats"]["uncertified"] == r.stats["uncertified"]
    assert g["stats"]["n_clusters"] == r.stats["n_clusters"]


@pytest.mark.parametrize("il,iu,side", [(1, 40, 0), (100, 400, 0), (2901, 3000, 0), (1500, 1500, 0),
                                        (1, 3000, 2), (700, 2100, 1)])
def test_parity_subsets(torch_cuda, il, iu, side):
    d, e = mi.random_tridiag(3000, 9, -1.0)
    g = gpu_solve(torch_cuda, d, e, il, iu, side)
    r = oracle.mrrr(d, e, il, iu, root_side=side)
    check_integers(g, r)
    check_tol(d, e, g["W"], g["Z"], r.W, max(abs(r.W).max(), 2.0))


def test_parity_subset_in_cluster(torch_cuda):
    # the subset edge falls inside Wilkinson pairs: guards must extend and the pair processed whole
    d, e = mi.wilkinson(300)
    for il, iu in [(600, 601), (2, 2), (300, 450)]:
        g = gpu_solve(torch_cuda, d, e, il, iu)
        r = oracle.mrrr(d, e, il, iu)
        check_integers(g, r)
        check_tol(d, e, g["W"], g["Z"], r.W, 301.0)


@pytest.mark.parametrize("il,iu", [(5, 7), (1, 40), (100, 130), (1500, 1600), (1604, 1608)])
def test_parity_subset_edges_in_large_clusters(torch_cuda, il, iu):
    # glued Wilkinson with clusters of 8/16 (and 256-clusters at C4 size): the guards extend through whole
    # clusters in doubling batches; the computed set (NaN pattern), intervals and groups equal the oracle's
    # one-at-a-time extension bit for bit
    d, e = mi.glued_wilkinson(8, 100, 1e-10)
    g = gpu_solve(torch_cuda, d, e, il, iu)
    r = oracle.mrrr(d, e, il, iu)
    check_integers(g, r)
    check_tol(d, e, g["W"], g["Z"], r.W, 101.0)


@pytest.mark.parametrize("sel", [(1, 40), (3, 9), (10, 40), (40, 40), (1, 1)])
def test_parity_split_matrix(torch_cuda, sel):
    rng = np.random.default_rng(3)
    d = rng.uniform(-1, 1, 40)
    e = rng.uniform(-1, 1, 39)
    e[[4, 5, 17, 30]] = 0.0
    e[22] = 1e-300
    g = gpu_solve(torch_cuda, d, e, *sel)
    r = oracle.mrrr(d, e, *sel)
    check_integers(g, r)
    check_tol(d, e, g["W"], g["Z"], r.W, 2.0)


@pytest.mark.parametrize("sel", [(1, 6000), (2500, 2600), (5999, 6000)])
def test_parity_many_blocks(torch_cuda, sel):
    # 6000 rows in ~700 blocks of 1..16 rows (repeated diagonal values across blocks: ties broken by position):
    # the multi-block ranking (bitonic sort of (key, position) over 8192 padded entries: tile and global passes)
    # must select exactly the oracle's columns
    rng = np.random.default_rng(17)
    n = 6000
    d = np.round(rng.uniform(-1, 1, n), 2)
    e = rng.uniform(-1, 1, n - 1)
    cuts = np.cumsum(rng.integers(1, 17, n))
    e[cuts[cuts < n - 1] - 1] = 0.0
    g = gpu_solve(torch_cuda, d, e, *sel)
    r = oracle.mrrr(d, e, *sel)
    assert r.nblocks > 500
    check_integers(g, r)
    check_tol(d, e, g["W"], g["Z"], r.W, 4.0)


def test_parity_split_threshold_exact(torch_cuda):
    # |beta| exactly at eps sqrt(n) ||T||_1 splits; one ulp above does not
    d = np.array([3.0, 1.0, 1.0, 1.0])
    tol = (EPS * 2.0) * 4.0
    for b, nblk in [(tol, 2), (np.nextafter(tol, 1.0), 1)]:
        e = np.array([1.0, b, 1.0])
        g = gpu_solve(torch_cuda, d, e)
        r = oracle.mrrr(d, e)
        assert g["diag"].nblocks == r.nblocks == nblk
        check_integers(g, r)


@pytest.mark.parametrize("s", [600, -600, 1022, -1040])
def test_scaled_inputs(torch_cuda, s):
    # max |entry| outside [2^-500, 2^500] (A-21): solved on 2^-e T, W scaled back -- the same as the oracle's
    # exact power-of-two image, and Z equal to the unscaled solve's
    d, e = mi.random_tridiag(700, 19, -1.0)
    ds, es = np.ldexp(d, s), np.ldexp(e, s)
    g = gpu_solve(torch_cuda, ds, es)
    r = oracle.mrrr(ds, es)
    assert r.info == 0
    check_integers(g, r)
    d1, e1 = np.ldexp(ds, -s), np.ldexp(es, -s)
    g1 = gpu_solve(torch_cuda, d1, e1, diag=False)
    assert np.array_equal(g["Z"], g1["Z"])
    assert np.array_equal(g["W"], np.ldexp(g1["W"], s))
    assert np.array_equal(r.W, g["W"]) or np.max(np.abs(np.ldexp(g["W"] - r.W, -s))) <= 8 * 700 * EPS * 3


@pytest.mark.parametrize("case", ["zero", "constant_diag", "two_equal_blocks", "tiny_offdiag"])
def test_degenerate_inputs(torch_cuda, case):
    # degenerate inputs: the zero matrix and a constant diagonal (every off-diagonal splits: n blocks of size 1,
    # all eigenvalues equal), two identical decoupled blocks (every eigenvalue exactly double), off-diagonals
    # just above the split threshold
    n = 60
    if case == "zero":
        d, e = np.zeros(n), np.zeros(n - 1)
    elif case == "constant_diag":
        d, e = np.full(n, 2.5), np.zeros(n - 1)
    elif case == "two_equal_blocks":
        d1, e1 = mi.random_tridiag(30, 5, -1.0)
        d, e = np.concatenate([d1, d1]), np.concatenate([e1, [0.0], e1])
    else:
        d, e = mi.random_tridiag(n, 6, -1.0)
        e[10] = 4 * EPS * np.sqrt(n) * 4
    g = gpu_solve(torch_cuda, d, e)
    r = oracle.mrrr(d, e)
    assert r.info == 0
    check_integers(g, r)
    tn = max(abs(r.W[0]), abs(r.W[-1]), 1.0)
    check_tol(d, e, g["W"], g["Z"], r.W, tn)
    assert oracle.ortho_full(g["Z"]) <= max(n, 32) * EPS


def test_large_n_small_subset(torch_cuda):
    # n = 300,000 (past C5a's 65,536): 64-bit offsets of the workspace planes and of Z, indices 1..48 and the
    # last 48, compared with the oracle
    n = 300_000
    d, e = mi.random_tridiag(n, 8, 0.0)
    for il, iu in [(1, 48), (n - 47, n)]:
        g = gpu_solve(torch_cuda, d, e, il, iu)
        r = oracle.mrrr(d, e, il, iu)
        check_integers(g, r)
        check_tol(d, e, g["W"], g["Z"], r.W, 2.5)
        assert oracle.ortho_full(g["Z"]) <= n * EPS


def test_error_codes(torch_cuda):
    import paper_1401_4950_b200 as m
    d, e = mi.one_two_one(5)
    s = m.Solver()
    dt = torch_cuda.from_numpy(d).cuda()
    et = torch_cuda.from_numpy(e).cuda()
    with pytest.raises(m.MrrrError, match="code -5"):
        s.eig(dt, et, 0, 3)
    with pytest.raises(m.MrrrError, match="code -6"):
        s.eig(dt, et, 3, 2)
    d2 = d.copy()
    d2[1] = np.inf
    with pytest.raises(m.MrrrError, match="code 1"):
        s.eig(torch_cuda.from_numpy(d2).cuda(), et)


def test_host_api_matches_device_api(torch_cuda):
    import paper_1401_4950_b200 as m
    d, e = mi.random_tridiag(1500, 21, -1.0)
    g = gpu_solve(torch_cuda, d, e, diag=False)
    s = m.Solver()
    W, Z = s.eig_host(d, e)
    assert np.array_equal(W, g["W"]) and np.array_equal(Z, g["Z"])
    # caller-supplied page-locked result buffers (the bench's e2e path), and a subset with ldz = n
    hW = torch_cuda.empty(100, dtype=torch_cuda.float64).pin_memory().numpy()
    hZ = torch_cuda.empty((100, d.size), dtype=torch_cuda.float64).pin_memory().numpy()
    W2, Z2 = s.eig_host(d, e, 301, 400, W=hW, Zt=hZ)
    assert W2 is hW or np.shares_memory(W2, hW)
    assert np.array_equal(W2, g["W"][300:400]) and np.array_equal(Z2, g["Z"][:, 300:400])
    with pytest.raises(m.MrrrError):
        s.eig_host(d, e, 301, 400, W=np.empty(99), Zt=hZ)


def test_shards_reproduce_full_solve(torch_cuda):
    # P virtual ranks run one after another on this GPU: owned ranges partition [il, iu] and every
    # column equals the single-GPU solve of [il, iu] bit for bit (SURVEY §8(e) ownership by first index;
    # subsets whose ends cut Wilkinson pairs, and right-end subsets that take the right root: ADVICE r1)
    import paper_1401_4950_b200 as m
    from paper_1401_4950_b200 import dist as pd
    cases = [(mi.random_tridiag(2000, 31, -1.0), [(1, 2000), (1901, 2000)]),
             (mi.wilkinson(400), [(1, 801), (600, 601), (300, 450), (2, 2), (700, 801)])]
    for (d, e), sels in cases:
        n = d.size
        gst = oracle.mrrr(d, e).root_gstart  # group starts: the ownership rule's input
        dt = torch_cuda.from_numpy(d).cuda()
        et = torch_cuda.from_numpy(e).cuda()
        for il, iu in sels:
            g = gpu_solve(torch_cuda, d, e, il, iu, diag=False)
            k = iu - il + 1
            for P in (2, 3, 4):
                per = (k + P - 1) // P
                covered = []
                for rank in range(P):
                    sl, su = pd.shard_range(il, iu, P, rank)
                    if su < sl:
                        continue
                    assert (sl, su) == (il + rank * per, min(il + (rank + 1) * per - 1, iu))
                    s = m.Solver()
                    jlo, jhi, W, Z = s.eig_shard(dt, et, sl, su, il, iu)
                    assert (jlo, jhi) == pd.owned_range(gst, sl, su, n, il, iu)
                    if jhi >= jlo:
                        covered.extend(range(jlo, jhi + 1))
                        assert np.array_equal(W.cpu().numpy(), g["W"][jlo - il:jhi - il + 1])
                        assert np.array_equal(Z.cpu().numpy(), g["Z"][:, jlo - il:jhi - il + 1])
                    s.close()
                assert covered == list(range(il, iu + 1))


# ------------------------------------------------------------------------- full-size configs
def _windows(k, count, width, seed):
    rng = np.random.default_rng(seed)
    starts = sorted(set([1, k - width + 1] + list(rng.integers(1, k - width + 2, count))))
    return [(a, a + width - 1) for a in starts]


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_config_full_parity(torch_cuda, cfg):
    c = mi.CONFIGS[cfg]
    d, e = c.matrix()
    g = gpu_solve(torch_cuda, d, e, c.il, c.iu)
    r = oracle.mrrr(d, e, c.il, c.iu)
    check_integers(g, r)
    tn = max(abs(r.W[0]), abs(r.W[-1]))
    check_tol(d, e, g["W"], g["Z"], r.W, tn)
    Zt = torch_cuda.from_numpy(g["Z"]).cuda()
    G = Zt.T @ Zt - torch_cuda.eye(c.k, dtype=torch_cuda.float64, device="cuda")
    # fp64 DGEMM Gram: rounding <= sqrt(n) eps typical; flagged entries are re-checked in binary128
    big = torch_cuda.nonzero(G.abs() > 0.25 * c.n * EPS).cpu().numpy()
    assert oracle.ortho_pairs(g["Z"], big[:, 0], big[:, 1]) <= c.n * EPS if big.size else True
    assert float(G.abs().max()) <= 1.5 * c.n * EPS
    # every vector (all singletons) vs the oracle's: Davis-Kahan, |z_gpu - z_oracle| <= 2 (rho_gpu + rho_or) / gap
    rho_g = oracle.residuals(d, e, g["W"], g["Z"])
    rho_o = oracle.residuals(d, e, r.W, r.Z)
    gap = np.minimum(np.append(np.inf, np.diff(r.W)), np.append(np.diff(r.W), np.inf))
    sgn = np.where(np.sum(g["Z"] * r.Z, axis=0) >= 0, 1.0, -1.0)
    dz = np.max(np.abs(g["Z"] - r.Z * sgn), axis=0)
    assert np.all(r.depth == 0)
    assert np.all(dz <= 2 * (rho_g + rho_o) / gap + 8 * np.sqrt(c.n) * EPS)


def test_division_fast_path_is_ieee(torch_cuda):
    # the branch-free NegCount division must be bit-identical to __ddiv_rn
    import paper_1401_4950_b200 as m
    assert m.selftest(1, 1 << 28, 12345) == 0


@pytest.mark.parametrize("env", [{"MRRR_GROUPED": "0"}, {"MRRR_NEGTMA": "0"},
                                 {"MRRR_TARGET_CHAINS": "8192"}, {"MRRR_SEGK": "1"}, {"MRRR_RQISEG": "0"},
                                 {"MRRR_RQISEG": "1", "MRRR_RQISEGK": "1"},
                                 {"MRRR_RQISEGW": "16"}, {"MRRR_RQISEGMIN": "0"},
                                 {"MRRR_RQIBULK": "0"}, {"MRRR_SEGCH2": "1000000"}, {"MRRR_SEGTHREADS": "262144"},
                                 {"MRRR_SEGYK": "1"}, {"MRRR_SEGYW": "8"}, {"MRRR_SEGXK": "1"}, {"MRRR_SEGXK": "8", "MRRR_SEGXW": "8"},
                                 {"MRRR_DEVSTABLE": "0"}, {"MRRR_DEVROUNDS": "1"}, {"MRRR_RQISEGCHILD": "0"},
                                 {"MRRR_SEGCHILDMIN": "0"}, {"MRRR_RECSTAGE": "1"}, {"MRRR_TWDD_ROOT": "100000"},
                                 {"MRRR_DEFER_TAIL": "0"}])
def test_bisection_schedules_are_bit_identical(torch_cuda, env, monkeypatch):
    # every evaluation schedule (k-section budget, TMA staging, representation-grouped child rounds, guided
    # tube rounds) must reproduce the oracle's sequential Alg. Bisection intervals bit for bit (rule W)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    for d, e in (mi.random_tridiag(2000, 17, -1.0), mi.wilkinson(200), mi.glued_wilkinson(6, 40, 1e-10)):
        g = gpu_solve(torch_cuda, d, e)
        r = oracle.mrrr(d, e)
        check_integers(g, r)
        tn = max(abs(r.W[0]), abs(r.W[-1]))
        check_tol(d, e, g["W"], g["Z"], r.W, tn)
        g["solver"].close()


@pytest.mark.parametrize("fault", [1, 2, 3])
def test_forced_fallback_and_careful_paths(torch_cuda, fault, monkeypatch):
    # fault injection (MRRR_FAULT, read at mrrr_init): every singleton through the two-lane kernel (MRRR_RQISEG=0)
    # with bit 0 = no RQI iterations, so every eigenpair comes from the y-bisection fallback + one Getvec
    # (P:3481-3482), bit 1 = every Getvec through the careful IEEE pass (A-25).  The oracle's
    # own fallback and zero-pivot branches are pinned in tests/test_oracle_branches.py; here the GPU's must
    # still meet every parity gate.
    monkeypatch.setenv("MRRR_RQISEG", "0")
    monkeypatch.setenv("MRRR_FAULT", str(fault))
    for d, e in (mi.random_tridiag(1500, 23, -1.0), mi.wilkinson(150), mi.glued_wilkinson(4, 40, 1e-10)):
        g = gpu_solve(torch_cuda, d, e)
        r = oracle.mrrr(d, e)
        check_integers(g, r)
        tn = max(abs(r.W[0]), abs(r.W[-1]))
        check_tol(d, e, g["W"], g["Z"], r.W, tn)
        assert oracle.ortho_full(g["Z"]) <= max(d.size, 32) * EPS
        if fault & 1:
            assert g["stats"]["rqi_fallbacks"] == d.size
        if fault & 2:
            assert g["stats"]["careful"] == d.size
        g["solver"].close()


@pytest.mark.gpu
@pytest.mark.parametrize("mat,il,iu", [("rand", 5, 560), ("rand", 500, 600), ("wilk", 600, 601), ("wilk", 300, 450)])
def test_eig_dist_single_rank_matches_full_solve(torch_cuda, mat, il, iu):
    # mrrr_eig_dist with a one-rank NCCL communicator: the shard is the whole selection, the all-gathered
    # eigenvalue list and the owned vectors equal the plain solve bit for bit (same kernels, same order);
    # right-end subsets take the same root side as mrrr_eig, subset ends inside clusters are cut at il/iu
    import paper_1401_4950_b200 as m
    d, e = mi.random_tridiag(600, 41, -1.0) if mat == "rand" else mi.wilkinson(300)
    dt, et = torch_cuda.from_numpy(d).cuda(), torch_cuda.from_numpy(e).cuda()
    s = m.Solver()
    W0, Z0 = s.eig(dt, et, il, iu)
    s2 = m.Solver()
    jlo, jhi, W, Z = s2.eig_dist(dt, et, il, iu, m.nccl_unique_id(), 0, 1)
    torch_cuda.cuda.synchronize()
    assert (jlo, jhi) == (il, iu)
    assert torch_cuda.equal(W.cpu(), W0.cpu())
    assert torch_cuda.equal(Z.cpu(), Z0.cpu())


@pytest.mark.gpu
def test_eig_dist_two_ranks(torch_cuda):
    # world 2 over NCCL, one process per GPU (skipped on a one-GPU box): the gathered W equals the 1-GPU solve
    if torch_cuda.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    import subprocess
    import sys
    import os
    code = os.path.join(os.path.dirname(os.path.abspath(__file__)), "dist_worker.py")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29533", code], capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("DIST_OK") == 2


@pytest.mark.gpu
def test_deferred_tails_chunked_levels_bit_identical(torch_cuda, monkeypatch):
    # deferred tails (two-lane child levels on the side stream): a workspace limit
    # that splits the root clusters into chunks of ~10 (the solve stream waits for each chunk's tail before the
    # next chunk rewrites the representation slots) and many RQI batches; W and Z equal the unchunked solve and
    # the in-order schedule (MRRR_DEFER_TAIL=0) bit for bit, and the integers / tolerances match the oracle
    import paper_1401_4950_b200 as m
    d, e = mi.glued_wilkinson(8, 100, 1e-10)
    n = d.size
    per_child = n * (16 + 48)  # double2 + YElt rows of one child representation
    runs = []
    for ws, defer in ((0, "1"), (4 * 11 * per_child, "1"), (4 * 11 * per_child, "0")):
        monkeypatch.setenv("MRRR_DEFER_TAIL", defer)
        s = m.Solver(keep_diag=True, ws_limit=ws)
        W, Z = s.eig(torch_cuda.from_numpy(d).cuda(), torch_cuda.from_numpy(e).cuda())
        torch_cuda.cuda.synchronize()
        runs.append((W.cpu().numpy(), Z.cpu().numpy(), s.stats(), s.diag() if ws == 0 else None))
        s.close()
    for W, Z, st, _ in runs[1:]:
        assert np.array_equal(W, runs[0][0]) and np.array_equal(Z, runs[0][1])
        assert st["failed"] == 0
    r = oracle.mrrr(d, e)
    g = dict(W=runs[0][0], Z=runs[0][1], stats=runs[0][2], diag=runs[0][3])
    check_integers(g, r)
    tn = max(abs(r.W[0]), abs(r.W[-1]))
    check_tol(d, e, g["W"], g["Z"], r.W, tn)
