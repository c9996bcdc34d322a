"""ctypes front end of the CPU oracle (oracle/mrrr_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
``bench.py`` (cpu_baseline leg and ``--impl reference``).  The product package
``paper_1401_4950_b200`` never imports this module, and this module never
imports the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "mrrr_oracle.c")
LIB = os.path.join(HERE, "liboracle.so")
LIB_SD = os.path.join(HERE, "liboracle_sd.so")  # the same source with -DORACLE_SD: single/double realisation

CFLAGS = ["-O2", "-std=gnu11", "-fopenmp", "-fPIC", "-shared", "-ffp-contract=off",
          "-fno-fast-math", "-fexcess-precision=standard"]

STAT_NAMES = ["d_max", "n_clusters", "largest_cluster", "uncertified", "shift_attempts", "rqi_iters",
              "rqi_fallbacks", "bracket_fixes", "root_backoffs", "failed", "negcount_x", "negcount_y",
              "getvec_calls", "zero_pivots", "early_stops", "support_rows"]


def build(force: bool = False) -> str:
    for out, extra in ((LIB, []), (LIB_SD, ["-DORACLE_SD"])):
        if force or not os.path.exists(out) or os.path.getmtime(out) < os.path.getmtime(SRC):
            subprocess.check_call(["gcc", *CFLAGS, *extra, "-o", out, SRC, "-lquadmath", "-lm"])
    return LIB


class _Opts(C.Structure):
    _fields_ = [("gaptol", C.c_double), ("seed", C.c_uint64), ("root_side", C.c_int32), ("threads", C.c_int32),
                ("roots_only", C.c_int32), ("early_stop", C.c_int32), ("support", C.c_int32)]


class _Diag(C.Structure):
    _fields_ = [(nm, C.c_void_p) for nm in
                ("nblocks", "block_start", "mu", "side", "root_lo", "root_hi", "root_gstart", "depth",
                 "grp_first", "grp_last", "fin_lo", "fin_hi", "stats")]


_libs = {}
_dp = C.POINTER(C.c_double)
_i64 = C.c_int64


def lib(sd: bool = False):
    """The double/quadruple oracle, or (sd=True) the single/double realisation built from the same source."""
    if sd not in _libs:
        build()
        L = C.CDLL(LIB_SD if sd else LIB)
        L.oracle_mrrr.restype = C.c_int
        L.oracle_mrrr.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, _i64, C.POINTER(_Opts), C.c_void_p,
                                  C.c_void_p, _i64, C.POINTER(_Diag)]
        L.oracle_xi.restype = C.c_double
        L.oracle_xi.argtypes = [C.c_uint64, C.c_uint64]
        L.oracle_norm1.restype = C.c_double
        L.oracle_norm1.argtypes = [_i64, C.c_void_p, C.c_void_p]
        L.oracle_split.restype = _i64
        L.oracle_split.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_gershgorin.restype = None
        L.oracle_gershgorin.argtypes = [_i64, C.c_void_p, C.c_void_p, _dp, _dp, _dp]
        L.oracle_negcount_x.restype = _i64
        L.oracle_negcount_x.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_double]
        L.oracle_negcount_t_q.restype = _i64
        L.oracle_negcount_t_q.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_double, C.c_double]
        L.oracle_bisect_x.restype = None
        L.oracle_bisect_x.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, C.c_double, _dp, _dp]
        L.oracle_dyadic_widen.restype = None
        L.oracle_dyadic_widen.argtypes = [C.c_double, C.c_double, _dp, _dp]
        L.oracle_is_boundary.restype = C.c_int
        L.oracle_is_boundary.argtypes = [C.c_double] * 5
        L.oracle_root_x.restype = C.c_int
        L.oracle_root_x.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_int, _dp, C.c_void_p, C.c_void_p, _dp,
                                    _dp, C.POINTER(C.c_int)]
        L.oracle_root_y.restype = C.c_int
        L.oracle_root_y.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, _i64, C.c_int, C.c_uint64, _dp] + \
            [C.c_void_p] * 6
        L.oracle_dstqds.restype = None
        L.oracle_dstqds.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_double] + [C.c_void_p] * 4
        L.oracle_dqds.restype = None
        L.oracle_dqds.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_double] + [C.c_void_p] * 3
        L.oracle_getvec.restype = None
        L.oracle_getvec.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_double, C.c_double, C.POINTER(_i64),
                                    C.c_void_p, _dp, _dp, C.POINTER(_i64)]
        L.oracle_residuals.restype = None
        L.oracle_residuals.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, C.c_void_p, C.c_void_p, _i64,
                                       C.c_void_p]
        L.oracle_ortho_full.restype = C.c_double
        L.oracle_ortho_full.argtypes = [_i64, _i64, C.c_void_p, _i64]
        L.oracle_ortho_pairs.restype = C.c_double
        L.oracle_ortho_pairs.argtypes = [_i64, C.c_void_p, _i64, _i64, C.c_void_p, C.c_void_p]
        L.oracle_jacobi.restype = None
        L.oracle_jacobi.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_maxd.restype = C.c_int
        L.oracle_negcount_x_many.restype = None
        L.oracle_negcount_x_many.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, C.c_void_p, C.c_void_p]
        L.oracle_jacobi_ldl.restype = None
        L.oracle_jacobi_ldl.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_stats_read.restype = None
        L.oracle_stats_read.argtypes = [C.c_void_p]
        L.oracle_stats_reset.restype = None
        L.oracle_stats_reset.argtypes = []
        L.oracle_bracket_x.restype = _i64
        L.oracle_bracket_x.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, _dp, _dp]
        L.oracle_bracket_y.restype = _i64
        L.oracle_bracket_y.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, _dp, _dp]
        L.oracle_bisect_y_full.restype = None
        L.oracle_bisect_y_full.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, C.c_double, C.c_double, _dp, _dp]
        L.oracle_rqi.restype = None
        L.oracle_rqi.argtypes = [_i64, C.c_void_p, C.c_void_p, _i64, C.c_double, C.c_double, C.c_double, C.c_int32, _dp,
                                 C.c_void_p, C.POINTER(_i64), C.POINTER(_i64)]
        L.oracle_es_rtol.restype = C.c_double
        L.oracle_es_rtol.argtypes = [_i64, C.c_double]
        L.oracle_es_stop.restype = C.c_int
        L.oracle_es_stop.argtypes = [C.c_double] * 7
        L.oracle_root_x_from.restype = C.c_int
        L.oracle_root_x_from.argtypes = [_i64, C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_double, _dp,
                                         C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
        _libs[sd] = L
    return _libs[sd]


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data if a is not None else None


@dataclass
class OracleResult:
    W: np.ndarray
    Z: np.ndarray | None
    info: int
    nblocks: int
    block_start: np.ndarray
    mu: np.ndarray
    side: np.ndarray
    root_lo: np.ndarray
    root_hi: np.ndarray
    root_gstart: np.ndarray
    depth: np.ndarray
    grp_first: np.ndarray
    grp_last: np.ndarray
    fin_lo: np.ndarray
    fin_hi: np.ndarray
    stats: dict = field(default_factory=dict)


def mrrr(d, e, il: int | None = None, iu: int | None = None, *, gaptol: float | None = None, seed: int = 0,
         root_side: int = 0, threads: int = 0, roots_only: bool = False, sd: bool = False,
         early_stop: bool = False, support: bool = False) -> OracleResult:
    """Eigenpairs il..iu (1-based, inclusive) of the tridiagonal (d, e) by the oracle.  roots_only: stop after
    the root bisection (S1-S5): only nblocks/block_start/mu/side/root_lo/root_hi/root_gstart are filled.
    sd: the single/double realisation (liboracle_sd.so, gaptol 1e-5 by default); its inputs are
    the binary32 values (pass them as float32 or as their exact float64 images) and W, Z come back in float64
    before the final binary32 rounding (float32 of them is the realisation's output).  early_stop: the early
    classification stop of the root bisection (S5', A-41).  support: numerical-support
    truncation of every singleton vector (S10', Getvec remark (2) P:3459-3463, A-42)."""
    d = _f64(d)
    n = d.size
    e = _f64(e) if n > 1 else np.zeros(1)
    il = 1 if il is None else int(il)
    iu = n if iu is None else int(iu)
    k = iu - il + 1
    L = lib(sd)
    maxd = L.oracle_maxd()
    if gaptol is None:
        gaptol = 0.0 if sd else 1e-10
    W = np.zeros(k)
    Z = np.zeros((k, n))  # column j of the Fortran-style Z is row j here (ldz = n)
    nblocks = np.zeros(1, np.int32)
    bstart = np.zeros(n + 1, np.int32)
    mu = np.zeros(n)
    side = np.zeros(n, np.int32)
    rlo = np.zeros(n)
    rhi = np.zeros(n)
    rgs = np.zeros(n, np.int32)
    depth = np.zeros(k, np.int32)
    gf = np.zeros(maxd * k, np.int32)
    gl = np.zeros(maxd * k, np.int32)
    flo = np.zeros(k)
    fhi = np.zeros(k)
    st = np.zeros(16, np.int64)
    dg = _Diag(*[_ptr(a) for a in (nblocks, bstart, mu, side, rlo, rhi, rgs, depth, gf, gl, flo, fhi, st)])
    op = _Opts(gaptol, seed, root_side, threads, int(roots_only), int(early_stop), int(support))
    info = L.oracle_mrrr(n, _ptr(d), _ptr(e), il, iu, C.byref(op), _ptr(W), _ptr(Z), n, C.byref(dg))
    nbk = int(nblocks[0])
    return OracleResult(W=W, Z=Z.T, info=info, nblocks=nbk, block_start=bstart[:nbk + 1].copy(),
                        mu=mu[:nbk].copy(), side=side[:nbk].copy(), root_lo=rlo, root_hi=rhi, root_gstart=rgs,
                        depth=depth, grp_first=gf.reshape(maxd, k), grp_last=gl.reshape(maxd, k), fin_lo=flo,
                        fin_hi=fhi, stats={nm: int(st[i]) for i, nm in enumerate(STAT_NAMES)})


# ---------------------------------------------------------------- unit wrappers
def es_rtol(n: int, rtol: float, *, sd: bool = False) -> float:
    """Stage-1 tolerance of the early classification stop (S5', A-41)."""
    return lib(sd).oracle_es_rtol(n, rtol)


def es_stop(left, mid, right, gaptol: float, *, sd: bool = False) -> bool:
    """The early-stop test of an index from the stage-1 intervals (lo, hi) of it and its two neighbours."""
    return bool(lib(sd).oracle_es_stop(left[0], left[1], mid[0], mid[1], right[0], right[1], gaptol))


def xi(seed: int, idx: int, *, sd: bool = False) -> float:
    return lib(sd).oracle_xi(seed, idx)


def norm1(d, e) -> float:
    d, e = _f64(d), _f64(e)
    return lib().oracle_norm1(d.size, _ptr(d), _ptr(e))


def split(d, e, *, sd: bool = False) -> np.ndarray:
    d, e = _f64(d), _f64(e)
    st = np.zeros(d.size + 1, np.int32)
    nb = lib(sd).oracle_split(d.size, _ptr(d), _ptr(e), _ptr(st))
    return st[:nb + 1].copy()


def gershgorin(d, e, *, sd: bool = False):
    d, e = _f64(d), _f64(e)
    gl, gu, t = C.c_double(), C.c_double(), C.c_double()
    lib(sd).oracle_gershgorin(d.size, _ptr(d), _ptr(e), C.byref(gl), C.byref(gu), C.byref(t))
    return gl.value, gu.value, t.value


def negcount_x(dx, dllx, sigma: float, *, sd: bool = False) -> int:
    dx, dllx = _f64(dx), _f64(dllx)
    return lib(sd).oracle_negcount_x(dx.size, _ptr(dx), _ptr(dllx), sigma)


def negcount_x_many(dx, dllx, sigmas) -> np.ndarray:
    dx, dllx, sg = _f64(dx), _f64(dllx), _f64(sigmas)
    out = np.zeros(sg.size, np.int64)
    lib().oracle_negcount_x_many(dx.size, _ptr(dx), _ptr(dllx), sg.size, _ptr(sg), _ptr(out))
    return out


def negcount_t(d, e, sigma: float, mu: float = 0.0) -> int:
    """Eigenvalues of T below mu + sigma, Sturm count in binary128 (Alg. negcountT)."""
    d, e = _f64(d), _f64(e) if len(d) > 1 else np.zeros(1)
    return lib().oracle_negcount_t_q(d.size, _ptr(d), _ptr(e), mu, sigma)


def bisect_x(dx, dllx, j: int, lo: float, hi: float, rtol: float, *, sd: bool = False):
    dx, dllx = _f64(dx), _f64(dllx)
    a, b = C.c_double(lo), C.c_double(hi)
    lib(sd).oracle_bisect_x(dx.size, _ptr(dx), _ptr(dllx), j, rtol, C.byref(a), C.byref(b))
    return a.value, b.value


def dyadic_widen(lo: float, hi: float):
    a, b = C.c_double(), C.c_double()
    lib().oracle_dyadic_widen(lo, hi, C.byref(a), C.byref(b))
    return a.value, b.value


def is_boundary(lo1, hi1, lo2, hi2, gaptol=1e-10) -> bool:
    return bool(lib().oracle_is_boundary(lo1, hi1, lo2, hi2, gaptol))


def root_x(d, e, left: bool = True):
    d, e = _f64(d), _f64(e)
    n = d.size
    mu, gl, gu = C.c_double(), C.c_double(), C.c_double()
    bo = C.c_int()
    dx = np.zeros(n)
    lx = np.zeros(n)
    rc = lib().oracle_root_x(n, _ptr(d), _ptr(e), int(left), C.byref(mu), _ptr(dx), _ptr(lx), C.byref(gl),
                             C.byref(gu), C.byref(bo))
    return dict(rc=rc, mu=mu.value, d=dx, l=lx[:n - 1].copy(), gl=gl.value, gu=gu.value, backoffs=bo.value)


def root_y(d, e, left: bool = True, seed: int = 0, s: int = 0, nb: int | None = None, *, sd: bool = False):
    d, e = _f64(d), _f64(e)
    n = d.size
    nb = n - s if nb is None else nb
    mu = C.c_double()
    arrs = [np.zeros(nb) for _ in range(6)]
    rc = lib(sd).oracle_root_y(n, _ptr(d), _ptr(e), s, nb, int(left), seed, C.byref(mu), *[_ptr(a) for a in arrs])
    dh, dl, lh, ll, dx, dllx = arrs
    return dict(rc=rc, mu=mu.value, d_hi=dh, d_lo=dl, l_hi=lh, l_lo=ll, dx=dx, dllx=dllx)


def dstqds(d, l, tau: float, *, sd: bool = False):
    d, l = _f64(d), _f64(l)
    n = d.size
    lpad = np.zeros(n)
    lpad[:n - 1] = l
    dph, dpl, lph, sh = (np.zeros(n) for _ in range(4))
    lib(sd).oracle_dstqds(n, _ptr(d), _ptr(lpad), tau, _ptr(dph), _ptr(dpl), _ptr(lph), _ptr(sh))
    return dph, lph[:n - 1], sh


def dqds(d, l, tau: float, *, sd: bool = False):
    d, l = _f64(d), _f64(l)
    n = d.size
    lpad = np.zeros(n)
    lpad[:n - 1] = l
    om, um, p = (np.zeros(n) for _ in range(3))
    lib(sd).oracle_dqds(n, _ptr(d), _ptr(lpad), tau, _ptr(om), _ptr(um), _ptr(p))
    return om, um[:n - 1], p


def getvec(d, l, lam_hi: float, lam_lo: float = 0.0, r: int = 0, *, sd: bool = False):
    d, l = _f64(d), _f64(l)
    n = d.size
    lpad = np.zeros(n)
    lpad[:n - 1] = l
    z = np.zeros(n)
    rr = C.c_int64(r)
    g, zz = C.c_double(), C.c_double()
    c = C.c_int64()
    lib(sd).oracle_getvec(n, _ptr(d), _ptr(lpad), lam_hi, lam_lo, C.byref(rr), _ptr(z), C.byref(g), C.byref(zz),
                        C.byref(c))
    return dict(z=z, gamma=g.value, zz=zz.value, r=rr.value, c=c.value)


def residuals(d, e, W, Z) -> np.ndarray:
    """||T z_j - W_j z_j||_2 in binary128; Z is (n, k) column-major in spirit."""
    d, e, W = _f64(d), _f64(e), _f64(W)
    Zc = np.asfortranarray(Z, dtype=np.float64)
    n, k = Zc.shape
    res = np.zeros(k)
    lib().oracle_residuals(n, _ptr(d), _ptr(e), k, _ptr(W), Zc.ctypes.data, n, _ptr(res))
    return res


def ortho_full(Z) -> float:
    Zc = np.asfortranarray(Z, dtype=np.float64)
    n, k = Zc.shape
    return lib().oracle_ortho_full(n, k, Zc.ctypes.data, n)


def ortho_pairs(Z, pi, pj) -> float:
    Zc = np.asfortranarray(Z, dtype=np.float64)
    n, _ = Zc.shape
    pi = np.ascontiguousarray(pi, dtype=np.int64)
    pj = np.ascontiguousarray(pj, dtype=np.int64)
    return lib().oracle_ortho_pairs(n, Zc.ctypes.data, n, pi.size, _ptr(pi), _ptr(pj))


def jacobi(d, e) -> np.ndarray:
    """Eigenvalues (ascending) of the dense T by cyclic Jacobi in binary128, returned (hi, lo)."""
    d, e = _f64(d), _f64(e) if len(d) > 1 else np.zeros(1)
    n = d.size
    hi, lo = np.zeros(n), np.zeros(n)
    lib().oracle_jacobi(n, _ptr(d), _ptr(e), _ptr(hi), _ptr(lo))
    return hi, lo


# ------------------------------------------------------- branch pins (tests/test_oracle_branches.py)
def _lpad(d, l):
    d = _f64(d)
    lp = np.zeros(d.size)
    lp[:d.size - 1] = _f64(l)
    return d, lp


def jacobi_ldl(d, l):
    """Eigenvalues (ascending, hi/lo) of L D L^T multiplied out in binary128, by cyclic Jacobi."""
    d, lp = _lpad(d, l)
    hi, lo = np.zeros(d.size), np.zeros(d.size)
    lib().oracle_jacobi_ldl(d.size, _ptr(d), _ptr(lp), _ptr(hi), _ptr(lo))
    return hi, lo


def stats_read() -> dict:
    st = np.zeros(16, np.int64)
    lib().oracle_stats_read(_ptr(st))
    return {nm: int(st[i]) for i, nm in enumerate(STAT_NAMES)}


def stats_reset():
    lib().oracle_stats_reset()


def bracket_x(dx, dllx, j: int, lo: float, hi: float):
    dx, dllx = _f64(dx), _f64(dllx)
    a, b = C.c_double(lo), C.c_double(hi)
    fixes = lib().oracle_bracket_x(dx.size, _ptr(dx), _ptr(dllx), j, C.byref(a), C.byref(b))
    return a.value, b.value, fixes


def bracket_y(d, l, j: int, lo: float, hi: float, *, sd: bool = False):
    d, lp = _lpad(d, l)
    a, b = C.c_double(lo), C.c_double(hi)
    fixes = lib(sd).oracle_bracket_y(d.size, _ptr(d), _ptr(lp), j, C.byref(a), C.byref(b))
    return a.value, b.value, fixes


def bisect_y_full(d, l, j: int, lo: float, hi: float, *, sd: bool = False):
    d, lp = _lpad(d, l)
    a, b = C.c_double(), C.c_double()
    lib(sd).oracle_bisect_y_full(d.size, _ptr(d), _ptr(lp), j, lo, hi, C.byref(a), C.byref(b))
    return a.value, b.value


def rqi(d, l, j: int, lo: float, hi: float, gap: float, *, sd: bool = False, support: bool = False):
    d, lp = _lpad(d, l)
    W = C.c_double()
    z = np.zeros(d.size)
    it, fb = C.c_int64(), C.c_int64()
    lib(sd).oracle_rqi(d.size, _ptr(d), _ptr(lp), j, lo, hi, gap, int(support), C.byref(W), _ptr(z), C.byref(it), C.byref(fb))
    return dict(W=W.value, z=z, iters=it.value, fallbacks=fb.value)


def root_x_from(d, e, left: bool, mu0: float, t: float):
    d, e = _f64(d), _f64(e)
    n = d.size
    mu = C.c_double()
    bo = C.c_int()
    dx, lx = np.zeros(n), np.zeros(n)
    rc = lib().oracle_root_x_from(n, _ptr(d), _ptr(e), int(left), mu0, t, C.byref(mu), _ptr(dx), _ptr(lx),
                                  C.byref(bo))
    return dict(rc=rc, mu=mu.value, d=dx, l=lx[:n - 1].copy(), backoffs=bo.value)
