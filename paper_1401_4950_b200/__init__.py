"""B200-native mixed-precision MRRR tridiagonal eigensolver (arXiv 1401.4950).

Thin ctypes binding of ``libmrrr.so`` (C ABI in ``include/mrrr.h``): argument
marshalling only.  Every step of the solve runs in the sm_100a kernels of
``csrc/``; there is no CPU fallback -- importing works without a GPU, but
creating a solver raises if the library or a CUDA device is missing.

    import torch, paper_1401_4950_b200 as mrrr
    s = mrrr.Solver()
    W, Z = s.eig(d_cuda, e_cuda)          # all pairs; Z is (n, k), column j <-> W[j]
    W, Z = s.eig(d_cuda, e_cuda, 1, 100)  # indices 1..100 (1-based, inclusive)
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MRRR_LIB") or os.path.join(HERE, "libmrrr.so")

KEEP_DIAG = 1
EARLY_STOP = 2  # MRRR_EARLY_STOP (include/mrrr.h): early classification stop of the root bisection
FULL_SUPPORT = 4  # MRRR_FULL_SUPPORT: store the whole Getvec recurrence (no numerical-support truncation, A-42)
MAXD = 8
NSTATS = 37
STAT_NAMES = ["d_max", "n_clusters", "largest_cluster", "uncertified", "shift_attempts", "rqi_iters",
              "rqi_fallbacks", "bracket_fixes", "root_backoffs", "failed", "negcount_x", "negcount_y",
              "getvec_calls", "rounds", "launches", "nblocks", "qd_steps", "qdg_steps", "z_steps", "zw_steps",
              "negcount_x_alg", "negcount_y_alg", "rqi_reject_sign", "rqi_reject_bracket", "rqi_handover", "ho_twist", "ho_fixed", "ho_rqc", "qd_light", "twist_rows", "seg_wide", "careful",
              "xg_fallback_chains", "xg_fallback_segments", "early_stops", "root_fallback_chains", "zwin_reruns"]
TIME_NAMES = ["total", "split_root", "root_bisection", "classification", "clusters", "singletons",
              "rqi_ms_per_launch", "rqi_launches", "negcount_ms_per_launch", "negcount_launches", "t10", "t11"]


class MrrrError(RuntimeError):
    pass


class _Opts(C.Structure):
    _fields_ = [("device", C.c_int32), ("root_side", C.c_int32), ("stream", C.c_void_p), ("gaptol", C.c_double),
                ("seed", C.c_uint64), ("flags", C.c_uint32), ("reserved", C.c_uint32), ("ws_limit", C.c_int64)]


class _Diag(C.Structure):
    _fields_ = [(nm, C.c_void_p) for nm in ("nblocks", "block_start", "mu", "side", "root_lo", "root_hi",
                                            "root_gstart", "depth", "grp_first", "grp_last", "fin_lo", "fin_hi")]


_lib = None


def load() -> C.CDLL:
    """Load libmrrr.so; raises if it was not built (run __graft_entry__.build())."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise MrrrError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        i64, vp = C.c_int64, C.c_void_p
        L.mrrr_init.argtypes = [C.POINTER(vp), C.POINTER(_Opts)]
        L.mrrr_eig.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, i64]
        L.mrrr_eig_host.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, i64]
        L.mrrr_seig.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, i64]
        L.mrrr_seig_host.argtypes = [vp, vp, vp, i64, i64, i64, vp, vp, i64]
        L.mrrr_eig_shard.argtypes = [vp, vp, vp, i64, i64, i64, i64, i64, vp, vp, i64, i64, C.POINTER(i64),
                                      C.POINTER(i64)]
        L.mrrr_get_stats.argtypes = [vp, vp, C.c_int32]
        L.mrrr_get_times.argtypes = [vp, vp, C.c_int32]
        L.mrrr_get_diag.argtypes = [vp, C.POINTER(_Diag)]
        L.mrrr_shard_owner.argtypes = [vp, i64, i64, i64, i64, i64, i64, C.POINTER(i64), C.POINTER(i64)]
        L.mrrr_shard_owner.restype = C.c_int
        L.mrrr_selftest.argtypes = [C.c_int, i64, C.c_uint64, C.POINTER(i64)]
        L.mrrr_selftest.restype = C.c_int
        L.mrrr_strerror.argtypes = [C.c_int]
        L.mrrr_strerror.restype = C.c_char_p
        L.mrrr_destroy.argtypes = [vp]
        L.mrrr_nccl_unique_id.argtypes = [vp]
        L.mrrr_eig_dist.argtypes = [vp, vp, C.c_int32, C.c_int32, vp, vp, i64, i64, i64, vp, vp, i64, i64,
                                    C.POINTER(i64), C.POINTER(i64)]
        for f in ("mrrr_init", "mrrr_eig", "mrrr_eig_host", "mrrr_eig_shard", "mrrr_get_stats", "mrrr_get_times",
                  "mrrr_get_diag", "mrrr_destroy", "mrrr_nccl_unique_id", "mrrr_eig_dist", "mrrr_seig",
                  "mrrr_seig_host"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


EXPORTED = ["mrrr_init", "mrrr_eig", "mrrr_eig_host", "mrrr_eig_shard", "mrrr_get_stats", "mrrr_get_diag",
            "mrrr_get_times", "mrrr_selftest", "mrrr_shard_owner", "mrrr_strerror", "mrrr_destroy",
            "mrrr_nccl_unique_id", "mrrr_eig_dist", "mrrr_seig", "mrrr_seig_host"]


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for :meth:`Solver.eig_dist` (create on one rank, send to all)."""
    buf = C.create_string_buffer(128)
    _check(load().mrrr_nccl_unique_id(buf), "mrrr_nccl_unique_id")
    return buf.raw


def selftest(which: int, n: int, seed: int = 1) -> int:
    """Run a built-in device self test; returns the number of mismatches (see include/mrrr.h)."""
    bad = C.c_int64()
    _check(load().mrrr_selftest(which, n, seed, C.byref(bad)), "mrrr_selftest")
    return bad.value


def _check(rc: int, what: str):
    if rc != 0:
        msg = load().mrrr_strerror(rc).decode()
        raise MrrrError(f"{what} failed with code {rc}: {msg}")


@dataclass
class Diag:
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


class Solver:
    """One libmrrr handle (one device, one stream)."""

    def __init__(self, device: int | None = None, gaptol: float = 0.0, seed: int = 0, root_side: int = 0,
                 keep_diag: bool = False, stream: int | None = None, ws_limit: int = 0,
                 early_stop: bool = False, full_support: bool = False):
        L = load()
        self._h = C.c_void_p()
        flags = ((KEEP_DIAG if keep_diag else 0) | (EARLY_STOP if early_stop else 0)
                 | (FULL_SUPPORT if full_support else 0))
        o = _Opts(-1 if device is None else int(device), int(root_side), stream, float(gaptol), int(seed),
                  flags, 0, int(ws_limit))
        _check(L.mrrr_init(C.byref(self._h), C.byref(o)), "mrrr_init")
        self.keep_diag = keep_diag
        self._last = (0, 0)

    # -------------------------------------------------------------- solves
    def eig(self, d, e, il: int | None = None, iu: int | None = None, W=None, Z=None):
        """Device solve: d, e are float64 CUDA tensors.  Returns (W, Z) with Z of shape (n, k) (a
        column-major view: Z[:, j] is contiguous)."""
        return self._eig_dev(d, e, il, iu, W, Z, single=False)

    def seig(self, d, e, il: int | None = None, iu: int | None = None, W=None, Z=None):
        """Single/double realisation (mrrr_seig): d, e float32 CUDA tensors in, float32 (W, Z)
        out, binary64 inside, gaptol 1e-5."""
        return self._eig_dev(d, e, il, iu, W, Z, single=True)

    def _eig_dev(self, d, e, il, iu, W, Z, single: bool):
        import torch
        dt = torch.float32 if single else torch.float64
        tn = "float32" if single else "float64"
        n = d.numel()
        il = 1 if il is None else int(il)
        iu = n if iu is None else int(iu)
        k = max(iu - il + 1, 0)
        if not (d.is_cuda and d.dtype == dt and d.is_contiguous()):
            raise MrrrError(f"d must be a contiguous {tn} CUDA tensor")
        if n > 1 and not (e.is_cuda and e.dtype == dt and e.is_contiguous()):
            raise MrrrError(f"e must be a contiguous {tn} CUDA tensor")
        if W is None:
            W = torch.empty(k, dtype=dt, device=d.device)
        if Z is None:
            Zt = torch.empty((k, n), dtype=dt, device=d.device)
        elif Z.dim() == 2 and tuple(Z.shape) == (n, k) and Z.stride() == (1, n):
            Zt = Z.T  # a column-major (n, k) view (e.g. the Z returned by an earlier call)
        elif Z.dim() == 2 and tuple(Z.shape) == (k, n) and Z.is_contiguous():
            Zt = Z    # row j of the (k, n) buffer receives eigenvector j
        else:
            raise MrrrError("Z must be a contiguous (k, n) buffer or a column-major (n, k) view")
        if not (Zt.is_cuda and Zt.dtype == dt and W.dtype == dt) or W.numel() < k:
            raise MrrrError(f"W, Z must be {tn} CUDA buffers of k and k x n entries")
        ep = e.data_ptr() if (e is not None and e.numel()) else None
        fn = "mrrr_seig" if single else "mrrr_eig"
        rc = getattr(load(), fn)(self._h, d.data_ptr(), ep, n, il, iu, W.data_ptr(), Zt.data_ptr(), n)
        _check(rc, fn)
        self._last = (n, k)
        return W, Zt.T

    def eig_host(self, d: np.ndarray, e: np.ndarray, il: int | None = None, iu: int | None = None,
                 W: np.ndarray | None = None, Zt: np.ndarray | None = None, single: bool = False):
        """Host solve (copies inside the call): d, e host arrays in, (W, Z[n, k]) host arrays out.  W (k,) and
        Zt (k, n) may be supplied (e.g. page-locked buffers for full-speed copies).  single: the
        single/double realisation (mrrr_seig_host; float32 arrays in and out)."""
        dt = np.float32 if single else np.float64
        d = np.ascontiguousarray(d, dtype=dt)
        n = d.size
        e = np.ascontiguousarray(e, dtype=dt) if n > 1 else np.zeros(1, dt)
        il = 1 if il is None else int(il)
        iu = n if iu is None else int(iu)
        k = iu - il + 1
        if W is None:
            W = np.empty(k, dt)
        if Zt is None:
            Zt = np.empty((k, n), dt)
        if W.shape != (k,) or Zt.shape != (k, n) or W.dtype != dt or Zt.dtype != dt \
                or not (W.flags.c_contiguous and Zt.flags.c_contiguous):
            raise MrrrError(f"W must be {dt.__name__} (k,), Zt {dt.__name__} C-contiguous (k, n)")
        fn = "mrrr_seig_host" if single else "mrrr_eig_host"
        rc = getattr(load(), fn)(self._h, d.ctypes.data, e.ctypes.data, n, il, iu, W.ctypes.data, Zt.ctypes.data, n)
        _check(rc, fn)
        self._last = (n, k)
        return W, Zt.T

    def eig_shard(self, d, e, sl: int, su: int, il: int | None = None, iu: int | None = None,
                  ncols_cap: int | None = None):
        """Multi-GPU shard [sl, su] of the selection [il, iu] (default all pairs): eigenpairs of the units
        (root groups cut to [il, iu]) that start in [sl, su]; returns (jlo, jhi, W, Z)."""
        import torch
        n = d.numel()
        il = 1 if il is None else int(il)
        iu = n if iu is None else int(iu)
        cap = (su - sl + 1) * 2 + 64 if ncols_cap is None else ncols_cap
        cap = max(min(cap, iu - il + 1), 1)
        W = torch.empty(cap, dtype=torch.float64, device=d.device)
        Zt = torch.empty((cap, n), dtype=torch.float64, device=d.device)
        jlo, jhi = C.c_int64(), C.c_int64()
        rc = load().mrrr_eig_shard(self._h, d.data_ptr(), e.data_ptr() if n > 1 else None, n, il, iu, int(sl),
                                   int(su), W.data_ptr(), Zt.data_ptr(), n, cap, C.byref(jlo), C.byref(jhi))
        _check(rc, "mrrr_eig_shard")
        m = max(jhi.value - jlo.value + 1, 0)
        self._last = (n, m)
        return jlo.value, jhi.value, W[:m], Zt[:m].T

    def eig_dist(self, d, e, il: int, iu: int, nccl_id: bytes, rank: int, world: int,
                 ncols_cap: int | None = None):
        """Multi-GPU solve through libmrrr's own NCCL all-gather (mrrr_eig_dist): every rank gets all
        k = iu - il + 1 eigenvalues in W and its owned eigenvectors; returns (jlo, jhi, W, Z_local)."""
        import torch
        n = d.numel()
        k = iu - il + 1
        per = -(-k // world)
        cap = max(min(per * 2 + 64 if ncols_cap is None else ncols_cap, k), 1)
        W = torch.empty(k, dtype=torch.float64, device=d.device)
        Zt = torch.empty((cap, n), dtype=torch.float64, device=d.device)
        jlo, jhi = C.c_int64(), C.c_int64()
        idb = C.create_string_buffer(bytes(nccl_id), 128)
        rc = load().mrrr_eig_dist(self._h, idb, int(rank), int(world), d.data_ptr(),
                                  e.data_ptr() if n > 1 else None, n, int(il), int(iu), W.data_ptr(),
                                  Zt.data_ptr(), n, cap, C.byref(jlo), C.byref(jhi))
        _check(rc, "mrrr_eig_dist")
        m = max(jhi.value - jlo.value + 1, 0)
        self._last = (n, m)
        return jlo.value, jhi.value, W, Zt[:m].T

    # -------------------------------------------------------------- results
    def stats(self) -> dict:
        s = np.zeros(NSTATS, np.int64)
        _check(load().mrrr_get_stats(self._h, s.ctypes.data, NSTATS), "mrrr_get_stats")
        return {nm: int(s[i]) for i, nm in enumerate(STAT_NAMES)}

    def times(self) -> dict:
        t = np.zeros(12)
        _check(load().mrrr_get_times(self._h, t.ctypes.data, 12), "mrrr_get_times")
        return {nm: float(t[i]) for i, nm in enumerate(TIME_NAMES)}

    def diag(self) -> Diag:
        n, k = self._last
        a = dict(nblocks=np.zeros(1, np.int32), block_start=np.zeros(n + 1, np.int32), mu=np.zeros(n),
                 side=np.zeros(n, np.int32), root_lo=np.zeros(n), root_hi=np.zeros(n),
                 root_gstart=np.zeros(n, np.int32), depth=np.zeros(k, np.int32),
                 grp_first=np.zeros(MAXD * k, np.int32), grp_last=np.zeros(MAXD * k, np.int32), fin_lo=np.zeros(k),
                 fin_hi=np.zeros(k))
        g = _Diag(*[a[f].ctypes.data for f, _ in _Diag._fields_])
        _check(load().mrrr_get_diag(self._h, C.byref(g)), "mrrr_get_diag")
        nb = int(a["nblocks"][0])
        return Diag(nblocks=nb, block_start=a["block_start"][:nb + 1], mu=a["mu"][:nb], side=a["side"][:nb],
                    root_lo=a["root_lo"], root_hi=a["root_hi"], root_gstart=a["root_gstart"], depth=a["depth"],
                    grp_first=a["grp_first"].reshape(MAXD, k), grp_last=a["grp_last"].reshape(MAXD, k),
                    fin_lo=a["fin_lo"], fin_hi=a["fin_hi"])

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            load().mrrr_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def eig(d, e, il=None, iu=None, **kw):
    """One-shot convenience: device tensors in, (W, Z) out."""
    s = Solver(**kw)
    try:
        return s.eig(d, e, il, iu)
    finally:
        s.close()
