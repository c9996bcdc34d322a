"""Seeded synthetic tridiagonal inputs shared by the oracle tests, the GPU parity
tests and ``bench.py``.

This module holds NONE of the eigensolver's arithmetic: it only produces the
input diagonals ``d`` (alpha) and off-diagonals ``e`` (beta) of a symmetric
tridiagonal T (PAPER.md eq:thetridiagonal) from a written recipe.
Both sides of a parity check (``oracle/`` and the CUDA path) receive the same
bytes from here; neither side imports the other.

Recipes:

* SplitMix64 (Steele/Lea/Flood 2014).  The i-th output (i = 0, 1, ...) of the
  stream keyed by ``seed`` is ``mix(seed + (i + 1) * 0x9E3779B97F4A7C15 mod
  2^64)`` with the standard finaliser ``mix``.  A uniform double in [0, 1) is
  ``(x >> 11) * 2^-53`` (exact); uniform [-1, 1) is ``2u - 1`` (exact).
* C1  1-2-1 Toeplitz, n = 1000: d = 2, e = -1 (App. D).
* C2  random, n = 8192, seed 14014950: n draws for d (U[-1,1)), then n-1 draws
      for e (U[-1,1)).
* C3  Wilkinson W+ with m = 8192 (n = 16385): d_i = |m - i|, e = 1
      (App. D).
* C4  glued Wilkinson: 128 copies of W+_{201} (d = |100 - i|), e = 1 inside,
      glue e[201 b - 1] = 1e-10 for b = 1..127 (0-based e).
* C5  random, n = 65536, seed 14014951: d ~ U[-1,1), e ~ U[0,1)
      (C5a all pairs, C5b indices 1..6553).
* Families of App. D for the §8(f1) sweeps: 1-2-1, Clement (Kac), Wilkinson, Hermite, Legendre,
  Laguerre (readings A-23 in DESIGN.md), and the two prescribed-spectrum families Uniform
  (lambda_k = eps + (k-1)(1-eps)/(n-1)) and Geometric (lambda_k = eps^((n-k)/(n-1))), eps = 2^-53: T is the
  Householder tridiagonal form (LAPACK dsytrd) of Q diag(lambda) Q^T with Q the orthogonal factor of a
  seeded Gaussian matrix (the LAPACK test-matrix recipe the paper's Artificial set follows),
  computed with one BLAS thread so that the bytes do not depend on the host.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass
from typing import Callable

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int, start: int = 0) -> np.ndarray:
    """Outputs ``start .. start+count-1`` of the SplitMix64 stream keyed by ``seed``."""
    with np.errstate(over="ignore"):
        i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def uniform01(seed: int, count: int, start: int = 0) -> np.ndarray:
    """(x >> 11) * 2^-53: exact doubles in [0, 1)."""
    x = splitmix64(seed, count, start) >> np.uint64(11)
    return x.astype(np.float64) * (2.0 ** -53)


# ----------------------------------------------------------------------------
# generators: each returns (d, e) as contiguous float64 arrays
# ----------------------------------------------------------------------------

def one_two_one(n: int, offdiag: float = -1.0):
    return np.full(n, 2.0), np.full(max(n - 1, 0), offdiag)


def random_tridiag(n: int, seed: int, e_lo: float = -1.0):
    """d ~ U[-1,1); e ~ U[-1,1) if e_lo == -1 else U[0,1) (C2 / C5 recipes)."""
    u = uniform01(seed, 2 * n - 1)
    d = 2.0 * u[:n] - 1.0
    ue = u[n:]
    e = 2.0 * ue - 1.0 if e_lo == -1.0 else ue.copy()
    return np.ascontiguousarray(d), np.ascontiguousarray(e)


def wilkinson(m: int):
    n = 2 * m + 1
    i = np.arange(n, dtype=np.float64)
    return np.abs(m - i), np.ones(n - 1)


def glued_wilkinson(copies: int = 128, m: int = 100, glue: float = 1e-10):
    db, eb = wilkinson(m)
    bs = db.size
    d = np.tile(db, copies)
    e = np.ones(bs * copies - 1)
    for b in range(1, copies):
        e[bs * b - 1] = glue
    return d, e


def clement(n: int):
    k = np.arange(1, n, dtype=np.float64)
    return np.zeros(n), np.sqrt(k * (n - k))


def hermite(n: int):
    return np.zeros(n), np.sqrt(np.arange(1, n, dtype=np.float64))


def legendre(n: int):
    # beta_k = k / sqrt((2k-1)(2k+1)), k = 2..n  (A-23: n-1 values to positions 1..n-1)
    k = np.arange(2, n + 1, dtype=np.float64)
    return np.zeros(n), k / np.sqrt((2 * k - 1) * (2 * k + 1))


def laguerre(n: int):
    # diag (3,5,...,2n+1); off-diagonal (2,3,...,n) (A-23 extends the garbled n-2 list)
    return 2.0 * np.arange(1, n + 1, dtype=np.float64) + 1.0, np.arange(2, n + 1, dtype=np.float64)


def _prescribed_spectrum(lam: np.ndarray, seed: int):
    import scipy.linalg as sla
    from threadpoolctl import threadpool_limits
    n = lam.size
    with threadpool_limits(limits=1):
        g = np.random.default_rng(seed).standard_normal((n, n))
        q, r = np.linalg.qr(g)
        q = q * np.sign(np.diag(r))          # Haar-distributed orthogonal factor
        a = (q * lam) @ q.T
        a = (a + a.T) / 2
        c, d, e, tau, info = sla.lapack.dsytrd(a, lower=1)
    assert info == 0
    return np.ascontiguousarray(d), np.ascontiguousarray(e)


def uniform_spectrum(n: int, seed: int = 7239):
    """Uniform family (App. D): eigenvalues eps + (k-1)(1-eps)/(n-1), k = 1..n."""
    eps = 2.0 ** -53
    k = np.arange(1, n + 1, dtype=np.float64)
    return _prescribed_spectrum(eps + (k - 1) * (1 - eps) / (n - 1), seed)


def geometric_spectrum(n: int, seed: int = 7242):
    """Geometric family (App. D): eigenvalues eps^((n-k)/(n-1)), k = 1..n."""
    eps = 2.0 ** -53
    k = np.arange(1, n + 1, dtype=np.float64)
    return _prescribed_spectrum(eps ** ((n - k) / (n - 1)), seed)


# App. D families by name, each a function of n (Wilkinson: the odd size 2m+1 <= n+1)
FAMILIES = {
    "uniform": lambda n: uniform_spectrum(n),
    "geometric": lambda n: geometric_spectrum(n),
    "121": lambda n: one_two_one(n),
    "clement": lambda n: clement(n),
    "wilkinson": lambda n: wilkinson(n // 2),
    "hermite": lambda n: hermite(n),
    "legendre": lambda n: legendre(n),
    "laguerre": lambda n: laguerre(n),
}


def sha256(d: np.ndarray, e: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(d, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(e, dtype=np.float64).tobytes())
    return h.hexdigest()


@dataclass(frozen=True)
class Config:
    name: str
    n: int
    il: int
    iu: int
    make: Callable[[], tuple]
    note: str

    def matrix(self):
        d, e = self.make()
        return np.ascontiguousarray(d, dtype=np.float64), np.ascontiguousarray(e, dtype=np.float64)

    @property
    def k(self) -> int:
        return self.iu - self.il + 1


CONFIGS = {
    "C1": Config("C1", 1000, 1, 1000, lambda: one_two_one(1000), "1-2-1 Toeplitz n=1000, all pairs"),
    "C2": Config("C2", 8192, 1, 8192, lambda: random_tridiag(8192, 14014950, -1.0),
                 "random U[-1,1) n=8192 seed 14014950, all pairs"),
    "C3": Config("C3", 16385, 1, 16385, lambda: wilkinson(8192), "Wilkinson W+ m=8192, all pairs"),
    "C4": Config("C4", 25728, 1, 25728, lambda: glued_wilkinson(128, 100, 1e-10),
                 "128 x W+_201 glued by 1e-10, all pairs"),
    "C5a": Config("C5a", 65536, 1, 65536, lambda: random_tridiag(65536, 14014951, 0.0),
                  "random d~U[-1,1) e~U[0,1) n=65536 seed 14014951, all pairs"),
    "C5b": Config("C5b", 65536, 1, 6553, lambda: random_tridiag(65536, 14014951, 0.0),
                  "same matrix as C5a, indices 1..6553"),
}
