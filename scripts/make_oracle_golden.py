"""Write the oracle's full-size results for the BASELINE configurations C3, C4, C5b, C5a to
tests/golden/oracle_<cfg>.npz (calls only oracle/ and mrrr_inputs/; never the CUDA path).

The full oracle solves take minutes to an hour of CPU time, far too long for the GPU test run, so the GPU
parity tests (tests/test_gpu_fullsize.py) compare the CUDA path against these stored oracle outputs, and
check that the stored file belongs to the same input bytes and the same oracle source (SHA-256 of both).
C1 and C2 are cheap and are compared against a live oracle run.

    python scripts/make_oracle_golden.py [C3 C4 C5b C5a] [--threads N]

Stored per config: block starts, mu and side per block, every root interval (fp64 bits) and root group start,
depth / group extents per depth / final-node interval of every output index (the integer diagnostics the
parity gates compare bit for bit), W, and the oracle's statistics.  Final-node intervals are stored only
below the root (at depth 0 they are the root intervals).
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import mrrr_inputs as mi  # noqa: E402
import oracle  # noqa: E402


def input_sha(d, e):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(d, np.float64).tobytes())
    h.update(np.ascontiguousarray(e, np.float64).tobytes())
    return h.hexdigest()


def oracle_sha():
    with open(os.path.join(ROOT, "oracle", "mrrr_oracle.c"), "rb") as f:
        return hashlib.sha256(f.read()).hexdigest()


def golden_path(name):
    return os.path.join(ROOT, "tests", "golden", f"oracle_{name}.npz")


def make(name, threads):
    cfg = mi.CONFIGS[name]
    d, e = cfg.matrix()
    t0 = time.time()
    r = oracle.mrrr(d, e, cfg.il, cfg.iu, threads=threads)
    wall = time.time() - t0
    assert r.info == 0, r.info
    dmax = int(r.depth.max())
    below = r.depth > 0
    fin_lo = np.where(below, r.fin_lo, np.nan)
    fin_hi = np.where(below, r.fin_hi, np.nan)
    meta = dict(config=name, n=cfg.n, il=cfg.il, iu=cfg.iu, input_sha256=input_sha(d, e), oracle_sha256=oracle_sha(),
                gaptol=1e-10, seed=0, stats=r.stats, wall_s=wall, threads=threads, script="scripts/make_oracle_golden.py")
    np.savez_compressed(golden_path(name), meta=np.array(json.dumps(meta)), block_start=r.block_start, mu=r.mu,
                        side=r.side, root_lo=r.root_lo, root_hi=r.root_hi, root_gstart=r.root_gstart.astype(np.int8),
                        depth=r.depth.astype(np.int8), grp_first=r.grp_first[:dmax + 1], grp_last=r.grp_last[:dmax + 1],
                        fin_lo=fin_lo, fin_hi=fin_hi, W=r.W)
    print(f"{name}: {wall:.1f} s on {threads} threads, stats {r.stats}", flush=True)


def load(name):
    """The stored oracle result as a dict (meta decoded); raises FileNotFoundError if absent."""
    z = np.load(golden_path(name))
    out = {k: z[k] for k in z.files if k != "meta"}
    out["meta"] = json.loads(str(z["meta"]))
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", default=["C3", "C4", "C5b", "C5a"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    a = ap.parse_args()
    for c in a.configs:
        make(c, a.threads)
