"""The CPU oracle timed on the host it runs on: CPU model, core count, 1-thread and all-thread
wall times of C1 and C2 (all pairs), and all-thread times of the other configurations (C5a: root bisection of all
indices plus the full solve of a 6,553-index window, scaled -- the full C5a oracle solve takes ~10 min on 16 threads).

    python scripts/oracle_times.py > profiles/r02_oracle_times.txt
"""
import os
import platform
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mrrr_inputs as mi  # noqa: E402
import oracle  # noqa: E402


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


ncpu = os.cpu_count() or 1
print(f"host: {cpu_model()}, {ncpu} logical CPUs (nproc), oracle = oracle/mrrr_oracle.c (gcc -O2, OpenMP, binary128 y-path)")
print("config  k       n       threads  wall_s    entries/s")


def run(name, threads, il=None, iu=None, note=""):
    c = mi.CONFIGS[name]
    d, e = c.matrix()
    il = c.il if il is None else il
    iu = c.iu if iu is None else iu
    t0 = time.perf_counter()
    r = oracle.mrrr(d, e, il, iu, threads=threads)
    t = time.perf_counter() - t0
    assert r.info == 0
    k = iu - il + 1
    print(f"{name:6s}  {k:6d}  {c.n:6d}  {threads:7d}  {t:8.2f}  {k * c.n / t:10.3e}  {note}", flush=True)


run("C1", 1)
run("C1", ncpu)
run("C2", 1)
run("C2", ncpu)
for name in ("C3", "C4", "C5b"):
    run(name, ncpu)
run("C5a", ncpu, 1, 6553, "(window 1..6553 of C5a = C5b's work; the all-pairs solve is ~10x)")
