"""Build libmrrr.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import glob
import os
import shlex
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "mrrr.cu")
DEPS = sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")) + glob.glob(os.path.join(HERE, "csrc", "*.cuh"))) + \
    [os.path.join(ROOT, "include", "mrrr.h")]
LIB = os.path.join(HERE, "libmrrr.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


def nvcc():
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.exists(c) or c == "nvcc"):
            return c
    return "nvcc"


def build(force: bool = False, verbose: bool = False) -> str:
    stale = not os.path.exists(LIB) or any(os.path.getmtime(LIB) < os.path.getmtime(p) for p in DEPS)
    if force or stale:
        # MRRR_NVCC_EXTRA: developer experiments only (e.g. "-DMRRR_ZG=4"); the product build sets nothing
        cmd = [nvcc(), *NVCC_FLAGS, *shlex.split(os.environ.get("MRRR_NVCC_EXTRA", "")), "-o", LIB, SRC]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
