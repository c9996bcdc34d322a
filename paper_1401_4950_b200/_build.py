"""Build libmrrr.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(HERE, "csrc", "mrrr.cu")
DEPS = [os.path.join(HERE, "csrc", f) for f in ("mrrr.cu", "kernels.cuh", "kernels_vec.cuh", "kernels_rqi.cuh", "dd.cuh")] + \
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
        cmd = [nvcc(), *NVCC_FLAGS, "-o", LIB, SRC]
        if verbose:
            print(" ".join(cmd))
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
