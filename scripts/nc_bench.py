"""Driver of scripts/nc_bench.cu (developer microbenchmark; uses the oracle only to build a root representation)."""
import ctypes as C, os, sys, subprocess
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mrrr_inputs as mi, oracle
H = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(H, "nc_bench.so")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(H, "nc_bench.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-Xcompiler", "-fPIC",
                           "-shared", "-o", so, os.path.join(H, "nc_bench.cu")])
L = C.CDLL(so)
L.nc_bench.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
L.nc_divcheck.argtypes = [C.c_longlong, C.c_uint64, C.c_void_p]
L.nc_xu.argtypes = [C.c_int, C.c_int, C.c_void_p]
for kind, nm in ((0, "MUFU.RCP64H"), (1, "MUFU.RCP f32")):
    r = C.c_float()
    L.nc_xu(kind, 2000, C.byref(r))
    print(f"{nm}: {r.value:.1f} thread-ops/ns = {r.value / 148 / 1.965:.1f} per SM per clock", flush=True)
cfg = mi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
d, e = cfg.matrix()
R = oracle.root_x(d, e, True)
n = d.size
dx, lx = R["d"], R["l"]
dll = np.zeros(n); dll[:n - 1] = (dx[:n - 1] * lx) * lx
mx = np.ascontiguousarray(np.stack([dx, dll], 1).ravel())
P = 2.0 ** np.ceil(np.log2(R["gu"] - R["mu"]))
names = {0: "v0 branch/step", 1: "sticky divA", 2: "sticky divB", 3: "sticky divC", 4: "sticky divB pf4",
         5: "sticky divA pf4", 6: "smem divB", 7: "smem divA", 9: "2 chains/thread divB", 8: "careful __ddiv_rn",
         10: "smem div_f (f32 seed)"}
for nch in (65536, 122880, 245760):
    ref = None
    for v in (8, 6, 10, 7):
        cnt = np.zeros(nch, np.int32)
        ms = C.c_float()
        msp = C.pointer(ms)
        rc = L.nc_bench(mx.ctypes.data, n, nch, P, v, 3, msp, cnt.ctypes.data)
        if ref is None: ref = cnt.copy()
        print(f"n={n} nch={nch:7d} {names[v]:24s} {ms.value:8.3f} ms  {ms.value*1e6/(n-1):7.1f} ns/step  "
              f"mismatch={int(np.sum(cnt != ref))} rc={rc}", flush=True)
bad = (C.c_ulonglong * 3)()
N = int(sys.argv[2]) if len(sys.argv) > 2 else 4_000_000_000
for seed in (1, 2):
    rc = L.nc_divcheck(C.c_longlong(N), C.c_uint64(seed), bad)
    print(f"divcheck N={N} seed={seed}: mismatches vs __ddiv_rn divA={bad[0]} divB={bad[1]} div_f={bad[2]} rc={rc}", flush=True)
