"""Developer sweep of schedule knobs (env variables read at mrrr_init) on one config, in one process:

    python scripts/sweep_env.py C2 5 "" "MRRR_SEGK=16" "MRRR_SEGK=16 MRRR_SEGW=64"

prints ms per solve (median over reps, CUDA events, L2 flushed between solves) and the phase split.
A config name "sd:<cfg>" runs the single/double realisation (mrrr_seig) on the binary32 copy of <cfg>."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

SD = sys.argv[1].startswith("sd:")
if SD:
    sys.argv[1] = sys.argv[1][3:]
if sys.argv[1].startswith("fam:"):  # fam:<family>:<n>, all pairs
    _, fam, nn = sys.argv[1].split(":")
    _d, _e = mi.FAMILIES[fam](int(nn))
    cfg = mi.Config(f"{fam}{_d.size}", _d.size, 1, _d.size, lambda: (_d, _e), fam)
else:
    cfg = mi.CONFIGS[sys.argv[1]]
reps = int(sys.argv[2])
d, e = cfg.matrix()
fdt = np.float32 if SD else np.float64
dt, et = torch.from_numpy(d.astype(fdt)).cuda(), torch.from_numpy(e.astype(fdt)).cuda()
W = torch.empty(cfg.k, dtype=dt.dtype, device="cuda")
Z = torch.empty((cfg.k, cfg.n), dtype=dt.dtype, device="cuda")
flush = torch.empty(32 * 1024 * 1024, dtype=torch.float64, device="cuda")
base = dict(os.environ)
W0 = None
for spec in sys.argv[3:]:
    os.environ.clear()
    os.environ.update(base)
    for kv in spec.split():
        k, v = kv.split("=")
        os.environ[k] = v
    s = m.Solver()
    ts = []
    for r in range(reps + 2):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        (s.seig if SD else s.eig)(dt, et, cfg.il, cfg.iu, W=W, Z=Z)
        b.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(a.elapsed_time(b))
    Wc = W.cpu().numpy()
    same = "" if W0 is None else ("W=" if np.array_equal(Wc, W0) else f"dW={np.max(np.abs(Wc - W0)):.2e}")
    if W0 is None:
        W0 = Wc.copy()
    t = s.times()
    st = s.stats()
    print(f"{'sd:' if SD else ''}{cfg.name} [{spec or 'default'}] {np.median(ts):.3f} ms (min {min(ts):.3f}) | bis {t['root_bisection']:.2f} "
          f"clu {t['clusters']:.2f} sing {t['singletons']:.2f} | neg {t['negcount_ms_per_launch']*1e3:.1f} us x "
          f"{int(t['negcount_launches'])} | rqi {t['rqi_ms_per_launch']:.3f} x {int(t['rqi_launches'])} | "
          f"rounds {st['rounds']} launches {st['launches']} ho {st['rqi_handover']} "
          f"xgfb {st['xg_fallback_chains']}/{st['xg_fallback_segments']} rootfb {st['root_fallback_chains']} {same}", flush=True)
    s.close()
