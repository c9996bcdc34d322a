"""Kernel timeline of one solve (torch.profiler / CUPTI): per-kernel start and duration, and the idle gaps
between consecutive kernels (host round trips), summed by the kernel that follows the gap.

    python scripts/timeline.py C2 [sd]
"""
import sys
from collections import defaultdict

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
sd = len(sys.argv) > 2 and sys.argv[2] == "sd"
c = mi.CONFIGS[name]
d, e = c.matrix()
dt = np.float32 if sd else np.float64
d_, e_ = torch.from_numpy(d.astype(dt)).cuda(), torch.from_numpy(e.astype(dt)).cuda()
s = m.Solver()
f = s.seig if sd else s.eig
W = torch.empty(c.k, dtype=d_.dtype, device="cuda")
Z = torch.empty((c.k, c.n), dtype=d_.dtype, device="cuda")
for _ in range(3):
    f(d_, e_, c.il, c.iu, W=W, Z=Z)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    f(d_, e_, c.il, c.iu, W=W, Z=Z)
    torch.cuda.synchronize()
allev = list(prof.events())
ev = [x for x in allev if x.device_type.name == "CUDA"]
rt = sorted([x for x in allev if x.device_type.name == "CPU" and x.name.startswith("cuda")],
            key=lambda x: x.time_range.start)
ev.sort(key=lambda x: x.time_range.start)
t0 = ev[0].time_range.start
busy = sum(x.time_range.end - x.time_range.start for x in ev)
span = ev[-1].time_range.end - t0
gaps = defaultdict(float)
ngap = defaultdict(int)
prev_end = ev[0].time_range.end
prev_name = ev[0].name
big = []
for x in ev[1:]:
    g = x.time_range.start - prev_end
    if g > 0:
        key = x.name.split("(")[0][:40]
        gaps[key] += g
        ngap[key] += 1
        big.append((g, prev_name.split("(")[0][:30], key, (x.time_range.start - t0) / 1e3))
    prev_end = max(prev_end, x.time_range.end)
    prev_name = x.name
print(f"{name}{' sd' if sd else ''}: {len(ev)} device activities, span {span/1e3:.3f} ms, busy {busy/1e3:.3f} ms, "
      f"idle {(span-busy)/1e3:.3f} ms")
for k, v in sorted(gaps.items(), key=lambda kv: -kv[1])[:15]:
    print(f"  idle before {k:42s} {v/1e3:8.3f} ms over {ngap[k]} gaps")
print("  largest single gaps (us, after -> before, at ms):")
for g, a, b, at in sorted(big, reverse=True)[:8]:
    print(f"    {g:8.1f}  {a:30s} -> {b:40s} @ {at:.3f}")
# runtime API calls issued inside the largest gaps (what the host was doing while the GPU idled)
for g, a, b, at in sorted(big, reverse=True)[:4]:
    lo, hi = t0 + at * 1e3 - g, t0 + at * 1e3
    calls = [(x.name, (x.time_range.end - x.time_range.start)) for x in rt if x.time_range.end >= lo and x.time_range.start <= hi]
    print(f"    gap @ {at:.3f} ms: " + ", ".join(f"{nm}({d:.0f}us)" for nm, d in calls[:12]))
