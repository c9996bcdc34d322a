"""Kernel sequence of one solve (torch.profiler / CUPTI): start offset, duration and name of every device
activity, for reading a round structure by eye.

    python scripts/kseq.py C2 [sd] [es]     (es: MRRR_EARLY_STOP)
"""
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
sd = "sd" in sys.argv[2:]
es = "es" in sys.argv[2:]
c = mi.CONFIGS[name]
d, e = c.matrix()
dt = np.float32 if sd else np.float64
d_, e_ = torch.from_numpy(d.astype(dt)).cuda(), torch.from_numpy(e.astype(dt)).cuda()
s = m.Solver(early_stop=es)
f = s.seig if sd else s.eig
W = torch.empty(c.k, dtype=d_.dtype, device="cuda")
Z = torch.empty((c.k, c.n), dtype=d_.dtype, device="cuda")
for _ in range(3):
    f(d_, e_, c.il, c.iu, W=W, Z=Z)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    f(d_, e_, c.il, c.iu, W=W, Z=Z)
    torch.cuda.synchronize()
ev = sorted([x for x in prof.events() if x.device_type.name == "CUDA"], key=lambda x: x.time_range.start)
t0 = ev[0].time_range.start
for x in ev:
    print(f"{(x.time_range.start - t0) / 1e3:9.3f} {(x.time_range.end - x.time_range.start):9.1f}  {x.name[:90]}")
print(name, s.times(), s.stats())
