"""Run one warm-up and one profiled solve of a config (for ncu captures)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

cfg = mi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
d, e = cfg.matrix()
s = m.Solver()
dt, et = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
for _ in range(reps):
    W, Z = s.eig(dt, et, cfg.il, cfg.iu)
torch.cuda.synchronize()
print(cfg.name, s.times(), s.stats())
