"""Time one rank's share of an N-GPU run on one GPU: eigenpairs of the r-th of N contiguous index shards
(the per-rank work of `bench.py --gpus N`; the all-gather is not included).

    python scripts/shard_time.py C2 8 [reps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402
from paper_1401_4950_b200 import dist as pd  # noqa: E402

cfg = mi.CONFIGS[sys.argv[1]]
N = int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
d, e = cfg.matrix()
s = m.Solver()
dt, et = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
worst = 0.0
for r in (0, N // 2, N - 1):
    sl, su = pd.shard_range(cfg.il, cfg.iu, N, r)
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        s.eig_shard(dt, et, sl, su, cfg.il, cfg.iu)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = min(ts[1:])
    worst = max(worst, t)
    print(f"{cfg.name} N={N} rank {r} [{sl},{su}]: {t:.3f} ms  {s.times()}", flush=True)
print(f"{cfg.name} N={N}: max over the sampled ranks {worst:.3f} ms")
