"""One solve of a configuration for ncu launch lists: `python scripts/sd_once.py C3` (double/dd, mrrr_eig) or
`python scripts/sd_once.py sd:C2` (single/double, mrrr_seig on the binary32 copy of the matrix)."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "sd:C2"
sd = name.startswith("sd:")
c = mi.CONFIGS[name[3:] if sd else name]
d, e = c.matrix()
dt = np.float32 if sd else np.float64
d_, e_ = torch.from_numpy(d.astype(dt)).cuda(), torch.from_numpy(e.astype(dt)).cuda()
s = m.Solver()
(s.seig if sd else s.eig)(d_, e_, c.il, c.iu)
torch.cuda.synchronize()
print(s.times(), s.stats())
