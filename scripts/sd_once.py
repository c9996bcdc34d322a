"""One single/double solve of a configuration (binary32 copy of its matrix) -- for ncu launch lists."""
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402

c = mi.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
d, e = c.matrix()
d32 = torch.from_numpy(d.astype(np.float32)).cuda()
e32 = torch.from_numpy(e.astype(np.float32)).cuda()
s = m.Solver()
s.seig(d32, e32, c.il, c.iu)
torch.cuda.synchronize()
print(s.times(), s.stats())
