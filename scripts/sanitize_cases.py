import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import mrrr_inputs as mi, paper_1401_4950_b200 as m
cases = [(mi.random_tridiag(3000, 5, -1.0), [(1, 3000), (100, 400), (2901, 3000)]),
         (mi.wilkinson(300), [(1, 601), (300, 450), (590, 601)]),
         (mi.glued_wilkinson(8, 100, 1e-10), [(1, 1608), (100, 130), (1604, 1608)]),
         (mi.one_two_one(1500), [(1, 1500)]),
         (mi.random_tridiag(200, 7, -1.0), [(1, 200)])]
for (d, e), sels in cases:
    dt, et = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
    for il, iu in sels:
        s = m.Solver(keep_diag=True)
        W, Z = s.eig(dt, et, il, iu)
        torch.cuda.synchronize()
        s.diag()
        for P in (2, 3):
            from paper_1401_4950_b200 import dist as pd
            for r in range(P):
                sl, su = pd.shard_range(il, iu, P, r)
                if su >= sl:
                    s2 = m.Solver()
                    s2.eig_shard(dt, et, sl, su, il, iu)
                    s2.close()
        s.close()
print("SAN_DONE")
