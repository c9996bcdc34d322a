timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np, mrrr_inputs as mi, paper_1401_4950_b200 as m, oracle, time
d,e=mi.wilkinson(2048)
s=m.Solver(keep_diag=True)
W,Z=s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()); torch.cuda.synchronize()
r=oracle.mrrr(d,e); g=s.diag()
mm=np.flatnonzero(~((g.fin_lo==r.fin_lo)&(g.fin_hi==r.fin_hi)))
print('mismatch', len(mm), mm[:10], g.depth[mm[:10]], (g.fin_hi-g.fin_lo)[mm[:5]], (g.fin_lo-r.fin_lo)[mm[:5]])
"
cp scripts/libmrrr_prev.so paper_1401_4950_b200/libmrrr.so
echo prev:
timeout 200 python -c "
import sys; sys.path.insert(0,'.')
import torch, numpy as np, mrrr_inputs as mi, paper_1401_4950_b200 as m, oracle, time
d,e=mi.wilkinson(2048)
s=m.Solver(keep_diag=True)
W,Z=s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()); torch.cuda.synchronize()
r=oracle.mrrr(d,e); g=s.diag()
mm=np.flatnonzero(~((g.fin_lo==r.fin_lo)&(g.fin_hi==r.fin_hi)))
print('mismatch', len(mm), mm[:10])
"
