python -c "
import sys, os; sys.path.insert(0,'.')
import torch, numpy as np, mrrr_inputs as mi, paper_1401_4950_b200 as m
for env in [{'MRRR_SEGCHILDMIN':'1'}, {'MRRR_SEGCHILDMIN':'1','MRRR_RQISEGW':'1536'}, {'MRRR_SEGCHILDMIN':'1','MRRR_RQISEGK':'2'}]:
    os.environ.update(env)
    c=mi.CONFIGS['C4']; d,e=c.matrix(); s=m.Solver()
    for _ in range(2): W,Z=s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), c.il, c.iu)
    torch.cuda.synchronize(); st=s.stats(); t=s.times()
    print(env, {k:st[k] for k in ['rqi_handover','ho_twist','ho_fixed','ho_rqc','seg_wide']}, round(t['total'],2), round(t['rqi_ms_per_launch'],2))
    s.close()
"
