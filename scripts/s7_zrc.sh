O=gpurun_out
python scripts/sweep_env.py C2 5 "MRRR_ZWIN=0" "" "MRRR_ZWIN=128" "MRRR_ZWIN=192" "MRRR_ZWIN=384" > $O/s7_sweep.log 2>&1
python scripts/sweep_env.py C5b 3 "MRRR_ZWIN=0" "" "MRRR_ZWIN=128" >> $O/s7_sweep.log 2>&1
python -c "
import sys; sys.path.insert(0,'.')
import os, torch, numpy as np, mrrr_inputs as mi, paper_1401_4950_b200 as m
for zw in ['128','256']:
  os.environ['MRRR_ZWIN']=zw
  for cfg in ['C2','C5b']:
    c=mi.CONFIGS[cfg]; d,e=c.matrix(); s=m.Solver()
    W,Z=s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), c.il, c.iu); torch.cuda.synchronize()
    st=s.stats(); print(zw, cfg, 'zwin_reruns', st['zwin_reruns'], 'handover', st['rqi_handover'], 'iters', st['rqi_iters']); s.close()
" >> $O/s7_sweep.log 2>&1
cat $O/s7_sweep.log
