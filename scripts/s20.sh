O=gpurun_out
python -c "
import sys; sys.path.insert(0,'.')
import torch, mrrr_inputs as mi, paper_1401_4950_b200 as m
for cfg in ['C3','C4']:
    c=mi.CONFIGS[cfg]; d,e=c.matrix(); s=m.Solver()
    W,Z=s.eig(torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda(), c.il, c.iu); torch.cuda.synchronize()
    st=s.stats(); print(cfg, {k:st[k] for k in ['zwin_reruns','rqi_handover','rqi_iters','seg_wide']}); s.close()
"
timeout 1700 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_support.py tests/test_gpu_families.py -q -x > $O/s20_tests.log 2>&1; echo "tests rc=$?"; tail -3 $O/s20_tests.log
