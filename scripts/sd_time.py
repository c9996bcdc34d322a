import numpy as np, torch, sys
sys.path.insert(0, '.')
import mrrr_inputs as mi, paper_1401_4950_b200 as m
for cfg in ["C2", "C1", "C5b"]:
    c = mi.CONFIGS[cfg]; d, e = c.matrix()
    d32 = torch.from_numpy(d.astype(np.float32)).cuda(); e32 = torch.from_numpy(e.astype(np.float32)).cuda()
    s = m.Solver()
    k = c.iu - c.il + 1
    W = torch.empty(k, dtype=torch.float32, device='cuda'); Z = torch.empty((k, c.n), dtype=torch.float32, device='cuda')
    ts = []
    for r in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); a.record(); s.seig(d32, e32, c.il, c.iu, W=W, Z=Z); b.record(); torch.cuda.synchronize()
        if r >= 2: ts.append(a.elapsed_time(b))
    t = s.times(); st = s.stats()
    print(cfg, "sd ms", np.median(ts), "bis", round(t['root_bisection'],2), "sing", round(t['singletons'],2), "clu", round(t['clusters'],2), "ncl", st['n_clusters'], "ho", st['rqi_handover'], "rounds", st['rounds'], flush=True)
    s.close()
