"""Worker of tests/test_gpu_parity.py::test_eig_dist_two_ranks (launched by torch.distributed.run, one rank
per GPU): mrrr_eig_dist over a real NCCL communicator; every rank checks the gathered eigenvalue list and its
owned vectors against its own single-GPU solve of the same selection."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import mrrr_inputs as mi  # noqa: E402
import paper_1401_4950_b200 as m  # noqa: E402
from paper_1401_4950_b200 import dist as pd  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("gloo")
ident = pd.nccl_id_broadcast()
for (d, e), (il, iu) in [(mi.random_tridiag(3000, 5, -1.0), (1, 3000)), (mi.wilkinson(300), (300, 450)),
                         (mi.wilkinson(300), (590, 601))]:
    dt, et = torch.from_numpy(d).cuda(), torch.from_numpy(e).cuda()
    W0, Z0 = m.Solver().eig(dt, et, il, iu)
    jlo, jhi, W, Z = m.Solver().eig_dist(dt, et, il, iu, ident, rank, world)
    torch.cuda.synchronize()
    assert torch.equal(W.cpu(), W0.cpu())
    assert torch.equal(Z.cpu(), Z0[:, jlo - il:jhi - il + 1].cpu())
    spans = [None] * world
    dist.all_gather_object(spans, (jlo, jhi))
    got = [j for a, b in spans for j in range(a, b + 1)]
    assert got == list(range(il, iu + 1)), spans
print("DIST_OK", rank, flush=True)
dist.destroy_process_group()
