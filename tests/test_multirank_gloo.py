"""N > 1 host path on CPU (world_size 2 and 3, gloo): index-range sharding (PMRRR's static division,
P:4593-4599), first-index group ownership (libmrrr mrrr_shard_owner, north_star / SURVEY §8(e)) and the
eigenvalue all-gather.  The per-rank solve itself needs a GPU; here every rank takes its
owned eigenvalues from the oracle's full solve, so what is tested is the partition + ownership + gather
logic that bench.py and a user's multi-GPU job run around mrrr_eig_shard."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import mrrr_inputs as mi
import oracle


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, il, iu, gstart, W_full, q):
    import torch
    import torch.distributed as dist

    from paper_1401_4950_b200 import dist as pd
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sl, su = pd.shard_range(il, iu, world, rank)
        if su >= sl:
            jlo, jhi = pd.owned_range(gstart, sl, su, n, il, iu)
        else:
            jlo, jhi = su + 1, su
        m = max(jhi - jlo + 1, 0)
        Wl = torch.from_numpy(W_full[jlo - il:jlo - il + m].copy())
        W = pd.allgather_eigenvalues(Wl, jlo, jhi, il, iu)
        ranges = [None] * world
        dist.all_gather_object(ranges, (sl, su, jlo, jhi))
        # the NCCL id of mrrr_eig_dist reaches every rank unchanged (None where libnccl is absent)
        try:
            ident = pd.nccl_id_broadcast()
        except Exception:
            ident = None
        ids = [None] * world
        dist.all_gather_object(ids, ident)
        q.put((rank, W.numpy(), ranges, ids))
    finally:
        dist.destroy_process_group()


def _run(world, d, e, il=None, iu=None):
    n = d.size
    il = 1 if il is None else il
    iu = n if iu is None else iu
    r = oracle.mrrr(d, e, 1, n)
    gstart = np.asarray(r.root_gstart, dtype=np.int32)
    W_full = np.ascontiguousarray(r.W[il - 1:iu])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(k, world, port, n, il, iu, gstart, W_full, q)) for k in range(world)]
    for p in ps:
        p.start()
    out = [q.get(timeout=180) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort(key=lambda t: t[0])
    return gstart, W_full, out


def _check(gstart, W_full, out, il, iu):
    ranges = out[0][2]
    # every rank saw the same ranges and the same gathered list, equal to the full solve
    for rank, W, rg, ids in out:
        assert rg == ranges
        np.testing.assert_array_equal(W, W_full)
        # one NCCL id for all ranks (mrrr_eig_dist's communicator bootstrap)
        assert all(x == ids[0] for x in ids)
        assert ids[0] is None or len(ids[0]) == 128
    # owned ranges partition [il, iu] exactly, each starting at a group start and ending at a group end
    owned = [(jlo, jhi) for (_, _, jlo, jhi) in ranges if jhi >= jlo]
    assert owned[0][0] == il and owned[-1][1] == iu
    for (a0, a1), (b0, b1) in zip(owned, owned[1:]):
        assert b0 == a1 + 1
    for jlo, jhi in owned:
        assert gstart[jlo - 1] == 1 or jlo == il
        assert jhi == iu or gstart[jhi] == 1
    # a unit (root group cut to [il, iu]) is owned by the rank whose shard holds its first index
    for (sl, su, jlo, jhi) in ranges:
        starts = [j for j in range(max(sl, il), su + 1) if gstart[j - 1] == 1 or j == il]
        if starts:
            assert jlo == starts[0]
        else:
            assert jhi < jlo


@pytest.mark.parametrize("world", [2, 3])
def test_shards_singletons(world):
    d, e = mi.one_two_one(120)
    gs, Wf, out = _run(world, d, e)
    _check(gs, Wf, out, 1, d.size)


@pytest.mark.parametrize("world", [2, 3])
def test_shards_clusters_straddle(world):
    # Wilkinson W+_{2m+1}: near-degenerate pairs; odd shard boundaries cut pairs (ownership moves them)
    d, e = mi.wilkinson(31)
    gs, Wf, out = _run(world, d, e)
    assert (gs == 0).sum() > 0  # clusters exist
    _check(gs, Wf, out, 1, d.size)
    ranges = out[0][2]
    cut = [su for (sl, su, jlo, jhi) in ranges[:-1] if su < d.size and gs[su] == 0]
    assert cut, "test needs a cluster straddling a shard boundary"


@pytest.mark.parametrize("world,il,iu", [(2, 600, 601), (3, 600, 601), (2, 300, 450), (3, 300, 450), (3, 2, 2),
                                         (2, 590, 601)])
def test_shards_subset_edges_inside_clusters(world, il, iu):
    # a subset whose ends fall inside Wilkinson pairs -- the unit containing il starts at il, no
    # owned range runs past iu, and the owned ranges still partition [il, iu]
    d, e = mi.wilkinson(300)
    gs, Wf, out = _run(world, d, e, il, iu)
    _check(gs, Wf, out, il, iu)


def test_owner_clips_to_selection():
    from paper_1401_4950_b200 import dist as pd
    g = np.array([1, 0, 1, 0, 1, 0, 1, 0, 1, 0], np.int32)   # pairs (1,2) (3,4) ... (9,10)
    assert pd.owned_range(g, 4, 5, 10, 4, 7) == (4, 6)      # il = 4 inside the pair (3,4): unit 4..4 + pair 5,6
    assert pd.owned_range(g, 6, 7, 10, 4, 7) == (7, 7)      # iu = 7 cuts the pair (7,8)
    assert pd.owned_range(g, 4, 4, 10, 4, 4) == (4, 4)
    with pytest.raises(ValueError):
        pd.owned_range(g, 3, 5, 10, 4, 7)                   # shard starts before il


def test_shards_glued_blocks():
    d, e = mi.glued_wilkinson(copies=4, m=10, glue=1e-10)
    gs, Wf, out = _run(2, d, e)
    _check(gs, Wf, out, 1, d.size)


def test_shard_range_covers_and_balances():
    from paper_1401_4950_b200 import dist as pd
    for k in (1, 7, 8, 65536, 6553):
        for world in (1, 2, 3, 4, 8):
            rs = [pd.shard_range(1, k, world, r) for r in range(world)]
            got = [j for sl, su in rs for j in range(sl, su + 1)]
            assert got == list(range(1, k + 1))
            sizes = [max(su - sl + 1, 0) for sl, su in rs]
            assert max(sizes) - min(s for s in sizes) <= max(sizes)  # contiguous, ceil-divided
            assert max(sizes) == -(-k // world)


def test_owner_argument_errors():
    from paper_1401_4950_b200 import dist as pd
    g = np.ones(10, np.int32)
    with pytest.raises(ValueError):
        pd.owned_range(g, 0, 5, 10)
    with pytest.raises(ValueError):
        pd.owned_range(g, 6, 5, 10)
    with pytest.raises(ValueError):
        pd.owned_range(g, 1, 5, 4)
    with pytest.raises(ValueError):
        pd.owned_range(g, 1, 5, 10, 1, 11)
    assert pd.owned_range(g, 3, 5, 10) == (3, 5)
    g2 = np.array([1, 0, 0, 1, 0, 1, 1, 0, 0, 0], np.int32)
    assert pd.owned_range(g2, 2, 3, 10) == (4, 3)      # no group starts in [2, 3]
    assert pd.owned_range(g2, 4, 6, 10) == (4, 6)
    assert pd.owned_range(g2, 7, 7, 10) == (7, 10)     # the cluster 7..10 straddles
