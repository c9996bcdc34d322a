"""Multi-GPU plumbing of the MRRR hot path: one process per GPU, index-range shards.

The division follows PMRRR's static contiguous division of the k wanted indices (P:4593-4599,
P:4614-4615): rank p gets [il + p*ceil(k/P), il + (p+1)*ceil(k/P) - 1] ∩ [il, iu].  Every rank builds the
same root representation (bit-identical by construction) and bisects its shard plus guards; the rank
whose shard holds the FIRST index of a group (singleton or cluster) owns the whole group
(``mrrr_shard_owner`` in libmrrr, north_star), so no representation or interval crosses a process
boundary.  The only collective is the final gather of the eigenvalue list (P:4619-4621 gathers all
eigenvalues; here over NCCL on NVLink, or gloo in the CPU tests); Z stays column-sharded.

Everything here is host logic (argument marshalling and a torch.distributed collective); the solve
itself runs in libmrrr's kernels via :meth:`Solver.eig_shard`.
"""
from __future__ import annotations

import ctypes as C

import numpy as np


def shard_range(il: int, iu: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [sl, su] (1-based, inclusive) of [il, iu] for ``rank`` of ``world``; su < sl if
    the rank gets nothing (k < world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    k = iu - il + 1
    per = -(-k // world)
    sl = il + rank * per
    su = min(il + (rank + 1) * per - 1, iu)
    return sl, su


def owned_range(gstart: np.ndarray, sl: int, su: int, jmax: int, il: int = 1, iu: int | None = None) -> tuple[int, int]:
    """Owned index range of a shard [sl, su] of the selection [il, iu] under the first-index ownership rule
    (libmrrr mrrr_shard_owner, a host-only C ABI call).  ``gstart[j-1]`` is 1 iff index j starts a root
    group; units are root groups cut to [il, iu]."""
    from . import load
    g = np.ascontiguousarray(gstart, dtype=np.int32)
    iu = g.size if iu is None else iu
    jlo, jhi = C.c_int64(), C.c_int64()
    rc = load().mrrr_shard_owner(g.ctypes.data, g.size, il, iu, sl, su, jmax, C.byref(jlo), C.byref(jhi))
    if rc != 0:
        raise ValueError(f"mrrr_shard_owner failed with code {rc}")
    return jlo.value, jhi.value


def allgather_eigenvalues(W_local, jlo: int, jhi: int, il: int, iu: int, group=None):
    """Gather every rank's owned eigenvalues W[jlo..jhi] into the full list W[il..iu] on every rank.
    ``W_local`` is a float64 tensor on the process group's device (CUDA for NCCL, CPU for gloo).
    Returns the full tensor (length iu - il + 1)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    dev = W_local.device
    m = max(jhi - jlo + 1, 0)
    meta = torch.tensor([jlo, m], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    cap = max(int(x[1]) for x in metas)
    buf = torch.zeros(max(cap, 1), dtype=torch.float64, device=dev)
    if m:
        buf[:m] = W_local[:m]
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    W = torch.full((iu - il + 1,), float("nan"), dtype=torch.float64, device=dev)
    for x, p in zip(metas, parts):
        lo, cnt = int(x[0]), int(x[1])
        if cnt:
            W[lo - il:lo - il + cnt] = p[:cnt]
    return W


def nccl_id_broadcast(group=None) -> bytes:
    """The 128-byte NCCL id of :meth:`Solver.eig_dist`: created on rank 0 (libmrrr, run-time-loaded
    libnccl) and sent to every rank over the torch.distributed group (any backend)."""
    import torch.distributed as dist
    from . import nccl_unique_id
    box = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]
