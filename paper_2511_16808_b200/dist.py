"""Process-group plumbing for the slab-partitioned solve.

torch.distributed is used only to bootstrap: rank 0 draws the NCCL unique id
through the C-ABI (hmg_comm_nccl_unique_id) and broadcasts it; every rank then
opens its own libhmg communicator (hmg_comm_nccl).  All data-path collectives
(halos, dot-product allreduce, coarse allgather) run inside libhmg.
"""
from __future__ import annotations

import os

import numpy as np


def env_ranks():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def share_unique_id(make_id, group=None):
    """Rank 0 calls ``make_id()`` (128 bytes); the id is broadcast to every rank."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    buf = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid = make_id()
        assert len(uid) == 128
        buf = torch.frombuffer(bytearray(uid), dtype=torch.uint8).clone()
    backend = dist.get_backend(group)
    if backend == "nccl":
        buf = buf.cuda()
    dist.broadcast(buf, src=0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def nccl_comm(group=None):
    """libhmg NCCL communicator of this process (torch.distributed must be initialised)."""
    import torch.distributed as dist
    from . import hmg
    uid = share_unique_id(hmg.Comm.nccl_unique_id, group)
    return hmg.Comm.nccl(uid, dist.get_rank(group), dist.get_world_size(group))


def max_over_ranks(value, group=None, device=None):
    """Max of a float over the ranks (timing: the job is as slow as its slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def slab_rows(nodes_slab_axis, levels, nranks, rank, level=0, ghost=4):
    """This rank's global rows on ``level`` under hmg_slab_partition's rule."""
    from . import hmg
    lo, hi, dist = hmg.slab_partition(nodes_slab_axis, levels, nranks, ghost)
    if not dist[level]:
        return 0, int(hi[level, -1])
    return int(lo[level, rank]), int(hi[level, rank])


def split_rows(array, lo, hi, dim):
    """Rows [lo, hi) of the slab axis of a field shaped nodes[::-1] (z, y, x) / (y, x)."""
    a = np.asarray(array)
    return np.ascontiguousarray(a[lo:hi])
