"""Multi-rank host plumbing around spamm_multiply_mgpu (Sec. 3.4).

One process per GPU.  torch.distributed carries only host-side coordination (the NCCL
unique id, work vectors for the partitioner when a caller wants them, timing maxima);
the data path (input broadcast, norm-map all-gather, row-work all-reduce, C all-gather)
runs inside libspamm.so over NCCL.  All functions here are argument marshalling around
the C ABI; they work with any torch.distributed backend (gloo for CPU tests).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import spamm as sp


def nccl_comm(rank: int, world: int, group=None):
    """Create the library's NCCL communicator: rank 0 draws the unique id
    (spamm_nccl_unique_id), torch.distributed broadcasts it, every rank joins."""
    uid = [sp.spamm_nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0, group=group)
    return sp.spamm_nccl_comm_init(world, rank, uid[0])


def agree_unique_id(rank: int, world: int, group=None) -> bytes:
    """The 128-byte id every rank would pass to spamm_nccl_comm_init (no device needed)."""
    uid = [sp.spamm_nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0, group=group)
    return uid[0]


def balanced_cuts(local_row_work, nranks: int, group=None) -> list[int]:
    """Sum each rank's partial row-work vector (zeros outside its provisional rows) over
    the group and cut rows with spamm_partition_rows (Sec. 3.5.1 balance applied to the
    Sec. 3.4 row partition).  Every rank returns the identical cut list."""
    w = torch.as_tensor(local_row_work, dtype=torch.int64).clone()
    if nranks > 1:
        dist.all_reduce(w, op=dist.ReduceOp.SUM, group=group)
    return sp.spamm_partition_rows(w.tolist(), nranks)


def provisional_rows(n_rows: int, rank: int, nranks: int) -> tuple[int, int]:
    """Even split used before work counts exist (the paper's split)."""
    return n_rows * rank // nranks, n_rows * (rank + 1) // nranks


def max_over_ranks(x: float, group=None, device=None) -> float:
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
