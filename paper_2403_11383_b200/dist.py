"""torch.distributed plumbing for sample sharding over GPUs (one process per GPU).

The library shards the K samples of every robot by global sample index
(`shard_range`, the same formula as sbs_create in csrc/sbs_api.cpp) and combines
the ranks' records (MPPI, Naive or CEM) with one NCCL all-gather inside sbs_step; this module only
bootstraps the NCCL communicator (rank 0's ncclUniqueId broadcast over the
torch.distributed store) -- no method arithmetic here.
"""
from __future__ import annotations


def shard_range(K: int, rank: int, world: int) -> tuple[int, int]:
    """Global sample slice [k_begin, k_begin + K_local) owned by `rank`."""
    k_begin = K * rank // world
    return k_begin, K * (rank + 1) // world - k_begin


def bootstrap_nccl_id(rank: int, group=None) -> bytes:
    """Rank 0 draws an ncclUniqueId through the C ABI; every rank returns it."""
    import torch.distributed as dist

    from . import binding
    obj = [binding.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]
