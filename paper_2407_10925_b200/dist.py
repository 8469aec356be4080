"""Process-sharded runs (one process per GPU, launched by torchrun): the binary two-array half
table split over the WORLD_SIZE processes.

The library builds its own NCCL communicator from one ncclUniqueId; this module only creates the
id on rank 0 and broadcasts it through the torch process group (any backend), then creates the
handle collectively.  Every rank must call the handle's methods collectively.
"""
from __future__ import annotations

from .lcsb import Lcsb, lcsb_nccl_unique_id


def broadcast_id(raw: bytes | None, group=None) -> bytes:
    """Rank 0's bytes on every rank (torch.distributed.broadcast_object_list)."""
    import torch.distributed as dist
    obj = [raw if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def create_sharded(ell: int, dtype: str = "f32", rmode: str = "max", group=None,
                   stream=None) -> Lcsb:
    """Collective: every rank of the (torch) process group gets one shard of the sigma = d = 2
    two-array table of length-ell strings."""
    import torch.distributed as dist
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    nid = broadcast_id(lcsb_nccl_unique_id() if rank == 0 else None, group)
    return Lcsb(2, 2, ell, dtype=dtype, form="two_array", rmode=rmode, shards=ws, shard=rank,
                nccl_id=nid, stream=stream, torch_allocator=False)
