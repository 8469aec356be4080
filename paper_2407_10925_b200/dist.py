"""Process-sharded runs (one process per GPU, launched by torchrun): the binary two-array half
table split over the WORLD_SIZE processes.

Two transports for the library's three collectives (IPC-handle exchange at create, the per-sweep
barrier, the bound's scalar reductions):

* ``"nccl"``: the library builds its own NCCL communicator from one ncclUniqueId (created on rank
  0, broadcast here through the torch process group); barrier and reductions are NCCL
  all-reduces enqueued on the stream (asynchronous sweeps).  One GPU per rank.
* ``"host"``: the library calls back into :func:`comm_hooks` -- host collectives of the torch
  process group (gloo).  Each sweep ends with a stream synchronise and a host barrier, so no
  kernel ever waits on another rank: several ranks may share one GPU (the multi-process test on
  the single-GPU box, tests/test_multiprocess.py).

Every rank must call the handle's methods collectively.
"""
from __future__ import annotations

import ctypes

import numpy as np

from .lcsb import (ALLGATHER_FN, ALLREDUCE_FN, BARRIER_FN, Lcsb, LcsbCommHooks,
                   lcsb_nccl_unique_id)

_SIGN = np.uint64(1 << 63)


def broadcast_id(raw: bytes | None, group=None) -> bytes:
    """Rank 0's bytes on every rank (torch.distributed.broadcast_object_list)."""
    import torch.distributed as dist
    obj = [raw if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def allgather_bytes(mine: bytes, group=None) -> bytes:
    """Every rank's bytes (all the same length), concatenated in rank order."""
    import torch
    import torch.distributed as dist
    t = torch.frombuffer(bytearray(mine), dtype=torch.uint8)
    out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, t, group=group)
    return b"".join(bytes(o.numpy().tobytes()) for o in out)


def allreduce_max_u64(vals, group=None) -> np.ndarray:
    """Element-wise max over the ranks of unsigned 64-bit values (as int64 with the sign bit
    flipped, which preserves the order)."""
    import torch
    import torch.distributed as dist
    v = np.ascontiguousarray(vals, dtype=np.uint64) ^ _SIGN
    t = torch.from_numpy(v.view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.numpy().view(np.uint64) ^ _SIGN


def comm_hooks(group=None) -> LcsbCommHooks:
    """lcsb_comm_hooks over the torch process group (host collectives; gloo)."""
    import torch.distributed as dist

    def _allgather(mine, all_, nbytes, ctx):
        try:
            data = allgather_bytes(ctypes.string_at(mine, nbytes), group)
            ctypes.memmove(all_, data, len(data))
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed collective
            return 1

    def _barrier(ctx):
        try:
            dist.barrier(group=group)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    def _allreduce(vals, n, ctx):
        try:
            arr = np.ctypeslib.as_array(vals, shape=(n,))
            arr[:] = allreduce_max_u64(arr.copy(), group)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    h = LcsbCommHooks()
    h.allgather = ALLGATHER_FN(_allgather)
    h.barrier = BARRIER_FN(_barrier)
    h.allreduce_max_u64 = ALLREDUCE_FN(_allreduce)
    h.ctx = None
    h._keep = (h.allgather, h.barrier, h.allreduce_max_u64)  # the callbacks outlive the handle
    return h


def create_sharded(ell: int, dtype: str = "f32", rmode: str = "max", group=None,
                   stream=None, transport: str = "nccl", sigma: int = 2,
                   form: str = "auto", symmetry: int = -1, block_log4: int = 0,
                   offset_policy: int = 0) -> Lcsb:
    """Collective: every rank of the (torch) process group gets one shard of the d = 2 table of
    length-ell strings: sigma = 2 -- the symmetry-folded quarter table for l >= 12 (DESIGN.md
    §9c; the same kernels as one GPU) or the complement-folded half table (§9; symmetry = 1,
    and below l = 12); sigma = 4 -- the complement-folded q4 table, KS or two-array form
    (§9b).  offset_policy = 1: integer offsets (readings R23, R26; quarter table and sigma = 4;
    the min crosses the ranks before every sweep)."""
    import torch.distributed as dist
    if sigma not in (2, 4):
        raise ValueError("sharded tables exist for sigma = 2 and sigma = 4 (d = 2)")
    if sigma == 2:
        form = "two_array"
    ws = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if transport == "host":
        return Lcsb(sigma, 2, ell, dtype=dtype, form=form, rmode=rmode, shards=ws,
                    shard=rank, comm_hooks=comm_hooks(group), stream=stream,
                    torch_allocator=False, symmetry=symmetry, block_log4=block_log4,
                    offset_policy=offset_policy)
    if transport != "nccl":
        raise ValueError("transport must be 'nccl' or 'host'")
    nid = broadcast_id(lcsb_nccl_unique_id() if rank == 0 else None, group)
    return Lcsb(sigma, 2, ell, dtype=dtype, form=form, rmode=rmode, shards=ws, shard=rank,
                nccl_id=nid, stream=stream, torch_allocator=False, symmetry=symmetry,
                block_log4=block_log4, offset_policy=offset_policy)
