"""Host-side multi-rank plumbing (one process per GPU, torch.distributed).

Only bookkeeping lives here: which z-planes a rank owns, the NCCL unique-id
bootstrap for libsten's communicator, and max-over-ranks timing.  All data
movement of a solve (halo planes, scalar all-reduce) happens inside libsten.so.
"""
from __future__ import annotations

import os


def rank_env():
    """(rank, world_size, local_rank) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def slab_of(rank: int, world: int, nz_global: int):
    """z-slab decomposition: rank r owns planes [r*nz/G, (r+1)*nz/G),
    rank order = z order.  Returns (z0, nz_local)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    if nz_global % world:
        raise ValueError(f"nz_global={nz_global} not divisible by {world} ranks")
    nzl = nz_global // world
    return rank * nzl, nzl


def neighbours(rank: int, world: int):
    """(rank below in z or None, rank above in z or None)."""
    return (rank - 1 if rank > 0 else None), (rank + 1 if rank + 1 < world else None)


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string from `src` over the default process group."""
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def bootstrap_comm(sten_module, rank: int, world: int):
    """NCCL communicator of libsten: rank 0 draws the unique id, everyone receives it
    over torch.distributed, then each rank joins (sten_comm_create)."""
    uid = broadcast_bytes(sten_module.comm_unique_id() if rank == 0 else None)
    return sten_module.comm_create(uid, world, rank)


def max_over_ranks(value: float, device=None) -> float:
    """All-reduce MAX of a per-rank time (the bench reports the slowest rank)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())
