"""Chain sharding across ranks.

A chain of submeshes is sequential, so the only parallel unit across GPUs is
the independent mesh (one chain each).  Each rank runs its contiguous slice of
the meshes through ``smg_run_chains`` with no data-path collective; afterwards
the per-mesh results (reconstructions, coefficients) are gathered to every rank
with one all-gather (NCCL over NVLink on the GPU box, gloo in the CPU tests).
The reference has no multi-process path: one call of
compute_block_bases_fixed_sizes (pipeline.hpp:144) carries one mesh, and a
batch of meshes is a serial sequence of such calls; ranks here split that
sequence.
"""
from __future__ import annotations

from typing import List, Sequence


def shard_meshes(total: int, world: int, rank: int) -> List[int]:
    """Contiguous, balanced mesh ids of ``rank``: the first ``total % world``
    ranks get one extra mesh.  Empty when ``total < world`` for the tail ranks."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError(f"invalid rank {rank} of world {world}")
    if total < 0:
        raise ValueError("negative mesh count")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    count = base + (1 if rank < extra else 0)
    return list(range(start, start + count))


def shard_counts(total: int, world: int) -> List[int]:
    return [len(shard_meshes(total, world, r)) for r in range(world)]


def gather_meshes(local, total: int, group=None):
    """All-gather per-mesh result rows to every rank, in global mesh order.

    ``local`` is a tensor of shape (len(shard_meshes(total, world, rank)), *row);
    the result has shape (total, *row).  Ragged shards are padded to the largest
    shard for the collective and trimmed afterwards.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    counts = shard_counts(total, world)
    if local.shape[0] != counts[rank]:
        raise ValueError(f"rank {rank} holds {local.shape[0]} meshes, shard has {counts[rank]}")
    width = max(counts) if counts else 0
    row = tuple(local.shape[1:])
    if local.shape[0] == width:
        padded = local.contiguous()
    else:
        padded = torch.zeros((width,) + row, dtype=local.dtype, device=local.device)
        padded[: local.shape[0]] = local
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def owner_of(mesh_id: int, total: int, world: int) -> int:
    """Rank that runs ``mesh_id``."""
    if not (0 <= mesh_id < total):
        raise ValueError("mesh id out of range")
    for r in range(world):
        ids = shard_meshes(total, world, r)
        if ids and ids[0] <= mesh_id <= ids[-1]:
            return r
    raise AssertionError("unreachable")


__all__: Sequence[str] = ("shard_meshes", "shard_counts", "gather_meshes", "owner_of")
