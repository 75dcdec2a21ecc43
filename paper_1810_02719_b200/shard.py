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


class LibComm:
    """The library's own NCCL communicator (smg_comm_create): rank 0 makes the
    unique id (smg_comm_unique_id), the caller's process group broadcasts it,
    and smg_gather_meshes all-gathers per-mesh rows on the context stream --
    the C++ host path a reference-side caller (C++ / MPI) would use directly."""

    def __init__(self, ctx, world: int, rank: int, broadcast=None):
        import ctypes as C
        import numpy as np
        self.ctx, self.world, self.rank = ctx, world, rank
        uid = np.zeros(128, np.uint8)
        if rank == 0:
            ctx.check(ctx.lib.smg_comm_unique_id(ctx.handle, uid.ctypes.data))
        if world > 1:
            if broadcast is None:
                raise ValueError("world > 1 needs a broadcast of the unique id")
            uid = broadcast(uid)
        self.handle = C.c_void_p()
        ctx.check(ctx.lib.smg_comm_create(ctx.handle, uid.ctypes.data, world, rank, C.byref(self.handle)))

    def gather(self, local, out, total: int, row_doubles: int) -> None:
        """device pointers (ints) or objects with data_ptr()"""
        lp = local.data_ptr() if hasattr(local, "data_ptr") else local
        op = out.data_ptr() if hasattr(out, "data_ptr") else out
        self.ctx.check(self.ctx.lib.smg_gather_meshes(self.ctx.handle, self.handle, int(total), int(row_doubles),
                                                      lp, op))

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.ctx.lib.smg_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def torch_broadcast(uid):
    """broadcast a uint8 numpy array from rank 0 over the default process group"""
    import numpy as np
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.from_numpy(uid.copy()).to(dev)
    dist.broadcast(t, 0)
    return np.ascontiguousarray(t.cpu().numpy())


__all__: Sequence[str] = ("shard_meshes", "shard_counts", "gather_meshes", "owner_of", "LibComm", "torch_broadcast")
