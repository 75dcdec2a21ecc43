"""N>1 host path on CPU: mesh sharding + the all-gather of per-mesh results,
world_size 2 over gloo (the GPU box uses NCCL for the same calls; bench.py).

Each rank runs the oracle chain (test infrastructure, the checker) on its own
meshes and the gathered reconstructions must equal a single-process run.
"""
import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from paper_1810_02719_b200 import shard, synth  # noqa: E402


def test_shard_partition_properties():
    for total in range(0, 20):
        for world in range(1, 9):
            ids = [shard.shard_meshes(total, world, r) for r in range(world)]
            flat = [i for part in ids for i in part]
            assert flat == list(range(total))
            sizes = [len(p) for p in ids]
            assert max(sizes) - min(sizes) <= 1
            for r, part in enumerate(ids):
                for i in part:
                    assert shard.owner_of(i, total, world) == r
    with pytest.raises(ValueError):
        shard.shard_meshes(4, 2, 2)
    with pytest.raises(ValueError):
        shard.owner_of(5, 5, 2)


def _recon(mesh_id):
    import specmesh_oracle as O
    W = H = 16
    base = synth.grid_mesh(W, H, 900 + mesh_id, 0.01)
    seg = synth.grid_tiles(W, H, 8, 8)
    subs = O.build_submeshes(base.adj_offsets, base.adj_cols, seg.members)
    cfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=10, iterations=1, shift_scale=1e-3)
    bb = O.compute_block_bases_fixed_sizes(base.vertices, subs, np.arange(len(subs)), cfg, [10] * len(subs))
    return O.coarse_reconstruct_points(bb, base.vertices).reshape(-1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, total, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ids = shard.shard_meshes(total, world, rank)
        rows = [_recon(i) for i in ids]
        width = 3 * 16 * 16
        local = torch.from_numpy(np.stack(rows)) if rows else torch.zeros((0, width), dtype=torch.float64)
        out = shard.gather_meshes(local, total)
        q.put((rank, out.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("total", [2, 3])
def test_gather_matches_single_process(total):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = np.stack([_recon(i) for i in range(total)])
    for r in range(2):
        assert got[r].shape == expect.shape
        np.testing.assert_array_equal(got[r], expect)


def test_library_shard_range_matches():
    """smg_shard_range (the C++ host's sharding, include/specmesh_gpu.h) gives the
    same slices as shard.shard_meshes -- host-only, no GPU needed."""
    import ctypes as C
    from paper_1810_02719_b200 import _abi
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("libspecmesh_b200.so not built")
    lib = _abi.load()
    f, c = C.c_int32(), C.c_int32()
    for total in range(0, 70):
        for world in range(1, 9):
            for r in range(world):
                assert lib.smg_shard_range(total, world, r, C.byref(f), C.byref(c)) == 0
                assert list(range(f.value, f.value + c.value)) == shard.shard_meshes(total, world, r)
    assert lib.smg_shard_range(4, 2, 2, C.byref(f), C.byref(c)) == 2
