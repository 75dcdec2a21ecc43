"""F1: segmentation on the GPU (smg_partition_mesh / smg_expand_overlaps /
smg_order_submeshes / smg_segment_mesh) bit-exact against the oracle's
restatement of partition.hpp:58-307 / pipeline.hpp:131-138 -- assignment,
member lists and order -- on C2, C3 and a C5 mesh at k in {8, 64}, the hand
traces of test_oracle_segmentation, and the reference's error texts; then
compute_block_bases without a Segmentation (the reference's own flow,
pipeline.hpp:198-201) equals the chain over the explicit segmentation."""
import time

import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_1810_02719_b200")

from test_oracle_segmentation import path_graph  # noqa: E402


def graph_mesh(offs, cols):
    n = len(offs) - 1
    return synth.Mesh(np.zeros((n, 3)), np.zeros((0, 3), np.int32), np.asarray(offs, np.int32),
                      np.asarray(cols, np.int32))


def test_partition_hand_traces(ctx):
    offs, cols = path_graph(8)
    assert G.partition_mesh(graph_mesh(offs, cols), 2, 1, ctx=ctx).tolist() == [0, 0, 0, 0, 1, 1, 1, 1]
    offs2 = np.concatenate([offs, offs[1:] + offs[-1]])
    cols2 = np.concatenate([cols, cols + 8])
    m2 = graph_mesh(offs2, cols2)
    assert G.partition_mesh(m2, 2, 1, ctx=ctx).tolist() == O.partition_mesh(offs2, cols2, 2, 1).assignment.tolist()
    chain = [np.arange(3 * i, 3 * i + 4) for i in range(5)]
    assert G.order_submeshes(chain, 3, ctx=ctx).tolist() == [2, 1, 3, 0, 4]
    assert G.order_submeshes([np.arange(4)], 7, ctx=ctx).tolist() == [0]
    p = O.Partition(np.asarray([0] * 5 + [1] * 5, np.int32), 2)
    o10, c10 = path_graph(10)
    mem = G.expand_overlaps(graph_mesh(o10, c10), p.assignment, 2, 1.5, ctx=ctx)
    assert [m.tolist() for m in mem] == [list(range(7)), list(range(3, 10))]


def test_segmentation_errors(ctx):
    offs, cols = path_graph(8)
    m = graph_mesh(offs, cols)
    with pytest.raises(G.InvalidArgument, match=r"part count k must satisfy 1 <= k <= n/4"):
        G.partition_mesh(m, 3, 1, ctx=ctx)
    o3 = np.concatenate([offs, offs[1:] + offs[-1], offs[1:] + 2 * offs[-1]])
    c3 = np.concatenate([cols, cols + 8, cols + 16])
    with pytest.raises(G.InvalidArgument, match=r"partition failed: k is incompatible with the mesh connectivity"):
        G.partition_mesh(graph_mesh(o3, c3), 2, 1, ctx=ctx)
    with pytest.raises(G.InvalidArgument, match=r"overlap growth must be >= 1.0"):
        G.expand_overlaps(m, np.asarray([0] * 4 + [1] * 4), 2, 0.5, ctx=ctx)
    with pytest.raises(G.InvalidArgument, match=r"partition has an empty part"):
        G.expand_overlaps(m, np.zeros(8, np.int32), 2, 1.0, ctx=ctx)


CASES = [("C2", 8), ("C2", 64), ("C3", 8), ("C3", 64), ("C5", 8), ("C5", 64)]


@pytest.mark.parametrize("name,k", CASES)
def test_segment_mesh_bit_exact(ctx, name, k):
    w = synth.config(name)
    seed = 17
    t0 = time.perf_counter()
    seg, a = G.segment_mesh(w.mesh, k, 1.15, seed, ctx=ctx, return_assignment=True)
    t_gpu = time.perf_counter() - t0
    part, members, seq = O.segment_mesh(w.mesh.adj_offsets, w.mesh.adj_cols, k, 1.15, seed)
    assert np.array_equal(a, part.assignment)
    assert len(seg.members) == len(members)
    for gm, om in zip(seg.members, members):
        assert np.array_equal(gm, om)
    assert np.array_equal(seg.sequence, seq)
    print(f"{name} k={k}: n_d={seg.block_size}, GPU segment_mesh {t_gpu * 1e3:.1f} ms")


def test_compute_block_bases_segments_itself(ctx):
    """compute_block_bases(mesh, cfg) with no Segmentation runs segment_mesh on
    the GPU first (pipeline.hpp:198-201): same results as the explicit path."""
    mesh = synth.small_grid(96, 64, 32, 32, seed=5, flip=4)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=40, iterations=1, shift_scale=1e-3, part_count=6,
                           growth=1.15, seed=4)
    a = G.compute_block_bases(mesh, None, cfg, ctx=ctx)
    seg = G.segment_mesh(mesh, 6, 1.15, 4, ctx=ctx)
    b = G.compute_block_bases(mesh, seg, cfg, ctx=ctx)
    assert np.array_equal(a.sequence, seg.sequence) and a.block_size == seg.block_size
    assert np.array_equal(a.reconstruction, b.reconstruction)
    for i in range(6):
        assert a.stats[i] == b.stats[i]
        assert np.array_equal(a.coefficients[i], b.coefficients[i])
    # and the chain over it matches the oracle's chain over the oracle's segmentation
    part, members, seq = O.segment_mesh(mesh.adj_offsets, mesh.adj_cols, 6, 1.15, 4)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, members)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=40, iterations=1, shift_scale=1e-3)
    ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seq, ocfg, [40] * 6)
    rec = O.coarse_reconstruct_points(ob, mesh.vertices)
    assert np.linalg.norm(a.reconstruction - rec, axis=1).max() <= 1e-9 * np.linalg.norm(rec, axis=1).max()
