"""GPU parity of the dynamic-mesh path (F3): denoise_dynamic (denoise.hpp:258-291)
and the batched frames stage coarse_reconstruct_points(frame, bases, mode)
(pipeline.hpp:300-305) against the CPU oracle on seeded frame sequences."""
import os

import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_1810_02719_b200")


def rel_err(a, b):
    return np.linalg.norm(a - b, axis=1).max() / np.linalg.norm(b, axis=1).max()


def sequence(W, H, frames, seed, flip=None):
    topo = synth.small_grid(W, H, 32, 32, seed=seed, flip=flip)
    verts = synth.grid_sequence(W, H, frames, seed, 0.01)
    return topo, [synth.Mesh(v, topo.faces, topo.adj_offsets, topo.adj_cols) for v in verts]


def overlapping_tiles(W, H, tw, step):
    """tw x H column strips starting every `step` columns: neighbouring strips
    overlap, so vertices have 2 owners with different local degrees."""
    members = []
    for x0 in range(0, W - tw + 1, step):
        xs = np.arange(x0, x0 + tw)
        ys = np.arange(H)
        members.append(np.sort((ys[:, None] * W + xs[None, :]).ravel()).astype(np.int32))
    return synth.Segmentation(members, np.arange(len(members), dtype=np.int32))


@pytest.mark.parametrize("mode", ["weighted", "simple"])
def test_denoise_dynamic_matches_oracle(ctx, mode):
    topo, frames = sequence(64, 64, 5, seed=11, flip=3)
    seg = synth.grid_tiles(64, 64, 32, 32)
    c = 40
    cfg = G.PipelineConfig(weighting="binary", subspace_size=c, iterations=1, shift_scale=1e-3)
    res = G.denoise_dynamic(frames, seg, cfg, [c] * seg.count, mode=mode, ctx=ctx)
    subs = O.build_submeshes(topo.adj_offsets, topo.adj_cols, seg.members)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=c, iterations=1, shift_scale=1e-3)
    ref, nb, _ = O.denoise_dynamic([f.vertices for f in frames], subs, seg.sequence, ocfg, [c] * seg.count,
                                   weighted=mode == "weighted")
    assert res.basis_blocks_computed == nb == seg.count
    assert len(res.frames) == len(frames)
    for got, want in zip(res.frames, ref):
        assert rel_err(got, want) < 1e-9
    assert res.timings["shared_basis"] > 0 and res.timings["frames"] > 0


@pytest.mark.parametrize("mode", ["weighted", "simple"])
def test_frames_stage_overlapping_blocks(ctx, mode):
    """Same bases on both sides (the oracle's): only the GEMM rounding differs.
    Overlapping strips make the degree weighting and the id-ordered sum matter."""
    topo, frames = sequence(96, 32, 3, seed=5, flip=9)
    seg = overlapping_tiles(96, 32, 32, 16)
    subs = O.build_submeshes(topo.adj_offsets, topo.adj_cols, seg.members)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=30, iterations=1, shift_scale=1e-3)
    ob = O.compute_block_bases_fixed_sizes(frames[0].vertices, subs, seg.sequence, ocfg, [30] * seg.count)
    bb = G.BlockBases(seg.sequence, [], ob.bases, None, None, {}, seg.block_size)
    got = G.coarse_reconstruct_frames(topo, seg, bb, [f.vertices for f in frames], mode=mode, ctx=ctx)
    for g, f in zip(got, frames):
        want = O.coarse_reconstruct_points(ob, f.vertices, weighted=mode == "weighted")
        assert rel_err(g, want) < 1e-12
    # weighted and simple differ on the shared columns
    other = G.coarse_reconstruct_frames(topo, seg, bb, [frames[0].vertices],
                                        mode="simple" if mode == "weighted" else "weighted", ctx=ctx)[0]
    assert np.abs(other - got[0]).max() > 0


def test_frames_stage_variable_sizes_and_batches(ctx, monkeypatch):
    """Per-block c (non-uniform basis offsets) and several frame batches (the
    last one partial)."""
    topo, frames = sequence(64, 64, 5, seed=21)
    seg = synth.grid_tiles(64, 64, 32, 32)
    sizes = [24, 40, 31, 16]
    subs = O.build_submeshes(topo.adj_offsets, topo.adj_cols, seg.members)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=24, iterations=1, shift_scale=1e-3)
    ob = O.compute_block_bases_fixed_sizes(frames[0].vertices, subs, seg.sequence, ocfg, sizes)
    bb = G.BlockBases(seg.sequence, [], ob.bases, None, None, {}, seg.block_size)
    monkeypatch.setenv("SMG_FRAMES_BATCH", "2")
    got = G.coarse_reconstruct_frames(topo, seg, bb, [f.vertices for f in frames], ctx=ctx)
    for g, f in zip(got, frames):
        assert rel_err(g, O.coarse_reconstruct_points(ob, f.vertices)) < 1e-12


def test_denoise_dynamic_variable_sizes(ctx):
    topo, frames = sequence(64, 64, 3, seed=8, flip=1)
    seg = synth.grid_tiles(64, 64, 32, 32)
    sizes = [30, 36, 30, 24]
    cfg = G.PipelineConfig(weighting="binary", subspace_size=30, iterations=1, shift_scale=1e-3)
    res = G.denoise_dynamic(frames, seg, cfg, sizes, ctx=ctx)
    subs = O.build_submeshes(topo.adj_offsets, topo.adj_cols, seg.members)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=30, iterations=1, shift_scale=1e-3)
    ref, _, _ = O.denoise_dynamic([f.vertices for f in frames], subs, seg.sequence, ocfg, sizes)
    for got, want in zip(res.frames, ref):
        assert rel_err(got, want) < 1e-9


def test_denoise_dynamic_connectivity_mismatch(ctx):
    topo, frames = sequence(64, 64, 2, seed=3)
    flipped = synth.small_grid(64, 64, 32, 32, seed=3, flip=4)
    frames[1] = synth.Mesh(frames[1].vertices, flipped.faces, flipped.adj_offsets, flipped.adj_cols)
    seg = synth.grid_tiles(64, 64, 32, 32)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=20, iterations=1, shift_scale=1e-3)
    with pytest.raises(G.InvalidArgument, match="frame 1 does not share the sequence connectivity"):
        G.denoise_dynamic(frames, seg, cfg, [20] * seg.count, ctx=ctx)


def test_frames_stage_uncovered_vertices(ctx):
    topo, frames = sequence(64, 64, 1, seed=3)
    seg = synth.grid_tiles(64, 64, 32, 32)
    part = synth.Segmentation(seg.members[:3], np.arange(3, dtype=np.int32))
    subs = O.build_submeshes(topo.adj_offsets, topo.adj_cols, part.members)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=10, iterations=1, shift_scale=1e-3)
    ob = O.compute_block_bases_fixed_sizes(frames[0].vertices, subs, part.sequence, ocfg, [10] * 3)
    bb = G.BlockBases(part.sequence, [], ob.bases, None, None, {}, part.block_size)
    with pytest.raises(G.InvalidArgument, match="reconstruction is missing 1024 vertices: 2080 2081"):
        G.coarse_reconstruct_frames(topo, part, bb, [frames[0].vertices], ctx=ctx)


def test_frames_stage_device_pointers(ctx):
    """smg_coarse_reconstruct_frames with device bases, frames and outputs equals
    the host-pointer call bit for bit."""
    import ctypes as C

    import torch
    from paper_1810_02719_b200 import _abi
    topo, frames = sequence(64, 64, 3, seed=17)
    seg = synth.grid_tiles(64, 64, 32, 32)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=24, iterations=1, shift_scale=1e-3)
    bb = G.compute_block_bases_fixed_sizes(frames[0], seg, cfg, [24] * seg.count, want_bases=True, ctx=ctx)
    want = G.coarse_reconstruct_frames(topo, seg, bb, [f.vertices for f in frames], ctx=ctx)
    dev = torch.device("cuda", 0)
    keep = []
    mv, sv = G._mesh_view(topo, keep), G._seg_view(seg, keep)
    k = seg.count
    sizes = np.full(k, 24, np.int32)
    offs = (np.arange(k + 1) * 24 * seg.block_size).astype(np.int64)
    data = torch.from_numpy(np.concatenate([b.ravel(order="F") for b in bb.bases])).to(dev)
    bv = _abi.smg_bases(k, sizes.ctypes.data, offs.ctypes.data, data.data_ptr(), 1)
    cols = [torch.from_numpy(np.ascontiguousarray(f.vertices[:, a])).to(dev) for f in frames for a in range(3)]
    xyz = (C.c_void_p * len(cols))(*[t.data_ptr() for t in cols])
    outs = [torch.empty(3 * topo.n, dtype=torch.float64, device=dev) for _ in frames]
    outp = (C.c_void_p * len(outs))(*[t.data_ptr() for t in outs])
    ctx.check(ctx.lib.smg_coarse_reconstruct_frames(ctx.handle, C.byref(mv), C.byref(sv), C.byref(bv), len(frames),
                                                    xyz, 1, 1, outp, 1))
    torch.cuda.synchronize()
    for o, w in zip(outs, want):
        assert np.array_equal(o.cpu().numpy().reshape(3, -1).T, w)


def test_denoise_dynamic_doi_bases(ctx):
    """DOI-chosen per-block sizes (cfg.basis_mode = doi, no sizes): the frames
    stage runs on the variable-c bases and equals the per-frame projection of
    those bases."""
    topo, frames = sequence(64, 64, 3, seed=19, flip=2)
    seg = synth.grid_tiles(64, 64, 32, 32)
    cfg = G.PipelineConfig(weighting="binary", basis_mode="doi", subspace_size=8, c_min=4, c_max=48,
                           eps_low=2e-3, eps_high=2e-2, shift_scale=1e-3)
    res = G.denoise_dynamic(frames, seg, cfg, ctx=ctx)
    bb = G.compute_block_bases(frames[0], seg, cfg, want_bases=True, ctx=ctx)
    want = G.coarse_reconstruct_frames(topo, seg, bb, [f.vertices for f in frames], ctx=ctx)
    for got, w in zip(res.frames, want):
        assert rel_err(got, w) < 1e-12
    assert len({b.shape[1] for b in bb.bases}) >= 1


def test_denoise_dynamic_single_frame_equals_chain(ctx):
    """One frame: denoise_dynamic is the coarse pass of that frame."""
    topo, frames = sequence(64, 64, 1, seed=23, flip=5)
    seg = synth.grid_tiles(64, 64, 32, 32)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=30, iterations=1, shift_scale=1e-3)
    res = G.denoise_dynamic(frames, seg, cfg, [30] * seg.count, ctx=ctx)
    bb = G.compute_block_bases_fixed_sizes(frames[0], seg, cfg, [30] * seg.count, ctx=ctx)
    assert rel_err(res.frames[0], bb.reconstruction) < 1e-12
