"""CPU checks of the oracle's dynamic-mesh restatement (denoise.hpp:258-291) and
of the frame-sequence generator (test infrastructure for test_gpu_frames)."""
import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth


def small_problem(frames):
    topo = synth.small_grid(32, 32, 16, 16, seed=4, flip=2)
    seg = synth.grid_tiles(32, 32, 16, 16)
    subs = O.build_submeshes(topo.adj_offsets, topo.adj_cols, seg.members)
    verts = synth.grid_sequence(32, 32, frames, 4, 0.01)
    cfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=12, iterations=1, shift_scale=1e-3)
    return topo, seg, subs, verts, cfg


def test_sequence_shares_grid_and_moves():
    v = synth.grid_sequence(16, 8, 3, 9, 0.0)
    assert all(f.shape == (128, 3) for f in v)
    assert np.array_equal(v[0][:, :2], v[2][:, :2])  # xy fixed, only heights move
    assert np.abs(v[0][:, 2] - v[2][:, 2]).max() > 0


def test_denoise_dynamic_bases_from_first_frame():
    _, seg, subs, verts, cfg = small_problem(3)
    out, nb, bb = O.denoise_dynamic(verts, subs, seg.sequence, cfg, [12] * seg.count)
    assert nb == seg.count == 4
    # frame 0 equals the plain coarse pass; later frames reuse frame 0's bases
    assert np.array_equal(out[0], O.coarse_reconstruct_points(bb, verts[0]))
    assert np.array_equal(out[2], O.coarse_reconstruct_points(bb, verts[2]))
    # the projection is linear in the coordinates
    mix = O.coarse_reconstruct_points(bb, 0.25 * verts[1] + 0.75 * verts[2])
    assert np.abs(mix - (0.25 * out[1] + 0.75 * out[2])).max() < 1e-12 * np.abs(mix).max()


def test_denoise_dynamic_identical_frames_and_idempotence():
    _, seg, subs, verts, cfg = small_problem(1)
    out, _, bb = O.denoise_dynamic([verts[0], verts[0].copy()], subs, seg.sequence, cfg, [12] * seg.count)
    assert np.array_equal(out[0], out[1])
    # disjoint tiles: projecting the reconstruction again changes nothing
    again = O.coarse_reconstruct_points(bb, out[0])
    assert np.abs(again - out[0]).max() < 1e-12 * np.abs(out[0]).max()


def test_denoise_dynamic_errors():
    _, seg, subs, verts, cfg = small_problem(1)
    with pytest.raises(O.InvalidArgument, match="at least one frame"):
        O.denoise_dynamic([], subs, seg.sequence, cfg, [12] * seg.count)
    with pytest.raises(O.InvalidArgument, match="frame 1 does not share the sequence connectivity"):
        O.denoise_dynamic([verts[0], verts[0][:100]], subs, seg.sequence, cfg, [12] * seg.count)
