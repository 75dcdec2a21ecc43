"""CPU, only where the reference sources are present (this container): the reference's OWN
code, compiled by `make refharness` over oracle/eigen_shim, run live on fresh seeded inputs
and compared with the numpy oracle -- beyond the committed fixtures, any seed.  Skipped on
the GPU box (no /root/reference there; the fixtures under tests/golden/ stand in)."""
import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth

R = pytest.importorskip("ref_binding")
if not R.available():
    pytest.skip("oracle/_ref/libspecmesh_ref.so not built (needs /root/reference)", allow_module_level=True)


@pytest.mark.parametrize("seed,flip,c,t", [(17, 3, 24, 1), (23, None, 40, 2)])
def test_fixed_chain_live(seed, flip, c, t):
    mesh = synth.small_grid(96, 64, 32, 32, seed=seed, flip=flip)
    seg = synth.grid_tiles(96, 64, 32, 32)
    rm = R.Mesh(mesh.vertices, mesh.faces)
    offs, cols = rm.edges_csr()
    assert np.array_equal(offs, mesh.adj_offsets) and np.array_equal(cols, mesh.adj_cols)  # build_edges
    rs = R.Segmentation.from_members(rm, seg.members, seg.sequence)
    bb = R.chain_fixed(rm, rs, R.default_config(weighting=R.BINARY, subspace_size=c, iterations=t, shift_scale=1e-3),
                       [c] * seg.count)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence,
                                           O.PipelineConfig(weighting=O.BINARY, subspace_size=c, iterations=t,
                                                            shift_scale=1e-3), [c] * seg.count)
    for i in range(seg.count):
        assert O.max_principal_angle(bb.basis(i), ob.bases[i]) < 1e-8
        assert abs(bb.stats(i)["residual_rms"] - ob.stats[i].residual_rms) <= 1e-9 * ob.stats[i].residual_rms
        co = O.gft(ob.bases[i], subs[i].local_coords(mesh.vertices))
        assert np.abs(np.abs(bb.coefficients(i)) - np.abs(co)).max() <= 1e-8 * np.abs(co).max()
    rec = O.coarse_reconstruct_points(ob, mesh.vertices)
    assert np.linalg.norm(bb.reconstruct() - rec, axis=1).max() <= 1e-9 * np.linalg.norm(rec, axis=1).max()


@pytest.mark.parametrize("k,seed", [(4, 1), (6, 9)])
def test_segment_mesh_live(k, seed):
    mesh = synth.small_grid(48, 40, 16, 8, seed=5, flip=2)
    rm = R.Mesh(mesh.vertices, mesh.faces)
    seg = R.Segmentation.segment_mesh(rm, R.default_config(part_count=k, growth=1.2, seed=seed))
    part, members, order = O.segment_mesh(mesh.adj_offsets, mesh.adj_cols, k, 1.2, seed)
    assert np.array_equal(seg.assignment(), part.assignment)
    assert all(np.array_equal(a, b) for a, b in zip(seg.members(), members))
    assert np.array_equal(seg.order(), order)


def test_primitives_live():
    mesh = synth.sphere_mesh(3, 13)
    seg = synth.sphere_blocks(mesh, bands=4, block=128)
    rm = R.Mesh(mesh.vertices, mesh.faces)
    rs = R.Segmentation.from_members(rm, seg.members, seg.sequence)
    sub = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)[2]
    for wt_r, wt_o in ((R.BINARY, O.BINARY), (R.DISTANCE, O.DISTANCE)):
        offs, cols, vals, tr, de = rs.laplacian(2, wt_r, 1e-3)
        lap = O.build_laplacian(sub, mesh.vertices, wt_o)
        assert np.array_equal(offs, lap.rowptr) and np.array_equal(cols, lap.cols) and np.array_equal(vals, lap.vals)
        assert tr == lap.trace() and de == O.default_shift(lap, 1e-3)
    rng = np.random.Generator(np.random.PCG64(3))
    block = rng.standard_normal((seg.members[2].size, 12))
    assert np.abs(R.orthonormalize(block) - O.orthonormalize(block)).max() <= 1e-12
    lap = O.build_laplacian(sub, mesh.vertices, O.DISTANCE)
    y = O.ShiftedInverseOperator(lap, O.default_shift(lap, 1e-3), 2).apply(block)
    assert np.abs(rs.apply(2, R.DISTANCE, 1e-3, 2, block) - y).max() <= 1e-11 * np.abs(y).max()
    q = O.orthonormalize(block)
    rot, _ = np.linalg.qr(rng.standard_normal((12, 12)))
    other = O.orthonormalize(rng.standard_normal(block.shape))
    assert R.max_principal_angle(q, q @ rot) < 1e-13  # the same span
    assert abs(R.max_principal_angle(q, other) - O.max_principal_angle(q, other)) < 1e-12
    with pytest.raises(R.RefError, match="rank deficient"):
        R.orthonormalize(np.ones((8, 2)))
