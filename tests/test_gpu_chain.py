"""GPU parity of the chain (compute_block_bases_fixed_sizes / compute_block_bases
+ coarse_reconstruct_points) against the CPU oracle on seeded inputs."""
import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_1810_02719_b200")


def run_both(ctx, mesh, seg, c, t=1, scale=1e-3, want_bases=True):
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=c, iterations=t, shift_scale=scale)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=c, iterations=t, shift_scale=scale)
    bb = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [c] * seg.count, want_bases=want_bases, ctx=ctx)
    ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence, ocfg, [c] * seg.count)
    return bb, ob


def check_parity(mesh, bb, ob, angle_tol=1e-8, recon_tol=1e-9):
    k = len(ob.bases)
    angles = [O.max_principal_angle(bb.bases[i], ob.bases[i]) for i in range(k)]
    assert max(angles) < angle_tol, max(angles)
    rec = O.coarse_reconstruct_points(ob, mesh.vertices)
    err = np.linalg.norm(bb.reconstruction - rec, axis=1).max() / np.linalg.norm(rec, axis=1).max()
    assert err < recon_tol, err
    for i in range(k):
        assert bb.stats[i].subspace_size == ob.stats[i].subspace_size
        assert bb.stats[i].oi_iterations == ob.stats[i].oi_iterations
        assert abs(bb.stats[i].residual_rms - ob.stats[i].residual_rms) <= 1e-9 * max(ob.stats[i].residual_rms, 1e-300)
        co = O.gft(ob.bases[i], ob.submeshes[i].local_coords(mesh.vertices))
        # coefficients carry the sign convention (spectral.hpp:72-85).  Columns
        # whose two largest magnitudes tie to rounding (mirror-symmetric grid
        # eigenvectors) have an implementation-dependent sign: align those only.
        ub, uo = bb.bases[i], ob.bases[i]
        s = np.sign(np.sum(ub * uo, axis=0))
        mags = np.sort(np.abs(uo), axis=0)
        tie = (mags[-1] - mags[-2]) <= 1e-9 * mags[-1]
        assert np.all((s > 0) | tie), "sign convention differs on a column without a magnitude tie"
        assert np.abs(bb.coefficients[i] * s[:, None] - co).max() <= 1e-8 * np.abs(co).max()
        assert np.abs(ub.T @ ub - np.eye(ub.shape[1])).max() < 1e-12


def test_chain_grid_identical_tiles(ctx):
    mesh = synth.small_grid(128, 128, 32, 32, seed=2)
    seg = synth.grid_tiles(128, 128, 32, 32)
    bb, ob = run_both(ctx, mesh, seg, 100)
    check_parity(mesh, bb, ob)


def test_chain_grid_flipped_tiles(ctx):
    """Per-quad diagonal flips make every tile's Laplacian differ, so the warm
    start carry is exercised (SURVEY.md §0 finding 3)."""
    mesh = synth.small_grid(128, 64, 32, 32, seed=4, flip=8)
    seg = synth.grid_tiles(128, 64, 32, 32)
    bb, ob = run_both(ctx, mesh, seg, 60, t=2)
    check_parity(mesh, bb, ob)


def test_chain_wide_tiles(ctx):
    mesh = synth.small_grid(128, 64, 64, 32, seed=6, flip=3)
    seg = synth.grid_tiles(128, 64, 64, 32)
    bb, ob = run_both(ctx, mesh, seg, 200)
    check_parity(mesh, bb, ob)


def test_chain_sphere_blocks(ctx):
    """Icosphere blocks (RCM ordering, overlapping submeshes, stitched)."""
    mesh = synth.sphere_mesh(5, 11)
    seg = synth.sphere_blocks(mesh, bands=16, block=256)
    bb, ob = run_both(ctx, mesh, seg, 40)
    check_parity(mesh, bb, ob)


def test_chain_reference_default_shift_throws_same_column(ctx):
    """shift_scale = 1e-8 (reference default) makes the reference throw "rank
    deficient at column k" (SURVEY.md §0 finding 2); the GPU reports the same k."""
    mesh = synth.small_grid(64, 64, 32, 32, seed=2)
    seg = synth.grid_tiles(64, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    ocfg = O.PipelineConfig(weighting=O.BINARY, subspace_size=40, iterations=1, shift_scale=1e-8)
    with pytest.raises(O.Error) as eo:
        O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence, ocfg, [40] * seg.count)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=40, iterations=1, shift_scale=1e-8)
    with pytest.raises(G.SpecmeshError) as eg:
        G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40] * seg.count, ctx=ctx)
    assert str(eg.value) == str(eo.value)


def test_chain_invalid_arguments(ctx):
    mesh = synth.small_grid(64, 64, 32, 32, seed=2)
    seg = synth.grid_tiles(64, 64, 32, 32)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=40, iterations=1, shift_scale=1e-3)
    with pytest.raises(G.InvalidArgument, match="subspace size out of range for block"):
        G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40, 40, 2000, 40], ctx=ctx)
    with pytest.raises(G.InvalidArgument, match="need one subspace size per block"):
        G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40] * 3, ctx=ctx)
    bad = synth.Segmentation([seg.members[0], seg.members[1][:500]], np.array([0, 1], np.int32))
    with pytest.raises(G.InvalidArgument, match="initial basis does not match the operator size"):
        G.compute_block_bases_fixed_sizes(mesh, bad, cfg, [40, 40], ctx=ctx)
    hole = synth.Segmentation(seg.members[:3], np.array([0, 1, 2], np.int32))
    with pytest.raises(G.InvalidArgument, match="reconstruction is missing 1024 vertices"):
        G.compute_block_bases_fixed_sizes(mesh, hole, cfg, [40] * 3, ctx=ctx)


def test_chain_variable_sizes_shrink_and_grow(ctx):
    """sizes_in_order with shrink (leading columns) and growth (seeded
    libstdc++ Gaussian columns + orthonormalize) -- resize_basis, pipeline.hpp:97-109."""
    mesh = synth.small_grid(128, 64, 32, 32, seed=4, flip=8)
    seg = synth.grid_tiles(128, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    sizes = [40, 30, 30, 50, 45, 60, 60, 20]
    cfg = G.PipelineConfig(weighting="binary", iterations=1, shift_scale=1e-3)
    ocfg = O.PipelineConfig(weighting=O.BINARY, iterations=1, shift_scale=1e-3)
    bb = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, sizes, want_bases=True, ctx=ctx)
    ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence, ocfg, sizes)
    check_parity(mesh, bb, ob)


def test_chain_grows_at_position_one(ctx):
    """Growth right after the first basis: the appended columns follow the
    first block's sign-fixed basis (resize_basis, pipeline.hpp:97-109)."""
    mesh = synth.small_grid(64, 64, 32, 32, seed=8, flip=1)
    seg = synth.grid_tiles(64, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    sizes = [30, 36, 30, 24]
    cfg = G.PipelineConfig(weighting="binary", iterations=1, shift_scale=1e-3)
    ocfg = O.PipelineConfig(weighting=O.BINARY, iterations=1, shift_scale=1e-3)
    bb = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, sizes, want_bases=True, ctx=ctx)
    ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence, ocfg, sizes)
    check_parity(mesh, bb, ob)


@pytest.mark.parametrize("kw", [
    dict(subspace_size=60, c_min=10, c_max=200, eps_low=2e-3, eps_high=2e-2, shift_scale=1e-3),
    # c pinned (c_min = c_max): no adjustment possible, blocks above the band end unconverged
    dict(subspace_size=30, c_min=30, c_max=30, eps_low=1e-4, eps_high=1e-3, shift_scale=1e-3),
    # a band above every residual: every block shrinks towards c_min
    dict(subspace_size=40, c_min=20, c_max=60, eps_low=0.5, eps_high=0.9, shift_scale=1e-3),
])
def test_doi_chain_decisions_match(ctx, kw):
    """DOI chain with a band each block meets in a few steps: per-block c,
    iteration count and convergence flags equal the oracle's."""
    mesh = synth.small_grid(128, 64, 32, 32, seed=4, flip=8)
    seg = synth.grid_tiles(128, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    cfg = G.PipelineConfig(weighting="binary", basis_mode="doi", **kw)
    ocfg = O.PipelineConfig(weighting=O.BINARY, **kw)
    bb = G.compute_block_bases(mesh, seg, cfg, want_bases=True, ctx=ctx)
    ob = O.compute_block_bases_doi(mesh.vertices, subs, seg.sequence, ocfg)
    for i in range(seg.count):
        g, o = bb.stats[i], ob.stats[i]
        assert (g.subspace_size, g.oi_iterations, g.converged) == (o.subspace_size, o.oi_iterations, o.converged)
        assert abs(g.doi_residual - o.doi_residual) <= 1e-6 * o.doi_residual


@pytest.mark.parametrize("nchains,sizes", [(3, None), (5, [60, 80, 80, 70])])
def test_batched_chains_equal_single_chains(ctx, nchains, sizes):
    """smg_run_chains (config 5's per-GPU shard) matches running each chain
    alone.  Chains are independent and every reduction has a fixed order; the
    first-submesh subspace iteration runs as many rounds as the slowest chain of
    the batch needs, so agreement is to the first-basis tolerance, not bitwise.
    Five chains run as two chain groups on their own streams (with a growth at
    position 1: each group re-signs its share of the first basis)."""
    meshes = [synth.small_grid(128, 64, 64, 32, seed=s, flip=s) for s in range(1, nchains + 1)]
    seg = synth.grid_tiles(128, 64, 64, 32)
    sizes = sizes or [80] * seg.count
    cfg = G.PipelineConfig(weighting="binary", subspace_size=80, iterations=1, shift_scale=1e-3)
    batch = G.run_chains(meshes, [seg] * nchains, cfg, sizes, ctx=ctx)
    for m, b in zip(meshes, batch):
        single = G.compute_block_bases_fixed_sizes(m, seg, cfg, sizes, ctx=ctx)
        r = single.reconstruction
        assert np.linalg.norm(b.reconstruction - r, axis=1).max() <= 1e-10 * np.linalg.norm(r, axis=1).max()
        for i in range(seg.count):
            assert abs(single.stats[i].residual_rms - b.stats[i].residual_rms) <= 1e-10 * single.stats[i].residual_rms


def test_fused_chebyshev_filter_bit_identical(ctx, monkeypatch):
    """The fused first-basis filter (all degree steps in one launch, iterates in
    shared memory) performs the per-step SpMM path's arithmetic exactly."""
    mesh = synth.small_grid(64, 64, 32, 32, seed=6, flip=2)
    seg = synth.grid_tiles(64, 64, 32, 32)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=40, iterations=1, shift_scale=1e-3)
    fused = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40] * seg.count, want_bases=True, ctx=ctx)
    monkeypatch.setenv("SMG_CHEB_UNFUSED", "1")
    plain = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40] * seg.count, want_bases=True, ctx=ctx)
    for a, b in zip(fused.bases, plain.bases):
        assert np.array_equal(a, b)
    assert np.array_equal(fused.reconstruction, plain.reconstruction)


@pytest.mark.parametrize("tw,th,c", [(4, 4, 16), (4, 4, 1), (4, 4, 4), (8, 4, 5), (2, 2, 2), (2, 2, 4), (5, 5, 7),
                                     (40, 4, 20), (6, 8, 48), (48, 8, 64)])
def test_tiny_tiles_and_full_bases(ctx, tw, th, c):
    """Edge sizes: 4- and 16-vertex tiles, c = 1 and c = n_d (the basis spans
    the whole block, so the reconstruction is exact).  When the first-basis
    subspace is the whole block its single Rayleigh-Ritz is final (not a
    2-sweep bootstrap).  (A 2x2 tile has eigenvalues 0, 2, 4, 4: c = 3 would cut
    a degenerate pair, where no basis is determined.)"""
    W, H = 4 * tw, 2 * th
    mesh = synth.small_grid(W, H, tw, th, seed=5, flip=3)
    seg = synth.grid_tiles(W, H, tw, th)
    bb, ob = run_both(ctx, mesh, seg, c)
    if c < tw * th:
        check_parity(mesh, bb, ob)
        return
    for i in range(seg.count):
        assert O.max_principal_angle(bb.bases[i], ob.bases[i]) < 1e-8
        assert bb.stats[i].residual_rms <= 1e-12 * np.abs(mesh.vertices).max()
    assert np.abs(bb.reconstruction - mesh.vertices).max() <= 1e-11 * np.abs(mesh.vertices).max()


def test_chain_distance_weighting(ctx):
    """The reference's default weighting (1 / |v_i - v_j|^2 off the diagonal,
    spectral.hpp:48-59): chain parity against the oracle (first basis through
    the per-step SpMM filter, not the binary-pattern fused one)."""
    mesh = synth.small_grid(64, 64, 32, 32, seed=9, flip=6)
    seg = synth.grid_tiles(64, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    cfg = G.PipelineConfig(weighting="distance", subspace_size=40, iterations=1, shift_scale=1e-3)
    ocfg = O.PipelineConfig(weighting=O.DISTANCE, subspace_size=40, iterations=1, shift_scale=1e-3)
    bb = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40] * seg.count, want_bases=True, ctx=ctx)
    ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence, ocfg, [40] * seg.count)
    check_parity(mesh, bb, ob)


@pytest.mark.parametrize("dense_limit", [512, 1023])
def test_chain_cold_start_first_basis(ctx, dense_limit):
    """n_d > dense_limit: the first basis is the reference's cold start,
    random_orthonormal_basis(n_d, c, seed ^ 0x9E3779B97F4A7C15) followed by
    initial_iterations OI steps (pipeline.hpp:118-119, spectral.hpp:134-141);
    the Gaussian draws are libstdc++'s, so GPU and oracle start from the same
    block and track the same iterates."""
    mesh = synth.small_grid(64, 64, 32, 32, seed=9, flip=4)
    seg = synth.grid_tiles(64, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    kw = dict(subspace_size=24, iterations=1, shift_scale=1e-3, dense_limit=dense_limit, initial_iterations=12)
    cfg = G.PipelineConfig(weighting="binary", **kw)
    ocfg = O.PipelineConfig(weighting=O.BINARY, **kw)
    bb = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [24] * seg.count, want_bases=True, ctx=ctx)
    ob = O.compute_block_bases_fixed_sizes(mesh.vertices, subs, seg.sequence, ocfg, [24] * seg.count)
    check_parity(mesh, bb, ob)
    # the cold start is not the dense eigenbasis: 12 R^2 steps from a random block
    dense = O.bottom_subspace(O.dense_eigendecomposition(O.build_laplacian(subs[0], mesh.vertices, O.BINARY)), 24)
    assert O.max_principal_angle(ob.bases[0], dense) > 1e-6


def test_run_info_and_doi_host_loop(ctx, monkeypatch):
    """smg_last_run_info reports the factorisation the library chose; the
    host-driven DOI loop (SMG_DOI_NOGRAPH, for profilers) takes the same
    decisions as the CUDA-graph WHILE loop, step for step."""
    mesh = synth.small_grid(128, 64, 32, 32, seed=4, flip=8)
    seg = synth.grid_tiles(128, 64, 32, 32)
    cfg = G.PipelineConfig(weighting="binary", subspace_size=40, iterations=1, shift_scale=1e-3)
    G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [40] * seg.count, ctx=ctx)
    info = ctx.last_run_info()
    assert info["chains"] == 1 and info["positions"] == seg.count and info["block_width"] in (32, 33, 48, 64)
    assert info["ordering"] in ("natural", "geometric", "rcm")
    dcfg = G.PipelineConfig(weighting="binary", basis_mode="doi", subspace_size=10, c_min=5, c_max=120,
                            eps_low=3e-4, eps_high=3e-3, shift_scale=1e-3)
    ctx.doi_trace(True)
    a = G.compute_block_bases(mesh, seg, dcfg, ctx=ctx)
    ta = ctx.read_doi_trace()
    ctx.doi_trace(True)
    monkeypatch.setenv("SMG_DOI_NOGRAPH", "1")
    b = G.compute_block_bases(mesh, seg, dcfg, ctx=ctx)
    tb = ctx.read_doi_trace()
    ctx.doi_trace(False)
    assert [s.subspace_size for s in a.stats] == [s.subspace_size for s in b.stats]
    assert [s.oi_iterations for s in a.stats] == [s.oi_iterations for s in b.stats]
    assert np.array_equal(ta[0], tb[0]) and np.array_equal(ta[1], tb[1])
    assert np.allclose(ta[2], tb[2], rtol=1e-12, atol=0)
    assert np.array_equal(a.reconstruction, b.reconstruction)
