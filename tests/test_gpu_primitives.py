"""GPU parity of the L3 primitives against the CPU oracle, through the C ABI.

Tolerances (BASELINE.json north_star): CSR bit-exact; tracked subspaces by the
largest principal angle <= 1e-8; reconstructions <= 1e-9 relative (normwise);
plus the SPEC.md known answers on the GPU path."""
import math

import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_1810_02719_b200")


@pytest.fixture(scope="module")
def grid():
    mesh = synth.small_grid(64, 64, 32, 32, seed=3, flip=5)
    seg = synth.grid_tiles(64, 64, 32, 32)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    return mesh, seg, subs


@pytest.fixture(scope="module")
def sphere():
    mesh = synth.sphere_mesh(5, 11)
    seg = synth.sphere_blocks(mesh, bands=16, block=256)
    subs = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)
    return mesh, seg, subs


def _op(ctx, lap, scale=1e-3, z=2):
    d = O.default_shift(lap, scale)
    return G.ShiftedInverseOperator(lap.rowptr, lap.cols, lap.vals, d, z, ctx=ctx), O.ShiftedInverseOperator(lap, d, z)


@pytest.mark.parametrize("weighting", ["binary", "distance"])
def test_laplacian_bit_exact_grid(ctx, grid, weighting):
    mesh, seg, subs = grid
    for t in (0, 3):
        lap = O.build_laplacian(subs[t], mesh.vertices, weighting)
        rp, c, v, tr = G.build_laplacian(mesh, seg.members[t], weighting, ctx=ctx)
        assert np.array_equal(rp, lap.rowptr) and np.array_equal(c, lap.cols)
        assert np.array_equal(v, lap.vals)  # bit-exact, incl. 1/d^2 weights
        assert tr == lap.trace()


def test_laplacian_bit_exact_sphere_blocks(ctx, sphere):
    mesh, seg, subs = sphere
    for t in (0, 7, seg.count - 1):
        lap = O.build_laplacian(subs[t], mesh.vertices, "binary")
        rp, c, v, tr = G.build_laplacian(mesh, seg.members[t], "binary", ctx=ctx)
        assert np.array_equal(rp, lap.rowptr) and np.array_equal(c, lap.cols) and np.array_equal(v, lap.vals)


def test_coincident_vertices_error(ctx):
    faces = np.array([[0, 1, 2]], np.int32)
    offs, cols = synth.build_edges(faces, 3)
    mesh = synth.Mesh(np.array([[0.0, 0, 0], [0.0, 0, 0], [1.0, 0, 0]]), faces, offs, cols)
    with pytest.raises(G.SpecmeshError, match="coincident connected vertices 0 and 1 make the distance weight singular"):
        G.build_laplacian(mesh, [0, 1, 2], "distance", ctx=ctx)


def test_shifted_inverse_known_answer(ctx):
    rp = np.array([0, 2, 4], np.int32)
    c = np.array([0, 1, 0, 1], np.int32)
    v = np.array([1.0, -1.0, -1.0, 1.0])
    op1 = G.ShiftedInverseOperator(rp, c, v, 1.0, 1, ctx=ctx)
    assert np.allclose(op1.apply(np.array([[1.0], [0.0]]))[:, 0], [2 / 3, 1 / 3], atol=1e-15)
    op2 = G.ShiftedInverseOperator(rp, c, v, 1.0, 2, ctx=ctx)
    b = np.array([[1.0, 0.3], [0.0, -2.0]])
    assert np.abs(op2.apply(b) - op1.apply(op1.apply(b))).max() < 1e-12


def test_operator_apply_matches_oracle(ctx, grid, sphere):
    rng = np.random.default_rng(0)
    for mesh, seg, subs in (grid, sphere):
        lap = O.build_laplacian(subs[1], mesh.vertices, "binary")
        g, o = _op(ctx, lap)
        b = rng.standard_normal((lap.size(), 24))
        for fn in ("apply", "apply_once"):
            y, yo = getattr(g, fn)(b), getattr(o, fn)(b)
            assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < 1e-12
        y = g.spmm(b)
        yo = (lap.to_scipy() + g.shift() * np.eye(lap.size())) @ b
        assert np.abs(y - yo).max() < 1e-12


def test_operator_indefinite_distance_weighting(ctx, grid):
    """Distance weights on a unit grid make L indefinite (SURVEY finding 7); the
    reference's no-pivot LDL^T accepts negative pivots and so does the signed
    block factor."""
    mesh, seg, subs = grid
    v = mesh.vertices.copy()
    v[:, :2] *= 0.5  # edge length < 1 => 1/d^2 > 1 > degree share
    lap = O.build_laplacian(subs[0], v, "distance")
    g, o = _op(ctx, lap, scale=1e-3, z=1)
    b = np.random.default_rng(1).standard_normal((lap.size(), 8))
    y, yo = g.apply(b), o.apply(b)
    assert np.linalg.norm(y - yo) / np.linalg.norm(yo) < 1e-9


def test_orthonormalize_known_answers(ctx):
    q = G.orthonormalize(np.array([[2.0, 0], [0, 3.0], [0, 0]]), ctx=ctx)
    assert np.allclose(q, [[1.0, 0], [0, 1.0], [0, 0]], atol=1e-15)
    b = np.random.default_rng(1).standard_normal((100, 8))
    q = G.orthonormalize(b, ctx=ctx)
    assert np.abs(q.T @ q - np.eye(8)).max() < 1e-12
    assert np.abs(q - O.orthonormalize(b)).max() < 1e-12  # same sign convention


@pytest.mark.parametrize("col", [1, 3, 7])
def test_orthonormalize_rank_deficiency_error_parity(ctx, col):
    b = np.random.default_rng(col).standard_normal((64, 10))
    b[:, col] = b[:, 0] * 0.5 + b[:, col - 1]
    with pytest.raises(O.Error) as eo:
        O.orthonormalize(b)
    with pytest.raises(G.SpecmeshError) as eg:
        G.orthonormalize(b, ctx=ctx)
    assert str(eg.value) == str(eo.value) == f"orthonormalize: block is rank deficient at column {col}"


def test_rank_test_resolution_divergence(ctx):
    """Known deviation: two unit columns at an angle of 1e-7.
    Householder QR gives |r_11| = sin(1e-7) ~ 1e-7 >= 1e-13 ||V||_F, so the
    reference passes; the column-scaled Cholesky pivot is 1 - cos^2 ~ 1e-14,
    below the Gram's resolution (1e-12), and the GPU reports rank deficiency
    at column 1.  Larger angles (1e-5) pass on both."""
    rng = np.random.default_rng(3)
    e, f = np.linalg.qr(rng.standard_normal((64, 2)))[0].T
    for theta, gpu_fails in ((1e-7, True), (1e-5, False)):
        b = np.stack([e, np.cos(theta) * e + np.sin(theta) * f], axis=1)
        qo = O.orthonormalize(b)  # the reference's test passes
        if gpu_fails:
            with pytest.raises(G.SpecmeshError, match="rank deficient at column 1"):
                G.orthonormalize(b, ctx=ctx)
        else:
            q = G.orthonormalize(b, ctx=ctx)
            assert np.abs(q.T @ q - np.eye(2)).max() < 1e-9
            assert O.max_principal_angle(q, qo) < 1e-6


@pytest.mark.parametrize("c", [33, 300, 512])
def test_orthonormalize_wide_blocks(ctx, c):
    """Multi-panel CholeskyQR2 up to the 512-column limit, graded column norms."""
    rng = np.random.default_rng(c)
    b = rng.standard_normal((2048, c)) * np.logspace(0, -6, c)
    q = G.orthonormalize(b, ctx=ctx)
    assert np.abs(q.T @ q - np.eye(c)).max() < 1e-12
    assert np.abs(q - O.orthonormalize(b)).max() < 1e-10


@pytest.mark.parametrize("c", [200, 256, 320, 400])
def test_orthonormalize_ill_conditioned_second_pass(ctx, c):
    """Conditioning that column scaling cannot remove (kappa = 1e5 spread over
    mixed columns): the second CholeskyQR pass is not near-identity, so its
    Cholesky forms the full inverse -- on one CTA (c <= 224) or split over a
    4-CTA cluster with strided s-sums (c > 224, one chain)."""
    rng = np.random.default_rng(100 + c)
    u, _ = np.linalg.qr(rng.standard_normal((2048, c)))
    w, _ = np.linalg.qr(rng.standard_normal((c, c)))
    b = (u * np.logspace(0, -5, c)) @ w.T
    q = G.orthonormalize(b, ctx=ctx)
    assert np.abs(q.T @ q - np.eye(c)).max() < 1e-12
    assert np.abs(q - O.orthonormalize(b)).max() < 1e-8


def test_orthonormalize_errors(ctx):
    with pytest.raises(G.SpecmeshError, match=r"rank deficient \(all zero\)"):
        G.orthonormalize(np.zeros((5, 2)), ctx=ctx)
    with pytest.raises(G.InvalidArgument, match="block must be tall"):
        G.orthonormalize(np.ones((2, 3)), ctx=ctx)


def test_orthogonal_iteration(ctx, grid):
    mesh, seg, subs = grid
    lap = O.build_laplacian(subs[0], mesh.vertices, "binary")
    g, o = _op(ctx, lap)
    w, u = O.dense_eigendecomposition(lap)
    assert O.max_principal_angle(G.orthogonal_iteration(g, u[:, :40], 3), u[:, :40]) < 1e-10
    init = O.orthonormalize(np.random.default_rng(2).standard_normal((lap.size(), 30)))
    ug = G.orthogonal_iteration(g, init, 4)
    uo = O.orthogonal_iteration(o, init, 4)
    assert O.max_principal_angle(ug, uo) < 1e-10
    assert np.abs(ug - uo).max() < 1e-8  # same sign convention
    with pytest.raises(G.InvalidArgument, match="t_max must be nonnegative"):
        G.orthogonal_iteration(g, init, -1)


@pytest.mark.parametrize("case,c", [("grid", 40), ("grid", 100), ("sphere", 60), ("wide", 200), ("grid", 400),
                                    ("wide", 440)])
def test_first_basis_matches_dense_eig(ctx, grid, sphere, case, c):
    """bottom_subspace(dense_eigendecomposition(L), c) (spectral.hpp:92-117)."""
    if case == "wide":
        mesh = synth.small_grid(64, 32, 64, 32, seed=9)
        seg = synth.grid_tiles(64, 32, 64, 32)
        sub = O.build_submeshes(mesh.adj_offsets, mesh.adj_cols, seg.members)[0]
    else:
        mesh, seg, subs = grid if case == "grid" else sphere
        sub = subs[2]
    lap = O.build_laplacian(sub, mesh.vertices, "binary")
    g, _ = _op(ctx, lap)
    w, u = O.dense_eigendecomposition(lap)
    ug, ev = G.bottom_subspace(g, c, return_eigenvalues=True)
    assert O.max_principal_angle(ug, u[:, :c]) < 1e-9
    assert np.abs(ev - w[:c]).max() < 1e-10
    assert np.abs(ug.T @ ug - np.eye(c)).max() < 1e-12


def test_gft_igft(ctx, grid):
    mesh, seg, subs = grid
    lap = O.build_laplacian(subs[0], mesh.vertices, "binary")
    w, u = O.dense_eigendecomposition(lap)
    x = subs[0].local_coords(mesh.vertices)
    for c in (10, 100):
        cg = G.gft(u[:, :c], x, ctx=ctx)
        co = O.gft(u[:, :c], x)
        assert np.abs(cg - co).max() <= 1e-12 * np.abs(co).max()
        xh = G.igft(u[:, :c], co, ctx=ctx)
        assert np.abs(xh - O.igft(u[:, :c], co)).max() <= 1e-12 * np.abs(x).max()
    e1 = np.zeros((lap.size(), 3))
    e1[:, 0] = u[:, 0]
    assert np.allclose(G.gft(u[:, :5], e1, ctx=ctx)[:, 0], np.eye(5)[0], atol=1e-14)
    rt = G.igft(u, G.gft(u, x, ctx=ctx), ctx=ctx)
    assert np.abs(rt - x).max() < 1e-10


@pytest.mark.parametrize("t_max", [1, 2, 4, 6])
def test_dynamic_oi_step_parity(ctx, grid, t_max):
    """Step-level DOI parity.  DOI's raw-append + R^z growth is exponentially
    sensitive to rounding (two CPU restatements differ by 0.8 rad after 30 steps;
    DESIGN.md), so the basis is compared over the first steps and the decisions
    (c, iterations, converged) must match exactly."""
    mesh, seg, subs = grid
    lap = O.build_laplacian(subs[0], mesh.vertices, "binary")
    g, o = _op(ctx, lap)
    w, u = O.dense_eigendecomposition(lap)
    x = subs[0].local_coords(mesh.vertices)
    rg = G.dynamic_oi(g, u[:, :20], x, 1e-3, 1e-2, 5, 200, t_max)
    ro = O.dynamic_oi(o, u[:, :20], x, 1e-3, 1e-2, 5, 200, t_max)
    assert (rg.basis.shape, rg.iterations, rg.converged) == (ro.basis.shape, ro.iterations, ro.converged)
    assert abs(rg.residual - ro.residual) <= 1e-9 * ro.residual
    assert O.max_principal_angle(rg.basis, ro.basis) < 1e-8


def test_dynamic_oi_known_answers(ctx):
    n = 30
    rp, cols, vals = [0], [], []
    for i in range(n):
        nb = [j for j in (i - 1, i + 1) if 0 <= j < n]
        row = sorted(nb + [i])
        cols += row
        vals += [float(len(nb)) if j == i else -1.0 for j in row]
        rp.append(len(cols))
    lap = O.Laplacian(np.array(rp), np.array(cols), np.array(vals), "binary")
    w, u = O.dense_eigendecomposition(lap)
    g = G.ShiftedInverseOperator(lap.rowptr, lap.cols, lap.vals, 1e-2, 2, ctx=ctx)
    coords = np.random.default_rng(4).standard_normal((n, 3))
    r = G.dynamic_oi(g, u[:, :10], coords, 1e-9, 1e9, 2, 30, 10)  # band met at t=1
    assert r.iterations == 1 and r.basis.shape[1] == 10 and r.converged
    r = G.dynamic_oi(g, u, coords, 1e-12, 1e-9, 2, 30, 5)  # c = n_d: e = 0, below band -> shrinks
    ro = O.dynamic_oi(O.ShiftedInverseOperator(lap, 1e-2, 2), u, coords, 1e-12, 1e-9, 2, 30, 5)
    assert (r.basis.shape, r.iterations, r.converged) == (ro.basis.shape, ro.iterations, ro.converged)
    with pytest.raises(G.InvalidArgument, match="need 0 < eps_low < eps_high"):
        G.dynamic_oi(g, u[:, :10], coords, 1e-2, 1e-3, 2, 30, 5)
    with pytest.raises(G.InvalidArgument, match="need c_min <= init subspace size <= c_max"):
        G.dynamic_oi(g, u[:, :10], coords, 1e-3, 1e-2, 12, 30, 5)


def test_one_step_parity_sphere_chain(ctx, sphere):
    """SURVEY.md §4.3 one-step mode: the oracle's U_{i-1} fed into the GPU's
    OI step i on icosphere blocks (RCM-ordered, some disconnected)."""
    mesh, seg, subs = sphere
    prev = None
    worst = 0.0
    for i in range(6):
        lap = O.build_laplacian(subs[i], mesh.vertices, "binary")
        g, o = _op(ctx, lap)
        if prev is None:
            prev = O.bottom_subspace(O.dense_eigendecomposition(lap), 30)
            continue
        ug = G.orthogonal_iteration(g, prev, 1)
        uo = O.orthogonal_iteration(o, prev, 1)
        worst = max(worst, O.max_principal_angle(ug, uo))
        prev = uo
    assert worst < 1e-10


@pytest.mark.parametrize("env", [{"SMG_FB_BOOT_SWEEPS": "1"}, {"SMG_FIRST_BASIS": "si"}])
def test_first_basis_fallback_paths(ctx, grid, monkeypatch, env):
    """A filter planned from one bootstrap Jacobi sweep over-amplifies at c = 400
    of 1024 (the single-pass CholeskyQR breaks down) and the first basis retries
    shift-invert only; SMG_FIRST_BASIS=si runs that path directly.  Both must
    still give bottom_subspace(dense_eigendecomposition(L), c)."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    mesh, seg, subs = grid
    lap = O.build_laplacian(subs[2], mesh.vertices, "binary")
    g, _ = _op(ctx, lap)
    w, u = O.dense_eigendecomposition(lap)
    c = 400
    ug, ev = G.bottom_subspace(g, c, return_eigenvalues=True)
    assert O.max_principal_angle(ug, u[:, :c]) < 1e-9
    assert np.abs(ev - w[:c]).max() < 1e-10


@pytest.mark.parametrize("rows,cols", [(2048, 200), (1026, 60), (4096, 399), (700, 512), (64, 7)])
def test_orthonormality_probe_tracks_the_exact_norm(ctx, rows, cols):
    """The adaptive CholeskyQR2 decides its pass-2 skip from a one-pass randomized estimate of
    ||Q^T Q - I||_F (probe.cu, 8 fixed +-1 vectors).  Against the exact norm: an orthonormal
    block sits at rounding level; a block with a known departure E (dense, or concentrated in
    one entry -- the estimator's worst case) is estimated within the Hutchinson spread; odd
    widths, the width limit and row counts that are not multiples of the 32-row stage."""
    rng = np.random.Generator(np.random.PCG64(rows * 1000 + cols))
    q, _ = np.linalg.qr(rng.standard_normal((rows, cols)))
    assert G.orthonormality_estimate(q, ctx=ctx) < 1e-13
    # dense symmetric departure: Q (I + S) with ||S||_F = 1e-9  ->  Q^T Q - I ~ 2 S
    s = rng.standard_normal((cols, cols))
    s = (s + s.T) / 2
    s *= 1e-9 / np.linalg.norm(s)
    p = q @ (np.eye(cols) + s)
    exact = np.linalg.norm(p.T @ p - np.eye(cols))
    est = G.orthonormality_estimate(p, ctx=ctx)
    assert 0.6 * exact <= est <= 1.6 * exact, (est, exact)
    # rank-one departure (one column scaled): every probe sees it with weight 1
    p = q.copy()
    p[:, cols // 2] *= 1 + 1e-8
    exact = np.linalg.norm(p.T @ p - np.eye(cols))
    est = G.orthonormality_estimate(p, ctx=ctx)
    assert 0.9 * exact <= est <= 1.1 * exact, (est, exact)
    # two nearly parallel columns: far above any skip threshold
    p = q.copy()
    p[:, 0] = p[:, 1]
    assert G.orthonormality_estimate(p, ctx=ctx) > 0.5
