"""Pins the CPU oracle to the reference's only known answers: the SPEC.md
examples and invariants for the path and libstdc++'s
own RNG draws (the reference ships no tests or golden vectors)."""
import math
import os
import subprocess

import numpy as np
import pytest

import specmesh_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def edge_submesh():
    return O.Submesh(np.array([0, 1]), [np.array([1]), np.array([0])], np.array([1, 1]))


def test_laplacian_unit_edge():
    v = np.array([[0.0, 0, 0], [1.0, 0, 0]])
    for w in (O.BINARY, O.DISTANCE):
        lap = O.build_laplacian(edge_submesh(), v, w)
        assert np.array_equal(lap.dense(), [[1.0, -1.0], [-1.0, 1.0]])


def test_laplacian_edge_length_two():
    v = np.array([[0.0, 0, 0], [2.0, 0, 0]])
    lap = O.build_laplacian(edge_submesh(), v, O.DISTANCE)
    assert np.array_equal(lap.dense(), [[1.0, -0.25], [-0.25, 1.0]])


def test_laplacian_unit_triangle_row_sums():
    # SPEC's derivation "1*3 - 2*1 = 1" contradicts its own D_ii = |N(i)| (= 2 in a
    # triangle) and the code (spectral.hpp:46): with unit sides every row sums to
    # 2 - 2*1 = 0.  The oracle follows the code.
    v = np.array([[0.0, 0, 0], [1.0, 0, 0], [0.5, math.sqrt(3) / 2, 0]])
    sub = O.Submesh(np.arange(3), [np.array([1, 2]), np.array([0, 2]), np.array([0, 1])], np.array([2, 2, 2]))
    lap = O.build_laplacian(sub, v, O.DISTANCE)
    assert np.allclose(lap.dense().sum(axis=1), 0.0, atol=1e-12)
    assert np.allclose(np.diag(lap.dense()), 2.0)


def test_coincident_vertices_error():  # spectral.hpp:53-57
    v = np.array([[0.0, 0, 0], [0.0, 0, 0]])
    with pytest.raises(O.Error, match="coincident connected vertices 0 and 1"):
        O.build_laplacian(edge_submesh(), v, O.DISTANCE)


def test_dense_eig_unit_edge():
    lap = O.build_laplacian(edge_submesh(), np.array([[0.0, 0, 0], [1.0, 0, 0]]), O.BINARY)
    w, u = O.dense_eigendecomposition(lap)
    assert np.allclose(w, [0.0, 2.0], atol=1e-14)
    assert np.allclose(u[:, 0], [1 / math.sqrt(2), 1 / math.sqrt(2)], atol=1e-14)


def path_laplacian(n):
    adj = [np.array([j for j in (i - 1, i + 1) if 0 <= j < n]) for i in range(n)]
    sub = O.Submesh(np.arange(n), adj, np.array([a.size for a in adj]))
    return O.build_laplacian(sub, np.zeros((n, 3)), O.BINARY)


def test_dense_eig_path_graph():
    w, u = O.dense_eigendecomposition(path_laplacian(4))
    expect = [2 - 2 * math.cos(k * math.pi / 4) for k in range(4)]
    assert np.allclose(w, expect, atol=1e-12)
    assert np.abs(u.T @ u - np.eye(4)).max() < 1e-10


def test_shifted_inverse_2x2():
    lap = O.build_laplacian(edge_submesh(), np.array([[0.0, 0, 0], [1.0, 0, 0]]), O.BINARY)
    op1 = O.ShiftedInverseOperator(lap, 1.0, 1)
    assert np.allclose(op1.apply(np.array([[1.0], [0.0]]))[:, 0], [2 / 3, 1 / 3], atol=1e-15)
    op2 = O.ShiftedInverseOperator(lap, 1.0, 2)
    b = np.array([[1.0, 0.3], [0.0, -2.0]])
    assert np.abs(op2.apply(b) - op1.apply(op1.apply(b))).max() < 1e-12


def test_shifted_inverse_spectrum_identity():
    lap = path_laplacian(50)
    w, u = O.dense_eigendecomposition(lap)
    op = O.ShiftedInverseOperator(lap, 0.1, 1)
    R = op.apply(np.eye(50))
    assert np.allclose(np.linalg.eigvalsh(R)[::-1], 1.0 / (w + 0.1), rtol=1e-8)


def test_orthonormalize_axis():
    q = O.orthonormalize(np.array([[2.0, 0], [0, 3.0], [0, 0]]))
    assert np.array_equal(q, [[1.0, 0], [0, 1.0], [0, 0]])


def test_orthonormalize_random_span():
    b = np.random.default_rng(1).standard_normal((100, 8))
    q = O.orthonormalize(b)
    assert np.abs(q.T @ q - np.eye(8)).max() < 1e-12
    pq = q @ q.T
    pb = b @ np.linalg.solve(b.T @ b, b.T)
    assert np.abs(pq - pb).max() < 1e-10


def test_orthonormalize_rank_deficient():  # spectral.hpp:124-128
    b = np.random.default_rng(2).standard_normal((20, 4))
    b[:, 3] = b[:, 1]
    with pytest.raises(O.Error, match="rank deficient at column 3"):
        O.orthonormalize(b)
    with pytest.raises(O.Error, match=r"rank deficient \(all zero\)"):
        O.orthonormalize(np.zeros((5, 2)))
    with pytest.raises(O.InvalidArgument, match="block must be tall"):
        O.orthonormalize(np.ones((2, 3)))


def test_oi_fixed_point_and_convergence():
    lap = path_laplacian(200)
    w, u = O.dense_eigendecomposition(lap)
    op = O.ShiftedInverseOperator(lap, 1e-3, 2)
    assert O.max_principal_angle(O.orthogonal_iteration(op, u[:, :8], 3), u[:, :8]) < 1e-10
    init = O.orthonormalize(np.random.default_rng(3).standard_normal((200, 8)))
    v = init
    for _ in range(40):
        v = O.orthogonal_iteration(op, v, 1)
        assert np.linalg.norm(v.T @ v - np.eye(8)) < 1e-10
    assert O.max_principal_angle(v, u[:, :8]) < 1e-6


def test_doi_known_answers():
    lap = path_laplacian(30)
    w, u = O.dense_eigendecomposition(lap)
    op = O.ShiftedInverseOperator(lap, 1e-2, 2)
    coords = np.random.default_rng(4).standard_normal((30, 3))
    full = O.projection_residual(u, coords)
    assert np.abs(full).max() < 1e-10
    r = O.dynamic_oi(op, u[:, :10], coords, 1e-9, 1e9, 2, 30, 10)
    assert r.iterations == 1 and r.basis.shape[1] == 10 and r.converged


def test_gft_igft_known_answers():
    lap = path_laplacian(40)
    w, u = O.dense_eigendecomposition(lap)
    uc = u[:, :6]
    x = np.zeros((40, 3))
    x[:, 0] = uc[:, 0]
    c = O.gft(uc, x)
    assert np.allclose(c[:, 0], np.eye(6)[0], atol=1e-14) and np.allclose(c[:, 1:], 0)
    ortho = np.zeros((40, 3))
    ortho[:, 1] = u[:, 20]
    assert np.abs(O.gft(uc, ortho)).max() < 1e-13
    v = np.random.default_rng(5).standard_normal((40, 3))
    assert np.abs(O.igft(u, O.gft(u, v)) - v).max() < 1e-10
    errs = [np.linalg.norm(v - O.igft(u[:, :k], O.gft(u[:, :k], v))) for k in range(1, 41)]
    assert all(errs[i + 1] <= errs[i] + 1e-12 for i in range(39))


def test_weighted_stitch_degrees():
    subs = [O.Submesh(np.array([0]), [np.array([])], np.array([d])) for d in (4, 5, 6)]
    p = [np.array([[1.0, 2.0, 3.0]]), np.array([[4.0, -1.0, 0.5]]), np.array([[0.0, 7.0, -2.0]])]
    out = O.reconstruct_weighted(subs, p, 1)
    assert np.allclose(out[0], (4 * p[0][0] + 5 * p[1][0] + 6 * p[2][0]) / 15)
    with pytest.raises(O.InvalidArgument, match="reconstruction is missing 1 vertices: 1"):
        O.reconstruct_weighted(subs[:1], p[:1], 2)


def test_sign_convention_first_index_wins():  # spectral.hpp:72-85
    a = np.array([[-1.0, 2.0], [1.0, -2.0], [0.5, 0.0]])
    O.apply_sign_convention(a)
    assert np.array_equal(a, [[1.0, 2.0], [-1.0, -2.0], [-0.5, 0.0]])


def test_basis_dump_roundtrip(tmp_path):  # spectral.hpp:312-365
    b = np.random.default_rng(6).standard_normal((7, 3))
    p = str(tmp_path / "b.smb")
    O.write_basis(b, p)
    raw = open(p, "rb").read()
    assert raw[:8] == b"SMBASIS1" and len(raw) == 24 + 7 * 3 * 8
    assert np.array_equal(O.read_basis(p), b)


def _rng_ref():
    exe = os.path.join(ROOT, "oracle", "_ref", "rng_ref")
    if not os.path.exists(exe):
        subprocess.run(["g++", "-O2", "-std=c++17", "-o", exe, os.path.join(ROOT, "oracle", "rng_ref.cpp")],
                       check=True)
    return exe


@pytest.mark.parametrize("seed", [1, 42, 0x9E3779B97F4A7C15 ^ 1, 1 + 0x5851F42D4C957F2D * 3])
def test_rng_pinned_to_libstdcxx(seed):
    """mt19937_64 + normal_distribution exactly as the reference's libstdc++."""
    seed &= (1 << 64) - 1
    out = subprocess.run([_rng_ref(), str(seed), "64"], capture_output=True, text=True, check=True).stdout
    us = [int(l.split()[1]) for l in out.splitlines() if l.startswith("u ")]
    gs = [float.fromhex(l.split()[1]) for l in out.splitlines() if l.startswith("g ")]
    r = O.MT19937_64(seed)
    assert [r() for _ in range(64)] == us
    r = O.MT19937_64(seed)
    g = O.NormalDistribution()
    assert [g(r) for _ in range(64)] == gs
