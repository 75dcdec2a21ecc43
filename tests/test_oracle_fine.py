"""CPU checks of the oracle's fine-denoising restatement (denoise.hpp:11-180,
mesh.hpp:87-116) on known answers and invariants."""
import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth


def test_face_geometry_known_answer():
    v = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [0.0, 0.0, 0.0]])
    f = np.array([[0, 1, 2], [0, 1, 3]])
    cen, nrm, area, deg = O.face_geometry(v, f)
    assert np.allclose(cen[0], [1 / 3, 1 / 3, 0.0], rtol=0, atol=1e-16)
    assert nrm[0].tolist() == [0.0, 0.0, 1.0] and area[0] == 0.5
    assert nrm[1].tolist() == [0.0, 0.0, 0.0] and area[1] == 0.0 and deg.tolist() == [1]


def test_ring_adjacency():
    f = np.array([[0, 1, 2], [1, 3, 2], [3, 4, 5]])
    ring = O.face_ring_adjacency(f, 6, 1)
    assert [r.tolist() for r in ring] == [[0, 1], [0, 1, 2], [1, 2]]
    ring2 = O.face_ring_adjacency(f, 6, 2)
    assert [r.tolist() for r in ring2] == [[0, 1, 2], [0, 1, 2], [0, 1, 2]]
    with pytest.raises(O.InvalidArgument, match="ring depth must be at least 1"):
        O.face_ring_adjacency(f, 6, 0)


def test_flat_mesh_is_a_fixed_point():
    m = synth.small_grid(12, 9, 12, 9, seed=1, flip=2)
    v = m.vertices.copy()
    v[:, 2] = 0.0
    out, nrm = O.fine_denoise(v, m.faces, O.BilateralParams())
    assert np.array_equal(out, v)
    assert np.all(nrm[:, 2] == 1.0)


def test_denoise_reduces_roughness_and_errors():
    m = synth.small_grid(16, 16, 16, 16, seed=2)
    v = m.vertices.copy()
    v[:, 2] = 0.05 * np.random.default_rng(3).standard_normal(v.shape[0])
    out, _ = O.fine_denoise(v, m.faces, O.BilateralParams(normal_iterations=3, vertex_iterations=5))
    assert np.abs(out[:, 2]).mean() < np.abs(v[:, 2]).mean()
    with pytest.raises(O.InvalidArgument, match="sigma_range must be positive"):
        O.BilateralParams(sigma_range=0.0).validate()
    with pytest.raises(O.InvalidArgument, match="iteration counts and ring depth must be positive"):
        O.BilateralParams(vertex_iterations=0).validate()
    with pytest.raises(O.InvalidArgument, match="mesh has no adjacent face pairs"):
        O.fine_denoise(np.eye(3), np.array([[0, 1, 2]]), O.BilateralParams())
