"""GPU parity of fine denoising (F4, denoise.hpp:172-178) against the oracle:
geometry is computed with the reference's operation order and no FMA
contraction, the sums run in the reference's order; the only difference is
the device exp() (<= 1 ulp), so vertices and normals agree to ~1e-13."""
import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import synth

pytestmark = pytest.mark.gpu

G = pytest.importorskip("paper_1810_02719_b200")


def noisy_grid(W=40, H=30, seed=5, amp=0.05):
    m = synth.small_grid(W, H, W, H, seed=seed, flip=seed)
    v = m.vertices.copy()
    v[:, 2] = 0.2 * v[:, 2] + amp * np.random.default_rng(seed).standard_normal(v.shape[0])
    return v, m.faces


def check(v, f, gp, op, tol=1e-12):
    got, gn = G.fine_denoise(v, f, gp, return_normals=True)
    want, wn = O.fine_denoise(v, f, op)
    scale = np.abs(want).max()
    assert np.abs(got - want).max() <= tol * scale
    assert np.abs(gn - wn).max() <= tol
    return got


@pytest.mark.parametrize("kw", [{}, {"sigma_spatial": 1.5}, {"ring_depth": 2, "normal_iterations": 3},
                                {"ring_depth": 3, "normal_iterations": 2, "vertex_iterations": 3},
                                {"sigma_range": 0.2, "vertex_iterations": 4}])
def test_fine_denoise_grid(ctx, kw):
    v, f = noisy_grid()
    check(v, f, G.BilateralParams(**kw), O.BilateralParams(**kw))


def test_fine_denoise_sphere(ctx):
    m = synth.sphere_mesh(3, seed=7)
    check(m.vertices, m.faces, G.BilateralParams(), O.BilateralParams())


def test_degenerate_faces(ctx):
    """A collapsed vertex makes zero-area faces: they neither contribute nor
    get updated (denoise.hpp:84-86)."""
    v, f = noisy_grid(20, 20, seed=9)
    v[45] = v[44]
    _, _, area, deg = O.face_geometry(v, f)
    assert deg.size > 0
    check(v, f, G.BilateralParams(), O.BilateralParams())


def test_fine_denoise_errors(ctx):
    v, f = noisy_grid(8, 8, seed=1)
    with pytest.raises(G.InvalidArgument, match="sigma_range must be positive"):
        G.fine_denoise(v, f, G.BilateralParams(sigma_range=0.0))
    with pytest.raises(G.InvalidArgument, match="iteration counts and ring depth must be positive"):
        G.fine_denoise(v, f, G.BilateralParams(ring_depth=0))
    with pytest.raises(G.InvalidArgument, match="sigma_spatial must be positive"):
        G.fine_denoise(v, f, G.BilateralParams(sigma_spatial=-1.0))
    with pytest.raises(G.InvalidArgument, match="mesh has no adjacent face pairs"):
        G.fine_denoise(np.eye(3), np.array([[0, 1, 2]]), G.BilateralParams())
    bad = f.copy()
    bad[3, 1] = v.shape[0]
    with pytest.raises(G.InvalidArgument, match="face 3 references a vertex out of range"):
        G.fine_denoise(v, bad, G.BilateralParams())


def test_fine_denoise_device_pointers(ctx):
    """on_device = 1: device-resident inputs and outputs give the host path's result."""
    import ctypes as C

    import torch
    from paper_1810_02719_b200 import _abi
    v, f = noisy_grid(24, 20, seed=4)
    want, wn = G.fine_denoise(v, f, G.BilateralParams(), return_normals=True, ctx=ctx)
    dev = torch.device("cuda", 0)
    xyz = [torch.from_numpy(np.ascontiguousarray(v[:, a])).to(dev) for a in range(3)]
    df = torch.from_numpy(np.ascontiguousarray(f, dtype=np.int32)).to(dev)
    out = torch.empty(3 * v.shape[0], dtype=torch.float64, device=dev)
    nrm = torch.empty(3 * f.shape[0], dtype=torch.float64, device=dev)
    bp = _abi.smg_bilateral_params()
    ctx.lib.smg_default_bilateral_params(C.byref(bp))
    ctx.check(ctx.lib.smg_fine_denoise(ctx.handle, v.shape[0], xyz[0].data_ptr(), xyz[1].data_ptr(),
                                       xyz[2].data_ptr(), f.shape[0], df.data_ptr(), C.byref(bp), out.data_ptr(),
                                       nrm.data_ptr(), 1))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().reshape(3, -1).T, want)
    assert np.array_equal(nrm.cpu().numpy().reshape(3, -1).T, wn)
