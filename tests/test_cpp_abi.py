"""The C ABI called from compiled C++ through include/specmesh_gpu.hpp
(tests/cpp/abi_chain.cpp, built by `make`), not from ctypes: the same chain as
the Python path on the same inputs (pipeline.hpp:144-194, :245-285)."""
import os
import struct
import subprocess

import numpy as np
import pytest

from paper_1810_02719_b200 import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "build", "abi_chain")


def write_input(path, mesh, seg, mode, c, t, c_min=1, c_max=0, eps=(1e-5, 1e-4), scale=1e-3):
    nd = seg.block_size
    with open(path, "wb") as f:
        f.write(struct.pack("<q", mesh.n))
        f.write(struct.pack("<8i", int(mesh.adj_offsets[-1]), seg.count, nd, mode, c, t, c_min, c_max))
        f.write(struct.pack("<3d", eps[0], eps[1], scale))
        f.write(np.ascontiguousarray(mesh.vertices.T, dtype="<f8").tobytes())
        f.write(np.asarray(mesh.adj_offsets, dtype="<i4").tobytes())
        f.write(np.asarray(mesh.adj_cols, dtype="<i4").tobytes())
        for m in seg.members:
            f.write(np.sort(np.asarray(m)).astype("<i4").tobytes())
        f.write(np.asarray(seg.sequence, dtype="<i4").tobytes())


def read_output(path, k, n):
    data = open(path, "rb").read()
    (status,) = struct.unpack_from("<i", data, 0)
    if status != 0:
        return status, data[4:].decode(), None
    off, tiles = 4, []
    for _ in range(k):
        c, rms, doi, conv, its = struct.unpack_from("<iddii", data, off)
        off += struct.calcsize("<iddii")
        coef = np.frombuffer(data, "<f8", 3 * c, off).reshape(3, c).T
        off += 24 * c
        tiles.append((c, rms, doi, conv, its, coef))
    recon = np.frombuffer(data, "<f8", 3 * n, off).reshape(3, n).T
    return status, tiles, recon


def test_cpp_caller_builds_and_reports_status(tmp_path):
    """CPU: the compiled caller links against the library; a bad input is the
    reference's InvalidArgument (status 2) with its text, and without a GPU
    smg_create fails cleanly (status 3) -- no CPU fallback."""
    assert os.path.exists(EXE), "build/abi_chain missing: run make"
    bad = tmp_path / "bad.bin"
    bad.write_bytes(b"")
    out = tmp_path / "o.bin"
    r = subprocess.run([EXE, str(bad), str(out)])
    assert r.returncode == 2
    assert read_output(str(out), 0, 0)[1] == "short input file"
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        mesh = synth.small_grid(64, 32, 32, 32, seed=3)
        seg = synth.grid_tiles(64, 32, 32, 32)
        inp = tmp_path / "in.bin"
        write_input(str(inp), mesh, seg, 0, 20, 1)
        r = subprocess.run([EXE, str(inp), str(out)])
        assert r.returncode == 3
        st, msg, _ = read_output(str(out), seg.count, mesh.n)
        assert st == 3 and "smg_create failed" in msg


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1])
def test_cpp_caller_matches_python_path(ctx, tmp_path, mode):
    import paper_1810_02719_b200 as G
    mesh = synth.small_grid(128, 64, 32, 32, seed=4, flip=8)
    seg = synth.grid_tiles(128, 64, 32, 32)
    inp, out = tmp_path / "in.bin", tmp_path / "out.bin"
    if mode == 0:
        write_input(str(inp), mesh, seg, 0, 60, 2)
        cfg = G.PipelineConfig(weighting="binary", subspace_size=60, iterations=2, shift_scale=1e-3)
        bb = G.compute_block_bases_fixed_sizes(mesh, seg, cfg, [60] * seg.count, ctx=ctx)
    else:
        kw = dict(subspace_size=20, c_min=10, c_max=120, eps_low=3e-4, eps_high=3e-3)
        write_input(str(inp), mesh, seg, 1, 20, 1, c_min=10, c_max=120, eps=(3e-4, 3e-3))
        cfg = G.PipelineConfig(weighting="binary", basis_mode="doi", shift_scale=1e-3, **kw)
        bb = G.compute_block_bases(mesh, seg, cfg, ctx=ctx)
    r = subprocess.run([EXE, str(inp), str(out)])
    assert r.returncode == 0
    st, tiles, recon = read_output(str(out), seg.count, mesh.n)
    assert st == 0
    # same library, same kernels, same inputs: identical results
    assert np.array_equal(recon, bb.reconstruction)
    for i, (c, rms, doi, conv, its, coef) in enumerate(tiles):
        s = bb.stats[i]
        assert (c, rms, doi, bool(conv), its) == (s.subspace_size, s.residual_rms, s.doi_residual, s.converged,
                                                 s.oi_iterations)
        assert np.array_equal(coef, bb.coefficients[i])
