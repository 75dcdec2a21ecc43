"""CPU tests: synthetic config inputs (sizes quoted in SURVEY.md §8(a) A1) and
the C-ABI shared library (loads, exports every symbol include/specmesh_gpu.h
declares -- no compute calls without a GPU)."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_1810_02719_b200 import _abi, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_grid_edge_counts():
    m = synth.grid_mesh(256, 256, 1, 0.005)
    assert m.n == 65536 and m.adj_cols.size // 2 == 195585  # C2 |E|
    m5 = synth.grid_mesh(512, 512, 5000, 0.01)
    assert m5.adj_cols.size // 2 == 784385  # C5 |E|
    # neighbour lists sorted, symmetric, no self loops (mesh.hpp:52-70)
    for v in (0, 257, 65535):
        nb = m.neighbors(v)
        assert np.all(np.diff(nb) > 0) and v not in nb
        for w in nb:
            assert v in m.neighbors(w)


def test_grid_tiles_cover_and_order():
    seg = synth.grid_tiles(256, 256, 32, 32)
    assert seg.count == 64 and seg.block_size == 1024
    allm = np.sort(np.concatenate(seg.members))
    assert np.array_equal(allm, np.arange(65536))
    seg5 = synth.grid_tiles(512, 512, 64, 32)
    assert seg5.count == 128 and seg5.block_size == 2048


def test_icosphere_blocks():
    m = synth.sphere_mesh(7, 303)
    assert m.n == 163842 and m.faces.shape[0] == 327680 and m.adj_cols.size // 2 == 491520
    seg = synth.sphere_blocks(m)
    assert seg.count == 160 and seg.block_size == 1026
    assert all(s.size == 1026 for s in seg.members)
    assert np.unique(np.concatenate(seg.members)).size == m.n  # every vertex covered


def test_flip_variant_differs():
    a = synth.small_grid(64, 64, 32, 32, seed=3)
    b = synth.small_grid(64, 64, 32, 32, seed=3, flip=5)
    assert a.adj_cols.size == b.adj_cols.size and not np.array_equal(a.adj_cols, b.adj_cols)


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "specmesh_gpu.h")).read()
    return sorted(set(re.findall(r"\b(smg_[a-z_]+)\s*\(", txt)))


def test_header_matches_binding_list():
    assert header_symbols() == sorted(_abi.EXPORTED)


def test_library_loads_and_exports_all_symbols():
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("libspecmesh_b200.so not built")
    lib = ctypes.CDLL(_abi.LIB_PATH)
    for name in header_symbols():
        assert hasattr(lib, name), name
    lib = _abi.load()
    assert lib.smg_abi_version() == 2
    # host-only entry points (no device work)
    assert lib.smg_default_shift(5890.0, 1024, 1e-3) == max(1e-3 * (5890.0 / 1024), 1e-300)
    cfg = _abi.smg_pipeline_config()
    lib.smg_default_config(ctypes.byref(cfg))
    assert (cfg.power, cfg.iterations, cfg.dense_limit, cfg.shift_scale, cfg.weighting) == (2, 2, 4096, 1e-8, 1)
    assert (cfg.part_count, cfg.growth) == (8, 1.15)  # pipeline.hpp:42-43


def test_no_gpu_create_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    if not os.path.exists(_abi.LIB_PATH):
        pytest.skip("libspecmesh_b200.so not built")
    import paper_1810_02719_b200 as G
    with pytest.raises(G.SpecmeshError, match="no usable sm_100 GPU"):
        G.Context(0)
