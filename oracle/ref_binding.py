"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libspecmesh_ref.so.

That library is the reference's own headers (/root/reference/proj/include,
compiled where they lie, never copied) over ``oracle/eigen_shim`` -- a stand-in
for the Eigen dependency, which is absent from this image (see
``oracle/eigen_shim/Eigen/mini_eigen.hpp`` for what that pins and what it does
not).  It exists only in a container that has /root/reference; the GPU box uses
the committed fixtures under tests/golden/ instead (tests/golden/make_ref_fixtures.py).
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libspecmesh_ref.so")

BINARY, DISTANCE = 0, 1
OI, DOI, SVD = 0, 1, 2


class RefError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class Config(C.Structure):
    """specmesh::PipelineConfig (pipeline.hpp:41-68)."""

    _fields_ = [
        ("part_count", C.c_int), ("growth", C.c_double), ("basis_mode", C.c_int), ("weighting", C.c_int),
        ("subspace_size", C.c_int), ("eps_low", C.c_double), ("eps_high", C.c_double), ("c_min", C.c_int),
        ("c_max", C.c_int), ("power", C.c_int), ("iterations", C.c_int), ("initial_iterations", C.c_int),
        ("doi_iterations", C.c_int), ("seed", C.c_ulonglong), ("dense_limit", C.c_int),
        ("shift_scale", C.c_double), ("threads", C.c_uint),
    ]


_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(LIB_PATH)
        _lib.ref_last_error.restype = C.c_char_p
        _lib.ref_mesh_edge_entries.restype = C.c_longlong
        _lib.ref_seg_adjacency_entries.restype = C.c_longlong
        _lib.ref_laplacian_nnz.restype = C.c_longlong
        _lib.ref_bases_timing.restype = C.c_double
        for name in ("ref_mesh_destroy", "ref_seg_destroy", "ref_bases_destroy", "ref_seg_assignment",
                     "ref_seg_members", "ref_seg_order", "ref_bases_members", "ref_bases_order",
                     "ref_bases_basis", "ref_bases_stats", "ref_mesh_edges_csr", "ref_default_config"):
            getattr(_lib, name).restype = None
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise RefError(status, lib().ref_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _col(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def default_config(**kw) -> Config:
    c = Config()
    lib().ref_default_config(C.byref(c))
    for k, v in kw.items():
        if not hasattr(c, k):
            raise AttributeError(k)
        setattr(c, k, v)
    return c


class Mesh:
    def __init__(self, vertices: np.ndarray, faces: np.ndarray):
        v = np.ascontiguousarray(vertices, dtype=np.float64)
        f = np.ascontiguousarray(faces, dtype=np.int32)
        self.n = int(v.shape[0])
        self.h = C.c_void_p()
        _check(lib().ref_mesh_create(self.n, _p(v), int(f.shape[0]), _p(f), C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_mesh_destroy(self.h)
            self.h = None

    def edges_csr(self):
        """build_edges (mesh.hpp:52-70) as CSR."""
        nnz = lib().ref_mesh_edge_entries(self.h)
        offs = np.zeros(self.n + 1, dtype=np.int64)
        cols = np.zeros(nnz, dtype=np.int32)
        lib().ref_mesh_edges_csr(self.h, _p(offs), _p(cols))
        return offs, cols


class Segmentation:
    def __init__(self, handle, mesh: Mesh):
        self.h = handle
        self.mesh = mesh

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_seg_destroy(self.h)
            self.h = None

    @classmethod
    def segment_mesh(cls, mesh: Mesh, cfg: Config) -> "Segmentation":
        h = C.c_void_p()
        _check(lib().ref_segment_mesh(mesh.h, C.byref(cfg), C.byref(h)))
        return cls(h, mesh)

    @classmethod
    def from_members(cls, mesh: Mesh, members: Sequence[np.ndarray], sequence) -> "Segmentation":
        offs = np.zeros(len(members) + 1, dtype=np.int64)
        offs[1:] = np.cumsum([len(m) for m in members])
        ids = np.ascontiguousarray(np.concatenate(members), dtype=np.int32)
        seq = np.ascontiguousarray(sequence, dtype=np.int32)
        h = C.c_void_p()
        _check(lib().ref_segmentation_from_members(mesh.h, len(members), _p(offs), _p(ids), _p(seq), C.byref(h)))
        return cls(h, mesh)

    @property
    def count(self) -> int:
        return lib().ref_seg_count(self.h)

    def assignment(self) -> np.ndarray:
        out = np.zeros(self.mesh.n, dtype=np.int32)
        lib().ref_seg_assignment(self.h, _p(out))
        return out

    def members(self) -> List[np.ndarray]:
        res = []
        for i in range(self.count):
            m = np.zeros(lib().ref_seg_size(self.h, i), dtype=np.int32)
            lib().ref_seg_members(self.h, i, _p(m))
            res.append(m)
        return res

    def order(self) -> np.ndarray:
        out = np.zeros(self.count, dtype=np.int32)
        lib().ref_seg_order(self.h, _p(out))
        return out

    def laplacian(self, sid: int, weighting: int, shift_scale: float):
        """(offsets, cols, vals, trace, delta) of build_laplacian / default_shift."""
        n = lib().ref_seg_size(self.h, sid)
        nnz = lib().ref_laplacian_nnz(self.h, sid)
        offs = np.zeros(n + 1, dtype=np.int32)
        cols = np.zeros(nnz, dtype=np.int32)
        vals = np.zeros(nnz, dtype=np.float64)
        tr, de = C.c_double(), C.c_double()
        _check(lib().ref_laplacian(self.mesh.h, self.h, sid, weighting, C.c_double(shift_scale), _p(offs), _p(cols),
                                   _p(vals), C.byref(tr), C.byref(de)))
        return offs, cols, vals, tr.value, de.value

    def apply(self, sid: int, weighting: int, shift_scale: float, z: int, block: np.ndarray) -> np.ndarray:
        b = _col(block)
        out = np.zeros_like(b, order="F")
        _check(lib().ref_apply(self.mesh.h, self.h, sid, weighting, C.c_double(shift_scale), z, b.shape[1], _p(b),
                               _p(out)))
        return out

    def bottom_subspace(self, sid: int, weighting: int, c: int):
        n = lib().ref_seg_size(self.h, sid)
        ev = np.zeros(n)
        basis = np.zeros((n, c), order="F")
        _check(lib().ref_bottom_subspace(self.mesh.h, self.h, sid, weighting, c, _p(ev), _p(basis)))
        return ev, basis

    def orthogonal_iteration(self, sid: int, weighting: int, shift_scale: float, z: int, init: np.ndarray,
                             t_max: int) -> np.ndarray:
        b = _col(init)
        out = np.zeros_like(b, order="F")
        _check(lib().ref_orthogonal_iteration(self.mesh.h, self.h, sid, weighting, C.c_double(shift_scale), z,
                                              b.shape[1], _p(b), t_max, _p(out)))
        return out

    def dynamic_oi(self, sid: int, weighting: int, shift_scale: float, z: int, init: np.ndarray, eps_low: float,
                   eps_high: float, c_min: int, c_max: int, t_max: int):
        b = _col(init)
        n = b.shape[0]
        out = np.zeros((n, c_max), order="F")
        oc, it, conv, res = C.c_int(), C.c_int(), C.c_int(), C.c_double()
        _check(lib().ref_dynamic_oi(self.mesh.h, self.h, sid, weighting, C.c_double(shift_scale), z, b.shape[1], _p(b),
                                    C.c_double(eps_low), C.c_double(eps_high), c_min, c_max, t_max, _p(out),
                                    C.byref(oc), C.byref(it), C.byref(conv), C.byref(res)))
        return np.ascontiguousarray(out[:, :oc.value]), it.value, bool(conv.value), res.value


class BlockBases:
    def __init__(self, handle, mesh: Mesh):
        self.h = handle
        self.mesh = mesh

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_bases_destroy(self.h)
            self.h = None

    @property
    def count(self) -> int:
        return lib().ref_bases_count(self.h)

    def members(self) -> List[np.ndarray]:
        res = []
        for i in range(self.count):
            m = np.zeros(lib().ref_bases_size(self.h, i), dtype=np.int32)
            lib().ref_bases_members(self.h, i, _p(m))
            res.append(m)
        return res

    def order(self) -> np.ndarray:
        out = np.zeros(self.count, dtype=np.int32)
        lib().ref_bases_order(self.h, _p(out))
        return out

    def basis(self, sid: int) -> np.ndarray:
        out = np.zeros((lib().ref_bases_size(self.h, sid), lib().ref_bases_c(self.h, sid)), order="F")
        lib().ref_bases_basis(self.h, sid, _p(out))
        return out

    def stats(self, sid: int) -> dict:
        s = np.zeros(5)
        lib().ref_bases_stats(self.h, int(sid), _p(s))
        return {"subspace_size": int(s[0]), "residual_rms": float(s[1]), "doi_residual": float(s[2]),
                "converged": bool(s[3]), "oi_iterations": int(s[4])}

    def coefficients(self, sid: int) -> np.ndarray:
        out = np.zeros((lib().ref_bases_c(self.h, sid), 3), order="F")
        _check(lib().ref_bases_coefficients(self.h, self.mesh.h, sid, _p(out)))
        return out

    def reconstruct(self, weighted: bool = True) -> np.ndarray:
        out = np.zeros((self.mesh.n, 3))
        _check(lib().ref_bases_reconstruct(self.h, self.mesh.h, int(weighted), _p(out)))
        return out

    def timing(self, stage: str) -> float:
        return lib().ref_bases_timing(self.h, stage.encode())


def chain_fixed(mesh: Mesh, seg: Segmentation, cfg: Config, sizes_in_order) -> BlockBases:
    """compute_block_bases_fixed_sizes (pipeline.hpp:144-194)."""
    sizes = np.ascontiguousarray(sizes_in_order, dtype=np.int32)
    h = C.c_void_p()
    _check(lib().ref_chain_fixed(mesh.h, seg.h, C.byref(cfg), _p(sizes), C.byref(h)))
    return BlockBases(h, mesh)


def chain(mesh: Mesh, cfg: Config) -> BlockBases:
    """compute_block_bases (pipeline.hpp:198-285): segments internally."""
    h = C.c_void_p()
    _check(lib().ref_chain(mesh.h, C.byref(cfg), C.byref(h)))
    return BlockBases(h, mesh)


def chain_doi_external(mesh: Mesh, seg: Segmentation, cfg: Config) -> BlockBases:
    """the DOI branch (pipeline.hpp:245-285) over an external segmentation (C4's tiles)."""
    h = C.c_void_p()
    _check(lib().ref_chain_doi_external(mesh.h, seg.h, C.byref(cfg), C.byref(h)))
    return BlockBases(h, mesh)


def orthonormalize(block: np.ndarray) -> np.ndarray:
    b = _col(block)
    out = np.zeros_like(b, order="F")
    _check(lib().ref_orthonormalize(b.shape[0], b.shape[1], _p(b), _p(out)))
    return out


def resize_basis(basis: np.ndarray, new_size: int, seed: int) -> np.ndarray:
    b = _col(basis)
    out = np.zeros((b.shape[0], new_size), order="F")
    _check(lib().ref_resize_basis(b.shape[0], b.shape[1], _p(b), new_size, C.c_ulonglong(seed), _p(out)))
    return out


def max_principal_angle(a: np.ndarray, b: np.ndarray) -> float:
    a, b = _col(a), _col(b)
    out = C.c_double()
    _check(lib().ref_max_principal_angle(a.shape[0], a.shape[1], _p(a), _p(b), C.byref(out)))
    return out.value


def compress(mesh: Mesh, cfg: Config, quant_bits: int) -> bytes:
    """serialize_encoded_mesh(compress_mesh(mesh, {cfg, quant_bits})) (compress.hpp:152-219, :378-420)."""
    n = C.c_longlong()
    _check(lib().ref_compress(mesh.h, C.byref(cfg), quant_bits, None, C.c_longlong(0), C.byref(n)))
    buf = np.zeros(n.value, dtype=np.uint8)
    _check(lib().ref_compress(mesh.h, C.byref(cfg), quant_bits, _p(buf), C.c_longlong(n.value), C.byref(n)))
    return buf.tobytes()


def decompress(data: bytes, n: int) -> np.ndarray:
    """decompress_mesh(parse_encoded_mesh(data)).vertices (compress.hpp:210-262, :422-474)."""
    buf = np.frombuffer(data, dtype=np.uint8).copy()
    out = np.zeros((n, 3))
    _check(lib().ref_decompress(_p(buf), C.c_longlong(buf.size), _p(out), n))
    return out


def fine_denoise(mesh: Mesh, nf: int, sigma_spatial=0.0, sigma_range=0.35, normal_iterations=5, vertex_iterations=10,
                 ring_depth=1):
    """fine_denoise (denoise.hpp:175-180) -> (vertices n x 3, filtered normals nf x 3)."""
    out = np.zeros((mesh.n, 3))
    nrm = np.zeros((nf, 3))
    _check(lib().ref_fine_denoise(mesh.h, C.c_double(sigma_spatial), C.c_double(sigma_range), normal_iterations,
                                  vertex_iterations, ring_depth, _p(out), _p(nrm)))
    return out, nrm


def denoise_dynamic(mesh: Mesh, frames: Sequence[np.ndarray], cfg: Config, weighted: bool = True):
    """denoise_dynamic (denoise.hpp:258-291); ``mesh`` is frame 0 (connectivity shared)."""
    x = np.ascontiguousarray(np.stack(frames), dtype=np.float64)
    out = np.zeros_like(x)
    nb = C.c_int()
    _check(lib().ref_denoise_dynamic(mesh.h, x.shape[0], _p(x), C.byref(cfg), int(weighted), _p(out), C.byref(nb)))
    return out, nb.value
