"""paper_1810_02719_b200 -- B200-native OI spectral path of arXiv 1810.02719.

Python mirror of the reference's path API (``specmesh`` C++ headers, cited
file:line in each function) on top of the C ABI of ``libspecmesh_b200.so``
(include/specmesh_gpu.h).  Same names, argument meaning and error behaviour:
preconditions raise :class:`InvalidArgument` (reference ``require``,
core.hpp:36-38) and numerical failures raise :class:`SpecmeshError` with the
reference's message text (core.hpp:18-22).  Matrices are numpy arrays in the
reference's orientation (n x c bases, n x 3 points).

Every compute call runs sm_100a kernels; nothing here falls back to the CPU.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import List, Optional, Sequence

import numpy as np

from . import _abi

__all__ = [
    "SpecmeshError", "InvalidArgument", "ParseError", "Context", "PipelineConfig", "BlockBases", "default_context",
    "build_laplacian", "default_shift", "ShiftedInverseOperator", "orthonormalize", "orthogonal_iteration",
    "dynamic_oi", "bottom_subspace", "gft", "igft", "compute_block_bases_fixed_sizes", "compute_block_bases",
    "run_chains", "coarse_reconstruct_points", "coarse_reconstruct_frames", "DynamicDenoiseResult",
    "denoise_dynamic", "BilateralParams", "fine_denoise",
]


class SpecmeshError(RuntimeError):
    """specmesh::Error (core.hpp:18-22)."""


class InvalidArgument(SpecmeshError):
    """specmesh::InvalidArgument (core.hpp:24-28)."""


class ParseError(SpecmeshError):
    """specmesh::ParseError (core.hpp:30-34)."""


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else C.c_void_p(a.ctypes.data)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _colmajor(a: np.ndarray) -> np.ndarray:
    """Eigen column-major storage of an (rows, cols) array."""
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


class Context:
    """One CUDA device + stream (smg_create)."""

    def __init__(self, device: int = 0):
        self.lib = _abi.load()
        h = C.c_void_p()
        st = self.lib.smg_create(device, C.byref(h))
        if st != _abi.SMG_OK:
            raise SpecmeshError(f"smg_create failed on device {device} (status {st}): no usable sm_100 GPU")
        self.handle = h
        self.device = device

    def check(self, status: int) -> None:
        if status == _abi.SMG_OK:
            return
        msg = self.lib.smg_last_error(self.handle).decode()
        if status == _abi.SMG_INVALID_ARGUMENT:
            raise InvalidArgument(msg)
        if status == _abi.SMG_PARSE_ERROR:
            raise ParseError(msg)
        raise SpecmeshError(msg)

    def doi_trace(self, on: bool = True) -> None:
        """Start (clear) or stop the DOI step log (smg_doi_trace_enable)."""
        self.check(self.lib.smg_doi_trace_enable(self.handle, 1 if on else 0))

    def read_doi_trace(self):
        """(position, subspace size the step ran with, residual) per logged DOI step."""
        n = C.c_int64()
        self.check(self.lib.smg_doi_trace_read(self.handle, 0, None, None, None, C.byref(n)))
        pos = np.zeros(n.value, np.int32)
        c = np.zeros(n.value, np.int32)
        r = np.zeros(n.value, np.float64)
        if n.value:
            self.check(self.lib.smg_doi_trace_read(self.handle, n.value, _ptr(pos), _ptr(c), _ptr(r), C.byref(n)))
        return pos, c, r

    def last_run_info(self) -> dict:
        """What the last chain call chose (smg_last_run_info): block width,
        ordering (natural / geometric / rcm), chain groups, batch shape."""
        ri = _abi.smg_run_info()
        self.check(self.lib.smg_last_run_info(self.handle, C.byref(ri)))
        return {"block_width": ri.block_width, "ordering": ["natural", "geometric", "rcm"][ri.ordering],
                "chain_groups": ri.chain_groups, "chains": ri.chains, "positions": ri.positions}

    def close(self) -> None:
        if getattr(self, "handle", None):
            self.lib.smg_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


@dataclasses.dataclass
class PipelineConfig:
    """PipelineConfig (pipeline.hpp:41-68), path fields, reference defaults."""

    weighting: str = "distance"
    basis_mode: str = "oi"
    subspace_size: int = 16
    eps_low: float = 0.004
    eps_high: float = 0.04
    c_min: int = 2
    c_max: int = 0
    power: int = 2
    iterations: int = 2
    initial_iterations: int = 60
    doi_iterations: int = 0
    seed: int = 1
    dense_limit: int = 4096
    shift_scale: float = 1e-8
    part_count: int = 8      # segment_mesh k (used when no Segmentation is given)
    growth: float = 1.15     # overlap factor

    def to_c(self) -> _abi.smg_pipeline_config:
        if self.weighting not in _abi.WEIGHTING:
            raise InvalidArgument(f"unknown weighting '{self.weighting}' (expected binary|distance)")
        if self.basis_mode not in _abi.BASIS_MODE:
            raise InvalidArgument(f"unknown basis mode '{self.basis_mode}' (expected oi|doi)")
        return _abi.smg_pipeline_config(
            _abi.WEIGHTING[self.weighting], _abi.BASIS_MODE[self.basis_mode], self.subspace_size, self.eps_low,
            self.eps_high, self.c_min, self.c_max, self.power, self.iterations, self.initial_iterations,
            self.doi_iterations, self.seed & ((1 << 64) - 1), self.dense_limit, self.shift_scale, self.part_count,
            self.growth)


# ------------------------------------------------------------------ L3 primitives

def _mesh_view(mesh, keep: list) -> _abi.smg_mesh:
    x = _f64(mesh.vertices[:, 0])
    y = _f64(mesh.vertices[:, 1])
    z = _f64(mesh.vertices[:, 2])
    offs = _i32(mesh.adj_offsets)
    cols = _i32(mesh.adj_cols)
    keep += [x, y, z, offs, cols]
    return _abi.smg_mesh(mesh.n, x.ctypes.data, y.ctypes.data, z.ctypes.data, offs.ctypes.data,
                         cols.ctypes.data, 0)


def _seg_view(seg, keep: list) -> _abi.smg_segmentation:
    offs, ids = seg.flat()
    seq = _i32(seg.sequence)
    keep += [offs, ids, seq]
    return _abi.smg_segmentation(seg.count, offs.ctypes.data, ids.ctypes.data, int(seq.size), seq.ctypes.data, 0)


def build_laplacian(mesh, members, weighting: str = "distance", ctx: Optional[Context] = None):
    """build_submesh adjacency + build_laplacian (partition.hpp:169-184,
    spectral.hpp:39-68).  Returns (rowptr, cols, vals, trace) of L = D - C."""
    ctx = ctx or default_context()
    keep: list = []
    mv = _mesh_view(mesh, keep)
    mem = _i32(np.sort(np.asarray(members)))
    n = int(mem.size)
    cap = int(n + np.diff(mesh.adj_offsets)[mem].sum())
    rowptr = np.empty(n + 1, np.int32)
    cols = np.empty(cap, np.int32)
    vals = np.empty(cap, np.float64)
    nnz = C.c_int64()
    tr = C.c_double()
    ctx.check(ctx.lib.smg_build_laplacian(ctx.handle, C.byref(mv), _ptr(mem), n, _abi.WEIGHTING[weighting],
                                          _ptr(rowptr), _ptr(cols), _ptr(vals), cap, C.byref(nnz), C.byref(tr)))
    k = nnz.value
    return rowptr, cols[:k].copy(), vals[:k].copy(), tr.value


def default_shift(trace: float, n: int, scale: float = 1e-8) -> float:
    """default_shift (spectral.hpp:193-196)."""
    return _abi.load().smg_default_shift(trace, n, scale)


class ShiftedInverseOperator:
    """ShiftedInverseOperator (spectral.hpp:145-190) on the GPU block factor."""

    def __init__(self, rowptr, cols, vals, delta: float, z: int, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self._rp, self._c, self._v = _i32(rowptr), _i32(cols), _f64(vals)
        self.n = int(self._rp.size - 1)
        self.shift_, self.power_ = float(delta), int(z)
        h = C.c_void_p()
        self.ctx.check(self.ctx.lib.smg_operator_create(self.ctx.handle, self.n, _ptr(self._rp), _ptr(self._c),
                                                        _ptr(self._v), self.shift_, self.power_, C.byref(h)))
        self.handle = h

    def size(self) -> int:
        return self.n

    def shift(self) -> float:
        return self.shift_

    def power(self) -> int:
        return self.power_

    def _call(self, block: np.ndarray, once: int) -> np.ndarray:
        block = np.asarray(block, dtype=np.float64)
        if block.ndim != 2 or block.shape[0] != self.n:
            raise InvalidArgument("operator/block dimension mismatch")
        b = _colmajor(block)
        out = np.empty_like(b, order="F")
        self.ctx.check(self.ctx.lib.smg_operator_apply(self.ctx.handle, self.handle, b.shape[1], _ptr(b),
                                                       _ptr(out), once))
        return np.ascontiguousarray(out)

    def apply_once(self, block):
        return self._call(block, 1)

    def apply(self, block):
        return self._call(block, 0)

    def spmm(self, block):
        """(L + delta I) X -- CSR SpMM kernel (K4)."""
        b = _colmajor(block)
        out = np.empty_like(b, order="F")
        self.ctx.check(self.ctx.lib.smg_operator_spmm(self.ctx.handle, self.handle, b.shape[1], _ptr(b),
                                                      _ptr(out)))
        return np.ascontiguousarray(out)

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.ctx.lib.smg_operator_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def orthonormalize(block, ctx: Optional[Context] = None) -> np.ndarray:
    """orthonormalize (spectral.hpp:120-132): CholeskyQR2 + rank test + sign convention."""
    ctx = ctx or default_context()
    block = np.asarray(block, dtype=np.float64)
    rows, cols = block.shape
    b = _colmajor(block)
    q = np.empty_like(b, order="F")
    ctx.check(ctx.lib.smg_orthonormalize(ctx.handle, rows, cols, _ptr(b), _ptr(q)))
    return np.ascontiguousarray(q)


def orthonormality_estimate(block, ctx: Optional[Context] = None) -> float:
    """The adaptive CholeskyQR2's one-pass estimate of ||Q^T Q - I||_F (probe.cu; diagnostics)."""
    ctx = ctx or default_context()
    b = _colmajor(np.asarray(block, dtype=np.float64))
    est = C.c_double()
    ctx.check(ctx.lib.smg_orthonormality_estimate(ctx.handle, b.shape[0], b.shape[1], _ptr(b), C.byref(est)))
    return est.value


def orthogonal_iteration(op: ShiftedInverseOperator, init, t_max: int) -> np.ndarray:
    """orthogonal_iteration (spectral.hpp:204-211)."""
    init = np.asarray(init, dtype=np.float64)
    if init.shape[0] != op.n:
        raise InvalidArgument("initial basis does not match the operator size")
    b = _colmajor(init)
    out = np.empty_like(b, order="F")
    op.ctx.check(op.ctx.lib.smg_orthogonal_iteration(op.ctx.handle, op.handle, b.shape[1], _ptr(b), int(t_max),
                                                     _ptr(out)))
    return np.ascontiguousarray(out)


@dataclasses.dataclass
class DoiResult:
    """DoiResult (spectral.hpp:233-238)."""

    basis: np.ndarray
    converged: bool
    residual: float
    iterations: int


def dynamic_oi(op: ShiftedInverseOperator, init, coords, eps_low: float, eps_high: float, c_min: int, c_max: int,
               t_max: int) -> DoiResult:
    """dynamic_oi (spectral.hpp:244-287) -- the loop runs on the device."""
    init = np.asarray(init, dtype=np.float64)
    coords = np.asarray(coords, dtype=np.float64)
    if coords.shape[0] != op.n:
        raise InvalidArgument("coordinate/operator dimension mismatch")
    b = _colmajor(init)
    x = _colmajor(coords)
    cap = max(int(c_max), b.shape[1])
    out = np.empty((op.n, cap), order="F")
    c_out, conv, it = C.c_int32(), C.c_int32(), C.c_int32()
    res = C.c_double()
    op.ctx.check(op.ctx.lib.smg_dynamic_oi(op.ctx.handle, op.handle, b.shape[1], _ptr(b), _ptr(x), eps_low,
                                           eps_high, c_min, c_max, t_max, _ptr(out), C.byref(c_out),
                                           C.byref(conv), C.byref(res), C.byref(it)))
    c = c_out.value
    basis = np.ascontiguousarray(out.reshape(-1, order="F")[:op.n * c].reshape((op.n, c), order="F"))
    return DoiResult(basis, bool(conv.value), res.value, it.value)


def bottom_subspace(op: ShiftedInverseOperator, c: int, return_eigenvalues: bool = False):
    """bottom_subspace(dense_eigendecomposition(L), c) (spectral.hpp:92-117),
    produced on the GPU (shift-invert subspace iteration + Rayleigh-Ritz)."""
    out = np.empty((op.n, c), order="F")
    ev = np.empty(c)
    op.ctx.check(op.ctx.lib.smg_bottom_subspace(op.ctx.handle, op.handle, int(c), _ptr(out), _ptr(ev)))
    u = np.ascontiguousarray(out)
    return (u, ev) if return_eigenvalues else u


def gft(basis, coords, ctx: Optional[Context] = None) -> np.ndarray:
    """gft (spectral.hpp:290-293): C = U^T X."""
    ctx = ctx or default_context()
    basis = np.asarray(basis, dtype=np.float64)
    coords = np.asarray(coords, dtype=np.float64)
    if coords.shape[0] != basis.shape[0]:
        raise InvalidArgument("coordinate/basis dimension mismatch")
    u, x = _colmajor(basis), _colmajor(coords)
    out = np.empty((basis.shape[1], 3), order="F")
    ctx.check(ctx.lib.smg_gft(ctx.handle, basis.shape[0], basis.shape[1], _ptr(u), _ptr(x), _ptr(out)))
    return np.ascontiguousarray(out)


def igft(basis, coeffs, ctx: Optional[Context] = None) -> np.ndarray:
    """igft (spectral.hpp:295-298): X^ = U C."""
    ctx = ctx or default_context()
    basis = np.asarray(basis, dtype=np.float64)
    coeffs = np.asarray(coeffs, dtype=np.float64)
    if coeffs.shape[0] != basis.shape[1]:
        raise InvalidArgument("coefficient/basis dimension mismatch")
    u, cf = _colmajor(basis), _colmajor(coeffs)
    out = np.empty((basis.shape[0], 3), order="F")
    ctx.check(ctx.lib.smg_igft(ctx.handle, basis.shape[0], basis.shape[1], _ptr(u), _ptr(cf), _ptr(out)))
    return np.ascontiguousarray(out)


# ------------------------------------------------------------------ L4 chain

@dataclasses.dataclass
class BlockStats:
    """BlockStats (pipeline.hpp:70-76)."""

    subspace_size: int
    residual_rms: float
    doi_residual: float
    converged: bool
    oi_iterations: int


@dataclasses.dataclass
class BlockBases:
    """BlockBases (pipeline.hpp:78-92) + the path outputs: per-id coefficients
    (gft) and the stitched coarse reconstruction (coarse_reconstruct_points)."""

    sequence: np.ndarray
    stats: List[BlockStats]
    bases: Optional[List[np.ndarray]]
    coefficients: Optional[List[np.ndarray]]
    reconstruction: Optional[np.ndarray]
    timings: dict
    block_size: int

    def sizes_in_order(self) -> List[int]:
        return [self.stats[i].subspace_size for i in self.sequence]


class _Out:
    def __init__(self, k: int, n_d: int, nv: int, cap_c: int, want_bases: bool, want_coeffs: bool,
                 want_recon: bool):
        self.ss = np.zeros(k, np.int32)
        self.rms = np.zeros(k)
        self.doi = np.zeros(k)
        self.conv = np.zeros(k, np.int32)
        self.it = np.zeros(k, np.int32)
        self.recon = np.zeros(nv * 3) if want_recon else None
        self.coef = np.zeros(k * cap_c * 3) if want_coeffs else None
        self.coef_off = np.zeros(k + 1, np.int64)
        self.bases = np.zeros(k * cap_c * n_d) if want_bases else None
        self.basis_off = np.zeros(k + 1, np.int64)
        self.k, self.n_d, self.nv = k, n_d, nv

    def c(self) -> _abi.smg_chain_output:
        o = _abi.smg_chain_output()
        o.subspace_size = self.ss.ctypes.data
        o.residual_rms = self.rms.ctypes.data
        o.doi_residual = self.doi.ctypes.data
        o.converged = self.conv.ctypes.data
        o.oi_iterations = self.it.ctypes.data
        o.reconstruction = None if self.recon is None else self.recon.ctypes.data
        o.coefficients = None if self.coef is None else self.coef.ctypes.data
        o.coefficients_capacity = 0 if self.coef is None else self.coef.size
        o.coefficient_offsets = self.coef_off.ctypes.data
        o.bases = None if self.bases is None else self.bases.ctypes.data
        o.bases_capacity = 0 if self.bases is None else self.bases.size
        o.basis_offsets = self.basis_off.ctypes.data
        o.on_device = 0
        self._c = o
        return o

    def result(self, sequence) -> BlockBases:
        o = self._c
        stats = [BlockStats(int(self.ss[i]), float(self.rms[i]), float(self.doi[i]), bool(self.conv[i]),
                            int(self.it[i])) for i in range(self.k)]
        coeffs = None
        if self.coef is not None:
            coeffs = [self.coef[self.coef_off[i]:self.coef_off[i + 1]].reshape((3, -1)).T.copy()
                      for i in range(self.k)]
        bases = None
        if self.bases is not None:
            bases = [self.bases[self.basis_off[i]:self.basis_off[i + 1]].reshape((-1, self.n_d)).T.copy()
                     for i in range(self.k)]
        recon = None if self.recon is None else self.recon.reshape((3, self.nv)).T.copy()
        names = ["laplacian", "factorize", "basis", "basis_total", "project", "total"]
        timings = {nm: float(o.timings[i]) for i, nm in enumerate(names)}
        return BlockBases(np.asarray(sequence), stats, bases, coeffs, recon, timings, self.n_d)


def compute_block_bases_fixed_sizes(mesh, seg, cfg: PipelineConfig, sizes_in_order: Sequence[int],
                                    want_bases: bool = False, want_coeffs: bool = True, want_recon: bool = True,
                                    ctx: Optional[Context] = None) -> BlockBases:
    """compute_block_bases_fixed_sizes (pipeline.hpp:144-194) followed by
    coarse_reconstruct_points (pipeline.hpp:300-305) when ``want_recon``."""
    ctx = ctx or default_context()
    sizes = _i32(sizes_in_order)
    if sizes.size != seg.count:
        raise InvalidArgument("need one subspace size per block")
    keep: list = []
    mv, sv = _mesh_view(mesh, keep), _seg_view(seg, keep)
    out = _Out(seg.count, seg.block_size, mesh.n, int(sizes.max()), want_bases, want_coeffs, want_recon)
    oc = out.c()
    cc = cfg.to_c()
    ctx.check(ctx.lib.smg_compute_block_bases_fixed_sizes(ctx.handle, C.byref(mv), C.byref(sv), C.byref(cc),
                                                          _ptr(sizes), C.byref(oc)))
    return out.result(seg.sequence)


def compute_block_bases(mesh, seg, cfg: PipelineConfig, want_bases: bool = False, want_coeffs: bool = True,
                        want_recon: bool = True, ctx: Optional[Context] = None) -> BlockBases:
    """compute_block_bases (pipeline.hpp:198-287), OI or DOI.  ``seg=None`` is
    the reference's own flow: the mesh is segmented on the GPU first
    (segment_mesh with cfg.part_count / growth / seed, pipeline.hpp:201); the
    result's ``sequence`` / ``block_size`` are the segmentation's (call
    segment_mesh for the member lists).  Bases need an explicit segmentation."""
    ctx = ctx or default_context()
    if seg is None:
        if want_bases:
            raise InvalidArgument("want_bases needs an explicit segmentation (segment_mesh)")
        keep = []
        mv = _mesh_view(mesh, keep)
        k = int(cfg.part_count)
        cap = cfg.subspace_size
        if cfg.basis_mode == "doi":
            cap = cfg.c_max if cfg.c_max > 0 else max(64, 2 * cfg.subspace_size)
        out = _Out(k, 0, mesh.n, max(cap, 1), False, want_coeffs, want_recon)
        oc = out.c()
        seq = np.zeros(k, np.int32)
        oc.sequence_out = seq.ctypes.data
        cc = cfg.to_c()
        ctx.check(ctx.lib.smg_compute_block_bases(ctx.handle, C.byref(mv), None, C.byref(cc), C.byref(oc)))
        out.n_d = int(oc.block_size)
        return out.result(seq)
    keep: list = []
    mv, sv = _mesh_view(mesh, keep), _seg_view(seg, keep)
    n_d = seg.block_size
    if cfg.basis_mode == "doi":
        cm = cfg.c_max if cfg.c_max > 0 else max(64, 2 * cfg.subspace_size)
        cap = min(cm, n_d)
    else:
        cap = cfg.subspace_size
    out = _Out(seg.count, n_d, mesh.n, max(cap, 1), want_bases, want_coeffs, want_recon)
    oc = out.c()
    cc = cfg.to_c()
    ctx.check(ctx.lib.smg_compute_block_bases(ctx.handle, C.byref(mv), C.byref(sv), C.byref(cc), C.byref(oc)))
    return out.result(seg.sequence)


# ------------------------------------------------------------------ segmentation (F1)

def partition_mesh(mesh, k: int, seed: int = 1, ctx: Optional[Context] = None) -> np.ndarray:
    """partition_mesh (partition.hpp:84-159) on the GPU: per-vertex part id."""
    ctx = ctx or default_context()
    keep: list = []
    mv = _mesh_view(mesh, keep)
    a = np.empty(mesh.n, np.int32)
    ctx.check(ctx.lib.smg_partition_mesh(ctx.handle, C.byref(mv), int(k), seed & ((1 << 64) - 1), _ptr(a)))
    return a


def expand_overlaps(mesh, assignment, k: int, growth: float, ctx: Optional[Context] = None) -> List[np.ndarray]:
    """expand_overlaps (partition.hpp:205-253) on the GPU: k sorted member lists of n_d."""
    ctx = ctx or default_context()
    keep: list = []
    mv = _mesh_view(mesh, keep)
    a = _i32(assignment)
    nd = C.c_int32()
    st = ctx.lib.smg_expand_overlaps(ctx.handle, C.byref(mv), _ptr(a), int(k), float(growth), None, 0, C.byref(nd))
    if nd.value <= 0:
        ctx.check(st)
    mem = np.empty(int(k) * nd.value, np.int32)
    ctx.check(ctx.lib.smg_expand_overlaps(ctx.handle, C.byref(mv), _ptr(a), int(k), float(growth), _ptr(mem),
                                          mem.size, C.byref(nd)))
    return [mem[i * nd.value:(i + 1) * nd.value].copy() for i in range(int(k))]


def order_submeshes(members: Sequence[np.ndarray], seed: int = 1, ctx: Optional[Context] = None) -> np.ndarray:
    """order_submeshes (partition.hpp:258-307) on the GPU."""
    ctx = ctx or default_context()
    offs = np.zeros(len(members) + 1, np.int32)
    offs[1:] = np.cumsum([len(m) for m in members])
    flat = _i32(np.concatenate([np.asarray(m) for m in members])) if len(members) else np.zeros(0, np.int32)
    seq = np.empty(len(members), np.int32)
    ctx.check(ctx.lib.smg_order_submeshes(ctx.handle, len(members), _ptr(offs), _ptr(flat), seed & ((1 << 64) - 1),
                                          _ptr(seq)))
    return seq


def segment_mesh(mesh, part_count: int = 8, growth: float = 1.15, seed: int = 1, ctx: Optional[Context] = None,
                 return_assignment: bool = False):
    """segment_mesh (pipeline.hpp:131-138) on the GPU -> synth.Segmentation
    (sorted member lists by submesh id + the SubmeshOrder sequence)."""
    from .synth import Segmentation
    ctx = ctx or default_context()
    keep: list = []
    mv = _mesh_view(mesh, keep)
    nd = C.c_int32()
    k = int(part_count)
    seq = np.empty(k, np.int32)
    a = np.empty(mesh.n, np.int32)
    # parts stay near cap = int(ceil(n/k) * 1.1) (beyond it only once every part is capped):
    # size the member buffer for that (a second call only in the rare case)
    cap = int(math.ceil(mesh.n / max(k, 1)) * 1.1) if k >= 1 else 1
    guess = max(1, min(mesh.n, int(math.floor(float(growth) * 2 * cap)) + 1))
    mem = np.empty(max(k, 1) * guess, np.int32)
    st = ctx.lib.smg_segment_mesh(ctx.handle, C.byref(mv), k, float(growth), seed & ((1 << 64) - 1), _ptr(a),
                                  _ptr(mem), mem.size, C.byref(nd), _ptr(seq))
    if st != _abi.SMG_OK:
        if nd.value <= 0 or k * nd.value <= mem.size:
            ctx.check(st)
        mem = np.empty(k * nd.value, np.int32)
        ctx.check(ctx.lib.smg_segment_mesh(ctx.handle, C.byref(mv), k, float(growth), seed & ((1 << 64) - 1),
                                           _ptr(a), _ptr(mem), mem.size, C.byref(nd), _ptr(seq)))
    segm = Segmentation([mem[i * nd.value:(i + 1) * nd.value].copy() for i in range(int(part_count))], seq)
    return (segm, a) if return_assignment else segm


def run_chains(meshes, segs, cfg: PipelineConfig, sizes_in_order: Sequence[int], want_bases: bool = False,
               want_coeffs: bool = True, want_recon: bool = True, ctx: Optional[Context] = None) -> List[BlockBases]:
    """Independent fixed-size chains in lockstep on one GPU (smg_run_chains)."""
    ctx = ctx or default_context()
    sizes = _i32(sizes_in_order)
    keep: list = []
    B = len(meshes)
    mvs = (_abi.smg_mesh * B)(*[_mesh_view(m, keep) for m in meshes])
    svs = (_abi.smg_segmentation * B)(*[_seg_view(s, keep) for s in segs])
    outs = [_Out(s.count, s.block_size, m.n, int(sizes.max()), want_bases, want_coeffs, want_recon)
            for m, s in zip(meshes, segs)]
    ocs = (_abi.smg_chain_output * B)(*[o.c() for o in outs])
    cc = cfg.to_c()
    ctx.check(ctx.lib.smg_run_chains(ctx.handle, B, mvs, svs, C.byref(cc), _ptr(sizes), ocs))
    res = []
    for i, (o, s) in enumerate(zip(outs, segs)):
        o._c = ocs[i]
        res.append(o.result(s.sequence))
    return res


def coarse_reconstruct_points(bb: BlockBases) -> np.ndarray:
    """coarse_reconstruct_points (pipeline.hpp:300-305) -- computed on the GPU by
    the chain call (want_recon=True); this accessor returns it."""
    if bb.reconstruction is None:
        raise InvalidArgument("the chain was run without want_recon")
    return bb.reconstruction


# ------------------------------------------------------------------ F3 dynamic meshes

def _frame_tables(frames, n: int, keep: list):
    """x_0, y_0, z_0, x_1, ... host pointers of (n, 3) frame arrays + SoA outputs."""
    xyz = (C.c_void_p * (3 * len(frames)))()
    outs = []
    outp = (C.c_void_p * len(frames))()
    for f, v in enumerate(frames):
        v = np.asarray(v, dtype=np.float64)
        if v.shape != (n, 3):
            raise InvalidArgument(f"frame {f} has shape {v.shape}, expected ({n}, 3)")
        for a in range(3):
            col = _f64(v[:, a])
            keep.append(col)
            xyz[3 * f + a] = col.ctypes.data
        o = np.zeros(3 * n)
        outs.append(o)
        outp[f] = o.ctypes.data
    return xyz, outp, outs


def coarse_reconstruct_frames(mesh, seg, bb: BlockBases, frames, mode: str = "weighted",
                              ctx: Optional[Context] = None) -> List[np.ndarray]:
    """coarse_reconstruct_points(frame, bases, mode) (pipeline.hpp:300-305) for
    every frame of a sequence sharing ``mesh``'s connectivity -- the frames stage
    of denoise_dynamic (denoise.hpp:280-288), batched on the GPU."""
    ctx = ctx or default_context()
    if bb.bases is None:
        raise InvalidArgument("the chain was run without want_bases")
    if mode not in _abi.AVERAGE_MODE:
        raise InvalidArgument(f"unknown average mode '{mode}' (expected simple|weighted)")
    keep: list = []
    mv, sv = _mesh_view(mesh, keep), _seg_view(seg, keep)
    k = len(bb.bases)
    sizes = _i32([b.shape[1] for b in bb.bases])
    offs = np.zeros(k + 1, np.int64)
    offs[1:] = np.cumsum([b.size for b in bb.bases])
    data = np.concatenate([np.asarray(b, np.float64).ravel(order="F") for b in bb.bases])
    bv = _abi.smg_bases(k, sizes.ctypes.data, offs.ctypes.data, data.ctypes.data, 0)
    xyz, outp, outs = _frame_tables(frames, mesh.n, keep)
    ctx.check(ctx.lib.smg_coarse_reconstruct_frames(ctx.handle, C.byref(mv), C.byref(sv), C.byref(bv), len(frames),
                                                    xyz, 0, _abi.AVERAGE_MODE[mode], outp, 0))
    return [o.reshape((3, mesh.n)).T.copy() for o in outs]


@dataclasses.dataclass
class DynamicDenoiseResult:
    """DynamicDenoiseResult (denoise.hpp:251-256): per-frame vertices (the
    connectivity is unchanged), basis computations (= k), stage seconds."""

    frames: List[np.ndarray]
    basis_blocks_computed: int
    timings: dict


def denoise_dynamic(frames, seg, cfg: PipelineConfig, sizes_in_order: Optional[Sequence[int]] = None,
                    mode: str = "weighted", ctx: Optional[Context] = None) -> DynamicDenoiseResult:
    """denoise_dynamic (denoise.hpp:258-291) over an external segmentation:
    bases from frames[0], then every frame's coarse projection.  ``frames``
    are meshes sharing one connectivity (``vertices``, ``adj_offsets``,
    ``adj_cols``)."""
    ctx = ctx or default_context()
    if len(frames) == 0:
        raise InvalidArgument("dynamic denoising needs at least one frame")
    if mode not in _abi.AVERAGE_MODE:
        raise InvalidArgument(f"unknown average mode '{mode}' (expected simple|weighted)")
    keep: list = []
    mvs = (_abi.smg_mesh * len(frames))(*[_mesh_view(m, keep) for m in frames])
    sv = _seg_view(seg, keep)
    sizes = None if sizes_in_order is None else _i32(sizes_in_order)
    if sizes is not None and sizes.size != seg.count:
        raise InvalidArgument("need one subspace size per block")
    n = frames[0].n
    outs = [np.zeros(3 * n) for _ in frames]
    outp = (C.c_void_p * len(frames))(*[o.ctypes.data for o in outs])
    nb = C.c_int32()
    tm = np.zeros(3)
    cc = cfg.to_c()
    ctx.check(ctx.lib.smg_denoise_dynamic(ctx.handle, len(frames), mvs, C.byref(sv), C.byref(cc), _ptr(sizes),
                                          _abi.AVERAGE_MODE[mode], outp, 0, C.byref(nb), tm.ctypes.data_as(
                                              _abi.c_double_p)))
    return DynamicDenoiseResult([o.reshape((3, n)).T.copy() for o in outs], int(nb.value),
                                {"shared_basis": float(tm[0]), "frames": float(tm[1]), "total": float(tm[2])})


# ------------------------------------------------------------------ F4 fine denoising

@dataclasses.dataclass
class BilateralParams:
    """BilateralParams (denoise.hpp:11-24), reference defaults."""

    sigma_spatial: float = 0.0
    sigma_range: float = 0.35
    normal_iterations: int = 5
    vertex_iterations: int = 10
    ring_depth: int = 1


def fine_denoise(vertices, faces, params: Optional[BilateralParams] = None, return_normals: bool = False,
                 ctx: Optional[Context] = None):
    """fine_denoise (denoise.hpp:172-178) on the GPU: bilateral filtering of
    the face normals over face rings, then vertex repositioning.  Returns the
    n x 3 vertices (and the filtered face normals when ``return_normals``)."""
    ctx = ctx or default_context()
    params = params or BilateralParams()
    v = np.asarray(vertices, dtype=np.float64)
    f = _i32(np.asarray(faces).reshape(-1, 3))
    n, nf = v.shape[0], f.shape[0]
    xs = [_f64(v[:, a]) for a in range(3)]
    out = np.zeros(3 * n)
    nrm = np.zeros(3 * nf) if return_normals else None
    bp = _abi.smg_bilateral_params(params.sigma_spatial, params.sigma_range, params.normal_iterations,
                                   params.vertex_iterations, params.ring_depth)
    ctx.check(ctx.lib.smg_fine_denoise(ctx.handle, n, _ptr(xs[0]), _ptr(xs[1]), _ptr(xs[2]), nf, _ptr(f),
                                       C.byref(bp), _ptr(out), _ptr(nrm), 0))
    res = out.reshape((3, n)).T.copy()
    if return_normals:
        return res, nrm.reshape((3, nf)).T.copy()
    return res
