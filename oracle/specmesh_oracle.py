"""CPU oracle: a numpy/scipy restatement of the reference's hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker or the timed CPU baseline -- never as the thing
measured or shipped.  The product path (``paper_1810_02719_b200``) never imports
it and fails loudly without its CUDA library.

What it restates (reference = /root/reference/proj/include/specmesh, cited file:line):
  * build_submesh             partition.hpp:169-197  (local order = ascending id)
  * build_laplacian           spectral.hpp:39-68     (L = D - C, D_ii = |N(i)|)
  * Laplacian.trace / default_shift   spectral.hpp:32-36, :193-196
  * ShiftedInverseOperator    spectral.hpp:145-190   (R^z by z factor solves)
  * apply_sign_convention     spectral.hpp:72-85
  * dense_eigendecomposition / bottom_subspace   spectral.hpp:92-117
  * orthonormalize            spectral.hpp:120-132   (Householder QR, rank test)
  * random_orthonormal_basis  spectral.hpp:134-141
  * orthogonal_iteration      spectral.hpp:204-211
  * projection_residual(_rms), bounding_box_diagonal   spectral.hpp:216-231
  * dynamic_oi                spectral.hpp:244-287
  * gft / igft                spectral.hpp:290-298
  * max_principal_angle       spectral.hpp:303-309
  * write_basis / read_basis  spectral.hpp:312-365  (SMBASIS1)
  * PipelineConfig            pipeline.hpp:41-68
  * resize_basis              pipeline.hpp:97-109
  * initial_block_basis       pipeline.hpp:113-120
  * compute_block_bases_fixed_sizes   pipeline.hpp:144-194
  * compute_block_bases (DOI branch)  pipeline.hpp:245-285, with an external
    Segmentation (the reference segments internally, :201)
  * project_blocks / coarse_reconstruct_points   pipeline.hpp:290-305
  * reconstruct_weighted      partition.hpp:311-355
  * hop_distances / partition_mesh   partition.hpp:58-75, :84-159  (farthest-point
    seeds, greedy smallest-part growth, exact tie rules)
  * overlap_target_size / expand_overlaps   partition.hpp:162-165, :205-253
  * order_submeshes           partition.hpp:258-307
  * segment_mesh              pipeline.hpp:131-138

Third-party dependency: the reference's arithmetic comes from Eigen (version
unpinned; absent from this image and the GPU box -- SURVEY.md §8(c)).  Its
published algorithms are restated with
LAPACK through scipy: SimplicialLDLT (AMD order, no pivoting) -> banded Cholesky
(LAPACK dpbtrf/dpbtrs) in natural or RCM order, with a no-pivot banded LDL^T for
indefinite matrices (what Eigen's LDL^T tolerates); HouseholderQR ->
LAPACK dgeqrf/dorgqr; SelfAdjointEigenSolver -> LAPACK dsyevd.  They differ from
Eigen only in rounding.

Parity pin: the reference ships no tests, fixtures or golden vectors, but its own
unmodified headers run in this container over oracle/eigen_shim (a stand-in for the
Eigen API subset they use; oracle/ref_harness.cpp, `make refharness`).  Their outputs
on the seeded configurations are committed as tests/golden/ref_* (made by
tests/golden/make_ref_fixtures.py) and tests/test_ref_fixtures.py holds this oracle to
them: edges, partitions, member lists, orders, CSR patterns and values (1/d^2
included), traces, shifts, DOI decisions and exception texts identical; subspace
angles <= 1e-8, reconstructions <= 1e-9, coefficients <= 1e-8 on C1, C2, C3, a whole
C5 chain and the widened rows.  That pins every line of the reference's own code;
what stays unpinned is only the rounding of Eigen's inner kernels (the shim restates
them too -- see its header).  Also pinned: the SPEC.md known-answer examples
(tests/test_oracle_known_answers.py) and the RNG, bit-exact against
libstdc++'s std::mt19937_64 / std::normal_distribution (oracle/rng_ref.cpp).
"""
from __future__ import annotations

import dataclasses
import math
import struct
import time
from typing import Dict, List, Optional, Sequence

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
from scipy.sparse.csgraph import dijkstra, reverse_cuthill_mckee


class Error(RuntimeError):
    """core.hpp:18-22"""


class InvalidArgument(Error):
    """core.hpp:24-28"""


class ParseError(Error):
    """core.hpp:30-34"""


def require(cond: bool, message: str) -> None:
    """core.hpp:36-38"""
    if not cond:
        raise InvalidArgument(message)


BINARY = "binary"
DISTANCE = "distance"

# --------------------------------------------------------------------------
# RNG: libstdc++ std::mt19937_64 + std::normal_distribution (polar method)

_MASK = (1 << 64) - 1


class MT19937_64:
    """std::mt19937_64 (Matsumoto-Nishimura 64-bit parameters)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & _MASK
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & _MASK
        self.idx = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & _MASK


class NormalDistribution:
    """libstdc++ normal_distribution<double>(0,1): Marsaglia polar method,
    second deviate cached; uniforms via generate_canonical<double,53>."""

    def __init__(self):
        self.saved = None

    @staticmethod
    def _canonical(rng: MT19937_64) -> float:
        r = float(rng()) / 18446744073709551616.0
        if r >= 1.0:
            r = math.nextafter(1.0, 0.0)
        return r

    def __call__(self, rng: MT19937_64) -> float:
        if self.saved is not None:
            v, self.saved = self.saved, None
            return v
        while True:
            x = 2.0 * self._canonical(rng) - 1.0
            y = 2.0 * self._canonical(rng) - 1.0
            r2 = x * x + y * y
            if not (r2 > 1.0 or r2 == 0.0):
                break
        mult = math.sqrt(-2.0 * math.log(r2) / r2)
        self.saved = x * mult
        return y * mult


def gaussian_block(rows: int, cols: int, seed: int) -> np.ndarray:
    """Column-major fill order of spectral.hpp:138-139 / pipeline.hpp:106-107."""
    rng = MT19937_64(seed)
    g = NormalDistribution()
    out = np.empty((rows, cols))
    for j in range(cols):
        for i in range(rows):
            out[i, j] = g(rng)
    return out


# --------------------------------------------------------------------------
# submesh + Laplacian

@dataclasses.dataclass
class Submesh:
    """partition.hpp:34-47 (local faces omitted: not read by the path)."""

    global_indices: np.ndarray
    local_adjacency: List[np.ndarray]
    local_degrees: np.ndarray

    def size(self) -> int:
        return int(self.global_indices.size)

    def local_coords(self, vertices: np.ndarray) -> np.ndarray:
        return vertices[self.global_indices]


def build_submesh(adj_offsets: np.ndarray, adj_cols: np.ndarray, members) -> Submesh:
    """partition.hpp:169-184: sort members, induced adjacency in neighbour-list order."""
    g = np.sort(np.asarray(members, dtype=np.int64))
    adj = []
    for gi in g:
        nb = adj_cols[adj_offsets[gi]:adj_offsets[gi + 1]]
        pos = np.searchsorted(g, nb)
        pos = np.minimum(pos, g.size - 1)
        inside = g[pos] == nb
        adj.append(pos[inside].astype(np.int64))
    deg = np.array([a.size for a in adj], dtype=np.int64)
    return Submesh(g, adj, deg)


@dataclasses.dataclass
class Laplacian:
    """spectral.hpp:27-37; CSR of the symmetric matrix (== Eigen's CSC arrays)."""

    rowptr: np.ndarray
    cols: np.ndarray
    vals: np.ndarray
    weighting: str

    def size(self) -> int:
        return int(self.rowptr.size - 1)

    def trace(self) -> float:
        n = self.size()
        t = 0.0
        for i in range(n):
            s, e = self.rowptr[i], self.rowptr[i + 1]
            k = np.nonzero(self.cols[s:e] == i)[0]
            t += float(self.vals[s + k[0]]) if k.size else 0.0
        return t

    def to_scipy(self) -> sp.csr_matrix:
        n = self.size()
        return sp.csr_matrix((self.vals, self.cols, self.rowptr), shape=(n, n))

    def dense(self) -> np.ndarray:
        return self.to_scipy().toarray()


def build_laplacian(sub: Submesh, vertices: np.ndarray, weighting: str) -> Laplacian:
    """spectral.hpp:39-68.  setFromTriplets sorts each column by row; for the
    symmetric L those are our CSR rows sorted by column."""
    n = sub.size()
    require(n >= 2, "submesh must have at least 2 vertices")
    rowptr = np.zeros(n + 1, dtype=np.int64)
    cols_l, vals_l = [], []
    for i in range(n):
        nb = sub.local_adjacency[i]
        w = np.ones(nb.size)
        if weighting == DISTANCE:
            gi = sub.global_indices[i]
            for t, j in enumerate(nb):
                gj = sub.global_indices[j]
                dx = vertices[gi, 0] - vertices[gj, 0]
                dy = vertices[gi, 1] - vertices[gj, 1]
                dz = vertices[gi, 2] - vertices[gj, 2]
                d2 = (dx * dx + dy * dy) + dz * dz
                with np.errstate(divide="ignore"):
                    inv = 1.0 / d2 if d2 != 0.0 else math.inf
                if not (d2 > 0.0) or not math.isfinite(inv):
                    raise Error(f"coincident connected vertices {gi} and {gj} make the "
                                "distance weight singular")
                w[t] = inv
        c = np.concatenate([[i], nb])
        v = np.concatenate([[float(sub.local_degrees[i])], -w])
        order = np.argsort(c, kind="stable")
        cols_l.append(c[order])
        vals_l.append(v[order])
        rowptr[i + 1] = rowptr[i] + c.size
    return Laplacian(rowptr, np.concatenate(cols_l), np.concatenate(vals_l), weighting)


def default_shift(lap: Laplacian, scale: float = 1e-8) -> float:
    """spectral.hpp:193-196 -- operation order scale * (trace / n) kept."""
    mean_diag = lap.trace() / float(lap.size())
    return max(scale * mean_diag, 1e-300)


# --------------------------------------------------------------------------
# shifted-inverse operator

class ShiftedInverseOperator:
    """spectral.hpp:145-190.  Factor of L + delta*I in natural order (grid
    tiles are banded there) or RCM order, banded Cholesky via LAPACK; a no-pivot
    banded LDL^T takes over when the matrix is not positive definite."""

    # RCM is tried when the natural bandwidth exceeds this (96: grid tiles keep
    # their natural order).  The CPU baseline lowers it to 0 so a 32x64 tile is
    # factored at bandwidth 33 like the GPU's geometric ordering (bench.py).
    rcm_above = 96

    def __init__(self, lap: Laplacian, delta: float, z: int):
        require(delta > 0.0, "shift delta must be positive")
        require(z >= 1, "power z must be at least 1")
        self.shift_, self.power_, self.size_ = delta, z, lap.size()
        a = lap.to_scipy().tocsr().copy()
        a = a + delta * sp.identity(self.size_, format="csr")
        a = a.tocsr()
        a.sort_indices()
        perm = np.arange(self.size_)
        bw = self._bandwidth(a)
        if bw > self.rcm_above:
            p = reverse_cuthill_mckee(a, symmetric_mode=True)
            ap = a[p][:, p].tocsr()
            if self._bandwidth(ap) < bw:
                perm, a, bw = p, ap, self._bandwidth(ap)
        self.perm = perm
        self.bw = bw
        n = self.size_
        ab = np.zeros((bw + 1, n))
        coo = a.tocoo()
        lower = coo.row >= coo.col
        ab[coo.row[lower] - coo.col[lower], coo.col[lower]] = coo.data[lower]
        self.ldl = None
        try:
            self.cb = sla.cholesky_banded(ab, lower=True)
        except np.linalg.LinAlgError:
            self.cb = None
            self.ldl = self._banded_ldlt(a.toarray(), bw)

    @staticmethod
    def _bandwidth(a) -> int:
        coo = a.tocoo()
        return int(np.abs(coo.row - coo.col).max()) if coo.nnz else 0

    @staticmethod
    def _banded_ldlt(A: np.ndarray, bw: int):
        n = A.shape[0]
        L = np.eye(n)
        d = np.zeros(n)
        for j in range(n):
            lo = max(0, j - bw)
            dj = A[j, j] - np.dot(L[j, lo:j] ** 2, d[lo:j])
            if dj == 0.0 or not math.isfinite(dj):
                raise Error("sparse factorization of the shifted Laplacian failed")
            d[j] = dj
            hi = min(n, j + bw + 1)
            L[j + 1:hi, j] = (A[j + 1:hi, j] - L[j + 1:hi, lo:j] @ (d[lo:j] * L[j, lo:j])) / dj
        return L, d

    def size(self) -> int:
        return self.size_

    def shift(self) -> float:
        return self.shift_

    def power(self) -> int:
        return self.power_

    def _solve(self, b: np.ndarray) -> np.ndarray:
        bp = b[self.perm]
        if self.cb is not None:
            xp = sla.cho_solve_banded((self.cb, True), bp, check_finite=False)
        else:
            L, d = self.ldl
            y = sla.solve_triangular(L, bp, lower=True, unit_diagonal=True)
            y = y / (d[:, None] if y.ndim == 2 else d)
            xp = sla.solve_triangular(L.T, y, lower=False, unit_diagonal=True)
        x = np.empty_like(xp)
        x[self.perm] = xp
        return x

    def apply_once(self, block: np.ndarray) -> np.ndarray:
        require(block.shape[0] == self.size_, "operator/block dimension mismatch")
        return self._solve(block)

    def apply(self, block: np.ndarray) -> np.ndarray:
        out = self.apply_once(block)
        for _ in range(1, self.power_):
            out = self._solve(out)
        return out


# --------------------------------------------------------------------------
# dense linear algebra

def apply_sign_convention(cols: np.ndarray) -> np.ndarray:
    """spectral.hpp:72-85: per column argmax |.| (strict >, first index wins),
    flip if that entry is negative.  In place; returns the array."""
    if cols.shape[0] == 0:
        return cols
    at = np.argmax(np.abs(cols), axis=0)  # first occurrence of the maximum
    neg = cols[at, np.arange(cols.shape[1])] < 0.0
    cols[:, neg] *= -1.0
    return cols


def dense_eigendecomposition(lap: Laplacian, dense_limit: int = 4096):
    """spectral.hpp:92-104 -> (ascending eigenvalues, sign-fixed eigenvectors)."""
    require(lap.size() <= dense_limit, "submesh size exceeds the dense eigendecomposition limit")
    w, v = np.linalg.eigh(lap.dense())
    if not np.all(np.isfinite(w)):
        raise Error("dense eigendecomposition failed to converge")
    return w, apply_sign_convention(np.ascontiguousarray(v))


def bottom_subspace(spectrum, c: int) -> np.ndarray:
    """spectral.hpp:114-117"""
    require(1 <= c <= spectrum[1].shape[1], "subspace size out of range")
    return spectrum[1][:, :c].copy()


def orthonormalize(block: np.ndarray) -> np.ndarray:
    """spectral.hpp:120-132"""
    rows, cols = block.shape
    require(cols >= 1 and rows >= cols, "block must be tall (rows >= cols >= 1)")
    scale = float(np.linalg.norm(block))
    if scale == 0.0:
        raise Error("orthonormalize: block is rank deficient (all zero)")
    q, r = sla.qr(block, mode="economic", check_finite=False)
    d = np.abs(np.diag(r))
    bad = np.nonzero(d < 1e-13 * scale)[0]
    if bad.size:
        raise Error(f"orthonormalize: block is rank deficient at column {int(bad[0])}")
    return apply_sign_convention(np.ascontiguousarray(q))


def random_orthonormal_basis(rows: int, c: int, seed: int) -> np.ndarray:
    """spectral.hpp:134-141"""
    return orthonormalize(gaussian_block(rows, c, seed))


def orthogonal_iteration(op: ShiftedInverseOperator, init: np.ndarray, t_max: int) -> np.ndarray:
    """spectral.hpp:204-211"""
    require(init.shape[0] == op.size(), "initial basis does not match the operator size")
    require(t_max >= 0, "t_max must be nonnegative")
    u = init
    for _ in range(t_max):
        u = orthonormalize(op.apply(u))
    return u


def projection_residual(basis: np.ndarray, coords: np.ndarray) -> np.ndarray:
    """spectral.hpp:216-220: e = s - U (U^T s), s = x + y + z."""
    require(coords.shape[0] == basis.shape[0], "coordinate/basis dimension mismatch")
    summed = coords.sum(axis=1)
    return summed - basis @ (basis.T @ summed)


def projection_residual_rms(basis: np.ndarray, coords: np.ndarray) -> float:
    """spectral.hpp:223-226"""
    residual = coords - basis @ (basis.T @ coords)
    return math.sqrt(float(np.sum(residual * residual)) / float(coords.size))


def bounding_box_diagonal(coords: np.ndarray) -> float:
    """spectral.hpp:228-231"""
    if coords.shape[0] == 0:
        return 0.0
    return float(np.linalg.norm(coords.max(axis=0) - coords.min(axis=0)))


@dataclasses.dataclass
class DoiResult:
    """spectral.hpp:233-238"""

    basis: np.ndarray
    converged: bool = False
    residual: float = 0.0
    iterations: int = 0


def dynamic_oi(op, init, coords, eps_low, eps_high, c_min, c_max, t_max, trace=None) -> DoiResult:
    """spectral.hpp:244-287.  ``trace`` (test hook): a list that receives
    (subspace size the step ran with, residual) for every step."""
    require(eps_low > 0.0 and eps_low < eps_high, "need 0 < eps_low < eps_high")
    require(c_min >= 1 and c_min <= init.shape[1] and init.shape[1] <= c_max,
            "need c_min <= init subspace size <= c_max")
    require(c_max <= op.size(), "c_max cannot exceed the submesh size")
    require(coords.shape[0] == op.size(), "coordinate/operator dimension mismatch")
    scale = bounding_box_diagonal(coords)
    if scale == 0.0:
        scale = 1.0
    u = init
    appended_raw = False
    res = DoiResult(basis=init)
    for t in range(1, t_max + 1):
        u = orthonormalize(op.apply(u))
        appended_raw = False
        res.iterations = t
        e = projection_residual(u, coords)
        en = float(np.linalg.norm(e))
        res.residual = en / scale
        if trace is not None:
            trace.append((u.shape[1], res.residual))
        if res.residual > eps_high:
            if u.shape[1] >= c_max:
                break
            u = np.concatenate([u, (e / en)[:, None]], axis=1)
            appended_raw = True
        elif res.residual < eps_low:
            if u.shape[1] <= c_min:
                res.converged = True
                break
            u = u[:, :-1].copy()
        else:
            res.converged = True
            break
    if appended_raw:
        u = orthonormalize(u)
    res.basis = u
    return res


def gft(basis: np.ndarray, coords: np.ndarray) -> np.ndarray:
    """spectral.hpp:290-293"""
    require(coords.shape[0] == basis.shape[0], "coordinate/basis dimension mismatch")
    return basis.T @ coords


def igft(basis: np.ndarray, coeffs: np.ndarray) -> np.ndarray:
    """spectral.hpp:295-298"""
    require(coeffs.shape[0] == basis.shape[1], "coefficient/basis dimension mismatch")
    return basis @ coeffs


def max_principal_angle(a: np.ndarray, b: np.ndarray) -> float:
    """spectral.hpp:303-309"""
    require(a.shape == b.shape, "principal angles need equally shaped bases")
    residual = a - b @ (b.T @ a)
    s = float(np.linalg.svd(residual, compute_uv=False)[0]) if residual.size else 0.0
    return math.asin(min(max(s, 0.0), 1.0))


BASIS_MAGIC = b"SMBASIS1"


def write_basis(basis: np.ndarray, path: str) -> None:
    """spectral.hpp:337-347: magic, u64 rows, u64 cols, row-major f64 LE."""
    with open(path, "wb") as f:
        f.write(BASIS_MAGIC)
        f.write(struct.pack("<QQ", basis.shape[0], basis.shape[1]))
        f.write(np.ascontiguousarray(basis, dtype="<f8").tobytes())


def read_basis(path: str) -> np.ndarray:
    """spectral.hpp:349-365"""
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != BASIS_MAGIC:
        raise ParseError(f"{path}: not a basis dump")
    if len(data) < 24:
        raise ParseError(f"{path}: bad basis header")
    rows, cols = struct.unpack("<QQ", data[8:24])
    if rows < 1 or cols < 1 or cols > rows:
        raise ParseError(f"{path}: bad basis header")
    body = data[24:]
    if len(body) < rows * cols * 8:
        raise ParseError(f"{path}: truncated basis dump")
    return np.frombuffer(body[:rows * cols * 8], dtype="<f8").reshape(rows, cols).copy()


# --------------------------------------------------------------------------
# pipeline

@dataclasses.dataclass
class PipelineConfig:
    """pipeline.hpp:41-68 (segmentation fields unused: Segmentation is an input)."""

    weighting: str = DISTANCE
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

    def resolve_c_max(self, block_size: int) -> int:
        cm = self.c_max if self.c_max > 0 else max(64, 2 * self.subspace_size)
        return min(cm, block_size)

    def resolve_doi_iterations(self, resolved_c_max: int) -> int:
        if self.doi_iterations > 0:
            return self.doi_iterations
        return (resolved_c_max - self.c_min) + 16


@dataclasses.dataclass
class BlockStats:
    """pipeline.hpp:70-76"""

    subspace_size: int = 0
    residual_rms: float = 0.0
    doi_residual: float = 0.0
    converged: bool = True
    oi_iterations: int = 0


@dataclasses.dataclass
class BlockBases:
    """pipeline.hpp:78-92"""

    submeshes: List[Submesh]
    sequence: np.ndarray
    bases: List[Optional[np.ndarray]]
    stats: List[BlockStats]
    timings: Dict[str, float]
    block_size: int

    def sizes_in_order(self) -> List[int]:
        return [self.bases[i].shape[1] for i in self.sequence]


def _add(t: Dict[str, float], k: str, v: float) -> None:
    t[k] = t.get(k, 0.0) + v


def resize_basis(basis: np.ndarray, new_size: int, seed: int) -> np.ndarray:
    """pipeline.hpp:97-109"""
    old = basis.shape[1]
    if new_size == old:
        return basis
    require(1 <= new_size <= basis.shape[0], "subspace size out of range")
    if new_size < old:
        return basis[:, :new_size].copy()
    grown = np.empty((basis.shape[0], new_size))
    grown[:, :old] = basis
    grown[:, old:] = gaussian_block(basis.shape[0], new_size - old, seed)
    return orthonormalize(grown)


def initial_block_basis(lap: Laplacian, op: ShiftedInverseOperator, c: int,
                        cfg: PipelineConfig) -> np.ndarray:
    """pipeline.hpp:113-120"""
    if lap.size() <= cfg.dense_limit:
        return bottom_subspace(dense_eigendecomposition(lap, cfg.dense_limit), c)
    cold = random_orthonormal_basis(lap.size(), c, cfg.seed ^ 0x9E3779B97F4A7C15)
    return orthogonal_iteration(op, cold, cfg.initial_iterations)


def _pos_seed(cfg: PipelineConfig, pos: int) -> int:
    return (cfg.seed + 0x5851F42D4C957F2D * pos) & _MASK


def build_submeshes(adj_offsets, adj_cols, members: Sequence[np.ndarray]) -> List[Submesh]:
    return [build_submesh(adj_offsets, adj_cols, m) for m in members]


def compute_block_bases_fixed_sizes(vertices, submeshes: List[Submesh], sequence, cfg: PipelineConfig,
                                    sizes_in_order: Sequence[int], keep_bases: bool = True,
                                    init_basis: Optional[np.ndarray] = None) -> BlockBases:
    """pipeline.hpp:144-194.  ``init_basis`` (test hook) replaces the dense
    first-submesh basis, used by the one-step parity mode."""
    require(len(sizes_in_order) == len(sequence), "need one subspace size per block")
    k = len(submeshes)
    res = BlockBases(submeshes, np.asarray(sequence), [None] * k, [BlockStats() for _ in range(k)],
                     {}, submeshes[0].size() if submeshes else 0)
    t_all = time.perf_counter()
    previous = None
    for pos, sid in enumerate(sequence):
        sub = submeshes[sid]
        c = int(sizes_in_order[pos])
        require(1 <= c <= sub.size(), "subspace size out of range for block")
        t0 = time.perf_counter()
        lap = build_laplacian(sub, vertices, cfg.weighting)
        _add(res.timings, "laplacian", time.perf_counter() - t0)
        t0 = time.perf_counter()
        op = ShiftedInverseOperator(lap, default_shift(lap, cfg.shift_scale), cfg.power)
        _add(res.timings, "factorize", time.perf_counter() - t0)
        t0 = time.perf_counter()
        if pos == 0:
            basis = init_basis if init_basis is not None else initial_block_basis(lap, op, c, cfg)
        else:
            warm = resize_basis(previous, c, _pos_seed(cfg, pos))
            basis = orthogonal_iteration(op, warm, cfg.iterations)
        _add(res.timings, "basis", time.perf_counter() - t0)
        if pos == 0:
            _add(res.timings, "first_basis", time.perf_counter() - t0)
        st = res.stats[sid]
        st.subspace_size = c
        st.oi_iterations = 0 if pos == 0 else cfg.iterations
        st.residual_rms = projection_residual_rms(basis, sub.local_coords(vertices))
        previous = basis
        res.bases[sid] = basis if keep_bases else None
    _add(res.timings, "basis_total", time.perf_counter() - t_all)
    return res


def compute_block_bases_doi(vertices, submeshes: List[Submesh], sequence, cfg: PipelineConfig,
                            keep_bases: bool = True, trace=None, on_block=None,
                            operator_factory=None) -> BlockBases:
    """pipeline.hpp:245-285 (DOI branch), over an external segmentation.
    ``trace`` (test hook): list receiving (position, c, residual) per DOI step;
    ``on_block(pos, sid, basis)`` is called after every block;
    ``operator_factory(lap, delta, z)`` replaces ShiftedInverseOperator (a
    second restatement of the solve, to measure rounding sensitivity)."""
    k = len(submeshes)
    res = BlockBases(submeshes, np.asarray(sequence), [None] * k, [BlockStats() for _ in range(k)],
                     {}, submeshes[0].size() if submeshes else 0)
    t_all = time.perf_counter()
    previous = None
    for pos, sid in enumerate(sequence):
        sub = submeshes[sid]
        c_max = cfg.resolve_c_max(sub.size())
        doi_t = cfg.resolve_doi_iterations(c_max)
        t0 = time.perf_counter()
        lap = build_laplacian(sub, vertices, cfg.weighting)
        _add(res.timings, "laplacian", time.perf_counter() - t0)
        t0 = time.perf_counter()
        op = (operator_factory or ShiftedInverseOperator)(lap, default_shift(lap, cfg.shift_scale), cfg.power)
        _add(res.timings, "factorize", time.perf_counter() - t0)
        t0 = time.perf_counter()
        if pos == 0:
            c0 = min(max(cfg.subspace_size, cfg.c_min), c_max)
            init = initial_block_basis(lap, op, c0, cfg)
        else:
            c_init = min(max(previous.shape[1], cfg.c_min), c_max)
            init = resize_basis(previous, c_init, _pos_seed(cfg, pos))
        coords = sub.local_coords(vertices)
        steps = [] if trace is not None else None
        doi = dynamic_oi(op, init, coords, cfg.eps_low, cfg.eps_high, cfg.c_min, c_max, doi_t, trace=steps)
        if trace is not None:
            trace.extend((pos, c, r) for c, r in steps)
        _add(res.timings, "basis", time.perf_counter() - t0)
        st = res.stats[sid]
        st.subspace_size = doi.basis.shape[1]
        st.doi_residual = doi.residual
        st.converged = doi.converged
        st.oi_iterations = doi.iterations
        st.residual_rms = projection_residual_rms(doi.basis, coords)
        previous = doi.basis
        res.bases[sid] = doi.basis if keep_bases else None
        if on_block is not None:
            on_block(pos, sid, doi.basis)
    _add(res.timings, "basis_total", time.perf_counter() - t_all)
    return res


def project_blocks(bb: BlockBases, vertices: np.ndarray) -> List[np.ndarray]:
    """pipeline.hpp:290-297 (loops over submesh id)."""
    out = []
    for sid, sub in enumerate(bb.submeshes):
        coords = sub.local_coords(vertices)
        out.append(igft(bb.bases[sid], gft(bb.bases[sid], coords)))
    return out


def block_coefficients(bb: BlockBases, vertices: np.ndarray) -> List[np.ndarray]:
    return [gft(bb.bases[s], sub.local_coords(vertices)) for s, sub in enumerate(bb.submeshes)]


def reconstruct_weighted(submeshes: List[Submesh], local_results: List[np.ndarray], n: int,
                         weighted: bool = True) -> np.ndarray:
    """partition.hpp:311-355"""
    require(len(submeshes) == len(local_results), "submesh and result lists must have equal length")
    out = np.zeros((n, 3))
    wsum = np.zeros(n)
    copies = np.zeros(n, dtype=np.int64)
    fallback = np.zeros((n, 3))
    for sub, loc in zip(submeshes, local_results):
        require(loc.shape[0] == sub.size(), "local result size does not match its submesh")
        g = sub.global_indices
        w = sub.local_degrees.astype(np.float64) if weighted else np.ones(g.size)
        out[g] += w[:, None] * loc
        wsum[g] += w
        fallback[g] += loc
        copies[g] += 1
    unc = np.nonzero(copies == 0)[0]
    if unc.size:
        msg = f"reconstruction is missing {unc.size} vertices:" + "".join(f" {int(v)}" for v in unc[:16])
        if unc.size > 16:
            msg += " ..."
        raise InvalidArgument(msg)
    pos = wsum > 0.0
    out[pos] /= wsum[pos][:, None]
    out[~pos] = fallback[~pos] / copies[~pos][:, None]
    return out


def coarse_reconstruct_points(bb: BlockBases, vertices: np.ndarray, weighted: bool = True) -> np.ndarray:
    """pipeline.hpp:300-305"""
    return reconstruct_weighted(bb.submeshes, project_blocks(bb, vertices), vertices.shape[0], weighted)


def denoise_dynamic(frames: List[np.ndarray], submeshes: List[Submesh], sequence, cfg: "PipelineConfig",
                    sizes_in_order, weighted: bool = True):
    """denoise.hpp:258-291 with an external segmentation: bases computed once
    from the first frame (:276-277), then coarse_reconstruct_points of every frame
    (:280-288).  Returns (frames, basis_blocks_computed, bases)."""
    require(len(frames) > 0, "dynamic denoising needs at least one frame")
    n = frames[0].shape[0]
    for i in range(1, len(frames)):
        if frames[i].shape[0] != n:
            raise InvalidArgument(f"frame {i} does not share the sequence connectivity")
    bb = compute_block_bases_fixed_sizes(frames[0], submeshes, sequence, cfg, sizes_in_order)
    out = [coarse_reconstruct_points(bb, v, weighted) for v in frames]
    return out, len(bb.bases), bb


# --------------------------------------------------------------------------
# F2 spectral codec (compress.hpp)

@dataclasses.dataclass
class EncodedBlock:
    """compress.hpp:17-25."""

    submesh_id: int = 0
    subspace_size: int = 0
    coeff_min: List[float] = dataclasses.field(default_factory=lambda: [0.0, 0.0, 0.0])
    coeff_max: List[float] = dataclasses.field(default_factory=lambda: [0.0, 0.0, 0.0])
    constant_axis: List[int] = dataclasses.field(default_factory=lambda: [0, 0, 0])
    values: List[int] = dataclasses.field(default_factory=list)  # axis-major: c x, c y, c z


def bits_per_vertex(quant_bits: int, subspace_size: int, block_count: int, vertex_count: int) -> float:
    """compress.hpp:28-31"""
    require(quant_bits > 0 and subspace_size > 0 and block_count > 0 and vertex_count > 0,
            "bits_per_vertex arguments must be positive")
    return 3.0 * quant_bits * subspace_size * block_count / float(vertex_count)


def encode_coefficients(coefficients: np.ndarray, quant_bits: int, submesh_id: int = 0) -> EncodedBlock:
    """compress.hpp:36-62 after the gft (:40): per-axis range, step = (hi-lo)/2^q,
    value = clamp(long((x - lo) / step), 0, 2^q - 1); constant axes send nothing.
    Python floats are IEEE doubles without FMA contraction, int() truncates toward
    zero like static_cast<long>."""
    require(1 <= quant_bits <= 16, "quantization bits must be in [1,16]")
    c = int(coefficients.shape[0])
    levels = 1 << quant_bits
    blk = EncodedBlock(submesh_id=submesh_id, subspace_size=c, values=[0] * (3 * c))
    for axis in range(3):
        col = [float(v) for v in coefficients[:, axis]]
        lo, hi = min(col), max(col)
        blk.coeff_min[axis] = lo
        blk.coeff_max[axis] = hi
        if not (hi > lo):
            blk.constant_axis[axis] = 1
            continue
        step = (hi - lo) / levels
        for i in range(c):
            q = int((col[i] - lo) / step)
            blk.values[axis * c + i] = min(max(q, 0), levels - 1)
    return blk


def encode_block(sub: Submesh, vertices: np.ndarray, basis: np.ndarray, quant_bits: int,
                 submesh_id: int = 0) -> EncodedBlock:
    """compress.hpp:33-62"""
    require(1 <= quant_bits <= 16, "quantization bits must be in [1,16]")
    require(basis.shape[0] == sub.size(), "basis does not match the submesh size")
    return encode_coefficients(gft(basis, sub.local_coords(vertices)), quant_bits, submesh_id)


def dequantize_block(block: EncodedBlock, quant_bits: int) -> np.ndarray:
    """compress.hpp:64-80: lo + (q + 0.5) * step."""
    c = block.subspace_size
    levels = 1 << quant_bits
    out = np.zeros((c, 3))
    for axis in range(3):
        if block.constant_axis[axis]:
            out[:, axis] = block.coeff_min[axis]
            continue
        step = (block.coeff_max[axis] - block.coeff_min[axis]) / levels
        for i in range(c):
            out[i, axis] = block.coeff_min[axis] + (block.values[axis * c + i] + 0.5) * step
    return out


def decode_block(block: EncodedBlock, basis: np.ndarray, quant_bits: int) -> np.ndarray:
    """compress.hpp:84-89"""
    if basis.shape[1] != block.subspace_size:
        raise Error("decode_block: basis subspace size does not match the block")
    return igft(basis, dequantize_block(block, quant_bits))


@dataclasses.dataclass
class EncodedMesh:
    """compress.hpp:100-150 (config echo + connectivity + blocks in order)."""

    version: int = 1
    basis_mode: int = 0  # BasisMode::OI
    quant_bits: int = 12
    part_count: int = 0
    growth: float = 1.15
    subspace_size: int = 0
    eps_low: float = 0.0
    eps_high: float = 0.0
    c_min: int = 0
    c_max: int = 0
    power: int = 2
    iterations: int = 2
    initial_iterations: int = 60
    seed: int = 1
    dense_limit: int = 4096
    shift_scale: float = 1e-8
    vertex_count: int = 0
    faces: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros((0, 3), np.int32))
    blocks: List[EncodedBlock] = dataclasses.field(default_factory=list)

    def total_bpv(self) -> float:
        """compress.hpp:145-150"""
        bits = sum(3 * self.quant_bits * b.subspace_size for b in self.blocks)
        return bits / self.vertex_count


def compress_mesh(vertices: np.ndarray, faces: np.ndarray, submeshes: List[Submesh], sequence,
                  cfg: PipelineConfig, quant_bits: int, sizes_in_order=None, doi: bool = False):
    """compress.hpp:152-219 with an external segmentation: Binary weighting
    (:157); DOI only picks the sizes (:162-166); the transmitted bases are the
    fixed-size OI chain (:168-174); blocks in order sequence (:208-212)."""
    cfg = dataclasses.replace(cfg, weighting=BINARY)
    k = len(submeshes)
    if sizes_in_order is None:
        if doi:
            probe = compute_block_bases_doi(vertices, submeshes, sequence, cfg)
            sizes_in_order = [probe.stats[i].subspace_size for i in sequence]
        else:
            sizes_in_order = [cfg.subspace_size] * k
    bb = compute_block_bases_fixed_sizes(vertices, submeshes, sequence, cfg, sizes_in_order)
    enc = EncodedMesh(basis_mode=1 if doi else 0, quant_bits=quant_bits, part_count=k,
                      subspace_size=cfg.subspace_size, eps_low=cfg.eps_low, eps_high=cfg.eps_high,
                      c_min=cfg.c_min, c_max=cfg.c_max, power=cfg.power, iterations=cfg.iterations,
                      initial_iterations=cfg.initial_iterations, seed=cfg.seed, dense_limit=cfg.dense_limit,
                      shift_scale=cfg.shift_scale, vertex_count=int(vertices.shape[0]),
                      faces=np.asarray(faces, np.int32))
    for sid in sequence:
        enc.blocks.append(encode_block(submeshes[sid], vertices, bb.bases[sid], quant_bits, int(sid)))
    return enc, bb


def replay_config(enc: EncodedMesh) -> PipelineConfig:
    """compress.hpp:125-143"""
    return PipelineConfig(weighting=BINARY, subspace_size=enc.subspace_size, eps_low=enc.eps_low,
                          eps_high=enc.eps_high, c_min=enc.c_min, c_max=enc.c_max, power=enc.power,
                          iterations=enc.iterations, initial_iterations=enc.initial_iterations, seed=enc.seed,
                          dense_limit=enc.dense_limit, shift_scale=enc.shift_scale)


def decompress_mesh(enc: EncodedMesh, submeshes: List[Submesh], sequence):
    """compress.hpp:221-256: replay the chain from connectivity alone (zero
    coordinates, :224-226), decode every block, stitch Weighted."""
    cfg = replay_config(enc)
    zero = np.zeros((enc.vertex_count, 3))
    sizes = [b.subspace_size for b in enc.blocks]
    if len(enc.blocks) != len(sequence):
        raise ParseError("encoded block count does not match the replayed segmentation")
    bb = compute_block_bases_fixed_sizes(zero, submeshes, sequence, cfg, sizes)
    locals_: List[Optional[np.ndarray]] = [None] * len(submeshes)
    for pos, blk in enumerate(enc.blocks):
        if blk.submesh_id >= len(locals_) or int(sequence[pos]) != blk.submesh_id:
            raise ParseError("encoded block order does not match the replayed segmentation")
        locals_[blk.submesh_id] = decode_block(blk, bb.bases[blk.submesh_id], enc.quant_bits)
    return reconstruct_weighted(submeshes, locals_, enc.vertex_count, True)


CODEC_MAGIC = b"SPECMSH1"


class _BitPacker:
    """compress.hpp:334-360: MSB first, pad_to_byte shifts the tail left."""

    def __init__(self, out: bytearray):
        self.out, self.buffer, self.filled = out, 0, 0

    def put(self, value: int, bits: int) -> None:
        for b in range(bits - 1, -1, -1):
            self.buffer = ((self.buffer << 1) | ((value >> b) & 1)) & 0xFF
            self.filled += 1
            if self.filled == 8:
                self._flush()

    def pad_to_byte(self) -> None:
        if self.filled > 0:
            self.buffer = (self.buffer << (8 - self.filled)) & 0xFF
            self._flush()

    def _flush(self) -> None:
        self.out.append(self.buffer)
        self.buffer, self.filled = 0, 0


def pack_block_values(block: EncodedBlock, quant_bits: int) -> bytes:
    """The payload one block contributes (compress.hpp:415-423)."""
    out = bytearray()
    pk = _BitPacker(out)
    c = block.subspace_size
    for a in range(3):
        if block.constant_axis[a]:
            continue
        for i in range(c):
            pk.put(block.values[a * c + i], quant_bits)
    pk.pad_to_byte()
    return bytes(out)


def serialize_encoded_mesh(enc: EncodedMesh) -> bytes:
    """compress.hpp:392-426: little endian, coefficients bit-packed MSB first."""
    o = bytearray(CODEC_MAGIC)
    o += struct.pack("<IBBH", enc.version, enc.basis_mode, 0, enc.quant_bits)
    o += struct.pack("<IdI", enc.part_count, enc.growth, enc.subspace_size)
    o += struct.pack("<dd", enc.eps_low, enc.eps_high)
    o += struct.pack("<IIIII", enc.c_min, enc.c_max, enc.power, enc.iterations, enc.initial_iterations)
    o += struct.pack("<QId", enc.seed, enc.dense_limit, enc.shift_scale)
    faces = np.asarray(enc.faces, np.int64).reshape(-1, 3)
    o += struct.pack("<II", enc.vertex_count, faces.shape[0])
    o += faces.astype("<u4").tobytes()
    o += struct.pack("<I", len(enc.blocks))
    for b in enc.blocks:
        o += struct.pack("<IIB", b.submesh_id, b.subspace_size,
                         b.constant_axis[0] | (b.constant_axis[1] << 1) | (b.constant_axis[2] << 2))
        o += struct.pack("<3d", *b.coeff_min)
        o += struct.pack("<3d", *b.coeff_max)
        o += pack_block_values(b, enc.quant_bits)
    return bytes(o)


class _Reader:
    """compress.hpp:294-332 (ByteReader) + :362-386 (BitUnpacker)."""

    def __init__(self, data: bytes):
        self.data, self.at = data, 0

    def take(self, n: int) -> bytes:
        if self.at + n > len(self.data):
            raise ParseError("bitstream truncated")
        v = self.data[self.at:self.at + n]
        self.at += n
        return v

    def unpack(self, fmt: str):
        return struct.unpack(fmt, self.take(struct.calcsize(fmt)))


def parse_encoded_mesh(data: bytes) -> EncodedMesh:
    """compress.hpp:428-474"""
    r = _Reader(bytes(data))
    if r.take(8) != CODEC_MAGIC:
        raise ParseError("not a specmesh bitstream (bad magic)")
    enc = EncodedMesh()
    (enc.version,) = r.unpack("<I")
    if enc.version != 1:
        raise ParseError("unsupported bitstream version")
    enc.basis_mode, _w, enc.quant_bits = r.unpack("<BBH")
    if enc.quant_bits < 1 or enc.quant_bits > 16:
        raise ParseError("bitstream has invalid quantization bits")
    enc.part_count, enc.growth, enc.subspace_size = r.unpack("<IdI")
    enc.eps_low, enc.eps_high = r.unpack("<dd")
    enc.c_min, enc.c_max, enc.power, enc.iterations, enc.initial_iterations = r.unpack("<IIIII")
    enc.seed, enc.dense_limit, enc.shift_scale = r.unpack("<QId")
    enc.vertex_count, nf = r.unpack("<II")
    enc.faces = np.frombuffer(r.take(12 * nf), "<u4").astype(np.int32).reshape(nf, 3)
    (nb,) = r.unpack("<I")
    q = enc.quant_bits
    for _ in range(nb):
        b = EncodedBlock()
        b.submesh_id, b.subspace_size, flags = r.unpack("<IIB")
        b.constant_axis = [(flags >> a) & 1 for a in range(3)]
        b.coeff_min = list(r.unpack("<3d"))
        b.coeff_max = list(r.unpack("<3d"))
        b.values = [0] * (3 * b.subspace_size)
        buf, filled = 0, 0
        for a in range(3):
            if b.constant_axis[a]:
                continue
            for i in range(b.subspace_size):
                v = 0
                for _bit in range(q):
                    if filled == 0:
                        buf = r.take(1)[0]
                        filled = 8
                    v = (v << 1) | ((buf >> (filled - 1)) & 1)
                    filled -= 1
                b.values[a * b.subspace_size + i] = v
        enc.blocks.append(b)
    if r.at != len(r.data):
        raise ParseError("trailing bytes after bitstream payload")
    return enc


# --------------------------------------------------------------------------
# F4 fine denoising (denoise.hpp:11-180, mesh.hpp:87-116)

@dataclasses.dataclass
class BilateralParams:
    """denoise.hpp:11-24"""

    sigma_spatial: float = 0.0
    sigma_range: float = 0.35
    normal_iterations: int = 5
    vertex_iterations: int = 10
    ring_depth: int = 1

    def validate(self) -> None:
        require(self.sigma_spatial >= 0.0, "sigma_spatial must be positive (or 0 for automatic)")
        require(self.sigma_range > 0.0, "sigma_range must be positive")
        require(self.normal_iterations > 0 and self.vertex_iterations > 0 and self.ring_depth > 0,
                "iteration counts and ring depth must be positive")


def _sq3(dx, dy, dz):
    """squaredNorm of a 3-vector, (x*x + y*y) + z*z."""
    return (dx * dx + dy * dy) + dz * dz


def face_geometry(vertices: np.ndarray, faces: np.ndarray):
    """mesh.hpp:94-116: centroids ((a+b)+c)/3, unit normals of (b-a)x(c-a), areas
    0.5|cross|, degenerate faces (zero cross) get a zero normal.  Component-wise
    scalar arithmetic in the reference's order."""
    f = np.asarray(faces, np.int64)
    a, b, c = vertices[f[:, 0]], vertices[f[:, 1]], vertices[f[:, 2]]
    cen = ((a + b) + c) / 3.0
    u, v = b - a, c - a
    cx = u[:, 1] * v[:, 2] - u[:, 2] * v[:, 1]
    cy = u[:, 2] * v[:, 0] - u[:, 0] * v[:, 2]
    cz = u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0]
    norm = np.sqrt(_sq3(cx, cy, cz))
    areas = 0.5 * norm
    nrm = np.zeros((f.shape[0], 3))
    ok = norm > 0.0
    nrm[ok, 0] = cx[ok] / norm[ok]
    nrm[ok, 1] = cy[ok] / norm[ok]
    nrm[ok, 2] = cz[ok] / norm[ok]
    return cen, nrm, areas, np.nonzero(~ok)[0]


def faces_of_vertex(faces: np.ndarray, n: int) -> List[np.ndarray]:
    """denoise.hpp:43-45 / :152-154: incident faces per vertex, ascending."""
    out: List[list] = [[] for _ in range(n)]
    for fi, fv in enumerate(np.asarray(faces)):
        for k in range(3):
            out[int(fv[k])].append(fi)
    return [np.asarray(l, np.int64) for l in out]


def face_ring_adjacency(faces: np.ndarray, n: int, depth: int = 1) -> List[np.ndarray]:
    """denoise.hpp:39-65: faces sharing >= 1 vertex (self included), sorted unique;
    `depth` repeats the expansion."""
    require(depth >= 1, "ring depth must be at least 1")
    fov = faces_of_vertex(faces, n)
    f = np.asarray(faces)
    ring = [np.unique(np.concatenate([fov[int(f[i, 0])], fov[int(f[i, 1])], fov[int(f[i, 2])]]))
            for i in range(f.shape[0])]
    for _ in range(1, depth):
        ring = [np.unique(np.concatenate([ring[g] for g in ring[i]])) for i in range(f.shape[0])]
    return ring


def _padded(lists: List[np.ndarray]):
    width = max(len(l) for l in lists) if lists else 0
    idx = np.zeros((len(lists), width), np.int64)
    valid = np.zeros((len(lists), width), bool)
    for i, l in enumerate(lists):
        idx[i, :len(l)] = l
        valid[i, :len(l)] = True
    return idx, valid


def default_sigma_spatial(centroids: np.ndarray, ring: List[np.ndarray]) -> float:
    """denoise.hpp:67-83: mean centroid distance over adjacent pairs g > f,
    summed in (f, g) order."""
    total, count = 0.0, 0
    for fi, lst in enumerate(ring):
        g = lst[lst > fi]
        if g.size == 0:
            continue
        d = centroids[g] - centroids[fi]
        dist = np.sqrt(_sq3(d[:, 0], d[:, 1], d[:, 2]))
        for v in dist:
            total += float(v)
        count += int(g.size)
    require(count > 0, "mesh has no adjacent face pairs")
    return total / count


def bilateral_normals(centroids, normals, areas, degenerate, ring, params: BilateralParams) -> np.ndarray:
    """denoise.hpp:87-127: Jacobi sweeps; per face acc += ((A_g * ks) * kr) * n_g
    over its ring in ascending order (zero-area faces skipped), normalised when
    nonzero; degenerate faces are not updated."""
    params.validate()
    sigma_s = params.sigma_spatial if params.sigma_spatial > 0.0 else default_sigma_spatial(centroids, ring)
    idx, valid = _padded(ring)
    nf = normals.shape[0]
    deg = np.zeros(nf, bool)
    deg[np.asarray(degenerate, np.int64)] = True
    cur = normals.copy()
    two_s = 2.0 * sigma_s * sigma_s
    two_r = 2.0 * params.sigma_range * params.sigma_range
    for _ in range(params.normal_iterations):
        acc = np.zeros((nf, 3))
        for r in range(idx.shape[1]):
            g = idx[:, r]
            use = valid[:, r] & (areas[g] > 0.0)
            dc = centroids - centroids[g]
            ks = np.exp(-_sq3(dc[:, 0], dc[:, 1], dc[:, 2]) / two_s)
            dn = cur - cur[g]
            kr = np.exp(-_sq3(dn[:, 0], dn[:, 1], dn[:, 2]) / two_r)
            w = (areas[g] * ks) * kr
            contrib = w[:, None] * cur[g]
            acc[use] += contrib[use]
        norm = np.sqrt(_sq3(acc[:, 0], acc[:, 1], acc[:, 2]))
        nxt = cur.copy()
        upd = (~deg) & (norm > 0.0)
        nxt[upd] = acc[upd] / norm[upd][:, None]
        cur = nxt
    return cur


def update_vertices(vertices: np.ndarray, faces: np.ndarray, target_normals: np.ndarray,
                    vertex_iterations: int) -> np.ndarray:
    """denoise.hpp:133-165: per pass, centroids from the current vertices, then
    v += (1/|F_v|) sum_{f in F_v, ascending} n_f (n_f . (m_f - v))."""
    f = np.asarray(faces, np.int64)
    require(target_normals.shape[0] == f.shape[0], "one target normal per face required")
    require(vertex_iterations >= 0, "vertex iterations must be nonnegative")
    fov = faces_of_vertex(faces, vertices.shape[0])
    idx, valid = _padded(fov)
    cnt = valid.sum(axis=1)
    out = vertices.copy()
    for _ in range(vertex_iterations):
        cen = ((out[f[:, 0]] + out[f[:, 1]]) + out[f[:, 2]]) / 3.0
        delta = np.zeros_like(out)
        for r in range(idx.shape[1]):
            fi = idx[:, r]
            use = valid[:, r]
            nrm = target_normals[fi]
            d = cen[fi] - out
            dot = (nrm[:, 0] * d[:, 0] + nrm[:, 1] * d[:, 1]) + nrm[:, 2] * d[:, 2]
            delta[use] += (nrm * dot[:, None])[use]
        has = cnt > 0
        nxt = out.copy()
        nxt[has] = out[has] + delta[has] / cnt[has][:, None].astype(np.float64)
        out = nxt
    return out


def fine_denoise(vertices: np.ndarray, faces: np.ndarray, params: BilateralParams):
    """denoise.hpp:172-178; returns (vertices, filtered normals)."""
    cen, nrm, areas, degenerate = face_geometry(vertices, faces)
    ring = face_ring_adjacency(faces, vertices.shape[0], params.ring_depth)
    filtered = bilateral_normals(cen, nrm, areas, degenerate, ring, params)
    return update_vertices(vertices, faces, filtered, params.vertex_iterations), filtered


# --------------------------------------------------------------------------
# segmentation (partition.hpp:58-307, pipeline.hpp:131-138)

_INT_MAX = 2 ** 31 - 1


def hop_distances(adj_offsets, adj_cols, sources) -> np.ndarray:
    """partition.hpp:58-75: multi-source BFS hop distances, unreachable =
    INT_MAX (scipy's unweighted multi-source Dijkstra = BFS, min over sources)."""
    n = len(adj_offsets) - 1
    g = sp.csr_matrix((np.ones(len(adj_cols)), np.asarray(adj_cols), np.asarray(adj_offsets)), shape=(n, n))
    d = dijkstra(g, unweighted=True, indices=list(sources), min_only=True)
    out = np.full(n, _INT_MAX, dtype=np.int64)
    fin = np.isfinite(d)
    out[fin] = d[fin].astype(np.int64)
    return out


@dataclasses.dataclass
class Partition:
    """partition.hpp:20-29"""

    assignment: np.ndarray  # per-vertex part id
    part_count: int

    def part_sizes(self) -> List[int]:
        return list(np.bincount(self.assignment, minlength=self.part_count))


def partition_mesh(adj_offsets, adj_cols, k: int, seed: int) -> Partition:
    """partition.hpp:84-159: farthest-point seeds (first = mt19937_64(seed)()
    mod n; then the lowest-id vertex at the largest hop distance from all
    seeds, unreachable first), then greedy region growing: always the
    smallest part (lowest id on ties) with a nonempty frontier and size below
    cap = int(ceil(n/k) * 1.1) (any frontier if all are capped) takes the
    first unassigned neighbour of its frontier's front vertex."""
    offs = np.asarray(adj_offsets, dtype=np.int64)
    cols = np.asarray(adj_cols, dtype=np.int64)
    n = len(offs) - 1
    require(k >= 1 and k <= n // 4, "part count k must satisfy 1 <= k <= n/4")
    rng = MT19937_64(seed)
    seeds = [int(rng() % n)]
    while len(seeds) < k:
        dist = hop_distances(offs, cols, seeds)
        seeds.append(int(np.argmax(dist)))  # first index of the maximum
    cap = int(math.ceil(n / k) * 1.1)
    assignment = [-1] * n
    frontier = [[] for _ in range(k)]  # deque as list + head index
    head = [0] * k
    sizes = [0] * k
    assigned = 0
    for p in range(k):
        assignment[seeds[p]] = p
        sizes[p] = 1
        assigned += 1
        frontier[p].append(seeds[p])
    offs_l, cols_l = offs.tolist(), cols.tolist()

    def pick(respect_cap):
        best = -1
        for p in range(k):
            if head[p] >= len(frontier[p]):
                continue
            if respect_cap and sizes[p] >= cap:
                continue
            if best == -1 or sizes[p] < sizes[best]:
                best = p
        return best

    while assigned < n:
        p = pick(True)
        if p == -1:
            p = pick(False)
        if p == -1:
            raise InvalidArgument("partition failed: k is incompatible with the mesh connectivity "
                                  "(a component ended up without a seed)")
        fr = frontier[p]
        grew = False
        while head[p] < len(fr) and not grew:
            v = fr[head[p]]  # front; popped only when it has no unassigned neighbour left
            for j in range(offs_l[v], offs_l[v + 1]):
                w = cols_l[j]
                if assignment[w] != -1:
                    continue
                assignment[w] = p
                sizes[p] += 1
                assigned += 1
                fr.append(w)
                grew = True
                break
            if not grew:
                head[p] += 1
    return Partition(np.asarray(assignment, dtype=np.int32), k)


def overlap_target_size(max_raw_part_size: int, growth: float) -> int:
    """partition.hpp:162-165"""
    require(growth >= 1.0, "overlap growth must be >= 1.0")
    return int(math.floor(growth * max_raw_part_size))


def expand_overlaps(adj_offsets, adj_cols, partition: Partition, growth: float) -> List[np.ndarray]:
    """partition.hpp:205-253: every part grows by BFS rings to exactly
    n_d = floor(growth * max part size) vertices; the last ring is trimmed by
    ascending id; an exhausted component is padded with the smallest unused
    ids.  Returns the sorted member lists (build_submesh sorts, :170)."""
    offs = np.asarray(adj_offsets, dtype=np.int64)
    cols = np.asarray(adj_cols, dtype=np.int64)
    n = len(offs) - 1
    sizes = partition.part_sizes()
    for p in range(partition.part_count):
        require(sizes[p] > 0, "partition has an empty part")
    target = overlap_target_size(max(sizes), growth)
    require(target <= n, "target submesh size exceeds the vertex count")
    out = []
    for p in range(partition.part_count):
        member = np.zeros(n, dtype=bool)
        members = np.nonzero(partition.assignment == p)[0]
        member[members] = True
        count = members.size
        parts = [members]
        ring = members
        while count < target:
            nb = np.concatenate([cols[offs[v]:offs[v + 1]] for v in ring]) if ring.size else np.zeros(0, np.int64)
            nxt = np.unique(nb[~member[nb]])  # sorted, deduplicated
            if nxt.size == 0:
                break
            member[nxt] = True  # "seen" marks the whole ring, even the trimmed part
            room = target - count
            take = nxt[:room]
            parts.append(take)
            count += take.size
            ring = take
        if count < target:
            pad = np.nonzero(~member)[0][:target - count]
            parts.append(pad)
        out.append(np.sort(np.concatenate(parts)).astype(np.int32))
    return out


def order_submeshes(members: Sequence[np.ndarray], seed: int) -> np.ndarray:
    """partition.hpp:258-307: initial submesh mt19937_64(seed)() mod k, then
    BFS over the shared-vertex adjacency graph, neighbours in ascending id,
    restarting at the smallest unvisited id."""
    k = len(members)
    require(k > 0, "cannot order an empty submesh list")
    owners: Dict[int, List[int]] = {}
    for s_, m in enumerate(members):
        for g in np.asarray(m).tolist():
            owners.setdefault(g, []).append(s_)
    adj = [set() for _ in range(k)]
    for lst in owners.values():
        for a in range(len(lst)):
            for b in range(a + 1, len(lst)):
                adj[lst[a]].add(lst[b])
                adj[lst[b]].add(lst[a])
    adjl = [sorted(a) for a in adj]
    initial = int(MT19937_64(seed)() % k)
    seq, visited, queue = [], [False] * k, []
    qh = 0

    def visit(s_):
        visited[s_] = True
        seq.append(s_)
        queue.append(s_)

    visit(initial)
    nxt = 0
    while len(seq) < k:
        if qh >= len(queue):
            while visited[nxt]:
                nxt += 1
            visit(nxt)
            continue
        s_ = queue[qh]
        qh += 1
        for t in adjl[s_]:
            if not visited[t]:
                visit(t)
    return np.asarray(seq, dtype=np.int32)


def segment_mesh(adj_offsets, adj_cols, part_count: int, growth: float, seed: int):
    """pipeline.hpp:131-138 -> (Partition, sorted member lists, sequence)."""
    part = partition_mesh(adj_offsets, adj_cols, part_count, seed)
    members = expand_overlaps(adj_offsets, adj_cols, part, growth)
    return part, members, order_submeshes(members, seed)
