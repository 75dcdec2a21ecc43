"""Seeded synthetic inputs for the five BASELINE.json configurations.

This is input preparation, not part of the measured path: it builds the mesh
(vertices SoA + faces), the ``build_edges`` neighbour lists as CSR
(mesh.hpp:52-70: union of face edges, each list sorted ascending, no
duplicates) and the segmentation (submesh member lists + visiting order) that
the reference's ``compute_block_bases_fixed_sizes`` (pipeline.hpp:144) takes as
its ``Segmentation`` argument.  BASELINE.json names no dataset; the shapes,
sizes and value distributions below follow the config text and SURVEY.md §8(d).

Pinned conventions (SURVEY.md §8(d) "Pinned parameters", echoed in DESIGN.md):
  * grids: W x H vertices, id = y*W + x, integer xy spacing; each quad
    (x,y),(x+1,y),(x,y+1),(x+1,y+1) split along its main diagonal into faces
    (a,b,d), (a,d,c);  z = sum_{k<3} sin(2*pi*(fx_k*x/(W-1) + fy_k*y/(H-1)) + phi_k)
    with fx_k, fy_k ~ U[1,4] cycles over the extent, phi_k ~ U[0, 2*pi), plus
    N(0, sigma^2) on z.
  * grid tiles are row-major (tile id = ty * tiles_x + tx), visited in id order.
  * icosphere: level-7 midpoint subdivision of the icosahedron built from the
    cyclic permutations of (0, +-1, +-phi); radial displacement 0.05 * a seeded
    degree<=4 polynomial restricted to the sphere (= span of real spherical
    harmonics l<=4) normalised to max |h| = 1; then N(0, (0.3*mean edge)^2)
    along the area-weighted vertex normal.  Partition: band = min(64*theta/pi, 63),
    azimuth = atan2(y, x); stable sort by (band, azimuth, id); contiguous parts of
    1024 with the 2 leftover vertices in the last part (1026); every part is then
    equalised by the reference's own ``expand_overlaps`` (partition.hpp:205-253)
    with growth 1.0, so n_d = 1026 and 160 submeshes visited in part order.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

import numpy as np


@dataclasses.dataclass
class Mesh:
    """``Mesh`` (mesh.hpp:18-37) + ``EdgeSet`` (mesh.hpp:40-50) as flat arrays."""

    vertices: np.ndarray  # (n, 3) float64, row per vertex
    faces: np.ndarray  # (n_f, 3) int32
    adj_offsets: np.ndarray  # (n+1,) int32
    adj_cols: np.ndarray  # (2|E|,) int32, each list sorted ascending

    @property
    def n(self) -> int:
        return int(self.vertices.shape[0])

    def neighbors(self, v: int) -> np.ndarray:
        return self.adj_cols[self.adj_offsets[v]:self.adj_offsets[v + 1]]


@dataclasses.dataclass
class Segmentation:
    """``Segmentation`` (pipeline.hpp:125-129) reduced to what the path reads:
    sorted member lists per submesh id and the visiting order."""

    members: List[np.ndarray]  # per submesh id, sorted ascending int32
    sequence: np.ndarray  # permutation of submesh ids (SubmeshOrder)

    @property
    def count(self) -> int:
        return len(self.members)

    @property
    def block_size(self) -> int:
        return int(self.members[0].size)

    def flat(self):
        offs = np.zeros(self.count + 1, dtype=np.int32)
        offs[1:] = np.cumsum([m.size for m in self.members])
        ids = np.concatenate(self.members).astype(np.int32)
        return offs, ids


@dataclasses.dataclass
class Workload:
    name: str
    mesh: Mesh
    seg: Segmentation
    c: int  # fixed c, or initial c for DOI
    iterations: int  # OI t per tile (0 for DOI)
    doi: bool = False
    c_min: int = 0
    c_max: int = 0
    eps_low: float = 0.0
    eps_high: float = 0.0


def build_edges(faces: np.ndarray, n: int):
    """mesh.hpp:52-70 as CSR: union of face edges, neighbour lists sorted, deduped."""
    f = faces.astype(np.int64)
    a, b, c = f[:, 0], f[:, 1], f[:, 2]
    src = np.concatenate([a, b, b, c, c, a])
    dst = np.concatenate([b, a, c, b, a, c])
    key = np.unique(src * n + dst)
    src = key // n
    dst = key % n
    offs = np.zeros(n + 1, dtype=np.int64)
    np.add.at(offs, src + 1, 1)
    offs = np.cumsum(offs)
    return offs.astype(np.int32), dst.astype(np.int32)


def _grid_faces(W: int, H: int) -> np.ndarray:
    x, y = np.meshgrid(np.arange(W - 1), np.arange(H - 1))
    x = x.ravel()
    y = y.ravel()
    a = y * W + x
    b = a + 1
    c = a + W
    d = a + W + 1
    f1 = np.stack([a, b, d], axis=1)
    f2 = np.stack([a, d, c], axis=1)
    # faces of one quad adjacent: (a,b,d), (a,d,c) per quad in row-major quad order
    return np.stack([f1, f2], axis=1).reshape(-1, 3).astype(np.int32)


def grid_mesh(W: int, H: int, seed: int, sigma: float) -> Mesh:
    faces = _grid_faces(W, H)
    offs, cols = build_edges(faces, W * H)
    return Mesh(grid_vertices(W, H, seed, sigma), faces, offs, cols)


def grid_vertices(W: int, H: int, seed: int, sigma: float) -> np.ndarray:
    """Vertices of the seeded height-field grid (connectivity is seed independent)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    fx = rng.uniform(1.0, 4.0, size=3)
    fy = rng.uniform(1.0, 4.0, size=3)
    phi = rng.uniform(0.0, 2.0 * math.pi, size=3)
    ids = np.arange(W * H)
    x = (ids % W).astype(np.float64)
    y = (ids // W).astype(np.float64)
    z = np.zeros(W * H)
    for k in range(3):
        z += np.sin(2.0 * math.pi * (fx[k] * x / (W - 1) + fy[k] * y / (H - 1)) + phi[k])
    z += rng.normal(0.0, sigma, size=W * H)
    return np.stack([x, y, z], axis=1)


def grid_sequence(W: int, H: int, frames: int, seed: int, sigma: float, drift: float = 0.05) -> List[np.ndarray]:
    """A dynamic mesh (frames sharing the grid connectivity, denoise.hpp:248-256):
    the seeded sinusoid surface with per-sinusoid phases advancing by ``drift``
    times a seeded rate each frame, fresh N(0, sigma^2) noise per frame."""
    rng = np.random.Generator(np.random.PCG64(seed))
    fx = rng.uniform(1.0, 4.0, size=3)
    fy = rng.uniform(1.0, 4.0, size=3)
    phi = rng.uniform(0.0, 2.0 * math.pi, size=3)
    rate = rng.uniform(-1.0, 1.0, size=3)
    ids = np.arange(W * H)
    x = (ids % W).astype(np.float64)
    y = (ids // W).astype(np.float64)
    out = []
    for t in range(frames):
        z = np.zeros(W * H)
        for k in range(3):
            z += np.sin(2.0 * math.pi * (fx[k] * x / (W - 1) + fy[k] * y / (H - 1)) + phi[k] + drift * rate[k] * t)
        z += rng.normal(0.0, sigma, size=W * H)
        out.append(np.stack([x, y, z], axis=1))
    return out


def grid_tiles(W: int, H: int, tw: int, th: int) -> Segmentation:
    """Row-major tiles of tw (x) by th (y) vertices; local order ascending id."""
    assert W % tw == 0 and H % th == 0
    members = []
    for ty in range(H // th):
        for tx in range(W // tw):
            xs = np.arange(tx * tw, (tx + 1) * tw)
            ys = np.arange(ty * th, (ty + 1) * th)
            m = (ys[:, None] * W + xs[None, :]).ravel().astype(np.int32)
            members.append(np.sort(m))
    return Segmentation(members, np.arange(len(members), dtype=np.int32))


# --------------------------------------------------------------------------
# icosphere (config 3)

def _icosahedron():
    p = (1.0 + math.sqrt(5.0)) / 2.0
    v = np.array([
        [-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0],
        [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
        [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1],
    ], dtype=np.float64)
    f = np.array([
        [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
        [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
        [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
        [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1],
    ], dtype=np.int64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v, f


def icosphere(level: int):
    v, f = _icosahedron()
    for _ in range(level):
        nv = v.shape[0]
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]], axis=0)
        e.sort(axis=1)
        key = e[:, 0] * (nv + 1) + e[:, 1]
        uniq, inv = np.unique(key, return_inverse=True)
        ea = uniq // (nv + 1)
        eb = uniq % (nv + 1)
        mid = v[ea] + v[eb]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        m = f.shape[0]
        ab = nv + inv[:m]
        bc = nv + inv[m:2 * m]
        ca = nv + inv[2 * m:]
        a, b, c = f[:, 0], f[:, 1], f[:, 2]
        f = np.stack([
            np.stack([a, ab, ca], 1), np.stack([b, bc, ab], 1),
            np.stack([c, ca, bc], 1), np.stack([ab, bc, ca], 1)], axis=1).reshape(-1, 3)
        v = np.concatenate([v, mid], axis=0)
    return v, f.astype(np.int32)


def _vertex_normals(v: np.ndarray, f: np.ndarray) -> np.ndarray:
    a, b, c = v[f[:, 0]], v[f[:, 1]], v[f[:, 2]]
    fn = np.cross(b - a, c - a)  # area-weighted (x2)
    vn = np.zeros_like(v)
    for k in range(3):
        np.add.at(vn, f[:, k], fn)
    return vn / np.linalg.norm(vn, axis=1, keepdims=True)


def mean_edge_length(v: np.ndarray, offs: np.ndarray, cols: np.ndarray) -> float:
    src = np.repeat(np.arange(v.shape[0]), np.diff(offs))
    keep = cols > src
    d = np.linalg.norm(v[src[keep]] - v[cols[keep]], axis=1)
    return float(d.mean())


def sphere_mesh(level: int, seed: int, amplitude: float = 0.05, noise: float = 0.3) -> Mesh:
    rng = np.random.Generator(np.random.PCG64(seed))
    v, f = icosphere(level)
    # degree <= 4 polynomial on the sphere == span of real SH with l <= 4
    exps = [(i, j, k) for d in range(1, 5) for i in range(d + 1) for j in range(d + 1 - i)
            for k in [d - i - j]]
    coef = rng.normal(0.0, 1.0, size=len(exps))
    h = np.zeros(v.shape[0])
    for cf, (i, j, k) in zip(coef, exps):
        h += cf * v[:, 0] ** i * v[:, 1] ** j * v[:, 2] ** k
    h /= np.abs(h).max()
    v = v * (1.0 + amplitude * h)[:, None]
    offs, cols = build_edges(f, v.shape[0])
    ell = mean_edge_length(v, offs, cols)
    nrm = _vertex_normals(v, f)
    v = v + nrm * rng.normal(0.0, noise * ell, size=v.shape[0])[:, None]
    return Mesh(v, f, offs, cols)


def expand_overlaps(mesh: Mesh, assignment: np.ndarray, part_count: int, growth: float):
    """partition.hpp:205-253 restated: BFS rings over the part boundary, last
    ring trimmed by ascending id, padding with the smallest unused ids."""
    n = mesh.n
    sizes = np.bincount(assignment, minlength=part_count)
    assert (sizes > 0).all(), "partition has an empty part"
    target = int(math.floor(growth * int(sizes.max())))
    assert target <= n
    out = []
    for p in range(part_count):
        member = np.zeros(n, dtype=bool)
        members = list(np.nonzero(assignment == p)[0])
        member[members] = True
        ring = list(members)
        while len(members) < target:
            nxt = []
            for v in ring:
                for w in mesh.neighbors(v):
                    if not member[w]:
                        member[w] = True
                        nxt.append(int(w))
            if not nxt:
                break
            nxt.sort()
            room = target - len(members)
            if len(nxt) > room:
                nxt = nxt[:room]
            members.extend(nxt)
            ring = nxt
        v = 0
        while len(members) < target and v < n:
            if not member[v]:
                member[v] = True
                members.append(v)
            v += 1
        out.append(np.sort(np.asarray(members, dtype=np.int32)))
    return out


def sphere_blocks(mesh: Mesh, bands: int = 64, block: int = 1024) -> Segmentation:
    v = mesh.vertices
    r = np.linalg.norm(v, axis=1)
    theta = np.arccos(np.clip(v[:, 2] / r, -1.0, 1.0))
    band = np.minimum(np.floor(bands * theta / math.pi), bands - 1).astype(np.int64)
    azim = np.arctan2(v[:, 1], v[:, 0])
    ids = np.arange(mesh.n)
    order = np.lexsort((ids, azim, band))  # primary band, then azimuth, then id
    parts = mesh.n // block
    assignment = np.empty(mesh.n, dtype=np.int64)
    pos = np.arange(mesh.n)
    assignment[order] = np.minimum(pos // block, parts - 1)
    members = expand_overlaps(mesh, assignment, parts, 1.0)
    return Segmentation(members, np.arange(parts, dtype=np.int32))


# --------------------------------------------------------------------------
# the five configurations (BASELINE.json "configs")

DOI_BAND = (1e-5, 1e-4)  # eps_low, eps_high


def config(name: str, mesh_index: int = 0, seed: Optional[int] = None) -> Workload:
    name = name.upper()
    if name == "C1":
        m = grid_mesh(32, 32, seed if seed is not None else 101, 0.01)
        return Workload("C1", m, grid_tiles(32, 32, 32, 32), c=40, iterations=10)
    if name == "C2":
        m = grid_mesh(256, 256, seed if seed is not None else 202, 0.005)
        return Workload("C2", m, grid_tiles(256, 256, 32, 32), c=100, iterations=1)
    if name == "C3":
        m = sphere_mesh(7, seed if seed is not None else 303)
        return Workload("C3", m, sphere_blocks(m), c=60, iterations=1)
    if name == "C4":
        m = grid_mesh(1024, 1024, seed if seed is not None else 404, 0.01)
        return Workload("C4", m, grid_tiles(1024, 1024, 64, 64), c=20, iterations=0, doi=True,
                        c_min=20, c_max=400, eps_low=DOI_BAND[0], eps_high=DOI_BAND[1])
    if name == "C5":
        s = (seed if seed is not None else 5000) + mesh_index
        m = grid_mesh(512, 512, s, 0.01)
        return Workload("C5", m, grid_tiles(512, 512, 64, 32), c=200, iterations=1)
    raise ValueError(f"unknown config {name}")


def small_grid(W: int, H: int, tw: int, th: int, seed: int = 7, sigma: float = 0.01,
               flip: Optional[int] = None) -> Mesh:
    """Small grids for parity tests.  ``flip`` seeds a per-quad diagonal flip so
    tiles differ (SURVEY.md §0 finding 3: identical tiles hide carry bugs)."""
    m = grid_mesh(W, H, seed, sigma)
    if flip is None:
        return m
    rng = np.random.Generator(np.random.PCG64(flip))
    faces = m.faces.reshape(-1, 2, 3).copy()
    fl = rng.random(faces.shape[0]) < 0.5
    q = np.nonzero(fl)[0]
    a = faces[q, 0, 0]
    b = faces[q, 0, 1]
    d = faces[q, 0, 2]
    c = faces[q, 1, 2]
    faces[q, 0] = np.stack([a, b, c], 1)
    faces[q, 1] = np.stack([b, d, c], 1)
    faces = faces.reshape(-1, 3)
    offs, cols = build_edges(faces, m.n)
    return Mesh(m.vertices, faces, offs, cols)
