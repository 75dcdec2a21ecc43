"""F2: the spectral codec (compress.hpp) over the GPU chain.

compress_mesh / decompress_mesh mirror compress.hpp:152-256 with an external
Segmentation (the reference segments internally, compress.hpp:168-174 /
:242-244): the basis chain, the per-block quantisation and the MSB-first
bit-packing run on the GPU (smg_compress_blocks); decoding replays the chain
from connectivity alone and dequantises straight from the packed payload
(smg_decompress_blocks).  serialize_encoded_mesh / parse_encoded_mesh write
and read the reference's SPECMSH1 container (compress.hpp:378-474) byte for
byte: the header is host byte work, each block's payload is the GPU's packed
bytes.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import struct
from typing import List, Optional, Sequence

import numpy as np

from . import _abi
from . import (Context, InvalidArgument, ParseError, PipelineConfig, _i32, _mesh_view, _ptr, _seg_view,
               default_context)

__all__ = ["ParseError", "CompressionConfig", "EncodedBlock", "EncodedMesh", "bits_per_vertex", "compress_mesh",
           "decompress_mesh", "serialize_encoded_mesh", "parse_encoded_mesh", "write_encoded_mesh",
           "read_encoded_mesh"]

MAGIC = b"SPECMSH1"  # compress.hpp:263


@dataclasses.dataclass
class CompressionConfig:
    """compress.hpp:94-97"""

    pipeline: PipelineConfig = dataclasses.field(default_factory=PipelineConfig)
    quant_bits: int = 12


@dataclasses.dataclass
class EncodedBlock:
    """compress.hpp:17-25, plus ``payload``: the block's packed values exactly as
    they appear in the bitstream."""

    submesh_id: int
    subspace_size: int
    coeff_min: List[float]
    coeff_max: List[float]
    constant_axis: List[int]
    payload: bytes
    quant_bits: int

    @property
    def values(self) -> np.ndarray:
        """EncodedBlock.values (axis-major, zeros on constant axes), unpacked."""
        c, q = self.subspace_size, self.quant_bits
        out = np.zeros(3 * c, np.uint16)
        live = [a for a in range(3) if not self.constant_axis[a]]
        if live:
            bits = np.unpackbits(np.frombuffer(self.payload, np.uint8))[:len(live) * c * q].reshape(-1, q)
            vals = (bits.astype(np.uint32) << np.arange(q - 1, -1, -1, dtype=np.uint32)).sum(axis=1)
            for r, a in enumerate(live):
                out[a * c:(a + 1) * c] = vals[r * c:(r + 1) * c]
        return out


@dataclasses.dataclass
class EncodedMesh:
    """compress.hpp:100-150"""

    version: int = 1
    basis_mode: int = 0
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

    def replay_config(self) -> PipelineConfig:
        """compress.hpp:125-143 (Binary: the decoder has no coordinates)."""
        return PipelineConfig(weighting="binary", basis_mode="oi", subspace_size=self.subspace_size,
                              eps_low=self.eps_low, eps_high=self.eps_high, c_min=self.c_min, c_max=self.c_max,
                              power=self.power, iterations=self.iterations,
                              initial_iterations=self.initial_iterations, seed=self.seed,
                              dense_limit=self.dense_limit, shift_scale=self.shift_scale)

    def total_bpv(self) -> float:
        """compress.hpp:145-150"""
        return sum(3 * self.quant_bits * b.subspace_size for b in self.blocks) / self.vertex_count


def bits_per_vertex(quant_bits: int, subspace_size: int, block_count: int, vertex_count: int) -> float:
    """compress.hpp:28-31"""
    if not (quant_bits > 0 and subspace_size > 0 and block_count > 0 and vertex_count > 0):
        raise InvalidArgument("bits_per_vertex arguments must be positive")
    return 3.0 * quant_bits * subspace_size * block_count / float(vertex_count)


class _Blocks:
    """smg_encoded_blocks backing arrays."""

    def __init__(self, k: int, q: int, cap_values: int, cap_payload: int):
        self.k = k
        self.ids = np.zeros(k, np.uint32)
        self.cs = np.zeros(k, np.uint32)
        self.lo = np.zeros(3 * k)
        self.hi = np.zeros(3 * k)
        self.flags = np.zeros(k, np.uint8)
        self.values = np.zeros(max(cap_values, 1), np.uint16)
        self.payload = np.zeros(max(cap_payload, 1), np.uint8)
        self.poff = np.zeros(k + 1, np.int64)
        self.c = _abi.smg_encoded_blocks(k, q, self.ids.ctypes.data, self.cs.ctypes.data, self.lo.ctypes.data,
                                         self.hi.ctypes.data, self.flags.ctypes.data, self.values.ctypes.data,
                                         self.payload.ctypes.data, self.payload.size, self.poff.ctypes.data)


def compress_mesh(mesh, seg, config: CompressionConfig, sizes_in_order: Optional[Sequence[int]] = None,
                  ctx: Optional[Context] = None) -> EncodedMesh:
    """compress_mesh (compress.hpp:152-219) over an external segmentation.
    ``mesh`` carries ``faces`` (stored in the container) and the EdgeSet CSR."""
    ctx = ctx or default_context()
    cfg = dataclasses.replace(config.pipeline, weighting="binary")
    q = config.quant_bits
    if not (1 <= q <= 16):
        raise InvalidArgument("quantization bits must be in [1,16]")
    k = seg.count
    keep: list = []
    mv, sv = _mesh_view(mesh, keep), _seg_view(seg, keep)
    sizes = None if sizes_in_order is None else _i32(sizes_in_order)
    if cfg.basis_mode == "doi":
        cm = cfg.c_max if cfg.c_max > 0 else max(64, 2 * cfg.subspace_size)
        cap_c = min(cm, seg.block_size)
    else:
        cap_c = int(sizes.max()) if sizes is not None else cfg.subspace_size
    cap_values = 3 * k * cap_c
    cap_payload = k * ((3 * cap_c * q + 7) // 8)
    blk = _Blocks(k, q, cap_values, cap_payload)
    cc = cfg.to_c()
    ctx.check(ctx.lib.smg_compress_blocks(ctx.handle, C.byref(mv), C.byref(sv), C.byref(cc), _ptr(sizes), q,
                                          C.byref(blk.c)))
    enc = EncodedMesh(basis_mode=_abi.BASIS_MODE[cfg.basis_mode], quant_bits=q, part_count=k,
                      subspace_size=cfg.subspace_size, eps_low=cfg.eps_low, eps_high=cfg.eps_high, c_min=cfg.c_min,
                      c_max=cfg.c_max, power=cfg.power, iterations=cfg.iterations,
                      initial_iterations=cfg.initial_iterations, seed=cfg.seed, dense_limit=cfg.dense_limit,
                      shift_scale=cfg.shift_scale, vertex_count=mesh.n, faces=np.asarray(mesh.faces, np.int32))
    for p in range(k):
        enc.blocks.append(EncodedBlock(int(blk.ids[p]), int(blk.cs[p]), [float(v) for v in blk.lo[3 * p:3 * p + 3]],
                                       [float(v) for v in blk.hi[3 * p:3 * p + 3]],
                                       [(int(blk.flags[p]) >> a) & 1 for a in range(3)],
                                       blk.payload[blk.poff[p]:blk.poff[p + 1]].tobytes(), q))
    return enc


def decompress_mesh(encoded: EncodedMesh, seg, topology=None, ctx: Optional[Context] = None) -> np.ndarray:
    """decompress_mesh (compress.hpp:221-256) over an external segmentation:
    replays the chain from the connectivity (``topology``'s EdgeSet CSR, or the
    container's faces through build_edges, mesh.hpp:52-70), decodes on the GPU,
    stitches with degree weights.  Returns the n x 3 vertices."""
    ctx = ctx or default_context()
    from . import synth
    if topology is None:
        offs, cols = synth.build_edges(np.asarray(encoded.faces), encoded.vertex_count)
        topology = synth.Mesh(np.zeros((encoded.vertex_count, 3)), np.asarray(encoded.faces), offs, cols)
    keep: list = []
    mv, sv = _mesh_view(topology, keep), _seg_view(seg, keep)
    k = len(encoded.blocks)
    blk = _Blocks(k, encoded.quant_bits, 0, sum(len(b.payload) for b in encoded.blocks))
    for p, b in enumerate(encoded.blocks):
        blk.ids[p], blk.cs[p] = b.submesh_id, b.subspace_size
        blk.lo[3 * p:3 * p + 3] = b.coeff_min
        blk.hi[3 * p:3 * p + 3] = b.coeff_max
        blk.flags[p] = b.constant_axis[0] | (b.constant_axis[1] << 1) | (b.constant_axis[2] << 2)
        blk.poff[p + 1] = blk.poff[p] + len(b.payload)
        blk.payload[blk.poff[p]:blk.poff[p + 1]] = np.frombuffer(b.payload, np.uint8)
    blk.c.values = None
    out = np.zeros(3 * encoded.vertex_count)
    cc = encoded.replay_config().to_c()
    ctx.check(ctx.lib.smg_decompress_blocks(ctx.handle, C.byref(mv), C.byref(sv), C.byref(cc), C.byref(blk.c),
                                            out.ctypes.data, 0))
    return out.reshape((3, encoded.vertex_count)).T.copy()


def serialize_encoded_mesh(enc: EncodedMesh) -> bytes:
    """compress.hpp:392-426 (little endian; block payloads as packed on the GPU)."""
    o = bytearray(MAGIC)
    o += struct.pack("<IBBH", enc.version, enc.basis_mode, 0, enc.quant_bits)
    o += struct.pack("<IdI", enc.part_count, enc.growth, enc.subspace_size)
    o += struct.pack("<dd", enc.eps_low, enc.eps_high)
    o += struct.pack("<IIIII", enc.c_min, enc.c_max, enc.power, enc.iterations, enc.initial_iterations)
    o += struct.pack("<QId", enc.seed & ((1 << 64) - 1), enc.dense_limit, enc.shift_scale)
    faces = np.asarray(enc.faces, np.int64).reshape(-1, 3)
    o += struct.pack("<II", enc.vertex_count, faces.shape[0])
    o += faces.astype("<u4").tobytes()
    o += struct.pack("<I", len(enc.blocks))
    for b in enc.blocks:
        o += struct.pack("<IIB", b.submesh_id, b.subspace_size,
                         b.constant_axis[0] | (b.constant_axis[1] << 1) | (b.constant_axis[2] << 2))
        o += struct.pack("<3d", *b.coeff_min)
        o += struct.pack("<3d", *b.coeff_max)
        o += b.payload
    return bytes(o)


def parse_encoded_mesh(data: bytes) -> EncodedMesh:
    """compress.hpp:428-474, with the reference's ParseError messages."""
    data = bytes(data)
    at = [0]

    def take(n):
        if at[0] + n > len(data):
            raise ParseError("bitstream truncated")
        v = data[at[0]:at[0] + n]
        at[0] += n
        return v

    def un(fmt):
        return struct.unpack(fmt, take(struct.calcsize(fmt)))

    if take(8) != MAGIC:
        raise ParseError("not a specmesh bitstream (bad magic)")
    e = EncodedMesh()
    (e.version,) = un("<I")
    if e.version != 1:
        raise ParseError("unsupported bitstream version")
    e.basis_mode, _w, e.quant_bits = un("<BBH")
    if e.quant_bits < 1 or e.quant_bits > 16:
        raise ParseError("bitstream has invalid quantization bits")
    e.part_count, e.growth, e.subspace_size = un("<IdI")
    e.eps_low, e.eps_high = un("<dd")
    e.c_min, e.c_max, e.power, e.iterations, e.initial_iterations = un("<IIIII")
    e.seed, e.dense_limit, e.shift_scale = un("<QId")
    e.vertex_count, nf = un("<II")
    e.faces = np.frombuffer(take(12 * nf), "<u4").astype(np.int32).reshape(nf, 3)
    (nb,) = un("<I")
    for _ in range(nb):
        sid, c, flags = un("<IIB")
        lo = list(un("<3d"))
        hi = list(un("<3d"))
        const = [(flags >> a) & 1 for a in range(3)]
        nbytes = ((3 - sum(const)) * c * e.quant_bits + 7) // 8
        e.blocks.append(EncodedBlock(sid, c, lo, hi, const, take(nbytes), e.quant_bits))
    if at[0] != len(data):
        raise ParseError("trailing bytes after bitstream payload")
    return e


def write_encoded_mesh(enc: EncodedMesh, path: str) -> None:
    """compress.hpp:476-483"""
    with open(path, "wb") as f:
        f.write(serialize_encoded_mesh(enc))


def read_encoded_mesh(path: str) -> EncodedMesh:
    """compress.hpp:485-491"""
    try:
        with open(path, "rb") as f:
            return parse_encoded_mesh(f.read())
    except OSError:
        raise ParseError(f"cannot open '{path}'") from None
