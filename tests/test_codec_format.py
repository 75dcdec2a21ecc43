"""CPU checks of the SPECMSH1 container (compress.hpp:378-474): the oracle's
restatement against hand-derived bytes, and the package's host serializer /
parser against the oracle (no GPU: payloads come from the oracle's packer)."""
import struct

import numpy as np
import pytest

import specmesh_oracle as O
from paper_1810_02719_b200 import codec as K


def test_bitpacker_known_answer():
    # q = 3: 5, 2, 7 -> 101 010 111 -> 0b10101011, 0b1 + 7 pad zeros
    b = O.EncodedBlock(0, 1, [0.0] * 3, [1.0] * 3, [0, 0, 0], [5, 2, 7])
    assert O.pack_block_values(b, 3) == bytes([0b10101011, 0b10000000])
    # constant y axis: only x and z values are sent
    b = O.EncodedBlock(0, 2, [0.0] * 3, [1.0] * 3, [0, 1, 0], [1, 0, 9, 9, 3, 2])
    assert O.pack_block_values(b, 4) == bytes([0x10, 0x32])


def test_encode_known_answer():
    coeffs = np.array([[0.0, 1.0, 2.0], [1.0, 1.0, 4.0], [0.5, 1.0, 3.0], [0.25, 1.0, 2.0]])
    b = O.encode_coefficients(coeffs, 2)
    # x: lo 0, hi 1, step 0.25 -> 0, 4 (clamped to 3), 2, 1; y constant; z: step 0.5 -> 0, 4->3, 2, 0
    assert b.values == [0, 3, 2, 1, 0, 0, 0, 0, 0, 3, 2, 0]
    assert b.constant_axis == [0, 1, 0]
    d = O.dequantize_block(b, 2)
    assert d[:, 0].tolist() == [0.125, 0.875, 0.625, 0.375]
    assert d[:, 1].tolist() == [1.0] * 4
    assert d[:, 2].tolist() == [2.25, 3.75, 3.25, 2.25]


def small_encoded():
    faces = np.array([[0, 1, 2], [1, 3, 2]], np.int32)
    enc = O.EncodedMesh(quant_bits=5, part_count=2, subspace_size=3, vertex_count=4, faces=faces, seed=77,
                        shift_scale=1e-3)
    enc.blocks = [O.EncodedBlock(1, 3, [-1.0, 0.0, 2.0], [1.0, 0.0, 3.0], [0, 1, 0], [31, 0, 7, 0, 0, 0, 1, 2, 3]),
                  O.EncodedBlock(0, 2, [0.5, 0.5, 0.5], [0.5, 0.5, 0.5], [1, 1, 1], [0] * 6)]
    return enc


def test_serialize_layout_and_round_trip():
    enc = small_encoded()
    data = O.serialize_encoded_mesh(enc)
    assert data[:8] == b"SPECMSH1"
    assert struct.unpack_from("<IBBH", data, 8) == (1, 0, 0, 5)
    # header 8+4+1+1+2+4+8+4+8+8+20+8+4+8+4+4 = 96, faces 24, block count 4
    assert len(data) == 96 + 24 + 4 + (4 + 4 + 1 + 48 + 4) + (4 + 4 + 1 + 48)
    back = O.parse_encoded_mesh(data)
    assert O.serialize_encoded_mesh(back) == data
    assert back.blocks[0].values == enc.blocks[0].values
    assert np.array_equal(back.faces, enc.faces)


def test_package_serializer_matches_oracle():
    enc = small_encoded()
    data = O.serialize_encoded_mesh(enc)
    pk = K.parse_encoded_mesh(data)
    assert K.serialize_encoded_mesh(pk) == data
    for b, ob in zip(pk.blocks, enc.blocks):
        assert b.payload == O.pack_block_values(ob, enc.quant_bits)
        assert b.values.tolist() == [v if not ob.constant_axis[i // ob.subspace_size] else 0
                                     for i, v in enumerate(ob.values)]
    assert pk.total_bpv() == pytest.approx(enc.total_bpv())


@pytest.mark.parametrize("parse", [O.parse_encoded_mesh, K.parse_encoded_mesh])
def test_parse_errors(parse):
    data = O.serialize_encoded_mesh(small_encoded())
    err = (O.ParseError, K.ParseError)
    with pytest.raises(err, match="bad magic"):
        parse(b"XPECMSH1" + data[8:])
    with pytest.raises(err, match="bitstream truncated"):
        parse(data[:-1])
    with pytest.raises(err, match="trailing bytes"):
        parse(data + b"\0")
    with pytest.raises(err, match="unsupported bitstream version"):
        parse(data[:8] + struct.pack("<I", 2) + data[12:])
    with pytest.raises(err, match="invalid quantization bits"):
        parse(data[:14] + struct.pack("<H", 17) + data[16:])


def test_bits_per_vertex():
    assert O.bits_per_vertex(12, 100, 64, 65536) == K.bits_per_vertex(12, 100, 64, 65536) == 3.515625
    with pytest.raises(Exception, match="must be positive"):
        K.bits_per_vertex(0, 1, 1, 1)
