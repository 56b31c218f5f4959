"""SURVEY 8f "next": SHCF coefficient files (transform.hpp:39-52,
transform.cpp:127-269). The library's writer must produce the reference's
bytes for the same stack, its reader must return the stack bit-exactly and
reject malformed streams with the reference's error classes; a GPU forward
stack written by the library must read back through the reference format."""
import struct

import numpy as np
import pytest

from conftest import golden, rel_l2
import paper_1402_5670_b200 as P

pytestmark = pytest.mark.gpu


def _system(g):
    b = g["bands"]
    prof = P.ScaleProfile.from_levels(list(g["levels"]))
    if b.ndim == 3:
        return P.build_system_2d(b.shape[1], b.shape[2], prof)
    return P.build_system_3d(b.shape[1:], prof)


@pytest.mark.parametrize("name", ["shcf_2d_16_01", "shcf_3d_8x12x10_0"])
def test_serialize_is_byte_identical(cuda, name):
    g = golden(name)
    s = _system(g)
    assert P.serialize(g["bands"], s) == g["shcf"].tobytes()


@pytest.mark.parametrize("name", ["shcf_2d_16_01", "shcf_3d_8x12x10_0"])
def test_deserialize_round_trip(cuda, name):
    g = golden(name)
    s = _system(g)
    back = P.deserialize(g["shcf"].tobytes(), s)
    np.testing.assert_array_equal(back, g["bands"])


@pytest.mark.parametrize("name", ["shcf_2d_16_01", "shcf_3d_8x12x10_0"])
def test_gpu_forward_serialized(cuda, name):
    # GPU stack -> SHCF -> parse: same header/records as the reference, data within parity tolerance
    g = golden(name)
    s = _system(g)
    ref_bytes = g["shcf"].tobytes()
    f = P.inverse(g["bands"], s)  # any signal whose forward we compare against forward on the GPU
    stack = P.forward(f, s)
    data = P.serialize(stack, s)
    hdr = len(ref_bytes) - g["bands"].size * 8
    assert data[:hdr] == ref_bytes[:hdr]
    back = np.frombuffer(data[hdr:], dtype="<f8").reshape(g["bands"].shape)
    np.testing.assert_array_equal(back, stack)


def test_deserialize_errors(cuda):
    g = golden("shcf_2d_16_01")
    s = _system(g)
    good = g["shcf"].tobytes()
    with pytest.raises(P.FormatError):
        P.deserialize(b"SHCX" + good[4:], s)  # bad magic
    with pytest.raises(P.FormatError):
        P.deserialize(good[:4] + struct.pack("<H", 2) + good[6:], s)  # version
    with pytest.raises(P.FormatError):
        P.deserialize(good[:6] + bytes([4]) + good[7:], s)  # dimensionality
    with pytest.raises(P.FormatError):
        P.deserialize(good[:-8], s)  # truncated data
    with pytest.raises(P.FormatError):
        P.deserialize(good[:20], s)  # truncated records
    with pytest.raises(P.FormatError):
        bad = bytearray(good)
        bad[19] = 7  # first record's kind
        P.deserialize(bytes(bad), s)
    with pytest.raises(P.ShapeError):
        P.deserialize(good[:7] + struct.pack("<I", 32) + good[11:], s)  # rows differ from the system
    with pytest.raises(P.ShapeError):
        bad = bytearray(good)
        bad[20:24] = struct.pack("<i", 3)  # first record's scale
        P.deserialize(bytes(bad), s)
    s3 = P.build_system_3d((8, 12, 10), P.ScaleProfile.from_levels([0]))
    with pytest.raises(P.FormatError):
        P.deserialize(good, s3)  # a 2D stream into a 3D system
    with pytest.raises(P.ShapeError):
        P.serialize(g["bands"][:-1], s)


@pytest.mark.parametrize("shape,levels,chunk", [((64, 64), [0, 1, 1], 7), ((32, 32, 32), [0, 1], 10)])
def test_streamed_files(cuda, tmp_path, shape, levels, chunk):
    # decompose straight to / reconstruct straight from an SHCF file, chunk by chunk
    prof = P.ScaleProfile.from_levels(levels)
    s = P.build_system_2d(*shape, prof) if len(shape) == 2 else P.build_system_3d(shape, prof)
    f = np.random.default_rng(4).uniform(-1, 1, shape)
    path = str(tmp_path / "c.shcf")
    P.forward_to_file(f, s, path, chunk)
    stack = P.forward(f, s)
    assert open(path, "rb").read() == P.serialize(stack, s)
    r = P.inverse_from_file(path, s, chunk)
    want = P.inverse(stack, s)
    assert np.linalg.norm(r - want) / np.linalg.norm(want) <= 1e-13
    assert np.linalg.norm(r - f) / np.linalg.norm(f) <= 1e-10
    bad = tmp_path / "bad.shcf"
    bad.write_bytes(open(path, "rb").read()[:-8])
    with pytest.raises(P.FormatError):
        P.inverse_from_file(str(bad), s, chunk)
    with pytest.raises(P.FormatError):
        P.inverse_from_file(str(tmp_path / "missing.shcf"), s)
