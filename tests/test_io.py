"""Signal files at the edges of the path (SURVEY 8f "next"): the library's
PGM / SVOL writers produce the reference's bytes (image_io.cpp:77-159, golden
bytes written by the unmodified reference) and its readers parse them back,
with the reference's FormatError cases. Host-only calls: no GPU needed."""
import numpy as np
import pytest

from conftest import golden
import paper_1402_5670_b200 as P


def test_pgm_bytes_match_reference(tmp_path):
    g = golden("io_pgm_svol")
    for name, mv in (("pgm8", 255), ("pgm16", 4095)):
        p = str(tmp_path / f"{name}.pgm")
        P.save_pgm(g["img"] * (mv / 255.0), p, mv)
        assert open(p, "rb").read() == g[name].tobytes()
        im = P.load_pgm(p)
        assert im.maxval == mv
        np.testing.assert_array_equal(im.pixels, g[name + "_loaded"])


def test_svol_bytes_match_reference(tmp_path):
    g = golden("io_pgm_svol")
    p = str(tmp_path / "v.svol")
    P.save_svol(g["vol"], p)
    assert open(p, "rb").read() == g["svol"].tobytes()
    np.testing.assert_array_equal(P.load_svol(p), g["vol"])


def test_pgm_comments_and_errors(tmp_path):
    p = tmp_path / "c.pgm"
    p.write_bytes(b"P5 # comment\n3 # w\n2\n255\n" + bytes([1, 2, 3, 4, 5, 6]))
    im = P.load_pgm(str(p))
    np.testing.assert_array_equal(im.pixels, [[1, 2, 3], [4, 5, 6]])
    bad = {
        "magic.pgm": b"P2\n3 2\n255\n" + bytes(6),
        "trunc.pgm": b"P5\n3 2\n255\n" + bytes(5),
        "hdr.pgm": b"P5\n3 x\n255\n" + bytes(6),
        "zero.pgm": b"P5\n0 2\n255\n",
        "maxval.pgm": b"P5\n3 2\n70000\n" + bytes(12),
        "short.pgm": b"P5\n3",
    }
    for name, data in bad.items():
        (tmp_path / name).write_bytes(data)
        with pytest.raises(P.FormatError):
            P.load_pgm(str(tmp_path / name))
    with pytest.raises(P.FormatError):
        P.load_pgm(str(tmp_path / "missing.pgm"))
    with pytest.raises(P.FormatError):
        P.save_pgm(np.zeros((2, 2)), str(tmp_path / "x.pgm"), 0)


def test_svol_errors(tmp_path):
    good = bytearray(b"SVOL" + (1).to_bytes(2, "little") + b"".join(d.to_bytes(4, "little") for d in (1, 1, 2)))
    good += np.array([1.5, -2.0]).astype("<f8").tobytes()
    (tmp_path / "ok.svol").write_bytes(bytes(good))
    np.testing.assert_array_equal(P.load_svol(str(tmp_path / "ok.svol")), [[[1.5, -2.0]]])
    cases = {
        "magic.svol": b"SVOX" + bytes(good[4:]),
        "version.svol": bytes(good[:4]) + (2).to_bytes(2, "little") + bytes(good[6:]),
        "zero.svol": bytes(good[:6]) + (0).to_bytes(4, "little") + bytes(good[10:]),
        "trunc.svol": bytes(good[:-1]),
    }
    for name, data in cases.items():
        (tmp_path / name).write_bytes(data)
        with pytest.raises(P.FormatError):
            P.load_svol(str(tmp_path / name))


DESC = ["d2_512_1122", "d2_48x40_full_j1", "d2_32_legall", "d3_16_impulse", "d3_16x20x24_legall"]


@pytest.mark.parametrize("name", DESC)
def test_descriptor_text_round_trip(name):
    # read_descriptor / write_descriptor grammar (descriptor.cpp:48-126) on the reference's own texts
    text = str(golden("descriptors")[name + "_text"])
    d = P.SystemDescriptor.parse(text)
    assert d.text() == text


def test_descriptor_parse_errors(tmp_path):
    good = str(golden("descriptors")["d2_32_legall_text"])
    for bad in (good.replace("shearlet-system 1", "shearlet-system 2"), good.replace("dims 32 32", "dims 32"),
                good + "colour blue\n", good.replace("qmf -0.125", "qmf x"), "\n".join(good.splitlines()[:-1])):
        with pytest.raises(P.FormatError):
            P.SystemDescriptor.parse(bad)
    with pytest.raises(P.FormatError):
        P.read_descriptor(str(tmp_path / "missing.txt"))
    p = str(tmp_path / "d.txt")
    P.write_descriptor(P.SystemDescriptor.parse(good), p)
    assert open(p).read() == good
