"""System descriptors (SURVEY 8f "next"; descriptor.hpp:12-39): describe() of
a GPU-built system reproduces the reference's text, and a system rebuilt on the
GPU from the reference's text has the reference's filter bank (RMS pinned)."""
import numpy as np
import pytest

from conftest import golden, golden_fan
import paper_1402_5670_b200 as P

pytestmark = pytest.mark.gpu

LEGALL = P.QmfPair.from_lowpass([-0.125, 0.25, 0.75, 0.25, -0.125], 2)


def _build(name):
    prof = P.ScaleProfile.from_levels
    if name == "d2_512_1122":
        return P.build_system_2d(512, 512, prof([1, 1, 2, 2]))
    if name == "d2_48x40_full_j1":
        return P.build_system_2d(48, 40, prof([0, 1], 1), full_system=True)
    if name == "d2_32_legall":
        return P.build_system_2d(32, 32, prof([0, 1]), fan=golden_fan(2), qmf=LEGALL)
    if name == "d3_16_impulse":
        return P.build_system_3d((16, 16, 16), prof([0, 1]), fan="impulse")
    return P.build_system_3d((16, 20, 24), prof([0, 1]), qmf=LEGALL)


@pytest.mark.parametrize("name", ["d2_512_1122", "d2_48x40_full_j1", "d2_32_legall", "d3_16_impulse",
                                  "d3_16x20x24_legall"])
def test_describe_matches_reference(cuda, name):
    g = golden("descriptors")
    s = _build(name)
    d = P.describe(s)
    text = str(g[name + "_text"])
    if name == "d2_32_legall":  # maxflat_fan(2) carries provenance "dmaxflat2" -> "custom"
        assert d.fan_name == "custom"
    assert d.text() == text
    np.testing.assert_allclose(s.filter_norms, g[name + "_rms"], rtol=1e-12)


@pytest.mark.parametrize("name", ["d2_512_1122", "d2_48x40_full_j1", "d3_16_impulse", "d3_16x20x24_legall"])
def test_build_from_reference_descriptor(cuda, name):
    g = golden("descriptors")
    d = P.SystemDescriptor.parse(str(g[name + "_text"]))
    s = P.build_from_descriptor_3d(d) if d.is_3d else P.build_from_descriptor_2d(d)
    np.testing.assert_allclose(s.filter_norms, g[name + "_rms"], rtol=1e-12)
    assert P.describe(s).text() == d.text()
    with pytest.raises(P.FormatError):  # wrong kind
        (P.build_from_descriptor_2d if d.is_3d else P.build_from_descriptor_3d)(d)


def test_descriptor_fan_errors(cuda):
    g = golden("descriptors")
    d = P.SystemDescriptor.parse(str(g["d2_32_legall_text"]))
    with pytest.raises(P.FormatError):  # custom fans cannot be rebuilt (descriptor.cpp:134-135)
        P.build_from_descriptor_2d(d)
    d = P.SystemDescriptor.parse(str(g["d2_48x40_full_j1_text"]))
    d.fan_checksum ^= 1
    with pytest.raises(P.FormatError):
        P.build_from_descriptor_2d(d)
