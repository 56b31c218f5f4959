"""build_system_2d/3d with an explicit FanFilter / QmfPair (system2d.hpp:66-69,
system3d.hpp:68-71): the GPU-built filter bank and transforms against golden
outputs of the unmodified reference built with the same fan and QMF taps."""
import numpy as np
import pytest

from conftest import golden, rel_l2, sample_idx
import paper_1402_5670_b200 as P

pytestmark = pytest.mark.gpu


def _bank(g):
    fan = P.FanFilter(g["fan"], int(g["fan_c"][0]), int(g["fan_c"][1]), "test")
    qmf = P.QmfPair.from_lowpass(g["lowpass"], int(g["lowpass_c"])) if "lowpass" in g.files else None
    return fan, qmf


@pytest.mark.parametrize("name", ["bank_2d_32_fan2_legall", "bank_2d_48x40_fan3"])
def test_custom_bank_2d(cuda, name):
    g = golden(name)
    fan, qmf = _bank(g)
    f = g["f"]
    s = P.build_system_2d(f.shape[0], f.shape[1], P.ScaleProfile.from_levels(list(g["levels"])), fan=fan, qmf=qmf)
    np.testing.assert_array_equal(s.index_records[:, :3], g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-10)
    assert rel_l2(s.frame_weight, g["frame_weight"]) <= 1e-12
    bands = P.forward(f, s)
    assert rel_l2(bands, g["bands"]) <= 1e-10
    assert rel_l2(P.inverse(g["bands"], s), g["rec"]) <= 1e-10


def test_custom_bank_3d(cuda):
    g = golden("bank_3d_16_fan2_legall")
    fan, qmf = _bank(g)
    f = g["f"]
    s = P.build_system_3d(f.shape, P.ScaleProfile.from_levels(list(g["levels"])), fan=fan, qmf=qmf)
    np.testing.assert_array_equal(s.index_records, g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-10)
    np.testing.assert_allclose(s.frame_weight.reshape(-1)[sample_idx(f.size)], g["W_sample"], rtol=1e-10)
    bands = P.forward(f, s)
    flat = bands.reshape(bands.shape[0], -1)
    np.testing.assert_allclose(np.sqrt((flat * flat).sum(1)), g["band_l2"], rtol=1e-10)
    np.testing.assert_allclose(flat[:, sample_idx(flat.shape[1])], g["band_sample"], rtol=1e-9, atol=1e-12)
    assert rel_l2(P.inverse(bands, s), g["rec"]) <= 1e-10


def test_default_bank_equals_explicit(cuda):
    # passing the default fan explicitly builds the same system as the built-in default
    prof = P.ScaleProfile.from_levels([0, 1])
    a = P.build_system_2d(64, 64, prof)
    b = P.build_system_2d(64, 64, prof, fan=P.FanFilter.default())
    np.testing.assert_array_equal(a.filter_norms, b.filter_norms)
    f = np.random.default_rng(1).standard_normal((64, 64))
    np.testing.assert_array_equal(P.forward(f, a), P.forward(f, b))


def test_asymmetric_fan_2d_complex_3d_rejected(cuda):
    # 2D keeps complex filter tables for an off-centre fan (tests/test_gpu_asym.py);
    # the 3D factor tables assume real spectra, so 3D refuses it loudly
    fan = P.FanFilter(np.array([[0.0, 1.0, 0.5]]), 0, 0, "asym")
    s = P.build_system_2d(32, 32, P.ScaleProfile.from_levels([0, 1]), fan=fan)
    f = np.random.default_rng(1).uniform(-1, 1, (32, 32))
    assert rel_l2(P.inverse(P.forward(f, s), s), f) <= 1e-10
    with pytest.raises(P.DomainError):
        P.build_system_3d((16, 16, 16), P.ScaleProfile.from_levels([0, 1]), fan=fan)
    with pytest.raises(P.InvalidArgument):
        P.build_system_2d(32, 32, P.ScaleProfile.from_levels([0, 1]), fan=P.FanFilter(np.zeros((0, 3)), 0, 0))
