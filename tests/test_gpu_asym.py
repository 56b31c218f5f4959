"""Asymmetric fans (filters.hpp:64: any fan): the filters stay real in space
but their spectra are complex (Hermitian); the reference stores full complex
grids (system2d.hpp:38). Such a system keeps complex filter tables and runs
the generic 2D path; parity against the unmodified reference
(tests/golden/bank_2d_*_asym.npz from oracle/gen_golden.py --only asym)."""
import numpy as np
import pytest

from conftest import golden, rel_l2
import paper_1402_5670_b200 as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name", ["bank_2d_32_asym", "bank_2d_64_asym"])
def test_asymmetric_fan_matches_reference(cuda, name):
    import torch
    g = golden(name)
    fan = P.FanFilter(np.array(g["fan"]), int(g["fan_c"][0]), int(g["fan_c"][1]), "test-asym")
    f = g["f"]
    n = f.shape[0]
    s = P.build_system_2d(n, n, P.ScaleProfile.from_levels(list(g["levels"])), fan=fan)
    np.testing.assert_array_equal(s.index_records[:, :3], g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    np.testing.assert_allclose(s.frame_weight, g["frame_weight"], rtol=1e-12, atol=1e-14)
    psi1 = s.filter_freq(1)
    assert np.abs(psi1.imag).max() > 0.1  # genuinely complex
    assert np.abs(psi1 - g["filter1"]).max() <= 1e-12
    b = P.forward(f, s)
    assert rel_l2(b, g["bands"]) <= 1e-10
    assert rel_l2(P.inverse(b, s), g["rec"]) <= 1e-10
    sch = P.ThresholdSchedule(list(g["K"]), float(g["sigma"]))
    assert rel_l2(P.denoise(f, s, sch), g["den"]) <= 1e-10
    bt = P.forward(torch.from_numpy(f).to(cuda), s)
    assert rel_l2(bt.cpu().numpy(), g["bands"]) <= 1e-10
