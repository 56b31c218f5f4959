"""Parity sweep: many grid shapes, scale profiles, j0, full systems and both
fans against the numpy oracle (itself pinned to the reference), through the
fast and generic paths: forward, denoise (threshold support) and round trip."""
import numpy as np
import pytest

import paper_1402_5670_b200 as P
from oracle import shearlet_np as O

pytestmark = pytest.mark.gpu

CASES_2D = [
    ((8, 8), [0], 0, False), ((16, 24), [0, 1], 0, True), ((30, 18), [1], 1, False), ((64, 64), [1, 1], 0, False),
    ((48, 80), [0, 0, 1], 0, False), ((128, 128), [0, 1, 2], 0, False), ((100, 60), [2], 0, True),
    ((192, 192), [0, 1], 1, False), ((256, 256), [1, 1], 0, True), ((36, 36), [0, 1], 0, False),
]
CASES_3D = [((8, 8, 8), [0], 0, False), ((16, 12, 20), [0, 1], 0, False), ((24, 24, 24), [1], 0, True),
            ((64, 64, 64), [0, 1], 0, False), ((10, 16, 14), [0], 1, False)]


@pytest.mark.parametrize("shape,levels,j0,full", CASES_2D)
@pytest.mark.parametrize("fan", ["dmaxflat4", "impulse"])
def test_sweep_2d(cuda, shape, levels, j0, full, fan):
    prof = P.ScaleProfile.from_levels(levels, j0)
    s = P.build_system_2d(*shape, prof, fan=fan, full_system=full)
    o = O.build_system_2d(*shape, levels, j0, full, O.impulse_fan() if fan == "impulse" else None)
    f = np.random.default_rng(sum(shape) + len(levels)).uniform(-1, 1, shape)
    b = P.forward(f, s)
    ob = O.forward_2d(f, o)
    assert np.linalg.norm(b - ob) / np.linalg.norm(ob) <= 1e-10
    np.testing.assert_allclose(s.filter_norms, o.filter_norms, rtol=1e-12)
    sigma = 0.05
    K = [2.0 + 0.5 * i for i in range(len(levels))]
    sch = P.ThresholdSchedule(K, sigma, True)
    thr = O.hard_threshold(ob, o.index, j0, o.filter_norms, K, sigma)
    gthr = P.hard_threshold(b, sch, s)
    assert np.array_equal(gthr != 0, thr != 0)
    den = P.denoise(f, s, sch)
    ref = O.inverse_2d(thr, o)
    assert np.linalg.norm(den - ref) / np.linalg.norm(ref) <= 1e-10
    assert np.linalg.norm(P.inverse(b, s) - f) / np.linalg.norm(f) <= 1e-10


@pytest.mark.parametrize("shape,levels,j0,full", CASES_3D)
def test_sweep_3d(cuda, shape, levels, j0, full):
    prof = P.ScaleProfile.from_levels(levels, j0)
    s = P.build_system_3d(shape, prof, full_system=full)
    o = O.build_system_3d(shape, levels, j0, full)
    f = np.random.default_rng(sum(shape)).uniform(-1, 1, shape)
    b = P.forward(f, s)
    ob = O.forward_3d(f, o)
    assert np.linalg.norm(b - ob) / np.linalg.norm(ob) <= 1e-10
    K = [3.0 + 0.5 * i for i in range(len(levels))]
    sch = P.ThresholdSchedule(K, 0.05, True)
    thr = O.hard_threshold(ob, o.index, j0, o.filter_norms, K, 0.05)
    den = P.denoise(f, s, sch)
    ref = O.inverse_3d(thr, o)
    assert np.linalg.norm(den - ref) / np.linalg.norm(ref) <= 1e-10
    assert np.linalg.norm(P.inverse(b, s) - f) / np.linalg.norm(f) <= 1e-10
