"""The reference's acceptance criteria for this path (tests/acceptance.cpp),
run on the GPU path: criterion 1 (accuracy and time budget), 6 (noisy-input
PSNR pin), 7 (directional beats separable denoising, values pinned to the
unmodified reference) and 10 (module invariants)."""
import time

import numpy as np
import pytest

from conftest import golden
import paper_1402_5670_b200 as P
from oracle import shearlet_np as O

pytestmark = pytest.mark.gpu


def test_criterion1_accuracy_and_time(cuda):
    # acceptance.cpp:55-73: 128^2 [0,0,1,1] seed 1 and 32^3 [0,0,1] seed 2, round trip <= 1e-10 in < 5 s
    f = O.random_grid((128, 128), 1)
    t0 = time.perf_counter()
    s = P.build_system_2d(128, 128, P.ScaleProfile.from_levels([0, 0, 1, 1]))
    r = P.inverse(P.forward(f, s), s)
    assert time.perf_counter() - t0 < 5.0
    assert np.linalg.norm(r - f) / np.linalg.norm(f) <= 1e-10
    v = np.random.default_rng(2).uniform(-1, 1, (32, 32, 32))
    t0 = time.perf_counter()
    s3 = P.build_system_3d((32, 32, 32), P.ScaleProfile.from_levels([0, 0, 1]))
    r3 = P.inverse(P.forward(v, s3), s3)
    assert time.perf_counter() - t0 < 5.0
    assert np.linalg.norm(r3 - v) / np.linalg.norm(v) <= 1e-10


def test_criterion6_noisy_psnr_pin():
    # acceptance.cpp:165-171: sigma 40 on the 512^2 cartoon gives 16.06 +- 0.15 dB
    img = P.cartoon(512)
    p = P.psnr(img, P.add_gaussian_noise(img, 40.0, 7))
    assert abs(p - 16.06) <= 0.15


def test_criterion7_directional_beats_separable(cuda):
    # acceptance.cpp:173-191, PSNRs pinned to the reference's own values
    g = golden("acceptance_c7")
    img = P.cartoon(256)
    noisy = P.add_gaussian_noise(img, 30.0, 11)
    sch = P.ThresholdSchedule.defaults_2d(30.0)
    sl2 = P.build_system_2d(256, 256, P.ScaleProfile.from_levels([1, 1, 2, 2]))
    swt = P.build_system_2d(256, 256, P.ScaleProfile.from_levels([0, 0, 0, 0]), fan="impulse")
    p_noisy = P.psnr(img, noisy)
    p_sl2 = P.psnr(img, P.denoise(noisy, sl2, sch))
    p_swt = P.psnr(img, P.denoise(noisy, swt, sch))
    assert p_sl2 - p_noisy >= 6.0 and p_sl2 >= p_swt + 0.5
    assert abs(p_noisy - float(g["p_noisy"])) <= 1e-9
    assert abs(p_sl2 - float(g["p_sl2"])) <= 1e-6
    assert abs(p_swt - float(g["p_swt"])) <= 1e-6


def test_criterion10_invariants(cuda):
    # acceptance.cpp:279-369: Plancherel within the frame bounds, translation covariance
    s = P.build_system_2d(32, 32, P.ScaleProfile.from_levels([0, 1]))
    A, B = s.frame_bounds()
    f = O.random_grid((32, 32), 77)
    c = P.forward(f, s)
    e, e0 = float((c * c).sum()), float((f * f).sum())
    assert A * e0 * (1 - 1e-9) <= e <= B * e0 * (1 + 1e-9)
    sh = np.roll(f, (5, -3), axis=(0, 1))
    cs = P.forward(sh, s)
    assert np.abs(cs - np.roll(c, (5, -3), axis=(1, 2))).max() <= 1e-12 * np.abs(c).max()
