"""Q / Q_opt separation-quality metrics (apps.cpp:282-362):
GPU blurs through the single-band decomposition, pinned against the
unmodified reference's values."""
import numpy as np
import pytest

from conftest import golden
import paper_1402_5670_b200 as P

pytestmark = pytest.mark.gpu


def test_gaussian_kernel_matches_reference():
    g = golden("quality_q")
    np.testing.assert_array_equal(P.gaussian_kernel(2.0).taps, g["gauss2"])
    np.testing.assert_array_equal(P.gaussian_kernel(0.7).taps, g["gauss07"])
    with pytest.raises(P.DomainError):
        P.gaussian_kernel(0.0)


@pytest.mark.parametrize("name,sigma", [("s2", 2.0), ("s07", 0.7)])
def test_quality_matches_reference(cuda, name, sigma):
    g = golden("quality_q")
    gk = P.gaussian_kernel(sigma)
    q, d = P.quality_q_opt(g["rec"], g["truth"], gk)
    assert d == int(g[f"dopt_{name}"])
    assert abs(q - float(g[f"qopt_{name}"])) <= 1e-12 * float(g[f"qopt_{name}"])
    q40 = P.quality_q(g["rec"], g["truth"], 40.0, gk)
    assert abs(q40 - float(g[f"q40_{name}"])) <= 1e-12 * float(g[f"q40_{name}"])


def test_quality_generic_grid(cuda):
    # 96 x 80 has no specialised FFT plan: the generic mixed-radix path blurs
    g = golden("quality_q")
    q, d = P.quality_q_opt(g["rec"][:96, :80], g["truth"][:96, :80], P.gaussian_kernel(1.5))
    assert d == int(g["dopt_crop"])
    assert abs(q - float(g["qopt_crop"])) <= 1e-12 * float(g["qopt_crop"])


def test_quality_errors(cuda):
    g = golden("quality_q")
    with pytest.raises(P.DomainError):
        P.quality_q_opt(g["rec"], g["truth"] * 2.0)
    with pytest.raises(P.DegenerateTruthError):
        P.quality_q_opt(g["rec"], np.zeros_like(g["truth"]))
    with pytest.raises(P.DomainError):
        P.quality_q(g["rec"], g["truth"], -1.0)
    with pytest.raises(P.ShapeError):
        P.quality_q(g["rec"], g["truth"][:64], 1.0)
