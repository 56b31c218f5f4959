"""SURVEY 8f "next": the iterative-thresholding pipelines (inpaint, separate)
run as device-resident loops over the fused dec/thr/rec path; parity against
golden outputs of the unmodified reference (apps.cpp:179-280)."""
import numpy as np
import pytest

from conftest import golden, rel_l2
import paper_1402_5670_b200 as P

pytestmark = pytest.mark.gpu


def test_inpaint_matches_reference(cuda):
    import torch
    g = golden("it_inpaint128")
    s = P.build_system_2d(128, 128, P.ScaleProfile.from_levels(list(g["levels"])))
    cfg = P.InpaintConfig(iterations=int(g["iterations"]), delta_min=float(g["delta_min"]))
    out = P.inpaint(g["masked"], g["mask"], s, cfg)
    assert rel_l2(out, g["out"]) <= 1e-10
    out_dev = P.inpaint(torch.from_numpy(g["masked"]).to(cuda), torch.from_numpy(g["mask"]).to(cuda), s, cfg)
    assert rel_l2(out_dev.cpu().numpy(), g["out"]) <= 1e-10


def test_inpaint_errors(cuda):
    s = P.build_system_2d(32, 32, P.ScaleProfile.from_levels([0, 1]))
    x = np.zeros((32, 32))
    with pytest.raises(P.DegenerateMaskError):
        P.inpaint(x, np.zeros((32, 32)), s, P.InpaintConfig(iterations=4))
    with pytest.raises(P.DomainError):
        P.inpaint(x, np.full((32, 32), 0.5), s, P.InpaintConfig(iterations=4))
    with pytest.raises(P.ConfigError):
        P.inpaint(x, np.ones((32, 32)), s, P.InpaintConfig(iterations=1))
    with pytest.raises(P.ConfigError):
        P.inpaint(x, np.ones((32, 32)), s, P.InpaintConfig(iterations=4, delta_min=1.5))


def test_separate_matches_reference(cuda):
    g = golden("it_separate128")
    sd = P.build_system_2d(128, 128, P.ScaleProfile.from_levels(list(g["dir_levels"])))
    si = P.build_system_2d(128, 128, P.ScaleProfile.from_levels(list(g["iso_levels"])), fan="impulse")
    cfg = P.InpaintConfig(iterations=int(g["iterations"]), delta_min=float(g["delta_min"]))
    r = P.separate(g["signal"], sd, si, cfg)
    assert rel_l2(r.curvilinear, g["curves"]) <= 1e-10
    assert rel_l2(r.blobs, g["blobs"]) <= 1e-10


def test_inpaint_3d_matches_reference(cuda):
    # Signal3D inpaint (apps.hpp:70-72) through the same device-resident loop
    g = golden("it_inpaint3d32")
    s = P.build_system_3d((32, 32, 32), P.ScaleProfile.from_levels(list(g["levels"])))
    cfg = P.InpaintConfig(iterations=int(g["iterations"]), delta_min=float(g["delta_min"]))
    out = P.inpaint(g["masked"], g["mask"], s, cfg)
    assert rel_l2(out, g["out"]) <= 1e-10
