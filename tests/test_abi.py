"""CPU-side checks of the C ABI: the library loads, exports every symbol the
header declares, the Python mirror matches the reference API surface, and the
host-only entry points (input generators, error mapping) behave like the
reference. No kernel launches here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_1402_5670_b200 as P
from oracle import shearlet_np as O


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "shearlet_b200.h")).read()
    return sorted(set(re.findall(r"\b(sl_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = C.CDLL(P.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(P.EXPORTED_SYMBOLS) == syms


def test_version_and_last_error():
    L = P.lib()
    assert b"sm_100a" in L.sl_version()
    assert isinstance(L.sl_last_error(), bytes)


def test_null_handle_is_invalid_argument():
    L = P.lib()
    R = C.c_int()
    assert L.sl_redundancy(None, C.byref(R)) == 22
    with pytest.raises(P.InvalidArgument):
        P._check(L.sl_redundancy(None, C.byref(R)))


def test_error_code_mapping_matches_reference_classes():
    assert P._CODES[2] is P.ShapeError and P._CODES[3] is P.ConfigError
    assert P._CODES[5] is P.SingularFrameError and P._CODES[6] is P.UnsupportedSizeError
    for cls in P._CODES.values():
        assert issubclass(cls, P.Error)


def test_cartoon_matches_oracle_and_reference():
    np.testing.assert_array_equal(P.cartoon(64), O.cartoon(64))
    assert P.cartoon(256).sum() == golden("cfg1_cartoon256_11")["f_sum"]


def test_noise_matches_reference_generator():
    # cfg2 input: add_gaussian_noise(cartoon(512), 40, seed 7), apps.cpp:47-55
    noisy = P.add_gaussian_noise(P.cartoon(512), 40.0, 7)
    assert noisy.sum() == golden("cfg2_denoise512_1122")["f_sum"]
    assert np.array_equal(P.add_gaussian_noise(P.cartoon(16), 0.0, 3), P.cartoon(16))
    with pytest.raises(P.DomainError):
        P.add_gaussian_noise(P.cartoon(8), -1.0, 1)


def test_cartoon_volume_matches_reference():
    g = golden("cfg4_cartoonvol128_11")
    assert P.cartoon_volume(128).sum() == g["f_sum"]


def test_profiles_and_schedules():
    p = P.ScaleProfile.from_levels([1, 1, 2, 2])
    assert p.n_scales == 4 and p.top_level() == 4
    assert P.redundancy_2d(p) == 49 and P.redundancy_3d(P.ScaleProfile.from_levels([1, 1, 2])) == 292
    assert P.redundancy_3d(P.ScaleProfile.from_levels([0, 0, 1])) == 76
    assert P.ScaleProfile.parabolic(4, 1).shear_levels == [1, 1, 2, 2]
    assert P.ThresholdSchedule.defaults_2d(40).per_scale_factors == [2.5, 2.5, 2.5, 3.8]
    assert P.ThresholdSchedule.defaults_3d(40).per_scale_factors == [3.0, 3.0, 4.0]
    with pytest.raises(P.ConfigError):
        P.ScaleProfile.from_levels([1, -1])


def test_small_grid_rejected_before_device_work():
    with pytest.raises(P.UnsupportedSizeError):
        P.build_system_2d(4, 16, P.ScaleProfile.from_levels([0]))
    with pytest.raises(P.UnsupportedSizeError):
        P.build_system_3d((8, 8, 4), P.ScaleProfile.from_levels([0]))


def test_product_path_never_imports_oracle():
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_1402_5670_b200")):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".hpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle/", "").lower() or f == "__init__.py", f
                assert "import oracle" not in txt and "from oracle" not in txt, f
