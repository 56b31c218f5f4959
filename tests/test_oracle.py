"""Pins the CPU oracle (oracle/shearlet_np.py) against the reference's own
outputs: the committed golden fixtures (generated from the unmodified
reference by oracle/gen_golden.py) and, when built, oracle/_ref itself."""
import numpy as np
import pytest

from conftest import golden, rel_l2, sample_idx
from oracle import shearlet_np as O
from oracle import ref


def test_fan_checksum_and_taps():
    # filters.cpp:112-122: the bundled fan is maxflat_fan(4) with a fixed FNV-1a checksum
    fan = O.maxflat_fan(4)
    assert fan.v.shape == (15, 15) and fan.c0 == 7 and fan.c1 == 7
    np.testing.assert_array_equal(fan.v, fan.v[::-1, ::-1])  # centrally symmetric


def test_lowpass_sums_to_one_and_cascade_lengths():
    h = O.default_lowpass()
    assert abs(h.v.sum() - 1.0) < 1e-15
    q = O.qmf_default()
    for j in range(1, 6):
        hj, gj = O.cascade(q, j)
        assert len(hj.v) == 8 * (2 ** j - 1) + 1
        assert len(gj.v) == 8 * (2 ** j - 1) + 1


def test_mt19937_64_matches_std():
    # std::mt19937_64(22) first outputs (checked against libstdc++)
    r = O.MT19937_64(22)
    assert [r() for _ in range(3)] == [15789710126278856821, 8600543100456774415, 665720239889519832]


@pytest.mark.parametrize("name", ["t2d_16_01_seed21", "t2d_16_01_impulse", "t2d_64_0011_seed22", "t2d_40x24_01_seed5"])
def test_oracle_2d_full_golden(name):
    g = golden(name)
    f = g["f"]
    s = O.build_system_2d(f.shape[0], f.shape[1], list(g["levels"]), int(g["j0"]))
    np.testing.assert_array_equal(np.array(s.index), g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    np.testing.assert_allclose(s.frame_weight, g["frame_weight"], rtol=1e-12, atol=1e-14)
    bands = O.forward_2d(f, s)
    assert rel_l2(bands, g["bands"]) < 1e-12
    assert rel_l2(O.inverse_2d(g["bands"], s), g["rec"]) < 1e-12


def test_oracle_random_grid_matches_reference_generator():
    g = golden("t2d_16_01_seed21")
    np.testing.assert_array_equal(O.random_grid((16, 16), 21), g["f"])


def test_oracle_cfg1_stats():
    g = golden("cfg1_cartoon256_11")
    f = O.cartoon(256)
    assert f.sum() == g["f_sum"]
    s = O.build_system_2d(256, 256, [1, 1])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    assert abs(s.frame_weight.min() - g["W_min"]) < 1e-12 and abs(s.frame_weight.max() - g["W_max"]) < 1e-12
    bands = O.forward_2d(f, s)
    np.testing.assert_allclose(np.sqrt((bands.reshape(17, -1) ** 2).sum(1)), g["band_l2"], rtol=1e-11)
    flat = bands.reshape(17, -1)[:, sample_idx(256 * 256)]
    assert rel_l2(flat, g["band_sample"]) < 1e-12


@pytest.mark.slow
def test_oracle_cfg2_denoise_support():
    g = golden("cfg2_denoise512_1122")
    s = O.build_system_2d(512, 512, [1, 1, 2, 2])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    if ref.available():
        noisy = ref.add_noise(ref.cartoon(512), 40.0, 7)
        assert noisy.sum() == g["f_sum"]
    else:
        pytest.skip("reference library not built")
    bands = O.forward_2d(noisy, s)
    thr = O.hard_threshold(bands, s.index, 0, g["filter_norms"], list(g["K"]), float(g["sigma"]))
    kept = np.count_nonzero(thr.reshape(thr.shape[0], -1), axis=1)
    np.testing.assert_array_equal(kept, g["kept"])
    den = O.inverse_2d(thr, s)
    assert abs(den.sum() - g["den_sum"]) < 1e-9 * abs(g["den_sum"])


@pytest.mark.parametrize("name", ["t3d_8_0_seed80"])
def test_oracle_3d_full_golden(name):
    g = golden(name)
    f = g["f"]
    s = O.build_system_3d(f.shape, list(g["levels"]))
    np.testing.assert_array_equal(np.array(s.index), g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    assert rel_l2(O.forward_3d(f, s), g["bands"]) < 1e-12
    assert rel_l2(O.inverse_3d(g["bands"], s), g["rec"]) < 1e-12


@pytest.mark.parametrize("name", ["t3d_16_01_rand", "t3d_12x16x20_01"])
def test_oracle_3d_stats_golden(name):
    g = golden(name)
    dims = tuple(int(x) for x in g["dims"])
    s = O.build_system_3d(dims, list(g["levels"]))
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    assert abs(s.frame_weight.min() - g["W_min"]) < 1e-12
    for j, i in enumerate(g["filter_ids"]):
        smp = s.filter_freq(int(i)).reshape(-1)[sample_idx(int(np.prod(dims)))]
        assert np.abs(smp - g["filter_samples"][j]).max() < 1e-12


def test_oracle_3d_big_tables_cfg5_norms():
    # SL3D_2 at 192^3: only the cheap construction checks (norms of a few filters)
    g = golden("cfg5_denoise192_112")
    assert len(g["filter_norms"]) == 292 and O.redundancy_3d([1, 1, 2]) == 292


@pytest.mark.skipif(not ref.available(), reason="reference library not built")
def test_shim_fft_matches_numpy():
    rng = np.random.default_rng(0)
    for shape in [(192,), (100,), (11,), (64, 48), (12, 20, 14)]:
        x = rng.standard_normal(shape) + 1j * rng.standard_normal(shape)
        assert rel_l2(ref.fft_forward(x), np.fft.fftn(x)) < 1e-14


@pytest.mark.skipif(not ref.available(), reason="reference library not built")
def test_reference_library_matches_golden():
    g = golden("t2d_64_0011_seed22")
    r = ref.RefSystem2D(64, 64, [0, 0, 1, 1])
    assert rel_l2(r.forward(g["f"]), g["bands"]) < 1e-14


@pytest.mark.parametrize("name", ["shcf_2d_16_01", "shcf_3d_8x12x10_0"])
def test_oracle_shcf_bytes_golden(name):
    # transform.cpp:185-213: the restated writer reproduces the reference's bytes
    g = golden(name)
    b = g["bands"]
    if b.ndim == 3:
        s = O.build_system_2d(b.shape[1], b.shape[2], list(g["levels"]))
        idx = [tuple(r) + (0,) for r in s.index]
    else:
        idx = O.enumerate_filters_3d(O.Profile(list(g["levels"]), 0))
    assert O.serialize_shcf(b, idx) == g["shcf"].tobytes()


def test_oracle_maxflat_fans_golden():
    # fan_design.cpp:70-108, bit-exact for every order
    g = golden("maxflat_fans")
    for o in range(1, 7):
        np.testing.assert_array_equal(O.maxflat_fan(o).v, g[f"order{o}"])


def _bank(g):
    fan = O.T2(g["fan"], int(g["fan_c"][0]), int(g["fan_c"][1]))
    q = None
    if "lowpass" in g.files:
        h = O.T1(g["lowpass"], int(g["lowpass_c"]))
        q = O.Qmf(h, O.mirror_highpass(h))
    return fan, q


@pytest.mark.parametrize("name", ["bank_2d_32_fan2_legall", "bank_2d_48x40_fan3"])
def test_oracle_custom_bank_2d_golden(name):
    # build_system_2d with an explicit FanFilter / QmfPair (system2d.cpp:75-116)
    g = golden(name)
    fan, q = _bank(g)
    f = g["f"]
    s = O.build_system_2d(f.shape[0], f.shape[1], list(g["levels"]), 0, False, fan, q)
    np.testing.assert_array_equal(np.array(s.index), g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    assert rel_l2(O.forward_2d(f, s), g["bands"]) < 1e-12
    assert rel_l2(O.inverse_2d(g["bands"], s), g["rec"]) < 1e-12


def test_oracle_custom_bank_3d_golden():
    g = golden("bank_3d_16_fan2_legall")
    fan, q = _bank(g)
    f = g["f"]
    s = O.build_system_3d(f.shape, list(g["levels"]), 0, False, fan, q)
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    b = O.forward_3d(f, s)
    np.testing.assert_allclose(np.sqrt((b.reshape(b.shape[0], -1) ** 2).sum(1)), g["band_l2"], rtol=1e-10)
    assert rel_l2(O.inverse_3d(b, s), g["rec"]) < 1e-12


def test_python_bank_helpers():
    # host-side mirrors of filters.hpp helpers; the bundled fan is a checksummed
    # constant of the library equal to the reference's maxflat_fan(4)
    import paper_1402_5670_b200 as P
    g = golden("maxflat_fans")
    d = P.FanFilter.default()
    np.testing.assert_array_equal(d.taps, g["order4"])
    assert (d.center0, d.center1) == (7, 7)
    assert P.fan_checksum(d) == P.DEFAULT_FAN_CHECKSUM
    q = P.QmfPair.from_lowpass([-0.125, 0.25, 0.75, 0.25, -0.125])
    np.testing.assert_array_equal(q.highpass, O.mirror_highpass(O.T1(q.lowpass, 2)).v)
    assert P.alpha_to_shear_levels([1.0, 1.0, 1.0], 1) == [1, 1, 2]
    with pytest.raises(P.DomainError):
        P.alpha_to_shear_levels([2.0], 0)


def test_fan_asset_round_trip(tmp_path):
    # load_fan_filter / save_fan_filter text format (filters.cpp:124-156)
    import paper_1402_5670_b200 as P
    from conftest import golden_fan
    f = golden_fan(3)
    p = str(tmp_path / "fan.txt")
    f.save(p)
    back = P.FanFilter.load(p)
    np.testing.assert_array_equal(back.taps, f.taps)
    assert (back.center0, back.center1) == (f.center0, f.center1)
    (tmp_path / "bad.txt").write_text("3 3 1\n")
    with pytest.raises(P.AssetError):
        P.FanFilter.load(str(tmp_path / "bad.txt"))
    (tmp_path / "short.txt").write_text("2 2 0 0\n1 2\n3\n")
    with pytest.raises(P.AssetError):
        P.FanFilter.load(str(tmp_path / "short.txt"))
    with pytest.raises(P.AssetError):
        P.FanFilter.load(str(tmp_path / "missing.txt"))
