"""3D parity of the CUDA path (filters synthesised on the fly from factor
tables) against golden fixtures from the unmodified reference and the numpy
oracle; properties from test_transform.cpp:150-200, test_apps.cpp:317-335,
test_system3d.cpp and acceptance.cpp crit. 1."""
import numpy as np
import pytest

from conftest import golden, rel_l2, sample_idx
import paper_1402_5670_b200 as P
from oracle import shearlet_np as O

pytestmark = pytest.mark.gpu

_SYS = {}


def system(dims, levels, full=False, fan="dmaxflat4", shard=None):
    key = (tuple(dims), tuple(levels), full, fan, shard)
    if key not in _SYS:
        _SYS[key] = P.build_system_3d(dims, P.ScaleProfile.from_levels(levels), fan=fan, full_system=full,
                                      shard=shard)
    return _SYS[key]


def test_golden_8cubed_full(cuda):
    g = golden("t3d_8_0_seed80")
    f = g["f"]
    s = system(f.shape, [0])
    np.testing.assert_array_equal(s.index_records, g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    bands = P.forward(f, s)
    assert rel_l2(bands, g["bands"]) <= 1e-10
    assert np.abs(bands - g["bands"]).max() <= 1e-10
    assert rel_l2(P.inverse(g["bands"], s), g["rec"]) <= 1e-10


@pytest.mark.parametrize("name", ["t3d_16_01_rand", "t3d_12x16x20_01"])
def test_golden_stats(cuda, name):
    g = golden(name)
    dims = tuple(int(x) for x in g["dims"])
    s = system(dims, list(g["levels"]))
    np.testing.assert_array_equal(s.index_records, g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    A, B = s.frame_bounds()
    assert abs(A - g["W_min"]) < 1e-12 and abs(B - g["W_max"]) < 1e-12
    W = s.frame_weight.reshape(-1)[sample_idx(int(np.prod(dims)))]
    assert np.abs(W - g["W_sample"]).max() < 1e-12
    for j, i in enumerate(g["filter_ids"]):
        smp = s.filter_freq(int(i)).reshape(-1)[sample_idx(int(np.prod(dims)))]
        assert np.abs(smp - g["filter_samples"][j]).max() < 1e-12
    seed = 70 if name == "t3d_16_01_rand" else 3
    f = np.random.default_rng(seed).uniform(-1, 1, dims)
    assert abs(f.sum() - g["f_sum"]) < 1e-12
    bands = P.forward(f, s)
    np.testing.assert_allclose(np.sqrt((bands.reshape(len(bands), -1) ** 2).sum(1)), g["band_l2"], rtol=1e-10)
    assert rel_l2(bands.reshape(len(bands), -1)[:, sample_idx(f.size)], g["band_sample"]) <= 1e-10
    rec = P.inverse(bands, s)
    assert rel_l2(rec, f) <= 1e-10
    assert rel_l2(rec.reshape(-1)[sample_idx(f.size)], g["rec_sample"]) <= 1e-10


def test_vs_oracle_and_impulse(cuda):
    # test_transform.cpp:150-189 (16^3 [0,1]): round trip, impulse, Plancherel
    s = system((16, 16, 16), [0, 1])
    o = O.build_system_3d((16, 16, 16), [0, 1])
    f = np.random.default_rng(70).uniform(-1, 1, (16, 16, 16))
    assert rel_l2(P.forward(f, s), O.forward_3d(f, o)) <= 1e-10
    d = np.zeros((16, 16, 16)); d[0, 0, 0] = 1.0
    cb = P.forward(d, s)
    idx = (-np.arange(16)) % 16
    for i in range(0, s.redundancy(), 5):
        psi = np.real(np.fft.ifftn(o.filter_freq(i)))
        assert np.abs(cb[i] - psi[idx][:, idx][:, :, idx]).max() <= 1e-10
    A, B = s.frame_bounds()
    total = float(np.sum(P.forward(f, s) ** 2))
    e = float(np.sum(f * f))
    assert A * e * (1 - 1e-9) <= total <= B * e * (1 + 1e-9)


def test_32cubed_denoise_support(cuda):
    g = golden("t3d_32_001")
    s = system((32, 32, 32), [0, 0, 1])
    assert s.redundancy() == 76
    f = np.random.default_rng(2).uniform(-1, 1, (32, 32, 32))
    sch = P.ThresholdSchedule(list(g["K"]), float(g["sigma"]))
    den = P.denoise(f, s, sch)
    thr = P.hard_threshold(P.forward(f, s), sch, s)
    np.testing.assert_array_equal(np.count_nonzero(thr.reshape(76, -1), axis=1), g["kept"])
    assert abs(den.sum() - g["den_sum"]) <= 1e-10 * abs(g["den_sum"]) + 1e-12
    assert rel_l2(den.reshape(-1)[sample_idx(f.size)], g["den_sample"]) <= 1e-10


def test_denoise_sigma0_round_trip(cuda):
    # test_apps.cpp:317-335
    s = system((16, 16, 16), [0, 1])
    v = np.random.default_rng(7).uniform(0, 255, (16, 16, 16))
    assert rel_l2(P.denoise(v, s, P.ThresholdSchedule.defaults_3d(0.0, 2)), v) <= 1e-10


def test_cfg4_128_stats(cuda):
    import torch
    g = golden("cfg4_cartoonvol128_11")
    s = system((128, 128, 128), [1, 1])
    assert s.redundancy() == 99
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    f = P.cartoon_volume(128)
    ft = torch.from_numpy(f).to(cuda)
    bands = P.forward(ft, s)
    l2 = torch.sqrt((bands.reshape(99, -1) ** 2).sum(1)).cpu().numpy()
    np.testing.assert_allclose(l2, g["band_l2"], rtol=1e-10)
    si = torch.from_numpy(sample_idx(f.size)).to(cuda)
    assert rel_l2(bands.reshape(99, -1)[:, si].cpu().numpy(), g["band_sample"]) <= 1e-10
    rec = P.inverse(bands, s)
    assert (torch.linalg.norm(rec - ft) / torch.linalg.norm(ft)).item() <= 1e-10


@pytest.mark.slow
def test_cfg5_192_denoise_support(cuda):
    # SL3D_2 at 192^3 (R=292): identical kept support per band vs the reference
    import torch
    g = golden("cfg5_denoise192_112")
    s = system((192, 192, 192), [1, 1, 2])
    assert s.redundancy() == 292
    # the reference sums 7.1M squares sequentially (system3d.cpp:124-131): ~1e-12 relative rounding
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-10)
    A, B = s.frame_bounds()
    assert abs(A - g["W_min"]) < 1e-12 and abs(B - g["W_max"]) < 1e-12
    noisy = P.add_gaussian_noise(P.cartoon_volume(192), 40.0, 3)
    assert abs(noisy.sum() - g["f_sum"]) <= 1e-9 * abs(g["f_sum"])
    ft = torch.from_numpy(noisy).to(cuda)
    sch = P.ThresholdSchedule.defaults_3d(40.0)
    bands = P.forward(ft, s)
    l2 = torch.sqrt((bands.reshape(292, -1) ** 2).sum(1)).cpu().numpy()
    np.testing.assert_allclose(l2, g["band_l2"], rtol=1e-10)
    si = torch.from_numpy(sample_idx(noisy.size)).to(cuda)
    assert rel_l2(bands.reshape(292, -1)[:, si].cpu().numpy(), g["band_sample"]) <= 1e-10
    thr = P.hard_threshold(bands, sch, s)
    del bands
    kept = torch.count_nonzero(thr.reshape(292, -1), dim=1).cpu().numpy()
    np.testing.assert_array_equal(kept, g["kept"])
    den = P.inverse(thr, s)
    del thr
    d = den.cpu().numpy()
    assert abs(d.sum() - g["den_sum"]) <= 1e-10 * abs(g["den_sum"])
    assert rel_l2(d.reshape(-1)[sample_idx(d.size)], g["den_sample"]) <= 1e-10


def test_shards_sum_to_full(cuda):
    full = system((16, 16, 16), [0, 1])
    R = full.redundancy()
    f = np.random.default_rng(8).uniform(-1, 1, (16, 16, 16))
    cf = P.forward(f, full)
    parts = np.zeros((16, 16, 16))
    for lo, hi in [(0, 20), (20, 41), (41, R)]:
        s = system((16, 16, 16), [0, 1], shard=(lo, hi))
        c = P.forward(f, s)
        np.testing.assert_array_equal(c, cf[lo:hi])
        parts += P.inverse(c, s)
    assert rel_l2(parts, f) <= 1e-10


def test_gpu_construction_matches_oracle(cuda):
    # 3D factor tables built and expanded on the GPU vs the numpy restatement
    s = P.build_system_3d((32, 32, 32), P.ScaleProfile.from_levels([0, 0, 1]))
    o = O.build_system_3d((32, 32, 32), [0, 0, 1])
    np.testing.assert_allclose(s.filter_norms, o.filter_norms, rtol=1e-13)
    for i in (0, 1, 20, 40, 75):
        assert np.abs(s.filter_freq(i) - o.filter_freq(i)).max() <= 1e-13


def test_sharded_denoise_partials_sum_to_full(cuda):
    # denoise on a shard handle returns that shard's partial reconstruction
    # (linear after the per-band threshold), so shards sum to the full denoise
    import torch
    prof = P.ScaleProfile.from_levels([0, 1])
    full = P.build_system_3d((32, 32, 32), prof)
    R = full.redundancy()
    sch = P.ThresholdSchedule.defaults_3d(0.3, 2)
    x = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, (32, 32, 32))).to(cuda)
    want = P.denoise(x, full, sch).cpu().numpy()
    got = np.zeros_like(want)
    for lo, hi in ((0, R // 3), (R // 3, R - 5), (R - 5, R)):
        got += P.denoise(x, P.build_system_3d((32, 32, 32), prof, shard=(lo, hi)), sch).cpu().numpy()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12


def test_batched_api_3d(cuda):
    # batched entry points on a 3D system: frames over the workspace streams == per-volume calls
    import torch
    s = P.build_system_3d((64, 64, 64), P.ScaleProfile.from_levels([0, 1]))
    sch = P.ThresholdSchedule.defaults_3d(0.2, 2)
    rng = np.random.default_rng(9)
    vols = torch.from_numpy(rng.uniform(-1, 1, (3, 64, 64, 64))).to(cuda)
    den = P.denoise_batch(vols, s, sch)
    dec = P.forward_batch(vols, s, sch)
    rec = P.inverse_batch(dec, s)
    host = P.denoise_batch(vols.cpu().numpy(), s, sch)
    for i in range(3):
        one = P.denoise(vols[i], s, sch)
        assert (torch.linalg.norm(den[i] - one) / torch.linalg.norm(one)).item() <= 1e-12
        assert (torch.linalg.norm(rec[i] - one) / torch.linalg.norm(one)).item() <= 1e-12
        assert np.linalg.norm(host[i] - one.cpu().numpy()) <= 1e-12 * np.linalg.norm(host[i])


def test_largest_specialised_sizes_round_trip(cuda):
    # the largest fast-path grids: 2048^2 (2D) and 256^3 (3D); sigma 0 denoise == identity
    import torch
    for shape, lv in (((2048, 2048), [0, 1, 1]), ((256, 256, 256), [0, 1])):
        prof = P.ScaleProfile.from_levels(lv)
        s = P.build_system_2d(*shape, prof) if len(shape) == 2 else P.build_system_3d(shape, prof)
        f = torch.from_numpy(np.random.default_rng(3).uniform(-1, 1, shape)).to(cuda)
        r = P.inverse(P.forward(f, s), s)
        sch = (P.ThresholdSchedule.defaults_2d if len(shape) == 2 else P.ThresholdSchedule.defaults_3d)(0.0, len(lv))
        d = P.denoise(f, s, sch)
        assert (torch.linalg.norm(r - f) / torch.linalg.norm(f)).item() <= 1e-10
        assert (torch.linalg.norm(d - f) / torch.linalg.norm(f)).item() <= 1e-10
        del s, r, d
        torch.cuda.empty_cache()


@pytest.mark.parametrize("n,levels", [(64, [0, 1]), (128, [1, 1]), (192, [0, 0, 1]), (256, [0, 1])])
def test_three_pass_matches_five_pass(cuda, n, levels, monkeypatch):
    # the three-pass path (fast3d_split.cuh, default) against the five-pass
    # kernels (SLB_SPLIT3D=0): dec bands, rec and the fused denoise
    import torch
    prof = P.ScaleProfile.from_levels(levels)
    sch = P.ThresholdSchedule.defaults_3d(0.3, len(levels))
    x = torch.from_numpy(np.random.default_rng(n).uniform(-1, 1, (n, n, n))).to(cuda)
    got = {}
    for split in ("1", "0"):
        monkeypatch.setenv("SLB_SPLIT3D", split)  # knobs are read when the handle is created
        s = P.build_system_3d((n, n, n), prof)
        d, st = P.denoise(x, s, sch, return_stack=True)
        b = P.forward(x, s)
        r = P.inverse(b, s)
        got[split] = (d, st, b, r)
        del s
    (d1, st1, b1, r1), (d0, st0, b0, r0) = got["1"], got["0"]
    rel = lambda a, b: (torch.linalg.norm(a - b) / torch.linalg.norm(b)).item()  # noqa: E731
    assert rel(b1, b0) <= 1e-13 and rel(st1, st0) <= 1e-13
    assert rel(d1, d0) <= 1e-13 and rel(r1, r0) <= 1e-13
    assert rel(r1, x) <= 1e-10


@pytest.mark.parametrize("n,levels,env", [
    (64, [0, 1], {}),
    (64, [2, 2, 2], {"SLB_T3": "0"}),      # > 128 singleton groups: the launch lists split
    (128, [1, 1], {"SLB_CHUNK3": "7"}),     # chunk boundaries cut shear groups
    (192, [0, 0, 1], {}),
])
def test_shear_groups_match_per_band_passes(cuda, n, levels, env, monkeypatch):
    # passes A / C by shear groups (fast3d_group.cuh: one axis-0 FFT per group,
    # pyramid-3 bands in the axis-swapped frame) against one FFT per band
    # (SLB_GROUP3D=0): dec bands, the fused denoise and its stack, rec, and fp32
    import torch
    prof = P.ScaleProfile.from_levels(levels)
    sch = P.ThresholdSchedule.defaults_3d(0.3, len(levels))
    x = torch.from_numpy(np.random.default_rng(n + len(levels)).uniform(-1, 1, (n, n, n))).to(cuda)
    got = {}
    for grp in ("1", "0"):
        monkeypatch.setenv("SLB_GROUP3D", grp)  # knobs are read when the handle is created
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        s = P.build_system_3d((n, n, n), prof)
        d, st = P.denoise(x, s, sch, return_stack=True)
        b = P.forward(x, s)
        r = P.inverse(b, s)
        s32 = P.build_system_3d((n, n, n), prof, dtype="f32")
        d32 = P.denoise(x.float(), s32, P.ThresholdSchedule.defaults_3d(0.0, len(levels)))
        got[grp] = (d, st, b, r, d32)
        del s, s32
    (d1, st1, b1, r1, f1), (d0, st0, b0, r0, f0) = got["1"], got["0"]
    rel = lambda a, b: (torch.linalg.norm(a.double() - b.double()) / torch.linalg.norm(b.double())).item()  # noqa: E731
    assert rel(b1, b0) <= 1e-13 and rel(st1, st0) <= 1e-13
    assert rel(d1, d0) <= 1e-13 and rel(r1, r0) <= 1e-13
    assert rel(r1, x) <= 1e-10
    # thresholded support identical (values within the 1e-13 above)
    assert torch.equal(st1 != 0, st0 != 0)
    assert rel(f1, f0) <= 1e-5 and rel(f1, x) <= 1e-5
