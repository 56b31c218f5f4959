"""2D parity of the CUDA path (through the C ABI) against the reference:
golden fixtures generated from the unmodified reference, the numpy oracle,
and the reference test suite's properties (test_transform.cpp, test_apps.cpp,
test_system2d.cpp, acceptance.cpp). Tolerances: 1e-10 relative L2 (north_star)
unless the reference test states a tighter one."""
import numpy as np
import pytest

from conftest import golden, rel_l2, sample_idx
import paper_1402_5670_b200 as P
from oracle import shearlet_np as O

pytestmark = pytest.mark.gpu

_SYS = {}


def system(n0, n1, levels, j0=0, full=False, fan="dmaxflat4", shard=None):
    key = (n0, n1, tuple(levels), j0, full, fan, shard)
    if key not in _SYS:
        _SYS[key] = P.build_system_2d(n0, n1, P.ScaleProfile.from_levels(levels, j0), fan=fan,
                                      full_system=full, shard=shard)
    return _SYS[key]


@pytest.mark.parametrize("name", ["t2d_16_01_seed21", "t2d_16_01_impulse", "t2d_64_0011_seed22",
                                  "t2d_40x24_01_seed5"])
def test_golden_full(cuda, name):
    g = golden(name)
    f = g["f"]
    s = system(f.shape[0], f.shape[1], list(g["levels"]))
    assert s.redundancy() == len(g["index"])
    np.testing.assert_array_equal(s.index_records[:, :3], g["index"])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    np.testing.assert_allclose(s.frame_weight, g["frame_weight"], rtol=1e-12, atol=1e-14)
    bands = P.forward(f, s)
    assert rel_l2(bands, g["bands"]) <= 1e-10
    assert np.abs(bands - g["bands"]).max() <= 1e-10 * max(1.0, np.abs(f).max())
    rec = P.inverse(g["bands"], s)
    assert rel_l2(rec, g["rec"]) <= 1e-10
    assert rel_l2(rec, f) <= 1e-10


def test_filter_spectra_match_oracle(cuda):
    s = system(64, 64, [0, 0, 1, 1])
    o = O.build_system_2d(64, 64, [0, 0, 1, 1])
    for i in range(s.redundancy()):
        assert np.abs(s.filter_freq(i) - o.filters[i]).max() < 1e-12


def test_impulse_reproduces_reversed_taps(cuda):
    # test_transform.cpp:26-40
    s = system(16, 16, [0, 1])
    o = O.build_system_2d(16, 16, [0, 1])
    d = np.zeros((16, 16)); d[0, 0] = 1.0
    bands = P.forward(d, s)
    for i in range(s.redundancy()):
        psi = np.real(np.fft.ifft2(o.filters[i]))
        rev = psi[(-np.arange(16)) % 16][:, (-np.arange(16)) % 16]
        assert np.abs(bands[i] - rev).max() <= 1e-10


def test_constant_lands_in_lowpass(cuda):
    # test_transform.cpp:42-53
    s = system(32, 32, [0, 0])
    c = 37.5
    bands = P.forward(np.full((32, 32), c), s)
    for i, rec in enumerate(s.index):
        if rec[0] != 0:
            assert np.abs(bands[i]).max() <= 1e-6 * c


def test_linearity_zero_and_shape_errors(cuda):
    # test_transform.cpp:74-113
    s = system(32, 32, [0, 1])
    zero = np.zeros((s.redundancy(), 32, 32))
    assert np.linalg.norm(P.inverse(zero, s)) == 0.0
    rng = np.random.default_rng(31)
    f, g = rng.uniform(-1, 1, (32, 32)), rng.uniform(-1, 1, (32, 32))
    cf, cg = P.forward(f, s), P.forward(g, s)
    a, b = 0.7, -2.3
    lhs = P.inverse(a * cf + b * cg, s)
    assert np.abs(lhs - (a * P.inverse(cf, s) + b * P.inverse(cg, s))).max() <= 1e-12
    with pytest.raises(P.ShapeError):
        P.forward(np.zeros((16, 16)), s)
    with pytest.raises(P.ShapeError):
        P.inverse(np.zeros((s.redundancy() - 1, 32, 32)), s)


def test_plancherel_bounds(cuda):
    # test_transform.cpp:115-129
    s = system(64, 64, [0, 0, 1])
    A, B = s.frame_bounds()
    for seed in (50, 51, 52):
        f = np.random.default_rng(seed).uniform(-1, 1, (64, 64))
        total = float(np.sum(P.forward(f, s) ** 2))
        e = float(np.sum(f * f))
        assert A * e * (1 - 1e-9) <= total <= B * e * (1 + 1e-9)


def test_translation_covariance(cuda):
    # test_transform.cpp:131-148
    s = system(32, 32, [0, 1])
    f = np.random.default_rng(60).uniform(-1, 1, (32, 32))
    sh = np.roll(f, (5, 11), axis=(0, 1))
    cf, cs = P.forward(f, s), P.forward(sh, s)
    assert np.abs(np.roll(cf, (5, 11), axis=(1, 2)) - cs).max() <= 1e-12


def test_frame_weight_and_duals(cuda):
    # test_system2d.cpp:149-171: W = sum |psi|^2; sum gamma conj(psi) == 1
    s = system(64, 64, [0, 0, 1, 1])
    psi = np.stack([s.filter_freq(i) for i in range(s.redundancy())])
    W = np.sum(np.abs(psi) ** 2, axis=0)
    assert np.abs(W - s.frame_weight).max() <= 1e-12
    assert np.abs(np.sum(np.abs(psi) ** 2 / s.frame_weight, axis=0) - 1).max() <= 1e-12
    A, B = s.frame_bounds()
    assert 0 < A <= B and abs(A - W.min()) < 1e-14 and abs(B - W.max()) < 1e-14


def test_cfg1_stats(cuda):
    g = golden("cfg1_cartoon256_11")
    s = system(256, 256, [1, 1])
    f = P.cartoon(256)
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    A, B = s.frame_bounds()
    assert abs(A - g["W_min"]) < 1e-12 and abs(B - g["W_max"]) < 1e-12
    bands = P.forward(f, s)
    np.testing.assert_allclose(np.sqrt((bands.reshape(17, -1) ** 2).sum(1)), g["band_l2"], rtol=1e-10)
    assert rel_l2(bands.reshape(17, -1)[:, sample_idx(256 * 256)], g["band_sample"]) <= 1e-10
    rec = P.inverse(bands, s)
    assert rel_l2(rec, f) <= 1e-10
    assert rel_l2(rec.reshape(-1)[sample_idx(256 * 256)], g["rec_sample"]) <= 1e-10


def test_cfg2_denoise_support_identity(cuda):
    # 512^2 [1,1,2,2] (R=49), cartoon + noise(40, seed 7), defaults_2d(40)
    g = golden("cfg2_denoise512_1122")
    s = system(512, 512, [1, 1, 2, 2])
    np.testing.assert_allclose(s.filter_norms, g["filter_norms"], rtol=1e-12)
    noisy = P.add_gaussian_noise(P.cartoon(512), 40.0, 7)
    assert noisy.sum() == g["f_sum"]
    bands = P.forward(noisy, s)
    np.testing.assert_allclose(np.sqrt((bands.reshape(49, -1) ** 2).sum(1)), g["band_l2"], rtol=1e-10)
    sch = P.ThresholdSchedule.defaults_2d(40.0)
    thr = P.hard_threshold(bands, sch, s)
    kept = np.count_nonzero(thr.reshape(49, -1), axis=1)
    np.testing.assert_array_equal(kept, g["kept"])  # identical thresholded support
    den = P.inverse(thr, s)
    assert abs(den.sum() - g["den_sum"]) <= 1e-10 * abs(g["den_sum"])
    assert abs(np.sqrt((den * den).sum()) - g["den_l2"]) <= 1e-10 * g["den_l2"]
    assert rel_l2(den.reshape(-1)[sample_idx(512 * 512)], g["den_sample"]) <= 1e-10
    # fused denoise entry point == the composed one
    den2 = P.denoise(noisy, s, sch)
    assert rel_l2(den2, den) <= 1e-12
    # PSNR pins
    clean = P.cartoon(512)
    assert abs(P.psnr(clean, noisy) - 16.0868) < 1e-3
    assert abs(P.psnr(clean, den) - 32.7223) < 1e-3


def test_device_path_matches_host_path(cuda):
    import torch
    s = system(512, 512, [1, 1, 2, 2])
    f = P.add_gaussian_noise(P.cartoon(512), 40.0, 7)
    ft = torch.from_numpy(f).to(cuda)
    b_dev = P.forward(ft, s)
    b_host = P.forward(f, s)
    assert torch.equal(b_dev.cpu(), torch.from_numpy(b_host))
    sch = P.ThresholdSchedule.defaults_2d(40.0)
    fused = P.forward_thresholded(ft, s, sch)
    sep = P.hard_threshold(b_dev, sch, s)
    assert torch.equal(fused, sep)
    r_dev = P.inverse(fused, s)
    assert rel_l2(r_dev.cpu().numpy(), P.inverse(sep.cpu().numpy(), s)) == 0.0


def test_hard_threshold_semantics(cuda):
    # test_apps.cpp:53-95
    s = system(32, 32, [0, 1])
    f = np.random.default_rng(5).uniform(-1, 1, (32, 32))
    c = P.forward(f, s)
    same = P.hard_threshold(c, P.ThresholdSchedule([1.0, 1.0], 0.0), s)
    np.testing.assert_array_equal(same, c)  # sigma = 0 keeps everything
    sch = P.ThresholdSchedule([0.9, 1.3], 0.05)
    t1 = P.hard_threshold(c, sch, s)
    np.testing.assert_array_equal(t1[0], c[0])  # lowpass untouched
    np.testing.assert_array_equal(P.hard_threshold(t1, sch, s), t1)  # idempotent
    ref = O.hard_threshold(c, s.index, 0, s.filter_norms, sch.per_scale_factors, sch.sigma)
    np.testing.assert_array_equal(t1, ref)
    unscaled = P.ThresholdSchedule([2.0, 2.0], 1.0, False)
    x = np.zeros_like(c); x[1, 0, :3] = [3.0, -1.0, 5.0]
    np.testing.assert_array_equal(P.hard_threshold(x, unscaled, s)[1, 0, :3], [3.0, 0.0, 5.0])
    with pytest.raises(P.ConfigError):
        P.hard_threshold(c, P.ThresholdSchedule([1.0], 0.1), s)
    with pytest.raises(P.ConfigError):
        P.hard_threshold(c, P.ThresholdSchedule([1.0, 1.0], -0.1), s)
    with pytest.raises(P.ConfigError):
        P.hard_threshold(c, P.ThresholdSchedule([1.0, 0.0], 0.1), s)


def test_denoise_sigma0_round_trip_and_shift(cuda):
    # test_apps.cpp:97-123
    s = system(64, 64, [0, 0, 1])
    f = np.random.default_rng(9).uniform(0, 255, (64, 64))
    assert rel_l2(P.denoise(f, s, P.ThresholdSchedule.defaults_2d(0.0, 3)), f) <= 1e-10
    sch = P.ThresholdSchedule.defaults_2d(20.0, 3)
    d1 = P.denoise(f, s, sch)
    d2 = P.denoise(np.roll(f, (3, 7), axis=(0, 1)), s, sch)
    assert np.abs(np.roll(d1, (3, 7), axis=(0, 1)) - d2).max() <= 1e-10 * np.abs(d1).max()


def test_full_system_and_impulse_fan(cuda):
    # full_system keeps the boundary shears; impulse fan is the isotropic system
    for full, fan in [(True, "dmaxflat4"), (False, "impulse")]:
        s = system(32, 32, [0, 1], full=full, fan=fan)
        o = O.build_system_2d(32, 32, [0, 1], full=full, fan=O.impulse_fan() if fan == "impulse" else None)
        assert s.redundancy() == o.R
        np.testing.assert_allclose(s.filter_norms, o.filter_norms, rtol=1e-12)
        f = np.random.default_rng(4).uniform(-1, 1, (32, 32))
        assert rel_l2(P.forward(f, s), O.forward_2d(f, o)) <= 1e-10
        assert rel_l2(P.inverse(P.forward(f, s), s), f) <= 1e-10


@pytest.mark.parametrize("shape,levels", [((48, 80), [0, 1]), ((30, 50), [0, 0, 1]), ((36, 36), [1]),
                                          ((128, 96), [0, 1, 1]), ((27, 25), [0])])
def test_odd_and_mixed_radix_shapes(cuda, shape, levels):
    s = system(shape[0], shape[1], levels)
    o = O.build_system_2d(shape[0], shape[1], levels)
    f = np.random.default_rng(11).uniform(-1, 1, shape)
    assert rel_l2(P.forward(f, s), O.forward_2d(f, o)) <= 1e-10
    assert rel_l2(P.inverse(P.forward(f, s), s), f) <= 1e-10


def test_full_size_round_trips(cuda):
    # size-independent property at BASELINE sizes: exact reconstruction
    import torch
    for n, lv in [(512, [1, 1, 2, 2]), (1024, [1, 1, 2, 2])]:
        s = system(n, n, lv)
        f = torch.from_numpy(P.add_gaussian_noise(P.cartoon(n), 40.0, 1)).to(cuda)
        rec = P.inverse(P.forward(f, s), s)
        assert (torch.linalg.norm(rec - f) / torch.linalg.norm(f)).item() <= 1e-10


def test_shards_sum_to_full(cuda):
    # shearlet-index sharding: dec shards are slices, rec partials sum to the full rec
    full = system(64, 64, [0, 0, 1, 1])
    R = full.redundancy()
    f = np.random.default_rng(3).uniform(-1, 1, (64, 64))
    cf = P.forward(f, full)
    parts = np.zeros((64, 64))
    for lo, hi in [(0, 7), (7, 13), (13, R)]:
        s = system(64, 64, [0, 0, 1, 1], shard=(lo, hi))
        c = P.forward(f, s)
        np.testing.assert_array_equal(c, cf[lo:hi])
        parts += P.inverse(c, s)
    assert rel_l2(parts, f) <= 1e-10


def test_batched_api_matches_per_frame(cuda):
    import torch
    s = system(256, 256, [1, 1])
    sch = P.ThresholdSchedule.defaults_2d(30.0, 2)
    frames = np.stack([P.add_gaussian_noise(P.cartoon(256), 30.0, i) for i in range(5)])
    ft = torch.from_numpy(frames).to(cuda)
    s.set_streams(3)
    den_b = P.denoise_batch(ft, s, sch)
    dec_b = P.forward_batch(ft, s, sch)
    rec_b = P.inverse_batch(dec_b, s)
    host_b = P.denoise_batch(frames, s, sch)
    torch.cuda.synchronize()
    for i in range(5):
        one = P.denoise(ft[i], s, sch)
        # batched frames use the concurrent band grouping (G), a different summation association
        assert (torch.linalg.norm(den_b[i] - one) / torch.linalg.norm(one)).item() <= 1e-12
        assert torch.equal(rec_b[i], one)
        assert torch.equal(dec_b[i], P.forward_thresholded(ft[i], s, sch))
        assert np.linalg.norm(host_b[i] - one.cpu().numpy()) <= 1e-12 * np.linalg.norm(host_b[i])
    with pytest.raises(P.ShapeError):
        P.denoise_batch(ft[:, :128], s, sch)


@pytest.mark.parametrize("pipe,group", [("0", "1"), ("1", "1"), ("3", "1"), ("6", "1"), ("3", "2"), ("2", "3"),
                                        ("-1", "-1")])
def test_host_batch_pipelines_agree(cuda, monkeypatch, pipe, group):
    # the pipelined host batch (copy streams + SLB_HOST_PIPE compute streams,
    # SLB_PIPE_GROUP lock-step frames per stream, ragged last group) and the
    # per-frame fan-out return the per-frame result for every frame
    s = system(128, 128, [1, 2])
    sch = P.ThresholdSchedule.defaults_2d(25.0, 2)
    nfr = 7 if pipe != "-1" else 19  # auto schedule: >= 16 frames take head frame + lock-step pairs
    frames = np.stack([P.add_gaussian_noise(P.cartoon(128), 25.0, 40 + i) for i in range(nfr)])
    monkeypatch.setenv("SLB_HOST_PIPE", pipe)
    monkeypatch.setenv("SLB_PIPE_GROUP", group)
    sp = P.build_system_2d(128, 128, P.ScaleProfile.from_levels([1, 2]))  # knobs are read at creation
    got = P.denoise_batch(frames, sp, sch)
    for i in range(nfr):
        one = P.denoise(frames[i], s, sch)
        assert np.linalg.norm(got[i] - one) <= 1e-12 * np.linalg.norm(one)


@pytest.mark.parametrize("shape,levels", [((64, 64), [0, 0, 1, 1]), ((128, 128), [1, 1, 2]), ((48, 80), [0, 1])])
def test_gpu_construction_matches_oracle(cuda, shape, levels):
    # cascades (two-scale refinement), upsampling, separable convolutions, the
    # digital shear, embedding and FFTs all run on the GPU (csrc/gpu_taps.cuh,
    # build.cuh); the numpy restatement of the reference's filter algebra is the check
    s = P.build_system_2d(*shape, P.ScaleProfile.from_levels(levels))
    o = O.build_system_2d(shape[0], shape[1], levels)
    np.testing.assert_allclose(s.filter_norms, o.filter_norms, rtol=1e-13)
    for i in range(s.redundancy()):
        assert np.abs(s.filter_freq(i) - o.filters[i]).max() <= 1e-13


def test_duals_match_oracle(cuda):
    # duals() / dual_freq (system2d.cpp:128-148): psi_hat_i / W
    g = golden("t2d_16_01_seed21")
    s = P.build_system_2d(16, 16, P.ScaleProfile.from_levels([0, 1]))
    o = O.build_system_2d(16, 16, [0, 1])
    d = s.duals()
    assert len(d) == s.redundancy() == len(s.filters)
    for i in range(s.redundancy()):
        assert np.abs(d[i] - o.filters[i] / o.frame_weight).max() < 1e-12
    np.testing.assert_allclose(s.frame_weight, g["frame_weight"], rtol=1e-12)


def test_run_to_run_bit_identical(cuda):
    # DESIGN 6: band-order sums, deterministic slot / accumulator order -> repeated
    # calls (batched over streams, lone frames, 3D groups) are bitwise identical
    import torch
    s = P.build_system_2d(512, 512, P.ScaleProfile.from_levels([1, 1, 2, 2]))
    sch = P.ThresholdSchedule.defaults_2d(40.0)
    x = torch.from_numpy(np.stack([P.add_gaussian_noise(P.cartoon(512), 40.0, i) for i in range(8)])).to(cuda)
    a = P.denoise_batch(x, s, sch)
    for _ in range(3):
        assert torch.equal(P.denoise_batch(x, s, sch), a)
    one = P.denoise(x[0], s, sch)
    assert torch.equal(P.denoise(x[0], s, sch), one)
    s3 = P.build_system_3d((64, 64, 64), P.ScaleProfile.from_levels([0, 1]))
    v = torch.from_numpy(np.random.default_rng(2).uniform(-1, 1, (64, 64, 64))).to(cuda)
    sch3 = P.ThresholdSchedule.defaults_3d(0.2, 2)
    d3 = P.denoise(v, s3, sch3)
    assert torch.equal(P.denoise(v, s3, sch3), d3)


def test_stack_free_denoise_same_result(cuda):
    # sl_set_stack_output(0): the fused denoise never writes the stack; same reconstruction
    import torch
    for shape, lv, mk in (((512, 512), [1, 1, 2, 2], P.build_system_2d), ((64, 64, 64), [0, 1], P.build_system_3d),
                          ((128, 128, 128), [0, 1], P.build_system_3d), ((192, 192, 192), [0], P.build_system_3d)):
        prof = P.ScaleProfile.from_levels(lv)
        s = mk(*shape, prof) if len(shape) == 2 else mk(shape, prof)
        sch = (P.ThresholdSchedule.defaults_2d if len(shape) == 2 else P.ThresholdSchedule.defaults_3d)(0.2, len(lv))
        x = torch.from_numpy(np.random.default_rng(6).uniform(-1, 1, (3,) + shape)).to(cuda)
        want = P.denoise_batch(x, s, sch)
        one = P.denoise(x[0], s, sch)
        s.set_stack_output(False)
        assert torch.equal(P.denoise_batch(x, s, sch), want)
        assert torch.equal(P.denoise(x[0], s, sch), one)
        s.set_stack_output(True)
