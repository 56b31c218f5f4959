"""oracle/gen_golden.py -- TEST INFRASTRUCTURE ONLY.

Generates the committed golden fixtures under tests/golden/ from the
UNMODIFIED reference library (oracle/_ref/libshearlet_ref.so, built from
/root/reference by `make -C oracle ref`). Run here, in the container that has
/root/reference; the GPU box only reads the committed .npz files.

    python oracle/gen_golden.py [--big]

Each fixture stores the inputs (or the recipe to regenerate them with the
reference's own generators), and the reference's outputs either in full
(small grids) or as per-band statistics plus a fixed strided sample
(large grids), so the files stay small.
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import ref  # noqa: E402
from oracle import shearlet_np as O  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def sample_idx(n, k=257):
    """Fixed strided sample of k flat indices in [0, n)."""
    return (np.arange(k, dtype=np.int64) * 7919) % n


def kept_fingerprint(bands):
    """Per band (count, sum of kept flat indices, sum of (index mod 1000003)^2):
    a position fingerprint of the thresholded support (same as
    oracle/ref_capi.cpp ref_denoise_3d_stats and tests/conftest.py)."""
    flat = bands.reshape(bands.shape[0], -1)
    out = np.zeros((flat.shape[0], 3), dtype=np.int64)
    for i in range(flat.shape[0]):
        idx = np.flatnonzero(flat[i]).astype(np.int64)
        r = idx % 1000003
        out[i] = (idx.size, idx.sum(), (r * r).sum())
    return out


def band_stats(bands):
    flat = bands.reshape(bands.shape[0], -1)
    return {
        "band_l2": np.sqrt(np.sum(flat * flat, axis=1)),
        "band_sum": np.sum(flat, axis=1),
        "band_sample": flat[:, sample_idx(flat.shape[1])],
    }


def save(name, **kw):
    os.makedirs(OUT, exist_ok=True)
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **kw)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def gen_2d_full(name, n, levels, f, j0=0):
    s = ref.RefSystem2D(n, n, levels, j0=j0)
    bands = s.forward(f)
    rec = s.inverse(bands)
    save(name, f=f, levels=np.array(levels), j0=j0, index=s.index(), filter_norms=s.filter_norms(),
         frame_weight=s.frame_weight(), bands=bands, rec=rec)


def gen_2d_stats(name, n, levels, f, K=None, sigma=None, j0=0):
    s = ref.RefSystem2D(n, n, levels, j0=j0)
    bands = s.forward(f)
    rec = s.inverse(bands)
    W = s.frame_weight()
    kw = dict(levels=np.array(levels), j0=j0, index=s.index(), filter_norms=s.filter_norms(),
              W_min=W.min(), W_max=W.max(), W_sample=W.reshape(-1)[sample_idx(W.size)],
              f_sum=f.sum(), f_l2=np.sqrt((f * f).sum()),
              rec_sample=rec.reshape(-1)[sample_idx(rec.size)],
              rec_relerr=np.linalg.norm(rec - f) / np.linalg.norm(f), **band_stats(bands))
    if K is not None:
        thr = s.hard_threshold(bands, K, sigma)
        kept = np.count_nonzero(thr.reshape(thr.shape[0], -1), axis=1)
        den = s.inverse(thr)
        kw.update(K=np.array(K), sigma=sigma, kept=kept, kept_fp=kept_fingerprint(thr),
                  den_sample=den.reshape(-1)[sample_idx(den.size)], den_sum=den.sum(),
                  den_l2=np.sqrt((den * den).sum()))
    save(name, **kw)
    return s, bands


def gen_3d(name, dims, levels, f, K=None, sigma=None, full=False, threads=0):
    t = time.time()
    s = ref.RefSystem3D(dims, levels, threads=threads)
    W = s.frame_weight()
    kw = dict(dims=np.array(dims), levels=np.array(levels), index=s.index(),
              filter_norms=s.filter_norms(), W_min=W.min(), W_max=W.max(),
              W_sample=W.reshape(-1)[sample_idx(W.size)], f_sum=f.sum())
    print(f"  built {dims} {levels} R={s.R} in {time.time() - t:.1f}s")
    # a few filters, sampled, to pin the on-the-fly synthesis
    fi = [0, 1, s.R // 3, s.R // 2, s.R - 1]
    kw["filter_ids"] = np.array(fi)
    kw["filter_samples"] = np.stack([s.filter(i).reshape(-1)[sample_idx(W.size)] for i in fi])
    if K is not None and not full:
        si = sample_idx(W.size)
        den, kept, l2, smp = s.denoise_stats(f, K, sigma, si, threads=threads)
        fp = np.concatenate([kept[:, None], s.last_kept_fp], axis=1)
        kw.update(K=np.array(K), sigma=sigma, kept=kept, kept_fp=fp, band_l2=l2, band_sample=smp,
                  den_sample=den.reshape(-1)[si], den_sum=den.sum(), den_l2=np.sqrt((den * den).sum()))
    elif full:
        bands = s.forward(f, threads=threads)
        rec = s.inverse(bands, threads=threads)
        kw.update(f=f, bands=bands, rec=rec)
    else:
        bands = s.forward(f, threads=threads)
        rec = s.inverse(bands, threads=threads)
        kw.update(rec_sample=rec.reshape(-1)[sample_idx(rec.size)],
                  rec_relerr=np.linalg.norm(rec - f) / np.linalg.norm(f), **band_stats(bands))
    print(f"  done in {time.time() - t:.1f}s")
    save(name, **kw)


LEGALL_LOWPASS = np.array([-0.125, 0.25, 0.75, 0.25, -0.125])  # symmetric 5-tap, sums to 1


def gen_banks():
    """Custom FanFilter / QmfPair systems (build_system_2d/3d with explicit fan, qmf)."""
    fan2 = ref.maxflat_fan(2)
    q = (LEGALL_LOWPASS, 2)
    s = ref.RefSystem2D(32, 32, [0, 1], fan=fan2, qmf=q)
    f = O.random_grid((32, 32), 9)
    b = s.forward(f)
    save("bank_2d_32_fan2_legall", f=f, levels=np.array([0, 1]), fan=fan2[0], fan_c=np.array(fan2[1:]),
         lowpass=LEGALL_LOWPASS, lowpass_c=2, index=s.index(), filter_norms=s.filter_norms(),
         frame_weight=s.frame_weight(), bands=b, rec=s.inverse(b))
    fan3 = ref.maxflat_fan(3)
    s = ref.RefSystem2D(48, 40, [1, 1], fan=fan3)
    f = O.random_grid((48, 40), 10)
    b = s.forward(f)
    save("bank_2d_48x40_fan3", f=f, levels=np.array([1, 1]), fan=fan3[0], fan_c=np.array(fan3[1:]),
         index=s.index(), filter_norms=s.filter_norms(), frame_weight=s.frame_weight(), bands=b,
         rec=s.inverse(b))
    s3 = ref.RefSystem3D((16, 16, 16), [0, 1], fan=fan2, qmf=q)
    f = np.random.default_rng(12).uniform(-1, 1, (16, 16, 16))
    b = s3.forward(f)
    save("bank_3d_16_fan2_legall", f=f, levels=np.array([0, 1]), fan=fan2[0], fan_c=np.array(fan2[1:]),
         lowpass=LEGALL_LOWPASS, lowpass_c=2, index=s3.index(), filter_norms=s3.filter_norms(),
         W_sample=s3.frame_weight().reshape(-1)[sample_idx(f.size)], rec=s3.inverse(b), **band_stats(b))
    # fan_design::maxflat_fan(order), orders 1..6 (fan_design.cpp:70-108)
    save("maxflat_fans", **{f"order{o}": ref.maxflat_fan(o)[0] for o in range(1, 7)})


def gen_asym():
    """An asymmetric fan (maxflat_fan(2) with its centre moved off the middle):
    the filters are real in space but not centrally symmetric, so psi_hat is
    complex (Hermitian) -- the reference stores full complex grids
    (system2d.hpp:38) and accepts any fan (filters.hpp:64)."""
    t, c0, c1 = ref.maxflat_fan(2)
    fan = (t, c0 + 1, c1)
    for n, lv, name in ((32, [0, 1], "bank_2d_32_asym"), (64, [0, 0, 1], "bank_2d_64_asym")):
        s = ref.RefSystem2D(n, n, lv, fan=fan)
        f = O.random_grid((n, n), 13 + n)
        b = s.forward(f)
        K = [2.0] * len(lv)
        thr = s.hard_threshold(b, K, 0.2)
        save(name, f=f, levels=np.array(lv), fan=t, fan_c=np.array([c0 + 1, c1]), index=s.index(),
             filter_norms=s.filter_norms(), frame_weight=s.frame_weight(), bands=b, rec=s.inverse(b),
             K=np.array(K), sigma=0.2, den=s.inverse(thr), filter1=s.filter(1))


def gen_io():
    """PGM (8/16-bit) and SVOL bytes written by the reference (image_io.cpp:77-159)."""
    import tempfile
    d = tempfile.mkdtemp()
    img = ref.add_noise(ref.cartoon(48), 40.0, 5)[:40, :]  # 40 x 48, values outside [0, 255] too
    vol = np.random.default_rng(4).uniform(-2, 2, (5, 6, 7))
    out = {"img": img, "vol": vol}
    for name, mv in (("pgm8", 255), ("pgm16", 4095)):
        p = os.path.join(d, name + ".pgm")
        ref.save_pgm(img * (mv / 255.0), p, mv)
        out[name] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
        out[name + "_loaded"] = ref.load_pgm(p)[0]
    p = os.path.join(d, "v.svol")
    ref.save_svol(vol, p)
    out["svol"] = np.frombuffer(open(p, "rb").read(), dtype=np.uint8)
    save("io_pgm_svol", **out)


def gen_descriptors():
    """describe() + write_descriptor() texts of the reference (descriptor.cpp:30-67), and the
    RMS of systems rebuilt from them (build_from_descriptor_2d/3d)."""
    systems = {
        "d2_512_1122": ref.RefSystem2D(512, 512, [1, 1, 2, 2]),
        "d2_48x40_full_j1": ref.RefSystem2D(48, 40, [0, 1], j0=1, full=True),
        "d2_32_legall": ref.RefSystem2D(32, 32, [0, 1], qmf=(LEGALL_LOWPASS, 2), fan=ref.maxflat_fan(2)),
        "d3_16_impulse": ref.RefSystem3D((16, 16, 16), [0, 1], impulse_fan=True),
        "d3_16x20x24_legall": ref.RefSystem3D((16, 20, 24), [0, 1], qmf=(LEGALL_LOWPASS, 2)),
    }
    out = {}
    for k, sy in systems.items():
        out[k + "_text"] = np.array(ref.descriptor_text(sy))
        out[k + "_rms"] = sy.filter_norms()
    save("descriptors", **out)


def gen_quality():
    """quality_q / quality_q_opt (apps.cpp:289-362) on the separation fixture's curves."""
    g = np.load(os.path.join(OUT, "it_separate128.npz"))
    truth = (np.abs(ref.curves_plus_dots(128)) > 100.0).astype(np.float64)
    rec = np.abs(g["curves"])
    out = {"rec": rec, "truth": truth, "gauss2": ref.gaussian_kernel(2.0)[0], "gauss07": ref.gaussian_kernel(0.7)[0]}
    for name, sigma in (("s2", 2.0), ("s07", 0.7)):
        q, d = ref.quality_q_opt(rec, truth, sigma)
        out[f"qopt_{name}"], out[f"dopt_{name}"] = q, d
        out[f"q40_{name}"] = ref.quality_q(rec, truth, 40.0, sigma)
    # non-power-of-two grid (generic FFT path): 96 x 80 crop
    out["qopt_crop"], out["dopt_crop"] = ref.quality_q_opt(rec[:96, :80], truth[:96, :80], 1.5)
    save("quality_q", **out)


def gen_acceptance():
    """acceptance.cpp criterion 7 (173-191): 256^2 cartoon, sigma 30, seed 11;
    SL2D_2 vs the separable system ([0,0,0,0], impulse fan), PSNRs from the reference."""
    img = ref.cartoon(256)
    noisy = ref.add_noise(img, 30.0, 11)
    K = [2.5, 2.5, 2.5, 3.8]
    sl2 = ref.RefSystem2D(256, 256, [1, 1, 2, 2])
    swt = ref.RefSystem2D(256, 256, [0, 0, 0, 0], impulse_fan=True)
    save("acceptance_c7", p_noisy=ref.psnr(img, noisy), p_sl2=ref.psnr(img, sl2.denoise(noisy, K, 30.0)),
         p_swt=ref.psnr(img, swt.denoise(noisy, K, 30.0)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true", help="also the 128^3 / 192^3 fixtures")
    ap.add_argument("--only", choices=["cfg2", "cfg5", "asym"], help="regenerate one fixture")
    a = ap.parse_args()
    if not ref.available():
        sys.exit("build the reference first: make -C oracle ref")
    if a.only == "cfg2":
        noisy = ref.add_noise(ref.cartoon(512), 40.0, 7)
        gen_2d_stats("cfg2_denoise512_1122", 512, [1, 1, 2, 2], noisy, K=[2.5, 2.5, 2.5, 3.8], sigma=40.0)
        return
    if a.only == "asym":
        gen_asym()
        return
    if a.only == "cfg5":
        noisy3 = ref.add_noise(ref.cartoon_volume(192), 40.0, 3)
        gen_3d("cfg5_denoise192_112", (192, 192, 192), [1, 1, 2], noisy3, K=[3.0, 3.0, 4.0], sigma=40.0)
        return

    # test_transform.cpp:55-64 (naive-correlation pin): 16^2 [0,1] seed 21
    gen_2d_full("t2d_16_01_seed21", 16, [0, 1], O.random_grid((16, 16), 21))
    # test_transform.cpp:26-40 impulse at 16^2 [0,1]
    imp = np.zeros((16, 16)); imp[0, 0] = 1.0
    gen_2d_full("t2d_16_01_impulse", 16, [0, 1], imp)
    # test_transform.cpp:66-72 round trip 64^2 [0,0,1,1] seed 22
    gen_2d_full("t2d_64_0011_seed22", 64, [0, 0, 1, 1], O.random_grid((64, 64), 22))
    # non-square grid (drop-in generality): 40 x 24 [0,1], seed 5
    s = ref.RefSystem2D(40, 24, [0, 1])
    f = O.random_grid((40, 24), 5)
    b = s.forward(f)
    save("t2d_40x24_01_seed5", f=f, levels=np.array([0, 1]), j0=0, index=s.index(),
         filter_norms=s.filter_norms(), frame_weight=s.frame_weight(), bands=b, rec=s.inverse(b))
    # cfg1: cartoon 256^2 [1,1] round trip
    gen_2d_stats("cfg1_cartoon256_11", 256, [1, 1], ref.cartoon(256))
    # cfg2: cartoon 512 + noise(sigma 40, seed 7), [1,1,2,2], defaults_2d(40)
    noisy = ref.add_noise(ref.cartoon(512), 40.0, 7)
    s2, _ = gen_2d_stats("cfg2_denoise512_1122", 512, [1, 1, 2, 2], noisy, K=[2.5, 2.5, 2.5, 3.8], sigma=40.0)
    # 3D: test_transform.cpp:150-189 16^3 [0,1]; 8^3 [0] seed 80 (naive pin)
    gen_3d("t3d_8_0_seed80", (8, 8, 8), [0], np.random.default_rng(80).uniform(-1, 1, (8, 8, 8)), full=True)
    gen_3d("t3d_16_01_rand", (16, 16, 16), [0, 1], np.random.default_rng(70).uniform(-1, 1, (16, 16, 16)))
    gen_3d("t3d_12x16x20_01", (12, 16, 20), [0, 1], np.random.default_rng(3).uniform(-1, 1, (12, 16, 20)))
    # acceptance crit.1 3D shape 32^3 [0,0,1]
    gen_3d("t3d_32_001", (32, 32, 32), [0, 0, 1], np.random.default_rng(2).uniform(-1, 1, (32, 32, 32)),
           K=[3.0, 3.0, 4.0], sigma=0.3)
    # SURVEY 8f "next": iterative pipelines (apps.cpp:179-280)
    s = ref.RefSystem2D(128, 128, [0, 1, 1])
    mask = ref.random_mask(128, 128, 0.3, 5)
    masked = ref.cartoon(128) * mask
    rec = s.inpaint(masked, mask, 12)
    save("it_inpaint128", masked=masked, mask=mask, levels=np.array([0, 1, 1]), iterations=12, delta_min=0.01,
         out=rec)
    # 3D inpainting (apps.hpp:70-72): 32^3 [0,1], 30 % of the voxels observed
    s3 = ref.RefSystem3D((32, 32, 32), [0, 1])
    mask3 = (np.random.default_rng(6).uniform(size=(32, 32, 32)) < 0.3).astype(np.float64)
    masked3 = ref.cartoon_volume(32) * mask3
    save("it_inpaint3d32", masked=masked3, mask=mask3, levels=np.array([0, 1]), iterations=6, delta_min=0.01,
         out=s3.inpaint(masked3, mask3, 6))
    sd = ref.RefSystem2D(128, 128, [0, 1])
    si = ref.RefSystem2D(128, 128, [0, 0], impulse_fan=True)
    sig = ref.curves_plus_dots(128)
    c, b = sd.separate(si, sig, 10)
    save("it_separate128", signal=sig, dir_levels=np.array([0, 1]), iso_levels=np.array([0, 0]), iterations=10,
         delta_min=0.01, curves=c, blobs=b)
    # SURVEY 8f "next": SHCF coefficient files (transform.cpp:127-269), bytes from the reference serialize()
    s = ref.RefSystem2D(16, 16, [0, 1])
    b = s.forward(O.random_grid((16, 16), 21))
    save("shcf_2d_16_01", levels=np.array([0, 1]), bands=b,
         shcf=np.frombuffer(ref.serialize(s, b), dtype=np.uint8))
    s3 = ref.RefSystem3D((8, 12, 10), [0])
    b3 = s3.forward(np.random.default_rng(11).uniform(-1, 1, (8, 12, 10)))
    save("shcf_3d_8x12x10_0", levels=np.array([0]), bands=b3,
         shcf=np.frombuffer(ref.serialize(s3, b3), dtype=np.uint8))
    gen_banks()
    gen_asym()
    gen_io()
    gen_descriptors()
    gen_quality()
    gen_acceptance()
    if a.big:
        # cfg4: cartoon_volume(128), [1,1]
        gen_3d("cfg4_cartoonvol128_11", (128, 128, 128), [1, 1], ref.cartoon_volume(128))
        # cfg5: cartoon_volume(192) + noise(40, seed 3), SL3D_2 [1,1,2], defaults_3d(40)
        noisy3 = ref.add_noise(ref.cartoon_volume(192), 40.0, 3)
        gen_3d("cfg5_denoise192_112", (192, 192, 192), [1, 1, 2], noisy3, K=[3.0, 3.0, 4.0], sigma=40.0)


if __name__ == "__main__":
    main()
