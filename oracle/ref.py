"""oracle/ref.py -- TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/_ref/libshearlet_ref.so: the UNMODIFIED reference
library (/root/reference/proj/core/src, compiled by oracle/Makefile with our
FFTW-API shim). Used by tests/, oracle/gen_golden.py and bench.py's
cpu_baseline / --impl reference legs only -- never by the product path.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libshearlet_ref.so")

_lib = None


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} not built (make -C oracle ref)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        dp = C.POINTER(C.c_double)
        ip = C.POINTER(C.c_int)
        L.ref_last_error.restype = C.c_char_p
        L.ref_build_2d.argtypes = [C.c_int, C.c_int, ip, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(P)]
        L.ref_build_3d.argtypes = [C.c_int, C.c_int, C.c_int, ip, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(P)]
        for n in ("ref_free_2d", "ref_free_3d"):
            getattr(L, n).argtypes = [P]
        for n in ("ref_redundancy_2d", "ref_redundancy_3d"):
            getattr(L, n).argtypes = [P]
            getattr(L, n).restype = C.c_int
        for n in ("ref_index_2d", "ref_index_3d"):
            getattr(L, n).argtypes = [P, ip]
        for n in ("ref_filter_norms_2d", "ref_filter_norms_3d", "ref_frame_weight_2d", "ref_frame_weight_3d"):
            getattr(L, n).argtypes = [P, dp]
        L.ref_filter_2d.argtypes = [P, C.c_int, dp]
        L.ref_filter_3d.argtypes = [P, C.c_int, dp]
        for d in ("2d", "3d"):
            getattr(L, f"ref_forward_{d}").argtypes = [P, dp, dp, C.c_int]
            getattr(L, f"ref_inverse_{d}").argtypes = [P, dp, C.c_int, dp, C.c_int]
            getattr(L, f"ref_hard_threshold_{d}").argtypes = [P, dp, C.c_int, dp, C.c_int, C.c_double, C.c_int, dp]
            getattr(L, f"ref_denoise_{d}").argtypes = [P, dp, dp, C.c_int, C.c_double, C.c_int, dp, C.c_int]
        L.ref_denoise_3d_stats.argtypes = [P, dp, dp, C.c_int, C.c_double, C.c_int, dp, C.POINTER(C.c_longlong), dp, dp, C.POINTER(C.c_longlong), C.c_int, C.c_int, C.POINTER(C.c_longlong)]
        L.ref_inpaint_2d.argtypes = [P, dp, dp, C.c_int, C.c_double, C.c_double, C.c_int, dp, C.c_int]
        L.ref_inpaint_3d.argtypes = [P, dp, dp, C.c_int, C.c_double, C.c_double, C.c_int, dp, C.c_int]
        L.ref_separate_2d.argtypes = [P, P, dp, C.c_int, C.c_double, C.c_double, C.c_int, dp, dp, C.c_int]
        L.ref_random_mask.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint64, dp]
        L.ref_curves_plus_dots.argtypes = [C.c_int, dp]
        L.ref_cartoon.argtypes = [C.c_int, dp]
        L.ref_cartoon_volume.argtypes = [C.c_int, dp]
        L.ref_add_noise_2d.argtypes = [C.c_int, C.c_int, dp, C.c_double, C.c_uint64, dp]
        L.ref_add_noise_3d.argtypes = [C.c_int, C.c_int, C.c_int, dp, C.c_double, C.c_uint64, dp]
        L.ref_psnr_2d.argtypes = [C.c_int, C.c_int, dp, dp]
        L.ref_psnr_2d.restype = C.c_double
        L.ref_fft_forward.argtypes = [C.c_int, ip, dp]
        bank = [dp, C.c_int, C.c_int, dp, C.c_int, C.c_int, dp, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_build_2d_bank.argtypes = [C.c_int] * 2 + [ip] + [C.c_int] * 3 + bank + [C.c_int, C.POINTER(P)]
        L.ref_build_3d_bank.argtypes = [C.c_int] * 3 + [ip] + [C.c_int] * 3 + bank + [C.c_int, C.POINTER(P)]
        L.ref_maxflat_fan.argtypes = [C.c_int, dp, C.c_longlong, ip]
        L.ref_write_descriptor_2d.argtypes = [P, C.c_char_p]
        L.ref_write_descriptor_3d.argtypes = [P, C.c_char_p]
        L.ref_build_from_descriptor.argtypes = [C.c_char_p, ip, C.POINTER(P)]
        L.ref_gaussian_kernel.argtypes = [C.c_double, dp, C.c_longlong, ip]
        L.ref_quality_q_opt.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, dp, ip]
        L.ref_quality_q.argtypes = [C.c_int, C.c_int, dp, dp, C.c_double, C.c_double, dp]
        L.ref_save_pgm.argtypes = [dp, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.ref_load_pgm.argtypes = [C.c_char_p, dp, C.c_longlong, ip]
        L.ref_save_svol.argtypes = [dp, C.c_int, C.c_int, C.c_int, C.c_char_p]
        for d in ("2d", "3d"):
            getattr(L, f"ref_serialize_{d}").argtypes = [P, dp, C.c_int, C.c_char_p, C.c_longlong]
            getattr(L, f"ref_serialize_{d}").restype = C.c_longlong
        L.ref_deserialize.argtypes = [C.c_char_p, C.c_longlong, ip, ip, dp, C.c_longlong]
        L.ref_deserialize.restype = C.c_int
        _lib = L
    return _lib


def _dp(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _ip(a: np.ndarray):
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _bank_args(fan, qmf):
    """fan = (taps2d, c0, c1) or None (default fan); qmf = (lowpass, c) or (lowpass, c, highpass, hc) or None."""
    keep = []
    if qmf is None:
        q = [None, 0, 0, None, 0, 0]
    else:
        lp = np.ascontiguousarray(qmf[0], dtype=np.float64)
        keep.append(lp)
        q = [_dp(lp), len(lp), int(qmf[1]), None, 0, 0]
        if len(qmf) > 2:
            hp = np.ascontiguousarray(qmf[2], dtype=np.float64)
            keep.append(hp)
            q[3:] = [_dp(hp), len(hp), int(qmf[3])]
    if fan is None:
        f = [None, 0, 0, 0, 0]
    else:
        t = np.ascontiguousarray(fan[0], dtype=np.float64)
        keep.append(t)
        f = [_dp(t), t.shape[0], t.shape[1], int(fan[1]), int(fan[2])]
    return q + f, keep


def maxflat_fan(order):
    """fan_design::maxflat_fan(order) from the reference -> (taps, c0, c1)."""
    dims = np.zeros(4, dtype=np.int32)
    _check(lib().ref_maxflat_fan(order, None, 0, _ip(dims)))
    t = np.zeros((dims[0], dims[1]))
    _check(lib().ref_maxflat_fan(order, _dp(t), t.size, _ip(dims)))
    return t, int(dims[2]), int(dims[3])


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"reference error {code}: {msg}")
        self.code = code


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


class RefSystem2D:
    """Reference ShearletSystem2D (core/include/shearlet/system2d.hpp:29-51)."""

    def __init__(self, rows, cols, levels, j0=0, full=False, impulse_fan=False, threads=0, fan=None, qmf=None):
        L = lib()
        lv = np.asarray(levels, dtype=np.int32)
        h = C.c_void_p()
        if fan is None and qmf is None:
            _check(L.ref_build_2d(rows, cols, _ip(lv), len(lv), j0, int(full), int(impulse_fan), threads, C.byref(h)))
        else:
            args, self._keep = _bank_args(fan, qmf)
            _check(L.ref_build_2d_bank(rows, cols, _ip(lv), len(lv), j0, int(full), *args, threads, C.byref(h)))
        self.h = h
        self.rows, self.cols = rows, cols
        self.shape = (rows, cols)
        self.n_scales = len(lv)
        self.R = L.ref_redundancy_2d(h)

    def __del__(self):
        try:
            lib().ref_free_2d(self.h)
        except Exception:
            pass

    def index(self):
        rec = np.zeros((self.R, 3), dtype=np.int32)
        lib().ref_index_2d(self.h, _ip(rec))
        return rec

    def filter_norms(self):
        out = np.zeros(self.R)
        lib().ref_filter_norms_2d(self.h, _dp(out))
        return out

    def frame_weight(self):
        out = np.zeros(self.shape)
        lib().ref_frame_weight_2d(self.h, _dp(out))
        return out

    def filter(self, i):
        out = np.zeros(self.shape + (2,))
        lib().ref_filter_2d(self.h, i, _dp(out))
        return out[..., 0] + 1j * out[..., 1]

    def forward(self, f, threads=0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        out = np.zeros((self.R,) + self.shape)
        _check(lib().ref_forward_2d(self.h, _dp(f), _dp(out), threads))
        return out

    def inverse(self, bands, threads=0):
        bands = np.ascontiguousarray(bands, dtype=np.float64)
        out = np.zeros(self.shape)
        _check(lib().ref_inverse_2d(self.h, _dp(bands), bands.shape[0], _dp(out), threads))
        return out

    def hard_threshold(self, bands, K, sigma, scaled=True):
        bands = np.ascontiguousarray(bands, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        out = np.zeros_like(bands)
        _check(lib().ref_hard_threshold_2d(self.h, _dp(bands), bands.shape[0], _dp(K), len(K), sigma, int(scaled), _dp(out)))
        return out

    def denoise(self, f, K, sigma, scaled=True, threads=0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        out = np.zeros(self.shape)
        _check(lib().ref_denoise_2d(self.h, _dp(f), _dp(K), len(K), sigma, int(scaled), _dp(out), threads))
        return out

    def inpaint(self, masked, mask, iterations, delta_init=-1.0, delta_min=0.01, scaled=True, threads=0):
        masked = np.ascontiguousarray(masked, dtype=np.float64)
        mask = np.ascontiguousarray(mask, dtype=np.float64)
        out = np.zeros(self.shape)
        _check(lib().ref_inpaint_2d(self.h, _dp(masked), _dp(mask), iterations, delta_init, delta_min, int(scaled),
                                    _dp(out), threads))
        return out

    def separate(self, iso, signal, iterations, delta_init=-1.0, delta_min=0.01, scaled=True, threads=0):
        signal = np.ascontiguousarray(signal, dtype=np.float64)
        c, b = np.zeros(self.shape), np.zeros(self.shape)
        _check(lib().ref_separate_2d(self.h, iso.h, _dp(signal), iterations, delta_init, delta_min, int(scaled),
                                     _dp(c), _dp(b), threads))
        return c, b


class RefSystem3D:
    """Reference ShearletSystem3D (core/include/shearlet/system3d.hpp:32-61)."""

    def __init__(self, dims, levels, j0=0, full=False, impulse_fan=False, threads=0, fan=None, qmf=None):
        L = lib()
        lv = np.asarray(levels, dtype=np.int32)
        h = C.c_void_p()
        n0, n1, n2 = dims
        if fan is None and qmf is None:
            _check(L.ref_build_3d(n0, n1, n2, _ip(lv), len(lv), j0, int(full), int(impulse_fan), threads,
                                  C.byref(h)))
        else:
            args, self._keep = _bank_args(fan, qmf)
            _check(L.ref_build_3d_bank(n0, n1, n2, _ip(lv), len(lv), j0, int(full), *args, threads, C.byref(h)))
        self.h = h
        self.shape = tuple(dims)
        self.n_scales = len(lv)
        self.R = L.ref_redundancy_3d(h)

    def __del__(self):
        try:
            lib().ref_free_3d(self.h)
        except Exception:
            pass

    def index(self):
        rec = np.zeros((self.R, 4), dtype=np.int32)
        lib().ref_index_3d(self.h, _ip(rec))
        return rec

    def filter_norms(self):
        out = np.zeros(self.R)
        lib().ref_filter_norms_3d(self.h, _dp(out))
        return out

    def frame_weight(self):
        out = np.zeros(self.shape)
        lib().ref_frame_weight_3d(self.h, _dp(out))
        return out

    def filter(self, i):
        out = np.zeros(self.shape + (2,))
        _check(lib().ref_filter_3d(self.h, i, _dp(out)))
        return out[..., 0] + 1j * out[..., 1]

    def forward(self, f, threads=0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        out = np.zeros((self.R,) + self.shape)
        _check(lib().ref_forward_3d(self.h, _dp(f), _dp(out), threads))
        return out

    def inverse(self, bands, threads=0):
        bands = np.ascontiguousarray(bands, dtype=np.float64)
        out = np.zeros(self.shape)
        _check(lib().ref_inverse_3d(self.h, _dp(bands), bands.shape[0], _dp(out), threads))
        return out

    def hard_threshold(self, bands, K, sigma, scaled=True):
        bands = np.ascontiguousarray(bands, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        out = np.zeros_like(bands)
        _check(lib().ref_hard_threshold_3d(self.h, _dp(bands), bands.shape[0], _dp(K), len(K), sigma, int(scaled), _dp(out)))
        return out

    def denoise(self, f, K, sigma, scaled=True, threads=0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        out = np.zeros(self.shape)
        _check(lib().ref_denoise_3d(self.h, _dp(f), _dp(K), len(K), sigma, int(scaled), _dp(out), threads))
        return out

    def inpaint(self, masked, mask, iterations, delta_init=-1.0, delta_min=0.01, scaled=True, threads=0):
        masked = np.ascontiguousarray(masked, dtype=np.float64)
        mask = np.ascontiguousarray(mask, dtype=np.float64)
        out = np.zeros(self.shape)
        _check(lib().ref_inpaint_3d(self.h, _dp(masked), _dp(mask), iterations, delta_init, delta_min, int(scaled),
                                    _dp(out), threads))
        return out

    def denoise_stats(self, f, K, sigma, sample_idx, scaled=True, threads=0):
        f = np.ascontiguousarray(f, dtype=np.float64)
        K = np.ascontiguousarray(K, dtype=np.float64)
        si = np.ascontiguousarray(sample_idx, dtype=np.int64)
        out = np.zeros(self.shape)
        kept = np.zeros(self.R, dtype=np.int64)
        l2 = np.zeros(self.R)
        smp = np.zeros((self.R, len(si)))
        fp = np.zeros((self.R, 2), dtype=np.int64)
        LL = C.POINTER(C.c_longlong)
        _check(lib().ref_denoise_3d_stats(self.h, _dp(f), _dp(K), len(K), sigma, int(scaled), _dp(out),
                                          kept.ctypes.data_as(LL), _dp(l2), _dp(smp), si.ctypes.data_as(LL),
                                          len(si), threads, fp.ctypes.data_as(LL)))
        self.last_kept_fp = fp
        return out, kept, l2, smp


def _serialize(fn, h, bands):
    bands = np.ascontiguousarray(bands, dtype=np.float64)
    n = fn(h, _dp(bands), bands.shape[0], None, 0)
    if n < 0:
        _check(int(-n))
    buf = C.create_string_buffer(int(n))
    fn(h, _dp(bands), bands.shape[0], buf, n)
    return buf.raw


def serialize(system, bands) -> bytes:
    """Reference serialize() (transform.cpp:185-213) of a stack on `system`."""
    fn = lib().ref_serialize_2d if isinstance(system, RefSystem2D) else lib().ref_serialize_3d
    return _serialize(fn, system.h, bands)


def deserialize(data: bytes):
    """Reference deserialize_2d/3d (transform.cpp:216-269) -> bands [count][dims]."""
    nd, dims = C.c_int(), np.zeros(3, dtype=np.int32)
    nb = lib().ref_deserialize(data, len(data), C.byref(nd), _ip(dims), None, 0)
    if nb < 0:
        _check(-nb)
    shape = tuple(int(d) for d in dims[: nd.value])
    out = np.zeros((nb,) + shape)
    lib().ref_deserialize(data, len(data), C.byref(nd), _ip(dims), _dp(out), out.size)
    return out


def descriptor_text(system) -> str:
    """write_descriptor(describe(system)) (descriptor.cpp:30-67) -> text."""
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "sys.txt")
        fn = lib().ref_write_descriptor_2d if isinstance(system, RefSystem2D) else lib().ref_write_descriptor_3d
        _check(fn(system.h, p.encode()))
        return open(p).read()


def gaussian_kernel(sigma):
    info = np.zeros(2, dtype=np.int32)
    _check(lib().ref_gaussian_kernel(sigma, None, 0, _ip(info)))
    t = np.zeros((info[0], info[0]))
    _check(lib().ref_gaussian_kernel(sigma, _dp(t), t.size, _ip(info)))
    return t, int(info[1])


def quality_q_opt(rec, truth, sigma):
    rec = np.ascontiguousarray(rec, dtype=np.float64)
    truth = np.ascontiguousarray(truth, dtype=np.float64)
    q, d = C.c_double(), C.c_int()
    _check(lib().ref_quality_q_opt(rec.shape[0], rec.shape[1], _dp(rec), _dp(truth), sigma, C.byref(q), C.byref(d)))
    return q.value, d.value


def quality_q(rec, truth, delta, sigma):
    rec = np.ascontiguousarray(rec, dtype=np.float64)
    truth = np.ascontiguousarray(truth, dtype=np.float64)
    q = C.c_double()
    _check(lib().ref_quality_q(rec.shape[0], rec.shape[1], _dp(rec), _dp(truth), delta, sigma, C.byref(q)))
    return q.value


def save_pgm(px, path, maxval=255):
    px = np.ascontiguousarray(px, dtype=np.float64)
    _check(lib().ref_save_pgm(_dp(px), px.shape[0], px.shape[1], path.encode(), maxval))


def load_pgm(path):
    info = np.zeros(3, dtype=np.int32)
    _check(lib().ref_load_pgm(path.encode(), None, 0, _ip(info)))
    out = np.zeros((info[0], info[1]))
    _check(lib().ref_load_pgm(path.encode(), _dp(out), out.size, _ip(info)))
    return out, int(info[2])


def save_svol(v, path):
    v = np.ascontiguousarray(v, dtype=np.float64)
    _check(lib().ref_save_svol(_dp(v), *v.shape, path.encode()))


def random_mask(rows, cols, keep, seed):
    out = np.zeros((rows, cols))
    lib().ref_random_mask(rows, cols, keep, seed, _dp(out))
    return out


def curves_plus_dots(n):
    out = np.zeros((n, n))
    lib().ref_curves_plus_dots(n, _dp(out))
    return out


def cartoon(n):
    out = np.zeros((n, n))
    lib().ref_cartoon(n, _dp(out))
    return out


def cartoon_volume(n):
    out = np.zeros((n, n, n))
    lib().ref_cartoon_volume(n, _dp(out))
    return out


def add_noise(x, sigma, seed):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    if x.ndim == 2:
        lib().ref_add_noise_2d(x.shape[0], x.shape[1], _dp(x), sigma, seed, _dp(out))
    else:
        lib().ref_add_noise_3d(*x.shape, _dp(x), sigma, seed, _dp(out))
    return out


def psnr(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return lib().ref_psnr_2d(a.shape[0], a.shape[1], _dp(a), _dp(b))


def fft_forward(x: np.ndarray) -> np.ndarray:
    """Unnormalized forward DFT through the reference wrapper + our shim."""
    x = np.ascontiguousarray(x, dtype=np.complex128)
    buf = np.stack([x.real, x.imag], axis=-1).copy()
    dims = np.asarray(x.shape, dtype=np.int32)
    lib().ref_fft_forward(x.ndim, _ip(dims), _dp(buf))
    return buf[..., 0] + 1j * buf[..., 1]
