"""oracle/shearlet_np.py -- TEST INFRASTRUCTURE ONLY (CPU checker).

A plain numpy restatement of the reference's algorithm for the hot path:
system construction (tap algebra, fan design, digital shear, periodic
embedding), the undecimated forward/inverse transform and the RMS-scaled hard
threshold. Every function cites the reference file:line it restates
(paths relative to /root/reference/proj/core/). numpy.fft (pocketfft) stands
in for FFTW (FFTW is absent from the image; the reference only relies on the
unnormalized DFT definition, src/fft.cpp:45-50).

This module is pinned two ways (tests/test_oracle.py):
  * against the reference itself, compiled from its own sources into
    oracle/_ref/libshearlet_ref.so (when present), and
  * against the committed golden fixtures in tests/golden/, generated from
    that same library by oracle/gen_golden.py.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
it, and only as the checker. The product path never imports it.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------- taps
# A 1D tap set is (v: np.ndarray, center: int); taps[center] sits at n = 0
# (include/shearlet/taps.hpp:13-24). A 2D tap set is (v: 2D array, c0, c1).


@dataclass
class T1:
    v: np.ndarray
    c: int


@dataclass
class T2:
    v: np.ndarray
    c0: int
    c1: int


def conv(a: T1, b: T1) -> T1:  # src/taps.cpp:7-15
    return T1(np.convolve(a.v, b.v), a.c + b.c)


def upsample(a: T1, f: int) -> T1:  # src/taps.cpp:17-24
    if f == 1:
        return T1(a.v.copy(), a.c)
    out = np.zeros((len(a.v) - 1) * f + 1)
    out[::f] = a.v
    return T1(out, a.c * f)


def reversed_taps(a: T1) -> T1:  # src/taps.cpp:26-31
    return T1(a.v[::-1].copy(), len(a.v) - 1 - a.c)


def outer(a: T1, b: T1) -> T2:  # src/taps.cpp:39-48
    return T2(np.outer(a.v, b.v), a.c, b.c)


def conv_axis(g: T2, t: T1, axis: int) -> T2:  # src/taps.cpp:50-76
    n0, n1 = g.v.shape
    L = len(t.v)
    if axis == 0:
        out = np.zeros((n0 + L - 1, n1))
        for k in range(L):
            if t.v[k] != 0.0:
                out[k:k + n0, :] += g.v * t.v[k]
        return T2(out, g.c0 + t.c, g.c1)
    out = np.zeros((n0, n1 + L - 1))
    for k in range(L):
        if t.v[k] != 0.0:
            out[:, k:k + n1] += g.v * t.v[k]
    return T2(out, g.c0, g.c1 + t.c)


def upsample2(g: T2, f0: int, f1: int) -> T2:  # src/taps.cpp:78-88
    if f0 == 1 and f1 == 1:
        return T2(g.v.copy(), g.c0, g.c1)
    n0, n1 = g.v.shape
    out = np.zeros(((n0 - 1) * f0 + 1, (n1 - 1) * f1 + 1))
    out[::f0, ::f1] = g.v
    return T2(out, g.c0 * f0, g.c1 * f1)


def transposed(g: T2) -> T2:  # src/taps.cpp:90-99
    return T2(g.v.T.copy(), g.c1, g.c0)


def embed_periodic_2d(t: T2, n0: int, n1: int) -> np.ndarray:  # src/taps.cpp:101-111
    out = np.zeros((n0, n1))
    r0 = (np.arange(t.v.shape[0]) - t.c0) % n0
    r1 = (np.arange(t.v.shape[1]) - t.c1) % n1
    np.add.at(out, (r0[:, None], r1[None, :]), t.v)
    return out


def embed_periodic_1d(t: T1, n: int) -> np.ndarray:  # src/taps.cpp:113-118
    out = np.zeros(n)
    np.add.at(out, (np.arange(len(t.v)) - t.c) % n, t.v)
    return out


# ----------------------------------------------------------------- filters
def default_lowpass() -> T1:  # src/filters.cpp:12-20
    r2 = math.sqrt(2.0)
    a = (7.0 - 4.0 * r2) / 128.0
    b = (8.0 * r2 - 13.0) / 64.0
    c = (8.0 - 8.0 * r2) / 64.0
    d = (29.0 - 8.0 * r2) / 64.0
    e = (9.0 + 20.0 * r2) / 64.0
    return T1(np.array([a, b, c, d, e, d, c, b, a]), 4)


def mirror_highpass(h: T1) -> T1:  # src/filters.cpp:22-30
    n = np.arange(len(h.v)) - h.c
    return T1(np.where(n & 1, -h.v, h.v), h.c)


@dataclass
class Qmf:  # include/shearlet/filters.hpp:14-22
    lowpass: T1
    highpass: T1


def qmf_default() -> Qmf:  # src/filters.cpp:32-38
    h = default_lowpass()
    return Qmf(h, mirror_highpass(h))


def cascade(q: Qmf, level: int):  # src/filters.cpp:40-63 -> (h_j, g_j)
    if level < 0:
        raise ValueError("cascade: negative level")
    if level == 0:
        imp = T1(np.array([1.0]), 0)
        return imp, imp
    h = T1(q.lowpass.v.copy(), q.lowpass.c)
    for j in range(1, level):
        h = conv(h, upsample(q.lowpass, 1 << j))
    g = upsample(q.highpass, 1 << (level - 1))
    if level > 1:
        hp = T1(q.lowpass.v.copy(), q.lowpass.c)
        for j in range(1, level - 1):
            hp = conv(hp, upsample(q.lowpass, 1 << j))
        g = conv(g, hp)
    return h, g


def shear_interpolation_taps(q: Qmf, level: int) -> T1:  # src/filters.cpp:80-83
    h, _ = cascade(q, level)
    return T1(h.v * (math.sqrt(2.0) ** level), h.c)


# fan design: src/fan_design.cpp
def _combine(a: T2, sa: float, b: T2, sb: float) -> T2:  # fan_design.cpp:10-31
    lo0 = min(-a.c0, -b.c0)
    hi0 = max(a.v.shape[0] - 1 - a.c0, b.v.shape[0] - 1 - b.c0)
    lo1 = min(-a.c1, -b.c1)
    hi1 = max(a.v.shape[1] - 1 - a.c1, b.v.shape[1] - 1 - b.c1)
    out = np.zeros((hi0 - lo0 + 1, hi1 - lo1 + 1))
    o0, o1 = -a.c0 - lo0, -a.c1 - lo1
    out[o0:o0 + a.v.shape[0], o1:o1 + a.v.shape[1]] += sa * a.v
    o0, o1 = -b.c0 - lo0, -b.c1 - lo1
    out[o0:o0 + b.v.shape[0], o1:o1 + b.v.shape[1]] += sb * b.v
    return T2(out, -lo0, -lo1)


def _conv2(a: T2, b: T2) -> T2:  # fan_design.cpp:33-46
    n0 = a.v.shape[0] + b.v.shape[0] - 1
    n1 = a.v.shape[1] + b.v.shape[1] - 1
    out = np.zeros((n0, n1))
    for i in range(a.v.shape[0]):
        for j in range(a.v.shape[1]):
            x = a.v[i, j]
            if x != 0.0:
                out[i:i + b.v.shape[0], j:j + b.v.shape[1]] += x * b.v
    return T2(out, a.c0 + b.c0, a.c1 + b.c1)


def _lagrange_halfsample_weights(order: int):  # fan_design.cpp:48-65
    nn = 2 * order
    w = []
    for i in range(nn):
        xi = float(i - order + 1)
        prod = 1.0
        for j in range(nn):
            if j == i:
                continue
            xj = float(j - order + 1)
            prod *= (0.5 - xj) / (xi - xj)
        w.append(prod)
    return w


def maxflat_fan(order: int = 4) -> T2:  # fan_design.cpp:70-108
    kappa = T2(np.zeros((3, 3)), 1, 1)
    kappa.v[0, 1] = kappa.v[2, 1] = kappa.v[1, 0] = kappa.v[1, 2] = 0.25
    w = _lagrange_halfsample_weights(order)
    diamond = T2(np.array([[0.5]]), 0, 0)
    t_prev = T2(np.array([[1.0]]), 0, 0)
    t_cur = kappa
    for m in range(1, 2 * order):
        if m & 1:
            hm = w[order - 1 + (m + 1) // 2] / 2.0
            diamond = _combine(diamond, 1.0, t_cur, 2.0 * hm)
        t_next = _combine(_conv2(kappa, t_cur), 2.0, t_prev, -1.0)
        t_prev, t_cur = t_cur, t_next
    n0 = np.arange(diamond.v.shape[0]) - diamond.c0
    v = diamond.v.copy()
    odd = (n0 & 1).astype(bool)
    v[odd, :] = np.where(v[odd, :] != 0.0, -v[odd, :], v[odd, :])
    return T2(v, diamond.c0, diamond.c1)


def impulse_fan() -> T2:  # src/filters.cpp:85-87
    return T2(np.array([[1.0]]), 0, 0)


# ----------------------------------------------------------------- digital shear
def digital_shear_taps(t: T2, k: int, d: int, interp: T1) -> T2:  # src/shear.cpp:222-281
    kmax = 1 << d
    if abs(k) > kmax:
        raise ValueError("digital_shear_taps: |k| exceeds 2^d")

    def shear_support(inp: T2, kk: int) -> T2:  # shear.cpp:229-251
        if kk == 0:
            return inp
        n0, n1 = inp.v.shape
        lo1, hi1 = -inp.c1, n1 - 1 - inp.c1
        lo0in, hi0in = -inp.c0, n0 - 1 - inp.c0
        lo0 = min(lo0in - kk * lo1, lo0in - kk * hi1)
        hi0 = max(hi0in - kk * lo1, hi0in - kk * hi1)
        out = np.zeros((hi0 - lo0 + 1, n1))
        c0 = -lo0
        a0 = np.arange(n0) - inp.c0
        for j in range(n1):
            b1 = j - inp.c1
            out[a0 - kk * b1 + c0, j] = inp.v[:, j]
        return T2(out, c0, inp.c1)

    if d == 0:
        return shear_support(t, k)
    f = 1 << d
    up = upsample2(t, f, 1)
    up = conv_axis(up, interp, 0)
    up = shear_support(up, k)
    up = conv_axis(up, reversed_taps(interp), 0)
    lo = -up.c0
    hi = up.v.shape[0] - 1 - up.c0
    qlo = -((-lo) // f)  # ceil_div
    qhi = hi // f        # floor_div
    rows = np.arange(qlo, qhi + 1) * f + up.c0
    return T2(up.v[rows, :].copy(), -qlo, up.c1)


# ----------------------------------------------------------------- profiles
@dataclass
class Profile:  # include/shearlet/filters.hpp:79-92
    levels: list
    j0: int = 0

    @property
    def n_scales(self):
        return len(self.levels)

    @property
    def top_level(self):
        return self.j0 + len(self.levels)


# ----------------------------------------------------------------- 2D system
def enumerate_filters_2d(p: Profile, full=False):  # src/system2d.cpp:59-73
    idx = [(0, -1, 0)]  # (kind, scale, shear); kind 0 lowpass, 1 horiz, 2 vert
    for s, d in enumerate(p.levels):
        j = p.j0 + s
        km = 1 << d
        for k in range(-km, km + 1):
            idx.append((1, j, k))
        for k in range(-km, km + 1):
            if not full and abs(k) == km:
                continue
            idx.append((2, j, k))
    return idx


def build_shearlet_taps(j, k, d, J, fan: T2, q: Qmf) -> T2:  # src/system2d.cpp:21-37
    lg = J - j
    lh = J - (j - d)
    p = upsample2(fan, 1 << (J - j - 1), 1 << lh)
    qq = conv_axis(p, cascade(q, lg)[1], 0)
    qq = conv_axis(qq, cascade(q, lh)[0], 1)
    return digital_shear_taps(qq, k, d, shear_interpolation_taps(q, d))


@dataclass
class System2D:  # include/shearlet/system2d.hpp:29-51
    rows: int
    cols: int
    profile: Profile
    index: list
    filters: np.ndarray            # [R, rows, cols] complex128
    frame_weight: np.ndarray       # [rows, cols]
    filter_norms: np.ndarray       # [R]

    @property
    def R(self):
        return len(self.index)


def build_system_2d(rows, cols, levels, j0=0, full=False, fan=None, q=None) -> System2D:
    # src/system2d.cpp:75-116
    p = Profile(list(levels), j0)
    fan = maxflat_fan(4) if fan is None else fan
    q = qmf_default() if q is None else q
    idx = enumerate_filters_2d(p, full)
    J = p.top_level
    filt = np.zeros((len(idx), rows, cols), dtype=np.complex128)
    for i, (kind, j, k) in enumerate(idx):
        if kind == 0:
            hJ = cascade(q, J)[0]
            t = outer(hJ, hJ)
        else:
            d = p.levels[j - p.j0]
            t = build_shearlet_taps(j, k, d, J, fan, q)
            if kind == 2:
                t = transposed(t)
        filt[i] = np.fft.fft2(embed_periodic_2d(t, rows, cols))
    W = np.sum(np.abs(filt) ** 2, axis=0)                       # system2d.cpp:118-126
    norms = np.sqrt(np.sum(np.abs(filt) ** 2, axis=(1, 2)) / (rows * cols))  # :108-114
    return System2D(rows, cols, p, idx, filt, W, norms)


def forward_2d(f, s: System2D):  # src/transform.cpp:13-37
    F = np.fft.fft2(f)
    return np.real(np.fft.ifft2(np.conj(s.filters) * F[None], axes=(1, 2)))


def inverse_2d(bands, s: System2D):  # src/transform.cpp:63-92 (+ duals, system2d.cpp:128-148)
    B = np.fft.fft2(bands, axes=(1, 2))
    acc = np.sum(B * (s.filters / s.frame_weight[None]), axis=0)
    return np.real(np.fft.ifft2(acc))


# ----------------------------------------------------------------- 3D system
def redundancy_3d(levels, full=False):  # src/system3d.cpp:27-35
    r = 1
    for d in levels:
        qd = 2 * (1 << d) + 1
        r += 3 * qd * qd if full else 3 * qd * qd - 6 * qd + 4
    return r


def enumerate_filters_3d(p: Profile, full=False):  # src/system3d.cpp:58-80
    idx = [(0, -1, 0, 0)]  # (kind 0/3/4/5, scale, k1, k2)
    for s, d in enumerate(p.levels):
        j = p.j0 + s
        K = 1 << d
        for kind in (3, 4, 5):
            for k1 in range(-K, K + 1):
                for k2 in range(-K, K + 1):
                    if not full:
                        if kind == 4 and abs(k1) == K:
                            continue
                        if kind == 5 and (abs(k1) == K or abs(k2) == K):
                            continue
                    idx.append((kind, j, k1, k2))
    return idx


_PYR_AXES = {3: (0, 1, 2), 4: (1, 0, 2), 5: (2, 0, 1)}  # src/system3d.cpp:43-54


def build_phi_component(j, k, d, J, fan: T2, q: Qmf) -> T2:  # src/system3d.cpp:13-25
    lh = J - (j - d)
    p = upsample2(fan, 1 << (J - j - 1), 1 << lh)
    qq = conv_axis(p, cascade(q, lh)[0], 1)
    return digital_shear_taps(qq, k, d, shear_interpolation_taps(q, d))


@dataclass
class System3D:  # include/shearlet/system3d.hpp:32-61
    dims: tuple
    profile: Profile
    index: list
    lowpass_taps: T1
    scales: list                   # per scale: (d, highpass T1, [phi T2 for k=-K..K])
    frame_weight: np.ndarray = None
    filter_norms: np.ndarray = None

    @property
    def R(self):
        return len(self.index)

    def filter_freq(self, i):  # src/system3d.cpp:144-186
        kind, j, k1, k2 = self.index[i]
        n = self.dims
        if kind == 0:
            h = [np.fft.fft(embed_periodic_1d(self.lowpass_taps, n[a])) for a in range(3)]
            return h[0][:, None, None] * h[1][None, :, None] * h[2][None, None, :]
        d, g_taps, phis = self.scales[j - self.profile.j0]
        K = 1 << d
        pa, s1a, s2a = _PYR_AXES[kind]
        g = np.fft.fft(embed_periodic_1d(g_taps, n[pa]))
        p1 = np.fft.fft2(embed_periodic_2d(phis[k1 + K], n[pa], n[s1a]))
        p2 = np.fft.fft2(embed_periodic_2d(phis[k2 + K], n[pa], n[s2a]))
        # product indexed (p, s1, s2) then permuted to (0, 1, 2)
        prod = g[:, None, None] * p1[:, :, None] * p2[:, None, :]
        perm = np.argsort([pa, s1a, s2a])
        return np.transpose(prod, perm)


def build_system_3d(dims, levels, j0=0, full=False, fan=None, q=None) -> System3D:
    # src/system3d.cpp:82-142
    p = Profile(list(levels), j0)
    fan = maxflat_fan(4) if fan is None else fan
    q = qmf_default() if q is None else q
    idx = enumerate_filters_3d(p, full)
    J = p.top_level
    scales = []
    for s, d in enumerate(p.levels):
        j = j0 + s
        K = 1 << d
        phis = [build_phi_component(j, k, d, J, fan, q) for k in range(-K, K + 1)]
        scales.append((d, cascade(q, J - j)[1], phis))
    sys = System3D(tuple(dims), p, idx, cascade(q, J)[0], scales)
    W = np.zeros(dims)
    norms = np.zeros(len(idx))
    N = float(np.prod(dims))
    for i in range(len(idx)):
        m = np.abs(sys.filter_freq(i)) ** 2
        W += m
        norms[i] = math.sqrt(m.sum() / N)
    sys.frame_weight = W
    sys.filter_norms = norms
    return sys


def forward_3d(f, s: System3D):  # src/transform.cpp:39-61
    F = np.fft.fftn(f)
    out = np.zeros((s.R,) + tuple(s.dims))
    for i in range(s.R):
        out[i] = np.real(np.fft.ifftn(np.conj(s.filter_freq(i)) * F))
    return out


def inverse_3d(bands, s: System3D):  # src/transform.cpp:94-125
    acc = np.zeros(s.dims, dtype=np.complex128)
    for i in range(s.R):
        acc += np.fft.fftn(bands[i]) * s.filter_freq(i) / s.frame_weight
    return np.real(np.fft.ifftn(acc))


# ----------------------------------------------------------------- threshold
def defaults_2d(sigma, n_scales=4):  # src/apps.cpp:92-96
    k = [2.5] * n_scales
    if n_scales > 0:
        k[-1] = 3.8
    return k, sigma


def defaults_3d(sigma, n_scales=3):  # src/apps.cpp:97-101
    k = [3.0] * n_scales
    if n_scales > 0:
        k[-1] = 4.0
    return k, sigma


def band_thresholds(index, j0, filter_norms, K, sigma, scaled=True):
    """delta_i per band (apps.cpp:73-76); -1 marks the untouched lowpass."""
    out = np.full(len(index), -1.0)
    for i, rec in enumerate(index):
        scale = rec[1]
        if scale < 0:
            continue
        dlt = K[scale - j0] * sigma
        if scaled:
            dlt *= filter_norms[i]
        out[i] = dlt
    return out


def hard_threshold(bands, index, j0, filter_norms, K, sigma, scaled=True):
    # src/apps.cpp:57-81: keep |x| >= delta, lowpass untouched
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    out = bands.copy()
    d = band_thresholds(index, j0, filter_norms, K, sigma, scaled)
    for i in range(len(index)):
        if d[i] < 0:
            continue
        b = out[i]
        b[np.abs(b) < d[i]] = 0.0
    return out


# ----------------------------------------------------------------- inputs
class MT19937_64:
    """std::mt19937_64 (C++ [rand.predef]); the reference's RNG (apps.cpp:17-45,
    phantoms.cpp:110-130, tests/oracles.hpp:175-190)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            prev = self.mt[i - 1]
            self.mt[i] = (6364136223846793005 * (prev ^ (prev >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.idx = 312

    def _twist(self):
        mt = self.mt
        UM, LM = 0xFFFFFFFF80000000, 0x7FFFFFFF
        A = 0xB5026F5AA96619E9
        for i in range(312):
            x = (mt[i] & UM) | (mt[(i + 1) % 312] & LM)
            xa = x >> 1
            if x & 1:
                xa ^= A
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.idx = 0

    def __call__(self) -> int:
        if self.idx >= 312:
            self._twist()
        y = self.mt[self.idx]
        self.idx += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF



def serialize_shcf(bands, index) -> bytes:  # src/transform.cpp:185-213
    """SHCF bytes: "SHCF", u16 1, u8 ndim, u32 dims, u32 count, records
    (u8 kind, i32 scale, i32 k1/shear, i32 k2/0), then f64 LE row-major."""
    import struct
    bands = np.ascontiguousarray(bands, dtype="<f8")
    nd = bands.ndim - 1
    out = [b"SHCF", struct.pack("<HB", 1, nd), struct.pack("<%dI" % nd, *bands.shape[1:]),
           struct.pack("<I", bands.shape[0])]
    for r in index:
        out.append(struct.pack("<Biii", r[0], r[1], r[2], r[3] if len(r) > 3 else 0))
    out.append(bands.tobytes())
    return b"".join(out)


def random_grid(shape, seed):
    """U[-1,1) grid, tests/oracles.hpp:175-190 (pure Python: small sizes only)."""
    rng = MT19937_64(seed)
    n = int(np.prod(shape))
    v = np.array([2.0 * (rng() * 2.0 ** -64) - 1.0 for _ in range(n)])
    return v.reshape(shape)


def cartoon(n):  # src/phantoms.cpp:14-36
    i = np.arange(n, dtype=np.float64)[:, None]
    j = np.arange(n, dtype=np.float64)[None, :]
    x = i / n - 0.5 + 0 * j
    y = j / n - 0.5 + 0 * i
    img = np.full((n, n), 32.0)
    img[y > 0.12 + 0.18 * np.sin(5.0 * x)] = 96.0
    u = 0.8 * (x + 0.12) + 0.6 * (y + 0.18)
    v = -0.6 * (x + 0.12) + 0.8 * (y + 0.18)
    img[(u / 0.28) ** 2 + (v / 0.16) ** 2 < 1.0] = 200.0
    r2 = (x - 0.22) ** 2 + (y - 0.2) ** 2
    img[r2 < 0.16 ** 2] = 150.0
    img[r2 < 0.055 ** 2] = 60.0
    img[(np.abs(x + 0.3) < 0.06) & (np.abs(y + 0.32) < 0.06)] = 255.0
    return img


def psnr(ref, test):  # src/apps.cpp:125-135
    e = np.sqrt(np.sum((ref - test) ** 2))
    if e == 0:
        return math.inf
    return 20.0 * math.log10(255.0 * math.sqrt(ref.size) / e)
