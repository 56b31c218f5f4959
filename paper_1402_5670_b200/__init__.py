"""paper_1402_5670_b200 -- B200-native digital shearlet dec/rec hot path.

Python host mirror of the reference's C++ API for this path
(/root/reference/proj/core/include/shearlet/{system2d,system3d,transform,apps}.hpp),
bound through the C ABI in include/shearlet_b200.h (libshearlet_b200.so, built
in-tree by __graft_entry__.build()). Names, argument meaning and error classes
follow the reference:

    build_system_2d(rows, cols, ScaleProfile, fan, full_system)  system2d.hpp:66-69
    build_system_3d(dims, ScaleProfile, fan, full_system)        system3d.hpp:68-71
    forward(f, sys) / inverse(coeffs, sys)                       transform.hpp:27-37
    hard_threshold(coeffs, schedule, sys), denoise(...)          apps.hpp:31-44
    ThresholdSchedule.defaults_2d / defaults_3d                  apps.hpp:19-29
    sys.filter_norms (RMS), sys.frame_weight, sys.frame_bounds() system2d.hpp:29-51

Arrays: numpy float64 arrays run the host-pointer entry points (value
semantics, like the reference); CUDA torch tensors run the device-pointer
entry points on the current torch stream and return CUDA tensors. There is
no CPU fallback: without the built library every call raises.
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SLB_LIB", os.path.join(_HERE, "libshearlet_b200.so"))  # SLB_LIB: dev variants

# ------------------------------------------------------------------ errors
# errors.hpp:9-56


class Error(RuntimeError):
    pass


class DomainError(Error):
    pass


class ShapeError(Error):
    pass


class ConfigError(Error):
    pass


class AssetError(Error):
    pass


class FormatError(Error):
    pass


class SingularFrameError(Error):
    pass


class UnsupportedSizeError(Error):
    pass


class DegenerateMaskError(Error):
    pass


class DegenerateTruthError(Error):
    pass


class NcclError(Error):
    """NCCL failure or libnccl.so.2 not loadable (SL_ERR_NCCL)."""


class CudaError(Error):
    pass


class InvalidArgument(Error):
    pass


_CODES = {1: Error, 2: ShapeError, 3: ConfigError, 4: DomainError, 5: SingularFrameError,
          6: UnsupportedSizeError, 7: AssetError, 8: FormatError, 9: DegenerateMaskError, 10: DegenerateTruthError, 20: CudaError,
          21: NcclError, 22: InvalidArgument}

# ------------------------------------------------------------------ library
_lib = None


class _DevLib:
    """SLB_LIB variant wrapper: symbols the variant does not export bind to a stub."""

    class _Missing:
        argtypes = restype = None

        def __call__(self, *a):
            raise AttributeError("entry point missing from this SLB_LIB variant")

    def __init__(self, lib):
        object.__setattr__(self, "_l", lib)

    def __getattr__(self, name):
        try:
            return getattr(self._l, name)
        except AttributeError:
            m = _DevLib._Missing()
            object.__setattr__(self, name, m)
            return m


def lib():
    """Load libshearlet_b200.so; raises loudly if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(there is no CPU fallback for the shearlet hot path)")
    L = C.CDLL(LIB_PATH)
    if "SLB_LIB" in os.environ:
        L = _DevLib(L)  # A/B variants built from older commits may lack newer entry points
    P = C.c_void_p
    i = C.c_int
    dp = C.POINTER(C.c_double)
    ip = C.POINTER(C.c_int)
    L.sl_version.restype = C.c_char_p
    L.sl_last_error.restype = C.c_char_p
    L.sl_device_count.argtypes = [ip]
    L.sl_system_create_2d.argtypes = [i, i, ip, i, i, i, i, i, i, i, C.POINTER(P)]
    L.sl_system_create_3d.argtypes = [i, i, i, ip, i, i, i, i, i, i, i, C.POINTER(P)]
    bank = [dp, i, i, dp, i, i, dp, i, i, i, i, C.c_char_p]
    L.sl_system_create_2d_ex.argtypes = [i, i, ip, i, i, i] + bank + [i, i, i, C.POINTER(P)]
    L.sl_system_create_3d_ex.argtypes = [i, i, i, ip, i, i, i] + bank + [i, i, i, C.POINTER(P)]
    L.sl_default_fan.argtypes = [dp, C.c_int64, ip, ip, ip, ip]
    L.sl_describe.argtypes = [P, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)]
    L.sl_system_create_from_descriptor.argtypes = [C.c_char_p, i, i, i, i, C.POINTER(P)]
    L.sl_system_destroy.argtypes = [P]
    L.sl_ndim.argtypes = [P, ip, C.POINTER(C.c_int64)]
    L.sl_redundancy.argtypes = [P, ip]
    L.sl_shard.argtypes = [P, ip, ip]
    L.sl_index.argtypes = [P, C.POINTER(C.c_int32)]
    L.sl_filter_norms.argtypes = [P, dp]
    L.sl_frame_weight.argtypes = [P, dp]
    L.sl_frame_bounds.argtypes = [P, dp, dp]
    L.sl_filter_spectrum.argtypes = [P, i, dp]
    L.sl_sheardec_dev.argtypes = [P, P, P, P]
    L.sl_sheardec_threshold_dev.argtypes = [P, P, P, dp, i, C.c_double, i, P]
    L.sl_shearrec_dev.argtypes = [P, P, i, P, P]
    L.sl_hard_threshold_dev.argtypes = [P, P, P, i, dp, i, C.c_double, i, P]
    L.sl_denoise_dev.argtypes = [P, P, P, dp, i, C.c_double, i, P]
    L.sl_denoise_stack_dev.argtypes = [P, P, P, P, dp, i, C.c_double, i, P]
    L.sl_sheardec_host.argtypes = [P, dp, dp]
    L.sl_shearrec_host.argtypes = [P, dp, i, dp]
    L.sl_hard_threshold_host.argtypes = [P, dp, dp, i, dp, i, C.c_double, i]
    L.sl_denoise_host.argtypes = [P, dp, dp, dp, i, C.c_double, i]
    L.sl_set_stack_output.argtypes = [P, i]
    L.sl_set_streams.argtypes = [P, i]
    L.sl_sheardec_batch_dev.argtypes = [P, P, i, P, dp, i, C.c_double, i, P]
    L.sl_shearrec_batch_dev.argtypes = [P, P, i, P, P]
    L.sl_denoise_batch_dev.argtypes = [P, P, i, P, dp, i, C.c_double, i, P]
    L.sl_denoise_batch_stack_dev.argtypes = [P, P, i, P, P, dp, i, C.c_double, i, P]
    L.sl_denoise_batch_host.argtypes = [P, dp, i, dp, dp, i, C.c_double, i]
    L.sl_inpaint_dev.argtypes = [P, P, P, P, i, C.c_double, C.c_double, i, P]
    L.sl_inpaint_host.argtypes = [P, dp, dp, dp, i, C.c_double, C.c_double, i]
    L.sl_separate_dev.argtypes = [P, P, P, P, P, i, C.c_double, C.c_double, i, P]
    L.sl_separate_host.argtypes = [P, P, dp, dp, dp, i, C.c_double, C.c_double, i]
    L.sl_shcf_size.argtypes = [P, i, C.POINTER(C.c_size_t)]
    L.sl_shcf_serialize.argtypes = [P, dp, i, C.c_char_p, C.c_size_t]
    L.sl_shcf_deserialize.argtypes = [P, C.c_char_p, C.c_size_t, dp, i]
    L.sl_shcf_forward_file.argtypes = [P, dp, C.c_char_p, i]
    L.sl_shcf_inverse_file.argtypes = [P, C.c_char_p, dp, i]
    L.sl_load_pgm.argtypes = [C.c_char_p, dp, C.c_int64, ip, ip, ip]
    L.sl_save_pgm.argtypes = [dp, i, i, C.c_char_p, i]
    L.sl_load_svol.argtypes = [C.c_char_p, dp, C.c_int64, C.POINTER(C.c_int64)]
    L.sl_save_svol.argtypes = [dp, C.POINTER(C.c_int64), C.c_char_p]
    L.sl_gaussian_kernel.argtypes = [C.c_double, dp, C.c_int64, ip, ip]
    L.sl_binarize.argtypes = [dp, dp, C.c_int64, C.c_double]
    kern = [dp, i, i, i, i, i]
    L.sl_quality_q.argtypes = [i, i, dp, dp, C.c_double] + kern + [dp]
    L.sl_quality_q_opt.argtypes = [i, i, dp, dp] + kern + [dp, ip, dp]
    L.sl_profile.argtypes = [P, i]
    L.sl_pass_stats.argtypes = [P, i, C.c_char_p, dp, C.POINTER(C.c_int64), C.POINTER(C.c_int64), ip]
    L.sl_launch_count.argtypes = [P, C.POINTER(C.c_int64)]
    L.sl_system_set_precision.argtypes = [P, i]
    L.sl_sheardec_f32_dev.argtypes = [P, P, P, dp, i, C.c_double, i, P]
    L.sl_shearrec_f32_dev.argtypes = [P, P, i, P, P]
    L.sl_denoise_f32_dev.argtypes = [P, P, P, P, dp, i, C.c_double, i, P]
    L.sl_denoise_batch_f32_dev.argtypes = [P, P, i, P, P, dp, i, C.c_double, i, P]
    u8 = C.c_char_p
    L.sl_comm_unique_id.argtypes = [u8]
    L.sl_comm_create.argtypes = [u8, i, i, i, C.POINTER(P)]
    L.sl_comm_destroy.argtypes = [P]
    L.sl_comm_info.argtypes = [P, ip, ip, ip]
    L.sl_partition.argtypes = [C.c_int64, i, i, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
    L.sl_system_set_comm.argtypes = [P, P, i]
    L.sl_denoise_dist_dev.argtypes = [P, P, P, dp, i, C.c_double, i, i, P]
    L.sl_denoise_batch_dist_dev.argtypes = [P, P, i, P, dp, i, C.c_double, i, P]
    L.sl_denoise_batch_dist_host.argtypes = [P, dp, i, dp, dp, i, C.c_double, i]
    L.sl_phantom_cartoon.argtypes = [i, dp]
    L.sl_phantom_cartoon_volume.argtypes = [i, dp]
    L.sl_add_gaussian_noise.argtypes = [dp, dp, C.c_int64, C.c_double, C.c_uint64]
    _lib = L
    return L


EXPORTED_SYMBOLS = [
    "sl_version", "sl_last_error", "sl_device_count", "sl_system_create_2d", "sl_system_create_3d",
    "sl_system_destroy", "sl_ndim", "sl_redundancy", "sl_shard", "sl_index", "sl_filter_norms",
    "sl_frame_weight", "sl_frame_bounds", "sl_filter_spectrum", "sl_sheardec_dev", "sl_sheardec_threshold_dev",
    "sl_shearrec_dev", "sl_hard_threshold_dev", "sl_denoise_dev", "sl_denoise_stack_dev", "sl_sheardec_host", "sl_shearrec_host",
    "sl_hard_threshold_host", "sl_denoise_host", "sl_profile", "sl_pass_stats", "sl_launch_count",
    "sl_set_streams", "sl_set_stack_output", "sl_sheardec_batch_dev", "sl_shearrec_batch_dev", "sl_denoise_batch_dev",
    "sl_denoise_batch_stack_dev", "sl_denoise_batch_host", "sl_inpaint_dev", "sl_inpaint_host", "sl_separate_dev", "sl_separate_host",
    "sl_shcf_size", "sl_shcf_serialize", "sl_shcf_deserialize", "sl_shcf_forward_file", "sl_shcf_inverse_file",
    "sl_system_create_2d_ex", "sl_system_create_3d_ex", "sl_default_fan",
    "sl_describe", "sl_system_create_from_descriptor",
    "sl_gaussian_kernel", "sl_binarize", "sl_quality_q", "sl_quality_q_opt",
    "sl_load_pgm", "sl_save_pgm", "sl_load_svol", "sl_save_svol",
    "sl_phantom_cartoon", "sl_phantom_cartoon_volume",
    "sl_add_gaussian_noise",
    "sl_system_set_precision", "sl_sheardec_f32_dev", "sl_shearrec_f32_dev", "sl_denoise_f32_dev",
    "sl_denoise_batch_f32_dev",
    "sl_comm_unique_id", "sl_comm_create", "sl_comm_destroy", "sl_comm_info", "sl_partition", "sl_system_set_comm",
    "sl_denoise_dist_dev", "sl_denoise_batch_dist_dev", "sl_denoise_batch_dist_host",
]


def _check(rc: int):
    if rc != 0:
        msg = lib().sl_last_error().decode()
        raise _CODES.get(rc, Error)(msg)


def _dp(a: np.ndarray):
    if a.dtype != np.float64 or not a.flags.c_contiguous:
        raise InvalidArgument("expected a C-contiguous float64 array")
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _is_cuda_tensor(x) -> bool:
    return type(x).__module__.startswith("torch") and getattr(x, "is_cuda", False)


def _stream_ptr(device: int):
    import torch
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


# ------------------------------------------------------------------ profiles
@dataclass
class ScaleProfile:
    """filters.hpp:79-92."""
    shear_levels: List[int]
    coarsest_scale_offset: int = 0

    @property
    def n_scales(self) -> int:
        return len(self.shear_levels)

    def top_level(self) -> int:
        return self.coarsest_scale_offset + self.n_scales

    def validate(self):  # filters.cpp:168-176
        if self.coarsest_scale_offset < 0:
            raise ConfigError("ScaleProfile: coarsest scale offset must be >= 0")
        if any(d < 0 for d in self.shear_levels):
            raise ConfigError("ScaleProfile: shear levels must be >= 0")

    @staticmethod
    def from_levels(levels: Sequence[int], j0: int = 0) -> "ScaleProfile":
        p = ScaleProfile(list(int(x) for x in levels), int(j0))
        p.validate()
        return p

    @staticmethod
    def parabolic(n_scales: int, j0: int = 1) -> "ScaleProfile":  # d_j = ceil(j/2)
        return ScaleProfile.from_levels([(j0 + i + 1) // 2 for i in range(n_scales)], j0)


@dataclass
class ThresholdSchedule:
    """apps.hpp:19-29."""
    per_scale_factors: List[float]
    sigma: float = 0.0
    scale_by_filter_norm: bool = True

    @staticmethod
    def defaults_2d(sigma: float, n_scales: int = 4) -> "ThresholdSchedule":
        k = [2.5] * n_scales
        if n_scales > 0:
            k[-1] = 3.8
        return ThresholdSchedule(k, sigma, True)

    @staticmethod
    def defaults_3d(sigma: float, n_scales: int = 3) -> "ThresholdSchedule":
        k = [3.0] * n_scales
        if n_scales > 0:
            k[-1] = 4.0
        return ThresholdSchedule(k, sigma, True)


# ------------------------------------------------------------------ systems
class _System:
    ndim = 0

    def __init__(self, handle, profile: ScaleProfile, full_system: bool, device: int):
        self._h = handle
        self.profile = profile
        self.full_system = full_system
        self.device = device
        L = lib()
        R = C.c_int()
        _check(L.sl_redundancy(self._h, C.byref(R)))
        self._R = R.value
        lo, hi = C.c_int(), C.c_int()
        _check(L.sl_shard(self._h, C.byref(lo), C.byref(hi)))
        self.shard = (lo.value, hi.value)
        rec = np.zeros((self._R, 4), dtype=np.int32)
        _check(L.sl_index(self._h, rec.ctypes.data_as(C.POINTER(C.c_int32))))
        self.index_records = rec
        rms = np.zeros(self._R)
        _check(L.sl_filter_norms(self._h, _dp(rms)))
        self.filter_norms = rms
        self._W = None

    def __del__(self):
        try:
            if self._h:
                lib().sl_system_destroy(self._h)
                self._h = None
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    def redundancy(self) -> int:
        return self._R

    @property
    def n_bands(self) -> int:
        return self.shard[1] - self.shard[0]

    @property
    def frame_weight(self) -> np.ndarray:
        if self._W is None:
            w = np.zeros(self.shape)
            _check(lib().sl_frame_weight(self._h, _dp(w)))
            self._W = w
        return self._W

    def frame_bounds(self):
        a, b = C.c_double(), C.c_double()
        _check(lib().sl_frame_bounds(self._h, C.byref(a), C.byref(b)))
        return a.value, b.value

    # ---- instrumentation (bench.py) ----
    def set_profiling(self, enable: bool = True):
        _check(lib().sl_profile(self._h, int(enable)))

    def pass_stats(self):
        n = C.c_int()
        names = C.create_string_buffer(32 * 64)
        ms = np.zeros(64)
        cnt = np.zeros(64, dtype=np.int64)
        units = np.zeros(64, dtype=np.int64)
        _check(lib().sl_pass_stats(self._h, 64, names, _dp(ms), cnt.ctypes.data_as(C.POINTER(C.c_int64)),
                                   units.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(n)))
        raw = names.raw
        return {raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): (float(ms[i]), int(cnt[i]), int(units[i]))
                for i in range(n.value)}

    def set_comm(self, comm: Optional["Comm"], shard_bands: bool = True):
        """Attach a multi-GPU communicator (None detaches). shard_bands: this
        rank keeps only its band range (3D / single frames); False keeps the
        whole bank (2D batches shard by image)."""
        _check(lib().sl_system_set_comm(self._h, comm.handle if comm else None, int(bool(comm) and shard_bands)))
        lo, hi = C.c_int(), C.c_int()
        _check(lib().sl_shard(self._h, C.byref(lo), C.byref(hi)))
        self.shard = (lo.value, hi.value)
        self._comm = comm  # keeps the communicator alive while attached

    def set_stack_output(self, materialize: bool = True):
        """Fused denoise writes the thresholded stack (default, as the reference) or not."""
        _check(lib().sl_set_stack_output(self._h, int(materialize)))

    def set_streams(self, n: int):
        """Concurrent internal streams used by the batched entry points."""
        _check(lib().sl_set_streams(self._h, int(n)))

    def launch_count(self) -> int:
        c = C.c_int64()
        _check(lib().sl_launch_count(self._h, C.byref(c)))
        return c.value

    def filter_freq(self, i: int) -> np.ndarray:
        """psi_hat_i on the full grid (filters[i], system2d.hpp:38; filter_freq, system3d.cpp:144-186)."""
        out = np.zeros(self.shape + (2,))
        _check(lib().sl_filter_spectrum(self._h, int(i), _dp(out)))
        return out[..., 0] + 1j * out[..., 1]

    def dual_freq(self, i: int) -> np.ndarray:
        """psi_hat_i / W (dual_freq, system3d.cpp:188-195; duals()[i], system2d.cpp:128-148)."""
        W = self.frame_weight
        if W.min() < 1e-12:
            raise SingularFrameError("duals: frame weight below 1e-12")
        return self.filter_freq(i) / W

    def duals(self):
        """All dual spectra (system2d.hpp:45); materialised on request, R full complex grids."""
        return [self.dual_freq(i) for i in range(self._R)]

    @property
    def filters(self):
        """All filter spectra as full complex grids (system2d.hpp:38), materialised on request."""
        return [self.filter_freq(i) for i in range(self._R)]


class ShearletSystem2D(_System):
    """system2d.hpp:29-51 (filters live on the GPU as real Hermitian halves)."""
    ndim = 2

    def __init__(self, handle, rows, cols, profile, full_system, device):
        self.rows, self.cols = rows, cols
        self.shape = (rows, cols)
        super().__init__(handle, profile, full_system, device)
        # FilterIndex2D records: (kind, scale, shear)
        self.index = [(int(k), int(s), int(sh)) for k, s, sh, _ in self.index_records]


class ShearletSystem3D(_System):
    """system3d.hpp:32-61 (filters synthesised on the fly from factor tables)."""
    ndim = 3

    def __init__(self, handle, dims, profile, full_system, device):
        self.dims = tuple(dims)
        self.shape = tuple(dims)
        super().__init__(handle, profile, full_system, device)
        self.index = [(int(k), int(s), int(a), int(b)) for k, s, a, b in self.index_records]


def _levels_arg(profile: ScaleProfile):
    lv = np.asarray(profile.shear_levels, dtype=np.int32)
    return lv, lv.ctypes.data_as(C.POINTER(C.c_int))


def alpha_to_shear_levels(alpha: Sequence[float], j0: int) -> List[int]:  # filters.cpp:196-207
    out = []
    for i, a in enumerate(alpha):
        if not (0.0 < a < 2.0):
            raise DomainError("alpha_to_shear_levels: alpha must lie in (0, 2)")
        out.append(int(math.ceil((2.0 - a) * (j0 + i) / 2.0)))
    return out


@dataclass
class QmfPair:
    """Quadrature-mirror pair (filters.hpp:14-21): 1D taps with a centre index."""
    lowpass: np.ndarray
    highpass: np.ndarray
    lowpass_center: int
    highpass_center: int

    @staticmethod
    def from_lowpass(taps: Sequence[float], center: Optional[int] = None) -> "QmfPair":
        """g(n) = (-1)^n h(n), n counted from the centre (filters.cpp:22-34)."""
        h = np.asarray(taps, dtype=np.float64).copy()
        c = len(h) // 2 if center is None else int(center)
        g = np.array([(-v if (i - c) % 2 else v) for i, v in enumerate(h)], dtype=np.float64)
        return QmfPair(h, g, c, c)

    @staticmethod
    def maximally_flat_9tap() -> Optional["QmfPair"]:
        return None  # the library's built-in default (filters.cpp:12-20, 36-38)


@dataclass
class FanFilter:
    """2D directional fan filter with provenance (filters.hpp:51-67)."""
    taps: np.ndarray
    center0: int
    center1: int
    provenance: str = ""

    @staticmethod
    def impulse() -> "FanFilter":
        return FanFilter(np.ones((1, 1)), 0, 0, "impulse")

    @staticmethod
    def default() -> "FanFilter":
        """default_fan_filter() (filters.cpp:112-122): the bundled dmaxflat4 fan, checksum-verified."""
        r, c, c0, c1 = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(lib().sl_default_fan(None, 0, C.byref(r), C.byref(c), C.byref(c0), C.byref(c1)))
        t = np.zeros((r.value, c.value))
        _check(lib().sl_default_fan(_dp(t), t.size, None, None, None, None))
        f = FanFilter(t, c0.value, c1.value, "dmaxflat4")
        if fan_checksum(f) != DEFAULT_FAN_CHECKSUM:
            raise AssetError("default_fan_filter: checksum mismatch on bundled fan filter")
        return f

    @staticmethod
    def load(path: str) -> "FanFilter":
        """load_fan_filter (filters.cpp:124-140): "rows cols c0 c1" then rows of taps."""
        try:
            with open(path) as fh:
                words = fh.read().split()
        except OSError:
            raise AssetError("fan filter asset not readable: " + path)
        try:
            rows, cols, c0, c1 = int(words[0]), int(words[1]), int(words[2]), int(words[3])
        except (IndexError, ValueError):
            raise AssetError("fan filter asset header corrupt: " + path)
        if rows <= 0 or cols <= 0:
            raise AssetError("fan filter asset header corrupt: " + path)
        try:
            vals = [float(w) for w in words[4:4 + rows * cols]]
        except ValueError:
            raise AssetError("fan filter asset truncated: " + path)
        if len(vals) < rows * cols:
            raise AssetError("fan filter asset truncated: " + path)
        return FanFilter(np.array(vals).reshape(rows, cols), c0, c1, "file:" + path)

    def save(self, path: str):
        """save_fan_filter (filters.cpp:142-156)."""
        try:
            with open(path, "w") as fh:
                fh.write(f"{self.taps.shape[0]} {self.taps.shape[1]} {self.center0} {self.center1}\n")
                for row in self.taps:
                    fh.write(" ".join(repr(float(v)) for v in row) + "\n")
        except OSError:
            raise AssetError("cannot write fan filter asset: " + path)


DEFAULT_FAN_CHECKSUM = 0xB942F71DC884B1BA  # filters.cpp:113-116


def fan_checksum(fan: "FanFilter") -> int:
    """FNV-1a 64 over dims, centres and little-endian tap bytes (filters.cpp:89-110)."""
    h = 1469598103934665603
    meta = np.array([fan.taps.shape[0], fan.taps.shape[1], fan.center0 & 0xFFFFFFFFFFFFFFFF,
                     fan.center1 & 0xFFFFFFFFFFFFFFFF], dtype="<u8").tobytes()
    for b in meta + np.ascontiguousarray(fan.taps, dtype="<f8").tobytes():
        h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def _bank_args(fan, qmf):
    """(lowpass, len, c, highpass, len, c, fan, rows, cols, c0, c1) ctypes args; keeps arrays alive."""
    keep = []
    if qmf is None:
        q = [None, 0, 0, None, 0, 0]
    else:
        lp = np.ascontiguousarray(qmf.lowpass, dtype=np.float64)
        hp = np.ascontiguousarray(qmf.highpass, dtype=np.float64)
        keep += [lp, hp]
        q = [_dp(lp), len(lp), int(qmf.lowpass_center), _dp(hp), len(hp), int(qmf.highpass_center)]
    if fan is None or isinstance(fan, str):
        if fan not in (None, "dmaxflat4", "impulse"):
            raise ConfigError(f"unknown fan filter {fan!r}")
        fan = FanFilter.impulse() if fan == "impulse" else None
    if fan is None:
        f = [None, 0, 0, 0, 0, None]
    else:
        t = np.ascontiguousarray(fan.taps, dtype=np.float64)
        keep.append(t)
        f = [_dp(t), t.shape[0], t.shape[1], int(fan.center0), int(fan.center1), fan.provenance.encode()]
    return q + f, keep


def build_system_2d(rows: int, cols: int, profile: ScaleProfile, fan=None, qmf: Optional[QmfPair] = None,
                    full_system: bool = False, device: int = 0, shard=None, dtype: str = "f64") -> ShearletSystem2D:
    """build_system_2d (system2d.hpp:66-69). fan: None/"dmaxflat4" (default_fan_filter), "impulse" or a
    FanFilter; qmf: None (maximally_flat_9tap) or a QmfPair. dtype "f32" also prepares the optional
    fp32 mode (float32 CUDA tensors then run the fp32 kernels; fp64 stays available)."""
    profile.validate()
    lv, lvp = _levels_arg(profile)
    h = C.c_void_p()
    lo, hi = (0, -1) if shard is None else shard
    args, _keep = _bank_args(fan, qmf)
    _check(lib().sl_system_create_2d_ex(int(rows), int(cols), lvp, len(lv), profile.coarsest_scale_offset,
                                        int(full_system), *args, int(device), int(lo), int(hi), C.byref(h)))
    sys = ShearletSystem2D(h, rows, cols, profile, full_system, device)
    if dtype == "f32":
        _check(lib().sl_system_set_precision(h, 32))
    elif dtype != "f64":
        raise ConfigError("dtype must be 'f64' or 'f32'")
    return sys


def build_system_3d(dims, profile: ScaleProfile, fan=None, qmf: Optional[QmfPair] = None,
                    full_system: bool = False, device: int = 0, shard=None, dtype: str = "f64") -> ShearletSystem3D:
    """build_system_3d (system3d.hpp:68-71); fan / qmf as build_system_2d. dtype "f32" enables the
    optional fp32 fused denoise (float32 CUDA volumes) on cubic 64/128/192/256 grids."""
    profile.validate()
    lv, lvp = _levels_arg(profile)
    h = C.c_void_p()
    n0, n1, n2 = (int(x) for x in dims)
    lo, hi = (0, -1) if shard is None else shard
    args, _keep = _bank_args(fan, qmf)
    _check(lib().sl_system_create_3d_ex(n0, n1, n2, lvp, len(lv), profile.coarsest_scale_offset,
                                        int(full_system), *args, int(device), int(lo), int(hi), C.byref(h)))
    sys = ShearletSystem3D(h, (n0, n1, n2), profile, full_system, device)
    if dtype == "f32":
        _check(lib().sl_system_set_precision(h, 32))
    elif dtype != "f64":
        raise ConfigError("dtype must be 'f64' or 'f32'")
    return sys


def redundancy_2d(profile: ScaleProfile, full_system: bool = False) -> int:  # system2d.cpp:49-57
    profile.validate()
    r = 1
    for d in profile.shear_levels:
        per = 2 * (1 << d) + 1
        r += 2 * per if full_system else 2 * per - 2
    return r


def redundancy_3d(profile: ScaleProfile, full_system: bool = False) -> int:  # system3d.cpp:27-35
    profile.validate()
    r = 1
    for d in profile.shear_levels:
        q = 2 * (1 << d) + 1
        r += 3 * q * q if full_system else 3 * q * q - 6 * q + 4
    return r


# ------------------------------------------------------------------ descriptors
@dataclass
class SystemDescriptor:
    """descriptor.hpp:14-23: enough to rebuild a system bit-identically."""
    is_3d: bool = False
    dims: tuple = (0, 0)
    j0: int = 0
    shear_levels: List[int] = field(default_factory=list)
    full_system: bool = False
    qmf_lowpass: Optional[np.ndarray] = None
    qmf_center: int = 0
    fan_name: str = ""
    fan_checksum: int = 0

    def text(self) -> str:
        """write_descriptor's text (descriptor.cpp:48-67)."""
        lines = ["shearlet-system 1", "dims " + " ".join(str(int(d)) for d in self.dims), f"j0 {self.j0}",
                 "shear_levels" + "".join(f" {v}" for v in self.shear_levels),
                 f"full_system {1 if self.full_system else 0}", f"qmf_center {self.qmf_center}",
                 "qmf" + "".join(" %.17g" % v for v in self.qmf_lowpass),
                 f"fan {self.fan_name} {self.fan_checksum:x}"]
        return "\n".join(lines) + "\n"

    @staticmethod
    def parse(text: str) -> "SystemDescriptor":
        """read_descriptor's grammar (descriptor.cpp:69-126)."""
        d = SystemDescriptor()
        seen = set()
        for line in text.splitlines():
            w = line.split()
            if not w or w[0].startswith("#"):
                continue
            key, rest = w[0], w[1:]
            try:
                if key == "shearlet-system":
                    if not rest or int(rest[0]) != 1:
                        raise FormatError("descriptor: unsupported version")
                elif key == "dims":
                    if len(rest) not in (2, 3):
                        raise FormatError("descriptor: dims must have 2 or 3 entries")
                    d.dims, d.is_3d = tuple(int(x) for x in rest), len(rest) == 3
                elif key == "j0":
                    d.j0 = int(rest[0])
                elif key == "shear_levels":
                    d.shear_levels = [int(x) for x in rest]
                elif key == "full_system":
                    d.full_system = int(rest[0]) != 0
                elif key == "qmf_center":
                    d.qmf_center = int(rest[0])
                elif key == "qmf":
                    if not rest:
                        raise FormatError("descriptor: empty qmf taps")
                    d.qmf_lowpass = np.array([float(x) for x in rest])
                elif key == "fan":
                    d.fan_name, d.fan_checksum = rest[0], int(rest[1], 16)
                else:
                    raise FormatError(f"descriptor: unknown key '{key}'")
            except (IndexError, ValueError):
                raise FormatError(f"descriptor: bad {key} line")
            seen.add(key)
        if not {"shearlet-system", "dims", "shear_levels", "qmf", "fan"} <= seen:
            raise FormatError("descriptor: missing required fields")
        return d


def describe(sys: "_System") -> SystemDescriptor:
    """describe(sys) (descriptor.cpp:30-46), from the library's record of the build."""
    n = C.c_size_t()
    _check(lib().sl_describe(sys.handle, None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().sl_describe(sys.handle, buf, n.value + 1, C.byref(n)))
    return SystemDescriptor.parse(buf.value.decode())


def write_descriptor(d: SystemDescriptor, path: str):
    try:
        with open(path, "w") as fh:
            fh.write(d.text())
    except OSError:
        raise FormatError("cannot write system descriptor: " + path)


def read_descriptor(path: str) -> SystemDescriptor:
    try:
        with open(path) as fh:
            text = fh.read()
    except OSError:
        raise FormatError("cannot open system descriptor: " + path)
    return SystemDescriptor.parse(text)


def _from_descriptor(d: SystemDescriptor, ndim: int, device: int, shard):
    h = C.c_void_p()
    lo, hi = (0, -1) if shard is None else shard
    _check(lib().sl_system_create_from_descriptor(d.text().encode(), ndim, int(device), int(lo), int(hi),
                                                  C.byref(h)))
    return h


def build_from_descriptor_2d(d: SystemDescriptor, device: int = 0, shard=None) -> "ShearletSystem2D":
    """build_from_descriptor_2d (descriptor.cpp:142-147)."""
    h = _from_descriptor(d, 2, device, shard)
    prof = ScaleProfile(list(d.shear_levels), d.j0)
    return ShearletSystem2D(h, d.dims[0], d.dims[1], prof, d.full_system, device)


def build_from_descriptor_3d(d: SystemDescriptor, device: int = 0, shard=None) -> "ShearletSystem3D":
    """build_from_descriptor_3d (descriptor.cpp:149-154)."""
    h = _from_descriptor(d, 3, device, shard)
    prof = ScaleProfile(list(d.shear_levels), d.j0)
    return ShearletSystem3D(h, tuple(d.dims), prof, d.full_system, device)


# ------------------------------------------------------------------ transforms
def _check_signal(f, sys: _System, what: str):
    if tuple(f.shape) != tuple(sys.shape):
        raise ShapeError(f"{what}: signal dims do not match the system grid")


def _k_arg(schedule: ThresholdSchedule):
    K = np.ascontiguousarray(schedule.per_scale_factors, dtype=np.float64)
    return K, K.ctypes.data_as(C.POINTER(C.c_double))


def _is_f32(x) -> bool:
    import torch
    return _is_cuda_tensor(x) and x.dtype == torch.float32


def forward(f, sys: _System, threads: int = 0):
    """Undecimated analysis band_i = Re IDFT(conj(psi_i) DFT(f)) (transform.hpp:27-31).

    Returns the coefficient stack [n_bands, *dims] (numpy or CUDA tensor, like f).
    `threads` is accepted for API parity; the GPU grid replaces host threads."""
    _check_signal(f, sys, "forward")
    L = lib()
    if _is_f32(f):  # fp32 mode (sys built with dtype="f32")
        import torch
        f = f.contiguous()
        out = torch.empty((sys.n_bands,) + tuple(sys.shape), dtype=torch.float32, device=f.device)
        _check(L.sl_sheardec_f32_dev(sys.handle, C.c_void_p(f.data_ptr()), C.c_void_p(out.data_ptr()), None, 0,
                                     0.0, 0, _stream_ptr(f.device.index)))
        return out
    if _is_cuda_tensor(f):
        import torch
        f = f.contiguous().to(torch.float64)
        out = torch.empty((sys.n_bands,) + tuple(sys.shape), dtype=torch.float64, device=f.device)
        _check(L.sl_sheardec_dev(sys.handle, C.c_void_p(f.data_ptr()), C.c_void_p(out.data_ptr()),
                                 _stream_ptr(f.device.index)))
        return out
    f = np.ascontiguousarray(f, dtype=np.float64)
    out = np.empty((sys.n_bands,) + tuple(sys.shape))
    _check(L.sl_sheardec_host(sys.handle, _dp(f), _dp(out)))
    return out


def inverse(coeffs, sys: _System, threads: int = 0):
    """Exact synthesis f = Re IDFT(sum_i DFT(c_i) psi_i / W) (transform.hpp:33-37)."""
    if tuple(coeffs.shape[1:]) != tuple(sys.shape) or coeffs.shape[0] != sys.n_bands:
        raise ShapeError("inverse: coefficient stack does not match the system")
    L = lib()
    if _is_f32(coeffs):
        import torch
        coeffs = coeffs.contiguous()
        out = torch.empty(tuple(sys.shape), dtype=torch.float32, device=coeffs.device)
        _check(L.sl_shearrec_f32_dev(sys.handle, C.c_void_p(coeffs.data_ptr()), int(coeffs.shape[0]),
                                     C.c_void_p(out.data_ptr()), _stream_ptr(coeffs.device.index)))
        return out
    if _is_cuda_tensor(coeffs):
        import torch
        coeffs = coeffs.contiguous().to(torch.float64)
        out = torch.empty(tuple(sys.shape), dtype=torch.float64, device=coeffs.device)
        _check(L.sl_shearrec_dev(sys.handle, C.c_void_p(coeffs.data_ptr()), int(coeffs.shape[0]),
                                 C.c_void_p(out.data_ptr()), _stream_ptr(coeffs.device.index)))
        return out
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.empty(tuple(sys.shape))
    _check(L.sl_shearrec_host(sys.handle, _dp(coeffs), int(coeffs.shape[0]), _dp(out)))
    return out


def hard_threshold(coeffs, schedule: ThresholdSchedule, sys: _System):
    """Zero |x| < K_j sigma (RMS_i); lowpass untouched; returns a new stack (apps.hpp:31-38)."""
    K, Kp = _k_arg(schedule)
    L = lib()
    if _is_cuda_tensor(coeffs):
        import torch
        coeffs = coeffs.contiguous()
        out = torch.empty_like(coeffs)
        _check(L.sl_hard_threshold_dev(sys.handle, C.c_void_p(coeffs.data_ptr()), C.c_void_p(out.data_ptr()),
                                       int(coeffs.shape[0]), Kp, len(K), float(schedule.sigma),
                                       int(schedule.scale_by_filter_norm), _stream_ptr(coeffs.device.index)))
        return out
    coeffs = np.ascontiguousarray(coeffs, dtype=np.float64)
    out = np.empty_like(coeffs)
    _check(L.sl_hard_threshold_host(sys.handle, _dp(coeffs), _dp(out), int(coeffs.shape[0]), Kp, len(K),
                                    float(schedule.sigma), int(schedule.scale_by_filter_norm)))
    return out


def forward_thresholded(f, sys: _System, schedule: ThresholdSchedule):
    """forward() with hard_threshold() fused into the dec epilogue (CUDA tensors)."""
    _check_signal(f, sys, "forward")
    import torch
    K, Kp = _k_arg(schedule)
    f = f.contiguous().to(torch.float64)
    out = torch.empty((sys.n_bands,) + tuple(sys.shape), dtype=torch.float64, device=f.device)
    _check(lib().sl_sheardec_threshold_dev(sys.handle, C.c_void_p(f.data_ptr()), C.c_void_p(out.data_ptr()),
                                           Kp, len(K), float(schedule.sigma), int(schedule.scale_by_filter_norm),
                                           _stream_ptr(f.device.index)))
    return out


def denoise(noisy, sys: _System, schedule: ThresholdSchedule, threads: int = 0, return_stack: bool = False):
    """inverse(hard_threshold(forward(noisy))) (apps.hpp:40-43, apps.cpp:114-121),
    fused on the device. return_stack=True (CUDA tensors) also returns the
    thresholded stack the fused pass wrote: (denoised, stack)."""
    _check_signal(noisy, sys, "forward")
    K, Kp = _k_arg(schedule)
    L = lib()
    if _is_f32(noisy):
        import torch
        noisy = noisy.contiguous()
        out = torch.empty_like(noisy)
        stack = torch.empty((sys.n_bands,) + tuple(sys.shape), dtype=torch.float32, device=noisy.device) \
            if return_stack else None
        _check(L.sl_denoise_f32_dev(sys.handle, C.c_void_p(noisy.data_ptr()),
                                    C.c_void_p(stack.data_ptr() if stack is not None else None),
                                    C.c_void_p(out.data_ptr()), Kp, len(K), float(schedule.sigma),
                                    int(schedule.scale_by_filter_norm), _stream_ptr(noisy.device.index)))
        return (out, stack) if return_stack else out
    if _is_cuda_tensor(noisy):
        import torch
        noisy = noisy.contiguous().to(torch.float64)
        out = torch.empty_like(noisy)
        args = (Kp, len(K), float(schedule.sigma), int(schedule.scale_by_filter_norm), _stream_ptr(noisy.device.index))
        if return_stack:
            stack = torch.empty((sys.n_bands,) + tuple(sys.shape), dtype=torch.float64, device=noisy.device)
            _check(L.sl_denoise_stack_dev(sys.handle, C.c_void_p(noisy.data_ptr()), C.c_void_p(stack.data_ptr()),
                                          C.c_void_p(out.data_ptr()), *args))
            return out, stack
        _check(L.sl_denoise_dev(sys.handle, C.c_void_p(noisy.data_ptr()), C.c_void_p(out.data_ptr()), *args))
        return out
    if return_stack:
        raise InvalidArgument("return_stack needs a CUDA tensor input")
    noisy = np.ascontiguousarray(noisy, dtype=np.float64)
    out = np.empty_like(noisy)
    _check(L.sl_denoise_host(sys.handle, _dp(noisy), _dp(out), Kp, len(K), float(schedule.sigma),
                             int(schedule.scale_by_filter_norm)))
    return out


def _check_batch(x, sys: _System):
    if x.ndim != sys.ndim + 1 or tuple(x.shape[1:]) != tuple(sys.shape):
        raise ShapeError("batch: expected [nframes, *dims] matching the system grid")


def forward_batch(frames, sys: _System, schedule: Optional[ThresholdSchedule] = None):
    """forward() (optionally + fused hard_threshold) of [nframes, *dims] CUDA frames -> [nframes, nb, *dims]."""
    _check_batch(frames, sys)
    import torch
    frames = frames.contiguous().to(torch.float64)
    out = torch.empty((frames.shape[0], sys.n_bands) + tuple(sys.shape), dtype=torch.float64, device=frames.device)
    if schedule is None:
        Kp, nK, sg, sc = None, 0, 0.0, 0
    else:
        K, Kp = _k_arg(schedule)
        nK, sg, sc = len(K), float(schedule.sigma), int(schedule.scale_by_filter_norm)
    _check(lib().sl_sheardec_batch_dev(sys.handle, C.c_void_p(frames.data_ptr()), int(frames.shape[0]),
                                       C.c_void_p(out.data_ptr()), Kp, nK, sg, sc, _stream_ptr(frames.device.index)))
    return out


def inverse_batch(coeffs, sys: _System):
    """inverse() of [nframes, nb, *dims] CUDA stacks -> [nframes, *dims]."""
    if coeffs.ndim != sys.ndim + 2 or coeffs.shape[1] != sys.n_bands or tuple(coeffs.shape[2:]) != tuple(sys.shape):
        raise ShapeError("inverse_batch: coefficient stacks do not match the system")
    import torch
    coeffs = coeffs.contiguous().to(torch.float64)
    out = torch.empty((coeffs.shape[0],) + tuple(sys.shape), dtype=torch.float64, device=coeffs.device)
    _check(lib().sl_shearrec_batch_dev(sys.handle, C.c_void_p(coeffs.data_ptr()), int(coeffs.shape[0]),
                                       C.c_void_p(out.data_ptr()), _stream_ptr(coeffs.device.index)))
    return out


def denoise_batch(frames, sys: _System, schedule: ThresholdSchedule, return_stacks: bool = False):
    """denoise() of [nframes, *dims] frames; CUDA tensors stay on the device, numpy
    arrays go through the host entry point (H2D + dec/thr/rec + D2H).
    return_stacks=True (CUDA) also returns the [nframes, nb, *dims] thresholded stacks."""
    _check_batch(frames, sys)
    K, Kp = _k_arg(schedule)
    args = (Kp, len(K), float(schedule.sigma), int(schedule.scale_by_filter_norm))
    if _is_f32(frames):
        import torch
        frames = frames.contiguous()
        out = torch.empty_like(frames)
        st = torch.empty((frames.shape[0], sys.n_bands) + tuple(sys.shape), dtype=torch.float32,
                         device=frames.device) if return_stacks else None
        _check(lib().sl_denoise_batch_f32_dev(sys.handle, C.c_void_p(frames.data_ptr()), int(frames.shape[0]),
                                              C.c_void_p(st.data_ptr() if st is not None else None),
                                              C.c_void_p(out.data_ptr()), *args, _stream_ptr(frames.device.index)))
        return (out, st) if return_stacks else out
    if _is_cuda_tensor(frames):
        import torch
        frames = frames.contiguous().to(torch.float64)
        out = torch.empty_like(frames)
        if return_stacks:
            st = torch.empty((frames.shape[0], sys.n_bands) + tuple(sys.shape), dtype=torch.float64,
                             device=frames.device)
            _check(lib().sl_denoise_batch_stack_dev(sys.handle, C.c_void_p(frames.data_ptr()), int(frames.shape[0]),
                                                    C.c_void_p(st.data_ptr()), C.c_void_p(out.data_ptr()), *args,
                                                    _stream_ptr(frames.device.index)))
            return out, st
        _check(lib().sl_denoise_batch_dev(sys.handle, C.c_void_p(frames.data_ptr()), int(frames.shape[0]),
                                          C.c_void_p(out.data_ptr()), *args, _stream_ptr(frames.device.index)))
        return out
    if return_stacks:
        raise InvalidArgument("return_stacks needs CUDA tensor frames")
    frames = np.ascontiguousarray(frames, dtype=np.float64)
    out = np.empty_like(frames)
    _check(lib().sl_denoise_batch_host(sys.handle, _dp(frames), int(frames.shape[0]), _dp(out), *args))
    return out


# ------------------------------------------------------------------ multi-GPU
def partition(count: int, nranks: int, rank: int):
    """[lo, hi) of `rank` in the balanced contiguous split the library uses."""
    lo, hi = C.c_int64(), C.c_int64()
    _check(lib().sl_partition(int(count), int(nranks), int(rank), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


class Comm:
    """NCCL communicator owned by the library (one process per GPU)."""

    def __init__(self, unique_id: bytes, nranks: int, rank: int, device: int):
        h = C.c_void_p()
        _check(lib().sl_comm_create(bytes(unique_id), int(nranks), int(rank), int(device), C.byref(h)))
        self.handle, self.nranks, self.rank, self.device = h, nranks, rank, device

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        _check(lib().sl_comm_unique_id(buf))
        return buf.raw

    def __del__(self):
        try:
            if self.handle:
                lib().sl_comm_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def denoise_dist(x, sys: _System, schedule: ThresholdSchedule, root: int = 0):
    """Sharded fused denoise across the ranks of sys's communicator: x (CUDA,
    read on the root, overwritten by the broadcast elsewhere) -> the full
    denoised signal on the root (an unspecified buffer elsewhere)."""
    import torch
    K, Kp = _k_arg(schedule)
    x = x.contiguous().to(torch.float64)
    out = torch.empty_like(x)
    _check(lib().sl_denoise_dist_dev(sys.handle, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()), Kp, len(K),
                                     float(schedule.sigma), int(schedule.scale_by_filter_norm), int(root),
                                     _stream_ptr(x.device.index)))
    return out


def denoise_batch_dist(frames, sys: _System, schedule: ThresholdSchedule, out=None):
    """This rank's share (partition(nframes, ...)) of a globally indexed batch;
    the other frames of `out` are left untouched. No collective."""
    _check_batch(frames, sys)
    K, Kp = _k_arg(schedule)
    args = (Kp, len(K), float(schedule.sigma), int(schedule.scale_by_filter_norm))
    if _is_cuda_tensor(frames):
        import torch
        frames = frames.contiguous().to(torch.float64)
        out = torch.zeros_like(frames) if out is None else out
        _check(lib().sl_denoise_batch_dist_dev(sys.handle, C.c_void_p(frames.data_ptr()), int(frames.shape[0]),
                                               C.c_void_p(out.data_ptr()), *args, _stream_ptr(frames.device.index)))
        return out
    frames = np.ascontiguousarray(frames, dtype=np.float64)
    out = np.zeros_like(frames) if out is None else out
    _check(lib().sl_denoise_batch_dist_host(sys.handle, _dp(frames), int(frames.shape[0]), _dp(out), *args))
    return out


# ------------------------------------------------------------------ SHCF files
def serialize(coeffs, sys: _System) -> bytes:
    """SHCF bytes of a coefficient stack (transform.hpp:45-46), identical to the reference."""
    c = np.ascontiguousarray(coeffs.cpu().numpy() if _is_cuda_tensor(coeffs) else coeffs, dtype=np.float64)
    if c.ndim != sys.ndim + 1 or tuple(c.shape[1:]) != tuple(sys.shape):
        raise ShapeError(f"serialize: stack shape {c.shape} does not match the system {sys.shape}")
    n = C.c_size_t()
    _check(lib().sl_shcf_size(sys.handle, int(c.shape[0]), C.byref(n)))
    buf = C.create_string_buffer(n.value)
    _check(lib().sl_shcf_serialize(sys.handle, _dp(c), int(c.shape[0]), buf, n.value))
    return buf.raw


def deserialize(data: bytes, sys: _System) -> np.ndarray:
    """Coefficient stack from SHCF bytes, validated against the system (transform.hpp:50-52)."""
    out = np.empty((sys.n_bands,) + tuple(sys.shape))
    _check(lib().sl_shcf_deserialize(sys.handle, data, len(data), _dp(out), sys.n_bands))
    return out


def forward_to_file(f, sys: _System, path: str, bands_per_chunk: int = 0):
    """forward(f) written straight to an SHCF file, a chunk of bands at a time (the
    stack is never held whole); same bytes as serialize(forward(f), sys)."""
    x = np.ascontiguousarray(f.cpu().numpy() if _is_cuda_tensor(f) else f, dtype=np.float64)
    _check_signal(x, sys, "forward")
    _check(lib().sl_shcf_forward_file(sys.handle, _dp(x), os.fsencode(path), int(bands_per_chunk)))


def inverse_from_file(path: str, sys: _System, bands_per_chunk: int = 0) -> np.ndarray:
    """inverse() of an SHCF file, streamed a chunk of bands at a time."""
    out = np.empty(tuple(sys.shape))
    _check(lib().sl_shcf_inverse_file(sys.handle, os.fsencode(path), _dp(out), int(bands_per_chunk)))
    return out


# ------------------------------------------------------------------ signal files
@dataclass
class PgmImage:
    """image_io.hpp:9-15: pixels [rows][cols] (axis 0 = image rows), maxval."""
    pixels: np.ndarray
    maxval: int = 255


def load_pgm(path: str) -> PgmImage:
    """load_pgm (image_io.cpp:43-75): binary P5, 8- or 16-bit."""
    r, c, m = C.c_int(), C.c_int(), C.c_int()
    b = os.fsencode(path)
    _check(lib().sl_load_pgm(b, None, 0, C.byref(r), C.byref(c), C.byref(m)))
    px = np.empty((r.value, c.value))
    _check(lib().sl_load_pgm(b, _dp(px), px.size, None, None, None))
    return PgmImage(px, m.value)


def save_pgm(pixels, path: str, maxval: int = 255):
    """save_pgm (image_io.cpp:77-100): rounds and clamps to [0, maxval]."""
    px = np.ascontiguousarray(pixels, dtype=np.float64)
    if px.ndim != 2:
        raise ShapeError("save_pgm: pixels must be 2D")
    _check(lib().sl_save_pgm(_dp(px), px.shape[0], px.shape[1], os.fsencode(path), int(maxval)))


def load_svol(path: str) -> np.ndarray:
    """load_svol (image_io.cpp:125-143)."""
    d = (C.c_int64 * 3)()
    b = os.fsencode(path)
    _check(lib().sl_load_svol(b, None, 0, d))
    v = np.empty(tuple(d))
    _check(lib().sl_load_svol(b, _dp(v), v.size, d))
    return v


def save_svol(volume, path: str):
    """save_svol (image_io.cpp:145-159)."""
    v = np.ascontiguousarray(volume, dtype=np.float64)
    if v.ndim != 3:
        raise ShapeError("save_svol: volume must be 3D")
    _check(lib().sl_save_svol(_dp(v), (C.c_int64 * 3)(*v.shape), os.fsencode(path)))


# ------------------------------------------------------------------ quality metrics
def gaussian_kernel(sigma_pixels: float = 2.0) -> "FanFilter":
    """gaussian_kernel (apps.cpp:289-306): L1-normalised taps, radius ceil(4 sigma); returned as
    Taps2d-like (taps, center0, center1)."""
    n, c = C.c_int(), C.c_int()
    _check(lib().sl_gaussian_kernel(float(sigma_pixels), None, 0, C.byref(n), C.byref(c)))
    t = np.empty((n.value, n.value))
    _check(lib().sl_gaussian_kernel(float(sigma_pixels), _dp(t), t.size, None, None))
    return FanFilter(t, c.value, c.value, f"gaussian{sigma_pixels}")


def binarize(signal, delta: float) -> np.ndarray:
    """binarize (apps.cpp:282-287): 1 where |g| >= delta, else 0."""
    x = np.ascontiguousarray(signal, dtype=np.float64)
    out = np.empty_like(x)
    _check(lib().sl_binarize(_dp(x), _dp(out), x.size, float(delta)))
    return out


def _quality_args(recovered, truth, gaussian):
    r = np.ascontiguousarray(recovered, dtype=np.float64)
    t = np.ascontiguousarray(truth, dtype=np.float64)
    if r.shape != t.shape or r.ndim != 2:
        raise ShapeError("quality_q: dimension mismatch")
    g = gaussian_kernel(2.0) if gaussian is None else gaussian
    k = np.ascontiguousarray(g.taps, dtype=np.float64)
    return r, t, k, g


def quality_q(recovered, truth, delta: float, gaussian=None, device: int = 0) -> float:
    """quality_q (apps.cpp:309-326); the blurs run on the GPU."""
    r, t, k, g = _quality_args(recovered, truth, gaussian)
    q = C.c_double()
    _check(lib().sl_quality_q(r.shape[0], r.shape[1], _dp(r), _dp(t), float(delta), _dp(k), k.shape[0], k.shape[1],
                              int(g.center0), int(g.center1), int(device), C.byref(q)))
    return q.value


def quality_q_opt(recovered, truth, gaussian=None, device: int = 0, return_all: bool = False):
    """quality_q_opt (apps.cpp:328-360): (min Q over delta = 0..255, argmin); 256 blurs batched on the GPU."""
    r, t, k, g = _quality_args(recovered, truth, gaussian)
    q, d = C.c_double(), C.c_int()
    allq = np.empty(256)
    _check(lib().sl_quality_q_opt(r.shape[0], r.shape[1], _dp(r), _dp(t), _dp(k), k.shape[0], k.shape[1],
                                  int(g.center0), int(g.center1), int(device), C.byref(q), C.byref(d), _dp(allq)))
    return (q.value, d.value, allq) if return_all else (q.value, d.value)


# ------------------------------------------------------------------ iterative pipelines
@dataclass
class InpaintConfig:
    """apps.hpp:46-51."""
    iterations: int = 100
    delta_init: float = -1.0   # < 0: largest (RMS-scaled) coefficient of the input
    delta_min: float = 0.01
    scale_by_filter_norm: bool = True


def inpaint(masked_signal, mask, sys: _System, config: InpaintConfig = InpaintConfig(), threads: int = 0):
    """Iterative-thresholding inpainting (apps.hpp:59-76, apps.cpp:179-235); the loop runs on the GPU."""
    if tuple(mask.shape) != tuple(masked_signal.shape):
        raise ShapeError("inpaint: mask dims must match the signal")
    _check_signal(masked_signal, sys, "inpaint")
    args = (int(config.iterations), float(config.delta_init), float(config.delta_min),
            int(config.scale_by_filter_norm))
    L = lib()
    if _is_cuda_tensor(masked_signal):
        import torch
        x = masked_signal.contiguous().to(torch.float64)
        m = mask.contiguous().to(torch.float64)
        out = torch.empty_like(x)
        _check(L.sl_inpaint_dev(sys.handle, C.c_void_p(x.data_ptr()), C.c_void_p(m.data_ptr()),
                                C.c_void_p(out.data_ptr()), *args, _stream_ptr(x.device.index)))
        return out
    x = np.ascontiguousarray(masked_signal, dtype=np.float64)
    m = np.ascontiguousarray(mask, dtype=np.float64)
    out = np.empty_like(x)
    _check(L.sl_inpaint_host(sys.handle, _dp(x), _dp(m), _dp(out), *args))
    return out


@dataclass
class SeparationResult:
    """apps.hpp:78-81."""
    curvilinear: object
    blobs: object


def separate(signal, directional: ShearletSystem2D, isotropic: ShearletSystem2D,
             config: InpaintConfig = InpaintConfig(), threads: int = 0) -> SeparationResult:
    """Joint iterative thresholding over two systems (apps.hpp:83-90, apps.cpp:237-280)."""
    if tuple(signal.shape) != tuple(directional.shape) or tuple(signal.shape) != tuple(isotropic.shape):
        raise ShapeError("separate: both systems must match the signal dims")
    args = (int(config.iterations), float(config.delta_init), float(config.delta_min),
            int(config.scale_by_filter_norm))
    L = lib()
    if _is_cuda_tensor(signal):
        import torch
        x = signal.contiguous().to(torch.float64)
        c, b = torch.empty_like(x), torch.empty_like(x)
        _check(L.sl_separate_dev(directional.handle, isotropic.handle, C.c_void_p(x.data_ptr()),
                                 C.c_void_p(c.data_ptr()), C.c_void_p(b.data_ptr()), *args,
                                 _stream_ptr(x.device.index)))
        return SeparationResult(c, b)
    x = np.ascontiguousarray(signal, dtype=np.float64)
    c, b = np.empty_like(x), np.empty_like(x)
    _check(L.sl_separate_host(directional.handle, isotropic.handle, _dp(x), _dp(c), _dp(b), *args))
    return SeparationResult(c, b)


# ------------------------------------------------------------------ inputs
def cartoon(n: int) -> np.ndarray:
    """phantoms::cartoon (phantoms.cpp:14-36)."""
    out = np.empty((n, n))
    _check(lib().sl_phantom_cartoon(int(n), _dp(out)))
    return out


def cartoon_volume(n: int) -> np.ndarray:
    """phantoms::cartoon_volume (phantoms.cpp:91-108)."""
    out = np.empty((n, n, n))
    _check(lib().sl_phantom_cartoon_volume(int(n), _dp(out)))
    return out


def add_gaussian_noise(x: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """add_gaussian_noise (apps.cpp:47-55): mt19937_64 + Box-Muller."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _check(lib().sl_add_gaussian_noise(_dp(x), _dp(out), x.size, float(sigma), int(seed)))
    return out


def psnr(reference: np.ndarray, test: np.ndarray) -> float:
    """20 log10(255 sqrt(N) / ||ref - test||) (apps.cpp:125-135)."""
    if reference.shape != test.shape:
        raise ShapeError("psnr: dimension mismatch")
    e2 = float(np.sum((reference - test) ** 2))
    if e2 == 0.0:
        return float("inf")
    return 20.0 * np.log10(255.0 * np.sqrt(reference.size) / np.sqrt(e2))
