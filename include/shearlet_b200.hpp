// shearlet_b200.hpp -- header-only C++ host API over the C ABI.
//
// Mirrors the reference's C++ interface for the hot path
// (/root/reference/proj/core/include/shearlet/{system2d,system3d,transform,apps,errors}.hpp):
// same function names and argument meaning, the same exception hierarchy, and
// value semantics on host containers. Signals are row-major std::vector<double>
// (axis 0 slowest), stacks are contiguous [R][dims...].
#pragma once

#include <array>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "shearlet_b200.h"

namespace shearlet_b200 {

// errors.hpp:9-56
struct Error : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : Error { using Error::Error; };
struct ShapeError : Error { using Error::Error; };
struct ConfigError : Error { using Error::Error; };
struct AssetError : Error { using Error::Error; };
struct FormatError : Error { using Error::Error; };
struct SingularFrameError : Error { using Error::Error; };
struct UnsupportedSizeError : Error { using Error::Error; };
struct DegenerateMaskError : Error { using Error::Error; };
struct DegenerateTruthError : Error { using Error::Error; };
struct CudaError : Error { using Error::Error; };
struct NcclError : Error { using Error::Error; };

inline void check(int rc) {
    if (rc == SL_OK) return;
    const std::string m = sl_last_error();
    switch (rc) {
        case SL_ERR_SHAPE: throw ShapeError(m);
        case SL_ERR_CONFIG: throw ConfigError(m);
        case SL_ERR_DOMAIN: throw DomainError(m);
        case SL_ERR_SINGULAR_FRAME: throw SingularFrameError(m);
        case SL_ERR_UNSUPPORTED_SIZE: throw UnsupportedSizeError(m);
        case SL_ERR_ASSET: throw AssetError(m);
        case SL_ERR_FORMAT: throw FormatError(m);
        case SL_ERR_DEGENERATE_MASK: throw DegenerateMaskError(m);
        case SL_ERR_DEGENERATE_TRUTH: throw DegenerateTruthError(m);
        case SL_ERR_CUDA: throw CudaError(m);
        case SL_ERR_NCCL: throw NcclError(m);
        default: throw Error(m);
    }
}

// ScaleProfile::from_levels (filters.hpp:79-92)
struct ScaleProfile {
    std::vector<int> shear_levels;
    int coarsest_scale_offset = 0;
    static ScaleProfile from_levels(std::vector<int> levels, int j0 = 0) { return {std::move(levels), j0}; }
    int n_scales() const { return static_cast<int>(shear_levels.size()); }
};

// ThresholdSchedule (apps.hpp:19-29)
struct ThresholdSchedule {
    std::vector<double> per_scale_factors;
    double sigma = 0.0;
    bool scale_by_filter_norm = true;
    static ThresholdSchedule defaults_2d(double sigma, int n_scales = 4) {
        std::vector<double> k(static_cast<size_t>(n_scales), 2.5);
        if (n_scales > 0) k.back() = 3.8;
        return {k, sigma, true};
    }
    static ThresholdSchedule defaults_3d(double sigma, int n_scales = 3) {
        std::vector<double> k(static_cast<size_t>(n_scales), 3.0);
        if (n_scales > 0) k.back() = 4.0;
        return {k, sigma, true};
    }
};

struct FilterIndex {  // kind, scale, k1 (2D shear), k2
    int kind, scale, k1, k2;
};

// ShearletSystem2D / 3D: owns the device-resident filter bank.
class ShearletSystem {
  public:
    explicit ShearletSystem(sl_system* h) : h_(h, &sl_system_destroy) {
        int nd = 0;
        int64_t d[3];
        check(sl_ndim(h, &nd, d));
        ndim_ = nd;
        for (int a = 0; a < 3; ++a) dims_[static_cast<size_t>(a)] = static_cast<size_t>(d[a]);
        int R = 0, lo = 0, hi = 0;
        check(sl_redundancy(h, &R));
        check(sl_shard(h, &lo, &hi));
        R_ = R;
        nb_ = hi - lo;
        std::vector<int32_t> rec(static_cast<size_t>(4 * R));
        check(sl_index(h, rec.data()));
        for (int i = 0; i < R; ++i)
            index.push_back({rec[4 * i], rec[4 * i + 1], rec[4 * i + 2], rec[4 * i + 3]});
        filter_norms.resize(static_cast<size_t>(R));
        check(sl_filter_norms(h, filter_norms.data()));
    }
    sl_system* handle() const { return h_.get(); }
    std::size_t redundancy() const { return static_cast<std::size_t>(R_); }
    std::size_t n_bands() const { return static_cast<std::size_t>(nb_); }
    std::size_t size() const { return ndim_ == 2 ? dims_[0] * dims_[1] : dims_[0] * dims_[1] * dims_[2]; }
    int ndim() const { return ndim_; }
    /// optional fp32 mode (2D fast-path grids): prepares the float tables
    void set_precision(int bits) const { check(sl_system_set_precision(h_.get(), bits)); }
    std::pair<double, double> frame_bounds() const {
        double a, b;
        check(sl_frame_bounds(h_.get(), &a, &b));
        return {a, b};
    }
    std::vector<double> frame_weight() const {
        std::vector<double> w(size());
        check(sl_frame_weight(h_.get(), w.data()));
        return w;
    }
    std::vector<FilterIndex> index;
    std::vector<double> filter_norms;  // RMS

  private:
    std::unique_ptr<sl_system, int (*)(sl_system*)> h_;
    int ndim_ = 0, R_ = 0, nb_ = 0;
    std::array<std::size_t, 3> dims_{1, 1, 1};
};

// build_system_2d / build_system_3d (system2d.hpp:66-69, system3d.hpp:68-71)
inline ShearletSystem build_system_2d(std::size_t rows, std::size_t cols, const ScaleProfile& p,
                                      bool impulse_fan = false, bool full_system = false, int device = 0) {
    sl_system* h = nullptr;
    check(sl_system_create_2d(static_cast<int>(rows), static_cast<int>(cols), p.shear_levels.data(), p.n_scales(),
                              p.coarsest_scale_offset, full_system, impulse_fan, device, 0, -1, &h));
    return ShearletSystem(h);
}
inline ShearletSystem build_system_3d(std::array<std::size_t, 3> d, const ScaleProfile& p, bool impulse_fan = false,
                                      bool full_system = false, int device = 0) {
    sl_system* h = nullptr;
    check(sl_system_create_3d(static_cast<int>(d[0]), static_cast<int>(d[1]), static_cast<int>(d[2]),
                              p.shear_levels.data(), p.n_scales(), p.coarsest_scale_offset, full_system, impulse_fan,
                              device, 0, -1, &h));
    return ShearletSystem(h);
}

// Explicit filter bank (filters.hpp:14-67): 1D QMF taps and a 2D fan, each with a centre.
struct Taps1d {
    std::vector<double> v;
    int center = 0;
};
struct QmfPair {
    Taps1d lowpass, highpass;  // highpass empty = mirror_highpass(lowpass)
    static QmfPair from_lowpass(Taps1d low) { return QmfPair{std::move(low), {}}; }
};
struct FanFilter {
    std::vector<double> taps;  // row-major rows x cols
    int rows = 0, cols = 0, center0 = 0, center1 = 0;
    std::string provenance = "custom";
    static FanFilter impulse() { return FanFilter{{1.0}, 1, 1, 0, 0, "impulse"}; }
    static FanFilter default_fan() {  // default_fan_filter(), the bundled dmaxflat4 constant
        FanFilter f;
        check(sl_default_fan(nullptr, 0, &f.rows, &f.cols, &f.center0, &f.center1));
        f.taps.resize(static_cast<std::size_t>(f.rows) * f.cols);
        check(sl_default_fan(f.taps.data(), static_cast<int64_t>(f.taps.size()), nullptr, nullptr, nullptr, nullptr));
        f.provenance = "dmaxflat4";
        return f;
    }
};
inline ShearletSystem build_system_2d(std::size_t rows, std::size_t cols, const ScaleProfile& p, const FanFilter& fan,
                                      const QmfPair& qmf, bool full_system = false, int device = 0) {
    sl_system* h = nullptr;
    const bool hp = !qmf.highpass.v.empty();
    check(sl_system_create_2d_ex(
        static_cast<int>(rows), static_cast<int>(cols), p.shear_levels.data(), p.n_scales(), p.coarsest_scale_offset,
        full_system, qmf.lowpass.v.empty() ? nullptr : qmf.lowpass.v.data(), static_cast<int>(qmf.lowpass.v.size()), qmf.lowpass.center,
        hp ? qmf.highpass.v.data() : nullptr, static_cast<int>(qmf.highpass.v.size()), qmf.highpass.center,
        fan.taps.empty() ? nullptr : fan.taps.data(), fan.rows, fan.cols, fan.center0, fan.center1,
        fan.provenance.c_str(), device, 0, -1, &h));
    return ShearletSystem(h);
}
inline ShearletSystem build_system_3d(std::array<std::size_t, 3> d, const ScaleProfile& p, const FanFilter& fan,
                                      const QmfPair& qmf, bool full_system = false, int device = 0) {
    sl_system* h = nullptr;
    const bool hp = !qmf.highpass.v.empty();
    check(sl_system_create_3d_ex(
        static_cast<int>(d[0]), static_cast<int>(d[1]), static_cast<int>(d[2]), p.shear_levels.data(), p.n_scales(),
        p.coarsest_scale_offset, full_system, qmf.lowpass.v.empty() ? nullptr : qmf.lowpass.v.data(), static_cast<int>(qmf.lowpass.v.size()),
        qmf.lowpass.center, hp ? qmf.highpass.v.data() : nullptr, static_cast<int>(qmf.highpass.v.size()),
        qmf.highpass.center, fan.taps.empty() ? nullptr : fan.taps.data(), fan.rows, fan.cols, fan.center0, fan.center1,
        fan.provenance.c_str(), device, 0, -1, &h));
    return ShearletSystem(h);
}

// forward / inverse (transform.hpp:27-37), value semantics
inline std::vector<double> forward(const std::vector<double>& f, const ShearletSystem& s) {
    if (f.size() != s.size()) throw ShapeError("forward: signal dims do not match the system grid");
    std::vector<double> c(s.n_bands() * s.size());
    check(sl_sheardec_host(s.handle(), f.data(), c.data()));
    return c;
}
inline std::vector<double> inverse(const std::vector<double>& coeffs, const ShearletSystem& s) {
    if (coeffs.size() != s.n_bands() * s.size())
        throw ShapeError("inverse: coefficient stack does not match the system");
    std::vector<double> f(s.size());
    check(sl_shearrec_host(s.handle(), coeffs.data(), static_cast<int>(s.n_bands()), f.data()));
    return f;
}
// hard_threshold / denoise (apps.hpp:31-44)
inline std::vector<double> hard_threshold(const std::vector<double>& coeffs, const ThresholdSchedule& sch,
                                          const ShearletSystem& s) {
    std::vector<double> out(coeffs.size());
    check(sl_hard_threshold_host(s.handle(), coeffs.data(), out.data(),
                                 static_cast<int>(coeffs.size() / std::max<std::size_t>(1, s.size())),
                                 sch.per_scale_factors.data(), static_cast<int>(sch.per_scale_factors.size()),
                                 sch.sigma, sch.scale_by_filter_norm));
    return out;
}
inline std::vector<double> denoise(const std::vector<double>& noisy, const ShearletSystem& s,
                                   const ThresholdSchedule& sch) {
    if (noisy.size() != s.size()) throw ShapeError("forward: signal dims do not match the system grid");
    std::vector<double> out(s.size());
    check(sl_denoise_host(s.handle(), noisy.data(), out.data(), sch.per_scale_factors.data(),
                          static_cast<int>(sch.per_scale_factors.size()), sch.sigma, sch.scale_by_filter_norm));
    return out;
}

// Iterative thresholding (apps.hpp:46-90): the whole loop runs on the device
struct InpaintConfig {
    int iterations = 100;
    double delta_init = -1.0;  // < 0: the largest (RMS-scaled) coefficient of the input
    double delta_min = 0.01;
    bool scale_by_filter_norm = true;
};
inline std::vector<double> inpaint(const std::vector<double>& masked, const std::vector<double>& mask,
                                   const ShearletSystem& s, const InpaintConfig& c = InpaintConfig()) {
    if (masked.size() != s.size() || mask.size() != s.size()) throw ShapeError("inpaint: dims do not match the system");
    std::vector<double> out(s.size());
    check(sl_inpaint_host(s.handle(), masked.data(), mask.data(), out.data(), c.iterations, c.delta_init, c.delta_min,
                          c.scale_by_filter_norm));
    return out;
}
struct SeparationResult {
    std::vector<double> curvilinear, blobs;
};
inline SeparationResult separate(const std::vector<double>& signal, const ShearletSystem& directional,
                                 const ShearletSystem& isotropic, const InpaintConfig& c = InpaintConfig()) {
    if (signal.size() != directional.size()) throw ShapeError("separate: dims do not match the system");
    SeparationResult r{std::vector<double>(signal.size()), std::vector<double>(signal.size())};
    check(sl_separate_host(directional.handle(), isotropic.handle(), signal.data(), r.curvilinear.data(),
                           r.blobs.data(), c.iterations, c.delta_init, c.delta_min, c.scale_by_filter_norm));
    return r;
}

// SHCF coefficient files (transform.hpp:39-52): bytes of serialize() / deserialize_2d/3d
inline std::vector<unsigned char> serialize(const std::vector<double>& coeffs, const ShearletSystem& s) {
    if (coeffs.size() != s.n_bands() * s.size()) throw ShapeError("serialize: stack does not match the system");
    std::size_t n = 0;
    check(sl_shcf_size(s.handle(), static_cast<int>(s.n_bands()), &n));
    std::vector<unsigned char> out(n);
    check(sl_shcf_serialize(s.handle(), coeffs.data(), static_cast<int>(s.n_bands()), out.data(), n));
    return out;
}
inline std::vector<double> deserialize(const std::vector<unsigned char>& bytes, const ShearletSystem& s) {
    std::vector<double> c(s.n_bands() * s.size());
    check(sl_shcf_deserialize(s.handle(), bytes.data(), bytes.size(), c.data(), static_cast<int>(s.n_bands())));
    return c;
}

// Streamed SHCF files: decompose to / reconstruct from a file a chunk of bands at a time
inline void forward_to_file(const std::vector<double>& f, const ShearletSystem& s, const std::string& path,
                            int bands_per_chunk = 0) {
    if (f.size() != s.size()) throw ShapeError("forward: signal dims do not match the system grid");
    check(sl_shcf_forward_file(s.handle(), f.data(), path.c_str(), bands_per_chunk));
}
inline std::vector<double> inverse_from_file(const std::string& path, const ShearletSystem& s,
                                             int bands_per_chunk = 0) {
    std::vector<double> out(s.size());
    check(sl_shcf_inverse_file(s.handle(), path.c_str(), out.data(), bands_per_chunk));
    return out;
}

// System descriptors (descriptor.hpp:12-39): write_descriptor(describe(s)) text, rebuild from text
inline std::string describe(const ShearletSystem& s) {
    std::size_t n = 0;
    check(sl_describe(s.handle(), nullptr, 0, &n));
    std::string t(n + 1, '\0');
    check(sl_describe(s.handle(), t.data(), t.size(), &n));
    t.resize(n);
    return t;
}
inline ShearletSystem build_from_descriptor(const std::string& text, int device = 0) {
    sl_system* h = nullptr;
    check(sl_system_create_from_descriptor(text.c_str(), 0, device, 0, -1, &h));
    return ShearletSystem(h);
}

// Signal files (image_io.hpp:9-24)
struct PgmImage {
    std::vector<double> pixels;  // rows x cols, axis 0 = image rows
    int rows = 0, cols = 0, maxval = 255;
};
inline PgmImage load_pgm(const std::string& path) {
    PgmImage im;
    check(sl_load_pgm(path.c_str(), nullptr, 0, &im.rows, &im.cols, &im.maxval));
    im.pixels.resize(static_cast<std::size_t>(im.rows) * im.cols);
    check(sl_load_pgm(path.c_str(), im.pixels.data(), static_cast<int64_t>(im.pixels.size()), nullptr, nullptr,
                      nullptr));
    return im;
}
inline void save_pgm(const std::vector<double>& pixels, int rows, int cols, const std::string& path,
                     int maxval = 255) {
    if (pixels.size() != static_cast<std::size_t>(rows) * cols) throw ShapeError("save_pgm: pixel count");
    check(sl_save_pgm(pixels.data(), rows, cols, path.c_str(), maxval));
}
inline std::vector<double> load_svol(const std::string& path, std::array<std::size_t, 3>* dims) {
    int64_t d[3] = {0, 0, 0};
    check(sl_load_svol(path.c_str(), nullptr, 0, d));
    std::vector<double> v(static_cast<std::size_t>(d[0] * d[1] * d[2]));
    check(sl_load_svol(path.c_str(), v.data(), static_cast<int64_t>(v.size()), d));
    if (dims) *dims = {static_cast<std::size_t>(d[0]), static_cast<std::size_t>(d[1]), static_cast<std::size_t>(d[2])};
    return v;
}
inline void save_svol(const std::vector<double>& v, std::array<std::size_t, 3> dims, const std::string& path) {
    if (v.size() != dims[0] * dims[1] * dims[2]) throw ShapeError("save_svol: sample count");
    const int64_t d[3] = {static_cast<int64_t>(dims[0]), static_cast<int64_t>(dims[1]), static_cast<int64_t>(dims[2])};
    check(sl_save_svol(v.data(), d, path.c_str()));
}

// Separation quality (apps.hpp:86-101): Gaussian taps (size x size, centre) and Q / Q_opt
struct GaussianKernel {
    std::vector<double> taps;
    int size = 0, center = 0;
};
inline GaussianKernel gaussian_kernel(double sigma_pixels = 2.0) {
    GaussianKernel g;
    check(sl_gaussian_kernel(sigma_pixels, nullptr, 0, &g.size, &g.center));
    g.taps.resize(static_cast<std::size_t>(g.size) * g.size);
    check(sl_gaussian_kernel(sigma_pixels, g.taps.data(), static_cast<int64_t>(g.taps.size()), nullptr, nullptr));
    return g;
}
inline double quality_q(const std::vector<double>& recovered, const std::vector<double>& truth, int rows, int cols,
                        double delta, const GaussianKernel& g, int device = 0) {
    if (recovered.size() != truth.size() || recovered.size() != static_cast<std::size_t>(rows) * cols)
        throw ShapeError("quality_q: dimension mismatch");
    double q = 0.0;
    check(sl_quality_q(rows, cols, recovered.data(), truth.data(), delta, g.taps.data(), g.size, g.size, g.center,
                       g.center, device, &q));
    return q;
}
inline std::pair<double, int> quality_q_opt(const std::vector<double>& recovered, const std::vector<double>& truth,
                                            int rows, int cols, const GaussianKernel& g, int device = 0) {
    if (recovered.size() != truth.size() || recovered.size() != static_cast<std::size_t>(rows) * cols)
        throw ShapeError("quality_q_opt: dimension mismatch");
    double q = 0.0;
    int d = 0;
    check(sl_quality_q_opt(rows, cols, recovered.data(), truth.data(), g.taps.data(), g.size, g.size, g.center,
                           g.center, device, &q, &d, nullptr));
    return {q, d};
}

// ---- fused denoise returning the thresholded stack (host value semantics over
// a device round trip is the _host entry points' job; this one takes device
// pointers, as a caller already holding device buffers would)
inline void denoise_with_stack_dev(const ShearletSystem& s, const double* d_in, double* d_stack, double* d_out,
                                   const ThresholdSchedule& sch, void* stream = nullptr) {
    check(sl_denoise_stack_dev(s.handle(), d_in, d_stack, d_out, sch.per_scale_factors.data(),
                               static_cast<int>(sch.per_scale_factors.size()), sch.sigma,
                               sch.scale_by_filter_norm ? 1 : 0, stream));
}

// ---- multi-GPU: one process per GPU, the library's own NCCL communicator
class Comm {
  public:
    static std::vector<unsigned char> unique_id() {
        std::vector<unsigned char> id(128);
        check(sl_comm_unique_id(id.data()));
        return id;
    }
    Comm(const std::vector<unsigned char>& id, int nranks, int rank, int device) : c_(nullptr, &sl_comm_destroy) {
        if (id.size() != 128) throw ConfigError("Comm: the NCCL unique id has 128 bytes");
        sl_comm* c = nullptr;
        check(sl_comm_create(id.data(), nranks, rank, device, &c));
        c_.reset(c);
    }
    sl_comm* handle() const { return c_.get(); }

  private:
    std::unique_ptr<sl_comm, int (*)(sl_comm*)> c_;
};
/// attach (shard_bands: 3D / single frames) or detach (comm = nullptr)
inline void set_comm(const ShearletSystem& s, const Comm* comm, bool shard_bands = true) {
    check(sl_system_set_comm(s.handle(), comm ? comm->handle() : nullptr, shard_bands ? 1 : 0));
}
/// sharded fused denoise; d_in read on the root, d_out written on the root
inline void denoise_dist_dev(const ShearletSystem& s, const double* d_in, double* d_out, const ThresholdSchedule& sch,
                             int root = 0, void* stream = nullptr) {
    check(sl_denoise_dist_dev(s.handle(), d_in, d_out, sch.per_scale_factors.data(),
                              static_cast<int>(sch.per_scale_factors.size()), sch.sigma,
                              sch.scale_by_filter_norm ? 1 : 0, root, stream));
}

}  // namespace shearlet_b200
