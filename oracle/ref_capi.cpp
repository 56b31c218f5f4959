// oracle/ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A flat C wrapper over the UNMODIFIED reference library, compiled from
// /root/reference/proj/core/src/*.cpp by oracle/Makefile into
// oracle/_ref/libshearlet_ref.so. It exists so Python tests, the golden
// generator (oracle/gen_golden.py) and bench.py's cpu_baseline leg can drive
// the reference's own public API (system2d.hpp:66-69, system3d.hpp:68-71,
// transform.hpp:27-37, apps.hpp:16-44) through ctypes. Only the call
// plumbing lives here; every number comes from the reference code.
#include <cstdint>
#include <cmath>
#include <cstring>
#include <exception>
#include <sstream>
#include <string>
#include <vector>

#include "shearlet/apps.hpp"
#include "shearlet/descriptor.hpp"
#include "shearlet/fft.hpp"
#include "shearlet/image_io.hpp"
#include "shearlet/phantoms.hpp"
#include "shearlet/system2d.hpp"
#include "shearlet/system3d.hpp"
#include "shearlet/transform.hpp"

using namespace shearlet;

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ShapeError& e) { g_err = e.what(); return 2; }
    catch (const ConfigError& e) { g_err = e.what(); return 3; }
    catch (const DomainError& e) { g_err = e.what(); return 4; }
    catch (const SingularFrameError& e) { g_err = e.what(); return 5; }
    catch (const UnsupportedSizeError& e) { g_err = e.what(); return 6; }
    catch (const AssetError& e) { g_err = e.what(); return 7; }
    catch (const FormatError& e) { g_err = e.what(); return 8; }
    catch (const DegenerateMaskError& e) { g_err = e.what(); return 9; }
    catch (const DegenerateTruthError& e) { g_err = e.what(); return 10; }
    catch (const Error& e) { g_err = e.what(); return 1; }
    catch (const std::exception& e) { g_err = e.what(); return 99; }
}

const QmfPair& qmf() {
    static const QmfPair q = QmfPair::maximally_flat_9tap();
    return q;
}
FanFilter fan_for(int impulse_fan) {
    return impulse_fan ? FanFilter::impulse() : default_fan_filter();
}
QmfPair qmf_of(const double* lp, int lpn, int lpc, const double* hp, int hpn, int hpc) {
    if (!lp) return qmf();
    QmfPair q = QmfPair::from_lowpass(Taps1d{std::vector<double>(lp, lp + lpn), lpc});
    if (hp) q.highpass = Taps1d{std::vector<double>(hp, hp + hpn), hpc};
    return q;
}
FanFilter fan_of(const double* f, int fr, int fc, int fc0, int fc1) {
    if (!f) return default_fan_filter();
    Taps2d t;
    t.v = RealGrid2(static_cast<std::size_t>(fr), static_cast<std::size_t>(fc));
    std::memcpy(t.v.data(), f, sizeof(double) * static_cast<std::size_t>(fr * fc));
    t.center0 = fc0;
    t.center1 = fc1;
    return FanFilter{t, "custom"};
}
ScaleProfile profile_of(const int* levels, int n, int j0) {
    return ScaleProfile::from_levels(std::vector<int>(levels, levels + n), j0);
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ---------------------------------------------------------------- 2D
int ref_build_2d(int rows, int cols, const int* levels, int n_scales, int j0, int full,
                 int impulse_fan, int threads, void** out) {
    return guard([&] {
        auto* s = new ShearletSystem2D(build_system_2d(
            static_cast<std::size_t>(rows), static_cast<std::size_t>(cols),
            profile_of(levels, n_scales, j0), fan_for(impulse_fan), qmf(), full != 0, threads));
        *out = s;
    });
}
// build_system_2d/3d with an explicit FanFilter + QmfPair (system2d.hpp:66-69)
int ref_build_2d_bank(int rows, int cols, const int* levels, int n_scales, int j0, int full, const double* lp, int lpn,
                      int lpc, const double* hp, int hpn, int hpc, const double* fan, int fr, int fc, int fc0, int fc1,
                      int threads, void** out) {
    return guard([&] {
        auto* s = new ShearletSystem2D(build_system_2d(
            static_cast<std::size_t>(rows), static_cast<std::size_t>(cols), profile_of(levels, n_scales, j0),
            fan_of(fan, fr, fc, fc0, fc1), qmf_of(lp, lpn, lpc, hp, hpn, hpc), full != 0, threads));
        *out = s;
    });
}
int ref_build_3d_bank(int n0, int n1, int n2, const int* levels, int n_scales, int j0, int full, const double* lp,
                      int lpn, int lpc, const double* hp, int hpn, int hpc, const double* fan, int fr, int fc, int fc0,
                      int fc1, int threads, void** out) {
    return guard([&] {
        auto* s = new ShearletSystem3D(build_system_3d(
            {static_cast<std::size_t>(n0), static_cast<std::size_t>(n1), static_cast<std::size_t>(n2)},
            profile_of(levels, n_scales, j0), fan_of(fan, fr, fc, fc0, fc1), qmf_of(lp, lpn, lpc, hp, hpn, hpc),
            full != 0, threads));
        *out = s;
    });
}
// fan_design::maxflat_fan(order) -> taps (cap doubles), dims and centres
int ref_maxflat_fan(int order, double* out, long long cap, int* dims) {
    return guard([&] {
        const Taps2d t = fan_design::maxflat_fan(order);
        dims[0] = static_cast<int>(t.size0());
        dims[1] = static_cast<int>(t.size1());
        dims[2] = static_cast<int>(t.center0);
        dims[3] = static_cast<int>(t.center1);
        if (out && cap >= static_cast<long long>(t.size0() * t.size1()))
            std::memcpy(out, t.v.data(), sizeof(double) * t.size0() * t.size1());
    });
}

void ref_free_2d(void* h) { delete static_cast<ShearletSystem2D*>(h); }
int ref_redundancy_2d(void* h) { return static_cast<int>(static_cast<ShearletSystem2D*>(h)->redundancy()); }

// index records: kind, scale, shear (3 ints per filter)
void ref_index_2d(void* h, int* rec) {
    const auto& s = *static_cast<ShearletSystem2D*>(h);
    for (std::size_t i = 0; i < s.index.size(); ++i) {
        rec[3 * i] = static_cast<int>(s.index[i].kind);
        rec[3 * i + 1] = s.index[i].scale;
        rec[3 * i + 2] = static_cast<int>(s.index[i].shear);
    }
}
void ref_filter_norms_2d(void* h, double* out) {
    const auto& s = *static_cast<ShearletSystem2D*>(h);
    std::memcpy(out, s.filter_norms.data(), sizeof(double) * s.filter_norms.size());
}
void ref_frame_weight_2d(void* h, double* out) {
    const auto& s = *static_cast<ShearletSystem2D*>(h);
    std::memcpy(out, s.frame_weight.data(), sizeof(double) * s.frame_weight.size());
}
// full complex spectrum of filter i, interleaved re/im
void ref_filter_2d(void* h, int i, double* out) {
    const auto& s = *static_cast<ShearletSystem2D*>(h);
    std::memcpy(out, s.filters[static_cast<std::size_t>(i)].data(),
                sizeof(double) * 2 * s.filters[static_cast<std::size_t>(i)].size());
}

int ref_forward_2d(void* h, const double* f, double* bands, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem2D*>(h);
        Signal2D in(s.rows, s.cols);
        std::memcpy(in.data(), f, sizeof(double) * in.size());
        const auto c = forward(in, s, threads);
        const std::size_t n = in.size();
        for (std::size_t i = 0; i < c.bands.size(); ++i)
            std::memcpy(bands + i * n, c.bands[i].data(), sizeof(double) * n);
    });
}

namespace {
CoefficientStack2D stack2_of(const ShearletSystem2D& s, const double* bands, int nb) {
    CoefficientStack2D c;
    c.rows = s.rows;
    c.cols = s.cols;
    c.index = s.index;
    c.bands.assign(static_cast<std::size_t>(nb), RealGrid2(s.rows, s.cols));
    const std::size_t n = s.rows * s.cols;
    for (std::size_t i = 0; i < c.bands.size(); ++i)
        std::memcpy(c.bands[i].data(), bands + i * n, sizeof(double) * n);
    return c;
}
CoefficientStack3D stack3_of(const ShearletSystem3D& s, const double* bands, int nb) {
    CoefficientStack3D c;
    c.dims = s.dims;
    c.index = s.index;
    c.bands.assign(static_cast<std::size_t>(nb), RealGrid3(s.dims[0], s.dims[1], s.dims[2]));
    const std::size_t n = s.dims[0] * s.dims[1] * s.dims[2];
    for (std::size_t i = 0; i < c.bands.size(); ++i)
        std::memcpy(c.bands[i].data(), bands + i * n, sizeof(double) * n);
    return c;
}
} // namespace

int ref_inverse_2d(void* h, const double* bands, int nb, double* out, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem2D*>(h);
        const auto r = inverse(stack2_of(s, bands, nb), s, threads);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

int ref_hard_threshold_2d(void* h, const double* bands, int nb, const double* K, int nK,
                          double sigma, int scaled, double* out) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem2D*>(h);
        ThresholdSchedule sch{std::vector<double>(K, K + nK), sigma, scaled != 0};
        const auto r = hard_threshold(stack2_of(s, bands, nb), sch, s);
        const std::size_t n = s.rows * s.cols;
        for (std::size_t i = 0; i < r.bands.size(); ++i)
            std::memcpy(out + i * n, r.bands[i].data(), sizeof(double) * n);
    });
}

int ref_denoise_2d(void* h, const double* in, const double* K, int nK, double sigma,
                   int scaled, double* out, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem2D*>(h);
        Signal2D f(s.rows, s.cols);
        std::memcpy(f.data(), in, sizeof(double) * f.size());
        ThresholdSchedule sch{std::vector<double>(K, K + nK), sigma, scaled != 0};
        const auto r = denoise(f, s, sch, threads);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

// ---------------------------------------------------------------- 3D
int ref_build_3d(int n0, int n1, int n2, const int* levels, int n_scales, int j0, int full,
                 int impulse_fan, int threads, void** out) {
    return guard([&] {
        auto* s = new ShearletSystem3D(build_system_3d(
            {static_cast<std::size_t>(n0), static_cast<std::size_t>(n1),
             static_cast<std::size_t>(n2)},
            profile_of(levels, n_scales, j0), fan_for(impulse_fan), qmf(), full != 0, threads));
        *out = s;
    });
}
void ref_free_3d(void* h) { delete static_cast<ShearletSystem3D*>(h); }
int ref_redundancy_3d(void* h) { return static_cast<int>(static_cast<ShearletSystem3D*>(h)->redundancy()); }
void ref_index_3d(void* h, int* rec) {
    const auto& s = *static_cast<ShearletSystem3D*>(h);
    for (std::size_t i = 0; i < s.index.size(); ++i) {
        rec[4 * i] = static_cast<int>(s.index[i].kind);
        rec[4 * i + 1] = s.index[i].scale;
        rec[4 * i + 2] = static_cast<int>(s.index[i].k1);
        rec[4 * i + 3] = static_cast<int>(s.index[i].k2);
    }
}
void ref_filter_norms_3d(void* h, double* out) {
    const auto& s = *static_cast<ShearletSystem3D*>(h);
    std::memcpy(out, s.filter_norms.data(), sizeof(double) * s.filter_norms.size());
}
void ref_frame_weight_3d(void* h, double* out) {
    const auto& s = *static_cast<ShearletSystem3D*>(h);
    std::memcpy(out, s.frame_weight.data(), sizeof(double) * s.frame_weight.size());
}
int ref_filter_3d(void* h, int i, double* out) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem3D*>(h);
        const auto g = s.filter_freq(static_cast<std::size_t>(i));
        std::memcpy(out, g.data(), sizeof(double) * 2 * g.size());
    });
}
// per-scale factor tables (taps): highpass length/center, phi shapes
int ref_scale_info_3d(void* h, int s, int* info) {
    return guard([&] {
        const auto& sys = *static_cast<ShearletSystem3D*>(h);
        const auto& sc = sys.scales.at(static_cast<std::size_t>(s));
        info[0] = sc.d;
        info[1] = static_cast<int>(sc.highpass.size());
        info[2] = static_cast<int>(sc.highpass.center);
        info[3] = static_cast<int>(sc.phi.size());
    });
}

int ref_forward_3d(void* h, const double* f, double* bands, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem3D*>(h);
        Signal3D in(s.dims[0], s.dims[1], s.dims[2]);
        std::memcpy(in.data(), f, sizeof(double) * in.size());
        const auto c = forward(in, s, threads);
        const std::size_t n = in.size();
        for (std::size_t i = 0; i < c.bands.size(); ++i)
            std::memcpy(bands + i * n, c.bands[i].data(), sizeof(double) * n);
    });
}
int ref_inverse_3d(void* h, const double* bands, int nb, double* out, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem3D*>(h);
        const auto r = inverse(stack3_of(s, bands, nb), s, threads);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}
int ref_hard_threshold_3d(void* h, const double* bands, int nb, const double* K, int nK,
                          double sigma, int scaled, double* out) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem3D*>(h);
        ThresholdSchedule sch{std::vector<double>(K, K + nK), sigma, scaled != 0};
        const auto r = hard_threshold(stack3_of(s, bands, nb), sch, s);
        const std::size_t n = s.dims[0] * s.dims[1] * s.dims[2];
        for (std::size_t i = 0; i < r.bands.size(); ++i)
            std::memcpy(out + i * n, r.bands[i].data(), sizeof(double) * n);
    });
}
int ref_denoise_3d(void* h, const double* in, const double* K, int nK, double sigma,
                   int scaled, double* out, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem3D*>(h);
        Signal3D f(s.dims[0], s.dims[1], s.dims[2]);
        std::memcpy(f.data(), in, sizeof(double) * f.size());
        ThresholdSchedule sch{std::vector<double>(K, K + nK), sigma, scaled != 0};
        const auto r = denoise(f, s, sch, threads);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}


// forward -> hard_threshold -> inverse, also reporting per-band L2 norms of the
// forward stack and kept counts of the thresholded stack (for big fixtures
// where the stack itself is too large to hand back).
int ref_denoise_3d_stats(void* h, const double* in, const double* K, int nK, double sigma,
                         int scaled, double* out, long long* kept, double* band_l2,
                         double* band_sample, const long long* sample_idx, int n_sample,
                         int threads, long long* kept_fp) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem3D*>(h);
        Signal3D f(s.dims[0], s.dims[1], s.dims[2]);
        std::memcpy(f.data(), in, sizeof(double) * f.size());
        ThresholdSchedule sch{std::vector<double>(K, K + nK), sigma, scaled != 0};
        CoefficientStack3D c = forward(f, s, threads);
        for (std::size_t i = 0; i < c.bands.size(); ++i) {
            double e = 0.0;
            for (double x : c.bands[i].raw()) e += x * x;
            band_l2[i] = std::sqrt(e);
            for (int q = 0; q < n_sample; ++q)
                band_sample[i * static_cast<std::size_t>(n_sample) + static_cast<std::size_t>(q)] =
                    c.bands[i].raw()[static_cast<std::size_t>(sample_idx[q])];
        }
        CoefficientStack3D t = hard_threshold(c, sch, s);
        c = CoefficientStack3D{};
        for (std::size_t i = 0; i < t.bands.size(); ++i) {
            long long k = 0, s1 = 0, s2 = 0;
            const auto& raw = t.bands[i].raw();
            for (std::size_t e = 0; e < raw.size(); ++e) {
                if (raw[e] == 0.0) continue;
                ++k;
                const long long id = static_cast<long long>(e), r = id % 1000003;
                s1 += id;  // kept-position fingerprint (tests/conftest.py kept_fingerprint)
                s2 += r * r;
            }
            kept[i] = k;
            if (kept_fp) {
                kept_fp[2 * i] = s1;
                kept_fp[2 * i + 1] = s2;
            }
        }
        const auto r = inverse(t, s, threads);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}

// ---------------------------------------------------------------- iterative pipelines
int ref_inpaint_2d(void* h, const double* masked, const double* mask, int iterations, double delta_init,
                   double delta_min, int scaled, double* out, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem2D*>(h);
        Signal2D x(s.rows, s.cols), m(s.rows, s.cols);
        std::memcpy(x.data(), masked, sizeof(double) * x.size());
        std::memcpy(m.data(), mask, sizeof(double) * m.size());
        InpaintConfig cfg;
        cfg.iterations = iterations;
        cfg.delta_init = delta_init;
        cfg.delta_min = delta_min;
        cfg.scale_by_filter_norm = scaled != 0;
        const auto r = inpaint(x, m, s, cfg, threads);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}
int ref_inpaint_3d(void* h, const double* masked, const double* mask, int iterations, double delta_init,
                   double delta_min, int scaled, double* out, int threads) {
    return guard([&] {
        const auto& s = *static_cast<ShearletSystem3D*>(h);
        Signal3D x(s.dims[0], s.dims[1], s.dims[2]), m(s.dims[0], s.dims[1], s.dims[2]);
        std::memcpy(x.data(), masked, sizeof(double) * x.size());
        std::memcpy(m.data(), mask, sizeof(double) * m.size());
        InpaintConfig cfg;
        cfg.iterations = iterations;
        cfg.delta_init = delta_init;
        cfg.delta_min = delta_min;
        cfg.scale_by_filter_norm = scaled != 0;
        const auto r = inpaint(x, m, s, cfg, threads);
        std::memcpy(out, r.data(), sizeof(double) * r.size());
    });
}
int ref_separate_2d(void* hd, void* hi, const double* signal, int iterations, double delta_init, double delta_min,
                    int scaled, double* curves, double* blobs, int threads) {
    return guard([&] {
        const auto& d = *static_cast<ShearletSystem2D*>(hd);
        const auto& i = *static_cast<ShearletSystem2D*>(hi);
        Signal2D x(d.rows, d.cols);
        std::memcpy(x.data(), signal, sizeof(double) * x.size());
        InpaintConfig cfg;
        cfg.iterations = iterations;
        cfg.delta_init = delta_init;
        cfg.delta_min = delta_min;
        cfg.scale_by_filter_norm = scaled != 0;
        const auto r = separate(x, d, i, cfg, threads);
        std::memcpy(curves, r.curvilinear.data(), sizeof(double) * x.size());
        std::memcpy(blobs, r.blobs.data(), sizeof(double) * x.size());
    });
}
// ---------------------------------------------------------------- SHCF files
// serialize() (transform.hpp:44-45) into a caller buffer; returns the byte
// count (call with out == nullptr to size), or -code on error.
long long ref_serialize_2d(void* h, const double* bands, int nb, unsigned char* out, long long cap) {
    std::string bytes;
    const int rc = guard([&] {
        std::ostringstream os(std::ios::binary);
        serialize(stack2_of(*static_cast<ShearletSystem2D*>(h), bands, nb), os);
        bytes = os.str();
    });
    if (rc) return -rc;
    if (out && cap >= static_cast<long long>(bytes.size())) std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<long long>(bytes.size());
}
long long ref_serialize_3d(void* h, const double* bands, int nb, unsigned char* out, long long cap) {
    std::string bytes;
    const int rc = guard([&] {
        std::ostringstream os(std::ios::binary);
        serialize(stack3_of(*static_cast<ShearletSystem3D*>(h), bands, nb), os);
        bytes = os.str();
    });
    if (rc) return -rc;
    if (out && cap >= static_cast<long long>(bytes.size())) std::memcpy(out, bytes.data(), bytes.size());
    return static_cast<long long>(bytes.size());
}
// deserialize_2d/3d (transform.hpp:50-51): bands out (nb*size doubles), dims
// out, returns band count or -code.
int ref_deserialize(const unsigned char* in, long long len, int* ndim, int* dims, double* bands, long long cap) {
    int nb = 0;
    const int rc = guard([&] {
        std::istringstream is(std::string(reinterpret_cast<const char*>(in), static_cast<std::size_t>(len)),
                              std::ios::binary);
        const int d = shcf_dimensionality(is);
        is.seekg(0);
        *ndim = d;
        if (d == 2) {
            const auto c = deserialize_2d(is);
            dims[0] = static_cast<int>(c.rows); dims[1] = static_cast<int>(c.cols); dims[2] = 1;
            nb = static_cast<int>(c.bands.size());
            const std::size_t n = c.rows * c.cols;
            if (bands && cap >= static_cast<long long>(n * c.bands.size()))
                for (std::size_t i = 0; i < c.bands.size(); ++i)
                    std::memcpy(bands + i * n, c.bands[i].data(), sizeof(double) * n);
        } else {
            const auto c = deserialize_3d(is);
            for (int a = 0; a < 3; ++a) dims[a] = static_cast<int>(c.dims[a]);
            nb = static_cast<int>(c.bands.size());
            const std::size_t n = c.dims[0] * c.dims[1] * c.dims[2];
            if (bands && cap >= static_cast<long long>(n * c.bands.size()))
                for (std::size_t i = 0; i < c.bands.size(); ++i)
                    std::memcpy(bands + i * n, c.bands[i].data(), sizeof(double) * n);
        }
    });
    return rc ? -rc : nb;
}

// ---------------------------------------------------------------- PGM / SVOL (image_io.hpp:9-24)
int ref_save_pgm(const double* px, int rows, int cols, const char* path, int maxval) {
    return guard([&] {
        Signal2D s(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
        std::memcpy(s.data(), px, sizeof(double) * s.size());
        save_pgm(s, path, maxval);
    });
}
int ref_load_pgm(const char* path, double* out, long long cap, int* info) {
    return guard([&] {
        const PgmImage im = load_pgm(path);
        info[0] = static_cast<int>(im.pixels.size0());
        info[1] = static_cast<int>(im.pixels.size1());
        info[2] = im.maxval;
        if (out && cap >= static_cast<long long>(im.pixels.size()))
            std::memcpy(out, im.pixels.data(), sizeof(double) * im.pixels.size());
    });
}
int ref_save_svol(const double* v, int n0, int n1, int n2, const char* path) {
    return guard([&] {
        Signal3D s(static_cast<std::size_t>(n0), static_cast<std::size_t>(n1), static_cast<std::size_t>(n2));
        std::memcpy(s.data(), v, sizeof(double) * s.size());
        save_svol(s, path);
    });
}

// ---------------------------------------------------------------- descriptors (descriptor.hpp:25-39)
int ref_write_descriptor_2d(void* h, const char* path) {
    return guard([&] { write_descriptor(describe(*static_cast<ShearletSystem2D*>(h)), path); });
}
int ref_write_descriptor_3d(void* h, const char* path) {
    return guard([&] { write_descriptor(describe(*static_cast<ShearletSystem3D*>(h)), path); });
}
// read_descriptor + build_from_descriptor_2d/3d; *is3d tells which handle kind came back
int ref_build_from_descriptor(const char* path, int* is3d, void** out) {
    return guard([&] {
        const SystemDescriptor d = read_descriptor(path);
        *is3d = d.is_3d ? 1 : 0;
        if (d.is_3d)
            *out = new ShearletSystem3D(build_from_descriptor_3d(d));
        else
            *out = new ShearletSystem2D(build_from_descriptor_2d(d));
    });
}

// ---------------------------------------------------------------- Q metrics (apps.hpp:92-101)
int ref_gaussian_kernel(double sigma, double* out, long long cap, int* info) {
    return guard([&] {
        const Taps2d t = gaussian_kernel(sigma);
        info[0] = static_cast<int>(t.size0());
        info[1] = static_cast<int>(t.center0);
        if (out && cap >= static_cast<long long>(t.size0() * t.size1()))
            std::memcpy(out, t.v.data(), sizeof(double) * t.size0() * t.size1());
    });
}
int ref_quality_q_opt(int rows, int cols, const double* rec, const double* truth, double sigma, double* q, int* delta) {
    return guard([&] {
        Signal2D r(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols)), t(r.size0(), r.size1());
        std::memcpy(r.data(), rec, sizeof(double) * r.size());
        std::memcpy(t.data(), truth, sizeof(double) * t.size());
        const auto res = quality_q_opt(r, t, gaussian_kernel(sigma));
        *q = res.first;
        *delta = res.second;
    });
}
int ref_quality_q(int rows, int cols, const double* rec, const double* truth, double d, double sigma, double* q) {
    return guard([&] {
        Signal2D r(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols)), t(r.size0(), r.size1());
        std::memcpy(r.data(), rec, sizeof(double) * r.size());
        std::memcpy(t.data(), truth, sizeof(double) * t.size());
        *q = quality_q(r, t, d, gaussian_kernel(sigma));
    });
}

void ref_random_mask(int rows, int cols, double keep, std::uint64_t seed, double* out) {
    const auto m = phantoms::random_mask(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols), keep, seed);
    std::memcpy(out, m.data(), sizeof(double) * m.size());
}
void ref_curves_plus_dots(int n, double* out) {
    const auto g = phantoms::curves_plus_dots(static_cast<std::size_t>(n));
    std::memcpy(out, g.data(), sizeof(double) * g.size());
}

// ---------------------------------------------------------------- inputs
void ref_cartoon(int n, double* out) {
    const auto g = phantoms::cartoon(static_cast<std::size_t>(n));
    std::memcpy(out, g.data(), sizeof(double) * g.size());
}
void ref_cartoon_volume(int n, double* out) {
    const auto g = phantoms::cartoon_volume(static_cast<std::size_t>(n));
    std::memcpy(out, g.data(), sizeof(double) * g.size());
}
void ref_add_noise_2d(int rows, int cols, const double* in, double sigma, std::uint64_t seed,
                      double* out) {
    Signal2D s(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols));
    std::memcpy(s.data(), in, sizeof(double) * s.size());
    const auto r = add_gaussian_noise(s, sigma, seed);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
}
void ref_add_noise_3d(int n0, int n1, int n2, const double* in, double sigma, std::uint64_t seed,
                      double* out) {
    Signal3D s(static_cast<std::size_t>(n0), static_cast<std::size_t>(n1), static_cast<std::size_t>(n2));
    std::memcpy(s.data(), in, sizeof(double) * s.size());
    const auto r = add_gaussian_noise(s, sigma, seed);
    std::memcpy(out, r.data(), sizeof(double) * r.size());
}
double ref_psnr_2d(int rows, int cols, const double* a, const double* b) {
    Signal2D x(static_cast<std::size_t>(rows), static_cast<std::size_t>(cols)), y(x);
    std::memcpy(x.data(), a, sizeof(double) * x.size());
    std::memcpy(y.data(), b, sizeof(double) * y.size());
    return psnr(x, y);
}
// raw 1D/2D/3D complex FFT through the reference wrapper (validates the shim)
void ref_fft_forward(int rank, const int* dims, double* data) {
    std::size_t n = 1;
    for (int a = 0; a < rank; ++a) n *= static_cast<std::size_t>(dims[a]);
    if (rank == 1) {
        std::vector<std::complex<double>> v(n);
        std::memcpy(v.data(), data, 16 * n);
        fft::forward(v);
        std::memcpy(data, v.data(), 16 * n);
    } else if (rank == 2) {
        ComplexGrid2 g(static_cast<std::size_t>(dims[0]), static_cast<std::size_t>(dims[1]));
        std::memcpy(g.data(), data, 16 * n);
        fft::forward(g);
        std::memcpy(data, g.data(), 16 * n);
    } else {
        ComplexGrid3 g(static_cast<std::size_t>(dims[0]), static_cast<std::size_t>(dims[1]),
                       static_cast<std::size_t>(dims[2]));
        std::memcpy(g.data(), data, 16 * n);
        fft::forward(g);
        std::memcpy(data, g.data(), 16 * n);
    }
}

} // extern "C"
