// integration/transform_b200.cpp -- the reference-side binding a maintainer
// adds to /root/reference/proj/core: the
// reference's own forward / inverse / denoise (transform.hpp:27-37,
// apps.hpp:40-44) implemented over the C ABI of libshearlet_b200.so, so
// every existing caller -- the CLI, inpaint / separate (apps.cpp:179-280),
// the test and acceptance suites -- runs the B200 path unchanged.
//
// Built by integration/Makefile against the UNMODIFIED reference sources
// (the reference's definitions of these five functions are made weak in its
// compiled objects, so these win at link time); nothing from the reference
// is copied here.
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "shearlet/apps.hpp"
#include "shearlet/errors.hpp"
#include "shearlet/transform.hpp"
#include "shearlet_b200.h"

namespace shearlet {
namespace {

void check(int rc) {
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
        default: throw Error(m);
    }
}

// One device handle per distinct filter bank. The key is the bank's content
// (grid, profile, full flag, QMF taps, fan taps), not the system's address:
// a system rebuilt at a recycled address with other parameters gets its own
// handle, and equal systems share one (their filters are identical).
struct Handle {
    sl_system* h = nullptr;
    ~Handle() {
        if (h) sl_system_destroy(h);
    }
};

template <class Sys>
std::string bank_key(const Sys& s, const std::vector<std::size_t>& dims) {
    std::ostringstream k;
    k.precision(17);
    for (std::size_t d : dims) k << d << 'x';
    k << '|' << s.profile.coarsest_scale_offset << ':';
    for (int l : s.profile.shear_levels) k << l << ',';
    k << '|' << s.full_system << '|' << s.qmf.lowpass.center << ':';
    for (double v : s.qmf.lowpass.v) k << v << ',';
    k << '|' << s.qmf.highpass.center << ':';
    for (double v : s.qmf.highpass.v) k << v << ',';
    k << '|' << s.fan.taps.center0 << ',' << s.fan.taps.center1 << ':' << s.fan.taps.size0() << 'x'
      << s.fan.taps.size1() << ':';
    for (double v : s.fan.taps.v.raw()) k << v << ',';
    return k.str();
}

template <class Sys>
sl_system* device_system(const Sys& s, const std::vector<std::size_t>& dims) {
    static std::mutex mu;
    static std::map<std::string, std::unique_ptr<Handle>> cache;
    const std::string key = bank_key(s, dims);
    std::lock_guard<std::mutex> lk(mu);
    auto& slot = cache[key];
    if (slot) return slot->h;
    auto h = std::make_unique<Handle>();
    const auto& q = s.qmf;
    const auto& fan = s.fan.taps;
    const int n = s.profile.n_scales;
    const char* prov = s.fan.provenance.c_str();
    if (dims.size() == 2)
        check(sl_system_create_2d_ex(int(dims[0]), int(dims[1]), s.profile.shear_levels.data(), n,
                                     s.profile.coarsest_scale_offset, s.full_system, q.lowpass.v.data(),
                                     int(q.lowpass.size()), int(q.lowpass.center), q.highpass.v.data(),
                                     int(q.highpass.size()), int(q.highpass.center), fan.v.data(), int(fan.size0()),
                                     int(fan.size1()), int(fan.center0), int(fan.center1), prov, /*device=*/0, 0, -1,
                                     &h->h));
    else
        check(sl_system_create_3d_ex(int(dims[0]), int(dims[1]), int(dims[2]), s.profile.shear_levels.data(), n,
                                     s.profile.coarsest_scale_offset, s.full_system, q.lowpass.v.data(),
                                     int(q.lowpass.size()), int(q.lowpass.center), q.highpass.v.data(),
                                     int(q.highpass.size()), int(q.highpass.center), fan.v.data(), int(fan.size0()),
                                     int(fan.size1()), int(fan.center0), int(fan.center1), prov, /*device=*/0, 0, -1,
                                     &h->h));
    slot = std::move(h);
    return slot->h;
}

std::vector<std::size_t> dims_of(const ShearletSystem2D& s) { return {s.rows, s.cols}; }
std::vector<std::size_t> dims_of(const ShearletSystem3D& s) { return {s.dims[0], s.dims[1], s.dims[2]}; }

template <class Stack, class Sig, class Sys, class Band>
Stack forward_impl(const Sig& f, const Sys& sys, Stack out) {
    const std::size_t n = f.size(), nb = sys.index.size();
    std::vector<double> flat(nb * n);
    check(sl_sheardec_host(device_system(sys, dims_of(sys)), f.data(), flat.data()));
    out.index = sys.index;
    out.bands.reserve(nb);
    for (std::size_t i = 0; i < nb; ++i) {
        out.bands.push_back(Band(f));
        std::memcpy(out.bands.back().data(), flat.data() + i * n, n * sizeof(double));
    }
    return out;
}

template <class Sig, class Stack, class Sys>
Sig inverse_impl(const Stack& c, const Sys& sys, Sig out) {
    const std::size_t n = out.size();
    std::vector<double> flat(c.bands.size() * n);
    for (std::size_t i = 0; i < c.bands.size(); ++i) {
        if (c.bands[i].size() != n) throw ShapeError("inverse: band dims do not match the system grid");
        std::memcpy(flat.data() + i * n, c.bands[i].data(), n * sizeof(double));
    }
    check(sl_shearrec_host(device_system(sys, dims_of(sys)), flat.data(), int(c.bands.size()), out.data()));
    return out;
}

template <class Sig, class Sys>
Sig denoise_impl(const Sig& noisy, const Sys& sys, const ThresholdSchedule& s) {
    Sig out = noisy;
    check(sl_denoise_host(device_system(sys, dims_of(sys)), noisy.data(), out.data(), s.per_scale_factors.data(),
                          int(s.per_scale_factors.size()), s.sigma, s.scale_by_filter_norm ? 1 : 0));
    return out;
}

}  // namespace

CoefficientStack2D forward(const Signal2D& f, const ShearletSystem2D& sys, int /*threads*/) {
    if (f.size0() != sys.rows || f.size1() != sys.cols)
        throw ShapeError("forward: signal dims do not match the system grid");
    CoefficientStack2D out;
    out.rows = sys.rows;
    out.cols = sys.cols;
    return forward_impl<CoefficientStack2D, Signal2D, ShearletSystem2D, RealGrid2>(f, sys, std::move(out));
}

CoefficientStack3D forward(const Signal3D& f, const ShearletSystem3D& sys, int /*threads*/) {
    if (f.size0() != sys.dims[0] || f.size1() != sys.dims[1] || f.size2() != sys.dims[2])
        throw ShapeError("forward: signal dims do not match the system grid");
    CoefficientStack3D out;
    out.dims = sys.dims;
    return forward_impl<CoefficientStack3D, Signal3D, ShearletSystem3D, RealGrid3>(f, sys, std::move(out));
}

Signal2D inverse(const CoefficientStack2D& c, const ShearletSystem2D& sys, int /*threads*/) {
    if (c.rows != sys.rows || c.cols != sys.cols || c.bands.size() != sys.index.size())
        throw ShapeError("inverse: coefficient stack does not match the system");
    return inverse_impl(c, sys, Signal2D(sys.rows, sys.cols));
}

Signal3D inverse(const CoefficientStack3D& c, const ShearletSystem3D& sys, int /*threads*/) {
    if (c.dims != sys.dims || c.bands.size() != sys.index.size())
        throw ShapeError("inverse: coefficient stack does not match the system");
    return inverse_impl(c, sys, Signal3D(sys.dims[0], sys.dims[1], sys.dims[2]));
}

Signal2D denoise(const Signal2D& noisy, const ShearletSystem2D& sys, const ThresholdSchedule& s, int /*threads*/) {
    if (noisy.size0() != sys.rows || noisy.size1() != sys.cols)
        throw ShapeError("forward: signal dims do not match the system grid");
    return denoise_impl(noisy, sys, s);
}

Signal3D denoise(const Signal3D& noisy, const ShearletSystem3D& sys, const ThresholdSchedule& s, int /*threads*/) {
    if (noisy.size0() != sys.dims[0] || noisy.size1() != sys.dims[1] || noisy.size2() != sys.dims[2])
        throw ShapeError("forward: signal dims do not match the system grid");
    return denoise_impl(noisy, sys, s);
}

}  // namespace shearlet
