// Host-side filter-bank geometry (see taps.hpp for the reference mapping).
#include "taps.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

namespace slb {

Taps2 Taps2::zeros(std::size_t n0, std::size_t n1, long c0, long c1) {
    Taps2 t;
    t.n0 = n0;
    t.n1 = n1;
    t.v.assign(n0 * n1, 0.0);
    t.c0 = c0;
    t.c1 = c1;
    return t;
}

Taps2 Taps2::impulse() {
    Taps2 t = zeros(1, 1, 0, 0);
    t.v[0] = 1.0;
    return t;
}

Taps1 impulse1() { return Taps1{{1.0}, 0}; }

Taps1 conv(const Taps1& a, const Taps1& b) {
    Taps1 o;
    o.v.assign(a.size() + b.size() - 1, 0.0);
    for (std::size_t i = 0; i < a.size(); ++i) {
        const double x = a.v[i];
        for (std::size_t j = 0; j < b.size(); ++j) o.v[i + j] += x * b.v[j];
    }
    o.c = a.c + b.c;
    return o;
}

Taps1 upsample(const Taps1& a, std::size_t f) {
    if (f == 1) return a;
    Taps1 o;
    o.v.assign((a.size() - 1) * f + 1, 0.0);
    for (std::size_t i = 0; i < a.size(); ++i) o.v[i * f] = a.v[i];
    o.c = a.c * static_cast<long>(f);
    return o;
}

Taps1 reversed(const Taps1& a) {
    Taps1 o;
    o.v.assign(a.v.rbegin(), a.v.rend());
    o.c = static_cast<long>(a.size()) - 1 - a.c;
    return o;
}

Taps2 outer(const Taps1& a0, const Taps1& a1) {
    Taps2 o = Taps2::zeros(a0.size(), a1.size(), a0.c, a1.c);
    for (std::size_t i = 0; i < a0.size(); ++i)
        for (std::size_t j = 0; j < a1.size(); ++j) o.at(i, j) = a0.v[i] * a1.v[j];
    return o;
}

Taps2 conv_axis(const Taps2& g, const Taps1& t, int axis) {
    const std::size_t L = t.size();
    if (axis == 0) {
        Taps2 o = Taps2::zeros(g.n0 + L - 1, g.n1, g.c0 + t.c, g.c1);
        for (std::size_t i = 0; i < g.n0; ++i)
            for (std::size_t k = 0; k < L; ++k) {
                const double w = t.v[k];
                if (w == 0.0) continue;
                const double* src = &g.v[i * g.n1];
                double* dst = &o.v[(i + k) * o.n1];
                for (std::size_t j = 0; j < g.n1; ++j) dst[j] += src[j] * w;
            }
        return o;
    }
    Taps2 o = Taps2::zeros(g.n0, g.n1 + L - 1, g.c0, g.c1 + t.c);
    for (std::size_t i = 0; i < g.n0; ++i)
        for (std::size_t k = 0; k < L; ++k) {
            const double w = t.v[k];
            if (w == 0.0) continue;
            const double* src = &g.v[i * g.n1];
            double* dst = &o.v[i * o.n1 + k];
            for (std::size_t j = 0; j < g.n1; ++j) dst[j] += src[j] * w;
        }
    return o;
}

Taps2 upsample2(const Taps2& g, std::size_t f0, std::size_t f1) {
    if (f0 == 1 && f1 == 1) return g;
    Taps2 o = Taps2::zeros((g.n0 - 1) * f0 + 1, (g.n1 - 1) * f1 + 1, g.c0 * static_cast<long>(f0),
                           g.c1 * static_cast<long>(f1));
    for (std::size_t i = 0; i < g.n0; ++i)
        for (std::size_t j = 0; j < g.n1; ++j) o.at(i * f0, j * f1) = g.at(i, j);
    return o;
}

Taps2 transposed(const Taps2& g) {
    Taps2 o = Taps2::zeros(g.n1, g.n0, g.c1, g.c0);
    for (std::size_t i = 0; i < g.n0; ++i)
        for (std::size_t j = 0; j < g.n1; ++j) o.at(j, i) = g.at(i, j);
    return o;
}

Taps1 maxflat9_lowpass() {
    const double r2 = std::sqrt(2.0);
    const double a = (7.0 - 4.0 * r2) / 128.0;
    const double b = (8.0 * r2 - 13.0) / 64.0;
    const double c = (8.0 - 8.0 * r2) / 64.0;
    const double d = (29.0 - 8.0 * r2) / 64.0;
    const double e = (9.0 + 20.0 * r2) / 64.0;
    return Taps1{{a, b, c, d, e, d, c, b, a}, 4};
}

Taps1 mirror_highpass(const Taps1& h) {
    Taps1 g = h;
    for (std::size_t i = 0; i < g.size(); ++i)
        if ((static_cast<long>(i) - g.c) & 1) g.v[i] = -g.v[i];
    return g;
}

Qmf qmf_from_lowpass(const Taps1& h) { return Qmf{h, mirror_highpass(h)}; }

namespace {
// h * up2(h) * up4(h) * ... * up_{2^(n-1)}(h)
Taps1 lowpass_product(const Taps1& h, int n) {
    Taps1 acc = h;
    for (int j = 1; j < n; ++j) acc = conv(acc, upsample(h, std::size_t{1} << j));
    return acc;
}
}  // namespace

void cascade(const Qmf& q, int level, Taps1* h, Taps1* g) {
    if (level < 0) throw std::domain_error("cascade: negative level");
    if (level == 0) {
        if (h) *h = impulse1();
        if (g) *g = impulse1();
        return;
    }
    if (h) *h = lowpass_product(q.lowpass, level);
    if (g) {
        Taps1 up = upsample(q.highpass, std::size_t{1} << (level - 1));
        *g = level > 1 ? conv(up, lowpass_product(q.lowpass, level - 1)) : up;
    }
}

Taps1 shear_interp(const Qmf& q, int level) {
    if (level < 0) throw std::domain_error("shear_interp: negative level");
    Taps1 h;
    cascade(q, level, &h, nullptr);
    const double s = std::pow(std::sqrt(2.0), level);
    for (double& x : h.v) x *= s;
    return h;
}

// ---------------------------------------------------------------- fan
namespace {

// a*sa + b*sb on the union of the two supports.
Taps2 weighted_sum(const Taps2& a, double sa, const Taps2& b, double sb) {
    const long lo0 = std::min(-a.c0, -b.c0);
    const long hi0 = std::max(static_cast<long>(a.n0) - 1 - a.c0, static_cast<long>(b.n0) - 1 - b.c0);
    const long lo1 = std::min(-a.c1, -b.c1);
    const long hi1 = std::max(static_cast<long>(a.n1) - 1 - a.c1, static_cast<long>(b.n1) - 1 - b.c1);
    Taps2 o = Taps2::zeros(static_cast<std::size_t>(hi0 - lo0 + 1), static_cast<std::size_t>(hi1 - lo1 + 1),
                           -lo0, -lo1);
    auto add = [&o, lo0, lo1](const Taps2& x, double s) {
        const std::size_t off0 = static_cast<std::size_t>(-x.c0 - lo0);
        const std::size_t off1 = static_cast<std::size_t>(-x.c1 - lo1);
        for (std::size_t i = 0; i < x.n0; ++i)
            for (std::size_t j = 0; j < x.n1; ++j) o.at(i + off0, j + off1) += s * x.at(i, j);
    };
    add(a, sa);
    add(b, sb);
    return o;
}

Taps2 full_conv2(const Taps2& a, const Taps2& b) {
    Taps2 o = Taps2::zeros(a.n0 + b.n0 - 1, a.n1 + b.n1 - 1, a.c0 + b.c0, a.c1 + b.c1);
    for (std::size_t i = 0; i < a.n0; ++i)
        for (std::size_t j = 0; j < a.n1; ++j) {
            const double x = a.at(i, j);
            if (x == 0.0) continue;
            for (std::size_t p = 0; p < b.n0; ++p)
                for (std::size_t q = 0; q < b.n1; ++q) o.at(i + p, j + q) += x * b.at(p, q);
        }
    return o;
}

// Lagrange weights at the half-sample point for the 2N nodes -(N-1)..N.
std::vector<double> halfsample_weights(int order) {
    const int nodes = 2 * order;
    std::vector<double> w(static_cast<std::size_t>(nodes));
    for (int i = 0; i < nodes; ++i) {
        const double xi = static_cast<double>(i - order + 1);
        double p = 1.0;
        for (int j = 0; j < nodes; ++j) {
            if (j == i) continue;
            const double xj = static_cast<double>(j - order + 1);
            p *= (0.5 - xj) / (xi - xj);
        }
        w[static_cast<std::size_t>(i)] = p;
    }
    return w;
}

}  // namespace

Taps2 maxflat_fan(int order) {
    if (order < 1) throw std::domain_error("maxflat_fan: order must be >= 1");
    // McClellan kernel (cos w0 + cos w1)/2 and Chebyshev recursion
    // T_{m+1} = 2 kappa * T_m - T_{m-1}; odd terms weighted by the half-band taps.
    Taps2 kappa = Taps2::zeros(3, 3, 1, 1);
    kappa.at(0, 1) = kappa.at(2, 1) = kappa.at(1, 0) = kappa.at(1, 2) = 0.25;
    const std::vector<double> w = halfsample_weights(order);
    Taps2 diamond = Taps2::impulse();
    diamond.v[0] = 0.5;
    Taps2 t_prev = Taps2::impulse();
    Taps2 t_cur = kappa;
    for (int m = 1; m <= 2 * order - 1; ++m) {
        if (m & 1) {
            const double hm = w[static_cast<std::size_t>(order - 1 + (m + 1) / 2)] / 2.0;
            diamond = weighted_sum(diamond, 1.0, t_cur, 2.0 * hm);
        }
        Taps2 t_next = weighted_sum(full_conv2(kappa, t_cur), 2.0, t_prev, -1.0);
        t_prev = std::move(t_cur);
        t_cur = std::move(t_next);
    }
    // (-1)^{n0} modulation moves the diamond passband onto the horizontal fan.
    for (std::size_t i = 0; i < diamond.n0; ++i)
        if ((static_cast<long>(i) - diamond.c0) & 1)
            for (std::size_t j = 0; j < diamond.n1; ++j)
                if (diamond.at(i, j) != 0.0) diamond.at(i, j) = -diamond.at(i, j);
    return diamond;
}

std::uint64_t fan_checksum(const Taps2& t) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&h](const unsigned char* p, std::size_t n) {
        for (std::size_t i = 0; i < n; ++i) {
            h ^= p[i];
            h *= 1099511628211ull;
        }
    };
    const std::uint64_t meta[4] = {t.n0, t.n1, static_cast<std::uint64_t>(t.c0), static_cast<std::uint64_t>(t.c1)};
    for (std::uint64_t m : meta) {
        unsigned char le[8];
        for (int i = 0; i < 8; ++i) le[i] = static_cast<unsigned char>(m >> (8 * i));
        mix(le, 8);
    }
    for (double x : t.v) {
        std::uint64_t bits;
        std::memcpy(&bits, &x, 8);
        unsigned char le[8];
        for (int i = 0; i < 8; ++i) le[i] = static_cast<unsigned char>(bits >> (8 * i));
        mix(le, 8);
    }
    return h;
}

// ---------------------------------------------------------------- shear
namespace {
// Integer shear of the centred support: rel (a0, b1) -> (a0 - k*b1, b1).
Taps2 shear_support(const Taps2& in, long k) {
    if (k == 0) return in;
    const long lo1 = -in.c1, hi1 = static_cast<long>(in.n1) - 1 - in.c1;
    const long lo0i = -in.c0, hi0i = static_cast<long>(in.n0) - 1 - in.c0;
    const long lo0 = std::min(lo0i - k * lo1, lo0i - k * hi1);
    const long hi0 = std::max(hi0i - k * lo1, hi0i - k * hi1);
    Taps2 o = Taps2::zeros(static_cast<std::size_t>(hi0 - lo0 + 1), in.n1, -lo0, in.c1);
    for (std::size_t j = 0; j < in.n1; ++j) {
        const long b1 = static_cast<long>(j) - in.c1;
        for (std::size_t i = 0; i < in.n0; ++i) {
            const long a0 = static_cast<long>(i) - in.c0;
            o.at(static_cast<std::size_t>(a0 - k * b1 + o.c0), j) = in.at(i, j);
        }
    }
    return o;
}
long floor_div(long a, long b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
long ceil_div(long a, long b) { return a >= 0 ? (a + b - 1) / b : -((-a) / b); }
}  // namespace

Taps2 digital_shear_taps(const Taps2& t, long k, int d, const Taps1& interp) {
    if (d < 0) throw std::domain_error("digital_shear_taps: negative refinement level");
    const long kmax = 1L << d;
    if (k < -kmax || k > kmax) throw std::domain_error("digital_shear_taps: |k| exceeds 2^d");
    if (d == 0) return shear_support(t, k);
    const long f = 1L << d;
    Taps2 up = upsample2(t, static_cast<std::size_t>(f), 1);
    up = conv_axis(up, interp, 0);
    up = shear_support(up, k);
    up = conv_axis(up, reversed(interp), 0);
    const long lo = -up.c0, hi = static_cast<long>(up.n0) - 1 - up.c0;
    const long qlo = ceil_div(lo, f), qhi = floor_div(hi, f);
    Taps2 o = Taps2::zeros(static_cast<std::size_t>(qhi - qlo + 1), up.n1, -qlo, up.c1);
    for (long q = qlo; q <= qhi; ++q)
        std::memcpy(&o.v[static_cast<std::size_t>(q - qlo) * o.n1],
                    &up.v[static_cast<std::size_t>(q * f + up.c0) * up.n1], sizeof(double) * up.n1);
    return o;
}

// ---------------------------------------------------------------- systems
std::vector<Record> enumerate_2d(const Profile& p, bool full) {
    std::vector<Record> idx{{0, -1, 0, 0}};
    for (int s = 0; s < p.n_scales(); ++s) {
        const int j = p.j0 + s;
        const int K = 1 << p.levels[static_cast<std::size_t>(s)];
        for (int k = -K; k <= K; ++k) idx.push_back({1, j, k, 0});
        for (int k = -K; k <= K; ++k)
            if (full || (k != K && k != -K)) idx.push_back({2, j, k, 0});
    }
    return idx;
}

std::vector<Record> enumerate_3d(const Profile& p, bool full) {
    std::vector<Record> idx{{0, -1, 0, 0}};
    for (int s = 0; s < p.n_scales(); ++s) {
        const int j = p.j0 + s;
        const int K = 1 << p.levels[static_cast<std::size_t>(s)];
        for (int kind = 3; kind <= 5; ++kind)
            for (int k1 = -K; k1 <= K; ++k1)
                for (int k2 = -K; k2 <= K; ++k2) {
                    const bool b1 = (k1 == K || k1 == -K), b2 = (k2 == K || k2 == -K);
                    if (!full && kind == 4 && b1) continue;
                    if (!full && kind == 5 && (b1 || b2)) continue;
                    idx.push_back({kind, j, k1, k2});
                }
    }
    return idx;
}

std::size_t redundancy_2d(const Profile& p, bool full) { return enumerate_2d(p, full).size(); }
std::size_t redundancy_3d(const Profile& p, bool full) { return enumerate_3d(p, full).size(); }

Taps2 cone_taps(int j, long k, int d, int J, const Taps2& fan, const Qmf& q) {
    const int lg = J - j, lh = J - (j - d);
    if (d < 0) throw std::domain_error("cone_taps: negative shear level");
    if (lg < 1 || lh < 0) throw std::domain_error("cone_taps: scale out of range");
    Taps1 g, h;
    cascade(q, lg, nullptr, &g);
    cascade(q, lh, &h, nullptr);
    Taps2 p = upsample2(fan, std::size_t{1} << (J - j - 1), std::size_t{1} << lh);
    p = conv_axis(p, g, 0);
    p = conv_axis(p, h, 1);
    return digital_shear_taps(p, k, d, shear_interp(q, d));
}

Taps2 phi_taps(int j, long k, int d, int J, const Taps2& fan, const Qmf& q) {
    const int lh = J - (j - d);
    if (d < 0) throw std::domain_error("phi_taps: negative shear level");
    if (J - j < 1 || lh < 0) throw std::domain_error("phi_taps: scale out of range");
    Taps1 h;
    cascade(q, lh, &h, nullptr);
    Taps2 p = upsample2(fan, std::size_t{1} << (J - j - 1), std::size_t{1} << lh);
    p = conv_axis(p, h, 1);
    return digital_shear_taps(p, k, d, shear_interp(q, d));
}

}  // namespace slb
