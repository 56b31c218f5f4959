// Host-side filter-bank descriptions (see taps.hpp). No tap arithmetic here.
#include "taps.hpp"

#include <cmath>
#include <cstring>

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

Taps1 maxflat9_lowpass() {
    // h = (a, b, c, d, e, d, c, b, a), centre 4, with sqrt(2) closed forms
    const double s = std::sqrt(2.0);
    const double a = (7.0 - 4.0 * s) / 128.0, b = (8.0 * s - 13.0) / 64.0, c = (8.0 - 8.0 * s) / 64.0;
    const double d = (29.0 - 8.0 * s) / 64.0, e = (9.0 + 20.0 * s) / 64.0;
    return Taps1{{a, b, c, d, e, d, c, b, a}, 4};
}

Taps1 mirror_highpass(const Taps1& h) {
    Taps1 g = h;
    for (std::size_t i = 0; i < g.v.size(); ++i) {
        const long n = static_cast<long>(i) - g.c;
        if (n % 2 != 0) g.v[i] = -g.v[i];
    }
    return g;
}

Qmf qmf_from_lowpass(const Taps1& h) { return Qmf{h, mirror_highpass(h)}; }

namespace {
// Upper-left 8x8 quadrant of the 15x15 dmaxflat4 fan (centre (7, 7)); the
// table is symmetric under i0 -> 14 - i0 and i1 -> 14 - i1. Exact binary64
// values; default_fan() re-checks the FNV-1a checksum of the full table.
constexpr double kFanQuadrant[8][8] = {
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0x1.4000000000000p-17},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, -0x1.1800000000000p-14, 0.0},
    {0.0, 0.0, 0.0, 0.0, 0.0, 0x1.a400000000000p-13, 0.0, -0x1.6bffffffffffep-13},
    {0.0, 0.0, 0.0, 0.0, -0x1.5e00000000000p-12, 0.0, 0x1.d87ffffffffffp-10, 0.0},
    {0.0, 0.0, 0.0, 0x1.5e00000000000p-12, 0.0, -0x1.0ae0000000000p-8, 0.0, 0x1.59a0000000000p-8},
    {0.0, 0.0, -0x1.a400000000000p-13, 0.0, 0x1.0ae0000000000p-8, 0.0, -0x1.add8000000000p-6, 0.0},
    {0.0, 0x1.1800000000000p-14, 0.0, -0x1.d87ffffffffffp-10, 0.0, 0x1.add8000000000p-6, 0.0, -0x1.6053000000000p-3},
    {-0x1.4000000000000p-17, 0.0, 0x1.6bffffffffffep-13, 0.0, -0x1.59a0000000000p-8, 0.0, 0x1.6053000000000p-3,
     0x1.0000000000000p-1},
};
}  // namespace

Taps2 default_fan() {
    Taps2 t = Taps2::zeros(15, 15, 7, 7);
    for (std::size_t i = 0; i < 15; ++i)
        for (std::size_t j = 0; j < 15; ++j) t.at(i, j) = kFanQuadrant[i < 8 ? i : 14 - i][j < 8 ? j : 14 - j];
    return t;
}

std::uint64_t fan_checksum(const Taps2& t) {
    std::uint64_t h = 1469598103934665603ull;  // the reference's FNV-1a offset basis (filters.cpp:89-110)
    auto feed64 = [&h](std::uint64_t w) {     // little-endian bytes of one word
        for (int b = 0; b < 8; ++b) {
            h ^= (w >> (8 * b)) & 0xffu;
            h *= 0x100000001b3ull;  // FNV prime
        }
    };
    feed64(t.n0);
    feed64(t.n1);
    feed64(static_cast<std::uint64_t>(t.c0));
    feed64(static_cast<std::uint64_t>(t.c1));
    for (double x : t.v) {
        std::uint64_t w;
        std::memcpy(&w, &x, sizeof w);
        feed64(w);
    }
    return h;
}

// ---------------------------------------------------------------- filter order
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

}  // namespace slb
