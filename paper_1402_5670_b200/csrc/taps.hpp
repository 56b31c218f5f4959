// Host-side filter-bank geometry for the B200 shearlet path.
//
// Finite tap sets with declared centres, the QMF cascade, the maximally-flat
// fan, the aperiodic digital shear and the filter enumeration order. These
// feed the device-side system construction (system.cu), which embeds the
// taps periodically, FFTs them on the GPU and reduces W / RMS there.
//
// Semantics follow the reference's filter algebra (paths relative to
// /root/reference/proj/core): include/shearlet/taps.hpp:13-61,
// src/filters.cpp:12-83, src/fan_design.cpp:48-108, src/shear.cpp:222-281,
// src/system2d.cpp:21-73, src/system3d.cpp:13-80.
#pragma once

#include <cstdint>
#include <vector>

namespace slb {

/// 1D taps: v[c] sits at n = 0, v[i] at n = i - c.
struct Taps1 {
    std::vector<double> v;
    long c = 0;
    std::size_t size() const { return v.size(); }
};

/// 2D taps, row-major v[i0 * n1 + i1], centre (c0, c1).
struct Taps2 {
    std::size_t n0 = 0, n1 = 0;
    std::vector<double> v;
    long c0 = 0, c1 = 0;
    double& at(std::size_t i0, std::size_t i1) { return v[i0 * n1 + i1]; }
    double at(std::size_t i0, std::size_t i1) const { return v[i0 * n1 + i1]; }
    static Taps2 zeros(std::size_t n0, std::size_t n1, long c0, long c1);
    static Taps2 impulse();
};

Taps1 impulse1();
Taps1 conv(const Taps1& a, const Taps1& b);
Taps1 upsample(const Taps1& a, std::size_t f);
Taps1 reversed(const Taps1& a);
Taps2 outer(const Taps1& a0, const Taps1& a1);
Taps2 conv_axis(const Taps2& g, const Taps1& t, int axis);
Taps2 upsample2(const Taps2& g, std::size_t f0, std::size_t f1);
Taps2 transposed(const Taps2& g);

struct Qmf {
    Taps1 lowpass, highpass;
};
Taps1 maxflat9_lowpass();               // filters.cpp:12-20 closed form
Taps1 mirror_highpass(const Taps1& h);  // filters.cpp:22-30
Qmf qmf_from_lowpass(const Taps1& h);
/// Level-j iterated lowpass h_j and highpass g_j (filters.cpp:40-63).
void cascade(const Qmf& q, int level, Taps1* h, Taps1* g);
Taps1 shear_interp(const Qmf& q, int level);  // h_d * sqrt(2)^d (filters.cpp:80-83)

Taps2 maxflat_fan(int order);  // fan_design.cpp:70-108
std::uint64_t fan_checksum(const Taps2& t);  // FNV-1a 64 (filters.cpp:89-110)
constexpr std::uint64_t kDefaultFanChecksum = 0xb942f71dc884b1baull;

/// Aperiodic digital shear S^d_{k/2^d} on centred taps (shear.cpp:222-281).
Taps2 digital_shear_taps(const Taps2& t, long k, int d, const Taps1& interp);

// ---------------------------------------------------------------- systems
struct Profile {
    std::vector<int> levels;  // shear level d_j per scale
    int j0 = 0;
    int n_scales() const { return static_cast<int>(levels.size()); }
    int top() const { return j0 + n_scales(); }
};

/// Filter record, SHCF-compatible (transform.cpp:188-193): kind 0 lowpass,
/// 1/2 horizontal/vertical cone (2D), 3/4/5 pyramids (3D).
struct Record {
    int kind, scale, k1, k2;
};

std::vector<Record> enumerate_2d(const Profile& p, bool full);  // system2d.cpp:59-73
std::vector<Record> enumerate_3d(const Profile& p, bool full);  // system3d.cpp:58-80
std::size_t redundancy_2d(const Profile& p, bool full);
std::size_t redundancy_3d(const Profile& p, bool full);

/// Spatial taps of one 2D cone filter, horizontal orientation (system2d.cpp:21-37).
Taps2 cone_taps(int j, long k, int d, int J, const Taps2& fan, const Qmf& q);
/// 3D component taps: the 2D construction with the highpass replaced by an
/// impulse (system3d.cpp:13-25).
Taps2 phi_taps(int j, long k, int d, int J, const Taps2& fan, const Qmf& q);

}  // namespace slb
