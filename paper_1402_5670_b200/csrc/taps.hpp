// Host-side descriptions of the filter bank: tap containers, the QMF pair and
// fan asset (constants), the scale profile and the filter enumeration order.
// All tap arithmetic (cascades, upsampling, separable convolutions, the
// digital shear, embedding and FFTs) runs on the GPU: gpu_taps.cuh, build.cuh.
//
// Reference (paths relative to /root/reference/proj/core): tap containers
// include/shearlet/taps.hpp:13-61; QMF pair and fan asset src/filters.cpp:12-38,
// 86-122; filter order src/system2d.cpp:49-73, src/system3d.cpp:27-80.
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

struct Qmf {
    Taps1 lowpass, highpass;
};
Taps1 maxflat9_lowpass();               // closed-form 9-tap lowpass (filters.cpp:12-20)
Taps1 mirror_highpass(const Taps1& h);  // g[n] = (-1)^n h[n] (filters.cpp:22-30)
Qmf qmf_from_lowpass(const Taps1& h);

/// The bundled 15x15 "dmaxflat4" fan filter (filters.cpp:112-122), shipped as
/// a constant table and verified against its FNV-1a checksum.
Taps2 default_fan();
std::uint64_t fan_checksum(const Taps2& t);  // FNV-1a 64 over dims, centre, tap bytes (filters.cpp:86-110)
constexpr std::uint64_t kDefaultFanChecksum = 0xb942f71dc884b1baull;

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

}  // namespace slb
