// Host-side synthetic input generators.
#pragma once
#include <cmath>
#include <cstdint>
#include <cstddef>

namespace slb {

// ------------------------------------------------------------------ phantoms
// Deterministic inputs with the reference generators' definitions
// (phantoms.cpp:14-36, 91-108; apps.cpp:17-55).
static void cartoon(int n, double* img) {
    const double N = n;
    auto sq = [](double x) { return x * x; };
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            const double x = i / N - 0.5, y = j / N - 0.5;
            double v = 32.0;
            if (y > 0.12 + 0.18 * std::sin(5.0 * x)) v = 96.0;
            const double u = 0.8 * (x + 0.12) + 0.6 * (y + 0.18);
            const double w = -0.6 * (x + 0.12) + 0.8 * (y + 0.18);
            if (sq(u / 0.28) + sq(w / 0.16) < 1.0) v = 200.0;
            const double r2 = sq(x - 0.22) + sq(y - 0.2);
            if (r2 < sq(0.16)) v = 150.0;
            if (r2 < sq(0.055)) v = 60.0;
            if (std::fabs(x + 0.3) < 0.06 && std::fabs(y + 0.32) < 0.06) v = 255.0;
            img[static_cast<size_t>(i) * n + j] = v;
        }
}

static void cartoon_volume(int n, double* vol) {
    const double N = n;
    auto sq = [](double x) { return x * x; };
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            for (int k = 0; k < n; ++k) {
                const double x = i / N - 0.5, y = j / N - 0.5, z = k / N - 0.5;
                double v = 20.0;
                if (z > 0.1 + 0.15 * std::sin(4.0 * x) * std::cos(3.0 * y)) v = 90.0;
                if (sq(x + 0.1) + sq(y + 0.08) + sq(z + 0.1) < sq(0.24)) v = 190.0;
                if (sq(x - 0.2) / sq(0.2) + sq(y - 0.15) / sq(0.12) + sq(z) / sq(0.12) < 1.0) v = 140.0;
                vol[(static_cast<size_t>(i) * n + j) * n + k] = v;
            }
}

struct Mt64 {  // std::mt19937_64
    uint64_t mt[312];
    int idx = 312;
    explicit Mt64(uint64_t seed) {
        mt[0] = seed;
        for (int i = 1; i < 312; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
    }
    uint64_t operator()() {
        if (idx >= 312) {
            for (int i = 0; i < 312; ++i) {
                const uint64_t x = (mt[i] & 0xFFFFFFFF80000000ull) | (mt[(i + 1) % 312] & 0x7FFFFFFFull);
                uint64_t xa = x >> 1;
                if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
                mt[i] = mt[(i + 156) % 312] ^ xa;
            }
            idx = 0;
        }
        uint64_t y = mt[idx++];
        y ^= (y >> 29) & 0x5555555555555555ull;
        y ^= (y << 17) & 0x71D67FFFEDA60000ull;
        y ^= (y << 37) & 0xFFF7EEE000000000ull;
        y ^= y >> 43;
        return y;
    }
};


}  // namespace slb
