// oracle/fftw_shim/fftw_shim.cpp -- TEST INFRASTRUCTURE ONLY (CPU checker).
//
// O(N log N) mixed-radix FFT behind the FFTW3 API subset the reference uses
// (see fftw3.h in this directory). Restates FFTW's published DFT definition;
// no FFTW source is used (FFTW is not in the image).
//
// Design: every axis of a rank-1..3 row-major array is transformed by
// gathering a block of up to kBlock vectors into a contiguous [L][B] scratch,
// running a Stockham autosort FFT vectorised across the B lanes (radix 4, 2,
// 3, 5 and a generic odd-prime radix), and scattering back. Plans are
// immutable after creation; execution uses thread-local scratch, so
// concurrent fftw_execute_dft calls on distinct buffers are safe (the
// reference relies on that: core/src/fft.cpp:24-26).
#include "fftw3.h"

#include <cmath>
#include <complex>
#include <cstddef>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace {

using cd = std::complex<double>;
constexpr int kBlock = 16;

struct Stage {
    int radix;
    int ns;                 // product of the radices of earlier stages
    std::vector<cd> tw;     // tw[(r-1)*ns + (j % ns)] = w^(r * (j%ns)), r = 1..R-1
    std::vector<cd> roots;  // generic radix: exp(sign 2 pi i q / R), q = 0..R-1
};

struct Plan1D {
    int n = 0;
    int sign = -1;
    std::vector<Stage> stages;
};

cd unit_root(long long k, long long n, int sign) {
    // exp(sign * 2 pi i k / n) with the argument reduced in long double.
    k %= n;
    if (k < 0) k += n;
    const long double a = 2.0L * 3.141592653589793238462643383279502884L *
                          static_cast<long double>(k) / static_cast<long double>(n);
    return cd(static_cast<double>(cosl(a)), static_cast<double>(sign * sinl(a)));
}

Plan1D make_plan_1d(int n, int sign) {
    Plan1D p;
    p.n = n;
    p.sign = sign;
    std::vector<int> radices;
    int m = n;
    while (m % 4 == 0) { radices.push_back(4); m /= 4; }
    while (m % 2 == 0) { radices.push_back(2); m /= 2; }
    while (m % 3 == 0) { radices.push_back(3); m /= 3; }
    while (m % 5 == 0) { radices.push_back(5); m /= 5; }
    for (int f = 7; m > 1; f += 2)
        while (m % f == 0) { radices.push_back(f); m /= f; }
    int ns = 1;
    for (int r : radices) {
        Stage s;
        s.radix = r;
        s.ns = ns;
        s.tw.resize(static_cast<std::size_t>((r - 1) * ns));
        for (int q = 1; q < r; ++q)
            for (int t = 0; t < ns; ++t)
                s.tw[static_cast<std::size_t>((q - 1) * ns + t)] =
                    unit_root(static_cast<long long>(q) * t, static_cast<long long>(ns) * r, sign);
        if (r != 2 && r != 3 && r != 4 && r != 5) {
            s.roots.resize(static_cast<std::size_t>(r));
            for (int q = 0; q < r; ++q) s.roots[static_cast<std::size_t>(q)] = unit_root(q, r, sign);
        }
        p.stages.push_back(std::move(s));
        ns *= r;
    }
    return p;
}

// One Stockham stage on [n][B] data: x -> y.
void run_stage(const Stage& st, int n, int B, int sign, const cd* x, cd* y) {
    const int R = st.radix;
    const int ns = st.ns;
    const int stride = n / R;
    const double sg = static_cast<double>(sign);
    cd v[64];
    std::vector<cd> vg;
    for (int j = 0; j < stride; ++j) {
        const int t = j % ns;
        const int dst = (j / ns) * ns * R + t;
        for (int b = 0; b < B; ++b) {
            if (R == 4) {
                cd a0 = x[(j) * B + b];
                cd a1 = x[(j + stride) * B + b];
                cd a2 = x[(j + 2 * stride) * B + b];
                cd a3 = x[(j + 3 * stride) * B + b];
                if (ns > 1) {
                    a1 *= st.tw[static_cast<std::size_t>(t)];
                    a2 *= st.tw[static_cast<std::size_t>(ns + t)];
                    a3 *= st.tw[static_cast<std::size_t>(2 * ns + t)];
                }
                const cd s02 = a0 + a2, d02 = a0 - a2;
                const cd s13 = a1 + a3, d13 = a1 - a3;
                // multiply d13 by sign*i
                const cd rd13(-sg * d13.imag(), sg * d13.real());
                y[(dst) * B + b] = s02 + s13;
                y[(dst + ns) * B + b] = d02 + rd13;
                y[(dst + 2 * ns) * B + b] = s02 - s13;
                y[(dst + 3 * ns) * B + b] = d02 - rd13;
            } else if (R == 2) {
                cd a0 = x[(j) * B + b];
                cd a1 = x[(j + stride) * B + b];
                if (ns > 1) a1 *= st.tw[static_cast<std::size_t>(t)];
                y[(dst) * B + b] = a0 + a1;
                y[(dst + ns) * B + b] = a0 - a1;
            } else if (R == 3) {
                cd a0 = x[(j) * B + b];
                cd a1 = x[(j + stride) * B + b];
                cd a2 = x[(j + 2 * stride) * B + b];
                if (ns > 1) {
                    a1 *= st.tw[static_cast<std::size_t>(t)];
                    a2 *= st.tw[static_cast<std::size_t>(ns + t)];
                }
                const double c = -0.5, s = sg * 0.86602540378443864676;
                const cd sum = a1 + a2, dif = a1 - a2;
                const cd m = a0 + c * sum;
                const cd rot(-s * dif.imag(), s * dif.real());
                y[(dst) * B + b] = a0 + sum;
                y[(dst + ns) * B + b] = m + rot;
                y[(dst + 2 * ns) * B + b] = m - rot;
            } else if (R == 5) {
                cd a[5];
                for (int q = 0; q < 5; ++q) {
                    a[q] = x[(j + q * stride) * B + b];
                    if (q > 0 && ns > 1) a[q] *= st.tw[static_cast<std::size_t>((q - 1) * ns + t)];
                }
                const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
                const double s1 = sg * 0.95105651629515357212, s2 = sg * 0.58778525229247312917;
                const cd t1 = a[1] + a[4], t2 = a[2] + a[3];
                const cd t3 = a[1] - a[4], t4 = a[2] - a[3];
                const cd m1 = a[0] + c1 * t1 + c2 * t2;
                const cd m2 = a[0] + c2 * t1 + c1 * t2;
                const cd r1 = s1 * t3 + s2 * t4;  // times i
                const cd r2 = s2 * t3 - s1 * t4;  // times i
                const cd ir1(-r1.imag(), r1.real()), ir2(-r2.imag(), r2.real());
                y[(dst) * B + b] = a[0] + t1 + t2;
                y[(dst + ns) * B + b] = m1 + ir1;
                y[(dst + 4 * ns) * B + b] = m1 - ir1;
                y[(dst + 2 * ns) * B + b] = m2 + ir2;
                y[(dst + 3 * ns) * B + b] = m2 - ir2;
            } else {
                cd* a = R <= 64 ? v : (vg.resize(static_cast<std::size_t>(R)), vg.data());
                for (int q = 0; q < R; ++q) {
                    a[q] = x[(j + q * stride) * B + b];
                    if (q > 0 && ns > 1) a[q] *= st.tw[static_cast<std::size_t>((q - 1) * ns + t)];
                }
                for (int k = 0; k < R; ++k) {
                    cd s = 0.0;
                    for (int q = 0; q < R; ++q)
                        s += a[q] * st.roots[static_cast<std::size_t>((static_cast<long long>(q) * k) % R)];
                    y[(dst + k * ns) * B + b] = s;
                }
            }
        }
    }
}

void run_plan(const Plan1D& p, int B, cd* buf, cd* tmp) {
    cd* x = buf;
    cd* y = tmp;
    for (const Stage& st : p.stages) {
        run_stage(st, p.n, B, p.sign, x, y);
        std::swap(x, y);
    }
    if (x != buf) std::memcpy(buf, x, sizeof(cd) * static_cast<std::size_t>(p.n) * B);
}

} // namespace

struct fftw_plan_s {
    int rank = 0;
    int dims[3] = {1, 1, 1};
    int sign = -1;
    Plan1D axis[3];
};

extern "C" fftw_plan fftw_plan_dft(int rank, const int* n, fftw_complex*, fftw_complex*, int sign,
                                   unsigned) {
    if (rank < 1 || rank > 3) return nullptr;
    auto* p = new fftw_plan_s;
    p->rank = rank;
    p->sign = sign;
    for (int a = 0; a < rank; ++a) {
        if (n[a] < 1) { delete p; return nullptr; }
        p->dims[a] = n[a];
        p->axis[a] = make_plan_1d(n[a], sign);
    }
    return p;
}

extern "C" void fftw_destroy_plan(fftw_plan p) { delete p; }

extern "C" void fftw_execute_dft(const fftw_plan p, fftw_complex* in, fftw_complex* out) {
    cd* data = reinterpret_cast<cd*>(in);
    std::size_t total = 1;
    for (int a = 0; a < p->rank; ++a) total *= static_cast<std::size_t>(p->dims[a]);
    if (out != in) {
        std::memcpy(out, in, sizeof(cd) * total);
        data = reinterpret_cast<cd*>(out);
    }
    thread_local std::vector<cd> scratch_a, scratch_b;
    for (int a = 0; a < p->rank; ++a) {
        const int n = p->dims[a];
        if (n == 1) continue;
        std::size_t inner = 1, outer = 1;
        for (int q = a + 1; q < p->rank; ++q) inner *= static_cast<std::size_t>(p->dims[q]);
        for (int q = 0; q < a; ++q) outer *= static_cast<std::size_t>(p->dims[q]);
        const std::size_t need = static_cast<std::size_t>(n) * kBlock;
        if (scratch_a.size() < need) { scratch_a.resize(need); scratch_b.resize(need); }
        cd* sa = scratch_a.data();
        cd* sb = scratch_b.data();
        const Plan1D& plan = p->axis[a];
        if (inner > 1) {
            // vectors (o, c): element i at o*n*inner + i*inner + c; block over c.
            for (std::size_t o = 0; o < outer; ++o) {
                cd* slab = data + o * static_cast<std::size_t>(n) * inner;
                for (std::size_t c0 = 0; c0 < inner; c0 += kBlock) {
                    const int B = static_cast<int>(std::min<std::size_t>(kBlock, inner - c0));
                    for (int i = 0; i < n; ++i)
                        std::memcpy(sa + static_cast<std::size_t>(i) * B, slab + static_cast<std::size_t>(i) * inner + c0,
                                    sizeof(cd) * B);
                    run_plan(plan, B, sa, sb);
                    for (int i = 0; i < n; ++i)
                        std::memcpy(slab + static_cast<std::size_t>(i) * inner + c0, sa + static_cast<std::size_t>(i) * B,
                                    sizeof(cd) * B);
                }
            }
        } else {
            // contiguous rows; gather kBlock rows transposed into [n][B].
            for (std::size_t o0 = 0; o0 < outer; o0 += kBlock) {
                const int B = static_cast<int>(std::min<std::size_t>(kBlock, outer - o0));
                for (int b = 0; b < B; ++b) {
                    const cd* row = data + (o0 + b) * static_cast<std::size_t>(n);
                    for (int i = 0; i < n; ++i) sa[static_cast<std::size_t>(i) * B + b] = row[i];
                }
                run_plan(plan, B, sa, sb);
                for (int b = 0; b < B; ++b) {
                    cd* row = data + (o0 + b) * static_cast<std::size_t>(n);
                    for (int i = 0; i < n; ++i) row[i] = sa[static_cast<std::size_t>(i) * B + b];
                }
            }
        }
    }
}
