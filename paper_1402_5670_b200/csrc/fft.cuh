// fp64 mixed-radix Stockham FFT primitives for sm_100a (shared-memory resident).
//
// A CTA transforms V "lines" of length L staged in shared memory, laid out
// a[v * ld + i] (ld = L + 1 to keep the transposed tile loads bank-conflict
// free). Stages are radix 8/4/2/3/5 (+ a generic odd radix) with twiddles
// from a global table tw[k] = exp(-2 pi i k / L), so any L whose tile fits in
// shared memory is supported; DIR = -1 is the forward (FFTW_FORWARD, e^{-})
// transform and DIR = +1 the unnormalised inverse, matching the reference's
// DFT convention (core/include/shearlet/fft.hpp:9-10).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace slb {

constexpr int kMaxStages = 16;

struct FftPlan {
    int L = 0;
    int nst = 0;
    int radix[kMaxStages] = {};
    int ns[kMaxStages] = {};    // product of the earlier radices
    const double2* tw = nullptr;  // device table exp(-2 pi i k / L), k < L
    const float2* tw32 = nullptr; // the same table rounded to fp32 (fp32 mode)
};

// Complex arithmetic and butterflies, generic over the complex type: double2
// (the fp64 path, the reference's precision) or float2 (the optional fp32
// mode). Constants are rounded to the scalar type, so the fp64 instances are
// exactly the fp64 code they replace.
template <class C>
struct CTraits;
template <>
struct CTraits<double2> {
    using R = double;
    __device__ __forceinline__ static double2 mk(double a, double b) { return make_double2(a, b); }
};
template <>
struct CTraits<float2> {
    using R = float;
    __device__ __forceinline__ static float2 mk(float a, float b) { return make_float2(a, b); }
};
template <class C>
using RealOf = typename CTraits<C>::R;
template <class C>
__device__ __forceinline__ C mkc(RealOf<C> a, RealOf<C> b) {
    return CTraits<C>::mk(a, b);
}

template <class C>
__device__ __forceinline__ C cadd(C a, C b) {
    return mkc<C>(a.x + b.x, a.y + b.y);
}
template <class C>
__device__ __forceinline__ C csub(C a, C b) {
    return mkc<C>(a.x - b.x, a.y - b.y);
}
template <class C>
__device__ __forceinline__ C cmul(C a, C b) {
    return mkc<C>(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
template <class C>
__device__ __forceinline__ C cconj(C a) {
    return mkc<C>(a.x, -a.y);
}
template <class C>
__device__ __forceinline__ C cscale(C a, RealOf<C> s) {
    return mkc<C>(a.x * s, a.y * s);
}
// a * (DIR * i)
template <int DIR, class C>
__device__ __forceinline__ C mul_di(C a) {
    return DIR < 0 ? mkc<C>(a.y, -a.x) : mkc<C>(-a.y, a.x);
}

template <int DIR, class C>
__device__ __forceinline__ void bfly2(C& a0, C& a1) {
    const C t = a0;
    a0 = cadd(t, a1);
    a1 = csub(t, a1);
}

template <int DIR, class C>
__device__ __forceinline__ void bfly4(C& a0, C& a1, C& a2, C& a3) {
    const C s02 = cadd(a0, a2), d02 = csub(a0, a2);
    const C s13 = cadd(a1, a3), d13 = mul_di<DIR>(csub(a1, a3));
    a0 = cadd(s02, s13);
    a2 = csub(s02, s13);
    a1 = cadd(d02, d13);
    a3 = csub(d02, d13);
}

template <int DIR, class C>
__device__ __forceinline__ void bfly8(C* a) {
    using R = RealOf<C>;
    constexpr R r = R(0.70710678118654752440);
    // radix-2 across distance 4, twiddle, then two radix-4 on even/odd halves
    C b0 = cadd(a[0], a[4]), b4 = csub(a[0], a[4]);
    C b1 = cadd(a[1], a[5]), b5 = csub(a[1], a[5]);
    C b2 = cadd(a[2], a[6]), b6 = csub(a[2], a[6]);
    C b3 = cadd(a[3], a[7]), b7 = csub(a[3], a[7]);
    // w8^1 = (1 + DIR i)/sqrt2 ; w8^2 = DIR i ; w8^3 = (-1 + DIR i)/sqrt2
    b5 = mkc<C>(r * (b5.x - DIR * b5.y), r * (b5.y + DIR * b5.x));
    b6 = mul_di<DIR>(b6);
    b7 = mkc<C>(r * (-b7.x - DIR * b7.y), r * (-b7.y + DIR * b7.x));
    bfly4<DIR>(b0, b1, b2, b3);
    bfly4<DIR>(b4, b5, b6, b7);
    a[0] = b0; a[2] = b1; a[4] = b2; a[6] = b3;
    a[1] = b4; a[3] = b5; a[5] = b6; a[7] = b7;
}

template <int DIR, class C>
__device__ __forceinline__ void bfly3(C& a0, C& a1, C& a2) {
    using R = RealOf<C>;
    constexpr R s = R(0.86602540378443864676);
    const C sum = cadd(a1, a2), dif = csub(a1, a2);
    const C m = mkc<C>(a0.x - R(0.5) * sum.x, a0.y - R(0.5) * sum.y);
    const C rot = mul_di<DIR>(cscale(dif, s));
    a0 = cadd(a0, sum);
    a1 = cadd(m, rot);
    a2 = csub(m, rot);
}

template <int DIR, class C>
__device__ __forceinline__ void bfly5(C* a) {
    using R = RealOf<C>;
    constexpr R c1 = R(0.30901699437494742410), c2 = R(-0.80901699437494742410);
    constexpr R s1 = R(0.95105651629515357212), s2 = R(0.58778525229247312917);
    const C t1 = cadd(a[1], a[4]), t2 = cadd(a[2], a[3]);
    const C t3 = csub(a[1], a[4]), t4 = csub(a[2], a[3]);
    const C m1 = mkc<C>(a[0].x + c1 * t1.x + c2 * t2.x, a[0].y + c1 * t1.y + c2 * t2.y);
    const C m2 = mkc<C>(a[0].x + c2 * t1.x + c1 * t2.x, a[0].y + c2 * t1.y + c1 * t2.y);
    const C r1 = mul_di<DIR>(mkc<C>(s1 * t3.x + s2 * t4.x, s1 * t3.y + s2 * t4.y));
    const C r2 = mul_di<DIR>(mkc<C>(s2 * t3.x - s1 * t4.x, s2 * t3.y - s1 * t4.y));
    a[0] = cadd(a[0], cadd(t1, t2));
    a[1] = cadd(m1, r1);
    a[4] = csub(m1, r1);
    a[2] = cadd(m2, r2);
    a[3] = csub(m2, r2);
}

template <int DIR, class C>
__device__ __forceinline__ C twiddle(const C* __restrict__ tw, int k) {
    const C w = __ldg(tw + k);
    return DIR < 0 ? w : cconj(w);
}

// Stockham: stage (R, Ns) maps butterfly j: inputs x[j + r*L/R] (times
// w^{r*(j%Ns)} with w = e^{DIR 2 pi i/(Ns R)}), outputs y[(j/Ns)*Ns*R + j%Ns + r*Ns].
// Ping-pongs between a and b; returns the buffer holding the result.
// Must be called by all threads of the CTA (contains __syncthreads).
template <int DIR>
__device__ double2* smem_fft(double2* a, double2* b, int V, int ld, const FftPlan& p) {
    const int L = p.L;
    for (int s = 0; s < p.nst; ++s) {
        const int R = p.radix[s];
        const int Ns = p.ns[s];
        const int stride = L / R;
        const int twstep = L / (Ns * R);
        const int nb = V * stride;
        for (int t = threadIdx.x; t < nb; t += blockDim.x) {
            const int v = t / stride;
            const int j = t - v * stride;
            const int jm = j % Ns;
            const double2* src = a + v * ld + j;
            double2* dst = b + v * ld + (j - jm) * R + jm;
            double2 x[8];
            if (R == 8) {
#pragma unroll
                for (int r = 0; r < 8; ++r) x[r] = src[r * stride];
                if (Ns > 1) {
#pragma unroll
                    for (int r = 1; r < 8; ++r) x[r] = cmul(x[r], twiddle<DIR>(p.tw, r * jm * twstep));
                }
                bfly8<DIR>(x);
#pragma unroll
                for (int r = 0; r < 8; ++r) dst[r * Ns] = x[r];
            } else if (R == 4) {
#pragma unroll
                for (int r = 0; r < 4; ++r) x[r] = src[r * stride];
                if (Ns > 1) {
#pragma unroll
                    for (int r = 1; r < 4; ++r) x[r] = cmul(x[r], twiddle<DIR>(p.tw, r * jm * twstep));
                }
                bfly4<DIR>(x[0], x[1], x[2], x[3]);
#pragma unroll
                for (int r = 0; r < 4; ++r) dst[r * Ns] = x[r];
            } else if (R == 2) {
                x[0] = src[0];
                x[1] = src[stride];
                if (Ns > 1) x[1] = cmul(x[1], twiddle<DIR>(p.tw, jm * twstep));
                bfly2<DIR>(x[0], x[1]);
                dst[0] = x[0];
                dst[Ns] = x[1];
            } else if (R == 3) {
#pragma unroll
                for (int r = 0; r < 3; ++r) x[r] = src[r * stride];
                if (Ns > 1) {
                    x[1] = cmul(x[1], twiddle<DIR>(p.tw, jm * twstep));
                    x[2] = cmul(x[2], twiddle<DIR>(p.tw, 2 * jm * twstep));
                }
                bfly3<DIR>(x[0], x[1], x[2]);
#pragma unroll
                for (int r = 0; r < 3; ++r) dst[r * Ns] = x[r];
            } else if (R == 5) {
#pragma unroll
                for (int r = 0; r < 5; ++r) x[r] = src[r * stride];
                if (Ns > 1) {
#pragma unroll
                    for (int r = 1; r < 5; ++r) x[r] = cmul(x[r], twiddle<DIR>(p.tw, r * jm * twstep));
                }
                bfly5<DIR>(x);
#pragma unroll
                for (int r = 0; r < 5; ++r) dst[r * Ns] = x[r];
            } else {
                // generic odd radix: direct DFT, roots w_R^q = tw[q * L / R]
                const int rstep = L / R;
                for (int k = 0; k < R; ++k) {
                    double2 acc = make_double2(0.0, 0.0);
                    for (int r = 0; r < R; ++r) {
                        double2 xr = src[r * stride];
                        if (Ns > 1 && r > 0) xr = cmul(xr, twiddle<DIR>(p.tw, r * jm * twstep));
                        const int q = (int)(((long long)r * k) % R);
                        acc = cadd(acc, cmul(xr, twiddle<DIR>(p.tw, q * rstep)));
                    }
                    dst[k * Ns] = acc;
                }
            }
        }
        __syncthreads();
        double2* t = a;
        a = b;
        b = t;
    }
    return a;
}

}  // namespace slb
