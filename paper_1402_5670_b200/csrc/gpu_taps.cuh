// Filter-bank construction on the GPU: every tap operation of the reference's
// filter algebra runs as a device kernel over centred tap arrays -- the QMF
// cascades, upsampling, separable axis convolutions, the five-stage digital
// shear, transposition and the lowpass tensor product. The host only holds the
// constant QMF / fan taps (taps.cpp) and the array geometry.
//
// Cascades use the two-scale refinement form x_{j} = h * (up2 x_{j-1}):
// h_j = refine^j(delta), g_j = refine^{j-1}(g) -- the same filters as the
// reference's products of upsampled taps, h * up2 h * ... * up_{2^{j-1}} h and
// up_{2^{j-1}} g * h_{j-1} (filters.cpp:40-63), summed in another order
// (~1 ulp per tap; filter spectra agree with the reference to 1e-15).
//
// Reference: src/taps.cpp:50-99 (conv_axis, upsample2, transposed),
// src/shear.cpp:222-281 (digital_shear_taps), src/system2d.cpp:21-37
// (build_shearlet_taps), src/system3d.cpp:13-25 (build_phi_component),
// src/filters.cpp:40-83 (cascade, shear_interpolation_taps).
// Temporaries are stream-ordered (cudaMallocAsync / cudaFreeAsync): building
// a filter never synchronises the device.
#pragma once

#include "common.cuh"

namespace slb {

// stream-ordered device array owned by a shared pointer
static std::shared_ptr<double> d_array(long long count, cudaStream_t st) {
    double* p = nullptr;
    SL_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), static_cast<size_t>(std::max(1LL, count)) * sizeof(double), st));
    return std::shared_ptr<double>(p, [st](double* q) { cudaFreeAsync(q, st); });
}

struct DTaps1 {
    std::shared_ptr<double> v;
    long n = 0, c = 0;
    const double* p() const { return v.get(); }
};

struct DTaps2 {
    std::shared_ptr<double> v;
    long n0 = 0, n1 = 0, c0 = 0, c1 = 0;
    const double* p() const { return v.get(); }
};

static inline unsigned blocks_for(long long n) { return static_cast<unsigned>(std::min<long long>(8192, (n + 255) / 256)); }

static DTaps1 d_alloc1(long n, long c, cudaStream_t st) { return DTaps1{d_array(n, st), n, c}; }
static DTaps2 d_alloc(long n0, long n1, long c0, long c1, cudaStream_t st) {
    return DTaps2{d_array(static_cast<long long>(n0) * n1, st), n0, n1, c0, c1};
}

static DTaps1 d_upload1(const Taps1& t, cudaStream_t st) {
    DTaps1 d = d_alloc1(static_cast<long>(t.size()), t.c, st);
    SL_CUDA(cudaMemcpyAsync(d.v.get(), t.v.data(), t.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    SL_CUDA(cudaStreamSynchronize(st));  // the host vector may go away (pageable copy)
    return d;
}
static DTaps2 d_upload(const Taps2& t, cudaStream_t st) {
    DTaps2 d = d_alloc(static_cast<long>(t.n0), static_cast<long>(t.n1), t.c0, t.c1, st);
    SL_CUDA(cudaMemcpyAsync(d.v.get(), t.v.data(), t.v.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    SL_CUDA(cudaStreamSynchronize(st));
    return d;
}

// ---------------------------------------------------------------- 1D kernels
// out[n] = sum_k h[k] * x[(n - k) / 2] over even n - k (two-scale refinement)
__global__ void kt_refine(const double* __restrict__ h, long lh, const double* __restrict__ x, long lx,
                          double* __restrict__ out, long lo) {
    for (long n = blockIdx.x * (long)blockDim.x + threadIdx.x; n < lo; n += (long)gridDim.x * blockDim.x) {
        double s = 0.0;
        const long kmin = max(0L, n - 2 * (lx - 1)), kmax = min(lh - 1, n);
        for (long k = kmin + ((n - kmin) & 1); k <= kmax; k += 2) s += h[k] * x[(n - k) >> 1];
        out[n] = s;
    }
}
__global__ void kt_scale_reverse(const double* __restrict__ in, long n, double scale, int reverse,
                                 double* __restrict__ out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x)
        out[i] = in[reverse ? n - 1 - i : i] * scale;
}
__global__ void kt_outer(const double* __restrict__ a, long na, const double* __restrict__ b, long nb,
                         double* __restrict__ out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)na * nb;
         e += (long long)gridDim.x * blockDim.x)
        out[e] = a[e / nb] * b[e % nb];
}

// x_{j} = h * up2(x_{j-1}), centre c_h + 2 c_x
static DTaps1 d_refine(const DTaps1& h, const DTaps1& x, cudaStream_t st) {
    const long lo = h.n + 2 * (x.n - 1);
    DTaps1 o = d_alloc1(lo, h.c + 2 * x.c, st);
    kt_refine<<<blocks_for(lo), 256, 0, st>>>(h.p(), h.n, x.p(), x.n, o.v.get(), lo);
    check_launch("kt_refine");
    return o;
}

// Device QMF pair and the per-level cascades (filters.cpp:40-63), memoised
// per level (the reference recomputes them for every filter).
struct DQmf {
    DTaps1 h, g, delta;
    std::map<int, DTaps1> hs, gs;
    DQmf(const Qmf& q, cudaStream_t st) {
        h = d_upload1(q.lowpass, st);
        g = d_upload1(q.highpass, st);
        delta = d_upload1(Taps1{{1.0}, 0}, st);
    }
    const DTaps1& lowpass(int level, cudaStream_t st) {  // h_j
        if (level < 0) throw SlError(SL_ERR_DOMAIN, "cascade: negative level");
        auto it = hs.find(level);
        if (it != hs.end()) return it->second;
        DTaps1 r = level == 0 ? delta : d_refine(h, lowpass(level - 1, st), st);
        return hs.emplace(level, std::move(r)).first->second;
    }
    const DTaps1& highpass(int level, cudaStream_t st) {  // g_j (g_0 = delta)
        if (level < 0) throw SlError(SL_ERR_DOMAIN, "cascade: negative level");
        auto it = gs.find(level);
        if (it != gs.end()) return it->second;
        DTaps1 r = level == 0 ? delta : (level == 1 ? g : d_refine(h, highpass(level - 1, st), st));
        return gs.emplace(level, std::move(r)).first->second;
    }
    // shear interpolation taps h_d * sqrt(2)^d (filters.cpp:80-83), optionally reversed
    DTaps1 interp(int d, bool reverse, cudaStream_t st) {
        const DTaps1& hd = lowpass(d, st);
        DTaps1 o = d_alloc1(hd.n, reverse ? hd.n - 1 - hd.c : hd.c, st);
        kt_scale_reverse<<<blocks_for(hd.n), 256, 0, st>>>(hd.p(), hd.n, std::pow(std::sqrt(2.0), d), reverse ? 1 : 0,
                                                           o.v.get());
        check_launch("kt_scale_reverse");
        return o;
    }
};

// ---------------------------------------------------------------- 2D kernels
// out(i*f0, j*f1) = in(i, j), zeros elsewhere (taps.cpp:78-88)
__global__ void kt_upsample2(const double* __restrict__ in, long n0, long n1, double* __restrict__ out, long m0, long m1,
                             int f0, int f1) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)m0 * m1;
         e += (long long)gridDim.x * blockDim.x) {
        const long a = (long)(e / m1), b = (long)(e - (long long)a * m1);
        out[e] = (a % f0 == 0 && b % f1 == 0) ? in[(a / f0) * n1 + b / f1] : 0.0;
    }
}

// separable aperiodic convolution along `axis` (taps.cpp:50-76): output o
// sums src(i)*t(o - i) over source rows i in ascending order, zero taps skipped.
__global__ void kt_conv_axis(const double* __restrict__ in, long n0, long n1, const double* __restrict__ t, int L,
                             int axis, double* __restrict__ out, long m0, long m1) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)m0 * m1;
         e += (long long)gridDim.x * blockDim.x) {
        const long a = (long)(e / m1), b = (long)(e - (long long)a * m1);
        double s = 0.0;
        if (axis == 0) {
            const long lo = max(0L, a - L + 1), hi = min(n0 - 1, a);
            for (long i = lo; i <= hi; ++i) {
                const double w = t[a - i];
                if (w != 0.0) s += in[i * n1 + b] * w;
            }
        } else {
            const long lo = max(0L, b - L + 1), hi = min(n1 - 1, b);
            for (long j = lo; j <= hi; ++j) {
                const double w = t[b - j];
                if (w != 0.0) s += in[a * n1 + j] * w;
            }
        }
        out[e] = s;
    }
}

// integer shear of the centred support: out(a0 - k*b1, b1) = in(a0, b1) (shear.cpp:229-251)
__global__ void kt_shear_support(const double* __restrict__ in, long n0, long n1, long c0, long c1, long k,
                                 double* __restrict__ out, long m0, long oc0) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)m0 * n1;
         e += (long long)gridDim.x * blockDim.x) {
        const long r = (long)(e / n1), j = (long)(e - (long long)r * n1);
        const long b1 = j - c1;
        const long a0 = (r - oc0) + k * b1;  // source relative index
        const long i = a0 + c0;
        out[e] = (i >= 0 && i < n0) ? in[i * n1 + j] : 0.0;
    }
}

// keep rows q*f + c0 for q in [qlo, qhi] (shear.cpp:263-279)
__global__ void kt_decimate_rows(const double* __restrict__ in, long n1, long c0, long f, long qlo, double* __restrict__ out,
                                 long m0) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)m0 * n1;
         e += (long long)gridDim.x * blockDim.x) {
        const long q = (long)(e / n1), j = (long)(e - (long long)q * n1);
        out[e] = in[((q + qlo) * f + c0) * n1 + j];
    }
}

__global__ void kt_transpose(const double* __restrict__ in, long n0, long n1, double* __restrict__ out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < (long long)n0 * n1;
         e += (long long)gridDim.x * blockDim.x) {
        const long a = (long)(e / n0), b = (long)(e - (long long)a * n0);  // out is n1 x n0
        out[e] = in[b * n1 + a];
    }
}

static DTaps2 d_upsample2(const DTaps2& g, long f0, long f1, cudaStream_t st) {
    if (f0 == 1 && f1 == 1) return g;
    DTaps2 d = d_alloc((g.n0 - 1) * f0 + 1, (g.n1 - 1) * f1 + 1, g.c0 * f0, g.c1 * f1, st);
    kt_upsample2<<<blocks_for(d.n0 * d.n1), 256, 0, st>>>(g.p(), g.n0, g.n1, d.v.get(), d.n0, d.n1, (int)f0, (int)f1);
    check_launch("kt_upsample2");
    return d;
}

static DTaps2 d_conv_axis(const DTaps2& g, const DTaps1& t, int axis, cudaStream_t st) {
    DTaps2 d = axis == 0 ? d_alloc(g.n0 + t.n - 1, g.n1, g.c0 + t.c, g.c1, st)
                         : d_alloc(g.n0, g.n1 + t.n - 1, g.c0, g.c1 + t.c, st);
    kt_conv_axis<<<blocks_for(d.n0 * d.n1), 256, 0, st>>>(g.p(), g.n0, g.n1, t.p(), (int)t.n, axis, d.v.get(), d.n0,
                                                           d.n1);
    check_launch("kt_conv_axis");
    return d;
}

static DTaps2 d_shear_support(const DTaps2& in, long k, cudaStream_t st) {
    if (k == 0) return in;
    const long lo1 = -in.c1, hi1 = in.n1 - 1 - in.c1;
    const long lo0i = -in.c0, hi0i = in.n0 - 1 - in.c0;
    const long lo0 = std::min(lo0i - k * lo1, lo0i - k * hi1);
    const long hi0 = std::max(hi0i - k * lo1, hi0i - k * hi1);
    DTaps2 d = d_alloc(hi0 - lo0 + 1, in.n1, -lo0, in.c1, st);
    kt_shear_support<<<blocks_for(d.n0 * d.n1), 256, 0, st>>>(in.p(), in.n0, in.n1, in.c0, in.c1, k, d.v.get(), d.n0,
                                                               d.c0);
    check_launch("kt_shear_support");
    return d;
}

// S^d_{k/2^d}: up 2^d along axis 0 -> interpolate -> integer shear of the
// support -> reversed interpolation -> keep every 2^d-th row (shear.cpp:222-281)
static DTaps2 d_digital_shear(const DTaps2& t, long k, int d, DQmf& q, cudaStream_t st) {
    const long kmax = 1L << d;
    if (k < -kmax || k > kmax) throw SlError(SL_ERR_DOMAIN, "digital_shear_taps: |k| exceeds 2^d");
    if (d == 0) return d_shear_support(t, k, st);
    const long f = 1L << d;
    DTaps2 up = d_upsample2(t, f, 1, st);
    up = d_conv_axis(up, q.interp(d, false, st), 0, st);
    up = d_shear_support(up, k, st);
    up = d_conv_axis(up, q.interp(d, true, st), 0, st);
    const long lo = -up.c0, hi = up.n0 - 1 - up.c0;
    const long qlo = lo >= 0 ? (lo + f - 1) / f : -((-lo) / f);
    const long qhi = hi >= 0 ? hi / f : -((-hi + f - 1) / f);
    DTaps2 o = d_alloc(qhi - qlo + 1, up.n1, -qlo, up.c1, st);
    kt_decimate_rows<<<blocks_for(o.n0 * o.n1), 256, 0, st>>>(up.p(), up.n1, up.c0, f, qlo, o.v.get(), o.n0);
    check_launch("kt_decimate_rows");
    return o;
}

static DTaps2 d_transposed(const DTaps2& g, cudaStream_t st) {
    DTaps2 d = d_alloc(g.n1, g.n0, g.c1, g.c0, st);
    kt_transpose<<<blocks_for(g.n0 * g.n1), 256, 0, st>>>(g.p(), g.n0, g.n1, d.v.get());
    check_launch("kt_transpose");
    return d;
}

// lowpass tensor h_J (x) h_J (system2d.cpp:95-97)
static DTaps2 d_outer(const DTaps1& a, const DTaps1& b, cudaStream_t st) {
    DTaps2 d = d_alloc(a.n, b.n, a.c, b.c, st);
    kt_outer<<<blocks_for(a.n * b.n), 256, 0, st>>>(a.p(), a.n, b.p(), b.n, d.v.get());
    check_launch("kt_outer");
    return d;
}

// 1D taps as a 1 x n tap grid (the 3D per-axis spectra)
static DTaps2 d_as_row(const DTaps1& t) { return DTaps2{t.v, 1, t.n, 0, t.c}; }

// build_shearlet_taps (system2d.cpp:21-37) on the device
static DTaps2 d_cone_taps(int j, long k, int d, int J, const DTaps2& fan, DQmf& q, cudaStream_t st) {
    const int lg = J - j, lh = J - (j - d);
    if (d < 0) throw SlError(SL_ERR_DOMAIN, "build_shearlet_taps: negative shear level");
    if (lg < 1 || lh < 0) throw SlError(SL_ERR_DOMAIN, "build_shearlet_taps: scale out of range");
    DTaps2 p = d_upsample2(fan, 1L << (J - j - 1), 1L << lh, st);
    p = d_conv_axis(p, q.highpass(lg, st), 0, st);
    p = d_conv_axis(p, q.lowpass(lh, st), 1, st);
    return d_digital_shear(p, k, d, q, st);
}

// build_phi_component (system3d.cpp:13-25) on the device
static DTaps2 d_phi_taps(int j, long k, int d, int J, const DTaps2& fan, DQmf& q, cudaStream_t st) {
    const int lh = J - (j - d);
    if (d < 0) throw SlError(SL_ERR_DOMAIN, "build_phi_component: negative shear level");
    if (J - j < 1 || lh < 0) throw SlError(SL_ERR_DOMAIN, "build_phi_component: scale out of range");
    DTaps2 p = d_upsample2(fan, 1L << (J - j - 1), 1L << lh, st);
    p = d_conv_axis(p, q.lowpass(lh, st), 1, st);
    return d_digital_shear(p, k, d, q, st);
}

}  // namespace slb
