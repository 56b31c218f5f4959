// Filter-bank construction on the GPU: the 2D tap algebra of the reference
// (upsampling, separable axis convolutions, the five-stage digital shear,
// transposition) as device kernels over centred tap grids. Only the 1D QMF
// cascades (<= 249 taps, a scalar recurrence) and the checksummed 15x15 fan
// asset are formed on the host.
//
// Reference: src/taps.cpp:50-99 (conv_axis, upsample2, transposed),
// src/shear.cpp:222-281 (digital_shear_taps), src/system2d.cpp:21-37
// (build_shearlet_taps), src/system3d.cpp:13-25 (build_phi_component).
// Each gather sums its contributions in the reference's loop order.
#pragma once

#include "common.cuh"

namespace slb {

struct DTaps2 {
    std::unique_ptr<DBuf<double>> v = std::make_unique<DBuf<double>>();
    long n0 = 0, n1 = 0, c0 = 0, c1 = 0;
    const double* p() const { return v->p; }
};

static inline unsigned blocks_for(long long n) { return static_cast<unsigned>(std::min<long long>(8192, (n + 255) / 256)); }

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

static DTaps2 d_upload(const Taps2& t, cudaStream_t st) {
    DTaps2 d;
    d.n0 = static_cast<long>(t.n0);
    d.n1 = static_cast<long>(t.n1);
    d.c0 = t.c0;
    d.c1 = t.c1;
    d.v->upload(t.v.data(), t.v.size(), st);
    return d;
}

static DTaps2 d_alloc(long n0, long n1, long c0, long c1) {
    DTaps2 d;
    d.n0 = n0;
    d.n1 = n1;
    d.c0 = c0;
    d.c1 = c1;
    d.v->alloc(static_cast<size_t>(n0 * n1));
    return d;
}

static DTaps2 d_upsample2(const DTaps2& g, long f0, long f1, cudaStream_t st) {
    if (f0 == 1 && f1 == 1) {
        DTaps2 d = d_alloc(g.n0, g.n1, g.c0, g.c1);
        SL_CUDA(cudaMemcpyAsync(d.v->p, g.p(), sizeof(double) * g.n0 * g.n1, cudaMemcpyDeviceToDevice, st));
        return d;
    }
    DTaps2 d = d_alloc((g.n0 - 1) * f0 + 1, (g.n1 - 1) * f1 + 1, g.c0 * f0, g.c1 * f1);
    kt_upsample2<<<blocks_for(d.n0 * d.n1), 256, 0, st>>>(g.p(), g.n0, g.n1, d.v->p, d.n0, d.n1, (int)f0, (int)f1);
    check_launch("kt_upsample2");
    return d;
}

static DTaps2 d_conv_axis(const DTaps2& g, const Taps1& t, int axis, DBuf<double>& tbuf, cudaStream_t st) {
    const long L = static_cast<long>(t.size());
    tbuf.upload(t.v.data(), t.v.size(), st);
    DTaps2 d = axis == 0 ? d_alloc(g.n0 + L - 1, g.n1, g.c0 + t.c, g.c1) : d_alloc(g.n0, g.n1 + L - 1, g.c0, g.c1 + t.c);
    kt_conv_axis<<<blocks_for(d.n0 * d.n1), 256, 0, st>>>(g.p(), g.n0, g.n1, tbuf.p, (int)L, axis, d.v->p, d.n0, d.n1);
    check_launch("kt_conv_axis");
    SL_CUDA(cudaStreamSynchronize(st));  // tbuf is reused by the next call
    return d;
}

static DTaps2 d_shear_support(const DTaps2& in, long k, cudaStream_t st) {
    if (k == 0) return d_upsample2(in, 1, 1, st);
    const long lo1 = -in.c1, hi1 = in.n1 - 1 - in.c1;
    const long lo0i = -in.c0, hi0i = in.n0 - 1 - in.c0;
    const long lo0 = std::min(lo0i - k * lo1, lo0i - k * hi1);
    const long hi0 = std::max(hi0i - k * lo1, hi0i - k * hi1);
    DTaps2 d = d_alloc(hi0 - lo0 + 1, in.n1, -lo0, in.c1);
    kt_shear_support<<<blocks_for(d.n0 * d.n1), 256, 0, st>>>(in.p(), in.n0, in.n1, in.c0, in.c1, k, d.v->p, d.n0, d.c0);
    check_launch("kt_shear_support");
    return d;
}

static DTaps2 d_digital_shear(const DTaps2& t, long k, int d, const Taps1& interp, DBuf<double>& tbuf, cudaStream_t st) {
    const long kmax = 1L << d;
    if (k < -kmax || k > kmax) throw SlError(SL_ERR_DOMAIN, "digital_shear_taps: |k| exceeds 2^d");
    if (d == 0) return d_shear_support(t, k, st);
    const long f = 1L << d;
    DTaps2 up = d_upsample2(t, f, 1, st);
    up = d_conv_axis(up, interp, 0, tbuf, st);
    up = d_shear_support(up, k, st);
    up = d_conv_axis(up, reversed(interp), 0, tbuf, st);
    const long lo = -up.c0, hi = up.n0 - 1 - up.c0;
    const long qlo = lo >= 0 ? (lo + f - 1) / f : -((-lo) / f);
    const long qhi = hi >= 0 ? hi / f : -((-hi + f - 1) / f);
    DTaps2 o = d_alloc(qhi - qlo + 1, up.n1, -qlo, up.c1);
    kt_decimate_rows<<<blocks_for(o.n0 * o.n1), 256, 0, st>>>(up.p(), up.n1, up.c0, f, qlo, o.v->p, o.n0);
    check_launch("kt_decimate_rows");
    return o;
}

static DTaps2 d_transposed(const DTaps2& g, cudaStream_t st) {
    DTaps2 d = d_alloc(g.n1, g.n0, g.c1, g.c0);
    kt_transpose<<<blocks_for(g.n0 * g.n1), 256, 0, st>>>(g.p(), g.n0, g.n1, d.v->p);
    check_launch("kt_transpose");
    return d;
}

// build_shearlet_taps (system2d.cpp:21-37) on the device
static DTaps2 d_cone_taps(int j, long k, int d, int J, const DTaps2& fan, const Qmf& q, DBuf<double>& tbuf,
                          cudaStream_t st) {
    const int lg = J - j, lh = J - (j - d);
    if (d < 0) throw SlError(SL_ERR_DOMAIN, "build_shearlet_taps: negative shear level");
    if (lg < 1 || lh < 0) throw SlError(SL_ERR_DOMAIN, "build_shearlet_taps: scale out of range");
    Taps1 g, h;
    cascade(q, lg, nullptr, &g);
    cascade(q, lh, &h, nullptr);
    DTaps2 p = d_upsample2(fan, 1L << (J - j - 1), 1L << lh, st);
    p = d_conv_axis(p, g, 0, tbuf, st);
    p = d_conv_axis(p, h, 1, tbuf, st);
    return d_digital_shear(p, k, d, shear_interp(q, d), tbuf, st);
}

// build_phi_component (system3d.cpp:13-25) on the device
static DTaps2 d_phi_taps(int j, long k, int d, int J, const DTaps2& fan, const Qmf& q, DBuf<double>& tbuf,
                         cudaStream_t st) {
    const int lh = J - (j - d);
    if (d < 0) throw SlError(SL_ERR_DOMAIN, "build_phi_component: negative shear level");
    if (J - j < 1 || lh < 0) throw SlError(SL_ERR_DOMAIN, "build_phi_component: scale out of range");
    Taps1 h;
    cascade(q, lh, &h, nullptr);
    DTaps2 p = d_upsample2(fan, 1L << (J - j - 1), 1L << lh, st);
    p = d_conv_axis(p, h, 1, tbuf, st);
    return d_digital_shear(p, k, d, shear_interp(q, d), tbuf, st);
}

}  // namespace slb
