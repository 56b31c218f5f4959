// Q / Q_opt separation-quality metrics (apps.cpp:282-362):
// Q(delta) = || blur(truth) - blur(binarize(recovered, delta)) || / || blur(truth) ||
// with a periodic Gaussian blur done in the frequency domain. The blur is the
// hot path's own single-band decomposition: a one-filter "system" whose filter
// is the embedded Gaussian's (real, even) spectrum, so blur(x) = Re IDFT(K F)
// runs on the same FFT kernels. Q_opt binarises at delta = 0..255, blurs all
// 256 images as one batch spread over the handle's streams, and reduces the
// squared errors per image in a fixed order (deterministic).
#pragma once
#include <cmath>
#include <limits>

#include "build.cuh"
#include "transform.cuh"

namespace slb {

// gaussian_kernel (apps.cpp:289-306): L1-normalised taps, radius ceil(4 sigma)
static Taps2 gaussian_taps(double sigma) {
    if (!(sigma > 0.0)) throw SlError(SL_ERR_DOMAIN, "gaussian_kernel: sigma must be > 0");
    const int radius = static_cast<int>(std::ceil(4.0 * sigma));
    const size_t n = static_cast<size_t>(2 * radius + 1);
    Taps2 t = Taps2::zeros(n, n, radius, radius);
    double sum = 0.0;
    for (int i = -radius; i <= radius; ++i)
        for (int j = -radius; j <= radius; ++j) {
            const double v = std::exp(-(static_cast<double>(i) * i + static_cast<double>(j) * j) / (2.0 * sigma * sigma));
            t.at(static_cast<size_t>(i + radius), static_cast<size_t>(j + radius)) = v;
            sum += v;
        }
    for (double& v : t.v) v /= sum;
    return t;
}

// one-band blur system on an n0 x n1 grid: psi = real spectrum of the embedded kernel
static void build_blur_2d(System& s, const Taps2& kernel, cudaStream_t st) {
    s.index = {Record{0, -1, 0, 0}};
    s.R = 1;
    s.lo = 0;
    s.hi = 1;
    s.psi.alloc(static_cast<size_t>(s.nhalf));
    DBuf<double> dtaps, grid;
    DBuf<double2> spec;
    DBuf<unsigned long long> mx;
    mx.alloc(2);
    spectrum_2d_of_taps(s, kernel, s.n[0], s.n[1], dtaps, grid, spec, st);
    SL_CUDA(cudaMemsetAsync(mx.p, 0, 2 * sizeof(unsigned long long), st));
    k_take_real<<<256, 256, 0, st>>>(spec.p, s.psi.p, s.nhalf, s.ldh, s.H, mx.p);
    check_launch("k_take_real");
    unsigned long long hm[2];
    SL_CUDA(cudaMemcpyAsync(hm, mx.p, sizeof(hm), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    double im, re;
    std::memcpy(&im, &hm[0], 8);
    std::memcpy(&re, &hm[1], 8);
    if (re > 0 && im / re > s.knobs.real_tol)
        throw SlError(SL_ERR_DOMAIN, "quality: blur kernel spectrum is not real (kernel not centrally symmetric)");
    s.rms.assign(1, 0.0);
    if (fast2d_supported(s.knobs, s.n[0], s.n[1])) {
        s.fast2d = true;
        s.psiT.alloc(static_cast<size_t>(s.H) * s.n[0]);
        k_half_to_colmajor<<<std::min<long long>(8192, (s.H * (long long)s.n[0] + 255) / 256), 256, 0, st>>>(
            s.psi.p, s.psiT.p, 1, s.n[0], s.H, s.ldh);
        check_launch("k_half_to_colmajor");
    }
    SL_CUDA(cudaStreamSynchronize(st));
}

// out[d][i] = |x[i]| >= d0 + d ? 1 : 0  (binarize, apps.cpp:282-287)
__global__ void k_binarize(const double* __restrict__ x, long long n, double d0, int nd, double* __restrict__ out) {
    const long long tot = n * nd;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int d = static_cast<int>(e / n);
        const long long i = e - static_cast<long long>(d) * n;
        out[e] = fabs(x[i]) >= d0 + d ? 1.0 : 0.0;
    }
}

// part[d][b] = sum over this block's strided elements of (ref - y[d])^2
__global__ void k_sq_err(const double* __restrict__ ref, const double* __restrict__ y, long long n,
                         double* __restrict__ part) {
    __shared__ double red[256];
    const double* yd = y + blockIdx.y * n;
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double d = (ref ? ref[i] : 0.0) - yd[i];
        acc = fma(d, d, acc);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.y * gridDim.x + blockIdx.x] = red[0];
}

struct QualityResult {
    double q = 0.0;
    int delta = 0;
};

// Q at the given deltas (nd consecutive integers from d0, or the single value d0).
// Returns the best (smallest q, ties: smallest delta) and all q's in `all`.
template <class FanOut>
static QualityResult quality_run(System& blur, const double* rec_h, const double* truth_h, double d0, int nd,
                                 FanOut&& fan_out_fn, cudaStream_t st, std::vector<double>* all = nullptr) {
    const long long N = blur.nreal;
    for (long long i = 0; i < N; ++i)
        if (truth_h[i] != 0.0 && truth_h[i] != 1.0) throw SlError(SL_ERR_DOMAIN, "quality_q: truth must be binary");
    DBuf<double> truth, rec, ref, bin, blurred, part;
    truth.upload(truth_h, static_cast<size_t>(N), st);
    rec.upload(rec_h, static_cast<size_t>(N), st);
    ref.alloc(static_cast<size_t>(N));
    dec(blur, truth.p, ref.p, nullptr, st);  // blur(truth)
    const int nblk = 64;
    part.alloc(static_cast<size_t>(nblk) * std::max(nd, 1));
    k_sq_err<<<dim3(nblk, 1), 256, 0, st>>>(nullptr, ref.p, N, part.p);
    check_launch("k_sq_err");
    std::vector<double> hp(static_cast<size_t>(nblk));
    SL_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    double rn2 = 0.0;
    for (double v : hp) rn2 += v;
    const double ref_norm = std::sqrt(rn2);
    if (ref_norm == 0.0) throw SlError(SL_ERR_DEGENERATE_TRUTH, "quality_q: truth carries no energy");
    bin.alloc(static_cast<size_t>(N) * nd);
    blurred.alloc(static_cast<size_t>(N) * nd);
    k_binarize<<<1024, 256, 0, st>>>(rec.p, N, d0, nd, bin.p);
    check_launch("k_binarize");
    fan_out_fn(nd, [&](int d, cudaStream_t fst) {
        dec(blur, bin.p + static_cast<size_t>(d) * N, blurred.p + static_cast<size_t>(d) * N, nullptr, fst);
    });
    k_sq_err<<<dim3(nblk, nd), 256, 0, st>>>(ref.p, blurred.p, N, part.p);
    check_launch("k_sq_err");
    hp.resize(static_cast<size_t>(nblk) * nd);
    SL_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    QualityResult best{std::numeric_limits<double>::infinity(), 0};
    for (int d = 0; d < nd; ++d) {
        double e2 = 0.0;
        for (int b = 0; b < nblk; ++b) e2 += hp[static_cast<size_t>(d) * nblk + b];
        const double q = std::sqrt(e2) / ref_norm;
        if (all) all->push_back(q);
        if (q < best.q) best = {q, static_cast<int>(d0) + d};
    }
    return best;
}

}  // namespace slb
