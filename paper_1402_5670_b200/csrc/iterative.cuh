// Iterative-thresholding pipelines on the device (SURVEY.md 8f "next"):
// inpainting (apps.cpp:179-235) and geometric separation (apps.cpp:237-280).
// Every iteration is one fused dec -> uniform hard threshold -> rec, reusing
// the hot path; the residual updates are elementwise kernels and the whole
// loop stays on the GPU (no host round trips after the initial delta).
#pragma once
#include "transform.cuh"

namespace slb {

// residual = mask * (masked - est); residual += est   (apps.cpp:214-219)
__global__ void k_inpaint_residual(const double* __restrict__ masked, const double* __restrict__ mask,
                                   const double* __restrict__ est, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        double r = mask[i] * (masked[i] - est[i]);
        r += est[i];
        out[i] = r;
    }
}

// r = s - (c + b); arg0 = r + c; arg1 = r + b   (apps.cpp:262-272)
__global__ void k_separate_args(const double* __restrict__ sig, const double* __restrict__ c,
                                const double* __restrict__ b, double* __restrict__ arg0, double* __restrict__ arg1,
                                long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double r = sig[i] - (c[i] + b[i]);
        arg0[i] = r + c[i];
        arg1[i] = r + b[i];
    }
}

// per-band max |x| (bits of non-negative doubles order like unsigned ints)
__global__ void k_band_maxabs(const double* __restrict__ bands, long long n, unsigned long long* __restrict__ out) {
    const double* b = bands + (long long)blockIdx.y * n;
    double m = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        m = fmax(m, fabs(b[i]));
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out + blockIdx.y, (unsigned long long)__double_as_longlong(m));
}

static unsigned elem_blocks(long long n) { return static_cast<unsigned>(std::min<long long>(4096, (n + 255) / 256)); }

// max over bands of max|c_i| (/ RMS_i when scaled)  (apps.cpp:159-170)
static double max_band_amplitude(System& s, const double* stack, bool scaled, cudaStream_t st) {
    DBuf<unsigned long long> mx;
    mx.alloc(static_cast<size_t>(s.nb()));
    SL_CUDA(cudaMemsetAsync(mx.p, 0, sizeof(unsigned long long) * s.nb(), st));
    {
        LaunchScope ls(s, "band_maxabs", st, s.nb());
        k_band_maxabs<<<dim3(std::min<unsigned>(256, elem_blocks(s.nreal)), s.nb()), 256, 0, st>>>(stack, s.nreal, mx.p);
        check_launch("k_band_maxabs");
    }
    std::vector<unsigned long long> h(static_cast<size_t>(s.nb()));
    SL_CUDA(cudaMemcpyAsync(h.data(), mx.p, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    double m = 0.0;
    for (int i = 0; i < s.nb(); ++i) {
        double bm;
        std::memcpy(&bm, &h[static_cast<size_t>(i)], 8);
        const double nrm = s.rms[static_cast<size_t>(s.lo + i)];
        if (scaled && nrm > 0.0) bm /= nrm;
        m = std::max(m, bm);
    }
    return m;
}

// Per-iteration uniform thresholds delta_it * RMS_i (all bands, lowpass
// included: threshold_uniform, apps.cpp:149-157), uploaded once.
static void uniform_deltas(System& s, double delta0, double lambda, int iters, bool scaled, DBuf<double>& out,
                           cudaStream_t st) {
    std::vector<double> d(static_cast<size_t>(iters) * s.R);
    double delta = delta0;
    for (int it = 0; it < iters; ++it) {
        for (int i = 0; i < s.R; ++i)
            d[static_cast<size_t>(it) * s.R + i] = scaled ? delta * s.rms[static_cast<size_t>(i)] : delta;
        delta *= lambda;
    }
    out.alloc(d.size());
    SL_CUDA(cudaMemcpyAsync(out.p, d.data(), d.size() * sizeof(double), cudaMemcpyHostToDevice, st));
    SL_CUDA(cudaStreamSynchronize(st));  // host vector goes out of scope
}

static void validate_iter_config(int iterations, double delta_min) {
    if (iterations < 2) throw SlError(SL_ERR_CONFIG, "iterative thresholding needs at least 2 iterations");
    if (!(delta_min > 0.0 && delta_min < 1.0)) throw SlError(SL_ERR_CONFIG, "delta_min must lie in (0, 1)");
}

// inpaint (apps.cpp:179-235); masked/mask/out device pointers of the grid size.
static void inpaint(System& s, const double* masked, const double* mask, double* out, int iterations,
                    double delta_init, double delta_min, bool scaled, cudaStream_t st) {
    validate_iter_config(iterations, delta_min);
    if (s.nb() != s.R) throw SlError(SL_ERR_CONFIG, "inpaint needs the full (unsharded) system");
    // mask checks on the host copy (binary, masked signal vanishes off the mask)
    std::vector<double> hm(static_cast<size_t>(s.nreal)), hs(static_cast<size_t>(s.nreal));
    SL_CUDA(cudaMemcpyAsync(hm.data(), mask, hm.size() * 8, cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaMemcpyAsync(hs.data(), masked, hs.size() * 8, cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    bool any = false;
    for (size_t i = 0; i < hm.size(); ++i) {
        if (hm[i] != 0.0 && hm[i] != 1.0) throw SlError(SL_ERR_DOMAIN, "inpaint: mask must be binary");
        if (hm[i] == 1.0)
            any = true;
        else if (hs[i] != 0.0)
            throw SlError(SL_ERR_DOMAIN, "inpaint: masked signal must vanish off the mask");
    }
    if (!any) throw SlError(9, "inpaint: mask observes no pixels");
    s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
    double delta = delta_init;
    if (delta < 0.0) {
        dec(s, masked, s.stack.p, nullptr, st);
        delta = max_band_amplitude(s, s.stack.p, scaled, st);
    }
    const double lambda = std::pow(delta_min, 1.0 / static_cast<double>(iterations - 1));
    DBuf<double> dl, res;
    uniform_deltas(s, delta, lambda, iterations, scaled, dl, st);
    res.alloc(static_cast<size_t>(s.nreal));
    SL_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * s.nreal, st));  // estimate = 0
    // the per-iteration thresholded stacks are internal: the fused passes never
    // write them (bitwise the same result)
    for (int it = 0; it < iterations; ++it) {
        {
            LaunchScope ls(s, "inpaint_residual", st, 1);
            k_inpaint_residual<<<elem_blocks(s.nreal), 256, 0, st>>>(masked, mask, out, res.p, s.nreal);
            check_launch("k_inpaint_residual");
        }
        denoise(s, res.p, nullptr, out, dl.p + static_cast<size_t>(it) * s.R, st);
    }
    SL_CUDA(cudaStreamSynchronize(st));  // dl / res are freed on return
}

// separate (apps.cpp:237-280): curves with `dir`, blobs with `iso`.
static void separate(System& dir, System& iso, const double* signal, double* curves, double* blobs, int iterations,
                     double delta_init, double delta_min, bool scaled, cudaStream_t st) {
    validate_iter_config(iterations, delta_min);
    if (dir.ndim != 2 || iso.ndim != 2 || dir.n[0] != iso.n[0] || dir.n[1] != iso.n[1])
        throw SlError(SL_ERR_SHAPE, "separate: both systems must match the signal dims");
    if (dir.nb() != dir.R || iso.nb() != iso.R) throw SlError(SL_ERR_CONFIG, "separate needs full systems");
    dir.stack.alloc(static_cast<size_t>(dir.nb()) * dir.nreal);
    iso.stack.alloc(static_cast<size_t>(iso.nb()) * iso.nreal);
    double delta = delta_init;
    if (delta < 0.0) {
        dec(dir, signal, dir.stack.p, nullptr, st);
        const double m0 = max_band_amplitude(dir, dir.stack.p, scaled, st);
        dec(iso, signal, iso.stack.p, nullptr, st);
        const double m1 = max_band_amplitude(iso, iso.stack.p, scaled, st);
        delta = std::max(m0, m1);
    }
    const double lambda = std::pow(delta_min, 1.0 / static_cast<double>(iterations - 1));
    DBuf<double> d0, d1, a0, a1;
    uniform_deltas(dir, delta, lambda, iterations, scaled, d0, st);
    uniform_deltas(iso, delta, lambda, iterations, scaled, d1, st);
    a0.alloc(static_cast<size_t>(dir.nreal));
    a1.alloc(static_cast<size_t>(dir.nreal));
    SL_CUDA(cudaMemsetAsync(curves, 0, sizeof(double) * dir.nreal, st));
    SL_CUDA(cudaMemsetAsync(blobs, 0, sizeof(double) * dir.nreal, st));
    for (int it = 0; it < iterations; ++it) {
        {
            LaunchScope ls(dir, "separate_args", st, 1);
            k_separate_args<<<elem_blocks(dir.nreal), 256, 0, st>>>(signal, curves, blobs, a0.p, a1.p, dir.nreal);
            check_launch("k_separate_args");
        }
        denoise(dir, a0.p, nullptr, curves, d0.p + static_cast<size_t>(it) * dir.R, st);
        denoise(iso, a1.p, nullptr, blobs, d1.p + static_cast<size_t>(it) * iso.R, st);
    }
    SL_CUDA(cudaStreamSynchronize(st));
}

}  // namespace slb
