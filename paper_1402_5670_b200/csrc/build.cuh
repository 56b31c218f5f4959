// System construction on the GPU (2D filter bank, 3D factor tables, W, RMS).
#pragma once
#include "launch.cuh"
#include "gpu_taps.cuh"
#include "fast2d_host.cuh"
#include "fast3d_host.cuh"

namespace slb {

// ---- small build kernels ------------------------------------------------------
// Periodic embedding with wrap-around accumulation (taps.cpp:101-111): a
// deterministic gather, summing source taps in the reference's (i, j) order.
__global__ void k_embed2d(const double* __restrict__ taps, int t0, int t1, long long c0, long long c1,
                          double* __restrict__ out, int n0, int n1) {
    const long long total = (long long)n0 * n1;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
        const int r0 = (int)(e / n1), r1 = (int)(e - (long long)r0 * n1);
        // taps index a satisfies (a - c0) mod n0 == r0  ->  a = r0 + c0 + m*n0
        long long a0 = (r0 + c0) % n0;
        if (a0 < 0) a0 += n0;
        long long b0 = (r1 + c1) % n1;
        if (b0 < 0) b0 += n1;
        double s = 0.0;
        for (long long a = a0; a < t0; a += n0)
            for (long long b = b0; b < t1; b += n1) s += taps[a * t1 + b];
        out[e] = s;
    }
}

// half complex spectrum -> real table; records max |im| and max |re| into
// maxabs[0..1] (bits of non-negative doubles order like unsigned integers)
__global__ void k_take_real(const double2* __restrict__ in, double* __restrict__ out, long long nhalf, int ldh, int H,
                            unsigned long long* __restrict__ maxabs) {
    unsigned long long mi = 0, mr = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf; e += (long long)gridDim.x * blockDim.x) {
        const double2 z = in[e];
        const bool pad = (e % ldh) >= H;
        out[e] = pad ? 0.0 : z.x;
        if (!pad) {
            mi = max(mi, (unsigned long long)__double_as_longlong(fabs(z.y)));
            mr = max(mr, (unsigned long long)__double_as_longlong(fabs(z.x)));
        }
    }
    atomicMax(maxabs, mi);
    atomicMax(maxabs + 1, mr);
}

// full real n0 x n1 spectrum from a half spectrum [n0][ldh] of an even filter
// (X(-a, -b) = X(a, b)), then (optionally) its transpose right after it
__global__ void k_expand_even(const double2* __restrict__ half, int n0, int n1, int ldh, double* __restrict__ out,
                              int with_transpose, unsigned long long* __restrict__ maxabs) {
    const int H = n1 / 2 + 1;
    const long long tot = (long long)n0 * n1;
    unsigned long long mi = 0, mr = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int a = (int)(e / n1), b = (int)(e - (long long)a * n1);
        const double2 z = b < H ? half[(long long)a * ldh + b] : half[(long long)((n0 - a) % n0) * ldh + (n1 - b)];
        out[e] = z.x;
        if (with_transpose) out[tot + (long long)b * n0 + a] = z.x;
        mi = max(mi, (unsigned long long)__double_as_longlong(fabs(z.y)));
        mr = max(mr, (unsigned long long)__double_as_longlong(fabs(z.x)));
    }
    atomicMax(maxabs, mi);
    atomicMax(maxabs + 1, mr);
}

// min / max of W over the valid half entries (bit order of non-negative doubles)
__global__ void k_minmax_w(const double* __restrict__ W, long long nhalf, int ldh, int H,
                           unsigned long long* __restrict__ mm) {
    unsigned long long lo = ~0ull, hi = 0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf; e += (long long)gridDim.x * blockDim.x) {
        if ((e % ldh) >= H) continue;
        const unsigned long long v = (unsigned long long)__double_as_longlong(W[e]);  // W >= 0
        lo = min(lo, v);
        hi = max(hi, v);
    }
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
}

// W[e] = sum_i psi_i[e]^2 over all filters in index order (system2d.cpp:118-126).
__global__ void k_weight2d(const double* __restrict__ psi, int R, long long nhalf, double* __restrict__ W) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf; e += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < R; ++i) {
            const double v = psi[(long long)i * nhalf + e];
            s += v * v;
        }
        W[e] = s;
    }
}

template <class Filt>
__global__ void k_weight_synth(Filt f, int R, long long nhalf, int ldh, int H, double* __restrict__ W) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf; e += (long long)gridDim.x * blockDim.x) {
        double s = 0.0;
        if ((e % ldh) < H)
            for (int i = 0; i < R; ++i) {
                const double v = f.get(i, e);
                s += v * v;
            }
        W[e] = (e % ldh) < H ? s : 1.0;
    }
}

// Per-band energy sum_full |psi|^2 from the half spectrum: columns k = 0 and
// k = L/2 (L even) count once, the others twice (Hermitian symmetry).
// Deterministic two-level reduction: partial[band][block].
template <class Filt>
__global__ void k_energy(Filt f, long long nhalf, int ldh, int H, int L, double* __restrict__ partial) {
    __shared__ double red[256];
    const int band = blockIdx.y;
    double s = 0.0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf; e += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(e % ldh);
        if (k >= H) continue;
        const double v = f.get(band, e);
        const double m = (k == 0 || 2 * k == L) ? 1.0 : 2.0;
        s += m * v * v;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[(long long)band * gridDim.x + blockIdx.x] = red[0];
}

struct FiltTable2DGet {
    FiltTable2D t;
    __device__ __forceinline__ double get(int band, long long e) const { return t.get(band, e); }
};
// complex filter spectra (asymmetric fans)
struct FiltTable2DCplx {
    const double2* psi;
    long long nhalf;
    __device__ __forceinline__ double2 get(int band, long long e) const { return __ldg(psi + (long long)band * nhalf + e); }
};
// |psi| of complex spectra, for the W / RMS reductions (sum of |psi|^2)
struct FiltTable2DAbs {
    const double2* psi;
    long long nhalf;
    __device__ __forceinline__ double get(int band, long long e) const {
        const double2 z = __ldg(psi + (long long)band * nhalf + e);
        return sqrt(z.x * z.x + z.y * z.y);
    }
};
// half complex spectrum (pad columns zeroed) into the complex table
__global__ void k_take_complex(const double2* __restrict__ in, double2* __restrict__ out, long long nhalf, int ldh,
                               int H) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf; e += (long long)gridDim.x * blockDim.x)
        out[e] = (e % ldh) >= H ? make_double2(0.0, 0.0) : in[e];
}

// [R][n0][ldh] row-major real halves -> [R][H][n0] column-major (fast 2D path)
__global__ void k_half_to_colmajor(const double* __restrict__ in, double* __restrict__ out, int R, int n0, int H,
                                   int ldh) {
    const long long tot = (long long)R * H * n0;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int r0 = (int)(e % n0);
        const long long t = e / n0;
        const int k = (int)(t % H);
        const int b = (int)(t / H);
        out[e] = in[((long long)b * n0 + r0) * ldh + k];
    }
}

// ------------------------------------------------------------------ build helpers
// Embed device-resident centred taps into an n0 x n1 periodic grid (wrap-sum)
// and r2c it on the GPU into `spec` ([n0][ldh] Hermitian half).
static void spectrum_2d_of_dtaps(System& s, const double* dt, long t0, long t1, long c0, long c1, int n0, int n1,
                                 DBuf<double>& grid, DBuf<double2>& spec, cudaStream_t st) {
    const int H = n1 / 2 + 1, ldh = (H + 7) / 8 * 8;
    grid.alloc(static_cast<size_t>(n0) * n1);
    spec.alloc(static_cast<size_t>(n0) * ldh);
    k_embed2d<<<std::min<long long>(4096, ((long long)n0 * n1 + 255) / 256), 256, 0, st>>>(
        dt, static_cast<int>(t0), static_cast<int>(t1), c0, c1, grid.p, n0, n1);
    check_launch("k_embed2d");
    rows_r2c(s, grid.p, 0, spec.p, 0, n0, n1, H, ldh, 1, st);
    if (n0 > 1) {
        LineGeom g{};
        g.L = n0;
        g.istride = ldh;
        g.ostride = 0;
        g.cw = ldh;
        g.ldh = ldh;
        g.H = H;
        g.n1 = 0;
        g.nhalf = static_cast<long long>(n0) * ldh;
        lines<-1, kPlain>(s, spec.p, 0, spec.p, 0, g, 1, 1, NoFilt{}, 0, nullptr, st);
    }
}
static void spectrum_2d_of_taps(System& s, const Taps2& t, int n0, int n1, DBuf<double>& dtaps, DBuf<double>& grid,
                                DBuf<double2>& spec, cudaStream_t st) {
    dtaps.upload(t.v.data(), t.v.size(), st);
    spectrum_2d_of_dtaps(s, dtaps.p, static_cast<long>(t.n0), static_cast<long>(t.n1), t.c0, t.c1, n0, n1, grid, spec,
                         st);
}

// |Im|/|Re| of the filter spectra, from per-filter device maxima (one copy at the end)
static double worst_imag_ratio(const DBuf<unsigned long long>& mx, int count, int* which, cudaStream_t st) {
    std::vector<unsigned long long> hm(2 * static_cast<size_t>(count));
    SL_CUDA(cudaMemcpyAsync(hm.data(), mx.p, hm.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    double worst = 0.0;
    for (int i = 0; i < count; ++i) {
        double im, re;
        std::memcpy(&im, &hm[2 * static_cast<size_t>(i)], 8);
        std::memcpy(&re, &hm[2 * static_cast<size_t>(i) + 1], 8);
        if (re > 0 && im / re > worst) {
            worst = im / re;
            if (which) *which = i;
        }
    }
    return worst;
}

static void finish_rms(System& s, const double* partial, int nblocks, int R) {
    s.rms.assign(static_cast<size_t>(R), 0.0);
    for (int i = 0; i < R; ++i) {
        double e = 0.0;
        for (int b = 0; b < nblocks; ++b) e += partial[static_cast<size_t>(i) * nblocks + b];
        s.rms[static_cast<size_t>(i)] = std::sqrt(e / static_cast<double>(s.nreal));
    }
}

static void finish_W(System& s, cudaStream_t st) {
    DBuf<unsigned long long> mm;
    mm.alloc(2);
    const unsigned long long init[2] = {~0ull, 0ull};
    SL_CUDA(cudaMemcpyAsync(mm.p, init, sizeof(init), cudaMemcpyHostToDevice, st));
    k_minmax_w<<<512, 256, 0, st>>>(s.W.p, s.nhalf, s.ldh, s.H, mm.p);
    check_launch("k_minmax_w");
    unsigned long long h[2];
    SL_CUDA(cudaMemcpyAsync(h, mm.p, sizeof(h), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    std::memcpy(&s.Wmin, &h[0], 8);
    std::memcpy(&s.Wmax, &h[1], 8);
}

static void init_geometry(System& s) {
    s.L_last = s.n[s.ndim - 1];
    s.H = s.L_last / 2 + 1;
    s.ldh = (s.H + 7) / 8 * 8;
    s.nreal = 1;
    for (int a = 0; a < s.ndim; ++a) s.nreal *= s.n[a];
    s.nrows = static_cast<int>(s.nreal / s.L_last);
    s.nhalf = static_cast<long long>(s.nrows) * s.ldh;
    for (int a = 0; a < s.ndim; ++a)
        if (s.n[a] > kMaxLen)
            throw SlError(SL_ERR_UNSUPPORTED_SIZE, "grid axis longer than " + std::to_string(kMaxLen));
    // bands per chunk: keep the complex intermediate around 32 MiB (L2-resident)
    const double per = static_cast<double>(s.nhalf) * sizeof(double2);
    s.chunk = std::max(1, static_cast<int>((32.0 * 1024 * 1024) / per));
}

static void validate_profile(const Profile& p) {
    for (int d : p.levels)
        if (d < 0) throw SlError(SL_ERR_CONFIG, "ScaleProfile: shear levels must be >= 0");
    if (p.j0 < 0) throw SlError(SL_ERR_CONFIG, "ScaleProfile: coarsest scale offset must be >= 0");
}

static Taps2 fan_of(int impulse_fan) {
    if (impulse_fan) return Taps2::impulse();
    Taps2 f = default_fan();
    if (fan_checksum(f) != kDefaultFanChecksum)
        throw SlError(SL_ERR_ASSET, "default_fan_filter: checksum mismatch on bundled fan filter");
    return f;
}

// The filter bank a system is built from: FanFilter + QmfPair (system2d.hpp:66-69).
struct Bank {
    Taps2 fan;
    Qmf qmf;
    std::string fan_name;  // descriptor name: "dmaxflat4", "impulse" or "custom" (descriptor.cpp:12-15)
};
static Bank default_bank(int impulse_fan) {
    return Bank{fan_of(impulse_fan), qmf_from_lowpass(maxflat9_lowpass()), impulse_fan ? "impulse" : "dmaxflat4"};
}

static void set_shard(System& s, int lo, int hi) {
    if (hi < 0) hi = s.R;
    if (lo < 0 || hi > s.R || lo >= hi) throw SlError(SL_ERR_CONFIG, "shard range outside the filter bank");
    s.lo = lo;
    s.hi = hi;
}

// 2D bank (system2d.cpp:75-116): every filter's taps are built, embedded and
// r2c'd on the device; no host round trip until the bank is complete.
static void build_2d(System& s, const Bank& bank, cudaStream_t st) {
    validate_profile(s.prof);
    s.index = enumerate_2d(s.prof, s.full);
    s.R = static_cast<int>(s.index.size());
    const int J = s.prof.top();
    const int n0 = s.n[0], n1 = s.n[1];
    s.psi.alloc(static_cast<size_t>(s.R) * s.nhalf);
    DBuf<double> grid;
    DBuf<double2> spec;
    DBuf<unsigned long long> mx;
    mx.alloc(2 * static_cast<size_t>(s.R));
    SL_CUDA(cudaMemsetAsync(mx.p, 0, 2 * static_cast<size_t>(s.R) * sizeof(unsigned long long), st));
    DQmf q(bank.qmf, st);
    const DTaps2 dfan = d_upload(bank.fan, st);
    s.psiC.alloc(static_cast<size_t>(s.R) * s.nhalf);  // released again for real (symmetric) banks
    for (int i = 0; i < s.R; ++i) {
        const Record& r = s.index[static_cast<size_t>(i)];
        DTaps2 t;
        if (r.kind == 0) {
            const DTaps1& hJ = q.lowpass(J, st);
            t = d_outer(hJ, hJ, st);
        } else {
            const int d = s.prof.levels[static_cast<size_t>(r.scale - s.prof.j0)];
            t = d_cone_taps(r.scale, r.k1, d, J, dfan, q, st);
            if (r.kind == 2) t = d_transposed(t, st);
        }
        spectrum_2d_of_dtaps(s, t.p(), t.n0, t.n1, t.c0, t.c1, n0, n1, grid, spec, st);
        k_take_real<<<256, 256, 0, st>>>(spec.p, s.psi.p + static_cast<size_t>(i) * s.nhalf, s.nhalf, s.ldh, s.H,
                                         mx.p + 2 * i);
        check_launch("k_take_real");
        k_take_complex<<<256, 256, 0, st>>>(spec.p, s.psiC.p + static_cast<size_t>(i) * s.nhalf, s.nhalf, s.ldh, s.H);
        check_launch("k_take_complex");
    }
    int worst_i = -1;
    const double worst = worst_imag_ratio(mx, s.R, &worst_i, st);
    // centrally symmetric banks (every default and maxflat fan) have real
    // spectra: real tables and the fast path. Asymmetric fans keep the
    // complex (Hermitian) spectra the reference stores (system2d.hpp:38) and
    // run the generic path.
    s.cplx = worst > s.knobs.real_tol;
    s.W.alloc(static_cast<size_t>(s.nhalf));
    const int nblk = 128;
    DBuf<double> part;
    part.alloc(static_cast<size_t>(s.R) * nblk);
    if (s.cplx) {
        FiltTable2DAbs fa{s.psiC.p, s.nhalf};
        k_weight_synth<<<1024, 256, 0, st>>>(fa, s.R, s.nhalf, s.ldh, s.H, s.W.p);
        check_launch("k_weight_synth");
        k_energy<<<dim3(nblk, s.R), 256, 0, st>>>(fa, s.nhalf, s.ldh, s.H, s.L_last, part.p);
        check_launch("k_energy");
    } else {
        k_weight2d<<<1024, 256, 0, st>>>(s.psi.p, s.R, s.nhalf, s.W.p);
        check_launch("k_weight2d");
        FiltTable2DGet f{FiltTable2D{s.psi.p, s.nhalf}};
        k_energy<<<dim3(nblk, s.R), 256, 0, st>>>(f, s.nhalf, s.ldh, s.H, s.L_last, part.p);
        check_launch("k_energy");
    }
    std::vector<double> hp(static_cast<size_t>(s.R) * nblk);
    SL_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    finish_rms(s, hp.data(), nblk, s.R);
    finish_W(s, st);
    if (s.cplx) {
        s.psi.release();
    } else {
        s.psiC.release();
    }
    if (!s.cplx && fast2d_supported(s.knobs, s.n[0], s.n[1])) {
        s.fast2d = true;
        s.psiT.alloc(static_cast<size_t>(s.R) * s.H * s.n[0]);
        s.WT.alloc(static_cast<size_t>(s.H) * s.n[0]);
        const long long tot = static_cast<long long>(s.R) * s.H * s.n[0];
        k_half_to_colmajor<<<std::min<long long>(8192, (tot + 255) / 256), 256, 0, st>>>(s.psi.p, s.psiT.p, s.R, s.n[0],
                                                                                          s.H, s.ldh);
        check_launch("k_half_to_colmajor");
        k_half_to_colmajor<<<std::min<long long>(8192, (s.H * (long long)s.n[0] + 255) / 256), 256, 0, st>>>(
            s.W.p, s.WT.p, 1, s.n[0], s.H, s.ldh);
        check_launch("k_half_to_colmajor");
        SL_CUDA(cudaStreamSynchronize(st));
    }
}

// 3D factor tables (system3d.cpp:82-142): per scale the 1D ĝ spectra and the
// 2K+1 Φ̂ planes (plus transposed copies for axis-0 lookups), and ĥ_J per
// axis, all built, r2c'd and expanded to full real spectra on the device,
// straight into the table buffers. W and RMS stream every synthesised filter.
static void build_3d(System& s, const Bank& bank, cudaStream_t st) {
    validate_profile(s.prof);
    s.index = enumerate_3d(s.prof, s.full);
    s.R = static_cast<int>(s.index.size());
    const int J = s.prof.top();
    DQmf q(bank.qmf, st);
    const DTaps2 dfan = d_upload(bank.fan, st);
    // ---- table layout (host bookkeeping only)
    struct Job {
        DTaps2 taps;
        int np, ns;
        bool tab2;  // plane (+ transpose) in tab2, else a 1D spectrum in tab1
        long long off;
    };
    std::vector<Job> jobs;
    long long n1d = 0, n2d = 0;
    auto add_1d = [&](const DTaps1& t, int n) {
        jobs.push_back(Job{d_as_row(t), 1, n, false, n1d});
        n1d += n;
        return static_cast<int>(jobs.back().off);
    };
    std::map<std::pair<int, int>, int> cache2;  // (taps id, n_p * 65536 + n_s) -> off
    auto add_2d = [&](const DTaps2& t, int tid, int np, int ns) {
        const auto key = std::make_pair(tid, np * 65536 + ns);
        auto it = cache2.find(key);
        if (it != cache2.end()) return it->second;
        jobs.push_back(Job{t, np, ns, true, n2d});
        n2d += 2LL * np * ns;  // plane + its transpose
        cache2[key] = static_cast<int>(jobs.back().off);
        return cache2[key];
    };
    FiltSynth3D syn{};
    for (int a = 0; a < 3; ++a) {
        syn.n[a] = s.n[a];
        syn.lp_off[a] = add_1d(q.lowpass(J, st), s.n[a]);
    }
    struct ScaleTabs {
        int d;
        std::vector<DTaps2> phi;  // device-built component taps
        std::map<int, int> goff;  // axis length -> offset
    };
    std::vector<ScaleTabs> sc(static_cast<size_t>(s.prof.n_scales()));
    int tid = 0;
    std::vector<std::vector<int>> phi_id(sc.size());
    for (int si = 0; si < s.prof.n_scales(); ++si) {
        const int j = s.prof.j0 + si;
        const int d = s.prof.levels[static_cast<size_t>(si)];
        auto& S = sc[static_cast<size_t>(si)];
        S.d = d;
        const int K = 1 << d;
        for (int k = -K; k <= K; ++k) {
            S.phi.push_back(d_phi_taps(j, k, d, J, dfan, q, st));
            phi_id[static_cast<size_t>(si)].push_back(tid++);
        }
    }
    static const int axes[6][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}, {0, 1, 2}, {1, 0, 2}, {2, 0, 1}};
    std::vector<BandDesc3D> bd(static_cast<size_t>(s.R));
    for (int i = 0; i < s.R; ++i) {
        const Record& r = s.index[static_cast<size_t>(i)];
        BandDesc3D& b = bd[static_cast<size_t>(i)];
        b.kind = r.kind;
        if (r.kind == 0) continue;
        const int si = r.scale - s.prof.j0;
        auto& S = sc[static_cast<size_t>(si)];
        const int K = 1 << S.d;
        b.pa = axes[r.kind][0];
        b.s1 = axes[r.kind][1];
        b.s2 = axes[r.kind][2];
        const int np = s.n[b.pa];
        auto git = S.goff.find(np);
        if (git == S.goff.end()) git = S.goff.emplace(np, add_1d(q.highpass(J - r.scale, st), np)).first;
        b.g_off = git->second;
        b.p1_off = add_2d(S.phi[static_cast<size_t>(r.k1 + K)],
                          phi_id[static_cast<size_t>(si)][static_cast<size_t>(r.k1 + K)], np, s.n[b.s1]);
        b.p2_off = add_2d(S.phi[static_cast<size_t>(r.k2 + K)],
                          phi_id[static_cast<size_t>(si)][static_cast<size_t>(r.k2 + K)], np, s.n[b.s2]);
    }
    // ---- spectra on the device, written straight into the tables
    s.tab1.alloc(static_cast<size_t>(std::max(1LL, n1d)));
    s.tab2.alloc(static_cast<size_t>(std::max(1LL, n2d)));
    DBuf<unsigned long long> mx;
    mx.alloc(2 * jobs.size());
    SL_CUDA(cudaMemsetAsync(mx.p, 0, 2 * jobs.size() * sizeof(unsigned long long), st));
    DBuf<double> grid;
    DBuf<double2> spec;
    for (size_t k = 0; k < jobs.size(); ++k) {
        const Job& jb = jobs[k];
        spectrum_2d_of_dtaps(s, jb.taps.p(), jb.taps.n0, jb.taps.n1, jb.taps.c0, jb.taps.c1, jb.np, jb.ns, grid, spec,
                             st);
        const int ldh = (jb.ns / 2 + 1 + 7) / 8 * 8;
        double* dst = jb.tab2 ? s.tab2.p + jb.off : s.tab1.p + jb.off;
        k_expand_even<<<blocks_for(static_cast<long long>(jb.np) * jb.ns), 256, 0, st>>>(
            spec.p, jb.np, jb.ns, ldh, dst, jb.tab2 ? 1 : 0, mx.p + 2 * k);
        check_launch("k_expand_even");
    }
    if (worst_imag_ratio(mx, static_cast<int>(jobs.size()), nullptr, st) > s.knobs.real_tol)
        throw SlError(SL_ERR_DOMAIN, "filter spectra are not real (asymmetric fan); unsupported by this build");
    s.bands3.upload(bd.data(), bd.size(), st);
    s.bands3_host = bd;
    syn.bands = s.bands3.p;
    syn.tab1d = s.tab1.p;
    syn.tab2d = s.tab2.p;
    s.synth = syn;
    FiltSynth3DFlat f{syn, s.ldh};
    s.W.alloc(static_cast<size_t>(s.nhalf));
    k_weight_synth<<<2048, 256, 0, st>>>(f, s.R, s.nhalf, s.ldh, s.H, s.W.p);
    check_launch("k_weight_synth");
    const int nblk = 128;
    DBuf<double> part;
    part.alloc(static_cast<size_t>(s.R) * nblk);
    k_energy<<<dim3(nblk, s.R), 256, 0, st>>>(f, s.nhalf, s.ldh, s.H, s.L_last, part.p);
    check_launch("k_energy");
    std::vector<double> hp(static_cast<size_t>(s.R) * nblk);
    SL_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    finish_rms(s, hp.data(), nblk, s.R);
    finish_W(s, st);
    if (fast3d_supported(s.knobs, s.n)) {
        s.fast3d = true;
        const int n = s.n[0];
        const long long tot = static_cast<long long>(s.H) * n * n;
        s.WN.alloc(static_cast<size_t>(tot));
        k3_half_to_natural<<<std::min<long long>(8192, (tot + 255) / 256), 256, 0, st>>>(s.W.p, s.WN.p, n, s.H, s.ldh);
        check_launch("k3_half_to_natural");
        SL_CUDA(cudaStreamSynchronize(st));
    }
}


}  // namespace slb
