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

// half complex spectrum -> real table; records max |im| and max |re| (bits of
// non-negative doubles order like unsigned integers).
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
// Embed centred taps into an n0 x n1 periodic grid on the device and return
// its Hermitian-half spectrum [n0][ldh] in `spec` (GPU FFT).
static void spectrum_2d_of_dtaps(System& s, const double* dt, long t0, long t1, long c0, long c1, int n0, int n1,
                                 DBuf<double>& grid, DBuf<double2>& spec, cudaStream_t st);
static void spectrum_2d_of_taps(System& s, const Taps2& t, int n0, int n1, DBuf<double>& dtaps, DBuf<double>& grid,
                                DBuf<double2>& spec, cudaStream_t st) {
    dtaps.upload(t.v.data(), t.v.size(), st);
    spectrum_2d_of_dtaps(s, dtaps.p, static_cast<long>(t.n0), static_cast<long>(t.n1), t.c0, t.c1, n0, n1, grid, spec,
                         st);
}
// Embed device-resident centred taps into an n0 x n1 grid and r2c it (GPU).
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

// Full real spectrum (n0 x n1) of centred taps, expanded from the half by the
// even symmetry of symmetric taps; also returns max|im| / max|re| of the half.
static std::vector<double> real_spectrum_full(System& s, const DTaps2& t, int n0, int n1, double* im_ratio,
                                              cudaStream_t st) {
    DBuf<double> grid;
    DBuf<double2> spec;
    spectrum_2d_of_dtaps(s, t.p(), t.n0, t.n1, t.c0, t.c1, n0, n1, grid, spec, st);
    const int H = n1 / 2 + 1, ldh = (H + 7) / 8 * 8;
    std::vector<double2> h(static_cast<size_t>(n0) * ldh);
    SL_CUDA(cudaMemcpyAsync(h.data(), spec.p, h.size() * sizeof(double2), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    std::vector<double> full(static_cast<size_t>(n0) * n1);
    double mi = 0, mr = 0;
    for (int a = 0; a < n0; ++a)
        for (int b = 0; b < H; ++b) {
            const double2 z = h[static_cast<size_t>(a) * ldh + b];
            mi = std::max(mi, std::fabs(z.y));
            mr = std::max(mr, std::fabs(z.x));
        }
    for (int a = 0; a < n0; ++a)
        for (int b = 0; b < n1; ++b) {
            double v;
            if (b < H)
                v = h[static_cast<size_t>(a) * ldh + b].x;
            else
                v = h[static_cast<size_t>((n0 - a) % n0) * ldh + (n1 - b)].x;
            full[static_cast<size_t>(a) * n1 + b] = v;
        }
    *im_ratio = mr > 0 ? mi / mr : 0.0;
    return full;
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
    std::vector<double> w(static_cast<size_t>(s.nhalf));
    SL_CUDA(cudaMemcpyAsync(w.data(), s.W.p, w.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    double lo = INFINITY, hi = -INFINITY;
    for (long long e = 0; e < s.nhalf; ++e) {
        if ((e % s.ldh) >= s.H) continue;
        lo = std::min(lo, w[static_cast<size_t>(e)]);
        hi = std::max(hi, w[static_cast<size_t>(e)]);
    }
    s.Wmin = lo;
    s.Wmax = hi;
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
    Taps2 f = maxflat_fan(4);
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

static void build_2d(System& s, const Bank& bank, cudaStream_t st) {
    validate_profile(s.prof);
    const Taps2& fan = bank.fan;
    const Qmf& q = bank.qmf;
    s.index = enumerate_2d(s.prof, s.full);
    s.R = static_cast<int>(s.index.size());
    const int J = s.prof.top();
    const int n0 = s.n[0], n1 = s.n[1];
    s.psi.alloc(static_cast<size_t>(s.R) * s.nhalf);
    DBuf<double> dtaps, grid, tbuf;
    DBuf<double2> spec;
    DBuf<unsigned long long> mx;
    mx.alloc(2);
    const bool host_taps = std::getenv("SLB_HOST_TAPS") != nullptr;  // cross-check path
    const DTaps2 dfan = d_upload(fan, st);
    double worst = 0.0;
    int worst_i = -1;
    for (int i = 0; i < s.R; ++i) {
        const Record& r = s.index[static_cast<size_t>(i)];
        if (r.kind == 0) {
            Taps1 hJ;
            cascade(q, J, &hJ, nullptr);
            spectrum_2d_of_taps(s, outer(hJ, hJ), n0, n1, dtaps, grid, spec, st);
        } else if (host_taps) {
            const int d = s.prof.levels[static_cast<size_t>(r.scale - s.prof.j0)];
            Taps2 t = cone_taps(r.scale, r.k1, d, J, fan, q);
            if (r.kind == 2) t = transposed(t);
            spectrum_2d_of_taps(s, t, n0, n1, dtaps, grid, spec, st);
        } else {
            // upsampling, separable convolutions and the digital shear on the GPU
            const int d = s.prof.levels[static_cast<size_t>(r.scale - s.prof.j0)];
            DTaps2 t = d_cone_taps(r.scale, r.k1, d, J, dfan, q, tbuf, st);
            if (r.kind == 2) t = d_transposed(t, st);
            spectrum_2d_of_dtaps(s, t.p(), t.n0, t.n1, t.c0, t.c1, n0, n1, grid, spec, st);
        }
        SL_CUDA(cudaMemsetAsync(mx.p, 0, 2 * sizeof(unsigned long long), st));
        k_take_real<<<256, 256, 0, st>>>(spec.p, s.psi.p + static_cast<size_t>(i) * s.nhalf, s.nhalf, s.ldh, s.H, mx.p);
        check_launch("k_take_real");
        unsigned long long hm[2];
        SL_CUDA(cudaMemcpyAsync(hm, mx.p, sizeof(hm), cudaMemcpyDeviceToHost, st));
        SL_CUDA(cudaStreamSynchronize(st));
        double im, re;
        std::memcpy(&im, &hm[0], 8);
        std::memcpy(&re, &hm[1], 8);
        if (re > 0 && im / re > worst) {
            worst = im / re;
            worst_i = i;
        }
    }
    if (worst > s.knobs.real_tol)
        throw SlError(SL_ERR_DOMAIN, "filter spectra are not real (asymmetric fan; filter " + std::to_string(worst_i) +
                                         " has |im|/|re| = " + std::to_string(worst) + "); unsupported by this build");
    s.W.alloc(static_cast<size_t>(s.nhalf));
    k_weight2d<<<1024, 256, 0, st>>>(s.psi.p, s.R, s.nhalf, s.W.p);
    check_launch("k_weight2d");
    const int nblk = 128;
    DBuf<double> part;
    part.alloc(static_cast<size_t>(s.R) * nblk);
    FiltTable2DGet f{FiltTable2D{s.psi.p, s.nhalf}};
    k_energy<<<dim3(nblk, s.R), 256, 0, st>>>(f, s.nhalf, s.ldh, s.H, s.L_last, part.p);
    check_launch("k_energy");
    std::vector<double> hp(static_cast<size_t>(s.R) * nblk);
    SL_CUDA(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
    SL_CUDA(cudaStreamSynchronize(st));
    finish_rms(s, hp.data(), nblk, s.R);
    // pad entries of W are never read as divisors; set them to 1 for safety
    finish_W(s, st);
    if (fast2d_supported(s.knobs, s.n[0], s.n[1])) {
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

static void build_3d(System& s, const Bank& bank, cudaStream_t st) {
    validate_profile(s.prof);
    const Taps2& fan = bank.fan;
    const Qmf& q = bank.qmf;
    s.index = enumerate_3d(s.prof, s.full);
    s.R = static_cast<int>(s.index.size());
    const int J = s.prof.top();
    std::vector<double> tab1, tab2;
    double worst = 0.0;
    // 1D spectra: real even -> full length via symmetry.
    auto add_1d = [&](const Taps1& t, int n) {
        Taps2 t2 = Taps2::zeros(1, t.size(), 0, t.c);
        std::memcpy(t2.v.data(), t.v.data(), t.size() * sizeof(double));
        double r;
        std::vector<double> full = real_spectrum_full(s, d_upload(t2, st), 1, n, &r, st);
        worst = std::max(worst, r);
        const int off = static_cast<int>(tab1.size());
        tab1.insert(tab1.end(), full.begin(), full.end());
        return off;
    };
    std::map<std::pair<int, int>, int> cache2;  // (taps id, n_p * 65536 + n_s) -> off
    auto add_2d = [&](const DTaps2& t, int tid, int np, int ns) {
        const auto key = std::make_pair(tid, np * 65536 + ns);
        auto it = cache2.find(key);
        if (it != cache2.end()) return it->second;
        double r;
        std::vector<double> full = real_spectrum_full(s, t, np, ns, &r, st);
        worst = std::max(worst, r);
        const int off = static_cast<int>(tab2.size());
        tab2.insert(tab2.end(), full.begin(), full.end());
        // transposed copy right after the plane (ns x np): coalesced lookups
        // when the principal index runs along axis 0 (FiltSynth3D::get_d)
        for (int a = 0; a < ns; ++a)
            for (int p = 0; p < np; ++p) tab2.push_back(full[static_cast<size_t>(p) * ns + a]);
        cache2[key] = off;
        return off;
    };
    DBuf<double> tbuf;
    const DTaps2 dfan = d_upload(fan, st);
    Taps1 hJ;
    cascade(q, J, &hJ, nullptr);
    FiltSynth3D syn{};
    for (int a = 0; a < 3; ++a) {
        syn.n[a] = s.n[a];
        syn.lp_off[a] = add_1d(hJ, s.n[a]);
    }
    struct ScaleTabs {
        int d;
        Taps1 g;
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
        cascade(q, J - j, nullptr, &S.g);
        const int K = 1 << d;
        for (int k = -K; k <= K; ++k) {
            if (std::getenv("SLB_HOST_TAPS"))
                S.phi.push_back(d_upload(phi_taps(j, k, d, J, fan, q), st));
            else
                S.phi.push_back(d_phi_taps(j, k, d, J, dfan, q, tbuf, st));
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
        if (git == S.goff.end()) git = S.goff.emplace(np, add_1d(S.g, np)).first;
        b.g_off = git->second;
        b.p1_off = add_2d(S.phi[static_cast<size_t>(r.k1 + K)], phi_id[static_cast<size_t>(si)][static_cast<size_t>(r.k1 + K)],
                          np, s.n[b.s1]);
        b.p2_off = add_2d(S.phi[static_cast<size_t>(r.k2 + K)], phi_id[static_cast<size_t>(si)][static_cast<size_t>(r.k2 + K)],
                          np, s.n[b.s2]);
    }
    if (worst > s.knobs.real_tol)
        throw SlError(SL_ERR_DOMAIN, "filter spectra are not real (asymmetric fan); unsupported by this build");
    s.tab1.upload(tab1.data(), tab1.size(), st);
    s.tab2.upload(tab2.data(), tab2.size(), st);
    s.bands3.upload(bd.data(), bd.size(), st);
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
