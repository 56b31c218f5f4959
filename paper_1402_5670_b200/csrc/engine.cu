// B200 shearlet engine: system construction on the GPU, dec/rec orchestration
// and the C ABI declared in include/shearlet_b200.h.
//
// Reference mapping (under /root/reference/proj/core):
//   build_system_2d   src/system2d.cpp:75-116   -> System::build_2d
//   build_system_3d   src/system3d.cpp:82-142   -> System::build_3d
//   forward 2D/3D     src/transform.cpp:13-61   -> dec_2d / dec_3d
//   inverse 2D/3D     src/transform.cpp:63-125  -> rec_2d / rec_3d
//   hard_threshold    src/apps.cpp:57-112       -> deltas() + k_threshold / fused epilogue
//   denoise           src/apps.cpp:114-121      -> sl_denoise_dev
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/shearlet_b200.h"
#include "kernels.cuh"
#include "taps.hpp"

namespace slb {

// ------------------------------------------------------------------ errors
struct SlError : std::runtime_error {
    int code;
    SlError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SL_CUDA(x)                                                                                  \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess)                                                                      \
            throw SlError(SL_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));            \
    } while (0)

static void check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw SlError(SL_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------ device buffers
template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    DBuf() = default;
    DBuf(const DBuf&) = delete;
    DBuf& operator=(const DBuf&) = delete;
    ~DBuf() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    void alloc(size_t count) {
        if (count <= n && p) return;
        release();
        if (count == 0) return;
        SL_CUDA(cudaMalloc(&p, count * sizeof(T)));
        n = count;
    }
    // Synchronous upload (construction time only). The copy is ordered on the
    // stream that consumes it and completed before returning: a pageable
    // cudaMemcpy may return before its DMA lands, and kernels on a non-blocking
    // stream are not ordered after the legacy stream.
    void upload(const T* h, size_t count, cudaStream_t st) {
        SL_CUDA(cudaStreamSynchronize(st));
        alloc(count);
        SL_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, st));
        SL_CUDA(cudaStreamSynchronize(st));
    }
};

// ------------------------------------------------------------------ FFT plans
struct PlanHolder {
    FftPlan plan;
    DBuf<double2> tw;
};

static std::vector<int> factor_radices(int L) {
    std::vector<int> r;
    int m = L;
    while (m % 8 == 0) { r.push_back(8); m /= 8; }
    while (m % 4 == 0) { r.push_back(4); m /= 4; }
    while (m % 2 == 0) { r.push_back(2); m /= 2; }
    while (m % 3 == 0) { r.push_back(3); m /= 3; }
    while (m % 5 == 0) { r.push_back(5); m /= 5; }
    for (int f = 7; m > 1; f += 2)
        while (m % f == 0) { r.push_back(f); m /= f; }
    return r;
}

static void make_plan(int L, PlanHolder& ph, cudaStream_t st) {
    const std::vector<int> r = factor_radices(L);
    if (static_cast<int>(r.size()) > kMaxStages) throw SlError(SL_ERR_UNSUPPORTED_SIZE, "FFT length has too many factors");
    for (int x : r)
        if (x > 64) throw SlError(SL_ERR_UNSUPPORTED_SIZE, "FFT length has a prime factor > 64");
    ph.plan.L = L;
    ph.plan.nst = static_cast<int>(r.size());
    int ns = 1;
    for (size_t s = 0; s < r.size(); ++s) {
        ph.plan.radix[s] = r[s];
        ph.plan.ns[s] = ns;
        ns *= r[s];
    }
    std::vector<double2> tw(static_cast<size_t>(L));
    for (int k = 0; k < L; ++k) {
        const long double a = -2.0L * 3.141592653589793238462643383279502884L * k / L;
        tw[static_cast<size_t>(k)] = make_double2(static_cast<double>(cosl(a)), static_cast<double>(sinl(a)));
    }
    ph.tw.upload(tw.data(), tw.size(), st);
    ph.plan.tw = ph.tw.p;
}

// ------------------------------------------------------------------ launch helpers
static constexpr int kMaxLen = 4096;  // per-line FFT length limit (shared-memory tile)

struct LineCfg {
    int V;
    size_t smem;
    int threads;
};

// Lines per CTA so that a tile is ~4096 complex (64 KiB per ping-pong buffer).
static LineCfg line_cfg(int L, bool strided) {
    int V = std::max(1, 4096 / L);
    if (strided) V = std::max(V, 8);
    V = std::min(V, 64);
    while (V > 1 && 2ull * V * (L + 1) * sizeof(double2) > 200 * 1024) V /= 2;
    LineCfg c;
    c.V = V;
    c.smem = 2ull * V * (L + 1) * sizeof(double2);
    c.threads = 256;
    return c;
}

template <class K>
static void set_smem(K kern, size_t smem) {
    static std::mutex mu;
    static std::map<const void*, size_t> done;
    std::lock_guard<std::mutex> lk(mu);
    auto it = done.find(reinterpret_cast<const void*>(kern));
    if (it != done.end() && it->second >= smem) return;
    SL_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    done[reinterpret_cast<const void*>(kern)] = smem;
}

// ------------------------------------------------------------------ system
struct System {
    int ndim = 2;
    int n[3] = {1, 1, 1};
    int L_last = 0, H = 0, ldh = 0;
    long long nreal = 0, nhalf = 0;
    int nrows = 0;  // product of the leading dims
    Profile prof;
    bool full = false;
    int device = 0;
    std::vector<Record> index;
    int R = 0;
    int lo = 0, hi = 0;  // shard
    std::vector<double> rms;
    double Wmin = 0, Wmax = 0;

    std::map<int, std::unique_ptr<PlanHolder>> plans;
    DBuf<double> psi;   // 2D: [R][nhalf] real
    DBuf<double> W;     // [nhalf]
    // 3D synthesis tables
    DBuf<BandDesc3D> bands3;
    DBuf<double> tab1, tab2;
    FiltSynth3D synth{};
    // scratch
    DBuf<double2> F, inter, acc;
    DBuf<double> delta, stack, io_in, io_out;
    int chunk = 1;
    std::mutex mu;

    int nb() const { return hi - lo; }

    const FftPlan& plan(int L, cudaStream_t st) {
        auto it = plans.find(L);
        if (it != plans.end()) return it->second->plan;
        auto ph = std::make_unique<PlanHolder>();
        make_plan(L, *ph, st);
        const FftPlan& p = ph->plan;
        plans[L] = std::move(ph);
        return p;
    }
};

// ---- generic pass launchers ------------------------------------------------
static void rows_r2c(System& s, const double* src, long long sbs, double2* dst, long long dbs, int nrows, int L,
                     int H, int ldh, int nbatch, cudaStream_t st) {
    const FftPlan& p = s.plan(L, st);
    LineCfg c = line_cfg(L, false);
    set_smem(k_rows_r2c, c.smem);
    const int npairs = (nrows + 1) / 2;
    dim3 grid((npairs + c.V - 1) / c.V, nbatch);
    k_rows_r2c<<<grid, c.threads, c.smem, st>>>(src, sbs, dst, dbs, nrows, H, ldh, p, c.V);
    check_launch("k_rows_r2c");
}

static void rows_c2r(System& s, const double2* src, long long sbs, double* dst, long long dbs, int nrows, int L,
                     int H, int ldh, int nbatch, double scale, const double* delta, int band_base, cudaStream_t st) {
    const FftPlan& p = s.plan(L, st);
    LineCfg c = line_cfg(L, false);
    set_smem(k_rows_c2r, c.smem);
    const int npairs = (nrows + 1) / 2;
    dim3 grid((npairs + c.V - 1) / c.V, nbatch);
    k_rows_c2r<<<grid, c.threads, c.smem, st>>>(src, sbs, dst, dbs, nrows, H, ldh, p, c.V, scale, delta, band_base);
    check_launch("k_rows_c2r");
}

template <int DIR, int MODE, class Filt>
static void lines(System& s, const double2* src, long long sbs, double2* dst, long long dbs, const LineGeom& g,
                  int outer, int nbatch, const Filt& filt, int band_base, const double* W, cudaStream_t st) {
    const FftPlan& p = s.plan(g.L, st);
    LineCfg c = line_cfg(g.L, true);
    auto kern = k_lines<DIR, MODE, Filt>;
    set_smem(kern, c.smem);
    const int tiles = (g.cw + c.V - 1) / c.V;
    dim3 grid(outer * tiles, nbatch);
    kern<<<grid, c.threads, c.smem, st>>>(src, sbs, dst, dbs, g, p, c.V, filt, band_base, W);
    check_launch("k_lines");
}

// Geometry of the strided axes of a half spectrum.
static LineGeom geom_axis(const System& s, int axis, int* outer) {
    LineGeom g{};
    g.ldh = s.ldh;
    g.H = s.H;
    g.nhalf = s.nhalf;
    g.n1 = s.ndim == 3 ? s.n[1] : 0;
    if (s.ndim == 2) {
        g.L = s.n[0];
        g.istride = s.ldh;
        g.ostride = 0;
        g.cw = s.ldh;
        *outer = 1;
    } else if (axis == 0) {
        g.L = s.n[0];
        g.istride = static_cast<long long>(s.n[1]) * s.ldh;
        g.ostride = 0;
        g.cw = s.n[1] * s.ldh;
        *outer = 1;
    } else {
        g.L = s.n[1];
        g.istride = s.ldh;
        g.ostride = static_cast<long long>(s.n[1]) * s.ldh;
        g.cw = s.ldh;
        *outer = s.n[0];
    }
    return g;
}

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

// ------------------------------------------------------------------ build helpers
// Embed centred taps into an n0 x n1 periodic grid on the device and return
// its Hermitian-half spectrum [n0][ldh] in `spec` (GPU FFT).
static void spectrum_2d_of_taps(System& s, const Taps2& t, int n0, int n1, DBuf<double>& dtaps, DBuf<double>& grid,
                                DBuf<double2>& spec, cudaStream_t st) {
    const int H = n1 / 2 + 1, ldh = (H + 7) / 8 * 8;
    dtaps.upload(t.v.data(), t.v.size(), st);
    grid.alloc(static_cast<size_t>(n0) * n1);
    spec.alloc(static_cast<size_t>(n0) * ldh);
    k_embed2d<<<std::min<long long>(4096, ((long long)n0 * n1 + 255) / 256), 256, 0, st>>>(
        dtaps.p, static_cast<int>(t.n0), static_cast<int>(t.n1), t.c0, t.c1, grid.p, n0, n1);
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
static std::vector<double> real_spectrum_full(System& s, const Taps2& t, int n0, int n1, double* im_ratio,
                                              cudaStream_t st) {
    DBuf<double> dtaps, grid;
    DBuf<double2> spec;
    spectrum_2d_of_taps(s, t, n0, n1, dtaps, grid, spec, st);
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

// Filters must be real to this relative level (override: SLB_REAL_TOL, debugging only).
static double real_tol() {
    const char* e = std::getenv("SLB_REAL_TOL");
    return e ? std::atof(e) : 1e-9;
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

static void set_shard(System& s, int lo, int hi) {
    if (hi < 0) hi = s.R;
    if (lo < 0 || hi > s.R || lo >= hi) throw SlError(SL_ERR_CONFIG, "shard range outside the filter bank");
    s.lo = lo;
    s.hi = hi;
}

static void build_2d(System& s, int impulse_fan, cudaStream_t st) {
    validate_profile(s.prof);
    const Taps2 fan = fan_of(impulse_fan);
    const Qmf q = qmf_from_lowpass(maxflat9_lowpass());
    s.index = enumerate_2d(s.prof, s.full);
    s.R = static_cast<int>(s.index.size());
    const int J = s.prof.top();
    const int n0 = s.n[0], n1 = s.n[1];
    s.psi.alloc(static_cast<size_t>(s.R) * s.nhalf);
    DBuf<double> dtaps, grid;
    DBuf<double2> spec;
    DBuf<unsigned long long> mx;
    mx.alloc(2);
    double worst = 0.0;
    int worst_i = -1;
    for (int i = 0; i < s.R; ++i) {
        const Record& r = s.index[static_cast<size_t>(i)];
        Taps2 t;
        if (r.kind == 0) {
            Taps1 hJ;
            cascade(q, J, &hJ, nullptr);
            t = outer(hJ, hJ);
        } else {
            const int d = s.prof.levels[static_cast<size_t>(r.scale - s.prof.j0)];
            t = cone_taps(r.scale, r.k1, d, J, fan, q);
            if (r.kind == 2) t = transposed(t);
        }
        spectrum_2d_of_taps(s, t, n0, n1, dtaps, grid, spec, st);
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
    if (worst > real_tol())
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
}

static void build_3d(System& s, int impulse_fan, cudaStream_t st) {
    validate_profile(s.prof);
    const Taps2 fan = fan_of(impulse_fan);
    const Qmf q = qmf_from_lowpass(maxflat9_lowpass());
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
        std::vector<double> full = real_spectrum_full(s, t2, 1, n, &r, st);
        worst = std::max(worst, r);
        const int off = static_cast<int>(tab1.size());
        tab1.insert(tab1.end(), full.begin(), full.end());
        return off;
    };
    std::map<std::pair<int, int>, int> cache2;  // (taps id, n_p * 65536 + n_s) -> off
    auto add_2d = [&](const Taps2& t, int tid, int np, int ns) {
        const auto key = std::make_pair(tid, np * 65536 + ns);
        auto it = cache2.find(key);
        if (it != cache2.end()) return it->second;
        double r;
        std::vector<double> full = real_spectrum_full(s, t, np, ns, &r, st);
        worst = std::max(worst, r);
        const int off = static_cast<int>(tab2.size());
        tab2.insert(tab2.end(), full.begin(), full.end());
        cache2[key] = off;
        return off;
    };
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
        std::vector<Taps2> phi;
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
            S.phi.push_back(phi_taps(j, k, d, J, fan, q));
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
    if (worst > real_tol())
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
}

// ------------------------------------------------------------------ thresholds
// delta_i = K[scale - j0] * sigma (* RMS_i) for this handle's bands; -1 for the
// lowpass (untouched). Validation as hard_threshold_impl (apps.cpp:59-67).
static void deltas(System& s, const double* K, int nK, double sigma, int scaled, cudaStream_t st) {
    if (nK != s.prof.n_scales()) throw SlError(SL_ERR_CONFIG, "hard_threshold: schedule length must equal n_scales");
    if (sigma < 0.0) throw SlError(SL_ERR_CONFIG, "hard_threshold: sigma must be >= 0");
    for (int i = 0; i < nK; ++i)
        if (!(K[i] > 0.0)) throw SlError(SL_ERR_CONFIG, "hard_threshold: factors must be positive");
    std::vector<double> d(static_cast<size_t>(s.R), -1.0);
    for (int i = 0; i < s.R; ++i) {
        const Record& r = s.index[static_cast<size_t>(i)];
        if (r.scale < 0) continue;
        double dl = K[r.scale - s.prof.j0] * sigma;
        if (scaled) dl *= s.rms[static_cast<size_t>(i)];
        d[static_cast<size_t>(i)] = dl;
    }
    s.delta.alloc(d.size());
    SL_CUDA(cudaMemcpyAsync(s.delta.p, d.data(), d.size() * sizeof(double), cudaMemcpyHostToDevice, st));
}

// ------------------------------------------------------------------ transforms
static void forward_spectrum(System& s, const double* f, cudaStream_t st) {
    s.F.alloc(static_cast<size_t>(s.nhalf));
    rows_r2c(s, f, 0, s.F.p, 0, s.nrows, s.L_last, s.H, s.ldh, 1, st);
    if (s.ndim == 3) {
        int outer;
        LineGeom g1 = geom_axis(s, 1, &outer);
        lines<-1, kPlain>(s, s.F.p, 0, s.F.p, 0, g1, outer, 1, NoFilt{}, 0, nullptr, st);
    }
    int outer;
    LineGeom g0 = geom_axis(s, 0, &outer);
    lines<-1, kPlain>(s, s.F.p, 0, s.F.p, 0, g0, outer, 1, NoFilt{}, 0, nullptr, st);
}

template <class Filt>
static void dec_bands(System& s, const Filt& filt, double* out, const double* delta, cudaStream_t st) {
    const int nb = s.nb();
    const int C = std::min(s.chunk, nb);
    s.inter.alloc(static_cast<size_t>(C) * s.nhalf);
    const double scale = 1.0 / static_cast<double>(s.nreal);
    int outer0, outer1 = 1;
    LineGeom g0 = geom_axis(s, 0, &outer0);
    LineGeom g1{};
    if (s.ndim == 3) g1 = geom_axis(s, 1, &outer1);
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        lines<+1, kDecMul>(s, s.F.p, 0, s.inter.p, s.nhalf, g0, outer0, cb, filt, s.lo + b0, nullptr, st);
        if (s.ndim == 3)
            lines<+1, kPlain>(s, s.inter.p, s.nhalf, s.inter.p, s.nhalf, g1, outer1, cb, NoFilt{}, 0, nullptr, st);
        rows_c2r(s, s.inter.p, s.nhalf, out + static_cast<size_t>(b0) * s.nreal, s.nreal, s.nrows, s.L_last, s.H,
                 s.ldh, cb, scale, delta, s.lo + b0, st);
    }
}

template <class Filt>
static void rec_bands(System& s, const Filt& filt, const double* coeffs, double* out, cudaStream_t st) {
    const int nb = s.nb();
    const int C = std::min(s.chunk, nb);
    s.inter.alloc(static_cast<size_t>(C) * s.nhalf);
    s.acc.alloc(static_cast<size_t>(s.nhalf));
    int outer0, outer1 = 1;
    LineGeom g0 = geom_axis(s, 0, &outer0);
    LineGeom g1{};
    if (s.ndim == 3) g1 = geom_axis(s, 1, &outer1);
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        rows_r2c(s, coeffs + static_cast<size_t>(b0) * s.nreal, s.nreal, s.inter.p, s.nhalf, s.nrows, s.L_last, s.H,
                 s.ldh, cb, st);
        if (s.ndim == 3)
            lines<-1, kPlain>(s, s.inter.p, s.nhalf, s.inter.p, s.nhalf, g1, outer1, cb, NoFilt{}, 0, nullptr, st);
        lines<-1, kRecMul>(s, s.inter.p, s.nhalf, s.inter.p, s.nhalf, g0, outer0, cb, filt, s.lo + b0, nullptr, st);
        k_reduce_bands<<<1184, 256, 0, st>>>(s.acc.p, s.inter.p, s.nhalf, cb, b0 > 0);
        check_launch("k_reduce_bands");
    }
    // acc / W, then the inverse transform of the single accumulated spectrum
    lines<+1, kDivW>(s, s.acc.p, 0, s.acc.p, 0, g0, outer0, 1, NoFilt{}, 0, s.W.p, st);
    if (s.ndim == 3) lines<+1, kPlain>(s, s.acc.p, 0, s.acc.p, 0, g1, outer1, 1, NoFilt{}, 0, nullptr, st);
    rows_c2r(s, s.acc.p, 0, out, 0, s.nrows, s.L_last, s.H, s.ldh, 1, 1.0 / static_cast<double>(s.nreal), nullptr, 0,
             st);
}

static void dec(System& s, const double* f, double* out, const double* delta, cudaStream_t st) {
    forward_spectrum(s, f, st);
    if (s.ndim == 2)
        dec_bands(s, FiltTable2DGet{FiltTable2D{s.psi.p, s.nhalf}}, out, delta, st);
    else
        dec_bands(s, FiltSynth3DFlat{s.synth, s.ldh}, out, delta, st);
}

static void rec(System& s, const double* coeffs, double* out, cudaStream_t st) {
    if (s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
    if (s.ndim == 2)
        rec_bands(s, FiltTable2DGet{FiltTable2D{s.psi.p, s.nhalf}}, coeffs, out, st);
    else
        rec_bands(s, FiltSynth3DFlat{s.synth, s.ldh}, coeffs, out, st);
}

// materialise one synthesised 3D filter (half spectrum) for API queries
__global__ void k_synth_band(FiltSynth3DFlat f, int band, long long nhalf, double* out) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf; e += (long long)gridDim.x * blockDim.x)
        out[e] = ((e % f.ldh) < f.s.n[2] / 2 + 1) ? f.get(band, e) : 0.0;
}

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

// ====================================================================== C ABI
using namespace slb;

struct sl_system {
    System s;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return SL_OK;
    } catch (const SlError& e) {
        g_err = e.what();
        return e.code;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return SL_ERR_DOMAIN;
    } catch (const std::bad_alloc& e) {
        g_err = "host allocation failed";
        return SL_ERR_GENERIC;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SL_ERR_GENERIC;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) SL_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

System& sys_of(sl_system* h) {
    if (!h) throw SlError(SL_ERR_INVALID, "null system handle");
    return h->s;
}
const System& sys_of(const sl_system* h) {
    if (!h) throw SlError(SL_ERR_INVALID, "null system handle");
    return h->s;
}
cudaStream_t stream_of(void* st) { return static_cast<cudaStream_t>(st); }

void require_dev_ptr(const void* p, const char* what) {
    if (!p) throw SlError(SL_ERR_INVALID, std::string(what) + ": null pointer");
}

int create(int ndim, const int* n, const int* levels, int n_scales, int j0, int full, int impulse_fan, int device,
           int lo, int hi, sl_system** out) {
    return guard([&] {
        if (!out) throw SlError(SL_ERR_INVALID, "null output handle");
        *out = nullptr;
        if (n_scales < 0) throw SlError(SL_ERR_CONFIG, "ScaleProfile: n_scales must be >= 0");
        if (n_scales > 0 && !levels) throw SlError(SL_ERR_INVALID, "null levels");
        for (int a = 0; a < ndim; ++a)
            if (n[a] < 8)
                throw SlError(SL_ERR_UNSUPPORTED_SIZE, ndim == 2 ? "build_system_2d: grid must be at least 8x8"
                                                                 : "build_system_3d: each dim must be >= 8");
        DeviceGuard dg(device);
        auto h = std::make_unique<sl_system>();
        System& s = h->s;
        s.ndim = ndim;
        for (int a = 0; a < ndim; ++a) s.n[a] = n[a];
        s.prof.levels.assign(levels, levels + n_scales);
        s.prof.j0 = j0;
        s.full = full != 0;
        s.device = device;
        init_geometry(s);
        cudaStream_t st;
        SL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        try {
            if (ndim == 2)
                build_2d(s, impulse_fan, st);
            else
                build_3d(s, impulse_fan, st);
            SL_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        cudaStreamDestroy(st);
        set_shard(s, lo, hi);
        *out = h.release();
    });
}
}  // namespace

extern "C" {

const char* sl_version(void) { return "shearlet_b200 0.1 (sm_100a fp64)"; }
const char* sl_last_error(void) { return g_err.c_str(); }

int sl_device_count(int* count) {
    return guard([&] {
        if (!count) throw SlError(SL_ERR_INVALID, "null count");
        SL_CUDA(cudaGetDeviceCount(count));
    });
}

int sl_system_create_2d(int rows, int cols, const int* levels, int n_scales, int j0, int full_system, int impulse_fan,
                        int device, int shard_lo, int shard_hi, sl_system** out) {
    const int n[2] = {rows, cols};
    return create(2, n, levels, n_scales, j0, full_system, impulse_fan, device, shard_lo, shard_hi, out);
}

int sl_system_create_3d(int n0, int n1, int n2, const int* levels, int n_scales, int j0, int full_system,
                        int impulse_fan, int device, int shard_lo, int shard_hi, sl_system** out) {
    const int n[3] = {n0, n1, n2};
    return create(3, n, levels, n_scales, j0, full_system, impulse_fan, device, shard_lo, shard_hi, out);
}

int sl_system_destroy(sl_system* sys) {
    return guard([&] {
        if (!sys) return;
        DeviceGuard dg(sys->s.device);
        delete sys;
    });
}

int sl_ndim(const sl_system* h, int* ndim, int64_t dims[3]) {
    return guard([&] {
        const System& s = sys_of(h);
        if (ndim) *ndim = s.ndim;
        if (dims)
            for (int a = 0; a < 3; ++a) dims[a] = a < s.ndim ? s.n[a] : 1;
    });
}

int sl_redundancy(const sl_system* h, int* R) {
    return guard([&] {
        if (!R) throw SlError(SL_ERR_INVALID, "null R");
        *R = sys_of(h).R;
    });
}

int sl_shard(const sl_system* h, int* lo, int* hi) {
    return guard([&] {
        const System& s = sys_of(h);
        if (lo) *lo = s.lo;
        if (hi) *hi = s.hi;
    });
}

int sl_index(const sl_system* h, int32_t* rec) {
    return guard([&] {
        const System& s = sys_of(h);
        if (!rec) throw SlError(SL_ERR_INVALID, "null records");
        for (int i = 0; i < s.R; ++i) {
            const Record& r = s.index[static_cast<size_t>(i)];
            rec[4 * i] = r.kind;
            rec[4 * i + 1] = r.scale;
            rec[4 * i + 2] = r.k1;
            rec[4 * i + 3] = r.k2;
        }
    });
}

int sl_filter_norms(const sl_system* h, double* rms) {
    return guard([&] {
        const System& s = sys_of(h);
        if (!rms) throw SlError(SL_ERR_INVALID, "null output");
        std::memcpy(rms, s.rms.data(), s.rms.size() * sizeof(double));
    });
}

int sl_frame_bounds(const sl_system* h, double* A, double* B) {
    return guard([&] {
        const System& s = sys_of(h);
        if (A) *A = s.Wmin;
        if (B) *B = s.Wmax;
    });
}

int sl_frame_weight(const sl_system* h, double* w) {
    return guard([&] {
        const System& s = sys_of(h);
        if (!w) throw SlError(SL_ERR_INVALID, "null output");
        DeviceGuard dg(s.device);
        std::vector<double> half(static_cast<size_t>(s.nhalf));
        SL_CUDA(cudaMemcpy(half.data(), s.W.p, half.size() * sizeof(double), cudaMemcpyDeviceToHost));
        // expand the Hermitian half: W(-xi) = W(xi)
        const long long rows = s.nrows;
        const int L = s.L_last;
        for (long long r = 0; r < rows; ++r) {
            long long rr = 0;  // index of the negated leading coordinates
            if (s.ndim == 2) {
                rr = (s.n[0] - r) % s.n[0];
            } else {
                const long long i0 = r / s.n[1], i1 = r % s.n[1];
                rr = ((s.n[0] - i0) % s.n[0]) * s.n[1] + (s.n[1] - i1) % s.n[1];
            }
            for (int k = 0; k < L; ++k)
                w[r * L + k] = k < s.H ? half[static_cast<size_t>(r * s.ldh + k)]
                                       : half[static_cast<size_t>(rr * s.ldh + (L - k))];
        }
    });
}

int sl_filter_spectrum(sl_system* h, int i, double* out) {
    return guard([&] {
        System& s = sys_of(h);
        std::lock_guard<std::mutex> lk(s.mu);
        if (i < 0 || i >= s.R) throw SlError(SL_ERR_DOMAIN, "filter index out of range");
        if (!out) throw SlError(SL_ERR_INVALID, "null output");
        DeviceGuard dg(s.device);
        std::vector<double> half(static_cast<size_t>(s.nhalf));
        if (s.ndim == 2) {
            SL_CUDA(cudaMemcpy(half.data(), s.psi.p + static_cast<size_t>(i) * s.nhalf, half.size() * sizeof(double),
                               cudaMemcpyDeviceToHost));
        } else {
            // synthesise on the device through the same energy kernel path
            DBuf<double> tmp;
            tmp.alloc(static_cast<size_t>(s.nhalf));
            FiltSynth3DFlat f{s.synth, s.ldh};
            k_synth_band<<<1024, 256>>>(f, i, s.nhalf, tmp.p);
            check_launch("k_synth_band");
            SL_CUDA(cudaMemcpy(half.data(), tmp.p, half.size() * sizeof(double), cudaMemcpyDeviceToHost));
        }
        const long long rows = s.nrows;
        const int L = s.L_last;
        for (long long r = 0; r < rows; ++r) {
            long long rr;
            if (s.ndim == 2) {
                rr = (s.n[0] - r) % s.n[0];
            } else {
                const long long i0 = r / s.n[1], i1 = r % s.n[1];
                rr = ((s.n[0] - i0) % s.n[0]) * s.n[1] + (s.n[1] - i1) % s.n[1];
            }
            for (int k = 0; k < L; ++k) {
                out[2 * (r * L + k)] = k < s.H ? half[static_cast<size_t>(r * s.ldh + k)]
                                               : half[static_cast<size_t>(rr * s.ldh + (L - k))];
                out[2 * (r * L + k) + 1] = 0.0;
            }
        }
    });
}

int sl_sheardec_dev(sl_system* h, const double* f, double* coeffs, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(f, "sheardec input");
        require_dev_ptr(coeffs, "sheardec output");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        dec(s, f, coeffs, nullptr, stream_of(stream));
    });
}

int sl_sheardec_threshold_dev(sl_system* h, const double* f, double* coeffs, const double* K, int nK, double sigma,
                              int scaled, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(f, "sheardec input");
        require_dev_ptr(coeffs, "sheardec output");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        dec(s, f, coeffs, s.delta.p, stream_of(stream));
    });
}

int sl_shearrec_dev(sl_system* h, const double* coeffs, int nbands, double* f, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        if (nbands != s.nb()) throw SlError(SL_ERR_SHAPE, "inverse: coefficient stack does not match the system");
        require_dev_ptr(coeffs, "shearrec input");
        require_dev_ptr(f, "shearrec output");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        rec(s, coeffs, f, stream_of(stream));
    });
}

int sl_hard_threshold_dev(sl_system* h, const double* in, double* out, int nbands, const double* K, int nK,
                          double sigma, int scaled, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        if (nbands != s.nb()) throw SlError(SL_ERR_SHAPE, "hard_threshold: stack does not match the system");
        require_dev_ptr(in, "hard_threshold input");
        require_dev_ptr(out, "hard_threshold output");
        dim3 grid(static_cast<unsigned>(std::min<long long>(1024, (s.nreal + 255) / 256)), s.nb());
        k_threshold<<<grid, 256, 0, stream_of(stream)>>>(in, out, s.nreal, s.delta.p + s.lo);
        check_launch("k_threshold");
    });
}

int sl_denoise_dev(sl_system* h, const double* in, double* out, const double* K, int nK, double sigma, int scaled,
                   void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(in, "denoise input");
        require_dev_ptr(out, "denoise output");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
        dec(s, in, s.stack.p, s.delta.p, stream_of(stream));
        rec(s, s.stack.p, out, stream_of(stream));
    });
}

// ---- host-pointer variants ----------------------------------------------
int sl_sheardec_host(sl_system* h, const double* f, double* coeffs) {
    return guard([&] {
        System& s = sys_of(h);
        if (!f || !coeffs) throw SlError(SL_ERR_INVALID, "null host pointer");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        s.io_in.alloc(static_cast<size_t>(s.nreal));
        s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
        SL_CUDA(cudaMemcpy(s.io_in.p, f, s.nreal * sizeof(double), cudaMemcpyHostToDevice));
        dec(s, s.io_in.p, s.stack.p, nullptr, 0);
        SL_CUDA(cudaMemcpy(coeffs, s.stack.p, static_cast<size_t>(s.nb()) * s.nreal * sizeof(double),
                           cudaMemcpyDeviceToHost));
    });
}

int sl_shearrec_host(sl_system* h, const double* coeffs, int nbands, double* f) {
    return guard([&] {
        System& s = sys_of(h);
        if (nbands != s.nb()) throw SlError(SL_ERR_SHAPE, "inverse: coefficient stack does not match the system");
        if (!f || !coeffs) throw SlError(SL_ERR_INVALID, "null host pointer");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        s.io_out.alloc(static_cast<size_t>(s.nreal));
        s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
        SL_CUDA(cudaMemcpy(s.stack.p, coeffs, static_cast<size_t>(s.nb()) * s.nreal * sizeof(double),
                           cudaMemcpyHostToDevice));
        rec(s, s.stack.p, s.io_out.p, 0);
        SL_CUDA(cudaMemcpy(f, s.io_out.p, s.nreal * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int sl_hard_threshold_host(sl_system* h, const double* in, double* out, int nbands, const double* K, int nK,
                           double sigma, int scaled) {
    return guard([&] {
        System& s = sys_of(h);
        if (!in || !out) throw SlError(SL_ERR_INVALID, "null host pointer");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        deltas(s, K, nK, sigma, scaled, 0);
        if (nbands != s.nb()) throw SlError(SL_ERR_SHAPE, "hard_threshold: stack does not match the system");
        const size_t n = static_cast<size_t>(s.nb()) * s.nreal;
        s.stack.alloc(n);
        SL_CUDA(cudaMemcpy(s.stack.p, in, n * sizeof(double), cudaMemcpyHostToDevice));
        dim3 grid(static_cast<unsigned>(std::min<long long>(1024, (s.nreal + 255) / 256)), s.nb());
        k_threshold<<<grid, 256>>>(s.stack.p, s.stack.p, s.nreal, s.delta.p + s.lo);
        check_launch("k_threshold");
        SL_CUDA(cudaMemcpy(out, s.stack.p, n * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int sl_denoise_host(sl_system* h, const double* in, double* out, const double* K, int nK, double sigma, int scaled) {
    return guard([&] {
        System& s = sys_of(h);
        if (!in || !out) throw SlError(SL_ERR_INVALID, "null host pointer");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        deltas(s, K, nK, sigma, scaled, 0);
        s.io_in.alloc(static_cast<size_t>(s.nreal));
        s.io_out.alloc(static_cast<size_t>(s.nreal));
        s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
        SL_CUDA(cudaMemcpy(s.io_in.p, in, s.nreal * sizeof(double), cudaMemcpyHostToDevice));
        dec(s, s.io_in.p, s.stack.p, s.delta.p, 0);
        rec(s, s.stack.p, s.io_out.p, 0);
        SL_CUDA(cudaMemcpy(out, s.io_out.p, s.nreal * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int sl_phantom_cartoon(int n, double* out) {
    return guard([&] {
        if (n <= 0 || !out) throw SlError(SL_ERR_INVALID, "bad cartoon arguments");
        cartoon(n, out);
    });
}

int sl_phantom_cartoon_volume(int n, double* out) {
    return guard([&] {
        if (n <= 0 || !out) throw SlError(SL_ERR_INVALID, "bad cartoon_volume arguments");
        cartoon_volume(n, out);
    });
}

int sl_add_gaussian_noise(const double* in, double* out, int64_t count, double sigma, uint64_t seed) {
    return guard([&] {
        if (sigma < 0.0) throw SlError(SL_ERR_DOMAIN, "add_gaussian_noise: sigma must be >= 0");
        if (!in || !out) throw SlError(SL_ERR_INVALID, "null pointer");
        if (in != out) std::memcpy(out, in, static_cast<size_t>(count) * sizeof(double));
        if (sigma == 0.0) return;
        Mt64 rng(seed);
        bool have = false;
        double spare = 0.0;
        auto uni = [&rng] { return static_cast<double>(rng()) * 0x1.0p-64; };
        for (int64_t i = 0; i < count; ++i) {
            double g;
            if (have) {
                have = false;
                g = spare;
            } else {
                double u1;
                do {
                    u1 = uni();
                } while (u1 <= 0.0);
                const double u2 = uni();
                const double r = std::sqrt(-2.0 * std::log(u1));
                const double a = 2.0 * M_PI * u2;
                spare = r * std::sin(a);
                have = true;
                g = r * std::cos(a);
            }
            out[i] += sigma * g;
        }
    });
}

}  // extern "C"
