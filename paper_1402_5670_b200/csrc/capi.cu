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
#include "build.cuh"
#include "transform.cuh"
#include "phantoms.cuh"
#include "iterative.cuh"
#include "shcf.cuh"
#include "image_io.cuh"
#include "descriptor.cuh"
#include "quality.cuh"
#include "comm.cuh"

// ====================================================================== C ABI
using namespace slb;

struct sl_system {
    System s;
    sl_comm* comm = nullptr;  // sl_system_set_comm: multi-GPU (one process per GPU)
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

// Explicit taps -> Bank; NULL lowpass = QmfPair::maximally_flat_9tap(), NULL
// highpass = mirror_highpass(lowpass) (QmfPair::from_lowpass), NULL fan =
// default_fan_filter() (filters.cpp:32-38, 114-122).
Bank bank_of(const double* lp, int lp_len, int lp_c, const double* hp, int hp_len, int hp_c, const double* fan, int fr,
             int fc, int fc0, int fc1, const char* provenance) {
    Bank b = default_bank(0);
    if (lp) {
        if (lp_len < 1) throw SlError(SL_ERR_INVALID, "QmfPair: empty lowpass");
        b.qmf.lowpass = Taps1{std::vector<double>(lp, lp + lp_len), lp_c};
        b.qmf.highpass = mirror_highpass(b.qmf.lowpass);
    }
    if (hp) {
        if (hp_len < 1) throw SlError(SL_ERR_INVALID, "QmfPair: empty highpass");
        b.qmf.highpass = Taps1{std::vector<double>(hp, hp + hp_len), hp_c};
    }
    if (fan) {
        if (fr < 1 || fc < 1) throw SlError(SL_ERR_INVALID, "FanFilter: empty taps");
        Taps2 t = Taps2::zeros(static_cast<size_t>(fr), static_cast<size_t>(fc), fc0, fc1);
        std::memcpy(t.v.data(), fan, sizeof(double) * t.v.size());
        b.fan = std::move(t);
        const std::string pv = provenance ? provenance : "";
        b.fan_name = (pv == "dmaxflat4" || pv == "impulse") ? pv : "custom";
    }
    return b;
}

int create(int ndim, const int* n, const int* levels, int n_scales, int j0, int full, const Bank* bank_in, int device,
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
        s.qmf_lowpass = bank_in->qmf.lowpass.v;
        s.qmf_center = bank_in->qmf.lowpass.c;
        s.fan_name = bank_in->fan_name;
        s.fan_ck = fan_checksum(bank_in->fan);
        cudaStream_t st;
        SL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        try {
            if (ndim == 2)
                build_2d(s, *bank_in, st);
            else
                build_3d(s, *bank_in, st);
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
    Bank bank;
    const int rc = guard([&] { bank = default_bank(impulse_fan); });
    if (rc) return rc;
    return create(2, n, levels, n_scales, j0, full_system, &bank, device, shard_lo, shard_hi, out);
}

int sl_system_create_3d(int n0, int n1, int n2, const int* levels, int n_scales, int j0, int full_system,
                        int impulse_fan, int device, int shard_lo, int shard_hi, sl_system** out) {
    const int n[3] = {n0, n1, n2};
    Bank bank;
    const int rc = guard([&] { bank = default_bank(impulse_fan); });
    if (rc) return rc;
    return create(3, n, levels, n_scales, j0, full_system, &bank, device, shard_lo, shard_hi, out);
}

int sl_system_create_2d_ex(int rows, int cols, const int* levels, int n_scales, int j0, int full_system,
                           const double* lowpass, int lowpass_len, int lowpass_center, const double* highpass,
                           int highpass_len, int highpass_center, const double* fan, int fan_rows, int fan_cols,
                           int fan_c0, int fan_c1, const char* fan_provenance, int device, int shard_lo,
                           int shard_hi, sl_system** out) {
    const int n[2] = {rows, cols};
    Bank bank;
    const int rc = guard([&] {
        bank = bank_of(lowpass, lowpass_len, lowpass_center, highpass, highpass_len, highpass_center, fan, fan_rows,
                       fan_cols, fan_c0, fan_c1, fan_provenance);
    });
    if (rc) return rc;
    return create(2, n, levels, n_scales, j0, full_system, &bank, device, shard_lo, shard_hi, out);
}

int sl_system_create_3d_ex(int n0, int n1, int n2, const int* levels, int n_scales, int j0, int full_system,
                           const double* lowpass, int lowpass_len, int lowpass_center, const double* highpass,
                           int highpass_len, int highpass_center, const double* fan, int fan_rows, int fan_cols,
                           int fan_c0, int fan_c1, const char* fan_provenance, int device, int shard_lo,
                           int shard_hi, sl_system** out) {
    const int n[3] = {n0, n1, n2};
    Bank bank;
    const int rc = guard([&] {
        bank = bank_of(lowpass, lowpass_len, lowpass_center, highpass, highpass_len, highpass_center, fan, fan_rows,
                       fan_cols, fan_c0, fan_c1, fan_provenance);
    });
    if (rc) return rc;
    return create(3, n, levels, n_scales, j0, full_system, &bank, device, shard_lo, shard_hi, out);
}

int sl_describe(const sl_system* h, char* text, size_t cap, size_t* len) {
    return guard([&] {
        const System& s = sys_of(h);
        Descriptor d;
        d.ndim = s.ndim;
        for (int a = 0; a < s.ndim; ++a) d.dims[a] = s.n[a];
        d.j0 = s.prof.j0;
        d.levels = s.prof.levels;
        d.full = s.full;
        d.qmf = s.qmf_lowpass;
        d.qmf_center = s.qmf_center;
        d.fan_name = s.fan_name;
        d.fan_ck = s.fan_ck;
        const std::string t = descriptor_text(d);
        if (len) *len = t.size();
        if (text) {
            if (cap < t.size() + 1) throw SlError(SL_ERR_INVALID, "describe: buffer too small");
            std::memcpy(text, t.c_str(), t.size() + 1);
        }
    });
}

int sl_system_create_from_descriptor(const char* text, int ndim, int device, int shard_lo, int shard_hi,
                                     sl_system** out) {
    Bank bank;
    Descriptor d;
    const int rc = guard([&] {
        if (!text) throw SlError(SL_ERR_INVALID, "null descriptor text");
        d = descriptor_parse(text);
        if (ndim == 2 && d.ndim != 2) throw SlError(SL_ERR_FORMAT, "descriptor: expected a 2D system");
        if (ndim == 3 && d.ndim != 3) throw SlError(SL_ERR_FORMAT, "descriptor: expected a 3D system");
        for (int v : d.levels)
            if (v < 0) throw SlError(SL_ERR_CONFIG, "ScaleProfile: shear levels must be >= 0");
        bank.fan = descriptor_fan(d);
        bank.fan_name = d.fan_name;
        bank.qmf = qmf_from_lowpass(Taps1{d.qmf, d.qmf_center});
        for (int a = 0; a < d.ndim; ++a)
            if (d.dims[a] < 0 || d.dims[a] > (1 << 20)) throw SlError(SL_ERR_FORMAT, "descriptor: bad dims");
    });
    if (rc) return rc;
    const int n[3] = {static_cast<int>(d.dims[0]), static_cast<int>(d.dims[1]), static_cast<int>(d.dims[2])};
    return create(d.ndim, n, d.levels.data(), static_cast<int>(d.levels.size()), d.j0, d.full, &bank, device, shard_lo,
                  shard_hi, out);
}

int sl_default_fan(double* taps, int64_t cap, int* rows, int* cols, int* c0, int* c1) {
    return guard([&] {
        const Taps2 f = fan_of(0);  // the bundled constant, checksum-verified
        if (rows) *rows = static_cast<int>(f.n0);
        if (cols) *cols = static_cast<int>(f.n1);
        if (c0) *c0 = static_cast<int>(f.c0);
        if (c1) *c1 = static_cast<int>(f.c1);
        if (taps) {
            if (cap < static_cast<int64_t>(f.v.size())) throw SlError(SL_ERR_INVALID, "default_fan: buffer too small");
            std::memcpy(taps, f.v.data(), sizeof(double) * f.v.size());
        }
    });
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
        CallOrder co(s, 0);
        std::vector<double> half(static_cast<size_t>(s.nhalf));
        std::vector<double2> halfc;
        if (s.ndim == 2 && s.cplx) {
            // complex (Hermitian) spectrum of an asymmetric fan: psi(-xi) = conj(psi(xi))
            halfc.resize(static_cast<size_t>(s.nhalf));
            SL_CUDA(cudaMemcpy(halfc.data(), s.psiC.p + static_cast<size_t>(i) * s.nhalf, halfc.size() * sizeof(double2),
                               cudaMemcpyDeviceToHost));
            const long long rows = s.nrows;
            const int L = s.L_last;
            for (long long r = 0; r < rows; ++r) {
                const long long rr = (s.n[0] - r) % s.n[0];
                for (int k = 0; k < L; ++k) {
                    const bool lo = k < s.H;
                    const double2 z = lo ? halfc[static_cast<size_t>(r * s.ldh + k)]
                                         : halfc[static_cast<size_t>(rr * s.ldh + (L - k))];
                    out[2 * (r * L + k)] = z.x;
                    out[2 * (r * L + k) + 1] = lo ? z.y : -z.y;
                }
            }
            return;
        }
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
        CallOrder co(s, stream_of(stream));
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
        CallOrder co(s, stream_of(stream));
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
        CallOrder co(s, stream_of(stream));
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
        CallOrder co(s, stream_of(stream));
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        if (nbands != s.nb()) throw SlError(SL_ERR_SHAPE, "hard_threshold: stack does not match the system");
        require_dev_ptr(in, "hard_threshold input");
        require_dev_ptr(out, "hard_threshold output");
        dim3 grid(static_cast<unsigned>(std::min<long long>(1024, (s.nreal + 255) / 256)), s.nb());
        LaunchScope ls(s, "threshold", stream_of(stream), s.nb());
        k_threshold<<<grid, 256, 0, stream_of(stream)>>>(in, out, s.nreal, s.delta.p + s.lo);
        check_launch("k_threshold");
    });
}

// Fused dec -> threshold -> rec. `stack` (device, [nbands][dims]) receives the
// thresholded coefficient stack -- what hard_threshold(forward(in)) returns in
// the reference (apps.cpp:114-121) -- or is null: then the handle's scratch
// stack is written while sl_set_stack_output is on (the default, the
// reference's denoise materialises it) and nothing is written when it is off.
static void denoise_one(System& s, const double* in, double* stack, double* out, cudaStream_t st) {
    double* stk = stack;
    if (!stk && s.materialize) {
        s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
        stk = s.stack.p;
    }
    denoise(s, in, stk, out, s.delta.p, st);
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
        CallOrder co(s, stream_of(stream));
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        denoise_one(s, in, nullptr, out, stream_of(stream));
    });
}

int sl_denoise_stack_dev(sl_system* h, const double* in, double* stack, double* out, const double* K, int nK,
                         double sigma, int scaled, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(in, "denoise input");
        require_dev_ptr(stack, "denoise stack output");
        require_dev_ptr(out, "denoise output");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        denoise_one(s, in, stack, out, stream_of(stream));
    });
}

// ---- batched variants: frames fanned out over the handle's workspaces ----
}  // extern "C"
namespace {
// Runs per_frame(frame, stream) for every frame, spreading frames round-robin
// over min(nstreams, nframes) workspaces whose streams fork from / join into
// the caller's stream (workspace 0 runs on the caller's stream itself).
template <class Fn>
void fan_out(System& s, int nframes, cudaStream_t user, Fn&& per_frame) {
    const int K = std::max(1, std::min(s.nstreams, nframes));
    s.ensure_workspaces(K);
    if (K > 1) {
        SL_CUDA(cudaEventRecord(s.fork_ev, user));
        for (int k = 1; k < K; ++k) SL_CUDA(cudaStreamWaitEvent(s.ws[static_cast<size_t>(k)]->st, s.fork_ev, 0));
    }
    s.concurrency = K;
    try {
        for (int f = 0; f < nframes; ++f) {
            const int k = f % K;
            s.w = s.ws[static_cast<size_t>(k)].get();
            per_frame(f, k == 0 ? user : s.w->st);
        }
    } catch (...) {
        s.w = s.ws[0].get();
        s.concurrency = 1;
        throw;
    }
    s.w = s.ws[0].get();
    s.concurrency = 1;
    for (int k = 1; k < K; ++k) {
        System::Workspace& wk = *s.ws[static_cast<size_t>(k)];
        SL_CUDA(cudaEventRecord(wk.ev, wk.st));
        SL_CUDA(cudaStreamWaitEvent(user, wk.ev, 0));
    }
}
// Lock-step 2D batches (fast2d_fused.cuh denoise2d_fast_batch): all frames of
// a group pass through each kernel together on one stream. SLB_LOCKSTEP=0
// restores the per-frame fan-out over the workspace streams.
bool lockstep_batch(const System& s, int nframes) {
    return s.fast2d && nframes > 1 && s.knobs.lockstep != 0 && !s.knobs.denoise_unfused;
}
int lockstep_group(const System& s, int nframes) { return std::max(1, std::min(nframes, s.knobs.lockstep_frames)); }
// stack of frame group g: the caller's [frames][nb][dims] buffer, else the
// workspace scratch (only while the handle materialises the stack)
double* group_stack(System& s, double* user, long long f0, int group, long long sfs) {
    if (user) return user + f0 * sfs;
    if (!s.materialize) return nullptr;
    s.w->stack.alloc(static_cast<size_t>(group) * sfs);
    return s.w->stack.p;
}
void denoise_lockstep(System& s, const double* in, int nframes, double* user_stack, double* out, cudaStream_t st) {
    if (s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
    const int group = lockstep_group(s, nframes);
    const int ngroups = (nframes + group - 1) / group;
    const long long sfs = static_cast<long long>(s.nb()) * s.nreal;
    // groups spread over the workspace streams like single frames
    fan_out(s, ngroups, st, [&](int g, cudaStream_t fst) {
        const int f0 = g * group, nf = std::min(group, nframes - f0);
        const size_t off = static_cast<size_t>(f0) * s.nreal;
        double* stk = group_stack(s, user_stack, f0, group, sfs);
        const int conc = s.concurrency;
        s.concurrency = std::max(conc, 4);  // full-machine band grouping (fast2d_cfg)
        s.lockstep_cfg = true;
        denoise2d_fast_batch(s, in + off, s.nreal, nf, stk, sfs, out + off, s.nreal, s.delta.p, fst);
        s.lockstep_cfg = false;
        s.concurrency = conc;
    });
}
void denoise_batch(System& s, const double* in, int nframes, double* user_stack, double* out, cudaStream_t st) {
    if (lockstep_batch(s, nframes)) {
        denoise_lockstep(s, in, nframes, user_stack, out, st);
        return;
    }
    const long long sfs = static_cast<long long>(s.nb()) * s.nreal;
    fan_out(s, nframes, st, [&](int fr, cudaStream_t fst) {
        double* stk = group_stack(s, user_stack, fr, 1, sfs);
        denoise(s, in + static_cast<size_t>(fr) * s.nreal, stk, out + static_cast<size_t>(fr) * s.nreal, s.delta.p,
                fst);
    });
}
// Host buffers of the e2e call: pinned memory is used as is; pageable memory
// is page-locked for the duration of the call (cudaHostRegister) so the
// per-frame async copies overlap the kernels instead of serialising the loop.
struct HostPin {
    const void* p = nullptr;
    bool registered = false;
    HostPin(const void* ptr, size_t bytes) : p(ptr) {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, ptr) != cudaSuccess) {
            cudaGetLastError();
            a.type = cudaMemoryTypeUnregistered;
        }
        if (a.type == cudaMemoryTypeUnregistered && bytes > 0) {
            SL_CUDA(cudaHostRegister(const_cast<void*>(ptr), bytes, cudaHostRegisterDefault));
            registered = true;
        }
    }
    ~HostPin() {
        if (registered) cudaHostUnregister(const_cast<void*>(p));
    }
};
}  // namespace
extern "C" {

int sl_set_stack_output(sl_system* h, int materialize) {
    return guard([&] {
        System& s = sys_of(h);
        std::lock_guard<std::mutex> lk(s.mu);
        s.materialize = materialize != 0;
    });
}

int sl_set_streams(sl_system* h, int nstreams) {
    return guard([&] {
        System& s = sys_of(h);
        if (nstreams < 1 || nstreams > 16) throw SlError(SL_ERR_CONFIG, "nstreams must be in [1, 16]");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        s.nstreams = nstreams;
    });
}

int sl_sheardec_batch_dev(sl_system* h, const double* f, int nframes, double* coeffs, const double* K, int nK,
                          double sigma, int scaled, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(f, "sheardec input");
        require_dev_ptr(coeffs, "sheardec output");
        if (nframes < 0) throw SlError(SL_ERR_SHAPE, "negative frame count");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        cudaStream_t st = stream_of(stream);
        if (K) deltas(s, K, nK, sigma, scaled, st);
        const double* dl = K ? s.delta.p : nullptr;
        fan_out(s, nframes, st, [&](int fr, cudaStream_t fst) {
            dec(s, f + static_cast<size_t>(fr) * s.nreal, coeffs + static_cast<size_t>(fr) * s.nb() * s.nreal, dl, fst);
        });
    });
}

int sl_shearrec_batch_dev(sl_system* h, const double* coeffs, int nframes, double* f, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(coeffs, "shearrec input");
        require_dev_ptr(f, "shearrec output");
        if (nframes < 0) throw SlError(SL_ERR_SHAPE, "negative frame count");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        fan_out(s, nframes, stream_of(stream), [&](int fr, cudaStream_t fst) {
            rec(s, coeffs + static_cast<size_t>(fr) * s.nb() * s.nreal, f + static_cast<size_t>(fr) * s.nreal, fst);
        });
    });
}

int sl_denoise_batch_dev(sl_system* h, const double* in, int nframes, double* out, const double* K, int nK,
                         double sigma, int scaled, void* stream) {
    return sl_denoise_batch_stack_dev(h, in, nframes, nullptr, out, K, nK, sigma, scaled, stream);
}

int sl_denoise_batch_stack_dev(sl_system* h, const double* in, int nframes, double* stacks, double* out,
                               const double* K, int nK, double sigma, int scaled, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(in, "denoise input");
        require_dev_ptr(out, "denoise output");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        if (nframes < 0) throw SlError(SL_ERR_SHAPE, "negative frame count");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        cudaStream_t st = stream_of(stream);
        CallOrder co(s, st);
        deltas(s, K, nK, sigma, scaled, st);
        denoise_batch(s, in, nframes, stacks, out, st);
    });
}

// Host in/out (e2e): H2D of all frames, batched dec/thr/rec, D2H of the results.
int sl_denoise_batch_host(sl_system* h, const double* in, int nframes, double* out, const double* K, int nK,
                          double sigma, int scaled) {
    return guard([&] {
        System& s = sys_of(h);
        if (!in || !out) throw SlError(SL_ERR_INVALID, "null host pointer");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        if (nframes < 0) throw SlError(SL_ERR_SHAPE, "negative frame count");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, 0);
        const size_t n = static_cast<size_t>(nframes) * s.nreal;
        s.io_in.alloc(n);
        s.io_out.alloc(n);
        HostPin pin_in(in, n * sizeof(double)), pin_out(out, n * sizeof(double));
        cudaStream_t st = 0;
        deltas(s, K, nK, sigma, scaled, st);
        // measured (tools/e2e_ab.sh, 8 frames of 512^2): 3 compute streams
        // 6250 frames/s, 1: 4800, 4: 6100, 5-6: 6220, per-frame fan-out: 6100
        // schedule (profiles/r2_e2e_sweep.log, r2b_sweep_e2e_pipe.log): below 16
        // frames 3 compute streams of single frames; from 16 frames 3 streams of
        // lock-step groups of 4 frames with every band in one group (as the
        // device batch) after one single head frame (compute starts after one
        // frame's H2D) -- e2e 0.90 of the device batch at 32 frames
        const bool many = nframes >= 16;
        const int pipe = s.knobs.host_pipe >= 0 ? s.knobs.host_pipe : (s.fast2d ? 3 : 0);
        const long long sfs = static_cast<long long>(s.nb()) * s.nreal;
        if (pipe > 0 && nframes > 1) {
            // pipelined: all H2D in frame order on one copy stream, the fused
            // denoise of frame f on compute stream f % pipe once its H2D is
            // done, all D2H in frame order on a second copy stream -- frames
            // finish staggered, so the D2H overlaps the later frames' kernels
            const int P = std::min(pipe, nframes);
            s.ensure_workspaces(P + 3);
            s.ensure_pipe_events(2 * static_cast<size_t>(nframes));
            cudaStream_t cin = s.ws[static_cast<size_t>(P + 1)]->st, cout = s.ws[static_cast<size_t>(P + 2)]->st;
            SL_CUDA(cudaEventRecord(s.fork_ev, st));
            for (int k = 1; k <= P + 2; ++k) SL_CUDA(cudaStreamWaitEvent(s.ws[static_cast<size_t>(k)]->st, s.fork_ev, 0));
            const size_t fb = static_cast<size_t>(s.nreal) * sizeof(double);
            s.concurrency = s.knobs.pipe_conc >= 1 ? s.knobs.pipe_conc : P;  // band grouping of fast2d_cfg
            // SLB_PIPE_GROUP: lock-step frame groups per compute stream (one
            // launch per pass covers the group, as in the device batch)
            const int want_grp = s.knobs.pipe_group >= 1 ? s.knobs.pipe_group : (many ? 4 : 1);
            const int head = s.knobs.pipe_head >= 0 ? s.knobs.pipe_head : (many ? 1 : 0);
            // the last `tail` frames alone too: the compute streams finish single
            // frames instead of pairs, so less D2H is left after the last kernel
            const int tail = s.knobs.pipe_tail >= 0 ? s.knobs.pipe_tail : 0;
            const int grp = lockstep_batch(s, nframes) ? std::max(1, std::min(nframes, want_grp)) : 1;
            if (grp > 1 && s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
            // segments: the first `head` frames alone (compute starts after one
            // frame's H2D), then lock-step groups of grp frames
            std::vector<std::pair<int, int>> seg;
            for (int f0 = 0; f0 < nframes;) {
                const bool single = static_cast<int>(seg.size()) < head || nframes - f0 <= tail;
                const int nf = single ? 1 : std::min(grp, nframes - f0);
                seg.emplace_back(f0, nf);
                f0 += nf;
            }
            s.ensure_pipe_events(2 * seg.size());
            try {
                for (size_t g = 0; g < seg.size(); ++g) {
                    const int f0 = seg[g].first, nf = seg[g].second;
                    const size_t off = static_cast<size_t>(f0) * s.nreal;
                    cudaEvent_t ein = s.pipe_ev[2 * g], ec = s.pipe_ev[2 * g + 1];
                    SL_CUDA(cudaMemcpyAsync(s.io_in.p + off, in + off, nf * fb, cudaMemcpyHostToDevice, cin));
                    SL_CUDA(cudaEventRecord(ein, cin));
                    s.w = s.ws[static_cast<size_t>(1 + g % P)].get();
                    SL_CUDA(cudaStreamWaitEvent(s.w->st, ein, 0));
                    double* stk = group_stack(s, nullptr, 0, std::max(grp, nf), sfs);
                    if (nf > 1) {
                        s.lockstep_cfg = s.knobs.pipe_allbands != 0;  // all bands in one group (fast2d_cfg)
                        denoise2d_fast_batch(s, s.io_in.p + off, s.nreal, nf, stk, sfs, s.io_out.p + off, s.nreal,
                                             s.delta.p, s.w->st);
                        s.lockstep_cfg = false;
                    } else
                        denoise(s, s.io_in.p + off, stk, s.io_out.p + off, s.delta.p, s.w->st);
                    SL_CUDA(cudaEventRecord(ec, s.w->st));
                    SL_CUDA(cudaStreamWaitEvent(cout, ec, 0));
                    SL_CUDA(cudaMemcpyAsync(out + off, s.io_out.p + off, nf * fb, cudaMemcpyDeviceToHost, cout));
                }
            } catch (...) {
                s.w = s.ws[0].get();
                s.concurrency = 1;
                s.lockstep_cfg = false;
                throw;
            }
            s.w = s.ws[0].get();
            s.concurrency = 1;
            for (int k = 1; k <= P + 2; ++k) {
                System::Workspace& wk = *s.ws[static_cast<size_t>(k)];
                SL_CUDA(cudaEventRecord(wk.ev, wk.st));
                SL_CUDA(cudaStreamWaitEvent(st, wk.ev, 0));
            }
        } else {
            // per frame (or lock-step frame group) on its workspace stream: H2D ->
            // fused denoise -> D2H, so one group's copies overlap the other groups'
            // kernels (both copy engines busy); single frames measured better here
            // than lock-step pairs (SLB_LOCKSTEP_HOST=1: pairs)
            const bool lock = s.knobs.lockstep_host != 0;
            const int group = (lock && lockstep_batch(s, nframes)) ? lockstep_group(s, nframes) : 1;
            if (group > 1 && s.Wmin < 1e-12)
                throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
            const int ngroups = (nframes + group - 1) / group;
            fan_out(s, ngroups, st, [&](int g, cudaStream_t fst) {
                const int f0 = g * group, nf = std::min(group, nframes - f0);
                const size_t off = static_cast<size_t>(f0) * s.nreal;
                const size_t bytes = static_cast<size_t>(nf) * s.nreal * sizeof(double);
                SL_CUDA(cudaMemcpyAsync(s.io_in.p + off, in + off, bytes, cudaMemcpyHostToDevice, fst));
                double* stk = group_stack(s, nullptr, 0, group, sfs);
                if (group > 1) {
                    const int conc = s.concurrency;
                    s.concurrency = std::max(conc, 4);
                    denoise2d_fast_batch(s, s.io_in.p + off, s.nreal, nf, stk, sfs, s.io_out.p + off, s.nreal,
                                         s.delta.p, fst);
                    s.concurrency = conc;
                } else {
                    denoise(s, s.io_in.p + off, stk, s.io_out.p + off, s.delta.p, fst);
                }
                SL_CUDA(cudaMemcpyAsync(out + off, s.io_out.p + off, bytes, cudaMemcpyDeviceToHost, fst));
            });
        }
        SL_CUDA(cudaStreamSynchronize(st));
    });
}

// ---- host-pointer variants ----------------------------------------------
int sl_sheardec_host(sl_system* h, const double* f, double* coeffs) {
    return guard([&] {
        System& s = sys_of(h);
        if (!f || !coeffs) throw SlError(SL_ERR_INVALID, "null host pointer");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, 0);
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
        CallOrder co(s, 0);
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
        CallOrder co(s, 0);
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
        CallOrder co(s, 0);
        deltas(s, K, nK, sigma, scaled, 0);
        s.io_in.alloc(static_cast<size_t>(s.nreal));
        s.io_out.alloc(static_cast<size_t>(s.nreal));
        SL_CUDA(cudaMemcpy(s.io_in.p, in, s.nreal * sizeof(double), cudaMemcpyHostToDevice));
        denoise_one(s, s.io_in.p, nullptr, s.io_out.p, 0);
        SL_CUDA(cudaMemcpy(out, s.io_out.p, s.nreal * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

// ---- iterative pipelines (apps.hpp:46-90) ------------------------------------
int sl_inpaint_dev(sl_system* h, const double* masked, const double* mask, double* out, int iterations,
                   double delta_init, double delta_min, int scale_by_rms, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        require_dev_ptr(masked, "inpaint signal");
        require_dev_ptr(mask, "inpaint mask");
        require_dev_ptr(out, "inpaint output");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        inpaint(s, masked, mask, out, iterations, delta_init, delta_min, scale_by_rms != 0, stream_of(stream));
    });
}

int sl_inpaint_host(sl_system* h, const double* masked, const double* mask, double* out, int iterations,
                    double delta_init, double delta_min, int scale_by_rms) {
    return guard([&] {
        System& s = sys_of(h);
        if (!masked || !mask || !out) throw SlError(SL_ERR_INVALID, "null host pointer");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, 0);
        DBuf<double> dm, dk, dout;
        dm.alloc(static_cast<size_t>(s.nreal));
        dk.alloc(static_cast<size_t>(s.nreal));
        dout.alloc(static_cast<size_t>(s.nreal));
        SL_CUDA(cudaMemcpy(dm.p, masked, s.nreal * 8, cudaMemcpyHostToDevice));
        SL_CUDA(cudaMemcpy(dk.p, mask, s.nreal * 8, cudaMemcpyHostToDevice));
        inpaint(s, dm.p, dk.p, dout.p, iterations, delta_init, delta_min, scale_by_rms != 0, 0);
        SL_CUDA(cudaMemcpy(out, dout.p, s.nreal * 8, cudaMemcpyDeviceToHost));
    });
}

int sl_separate_dev(sl_system* directional, sl_system* isotropic, const double* signal, double* curves, double* blobs,
                    int iterations, double delta_init, double delta_min, int scale_by_rms, void* stream) {
    return guard([&] {
        System& d = sys_of(directional);
        System& i = sys_of(isotropic);
        if (d.device != i.device) throw SlError(SL_ERR_CONFIG, "separate: systems on different devices");
        require_dev_ptr(signal, "separate signal");
        require_dev_ptr(curves, "separate curves");
        require_dev_ptr(blobs, "separate blobs");
        std::lock_guard<std::mutex> lk(d.mu);
        std::unique_lock<std::mutex> lk2(i.mu, std::defer_lock);
        if (&d != &i) lk2.lock();
        DeviceGuard dg(d.device);
        CallOrder co(d, stream_of(stream));
        CallOrder co2(i, stream_of(stream));
        separate(d, i, signal, curves, blobs, iterations, delta_init, delta_min, scale_by_rms != 0,
                 stream_of(stream));
    });
}

int sl_separate_host(sl_system* directional, sl_system* isotropic, const double* signal, double* curves,
                     double* blobs, int iterations, double delta_init, double delta_min, int scale_by_rms) {
    return guard([&] {
        System& d = sys_of(directional);
        System& i = sys_of(isotropic);
        if (d.device != i.device) throw SlError(SL_ERR_CONFIG, "separate: systems on different devices");
        if (!signal || !curves || !blobs) throw SlError(SL_ERR_INVALID, "null host pointer");
        std::lock_guard<std::mutex> lk(d.mu);
        std::unique_lock<std::mutex> lk2(i.mu, std::defer_lock);
        if (&d != &i) lk2.lock();
        DeviceGuard dg(d.device);
        CallOrder co(d, 0);
        CallOrder co2(i, 0);
        DBuf<double> ds, dc, db;
        ds.alloc(static_cast<size_t>(d.nreal));
        dc.alloc(static_cast<size_t>(d.nreal));
        db.alloc(static_cast<size_t>(d.nreal));
        SL_CUDA(cudaMemcpy(ds.p, signal, d.nreal * 8, cudaMemcpyHostToDevice));
        separate(d, i, ds.p, dc.p, db.p, iterations, delta_init, delta_min, scale_by_rms != 0, 0);
        SL_CUDA(cudaMemcpy(curves, dc.p, d.nreal * 8, cudaMemcpyDeviceToHost));
        SL_CUDA(cudaMemcpy(blobs, db.p, d.nreal * 8, cudaMemcpyDeviceToHost));
    });
}

// ---- SHCF coefficient files (transform.hpp:39-52) --------------------------
int sl_shcf_size(const sl_system* h, int nbands, size_t* bytes) {
    return guard([&] {
        if (!bytes) throw SlError(SL_ERR_INVALID, "null size");
        *bytes = shcf_bytes(sys_of(h), nbands);
    });
}

int sl_shcf_serialize(const sl_system* h, const double* coeffs, int nbands, unsigned char* out, size_t cap) {
    return guard([&] {
        const System& s = sys_of(h);
        if (!coeffs || !out) throw SlError(SL_ERR_INVALID, "null pointer");
        if (cap < shcf_bytes(s, nbands)) throw SlError(SL_ERR_INVALID, "output buffer too small");
        shcf_serialize(s, coeffs, nbands, out);
    });
}

int sl_shcf_deserialize(const sl_system* h, const unsigned char* in, size_t len, double* coeffs, int nbands) {
    return guard([&] {
        const System& s = sys_of(h);
        if (!in || !coeffs) throw SlError(SL_ERR_INVALID, "null pointer");
        shcf_deserialize(s, in, len, coeffs, nbands);
    });
}

// ---- streamed SHCF files: decompose straight to / reconstruct straight from a file,
// a chunk of bands at a time (the stack never exists whole, on the host or device)
}  // extern "C"
namespace {
__global__ void k_add_inplace(double* __restrict__ acc, const double* __restrict__ x, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        acc[i] += x[i];
}
// restrict the handle to bands [lo, hi) for one chunk, restoring the shard after
struct ShardScope {
    System& s;
    int lo, hi;
    ShardScope(System& sys, int l, int h) : s(sys), lo(sys.lo), hi(sys.hi) {
        s.lo = l;
        s.hi = h;
    }
    ~ShardScope() {
        s.lo = lo;
        s.hi = hi;
    }
};
struct PinnedBuf {
    double* p = nullptr;
    explicit PinnedBuf(size_t count) { SL_CUDA(cudaMallocHost(&p, count * sizeof(double))); }
    ~PinnedBuf() {
        if (p) cudaFreeHost(p);
    }
};
struct File {
    std::FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};
int stream_chunk(const System& s, int chunk) {
    if (chunk > 0) return std::min(chunk, s.nb());
    const double per = static_cast<double>(s.nreal) * sizeof(double);
    return std::max(1, std::min(s.nb(), static_cast<int>((2.0 * 1024 * 1024 * 1024) / per)));  // ~2 GB per chunk
}
}  // namespace
extern "C" {

int sl_shcf_forward_file(sl_system* h, const double* f, const char* path, int bands_per_chunk) {
    return guard([&] {
        System& s = sys_of(h);
        if (!f || !path) throw SlError(SL_ERR_INVALID, "null argument");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, 0);
        File out(path, "wb");
        if (!out.f) throw SlError(SL_ERR_FORMAT, std::string("cannot write coefficient file: ") + path);
        std::vector<unsigned char> hdr(shcf_header_bytes(s, s.nb()));
        shcf_write_header(s, hdr.data());
        if (std::fwrite(hdr.data(), 1, hdr.size(), out.f) != hdr.size())
            throw SlError(SL_ERR_FORMAT, "coefficient file write failed");
        const int C = stream_chunk(s, bands_per_chunk);
        const size_t cn = static_cast<size_t>(C) * s.nreal;
        s.io_in.upload(f, static_cast<size_t>(s.nreal), 0);
        s.stack.alloc(cn);
        PinnedBuf host(cn);
        std::vector<unsigned char> bytes(cn * 8);
        const int lo0 = s.lo, hi0 = s.hi;
        for (int b0 = lo0; b0 < hi0; b0 += C) {
            const int b1 = std::min(hi0, b0 + C);
            const size_t count = static_cast<size_t>(b1 - b0) * s.nreal;
            {
                ShardScope sc(s, b0, b1);
                dec(s, s.io_in.p, s.stack.p, nullptr, 0);
            }
            SL_CUDA(cudaMemcpy(host.p, s.stack.p, count * sizeof(double), cudaMemcpyDeviceToHost));
            shcf_write_data(host.p, count, bytes.data());
            if (std::fwrite(bytes.data(), 1, count * 8, out.f) != count * 8)
                throw SlError(SL_ERR_FORMAT, "coefficient file write failed");
        }
    });
}

int sl_shcf_inverse_file(sl_system* h, const char* path, double* out, int bands_per_chunk) {
    return guard([&] {
        System& s = sys_of(h);
        if (!out || !path) throw SlError(SL_ERR_INVALID, "null argument");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, 0);
        if (s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
        File in(path, "rb");
        if (!in.f) throw SlError(SL_ERR_FORMAT, std::string("cannot open coefficient file: ") + path);
        std::vector<unsigned char> hdr(shcf_header_bytes(s, s.nb()));
        const size_t got = std::fread(hdr.data(), 1, hdr.size(), in.f);
        shcf_deserialize(s, hdr.data(), got, nullptr, s.nb());  // magic, version, dims, count, records
        const int C = stream_chunk(s, bands_per_chunk);
        const size_t cn = static_cast<size_t>(C) * s.nreal;
        s.stack.alloc(cn);
        s.io_out.alloc(static_cast<size_t>(s.nreal));
        s.io_in.alloc(static_cast<size_t>(s.nreal));
        SL_CUDA(cudaMemset(s.io_out.p, 0, static_cast<size_t>(s.nreal) * sizeof(double)));
        PinnedBuf host(cn);
        std::vector<unsigned char> bytes(cn * 8);
        const int lo0 = s.lo, hi0 = s.hi;
        for (int b0 = lo0; b0 < hi0; b0 += C) {
            const int b1 = std::min(hi0, b0 + C);
            const size_t count = static_cast<size_t>(b1 - b0) * s.nreal;
            if (std::fread(bytes.data(), 1, count * 8, in.f) != count * 8)
                throw SlError(SL_ERR_FORMAT, "coefficient stream truncated");
            shcf_read_data(bytes.data(), count, host.p);
            SL_CUDA(cudaMemcpy(s.stack.p, host.p, count * sizeof(double), cudaMemcpyHostToDevice));
            {
                ShardScope sc(s, b0, b1);
                rec(s, s.stack.p, s.io_in.p, 0);  // partial reconstruction of the chunk (linear)
            }
            k_add_inplace<<<1024, 256>>>(s.io_out.p, s.io_in.p, s.nreal);
            check_launch("k_add_inplace");
        }
        SL_CUDA(cudaMemcpy(out, s.io_out.p, static_cast<size_t>(s.nreal) * sizeof(double), cudaMemcpyDeviceToHost));
    });
}

int sl_load_pgm(const char* path, double* pixels, int64_t cap, int* rows, int* cols, int* maxval) {
    return guard([&] {
        if (!path) throw SlError(SL_ERR_INVALID, "null path");
        const PgmHeader hd = pgm_load(path, pixels, cap);
        if (rows) *rows = static_cast<int>(hd.rows);
        if (cols) *cols = static_cast<int>(hd.cols);
        if (maxval) *maxval = hd.maxval;
    });
}

int sl_save_pgm(const double* pixels, int rows, int cols, const char* path, int maxval) {
    return guard([&] {
        if (!path || !pixels) throw SlError(SL_ERR_INVALID, "null argument");
        if (rows < 0 || cols < 0) throw SlError(SL_ERR_SHAPE, "PGM: negative dims");
        pgm_save(pixels, static_cast<size_t>(rows), static_cast<size_t>(cols), path, maxval);
    });
}

int sl_load_svol(const char* path, double* volume, int64_t cap, int64_t dims[3]) {
    return guard([&] {
        if (!path || !dims) throw SlError(SL_ERR_INVALID, "null argument");
        long long d[3];
        svol_load(path, volume, cap, d);
        for (int a = 0; a < 3; ++a) dims[a] = d[a];
    });
}

int sl_save_svol(const double* volume, const int64_t dims[3], const char* path) {
    return guard([&] {
        if (!path || !volume || !dims) throw SlError(SL_ERR_INVALID, "null argument");
        long long d[3];
        for (int a = 0; a < 3; ++a) {
            if (dims[a] < 0 || dims[a] > 0xFFFFFFFFll) throw SlError(SL_ERR_SHAPE, "SVOL: dims out of range");
            d[a] = dims[a];
        }
        svol_save(volume, d, path);
    });
}

int sl_gaussian_kernel(double sigma, double* taps, int64_t cap, int* size, int* center) {
    return guard([&] {
        const Taps2 t = gaussian_taps(sigma);
        if (size) *size = static_cast<int>(t.n0);
        if (center) *center = static_cast<int>(t.c0);
        if (taps) {
            if (cap < static_cast<int64_t>(t.v.size())) throw SlError(SL_ERR_INVALID, "gaussian_kernel: buffer too small");
            std::memcpy(taps, t.v.data(), sizeof(double) * t.v.size());
        }
    });
}

int sl_binarize(const double* in, double* out, int64_t count, double delta) {
    return guard([&] {
        if (delta < 0.0) throw SlError(SL_ERR_DOMAIN, "binarize: delta must be >= 0");
        if (!in || !out || count < 0) throw SlError(SL_ERR_INVALID, "null argument");
        for (int64_t i = 0; i < count; ++i) out[i] = std::fabs(in[i]) >= delta ? 1.0 : 0.0;
    });
}

namespace {
// one-band blur system for the quality metrics, on `device`, with its own stream
struct BlurRun {
    sl_system h;
    cudaStream_t st = nullptr;
    BlurRun(int rows, int cols, const double* kernel, int kr, int kc, int kc0, int kc1, int device) {
        if (rows < 1 || cols < 1) throw SlError(SL_ERR_SHAPE, "quality_q: empty grid");
        if (!kernel || kr < 1 || kc < 1) throw SlError(SL_ERR_INVALID, "quality_q: empty blur kernel");
        System& s = h.s;
        s.ndim = 2;
        s.n[0] = rows;
        s.n[1] = cols;
        s.device = device;
        init_geometry(s);
        Taps2 t = Taps2::zeros(static_cast<size_t>(kr), static_cast<size_t>(kc), kc0, kc1);
        std::memcpy(t.v.data(), kernel, sizeof(double) * t.v.size());
        SL_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        build_blur_2d(s, t, st);
    }
    ~BlurRun() {
        if (st) cudaStreamDestroy(st);
    }
    QualityResult run(const double* rec, const double* truth, double d0, int nd, std::vector<double>* all) {
        System& s = h.s;
        return quality_run(
            s, rec, truth, d0, nd,
            [&](int n, auto&& fn) { fan_out(s, n, st, [&](int f, cudaStream_t fst) { fn(f, fst); }); }, st, all);
    }
};
}  // namespace

int sl_quality_q(int rows, int cols, const double* recovered, const double* truth, double delta, const double* kernel,
                 int kr, int kc, int kc0, int kc1, int device, double* q) {
    return guard([&] {
        if (!recovered || !truth || !q) throw SlError(SL_ERR_INVALID, "null argument");
        if (delta < 0.0) throw SlError(SL_ERR_DOMAIN, "binarize: delta must be >= 0");
        DeviceGuard dg(device);
        BlurRun b(rows, cols, kernel, kr, kc, kc0, kc1, device);
        *q = b.run(recovered, truth, delta, 1, nullptr).q;
    });
}

int sl_quality_q_opt(int rows, int cols, const double* recovered, const double* truth, const double* kernel, int kr,
                     int kc, int kc0, int kc1, int device, double* q, int* best_delta, double* q_all) {
    return guard([&] {
        if (!recovered || !truth || !q || !best_delta) throw SlError(SL_ERR_INVALID, "null argument");
        DeviceGuard dg(device);
        BlurRun b(rows, cols, kernel, kr, kc, kc0, kc1, device);
        std::vector<double> all;
        const QualityResult r = b.run(recovered, truth, 0.0, 256, &all);
        *q = r.q;
        *best_delta = r.delta;
        if (q_all) std::memcpy(q_all, all.data(), sizeof(double) * all.size());
    });
}

int sl_profile(sl_system* h, int enable) {
    return guard([&] {
        System& s = sys_of(h);
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        collect_profile(s);
        s.stats.clear();
        s.profiling = enable != 0;
    });
}

int sl_pass_stats(sl_system* h, int max_passes, char* names, double* ms_total, int64_t* launches, int64_t* units,
                  int* n_passes) {
    return guard([&] {
        System& s = sys_of(h);
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        collect_profile(s);
        int i = 0;
        for (const auto& kv : s.stats) {
            if (i >= max_passes) break;
            if (names) {
                std::memset(names + 32 * i, 0, 32);
                std::strncpy(names + 32 * i, kv.first.c_str(), 31);
            }
            if (ms_total) ms_total[i] = kv.second.ms;
            if (launches) launches[i] = kv.second.n;
            if (units) units[i] = kv.second.units;
            ++i;
        }
        if (n_passes) *n_passes = i;
    });
}

int sl_launch_count(const sl_system* h, int64_t* count) {
    return guard([&] {
        if (!count) throw SlError(SL_ERR_INVALID, "null count");
        *count = sys_of(h).launches;
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

// ---- optional fp32 mode (north_star: within 1e-5 of the fp64 reference) ----
}  // extern "C"
namespace {
__global__ void k_to_f32(const double* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = static_cast<float>(in[i]);
}
System& fp32_sys(sl_system* h) {
    System& s = sys_of(h);
    if (!s.fp32) throw SlError(SL_ERR_CONFIG, "fp32 entry point: call sl_system_set_precision(sys, 32) first");
    return s;
}
}  // namespace
extern "C" {

int sl_system_set_precision(sl_system* h, int bits) {
    return guard([&] {
        System& s = sys_of(h);
        if (bits != 32 && bits != 64) throw SlError(SL_ERR_CONFIG, "precision must be 32 or 64 bits");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, 0);
        if (bits == 64) {
            s.fp32 = false;
            s.psiT32.release();
            s.WT32.release();
            return;
        }
        if (s.fast3d && s.knobs.split3d) {  // 3D: the three passes in fp32, tables synthesised as before
            s.fp32 = true;
            return;
        }
        if (!s.fast2d)
            throw SlError(SL_ERR_UNSUPPORTED_SIZE,
                          "fp32 mode: square 2D grids of 64..2048 (power of two or 192) and cubic 3D grids of "
                          "64 / 128 / 192 / 256 only");
        const long long np = static_cast<long long>(s.R) * s.H * s.n[0], nw = static_cast<long long>(s.H) * s.n[0];
        s.psiT32.alloc(static_cast<size_t>(np));
        s.WT32.alloc(static_cast<size_t>(nw));
        k_to_f32<<<1024, 256>>>(s.psiT.p, s.psiT32.p, np);
        check_launch("k_to_f32");
        k_to_f32<<<256, 256>>>(s.WT.p, s.WT32.p, nw);
        check_launch("k_to_f32");
        SL_CUDA(cudaDeviceSynchronize());
        s.fp32 = true;
    });
}

int sl_sheardec_f32_dev(sl_system* h, const float* f, float* coeffs, const double* K, int nK, double sigma, int scaled,
                        void* stream) {
    return guard([&] {
        System& s = fp32_sys(h);
        if (s.ndim != 2) throw SlError(SL_ERR_CONFIG, "fp32 mode in 3D: the fused denoise (sl_denoise_f32_dev)");
        require_dev_ptr(f, "sheardec input");
        require_dev_ptr(coeffs, "sheardec output");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        if (K) deltas(s, K, nK, sigma, scaled, stream_of(stream));
        dec2d_fast_f32(s, f, coeffs, K ? s.delta.p : nullptr, stream_of(stream));
    });
}

int sl_shearrec_f32_dev(sl_system* h, const float* coeffs, int nbands, float* f, void* stream) {
    return guard([&] {
        System& s = fp32_sys(h);
        if (s.ndim != 2) throw SlError(SL_ERR_CONFIG, "fp32 mode in 3D: the fused denoise (sl_denoise_f32_dev)");
        if (nbands != s.nb()) throw SlError(SL_ERR_SHAPE, "inverse: coefficient stack does not match the system");
        require_dev_ptr(coeffs, "shearrec input");
        require_dev_ptr(f, "shearrec output");
        if (s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        rec2d_fast_f32(s, coeffs, f, stream_of(stream));
    });
}

int sl_denoise_f32_dev(sl_system* h, const float* in, float* stack, float* out, const double* K, int nK, double sigma,
                       int scaled, void* stream) {
    return guard([&] {
        System& s = fp32_sys(h);
        require_dev_ptr(in, "denoise input");
        require_dev_ptr(out, "denoise output");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        if (s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        float* stk = stack;
        if (!stk && s.materialize) {  // scratch stack, sized for fp64 (fp32 uses the front half)
            s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
            stk = reinterpret_cast<float*>(s.stack.p);
        }
        if (s.ndim == 3)
            denoise3d_fast_f32(s, in, stk, out, s.delta.p, stream_of(stream));
        else
            denoise2d_fast_f32(s, in, stk, out, s.delta.p, stream_of(stream));
    });
}

int sl_denoise_batch_f32_dev(sl_system* h, const float* in, int nframes, float* stacks, float* out, const double* K,
                             int nK, double sigma, int scaled, void* stream) {
    return guard([&] {
        System& s = fp32_sys(h);
        if (s.ndim != 2) throw SlError(SL_ERR_CONFIG, "fp32 mode in 3D: the fused denoise (sl_denoise_f32_dev)");
        require_dev_ptr(in, "denoise input");
        require_dev_ptr(out, "denoise output");
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        if (nframes < 0) throw SlError(SL_ERR_SHAPE, "negative frame count");
        if (s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        cudaStream_t st = stream_of(stream);
        CallOrder co(s, st);
        deltas(s, K, nK, sigma, scaled, st);
        const int group = lockstep_group(s, nframes);
        const int ngroups = (nframes + group - 1) / group;
        const long long sfs = static_cast<long long>(s.nb()) * s.nreal;
        fan_out(s, ngroups, st, [&](int g, cudaStream_t fst) {
            const int f0 = g * group, nf = std::min(group, nframes - f0);
            const size_t off = static_cast<size_t>(f0) * s.nreal;
            float* stk = nullptr;
            if (stacks) {
                stk = stacks + static_cast<size_t>(f0) * sfs;
            } else if (s.materialize) {
                s.w->stack.alloc(static_cast<size_t>(group) * sfs);
                stk = reinterpret_cast<float*>(s.w->stack.p);
            }
            const int conc = s.concurrency;
            s.concurrency = std::max(conc, 4);
            s.lockstep_cfg = true;
            denoise2d_fast_batch_f32(s, in + off, s.nreal, nf, stk, sfs, out + off, s.nreal, s.delta.p, fst);
            s.lockstep_cfg = false;
            s.concurrency = conc;
        });
    });
}

// ---- multi-GPU: NCCL communicators and the sharded hot path (comm.cuh) ----
int sl_comm_unique_id(unsigned char* id) {
    return guard([&] {
        if (!id) throw SlError(SL_ERR_INVALID, "null id buffer");
        ncclUniqueId u;
        SL_NCCL(nccl().getUniqueId(&u));
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

int sl_comm_create(const unsigned char* id, int nranks, int rank, int device, sl_comm** out) {
    return guard([&] {
        if (!id || !out) throw SlError(SL_ERR_INVALID, "null argument");
        *out = nullptr;
        long long lo, hi;
        shard_of(1, nranks, rank, &lo, &hi);  // validates nranks / rank
        DeviceGuard dg(device);
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        auto c = std::make_unique<sl_comm>();
        c->nranks = nranks;
        c->rank = rank;
        c->device = device;
        SL_NCCL(nccl().commInitRank(&c->comm, nranks, u, rank));
        *out = c.release();
    });
}

int sl_comm_destroy(sl_comm* comm) {
    return guard([&] {
        if (!comm) return;
        DeviceGuard dg(comm->device);
        if (comm->comm) SL_NCCL(nccl().commDestroy(comm->comm));
        delete comm;
    });
}

int sl_comm_info(const sl_comm* comm, int* nranks, int* rank, int* device) {
    return guard([&] {
        if (!comm) throw SlError(SL_ERR_INVALID, "null communicator");
        if (nranks) *nranks = comm->nranks;
        if (rank) *rank = comm->rank;
        if (device) *device = comm->device;
    });
}

int sl_partition(int64_t count, int nranks, int rank, int64_t* lo, int64_t* hi) {
    return guard([&] {
        if (count < 0) throw SlError(SL_ERR_SHAPE, "negative count");
        long long a, b;
        shard_of(count, nranks, rank, &a, &b);
        if (lo) *lo = a;
        if (hi) *hi = b;
    });
}

int sl_system_set_comm(sl_system* h, sl_comm* comm, int shard_bands) {
    return guard([&] {
        System& s = sys_of(h);
        std::lock_guard<std::mutex> lk(s.mu);
        if (comm && comm->device != s.device) throw SlError(SL_ERR_CONFIG, "communicator and system on different devices");
        h->comm = comm;
        if (comm && shard_bands) {
            long long lo, hi;
            shard_of(s.R, comm->nranks, comm->rank, &lo, &hi);
            if (lo >= hi) throw SlError(SL_ERR_CONFIG, "more ranks than shearlets");
            set_shard(s, static_cast<int>(lo), static_cast<int>(hi));
        } else {
            set_shard(s, 0, s.R);
        }
    });
}

int sl_denoise_dist_dev(sl_system* h, const double* in, double* out, const double* K, int nK, double sigma, int scaled,
                        int root, void* stream) {
    return guard([&] {
        System& s = sys_of(h);
        if (!h->comm) throw SlError(SL_ERR_CONFIG, "denoise_dist: no communicator (sl_system_set_comm)");
        if (root < 0 || root >= h->comm->nranks) throw SlError(SL_ERR_CONFIG, "denoise_dist: bad root rank");
        if (h->comm->rank == root) {
            require_dev_ptr(in, "denoise input");
            require_dev_ptr(out, "denoise output");
        }
        if (!K && nK > 0) throw SlError(SL_ERR_INVALID, "null K");
        std::lock_guard<std::mutex> lk(s.mu);
        DeviceGuard dg(s.device);
        CallOrder co(s, stream_of(stream));
        deltas(s, K, nK, sigma, scaled, stream_of(stream));
        denoise_dist(s, *h->comm, in ? in : s.io_in.p, out, root, stream_of(stream));
    });
}

// 2D frames shard by image: this rank denoises frames [lo, hi) of the
// nframes-frame batch (global in / out indexing), no collective.
int sl_denoise_batch_dist_host(sl_system* h, const double* in, int nframes, double* out, const double* K, int nK,
                               double sigma, int scaled) {
    long long lo = 0, hi = nframes;
    const int rc = guard([&] {
        if (!h) throw SlError(SL_ERR_INVALID, "null system handle");
        if (!h->comm) throw SlError(SL_ERR_CONFIG, "denoise_batch_dist: no communicator (sl_system_set_comm)");
        if (nframes < 0) throw SlError(SL_ERR_SHAPE, "negative frame count");
        shard_of(nframes, h->comm->nranks, h->comm->rank, &lo, &hi);
    });
    if (rc) return rc;
    if (hi <= lo) return SL_OK;
    const size_t off = static_cast<size_t>(lo) * static_cast<size_t>(h->s.nreal);
    return sl_denoise_batch_host(h, in + off, static_cast<int>(hi - lo), out + off, K, nK, sigma, scaled);
}

int sl_denoise_batch_dist_dev(sl_system* h, const double* in, int nframes, double* out, const double* K, int nK,
                              double sigma, int scaled, void* stream) {
    long long lo = 0, hi = nframes;
    const int rc = guard([&] {
        if (!h) throw SlError(SL_ERR_INVALID, "null system handle");
        if (!h->comm) throw SlError(SL_ERR_CONFIG, "denoise_batch_dist: no communicator (sl_system_set_comm)");
        if (nframes < 0) throw SlError(SL_ERR_SHAPE, "negative frame count");
        shard_of(nframes, h->comm->nranks, h->comm->rank, &lo, &hi);
    });
    if (rc) return rc;
    if (hi <= lo) return SL_OK;
    const size_t off = static_cast<size_t>(lo) * static_cast<size_t>(h->s.nreal);
    return sl_denoise_batch_stack_dev(h, in + off, static_cast<int>(hi - lo), nullptr, out + off, K, nK, sigma, scaled,
                                      stream);
}

}  // extern "C"
