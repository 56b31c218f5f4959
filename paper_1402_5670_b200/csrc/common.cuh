// Shared host-side infrastructure of the engine: errors, device buffers,
// FFT plans, launch configuration and the System handle.
#pragma once
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
    DBuf<float2> tw32;
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
    std::vector<float2> t32(tw.size());
    for (size_t k = 0; k < tw.size(); ++k) t32[k] = make_float2(static_cast<float>(tw[k].x), static_cast<float>(tw[k].y));
    ph.tw32.upload(t32.data(), t32.size(), st);
    ph.plan.tw32 = ph.tw32.p;
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

// ------------------------------------------------------------------ knobs
// A/B knobs, read once when a handle is created: no
// getenv on the launch paths. -1 = the measured default for the geometry.
static int env_knob(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}
struct Knobs {
    int group = -1, chunk = -1, group1 = -1, group2 = -1, chunk1 = -1;  // 2D band grouping (fast2d_cfg)
    int g3 = -1, chunk3 = -1;                                          // 3D band group / chunk
    int lockstep = 1, lockstep_frames = 4;                              // lock-step frame groups (device batch)
    int host_pipe = -1, pipe_conc = -1, pipe_group = -1, pipe_head = -1, pipe_tail = -1, lockstep_host = 0, pipe_allbands = 1;  // pipelined host batch (-1: auto)
    bool denoise_unfused = false, disable_fast2d = false, disable_fast3d = false;
    bool split3d = true;  // three-pass 3D kernels (fast3d_split.cuh); SLB_SPLIT3D=0 selects the five-pass ones
    bool group3d = true;  // shear-group passes A / C (fast3d_group.cuh); SLB_GROUP3D=0: one axis-0 FFT per band
    bool t3 = true;       // pyramid-3 bands in the transposed frame (SLB_T3=0: singleton groups)
    double real_tol = 1e-9;
    static Knobs from_env() {
        Knobs k;
        k.group = env_knob("SLB_GROUP", -1);
        k.chunk = env_knob("SLB_CHUNK", -1);
        k.group1 = env_knob("SLB_GROUP1", -1);
        k.group2 = env_knob("SLB_GROUP2", -1);
        k.chunk1 = env_knob("SLB_CHUNK1", -1);
        k.g3 = env_knob("SLB_G3", -1);
        k.chunk3 = env_knob("SLB_CHUNK3", -1);
        k.lockstep = env_knob("SLB_LOCKSTEP", 1);
        k.lockstep_frames = std::max(1, env_knob("SLB_LOCKSTEP_FRAMES", 4));
        k.host_pipe = env_knob("SLB_HOST_PIPE", -1);
        k.pipe_conc = env_knob("SLB_PIPE_CONC", -1);
        k.pipe_group = env_knob("SLB_PIPE_GROUP", -1);
        k.pipe_head = env_knob("SLB_PIPE_HEAD", -1);
        k.pipe_tail = env_knob("SLB_PIPE_TAIL", -1);
        k.lockstep_host = env_knob("SLB_LOCKSTEP_HOST", 0);
        k.pipe_allbands = env_knob("SLB_PIPE_ALLBANDS", 1);
        k.denoise_unfused = std::getenv("SLB_DENOISE_UNFUSED") != nullptr;
        k.disable_fast2d = std::getenv("SLB_DISABLE_FAST2D") != nullptr;
        k.disable_fast3d = std::getenv("SLB_DISABLE_FAST3D") != nullptr;
        k.split3d = env_knob("SLB_SPLIT3D", 1) != 0;
        k.group3d = env_knob("SLB_GROUP3D", 1) != 0;
        k.t3 = env_knob("SLB_T3", 1) != 0;
        if (const char* e = std::getenv("SLB_REAL_TOL")) k.real_tol = std::atof(e);
        return k;
    }
};
// knob value, or `dflt` where the knob is unset (< 1)
static inline int knob_or(int v, int dflt) { return v >= 1 ? v : dflt; }

// ------------------------------------------------------------------ system
struct System {
    Knobs knobs = Knobs::from_env();
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
    // what describe() reports (descriptor.hpp:14-23)
    std::vector<double> qmf_lowpass;
    long qmf_center = 0;
    std::string fan_name;
    uint64_t fan_ck = 0;

    std::map<int, std::unique_ptr<PlanHolder>> plans;
    DBuf<double> psi;   // 2D: [R][nhalf] real
    // asymmetric fans: complex (Hermitian) filter spectra [R][nhalf]; such a
    // system runs the generic 2D path (the fast path assumes real filters)
    bool cplx = false;
    DBuf<double2> psiC;
    // 2D fast path (fast2d.cuh): column-major halves psi^T [R][H][n0], W^T [H][n0]
    bool fast2d = false;
    DBuf<double> psiT, WT;
    // optional fp32 mode (sl_system_set_precision(32)): the same tables rounded
    // to float, used by the *_f32 entry points
    bool fp32 = false;
    DBuf<float> psiT32, WT32;
    // 3D fast path (fast3d.cuh): W in the natural [k2][k1][k0] layout
    bool fast3d = false;
    DBuf<double> WN;
    DBuf<double> W;     // [nhalf]
    // 3D synthesis tables
    DBuf<BandDesc3D> bands3;
    std::vector<BandDesc3D> bands3_host;  // the same descriptors (shear-group planning on the host)
    DBuf<double> tab1, tab2;
    FiltSynth3D synth{};
    // scratch: one workspace per concurrent stream (batched calls fan frames
    // out over several workspaces); `w` is the workspace the next pass uses.
    struct Workspace {
        DBuf<double2> F, inter, acc, slots;
        DBuf<double2> FT, accT;  // 3D transposed frame (pyramid-3 shear groups): F^T and its accumulator
        DBuf<double2> aux;  // fp32-mode 3D staging (float2 spectra viewed through double2 storage)
        DBuf<int> done;  // per column block: CTAs of the last rec chunk that finished (self-resetting)
        DBuf<double> stack;
        cudaStream_t st = nullptr;  // owned stream (workspaces > 0)
        cudaEvent_t ev = nullptr;
        ~Workspace() {
            if (ev) cudaEventDestroy(ev);
            if (st) cudaStreamDestroy(st);
        }
    };
    std::vector<std::unique_ptr<Workspace>> ws;
    Workspace* w = nullptr;
    int nstreams = 6;               // workspaces used by batched calls (measured: 6 best for 8-frame host batches)
    int concurrency = 1;            // frames in flight on other streams (set by batched calls)
    bool lockstep_cfg = false;      // a lock-step frame group is being issued (fast2d_cfg: all bands in one group)
    bool materialize = true;        // fused denoise writes the thresholded stack (sl_set_stack_output)
    cudaEvent_t fork_ev = nullptr;
    cudaEvent_t last_ev = nullptr;  // completion of the previous call on this handle (any stream)
    std::vector<cudaEvent_t> pipe_ev;  // per-frame H2D / compute-done events of pipelined host batches
    std::vector<cudaEvent_t> comm_ev;  // slab-ready events of the overlapped multi-GPU reduce
    DBuf<double> delta, stack, io_in, io_out;
    std::vector<double> delta_host;  // host copy of `delta` (deltas() skips unchanged uploads)
    int chunk = 1;
    std::mutex mu;

    // instrumentation: kernel launch count (always) and optional per-pass
    // CUDA-event timing (sl_profile); events are recorded on the launch stream.
    long long launches = 0;
    bool profiling = false;
    struct PendingEv {
        std::string name;
        cudaEvent_t a, b;
        long long units;
    };
    std::vector<PendingEv> pending;
    struct PassStat {
        double ms = 0;
        long long n = 0;
        long long units = 0;  // bands (or spectra) processed
    };
    std::map<std::string, PassStat> stats;

    int nb() const { return hi - lo; }

    System() {
        ws.emplace_back(new Workspace());
        w = ws[0].get();
    }
    ~System() {
        if (fork_ev) cudaEventDestroy(fork_ev);
        if (last_ev) cudaEventDestroy(last_ev);
        for (cudaEvent_t e : pipe_ev) cudaEventDestroy(e);
        for (cudaEvent_t e : comm_ev) cudaEventDestroy(e);
    }
    // Ensure n workspaces exist (1..n-1 with their own non-blocking streams).
    void ensure_pipe_events(size_t n) {
        while (pipe_ev.size() < n) {
            cudaEvent_t e;
            SL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            pipe_ev.push_back(e);
        }
    }
    void ensure_comm_events(size_t n) {
        while (comm_ev.size() < n) {
            cudaEvent_t e;
            SL_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            comm_ev.push_back(e);
        }
    }
    void ensure_workspaces(int n) {
        if (!fork_ev) SL_CUDA(cudaEventCreateWithFlags(&fork_ev, cudaEventDisableTiming));
        while (static_cast<int>(ws.size()) < n) {
            auto p = std::make_unique<Workspace>();
            SL_CUDA(cudaStreamCreateWithFlags(&p->st, cudaStreamNonBlocking));
            SL_CUDA(cudaEventCreateWithFlags(&p->ev, cudaEventDisableTiming));
            ws.push_back(std::move(p));
        }
    }

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

// Orders one API call after the previous call on the same handle, whatever
// stream each was issued on: the handle's scratch (workspaces, delta, stack,
// io buffers, self-resetting counters) is shared by all calls, and the host
// mutex only orders when work is queued, not when the GPU runs it.
struct CallOrder {
    System& s;
    cudaStream_t st;
    CallOrder(System& sys, cudaStream_t stream) : s(sys), st(stream) {
        if (!s.last_ev) SL_CUDA(cudaEventCreateWithFlags(&s.last_ev, cudaEventDisableTiming));
        else SL_CUDA(cudaStreamWaitEvent(st, s.last_ev, 0));
    }
    ~CallOrder() { cudaEventRecord(s.last_ev, st); }
};

// Brackets one kernel launch: counts it and, when profiling, records a
// start/stop event pair on the launch stream.
struct LaunchScope {
    System& s;
    cudaEvent_t a = nullptr, b = nullptr;
    cudaStream_t st;
    const char* name;
    long long units;
    LaunchScope(System& sys, const char* nm, cudaStream_t stream, long long u = 1)
        : s(sys), st(stream), name(nm), units(u) {
        ++s.launches;
        if (s.profiling) {
            SL_CUDA(cudaEventCreate(&a));
            SL_CUDA(cudaEventCreate(&b));
            SL_CUDA(cudaEventRecord(a, st));
        }
    }
    ~LaunchScope() {
        if (a) {
            cudaEventRecord(b, st);
            s.pending.push_back({name, a, b, units});
        }
    }
};

static void collect_profile(System& s) {
    for (auto& p : s.pending) {
        SL_CUDA(cudaEventSynchronize(p.b));
        float ms = 0;
        SL_CUDA(cudaEventElapsedTime(&ms, p.a, p.b));
        auto& st = s.stats[p.name];
        st.ms += ms;
        st.n += 1;
        st.units += p.units;
        cudaEventDestroy(p.a);
        cudaEventDestroy(p.b);
    }
    s.pending.clear();
}

}  // namespace slb
