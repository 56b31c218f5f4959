// Multi-GPU behind the library boundary: NCCL communicators (one process per
// GPU) and the sharded hot path.
//
// The reference's only parallel axis is the filter index (parallel_for,
// parallel.hpp:20-46; ordered partial sums, transform.cpp:69-91,101-124).
// Across GPUs it becomes: rank r owns the balanced contiguous band range
// shard_range(R, r, nranks); the input is broadcast from the root, every
// rank runs the fused dec -> threshold -> rec of its own bands, and the
// reconstruction -- linear in the coefficients -- is summed onto the root:
//   3D fast path : the half-spectrum accumulators sum_b FFT(thr c_b) psi_b
//                  (57 MB at 192^3) are ncclReduce'd, and the root alone
//                  divides by W and runs the final inverse FFT;
//   otherwise    : the partial reconstructions are ncclReduce'd.
// Batched 2D frames shard by image (frame_range) with no collective.
// libnccl.so.2 is loaded at run time (dlopen), so the library itself loads
// without NCCL; a missing NCCL surfaces as SL_ERR_NCCL.
#pragma once
#include <dlfcn.h>
#include <nccl.h>  // types and enums only; every symbol is resolved through dlsym

#include "transform.cuh"

namespace slb {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    std::string why;
    bool ok() const { return commInitRank != nullptr; }
};

static NcclApi load_nccl() {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
        return a;
    }
    a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
    a.reduce = reinterpret_cast<decltype(a.reduce)>(dlsym(h, "ncclReduce"));
    a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
    auto init = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
    if (!a.getUniqueId || !a.commDestroy || !a.broadcast || !a.reduce || !a.errorString || !init) {
        a.why = "libnccl.so.2 lacks an entry point";
        return a;
    }
    a.commInitRank = init;
    return a;
}

static NcclApi& nccl() {
    static NcclApi api = load_nccl();
    if (!api.ok()) throw SlError(SL_ERR_NCCL, api.why);
    return api;
}

#define SL_NCCL(x)                                                                                  \
    do {                                                                                            \
        ncclResult_t r_ = (x);                                                                      \
        if (r_ != ncclSuccess) throw SlError(SL_ERR_NCCL, std::string(#x) + ": " + nccl().errorString(r_)); \
    } while (0)

// [lo, hi) of `rank` in a balanced contiguous split of `count` items
static void shard_of(long long count, int nranks, int rank, long long* lo, long long* hi) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw SlError(SL_ERR_CONFIG, "bad rank / number of ranks");
    *lo = count * rank / nranks;
    *hi = count * (rank + 1) / nranks;
}

}  // namespace slb

struct sl_comm {
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0, device = 0;
};

namespace slb {

// the distributed fused denoise on this rank (see the file comment)
static void denoise_dist(System& s, sl_comm& c, const double* in, double* out, int root, cudaStream_t st) {
    NcclApi& api = nccl();
    if (s.Wmin < 1e-12) throw SlError(SL_ERR_SINGULAR_FRAME, "inverse: frame weight below 1e-12");
    s.io_in.alloc(static_cast<size_t>(s.nreal));
    SL_NCCL(api.broadcast(in, s.io_in.p, static_cast<size_t>(s.nreal), ncclFloat64, root, c.comm, st));
    double* stk = nullptr;
    if (s.materialize) {
        s.stack.alloc(static_cast<size_t>(s.nb()) * s.nreal);
        stk = s.stack.p;
    }
    if (s.fast3d && s.knobs.split3d && !s.knobs.denoise_unfused) {
        // the accumulator slab [k2lo, k2hi) is final once the last chunk's pass C
        // has covered it: its ncclReduce runs on the communication stream while
        // pass C works on the next slab (chunked reduce overlapping the last band group)
        s.ensure_workspaces(2);
        if (!s.comm_ev.size()) s.ensure_comm_events(8);
        cudaStream_t cs = s.ws[1]->st;
        const long long plane = static_cast<long long>(s.n[0]) * s.n[1];  // double2 per k2 plane (natural layout)
        int slab = 0;
        denoise3d_split_acc(s, s.io_in.p, stk, s.delta.p, st, [&](int k2lo, int k2hi) {
            cudaEvent_t ev = s.comm_ev[static_cast<size_t>(slab++ % 8)];
            SL_CUDA(cudaEventRecord(ev, st));
            SL_CUDA(cudaStreamWaitEvent(cs, ev, 0));
            double2* a = s.w->acc.p + k2lo * plane;
            SL_NCCL(api.reduce(a, a, static_cast<size_t>(2 * (k2hi - k2lo) * plane), ncclFloat64, ncclSum, root,
                               c.comm, cs));
        });
        cudaEvent_t done = s.comm_ev[static_cast<size_t>(slab % 8)];
        SL_CUDA(cudaEventRecord(done, cs));
        SL_CUDA(cudaStreamWaitEvent(st, done, 0));
        if (c.rank == root) finish3d_fast(s, out, st);
        return;
    }
    s.io_out.alloc(static_cast<size_t>(s.nreal));
    denoise(s, s.io_in.p, stk, s.io_out.p, s.delta.p, st);
    SL_NCCL(api.reduce(s.io_out.p, c.rank == root ? out : s.io_out.p, static_cast<size_t>(s.nreal), ncclFloat64,
                       ncclSum, root, c.comm, st));
}

}  // namespace slb
