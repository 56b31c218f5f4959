// Host side of the 2D denoise megakernel (mega2d.cuh): task list, counters, launch.
#pragma once
#include "fast2d_p_host.cuh"
#include "mega2d.cuh"

namespace slb {

// Experimental (SLB_MEGA=1): measured ~2x slower than the multi-stream
// per-pass kernels on B200 (per-task ticket/fence/dependency overhead), so the
// default batched path fans frames out over streams instead.
static bool mega2d_enabled(const System& s) {
    const char* e = std::getenv("SLB_MEGA");
    return s.fast2d && e && std::atoi(e) == 1;
}

struct MegaState {
    DBuf<int4> tasks;
    DBuf<int> counters;
    DBuf<double2> F, acc, ring;
    DBuf<double> stack;
    int ntasks = 0, nframes = -1, nb = -1, S = 0, lag = 0, ncnt = 0;
};

template <int L>
static void mega_denoise_t(System& s, MegaState& ms, const double* in, int nframes, double* stack, double* out,
                           const double* delta, cudaStream_t st) {
    using M = Mega<L>;
    const int n0 = s.n[0], H = s.H, nb = s.nb();
    const long long nhT = static_cast<long long>(H) * n0;
    const int row_blocks = (n0 + 2 * M::V - 1) / (2 * M::V);
    const int col_blocks = (H + M::LINES - 1) / M::LINES;
    const int lag = env_int("SLB_MEGA_LAG", 4);
    const int S = std::max(2 * lag + 2, env_int("SLB_MEGA_RING", 16));
    const int nseq = nframes * nb;
    // counter layout
    const int oF1 = 0, oF2 = oF1 + nframes, oD = oF2 + nframes, oR = oD + nseq, oC = oR + nseq, oChain = oC + nseq,
              oX = oChain + nframes * col_blocks, ncnt = oX + nframes + 1;
    if (ms.nframes != nframes || ms.nb != nb || ms.S != S || ms.lag != lag) {
        std::vector<int4> t;
        for (int f = 0; f < nframes; ++f) {
            for (int rb = 0; rb < row_blocks; ++rb) t.push_back({kF1, f, 0, rb});
            for (int cb = 0; cb < col_blocks; ++cb) t.push_back({kF2, f, 0, cb});
            for (int step = 0; step < nb + 2 * lag; ++step) {
                const int bd = step, br = step - lag, bc = step - 2 * lag;
                if (bd < nb)
                    for (int cb = 0; cb < col_blocks; ++cb) t.push_back({kD, f, bd, cb});
                if (br >= 0 && br < nb)
                    for (int rb = 0; rb < row_blocks; ++rb) t.push_back({kR, f, br, rb});
                if (bc >= 0 && bc < nb)
                    for (int cb = 0; cb < col_blocks; ++cb) t.push_back({kC, f, bc, cb});
            }
            for (int cb = 0; cb < col_blocks; ++cb) t.push_back({kX, f, 0, cb});
            for (int rb = 0; rb < row_blocks; ++rb) t.push_back({kY, f, 0, rb});
        }
        ms.tasks.upload(t.data(), t.size(), st);
        ms.ntasks = static_cast<int>(t.size());
        ms.nframes = nframes;
        ms.nb = nb;
        ms.S = S;
        ms.lag = lag;
    }
    ms.counters.alloc(static_cast<size_t>(ncnt) + 1);
    ms.F.alloc(static_cast<size_t>(nframes) * nhT);
    ms.acc.alloc(static_cast<size_t>(nframes) * nhT);
    ms.ring.alloc(static_cast<size_t>(S) * nhT);
    SL_CUDA(cudaMemsetAsync(ms.counters.p, 0, sizeof(int) * (static_cast<size_t>(ncnt) + 1), st));
    MegaArgs a{};
    a.tasks = ms.tasks.p;
    a.ntasks = ms.ntasks;
    a.ticket = ms.counters.p + ncnt;
    a.cnt = ms.counters.p;
    a.nframes = nframes;
    a.nb = nb;
    a.band0 = s.lo;
    a.n0 = n0;
    a.H = H;
    a.S = S;
    a.f = in;
    a.stack = stack;
    a.out = out;
    a.F = ms.F.p;
    a.acc = ms.acc.p;
    a.ring = ms.ring.p;
    a.psiT = s.psiT.p;
    a.WT = s.WT.p;
    a.delta = delta;
    a.scale = 1.0 / static_cast<double>(s.nreal);
    a.tw = s.plan(L, st).tw;
    a.row_blocks = row_blocks;
    a.col_blocks = col_blocks;
    a.oF1 = oF1;
    a.oF2 = oF2;
    a.oD = oD;
    a.oR = oR;
    a.oC = oC;
    a.oChain = oChain;
    a.oX = oX;
    const size_t smem = std::max(static_cast<size_t>(H) * 2 * M::V, static_cast<size_t>(M::LINES) * L) * sizeof(double2);
    set_smem(k2_denoise_mega<L>, smem);
    const int per = resident_blocks(k2_denoise_mega<L>, M::THREADS, smem);
    const int grid = std::min(ms.ntasks, per * sm_count());
    LaunchScope ls(s, "mega2d_denoise", st, static_cast<long long>(nframes) * nb);
    k2_denoise_mega<L><<<grid, M::THREADS, smem, st>>>(a);
    check_launch("k2_denoise_mega");
}

static void mega_denoise(System& s, MegaState& ms, const double* in, int nframes, double* stack, double* out,
                         const double* delta, cudaStream_t st) {
    switch (s.n[0]) {
        case 64: mega_denoise_t<64>(s, ms, in, nframes, stack, out, delta, st); break;
        case 128: mega_denoise_t<128>(s, ms, in, nframes, stack, out, delta, st); break;
        case 192: mega_denoise_t<192>(s, ms, in, nframes, stack, out, delta, st); break;
        case 256: mega_denoise_t<256>(s, ms, in, nframes, stack, out, delta, st); break;
        case 512: mega_denoise_t<512>(s, ms, in, nframes, stack, out, delta, st); break;
        case 1024: mega_denoise_t<1024>(s, ms, in, nframes, stack, out, delta, st); break;
        case 2048: mega_denoise_t<2048>(s, ms, in, nframes, stack, out, delta, st); break;
        default: throw SlError(SL_ERR_GENERIC, "mega2d: unsupported size");
    }
}

}  // namespace slb
