// Host orchestration of the specialised 3D path (kernels in fast3d.cuh).
#pragma once
#include <functional>
#include "fast2d_host.cuh"
#include "fast3d.cuh"
#include "fast2d_fused.cuh"
#include "fast3d_split.cuh"
#include "fast3d_group.cuh"

namespace slb {

static bool fast3d_supported(const Knobs& k, const int* n) {
    if (k.disable_fast3d) return false;
    if (n[0] != n[1] || n[1] != n[2]) return false;
    switch (n[0]) {
        case 64: case 128: case 192: case 256: return true;
        default: return false;
    }
}

// bands per chunk: the rotated intermediate of a chunk stays around 64 MiB,
// but at least SLB_G3 bands so the axis-0 passes can share F / the accumulator
// RMW across a band group.
// Larger groups measured faster all the way up (fewer, larger launches; F and
// the accumulator touched once per group): take as many bands as ~6 GB of
// rotated intermediate allows (192^3: ~100 bands, 128^3: all 99), split across
// the frames in flight, at least 16.
static int fast3d_group(const System& s) {
    if (s.knobs.g3 >= 1) return s.knobs.g3;
    const double per = static_cast<double>(s.H) * s.n[0] * s.n[1] * sizeof(double2);
    const double budget = 6.0 * 1024 * 1024 * 1024 / std::max(1, s.concurrency);
    return std::max(1, std::min(s.nb(), std::max(16, static_cast<int>(budget / per))));
}
static int fast3d_chunk(const System& s) {
    const double per = static_cast<double>(s.H) * s.n[0] * s.n[1] * sizeof(double2);
    return knob_or(s.knobs.chunk3, std::max(fast3d_group(s), static_cast<int>((64.0 * 1024 * 1024) / per)));
}

template <int n>
struct Fast3DLaunch {
    using RC = RowCfg<n>;
    using CC = ColCfg<n>;
    using AC = Ax0Cfg<n>;
    System& s;
    cudaStream_t st;
    int H;
    long long nT;
    const double2* tw;
    size_t row_smem, col_smem, ax_smem;
    int row_blocks, line_blocks, ax_blocks;
    Fast3DLaunch(System& sys, cudaStream_t stream) : s(sys), st(stream) {
        H = s.H;
        nT = static_cast<long long>(H) * n * n;
        tw = s.plan(n, st).tw;
        row_smem = row_smem_bytes<n>(H);
        col_smem = static_cast<size_t>(CC::LINES) * LineBuf<n, false>::N * sizeof(double2);
        ax_smem = static_cast<size_t>(AC::V) * LineBuf<n, false>::N * sizeof(double2);  // [n][V] tile; line buffers alias it
        row_blocks = (n * n + 2 * RC::V - 1) / (2 * RC::V);
        line_blocks = static_cast<int>((static_cast<long long>(H) * n + CC::LINES - 1) / CC::LINES);
        ax_blocks = H * (n / AC::V);
    }
    void rows_r2c(const double* src, long long sbs, double2* dst, int nb) {
        set_smem(k2_rows_r2c<n>, row_smem);
        LaunchScope ls(s, "f3_rows_r2c", st, nb);
        k2_rows_r2c<n><<<dim3(row_blocks, nb), RC::THREADS, row_smem, st>>>(src, sbs, dst, nT, n * n, H, tw);
        check_launch("k2_rows_r2c");
    }
    void rows_c2r(const double2* src, double* dst, long long dbs, int nb, const double* delta, int band0) {
        set_smem(k2_rows_c2r<n>, row_smem);
        LaunchScope ls(s, delta ? "f3_rows_c2r_thr" : "f3_rows_c2r", st, nb);
        k2_rows_c2r<n><<<dim3(row_blocks, nb), RC::THREADS, row_smem, st>>>(
            src, nT, dst, dbs, n * n, H, 1.0 / static_cast<double>(s.nreal), delta, band0, tw);
        check_launch("k2_rows_c2r");
    }
    // dec rows pass + threshold + rec rows pass (fast2d_fused.cuh) over n*n rows
    void rows_fused(double2* inter, double* band, long long bbs, int nb, const double* delta, int band0) {
        auto* k = band ? k2_rows_fused<n, true> : k2_rows_fused<n, false>;
        set_smem(k, row_smem);
        LaunchScope ls(s, "f3_rows_fused", st, nb);
        k<<<dim3(row_blocks, nb), RC::FUSED_THREADS, row_smem, st>>>(
            inter, nT, band, bbs, n * n, H, 1.0 / static_cast<double>(s.nreal), delta, band0, tw, CUtensorMap{}, 0, 0, 0);
        check_launch("k2_rows_fused");
    }
    template <int DIR>
    void axis1(double2* data, int nb) {
        set_smem(k3_lines_contig<n, DIR>, col_smem);
        LaunchScope ls(s, "f3_axis1", st, nb);
        k3_lines_contig<n, DIR><<<dim3(line_blocks, nb), CC::THREADS, col_smem, st>>>(data, nT, static_cast<long long>(H) * n,
                                                                                      tw);
        check_launch("k3_lines_contig");
    }
    template <int DIR, int MODE>
    void to_rot(const double2* src, long long sbs, double2* dst, int nb, int band0, const double* WN, const char* nm) {
        LaunchScope ls(s, nm, st, nb);
        const int G = MODE == kAx0DecMul ? std::min(fast3d_group(s), nb) : 1;
        const int groups = (nb + G - 1) / G;
        set_smem(k3_ax0_to_rot<n, DIR, MODE>, ax_smem);
        k3_ax0_to_rot<n, DIR, MODE><<<dim3(ax_blocks, groups), AC::THREADS, ax_smem, st>>>(
            src, sbs, dst, nT, H, s.synth, band0, G, nb, WN, tw);
        check_launch("k3_ax0_to_rot");
    }
    template <int DIR, int MODE>
    void from_rot(const double2* src, double2* dst, int nb, int band0, int accumulate, const char* nm) {
        const size_t smem = MODE == kAx0RecAcc ? ax_smem + static_cast<size_t>(AC::V) * n * sizeof(double2) : ax_smem;
        set_smem(k3_ax0_from_rot<n, DIR, MODE>, smem);
        LaunchScope ls(s, nm, st, nb);
        if (MODE == kAx0RecAcc) {
            // one launch per chunk; every CTA walks the chunk's bands in order
            k3_ax0_from_rot<n, DIR, MODE><<<dim3(ax_blocks, 1), AC::THREADS, smem, st>>>(
                src, nT, dst, nT, nb, s.synth, band0, accumulate, tw);
            check_launch("k3_ax0_from_rot");
            return;
        }
        k3_ax0_from_rot<n, DIR, MODE><<<dim3(ax_blocks, nb), AC::THREADS, ax_smem, st>>>(
            src, nT, dst, nT, nb, s.synth, band0, accumulate, tw);
        check_launch("k3_ax0_from_rot");
    }
};

template <int n>
static void dec3d_fast_t(System& s, const double* f, double* out, const double* delta, cudaStream_t st) {
    Fast3DLaunch<n> K(s, st);
    const int nb = s.nb();
    const int C = std::min(fast3d_chunk(s), nb);
    s.w->inter.alloc(static_cast<size_t>(C) * K.nT);
    s.w->F.alloc(static_cast<size_t>(K.nT));
    // F (natural layout) = FFT_0 FFT_1 R2C_2 f
    K.rows_r2c(f, 0, s.w->inter.p, 1);
    K.template axis1<-1>(s.w->inter.p, 1);
    K.template from_rot<-1, kAx0Plain>(s.w->inter.p, s.w->F.p, 1, 0, 0, "f3_ax0_fwd");
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        K.template to_rot<+1, kAx0DecMul>(s.w->F.p, 0, s.w->inter.p, cb, s.lo + b0, nullptr, "f3_ax0_dec");
        K.template axis1<+1>(s.w->inter.p, cb);
        K.rows_c2r(s.w->inter.p, out + static_cast<size_t>(b0) * s.nreal, s.nreal, cb, delta, s.lo + b0);
    }
}

template <int n>
static void rec3d_fast_t(System& s, const double* coeffs, double* out, cudaStream_t st) {
    Fast3DLaunch<n> K(s, st);
    const int nb = s.nb();
    const int C = std::min(fast3d_chunk(s), nb);
    s.w->inter.alloc(static_cast<size_t>(C) * K.nT);
    s.w->acc.alloc(static_cast<size_t>(K.nT));
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        K.rows_r2c(coeffs + static_cast<size_t>(b0) * s.nreal, s.nreal, s.w->inter.p, cb);
        K.template axis1<-1>(s.w->inter.p, cb);
        K.template from_rot<-1, kAx0RecAcc>(s.w->inter.p, s.w->acc.p, cb, s.lo + b0, b0 > 0, "f3_ax0_rec");
    }
    K.template to_rot<+1, kAx0DivW>(s.w->acc.p, 0, s.w->inter.p, 1, 0, s.WN.p, "f3_ax0_final");
    K.template axis1<+1>(s.w->inter.p, 1);
    K.rows_c2r(s.w->inter.p, out, 0, 1, nullptr, 0);
}

// denoise with the stack materialised: 5 passes per band instead of 6 and no
// band read-back (the thresholded rows feed the rec r2c in the same kernel)
template <int n>
static void denoise3d_fast_t(System& s, const double* f, double* stack, double* out, const double* delta,
                             cudaStream_t st) {
    Fast3DLaunch<n> K(s, st);
    const int nb = s.nb();
    const int C = std::min(fast3d_chunk(s), nb);
    s.w->inter.alloc(static_cast<size_t>(C) * K.nT);
    s.w->F.alloc(static_cast<size_t>(K.nT));
    s.w->acc.alloc(static_cast<size_t>(K.nT));
    K.rows_r2c(f, 0, s.w->inter.p, 1);
    K.template axis1<-1>(s.w->inter.p, 1);
    K.template from_rot<-1, kAx0Plain>(s.w->inter.p, s.w->F.p, 1, 0, 0, "f3_ax0_fwd");
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        K.template to_rot<+1, kAx0DecMul>(s.w->F.p, 0, s.w->inter.p, cb, s.lo + b0, nullptr, "f3_ax0_dec");
        K.template axis1<+1>(s.w->inter.p, cb);
        K.rows_fused(s.w->inter.p, (stack ? stack + static_cast<size_t>(b0) * s.nreal : nullptr), s.nreal, cb, delta, s.lo + b0);
        K.template axis1<-1>(s.w->inter.p, cb);
        K.template from_rot<-1, kAx0RecAcc>(s.w->inter.p, s.w->acc.p, cb, s.lo + b0, b0 > 0, "f3_ax0_rec");
    }
    K.template to_rot<+1, kAx0DivW>(s.w->acc.p, 0, s.w->inter.p, 1, 0, s.WN.p, "f3_ax0_final");
    K.template axis1<+1>(s.w->inter.p, 1);
    K.rows_c2r(s.w->inter.p, out, 0, 1, nullptr, 0);
}

// ---------------------------------------------------------------- three-pass path (fast3d_split.cuh)
// band group of pass A (F held in registers across it): about a quarter of the
// chunk, so the grid has ~4x the CTAs of one group per band chunk
static int split_group(const System& s, int cb) {
    if (s.knobs.g3 >= 1) return s.knobs.g3;
    return std::max(4, (cb + 3) / 4);
}

template <int n, class C = double2>
struct Split3DLaunch {
    using S = SplitShape<n>;
    System& s;
    cudaStream_t st;
    long long nT;
    const C* tw;
    static constexpr size_t AC_SMEM = S::AC_ELEMS * sizeof(C);
    static constexpr size_t REC_SMEM = (S::REC_DB ? 2 : 1) * S::AC_ELEMS * sizeof(C);
    static constexpr size_t B_SMEM = S::B_ELEMS * sizeof(C);
    Split3DLaunch(System& sys, cudaStream_t stream) : s(sys), st(stream) {
        nT = static_cast<long long>(s.H) * n * n;
        tw = Prec2D<C>::tw(s.plan(n, st));
    }
    void dec(const C* F, C* Z, int nb, int band0) {
        set_smem(k3s_dec<n, C>, AC_SMEM);
        const int G = std::min(nb, split_group(s, nb));
        LaunchScope ls(s, "f3s_dec", st, nb);
        k3s_dec<n, C><<<dim3(S::H * S::Q, (nb + G - 1) / G), S::AC_THREADS, AC_SMEM, st>>>(F, Z, nT, s.synth, band0, G,
                                                                                       nb, tw);
        check_launch("k3s_dec");
    }
    template <int MODE>
    void mid(C* Z, RealOf<C>* band, const RealOf<C>* bandin, int nb, const double* delta, int band0,
             const BandDesc3D* tb = nullptr) {
        auto* k = (MODE == kMidRec || band) ? k3s_mid<n, MODE, true, C> : k3s_mid<n, MODE, false, C>;
        set_smem(k, B_SMEM);
        LaunchScope ls(s, MODE == kMidFused ? "f3s_mid" : (MODE == kMidDec ? "f3s_mid_dec" : "f3s_mid_rec"), st, nb);
        k<<<dim3(n * (S::P / 2), nb), S::B_THREADS, B_SMEM, st>>>(Z, nT, band, s.nreal, bandin,
                                                                 RealOf<C>(1.0 / static_cast<double>(s.nreal)), delta,
                                                                 band0, tw, tb);
        check_launch("k3s_mid");
    }
    // shear-group passes (fast3d_group.cuh)
    static constexpr size_t G_SMEM = GroupShape<n>::template smem<C>();
    // the chunk's Z as the 5D tensor {re/im x a%4, q, a/4, i0, slot * H + k2}
    // (quad-interleaved rows) for the TMA copies of the grouped passes A / C
    static CUtensorMap zmap_of(const C* Z, const SplitGroups& g) {
        CUtensorMap zmap{};
        if constexpr (GroupShape<n>::template TMA_STORE<C>) {
            int slots = 0;
            for (int i = 0; i < g.count; ++i) slots = std::max(slots, g.first[i] + g.len[i] - g.zb0);
            const cuuint64_t zs = static_cast<cuuint64_t>(S::H) * slots;
            if constexpr (SplitLayout<n, C>::ZQUAD) {
                // {re/im x a%4, q, a/4, i0, slot * H + k2}: quad-interleaved rows, 64-byte swizzle
                const cuuint64_t dims[5] = {8, static_cast<cuuint64_t>(S::Q), static_cast<cuuint64_t>(S::P / 4),
                                            static_cast<cuuint64_t>(n), zs};
                const cuuint64_t strides[4] = {4 * sizeof(C), 4 * S::Q * sizeof(C), static_cast<cuuint64_t>(n) * sizeof(C),
                                               static_cast<cuuint64_t>(n) * n * sizeof(C)};
                const cuuint32_t box[5] = {8, 1, static_cast<cuuint32_t>(S::P / 4), static_cast<cuuint32_t>(n), 1};
                zmap = tma_map_f64(Z, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_64B);
            } else {
                // {re/im x a, q, 1, i0, slot * H + k2}: plain [q][a] rows of P * 16 = 128 bytes, 128-byte swizzle
                const cuuint64_t dims[5] = {2 * static_cast<cuuint64_t>(S::P), static_cast<cuuint64_t>(S::Q), 1,
                                            static_cast<cuuint64_t>(n), zs};
                const cuuint64_t strides[4] = {S::P * sizeof(C), static_cast<cuuint64_t>(n) * sizeof(C),
                                               static_cast<cuuint64_t>(n) * sizeof(C),
                                               static_cast<cuuint64_t>(n) * n * sizeof(C)};
                const cuuint32_t box[5] = {2 * static_cast<cuuint32_t>(S::P), 1, 1, static_cast<cuuint32_t>(n), 1};
                zmap = tma_map_f64(Z, 5, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
            }
        }
        return zmap;
    }
    void gdec(const C* F, C* Z, const SplitGroups& g) {
        if constexpr (n > 192) {
            throw SlError(SL_ERR_GENERIC, "shear-group passes: n <= 192");
        } else {
        if (g.count == 0) return;
        set_smem(k3g_dec<n, C>, G_SMEM);
        int nbands = 0;
        for (int i = 0; i < g.count; ++i) nbands += g.len[i];
        const CUtensorMap zmap = zmap_of(Z, g);
        LaunchScope ls(s, "f3g_dec", st, nbands);
        k3g_dec<n, C><<<dim3(g.count, S::H * S::Q), S::AC_THREADS, G_SMEM, st>>>(F, Z, nT, s.synth, g, tw, zmap);
        check_launch("k3g_dec");
        }
    }
    void grec(const C* Z, C* acc, const SplitGroups& g, int accumulate, int k2lo = 0, int k2hi = -1) {
        if constexpr (n > 192) {
            throw SlError(SL_ERR_GENERIC, "shear-group passes: n <= 192");
        } else {
        if (g.count == 0) return;
        constexpr size_t C_SMEM = GroupShape<n>::template smem_c<C>();
        set_smem(k3g_rec<n, C>, C_SMEM);
        if (k2hi < 0) k2hi = S::H;
        int nbands = 0;
        for (int i = 0; i < g.count; ++i) nbands += g.len[i];
        LaunchScope ls(s, "f3g_rec", st, nbands);
        const CUtensorMap zmap = zmap_of(Z, g);
        k3g_rec<n, C><<<dim3((k2hi - k2lo) * S::Q, 1), S::AC_THREADS, C_SMEM, st>>>(Z, nT, acc, s.synth, g, accumulate,
                                                                                   tw, zmap, k2lo * S::Q);
        check_launch("k3g_rec");
        }
    }
    // out[k2] (+)= in[k2]^T for planes [k2lo, k2hi)
    void transpose(const C* in, C* out, int add, int k2lo = 0, int k2hi = -1) {
        if (k2hi < 0) k2hi = S::H;
        if (k2hi <= k2lo) return;
        LaunchScope ls(s, "f3_transpose", st, 1);
        k3_plane_transpose<C><<<dim3((n + 31) / 32, (n + 31) / 32, k2hi - k2lo), dim3(32, 8), 0, st>>>(in, out, n, k2lo,
                                                                                                   add);
        check_launch("k3_plane_transpose");
    }
    void rec(const C* Z, C* acc, int nb, int band0, int accumulate, int k2lo = 0, int k2hi = -1) {
        set_smem(k3s_rec<n, C>, REC_SMEM);
        if (k2hi < 0) k2hi = S::H;
        LaunchScope ls(s, "f3s_rec", st, nb);
        k3s_rec<n, C><<<dim3((k2hi - k2lo) * S::Q, 1), S::AC_THREADS, REC_SMEM, st>>>(
            Z, nT, acc, nb, s.synth, band0, accumulate, tw, k2lo * S::Q);
        check_launch("k3s_rec");
    }
};

// F (natural layout) = FFT_0 FFT_1 R2C_2 f, with the five-pass kernels (once per call)
template <int n>
static void forward_natural(Fast3DLaunch<n>& K, System& s, const double* f) {
    s.w->inter.alloc(static_cast<size_t>(K.nT));
    s.w->F.alloc(static_cast<size_t>(K.nT));
    K.rows_r2c(f, 0, s.w->inter.p, 1);
    K.template axis1<-1>(s.w->inter.p, 1);
    K.template from_rot<-1, kAx0Plain>(s.w->inter.p, s.w->F.p, 1, 0, 0, "f3_ax0_fwd");
}
// out = Re IFFT(acc / W) / N
template <int n>
static void finish_rec(Fast3DLaunch<n>& K, System& s, double* out) {
    K.template to_rot<+1, kAx0DivW>(s.w->acc.p, 0, s.w->inter.p, 1, 0, s.WN.p, "f3_ax0_final");
    K.template axis1<+1>(s.w->inter.p, 1);
    K.rows_c2r(s.w->inter.p, out, 0, 1, nullptr, 0);
}

// fused denoise of this handle's bands up to the half-spectrum accumulator
// sum_b FFT(thr(band_b)) psi_b in s.w->acc (natural layout); out = null stops
// there (the distributed path reduces the accumulators across ranks first).
// slab_done(k2lo, k2hi), when set, runs after the last chunk's pass C has been
// issued for the accumulator slab [k2lo, k2hi) -- the slab is final on this
// rank from that point of the stream on (the multi-GPU reduce overlaps the rest)
using SlabHook = std::function<void(int, int)>;

// Passes A / C of a band chunk: per band (k3s_dec / k3s_rec) or by shear
// groups (k3g_dec / k3g_rec, fast3d_group.cuh; n <= 192), the pyramid-3 bands
// in the frame with axes 0 and 1 swapped (F^T in, accT out, folded back once).
template <int n, class C>
struct SplitPasses {
    System& s;
    Split3DLaunch<n, C>& S3;
    bool grouped = false, t3 = false;
    const C* F = nullptr;
    const C* FT = nullptr;
    C* acc = nullptr;
    C* accT = nullptr;
    bool acc_w = false, accT_w = false, folded = false;
    struct Chunk {
        std::vector<SplitGroups> norm, trans;
    };
    // F: the input spectrum (null for rec-only calls); acc: the accumulator
    // (null for dec-only calls). F^T / accT live in double2 workspaces (the
    // fp32 mode uses their front halves).
    SplitPasses(System& sys, Split3DLaunch<n, C>& l, const C* f, C* a) : s(sys), S3(l), F(f), acc(a) {
        grouped = s.knobs.group3d && n <= 192;
        if (grouped && s.knobs.t3)
            for (int b = s.lo; b < s.hi && !t3; ++b) t3 = s.bands3_host[static_cast<size_t>(b)].kind == 3;
        if (!t3) return;
        const size_t nT = static_cast<size_t>(S3.nT);
        if (F) {
            s.w->FT.alloc(nT);
            FT = reinterpret_cast<const C*>(s.w->FT.p);
            S3.transpose(F, reinterpret_cast<C*>(s.w->FT.p), 0);
        }
        if (acc) {
            s.w->accT.alloc(nT);
            accT = reinterpret_cast<C*>(s.w->accT.p);
        }
    }
    const BandDesc3D* tb() const { return t3 ? s.bands3.p : nullptr; }
    // shear groups of the global bands [gb0, gb0 + cb): consecutive bands of one
    // pyramid / scale / first shear (same shared row) form a group
    Chunk plan(int gb0, int cb) const {
        Chunk ck;
        if (!grouped) return ck;
        struct Prev {
            int band = -2, type = -1, p1 = -1, kind = -1;
        } pn, pt;
        for (int b = gb0; b < gb0 + cb; ++b) {
            const BandDesc3D& d = s.bands3_host[static_cast<size_t>(b)];
            const bool tr = t3 && d.kind == 3;
            const int type = d.kind == 0 ? kGrpLow : (d.kind == 3 ? (tr ? kGrpRowK1 : kGrpFull) : (d.kind == 4 ? kGrpRowK1 : kGrpRowK2));
            std::vector<SplitGroups>& v = tr ? ck.trans : ck.norm;
            Prev& pv = tr ? pt : pn;
            const bool ext = (type == kGrpRowK1 || type == kGrpRowK2) && pv.band == b - 1 && pv.type == type &&
                             pv.p1 == d.p1_off && pv.kind == d.kind && v.back().len[v.back().count - 1] < kMaxGroupLen;
            if (ext) {
                ++v.back().len[v.back().count - 1];
            } else {
                if (v.empty() || v.back().count == kMaxGroups) {
                    v.emplace_back();
                    std::memset(&v.back(), 0, sizeof(SplitGroups));
                    v.back().zb0 = gb0;
                }
                SplitGroups& g = v.back();
                g.first[g.count] = b;
                g.len[g.count] = 1;
                g.type[g.count] = static_cast<unsigned char>(type);
                ++g.count;
            }
            pv = Prev{b, type, d.p1_off, d.kind};
        }
        return ck;
    }
    void dec(C* Z, int gb0, int cb, const Chunk& ck) {
        if (!grouped) {
            S3.dec(F, Z, cb, gb0);
            return;
        }
        for (const SplitGroups& g : ck.norm) S3.gdec(F, Z, g);
        for (const SplitGroups& g : ck.trans) S3.gdec(FT, Z, g);
    }
    // pass C of the chunk for the accumulator planes [k2lo, k2hi)
    void rec(const C* Z, int gb0, int cb, const Chunk& ck, int k2lo = 0, int k2hi = -1) {
        if (!grouped) {
            S3.rec(Z, acc, cb, gb0, acc_w, k2lo, k2hi);
            return;
        }
        bool aw = acc_w, tw = accT_w;
        for (const SplitGroups& g : ck.norm) {
            S3.grec(Z, acc, g, aw, k2lo, k2hi);
            aw = true;
        }
        for (const SplitGroups& g : ck.trans) {
            S3.grec(Z, accT, g, tw, k2lo, k2hi);
            tw = true;
        }
    }
    void done_chunk(const Chunk& ck, int cb) {
        acc_w = acc_w || (grouped ? !ck.norm.empty() : cb > 0);
        accT_w = accT_w || !ck.trans.empty();
    }
    // acc (+)= accT^T for the planes [k2lo, k2hi); call after done_chunk of the last chunk
    void fold(int k2lo = 0, int k2hi = -1) {
        if (accT_w) S3.transpose(accT, acc, acc_w ? 1 : 0, k2lo, k2hi);
    }
};

// fused denoise of this handle's bands up to the half-spectrum accumulator
// sum_b FFT(thr(band_b)) psi_b in s.w->acc (natural layout); out = null stops
// there (the distributed path reduces the accumulators across ranks first).
// slab_done(k2lo, k2hi), when set, runs after the last chunk's pass C has been
// issued for the accumulator slab [k2lo, k2hi) -- the slab is final on this
// rank from that point of the stream on (the multi-GPU reduce overlaps the rest)
template <int n>
static void denoise3d_split_t(System& s, const double* f, double* stack, double* out, const double* delta,
                              cudaStream_t st, const SlabHook& slab_done = nullptr) {
    Fast3DLaunch<n> K(s, st);
    Split3DLaunch<n> S3(s, st);
    const int nb = s.nb();
    const int C = std::min(fast3d_chunk(s), nb);
    forward_natural<n>(K, s, f);
    s.w->inter.alloc(static_cast<size_t>(C) * K.nT);
    s.w->acc.alloc(static_cast<size_t>(K.nT));
    SplitPasses<n, double2> SP(s, S3, s.w->F.p, s.w->acc.p);
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        double* sb = stack ? stack + static_cast<size_t>(b0) * s.nreal : nullptr;
        const auto ck = SP.plan(s.lo + b0, cb);
        SP.dec(s.w->inter.p, s.lo + b0, cb, ck);
        S3.template mid<kMidFused>(s.w->inter.p, sb, nullptr, cb, delta, s.lo + b0, SP.tb());
        if (slab_done && b0 + cb >= nb) {
            constexpr int kSlabs = 4;
            const bool aw = SP.acc_w, tw = SP.accT_w;
            for (int j = 0; j < kSlabs; ++j) {
                const int lo = SplitShape<n>::H * j / kSlabs, hi = SplitShape<n>::H * (j + 1) / kSlabs;
                SP.acc_w = aw;
                SP.accT_w = tw;
                SP.rec(s.w->inter.p, s.lo + b0, cb, ck, lo, hi);
                SP.done_chunk(ck, cb);
                SP.fold(lo, hi);
                slab_done(lo, hi);
            }
            SP.folded = true;
        } else {
            SP.rec(s.w->inter.p, s.lo + b0, cb, ck);
            SP.done_chunk(ck, cb);
        }
    }
    if (!SP.folded) SP.fold();
    if (out) finish_rec<n>(K, s, out);
}

// out = Re IFFT(acc / W) / N of an accumulator in s.w->acc
template <int n>
static void finish3d_t(System& s, double* out, cudaStream_t st) {
    Fast3DLaunch<n> K(s, st);
    s.w->inter.alloc(static_cast<size_t>(K.nT));
    finish_rec<n>(K, s, out);
}

// fp32 mode (sl_system_set_precision(32)): the three passes on float2 spectra.
// The input's spectrum F and the final inverse of the accumulator -- one
// spectrum each per call, < 1 % of the work -- run in fp64 and are rounded.
__global__ void k_f32_to_f64(const float* __restrict__ in, double* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = static_cast<double>(in[i]);
}
__global__ void k_f64_to_f32(const double* __restrict__ in, float* __restrict__ out, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        out[i] = static_cast<float>(in[i]);
}
template <int n>
static void denoise3d_split_f32_t(System& s, const float* f, float* stack, float* out, const double* delta,
                                  cudaStream_t st) {
    Fast3DLaunch<n> K(s, st);
    Split3DLaunch<n, float2> S3(s, st);
    const int nb = s.nb();
    const int C = std::min(fast3d_chunk(s), nb);
    const long long nr = s.nreal;
    s.w->aux.alloc(static_cast<size_t>(K.nT) + static_cast<size_t>((nr + 1) / 2));
    double* f64 = reinterpret_cast<double*>(s.w->aux.p + K.nT);  // real staging after the fp32 spectra
    k_f32_to_f64<<<2048, 256, 0, st>>>(f, f64, nr);
    check_launch("k_f32_to_f64");
    forward_natural<n>(K, s, f64);  // s.w->F (double2)
    float2* F32 = reinterpret_cast<float2*>(s.w->aux.p);
    float2* acc32 = F32 + K.nT;  // second half of the aux block (K.nT float2 = K.nT / 2 double2)
    k_f64_to_f32<<<2048, 256, 0, st>>>(reinterpret_cast<const double*>(s.w->F.p), reinterpret_cast<float*>(F32),
                                       2 * K.nT);
    check_launch("k_f64_to_f32");
    s.w->inter.alloc(static_cast<size_t>(C) * K.nT);
    float2* Z = reinterpret_cast<float2*>(s.w->inter.p);
    SplitPasses<n, float2> SP(s, S3, F32, acc32);
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        float* sb = stack ? stack + static_cast<size_t>(b0) * nr : nullptr;
        const auto ck = SP.plan(s.lo + b0, cb);
        SP.dec(Z, s.lo + b0, cb, ck);
        S3.template mid<kMidFused>(Z, sb, nullptr, cb, delta, s.lo + b0, SP.tb());
        SP.rec(Z, s.lo + b0, cb, ck);
        SP.done_chunk(ck, cb);
    }
    SP.fold();
    s.w->acc.alloc(static_cast<size_t>(K.nT));
    k_f32_to_f64<<<2048, 256, 0, st>>>(reinterpret_cast<const float*>(acc32), reinterpret_cast<double*>(s.w->acc.p),
                                       2 * K.nT);
    check_launch("k_f32_to_f64");
    finish_rec<n>(K, s, f64);
    k_f64_to_f32<<<2048, 256, 0, st>>>(f64, out, nr);
    check_launch("k_f64_to_f32");
}

template <int n>
static void dec3d_split_t(System& s, const double* f, double* out, const double* delta, cudaStream_t st) {
    Fast3DLaunch<n> K(s, st);
    Split3DLaunch<n> S3(s, st);
    const int nb = s.nb();
    const int C = std::min(fast3d_chunk(s), nb);
    forward_natural<n>(K, s, f);
    s.w->inter.alloc(static_cast<size_t>(C) * K.nT);
    SplitPasses<n, double2> SP(s, S3, s.w->F.p, nullptr);
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        const auto ck = SP.plan(s.lo + b0, cb);
        SP.dec(s.w->inter.p, s.lo + b0, cb, ck);
        S3.template mid<kMidDec>(s.w->inter.p, out + static_cast<size_t>(b0) * s.nreal, nullptr, cb, delta, s.lo + b0,
                                 SP.tb());
    }
}

template <int n>
static void rec3d_split_t(System& s, const double* coeffs, double* out, cudaStream_t st) {
    Fast3DLaunch<n> K(s, st);
    Split3DLaunch<n> S3(s, st);
    const int nb = s.nb();
    const int C = std::min(fast3d_chunk(s), nb);
    s.w->inter.alloc(static_cast<size_t>(C) * K.nT);
    s.w->acc.alloc(static_cast<size_t>(K.nT));
    SplitPasses<n, double2> SP(s, S3, nullptr, s.w->acc.p);
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        const auto ck = SP.plan(s.lo + b0, cb);
        S3.template mid<kMidRec>(s.w->inter.p, nullptr, coeffs + static_cast<size_t>(b0) * s.nreal, cb, nullptr,
                                 s.lo + b0, SP.tb());
        SP.rec(s.w->inter.p, s.lo + b0, cb, ck);
        SP.done_chunk(ck, cb);
    }
    SP.fold();
    finish_rec<n>(K, s, out);
}

#define SLB_FAST3D_DISPATCH(FN, ...)                                        \
    switch (s.n[0]) {                                                       \
        case 64: FN<64>(__VA_ARGS__); break;                                \
        case 128: FN<128>(__VA_ARGS__); break;                              \
        case 192: FN<192>(__VA_ARGS__); break;                              \
        case 256: FN<256>(__VA_ARGS__); break;                              \
        default: throw SlError(SL_ERR_GENERIC, "fast3d: unsupported size"); \
    }

// the three-pass kernels by default (SLB_SPLIT3D=0: the five-pass ones, A/B)
static void dec3d_fast(System& s, const double* f, double* out, const double* delta, cudaStream_t st) {
    if (s.knobs.split3d) {
        SLB_FAST3D_DISPATCH(dec3d_split_t, s, f, out, delta, st)
    } else {
        SLB_FAST3D_DISPATCH(dec3d_fast_t, s, f, out, delta, st)
    }
}
static void rec3d_fast(System& s, const double* coeffs, double* out, cudaStream_t st) {
    if (s.knobs.split3d) {
        SLB_FAST3D_DISPATCH(rec3d_split_t, s, coeffs, out, st)
    } else {
        SLB_FAST3D_DISPATCH(rec3d_fast_t, s, coeffs, out, st)
    }
}

static void finish3d_fast(System& s, double* out, cudaStream_t st) { SLB_FAST3D_DISPATCH(finish3d_t, s, out, st) }

static void denoise3d_fast_f32(System& s, const float* f, float* stack, float* out, const double* delta,
                               cudaStream_t st) {
    SLB_FAST3D_DISPATCH(denoise3d_split_f32_t, s, f, stack, out, delta, st)
}

// the distributed variant: stop at the accumulator, calling slab_done per slab
static void denoise3d_split_acc(System& s, const double* f, double* stack, const double* delta, cudaStream_t st,
                                const SlabHook& slab_done) {
    switch (s.n[0]) {
        case 64: denoise3d_split_t<64>(s, f, stack, nullptr, delta, st, slab_done); break;
        case 128: denoise3d_split_t<128>(s, f, stack, nullptr, delta, st, slab_done); break;
        case 192: denoise3d_split_t<192>(s, f, stack, nullptr, delta, st, slab_done); break;
        case 256: denoise3d_split_t<256>(s, f, stack, nullptr, delta, st, slab_done); break;
        default: throw SlError(SL_ERR_GENERIC, "fast3d: unsupported size");
    }
}

static void denoise3d_fast(System& s, const double* f, double* stack, double* out, const double* delta,
                           cudaStream_t st) {
    if (s.knobs.split3d) {
        SLB_FAST3D_DISPATCH(denoise3d_split_t, s, f, stack, out, delta, st)
    } else {
        SLB_FAST3D_DISPATCH(denoise3d_fast_t, s, f, stack, out, delta, st)
    }
}

}  // namespace slb
