// Host orchestration of the specialised 2D path (kernels in fast2d.cuh).
#pragma once
#include <cstdlib>

#include "fast2d.cuh"
#include "launch.cuh"

namespace slb {

static bool fast2d_supported(const Knobs& k, int n0, int n1) {
    if (k.disable_fast2d) return false;
    if (n0 != n1) return false;
    switch (n0) {
        case 64: case 128: case 192: case 256: case 512: case 1024: case 2048: return true;
        default: return false;
    }
}

// Precision-specific tables of the fast 2D path: fp64 (the reference's
// precision) or the optional fp32 mode.
template <class C>
struct Prec2D;
template <>
struct Prec2D<double2> {
    static const double* psiT(const System& s) { return s.psiT.p; }
    static const double* WT(const System& s) { return s.WT.p; }
    static const double2* tw(const FftPlan& p) { return p.tw; }
};
template <>
struct Prec2D<float2> {
    static const float* psiT(const System& s) {
        if (!s.fp32) throw SlError(SL_ERR_CONFIG, "fp32 entry point on a system without fp32 tables (sl_system_set_precision)");
        return s.psiT32.p;
    }
    static const float* WT(const System& s) { return s.WT32.p; }
    static const float2* tw(const FftPlan& p) { return p.tw32; }
};
template <class C>
static C* ws_as(DBuf<double2>& b) {  // workspace buffers are sized for double2; float2 uses the front half
    return reinterpret_cast<C*>(b.p);
}

// Band grouping: G bands per column-pass CTA (F / accumulator reuse), C bands
// per chunk (one launch per pass and chunk).
struct Fast2DCfg {
    int G, C;
};
// Measured (tools/sweep2d.sh, tools/single2d.py): with >= 4 frames in flight on
// other streams the SMs stay busy, and G = 14-28 cuts the slot traffic of the rec
// sum (16 Nh per G bands) and the F re-reads, chunks of ~64 MiB; a lone frame
// takes every band in one chunk (up to 256 MiB) so each pass is one
// full-machine launch, G = 7 from 512^2 up.
static Fast2DCfg fast2d_cfg(const System& s) {
    if (s.lockstep_cfg) {
        // lock-step frame groups (4 frames): every band in one chunk and one
        // column group -- F and the accumulator stay in registers across all
        // bands, one slot per frame (512^2 +3 %, 256^2 +7 %, 1024^2 +1 % over
        // G = 28 / 64 MiB chunks; profiles/r2b_sweep_lockstep_r2c.log)
        const int G = knob_or(s.knobs.group, std::max(1, s.nb()));
        int C = knob_or(s.knobs.chunk, std::max(1, s.nb()));
        C = std::max(G, (C / G) * G);
        return {G, C};
    }
    const bool conc = s.concurrency >= 4;
    const double per = static_cast<double>(s.H) * s.n[0] * sizeof(double2);
    if (!conc) {
        // 2-3 frames in flight (the pipelined host batch's 3 compute streams):
        // G = 14 at 512^2 (e2e +2 % over 7, r1p tools/ab_group1.sh)
        const int G = s.concurrency > 1 ? knob_or(s.knobs.group2, s.n[0] >= 512 ? 14 : 4)
                                        : knob_or(s.knobs.group1, s.n[0] >= 512 ? 7 : 4);
        const int C = knob_or(s.knobs.chunk1, std::max(G, static_cast<int>((256.0 * 1024 * 1024) / per)));
        return {G, std::max(1, C)};
    }
    // G = 28 where 28 bands fit the 64 MiB chunk (512^2: one group per chunk,
    // +1.2 % over G = 14 after the register-resident column state, r1o sweep),
    // else 14 (1024^2: chunks of 14)
    const int cfit = std::max(1, static_cast<int>((64.0 * 1024 * 1024) / per));
    const int G = knob_or(s.knobs.group, cfit >= 28 ? 28 : 14);
    int C = knob_or(s.knobs.chunk, cfit);
    C = std::max(G, (C / G) * G);
    return {G, C};
}

template <int L0, int L1, class CX = double2>
static void dec2d_fast_t(System& s, const RealOf<CX>* f, RealOf<CX>* out, const double* delta, cudaStream_t st) {
    const int n0 = s.n[0], H = s.H;
    const long long nhT = static_cast<long long>(H) * n0;  // column-major half spectrum
    const Fast2DCfg cfg = fast2d_cfg(s);
    const int nb = s.nb();
    const int C = std::min(cfg.C, nb);
    s.w->inter.alloc(static_cast<size_t>(C) * nhT);
    s.w->F.alloc(static_cast<size_t>(nhT));
    const CX* tw0 = Prec2D<CX>::tw(s.plan(L0, st));
    const CX* tw1 = Prec2D<CX>::tw(s.plan(L1, st));
    using RC = RowCfg<L1>;
    using CC = ColCfg<L0>;
    const size_t row_smem = row_smem_bytes<L1, CX>(H);
    const size_t col_smem = col1_smem_bytes<L0, CX>();
    const size_t col2_smem = coldec_smem_bytes<L0, CX>();
    set_smem(k2_rows_r2c<L1, CX>, row_smem);
    set_smem(k2_rows_c2r<L1, CX>, row_smem);
    set_smem(k2_cols_sum<L0, -1, CX>, col_smem);
    set_smem(k2_cols_dec<L0, CX>, col2_smem);
    const int row_blocks = (n0 + 2 * RC::V - 1) / (2 * RC::V);
    const int col_blocks = (H + CC::LINES - 1) / CC::LINES;
    {  // F^T = FFT_0(FFT_1(f))
        LaunchScope ls(s, "f2_rows_r2c", st, 1);
        k2_rows_r2c<L1, CX><<<dim3(row_blocks, 1), RC::THREADS, row_smem, st>>>(f, 0, ws_as<CX>(s.w->inter), 0, n0, H, tw1);
        check_launch("k2_rows_r2c");
    }
    {
        LaunchScope ls(s, "f2_cols_fwd", st, 1);
        k2_cols_sum<L0, -1, CX><<<col_blocks, CC::THREADS, col_smem, st>>>(ws_as<CX>(s.w->inter), 0, 1, nullptr, ws_as<CX>(s.w->F), H, tw0);
        check_launch("k2_cols_sum");
    }
    const double scale = RealOf<CX>(1.0 / static_cast<double>(s.nreal));
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        const int groups = (cb + cfg.G - 1) / cfg.G;
        {
            LaunchScope ls(s, "f2_cols_dec", st, cb);
            k2_cols_dec<L0, CX><<<dim3(col_blocks, groups), CC::THREADS, col2_smem, st>>>(
                ws_as<CX>(s.w->F), Prec2D<CX>::psiT(s), nhT, ws_as<CX>(s.w->inter), nhT, H, s.lo + b0, cfg.G, cb, tw0);
            check_launch("k2_cols_dec");
        }
        {
            LaunchScope ls(s, delta ? "f2_rows_c2r_thr" : "f2_rows_c2r", st, cb);
            k2_rows_c2r<L1, CX><<<dim3(row_blocks, cb), RC::THREADS, row_smem, st>>>(
                ws_as<CX>(s.w->inter), nhT, out + static_cast<size_t>(b0) * s.nreal, s.nreal, n0, H, scale, delta, s.lo + b0, tw1);
            check_launch("k2_rows_c2r");
        }
    }
}

template <int L0, int L1, class CX = double2>
static void rec2d_fast_t(System& s, const RealOf<CX>* coeffs, RealOf<CX>* out, cudaStream_t st) {
    const int n0 = s.n[0], H = s.H;
    const long long nhT = static_cast<long long>(H) * n0;
    const Fast2DCfg cfg = fast2d_cfg(s);
    const int nb = s.nb();
    const int C = std::min(cfg.C, nb);
    s.w->inter.alloc(static_cast<size_t>(C) * nhT);
    int nslots = 0;
    for (int b0 = 0; b0 < nb; b0 += C) nslots += (std::min(C, nb - b0) + cfg.G - 1) / cfg.G;
    s.w->slots.alloc(static_cast<size_t>(nslots) * nhT);
    const CX* tw0 = Prec2D<CX>::tw(s.plan(L0, st));
    const CX* tw1 = Prec2D<CX>::tw(s.plan(L1, st));
    using RC = RowCfg<L1>;
    using CC = ColCfg<L0>;
    const size_t row_smem = row_smem_bytes<L1, CX>(H);
    const size_t col_smem = col1_smem_bytes<L0, CX>();
    const size_t col2_smem = coldec_smem_bytes<L0, CX>();
    set_smem(k2_rows_r2c<L1, CX>, row_smem);
    set_smem(k2_rows_c2r<L1, CX>, row_smem);
    set_smem(k2_cols_rec<L0, CX>, colrec_smem_bytes<L0, CX>());
    set_smem(k2_cols_sum<L0, +1, CX>, col_smem);
    const int row_blocks = (n0 + 2 * RC::V - 1) / (2 * RC::V);
    const int col_blocks = (H + CC::LINES - 1) / CC::LINES;
    if (s.w->done.n < static_cast<size_t>(col_blocks)) {  // zeroed once; the kernel resets its counters
        s.w->done.alloc(static_cast<size_t>(col_blocks));
        SL_CUDA(cudaMemsetAsync(s.w->done.p, 0, static_cast<size_t>(col_blocks) * sizeof(int), st));
    }
    int slot0 = 0;
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        const int groups = (cb + cfg.G - 1) / cfg.G;
        {
            LaunchScope ls(s, "f2_rows_r2c", st, cb);
            k2_rows_r2c<L1, CX><<<dim3(row_blocks, cb), RC::THREADS, row_smem, st>>>(
                coeffs + static_cast<size_t>(b0) * s.nreal, s.nreal, ws_as<CX>(s.w->inter), nhT, n0, H, tw1);
            check_launch("k2_rows_r2c");
        }
        {
            LaunchScope ls(s, "f2_cols_rec", st, cb);
            // the last chunk's CTAs also finish the reconstruction (k2_cols_rec)
            const bool fin = b0 + cb >= nb;
            k2_cols_rec<L0, CX><<<dim3(col_blocks, groups), CC::THREADS, colrec_smem_bytes<L0, CX>(), st>>>(
                ws_as<CX>(s.w->inter), nhT, Prec2D<CX>::psiT(s), nhT, ws_as<CX>(s.w->slots), nhT, H, s.lo + b0, cfg.G, cb, slot0, tw0,
                fin ? s.w->done.p : nullptr, nslots, Prec2D<CX>::WT(s), ws_as<CX>(s.w->inter));
            check_launch("k2_cols_rec");
        }
        slot0 += groups;
    }
    {
        LaunchScope ls(s, "f2_rows_c2r", st, 1);
        k2_rows_c2r<L1, CX><<<dim3(row_blocks, 1), RC::THREADS, row_smem, st>>>(
            ws_as<CX>(s.w->inter), 0, out, 0, n0, H, RealOf<CX>(1.0 / static_cast<double>(s.nreal)), nullptr, 0, tw1);
        check_launch("k2_rows_c2r");
    }
}

#define SLB_FAST2D_DISPATCH(FN, ...)                       \
    switch (s.n[0]) {                                      \
        case 64: FN<64, 64>(__VA_ARGS__); break;           \
        case 128: FN<128, 128>(__VA_ARGS__); break;        \
        case 192: FN<192, 192>(__VA_ARGS__); break;        \
        case 256: FN<256, 256>(__VA_ARGS__); break;        \
        case 512: FN<512, 512>(__VA_ARGS__); break;        \
        case 1024: FN<1024, 1024>(__VA_ARGS__); break;     \
        case 2048: FN<2048, 2048>(__VA_ARGS__); break;     \
        default: throw SlError(SL_ERR_GENERIC, "fast2d: unsupported size"); \
    }

#define SLB_FAST2D_DISPATCH_F32(FN, ...)                            \
    switch (s.n[0]) {                                               \
        case 64: FN<64, 64, float2>(__VA_ARGS__); break;            \
        case 128: FN<128, 128, float2>(__VA_ARGS__); break;         \
        case 192: FN<192, 192, float2>(__VA_ARGS__); break;         \
        case 256: FN<256, 256, float2>(__VA_ARGS__); break;         \
        case 512: FN<512, 512, float2>(__VA_ARGS__); break;         \
        case 1024: FN<1024, 1024, float2>(__VA_ARGS__); break;      \
        case 2048: FN<2048, 2048, float2>(__VA_ARGS__); break;      \
        default: throw SlError(SL_ERR_GENERIC, "fast2d: unsupported size"); \
    }

static void dec2d_fast(System& s, const double* f, double* out, const double* delta, cudaStream_t st) {
    SLB_FAST2D_DISPATCH(dec2d_fast_t, s, f, out, delta, st)
}
static void rec2d_fast(System& s, const double* coeffs, double* out, cudaStream_t st) {
    SLB_FAST2D_DISPATCH(rec2d_fast_t, s, coeffs, out, st)
}
static void dec2d_fast_f32(System& s, const float* f, float* out, const double* delta, cudaStream_t st) {
    SLB_FAST2D_DISPATCH_F32(dec2d_fast_t, s, f, out, delta, st)
}
static void rec2d_fast_f32(System& s, const float* coeffs, float* out, cudaStream_t st) {
    SLB_FAST2D_DISPATCH_F32(rec2d_fast_t, s, coeffs, out, st)
}

}  // namespace slb
