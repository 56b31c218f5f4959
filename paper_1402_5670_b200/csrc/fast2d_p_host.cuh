// Host orchestration of the persistent 2D kernels (fast2d_p.cuh).
#pragma once
#include "fast2d_host.cuh"
#include "fast2d_p.cuh"

namespace slb {

static int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        SL_CUDA(cudaGetDevice(&dev));
        SL_CUDA(cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev));
    }
    return n;
}

template <class Kern>
static int resident_blocks(Kern k, int threads, size_t smem) {
    int b = 0;
    SL_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, threads, smem));
    return std::max(1, b);
}

template <int L0, int L1>
struct Fast2DP {
    using RC = RowCfg<L1>;
    using CC = ColCfg<L0>;
    System& s;
    cudaStream_t st;
    int n0, H;
    long long nhT;
    const double2 *tw0, *tw1;
    size_t c2r_smem, r2c_smem, col_smem;
    int row_blocks, col_blocks;
    Fast2DP(System& sys, cudaStream_t stream) : s(sys), st(stream) {
        n0 = s.n[0];
        H = s.H;
        nhT = static_cast<long long>(H) * n0;
        tw0 = s.plan(L0, st).tw;
        tw1 = s.plan(L1, st).tw;
        c2r_smem = (2 * static_cast<size_t>(2 * RC::V) * H + static_cast<size_t>(RC::V) * L1) * sizeof(double2);
        r2c_smem = (static_cast<size_t>(2 * RC::V) * H + static_cast<size_t>(RC::V) * L1) * sizeof(double2);
        col_smem = static_cast<size_t>(CC::LINES) * L0 * sizeof(double2);
        row_blocks = (n0 + 2 * RC::V - 1) / (2 * RC::V);
        col_blocks = (H + CC::LINES - 1) / CC::LINES;
        set_smem(k2p_rows_c2r<L1>, c2r_smem);
        set_smem(k2p_rows_r2c<L1>, r2c_smem);
        set_smem(k2p_cols_dec<L0>, col_smem);
        set_smem(k2p_cols_rec<L0>, col_smem);
    }
    int row_grid(int nb, size_t smem, bool c2r) {
        const int per = c2r ? resident_blocks(k2p_rows_c2r<L1>, RC::THREADS, smem)
                            : resident_blocks(k2p_rows_r2c<L1>, RC::THREADS, smem);
        return std::max(1, std::min(nb * row_blocks, per * sm_count()));
    }
    int col_K(int nb, bool dec) {
        const int per = dec ? resident_blocks(k2p_cols_dec<L0>, CC::THREADS, col_smem)
                            : resident_blocks(k2p_cols_rec<L0>, CC::THREADS, col_smem);
        const int K = std::max(1, (per * sm_count()) / col_blocks);
        return std::max(1, std::min(K, nb));
    }
    void rows_r2c(const double* src, long long sbs, double2* dst, int nb, const char* nm) {
        LaunchScope ls(s, nm, st, nb);
        k2p_rows_r2c<L1><<<row_grid(nb, r2c_smem, false), RC::THREADS, r2c_smem, st>>>(src, sbs, dst, nhT, n0, H, nb,
                                                                                       tw1);
        check_launch("k2p_rows_r2c");
    }
    void rows_c2r(const double2* src, long long sbs, double* dst, long long dbs, int nb, const double* delta,
                  int band0, const char* nm) {
        LaunchScope ls(s, nm, st, nb);
        k2p_rows_c2r<L1><<<row_grid(nb, c2r_smem, true), RC::THREADS, c2r_smem, st>>>(
            src, sbs, dst, dbs, n0, H, 1.0 / static_cast<double>(s.nreal), delta, band0, nb, tw1);
        check_launch("k2p_rows_c2r");
    }
};

template <int L0, int L1>
static void dec2d_fastp_t(System& s, const double* f, double* out, const double* delta, cudaStream_t st) {
    Fast2DP<L0, L1> P(s, st);
    const int nb = s.nb();
    const Fast2DCfg cfg = fast2d_cfg(s);
    const int C = std::min(cfg.C, nb);
    s.w->inter.alloc(static_cast<size_t>(C) * P.nhT);
    s.w->F.alloc(static_cast<size_t>(P.nhT));
    using CC = ColCfg<L0>;
    set_smem(k2_cols_sum<L0, -1>, P.col_smem);
    P.rows_r2c(f, 0, s.w->inter.p, 1, "f2_rows_r2c");
    {
        LaunchScope ls(s, "f2_cols_fwd", st, 1);
        k2_cols_sum<L0, -1><<<P.col_blocks, CC::THREADS, P.col_smem, st>>>(s.w->inter.p, 0, 1, nullptr, s.w->F.p, P.H,
                                                                            P.tw0);
        check_launch("k2_cols_sum");
    }
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        const int K = P.col_K(cb, true);
        {
            LaunchScope ls(s, "f2_cols_dec", st, cb);
            k2p_cols_dec<L0><<<P.col_blocks * K, CC::THREADS, P.col_smem, st>>>(
                s.w->F.p, s.psiT.p, P.nhT, s.w->inter.p, P.nhT, P.H, s.lo + b0, cb, P.col_blocks, P.tw0);
            check_launch("k2p_cols_dec");
        }
        P.rows_c2r(s.w->inter.p, P.nhT, out + static_cast<size_t>(b0) * s.nreal, s.nreal, cb, delta, s.lo + b0,
                   delta ? "f2_rows_c2r_thr" : "f2_rows_c2r");
    }
}

template <int L0, int L1>
static void rec2d_fastp_t(System& s, const double* coeffs, double* out, cudaStream_t st) {
    Fast2DP<L0, L1> P(s, st);
    const int nb = s.nb();
    const Fast2DCfg cfg = fast2d_cfg(s);
    const int C = std::min(cfg.C, nb);
    s.w->inter.alloc(static_cast<size_t>(C) * P.nhT);
    int nslots = 0;
    for (int b0 = 0; b0 < nb; b0 += C) nslots += P.col_K(std::min(C, nb - b0), false);
    s.w->slots.alloc(static_cast<size_t>(nslots) * P.nhT);
    using CC = ColCfg<L0>;
    set_smem(k2_cols_sum<L0, +1>, P.col_smem);
    int slot0 = 0;
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        P.rows_r2c(coeffs + static_cast<size_t>(b0) * s.nreal, s.nreal, s.w->inter.p, cb, "f2_rows_r2c");
        const int K = P.col_K(cb, false);
        {
            LaunchScope ls(s, "f2_cols_rec", st, cb);
            k2p_cols_rec<L0><<<P.col_blocks * K, CC::THREADS, P.col_smem, st>>>(
                s.w->inter.p, P.nhT, s.psiT.p, P.nhT, s.w->slots.p, P.nhT, P.H, s.lo + b0, cb, P.col_blocks, slot0,
                P.tw0);
            check_launch("k2p_cols_rec");
        }
        slot0 += K;
    }
    {
        LaunchScope ls(s, "f2_cols_final", st, 1);
        k2_cols_sum<L0, +1><<<P.col_blocks, CC::THREADS, P.col_smem, st>>>(s.w->slots.p, P.nhT, nslots, s.WT.p,
                                                                            s.w->inter.p, P.H, P.tw0);
        check_launch("k2_cols_sum");
    }
    P.rows_c2r(s.w->inter.p, 0, out, 0, 1, nullptr, 0, "f2_rows_c2r");
}

static void dec2d_fastp(System& s, const double* f, double* out, const double* delta, cudaStream_t st) {
    SLB_FAST2D_DISPATCH(dec2d_fastp_t, s, f, out, delta, st)
}
static void rec2d_fastp(System& s, const double* coeffs, double* out, cudaStream_t st) {
    SLB_FAST2D_DISPATCH(rec2d_fastp_t, s, coeffs, out, st)
}

}  // namespace slb
