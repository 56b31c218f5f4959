// Pass launchers (rows r2c/c2r, strided lines) and half-spectrum geometry.
#pragma once
#include "common.cuh"

namespace slb {

// ---- generic pass launchers ------------------------------------------------
static void rows_r2c(System& s, const double* src, long long sbs, double2* dst, long long dbs, int nrows, int L,
                     int H, int ldh, int nbatch, cudaStream_t st) {
    const FftPlan& p = s.plan(L, st);
    LineCfg c = line_cfg(L, false);
    set_smem(k_rows_r2c, c.smem);
    const int npairs = (nrows + 1) / 2;
    dim3 grid((npairs + c.V - 1) / c.V, nbatch);
    LaunchScope ls(s, "rows_r2c", st, nbatch);
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
    LaunchScope ls(s, delta ? "rows_c2r_thr" : "rows_c2r", st, nbatch);
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
    static const char* names[4] = {"lines_plain", "lines_decmul", "lines_recmul", "lines_divw"};
    LaunchScope ls(s, names[MODE], st, nbatch);
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


}  // namespace slb
