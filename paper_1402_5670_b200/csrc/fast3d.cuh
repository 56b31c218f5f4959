// Specialised 3D dec / rec kernels for cubic grids with a RegPlan length.
//
// Half spectra (H = n2/2 + 1) live in two layouts, both without padding:
//   rotated  R[k2][i0][k1]  (k1 fastest) -- what the rows pass (axis 2,
//            pair-packed, reused from fast2d.cuh with n0*n1 rows) reads/writes
//   natural  N[k2][k1][k0]  (k0 fastest) -- F, the accumulator and W
// Passes:
//   axis 1 : contiguous lines of R, in place                     (k3_lines_contig)
//   axis 0 : N -> R  (contiguous load, rotated staged store)      (k3_ax0_to_rot)
//            R -> N  (rotated staged load, contiguous store/RMW)  (k3_ax0_from_rot)
// The 3D filter psi_b(k0, k1, k2) is synthesised in registers from the
// per-scale factor tables (system3d.cpp:144-186), so no filter bank is read.
#pragma once

#include "fast2d.cuh"
#include "kernels.cuh"

namespace slb {

// [L][V] staging tile, v XOR-swizzled with i0 (dense fills, conflict-free line reads)
template <int V>
__device__ __forceinline__ int aslot(int i0, int v) {
    return i0 * V + (v ^ (i0 & (V - 1)));
}

template <int L>
struct Ax0Cfg {
    static constexpr int T = RegPlan<L>::T;
#ifndef SLB_AX0_V
    static constexpr int V = 8;  // lines (consecutive k1) per CTA -> 128-byte rotated runs
#else
    static constexpr int V = SLB_AX0_V;
#endif
    static constexpr int THREADS = V * T;
    // occupancy targets (CTAs/SM, measured at 128^3 / 192^3; overridable for A/B builds)
#ifndef SLB_AX0_TO_MINB
    // N -> R (192: 4 CTAs, 128 registers with the F line held in registers --
    // 6 CTAs at <= 85 registers without it; 256: 4 CTAs of 256 threads, 64
    // registers: 36.2 vols/s at 256^3 vs 35.1 with 3 and 32.3 with 2)
    static constexpr int TO_MIN_BLOCKS = 4;
#else
    static constexpr int TO_MIN_BLOCKS = SLB_AX0_TO_MINB;
#endif
#ifndef SLB_AX0_FROM_MINB
    static constexpr int FROM_MIN_BLOCKS = 4;  // R -> N (192 with the filter prefetch: 4 beats 5)
#else
    static constexpr int FROM_MIN_BLOCKS = SLB_AX0_FROM_MINB;
#endif
#ifndef SLB_LINES_MINB
    static constexpr int LINES_MIN_BLOCKS = 5;
#else
    static constexpr int LINES_MIN_BLOCKS = SLB_LINES_MINB;
#endif
};

// ---------------------------------------------------------------- axis 1 (contiguous lines, in place)
template <int L, int DIR>
__global__ void __launch_bounds__(ColCfg<L>::THREADS, Ax0Cfg<L>::LINES_MIN_BLOCKS)
    k3_lines_contig(double2* __restrict__ data, long long bstride, long long nlines, const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E;
    extern __shared__ double2 lbuf[];
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const long long line = (long long)blockIdx.x * ColCfg<L>::LINES + li;
    const bool valid = line < nlines;
    double2* d = data + blockIdx.y * bstride + line * L;
    double2 x[E];
#pragma unroll
    for (int m = 0; m < E; ++m) x[m] = valid ? __ldcg(d + t + T * m) : make_double2(0.0, 0.0);
    reg_fft<L, DIR, false>(x, lbuf + li * LineBuf<L, false>::N, t, tw);
    if (valid) {
#pragma unroll
        for (int m = 0; m < E; ++m) __stcg(d + t + T * m, x[m]);
    }
}

// N -> R keeps the F line in registers across the band group at 128 / 192
// (4 CTAs/SM; with the per-line filter setup: ax0 dec -12 % at 192 vs 6 CTAs
// without it, -1.5 % at 128 together with no filter prefetch there)
#ifndef SLB_AX0_TO_REGF
#define SLB_AX0_TO_REGF(L) ((L) == 128 || (L) == 192)
#endif
#ifndef SLB_AX0_FROM_REGACC
#define SLB_AX0_FROM_REGACC 0  // A/B: R -> N band sum in registers
#endif
#ifndef SLB_AX0_LINEFILT
#define SLB_AX0_LINEFILT 1  // per-line filter setup (FiltSynth3D::ax0_line); 0: get_d per element (A/B)
#endif
// filter prefetch up to this line length (measured with the per-line filter
// setup: it pays only at 64 for N -> R and up to 128 for R -> N)
#ifndef SLB_AX0_PF_TO_MAXL
#define SLB_AX0_PF_TO_MAXL 64
#endif
#ifndef SLB_AX0_PF_FROM_MAXL
#define SLB_AX0_PF_FROM_MAXL 128
#endif

enum Ax0Mode : int {
    kAx0Plain = 0,   // no filter
    kAx0DecMul = 1,  // prologue x *= conj(psi) (psi real)
    kAx0RecAcc = 2,  // epilogue acc (+)= x * psi
    kAx0DivW = 3,    // prologue x /= W
};

// ---------------------------------------------------------------- axis 0: N -> R
// Line (k2, k1) = contiguous N[(k2*n + k1)*n + k0]; output element (k2, i0, k1)
// goes to R[(k2*n + i0)*n + k1], staged through the tile so each i0 writes V
// consecutive k1 (a 128-byte run).
template <int L, int DIR, int MODE>
__global__ void __launch_bounds__(Ax0Cfg<L>::THREADS, Ax0Cfg<L>::TO_MIN_BLOCKS)
    k3_ax0_to_rot(const double2* __restrict__ src, long long sbs, double2* __restrict__ dst, long long dbs, int H,
                  FiltSynth3D filt, int band0, int G, int nb, const double* __restrict__ WN,
                  const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E, V = Ax0Cfg<L>::V;
    constexpr int n = L;
    extern __shared__ double2 tile[];  // [L][V] tile; the V line buffers alias it
    const int lines_per_k2 = n / V;
    const int k2 = blockIdx.x / lines_per_k2;
    const int k1_0 = (blockIdx.x - k2 * lines_per_k2) * V;
    // DecMul: CTA y handles bands [g0, g0 + gn) of the chunk, re-reading the same
    // F lines (L1/L2 hits after the first band); other modes: one spectrum per y.
    const int g0 = MODE == kAx0DecMul ? blockIdx.y * G : 0;
    const int gn = MODE == kAx0DecMul ? min(G, nb - g0) : 1;
    if (MODE != kAx0DecMul) {
        src += blockIdx.y * sbs;
        dst += blockIdx.y * dbs;
    }
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const int k1 = k1_0 + li;
    const double2* s = src + ((long long)k2 * n + k1) * n;
    double2* lb = tile + li * LineBuf<L, false>::N;  // line exchange buffers alias the output tile
    // PF: the next band's filter values are synthesised while this band is in
    // the FFT (DecMul) / before the FFT (RecAcc); measured per direction
    constexpr bool PF = L <= SLB_AX0_PF_TO_MAXL;
    // REGF: DecMul's F line loaded once into registers for the whole band group
    constexpr bool REGF = MODE == kAx0DecMul && SLB_AX0_TO_REGF(L);
    double2 fr[E];
    if (REGF) {
#pragma unroll
        for (int m = 0; m < E; ++m) fr[m] = __ldg(s + t + T * m);
    }
    double pn[E];
    if (PF && MODE == kAx0DecMul) {
        const BandDesc3D bd = filt.bands[band0 + g0];
        const FiltSynth3D::Ax0Line fl = filt.ax0_line(bd, k1, k2);
#pragma unroll
        for (int m = 0; m < E; ++m) pn[m] = SLB_AX0_LINEFILT ? fl.at(t + T * m) : filt.get_d(bd, t + T * m, k1, k2);
    }
    for (int bb = 0; bb < gn; ++bb) {
        BandDesc3D bd{};
        if (MODE == kAx0DecMul) bd = filt.bands[band0 + g0 + bb];
        FiltSynth3D::Ax0Line fl{};
        if (MODE == kAx0DecMul && !PF) fl = filt.ax0_line(bd, k1, k2);
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k0 = t + T * m;
            double2 z = REGF ? fr[m] : (MODE == kAx0DecMul ? __ldg(s + k0) : __ldcg(s + k0));
            if (MODE == kAx0DecMul) {
                const double p = PF ? pn[m] : (SLB_AX0_LINEFILT ? fl.at(k0) : filt.get_d(bd, k0, k1, k2));
                z = make_double2(z.x * p, z.y * p);
            } else if (MODE == kAx0DivW) {
                const double w = __ldg(WN + ((long long)k2 * n + k1) * n + k0);
                z = make_double2(z.x / w, z.y / w);
            }
            x[m] = z;
        }
        if (PF && MODE == kAx0DecMul && bb + 1 < gn) {
            const BandDesc3D bn = filt.bands[band0 + g0 + bb + 1];
            const FiltSynth3D::Ax0Line fn = filt.ax0_line(bn, k1, k2);
#pragma unroll
            for (int m = 0; m < E; ++m) pn[m] = SLB_AX0_LINEFILT ? fn.at(t + T * m) : filt.get_d(bn, t + T * m, k1, k2);
        }
        if (bb > 0) __syncthreads();  // previous band's tile fully written out
        reg_fft<L, DIR, false>(x, lb, t, tw);
        __syncthreads();              // every line's FFT is done with the aliased buffers
        // publish into the [i0][v] tile, then write 128-byte rotated runs
#pragma unroll
        for (int m = 0; m < E; ++m) tile[aslot<V>(t + T * m, li)] = x[m];
        __syncthreads();
        double2* o = dst + (long long)(g0 + bb) * dbs + (long long)k2 * n * n + k1_0;
        for (int idx = threadIdx.x; idx < V * L; idx += blockDim.x) {
            const int i0 = idx / V, v = idx - i0 * V;
            __stcg(o + (long long)i0 * n + v, tile[aslot<V>(i0, v)]);
        }
    }
    (void)H;
}

// ---------------------------------------------------------------- axis 0: R -> N
// kAx0RecAcc: one CTA walks the chunk's bands [0, nbands) in order, summing
// FFT_0(x_b) psi_b in registers, then read-modify-writes the accumulator once
// (acc (+)= sum; deterministic, independent of the stream count). Other modes:
// one spectrum per blockIdx.y.
template <int L, int DIR, int MODE>
__global__ void __launch_bounds__(Ax0Cfg<L>::THREADS, Ax0Cfg<L>::FROM_MIN_BLOCKS)
    k3_ax0_from_rot(const double2* __restrict__ src, long long sbs, double2* __restrict__ dst, long long dbs, int nbands,
                    FiltSynth3D filt, int band0, int accumulate, const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E, V = Ax0Cfg<L>::V;
    constexpr int n = L;
    extern __shared__ double2 tile[];  // [L][V] tile (line buffers alias it) [+ V accumulator lines]
    const int lines_per_k2 = n / V;
    const int k2 = blockIdx.x / lines_per_k2;
    const int k1_0 = (blockIdx.x - k2 * lines_per_k2) * V;
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const int k1 = k1_0 + li;
    double2* lb = tile + li * LineBuf<L, false>::N;  // line exchange buffers alias the input tile (after the gather)
    if (MODE != kAx0RecAcc) {
        src += blockIdx.y * sbs;
        dst += blockIdx.y * dbs;
    }
    const int nb = MODE == kAx0RecAcc ? nbands : 1;
    // RecAcc: per-thread accumulator slots after the tile (acc[li][t + T m]),
    // registers stay free for the FFT line
    double2* acc = tile + V * LineBuf<L, false>::N + li * L;
    constexpr bool REGACC = MODE == kAx0RecAcc && SLB_AX0_FROM_REGACC;
    double2 ar[E];
    if (MODE == kAx0RecAcc) {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            ar[m] = make_double2(0.0, 0.0);
            if (!REGACC) acc[t + T * m] = ar[m];
        }
    }
    double2 x[E];
    for (int b = 0; b < nb; ++b) {
        const double2* si = src + (long long)b * sbs + (long long)k2 * n * n + k1_0;
        if (b > 0) __syncthreads();  // previous band's line buffers are free again
        for (int idx = threadIdx.x; idx < V * L; idx += blockDim.x) {
            const int i0 = idx / V, v = idx - i0 * V;
            cp_async16(tile + aslot<V>(i0, v), si + (long long)i0 * n + v);
        }
        cp_async_wait_all();
        __syncthreads();
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = tile[aslot<V>(t + T * m, li)];
        __syncthreads();  // all lines gathered: the tile becomes the line buffers
        constexpr bool PF = L <= SLB_AX0_PF_FROM_MAXL;  // see k3_ax0_to_rot
        double p[E];  // this band's filter values, synthesised before the FFT
        if (PF && MODE == kAx0RecAcc) {
            const BandDesc3D bd = filt.bands[band0 + b];
            const FiltSynth3D::Ax0Line fl = filt.ax0_line(bd, k1, k2);
#pragma unroll
            for (int m = 0; m < E; ++m) p[m] = SLB_AX0_LINEFILT ? fl.at(t + T * m) : filt.get_d(bd, t + T * m, k1, k2);
        }
        reg_fft<L, DIR, false>(x, lb, t, tw);
        if (MODE == kAx0RecAcc) {
            const BandDesc3D bd = filt.bands[band0 + b];
            FiltSynth3D::Ax0Line fl{};
            if (!PF) fl = filt.ax0_line(bd, k1, k2);
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const double p_ = PF ? p[m] : (SLB_AX0_LINEFILT ? fl.at(t + T * m) : filt.get_d(bd, t + T * m, k1, k2));
                double2 a = REGACC ? ar[m] : acc[t + T * m];
                a.x = fma(x[m].x, p_, a.x);
                a.y = fma(x[m].y, p_, a.y);
                if (REGACC)
                    ar[m] = a;
                else
                    acc[t + T * m] = a;
            }
            (void)bd;
        }
    }
    double2* d = dst + ((long long)k2 * n + k1) * n;
    if (MODE == kAx0RecAcc) {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            double2 v = REGACC ? ar[m] : acc[t + T * m];
            if (accumulate) {
                const double2 o = __ldcg(d + t + T * m);
                v = make_double2(o.x + v.x, o.y + v.y);
            }
            __stcg(d + t + T * m, v);
        }
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) __stcg(d + t + T * m, x[m]);
    }
}

// [i0][i1][ldh] row-major half (build layout) -> natural N[k2][k1][k0]
__global__ void k3_half_to_natural(const double* __restrict__ in, double* __restrict__ out, int n, int H, int ldh) {
    const long long tot = (long long)H * n * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot; e += (long long)gridDim.x * blockDim.x) {
        const int k0 = (int)(e % n);
        const long long r = e / n;
        const int k1 = (int)(r % n);
        const int k2 = (int)(r / n);
        out[e] = in[((long long)k0 * n + k1) * ldh + k2];
    }
}

}  // namespace slb
