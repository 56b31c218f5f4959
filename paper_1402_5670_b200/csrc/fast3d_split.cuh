// Three-pass 3D dec -> threshold -> rec for cubic grids n = P * Q.
//
// The half spectrum of a band (k2 < H = n/2 + 1 along the real axis 2) makes
// three HBM round trips instead of five: the axis-1 FFT is split four-step
// style, k1 = q + Q p and i1 = a + P c, so that
//   y[a + P c] = sum_q w_Q^{c q} w_n^{a q} sum_p w_P^{a p} X[q + Q p],
// and each half rides along with a full axis:
//   pass A (k3s_dec): per (k2, q): the P lines k1 = q + Q p of F * psi_b (F in
//            registers across a band group, psi synthesised per line) get
//            the axis-0 IFFT, then the length-P DFT across the lines and the
//            twiddle w_n^{a q}                                  -> Z[k2][i0][q][a]
//   pass B (k3s_mid): per (i0, a pair): the length-Q DFT across q gives the
//            2Q rows i1 = a + P c; axis-2 c2r, 1/N, hard threshold, band
//            store; r2c, length-Q DFT back                     -> Z'[k2][i0][q][a]
//   pass C (k3s_rec): per (k2, q): twiddle, length-P DFT, axis-0 FFT,
//            * psi_b, summed over the chunk's bands in registers -> acc (RMW once)
// Z / Z' have the size of one half spectrum per band (H n n double2); pass B
// works in place. Per band: 16 Nh (A) + 16 Nh + 8 N + 16 Nh (B) + 16 Nh (C)
// bytes, against 5 passes (80 Nh + 8 N) in fast3d.cuh.
// Reference: transform.cpp:39-61 (forward 3D), :94-125 (inverse 3D),
// apps.cpp:57-81,114-121 (threshold, denoise), system3d.cpp:144-186 (psi).
#pragma once

#include "fast3d.cuh"

namespace slb {

template <int L>
struct SplitCfg;
template <>
struct SplitCfg<64> {
    static constexpr int P = 8, Q = 8;
};
template <>
struct SplitCfg<128> {
    static constexpr int P = 8, Q = 16;
};
template <>
struct SplitCfg<192> {
    static constexpr int P = 12, Q = 16;
};
template <>
struct SplitCfg<256> {
    static constexpr int P = 16, Q = 16;
};

// padded line buffers (e + e/8: conflict-free strided Stockham stores) in the
// FFT exchanges of the split kernels; the tiles they alias grow to fit
#ifndef SLB_SPLIT_PAD
#define SLB_SPLIT_PAD 0
#endif

template <int L>
struct SplitShape {
    static constexpr int T = RegPlan<L>::T, P = SplitCfg<L>::P, Q = SplitCfg<L>::Q;
    static constexpr int LD = P + 1;                 // [L][P] tile row stride: 8 consecutive rows hit distinct banks
    static constexpr int AC_THREADS = P * T;         // passes A / C: P axis-0 lines
    static constexpr int B_THREADS = Q * T;          // pass B: Q pair-lines = 2Q rows
    static constexpr int H = L / 2 + 1;
    static constexpr bool PAD = SLB_SPLIT_PAD;
    static constexpr int LB = LineBuf<L, PAD>::N;    // line buffer stride (double2)
    static constexpr size_t AC_ELEMS = static_cast<size_t>((L * LD > P * LB) ? L * LD : P * LB);
    static constexpr size_t B_ELEMS = static_cast<size_t>((H * 2 * Q > Q * LB) ? H * 2 * Q : Q * LB);
    static constexpr size_t AC_SMEM = AC_ELEMS * sizeof(double2);  // fp64; the fp32 mode needs half
    static constexpr size_t B_SMEM = B_ELEMS * sizeof(double2);
#ifndef SLB_SPLIT_AC_MINB
    static constexpr int AC_MINB = L >= 256 ? 1 : (L == 192 ? 2 : 4);
#else
    static constexpr int AC_MINB = SLB_SPLIT_AC_MINB;
#endif
#ifndef SLB_SPLIT_DEC_PF
    static constexpr bool DEC_PF = false;  // pass A: next band's filter line prefetched (A/B)
#else
    static constexpr bool DEC_PF = SLB_SPLIT_DEC_PF;
#endif
#ifndef SLB_SPLIT_REC_DB
    static constexpr bool REC_DB = true;  // pass C: double-buffered cp.async band tiles
#else
    static constexpr bool REC_DB = SLB_SPLIT_REC_DB;
#endif
#ifndef SLB_SPLIT_ZQUAD
    // quad-interleaved Z rows (zrow): measured 192^3 +0.7 % (pass B -5 %, A / C +3-4 %), 128^3 -5 %
    static constexpr bool ZQUAD = L == 192;
#else
    static constexpr bool ZQUAD = SLB_SPLIT_ZQUAD;
#endif
#ifndef SLB_SPLIT_B_DIRECT
    // pass B's Q-DFTs straight from / to Z in registers (measured: 128^3 pass B -6 %, 192^3 +5 %)
    static constexpr bool B_DIRECT = L <= 128;
#else
    static constexpr bool B_DIRECT = SLB_SPLIT_B_DIRECT;
#endif
#ifndef SLB_SPLIT_B_SWZ
    static constexpr bool B_SWZ = true;  // the (k, e)-pair conflict-free tile swizzle (192^3 pass B -0.6 % with cp.async too)
#else
    static constexpr bool B_SWZ = SLB_SPLIT_B_SWZ;
#endif
#ifndef SLB_SPLIT_B_MINB
    // 192 (with the single-exchange rows, X1): 3 CTAs/SM at 80 registers, 128 B
    // spilled, measured +3.4 % on the 3D step over 2 at 128 (without X1 the same
    // cap spills 356 B and loses 10 %; profiles/r2b_ab_passB_minb3.log)
    static constexpr int B_MINB = L >= 256 ? 1 : 3;
#else
    static constexpr int B_MINB = SLB_SPLIT_B_MINB;
#endif

};

// Offset of (q, a) inside one n-long Z row. ZQUAD: a is split into quads
// a = 4 aq + ar and the row is [aq][q][ar], so pass A / C's per-(k2, q) tiles
// move 64-byte runs and pass B's per-(i0, a pair) tiles 32-byte chunks at a
// 64-byte stride (8 lines per warp access instead of 16 for pass B; 3 lines per
// i0 for A / C instead of 2). Otherwise [q][a]: 192-byte runs for A / C, 32-byte
// chunks at a P * 16-byte stride for B.
template <int P, int Q, bool QUAD>
__host__ __device__ __forceinline__ int zrow(int q, int a) {
    if constexpr (QUAD) {
        static_assert(P % 4 == 0, "quads of a");
        return (a >> 2) * (4 * Q) + q * 4 + (a & 3);
    } else {
        return q * P + a;
    }
}

// pass B occupancy: the fp32 mode keeps 3 CTAs/SM below 256 (measured 2.6 %
// faster than 2 at 192), fp64 takes SplitShape::B_MINB
template <int L, class C>
struct SplitMinB {
    static constexpr int value = sizeof(C) == 16 ? SplitShape<L>::B_MINB : (L >= 256 ? 1 : 3);
};
// layout choices per precision: the fp32 mode (8-byte elements) measured 7 %
// faster at 192^3 with neither the quad-interleaved Z rows nor the pass-B swizzle
// (profiles/r2_ab_f32_layout.log)
template <int L, class C>
struct SplitLayout {
    static constexpr bool ZQUAD = sizeof(C) == 16 && SplitShape<L>::ZQUAD;
    static constexpr bool B_SWZ = sizeof(C) == 16 && SplitShape<L>::B_SWZ;
    static constexpr bool B_DIRECT = sizeof(C) == 16 && SplitShape<L>::B_DIRECT;  // measured in fp64 only
#ifndef SLB_SPLIT_B_X1
    static constexpr bool X1 = true;  // 192-point pass-B rows with one exchange per FFT (fft192_a / _b)
#else
    static constexpr bool X1 = SLB_SPLIT_B_X1;
#endif
};

// pass A keeps its F lines in registers across the band group (1) or reloads
// them per band from L2 (0: 24 fewer registers at 192)
#ifndef SLB_SPLIT_REGF
#define SLB_SPLIT_REGF 1
#endif

template <int R, int DIR, class C>
__device__ __forceinline__ void dft_small(C (&v)[R]) {
    if constexpr (R == 8)
        bfly8<DIR>(v);
    else if constexpr (R == 12)
        bfly12<DIR>(v);
    else if constexpr (R == 16)
        bfly16<DIR>(v);
}

// ---------------------------------------------------------------- pass A
template <int L, class C = double2>
__global__ void __launch_bounds__(SplitShape<L>::AC_THREADS, SplitShape<L>::AC_MINB)
    k3s_dec(const C* __restrict__ F, C* __restrict__ Z, long long zbs, FiltSynth3D filt, int band0, int G,
            int nb, const C* __restrict__ tw) {
    using S = SplitShape<L>;
    constexpr int T = S::T, E = RegPlan<L>::E, P = S::P, Q = S::Q, LD = S::LD, n = L;
    SLB_DYN_SMEM(C, tile);  // [n][LD]; the P line buffers alias it
    const int k2 = blockIdx.x / Q, q = blockIdx.x - k2 * Q;
    const int g0 = blockIdx.y * G, gn = min(G, nb - g0);
    const int p = threadIdx.x / T, t = threadIdx.x - p * T;
    const int k1 = q + Q * p;
    const C* fl = F + ((long long)k2 * n + k1) * n;
    C fr[E];
    if (SLB_SPLIT_REGF) {
#pragma unroll
        for (int m = 0; m < E; ++m) fr[m] = __ldg(fl + t + T * m);
    }
    C* lb = tile + p * S::LB;
    // PF: band b+1's filter line is synthesised (table loads in flight) while band b is in the FFT
    constexpr bool PF = S::DEC_PF;
    double pn[E];
    if (PF && gn > 0) {
        const FiltSynth3D::Ax0Line f0 = filt.ax0_line(filt.bands[band0 + g0], k1, k2);
#pragma unroll
        for (int m = 0; m < E; ++m) pn[m] = f0.at(t + T * m);
    }
    for (int bb = 0; bb < gn; ++bb) {
        const BandDesc3D bd = filt.bands[band0 + g0 + bb];
        const FiltSynth3D::Ax0Line fline = filt.ax0_line(bd, k1, k2);
        C x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const double ps = PF ? pn[m] : fline.at(t + T * m);
            const C f = SLB_SPLIT_REGF ? fr[m] : __ldg(fl + t + T * m);
            x[m] = mkc<C>(f.x * RealOf<C>(ps), f.y * RealOf<C>(ps));
        }
        if (PF && bb + 1 < gn) {
            const FiltSynth3D::Ax0Line fn = filt.ax0_line(filt.bands[band0 + g0 + bb + 1], k1, k2);
#pragma unroll
            for (int m = 0; m < E; ++m) pn[m] = fn.at(t + T * m);
        }
        if (bb > 0) __syncthreads();  // the previous band's tile is copied out
        reg_fft<L, +1, S::PAD>(x, lb, t, tw);
        __syncthreads();  // every line is done with the aliased buffers
#pragma unroll
        for (int m = 0; m < E; ++m) tile[(t + T * m) * LD + p] = x[m];
        __syncthreads();
        // length-P DFT across the lines for each i0, twiddle w_n^{a q}
        for (int i0 = threadIdx.x; i0 < n; i0 += S::AC_THREADS) {
            C v[P];
#pragma unroll
            for (int pp = 0; pp < P; ++pp) v[pp] = tile[i0 * LD + pp];
            dft_small<P, +1>(v);
#pragma unroll
            for (int a = 0; a < P; ++a) tile[i0 * LD + a] = a == 0 ? v[0] : cmul(v[a], twiddle<+1>(tw, a * q));
        }
        __syncthreads();
        // the CTA's P * T threads cover T rows i0 of P entries per step (row
        // offsets by compile-time strides, no per-element division)
        const int sa = threadIdx.x % P, si0 = threadIdx.x / P;
        C* z = Z + (long long)(g0 + bb) * zbs + (long long)k2 * n * n + zrow<P, Q, SplitLayout<L, C>::ZQUAD>(q, sa) + (long long)si0 * n;
#pragma unroll 4
        for (int j = 0; j < n / T; ++j) __stcg(z + (long long)j * T * n, tile[(si0 + T * j) * LD + sa]);
    }
}

// Pass B tile [H][2Q]: slot rr of row k XOR-swizzled with a function of k mod 8
// that keeps the per-line accesses (8 consecutive k, fixed rr), the row copies
// (consecutive rr) and the (k, e)-pair Q-DFT accesses (4 consecutive k x 2 e,
// slot 2 j + e) bank-conflict free for 16-byte elements. DIRECT: the Q-DFTs
// read / write Z straight from / to registers (no cp.async staging, no tile
// round trip for the copy-out).
template <int Q, bool DIRECT>
__device__ __forceinline__ int bslot(int k, int rr) {
    if constexpr (DIRECT)
        return k * (2 * Q) + (rr ^ (((k & 3) << 1) | ((k >> 2) & 1)));
    else
        return tslot<Q>(k, rr);
}

// The pair-packed c2r input of rows (2 lq, 2 lq + 1) with each half-spectrum
// entry read from the tile once: x[k] = X[k] + i Y[k] (k < H) and
// x[L - k] = conj(X[k]) + i conj(Y[k]) are formed by the thread owning k; the
// mirrored values travel to their owner (lane (T - t) mod T, register E - 1 - u)
// by warp shuffles (lane 0 keeps its own, register E - u). Needs L = T E with
// T a power of two <= 32 and the mirrored registers m > (H - 1) / T.
#ifndef SLB_SPLIT_C2R_SHFL
#define SLB_SPLIT_C2R_SHFL 1
#endif
template <int L, int T, int E, int Q, bool DIRECT, class C>
__device__ __forceinline__ void c2r_pack_shfl(const C* __restrict__ tile, int lq, int t, C (&x)[E]) {
    constexpr int H = L / 2 + 1;
    constexpr int UD = (H - 1) / T;  // registers u < UD are direct on every lane; u = UD on lane 0 only (k = L/2 when T | L/2)
    static_assert(T <= 32 && (T & (T - 1)) == 0 && T * E == L, "one power-of-two warp segment per line");
    static_assert(L % 2 == 0 && (L / 2) % T == 0, "k = L/2 sits on lane 0");
    C mir[UD];
#pragma unroll
    for (int u = 0; u <= UD; ++u) {
        const int k = t + T * u;
        if (u < UD || t == 0) {
            C X = tile[bslot<Q, DIRECT>(k, 2 * lq)];
            C Y = tile[bslot<Q, DIRECT>(k, 2 * lq + 1)];
            if (u < UD) mir[u] = mkc<C>(X.x + Y.y, Y.x - X.y);  // the value at L - k
            if (k == 0 || 2 * k == L) {
                X.y = 0.0;
                Y.y = 0.0;
            }
            x[u] = mkc<C>(X.x - Y.y, X.y + Y.x);
        }
    }
    const int src = (T - t) & (T - 1);
#pragma unroll
    for (int m = UD; m < E; ++m) {
        // lane t >= 1: k = t + T m mirrors k' = (T - t) + T (E - 1 - m) on lane T - t
        C v;
        v.x = __shfl_sync(0xffffffffu, mir[E - 1 - m < UD ? E - 1 - m : 0].x, src, T);
        v.y = __shfl_sync(0xffffffffu, mir[E - 1 - m < UD ? E - 1 - m : 0].y, src, T);
        if (t != 0) {
            x[m] = v;
        } else if (m > UD) {
            x[m] = mir[E - m];  // lane 0: k = T m mirrors T (E - m), its own register
        }
    }
}

// ---------------------------------------------------------------- pass B
enum SplitMid : int {
    kMidFused = 0,  // Z -> c2r, threshold, band store, r2c -> Z' (denoise)
    kMidDec = 1,    // Z -> c2r, threshold, band store                (forward)
    kMidRec = 2,    // band rows -> r2c -> Z'                         (inverse)
};

// One pass-B work item (i0 = bx / (P/2), a pair, band bi) on the CTA's tile.
// (A persistent variant that overlapped the next item's tile load with the
// current item measured 6.7 % slower at 192^3, profiles/r2b_ab_passB_persistent.log:
// the resident CTAs per SM already overlap each other's load and compute phases;
// so did an L2 bulk prefetch of the tile one wave of CTAs ahead, 2-3.5 % slower,
// r2b_ab_passB_l2_prefetch.log.)
template <int L, int MODE, bool STORE, class C>
__device__ __forceinline__ void mid_item(C* __restrict__ tile, int bx, int bi, C* __restrict__ Z,
                                         long long zbs, RealOf<C>* __restrict__ band, long long bbs,
                                         const RealOf<C>* __restrict__ bandin, RealOf<C> scale,
                                         const double* __restrict__ delta, int band0, const C* __restrict__ tw,
                                         const BandDesc3D* __restrict__ tb) {
    using S = SplitShape<L>;
    constexpr int T = S::T, E = RegPlan<L>::E, P = S::P, Q = S::Q, H = S::H, n = L;
    constexpr int KPT = (H + T - 1) / T;
    const int i0 = bx / (P / 2), a0 = 2 * (bx - i0 * (P / 2));
    const int lq = threadIdx.x / T, t = threadIdx.x - lq * T;  // pair-line c = lq: rows i1, i1 + 1
    const int i1 = a0 + P * lq;
    // tb: pyramid-3 bands run in the frame with axes 0 and 1 swapped
    // (fast3d_group.cuh); their rows (i0, i1) are the coefficient's rows (i1, i0)
    const bool trs = tb != nullptr && tb[band0 + bi].kind == 3;
    const long long roff = trs ? ((long long)i1 * n + i0) * n : ((long long)i0 * n + i1) * n;
    const long long rstep = trs ? (long long)n * n : (long long)n;  // row i1 + 1
    C* zb = Z + (long long)bi * zbs + (long long)i0 * n + zrow<P, Q, SplitLayout<L, C>::ZQUAD>(0, a0);  // + k2 n n + q ZS + e
    constexpr int ZS = SplitLayout<L, C>::ZQUAD ? 4 : P;  // distance between consecutive q at fixed a
    C* lb = tile + lq * S::LB;
    constexpr int KST = S::B_THREADS / (2 * Q);  // k2 rows per tile-copy step
    [[maybe_unused]] const int sj = threadIdx.x % (2 * Q), sk2 = threadIdx.x / (2 * Q);
    // X1: 192-point rows with one exchange per FFT (fft192_a / fft192_b, 12 x 16)
    constexpr bool X1 = L == 192 && SplitLayout<L, C>::X1;
    C x[X1 ? 16 : E];
    auto& xe = *reinterpret_cast<C(*)[E]>(&x[0]);  // the 16-major view (x[m] = element t + T m)
    if constexpr (MODE != kMidRec) {
        if constexpr (SplitLayout<L, C>::B_DIRECT) {
            // length-Q DFT over q for each (k2, e) straight from Z (lane pairs e = 0, 1
            // read one 32-byte sector per q), result into slot 2c + e
            for (int idx = threadIdx.x; idx < 2 * H; idx += S::B_THREADS) {
                const int k2 = idx >> 1, e = idx & 1;
                const C* zq = zb + (long long)k2 * n * n + e;
                C v[Q];
#pragma unroll
                for (int j = 0; j < Q; ++j) v[j] = __ldcg(zq + j * ZS);
                dft_small<Q, +1>(v);
#pragma unroll
                for (int j = 0; j < Q; ++j) tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, 2 * j + e)] = v[j];
            }
        } else {
            // KST k2-rows of 2Q slots per step (thread -> fixed slot, no per-element division)
#pragma unroll 4
            for (int k2 = sk2; k2 < H; k2 += KST)
                cp_async_c(tile + bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, sj), zb + (long long)k2 * n * n + (sj >> 1) * ZS + (sj & 1));
            cp_async_wait_all();
            __syncthreads();
            // length-Q DFT over q for each (k2, e), in place: slot 2q + e -> 2c + e
            for (int idx = threadIdx.x; idx < 2 * H; idx += S::B_THREADS) {
                const int e = idx / H, k2 = idx - e * H;
                C v[Q];
#pragma unroll
                for (int j = 0; j < Q; ++j) v[j] = tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, 2 * j + e)];
                dft_small<Q, +1>(v);
#pragma unroll
                for (int j = 0; j < Q; ++j) tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, 2 * j + e)] = v[j];
            }
        }
        __syncthreads();
        // axis-2 c2r of the row pair (pair-packed, as k2_rows_c2r)
        if constexpr (T <= 32 && SLB_SPLIT_C2R_SHFL) {
            c2r_pack_shfl<L, T, E, Q, SplitLayout<L, C>::B_SWZ>(tile, lq, t, xe);
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const int k = t + T * m;
                C X, Y;
                if (k < H) {
                    X = tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k, 2 * lq)];
                    Y = tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k, 2 * lq + 1)];
                    if (k == 0 || 2 * k == L) {
                        X.y = 0.0;
                        Y.y = 0.0;
                    }
                    xe[m] = mkc<C>(X.x - Y.y, X.y + Y.x);
                } else {
                    X = tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(L - k, 2 * lq)];
                    Y = tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(L - k, 2 * lq + 1)];
                    xe[m] = mkc<C>(X.x + Y.y, Y.x - X.y);
                }
            }
        }
        __syncthreads();  // the tile becomes the line buffers
        const double dl = delta ? delta[band0 + bi] : -1.0;
        RealOf<C>* r0p = band + (long long)bi * bbs + roff;
        auto thr_store = [&](C& v, int pos) {
            RealOf<C> u = v.x * scale, w = v.y * scale;
            if (dl >= 0.0) {
                if (fabs(u) < dl) u = 0.0;
                if (fabs(w) < dl) w = 0.0;
            }
            if (STORE) {
                r0p[pos] = u;
                r0p[rstep + pos] = w;
            }
            v = mkc<C>(u, w);
        };
        if constexpr (X1) {
            fft192_a<+1>(x, lb, t, tw);  // -> 12-major
            if (t < 12) {
#pragma unroll
                for (int r = 0; r < 16; ++r) thr_store(x[r], t + 12 * r);
            }
        } else {
            reg_fft<L, +1, S::PAD>(xe, lb, t, tw);
#pragma unroll
            for (int m = 0; m < E; ++m) thr_store(xe[m], t + T * m);
        }
        if constexpr (MODE == kMidDec) return;
    } else {
        const RealOf<C>* r0p = bandin + (long long)bi * bbs + roff;
        if constexpr (X1) {
            if (t < 12) {
#pragma unroll
                for (int r = 0; r < 16; ++r) x[r] = mkc<C>(__ldg(r0p + t + 12 * r), __ldg(r0p + rstep + t + 12 * r));
            }
        } else {
#pragma unroll
            for (int m = 0; m < E; ++m) xe[m] = mkc<C>(__ldg(r0p + t + T * m), __ldg(r0p + rstep + t + T * m));
        }
    }
    // axis-2 r2c of the row pair (as k2_rows_r2c)
    if constexpr (X1)
        fft192_b<-1>(x, lb, t, tw);  // 12-major -> 16-major
    else
        reg_fft<L, -1, S::PAD>(xe, lb, t, tw);
    C zk[KPT], zm[KPT];
    if constexpr (T <= 32 && SLB_ROWS_SHFL) {
        mirror_pairs_shfl<L, T, E, KPT>(xe, zk, zm, t);  // warp shuffles, no shared-memory round trip
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) lb[swz<S::PAD, L, sizeof(C)>(t + T * m)] = xe[m];
        line_sync<T>();
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int k = t + T * u;
            if (k < H) {
                zk[u] = lb[swz<S::PAD, L, sizeof(C)>(k)];
                zm[u] = lb[swz<S::PAD, L, sizeof(C)>(k == 0 ? 0 : L - k)];
            }
        }
    }
    __syncthreads();  // all line buffers read before the tile is rewritten
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        const int k = t + T * u;
        if (k < H) {
            tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k, 2 * lq)] = mkc<C>(RealOf<C>(0.5) * (zk[u].x + zm[u].x), RealOf<C>(0.5) * (zk[u].y - zm[u].y));
            tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k, 2 * lq + 1)] = mkc<C>(RealOf<C>(0.5) * (zk[u].y + zm[u].y), RealOf<C>(0.5) * (zm[u].x - zk[u].x));
        }
    }
    __syncthreads();
    // length-Q DFT back over c for each (k2, e): slot 2c + e -> q
    if constexpr (SplitLayout<L, C>::B_DIRECT) {
        for (int idx = threadIdx.x; idx < 2 * H; idx += S::B_THREADS) {
            const int k2 = idx >> 1, e = idx & 1;
            C v[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j) v[j] = tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, 2 * j + e)];
            dft_small<Q, -1>(v);
            C* zq = zb + (long long)k2 * n * n + e;
#pragma unroll
            for (int j = 0; j < Q; ++j) __stcg(zq + j * ZS, v[j]);
        }
    } else {
        for (int idx = threadIdx.x; idx < 2 * H; idx += S::B_THREADS) {
            const int e = idx / H, k2 = idx - e * H;
            C v[Q];
#pragma unroll
            for (int j = 0; j < Q; ++j) v[j] = tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, 2 * j + e)];
            dft_small<Q, -1>(v);
#pragma unroll
            for (int j = 0; j < Q; ++j) tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, 2 * j + e)] = v[j];
        }
        __syncthreads();
#pragma unroll 4
        for (int k2 = sk2; k2 < H; k2 += KST)
            __stcg(zb + (long long)k2 * n * n + (sj >> 1) * ZS + (sj & 1), tile[bslot<Q, SplitLayout<L, C>::B_SWZ>(k2, sj)]);
    }
}

template <int L, int MODE, bool STORE, class C = double2>
__global__ void __launch_bounds__(SplitShape<L>::B_THREADS, SplitMinB<L, C>::value)
    k3s_mid(C* __restrict__ Z, long long zbs, RealOf<C>* __restrict__ band, long long bbs,
            const RealOf<C>* __restrict__ bandin, RealOf<C> scale, const double* __restrict__ delta, int band0,
            const C* __restrict__ tw, const BandDesc3D* __restrict__ tb = nullptr) {
    SLB_DYN_SMEM(C, tile);  // [H][2Q] bslot<Q>; line buffers alias it
    mid_item<L, MODE, STORE, C>(tile, blockIdx.x, blockIdx.y, Z, zbs, band, bbs, bandin, scale, delta, band0,
                                tw, tb);
}

// ---------------------------------------------------------------- pass C
template <int L, class C = double2>
__global__ void __launch_bounds__(SplitShape<L>::AC_THREADS, SplitShape<L>::AC_MINB)
    k3s_rec(const C* __restrict__ Z, long long zbs, C* __restrict__ acc, int nbands, FiltSynth3D filt,
            int band0, int accumulate, const C* __restrict__ tw, int bx0 = 0) {
    using S = SplitShape<L>;
    constexpr int T = S::T, E = RegPlan<L>::E, P = S::P, Q = S::Q, LD = S::LD, n = L;
    SLB_DYN_SMEM(C, tile);  // [n][LD]; the P line buffers alias it
    const int bx = blockIdx.x + bx0;  // k2-slab launches (the multi-GPU reduce overlaps the last one)
    const int k2 = bx / Q, q = bx - k2 * Q;
    const int p = threadIdx.x / T, t = threadIdx.x - p * T;
    const int k1 = q + Q * p;
    // DB: band b+1's tile is loaded (cp.async) into the second buffer while band
    // b goes through the DFT / FFT / accumulate in the first
    constexpr bool DB = S::REC_DB;
    const int sa = threadIdx.x % P, si0 = threadIdx.x / P;
    auto load = [&](int b, C* buf) {
        const C* z = Z + (long long)b * zbs + (long long)k2 * n * n + zrow<P, Q, SplitLayout<L, C>::ZQUAD>(q, sa) + (long long)si0 * n;
#pragma unroll 4
        for (int j = 0; j < n / T; ++j) cp_async_c(buf + (si0 + T * j) * LD + sa, z + (long long)j * T * n);
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    C ar[E];
#pragma unroll
    for (int m = 0; m < E; ++m) ar[m] = mkc<C>(0.0, 0.0);
    if (DB && nbands > 0) load(0, tile);
    for (int b = 0; b < nbands; ++b) {
        C* cur = DB ? tile + (b & 1) * S::AC_ELEMS : tile;
        if (b > 0) __syncthreads();  // the previous band's line buffers (and its tile) are free
        if (DB) {
            if (b + 1 < nbands) {
                load(b + 1, tile + ((b + 1) & 1) * S::AC_ELEMS);
                asm volatile("cp.async.wait_group 1;" ::: "memory");  // band b landed, b+1 in flight
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
        } else {
            load(b, cur);
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncthreads();
        // twiddle w_n^{-a q}, length-P DFT over a -> p, for each i0
        for (int i0 = threadIdx.x; i0 < n; i0 += S::AC_THREADS) {
            C v[P];
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const C u = cur[i0 * LD + a];
                v[a] = a == 0 ? u : cmul(u, twiddle<-1>(tw, a * q));
            }
            dft_small<P, -1>(v);
#pragma unroll
            for (int pp = 0; pp < P; ++pp) cur[i0 * LD + pp] = v[pp];
        }
        __syncthreads();
        C x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = cur[(t + T * m) * LD + p];
        __syncthreads();  // all lines gathered: the tile becomes the line buffers
        const BandDesc3D bd = filt.bands[band0 + b];
        const FiltSynth3D::Ax0Line fline = filt.ax0_line(bd, k1, k2);
        reg_fft<L, -1, S::PAD>(x, cur + p * S::LB, t, tw);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const double ps = fline.at(t + T * m);
            ar[m].x = fma(x[m].x, RealOf<C>(ps), ar[m].x);
            ar[m].y = fma(x[m].y, RealOf<C>(ps), ar[m].y);
        }
    }
    C* d = acc + ((long long)k2 * n + k1) * n;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        C v = ar[m];
        if (accumulate) {
            const C o = __ldcg(d + t + T * m);
            v = mkc<C>(o.x + v.x, o.y + v.y);
        }
        __stcg(d + t + T * m, v);
    }
}

}  // namespace slb
