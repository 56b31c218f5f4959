// Specialised 2D dec / rec kernels (register-resident FFT lines, compile-time
// lengths) for grids whose n0 and n1 both have a RegPlan.
//
// Layout: every half spectrum is stored column-major, X^T[k1][k0] with
// k1 < H = n1/2 + 1 and k0 < n0, so an axis-0 line is contiguous. The filter
// bank psi^T[b][k1][k0] (real) and W^T share that layout.
//
//   dec : cols_dec  (F^T * psi_b -> IFFT_0 -> inter^T[b])         per band group
//         rows_c2r  (inter^T -> pair-packed IFFT_1 -> 1/N, threshold -> band)
//   rec : rows_r2c  (band -> pair-packed FFT_1 -> inter^T[b])
//         cols_rec  (sum_{b in group} FFT_0(inter^T[b]) * psi_b -> slot)
//         cols_final(sum_slots / W -> IFFT_0 -> inter^T[0]) ; rows_c2r -> f
// The rows kernels stage the column-major intermediate through a
// [2V rows][H] shared tile (coalesced 2V*16-byte runs per k1); the pair's
// rows of that tile double as the line's FFT exchange buffer.
#pragma once

#include "fft_reg.cuh"

// r2c mirror pairs by warp shuffles where a line fits one warp segment (T <= 32)
#ifndef SLB_ROWS_SHFL
#define SLB_ROWS_SHFL 1
#endif

namespace slb {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
// one complex element: 16 bytes (double2, .cg: L2 only) or 8 bytes (float2, .ca)
template <class C>
__device__ __forceinline__ void cp_async_c(C* smem, const C* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    if constexpr (sizeof(C) == 16)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
    else
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}
// dynamic shared memory typed per instantiation (fp64 / fp32 kernels share the symbol)
#define SLB_DYN_SMEM(C, name)                                      \
    extern __shared__ __align__(16) unsigned char slb_dyn_smem[]; \
    C* name = reinterpret_cast<C*>(slb_dyn_smem)

__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Slot of (k, rr) in a [H][2V] tile: the rr index is XOR-swizzled with k so
// that both the dense global-order fills (consecutive rr) and the per-line
// reads (consecutive k, fixed rr) are bank-conflict free. 2V is a power of two.
template <int V>
__device__ __forceinline__ int tslot(int k, int rr) {
    return k * (2 * V) + (rr ^ (k & (2 * V - 1)));
}

// cols_dec: the FFTs' base twiddles loaded once per thread before the band
// loop (they depend only on the thread index) instead of per band: cols_dec
// -15 %; cols_rec (capped at 128 registers) spills with them and slows 38 %,
// so it keeps the table loads (profiles/r2b_ab_cols_twiddle_preload.log; at 3
// CTAs/SM without spills -35 %, r2b_ab_colrec_twpre_minb3.log; from a
// shared-memory copy of the table -11 %, r2b_ab_colrec_twiddles_smem.log)
#ifndef SLB_COL_TWPRE
#define SLB_COL_TWPRE 1
#endif
#ifndef SLB_COLREC_TWPRE
#define SLB_COLREC_TWPRE 0
#endif

// CTA shapes: rows kernels take V = 256 / T row pairs (256 threads; smem =
// [H][2V] tile + V line buffers); column kernels take 128 / T lines
// (128 threads, L * 16 B each).
template <int L>
struct RowCfg {
    static constexpr int T = RegPlan<L>::T;
#ifndef SLB_ROW_THREADS
    // 256 threads; 192 (the 3D rows pass) measured faster with 64 at 12 CTAs/SM
    // (fused rows -3 % vs 128 threads at 6, +18 % slower with 32 threads) and
    // 1024 with 512 at 2 CTAs/SM (2D 1024^2 +2.4 %)
    static constexpr int NT = L == 192 ? 64 : (L == 1024 ? 512 : 256);
    static constexpr int V = (NT / T) > 0 ? NT / T : 1;
#else
    static constexpr int V = (SLB_ROW_THREADS / T) > 0 ? SLB_ROW_THREADS / T : 1;
#endif
    static constexpr int THREADS = V * T;
    // the fused rows kernel: the same V row pairs with its own line split
    static constexpr int FUSED_T = FusedRowPlan<L>::T;
    static constexpr int FUSED_THREADS = V * FUSED_T;
#ifndef SLB_ROWS_PAD
    static constexpr bool PAD = false;  // padded line buffers in the fused rows kernel (A/B: -DSLB_ROWS_PAD=1)
#else
    static constexpr bool PAD = SLB_ROWS_PAD;
#endif
#ifndef SLB_FUSED_MINB
    // explicit occupancy targets (measured): without them ptxas takes 124-154
    // registers; 4 CTAs/SM (<= 64 registers) except 192 (12 CTAs of 64 threads,
    // <= 85 registers), 1024 (2 of 512 threads) and 2048 (2)
    static constexpr int FUSED_MIN_BLOCKS = L == 192 ? 12 : ((L == 2048 || L == 1024) ? 2 : 4);
#else
    static constexpr int FUSED_MIN_BLOCKS = SLB_FUSED_MINB;
#endif
};
template <int L>
struct ColCfg {
    static constexpr int T = ColPlan<L>::T;
#ifndef SLB_COL_THREADS
    static constexpr int LINES = (128 / T) > 0 ? 128 / T : 1;
#else
    static constexpr int LINES = (SLB_COL_THREADS / T) > 0 ? SLB_COL_THREADS / T : 1;
#endif
    static constexpr int THREADS = LINES * T;
#ifndef SLB_COL_MINB
    // measured: 4 CTAs/SM (<= 128 registers) beats 5 (<= 102) for the column passes
    static constexpr int MIN_BLOCKS = 65536 / (THREADS * 128) > 0 ? 65536 / (THREADS * 128) : 1;
#else
    static constexpr int MIN_BLOCKS = SLB_COL_MINB;
#endif
};

// dynamic shared memory of the kernels (line buffers padded, LineBuf<L>)
template <int L, class C = double2>
static size_t row_smem_bytes(int H) {  // [H][2V] tile; V padded line buffers alias it
    using RC = RowCfg<L>;
    return std::max(static_cast<size_t>(2 * RC::V) * H, static_cast<size_t>(RC::V) * LineBuf<L, RC::PAD>::N) * sizeof(C);
}
template <int L, class C = double2>
static size_t col1_smem_bytes() {  // one padded exchange buffer per line
    return static_cast<size_t>(ColCfg<L>::LINES) * LineBuf<L>::N * sizeof(C);
}
template <int L, class C = double2>
static size_t col2_smem_bytes() {  // exchange buffer + a second L-line (F column / accumulator)
    return static_cast<size_t>(ColCfg<L>::LINES) * (LineBuf<L>::N + L) * sizeof(C);
}

// accumulator in registers (measured: cols_rec<512> -6 %, <1024> -10 %); at
// 192 it spills under the 128-register cap, so that length keeps the
// shared-memory accumulator
template <int L>
struct ColRec {
#ifndef SLB_COLREC_REGACC
    static constexpr bool REGACC = L != 192;
#else
    static constexpr bool REGACC = SLB_COLREC_REGACC;
#endif
#ifndef SLB_COLREC_PF
    static constexpr bool PF = false;  // register prefetch of the next band (A/B)
#else
    static constexpr bool PF = SLB_COLREC_PF;
#endif
    // CPA: band b+1's line is copied (cp.async, double-buffered per line) while
    // band b is in the FFT. Measured: the kernel alone -5 %, but the 4-stream
    // lock-step batch -3 % (51 KB instead of 18 KB of smem per CTA crowds out the
    // concurrently resident passes; profiles/r2_ab_colrec_cpa.log) -> opt-in
#ifndef SLB_COLREC_CPA
    static constexpr bool CPA = false;
#else
    static constexpr bool CPA = !PF && REGACC && SLB_COLREC_CPA;
#endif
};
template <int L, class C = double2>
static size_t colrec_smem_bytes() {  // register accumulator: exchange buffers (+ 2 staged lines per line with CPA)
    if (ColRec<L>::CPA) return static_cast<size_t>(ColCfg<L>::LINES) * (LineBuf<L>::N + 2 * L) * sizeof(C);
    return ColRec<L>::REGACC ? col1_smem_bytes<L, C>() : col2_smem_bytes<L, C>();
}

// ---------------------------------------------------------------- rows c2r
// In : src[k1 * n0 + r] (column-major half spectrum), bands strided by sbs.
// Out: dst[r * L + i] real rows, scaled, optionally thresholded (delta >= 0).
template <int L, class C = double2>
__global__ void __launch_bounds__(RowCfg<L>::THREADS)
    k2_rows_c2r(const C* __restrict__ src, long long sbs, RealOf<C>* __restrict__ dst, long long dbs, int n0,
                int H, RealOf<C> scale, const double* __restrict__ delta, int band0, const C* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E, V = RowCfg<L>::V;
    using R = RealOf<C>;
    SLB_DYN_SMEM(C, tile);  // [H][2V] swizzled tile, then V line buffers of L
    const int r0 = blockIdx.x * 2 * V;
    src += blockIdx.y * sbs;
    dst += blockIdx.y * dbs;
    const int nrows = min(2 * V, n0 - r0);
    // all tile loads in flight at once (cp.async, 16 B each, L2 only); the
    // smem slot order follows the global order so each warp's writes are dense
    // thread -> fixed slot rr, k-rows strided by a compile-time step
    constexpr int KS = RowCfg<L>::THREADS / (2 * V);
    const int rr = threadIdx.x % (2 * V);
#pragma unroll 4
    for (int k = threadIdx.x / (2 * V); k < H; k += KS) {
        if (rr < nrows)
            cp_async_c(tile + tslot<V>(k, rr), src + (long long)k * n0 + r0 + rr);
        else
            tile[tslot<V>(k, rr)] = mkc<C>(0.0, 0.0);
    }
    cp_async_wait_all();
    __syncthreads();
    const int q = threadIdx.x / T, t = threadIdx.x - q * T;
    C x[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int k = t + T * m;
        C X, Y;
        if (k < H) {
            X = tile[tslot<V>(k, 2 * q)];
            Y = tile[tslot<V>(k, 2 * q + 1)];
            if (k == 0 || 2 * k == L) {
                X.y = 0.0;
                Y.y = 0.0;
            }
            x[m] = mkc<C>(X.x - Y.y, X.y + Y.x);  // X + iY
        } else {
            X = tile[tslot<V>(L - k, 2 * q)];
            Y = tile[tslot<V>(L - k, 2 * q + 1)];
            x[m] = mkc<C>(X.x + Y.y, Y.x - X.y);  // conj(X) + i conj(Y)
        }
    }
    // the tile is dead once every line has gathered its inputs: the line
    // exchange buffers alias it (H*2V >= V*L), halving shared memory per CTA
    __syncthreads();
    C* lb = tile + q * LineBuf<L, false>::N;
    reg_fft<L, +1, false>(x, lb, t, tw);
    const double dl = delta ? delta[band0 + blockIdx.y] : -1.0;
    const int ra = r0 + 2 * q;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        R a = x[m].x * scale, b = x[m].y * scale;
        if (dl >= 0.0) {
            if (fabs(a) < dl) a = 0.0;
            if (fabs(b) < dl) b = 0.0;
        }
        const int i = t + T * m;
        if (ra < n0) dst[(long long)ra * L + i] = a;
        if (ra + 1 < n0) dst[(long long)(ra + 1) * L + i] = b;
    }
}

// ---------------------------------------------------------------- rows r2c
// In : real rows src[r * L + i]; Out: column-major half spectrum dst[k1 * n0 + r].
template <int L, class C = double2>
__global__ void __launch_bounds__(RowCfg<L>::THREADS)
    k2_rows_r2c(const RealOf<C>* __restrict__ src, long long sbs, C* __restrict__ dst, long long dbs, int n0,
                int H, const C* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E, V = RowCfg<L>::V;
    using R = RealOf<C>;
    constexpr int KPT = (L / 2 + 1 + T - 1) / T;  // split outputs per thread
    SLB_DYN_SMEM(C, tile);            // [H][2V] swizzled tile, then V line buffers
    const int r0 = blockIdx.x * 2 * V;
    src += blockIdx.y * sbs;
    dst += blockIdx.y * dbs;
    const int q = threadIdx.x / T, t = threadIdx.x - q * T;
    const int ra = r0 + 2 * q;
    C x[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
        const int i = t + T * m;
        const R a = ra < n0 ? __ldg(src + (long long)ra * L + i) : R(0);
        const R b = ra + 1 < n0 ? __ldg(src + (long long)(ra + 1) * L + i) : R(0);
        x[m] = mkc<C>(a, b);
    }
    C* lb = tile + q * LineBuf<L, false>::N;  // line buffers alias the (not yet used) output tile
    reg_fft<L, -1, false>(x, lb, t, tw);
    // Z in registers (element t + T m); mirror pairs by warp shuffles, or
    // through the line buffer for lines wider than a warp
    C zk[KPT], zm[KPT];
    if constexpr (T <= 32 && SLB_ROWS_SHFL) {
        mirror_pairs_shfl<L, T, E, KPT>(x, zk, zm, t);
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) lb[swz<false, L, sizeof(C)>(t + T * m)] = x[m];
        line_sync<T>();
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int k = t + T * u;
            if (k < H) {
                zk[u] = lb[swz<false, L, sizeof(C)>(k)];
                zm[u] = lb[swz<false, L, sizeof(C)>(k == 0 ? 0 : L - k)];
            }
        }
    }
    __syncthreads();  // all line buffers read before the tile is written
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        const int k = t + T * u;
        if (k < H) {
            tile[tslot<V>(k, 2 * q)] = mkc<C>(R(0.5) * (zk[u].x + zm[u].x), R(0.5) * (zk[u].y - zm[u].y));      // X
            tile[tslot<V>(k, 2 * q + 1)] = mkc<C>(R(0.5) * (zk[u].y + zm[u].y), R(0.5) * (zm[u].x - zk[u].x));  // Y
        }
    }
    __syncthreads();
    const int nrows = min(2 * V, n0 - r0);
    constexpr int KS = RowCfg<L>::THREADS / (2 * V);
    const int rr = threadIdx.x % (2 * V);
#pragma unroll 4
    for (int k = threadIdx.x / (2 * V); k < H; k += KS)
        if (rr < nrows) __stcg(dst + (long long)k * n0 + r0 + rr, tile[tslot<V>(k, rr)]);
}

// ---------------------------------------------------------------- column lines
// Column k1 of a column-major half spectrum is the contiguous line src[k1 * L ...].

// dec: inter[b] = IFFT_0(F * psi_b) for the G bands of this CTA's group.
// F column in registers instead of shared memory at 3 CTAs/SM (measured per
// length: cols_dec<512> -4 %, <256> -8 %; <1024> +7 %, kept in shared memory)
template <int L>
struct ColDec {
#ifndef SLB_COLDEC_REGF
    static constexpr bool REGF = L == 256 || L == 512;
#else
    static constexpr bool REGF = SLB_COLDEC_REGF;
#endif
#ifndef SLB_COLDEC_MINB
    static constexpr int MIN_BLOCKS = REGF ? 3 : ColCfg<L>::MIN_BLOCKS;
#else
    static constexpr int MIN_BLOCKS = SLB_COLDEC_MINB;
#endif
};
template <int L, class C = double2>
static size_t coldec_smem_bytes() {
    return ColDec<L>::REGF ? col1_smem_bytes<L, C>() : col2_smem_bytes<L, C>();
}
template <int L, class C = double2>
__global__ void __launch_bounds__(ColCfg<L>::THREADS, ColDec<L>::MIN_BLOCKS)
    k2_cols_dec(const C* __restrict__ FT, const RealOf<C>* __restrict__ psiT, long long pbs,
                C* __restrict__ inter, long long ibs, int H, int band0, int G, int nb,
                const C* __restrict__ tw, long long fzs = 0, long long izs = 0) {
    FT += blockIdx.z * fzs;  // blockIdx.z: frame of a lock-step batch
    inter += blockIdx.z * izs;
    constexpr int T = ColPlan<L>::T, E = ColPlan<L>::E;
    using R = RealOf<C>;
    SLB_DYN_SMEM(C, lbuf);  // per line: [exchange L][F column L]
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const int k1 = blockIdx.x * ColCfg<L>::LINES + li;
    const bool valid = k1 < H;
    C* sm = lbuf + li * (LineBuf<L>::N + (ColDec<L>::REGF ? 0 : L));
    C* fs = sm + LineBuf<L>::N;
    C fr[E];
    if (ColDec<L>::REGF) {
#pragma unroll
        for (int m = 0; m < E; ++m) fr[m] = valid ? __ldg(FT + (long long)k1 * L + t + T * m) : mkc<C>(0.0, 0.0);
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            if (valid)
                cp_async_c(fs + t + T * m, FT + (long long)k1 * L + t + T * m);
            else
                fs[t + T * m] = mkc<C>(0.0, 0.0);
        }
        cp_async_wait_all();
    }
    const int g0 = blockIdx.y * G;
    const int gn = min(G, nb - g0);
    [[maybe_unused]] TwPreK<ColPlan<L>, L, +1, C> twp;
    if constexpr (SLB_COL_TWPRE) twp.load(tw, t);
    // psi of band b+1 is loaded while band b is in the FFT
    R p[E];
    {
        const R* ps = psiT + (long long)(band0 + g0) * pbs + (long long)k1 * L;
#pragma unroll
        for (int m = 0; m < E; ++m) p[m] = (valid && gn > 0) ? __ldg(ps + t + T * m) : R(0);
    }
    for (int bb = 0; bb < gn; ++bb) {
        const int b = g0 + bb;
        C x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const C fv = ColDec<L>::REGF ? fr[m] : fs[t + T * m];
            x[m] = mkc<C>(fv.x * p[m], fv.y * p[m]);  // conj(psi) * F, psi real
        }
        if (bb + 1 < gn) {
            const R* ps = psiT + (long long)(band0 + b + 1) * pbs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) p[m] = valid ? __ldg(ps + t + T * m) : R(0);
        }
        if constexpr (SLB_COL_TWPRE)
            reg_fft_pw<ColPlan<L>, L, +1>(x, sm, t, twp);
        else
            reg_fft_p<ColPlan<L>, L, +1>(x, sm, t, tw);
        if (valid) {
            C* o = inter + (long long)b * ibs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) __stcg(o + t + T * m, x[m]);
        }
        line_sync<T>();
    }
}

// final rec column pass for one line: IFFT_0((sum_s slot[s]) / W) -> out; also
// the plain forward column FFT (F = FFT_0 of the rows pass) when W == nullptr &&
// DIR < 0. Slots are summed in index order (deterministic).
template <int L, int DIR, class C = double2>
__device__ __forceinline__ void cols_sum_line(const C* __restrict__ slots, long long sbs, int nslots,
                                              const RealOf<C>* __restrict__ WT, C* __restrict__ out, int k1,
                                              bool valid, C* sm, int t, const C* __restrict__ tw) {
    constexpr int T = ColPlan<L>::T, E = ColPlan<L>::E;
    using R = RealOf<C>;
    C x[E];
#pragma unroll
    for (int m = 0; m < E; ++m) x[m] = mkc<C>(0.0, 0.0);
    if (valid) {
        // slots summed in order; two slots' loads in flight per step
        int s = 0;
        for (; s + 1 < nslots; s += 2) {
            const C* in0 = slots + (long long)s * sbs + (long long)k1 * L;
            const C* in1 = in0 + sbs;
            C u[E], v[E];
#pragma unroll
            for (int m = 0; m < E; ++m) {
                u[m] = __ldcg(in0 + t + T * m);
                v[m] = __ldcg(in1 + t + T * m);
            }
#pragma unroll
            for (int m = 0; m < E; ++m) x[m] = cadd(cadd(x[m], u[m]), v[m]);
        }
        for (; s < nslots; ++s) {
            const C* in = slots + (long long)s * sbs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) x[m] = cadd(x[m], __ldcg(in + t + T * m));
        }
        if (WT) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const R w = __ldg(WT + (long long)k1 * L + t + T * m);
                x[m] = mkc<C>(x[m].x / w, x[m].y / w);
            }
        }
    }
    reg_fft_p<ColPlan<L>, L, DIR>(x, sm, t, tw);
    if (valid) {
        C* o = out + (long long)k1 * L;
#pragma unroll
        for (int m = 0; m < E; ++m) __stcg(o + t + T * m, x[m]);
    }
}

// rec: slot[g] = sum_{b in group g} FFT_0(inter[b]) * psi_b.
#ifndef SLB_COLREC_MINB
#define SLB_COLREC_MINB ColCfg<L>::MIN_BLOCKS
#endif
template <int L, class C = double2>
__global__ void __launch_bounds__(ColCfg<L>::THREADS, SLB_COLREC_MINB)
    k2_cols_rec(const C* __restrict__ inter, long long ibs, const RealOf<C>* __restrict__ psiT, long long pbs,
                C* __restrict__ slots, long long sbs, int H, int band0, int G, int nb, int slot0,
                const C* __restrict__ tw, int* __restrict__ done, int nslots, const RealOf<C>* __restrict__ WT,
                C* __restrict__ fout, long long izs = 0, long long szs = 0, long long fozs = 0) {
    inter += blockIdx.z * izs;  // blockIdx.z: frame of a lock-step batch
    slots += blockIdx.z * szs;
    fout += blockIdx.z * fozs;
    if (done) done += blockIdx.z * gridDim.x;
    constexpr int T = ColPlan<L>::T, E = ColPlan<L>::E;
    using R = RealOf<C>;
    SLB_DYN_SMEM(C, lbuf);  // per line: [exchange L][accumulator L]
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const int k1 = blockIdx.x * ColCfg<L>::LINES + li;
    const bool valid = k1 < H;
    // per line: [exchange L] (+ [accumulator L] unless it lives in registers)
    C* sm = lbuf + li * (LineBuf<L>::N + (ColRec<L>::CPA ? 2 * L : (ColRec<L>::REGACC ? 0 : L)));
    C* acc = sm + LineBuf<L>::N;  // thread t owns acc[t + T m]
    C ar[E];
#pragma unroll
    for (int m = 0; m < E; ++m) {
        ar[m] = mkc<C>(0.0, 0.0);
        if (!ColRec<L>::REGACC) acc[t + T * m] = ar[m];
    }
    const int g0 = blockIdx.y * G;
    const int gn = min(G, nb - g0);
    // PF: band b+1's line and psi are loaded into registers while band b is in
    // the FFT (the kernel is DRAM-latency bound at ~4 warps per scheduler)
    constexpr bool PF = ColRec<L>::PF;
    C xn[E];
    R pn[E];
    if (PF && gn > 0) {
        const C* in = inter + (long long)g0 * ibs + (long long)k1 * L;
        const R* ps = psiT + (long long)(band0 + g0) * pbs + (long long)k1 * L;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            xn[m] = valid ? __ldcg(in + t + T * m) : mkc<C>(0.0, 0.0);
            pn[m] = valid ? __ldg(ps + t + T * m) : R(0);
        }
    }
    [[maybe_unused]] TwPreK<ColPlan<L>, L, -1, C> twp;
    if constexpr (SLB_COLREC_TWPRE) twp.load(tw, t);
    constexpr bool CPA = ColRec<L>::CPA;
    C* stg = sm + LineBuf<L>::N;  // CPA: two staged lines [2][L] after the exchange buffer
    auto stage = [&](int b, int buf) {  // each thread copies exactly the elements it reads back
        if (valid) {
            const C* in = inter + (long long)b * ibs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) cp_async_c(stg + buf * L + t + T * m, in + t + T * m);
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    if (CPA && gn > 0) stage(g0, 0);
    for (int bb = 0; bb < gn; ++bb) {
        const int b = g0 + bb;
        C x[E];
        R p[E];
        if (CPA) {
            if (bb + 1 < gn) {
                stage(b + 1, (bb + 1) & 1);
                asm volatile("cp.async.wait_group 1;" ::: "memory");  // band b landed, b+1 in flight
            } else {
                asm volatile("cp.async.wait_group 0;" ::: "memory");
            }
            const C* cur = stg + (bb & 1) * L;
#pragma unroll
            for (int m = 0; m < E; ++m) x[m] = valid ? cur[t + T * m] : mkc<C>(0.0, 0.0);
            const R* ps = psiT + (long long)(band0 + b) * pbs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) p[m] = valid ? __ldg(ps + t + T * m) : R(0);
        } else if (PF) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                x[m] = xn[m];
                p[m] = pn[m];
            }
            if (bb + 1 < gn) {
                const C* in = inter + (long long)(b + 1) * ibs + (long long)k1 * L;
                const R* ps = psiT + (long long)(band0 + b + 1) * pbs + (long long)k1 * L;
#pragma unroll
                for (int m = 0; m < E; ++m) {
                    xn[m] = valid ? __ldcg(in + t + T * m) : mkc<C>(0.0, 0.0);
                    pn[m] = valid ? __ldg(ps + t + T * m) : R(0);
                }
            }
        } else {
            const C* in = inter + (long long)b * ibs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) x[m] = valid ? __ldcg(in + t + T * m) : mkc<C>(0.0, 0.0);
            // the band's psi is loaded before the FFT so its latency overlaps it
            const R* ps = psiT + (long long)(band0 + b) * pbs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) p[m] = valid ? __ldg(ps + t + T * m) : R(0);
        }
        if constexpr (SLB_COLREC_TWPRE)
            reg_fft_pw<ColPlan<L>, L, -1>(x, sm, t, twp);
        else
            reg_fft_p<ColPlan<L>, L, -1>(x, sm, t, tw);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            C a = ColRec<L>::REGACC ? ar[m] : acc[t + T * m];
            a.x = fma(x[m].x, p[m], a.x);
            a.y = fma(x[m].y, p[m], a.y);
            if (ColRec<L>::REGACC)
                ar[m] = a;
            else
                acc[t + T * m] = a;
        }
        line_sync<T>();
    }
    if (valid) {
        C* o = slots + (long long)(slot0 + blockIdx.y) * sbs + (long long)k1 * L;
#pragma unroll
        for (int m = 0; m < E; ++m) __stcg(o + t + T * m, ColRec<L>::REGACC ? ar[m] : acc[t + T * m]);
    }
    if (done == nullptr) return;
    // last chunk: the CTA that finishes its column block last sums every slot
    // (in slot order, as k2_cols_sum), divides by W and runs the final IFFT_0,
    // so the reconstruction needs no separate sum launch
    __shared__ int last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const int prev = atomicAdd(done + blockIdx.x, 1);
        last = prev == static_cast<int>(gridDim.y) - 1;
        if (last) done[blockIdx.x] = 0;  // reset for the next call on this workspace
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    cols_sum_line<L, +1, C>(slots, sbs, nslots, WT, fout, k1, valid, sm, t, tw);
}

template <int L, int DIR, class C = double2>
__global__ void __launch_bounds__(ColCfg<L>::THREADS)
    k2_cols_sum(const C* __restrict__ slots, long long sbs, int nslots, const RealOf<C>* __restrict__ WT,
                C* __restrict__ out, int H, const C* __restrict__ tw, long long szs = 0,
                long long ozs = 0) {
    slots += blockIdx.z * szs;  // blockIdx.z: frame of a lock-step batch
    out += blockIdx.z * ozs;
    constexpr int T = ColPlan<L>::T;
    SLB_DYN_SMEM(C, lbuf);
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const int k1 = blockIdx.x * ColCfg<L>::LINES + li;
    cols_sum_line<L, DIR, C>(slots, sbs, nslots, WT, out, k1, k1 < H, lbuf + li * LineBuf<L>::N, t, tw);
}

}  // namespace slb
