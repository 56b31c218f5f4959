// Shear-group passes A / C of the three-pass 3D path (fast3d_split.cuh).
//
// Every 3D shearlet spectrum is a product of factors that each depend on two
// of the three frequency indices (system3d.cpp:144-186):
//   psi_b(k) = g(k_pa) Phi_{s1(b)}(k_pa, k_s1) Phi_{s2(b)}(k_pa, k_s2).
// On an axis-0 line (k1, k2 fixed) of a band whose principal axis is 1 or 2
// (pyramids 4 / 5) only Phi_{s1(b)}(k_pa, k0) varies, and it is the same for
// every band of the pyramid and scale with the same first shear -- the
// 2^l + 1 (or 2^l - 1) bands of one "shear group", consecutive in the band
// order (index loop k2 innermost, taps.cpp: enumerate_3d). So
//   dec: IFFT_0(F psi_b) = s_b(k1, k2) IFFT_0(F A)         (A = shared row)
//   rec: sum_b psi_b FFT_0(y_b) = A FFT_0(sum_b s_b(k1, k2) y_b)
// and passes A / C run ONE axis-0 FFT per group instead of one per band; per
// band only the length-P DFT across the CTA's lines (and its Z tile) is left.
// Pyramid-3 bands (principal axis 0) factor the same way after swapping axes 0
// and 1 of the problem: the spectrum F^T[k2][k0][k1] goes through the same
// kernels, pass B stores the coefficient rows transposed (k3s_mid, `tb`), and
// their reconstruction sums into a transposed accumulator that is added back
// once. The lowpass factors as hJ(k0) * (hJ(k1) hJ(k2)).
// Reference: transform.cpp:39-61,94-125 (forward / inverse 3D), apps.cpp:114-121.
#pragma once

#include "fast3d_split.cuh"
#include "tma.cuh"

namespace slb {

enum GroupType : int {
    kGrpFull = 0,  // one band, the full axis-0 filter line (pyramid 3 without the transposed frame)
    kGrpRowK1 = 1, // A = Phi_{s1}(k1, .), s_b = g(k1) Phi_{s2}(k1, k2)   (pyramid 4; pyramid 3 transposed)
    kGrpRowK2 = 2, // A = Phi_{s1}(k2, .), s_b = g(k2) Phi_{s2}(k2, k1)   (pyramid 5)
    kGrpLow = 3,   // A = hJ(.),           s_b = hJ(k1) hJ(k2)            (lowpass)
};
constexpr int kMaxGroups = 128;  // groups per launch (the host splits longer lists)
constexpr int kMaxGroupLen = 16; // bands per group (the host splits longer runs)

struct SplitGroups {
    int count;
    int zb0;  // global band index of Z slot 0 (the chunk's first band)
    int first[kMaxGroups];  // global band index of each group's first band
    unsigned char len[kMaxGroups];
    unsigned char type[kMaxGroups];
};

#ifndef SLB_GROUP_C_TMA3
#define SLB_GROUP_C_TMA3 1
#endif
template <int L>
struct GroupShape {
    using S = SplitShape<L>;
    static_assert(S::AC_THREADS >= L, "one thread per output row i0 in the across-line DFTs");
    static constexpr size_t SC_BYTES = static_cast<size_t>(kMaxGroupLen) * S::P * sizeof(double);
    template <class C>
    static constexpr size_t smem() {  // two [n][LD] tiles + the band scalars + 2 mbarriers (+ 1024-byte alignment for TMA)
        return 2 * S::AC_ELEMS * sizeof(C) + SC_BYTES + 16 + S::P * sizeof(C) + 1024;
    }
#ifndef SLB_GROUP_A_MINB
    static constexpr int A_MINB = 2;
#else
    static constexpr int A_MINB = SLB_GROUP_A_MINB;
#endif
#ifndef SLB_GROUP_TMA
#define SLB_GROUP_TMA 1
#endif
    // pass A's Z tiles leave through TMA bulk tensor stores (fp64, 192: the
    // quad-interleaved Z rows as a 5D tensor, 64-byte swizzled staging)
    template <class C>
    static constexpr bool TMA_STORE = SLB_GROUP_TMA && sizeof(C) == 16 &&
                                      ((L == 192 && SplitLayout<L, C>::ZQUAD) || (L == 128 && !SplitLayout<L, C>::ZQUAD));
    // slot of (i0, a) in a TMA-staged tile: dense [i0][a] rows of P * 16 bytes,
    // 64-byte swizzle for 192 (quad rows), 128-byte for 128 (plain rows)
    __device__ __forceinline__ static int tslot_tma(int i0, int a) {
        if constexpr (L == 192)
            return sw64_slot(i0 * (S::P * 16) + a * 16);
        else
            return sw128_slot(i0 * (S::P * 16) + a * 16);
    }
    // pass C: with TMA at 192 a three-stage ring of dense n x P tiles (two band
    // tiles in flight while one is reduced); otherwise as smem()
    template <class C>
    static constexpr int C_STAGES = (SLB_GROUP_C_TMA3 && L == 192 && TMA_STORE<C>) ? 3 : 2;
    template <class C>
    __host__ __device__ static constexpr size_t c_stage_elems() {
        return C_STAGES<C> == 3 ? static_cast<size_t>(L) * S::P : S::AC_ELEMS;
    }
    template <class C>
    static constexpr size_t smem_c() {
        return C_STAGES<C> * c_stage_elems<C>() * sizeof(C) + SC_BYTES + 32 + S::P * sizeof(C) + 1024;
    }
#ifndef SLB_GROUP_C_MINB
    static constexpr int C_MINB = 2;
#else
    static constexpr int C_MINB = SLB_GROUP_C_MINB;
#endif
};

// the group's shared axis-0 row (unscaled): A[k0], or the full filter line (kGrpFull)
struct GroupRow {
    const double* A;
    FiltSynth3D::Ax0Line full;
    bool is_full;
    __device__ __forceinline__ double at(int k0) const { return is_full ? full.at(k0) : __ldg(A + k0); }
};
__device__ __forceinline__ GroupRow group_row(const FiltSynth3D& f, const BandDesc3D& d, int type, int k1, int k2,
                                              int n) {
    GroupRow r{};
    r.is_full = type == kGrpFull;
    if (r.is_full)
        r.full = f.ax0_line(d, k1, k2);
    else if (type == kGrpLow)
        r.A = f.tab1d + f.lp_off[0];
    else
        r.A = f.tab2d + d.p1_off + static_cast<long long>(type == kGrpRowK1 ? k1 : k2) * n;
    return r;
}
// per-band, per-line scalar s_b(k1, k2)
__device__ __forceinline__ double group_scalar(const FiltSynth3D& f, const BandDesc3D& d, int type, int k1, int k2,
                                               int n) {
    switch (type) {
        case kGrpRowK1: return __ldg(f.tab1d + d.g_off + k1) * __ldg(f.tab2d + d.p2_off + (long long)k1 * n + k2);
        case kGrpRowK2: return __ldg(f.tab1d + d.g_off + k2) * __ldg(f.tab2d + d.p2_off + (long long)k2 * n + k1);
        case kGrpLow: return __ldg(f.tab1d + f.lp_off[1] + k1) * __ldg(f.tab1d + f.lp_off[2] + k2);
        default: return 1.0;
    }
}

// ---------------------------------------------------------------- pass A (groups)
// grid (group, k2 * Q + q): consecutive CTAs share the CTA's F lines in L2.
template <int L, class C = double2>
__global__ void __launch_bounds__(SplitShape<L>::AC_THREADS, GroupShape<L>::A_MINB)
    k3g_dec(const C* __restrict__ F, C* __restrict__ Z, long long zbs, FiltSynth3D filt,
            const __grid_constant__ SplitGroups grp, const C* __restrict__ tw, const __grid_constant__ CUtensorMap zmap) {
    using S = SplitShape<L>;
    using R = RealOf<C>;
    constexpr int T = S::T, E = RegPlan<L>::E, P = S::P, Q = S::Q, LD = S::LD, n = L;
    constexpr bool TMA = GroupShape<L>::template TMA_STORE<C>;
    SLB_DYN_SMEM(C, tile_raw);  // [2][n][LD] output tiles; the line buffers and the Y staging alias tile 0
    C* tile = reinterpret_cast<C*>((reinterpret_cast<uintptr_t>(tile_raw) + 1023) & ~uintptr_t(1023));
    R* sc = reinterpret_cast<R*>(tile + 2 * S::AC_ELEMS);  // [len][P]
    // the CTA's across-line DFT twiddles w_n^{a q} (q fixed per CTA): read as
    // shared-memory broadcasts instead of per-band table loads through L1
    C* twq = reinterpret_cast<C*>(reinterpret_cast<unsigned char*>(sc) + GroupShape<L>::SC_BYTES + 16);
    const int gi = blockIdx.x;
    const int k2 = blockIdx.y / Q, q = blockIdx.y - k2 * Q;
    if (threadIdx.x < P) twq[threadIdx.x] = twiddle<+1>(tw, threadIdx.x * q);  // published by the post-FFT barrier
    const int p = threadIdx.x / T, t = threadIdx.x - p * T;
    const int k1 = q + Q * p;
    const int b0 = grp.first[gi], nbg = grp.len[gi], type = grp.type[gi];
    // the group's shared line: IFFT_0(F * A)
    C x[E];
    {
        const BandDesc3D bd0 = filt.bands[b0];
        const GroupRow row = group_row(filt, bd0, type, k1, k2, n);
        const C* fl = F + ((long long)k2 * n + k1) * n;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const C f = __ldg(fl + t + T * m);
            const R a = R(row.at(t + T * m));
            x[m] = mkc<C>(f.x * a, f.y * a);
        }
    }
    for (int i = threadIdx.x; i < nbg * P; i += S::AC_THREADS) {  // groups of up to kMaxGroupLen bands
        const int bb = i / P, pp = i - bb * P;
        sc[i] = R(group_scalar(filt, filt.bands[b0 + bb], type, q + Q * pp, k2, n));
    }
    reg_fft<L, +1, S::PAD>(x, tile + p * S::LB, t, tw);
    __syncthreads();  // every line is done with the aliased buffers
#pragma unroll
    for (int m = 0; m < E; ++m) tile[(t + T * m) * LD + p] = x[m];
    __syncthreads();
    const int i0 = threadIdx.x;
    C y[P];
    if (i0 < n) {
#pragma unroll
        for (int pp = 0; pp < P; ++pp) y[pp] = tile[i0 * LD + pp];
    }
    const int sa = threadIdx.x % P, si0 = threadIdx.x / P;
    for (int bb = 0; bb < nbg; ++bb) {
        // band bb writes tile (bb + 1) & 1: tile 0 (the Y staging) is first
        // rewritten at bb = 1, after the bb = 0 barrier every Y read precedes
        C* buf = tile + ((bb + 1) & 1) * S::AC_ELEMS;
        if constexpr (TMA) {
            if (bb >= 2) {  // the bulk store issued from this tile at bb - 2 has read it
                if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                __syncthreads();
            }
        }
        if (i0 < n) {
            C v[P];
#pragma unroll
            for (int pp = 0; pp < P; ++pp) {
                const R s = type == kGrpFull ? R(1) : sc[bb * P + pp];
                v[pp] = mkc<C>(y[pp].x * s, y[pp].y * s);
            }
            dft_small<P, +1>(v);
#pragma unroll
            for (int a = 0; a < P; ++a) {
                const C w = a == 0 ? v[0] : cmul(v[a], twq[a]);
                if constexpr (TMA)
                    buf[GroupShape<L>::tslot_tma(i0, a)] = w;  // dense [i0][a], swizzled
                else
                    buf[i0 * LD + a] = w;
            }
        }
        if constexpr (TMA) {
            // Z[slot][k2][i0][a/4][q][a%4] as the 5D tensor (a%4 re/im, q, a/4, i0, slot * H + k2)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncthreads();
            if (threadIdx.x == 0) tma_store_5d(&zmap, buf, 0, q, 0, 0, (b0 + bb - grp.zb0) * S::H + k2);
            continue;
        }
        __syncthreads();
        // (32-byte STG.256 stores of a pairs measured 2 % slower here and in
        // pass B's copy-out: profiles/r2b_ab_stg256_pairs.log)
        C* z = Z + (long long)(b0 + bb - grp.zb0) * zbs + (long long)k2 * n * n +
               zrow<P, Q, SplitLayout<L, C>::ZQUAD>(q, sa) + (long long)si0 * n;
#pragma unroll 4
        for (int j = 0; j < n / T; ++j) __stcg(z + (long long)j * T * n, buf[(si0 + T * j) * LD + sa]);
    }
    if constexpr (TMA) {
        if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read before exit (stream order publishes the writes)
    }
}

// ---------------------------------------------------------------- pass C (groups)
// per (k2, q): for every group, sum_b s_b * (twiddle, length-P DFT of Z'_b) in
// registers (one thread per row i0), then one axis-0 FFT, * A, into acc.
template <int L, class C = double2>
__global__ void __launch_bounds__(SplitShape<L>::AC_THREADS, GroupShape<L>::C_MINB)
    k3g_rec(const C* __restrict__ Z, long long zbs, C* __restrict__ acc, FiltSynth3D filt,
            const __grid_constant__ SplitGroups grp, int accumulate, const C* __restrict__ tw,
            const __grid_constant__ CUtensorMap zmap, int bx0 = 0) {
    using S = SplitShape<L>;
    using R = RealOf<C>;
    constexpr int T = S::T, E = RegPlan<L>::E, P = S::P, Q = S::Q, LD = S::LD, n = L;
    // TMA: band tiles arrive by bulk tensor loads (dense [i0][a], swizzled) on
    // mbarriers -- NST = 3 stages at 192 (two tiles in flight), else 2;
    // without TMA cp.async into [n][LD] tiles
    constexpr bool TMA = GroupShape<L>::template TMA_STORE<C>;
    constexpr int NST = GroupShape<L>::template C_STAGES<C>;
    constexpr bool DENSE = NST == 3;  // group-end scratch in the dense swizzled layout (stages of exactly n P)
    constexpr size_t STG = GroupShape<L>::template c_stage_elems<C>();
    SLB_DYN_SMEM(C, tile_raw);  // [NST][stage] band tiles
    C* tile = reinterpret_cast<C*>((reinterpret_cast<uintptr_t>(tile_raw) + 1023) & ~uintptr_t(1023));
    R* sc = reinterpret_cast<R*>(tile + NST * STG);
    uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(sc) + GroupShape<L>::SC_BYTES);
    C* twq = reinterpret_cast<C*>(reinterpret_cast<unsigned char*>(sc) + GroupShape<L>::SC_BYTES + 32);
    const int bx = blockIdx.x + bx0;  // k2-slab launches (the multi-GPU reduce overlaps the last one)
    const int k2 = bx / Q, q = bx - k2 * Q;
    const int p = threadIdx.x / T, t = threadIdx.x - p * T;
    const int k1 = q + Q * p;
    const int i0 = threadIdx.x;
    const int sa = threadIdx.x % P, si0 = threadIdx.x / P;
    auto load = [&](int slot, int stage) {
        C* buf = tile + stage * STG;
        if constexpr (TMA) {
            if (threadIdx.x == 0)
                tma_load_5d(&zmap, buf, bars + stage, static_cast<unsigned>(n * P * sizeof(C)), 0, q, 0, 0,
                            slot * S::H + k2);
        } else {
            const C* z = Z + (long long)slot * zbs + (long long)k2 * n * n + zrow<P, Q, SplitLayout<L, C>::ZQUAD>(q, sa) +
                         (long long)si0 * n;
#pragma unroll 4
            for (int j = 0; j < n / T; ++j) cp_async_c(buf + (si0 + T * j) * LD + sa, z + (long long)j * T * n);
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    };
    // Z slot of the band `ahead` bands after (gi, bb) in the launch's flat order, or -1
    auto slot_ahead = [&](int gi, int bb, int ahead) {
        bb += ahead;
        while (gi < grp.count && bb >= grp.len[gi]) {
            bb -= grp.len[gi];
            ++gi;
        }
        return gi < grp.count ? grp.first[gi] + bb - grp.zb0 : -1;
    };
    if constexpr (TMA) {
        if (threadIdx.x == 0) {
#pragma unroll
            for (int st = 0; st < NST; ++st) mbar_init(bars + st, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();
    }
    if (threadIdx.x < P) twq[threadIdx.x] = twiddle<-1>(tw, threadIdx.x * q);  // published by the first band's barrier
    C ar[E];
#pragma unroll
    for (int m = 0; m < E; ++m) ar[m] = mkc<C>(0.0, 0.0);
    // prologue: the first NST - 1 bands in flight
#pragma unroll
    for (int st = 0; st + 1 < NST; ++st) {
        const int sl = slot_ahead(0, 0, st);
        if (sl >= 0) load(sl, st);
    }
    int it = 0;  // flat band counter (stage it % NST)
    for (int gi = 0; gi < grp.count; ++gi) {
        const int b0 = grp.first[gi], nbg = grp.len[gi], type = grp.type[gi];
        // the previous group's scalars were last read before its closing barriers
        for (int i = threadIdx.x; i < nbg * P; i += S::AC_THREADS) {
            const int bb = i / P, pp = i - bb * P;
            sc[i] = R(group_scalar(filt, filt.bands[b0 + bb], type, q + Q * pp, k2, n));
        }
        C ag[P];
#pragma unroll
        for (int pp = 0; pp < P; ++pp) ag[pp] = mkc<C>(0.0, 0.0);
        C* cur = tile;
        for (int bb = 0; bb < nbg; ++bb, ++it) {
            const int stage = it % NST;
            cur = tile + stage * STG;
            if constexpr (TMA) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic use -> TMA refill
            // stage (it + NST - 1) % NST is free (read by band it - 1 / the group
            // end); with TMA this barrier also publishes the group's scalars at it = 0
            if (it > 0 || TMA) __syncthreads();
            const int nslot = slot_ahead(gi, bb, NST - 1);
            if constexpr (TMA) {
                if (nslot >= 0) load(nslot, (it + NST - 1) % NST);
                mbar_wait_parity(bars + stage, static_cast<unsigned>(it / NST) & 1u);  // band it landed
            } else {
                if (nslot >= 0) {
                    load(nslot, (it + 1) & 1);
                    asm volatile("cp.async.wait_group 1;" ::: "memory");  // band it landed, the next in flight
                } else {
                    asm volatile("cp.async.wait_group 0;" ::: "memory");
                }
                __syncthreads();
            }
            if (i0 < n) {
                C v[P];
#pragma unroll
                for (int a = 0; a < P; ++a) {
                    const C u = TMA ? cur[GroupShape<L>::tslot_tma(i0, a)] : cur[i0 * LD + a];
                    v[a] = a == 0 ? u : cmul(u, twq[a]);
                }
                dft_small<P, -1>(v);
#pragma unroll
                for (int pp = 0; pp < P; ++pp) {
                    const R s = type == kGrpFull ? R(1) : sc[bb * P + pp];
                    ag[pp].x = fma(v[pp].x, s, ag[pp].x);
                    ag[pp].y = fma(v[pp].y, s, ag[pp].y);
                }
            }
        }
        // group end: the rows' sums back into lines through the last band's tile
        __syncthreads();  // every row read its last tile
        if (i0 < n) {
#pragma unroll
            for (int pp = 0; pp < P; ++pp) {
                if constexpr (DENSE)
                    cur[GroupShape<L>::tslot_tma(i0, pp)] = ag[pp];
                else
                    cur[i0 * LD + pp] = ag[pp];
            }
        }
        __syncthreads();
        C x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = DENSE ? cur[GroupShape<L>::tslot_tma(t + T * m, p)] : cur[(t + T * m) * LD + p];
        __syncthreads();  // all lines gathered: the tile becomes the line buffers
        const BandDesc3D bd0 = filt.bands[b0];
        const GroupRow row = group_row(filt, bd0, type, k1, k2, n);
        if constexpr (DENSE)
            reg_fft_xor<L, -1>(x, cur + p * L, t, tw);  // P lines of exactly n slots fill the stage
        else
            reg_fft<L, -1, S::PAD>(x, cur + p * S::LB, t, tw);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const R a = R(row.at(t + T * m));
            ar[m].x = fma(x[m].x, a, ar[m].x);
            ar[m].y = fma(x[m].y, a, ar[m].y);
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

// out[k2][a][b] = in[k2][b][a] (add: +=) for the planes k2 in [k2lo, k2hi):
// F -> F^T for the transposed frame, and the transposed accumulator back.
template <class C>
__global__ void k3_plane_transpose(const C* __restrict__ in, C* __restrict__ out, int n, int k2lo, int add) {
    __shared__ C tl[32][33];
    const int k2 = blockIdx.z + k2lo;
    const long long pb = (long long)k2 * n * n;
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = by + j, c = bx + threadIdx.x;
        if (r < n && c < n) tl[j][threadIdx.x] = __ldcs(in + pb + (long long)r * n + c);
    }
    __syncthreads();
    for (int j = threadIdx.y; j < 32; j += blockDim.y) {
        const int r = bx + j, c = by + threadIdx.x;  // out row = in column
        if (r < n && c < n) {
            C v = tl[threadIdx.x][j];
            C* o = out + pb + (long long)r * n + c;
            if (add) {
                const C w = *o;
                v = mkc<C>(w.x + v.x, w.y + v.y);
            }
            *o = v;
        }
    }
}

}  // namespace slb
