// Fused 2D denoise pipeline: dec rows pass + hard threshold + rec rows pass in
// one kernel, so a thresholded band is written once (the materialised stack)
// and never read back: 3 passes per band instead of 4.
//
//   cols_dec  : inter[b] = IFFT_0(F psi_b)                       (fast2d.cuh)
//   rows_fused: band_b = thr(IFFT_1(inter[b]) / N) -> stack;
//               inter[b] = FFT_1(band_b)  (in place, same tile)
//   cols_rec  : slot += FFT_0(inter[b]) psi_b                     (fast2d.cuh)
// Semantics = inverse(hard_threshold(forward(f))) (apps.cpp:114-121).
#pragma once

#include "fast2d_host.cuh"
#include "tma.cuh"

namespace slb {

// TMA tile load / store in the fused rows pass (fp64, 512): the tile [H][2V =
// 8] has 128-byte rows, and tslot<4>'s XOR of the 16-byte slot with k & 7 is
// exactly the TMA 128-byte swizzle, so the bulk tensor copies (two boxes of
// HB <= 256 rows) land in the layout the per-line code already reads.
#ifndef SLB_ROWS_TMA
#define SLB_ROWS_TMA 1
#endif
template <int L, class C>
struct RowsTma {
    static constexpr bool ON = SLB_ROWS_TMA && L == 512 && sizeof(C) == 16 && 2 * RowCfg<L>::V == 8;
    static constexpr int H = L / 2 + 1, HB = (H + 1) / 2;
    static constexpr size_t TILE_BYTES = static_cast<size_t>(2 * HB) * 8 * sizeof(C);  // 2 boxes of HB 128-byte rows
    static size_t smem(size_t plain) { return std::max(plain, TILE_BYTES) + 1024 + 16; }  // + alignment + mbarrier
};

// STORE = false: the stack is not materialised (sl_set_stack_output, band
// null); a separate instantiation so the stack-writing variant keeps its
// register allocation (a runtime null test spilled 136 B/thread at L = 128)
template <int L, bool STORE = true, class C = double2>
__global__ void __launch_bounds__(RowCfg<L>::FUSED_THREADS, RowCfg<L>::FUSED_MIN_BLOCKS)
    k2_rows_fused(C* __restrict__ inter, long long ibs, RealOf<C>* __restrict__ band, long long bbs, int n0, int H,
                  RealOf<C> scale, const double* __restrict__ delta, int band0, const C* __restrict__ tw,
                  const __grid_constant__ CUtensorMap tmap, int cstride, long long izs = 0, long long bzs = 0) {
    constexpr int T = FusedRowPlan<L>::T, E = FusedRowPlan<L>::E, V = RowCfg<L>::V;
    using R = RealOf<C>;
    constexpr int KPT = (L / 2 + 1 + T - 1) / T;
    constexpr bool TMA = RowsTma<L, C>::ON;
    SLB_DYN_SMEM(C, tile_raw);  // [H][2V] swizzled tile, then V line buffers
    C* tile = TMA ? reinterpret_cast<C*>((reinterpret_cast<uintptr_t>(tile_raw) + 1023) & ~uintptr_t(1023)) : tile_raw;
    [[maybe_unused]] uint64_t* bar = reinterpret_cast<uint64_t*>(reinterpret_cast<unsigned char*>(tile) + RowsTma<L, C>::TILE_BYTES);
    [[maybe_unused]] const int slot = blockIdx.y + blockIdx.z * cstride;  // band slot of the intermediate (TMA z)
    const int r0 = blockIdx.x * 2 * V;
    inter += blockIdx.y * ibs + blockIdx.z * izs;  // blockIdx.z: frame of a lock-step batch
    // STORE = false keeps a (never taken) runtime test on the stores: ptxas
    // allocates that body without spills, while deleting the stores outright
    // spills 24-296 B/thread; L = 2048 also spills less with the test
    // (measured -Xptxas -v for every L)
    constexpr bool kTest = !STORE || L == 2048;
    if (!kTest || band) band += blockIdx.y * bbs + blockIdx.z * bzs;
    const int nrows = min(2 * V, n0 - r0);
    // thread -> fixed slot rr, k-rows strided by a compile-time step
    constexpr int KS = RowCfg<L>::FUSED_THREADS / (2 * V);
    const int rr = threadIdx.x % (2 * V);
    if constexpr (TMA) {
        constexpr int HB = RowsTma<L, C>::HB;
        if (threadIdx.x == 0) {
            mbar_init(bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncthreads();  // the barrier is initialised before anyone waits on it
        if (threadIdx.x == 0) {
            mbar_expect_tx(bar, static_cast<unsigned>(RowsTma<L, C>::TILE_BYTES));
            tma_load_3d(&tmap, tile, bar, 2 * r0, 0, slot);  // rows past n0 / k past H zero-fill
            tma_load_3d(&tmap, tile + HB * 2 * V, bar, 2 * r0, HB, slot);
        }
        mbar_wait_parity(bar, 0);
    } else {
#pragma unroll 4
        for (int k = threadIdx.x / (2 * V); k < H; k += KS) {
            if (rr < nrows)
                cp_async_c(tile + tslot<V>(k, rr), inter + (long long)k * n0 + r0 + rr);
            else
                tile[tslot<V>(k, rr)] = mkc<C>(0.0, 0.0);
        }
        cp_async_wait_all();
        __syncthreads();
    }
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
            x[m] = mkc<C>(X.x - Y.y, X.y + Y.x);
        } else {
            X = tile[tslot<V>(L - k, 2 * q)];
            Y = tile[tslot<V>(L - k, 2 * q + 1)];
            x[m] = mkc<C>(X.x + Y.y, Y.x - X.y);
        }
    }
    __syncthreads();              // every line has gathered: the tile is dead
    constexpr bool PAD = RowCfg<L>::PAD;
    C* lb = tile + q * LineBuf<L, PAD>::N;   // line buffers alias it (smem sized for both)
    reg_fft_p<FusedRowPlan<L>, L, +1, PAD>(x, lb, t, tw);
    const double dl = delta[band0 + blockIdx.y];
    const int ra = r0 + 2 * q;
#pragma unroll
    for (int m = 0; m < E; ++m) {
        R a = x[m].x * scale, c = x[m].y * scale;
        if (dl >= 0.0) {
            if (fabs(a) < dl) a = 0.0;
            if (fabs(c) < dl) c = 0.0;
        }
        const int i = t + T * m;
        if (!kTest || band) {
            if (ra < n0) band[(long long)ra * L + i] = a;
            if (ra + 1 < n0) band[(long long)(ra + 1) * L + i] = c;
        }
        x[m] = mkc<C>(ra < n0 ? a : 0.0, ra + 1 < n0 ? c : R(0));  // rec input: the thresholded rows
    }
    reg_fft_p<FusedRowPlan<L>, L, -1, PAD>(x, lb, t, tw);
    C zk[KPT], zm[KPT];
    if constexpr (T <= 32 && SLB_ROWS_SHFL) {
        mirror_pairs_shfl<L, T, E, KPT>(x, zk, zm, t);  // warp shuffles, no shared-memory round trip
    } else {
#pragma unroll
        for (int m = 0; m < E; ++m) lb[swz<PAD, L, sizeof(C)>(t + T * m)] = x[m];
        line_sync<T>();
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int k = t + T * u;
            if (k < H) {
                zk[u] = lb[swz<PAD, L, sizeof(C)>(k)];
                zm[u] = lb[swz<PAD, L, sizeof(C)>(k == 0 ? 0 : L - k)];
            }
        }
    }
    __syncthreads();  // all line buffers read before the tile is rewritten
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        const int k = t + T * u;
        if (k < H) {
            tile[tslot<V>(k, 2 * q)] = mkc<C>(R(0.5) * (zk[u].x + zm[u].x), R(0.5) * (zk[u].y - zm[u].y));
            tile[tslot<V>(k, 2 * q + 1)] = mkc<C>(R(0.5) * (zk[u].y + zm[u].y), R(0.5) * (zm[u].x - zk[u].x));
        }
    }
    if constexpr (TMA) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0) {
            constexpr int HB = RowsTma<L, C>::HB;
            tma_store_3d(&tmap, tile, 2 * r0, 0, slot);  // out-of-range rows / k are clipped
            tma_store_3d(&tmap, tile + HB * 2 * V, 2 * r0, HB, slot);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // smem read before exit
        }
        return;
    }
    __syncthreads();
#pragma unroll 4
    for (int k = threadIdx.x / (2 * V); k < H; k += KS)
        if (rr < nrows) __stcg(inter + (long long)k * n0 + r0 + rr, tile[tslot<V>(k, rr)]);
}

// rows pass of the fused denoise (band = null: the stack is not materialised)
// the intermediate [slots][H][n0] complex as a 3D fp64 tensor for the TMA tile
// copies (cached per buffer / shape: launches reuse a handful of workspaces)
template <int L, class C>
static CUtensorMap rows_tmap(C* inter, int n0, int H, long long slots) {
    CUtensorMap m{};
    if constexpr (RowsTma<L, C>::ON) {
        static std::mutex mu;
        static std::map<std::tuple<const void*, int, int, long long>, CUtensorMap> cache;
        std::lock_guard<std::mutex> lk(mu);
        const auto key = std::make_tuple(static_cast<const void*>(inter), n0, H, slots);
        auto it = cache.find(key);
        if (it != cache.end()) return it->second;
        const cuuint64_t dims[3] = {2 * static_cast<cuuint64_t>(n0), static_cast<cuuint64_t>(H),
                                    static_cast<cuuint64_t>(slots)};
        const cuuint64_t strides[2] = {static_cast<cuuint64_t>(n0) * sizeof(C),
                                       static_cast<cuuint64_t>(n0) * H * sizeof(C)};
        const cuuint32_t box[3] = {2 * 2 * RowCfg<L>::V, static_cast<cuuint32_t>(RowsTma<L, C>::HB), 1};
        m = tma_map_f64(inter, 3, dims, strides, box, CU_TENSOR_MAP_SWIZZLE_128B);
        cache[key] = m;
    }
    return m;
}

// spectra of nhT complex values a workspace buffer holds
template <class C>
static long long ws_slots(const DBuf<double2>& b, long long nhT) {
    return static_cast<long long>(b.n * sizeof(double2) / sizeof(C)) / nhT;
}

// inter: `slots` band spectra [H][n0] back to back (bands at ibs, frames at izs = cstride * ibs)
template <int L, class C = double2>
static void launch_rows_fused(dim3 grid, size_t tile_smem, cudaStream_t st, C* inter, long long ibs,
                              RealOf<C>* band, long long bbs, int n0, int H, double scale, const double* delta,
                              int band0, const C* tw, long long izs, long long bzs, long long slots) {
    using RC = RowCfg<L>;
    auto* k = band ? k2_rows_fused<L, true, C> : k2_rows_fused<L, false, C>;
    const int cstride = izs > 0 ? static_cast<int>(izs / ibs) : 0;
    const size_t smem = RowsTma<L, C>::ON ? RowsTma<L, C>::smem(tile_smem) : tile_smem;
    const CUtensorMap tm = rows_tmap<L, C>(inter, n0, H, slots);
    set_smem(k, smem);
    k<<<grid, RC::FUSED_THREADS, smem, st>>>(inter, ibs, band, bbs, n0, H, scale, delta, band0, tw, tm, cstride, izs,
                                              bzs);
    check_launch("k2_rows_fused");
}

// denoise with the stack materialised in `stack` ([nb][n0][n1]).
template <int L0, int L1, class CX = double2>
static void denoise2d_fast_t(System& s, const RealOf<CX>* f, RealOf<CX>* stack, RealOf<CX>* out, const double* delta,
                             cudaStream_t st) {
    const int n0 = s.n[0], H = s.H;
    const long long nhT = static_cast<long long>(H) * n0;
    const Fast2DCfg cfg = fast2d_cfg(s);
    const int nb = s.nb();
    const int C = std::min(cfg.C, nb);
    s.w->inter.alloc(static_cast<size_t>(C) * nhT);
    s.w->F.alloc(static_cast<size_t>(nhT));
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
    set_smem(k2_cols_sum<L0, -1, CX>, col_smem);
    set_smem(k2_cols_sum<L0, +1, CX>, col_smem);
    set_smem(k2_cols_dec<L0, CX>, col2_smem);
    set_smem(k2_cols_rec<L0, CX>, colrec_smem_bytes<L0, CX>());
    const int row_blocks = (n0 + 2 * RC::V - 1) / (2 * RC::V);
    const int col_blocks = (H + CC::LINES - 1) / CC::LINES;
    if (s.w->done.n < static_cast<size_t>(col_blocks)) {  // zeroed once; the kernel resets its counters
        s.w->done.alloc(static_cast<size_t>(col_blocks));
        SL_CUDA(cudaMemsetAsync(s.w->done.p, 0, static_cast<size_t>(col_blocks) * sizeof(int), st));
    }
    {
        LaunchScope ls(s, "f2_rows_r2c", st, 1);
        k2_rows_r2c<L1, CX><<<dim3(row_blocks, 1), RC::THREADS, row_smem, st>>>(f, 0, ws_as<CX>(s.w->inter), 0, n0, H, tw1);
        check_launch("k2_rows_r2c");
    }
    {
        LaunchScope ls(s, "f2_cols_fwd", st, 1);
        k2_cols_sum<L0, -1, CX><<<col_blocks, CC::THREADS, col_smem, st>>>(ws_as<CX>(s.w->inter), 0, 1, nullptr, ws_as<CX>(s.w->F), H, tw0);
        check_launch("k2_cols_sum");
    }
    const RealOf<CX> scale = RealOf<CX>(1.0 / static_cast<double>(s.nreal));
    int slot0 = 0;
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
            LaunchScope ls(s, "f2_rows_fused", st, cb);
            launch_rows_fused<L1, CX>(dim3(row_blocks, cb), row_smem, st, ws_as<CX>(s.w->inter), nhT,
                                  (stack ? stack + static_cast<size_t>(b0) * s.nreal : nullptr), s.nreal, n0, H, scale,
                                  delta, s.lo + b0, tw1, 0, 0, ws_slots<CX>(s.w->inter, nhT));
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
        k2_rows_c2r<L1, CX><<<dim3(row_blocks, 1), RC::THREADS, row_smem, st>>>(ws_as<CX>(s.w->inter), 0, out, 0, n0, H, scale,
                                                                            nullptr, 0, tw1);
        check_launch("k2_rows_c2r");
    }
}

// Lock-step batch: nf frames advance through the same passes together, one
// launch per pass covering every frame (blockIdx.z), so each band's psi is read
// once from HBM for all frames (L2 hits for the rest) and launches/tails are
// amortised over the batch. Per-frame stacks at stack + f * sfs.
template <int L0, int L1, class CX = double2>
static void denoise2d_fast_batch_t(System& s, const RealOf<CX>* f, long long ffs, int nf, RealOf<CX>* stack,
                                   long long sfs, RealOf<CX>* out, long long ofs, const double* delta, cudaStream_t st) {
    const int n0 = s.n[0], H = s.H;
    const long long nhT = static_cast<long long>(H) * n0;
    const Fast2DCfg cfg = fast2d_cfg(s);
    const int nb = s.nb();
    const int C = std::min(cfg.C, nb);
    const long long izs = static_cast<long long>(C) * nhT;
    s.w->inter.alloc(static_cast<size_t>(nf) * izs);
    s.w->F.alloc(static_cast<size_t>(nf) * nhT);
    int nslots = 0;
    for (int b0 = 0; b0 < nb; b0 += C) nslots += (std::min(C, nb - b0) + cfg.G - 1) / cfg.G;
    const long long szs = static_cast<long long>(nslots) * nhT;
    s.w->slots.alloc(static_cast<size_t>(nf) * szs);
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
    set_smem(k2_cols_rec<L0, CX>, colrec_smem_bytes<L0, CX>());
    const int row_blocks = (n0 + 2 * RC::V - 1) / (2 * RC::V);
    const int col_blocks = (H + CC::LINES - 1) / CC::LINES;
    const size_t ndone = static_cast<size_t>(col_blocks) * nf;
    if (s.w->done.n < ndone) {  // zeroed once; the kernel resets its counters
        s.w->done.alloc(ndone);
        SL_CUDA(cudaMemsetAsync(s.w->done.p, 0, ndone * sizeof(int), st));
    }
    {  // F^T of every frame
        LaunchScope ls(s, "f2_rows_r2c", st, nf);
        k2_rows_r2c<L1, CX><<<dim3(row_blocks, nf), RC::THREADS, row_smem, st>>>(f, ffs, ws_as<CX>(s.w->inter), izs, n0, H, tw1);
        check_launch("k2_rows_r2c");
    }
    {
        LaunchScope ls(s, "f2_cols_fwd", st, nf);
        k2_cols_sum<L0, -1, CX><<<dim3(col_blocks, 1, nf), CC::THREADS, col_smem, st>>>(ws_as<CX>(s.w->inter), 0, 1, nullptr,
                                                                                  ws_as<CX>(s.w->F), H, tw0, izs, nhT);
        check_launch("k2_cols_sum");
    }
    const RealOf<CX> scale = RealOf<CX>(1.0 / static_cast<double>(s.nreal));
    int slot0 = 0;
    for (int b0 = 0; b0 < nb; b0 += C) {
        const int cb = std::min(C, nb - b0);
        const int groups = (cb + cfg.G - 1) / cfg.G;
        {
            LaunchScope ls(s, "f2_cols_dec", st, static_cast<long long>(cb) * nf);
            k2_cols_dec<L0, CX><<<dim3(col_blocks, groups, nf), CC::THREADS, col2_smem, st>>>(
                ws_as<CX>(s.w->F), Prec2D<CX>::psiT(s), nhT, ws_as<CX>(s.w->inter), nhT, H, s.lo + b0, cfg.G, cb, tw0, nhT, izs);
            check_launch("k2_cols_dec");
        }
        {
            LaunchScope ls(s, "f2_rows_fused", st, static_cast<long long>(cb) * nf);
            launch_rows_fused<L1, CX>(dim3(row_blocks, cb, nf), row_smem, st, ws_as<CX>(s.w->inter), nhT,
                                  (stack ? stack + static_cast<size_t>(b0) * s.nreal : nullptr), s.nreal, n0, H, scale,
                                  delta, s.lo + b0, tw1, izs, sfs, ws_slots<CX>(s.w->inter, nhT));
        }
        {
            LaunchScope ls(s, "f2_cols_rec", st, static_cast<long long>(cb) * nf);
            const bool fin = b0 + cb >= nb;
            k2_cols_rec<L0, CX><<<dim3(col_blocks, groups, nf), CC::THREADS, colrec_smem_bytes<L0, CX>(), st>>>(
                ws_as<CX>(s.w->inter), nhT, Prec2D<CX>::psiT(s), nhT, ws_as<CX>(s.w->slots), nhT, H, s.lo + b0, cfg.G, cb, slot0, tw0,
                fin ? s.w->done.p : nullptr, nslots, Prec2D<CX>::WT(s), ws_as<CX>(s.w->inter), izs, szs, izs);
            check_launch("k2_cols_rec");
        }
        slot0 += groups;
    }
    {
        LaunchScope ls(s, "f2_rows_c2r", st, nf);
        k2_rows_c2r<L1, CX><<<dim3(row_blocks, nf), RC::THREADS, row_smem, st>>>(ws_as<CX>(s.w->inter), izs, out, ofs, n0, H,
                                                                             scale, nullptr, 0, tw1);
        check_launch("k2_rows_c2r");
    }
}

static void denoise2d_fast_batch(System& s, const double* f, long long ffs, int nf, double* stack, long long sfs,
                                 double* out, long long ofs, const double* delta, cudaStream_t st) {
    SLB_FAST2D_DISPATCH(denoise2d_fast_batch_t, s, f, ffs, nf, stack, sfs, out, ofs, delta, st)
}

static void denoise2d_fast(System& s, const double* f, double* stack, double* out, const double* delta,
                           cudaStream_t st) {
    SLB_FAST2D_DISPATCH(denoise2d_fast_t, s, f, stack, out, delta, st)
}

// fp32 mode (sl_system_set_precision(32)): the same passes on float2 spectra
static void denoise2d_fast_f32(System& s, const float* f, float* stack, float* out, const double* delta,
                               cudaStream_t st) {
    SLB_FAST2D_DISPATCH_F32(denoise2d_fast_t, s, f, stack, out, delta, st)
}
static void denoise2d_fast_batch_f32(System& s, const float* f, long long ffs, int nf, float* stack, long long sfs,
                                     float* out, long long ofs, const double* delta, cudaStream_t st) {
    SLB_FAST2D_DISPATCH_F32(denoise2d_fast_batch_t, s, f, ffs, nf, stack, sfs, out, ofs, delta, st)
}

}  // namespace slb
