// 3D rows + axis-1 passes fused per i0-plane on a 2-CTA cluster.
//
// In the rotated layout R[k2][i0][k1] the i0-plane P[k2][k1] (k2 < H, k1 < n)
// is H contiguous rows of n complex values — 298 KB at n = 192, too large for
// one SM but not for a pair. CTA r of the cluster keeps k2-rows
// [r*H0, min(H, (r+1)*H0)) in shared memory (row pitch n+1 so column walks are
// bank-conflict free) and the pair runs, on the plane held on chip:
//   A  own rows : IFFT along k1 (axis 1)                    (global -> smem)
//   B  own i1 half of the columns, reading / writing the peer's rows through
//      distributed shared memory: pair-packed c2r along k2 (axis 2), x 1/N,
//      hard threshold, band write, r2c back                  (smem <-> DSMEM)
//   C  own rows : FFT along k1                               (smem -> global)
// replacing axis1<+1>, rows_fused and axis1<-1> (three HBM round trips of the
// plane) with one read and one write of the plane plus the band write.
// Semantics identical to those three passes (fast3d_host.cuh).
#pragma once
#include <cooperative_groups.h>

#include "fast2d.cuh"

namespace slb {

template <int L>
struct PlaneCfg {
    static constexpr int T = RegPlan<L>::T;
    static constexpr int E = RegPlan<L>::E;
    static constexpr int H = L / 2 + 1;
    static constexpr int H0 = (H + 1) / 2;      // k2-rows held by CTA 0 (CTA 1: H - H0)
    static constexpr int PITCH = L + 1;         // tile row pitch (double2)
    static constexpr int THREADS = 256;
    static constexpr int LINES = THREADS / T;   // concurrent FFT lines per CTA
    static constexpr size_t SMEM = (static_cast<size_t>(H0) * PITCH + static_cast<size_t>(LINES) * L) * sizeof(double2);
};

template <int L>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PlaneCfg<L>::THREADS, 1)
    k3_plane_fused(double2* __restrict__ rot, long long rbs, double* __restrict__ band, long long bbs, double scale,
                   const double* __restrict__ delta, int band0, const double2* __restrict__ tw) {
    namespace cg = cooperative_groups;
    using C = PlaneCfg<L>;
    constexpr int T = C::T, E = C::E, H = C::H, H0 = C::H0, PITCH = C::PITCH, n = L;
    constexpr int KPT = (H + T - 1) / T;
    extern __shared__ double2 smem[];
    double2* tile = smem;                          // [H0][PITCH]
    double2* lbase = smem + H0 * PITCH;            // LINES line buffers of L
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    double2* peer = cluster.map_shared_rank(tile, rank ^ 1);
    double2* tile0 = rank == 0 ? tile : peer;      // rows [0, H0)
    double2* tile1 = rank == 0 ? peer : tile;      // rows [H0, H)
    const int i0 = blockIdx.x >> 1;
    const int b = blockIdx.y;
    rot += b * rbs;
    if (band) band += b * bbs;
    const int k2lo = rank * H0;
    const int nrows = rank == 0 ? H0 : H - H0;
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    double2* lb = lbase + li * L;

    // ---- A: stage own rows (cp.async, all in flight), IFFT along k1 in place
    for (int idx = threadIdx.x; idx < nrows * n; idx += C::THREADS) {
        const int r = idx / n, c = idx - r * n;
        cp_async16(tile + r * PITCH + c, rot + ((long long)(k2lo + r) * n + i0) * n + c);
    }
    cp_async_wait_all();
    __syncthreads();
    // trip counts are uniform across the CTA (lines share warps and barriers);
    // lines past the last row compute on zeros and store nothing
    for (int r0 = 0; r0 < nrows; r0 += C::LINES) {
        const int r = r0 + li;
        const bool act = r < nrows;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = act ? tile[r * PITCH + t + T * m] : make_double2(0.0, 0.0);
        reg_fft<L, +1, false>(x, lb, t, tw);
        if (act) {
#pragma unroll
            for (int m = 0; m < E; ++m) tile[r * PITCH + t + T * m] = x[m];
        }
        line_sync<T>();
    }
    cluster.sync();  // both halves of the plane are in (i1, k2) order

    // ---- B: columns i1 of this CTA's half, pairs (i1, i1 + 1) per line
    auto at = [&](int k, int i1) -> double2* {
        return k < H0 ? tile0 + k * PITCH + i1 : tile1 + (k - H0) * PITCH + i1;
    };
    const double dl = delta[band0 + b];
    constexpr int HALF = n / 2;                    // columns per CTA
    static_assert((HALF / 2) % C::LINES == 0, "column pairs must split evenly over the lines");
    for (int p = li; p < HALF / 2; p += C::LINES) {
        const int ia = rank * HALF + 2 * p;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k = t + T * m;
            double2 X, Y;
            if (k < H) {
                X = *at(k, ia);
                Y = *at(k, ia + 1);
                if (k == 0 || 2 * k == L) {
                    X.y = 0.0;
                    Y.y = 0.0;
                }
                x[m] = make_double2(X.x - Y.y, X.y + Y.x);
            } else {
                X = *at(L - k, ia);
                Y = *at(L - k, ia + 1);
                x[m] = make_double2(X.x + Y.y, Y.x - X.y);
            }
        }
        reg_fft<L, +1, false>(x, lb, t, tw);
        double* ba = band + ((long long)i0 * n + ia) * n;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            double a = x[m].x * scale, c = x[m].y * scale;
            if (dl >= 0.0) {
                if (fabs(a) < dl) a = 0.0;
                if (fabs(c) < dl) c = 0.0;
            }
            const int i = t + T * m;
            if (band) {
                ba[i] = a;
                ba[n + i] = c;
            }
            x[m] = make_double2(a, c);  // rec input: the thresholded rows
        }
        line_sync<T>();
        reg_fft<L, -1, false>(x, lb, t, tw);
#pragma unroll
        for (int m = 0; m < E; ++m) lb[swz<false>(t + T * m)] = x[m];
        line_sync<T>();
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int k = t + T * u;
            if (k < H) {
                const double2 zk = lb[swz<false>(k)];
                const double2 zm = lb[swz<false>(k == 0 ? 0 : L - k)];
                *at(k, ia) = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
                *at(k, ia + 1) = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
            }
        }
        line_sync<T>();
    }
    cluster.sync();  // the peer's column writes into this tile are visible

    // ---- C: own rows, FFT along k1, back to the rotated layout
    for (int r0 = 0; r0 < nrows; r0 += C::LINES) {
        const int r = r0 + li;
        const bool act = r < nrows;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = act ? tile[r * PITCH + t + T * m] : make_double2(0.0, 0.0);
        reg_fft<L, -1, false>(x, lb, t, tw);
        if (act) {
            double2* o = rot + ((long long)(k2lo + r) * n + i0) * n;
#pragma unroll
            for (int m = 0; m < E; ++m) __stcg(o + t + T * m, x[m]);
        }
        line_sync<T>();
    }
}

}  // namespace slb
