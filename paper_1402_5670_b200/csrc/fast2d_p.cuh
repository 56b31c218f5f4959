// Persistent, software-pipelined variants of the 2D pass kernels (fast2d.cuh).
//
// rows passes : each CTA walks work items (band, row block) with stride
//               gridDim.x; the next item's column-major tile is prefetched by
//               cp.async into the other half of a double buffer while the
//               current one is transformed (c2r) / the next item's rows are
//               prefetched into registers (r2c).
// column passes: grid = column blocks x K; a CTA keeps one column block and
//               takes bands j, j+K, j+2K, ... so F (dec) and the accumulator
//               (rec) stay in registers; the next band's filter/spectrum is
//               loaded into registers before the current FFT runs.
#pragma once

#include "fast2d.cuh"

namespace slb {

template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }

// ---------------------------------------------------------------- rows c2r (persistent)
template <int L>
__global__ void __launch_bounds__(RowCfg<L>::THREADS)
    k2p_rows_c2r(const double2* __restrict__ src, long long sbs, double* __restrict__ dst, long long dbs, int n0,
                 int H, double scale, const double* __restrict__ delta, int band0, int nbands,
                 const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E, V = RowCfg<L>::V;
    extern __shared__ double2 sm[];  // tile0 [H][2V] | tile1 [H][2V] | V line buffers
    const int tile_elems = H * 2 * V;
    double2* bufs[2] = {sm, sm + tile_elems};
    double2* lb_base = sm + 2 * tile_elems;
    const int row_blocks = (n0 + 2 * V - 1) / (2 * V);
    const int total = nbands * row_blocks;
    auto issue = [&](int w, double2* buf) {
        const int b = w / row_blocks, rb = w - b * row_blocks;
        const int r0 = rb * 2 * V;
        const int nrows = min(2 * V, n0 - r0);
        const double2* s = src + b * sbs;
        for (int idx = threadIdx.x; idx < tile_elems; idx += blockDim.x) {
            const int k = idx / (2 * V), rr = idx - k * 2 * V;
            if (rr < nrows)
                cp_async16(buf + tslot<V>(k, rr), s + (long long)k * n0 + r0 + rr);
            else
                buf[tslot<V>(k, rr)] = make_double2(0.0, 0.0);
        }
    };
    const int q = threadIdx.x / T, t = threadIdx.x - q * T;
    double2* lb = lb_base + q * L;
    int w = blockIdx.x;
    if (w < total) issue(w, bufs[0]);
    cp_async_commit();
    for (int it = 0; w < total; w += gridDim.x, ++it) {
        double2* cur = bufs[it & 1];
        if (w + (int)gridDim.x < total) issue(w + gridDim.x, bufs[(it + 1) & 1]);
        cp_async_commit();
        cp_async_wait_group<1>();
        __syncthreads();
        const int b = w / row_blocks, rb = w - b * row_blocks;
        const int r0 = rb * 2 * V;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k = t + T * m;
            double2 X, Y;
            if (k < H) {
                X = cur[tslot<V>(k, 2 * q)];
                Y = cur[tslot<V>(k, 2 * q + 1)];
                if (k == 0 || 2 * k == L) {
                    X.y = 0.0;
                    Y.y = 0.0;
                }
                x[m] = make_double2(X.x - Y.y, X.y + Y.x);
            } else {
                X = cur[tslot<V>(L - k, 2 * q)];
                Y = cur[tslot<V>(L - k, 2 * q + 1)];
                x[m] = make_double2(X.x + Y.y, Y.x - X.y);
            }
        }
        reg_fft<L, +1>(x, lb, t, tw);
        const double dl = delta ? delta[band0 + b] : -1.0;
        const int ra = r0 + 2 * q;
        double* d = dst + b * dbs;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            double a = x[m].x * scale, c = x[m].y * scale;
            if (dl >= 0.0) {
                if (fabs(a) < dl) a = 0.0;
                if (fabs(c) < dl) c = 0.0;
            }
            const int i = t + T * m;
            if (ra < n0) d[(long long)ra * L + i] = a;
            if (ra + 1 < n0) d[(long long)(ra + 1) * L + i] = c;
        }
        __syncthreads();  // everyone is done with `cur` before it is refilled
    }
    cp_async_wait_group<0>();
}

// ---------------------------------------------------------------- rows r2c (persistent)
template <int L>
__global__ void __launch_bounds__(RowCfg<L>::THREADS)
    k2p_rows_r2c(const double* __restrict__ src, long long sbs, double2* __restrict__ dst, long long dbs, int n0,
                 int H, int nbands, const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E, V = RowCfg<L>::V;
    constexpr int KPT = (L / 2 + 1 + T - 1) / T;
    extern __shared__ double2 sm[];  // tile [H][2V] | V line buffers
    double2* tile = sm;
    const int row_blocks = (n0 + 2 * V - 1) / (2 * V);
    const int total = nbands * row_blocks;
    const int q = threadIdx.x / T, t = threadIdx.x - q * T;
    double2* lb = sm + H * 2 * V + q * L;
    double ra_[E], rb_[E];  // prefetched rows of the next item
    auto load = [&](int w) {
        const int b = w / row_blocks, rbk = w - b * row_blocks;
        const int ra = rbk * 2 * V + 2 * q;
        const double* s = src + b * sbs;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int i = t + T * m;
            ra_[m] = ra < n0 ? __ldg(s + (long long)ra * L + i) : 0.0;
            rb_[m] = ra + 1 < n0 ? __ldg(s + (long long)(ra + 1) * L + i) : 0.0;
        }
    };
    int w = blockIdx.x;
    if (w < total) load(w);
    for (; w < total; w += gridDim.x) {
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = make_double2(ra_[m], rb_[m]);
        if (w + (int)gridDim.x < total) load(w + gridDim.x);  // in flight during the FFT
        reg_fft<L, -1>(x, lb, t, tw);
#pragma unroll
        for (int m = 0; m < E; ++m) lb[swz(t + T * m)] = x[m];
        line_sync<T>();
        double2 zk[KPT], zm[KPT];
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int k = t + T * u;
            if (k < H) {
                zk[u] = lb[swz(k)];
                zm[u] = lb[swz(k == 0 ? 0 : L - k)];
            }
        }
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int k = t + T * u;
            if (k < H) {
                tile[tslot<V>(k, 2 * q)] = make_double2(0.5 * (zk[u].x + zm[u].x), 0.5 * (zk[u].y - zm[u].y));
                tile[tslot<V>(k, 2 * q + 1)] = make_double2(0.5 * (zk[u].y + zm[u].y), 0.5 * (zm[u].x - zk[u].x));
            }
        }
        __syncthreads();
        const int b = w / row_blocks, rbk = w - b * row_blocks;
        const int r0 = rbk * 2 * V;
        const int nrows = min(2 * V, n0 - r0);
        double2* d = dst + b * dbs;
        for (int idx = threadIdx.x; idx < H * 2 * V; idx += blockDim.x) {
            const int k = idx / (2 * V), rr = idx - k * 2 * V;
            if (rr < nrows) __stcg(d + (long long)k * n0 + r0 + rr, tile[tslot<V>(k, rr)]);
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- cols dec (persistent)
// grid.x = col_blocks * K; CTA (cb, j) transforms bands j, j+K, ... of the chunk.
template <int L>
__global__ void __launch_bounds__(ColCfg<L>::THREADS)
    k2p_cols_dec(const double2* __restrict__ FT, const double* __restrict__ psiT, long long pbs,
                 double2* __restrict__ inter, long long ibs, int H, int band0, int nb, int col_blocks,
                 const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E;
    extern __shared__ double2 lbuf[];
    const int K = gridDim.x / col_blocks;
    const int cb = blockIdx.x % col_blocks, j = blockIdx.x / col_blocks;
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const int k1 = cb * ColCfg<L>::LINES + li;
    const bool valid = k1 < H;
    const int kk = valid ? k1 : 0;  // clamp for safe (ignored) loads
    double2* sm = lbuf + li * L;
    double2 f[E];
#pragma unroll
    for (int m = 0; m < E; ++m) f[m] = __ldg(FT + (long long)kk * L + t + T * m);
    double p[E];
    if (j < nb) {
        const double* ps = psiT + (long long)(band0 + j) * pbs + (long long)kk * L;
#pragma unroll
        for (int m = 0; m < E; ++m) p[m] = __ldg(ps + t + T * m);
    }
    for (int b = j; b < nb; b += K) {
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = make_double2(f[m].x * p[m], f[m].y * p[m]);  // conj(psi) F, psi real
        if (b + K < nb) {  // next band's filter, in flight during the FFT
            const double* ps = psiT + (long long)(band0 + b + K) * pbs + (long long)kk * L;
#pragma unroll
            for (int m = 0; m < E; ++m) p[m] = __ldg(ps + t + T * m);
        }
        reg_fft<L, +1>(x, sm, t, tw);
        if (valid) {
            double2* o = inter + (long long)b * ibs + (long long)k1 * L;
#pragma unroll
            for (int m = 0; m < E; ++m) __stcg(o + t + T * m, x[m]);
        }
    }
}

// ---------------------------------------------------------------- cols rec (persistent)
// slot[slot0 + j] = sum_{b = j, j+K, ...} FFT_0(inter[b]) * psi_b for this CTA's columns.
template <int L>
__global__ void __launch_bounds__(ColCfg<L>::THREADS)
    k2p_cols_rec(const double2* __restrict__ inter, long long ibs, const double* __restrict__ psiT, long long pbs,
                 double2* __restrict__ slots, long long sbs, int H, int band0, int nb, int col_blocks, int slot0,
                 const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E;
    extern __shared__ double2 lbuf[];
    const int K = gridDim.x / col_blocks;
    const int cb = blockIdx.x % col_blocks, j = blockIdx.x / col_blocks;
    const int li = threadIdx.x / T, t = threadIdx.x - li * T;
    const int k1 = cb * ColCfg<L>::LINES + li;
    const bool valid = k1 < H;
    const int kk = valid ? k1 : 0;
    double2* sm = lbuf + li * L;
    double2 acc[E], xn[E];
    double p[E];
#pragma unroll
    for (int m = 0; m < E; ++m) acc[m] = make_double2(0.0, 0.0);
    if (j < nb) {
        const double2* in = inter + (long long)j * ibs + (long long)kk * L;
        const double* ps = psiT + (long long)(band0 + j) * pbs + (long long)kk * L;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            xn[m] = __ldcg(in + t + T * m);
            p[m] = __ldg(ps + t + T * m);
        }
    }
    for (int b = j; b < nb; b += K) {
        double2 x[E];
        double pc[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            x[m] = xn[m];
            pc[m] = p[m];
        }
        if (b + K < nb) {  // next band in flight during this FFT
            const double2* in = inter + (long long)(b + K) * ibs + (long long)kk * L;
            const double* ps = psiT + (long long)(band0 + b + K) * pbs + (long long)kk * L;
#pragma unroll
            for (int m = 0; m < E; ++m) {
                xn[m] = __ldcg(in + t + T * m);
                p[m] = __ldg(ps + t + T * m);
            }
        }
        reg_fft<L, -1>(x, sm, t, tw);
#pragma unroll
        for (int m = 0; m < E; ++m) {
            acc[m].x = fma(x[m].x, pc[m], acc[m].x);
            acc[m].y = fma(x[m].y, pc[m], acc[m].y);
        }
    }
    if (valid) {
        double2* o = slots + (long long)(slot0 + j) * sbs + (long long)k1 * L;
#pragma unroll
        for (int m = 0; m < E; ++m) __stcg(o + t + T * m, acc[m]);
    }
}

}  // namespace slb
