// Persistent "megakernel" for the fused 2D denoise of a batch of frames.
//
// One launch runs every pass of every frame as a stream of tasks handed out
// by a global ticket counter, so there are no kernel boundaries (launch ramp,
// tails, idle SMs) between passes. Tasks only ever wait on tasks with smaller
// tickets, through per-band completion counters (release: __threadfence +
// atomicAdd; acquire: ld.acquire.gpu spin), which makes the schedule
// deadlock-free for any number of resident CTAs.
//
// Per frame f (band b, column block cb of 4 columns, row block rb of 4 row pairs):
//   F1(f,rb)  rows r2c of f            -> acc[f] (temporary)
//   F2(f,cb)  cols FFT                 -> F[f]                 waits F1(f,*)
//   D(f,b,cb) IFFT_0(F psi_b)          -> ring[seq]           waits F2(f,*), ring slot free
//   R(f,b,rb) IFFT_1, /N, threshold    -> stack; FFT_1 -> ring waits D(f,b,*)
//   C(f,b,cb) acc += FFT_0(ring) psi_b (band order per cb)     waits R(f,b,*), C(f,b-1,cb)
//   X(f,cb)   IFFT_0(acc / W)          -> ring[...]           waits C(f,nb-1,cb)
//   Y(f,rb)   rows c2r, /N             -> out[f]               waits X(f,*)
// seq = f * nb + b indexes a ring of S intermediate spectra (L2-sized).
#pragma once

#include "fast2d.cuh"

namespace slb {

enum MegaTask : int { kF1 = 0, kF2 = 1, kD = 2, kR = 3, kC = 4, kX = 5, kY = 6 };

struct MegaArgs {
    const int4* tasks;  // {type, frame, band, block}
    int ntasks;
    int* ticket;        // [1]
    int* cnt;           // counters, see offsets below
    int nframes, nb, band0;
    int n0, H, S;       // rows, half columns, ring slots
    const double* f;    // [frames][n0][L]
    double* stack;      // [frames][nb][n0][L]
    double* out;        // [frames][n0][L]
    double2* F;         // [frames][H][n0]
    double2* acc;       // [frames][H][n0]
    double2* ring;      // [S][H][n0]
    const double* psiT; // [R][H][n0]
    const double* WT;   // [H][n0]
    const double* delta;
    double scale;
    const double2* tw;
    int row_blocks, col_blocks;
    // counter offsets
    int oF1, oF2, oD, oR, oC, oChain, oX;
};

__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void wait_geq(const int* p, int target) {
    if (threadIdx.x == 0) {
        int ns = 32;
        while (ld_acquire(p) < target) {
            __nanosleep(ns);
            ns = min(ns * 2, 1024);
        }
    }
    __syncthreads();
}

__device__ __forceinline__ void signal(int* p) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(p, 1);
    }
}

template <int L>
struct Mega {
    static constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E;
    static constexpr int V = 256 / T;        // row pairs per rows task / lines per cols task
    static constexpr int LINES = V;
    static constexpr int THREADS = 256;
    static constexpr int KPT = (L / 2 + 1 + T - 1) / T;

    // ---- rows: load the [H][2V] tile of a column-major half spectrum (cp.async)
    __device__ static void load_tile(double2* tile, const double2* src, int n0, int H, int r0) {
        const int nrows = min(2 * V, n0 - r0);
        for (int idx = threadIdx.x; idx < H * 2 * V; idx += blockDim.x) {
            const int k = idx / (2 * V), rr = idx - k * 2 * V;
            if (rr < nrows)
                cp_async16(tile + tslot<V>(k, rr), src + (long long)k * n0 + r0 + rr);
            else
                tile[tslot<V>(k, rr)] = make_double2(0.0, 0.0);
        }
        cp_async_wait_all();
        __syncthreads();
    }
    // gather pair-packed Z = X + iY (Hermitian completion) for line q
    __device__ static void gather_c2r(double2 (&x)[E], const double2* tile, int q, int t, int H) {
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int k = t + T * m;
            double2 X, Y;
            if (k < H) {
                X = tile[tslot<V>(k, 2 * q)];
                Y = tile[tslot<V>(k, 2 * q + 1)];
                if (k == 0 || 2 * k == L) {
                    X.y = 0.0;
                    Y.y = 0.0;
                }
                x[m] = make_double2(X.x - Y.y, X.y + Y.x);
            } else {
                X = tile[tslot<V>(L - k, 2 * q)];
                Y = tile[tslot<V>(L - k, 2 * q + 1)];
                x[m] = make_double2(X.x + Y.y, Y.x - X.y);
            }
        }
    }
    // r2c split of Z (in registers) into the tile rows 2q, 2q+1, then store the tile
    __device__ static void split_store(double2 (&x)[E], double2* tile, double2* lb, int q, int t, int H,
                                       double2* dst, int n0, int r0) {
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
        __syncthreads();
#pragma unroll
        for (int u = 0; u < KPT; ++u) {
            const int k = t + T * u;
            if (k < H) {
                tile[tslot<V>(k, 2 * q)] = make_double2(0.5 * (zk[u].x + zm[u].x), 0.5 * (zk[u].y - zm[u].y));
                tile[tslot<V>(k, 2 * q + 1)] = make_double2(0.5 * (zk[u].y + zm[u].y), 0.5 * (zm[u].x - zk[u].x));
            }
        }
        __syncthreads();
        const int nrows = min(2 * V, n0 - r0);
        for (int idx = threadIdx.x; idx < H * 2 * V; idx += blockDim.x) {
            const int k = idx / (2 * V), rr = idx - k * 2 * V;
            if (rr < nrows) __stcg(dst + (long long)k * n0 + r0 + rr, tile[tslot<V>(k, rr)]);
        }
    }

    // ---- task bodies
    __device__ __noinline__ static void rows_r2c_task(const MegaArgs& a, double2* tile, const double* src, double2* dst, int rb) {
        const int q = threadIdx.x / T, t = threadIdx.x - q * T;
        const int r0 = rb * 2 * V, ra = r0 + 2 * q;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int i = t + T * m;
            x[m] = make_double2(ra < a.n0 ? __ldg(src + (long long)ra * L + i) : 0.0,
                                ra + 1 < a.n0 ? __ldg(src + (long long)(ra + 1) * L + i) : 0.0);
        }
        double2* lb = tile + q * L;
        reg_fft<L, -1>(x, lb, t, a.tw);
        split_store(x, tile, lb, q, t, a.H, dst, a.n0, r0);
    }
    __device__ __noinline__ static void rows_c2r_task(const MegaArgs& a, double2* tile, const double2* src, double* dst, int rb) {
        const int r0 = rb * 2 * V;
        load_tile(tile, src, a.n0, a.H, r0);
        const int q = threadIdx.x / T, t = threadIdx.x - q * T;
        double2 x[E];
        gather_c2r(x, tile, q, t, a.H);
        __syncthreads();
        double2* lb = tile + q * L;
        reg_fft<L, +1>(x, lb, t, a.tw);
        const int ra = r0 + 2 * q;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const int i = t + T * m;
            if (ra < a.n0) dst[(long long)ra * L + i] = x[m].x * a.scale;
            if (ra + 1 < a.n0) dst[(long long)(ra + 1) * L + i] = x[m].y * a.scale;
        }
    }
    __device__ __noinline__ static void rows_fused_task(const MegaArgs& a, double2* tile, double2* inter, double* band, double dl,
                                           int rb) {
        const int r0 = rb * 2 * V;
        load_tile(tile, inter, a.n0, a.H, r0);
        const int q = threadIdx.x / T, t = threadIdx.x - q * T;
        double2 x[E];
        gather_c2r(x, tile, q, t, a.H);
        __syncthreads();
        double2* lb = tile + q * L;
        reg_fft<L, +1>(x, lb, t, a.tw);
        const int ra = r0 + 2 * q;
#pragma unroll
        for (int m = 0; m < E; ++m) {
            double u = x[m].x * a.scale, v = x[m].y * a.scale;
            if (fabs(u) < dl) u = 0.0;  // apps.cpp:77-78 (keep |x| >= delta)
            if (fabs(v) < dl) v = 0.0;
            const int i = t + T * m;
            if (ra < a.n0) band[(long long)ra * L + i] = u;
            if (ra + 1 < a.n0) band[(long long)(ra + 1) * L + i] = v;
            x[m] = make_double2(ra < a.n0 ? u : 0.0, ra + 1 < a.n0 ? v : 0.0);
        }
        reg_fft<L, -1>(x, lb, t, a.tw);
        split_store(x, tile, lb, q, t, a.H, inter, a.n0, r0);
    }
    // column tasks: 4 lines (columns k1) of a column-major half spectrum
    __device__ __noinline__ static void cols_fwd_task(const MegaArgs& a, double2* lbuf, const double2* src, double2* dst, int cb) {
        const int li = threadIdx.x / T, t = threadIdx.x - li * T;
        const int k1 = cb * LINES + li;
        const bool valid = k1 < a.H;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = valid ? __ldcg(src + (long long)k1 * L + t + T * m) : make_double2(0.0, 0.0);
        reg_fft<L, -1>(x, lbuf + li * L, t, a.tw);
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; ++m) __stcg(dst + (long long)k1 * L + t + T * m, x[m]);
        }
    }
    __device__ __noinline__ static void cols_dec_task(const MegaArgs& a, double2* lbuf, const double2* F, const double* psi,
                                         double2* dst, int cb) {
        const int li = threadIdx.x / T, t = threadIdx.x - li * T;
        const int k1 = cb * LINES + li;
        const bool valid = k1 < a.H;
        const int kk = valid ? k1 : 0;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const double2 fv = __ldcg(F + (long long)kk * L + t + T * m);
            const double p = valid ? __ldg(psi + (long long)kk * L + t + T * m) : 0.0;
            x[m] = make_double2(fv.x * p, fv.y * p);  // conj(psi) F, psi real
        }
        reg_fft<L, +1>(x, lbuf + li * L, t, a.tw);
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; ++m) __stcg(dst + (long long)k1 * L + t + T * m, x[m]);
        }
    }
    __device__ __noinline__ static void cols_rec_task(const MegaArgs& a, double2* lbuf, const double2* src, const double* psi,
                                         double2* acc, bool first, int cb) {
        const int li = threadIdx.x / T, t = threadIdx.x - li * T;
        const int k1 = cb * LINES + li;
        const bool valid = k1 < a.H;
        const int kk = valid ? k1 : 0;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) x[m] = __ldcg(src + (long long)kk * L + t + T * m);
        reg_fft<L, -1>(x, lbuf + li * L, t, a.tw);
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; ++m) {
                const double p = __ldg(psi + (long long)k1 * L + t + T * m);
                double2 s = first ? make_double2(0.0, 0.0) : __ldcg(acc + (long long)k1 * L + t + T * m);
                s.x = fma(x[m].x, p, s.x);
                s.y = fma(x[m].y, p, s.y);
                __stcg(acc + (long long)k1 * L + t + T * m, s);
            }
        }
    }
    __device__ __noinline__ static void cols_final_task(const MegaArgs& a, double2* lbuf, const double2* acc, double2* dst,
                                           int cb) {
        const int li = threadIdx.x / T, t = threadIdx.x - li * T;
        const int k1 = cb * LINES + li;
        const bool valid = k1 < a.H;
        const int kk = valid ? k1 : 0;
        double2 x[E];
#pragma unroll
        for (int m = 0; m < E; ++m) {
            const double2 v = __ldcg(acc + (long long)kk * L + t + T * m);
            const double w = __ldg(a.WT + (long long)kk * L + t + T * m);
            x[m] = make_double2(v.x / w, v.y / w);
        }
        reg_fft<L, +1>(x, lbuf + li * L, t, a.tw);
        if (valid) {
#pragma unroll
            for (int m = 0; m < E; ++m) __stcg(dst + (long long)k1 * L + t + T * m, x[m]);
        }
    }
};

template <int L>
__global__ void __launch_bounds__(256, 2) k2_denoise_mega(MegaArgs a) {
    using M = Mega<L>;
    extern __shared__ double2 smem[];  // max(tile [H][2V], 4 line buffers)
    __shared__ int s_ticket;
    const long long nhT = (long long)a.H * a.n0;
    const long long N = (long long)a.n0 * L;
    for (;;) {
        if (threadIdx.x == 0) s_ticket = atomicAdd(a.ticket, 1);
        __syncthreads();
        const int tk = s_ticket;
        __syncthreads();
        if (tk >= a.ntasks) break;
        const int4 task = a.tasks[tk];
        const int f = task.y, b = task.z, blk = task.w;
        const int seq = f * a.nb + b;
        double2* Ff = a.F + f * nhT;
        double2* accf = a.acc + f * nhT;
        switch (task.x) {
            case kF1:
                M::rows_r2c_task(a, smem, a.f + f * N, accf, blk);
                signal(a.cnt + a.oF1 + f);
                break;
            case kF2:
                wait_geq(a.cnt + a.oF1 + f, a.row_blocks);
                M::cols_fwd_task(a, smem, accf, Ff, blk);
                signal(a.cnt + a.oF2 + f);
                break;
            case kD: {
                wait_geq(a.cnt + a.oF2 + f, a.col_blocks);
                if (seq >= a.S) wait_geq(a.cnt + a.oC + (seq - a.S), a.col_blocks);  // ring slot free
                M::cols_dec_task(a, smem, Ff, a.psiT + (long long)(a.band0 + b) * nhT, a.ring + (seq % a.S) * nhT, blk);
                signal(a.cnt + a.oD + seq);
                break;
            }
            case kR: {
                wait_geq(a.cnt + a.oD + seq, a.col_blocks);
                M::rows_fused_task(a, smem, a.ring + (seq % a.S) * nhT,
                                   a.stack + ((long long)f * a.nb + b) * N, a.delta[a.band0 + b], blk);
                signal(a.cnt + a.oR + seq);
                break;
            }
            case kC: {
                wait_geq(a.cnt + a.oR + seq, a.row_blocks);
                wait_geq(a.cnt + a.oChain + f * a.col_blocks + blk, b);  // band order per column block
                M::cols_rec_task(a, smem, a.ring + (seq % a.S) * nhT, a.psiT + (long long)(a.band0 + b) * nhT, accf,
                                 b == 0, blk);
                signal(a.cnt + a.oC + seq);
                signal(a.cnt + a.oChain + f * a.col_blocks + blk);
                break;
            }
            case kX: {
                wait_geq(a.cnt + a.oChain + f * a.col_blocks + blk, a.nb);
                M::cols_final_task(a, smem, accf, Ff, blk);  // F[f] is free again: reuse as output
                signal(a.cnt + a.oX + f);
                break;
            }
            case kY: {
                wait_geq(a.cnt + a.oX + f, a.col_blocks);
                M::rows_c2r_task(a, smem, Ff, a.out + f * N, blk);
                break;
            }
        }
        __syncthreads();
    }
}

}  // namespace slb
