// Device kernels of the shearlet dec/rec hot path (sm_100a, fp64).
//
// Spectra live as Hermitian halves along the last (fastest) axis:
// [n0][ldh] (2D) or [n0][n1][ldh] (3D) double2, H = n_last/2 + 1 columns used,
// ldh = H rounded up to 8 so every row starts 128-byte aligned. The transform
// is split per axis:
//   rows pass  : the contiguous last axis; two real rows are packed into one
//                complex line (z = x + i y), so r2c/c2r cost one c2c each pair;
//   lines pass : a strided axis (axis 0 in 2D, axes 0/1 in 3D); V adjacent
//                lines form one coalesced tile.
// The shearlet multiply (dec prologue), the 1/N scale + hard threshold (dec
// epilogue), the filter multiply (rec epilogue) and the 1/W weight (rec
// prologue) are fused into those passes, so no standalone elementwise pass
// over the coefficient stack touches HBM.
//
// Reference mapping (paths under /root/reference/proj/core):
//   dec  = forward()  src/transform.cpp:13-61 (conj(psi) * F, IDFT, Re, 1/N)
//   rec  = inverse()  src/transform.cpp:63-125 (sum DFT(c) * psi / W, IDFT)
//   thr  = hard_threshold_impl  src/apps.cpp:57-81 (|x| < delta -> 0)
#pragma once

#include "fft.cuh"

namespace slb {

// ------------------------------------------------------------------ filters
// Real, even filter spectra (the reference's taps are centrally symmetric, so
// psi_hat is real up to rounding; checked at build time).
struct FiltTable2D {
    const double* psi;  // [R][nhalf]
    long long nhalf;
    __device__ __forceinline__ double get(int band, long long e) const {
        return __ldg(psi + (long long)band * nhalf + e);
    }
};

// 3D filters are synthesised on the fly from per-scale factor tables
// (src/system3d.cpp:144-186): psi = g[p] * Phi_k1[p, s1] * Phi_k2[p, s2]
// with the pyramid's axis permutation, or hJ (x) hJ (x) hJ for the lowpass.
struct BandDesc3D {
    int kind;         // 0 lowpass, 3/4/5 pyramid
    int pa, s1, s2;   // principal / secondary axes
    int g_off;        // offset of g (along axis pa) in tab1d
    int p1_off;       // offset of Phi_k1 plane (n[pa] x n[s1]) in tab2d
    int p2_off;       // offset of Phi_k2 plane (n[pa] x n[s2]) in tab2d
};

struct FiltSynth3D {
    const BandDesc3D* bands;
    const double* tab1d;   // 1D real spectra
    const double* tab2d;   // 2D real spectra (full planes, row-major)
    int n[3];
    int lp_off[3];         // lowpass hJ spectra per axis in tab1d
    __device__ __forceinline__ double get(int band, int i0, int i1, int i2) const {
        return get_d(bands[band], i0, i1, i2);
    }
    // descriptor already loaded (hoisted out of per-element loops)
    __device__ __forceinline__ double get_d(const BandDesc3D& d, int i0, int i1, int i2) const {
        if (d.kind == 0)
            return __ldg(tab1d + lp_off[0] + i0) * __ldg(tab1d + lp_off[1] + i1) * __ldg(tab1d + lp_off[2] + i2);
        auto pick = [=](int ax) { return ax == 0 ? i0 : (ax == 1 ? i1 : i2); };  // no local-memory array
        const int p = pick(d.pa), a = pick(d.s1), b = pick(d.s2);
        // selects, not n[d.s1]: a dynamic index into the by-value parameter
        // copies it to a local-memory frame (48 B/thread, L1 traffic per element)
        auto len = [&](int ax) { return ax == 0 ? n[0] : (ax == 1 ? n[1] : n[2]); };
        const int ns1 = len(d.s1), ns2 = len(d.s2);
        if (d.pa == 0) {
            // pyramid 1: the principal index runs along axis 0, the line direction
            // of the axis-0 passes -> read the transposed copy of each plane
            // (stored right after it) so consecutive threads hit consecutive entries
            const int np = n[0];
            return __ldg(tab1d + d.g_off + p) * __ldg(tab2d + d.p1_off + np * ns1 + a * np + p) *
                   __ldg(tab2d + d.p2_off + np * ns2 + b * np + p);
        }
        return __ldg(tab1d + d.g_off + p) * __ldg(tab2d + d.p1_off + p * ns1 + a) *
               __ldg(tab2d + d.p2_off + p * ns2 + b);
    }
    // An axis-0 line (k1, k2 fixed, k0 varying) of one band: only the factors
    // indexed by k0 are loaded per element, the others once per line. Value
    // = three ? (A[k0] B[k0]) C[k0] : (c1 A[k0]) c2 -- the same products in
    // the same order as get_d (IEEE multiplication commutes), so bit-identical.
    struct Ax0Line {
        const double *A, *B, *C;
        double c1, c2;
        bool three;
        __device__ __forceinline__ double at(int k0) const {
            return three ? (__ldg(A + k0) * __ldg(B + k0)) * __ldg(C + k0) : (c1 * __ldg(A + k0)) * c2;
        }
    };
    __device__ __forceinline__ Ax0Line ax0_line(const BandDesc3D& d, int k1, int k2) const {
        Ax0Line l{};
        if (d.kind == 0) {  // (hJ0[k0] hJ1[k1]) hJ2[k2]
            l.three = false;
            l.A = tab1d + lp_off[0];
            l.c1 = __ldg(tab1d + lp_off[1] + k1);
            l.c2 = __ldg(tab1d + lp_off[2] + k2);
            return l;
        }
        auto len = [&](int ax) { return ax == 0 ? n[0] : (ax == 1 ? n[1] : n[2]); };
        const int ns1 = len(d.s1), ns2 = len(d.s2);
        if (d.pa == 0) {  // every factor runs along k0 (transposed planes)
            const int np = n[0];
            const int a = d.s1 == 1 ? k1 : k2, b = d.s2 == 1 ? k1 : k2;
            l.three = true;
            l.A = tab1d + d.g_off;
            l.B = tab2d + d.p1_off + np * ns1 + a * np;
            l.C = tab2d + d.p2_off + np * ns2 + b * np;
            return l;
        }
        const int p = d.pa == 1 ? k1 : k2;
        const double g = __ldg(tab1d + d.g_off + p);
        l.three = false;
        if (d.s1 == 0) {  // (g Phi1[p][k0]) Phi2[p][b]
            const int b = d.s2 == 1 ? k1 : k2;
            l.A = tab2d + d.p1_off + p * ns1;
            l.c1 = g;
            l.c2 = __ldg(tab2d + d.p2_off + p * ns2 + b);
        } else {  // (g Phi1[p][a]) Phi2[p][k0]
            const int a = d.s1 == 1 ? k1 : k2;
            l.A = tab2d + d.p2_off + p * ns2;
            l.c1 = g * __ldg(tab2d + d.p1_off + p * ns1 + a);
            l.c2 = 1.0;
        }
        return l;
    }
};

// ------------------------------------------------------------------ rows pass
// Forward r2c of row pairs: z = x[2q] + i x[2q+1]; Z = FFT(z);
// X[k] = (Z[k] + conj Z[L-k]) / 2, Y[k] = (Z[k] - conj Z[L-k]) / (2i).
__global__ void k_rows_r2c(const double* __restrict__ src, long long src_bstride, double2* __restrict__ dst,
                           long long dst_bstride, int nrows, int H, int ldh, FftPlan p, int V) {
    extern __shared__ double2 smem[];
    const int L = p.L, ld = L + 1;
    double2* a = smem;
    double2* b = smem + V * ld;
    const int npairs = (nrows + 1) >> 1;
    const int q0 = blockIdx.x * V;
    src += blockIdx.y * src_bstride;
    dst += blockIdx.y * dst_bstride;
    for (int t = threadIdx.x; t < V * L; t += blockDim.x) {
        const int v = t / L, i = t - v * L;
        const int q = q0 + v;
        double x = 0.0, y = 0.0;
        if (q < npairs) {
            const int r = 2 * q;
            x = src[(long long)r * L + i];
            if (r + 1 < nrows) y = src[(long long)(r + 1) * L + i];
        }
        a[v * ld + i] = make_double2(x, y);
    }
    __syncthreads();
    const double2* Z = smem_fft<-1>(a, b, V, ld, p);
    for (int t = threadIdx.x; t < V * H; t += blockDim.x) {
        const int v = t / H, k = t - v * H;
        const int q = q0 + v;
        if (q >= npairs) continue;
        const double2 zk = Z[v * ld + k];
        const double2 zm = Z[v * ld + (k == 0 ? 0 : L - k)];
        const int r = 2 * q;
        dst[(long long)r * ldh + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        if (r + 1 < nrows) dst[(long long)(r + 1) * ldh + k] = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
    }
}

// Inverse c2r of row pairs with the 1/N scale and, when delta[band] >= 0, the
// hard threshold |x| < delta -> 0 (apps.cpp:77-78) fused into the store.
// X[0] and X[L/2] are projected to their real parts, which is exactly what
// taking Re of the full complex IDFT does (fft.cpp:113-118).
__global__ void k_rows_c2r(const double2* __restrict__ src, long long src_bstride, double* __restrict__ dst,
                           long long dst_bstride, int nrows, int H, int ldh, FftPlan p, int V, double scale,
                           const double* __restrict__ delta, int band_base) {
    extern __shared__ double2 smem[];
    const int L = p.L, ld = L + 1;
    double2* a = smem;
    double2* b = smem + V * ld;
    const int npairs = (nrows + 1) >> 1;
    const int q0 = blockIdx.x * V;
    src += blockIdx.y * src_bstride;
    dst += blockIdx.y * dst_bstride;
    for (int t = threadIdx.x; t < V * H; t += blockDim.x) {
        const int v = t / H, k = t - v * H;
        const int q = q0 + v;
        double2 X = make_double2(0.0, 0.0), Y = make_double2(0.0, 0.0);
        if (q < npairs) {
            const int r = 2 * q;
            X = src[(long long)r * ldh + k];
            if (r + 1 < nrows) Y = src[(long long)(r + 1) * ldh + k];
        }
        if (k == 0 || 2 * k == L) {
            X.y = 0.0;
            Y.y = 0.0;
        }
        // Z[k] = X[k] + i Y[k];  Z[L-k] = conj(X[k]) + i conj(Y[k])
        a[v * ld + k] = make_double2(X.x - Y.y, X.y + Y.x);
        if (k != 0 && 2 * k != L) a[v * ld + L - k] = make_double2(X.x + Y.y, Y.x - X.y);
    }
    __syncthreads();
    const double2* z = smem_fft<+1>(a, b, V, ld, p);
    const double dl = delta ? delta[band_base + blockIdx.y] : -1.0;
    for (int t = threadIdx.x; t < V * L; t += blockDim.x) {
        const int v = t / L, i = t - v * L;
        const int q = q0 + v;
        if (q >= npairs) continue;
        const double2 w = z[v * ld + i];
        double x = w.x * scale, y = w.y * scale;
        if (dl >= 0.0) {
            if (fabs(x) < dl) x = 0.0;
            if (fabs(y) < dl) y = 0.0;
        }
        const int r = 2 * q;
        dst[(long long)r * L + i] = x;
        if (r + 1 < nrows) dst[(long long)(r + 1) * L + i] = y;
    }
}

// ------------------------------------------------------------------ lines pass
enum LineMode : int {
    kPlain = 0,   // z = src
    kDecMul = 1,  // prologue: z = conj(psi) * F   (transform.cpp:29-30, 53-54)
    kRecMul = 2,  // epilogue: out = FFT(z) * psi   (transform.cpp:81-82, 115-116)
    kDivW = 3,    // prologue: z = src / W         (duals: system2d.cpp:128-140)
};

struct LineGeom {
    int L;            // transform length (points per line)
    long long istride;  // element stride between points
    long long ostride;  // stride between outer blocks
    int cw;           // padded lines per outer block (multiple of ldh)
    int ldh, H;       // pad test: (c % ldh) < H
    int n1;           // 3D: size of axis 1 (index decode); 0 for 2D
    long long nhalf;  // elements per spectrum (band stride)
};

// filter multiply of the generic lines pass: real (centrally symmetric
// filters) or complex (asymmetric fans) spectra; the dec side takes conj(psi)
template <bool CONJ>
__device__ __forceinline__ double2 filt_mul(double2 z, double p) {
    return cscale(z, p);
}
template <bool CONJ>
__device__ __forceinline__ double2 filt_mul(double2 z, double2 p) {
    return cmul(z, CONJ ? cconj(p) : p);
}

template <int DIR, int MODE, class Filt>
__global__ void k_lines(const double2* __restrict__ src, long long src_bstride, double2* __restrict__ dst,
                        long long dst_bstride, LineGeom g, FftPlan p, int V, Filt filt, int band_base,
                        const double* __restrict__ W) {
    extern __shared__ double2 smem[];
    const int L = p.L, ld = L + 1;
    double2* a = smem;
    double2* b = smem + V * ld;
    const int tiles_per_outer = (g.cw + V - 1) / V;
    const int o = blockIdx.x / tiles_per_outer;
    const int c0 = (blockIdx.x - o * tiles_per_outer) * V;
    const int band = band_base + blockIdx.y;
    const long long base = (long long)o * g.ostride + c0;
    src += blockIdx.y * src_bstride;
    dst += blockIdx.y * dst_bstride;
    // load: consecutive threads -> consecutive lines (contiguous in memory)
    for (int t = threadIdx.x; t < V * L; t += blockDim.x) {
        const int i = t / V, v = t - i * V;
        const int c = c0 + v;
        double2 z = make_double2(0.0, 0.0);
        if (c < g.cw && (c % g.ldh) < g.H) {
            const long long e = base + (long long)i * g.istride + v;
            z = src[e];
            if (MODE == kDecMul) {
                z = filt_mul<true>(z, filt.get(band, e));
            } else if (MODE == kDivW) {
                const double w = __ldg(W + e);
                z = make_double2(z.x / w, z.y / w);
            }
        }
        a[v * ld + i] = z;
    }
    __syncthreads();
    const double2* r = smem_fft<DIR>(a, b, V, ld, p);
    for (int t = threadIdx.x; t < V * L; t += blockDim.x) {
        const int i = t / V, v = t - i * V;
        const int c = c0 + v;
        if (c < g.cw && (c % g.ldh) < g.H) {
            const long long e = base + (long long)i * g.istride + v;
            double2 z = r[v * ld + i];
            if (MODE == kRecMul) z = filt_mul<false>(z, filt.get(band, e));
            dst[e] = z;
        }
    }
}

// Adapter giving the 3D synthesiser the same get(band, e) interface.
struct FiltSynth3DFlat {
    FiltSynth3D s;
    int ldh;
    __device__ __forceinline__ double get(int band, long long e) const {
        const int i2 = (int)(e % ldh);
        const long long t = e / ldh;
        const int i1 = (int)(t % s.n[1]);
        const int i0 = (int)(t / s.n[1]);
        return s.get(band, i0, i1, i2);
    }
};

struct NoFilt {
    __device__ __forceinline__ double get(int, long long) const { return 1.0; }
};

// ------------------------------------------------------------------ reductions
// acc[e] (+)= sum_b prod[b][e], bands summed in index order (deterministic).
__global__ void k_reduce_bands(double2* __restrict__ acc, const double2* __restrict__ prod, long long nhalf,
                               int nb, int accumulate) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < nhalf;
         e += (long long)gridDim.x * blockDim.x) {
        double2 s = accumulate ? acc[e] : make_double2(0.0, 0.0);
        for (int bnd = 0; bnd < nb; ++bnd) s = cadd(s, prod[(long long)bnd * nhalf + e]);
        acc[e] = s;
    }
}

// Standalone hard threshold (apps.cpp:57-81) for an existing stack, in/out of place.
__global__ void k_threshold(const double* __restrict__ in, double* __restrict__ out, long long n,
                            const double* __restrict__ delta) {
    const int band = blockIdx.y;
    const double dl = delta[band];
    const double* src = in + (long long)band * n;
    double* dst = out + (long long)band * n;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        const double x = src[e];
        dst[e] = (dl >= 0.0 && fabs(x) < dl) ? 0.0 : x;
    }
}

}  // namespace slb
