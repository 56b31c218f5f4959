// Register-resident fp64 Stockham FFT with compile-time radix plans.
//
// One line of length L is transformed by T threads, each holding E = L / T
// complex values in registers. Thread t holds elements t + T*m (m < E) both on
// entry and on exit, so global loads/stores of a line are coalesced across
// the T threads without any staging. Between radix stages the line goes
// through a private shared-memory buffer of L complex values (double2 in
// the fp64 path, float2 in the fp32 mode) with an XOR swizzle
// (e ^ ((e >> 3) & 7)) that makes both the strided Stockham writes and the
// contiguous reads bank-conflict free; lines of T <= 32 threads synchronise
// with __syncwarp, wider lines with a named barrier per line.
//
// Stage s (radix R, Ns = product of earlier radices) performs the Stockham
// butterfly j: inputs j + r*L/R (times w^{r*(j%Ns)}, w = e^{DIR 2 pi i/(Ns R)}),
// outputs (j - j%Ns)*R + j%Ns + r*Ns; thread t owns butterflies j = t + T*q.
#pragma once

#include "fft.cuh"

namespace slb {

template <int L>
struct RegPlan;  // T, E, NST, R[]

#define SLB_REG_PLAN(L_, T_, ...)                                     \
    template <>                                                       \
    struct RegPlan<L_> {                                              \
        static constexpr int T = T_;                                  \
        static constexpr int E = L_ / T_;                             \
        static constexpr int R[] = {__VA_ARGS__};                     \
        static constexpr int NST = sizeof(R) / sizeof(int);           \
    };

// E = 8 complex per thread (16 doubles) keeps kernels near 64-80 registers.
#ifndef SLB_WIDE_E
SLB_REG_PLAN(64, 8, 8, 8)
#ifndef SLB_PLAN128
SLB_REG_PLAN(128, 16, 8, 4, 4)
#else
SLB_PLAN128
#endif
SLB_REG_PLAN(256, 32, 8, 8, 4)
#if defined(SLB_PLAN512_WIDE)
SLB_REG_PLAN(512, 16, 32, 16)  // one exchange per line, 32 complex per thread
#elif !defined(SLB_PLAN512)
SLB_REG_PLAN(512, 64, 8, 8, 8)
#else
SLB_PLAN512
#endif
#ifndef SLB_PLAN1024
SLB_REG_PLAN(1024, 128, 8, 8, 4, 4)
#else
SLB_PLAN1024
#endif
SLB_REG_PLAN(2048, 256, 8, 8, 8, 4)
#ifndef SLB_PLAN192
SLB_REG_PLAN(192, 16, 12, 4, 4)  // radix 12 in registers: 2 exchanges instead of 3 (4,4,4,3)
#else
SLB_PLAN192
#endif
#else
SLB_REG_PLAN(64, 8, 8, 8)
SLB_REG_PLAN(128, 16, 8, 4, 4)
SLB_REG_PLAN(256, 16, 16, 16)
SLB_REG_PLAN(512, 32, 8, 8, 8)
SLB_REG_PLAN(1024, 64, 16, 8, 8)
SLB_REG_PLAN(2048, 128, 16, 16, 8)
SLB_REG_PLAN(192, 8, 8, 8, 3)
#endif
// plan of the fused rows kernel (k2_rows_fused): RegPlan<L> except 512, which
// runs 32 threads x 16 complex per line there (warp-synchronous exchanges, r2c
// mirror pairs by shuffles): measured 2D 512^2 batch +5 % over 64 x 8
// (profiles/r2_ab_fused_rowplan.log; -DSLB_FUSEDPLAN512_T64 restores 64 x 8)
template <int L>
struct FusedRowPlan : RegPlan<L> {};
#ifndef SLB_FUSEDPLAN512_T64
template <>
struct FusedRowPlan<512> {
    static constexpr int T = 32;
    static constexpr int E = 16;
    static constexpr int R[] = {8, 8, 8};
    static constexpr int NST = 3;
};
#endif
// 1024: 64 threads x 16 complex per line (radix 8, 8, 16: two exchanges
// instead of the (8, 8, 4, 4) RegPlan's three): 2D 1024^2 x 64 +8 %
// (profiles/r2b_ab_rows1024_plan.log; -DSLB_FUSEDPLAN1024_T128 restores 128 x 8)
#ifndef SLB_FUSEDPLAN1024_T128
template <>
struct FusedRowPlan<1024> {
    static constexpr int T = 64;
    static constexpr int E = 16;
    static constexpr int R[] = {8, 8, 16};
    static constexpr int NST = 3;
};
#endif
// plan of the 2D column kernels (k2_cols_dec / rec / sum): RegPlan<L> unless a
// column-specific split is selected (A/B: -DSLB_COLPLAN512_T32)
template <int L>
struct ColPlan : RegPlan<L> {};
#ifdef SLB_COLPLAN512_T32
template <>
struct ColPlan<512> {
    static constexpr int T = 32;
    static constexpr int E = 16;
    static constexpr int R[] = {8, 8, 8};
    static constexpr int NST = 3;
};
#endif
#undef SLB_REG_PLAN

template <int L>
constexpr int plan_ns(int s) {
    int ns = 1;
    for (int i = 0; i < s; ++i) ns *= RegPlan<L>::R[i];
    return ns;
}

// Line exchange buffers are padded by one slot per 8 elements: e -> e + e/8.
// Stockham stores (stride NS, or 8 consecutive elements per thread) and loads
// (stride L/R) are then bank-conflict free for 16-byte accesses, and every
// address is a per-thread base plus a compile-time offset (no per-access XOR).
// The rows kernels keep the unpadded XOR swizzle (PAD = false): their line
// buffers alias a staging tile sized for L-element lines, and measured faster.
// Length 192 (radix 12 first) uses e -> e + e/24 in both modes: the stride-12
// stores of the radix-12 stage (e = 12 t + r) land on 8 distinct 16-byte bank
// groups per quarter-warp (4 t + t/2 mod 8), which neither the XOR swizzle nor
// the e/8 pad achieves (both 2-way), and aligned runs of 8 stay distinct.
// Plans whose first radix is 16 or 32 (one thread holds 16t..16t+15 or
// 32t..32t+31 before the first store) XOR the 16-byte slot with e >> 4 / e >> 5
// instead, in both modes.
#ifndef SLB_SWZ192
#define SLB_SWZ192 1
#endif
template <int L>
struct SwzShift {
    static constexpr int value = RegPlan<L>::R[0] == 32 ? 5 : (RegPlan<L>::R[0] == 16 ? 4 : 3);
};
template <>
struct SwzShift<0> {
    static constexpr int value = 3;
};
template <bool PAD = true, int L = 0, int ESZ = 16>
__device__ __forceinline__ int swz(int e) {
    if constexpr (L == 192 && SLB_SWZ192 && ESZ == 16)  // fp32 (8-byte) lines: the XOR swizzle measured 4 % faster
        return e + static_cast<int>(static_cast<unsigned>(e) / 24u);
    else if constexpr (SwzShift<L>::value != 3)
        return e ^ ((e >> SwzShift<L>::value) & 7);
    else if constexpr (PAD)
        return e + (e >> 3);
    else
        return e ^ ((e >> 3) & 7);
}
template <int L, bool PAD = true>
struct LineBuf {
    static constexpr int N = (L == 192 && SLB_SWZ192) ? L + L / 24
                             : (SwzShift<L>::value != 3 ? L : (PAD ? L + L / 8 : L));  // double2 slots per line buffer
};

template <int T>
__device__ __forceinline__ void line_sync() {
    if constexpr (T <= 32) {
        __syncwarp();
    } else {
        // one named barrier per line (ids 1..15), T threads each
        asm volatile("bar.sync %0, %1;" ::"r"(1 + (int)(threadIdx.x / T)), "r"(T) : "memory");
    }
}

// radix-16 = 4 x 4 with internal twiddles w16^{n1 k2}
template <int DIR, class C>
__device__ __forceinline__ void bfly16(C* a) {
    using Rl = RealOf<C>;
    constexpr Rl c1 = Rl(0.92387953251128675613), s1 = Rl(0.38268343236508977173), r2 = Rl(0.70710678118654752440);
    // stage 1: four radix-4 over n2 (stride 4), n1 = 0..3
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) bfly4<DIR>(a[n1], a[n1 + 4], a[n1 + 8], a[n1 + 12]);
    // a[n1 + 4 k1] now holds sum_n2 x[n1 + 4 n2] w4^{n2 k1}; twiddle by w16^{n1 k1}
    auto tw = [](C v, Rl c, Rl s) {  // v * (c + DIR i s)
        return mkc<C>(v.x * c - DIR * v.y * s, v.y * c + DIR * v.x * s);
    };
    a[5] = tw(a[5], c1, s1);     // n1=1,k1=1: w^1
    a[9] = tw(a[9], r2, r2);     // n1=1,k1=2: w^2
    a[13] = tw(a[13], s1, c1);   // n1=1,k1=3: w^3
    a[6] = tw(a[6], r2, r2);     // n1=2,k1=1: w^2
    a[10] = mul_di<DIR>(a[10]);  // n1=2,k1=2: w^4
    a[14] = tw(a[14], -r2, r2);  // n1=2,k1=3: w^6
    a[7] = tw(a[7], s1, c1);     // n1=3,k1=1: w^3
    a[11] = tw(a[11], -r2, r2);  // n1=3,k1=2: w^6
    a[15] = tw(a[15], -c1, -s1); // n1=3,k1=3: w^9
    // stage 2: radix-4 over n1 for each k1; output index k1 + 4 k2
    C o[16];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        C b0 = a[4 * k1], b1 = a[4 * k1 + 1], b2 = a[4 * k1 + 2], b3 = a[4 * k1 + 3];
        bfly4<DIR>(b0, b1, b2, b3);
        o[k1] = b0;
        o[k1 + 4] = b1;
        o[k1 + 8] = b2;
        o[k1 + 12] = b3;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = o[i];
}

// radix-12 = 4 x 3: n = n1 + 3 n2, radix-4 over n2, twiddle w12^{n1 k1},
// radix-3 over n1; output index k1 + 4 k2
template <int DIR, class C>
__device__ __forceinline__ void bfly12(C* a) {
    using Rl = RealOf<C>;
    constexpr Rl h = Rl(0.86602540378443864676);  // sqrt(3)/2
    constexpr Rl half = Rl(0.5);
#pragma unroll
    for (int n1 = 0; n1 < 3; ++n1) bfly4<DIR>(a[n1], a[n1 + 3], a[n1 + 6], a[n1 + 9]);
    auto tw = [](C v, Rl c, Rl s) {  // v * (c + DIR i s)
        return mkc<C>(v.x * c - DIR * v.y * s, v.y * c + DIR * v.x * s);
    };
    a[4] = tw(a[4], h, half);     // n1=1,k1=1: w^1
    a[7] = tw(a[7], half, h);     // n1=1,k1=2: w^2
    a[10] = mul_di<DIR>(a[10]);   // n1=1,k1=3: w^3
    a[5] = tw(a[5], half, h);     // n1=2,k1=1: w^2
    a[8] = tw(a[8], -half, h);    // n1=2,k1=2: w^4
    a[11] = mkc<C>(-a[11].x, -a[11].y);  // n1=2,k1=3: w^6
    C o[12];
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
        C b0 = a[3 * k1], b1 = a[3 * k1 + 1], b2 = a[3 * k1 + 2];
        bfly3<DIR>(b0, b1, b2);
        o[k1] = b0;
        o[k1 + 4] = b1;
        o[k1 + 8] = b2;
    }
#pragma unroll
    for (int i = 0; i < 12; ++i) a[i] = o[i];
}

// radix-32 = radix-2 over two radix-16 halves (decimation in time):
// X[k] = E[k] + w32^k O[k], X[k+16] = E[k] - w32^k O[k].
template <int DIR, class C>
__device__ __forceinline__ void bfly32(C* a) {
    using Rl = RealOf<C>;
    C e[16], o[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
        e[i] = a[2 * i];
        o[i] = a[2 * i + 1];
    }
    bfly16<DIR>(e);
    bfly16<DIR>(o);
    constexpr double c[16] = {1.0,
                              0.98078528040323044913,
                              0.92387953251128675613,
                              0.83146961230254523708,
                              0.70710678118654752440,
                              0.55557023301960222474,
                              0.38268343236508977173,
                              0.19509032201612826785,
                              0.0,
                              -0.19509032201612826785,
                              -0.38268343236508977173,
                              -0.55557023301960222474,
                              -0.70710678118654752440,
                              -0.83146961230254523708,
                              -0.92387953251128675613,
                              -0.98078528040323044913};
#pragma unroll
    for (int k = 0; k < 16; ++k) {
        // w32^k = cos(2 pi k/32) + DIR i sin(2 pi k/32); sin(2 pi k/32) = cos(2 pi (8-k)/32)
        const Rl cs = Rl(c[k]);
        const Rl sn = Rl(k <= 8 ? c[8 - k] : c[k - 8]);
        const C t = k == 0 ? o[0] : mkc<C>(o[k].x * cs - DIR * o[k].y * sn, o[k].y * cs + DIR * o[k].x * sn);
        a[k] = cadd(e[k], t);
        a[k + 16] = csub(e[k], t);
    }
}

// Butterfly of radix R on x[q + B*r], r < R.
template <int R, int DIR, int E, class C>
__device__ __forceinline__ void bfly_strided(C (&x)[E], int q, int B) {
    C v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = x[q + B * r];
    if constexpr (R == 2) {
        bfly2<DIR>(v[0], v[1]);
    } else if constexpr (R == 3) {
        bfly3<DIR>(v[0], v[1], v[2]);
    } else if constexpr (R == 4) {
        bfly4<DIR>(v[0], v[1], v[2], v[3]);
    } else if constexpr (R == 8) {
        bfly8<DIR>(v);
    } else if constexpr (R == 12) {
        bfly12<DIR>(v);
    } else if constexpr (R == 16) {
        bfly16<DIR>(v);
    } else if constexpr (R == 32) {
        bfly32<DIR>(v);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) x[q + B * r] = v[r];
}

// product of the first S radices of plan PL
template <class PL, int S>
struct PlanNS {
    static constexpr int value = PlanNS<PL, S - 1>::value * PL::R[S - 1];
};
template <class PL>
struct PlanNS<PL, 0> {
    static constexpr int value = 1;
};

// Base twiddle w^{jm} of butterfly q of stage S: a table load by default, or
// a value the caller preloaded once (TwPreK: kernels that run many FFTs of the
// same thread layout -- the twiddles depend only on the thread index)
template <int DIR, class C>
struct TwTable {
    const C* __restrict__ tw;
    template <int S>
    __device__ __forceinline__ C get(int /*q*/, int idx) const { return twiddle<DIR>(tw, idx); }
};

// SWL: the length whose exchange swizzle the line buffer uses (0: the plain
// XOR swizzle, L slots per line, for buffers sized exactly L)
template <int L, int DIR, int S, bool PAD, class C = double2, class PL = RegPlan<L>, int SWL = L>
struct RegStage {
    using P = PL;
    static constexpr int R = P::R[S];
    static constexpr int E = P::E;
    static constexpr int T = P::T;
    static constexpr int B = E / R;
    static constexpr int NS = PlanNS<PL, S>::value;
    static_assert(E % R == 0, "radix must divide the per-thread element count");

    __device__ __forceinline__ static void run(C (&x)[E], C* sm, int t, const C* __restrict__ tw) {
        run_w(x, sm, t, TwTable<DIR, C>{tw});
    }
    template <class TW>
    __device__ __forceinline__ static void run_w(C (&x)[E], C* sm, int t, const TW& tws) {
#pragma unroll
        for (int q = 0; q < B; ++q) {
            const int j = t + T * q;
            const int jm = j % NS;
            if constexpr (NS > 1) {
                // one table load per butterfly; w^2..w^(R-1) by complex products
                // (error ~3 ulp, far inside the 1e-10 budget) instead of R-1
                // loads through the L1 data pipe
                const C w1 = tws.template get<S>(q, jm * (L / (NS * R)));
                C wp[R];
                wp[1] = w1;
#pragma unroll
                for (int r = 2; r < R; ++r) wp[r] = (r & 1) ? cmul(wp[r - 1], w1) : cmul(wp[r / 2], wp[r / 2]);
#pragma unroll
                for (int r = 1; r < R; ++r) x[q + B * r] = cmul(x[q + B * r], wp[r]);
            }
            bfly_strided<R, DIR>(x, q, B);
        }
        if constexpr (S + 1 < P::NST) {
#pragma unroll
            for (int q = 0; q < B; ++q) {
                const int j = t + T * q;
                const int jm = j % NS;
                const int base = (j - jm) * R + jm;
#pragma unroll
                for (int r = 0; r < R; ++r) sm[swz<PAD, SWL, sizeof(C)>(base + r * NS)] = x[q + B * r];
            }
            line_sync<T>();
            constexpr int R2 = P::R[S + 1];
            constexpr int B2 = E / R2;
#pragma unroll
            for (int q = 0; q < B2; ++q) {
                const int j = t + T * q;
#pragma unroll
                for (int r = 0; r < R2; ++r) x[q + B2 * r] = sm[swz<PAD, SWL, sizeof(C)>(j + r * (L / R2))];
            }
            line_sync<T>();
            RegStage<L, DIR, S + 1, PAD, C, PL, SWL>::run_w(x, sm, t, tws);
        }
    }
};

// per-thread base twiddles of every stage s >= 1 (B butterflies each) for plan PL
template <class PL, int S>
struct PlanTwCount {
    static constexpr int value = PlanTwCount<PL, S - 1>::value + PL::E / PL::R[S];
};
template <class PL>
struct PlanTwCount<PL, 0> {
    static constexpr int value = 0;
};

// base twiddles of plan PL / direction DIR for thread t, loaded once
template <class PL, int L, int DIR, class C>
struct TwPreK {
    static constexpr int N = PlanTwCount<PL, PL::NST - 1>::value;
    C w[N > 0 ? N : 1];
    __device__ __forceinline__ void load(const C* __restrict__ tw, int t) {
        fill<1>(tw, t);
    }
    template <int S>
    __device__ __forceinline__ void fill(const C* __restrict__ tw, int t) {
        if constexpr (S < PL::NST) {
            constexpr int R = PL::R[S], B = PL::E / R, NS = PlanNS<PL, S>::value;
#pragma unroll
            for (int q = 0; q < B; ++q) {
                const int jm = (t + PL::T * q) % NS;
                w[PlanTwCount<PL, S - 1>::value + q] = twiddle<DIR>(tw, jm * (L / (NS * R)));
            }
            fill<S + 1>(tw, t);
        }
    }
    template <int S>
    __device__ __forceinline__ C get(int q, int) const { return w[PlanTwCount<PL, S - 1>::value + q]; }
};

// Mirror pairs of a line held in registers (x[m] = Z[t + T m] on the T lanes
// of one warp segment, T <= 32): zk[u] = Z[k], zm[u] = Z[(L - k) mod L] for
// k = t + T u, by warp shuffles instead of a shared-memory round trip --
// (L - k) lives on lane (T - t) mod T at register E - 1 - u (lane 0: its own
// register (E - u) mod E). The r2c split of pair-packed rows needs exactly these.
template <int L, int T, int E, int KPT, class C>
__device__ __forceinline__ void mirror_pairs_shfl(const C (&x)[E], C (&zk)[KPT], C (&zm)[KPT], int t) {
    static_assert(T <= 32 && (T & (T - 1)) == 0 && T * E == L, "one power-of-two warp segment per line");
    static_assert(KPT <= E, "split outputs within the line");
    const int src = (T - t) & (T - 1);
#pragma unroll
    for (int u = 0; u < KPT; ++u) {
        zk[u] = x[u];
        C v;
        v.x = __shfl_sync(0xffffffffu, x[E - 1 - u].x, src, T);
        v.y = __shfl_sync(0xffffffffu, x[E - 1 - u].y, src, T);
        zm[u] = t == 0 ? x[(E - u) % E] : v;
    }
}

// 192-point lines with ONE shared-memory exchange (radix 12 x 16) on 16
// threads (the axis-2 rows of the 3D pass B), instead of the (12, 4, 4)
// RegPlan's two:
//   16-major layout: x[m] = element t + 16 m, m < 12, all 16 threads;
//   12-major layout: x[r] = element t + 12 r, r < 16, threads t < 12 only.
// fft192_a: 16-major in -> 12-major out (radix 12, exchange, radix 16);
// fft192_b: 12-major in -> 16-major out (radix 16, exchange, radix 12).
// Stockham stages as RegStage (w = e^{DIR 2 pi i / 192}); twiddle powers by a
// running product (~15 ulp, far inside the 1e-10 budget; 15 independent table
// loads instead measured 6 % slower on the 3D step,
// profiles/r2b_ab_fft192_twiddle_loads.log). Exchange slots:
// e + e/24 for the radix-12 stores / 12-major loads, e ^ ((e >> 4) & 7) for the
// radix-16 stores / 16-major loads (both conflict-free per quarter warp).
__device__ __forceinline__ int swz192a(int e) { return e + static_cast<int>(static_cast<unsigned>(e) / 24u); }
__device__ __forceinline__ int swz192b(int e) { return e ^ ((e >> 4) & 7); }
template <int DIR, class C>
__device__ __forceinline__ void fft192_a(C (&x)[16], C* sm, int t, const C* __restrict__ tw) {
    bfly12<DIR>(x);
#pragma unroll
    for (int k = 0; k < 12; ++k) sm[swz192a(12 * t + k)] = x[k];
    __syncwarp();
    if (t < 12) {
#pragma unroll
        for (int r = 0; r < 16; ++r) x[r] = sm[swz192a(t + 12 * r)];
        const C w1 = twiddle<DIR>(tw, t);
        C wr = w1;
#pragma unroll
        for (int r = 1; r < 16; ++r) {
            x[r] = cmul(x[r], wr);
            if (r + 1 < 16) wr = cmul(wr, w1);
        }
        bfly16<DIR>(x);
    }
    __syncwarp();
}
template <int DIR, class C>
__device__ __forceinline__ void fft192_b(C (&x)[16], C* sm, int t, const C* __restrict__ tw) {
    if (t < 12) {
        bfly16<DIR>(x);
#pragma unroll
        for (int k = 0; k < 16; ++k) sm[swz192b(16 * t + k)] = x[k];
    }
    __syncwarp();
#pragma unroll
    for (int m = 0; m < 12; ++m) x[m] = sm[swz192b(t + 16 * m)];
    const C w1 = twiddle<DIR>(tw, t);
    C wr = w1;
#pragma unroll
    for (int m = 1; m < 12; ++m) {
        x[m] = cmul(x[m], wr);
        if (m + 1 < 12) wr = cmul(wr, w1);
    }
    bfly12<DIR>(x);
    __syncwarp();
}

// In/out: x[m] = element t + T*m of the line. sm: the line's L-element buffer.
template <int L, int DIR, bool PAD = true, class C>
__device__ __forceinline__ void reg_fft(C (&x)[RegPlan<L>::E], C* sm, int t, const C* __restrict__ tw) {
    RegStage<L, DIR, 0, PAD, C>::run(x, sm, t, tw);
}
// the same over an unpadded line buffer of exactly L slots (plain XOR swizzle)
template <int L, int DIR, class C>
__device__ __forceinline__ void reg_fft_xor(C (&x)[RegPlan<L>::E], C* sm, int t, const C* __restrict__ tw) {
    RegStage<L, DIR, 0, false, C, RegPlan<L>, 0>::run(x, sm, t, tw);
}
// the same with an explicit plan (a kernel family may use another T / E split
// of the same length; the first radix must match RegPlan<L>'s for the swizzle)
template <class PL, int L, int DIR, bool PAD = true, class C>
__device__ __forceinline__ void reg_fft_p(C (&x)[PL::E], C* sm, int t, const C* __restrict__ tw) {
    static_assert(PL::R[0] == RegPlan<L>::R[0], "line-buffer swizzle follows RegPlan<L>'s first radix");
    RegStage<L, DIR, 0, PAD, C, PL>::run(x, sm, t, tw);
}
// ... with the base twiddles preloaded once per thread (TwPreK)
template <class PL, int L, int DIR, bool PAD = true, class C, class TW>
__device__ __forceinline__ void reg_fft_pw(C (&x)[PL::E], C* sm, int t, const TW& tws) {
    static_assert(PL::R[0] == RegPlan<L>::R[0], "line-buffer swizzle follows RegPlan<L>'s first radix");
    RegStage<L, DIR, 0, PAD, C, PL>::run_w(x, sm, t, tws);
}

}  // namespace slb
