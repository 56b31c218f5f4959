// L2 / HBM copy bandwidth and FFT-512 compute-only throughput microbenchmarks.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1402_5670_b200/csrc/fft_reg.cuh"
using namespace slb;

__global__ void copy_k(const double2* __restrict__ a, double2* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        __stcg(b + i, __ldcg(a + i));
}

template <int L>
__global__ void fft_only(double2* out, int iters, const double2* __restrict__ tw) {
    constexpr int T = RegPlan<L>::T, E = RegPlan<L>::E;
    extern __shared__ double2 sm[];
    const int li = threadIdx.x / T, t = threadIdx.x % T;
    double2 x[E];
    for (int m = 0; m < E; ++m) x[m] = make_double2(t + m, m);
    for (int i = 0; i < iters; ++i) reg_fft<L, -1>(x, sm + li * L, t, tw);
    double2 s = make_double2(0, 0);
    for (int m = 0; m < E; ++m) s = cadd(s, x[m]);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (long long mb : {8LL, 32LL, 64LL, 96LL, 1024LL}) {
        long long n = mb * 1024 * 1024 / 16;
        double2 *a, *b;
        cudaMalloc(&a, n * 16);
        cudaMalloc(&b, n * 16);
        cudaMemset(a, 0, n * 16);
        for (int r = 0; r < 3; ++r) copy_k<<<sms * 8, 256>>>(a, b, n);
        cudaEventRecord(e0);
        const int reps = 20;
        for (int r = 0; r < reps; ++r) copy_k<<<sms * 8, 256>>>(a, b, n);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("copy %lld MB: %.1f GB/s (read+write)\n", mb, 2.0 * n * 16 * reps / (ms * 1e-3) / 1e9);
        cudaFree(a);
        cudaFree(b);
    }
    // FFT-512 compute only
    double2* tw;
    cudaMalloc(&tw, 512 * 16);
    double2 h[512];
    for (int k = 0; k < 512; ++k) h[k] = make_double2(cos(-2 * M_PI * k / 512), sin(-2 * M_PI * k / 512));
    cudaMemcpy(tw, h, sizeof(h), cudaMemcpyHostToDevice);
    double2* out;
    cudaMalloc(&out, 1 << 26);
    for (int lines : {2, 4, 8}) {
        constexpr int T = RegPlan<512>::T;
        const int threads = lines * T;
        const size_t smem = lines * 512 * 16;
        cudaFuncSetAttribute(fft_only<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        for (int blocks : {sms * 2, sms * 4, sms * 8}) {
            const int iters = 200;
            fft_only<512><<<blocks, threads, smem>>>(out, 10, tw);
            cudaEventRecord(e0);
            fft_only<512><<<blocks, threads, smem>>>(out, iters, tw);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double ffts = double(blocks) * lines * iters;
            const double flops = ffts * 5.0 * 512 * 9;
            printf("fft512 lines/cta=%d blocks=%d: %.3f ms, %.2f M fft/s, %.1f TFLOP/s (5NlogN), %.0f clk/fft/SM  err=%s\n", lines,
                   blocks, ms, ffts / ms / 1e3, flops / ms / 1e9, (ms * 1e-3 * 1.965e9 * sms) / ffts,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
