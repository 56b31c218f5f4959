// FP64 throughput microbenchmark (DFMA and DADD), CUDA events.
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a, double b) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) {
                x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
                x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
            } else {
                x0 = x0 + a; x1 = x1 + b; x2 = x2 + a; x3 = x3 + b; x4 = x4 + a; x5 = x5 + b; x6 = x6 + a; x7 = x7 + b;
            }
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 8 * 1024);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 4096;
    for (int op = 0; op < 2; ++op)
        for (int threads : {256, 512, 1024}) {
            const int blocks = sms * 2;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (op == 0) k<0><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
                else k<1><<<blocks, threads>>>(out, iters, 0.999999, 1e-9);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
            }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double ops = double(blocks) * threads * iters * 64;
            const double flops = ops * (op == 0 ? 2 : 1);
            printf("%s threads=%d: %.2f ms, %.2f T%s/s (%.1f ops/clk/SM at 1.965 GHz)\n", op == 0 ? "DFMA" : "DADD", threads,
                   ms, flops / ms / 1e9, op == 0 ? "FLOP" : "OP", ops / (ms * 1e-3) / sms / 1.965e9);
        }
    return 0;
}
