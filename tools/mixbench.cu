// HBM bandwidth by read:write mix (the 3D pass B moves 1 read : 2 writes).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_r1w1(const double2* __restrict__ a, double2* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        __stcg(b + i, __ldcg(a + i));
}
__global__ void k_r1w2(const double2* __restrict__ a, double2* __restrict__ b, double2* __restrict__ c, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 v = __ldcg(a + i);
        __stcg(b + i, v);
        __stcg(c + i, make_double2(v.y, v.x));
    }
}
__global__ void k_w(double2* __restrict__ b, long long n) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        __stcg(b + i, make_double2(i, 0));
}
__global__ void k_r(const double2* __restrict__ a, double2* __restrict__ out, long long n) {
    double2 s = make_double2(0, 0);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double2 v = __ldcg(a + i);
        s.x += v.x;
        s.y += v.y;
    }
    if (s.x == 12345.0) out[0] = s;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const long long n = 1LL << 26;  // 1 GiB of double2
    double2 *a, *b, *c;
    cudaMalloc(&a, n * 16);
    cudaMalloc(&b, n * 16);
    cudaMalloc(&c, n * 16);
    cudaMemset(a, 0, n * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grid = sms * 8, blk = 256;
    for (int kind = 0; kind < 4; ++kind) {
        float best = 1e30f;
        for (int rep = 0; rep < 8; ++rep) {
            cudaEventRecord(e0);
            if (kind == 0) k_r1w1<<<grid, blk>>>(a, b, n);
            if (kind == 1) k_r1w2<<<grid, blk>>>(a, b, c, n);
            if (kind == 2) k_w<<<grid, blk>>>(b, n);
            if (kind == 3) k_r<<<grid, blk>>>(a, b, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double bytes = (kind == 0 ? 2.0 : kind == 1 ? 3.0 : 1.0) * n * 16;
        const char* nm[4] = {"read1:write1", "read1:write2", "write only", "read only"};
        printf("%-14s %8.1f GB/s\n", nm[kind], bytes / best / 1e6);
    }
    return 0;
}
