// Microbenchmark: issue/throughput of scalar FFMA vs packed FFMA2 (sm_100a) with 8
// independent chains per thread; prints Gop/s (FMA = 1 op per lane-component).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float *out, int iters) {
    float a[8];
    for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3f + j;
    const float b = 0.999f, c = 1e-4f;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
    float s = 0;
    for (int j = 0; j < 8; ++j) s += a[j];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_ffma2(float *out, int iters) {
    float2 a[4];
    for (int j = 0; j < 4; ++j) a[j] = make_float2(threadIdx.x * 1e-3f + 2 * j, threadIdx.x * 1e-3f + 2 * j + 1);
    const float2 b = make_float2(0.999f, 0.999f), c = make_float2(1e-4f, 1e-4f);
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int j = 0; j < 4; ++j) a[j] = __ffma2_rn(a[j], b, c);
    float s = 0;
    for (int j = 0; j < 4; ++j) s += a[j].x + a[j].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    float *out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(float));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 16, blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        cudaEventRecord(e0);
        k_ffma<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * iters * 8;
        printf("FFMA : %.3f ms  %.1f Gfma/s\n", ms, ops / ms / 1e6);
        cudaEventRecord(e0);
        k_ffma2<<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA2: %.3f ms  %.1f Gfma/s\n", ms, ops / ms / 1e6);
    }
    return 0;
}
