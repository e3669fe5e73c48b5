// Measured fp64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput of the B200, next to
// scripts/fp64_peak.cu's DFMA figure: is the fold-batched CV scan better off on DMMA?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/dmma_peak scripts/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
__global__ void k_dmma(double *out, int iters) {
    double acc[8][2];
    for (int k = 0; k < 8; k++) { acc[k][0] = 0.0; acc[k][1] = 0.0; }
    double a = threadIdx.x * 1e-3, b = 0.999;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) dmma(acc[k], a, b);
    }
    double s = 0;
    for (int k = 0; k < 8; k++) s += acc[k][0] + acc[k][1];
    if (s == 12345.678) out[0] = s;
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *o; cudaMalloc(&o, 8);
    const int iters = 4000;
    for (int threads : {128, 256, 512}) {
        const int blocks = nsm * (1024 / threads);
        k_dmma<<<blocks, threads>>>(o, 10);
        cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_dmma<<<blocks, threads>>>(o, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fmas = (double)blocks * (threads / 32) * iters * 8 * 256;   // 8 x 8 x 4 FMAs per mma
        printf("{\"threads\": %d, \"dmma_fma_per_s\": %.4e, \"dmma_tflops\": %.3f, \"ms\": %.3f, \"err\": \"%s\"}\n", threads,
               fmas / (ms * 1e-3), 2 * fmas / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
