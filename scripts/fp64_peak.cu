// Measured fp64 FMA throughput of the B200 (the ALU roofline of the fold-batched scan):
// every SM at full occupancy, 8 independent DFMA chains per thread.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/fp64_peak scripts/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double *out, int iters) {
    double a[8];
    for (int k = 0; k < 8; k++) a[k] = threadIdx.x * 1e-3 + k;
    const double b = 0.999999, c = 1e-7;
    for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < 8; k++) a[k] = fma(a[k], b, c);
    double s = 0;
    for (int k = 0; k < 8; k++) s += a[k];
    if (s == 12345.678) out[0] = s;
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    double *o; cudaMalloc(&o, 8);
    const int iters = 20000, threads = 512, blocks = nsm * 4;
    k_dfma<<<blocks, threads>>>(o, 100);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)blocks * threads * iters * 8;
    printf("{\"fp64_fma_per_s\": %.4e, \"fp64_tflops\": %.3f, \"ms\": %.3f}\n", fmas / (ms * 1e-3), 2 * fmas / (ms * 1e-3) / 1e12, ms);
    return 0;
}
