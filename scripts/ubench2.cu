// Warp-wide fp64 latency/throughput and a replica of the blocked-CD warp step.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma_warp(double *out, long long *cyc, int iters) {
    double a = out[threadIdx.x & 7], b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) a = fma(a, b, c);
    long long t1 = clock64();
    out[8 + threadIdx.x] = a;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void k_shfl_bcast(double *out, long long *cyc, int iters) {
    double v = out[threadIdx.x & 7];
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) v = __shfl_sync(0xffffffffu, v, i & 31) + 1e-9;
    long long t1 = clock64();
    out[8 + threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__device__ __forceinline__ double soft(double z, double g) { return z > g ? z - g : (z < -g ? z + g : 0.0); }
__global__ void k_phaseb(double *out, long long *cyc, int iters, double la, double inv) {
    const int lane = threadIdx.x & 31;
    double gv = out[lane & 7] + lane, bv = 0.0, Gs[32];
#pragma unroll
    for (int b = 0; b < 32; b++) Gs[b] = 1e-3 * (b + lane);
    long long t0 = clock64();
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int bp = 0; bp < 32; bp++) {
            const double zb = __shfl_sync(0xffffffffu, gv + bv, bp);
            const double bo = __shfl_sync(0xffffffffu, bv, bp);
            const double bn = soft(zb, la) * inv;
            const double d = bn - bo;
            if (d != 0.0) {
                if (lane > bp) gv = fma(-d, Gs[bp], gv);
                if (lane == bp) bv = bn;
            }
        }
    }
    long long t1 = clock64();
    out[8 + threadIdx.x] = gv + bv;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double *out; long long *cyc, h;
    cudaMalloc(&out, 8 * 2048); cudaMalloc(&cyc, 64); cudaMemset(out, 0, 8 * 2048);
    const int it = 4096;
    for (int T : {1, 32, 128, 512}) {
        k_dfma_warp<<<1, T>>>(out, cyc, it); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("dependent DFMA chain, %4d threads: %6.1f cycles/op\n", T, (double)h / it);
    }
    k_shfl_bcast<<<1, 32>>>(out, cyc, it); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("shfl(double) broadcast + DADD chain: %6.1f cycles/step\n", (double)h / it);
    k_phaseb<<<1, 32>>>(out, cyc, 128, 1e-4, 1.0); cudaDeviceSynchronize(); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("phase-B replica: %6.1f cycles/coordinate\n", (double)h / (128 * 32));
    return 0;
}
