// Micro-benchmarks of the latencies that bound the coordinate-descent kernels
// (one coordinate update = a dependent chain of fp64 ops + a CTA barrier
// (+ a warp reduction in the residual flavour)).  Build & run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench scripts/ubench.cu && ./ubench
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double *out, long long *cyc, int iters) {
    double a = out[0], b = 1.0000001, c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) a = fma(a, b, c);
    long long t1 = clock64();
    out[1] = a;
    cyc[0] = t1 - t0;
}
__global__ void k_dadd(double *out, long long *cyc, int iters) {
    double a = out[0], c = 1e-9;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) a = a + c;
    long long t1 = clock64();
    out[1] = a;
    cyc[0] = t1 - t0;
}
__global__ void k_ffma(double *out, long long *cyc, int iters) {
    float a = (float)out[0], b = 1.0000001f, c = 1e-9f;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) a = fmaf(a, b, c);
    long long t1 = clock64();
    out[1] = a;
    cyc[0] = t1 - t0;
}
__global__ void k_bar(double *out, long long *cyc, int iters) {
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
// barrier + a dependent smem read-modify-write (the Gram CD step skeleton)
__global__ void k_bar_smem(double *out, long long *cyc, int iters) {
    __shared__ double g[2][1024];
    g[0][threadIdx.x] = threadIdx.x;
    g[1][threadIdx.x] = 0;
    __syncthreads();
    double acc = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
        int cur = i & 1;
        double v = g[cur][i & 511];              // broadcast read
        double bn = v > 1.0 ? v - 1.0 : 0.0;
        g[cur ^ 1][threadIdx.x] = fma(-bn, 1e-3, g[cur][threadIdx.x]);
        __syncthreads();
        acc += bn;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[1] = acc; }
}
__global__ void k_shfl(double *out, long long *cyc, int iters) {
    double v = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        v *= 1e-3;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[1] = v; }
}
__global__ void k_chase(const long long *next, long long *cyc, int iters, long long *sink) {
    long long p = 0;
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) p = __ldcg(next + p);
    long long t1 = clock64();
    cyc[0] = t1 - t0;
    sink[0] = p;
}

int main() {
    double *out;
    long long *cyc, *h = new long long[1];
    cudaMalloc(&out, 64);
    cudaMalloc(&cyc, 64);
    cudaMemset(out, 0, 64);
    const int it = 10000;
    auto report = [&](const char *name, int per) {
        cudaDeviceSynchronize();
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("%-40s %8.1f cycles\n", name, (double)h[0] / it / per);
    };
    k_dfma<<<1, 1>>>(out, cyc, it); report("DFMA dependent latency", 1);
    k_dadd<<<1, 1>>>(out, cyc, it); report("DADD dependent latency", 1);
    k_ffma<<<1, 1>>>(out, cyc, it); report("FFMA dependent latency", 1);
    for (int T : {32, 128, 256, 512, 1024}) {
        k_bar<<<1, T>>>(out, cyc, it);
        char b[64];
        snprintf(b, 64, "__syncthreads, %d threads", T);
        report(b, 1);
    }
    for (int T : {128, 256, 512, 1024}) {
        k_bar_smem<<<1, T>>>(out, cyc, it);
        char b[64];
        snprintf(b, 64, "gram-step skeleton, %d threads", T);
        report(b, 1);
    }
    k_shfl<<<1, 32>>>(out, cyc, it); report("fp64 warp_sum (5 levels) + DMUL", 1);
    // pointer chase over 8 MB (L2) and 1 GB (HBM)
    for (long long bytes : {8LL << 20, 1LL << 30}) {
        long long n = bytes / 8;
        long long *hn = new long long[n];
        long long stride = 4099;                // jump across lines
        for (long long i = 0; i < n; i++) hn[i] = (i + stride * 16) % n;
        long long *dn;
        cudaMalloc(&dn, bytes);
        cudaMemcpy(dn, hn, bytes, cudaMemcpyHostToDevice);
        k_chase<<<1, 1>>>(dn, cyc, 2000, cyc + 2);   // warm
        k_chase<<<1, 1>>>(dn, cyc, it, cyc + 2);
        char b[64];
        snprintf(b, 64, "dependent LDG.cg latency, %lld MB", bytes >> 20);
        report(b, 1);
        cudaFree(dn);
        delete[] hn;
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SM clock attribute: %d kHz\n", clk);
    return 0;
}
