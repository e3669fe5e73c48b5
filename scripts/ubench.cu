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
    extern int ring_main(void);
    return ring_main();
}

// ---------------------------------------------------------------------------
// Prefetch-ring strategies for the Gram CD step (row of nW doubles from L2 per
// step, one CTA barrier per step).  Reported: cycles per step.
constexpr int NW = 512;
__global__ void k_ring_ldg(const double *G, long long *cyc, int steps, double *sink) {
    const int t = threadIdx.x, T = blockDim.x;
    double ring[8];
#pragma unroll
    for (int i = 0; i < 8; i++) ring[i] = __ldcg(G + (size_t)i * NW + t);
    double acc = 0;
    long long t0 = clock64();
    for (int q0 = 0; q0 < steps; q0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            acc = fma(acc, 0.999, ring[u]);
            __syncthreads();
            ring[u] = __ldcg(G + (size_t)((q0 + u + 8) % 512) * NW + t);
        }
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    sink[t] = acc;
    (void)T;
}
__device__ __forceinline__ void cp_async8(void *smem, const void *gmem) {
    unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N> __device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }
__global__ void k_ring_cpasync(const double *G, long long *cyc, int steps, double *sink) {
    __shared__ double ring[8][NW];
    const int t = threadIdx.x;
#pragma unroll
    for (int i = 0; i < 8; i++) { cp_async8(&ring[i][t], G + (size_t)i * NW + t); cp_commit(); }
    double acc = 0;
    long long t0 = clock64();
    for (int q = 0; q < steps; q++) {
        cp_wait<7>();
        acc = fma(acc, 0.999, ring[q & 7][t]);
        __syncthreads();
        cp_async8(&ring[q & 7][t], G + (size_t)((q + 8) % 512) * NW + t);
        cp_commit();
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    sink[t] = acc;
}
__device__ __forceinline__ void mbar_init(unsigned long long *b, int cnt) {
    asm volatile("mbarrier.init.shared.b64 [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_expect_tx_arrive(unsigned long long *b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
                 "r"(bytes));
}
__device__ __forceinline__ void bulk_g2s(void *smem, const void *gmem, unsigned bytes, unsigned long long *b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            (unsigned)__cvta_generic_to_shared(smem)),
        "l"(gmem), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(b))
        : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n LAB_WAIT:\n"
        " mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n"
        " @!p bra LAB_WAIT;\n}\n" ::"r"((unsigned)__cvta_generic_to_shared(b)),
        "r"(phase));
}
__global__ void k_ring_bulk(const double *G, long long *cyc, int steps, double *sink) {
    __shared__ __align__(128) double ring[8][NW];
    __shared__ __align__(8) unsigned long long bar[8];
    const int t = threadIdx.x;
    if (t == 0) {
        for (int i = 0; i < 8; i++) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
    }
    __syncthreads();
    if (t == 0)
        for (int i = 0; i < 8; i++) { mbar_expect_tx_arrive(&bar[i], NW * 8); bulk_g2s(ring[i], G + (size_t)i * NW, NW * 8, &bar[i]); }
    double acc = 0;
    long long t0 = clock64();
    for (int q = 0; q < steps; q++) {
        int st = q & 7;
        mbar_wait(&bar[st], (q >> 3) & 1);
        acc = fma(acc, 0.999, ring[st][t]);
        __syncthreads();
        if (t == 0) {
            mbar_expect_tx_arrive(&bar[st], NW * 8);
            bulk_g2s(ring[st], G + (size_t)((q + 8) % 512) * NW, NW * 8, &bar[st]);
        }
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    sink[t] = acc;
}

// faithful Gram step: broadcast read -> soft threshold -> smem RMW with the ring value -> barrier
__global__ void k_gstep_ldg(const double *G, long long *cyc, int steps, double *sink) {
    __shared__ double g[2][NW];
    const int t = threadIdx.x;
    g[0][t] = t; g[1][t] = 0;
    double ring[8];
#pragma unroll
    for (int i = 0; i < 8; i++) ring[i] = __ldcg(G + (size_t)i * NW + t);
    __syncthreads();
    int cur = 0;
    long long t0 = clock64();
    for (int q0 = 0; q0 < steps; q0 += 8) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
            int q = q0 + u;
            double v = g[cur][q & (NW - 1)];
            double bn = v > 1e-3 ? v - 1e-3 : 1e-9;
            g[cur ^ 1][t] = fma(-bn, ring[u], g[cur][t]);
            __syncthreads();
            cur ^= 1;
            ring[u] = __ldcg(G + (size_t)((q + 8) % 512) * NW + t);
        }
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    sink[t] = g[cur][t];
}
__global__ void k_gstep_cp(const double *G, long long *cyc, int steps, double *sink) {
    __shared__ double g[2][NW];
    __shared__ double ring[8][NW];
    const int t = threadIdx.x;
    g[0][t] = t; g[1][t] = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) { cp_async8(&ring[i][t], G + (size_t)i * NW + t); cp_commit(); }
    __syncthreads();
    int cur = 0;
    long long t0 = clock64();
    for (int q = 0; q < steps; q++) {
        double v = g[cur][q & (NW - 1)];
        double bn = v > 1e-3 ? v - 1e-3 : 1e-9;
        cp_wait<7>();
        g[cur ^ 1][t] = fma(-bn, ring[q & 7][t], g[cur][t]);
        __syncthreads();
        cur ^= 1;
        cp_async8(&ring[q & 7][t], G + (size_t)((q + 8) % 512) * NW + t);
        cp_commit();
    }
    long long t1 = clock64();
    if (t == 0) cyc[0] = t1 - t0;
    sink[t] = g[cur][t];
}

int ring_main() {
    double *G, *sink;
    long long *cyc, h;
    cudaMalloc(&G, (size_t)512 * NW * 8);
    cudaMemset(G, 0, (size_t)512 * NW * 8);
    cudaMalloc(&sink, 8 * 1024);
    cudaMalloc(&cyc, 64);
    const int steps = 8192;
    for (int T : {128, 256, 512}) {
        k_ring_ldg<<<1, T>>>(G, cyc, steps, sink); cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("ring LDG (scoreboard)      T=%4d  %7.1f cycles/step\n", T, (double)h / steps);
        k_ring_cpasync<<<1, T>>>(G, cyc, steps, sink); cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("ring cp.async + wait_group T=%4d  %7.1f cycles/step\n", T, (double)h / steps);
        k_ring_bulk<<<1, T>>>(G, cyc, steps, sink); cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("ring bulk-TMA + mbarrier   T=%4d  %7.1f cycles/step   (%s)\n", T, (double)h / steps,
               cudaGetErrorString(cudaGetLastError()));
        k_gstep_ldg<<<1, T>>>(G, cyc, steps, sink); cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("gram step, LDG ring        T=%4d  %7.1f cycles/step\n", T, (double)h / steps);
        k_gstep_cp<<<1, T>>>(G, cyc, steps, sink); cudaDeviceSynchronize();
        cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("gram step, cp.async ring   T=%4d  %7.1f cycles/step   (%s)\n", T, (double)h / steps,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
