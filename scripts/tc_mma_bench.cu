// Micro-benchmark: tcgen05.mma kind::i8 issue rate (M = 128, cta_group::1) by smem layout and N,
// operands static in shared memory (contents irrelevant), one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1701_05936_b200/csrc \
//        scripts/tc_mma_bench.cu -o /tmp/tc_mma_bench
#include "bl_tc.cuh"

#include <cstdio>

using namespace bl;

__device__ __forceinline__ void tc_mma(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
__host__ __device__ constexpr uint32_t tc_idesc(int N, bool s) { return tc_idesc(128, N, s); }

// layout: 0 no swizzle (LBO 128, SBO 512, 64-byte K rows in 8x16 core matrices), 1 SWIZZLE_64B (rows of
// 64 bytes, SBO 512), 2 SWIZZLE_128B (rows of 128 bytes, SBO 1024)
__device__ __forceinline__ uint64_t mk_desc(uint32_t saddr, int layout) {
    uint64_t d = (uint64_t)((saddr & 0x3FFFFu) >> 4) | (1ull << 46);
    if (layout == 0) d |= ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32);
    if (layout == 1) d |= ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) | (4ull << 61);
    if (layout == 2) d |= ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) | (2ull << 61);
    return d;
}

__device__ __forceinline__ void mma_f16(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
template <int N, int KIND, int M>
__global__ void __launch_bounds__(128, 1) k_bench(int iters, int layout, int per_commit, long long *out) {
    extern __shared__ uint8_t sm_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tsh;
    const int wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tsh)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tsh;
    if (threadIdx.x == 0) {
        const uint32_t base = smem_addr(sm);
        uint32_t ids = tc_idesc(N, true);
        ids = (ids & ~(0x1Fu << 24)) | ((uint32_t)(M >> 4) << 24);
        if (KIND == 1) ids = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; it++) {
            for (int q = 0; q < per_commit; q++) {
                // A: 6 planes of 128 rows, B: N rows; K step of 32 bytes
                const int ks = q & 1, a = (q >> 1) % 6;
                uint32_t aoff, boff;
                if (layout == 0) { aoff = a * 8192 + 256 * ks; boff = 49152 + 256 * ks; }
                else if (layout == 1) { aoff = a * 8192 + 32 * ks; boff = 49152 + 32 * ks; }
                else { aoff = (a % 3) * 16384 + 32 * ks; boff = 49152 + 32 * ks; }
                const uint32_t dt = tmem + (uint32_t)((a % (480 / N)) * N);
                if (KIND == 0) tc_mma(dt, mk_desc(base + aoff, layout), mk_desc(base + boff, layout), ids, q != 0);
                else mma_f16(dt, mk_desc(base + aoff, layout), mk_desc(base + boff, layout), ids, q != 0);
            }
            tc_commit(&bar);
            mbar_wait(&bar, ph);
            ph ^= 1;
        }
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (wid == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

template <int N, int KIND = 0, int M = 128>
void run(int layout, int per_commit) {
    long long *d, h;
    cudaMalloc(&d, 8);
    const int iters = 2000;
    const size_t smem = 65536 + 1024;
    cudaFuncSetAttribute(k_bench<N, KIND, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench<N, KIND, M><<<148, 128, smem>>>(10, layout, per_commit, d);
    k_bench<N, KIND, M><<<148, 128, smem>>>(iters, layout, per_commit, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / iters / per_commit;
    const int K = KIND == 0 ? 32 : 16;
    printf("%s M=%d N=%3d layout=%d mmas/commit=%2d: %.1f cycles per MMA = %.0f MAC/clk  %s\n", KIND ? "f16" : "i8 ", M, N,
           layout, per_commit, per, (double)M * N * K / per, cudaGetErrorString(e));
    cudaFree(d);
}

int main2();
int main(int argc, char **argv) {
    if (argc > 1) return main2();
    for (int layout = 0; layout < 2; layout++) {
        run<16>(layout, 48);
        run<64>(layout, 48);
        run<80>(layout, 48);
        run<128>(layout, 48);
        run<256>(layout, 48);
        run<80, 1>(layout, 48);
        run<256, 1>(layout, 48);
        run<80, 0, 64>(layout, 48);
        run<256, 0, 64>(layout, 48);
    }
    return 0;
}

// ---- cta_group::2 (M = 256 over an SM pair): per-instruction cost
__device__ __forceinline__ void mma_i8_2sm(uint32_t dtmem, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n"
        ::"r"(dtmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc));
}
template <int N, int TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(640, 1) k_bench2(int iters, int per_commit, long long *out) {
    __shared__ volatile int stop;
    extern __shared__ uint8_t sm_raw[];
    uint8_t *sm = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm_raw) + 1023) & ~(uintptr_t)1023);
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tsh;
    const int wid = threadIdx.x >> 5;
    unsigned rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    for (int i = threadIdx.x; i < 65536; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (threadIdx.x == 0) {
        stop = 0;
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (wid == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tsh)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    cluster_arrive();
    cluster_wait();
    tc_fence_after();
    const uint32_t tmem = tsh;
    if (wid >= 4 && out[1] != 0) {                  // store traffic: 16 warps, STS.32 into [64 KB, 112 KB)
        uint32_t *w = reinterpret_cast<uint32_t *>(sm + 65536);
        uint32_t v = threadIdx.x;
        int k = 0;
        const long long tend = clock64() + (long long)iters * per_commit * 180;
        if (out[1] == 1) {
            while (clock64() < tend) {
#pragma unroll 8
                for (int u = 0; u < 64; u++) { w[((k + u) * 512 + threadIdx.x - 128) % 12288] = v; v += 3; }
                k += 64;
            }
        } else {                                  // tcgen05.st traffic: x4 stores into columns 352 .. 447
            const uint32_t tl = tmem + ((uint32_t)(32 * (wid & 3)) << 16) + 352;
            while (clock64() < tend) {
#pragma unroll 4
                for (int u = 0; u < 24; u++) tc_st4(tl + 4 * u, v, v + 1, v + 2, v + 3);
                tc_wait_st();
                v += 7;
            }
        }
    }
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t base = smem_addr(sm);
        uint32_t ids = tc_idesc(N, true);
        ids = (ids & ~(0x1Fu << 24)) | ((uint32_t)(256 >> 4) << 24);
        long long t0 = clock64();
        uint32_t ph = 0;
        for (int it = 0; it < iters; it++) {
#pragma unroll 12
            for (int q = 0; q < per_commit; q++) {
                const int ks = q & 1, a = (q >> 1) % 6;
                const uint32_t aoff = a * 8192 + 256 * ks, boff = 49152 + 256 * ks;
                if (TS == 0)
                    mma_i8_2sm(tmem + (uint32_t)((a % (480 / N)) * N), mk_desc(base + aoff, 0), mk_desc(base + boff, 0), ids, q != 0);
                else   // A from TMEM columns 256 + 16 a + 8 ks, D in [0, 2N)
                    tc_mma2_ts(tmem + (uint32_t)((a / 3) * N), tmem + 256 + 16 * (a % 6) + 8 * ks, mk_desc(base + boff, 0), ids,
                               q != 0);
            }
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_addr(&bar)), "h"((uint16_t)3) : "memory");
            mbar_wait(&bar, ph);
            ph ^= 1;
        }
        long long t1 = clock64();
        if (blockIdx.x == 0) out[0] = t1 - t0;
    }
    __syncthreads();
    tc_fence_before();
    cluster_arrive();
    cluster_wait();
    if (wid == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}
template <int N, int ts = 0>
void run2(int per_commit, int sts) {
    long long *d, h;
    cudaMalloc(&d, 24);
    long long init[3] = {0, sts, ts};
    cudaMemcpy(d, init, 24, cudaMemcpyHostToDevice);
    const int iters = 2000;
    const size_t smem = 65536 + 65536 + 1024;
    cudaFuncSetAttribute(k_bench2<N, ts>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_bench2<N, ts><<<148, 640, smem>>>(10, per_commit, d);
    k_bench2<N, ts><<<148, 640, smem>>>(iters, per_commit, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double per = (double)h / iters / per_commit;
    printf("A=%s sts=%d per_commit=%d i8 cta_group::2 M=256 N=%3d: %.1f cycles per MMA = %.0f MAC/clk per SM  %s\n",
           ts ? "tmem" : "smem", sts, per_commit, N, per, 128.0 * N * 32 / per,
           cudaGetErrorString(e));
    cudaFree(d);
}
int main2() {
    run2<80>(48, 0);
    run2<96>(48, 0);
    run2<96>(12, 0);
    run2<96, 1>(48, 0);
    run2<96, 1>(12, 0);
    run2<96, 1>(48, 1);
    run2<96, 1>(48, 2);
    run2<96, 1>(12, 2);
    run2<160, 1>(48, 0);
    run2<256, 1>(48, 0);
    return 0;
}
