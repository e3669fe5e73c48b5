// Micro-benchmark of cross-CTA synchronisation inside a thread-block cluster
// (one step of the cluster CD = leader -> owners -> leader hand-off):
//   A  barrier.cluster.arrive.release + wait.acquire, all threads
//   B  cg::cluster_group::sync()
//   C  flag ping-pong: leader stores a sequence number into every owner's smem
//      (st.release.cluster), owners spin on it (ld.acquire.cluster), then each
//      owner stores its ack into the leader's smem; one thread per CTA.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/cluster_bench scripts/cluster_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__device__ __forceinline__ void st_rel(unsigned *p, unsigned v) {
    asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acq(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory");
    return v;
}
__device__ __forceinline__ unsigned mapa(const void *p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_rel_remote(unsigned addr, unsigned v) {
    asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

template <int V>
__global__ void k_sync(long long *cyc, int iters, const double *G) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ unsigned flag;               // owners: sequence from the leader
    __shared__ unsigned acks[16];           // leader: per-owner acks
    __shared__ double pub[2][32], loc[32], gl[512];
    long long arr = 0;
    double2 rv[8];
    for (int i = 0; i < 8; i++) rv[i] = make_double2(0, 0);
    const int rank = cl.block_rank(), R = cl.num_blocks();
    if (threadIdx.x < 16) acks[threadIdx.x] = 0;
    if (threadIdx.x == 0) flag = 0;
    for (int k = threadIdx.x; k < 512; k += blockDim.x) gl[k] = 0;
    cl.sync();
    if (V >= 3) asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    long long t0 = clock64();
    for (int i = 1; i <= iters; i++) {
        if (V == 0) {
            asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
            asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        } else if (V == 1) {
            cl.sync();
        } else if (V >= 3) {
            // D: owners pull 32 doubles from the leader, apply, store; E: + global prefetch after arrive
            asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
            if (rank == 0) {
                if (threadIdx.x < 32) pub[i & 1][threadIdx.x] = i + threadIdx.x;
            } else {
                if (threadIdx.x < 32) loc[threadIdx.x] = cl.map_shared_rank(&pub[0][0], 0)[((i - 1) & 1) * 32 + threadIdx.x];
                __syncthreads();
                double acc = gl[threadIdx.x];
                for (int k = 0; k < 8; k++) acc += loc[k] * rv[k].x;
                gl[threadIdx.x] = acc;
                __syncthreads();
            }
            long long a0 = clock64();
            asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
            arr += clock64() - a0;
            if (V == 4 && rank > 0)
                for (int k = 0; k < 8; k++) rv[k] = __ldcg(reinterpret_cast<const double2 *>(G + (size_t)(k * 1024 + 2 * threadIdx.x)));
            if (i == iters) asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
        } else {
            if (rank == 0) {
                if (threadIdx.x > 0 && threadIdx.x < R) st_rel_remote(mapa(&flag, threadIdx.x), (unsigned)i);
                if (threadIdx.x > 0 && threadIdx.x < R) { while (ld_acq(&acks[threadIdx.x]) < (unsigned)i) {} }
                __syncthreads();
            } else {
                if (threadIdx.x == 0) {
                    while (ld_acq(&flag) < (unsigned)i) {}
                    st_rel_remote(mapa(&acks[rank], 0), (unsigned)i);
                }
                __syncthreads();
            }
        }
    }
    long long t1 = clock64();
    if (rank == 0 && threadIdx.x == 0) cyc[0] = t1 - t0;
    if (rank == 1 && threadIdx.x == 0) cyc[1] = arr;
    if (gl[threadIdx.x] == 12345.0) cyc[2] = 1;
    cl.sync();
}

int main() {
    long long *c;
    cudaMalloc(&c, 64);
    double *G;
    cudaMalloc(&G, 8 << 20);
    cudaMemset(G, 0, 8 << 20);
    const char *nm[5] = {"barrier.cluster arrive/wait", "cg cluster.sync           ", "flag ping-pong (DSMEM)    ",
                         "D pull+apply+arrive/wait  ", "E D + global prefetch     "};
    for (int R : {2, 4, 8, 16}) {
        for (int v = 0; v < 5; v++) {
            const void *k = v == 0 ? (const void *)k_sync<0> : v == 1 ? (const void *)k_sync<1> : v == 2 ? (const void *)k_sync<2>
                          : v == 3 ? (const void *)k_sync<3> : (const void *)k_sync<4>;
            if (R > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            int iters = 2000;
            void *args[] = {&c, &iters, &G};
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(R);
            cfg.blockDim = dim3(256);
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = R; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            for (int w = 0; w < 2; w++) cudaLaunchKernelExC(&cfg, k, args);
            cudaDeviceSynchronize();
            long long h[2] = {0, 0};
            cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
            printf("R=%2d %s %.1f cycles/step  arrive(owner) %.1f (%s)\n", R, nm[v], (double)h[0] / iters, v >= 3 ? (double)h[1] / iters : 0.0,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
