// Micro-benchmark of the sequential 32-coordinate chain of the Gram CD block
// step, in isolation (one warp, data in shared memory).  Variants:
//   A  one thread, z[32] in registers, fully unrolled triangular updates
//   B  lane-parallel: lane c holds z_c; rolled loop over b, d broadcast by shfl
//   C  like B but the broadcast goes through shared memory
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/chain_bench scripts/chain_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double st_d(double zb, double bo, double la, double &bn) {
    const double bn1 = zb - la, bn2 = zb + la;
    const double d1 = bn1 - bo, d2 = bn2 - bo;
    const bool hi = zb > la, lo = zb < -la;
    bn = hi ? bn1 : (lo ? bn2 : 0.0);
    return hi ? d1 : (lo ? d2 : -bo);
}

template <int V>
__global__ void k_chain(const double *Gin, const double *zin, double *out, long long *cyc, int reps, double la) {
    __shared__ __align__(16) double Gd[32][32];
    __shared__ __align__(16) double zsh[32], bsh[32], dsh[32], bnsh[32];
    const int lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) Gd[e >> 5][e & 31] = Gin[e];
    if (threadIdx.x < 32) { zsh[lane] = zin[lane]; bsh[lane] = 0.0; }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    double acc = 0.0;
    long long t0 = clock64();
    for (int r = 0; r < reps; r++) {
        if (V == 0) {
            if (lane == 0) {
                double z[32];
#pragma unroll
                for (int b = 0; b < 32; b += 2) {
                    const double2 v = *reinterpret_cast<const double2 *>(zsh + b);
                    z[b] = v.x; z[b + 1] = v.y;
                }
#pragma unroll
                for (int b = 0; b < 32; b++) {
                    double bn;
                    const double d = st_d(z[b], bsh[b], la, bn);
                    dsh[b] = d;
                    bnsh[b] = bn;
#pragma unroll
                    for (int c = (b + 1) & ~1; c < 32; c += 2) {
                        const double2 gv = *reinterpret_cast<const double2 *>(&Gd[b][c]);
                        if (c > b) z[c] = fma(-d, gv.x, z[c]);
                        z[c + 1] = fma(-d, gv.y, z[c + 1]);
                    }
                }
            }
            __syncwarp();
            acc += dsh[lane];
            __syncwarp();
        } else if (V == 1) {
            double z = zsh[lane], bo = bsh[lane], keep = 0.0, dk = 0.0;
            double g = Gd[0][lane];
#pragma unroll 1
            for (int b = 0; b < 32; b++) {
                const double gn = Gd[(b + 1) & 31][lane];     // next row, off the chain
                double bn;
                const double dl = st_d(z, bo, la, bn);
                const double d = __shfl_sync(0xffffffffu, dl, b);
                if (lane == b) { keep = bn; dk = d; }
                z = fma(-d, g, z);
                g = gn;
            }
            acc += dk + keep;
        } else {
            double z = zsh[lane], bo = bsh[lane], keep = 0.0, dk = 0.0;
            double g = Gd[0][lane];
#pragma unroll 1
            for (int b = 0; b < 32; b++) {
                const double gn = Gd[(b + 1) & 31][lane];
                double bn;
                const double dl = st_d(z, bo, la, bn);
                if (lane == b) { dsh[b] = dl; keep = bn; dk = dl; }
                __syncwarp();
                const double d = dsh[b];
                z = fma(-d, g, z);
                g = gn;
            }
            acc += dk + keep;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
    out[threadIdx.x] = acc;
}

int main() {
    double hG[1024], hz[32];
    for (int i = 0; i < 32; i++) {
        hz[i] = 0.3 * ((i * 37) % 11 - 5);
        for (int j = 0; j < 32; j++) hG[i * 32 + j] = i == j ? 1.0 : 0.01 * (((i + 3) * (j + 7)) % 13 - 6);
    }
    double *G, *z, *o;
    long long *c;
    cudaMalloc(&G, 8192); cudaMalloc(&z, 256); cudaMalloc(&o, 8192); cudaMalloc(&c, 8);
    cudaMemcpy(G, hG, 8192, cudaMemcpyHostToDevice);
    cudaMemcpy(z, hz, 256, cudaMemcpyHostToDevice);
    const int reps = 200;
    const char *nm[3] = {"A single-thread unrolled", "B lane-parallel shfl   ", "C lane-parallel smem   "};
    for (int threads : {32, 256}) {
        for (int v = 0; v < 3; v++) {
            long long h;
            for (int w = 0; w < 2; w++) {
                if (v == 0) k_chain<0><<<1, threads>>>(G, z, o, c, reps, 0.1);
                if (v == 1) k_chain<1><<<1, threads>>>(G, z, o, c, reps, 0.1);
                if (v == 2) k_chain<2><<<1, threads>>>(G, z, o, c, reps, 0.1);
                cudaDeviceSynchronize();
            }
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            printf("%s threads=%3d  %.1f cycles/block  %.1f cycles/coordinate (%s)\n", nm[v], threads,
                   (double)h / reps, (double)h / reps / 32, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
