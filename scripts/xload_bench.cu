// Micro-benchmark: HBM read rate of the tcgen05 scan's X access pattern (a CTA streams a tile of
// 128 columns; each of 16 warps owns 32 columns x RT rows of every stage, one 32-byte load per
// lane per 8 rows), by rows per stage and register prefetch depth.  No conversion, no MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 scripts/xload_bench.cu -o /tmp/xload
#include <cstdio>
#include <cstdint>

template <int RT, int PD>   // RT rows per thread per stage (multiple of 8), PD stages of loads in flight
__global__ void __launch_bounds__(512, 1) k_load(const float *__restrict__ X, int64_t ld, int n, int64_t p, float *out) {
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int qq = w & 3, h = w >> 2;                 // 4 column quarters x 4 row groups
    constexpr int SR = 4 * RT;                        // rows per stage
    const int nst = (n + SR - 1) / SR;
    const int64_t ntiles = (p + 127) / 128;
    float acc = 0.f;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int64_t j = min(t * 128 + 32 * qq + lane, p - 1);
        const float *xc = X + j * ld + RT * h;
        float r[PD][RT];
        auto load = [&](float (&v)[RT], int s) {
#pragma unroll
            for (int i = 0; i < RT; i += 8) {
                const int64_t row = (int64_t)s * SR + RT * h + i;
                if (s < nst && row < ld)
                    asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                        : "=f"(v[i]), "=f"(v[i + 1]), "=f"(v[i + 2]), "=f"(v[i + 3]), "=f"(v[i + 4]), "=f"(v[i + 5]),
                          "=f"(v[i + 6]), "=f"(v[i + 7])
                        : "l"(xc + (int64_t)s * SR + i));
                else
                    for (int u = 0; u < 8; u++) v[i + u] = 0.f;
            }
        };
#pragma unroll
        for (int d = 0; d < PD - 1; d++) load(r[d], d);
        for (int s = 0; s < nst; s += PD) {
#pragma unroll
            for (int d = 0; d < PD; d++) {
                load(r[(d + PD - 1) % PD], s + d + PD - 1);
#pragma unroll
                for (int i = 0; i < RT; i++) acc += r[d][i];
            }
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

template <int RT, int PD>
void run(const float *X, int64_t ld, int n, int64_t p, float *o) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_load<RT, PD><<<148, 512>>>(X, ld, n, p, o);
    float best = 1e9f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(a);
        k_load<RT, PD><<<148, 512>>>(X, ld, n, p, o);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    printf("rows/thread/stage %3d (stage %4d rows), %d stages in flight: %.3f ms = %.0f GB/s  %s\n", RT, 4 * RT, PD, best,
           (double)n * p * 4 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    const int n = 10000;
    const int64_t ld = 10000, p = 200000;
    float *X, *o;
    cudaMalloc(&X, sizeof(float) * ld * p);
    cudaMemset(X, 0, sizeof(float) * ld * p);
    cudaMalloc(&o, 4);
    run<16, 2>(X, ld, n, p, o);
    run<16, 3>(X, ld, n, p, o);
    run<16, 4>(X, ld, n, p, o);
    run<32, 2>(X, ld, n, p, o);
    run<32, 3>(X, ld, n, p, o);
    run<64, 2>(X, ld, n, p, o);
    return 0;
}
