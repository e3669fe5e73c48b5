// Stand-alone timing of the Gram CD kernels (bl_kernels.cuh) on synthetic data:
// nW slots, G = I + small symmetric noise, every coordinate active, a fixed
// number of passes.  Prints SM cycles per coordinate visit for the blocked
// warp-chain kernel (v5) and the pipelined single-thread-chain kernel (v6), and
// the largest coefficient difference between the two (same cyclic order).
// Build on the CPU box, run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1701_05936_b200/csrc -I scripts -o scripts/cd_bench scripts/cd_bench.cu
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "bl_kernels.cuh"
#include "gram6_ref.cuh"
using namespace bl;

std::vector<double> run(int ver, int nW, int passes_wanted, double lam, int R = 8) {
    int ldG = (nW + 31) / 32 * 32;
    std::vector<double> G((size_t)ldG * ldG, 0.0), z(nW), beta(nW, 0.0), c(nW, 0.0), s(nW, 1.0);
    srand(1);
    for (int i = 0; i < nW; i++) {
        G[(size_t)i * ldG + i] = 1.0;
        for (int j = 0; j < i; j++) {
            double v = 0.02 * ((rand() / (double)RAND_MAX) - 0.5);
            G[(size_t)i * ldG + j] = G[(size_t)j * ldG + i] = v;
        }
        z[i] = (rand() / (double)RAND_MAX) - 0.5;
    }
    std::vector<int> Wst(nW), ord(nW);
    for (int i = 0; i < nW; i++) Wst[i] = ord[i] = i;
    double *dG, *dz, *dbeta, *ddb, *dbw, *dc, *ds;
    int *dW, *dord;
    RoundStatus *dst;
    cudaMalloc(&dG, 8 * G.size());
    cudaMalloc(&dz, 8 * nW); cudaMalloc(&dbeta, 8 * nW); cudaMalloc(&ddb, 8 * nW); cudaMalloc(&dbw, 24 * nW);
    cudaMalloc(&dc, 8 * nW); cudaMalloc(&ds, 8 * nW); cudaMalloc(&dW, 4 * nW); cudaMalloc(&dord, 4 * nW);
    cudaMalloc(&dst, sizeof(RoundStatus));
    double *dGA;
    cudaMalloc(&dGA, 8 * G.size() + 8 * 32 * (size_t)ldG + 8 * 4 * (size_t)ldG + 64);
    G7Work wk;
    wk.g = dGA + G.size() + 32 * (size_t)ldG;
    wk.dl = wk.g + ldG;
    wk.act = reinterpret_cast<int *>(wk.dl + ldG);
    wk.rl = wk.act + ldG;
    wk.inA = reinterpret_cast<uint8_t *>(wk.rl + ldG);
    cudaMemcpy(dG, G.data(), 8 * G.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dz, z.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dbeta, beta.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, c.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, s.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, Wst.data(), 4 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dord, ord.data(), 4 * nW, cudaMemcpyHostToDevice);
    CdGramArgs a{};
    a.Wst = dW; a.ord = dord; a.nW = nW; a.ldG = ldG; a.G = dG; a.z = dz; a.beta = dbeta; a.dbeta = ddb;
    a.lam_alpha = lam; a.inv_den = 1.0; a.tol = 0.0; a.floor_ = 0.0; a.max_iter = passes_wanted;
    a.betaW_out = dbw; a.c = dc; a.s = ds; a.st = dst;
    a.GA = dGA; a.MA = dGA + G.size();
    int nWp = (nW + 1) & ~1;
    size_t smem = (size_t)24 * nWp + 16;
    if (ver == 6) {
        cudaFuncSetAttribute(k_cd_gram6<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        k_cd_gram6<false><<<1, kGram6Threads, gram6_smem(nW)>>>(a);
    } else {
        const void *kern = R == 4 ? (const void *)k_cd_gram7<false, 4> : R == 16 ? (const void *)k_cd_gram7<false, 16>
                                                                               : (const void *)k_cd_gram7<false, 8>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        if (R > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        void *args[] = {&a, &wk};
        cudaError_t e = cudaLaunchKernel(kern, dim3(R), dim3(kG7Threads), args, gram7_smem(nW, R), 0);
        if (e != cudaSuccess) printf("launch: %s\n", cudaGetErrorString(e));
    }
    cudaDeviceSynchronize();
    RoundStatus h;
    cudaMemcpy(&h, dst, sizeof h, cudaMemcpyDeviceToHost);
    std::vector<double> out(nW);
    cudaMemcpy(out.data(), dbw, 8 * nW, cudaMemcpyDeviceToHost);
    printf("v%d R=%2d nW=%5d passes=%d visits=%lld updates=%lld  cycles/visit=%.1f  lead %.1f bulk %.1f build %.1f catch %.1f | retries %lld rebuilds %lld catchups %lld full %lld (%s)\n",
           ver, ver == 7 ? R : 1, nW, h.cd_passes, h.cd_visits, h.cd_updates, (double)h.cd_cycles / h.cd_visits,
           (double)h.cd_prof[0] / h.cd_visits, (double)h.cd_prof[1] / h.cd_visits, (double)h.cd_prof[2] / h.cd_visits,
           (double)h.cd_prof[3] / h.cd_visits, h.cd_cnt[0], h.cd_cnt[1], h.cd_cnt[2], h.cd_cnt[3],
           cudaGetErrorString(cudaGetLastError()));
    if (ver == 7) {
        printf("      leader (cycles/visit): zc %.1f  M %.1f  FS %.1f  tail %.1f | wait snap+stage %.1f | link wait %.1f  link %.1f\n",
               (double)h.cd_dbg[0] / h.cd_visits, (double)h.cd_dbg[1] / h.cd_visits, (double)h.cd_dbg[2] / h.cd_visits,
               (double)h.cd_dbg[3] / h.cd_visits, (double)h.cd_dbg[4] / h.cd_visits, (double)h.cd_dbg[5] / h.cd_visits,
               (double)h.cd_dbg[6] / h.cd_visits);
    }
    cudaFree(dG); cudaFree(dz); cudaFree(dbeta); cudaFree(ddb); cudaFree(dbw); cudaFree(dc); cudaFree(ds);
    cudaFree(dW); cudaFree(dord); cudaFree(dst); cudaFree(dGA);
    return out;
}

int main() {
    const int sizes[] = {64, 200, 600, 1000, 1500, 2500, 4000};
    const int passes[] = {200, 60, 30, 20, 12, 8, 6};
    for (int u = 0; u < 7; u++) {
        for (double lam : {1e-6, 0.2}) {
            auto b6 = run(6, sizes[u], passes[u], lam);
            for (int R : {8}) {
                auto b7 = run(7, sizes[u], passes[u], lam, R);
                double md = 0.0, mb = 0.0;
                int nz = 0;
                for (int i = 0; i < sizes[u]; i++) {
                    md = fmax(md, fabs(b6[i] - b7[i]));
                    mb = fmax(mb, fabs(b6[i]));
                    nz += b7[i] != 0.0;
                }
                printf("   lam=%g R=%d max|b6-b7| = %.3e (max|b| %.3e, nnz %d)\n", lam, R, md, mb, nz);
            }
        }
    }
    return 0;
}
