// Stand-alone timing of the Gram CD kernel (bl_kernels.cuh) on synthetic data:
// nW slots, G = I + small symmetric noise, every coordinate active.  Prints
// SM cycles per coordinate visit.  Build on the CPU box, run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1701_05936_b200/csrc -o scripts/cd_bench scripts/cd_bench.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "bl_kernels.cuh"
using namespace bl;

template <int KP, int D, bool V5 = false>
void run(int nW, int passes_wanted) {
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
    cudaMemcpy(dG, G.data(), 8 * G.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dz, z.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dbeta, beta.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dc, c.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(ds, s.data(), 8 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, Wst.data(), 4 * nW, cudaMemcpyHostToDevice);
    cudaMemcpy(dord, ord.data(), 4 * nW, cudaMemcpyHostToDevice);
    CdGramArgs a{};
    a.Wst = dW; a.ord = dord; a.nW = nW; a.ldG = ldG; a.G = dG; a.z = dz; a.beta = dbeta; a.dbeta = ddb;
    a.lam_alpha = 1e-6; a.inv_den = 1.0; a.tol = 0.0; a.floor_ = 0.0; a.max_iter = passes_wanted;
    a.betaW_out = dbw; a.c = dc; a.s = ds; a.st = dst;
    int nWp = (nW + 1) & ~1;
    size_t smem = (size_t)24 * nWp + 16;
    cudaFuncSetAttribute(k_cd_gram5<KP>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k_cd_gram5<KP><<<1, kGram5Threads, smem>>>(a);
    cudaDeviceSynchronize();
    RoundStatus h;
    cudaMemcpy(&h, dst, sizeof h, cudaMemcpyDeviceToHost);
    printf("%s KP=%d D=%d nW=%5d passes=%d visits=%lld updates=%lld  cycles/visit=%.1f  A %.1f B %.1f C %.1f (%s)\n", V5 ? "blocked  " : "per-coord", KP, D, nW,
           h.cd_passes, h.cd_visits, h.cd_updates, (double)h.cd_cycles / h.cd_visits,
           (double)h.cd_prof[0] / h.cd_visits, (double)h.cd_prof[1] / h.cd_visits, (double)h.cd_prof[2] / h.cd_visits,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(dG); cudaFree(dz); cudaFree(dbeta); cudaFree(ddb); cudaFree(dbw); cudaFree(dc); cudaFree(ds);
    cudaFree(dW); cudaFree(dord); cudaFree(dst);
}

int main() {
    run<1, 0, true>(200, 40);
    run<1, 0, true>(600, 40);
    run<2, 0, true>(1500, 20);
    run<4, 0, true>(4000, 6);
    return 0;
}
