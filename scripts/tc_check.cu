// Stand-alone check + timing of the tcgen05 fold-batched scan (bl_tc.cuh): z_f(j) = x_j^T r_f
// (c = 0, s = 1, K2 = 1) against a CPU fp64 dot product on sampled columns, then GB/s of X
// read on a large design.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1701_05936_b200/csrc \
//        scripts/tc_check.cu -o /tmp/tc_check && /tmp/tc_check [n p NF]
#include "bl_tc.cuh"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

using namespace bl;

#define CKC(x)                                                                                  \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);     \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

template <int NF>
const void *kern_n(int nb) {
    if constexpr (NF > 1) {
        if (nb < NF) return kern_n<NF - 1>(nb);
    }
    return (const void *)k_scan_batch_tc<NF>;
}

int main(int argc, char **argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 1000;
    const int64_t p = argc > 2 ? atoll(argv[2]) : 1000;
    const int NF = argc > 3 ? atoi(argv[3]) : 11;
    const int reps = argc > 4 ? atoi(argv[4]) : 5;
    const int64_t ld = (n + 3) / 4 * 4;
    printf("n=%d p=%lld NF=%d ld=%lld\n", n, (long long)p, NF, (long long)ld);
    // X: N(0,1) fp32 with a few scaled columns (digit scales differ per column) and a zero column
    float *dX;
    CKC(cudaMalloc(&dX, sizeof(float) * ld * p));
    {
        const int64_t CH = 4096;
        std::vector<float> h(ld * CH);
        std::mt19937_64 g(1);
        std::normal_distribution<float> nd;
        for (int64_t j0 = 0; j0 < p; j0 += CH) {
            const int64_t c = std::min(CH, p - j0);
            if (j0 == 0 || j0 + CH >= p) {
                for (int64_t u = 0; u < c * ld; u++) h[u] = nd(g);
                for (int64_t u = 0; u < c; u++) {
                    const float sc = (j0 + u) % 7 == 3 ? 1e-3f : (j0 + u) % 7 == 5 ? 300.f : 1.f;
                    for (int i = 0; i < ld; i++) h[u * ld + i] = i < n ? h[u * ld + i] * sc : 0.f;
                    if (j0 + u == 2) for (int i = 0; i < ld; i++) h[u * ld + i] = 0.f;
                }
            }
            CKC(cudaMemcpy(dX + j0 * ld, h.data(), sizeof(float) * c * ld, cudaMemcpyHostToDevice));
        }
    }
    std::vector<std::vector<double>> hr(NF, std::vector<double>(n));
    std::mt19937_64 g(2);
    std::normal_distribution<double> nd;
    for (int f = 0; f < NF; f++)
        for (int i = 0; i < n; i++) hr[f][i] = (i % (f + 2) == 0) ? 0.0 : nd(g) * (f == 3 ? 1e-6 : 1.0);
    double *dr, *dout, *dK1, *dc, *ds, *rsc;
    uint8_t *dflags;
    int *dcnt, *dlist;
    CKC(cudaMalloc(&dr, sizeof(double) * n * NF));
    CKC(cudaMalloc(&dout, sizeof(double) * p * NF));
    CKC(cudaMalloc(&dK1, sizeof(double)));
    CKC(cudaMemset(dK1, 0, sizeof(double)));
    CKC(cudaMalloc(&dc, sizeof(double) * p));
    CKC(cudaMalloc(&ds, sizeof(double) * p));
    CKC(cudaMalloc(&dflags, p));
    CKC(cudaMalloc(&dcnt, sizeof(int) * 4 * NF));
    CKC(cudaMalloc(&dlist, sizeof(int) * 16));
    CKC(cudaMalloc(&rsc, sizeof(double) * 16));
    CKC(cudaMemset(dc, 0, sizeof(double) * p));
    CKC(cudaMemset(dflags, 0, p));
    {
        std::vector<double> one(p, 1.0);
        CKC(cudaMemcpy(ds, one.data(), sizeof(double) * p, cudaMemcpyHostToDevice));
    }
    std::vector<FitScan> hf(NF);
    for (int f = 0; f < NF; f++) {
        CKC(cudaMemcpy(dr + (size_t)f * n, hr[f].data(), sizeof(double) * n, cudaMemcpyHostToDevice));
        FitScan &F = hf[f];
        memset(&F, 0, sizeof(F));
        F.r = dr + (size_t)f * n;
        F.K1 = dK1;
        F.K2 = 1.0;
        F.c = dc;
        F.s = ds;
        F.out = dout + (size_t)f * p;
        F.flags = dflags;
        F.wflag = dflags;
        F.thr_viol = 1e300;
        F.thr_strong = -1.0;
        F.viol = dlist; F.nviol = dcnt + 4 * f;
        F.strong = dlist; F.nstrong = dcnt + 4 * f + 1;
    }
    FitScan *dfs;
    CKC(cudaMalloc(&dfs, sizeof(FitScan) * NF));
    CKC(cudaMemcpy(dfs, hf.data(), sizeof(FitScan) * NF, cudaMemcpyHostToDevice));
    float *xsc;
    CKC(cudaMalloc(&xsc, sizeof(float) * p));
    int dev = 0, nsm = 0;
    CKC(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    k_xscale<<<nsm * 8, 256>>>(dX, ld, n, p, xsc);
    CKC(cudaGetLastError());
    const int nst = (n + kTcRows - 1) / kTcRows;
    const int bb = tc_bbytes(NF);
    int *dsum;
    CKC(cudaMalloc(&dsum, sizeof(int) * 6 * kTcMaxFits));
    int8_t *img;
    CKC(cudaMalloc(&img, (size_t)nst * bb));
    const void *kern = kern_n<kTcMaxFits>(NF);
    const size_t smem = tc_smem(NF);
    CKC(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = 2 * (int)std::min<int64_t>((p + 2 * kTcCols - 1) / (2 * kTcCols), nsm / 2);
    const int *nl = nullptr;
    auto run = [&]() {
        CKC(cudaMemsetAsync(img, 0, (size_t)nst * bb));
        k_rimg<<<NF, 1024>>>(dfs, n, tc_n(NF) / 2, img, rsc, dsum);
        const float *X = dX;
        int64_t ld_ = ld, p_ = p;
        int n_ = n;
        const int8_t *im = img;
        const double *rs = rsc;
        const int *dsm = dsum;
        void *args[] = {&X, &ld_, &n_, &p_, &dfs, &xsc, &im, &rs, &dsm, &nl, &nl};
        CKC(cudaLaunchKernel(kern, dim3(grid), dim3(kTcThreads), args, smem, 0));
    };
    run();
    CKC(cudaDeviceSynchronize());
    CKC(cudaGetLastError());
    // check sampled columns
    std::vector<int64_t> cols;
    for (int64_t j = 0; j < std::min<int64_t>(p, 300); j++) cols.push_back(j);
    for (int64_t j = std::max<int64_t>(300, p - 300); j < p; j++) cols.push_back(j);
    double worst = 0.0;
    std::vector<float> xc(n);
    std::vector<double> rn(NF, 0.0);
    for (int f = 0; f < NF; f++) {
        for (int i = 0; i < n; i++) rn[f] += hr[f][i] * hr[f][i];
        rn[f] = std::sqrt(rn[f]);
    }
    int shown = 0;
    for (int64_t j : cols) {
        CKC(cudaMemcpy(xc.data(), dX + j * ld, sizeof(float) * n, cudaMemcpyDeviceToHost));
        double xn = 0.0;
        for (int i = 0; i < n; i++) xn += (double)xc[i] * xc[i];
        xn = std::sqrt(xn);
        for (int f = 0; f < NF; f++) {
            double ref = 0.0;
            for (int i = 0; i < n; i++) ref += (double)xc[i] * hr[f][i];
            double got;
            CKC(cudaMemcpy(&got, dout + (size_t)f * p + j, sizeof(double), cudaMemcpyDeviceToHost));
            const double e = std::fabs(got - ref) / (xn * rn[f] + 1e-300);
            if (e > worst) worst = e;
            if (e > 1e-12 && shown < 10) {
                printf("  col %lld fit %d: got %.17g ref %.17g (rel to |x||r| %.3e)\n", (long long)j, f, got, ref, e);
                shown++;
            }
        }
    }
    printf("max |z - ref| / (|x_j| |r_f|) over %zu columns x %d fits: %.3e  %s\n", cols.size(), NF, worst,
           worst < 1e-12 ? "OK" : "FAIL");
    // timing
    cudaEvent_t e0, e1;
    CKC(cudaEventCreate(&e0));
    CKC(cudaEventCreate(&e1));
    float best = 1e30f, tot = 0.f;
    for (int r = 0; r < reps; r++) {
        CKC(cudaEventRecord(e0));
        run();
        CKC(cudaEventRecord(e1));
        CKC(cudaEventSynchronize(e1));
        float ms;
        CKC(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
        tot += ms;
    }
    const double bytes = (double)p * n * 4;
    printf("pass: best %.3f ms, mean %.3f ms; X read %.1f GB/s (best); %.2f TFLOP/s useful (2 n p NF)\n", best,
           tot / reps, bytes / best / 1e6, 2.0 * n * p * NF / best / 1e9);
    return worst < 1e-12 ? 0 : 2;
}
