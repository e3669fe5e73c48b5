// bl_tc.cuh -- NEXT-1 fold-batched scan of fp32 designs on the 5th-generation tensor
// cores (tcgen05.mma kind::i8 on SM pairs, accumulators in TMEM).  Citations as in
// bl_kernels.cuh.
//
// The contraction is the batched form of identity (3): for the K + 1 fits of a
// cross-validation round, D = X^T R, R = the fits' residuals (n x NF), every
// column of X read once for all fits.  It is evaluated EXACTLY in integers:
//
//   x_ij = 2^{E_j} y_ij,  |y| <= 1/2     (E_j per column, k_xscale)
//   y ~ c0 2^-22 + c1 2^-37,  c0 = rint(y 2^22), c1 = rint((y - c0 2^-22) 2^37)
//       (|c0| <= 2^21, |c1| <= 2^14; |y - y~| <= 2^-38: |x - x~| <= 2^{E_j - 38} <= 2^-36 max_i |x_ij|)
//   U0 = c0 + 2^22 (three u8 digit planes, byte j weighted 2^{8 j - 22}), U1 = c1 + 2^14 (two
//       u8 planes, 2^{8 j - 37}); the top byte of each carries the bias 64, removed exactly in
//       the epilogue with the residual digit sums
//   r_i ~ 2^{-S_f} R_i,  R = rint(r 2^{S_f}), |R| <= 2^46, six balanced base-256 digits (s8)
//       (|r - r~| <= 2^{-S_f - 1} <= 2^-46 max_i |r_i|)
//
// Products of X byte j and residual digit b have the weight of the "diagonal" s = j + b, so the
// byte planes of a chunk accumulate into ONE int32 accumulator per (fit, s) -- the B operand of
// byte plane j holds digit b = s - j in column (f, s) -- with no rounding at all (|.| <= n
// (255 + 255 + 96) 128 < 2^31 for n <= 27,000).  The epilogue removes the bias in int32, then
// recombines the 2 x 8 diagonals per (column, fit) in fp64 in a fixed order.  The result differs from the exact dot product of the fp32 x and fp64 r by at most
// 2^-36 max|x_j| ||r||_1 + 2^-46 max|r| ||x_j||_1 + the fp64 rounding of the recombination
// (k_scan_batch_tc).
//
// Why integers: the fp64 pipe (DMMA = DFMA rate, 36 TFLOP/s) puts an 11-fit pass at the ridge
// of the HBM roofline (5.5 flop / byte) -- k_scan_batch_mma reached 0.56 of it.  Measured on
// B200 (scripts/tc_mma_bench.cu): one tcgen05.mma kind::i8 costs ~137 cycles at cta_group::1
// for ANY N <= 256, but ~70 cycles at cta_group::2 (M = 256 over an SM pair) for N = 80 --
// rising to ~140 when the A operand's shared memory is also being written at full rate.  So
// the pass runs on CTA pairs, and the converters put the X digit planes straight into TENSOR
// memory (tcgen05.st; A operand from TMEM), leaving shared memory to the small B tiles:
// 12 pair-MMAs per 64-row stage against ~1390 cycles of HBM time for the pair's 2 x 32 KB of
// X.  The operand traffic into the tensor core (and the converters' writes of it) is what
// limits the MMAs, so X carries five digit planes (37 bits), not six.  The digit split costs
// 4 FFMA/FADD + 2.75 PRMT per element, also inside the HBM time.
//
// Roles (a cluster of 2 CTAs = one SM pair, persistent over 256-column tiles; CTA rank q owns
// tile columns 128 q .. 128 q + 127 = its 128 TMEM lanes):
//   warps 0-3   epilogue: tcgen05.ld of the 2 x N accumulator columns of their 32 TMEM
//               lanes, bias removal, recombination, identity (3), KKT / strong tests,
//               ballot-compacted lists (as k_scan_batch)
//   warps 4-19  converters: warp (lane quarter wid % 4, row group (wid - 4) / 4): column
//               32 (wid % 4) + lane, 16 rows of each stage -> registers (32-byte loads, two
//               stages ahead) -> five digit-plane words x 4 -> tcgen05.st into the stage's A
//               slot in TMEM (lane = column, 16 columns of 4 K-bytes per plane); converter 0
//               also bulk-copies (cp.async.bulk, mbarrier tx count) this CTA's half of the
//               stage's residual digit tiles (3 byte-plane variants x N / 2 rows: the
//               cta_group::2 B split), prepared once per pass by k_rimg
//   warp 20     TMEM allocation (cta_group::2); in rank 0, lane 0 issues the pair's MMAs and
//               commits; in rank 1, lane 0 relays "stage full" to rank 0's barrier
// Ring of kTcStages stages: A slots in TMEM (80 columns each), B slots in shared memory;
// barriers full (converter warps + bulk tx), pfull (rank 1's relay, in rank 0), empty
// (multicast commit), tfull (multicast commit), tempty (8 epilogue warps of the pair, in
// rank 0).  TMEM: [0, 2N) the two chunk accumulators, then the A slots (2 N + 320 <= 512).
#pragma once
#include "bl_kernels.cuh"

namespace bl {

constexpr int kTcCols = 128;                     // X columns per CTA (UMMA M = 256 per SM pair)
constexpr int kTcRows = 64;                      // rows (K bytes) per pipeline stage
constexpr int kTcStages = 4;                     // A slots in TMEM
constexpr int kTcXL = 5;                         // X digit planes (U0: 3 bytes, U1: 2 bytes)
constexpr int kTcRL = 6;                         // residual digits
constexpr int kTcDiag = 8;                       // diagonals s = byte + digit, 0 .. 7
constexpr int kTcConvWarps = 16;
constexpr int kTcThreads = 32 * (4 + 1 + kTcConvWarps);
constexpr int kTcMmaWarp = 4 + kTcConvWarps;     // warps 0-3 epilogue, 4-19 converters (whole warpgroups), 20 MMA
constexpr int kTcAcols = kTcXL * kTcRows / 4;    // TMEM columns of one A slot (80)
constexpr int kTcMaxFits = 12;                   // 8 * 12 = 96 = N; 2 N + 4 * 80 = 512 TMEM columns
__host__ __device__ constexpr int tc_n(int nf) { return ((kTcDiag * nf + 15) / 16) * 16; }
__host__ __device__ constexpr int tc_vbytes(int nf) { return tc_n(nf) / 2 * kTcRows; }     // one variant, one half
__host__ __device__ constexpr int tc_hbytes(int nf) { return 3 * tc_vbytes(nf); }          // one CTA's B slot
__host__ __device__ constexpr int tc_bbytes(int nf) { return 2 * tc_hbytes(nf); }          // a stage's image
__host__ __device__ constexpr size_t tc_smem(int nf) { return (size_t)kTcStages * tc_hbytes(nf) + 1024; }
// byte offset of (row m of the M / N dimension, k-th byte of K) in a K-major core-matrix
// tile of 64 K-bytes: 8 x 16-byte core matrices, LBO (next 16 K-bytes) = 128, SBO (next 8 rows) = 512
__host__ __device__ constexpr int tc_off(int m, int k) { return (m >> 3) * 512 + (k >> 4) * 128 + (m & 7) * 16 + (k & 15); }

// smem matrix descriptor (sm_100 version 1): no swizzle, K-major, LBO 128 B, SBO 512 B
__device__ __forceinline__ uint64_t tc_desc(uint32_t saddr) {
    return (uint64_t)((saddr & 0x3FFFFu) >> 4) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(512 >> 4) << 32) |
           (1ull << 46);
}
// instruction descriptor, kind::i8: D s32, A u8 (K-major), B s8 (K-major), M, N
__host__ __device__ constexpr uint32_t tc_idesc(int M, int N, bool a_signed) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// A from tensor memory (both CTAs' TMEM at column atmem), B from both CTAs' shared memory
__device__ __forceinline__ void tc_mma2_ts(uint32_t dtmem, uint32_t atmem, uint64_t bd, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n"
        ::"r"(dtmem), "r"(atmem), "l"(bd), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tc_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c),
                 "r"(d)
                 : "memory");
}
__device__ __forceinline__ void tc_st2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b) : "memory");
}
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// arrive on the barrier at this smem offset in BOTH CTAs of the pair once the issued MMAs retire
__device__ __forceinline__ void tc_commit2(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                 ::"r"(smem_addr(bar)), "h"((uint16_t)3) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_ld16(uint32_t taddr, int (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// waits with cluster-scope acquire (barriers that CTAs of the pair arrive on remotely); the
// _lazy variant backs off (epilogue / relay waits that are off the critical path)
__device__ __forceinline__ bool mbar_try_relaxed(uint64_t *bar, unsigned parity) {
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_addr(bar)), "r"(parity) : "memory");
    return ok != 0;
}
// waits on barriers that the other CTA of the pair arrives on: relaxed polling, then ONE
// cluster-scope acquire (an acquire per poll invalidates the SM's L1 every time); the _lazy
// variant backs off (waits off the critical path)
__device__ __forceinline__ void mbar_wait_cl(uint64_t *bar, unsigned parity) {
    while (!mbar_try_relaxed(bar, parity)) {
    }
    asm volatile("fence.acquire.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_lazy(uint64_t *bar, unsigned parity) {
    while (!mbar_try_relaxed(bar, parity)) __nanosleep(256);
    asm volatile("fence.acquire.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// E_j: max_i<n |x_ij| <= 2^{E_j - 1}; xsc_j = 2^{-E_j} (a zero column: 1).  One pass over X,
// once per design (the digits of a column are relative to the whole column, all folds).
__global__ void __launch_bounds__(256) k_xscale(const float *__restrict__ X, int64_t ld, int n, int64_t p,
                                                float *__restrict__ xsc) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = w0; j < p; j += nw) {
        const float *x = X + j * ld;
        float m = 0.f;
        for (int i = 4 * lane; i < n; i += 128) {
            const float4 v = __ldcs(reinterpret_cast<const float4 *>(x + i));
            m = fmaxf(m, fabsf(v.x));
            if (i + 1 < n) m = fmaxf(m, fabsf(v.y));
            if (i + 2 < n) m = fmaxf(m, fabsf(v.z));
            if (i + 3 < n) m = fmaxf(m, fabsf(v.w));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) xsc[j] = m > 0.f ? ldexpf(1.f, -(ilogbf(m) + 2)) : 1.f;
    }
}

// The residual digits of one pass: fit f (block f) -> rsc[f] = 2^{-S_f}; digit b of row i goes
// to column (f, s = b + j) of the B tile of X byte plane j (j = 0, 1, 2) -- the "diagonal"
// pairing -- in the K-major layout, image[stage][half][j][N/2 rows x 64 bytes] (columns
// 0 .. N/2 - 1 in half 0, the rest in half 1: the two CTAs' B halves); dsum[6 f + b] = sum_i
// d_ifb (exact int32).  The caller zeroes the image (rows >= n, unused columns stay zero).
__global__ void __launch_bounds__(1024) k_rimg(const FitScan *__restrict__ fits, int n, int nhalf,
                                               int8_t *__restrict__ img, double *__restrict__ rsc,
                                               int *__restrict__ dsum) {
    __shared__ double sh[32];
    __shared__ int ssum[kTcRL];
    const int f = blockIdx.x;
    const double *r = fits[f].r;
    if (threadIdx.x < kTcRL) ssum[threadIdx.x] = 0;
    double m = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) m = fmax(m, fabs(r[i]));
    m = block_max(m, sh);
    // |R| = |rint(r 2^S)| <= 2^46: max < 2^{ilogb(max) + 1}
    const int S = m > 0.0 ? 45 - ilogb(m) : 0;
    if (threadIdx.x == 0) rsc[f] = ldexp(1.0, -S);
    const int vb = nhalf * kTcRows;
    int ds[kTcRL] = {0, 0, 0, 0, 0, 0};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        long long R = llrint(ldexp(r[i], S));
        int8_t *t = img + (size_t)(i / kTcRows) * 6 * vb;
        const int k = i % kTcRows;
#pragma unroll
        for (int b = 0; b < kTcRL; b++) {
            const long long dg = ((R + 128) & 255) - 128;      // balanced digit in [-128, 127]
            R = (R - dg) >> 8;                                  // exact
#pragma unroll
            for (int j = 0; j < 3; j++) {
                const int nb = kTcDiag * f + b + j, h = nb >= nhalf;
                t[(3 * h + j) * vb + tc_off(nb - h * nhalf, k)] = (int8_t)dg;
            }
            ds[b] += (int)dg;
        }
    }
#pragma unroll
    for (int b = 0; b < kTcRL; b++) {
        const int v = warp_sum_i(ds[b]);
        if ((threadIdx.x & 31) == 0) atomicAdd(&ssum[b], v);
    }
    __syncthreads();
    if (threadIdx.x < kTcRL) dsum[kTcRL * f + threadIdx.x] = ssum[threadIdx.x];
}

// 2^e as a compile-time double (|e| < 1000)
__host__ __device__ constexpr double tc_pow2(int e) {
    double v = 1.0;
    for (int i = 0; i < (e < 0 ? -e : e); i++) v = e < 0 ? v * 0.5 : v * 2.0;
    return v;
}
template <int NF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    k_scan_batch_tc(const float *__restrict__ X, int64_t ld, int n, int64_t p, const FitScan *__restrict__ fits,
                    const float *__restrict__ xsc, const int8_t *__restrict__ rimg, const double *__restrict__ rsc,
                    const int *__restrict__ dsum, const int *__restrict__ list, const int *__restrict__ lctl) {
    constexpr int N = tc_n(NF);
    constexpr int VB = tc_vbytes(NF);
    constexpr int HB = tc_hbytes(NF);
    constexpr int ABASE = 2 * N;                               // TMEM column of A slot 0
    static_assert(NF >= 1 && NF <= kTcMaxFits && ABASE + kTcStages * kTcAcols <= 512, "TMEM budget");
    extern __shared__ uint8_t smt_raw[];
    __shared__ FitScan fs[NF];
    __shared__ double k1s[NF], rscs[NF];
    __shared__ int dss[kTcRL * NF];
    __shared__ __align__(8) uint64_t full_b[kTcStages], pfull_b[kTcStages], empty_b[kTcStages], tfull, tempty;
    __shared__ uint32_t tmem_sh;
    uint8_t *ring = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smt_raw) + 1023) & ~(uintptr_t)1023);
    const int tid = threadIdx.x, wid = tid >> 5, lane = tid & 31;
    uint32_t q;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(q));
    if (tid < NF) fs[tid] = fits[tid];
    if (tid < kTcRL * NF) dss[tid] = dsum[tid];
    if (tid == 0) {
        for (int s = 0; s < kTcStages; s++) {
            mbar_init(&full_b[s], kTcConvWarps + 1);           // converter warps + the bulk copy's arm
            mbar_init(&pfull_b[s], 1);                          // rank 1's relay (rank 0's copy used)
            mbar_init(&empty_b[s], 1);
        }
        mbar_init(&tfull, 1);
        mbar_init(&tempty, 8);                                  // the pair's 8 epilogue warps
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (wid == kTcMmaWarp) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_arrive();
    cluster_wait();
    tc_fence_after();
    if (tid < NF) {
        k1s[tid] = *fs[tid].K1;
        rscs[tid] = rsc[tid];
    }
    __syncthreads();
    const uint32_t tmem = tmem_sh;
    if (list && !lctl[1]) list = nullptr;
    const int64_t P = list ? (int64_t)lctl[0] : p;
    const int64_t ntiles = (P + 2 * kTcCols - 1) / (2 * kTcCols);
    const int64_t pair0 = blockIdx.x >> 1, npair = gridDim.x >> 1;
    const int nst = (n + kTcRows - 1) / kTcRows;
    auto colof = [&](int64_t pos) -> int64_t { return list ? (int64_t)list[pos] : pos; };

    if (wid >= 4 && wid < kTcMmaWarp) {
        // ---------------- converters: column m = 32 (wid % 4) + lane (= its TMEM lane), rows
        // 16 h .. 16 h + 15 of every stage, h = (wid - 4) / 4: two 32-byte loads per stage (four
        // 16-byte loads if ld % 8 != 0), held in registers two stages ahead (three sets in rotation)
        const int qq = wid & 3, h = (wid - 4) >> 2, m = 32 * qq + lane;
        const uint32_t tl = tmem + ((uint32_t)(32 * qq) << 16) + ABASE + 4 * h;
        const bool copier = wid == 4 && lane == 0;
        const bool v8ok = (ld & 7) == 0 && (reinterpret_cast<uintptr_t>(X) & 31) == 0;   // 32-byte aligned segments
        uint32_t g = 0;                                            // stage counter (all tiles)
        for (int64_t tile = pair0; tile < ntiles; tile += npair) {
            const int64_t jc = colof(min(tile * 2 * kTcCols + q * kTcCols + m, P - 1));   // past the end: ignored
            const float *xc = X + jc * ld + 16 * h;
            const float sc = xsc[jc];
            float4 xa[4], xb[4], xd[4];
            auto load = [&](float4 (&xr)[4], int s) {
                if (s >= nst) return;
                if (v8ok) {
#pragma unroll
                    for (int i = 0; i < 4; i += 2) {
                        const int64_t r = (int64_t)s * kTcRows + 16 * h + 4 * i;
                        if (r < ld)                                // ld % 8 == 0: 8 rows inside or outside together
                            asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                                : "=f"(xr[i].x), "=f"(xr[i].y), "=f"(xr[i].z), "=f"(xr[i].w), "=f"(xr[i + 1].x),
                                  "=f"(xr[i + 1].y), "=f"(xr[i + 1].z), "=f"(xr[i + 1].w)
                                : "l"(xc + (int64_t)s * kTcRows + 4 * i));
                        else
                            xr[i] = xr[i + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 4; i++) {
                        const int64_t r = (int64_t)s * kTcRows + 16 * h + 4 * i;   // ld % 4 == 0
                        xr[i] = r < ld ? __ldcs(reinterpret_cast<const float4 *>(xc + (int64_t)s * kTcRows + 4 * i))
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
                    }
                }
            };
            auto step = [&](float4 (&cur)[4], float4 (&nx2)[4], int s) {
                load(nx2, s + 2);                                  // two stages ahead
                const uint32_t slot = g % kTcStages, use = g / kTcStages;
                if (use > 0) mbar_wait(&empty_b[slot], (use - 1) & 1);
                if (copier) {                                      // this CTA's half of the residual digit tiles
                    mbar_arm(&full_b[slot], HB);
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                        ::"r"(smem_addr(ring + (size_t)slot * HB)), "l"(rimg + (size_t)s * 2 * HB + q * HB), "r"(HB),
                        "r"(smem_addr(&full_b[slot]))
                        : "memory");
                }
                tc_fence_after();                                  // after the empty wait: the MMAs read the slot
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {                   // rows 16 h + 8 hh .. + 7
                    uint32_t pw[kTcXL][2];                         // plane words of 4 rows each
#pragma unroll
                    for (int i2 = 0; i2 < 2; i2++) {
                        const float4 cv = cur[2 * hh + i2];
                        const float v[4] = {cv.x, cv.y, cv.z, cv.w};
                        uint32_t w[2][4];
#pragma unroll
                        for (int u = 0; u < 4; u++) {
                            // U0 = c0 + 2^22 in the low 24 bits of t0 (3.0 = 1.5 2^1: unit in the last place
                            // 2^-22), U1 = c1 + 2^14 in the low 16 bits of t1 (1.5 2^-14 + 2^-23: ulp 2^-37)
                            const float t0 = __fmaf_rn(v[u], sc, 3.0f);
                            const float h0 = __fsub_rn(t0, 3.0f);
                            const float y1 = __fmaf_rn(v[u], sc, -h0);
                            const float t1 = __fadd_rn(y1, 9.16719436645507812500e-05f);
                            w[0][u] = __float_as_uint(t0);
                            w[1][u] = __float_as_uint(t1);
                        }
#pragma unroll
                        for (int c = 0; c < 2; c++) {
                            const uint32_t p01 = __byte_perm(w[c][0], w[c][1], 0x5140);
                            const uint32_t p23 = __byte_perm(w[c][2], w[c][3], 0x5140);
                            pw[3 * c][i2] = __byte_perm(p01, p23, 0x5410);
                            pw[3 * c + 1][i2] = __byte_perm(p01, p23, 0x7632);
                        }
                        const uint32_t q01 = __byte_perm(w[0][0], w[0][1], 0x0062);
                        const uint32_t q23 = __byte_perm(w[0][2], w[0][3], 0x6200);
                        pw[2][i2] = __byte_perm(q01, q23, 0x7610);
                    }
#pragma unroll
                    for (int a = 0; a < kTcXL; a++)
                        tc_st2(tl + slot * kTcAcols + 16 * a + 2 * hh, pw[a][0], pw[a][1]);
                }
                tc_wait_st();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&full_b[slot]);
                ++g;
            };
            load(xa, 0);
            load(xb, 1);
            for (int s = 0; s < nst; s += 3) {
                step(xa, xd, s);
                if (s + 1 < nst) step(xb, xa, s + 1);
                if (s + 2 < nst) step(xd, xb, s + 2);
            }
        }
    } else if (wid == kTcMmaWarp) {
        if (lane == 0 && q == 0) {
            // ---------------- MMA issuer of the pair (rank 0)
            uint32_t g = 0, it = 0;
            const uint32_t idu = tc_idesc(2 * kTcCols, N, false);
            for (int64_t tile = pair0; tile < ntiles; tile += npair, ++it) {
                if (it > 0) mbar_wait_cl(&tempty, (it - 1) & 1);    // both epilogues have read D
                tc_fence_after();
                for (int s = 0; s < nst; s++, ++g) {
                    const uint32_t slot = g % kTcStages, use = g / kTcStages;
                    mbar_wait(&full_b[slot], use & 1);
                    mbar_wait_cl(&pfull_b[slot], use & 1);
                    tc_fence_after();
                    const uint32_t bbase = smem_addr(ring + (size_t)slot * HB);
                    const uint32_t abase = tmem + ABASE + slot * kTcAcols;
#pragma unroll
                    for (int a = 0; a < kTcXL; a++) {                // planes 0-2: U0 bytes, 3-4: U1 bytes
                        const int c = a < 3 ? 0 : 1, jb = a < 3 ? a : a - 3;
#pragma unroll
                        for (int ks = 0; ks < 2; ks++)              // K = 32 bytes (8 TMEM columns) per MMA
                            tc_mma2_ts(tmem + (uint32_t)(c * N), abase + 16 * a + 8 * ks,
                                       tc_desc(bbase + jb * VB + 256 * ks), idu, (s | ks | jb) != 0);
                    }
                    tc_commit2(&empty_b[slot]);                     // both CTAs' slot is free once these retire
                }
                tc_commit2(&tfull);
            }
        } else if (lane == 0) {
            // ---------------- rank 1: relay "my stage is full" to rank 0's pfull barrier
            uint32_t g = 0;
            for (int64_t tile = pair0; tile < ntiles; tile += npair)
                for (int s = 0; s < nst; s++, ++g) {
                    const uint32_t slot = g % kTcStages, use = g / kTcStages;
                    mbar_wait(&full_b[slot], use & 1);
                    mbar_arrive_remote(mapa(&pfull_b[slot], 0));
                }
        }
        __syncwarp();
    } else {
        // ---------------- epilogue: thread = TMEM lane 32 wid + lane = this CTA's tile column
        uint32_t it = 0;
        const uint32_t tl = tmem + ((uint32_t)(32 * wid) << 16);
        const uint32_t tempty0 = mapa(&tempty, 0);
        for (int64_t tile = pair0; tile < ntiles; tile += npair, ++it) {
            mbar_wait_lazy(&tfull, it & 1);
            tc_fence_after();
            double acc[NF];
#pragma unroll
            for (int f = 0; f < NF; f++) acc[f] = 0.0;
#pragma unroll
            for (int c = 0; c < 2; c++) {
#pragma unroll
                for (int c0 = 0; c0 < N / 16; c0++) {
                    int v[16];
                    tc_ld16(tl + (uint32_t)(c * N + 16 * c0), v);
                    tc_wait_ld();
#pragma unroll
                    for (int u = 0; u < 16; u++) {
                        const int nb = 16 * c0 + u, f = nb / kTcDiag, sd = nb % kTcDiag;
                        if (f < NF) {
                            // the top byte plane (U0 byte 2, U1 byte 1) carries +64: remove
                            // 64 sum_i d_{f, sd - top} exactly
                            const int top = 2 - c;
                            const int db = sd - top;
                            const int dv = (db >= 0 && db < kTcRL) ? v[u] - 64 * dss[kTcRL * f + db] : v[u];
                            acc[f] = fma((double)dv, tc_pow2(8 * sd - (c ? 37 : 22)), acc[f]);
                        }
                    }
                }
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_remote(tempty0);            // D may be overwritten by the next tile
            const int64_t jp = tile * 2 * kTcCols + q * kTcCols + 32 * wid + lane;
            const bool inr = jp < P;
            const int64_t j = inr ? colof(jp) : 0;
            const double e2 = inr ? 1.0 / (double)xsc[j] : 0.0;    // 2^{E_j}, exact
#pragma unroll
            for (int f = 0; f < NF; f++) {
                const FitScan &F = fs[f];
                bool isv = false, iss = false;
                if (inr) {
                    const double d = acc[f] * e2 * rscs[f];
                    const double sj = F.s[j];
                    const double z = sj > 0.0 ? (d - F.c[j] * k1s[f]) * F.K2 / sj : 0.0;
                    F.out[j] = z;
                    const double az = fabs(z);
                    const bool inw = F.wflag[j] != 0;
                    const uint8_t fl = F.flags[j];
                    isv = !inw && (fl & 1) && az > F.thr_viol;
                    iss = !inw && (fl & 2) && F.thr_strong >= 0.0 && az >= F.thr_strong && sj > 0.0;
                }
                warp_append(isv, (int)j, F.viol, F.nviol);
                warp_append(iss, (int)j, F.strong, F.nstrong);
            }
        }
    }
    tc_fence_before();
    cluster_arrive();                                              // both CTAs done: every MMA has retired
    cluster_wait();
    if (wid == kTcMmaWarp) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

}  // namespace bl
