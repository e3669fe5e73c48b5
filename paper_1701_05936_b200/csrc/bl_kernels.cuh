// bl_kernels.cuh -- sm_100a kernels of the lasso / elastic-net path (biglasso,
// arXiv 1701.05936).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n,
// Qk = DESIGN.md section 3 reading k, "a9" etc. = SURVEY.md 8(a) rows.
//
// Layout: X column-major in HBM, x_ij at X[j*ld + i],
// column starts 16-byte aligned; the standardised matrix is never formed --
// every kernel applies (x - c_j)/s_j on the fly or folds it into an epilogue
// through identities (1)-(3).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace bl {

constexpr int kWarp = 32;
constexpr int kScanThreads = 256;
constexpr int kCdRmax = 16;      // rows per thread in the CD kernel (n <= 16 * 1024)

enum Dt { DT_F64 = 0, DT_F32 = 1, DT_I8 = 2 };

// Scalars produced once per (y, row mask) by the preprocessing kernels and read
// by later kernels straight from device memory (no host round trip).
struct PrepScalars {
    double ybar, sum_yt, Y2, nt, inv_nt;
    double A;          // |a_j*| / n  (= alpha * lambda_max)
    double lmax;       // lambda_max
    double sigma;      // sign(a_j*)
    double c_star, s_star, inv_s_star;
    double sum_v;      // sum of the vector the last store-mode scan used
    long long jstar;   // local index of x_*, -1 if not on this shard
    int n_live;        // non-constant columns
    int pad;
};

// Per-round status written by the CD and scan kernels; mirrored to pinned host
// memory with ONE copy per KKT round.
struct RoundStatus {
    int nviol, nstrong, nscope, nsafe;
    int cd_passes, cd_status, nnz, pad;
    double rss, sumr, l1, l2;
    double sum_v;      // sum of the quantised residual (int8 limb path)
    long long cd_visits, cd_updates;   // coordinate visits / nonzero updates of the last solve
    long long cd_cycles;               // SM clock cycles inside the CD kernel (thread 0)
    long long cd_prof[4];              // Gram CD phase cycles: leader steps, bulk steps, G_AA/M builds, lazy catch-ups
    long long cd_cnt[8];               // Gram CD events: speculation retries, G_AA builds, catch-ups, full sweeps,
                                       //   Newton steps, CG iterations, Newton cycles, partial (sign-limited) steps
    long long cd_dbg[8];               // Gram CD sub-phase cycles (micro-benchmarks only)
    double b0;                         // logistic path: intercept on the standardised scale (in/out)
    int outer, irls_done;              // logistic path: IRLS iterations of the last solve; converged flag
    unsigned int blk_done, pad3;       // k_resid_apply's block counter (the last block reduces; self-resetting)
};

// ---------------------------------------------------------------- small helpers

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ long long warp_sum_ll(long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide sum, result broadcast to every thread.  `sh` >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double *sh) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = lane < nw ? sh[lane] : 0.0;
    t = warp_sum(t);
    return t;
}
__device__ __forceinline__ double block_max(double v, double *sh) {
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    v = warp_max(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = lane < nw ? sh[lane] : -1.0;
    return warp_max(t);
}

// Warp-aggregated append of `j` (when pred) to list[*count].
__device__ __forceinline__ void warp_append(bool pred, int j, int *list, int *count) {
    unsigned m = __ballot_sync(0xffffffffu, pred);
    if (!m) return;
    int lane = threadIdx.x & 31;
    int leader = __ffs(m) - 1;
    int base = 0;
    if (lane == leader) base = atomicAdd(count, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (pred) list[base + __popc(m & ((1u << lane) - 1u))] = j;
}

__device__ __forceinline__ double soft_threshold(double z, double g) {
    return z > g ? z - g : (z < -g ? z + g : 0.0);
}

template <typename T> __device__ __forceinline__ double to_d(T x) { return (double)x; }

// ------------------------------------------------- a2: column statistics (G1)
// One warp per column, 16-byte vector loads.  c_j = mean, s_j = population SD
// over the rows in `mask` (all rows when mask == nullptr).  fp32/fp64: shifted
// sums about the first used row's value (exactly 0 variance for constant
// columns); int8: exact integer sums.
template <typename T, bool MASK>
__global__ void __launch_bounds__(256) k_colstats(const T *__restrict__ X, int64_t ld, int n, int64_t p,
                                                  const uint8_t *__restrict__ mask, int i0, double nt,
                                                  double *__restrict__ c, double *__restrict__ s) {
    constexpr int V = 16 / sizeof(T);
    int lane = threadIdx.x & 31;
    int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = gw; j < p; j += nwarp) {
        const T *col = X + j * ld;
        if constexpr (sizeof(T) == 1) {
            long long s1 = 0, s2 = 0;
            int a1 = 0, a2 = 0;          // full 16-row chunks: 4-way byte dot products (dp4a), exact in int32
            int i = lane * V;
            if (!MASK)                   // four full 16-row chunks per lane and step: four loads in flight
                for (; i + 3 * 32 * V + V <= n; i += 4 * 32 * V) {
                    int4 raw[4];
#pragma unroll
                    for (int u = 0; u < 4; u++) raw[u] = __ldg(reinterpret_cast<const int4 *>(col + i + u * 32 * V));
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        a1 = __dp4a(raw[u].x, 0x01010101, a1); a2 = __dp4a(raw[u].x, raw[u].x, a2);
                        a1 = __dp4a(raw[u].y, 0x01010101, a1); a2 = __dp4a(raw[u].y, raw[u].y, a2);
                        a1 = __dp4a(raw[u].z, 0x01010101, a1); a2 = __dp4a(raw[u].z, raw[u].z, a2);
                        a1 = __dp4a(raw[u].w, 0x01010101, a1); a2 = __dp4a(raw[u].w, raw[u].w, a2);
                    }
                }
            for (; i < n; i += 32 * V) {
                int4 raw = __ldg(reinterpret_cast<const int4 *>(col + i));
                if (!MASK && i + V <= n) {
                    a1 = __dp4a(raw.x, 0x01010101, a1); a2 = __dp4a(raw.x, raw.x, a2);
                    a1 = __dp4a(raw.y, 0x01010101, a1); a2 = __dp4a(raw.y, raw.y, a2);
                    a1 = __dp4a(raw.z, 0x01010101, a1); a2 = __dp4a(raw.z, raw.z, a2);
                    a1 = __dp4a(raw.w, 0x01010101, a1); a2 = __dp4a(raw.w, raw.w, a2);
                    continue;
                }
                const int8_t *xb = reinterpret_cast<const int8_t *>(&raw);
#pragma unroll
                for (int e = 0; e < V; e++) {
                    bool use = (i + e < n) && (!MASK || mask[i + e]);
                    int x = use ? (int)xb[e] : 0;
                    s1 += x;
                    s2 += x * x;
                }
            }
            s1 += a1;                    // per lane <= 512 rows x 127^2 < 2^31 (n <= 16384)
            s2 += a2;
            s1 = warp_sum_ll(s1);
            s2 = warp_sum_ll(s2);
            if (lane == 0) {
                long long ntl = (long long)nt;
                long long num = ntl * s2 - s1 * s1;      // n^2 var, exact
                c[j] = (double)s1 / nt;
                s[j] = num <= 0 ? 0.0 : sqrt((double)num) / nt;
            }
        } else {
            // U 16-byte loads in flight per lane (independent partial sums, combined in a fixed
            // order): one load per lane and iteration left the HBM stream latency-bound (0.6 of
            // peak), four 0.75; eight cover a 1000-row fp32 column in one step
            constexpr int U = 8;
            const double K = to_d(col[i0]);
            double s1[U], s2[U];
#pragma unroll
            for (int u = 0; u < U; u++) s1[u] = s2[u] = 0.0;
            for (int i = lane * V; i < n; i += U * 32 * V) {
                T xv[U][V];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int iu = i + u * 32 * V;
                    if (iu < n) *reinterpret_cast<int4 *>(xv[u]) = __ldcs(reinterpret_cast<const int4 *>(col + iu));
                    else *reinterpret_cast<int4 *>(xv[u]) = make_int4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int iu = i + u * 32 * V;
#pragma unroll
                    for (int e = 0; e < V; e++) {
                        const bool use = (iu + e < n) && (!MASK || mask[iu + e]);
                        const double d = use ? to_d(xv[u][e]) - K : 0.0;
                        s1[u] += d;
                        s2[u] = fma(d, d, s2[u]);
                    }
                }
            }
            double t1 = ((s1[0] + s1[1]) + (s1[2] + s1[3])) + ((s1[4] + s1[5]) + (s1[6] + s1[7]));
            double t2 = ((s2[0] + s2[1]) + (s2[2] + s2[3])) + ((s2[4] + s2[5]) + (s2[6] + s2[7]));
            t1 = warp_sum(t1);
            t2 = warp_sum(t2);
            if (lane == 0) {
                double var = (t2 - t1 * t1 / nt) / nt;
                c[j] = K + t1 / nt;
                s[j] = (var > 0.0 && t2 != 0.0) ? sqrt(var) : 0.0;
            }
        }
    }
}

// ------------------------------------------- a2 for the K + 1 fits of a cross-validation, one pass
// Each row belongs to exactly one fold, and fit u's training rows are all rows but fold
// fit_fold[u] (-1: all rows).  Per column (one warp) the shifted sums of every fold's rows
// (shift K = x_0j) accumulate in this warp's shared-memory slots [fold][lane] (fold ids of the
// rows staged once per CTA); then fit u's sums = all folds' minus its held-out fold's, and
// c_j, s_j follow as in k_colstats (population SD).  One pass over X instead of K + 1.
template <typename T>
__global__ void __launch_bounds__(256) k_colstats_folds(const T *__restrict__ X, int64_t ld, int n, int64_t p,
                                                        const int8_t *__restrict__ fold, int K,
                                                        const int *__restrict__ fit_fold, int nf,
                                                        const double *__restrict__ nt, double *const *__restrict__ cs) {
    extern __shared__ __align__(16) double accs[];          // [8 warps][K][2][32]
    int8_t *fsm = reinterpret_cast<int8_t *>(accs + (size_t)8 * K * 64);
    constexpr int V = 16 / sizeof(T);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < n; i += blockDim.x) fsm[i] = fold[i];
    __syncthreads();
    double *acc = accs + (size_t)wid * K * 64;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t j = gw; j < p; j += nwarp) {
        const T *col = X + j * ld;
        for (int f = 0; f < K; f++) { acc[f * 64 + lane] = 0.0; acc[f * 64 + 32 + lane] = 0.0; }
        __syncwarp();
        const double Ks = to_d(col[0]);
        for (int i = lane * V; i < n; i += 32 * V) {
            T xv[V];
            *reinterpret_cast<int4 *>(xv) = __ldg(reinterpret_cast<const int4 *>(col + i));
#pragma unroll
            for (int e = 0; e < V; e++) {
                if (i + e < n) {
                    const double d = to_d(xv[e]) - Ks;
                    double *a = acc + fsm[i + e] * 64 + lane;
                    a[0] += d;
                    a[32] = fma(d, d, a[32]);
                }
            }
        }
        __syncwarp();
        double t1 = 0.0, t2 = 0.0, h1 = 0.0, h2 = 0.0;      // lane u < nf: fit u's held-out fold sums
        const int fu = lane < nf ? fit_fold[lane] : -1;
        for (int f = 0; f < K; f++) {
            const double f1 = warp_sum(acc[f * 64 + lane]), f2 = warp_sum(acc[f * 64 + 32 + lane]);
            t1 += f1;
            t2 += f2;
            if (f == fu) { h1 = f1; h2 = f2; }
        }
        if (lane < nf) {
            const double s1 = t1 - h1, s2 = t2 - h2, m = nt[lane];
            const double var = (s2 - s1 * s1 / m) / m;
            cs[2 * lane][j] = Ks + s1 / m;
            cs[2 * lane + 1][j] = (var > 0.0 && s2 != 0.0) ? sqrt(var) : 0.0;
        }
        __syncwarp();
    }
}

// ------------------------------------------- a2 helper: y~ = (y - ybar) on the rows
// One block.  Writes yt (ld entries, 0 outside the mask / beyond n), the
// full-row starting residual rfull = y - ybar (beta = 0) and the scalars.
__global__ void k_center_y(const double *__restrict__ y, int n, int ld, const uint8_t *__restrict__ mask,
                           double nt, double *__restrict__ yt, double *__restrict__ rfull, PrepScalars *ps) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        if (!mask || mask[i]) acc += y[i];
    double ybar = block_sum(acc, sh) / nt;
    double s1 = 0.0, s2 = 0.0;
    for (int i = threadIdx.x; i < ld; i += blockDim.x) {
        double v = (i < n && (!mask || mask[i])) ? y[i] - ybar : 0.0;
        yt[i] = v;
        rfull[i] = i < n ? y[i] - ybar : 0.0;   // every row: held-out rows keep y_i - ybar_train
        s1 += v;
        s2 = fma(v, v, s2);
    }
    s1 = block_sum(s1, sh);
    s2 = block_sum(s2, sh);
    if (threadIdx.x == 0) {
        ps->ybar = ybar;
        ps->sum_yt = s1;
        ps->Y2 = s2;
        ps->nt = nt;
        ps->inv_nt = 1.0 / nt;
        ps->sum_v = s1;
    }
}

// out = sum_i v_i (one block) -- the cached sum r of identity (3) for a
// caller-given residual ("we pre-compute and store sum_i r_i").
__global__ void k_vsum(const double *__restrict__ v, int n, double *__restrict__ out) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) acc += v[i];
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) *out = acc;
}

// ------------------------------------------------------- fused scan (G4, row a9)
// Raw dot d_j = sum_i x_ij v_i for a list of columns (or all columns), then the
// identity epilogue:  out_j = (d_j - c_j * K1) * K2 / s_j
//   a_j  : v = y~,          K1 = sum y~,  K2 = 1           (identity (2))
//   b_j  : v = x_* - c_*,   K1 = sum v,   K2 = 1/s_*       (identity (1))
//   z_j  : v = r,           K1 = sum r,   K2 = 1/n         (identity (3))
// In SCAN mode the same epilogue also runs the KKT-violation test at lambda_k
// and the strong-rule test for lambda_{k+1} and
// appends hits with warp-ballot aggregated atomics (order fixed later on the
// host by sorting; the SET is deterministic).
struct ScanArgs {
    const void *X;
    int64_t ld;
    int n;
    int64_t p;
    const int *list;          // nullptr => dense j0..p-1
    int64_t j0;               // first column of a dense range (streamed chunks of a host-resident design)
    int rev;                  // visit the columns in reverse order: consecutive KKT scans alternate
                              // direction, so each starts on the columns the previous one left in L2
    const int *nlist;         // device count of `list` (nullptr => nlist_host)
    int nlist_host;
    const double *v;          // fp64 vector, >= ld entries, zero beyond n (fp32/fp64 path)
    const int8_t *limbs;      // int8 path: 8 planes of `limb_ld` bytes
    int limb_ld;
    const double *limb_scale; // 2^-S
    const double *K1;         // device scalar
    const double *K2;         // device scalar (nullptr => K2v)
    double K2v;
    const double *c, *s;
    double *out;
    const long long *jfix;    // device: out[*jfix] = *fixval (b_j* = n exactly); nullptr none
    const double *fixval;
    // SCAN mode
    int scan;
    const uint8_t *flags;     // bit0 safe at lambda_k, bit1 safe at lambda_{k+1}
    const uint8_t *wflag;     // column already in the working set
    double thr_viol;          // alpha * lambda_k                     (strict >, Q11)
    double thr_strong;        // alpha * (2 lambda_{k+1} - lambda_k)  (>=, Q10); < 0 => off
    int *viol, *nviol, *strong, *nstrong;
};

__device__ __forceinline__ void scan_epilogue(const ScanArgs &a, int64_t j, double d, double K1, double K2) {
    double sj = a.s[j];
    double z = sj > 0.0 ? (d - a.c[j] * K1) * K2 / sj : 0.0;
    if (a.jfix && j == *a.jfix) z = *a.fixval;
    a.out[j] = z;
}

// fp32 / fp64 design: each warp owns C columns at a time; lane L covers rows
// [V*L + 32*V*t, ...) with 16-byte loads; v is staged in shared memory once per
// block and reused by every column of the block (register-blocked over C).
template <typename T, int C>
__global__ void __launch_bounds__(kScanThreads) k_scan_fp(ScanArgs a) {
    constexpr int V = 16 / sizeof(T);
    extern __shared__ __align__(16) double vs[];
    const int n = a.n;
    const int npad = (n + 32 * V - 1) / (32 * V) * (32 * V);
    for (int i = threadIdx.x; i < npad; i += blockDim.x) vs[i] = i < n ? a.v[i] : 0.0;
    __syncthreads();
    const double K1 = *a.K1;
    const double K2 = a.K2 ? *a.K2 : a.K2v;
    const int64_t m = a.list ? (a.nlist ? (int64_t)*a.nlist : (int64_t)a.nlist_host) : a.p - a.j0;
    // a scope list holding every column (BEDPP kept all, lambda < ~0.5 lambda_max) is read
    // as the dense range: same columns, no index indirection, sequential DRAM pages
    const int *__restrict__ list = (a.list && m == a.p) ? nullptr : a.list;
    const int64_t j0 = list ? 0 : a.j0;
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const T *X = reinterpret_cast<const T *>(a.X);
    for (int64_t g = gw * C; g < m; g += nwarp * C) {
        int64_t col[C];
        const T *ptr[C];
#pragma unroll
        for (int q = 0; q < C; q++) {
            int64_t idx = g + q < m ? g + q : m - 1;
            if (a.rev) idx = m - 1 - idx;
            col[q] = list ? (int64_t)list[idx] : j0 + idx;
            ptr[q] = X + col[q] * a.ld;
        }
        double acc[C];
#pragma unroll
        for (int q = 0; q < C; q++) acc[q] = 0.0;
        int i = lane * V;
        // main body: two 16-byte loads per column in flight per lane
        for (; i + 32 * V < n; i += 64 * V) {
            T x0[C][V], x1[C][V];
#pragma unroll
            for (int q = 0; q < C; q++) {
                *reinterpret_cast<int4 *>(x0[q]) = __ldcs(reinterpret_cast<const int4 *>(ptr[q] + i));
                *reinterpret_cast<int4 *>(x1[q]) =
                    __ldcs(reinterpret_cast<const int4 *>(ptr[q] + i + 32 * V));
            }
            double v0[V], v1[V];
#pragma unroll
            for (int e = 0; e < V; e += 2) {
                double2 t0 = *reinterpret_cast<const double2 *>(&vs[i + e]);
                double2 t1 = *reinterpret_cast<const double2 *>(&vs[i + 32 * V + e]);
                v0[e] = t0.x; v0[e + 1] = t0.y; v1[e] = t1.x; v1[e + 1] = t1.y;
            }
            // the second chunk may run past n: zero padding rows explicitly
            const bool tail1 = i + 32 * V + V > n;
#pragma unroll
            for (int q = 0; q < C; q++) {
#pragma unroll
                for (int e = 0; e < V; e++) acc[q] = fma(to_d(x0[q][e]), v0[e], acc[q]);
#pragma unroll
                for (int e = 0; e < V; e++) {
                    double xv = to_d(x1[q][e]);
                    if (tail1 && i + 32 * V + e >= n) xv = 0.0;
                    acc[q] = fma(xv, v1[e], acc[q]);
                }
            }
        }
        for (; i < n; i += 32 * V) {
            T x0[C][V];
#pragma unroll
            for (int q = 0; q < C; q++)
                *reinterpret_cast<int4 *>(x0[q]) = __ldcs(reinterpret_cast<const int4 *>(ptr[q] + i));
#pragma unroll
            for (int q = 0; q < C; q++)
#pragma unroll
                for (int e = 0; e < V; e++) {
                    double xv = (i + e < n) ? to_d(x0[q][e]) : 0.0;
                    acc[q] = fma(xv, vs[i + e], acc[q]);
                }
        }
#pragma unroll
        for (int q = 0; q < C; q++) acc[q] = warp_sum(acc[q]);
        // lane q finishes column q
        double d = acc[0];
#pragma unroll
        for (int q = 1; q < C; q++) d = lane == q ? acc[q] : d;
        const bool valid = lane < C && g + lane < m;
        int64_t j = col[0];
#pragma unroll
        for (int q = 1; q < C; q++) j = lane == q ? col[q] : j;
        bool isv = false, iss = false;
        if (valid) {
            scan_epilogue(a, j, d, K1, K2);
            if (a.scan) {
                double az = fabs(a.out[j]);
                bool inw = a.wflag[j] != 0;
                uint8_t f = a.flags ? a.flags[j] : 3;
                isv = !inw && (f & 1) && az > a.thr_viol;
                iss = !inw && (f & 2) && a.thr_strong >= 0.0 && az >= a.thr_strong && a.s[j] > 0.0;
            }
        }
        if (a.scan) {
            warp_append(isv, (int)j, a.viol, a.nviol);
            warp_append(iss, (int)j, a.strong, a.nstrong);
        }
    }
}

// ------------------------- lockstep CV: the union of the fits' BEDPP scopes
// Column j must be scanned in a round if any pending fit keeps it (safe at lambda_k or
// lambda_{k+1}: flags & 3).  k_scope_union compacts those columns (any order: every
// result of the scan is per column); k_scope_finish decides dense (the union covers more
// than half the columns) or list mode for k_scan_batch*, and records the columns each fit
// will have read in its RoundStatus.nscope (the local live count in dense mode).
__global__ void __launch_bounds__(256) k_scope_union(int64_t p, const uint8_t *const *__restrict__ flags, int nf,
                                                     int *__restrict__ list, int *__restrict__ count) {
    for (int64_t j0 = (int64_t)blockIdx.x * blockDim.x; j0 < p; j0 += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = j0 + threadIdx.x;
        bool any = false;
        if (j < p)
            for (int f = 0; f < nf && !any; f++) any = (flags[f][j] & 3) != 0;
        warp_append(any, (int)j, list, count);
    }
}
__global__ void k_scope_finish(int64_t p, const int *__restrict__ count, const int *const *__restrict__ nlive, int nf,
                               RoundStatus *const *__restrict__ st, int *__restrict__ use_list) {
    if (threadIdx.x != 0) return;
    const int cnt = *count;
    const int ul = 2 * (int64_t)cnt <= p;
    *use_list = ul;
    for (int f = 0; f < nf; f++) st[f]->nscope = ul ? cnt : *nlive[f];
}

// ------------------------- NEXT-1: fold-batched scan (lockstep cross-validation)
// SURVEY 8(f) NEXT-1.  The K+1 fits of a CV scan the same X with different
// residuals (each zero on its held-out rows) and fold-specific c, s (Q16); one
// pass over X serves them all: per column, nf dot products against residual
// chunks staged in shared memory, then each fit's identity-(3) epilogue with its
// own KKT / strong-rule tests and compacted lists (as k_scan_fp's SCAN mode).
// X traffic falls by the number of fits; the fp64 FMAs per byte rise by the
// same factor (cfg5: 11 FMAs per 4-byte element, near the fp64 ridge).
struct FitScan {
    const double *r;                 // residual, zero on unused rows (>= n entries)
    const double *K1;                // device: sum r
    double K2;                       // 1 / n_used
    const double *c, *s;
    double *out;                     // z
    const uint8_t *flags, *wflag;
    double thr_viol, thr_strong;
    int *viol, *nviol, *strong, *nstrong;
    const int8_t *limbs;             // int8 designs: the fit's quantised residual (8 digit planes x limb_ld)
    const double *limb_scale;        //   2^-S of the quantisation (K1 then points to the quantised sum)
};
constexpr int kBatchMax = 12;        // fits per launch
constexpr int kBatchRows = 128;      // rows per pipeline stage
constexpr int kBatchStages = 3;
constexpr int kBatchThreads = 128;   // 4 warps x 4 columns per CTA
constexpr int kBatchTile = 16;       // columns per CTA

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// dynamic shared memory of one CTA: kBatchStages x (NF residual rows + 16 x-columns) x kBatchRows
__host__ __device__ constexpr size_t batch_smem(int nf, int itemsize) {
    return (size_t)kBatchStages * kBatchRows * ((size_t)8 * nf + (size_t)itemsize * kBatchTile);
}

// One CTA = 4 warps x 4 columns.  Per stage of kBatchRows rows, cp.async brings the
// fits' residual rows and the tile's x rows into shared memory (3-stage ring);
// lane l multiplies rows l, l+32, ... (conflict-free 4- / 8-byte shared loads).
// NF = the exact number of fits of the launch (the fit loops unroll completely).
template <typename T, int NF>
__global__ void __launch_bounds__(kBatchThreads, 3) k_scan_batch(const T *__restrict__ X, int64_t ld, int n, int64_t p,
                                                                  const FitScan *__restrict__ fits, int nf_unused,
                                                                  const int *__restrict__ list, const int *__restrict__ lctl) {
    extern __shared__ __align__(16) double smb[];
    __shared__ FitScan fs[NF];
    __shared__ double k1s[NF];
    constexpr int RPL = kBatchRows / 32;
    constexpr int XE = 16 / sizeof(T);                          // x elements per 16-byte copy
    constexpr size_t STAGE_D = (size_t)NF * kBatchRows + (size_t)kBatchTile * kBatchRows * sizeof(T) / 8;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x < NF) fs[threadIdx.x] = fits[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < NF) k1s[threadIdx.x] = *fs[threadIdx.x].K1;
    const int nchunk = (n + kBatchRows - 1) / kBatchRows;
    // list mode (lctl = {count, use_list}): tile positions index the union scope list
    if (list && !lctl[1]) list = nullptr;
    const int64_t P = list ? (int64_t)lctl[0] : p;
    auto colof = [&](int64_t pos) -> int64_t { return list ? (int64_t)list[pos] : pos; };
    for (int64_t g0 = (int64_t)blockIdx.x * kBatchTile; g0 < P; g0 += (int64_t)gridDim.x * kBatchTile) {
        const int ntile = (int)min((int64_t)kBatchTile, P - g0);
        // stage chunk c into ring slot b: residual rows of every fit, x rows of every tile column
        auto stage = [&](int c, int b) {
            double *rs = smb + (size_t)b * STAGE_D;
            T *xs = reinterpret_cast<T *>(rs + NF * kBatchRows);
            const int i0 = c * kBatchRows;
            const bool full = i0 + kBatchRows <= n;
            for (int e = threadIdx.x; e < NF * kBatchRows / 2; e += kBatchThreads) {
                const int f = e / (kBatchRows / 2), i = 2 * (e - f * (kBatchRows / 2));
                double *dst = rs + f * kBatchRows + i;
                if (full) cp_async16(dst, fs[f].r + i0 + i);
                else { dst[0] = i0 + i < n ? fs[f].r[i0 + i] : 0.0; dst[1] = i0 + i + 1 < n ? fs[f].r[i0 + i + 1] : 0.0; }
            }
            constexpr int XC = kBatchRows / XE;                 // 16-byte copies per column
            for (int e = threadIdx.x; e < kBatchTile * XC; e += kBatchThreads) {
                const int q = e / XC, i = (e - q * XC) * XE;
                const T *src = X + colof(g0 + min(q, ntile - 1)) * ld + i0 + i;   // past-the-end columns: a valid column, ignored
                T *dst = xs + q * kBatchRows + i;
                if (i0 + i + XE <= ld) cp_async16(dst, src);
                else {
#pragma unroll
                    for (int u = 0; u < XE; u++) dst[u] = T(0);
                }
            }
            cp_async_commit();
        };
        double acc[4][NF];
#pragma unroll
        for (int q = 0; q < 4; q++)
#pragma unroll
            for (int f = 0; f < NF; f++) acc[q][f] = 0.0;
        __syncthreads();                                       // the previous tile's stages are consumed
        stage(0, 0);
        if (nchunk > 1) stage(1, 1); else cp_async_commit();
        for (int c = 0; c < nchunk; c++) {
            cp_async_wait<1>();                                 // chunk c has landed (c + 1 may be in flight)
            __syncthreads();
            if (c + 2 < nchunk) stage(c + 2, (c + 2) % kBatchStages); else cp_async_commit();
            const double *rs = smb + (size_t)(c % kBatchStages) * STAGE_D;
            const T *xs = reinterpret_cast<const T *>(rs + NF * kBatchRows) + (wid * 4) * kBatchRows;
            const bool tail = (c + 1) * kBatchRows > n;
#pragma unroll
            for (int u = 0; u < RPL; u++) {
                const int row = 32 * u + lane;
                double rv[NF];
#pragma unroll
                for (int f = 0; f < NF; f++) rv[f] = rs[f * kBatchRows + row];
                const bool ok = !tail || c * kBatchRows + row < n; // padding rows of X may hold anything
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const double xv = ok ? to_d(xs[q * kBatchRows + row]) : 0.0;
#pragma unroll
                    for (int f = 0; f < NF; f++) acc[q][f] = fma(xv, rv[f], acc[q][f]);
                }
            }
        }
        cp_async_wait<0>();
        const int64_t j0 = g0 + wid * 4;                       // tile position of this warp's first column
        const int nv = (int)max((int64_t)0, min((int64_t)4, P - j0));
        if (nv == 0) continue;
#pragma unroll
        for (int f = 0; f < NF; f++) {
            double d = 0.0;
#pragma unroll
            for (int q = 0; q < 4; q++) {
                const double sq = warp_sum(acc[q][f]);
                d = lane == q ? sq : d;
            }
            const FitScan &F = fs[f];
            bool isv = false, iss = false;
            const int64_t j = lane < nv ? colof(j0 + lane) : 0;
            if (lane < nv) {
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

// NEXT-1 on the fp64 tensor cores: the same contraction Z = X^T R (columns x fits, summed
// over the rows) as k_scan_batch, issued as mma.m8n8k4.f64 (DMMA: 256 FMAs per
// instruction; the measured DMMA rate equals the DFMA peak, scripts/dmma_peak.cu, but
// one instruction replaces 8 FMAs per lane and the operands are fragments, not a
// shared-memory load per FMA -- k_scan_batch was bound by shared-memory bandwidth).
// M = 8 columns, N = 8 fits, K = 4 rows; a warp owns 32 columns (4 m-tiles) and all
// fits (ceil(NF / 8) n-tiles).  The K index is permuted so that lane (g, t) covers rows
// 4t..4t+3 of a 16-row group over the group's 4 MMAs: its x fragment is ONE 16-byte
// global load (fp32) of column g, its residual fragments two 16-byte shared loads per
// fit.  Residual rows stream through a 3-stage cp.async ring (fit stride 66 doubles:
// conflict-free fragment loads); the accumulators land in a shared Z tile and the
// identity-(3) epilogue, tests and list compaction run as in k_scan_batch.
constexpr int kBMThreads = 256;              // 8 warps
#ifndef BL_BM_MT
#define BL_BM_MT 4
#endif
constexpr int kBMMT = BL_BM_MT;              // m-tiles (8 columns each) per warp
constexpr int kBMCols = 64 * kBMMT;          // columns per CTA tile (8 kBMMT per warp)
#ifndef BL_BM_ROWS
#define BL_BM_ROWS 64
#endif
#ifndef BL_BM_STAGES
#define BL_BM_STAGES 3
#endif
constexpr int kBMRows = BL_BM_ROWS;          // residual rows per stage (groups of 16)
constexpr int kBMStages = BL_BM_STAGES;
constexpr int kBMStride = kBMRows + 2;       // doubles per fit in a stage
constexpr int kBMZ = 17;                     // Z tile row stride (doubles)
__host__ __device__ constexpr size_t batch_mma_smem(int nf) {
    return (size_t)kBMStages * nf * kBMStride * 8 + (size_t)kBMCols * kBMZ * 8;
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

// raw x fragment of one lane: 4 consecutive rows of one column, kept unconverted while in flight
template <typename T> struct XFrag;
template <> struct XFrag<float> {
    float4 v;
    __device__ __forceinline__ void load(const float *p, bool ok) {
        v = ok ? __ldcs(reinterpret_cast<const float4 *>(p)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __device__ __forceinline__ double get(int u) const { return u == 0 ? v.x : u == 1 ? v.y : u == 2 ? v.z : v.w; }
};
template <> struct XFrag<double> {
    double2 a, b;
    __device__ __forceinline__ void load(const double *p, bool ok) {
        a = ok ? __ldcs(reinterpret_cast<const double2 *>(p)) : make_double2(0.0, 0.0);
        b = ok ? __ldcs(reinterpret_cast<const double2 *>(p + 2)) : make_double2(0.0, 0.0);
    }
    __device__ __forceinline__ double get(int u) const { return u == 0 ? a.x : u == 1 ? a.y : u == 2 ? b.x : b.y; }
};

#ifndef BL_BM_MINB
#define BL_BM_MINB 2
#endif
#ifndef BL_BM_NOREM
#define BL_BM_NOREM 0
#endif
template <typename T, int NF>
__global__ void __launch_bounds__(kBMThreads, BL_BM_MINB) k_scan_batch_mma(const T *__restrict__ X, int64_t ld, int n, int64_t p,
                                                                   const FitScan *__restrict__ fits, int nf_unused,
                                                                   const int *__restrict__ list, const int *__restrict__ lctl) {
    extern __shared__ __align__(16) double smb[];
    __shared__ FitScan fs[NF];
    __shared__ double k1s[NF];
    // fits 0..7 on the tensor cores; 1-4 further fits (cfg5: 11 = 8 + 3) as DFMAs on the same x
    // fragments instead of a second, mostly empty 8-fit MMA tile
    constexpr int NR = (!BL_BM_NOREM && NF > 8 && NF - 8 <= 4) ? NF - 8 : 0;
    constexpr int NT = NR ? 1 : (NF + 7) / 8, MT = kBMMT;
    constexpr int GPS = kBMRows / 16;                        // 16-row groups per stage
    constexpr int D = sizeof(T) == 4 ? 2 : 1;                // x groups in flight per lane (GPS % D == 0)
    double *ring = smb;
    double *Zs = smb + (size_t)kBMStages * NF * kBMStride;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    if (threadIdx.x < NF) fs[threadIdx.x] = fits[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < NF) k1s[threadIdx.x] = *fs[threadIdx.x].K1;
    const int nstage = (n + kBMRows - 1) / kBMRows;
    double *zw = Zs + (size_t)(8 * MT * wid) * kBMZ;             // this warp's 8 MT Z rows
    // list mode (lctl = {count, use_list}): tile positions index the union scope list
    if (list && !lctl[1]) list = nullptr;
    const int64_t P = list ? (int64_t)lctl[0] : p;
    auto colof = [&](int64_t pos) -> int64_t { return list ? (int64_t)list[pos] : pos; };
    for (int64_t col0 = (int64_t)blockIdx.x * kBMCols; col0 < P; col0 += (int64_t)gridDim.x * kBMCols) {
        auto stage = [&](int sidx, int b) {
            double *rs = ring + (size_t)b * NF * kBMStride;
            const int i0 = sidx * kBMRows;
            const bool full = i0 + kBMRows <= n;
            for (int e = threadIdx.x; e < NF * kBMRows / 2; e += kBMThreads) {
                const int f = e / (kBMRows / 2), i = 2 * (e - f * (kBMRows / 2));
                double *dst = rs + f * kBMStride + i;
                if (full) cp_async16(dst, fs[f].r + i0 + i);
                else { dst[0] = i0 + i < n ? fs[f].r[i0 + i] : 0.0; dst[1] = i0 + i + 1 < n ? fs[f].r[i0 + i + 1] : 0.0; }
            }
            cp_async_commit();
        };
        // this lane's columns (clamped: past-the-end columns read a valid column, ignored)
        const T *xc[MT];
#pragma unroll
        for (int mt = 0; mt < MT; mt++) xc[mt] = X + colof(min(col0 + 8 * MT * wid + 8 * mt + g, P - 1)) * ld;
        double acc[MT][NT][2];
        double accr[MT][NR > 0 ? NR : 1];
#pragma unroll
        for (int mt = 0; mt < MT; mt++) {
#pragma unroll
            for (int nt = 0; nt < NT; nt++) { acc[mt][nt][0] = 0.0; acc[mt][nt][1] = 0.0; }
#pragma unroll
            for (int f = 0; f < (NR > 0 ? NR : 1); f++) accr[mt][f] = 0.0;
        }
        __syncthreads();                                       // the previous tile's stages are consumed
        stage(0, 0);
        if (nstage > 1) stage(1, 1); else cp_async_commit();
        // x fragments D groups ahead (group q = rows 16q..16q+15; lane rows 16q + 4t .. + 3)
        XFrag<T> xr[D][MT];
        auto xload = [&](int slot, int q) {
            const int r = 16 * q + 4 * t;
            const bool ok = r < ld;                            // ld % 4 == 0: 4 rows are inside or outside together
#pragma unroll
            for (int mt = 0; mt < MT; mt++) xr[slot][mt].load(xc[mt] + r, ok);
        };
#pragma unroll
        for (int q = 0; q < D; q++)
            if (16 * q < n) xload(q, q);
        for (int sidx = 0; sidx < nstage; sidx++) {
            cp_async_wait<1>();
            __syncthreads();
            if (sidx + 2 < nstage) stage(sidx + 2, (sidx + 2) % kBMStages); else cp_async_commit();
            const double *rs = ring + (size_t)(sidx % kBMStages) * NF * kBMStride;
#pragma unroll
            for (int kg = 0; kg < GPS; kg++) {
                const int q = sidx * GPS + kg, r0 = 16 * q;
                if (r0 >= n) break;                                 // warp-uniform
                const int slot = kg % D;
                double xa[MT][4];
                const int rr = r0 + 4 * t;
#pragma unroll
                for (int mt = 0; mt < MT; mt++)
#pragma unroll
                    for (int u = 0; u < 4; u++) xa[mt][u] = rr + u < n ? xr[slot][mt].get(u) : 0.0;   // padding rows: anything
                if (r0 + 16 * D < n) xload(slot, q + D);
                double rb[NT][4];
#pragma unroll
                for (int nt = 0; nt < NT; nt++) {
                    const int f = 8 * nt + g;
                    if (f < NF) {
                        const double2 q0 = *reinterpret_cast<const double2 *>(rs + f * kBMStride + kg * 16 + 4 * t);
                        const double2 q1 = *reinterpret_cast<const double2 *>(rs + f * kBMStride + kg * 16 + 4 * t + 2);
                        rb[nt][0] = q0.x; rb[nt][1] = q0.y; rb[nt][2] = q1.x; rb[nt][3] = q1.y;
                    } else {
                        rb[nt][0] = rb[nt][1] = rb[nt][2] = rb[nt][3] = 0.0;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; u++)
#pragma unroll
                    for (int mt = 0; mt < MT; mt++)
#pragma unroll
                        for (int nt = 0; nt < NT; nt++) dmma884(acc[mt][nt], xa[mt][u], rb[nt][u]);
                if constexpr (NR > 0) {                            // fits 8.. : this lane's 4 rows, its 4 columns
#pragma unroll
                    for (int f = 0; f < NR; f++) {
                        const double2 q0 = *reinterpret_cast<const double2 *>(rs + (8 + f) * kBMStride + kg * 16 + 4 * t);
                        const double2 q1 = *reinterpret_cast<const double2 *>(rs + (8 + f) * kBMStride + kg * 16 + 4 * t + 2);
#pragma unroll
                        for (int mt = 0; mt < MT; mt++) {
                            double v = accr[mt][f];
                            v = fma(xa[mt][0], q0.x, v);
                            v = fma(xa[mt][1], q0.y, v);
                            v = fma(xa[mt][2], q1.x, v);
                            v = fma(xa[mt][3], q1.y, v);
                            accr[mt][f] = v;
                        }
                    }
                }
            }
        }
        cp_async_wait<0>();
        // accumulators -> this warp's Z rows: lane (g, t) holds Z[8 mt + g][8 nt + 2t, +1]
#pragma unroll
        for (int mt = 0; mt < MT; mt++)
#pragma unroll
            for (int nt = 0; nt < NT; nt++) {
                zw[(8 * mt + g) * kBMZ + 8 * nt + 2 * t] = acc[mt][nt][0];
                zw[(8 * mt + g) * kBMZ + 8 * nt + 2 * t + 1] = acc[mt][nt][1];
            }
        if constexpr (NR > 0) {                                    // sum the DFMA partials over the 4 row lanes
#pragma unroll
            for (int mt = 0; mt < MT; mt++)
#pragma unroll
                for (int f = 0; f < NR; f++) {
                    double v = accr[mt][f];
                    v += __shfl_xor_sync(0xffffffffu, v, 1);
                    v += __shfl_xor_sync(0xffffffffu, v, 2);
                    if (t == 0) zw[(8 * mt + g) * kBMZ + 8 + f] = v;
                }
        }
        __syncwarp();
        const int64_t jp = col0 + 8 * MT * wid + lane;         // tile position
        const bool inr = lane < 8 * MT && jp < P;
        const int64_t j = inr ? colof(jp) : 0;
#pragma unroll
        for (int f = 0; f < NF; f++) {
            const FitScan &F = fs[f];
            bool isv = false, iss = false;
            if (inr) {
                const double d = zw[lane * kBMZ + f];
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
        __syncwarp();
    }
}

// int8 design: exact integer dot products on the tensor cores.  The fp64 vector
// v is quantised once per scan to a 64-bit fixed-point integer R_i = round(v_i
// 2^S) (|R| < 2^62) split into 8 balanced base-256 digits (k_limbs); then
//   sum_i x_ij R_i = sum_l 256^l sum_i x_ij D_il
// and each inner sum is an s8 x s8 -> s32 MMA with no rounding at all.
// mma.m16n8k32: M = 16 columns, N = 8 limbs, K = 32 rows.  Lane (g, t) loads
// 16 contiguous rows of columns j0+g and j0+g+8; k-slot <-> row mapping is
// identical for A and B so any row order is valid (the sum is exact).
__device__ __forceinline__ void mma_s8(int (&d)[4], int a0, int a1, int a2, int a3, int b0, int b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void __launch_bounds__(kScanThreads) k_scan_i8(ScanArgs a) {
    extern __shared__ __align__(16) int8_t ls[];   // 8 planes x limb_ld
    const int LL = a.limb_ld;
    {
        const int4 *src = reinterpret_cast<const int4 *>(a.limbs);
        int4 *dst = reinterpret_cast<int4 *>(ls);
        for (int i = threadIdx.x; i < 8 * LL / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const double K1 = *a.K1;
    const double K2 = a.K2 ? *a.K2 : a.K2v;
    const double scale = *a.limb_scale;
    const int64_t m = a.list ? (a.nlist ? (int64_t)*a.nlist : (int64_t)a.nlist_host) : a.p - a.j0;
    // a scope list holding every column (BEDPP kept all, lambda < ~0.5 lambda_max) is read
    // as the dense range: same columns, no index indirection, sequential DRAM pages
    const int *__restrict__ list = (a.list && m == a.p) ? nullptr : a.list;
    const int64_t jd = list ? 0 : a.j0;
    const int lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarp = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int8_t *X = reinterpret_cast<const int8_t *>(a.X);
    const int ld = (int)a.ld;
    // per-lane 2^(8 l - S) weights for the two limbs this lane accumulates
    const double w0 = ldexp(scale, 16 * t), w1 = ldexp(scale, 16 * t + 8);
    for (int64_t g0 = gw * 16; g0 < m; g0 += nwarp * 16) {
        int64_t ia = g0 + g < m ? g0 + g : m - 1;
        int64_t ib = g0 + g + 8 < m ? g0 + g + 8 : m - 1;
        if (a.rev) { ia = m - 1 - ia; ib = m - 1 - ib; }
        int64_t ja = list ? (int64_t)list[ia] : jd + ia;
        int64_t jb = list ? (int64_t)list[ib] : jd + ib;
        const int8_t *pa = X + ja * a.ld, *pb = X + jb * a.ld;
        int acc[4] = {0, 0, 0, 0};
        const int8_t *lg = ls + g * LL + 16 * t;
        int r = 0;
        for (; r + 256 <= ld; r += 256) {     // four 64-row blocks per step: 8 loads in flight per lane
            int4 xa[4], xb[4], l[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                xa[u] = __ldcs(reinterpret_cast<const int4 *>(pa + r + 64 * u + 16 * t));
                xb[u] = __ldcs(reinterpret_cast<const int4 *>(pb + r + 64 * u + 16 * t));
            }
#pragma unroll
            for (int u = 0; u < 4; u++) l[u] = *reinterpret_cast<const int4 *>(lg + r + 64 * u);
#pragma unroll
            for (int u = 0; u < 4; u++) {
                mma_s8(acc, xa[u].x, xb[u].x, xa[u].y, xb[u].y, l[u].x, l[u].y);
                mma_s8(acc, xa[u].z, xb[u].z, xa[u].w, xb[u].w, l[u].z, l[u].w);
            }
        }
        for (; r + 128 <= ld; r += 128) {     // two 64-row blocks per step
            int4 xa0 = __ldcs(reinterpret_cast<const int4 *>(pa + r + 16 * t));
            int4 xb0 = __ldcs(reinterpret_cast<const int4 *>(pb + r + 16 * t));
            int4 xa1 = __ldcs(reinterpret_cast<const int4 *>(pa + r + 64 + 16 * t));
            int4 xb1 = __ldcs(reinterpret_cast<const int4 *>(pb + r + 64 + 16 * t));
            int4 l0 = *reinterpret_cast<const int4 *>(lg + r);
            int4 l1 = *reinterpret_cast<const int4 *>(lg + r + 64);
            mma_s8(acc, xa0.x, xb0.x, xa0.y, xb0.y, l0.x, l0.y);
            mma_s8(acc, xa0.z, xb0.z, xa0.w, xb0.w, l0.z, l0.w);
            mma_s8(acc, xa1.x, xb1.x, xa1.y, xb1.y, l1.x, l1.y);
            mma_s8(acc, xa1.z, xb1.z, xa1.w, xb1.w, l1.z, l1.w);
        }
        for (; r < ld; r += 64) {             // ragged tail (ld is a multiple of 16)
            bool in = r + 16 * t < ld;
            int4 xa0 = in ? __ldcs(reinterpret_cast<const int4 *>(pa + r + 16 * t)) : make_int4(0, 0, 0, 0);
            int4 xb0 = in ? __ldcs(reinterpret_cast<const int4 *>(pb + r + 16 * t)) : make_int4(0, 0, 0, 0);
            int4 l0 = *reinterpret_cast<const int4 *>(lg + r);
            mma_s8(acc, xa0.x, xb0.x, xa0.y, xb0.y, l0.x, l0.y);
            mma_s8(acc, xa0.z, xb0.z, xa0.w, xb0.w, l0.z, l0.w);
        }
        // acc[0], acc[1]: column ja, limbs 2t, 2t+1; acc[2], acc[3]: column jb
        double da = fma((double)acc[0], w0, (double)acc[1] * w1);
        double db = fma((double)acc[2], w0, (double)acc[3] * w1);
        da += __shfl_xor_sync(0xffffffffu, da, 1);
        db += __shfl_xor_sync(0xffffffffu, db, 1);
        da += __shfl_xor_sync(0xffffffffu, da, 2);
        db += __shfl_xor_sync(0xffffffffu, db, 2);
        // lanes t==0 finish column A, t==1 column B
        bool valid = (t == 0 && g0 + g < m) || (t == 1 && g0 + g + 8 < m);
        int64_t j = t == 0 ? ja : jb;
        double d = t == 0 ? da : db;
        bool isv = false, iss = false;
        if (valid) {
            scan_epilogue(a, j, d, K1, K2);
            if (a.scan) {
                double az = fabs(a.out[j]);
                bool inw = a.wflag[j] != 0;
                uint8_t f = a.flags ? a.flags[j] : 3;
                isv = !inw && (f & 1) && az > a.thr_viol;
                iss = !inw && (f & 2) && a.thr_strong >= 0.0 && az >= a.thr_strong && a.s[j] > 0.0;
            }
        }
        if (a.scan) {
            warp_append(isv, (int)j, a.viol, a.nviol);
            warp_append(iss, (int)j, a.strong, a.nstrong);
        }
    }
}

// NEXT-1 for int8 designs: the fold-batched scan on the integer tensor cores.  Every fit's
// residual is quantised to 8 digit planes (k_limbs, Q27); one pass over X serves all fits:
// per 32-row k-step a lane's A fragment (two columns x 16 rows, k_scan_i8's mapping) is loaded
// ONCE and multiplied by each fit's B fragment (its 8 digit planes x the same rows) --
// mma.m16n8k32.s8, exact int32 accumulation per fit.  The fits' digit planes stream through
// shared memory in 256-row chunks (double-buffered cp.async; the whole set would not fit at
// n = 2898 x 11 fits).  Epilogue per fit as k_scan_batch (identity (3) with the fit's c, s,
// quantised sum and 1/n_used; KKT / strong-rule tests; list compaction).
constexpr int kBIRows = 256;                   // rows per chunk
__host__ __device__ constexpr size_t batch_i8_smem(int nf) { return (size_t)2 * nf * 8 * kBIRows; }

template <int NF>
__global__ void __launch_bounds__(kScanThreads) k_scan_batch_i8(const int8_t *__restrict__ X, int64_t ld, int n, int64_t p,
                                                              const FitScan *__restrict__ fits, int limb_ld,
                                                              const int *__restrict__ list, const int *__restrict__ lctl) {
    extern __shared__ __align__(16) int8_t lsb[];      // [2][NF][8][kBIRows]
    __shared__ FitScan fs[NF];
    __shared__ double k1s[NF], scs[NF];
    if (threadIdx.x < NF) fs[threadIdx.x] = fits[threadIdx.x];
    __syncthreads();
    if (threadIdx.x < NF) { k1s[threadIdx.x] = *fs[threadIdx.x].K1; scs[threadIdx.x] = *fs[threadIdx.x].limb_scale; }
    if (list && !lctl[1]) list = nullptr;
    const int64_t P = list ? (int64_t)lctl[0] : p;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t = lane & 3;
    const int nchunk = (int)((ld + kBIRows - 1) / kBIRows);
    constexpr int STAGE = NF * 8 * kBIRows;
    // CTA tile = 8 warps x 16 columns
    for (int64_t c0 = (int64_t)blockIdx.x * 128; c0 < P; c0 += (int64_t)gridDim.x * 128) {
        const int64_t g0 = c0 + 16 * wid;
        const int64_t ia = min(g0 + g, P - 1), ib = min(g0 + g + 8, P - 1);
        const int64_t ja = list ? (int64_t)list[ia] : ia, jb = list ? (int64_t)list[ib] : ib;
        const int8_t *pa = X + ja * ld, *pb = X + jb * ld;
        int acc[NF][4];
#pragma unroll
        for (int f = 0; f < NF; f++) acc[f][0] = acc[f][1] = acc[f][2] = acc[f][3] = 0;
        auto stage = [&](int ch, int b) {
            int8_t *dst0 = lsb + (size_t)b * STAGE;
            const int r0 = ch * kBIRows;
            for (int e = threadIdx.x; e < NF * 8 * (kBIRows / 16); e += kScanThreads) {
                const int fl = e / (kBIRows / 16), q = e - fl * (kBIRows / 16);
                const int f = fl >> 3, l = fl & 7;
                int8_t *dst = dst0 + (size_t)fl * kBIRows + 16 * q;
                const int r = r0 + 16 * q;
                if (r + 16 <= limb_ld) cp_async16(dst, fs[f].limbs + (size_t)l * limb_ld + r);
                else *reinterpret_cast<int4 *>(dst) = make_int4(0, 0, 0, 0);
            }
            cp_async_commit();
        };
        __syncthreads();                                   // the previous tile's stages are consumed
        stage(0, 0);
        for (int ch = 0; ch < nchunk; ch++) {
            if (ch + 1 < nchunk) stage(ch + 1, (ch + 1) & 1); else cp_async_commit();
            cp_async_wait<1>();
            __syncthreads();
            const int8_t *st = lsb + (size_t)(ch & 1) * STAGE;
            const int r0 = ch * kBIRows;
#pragma unroll
            for (int u = 0; u < kBIRows / 64; u++) {
                const int r = r0 + 64 * u + 16 * t;
                const bool in = r < ld;                     // ld % 16 == 0: 16 rows in or out together
                const int4 xa = in ? __ldcs(reinterpret_cast<const int4 *>(pa + r)) : make_int4(0, 0, 0, 0);
                const int4 xb = in ? __ldcs(reinterpret_cast<const int4 *>(pb + r)) : make_int4(0, 0, 0, 0);
#pragma unroll
                for (int f = 0; f < NF; f++) {
                    const int4 l = *reinterpret_cast<const int4 *>(st + (size_t)(f * 8 + g) * kBIRows + 64 * u + 16 * t);
                    mma_s8(acc[f], xa.x, xb.x, xa.y, xb.y, l.x, l.y);
                    mma_s8(acc[f], xa.z, xb.z, xa.w, xb.w, l.z, l.w);
                }
            }
            __syncthreads();                               // stage (ch & 1) is rewritten at ch + 2
        }
        cp_async_wait<0>();
        // acc[f][0], acc[f][1]: column ja, limbs 2t, 2t+1; acc[f][2], acc[f][3]: column jb
        const bool valid = (t == 0 && g0 + g < P) || (t == 1 && g0 + g + 8 < P);
        const int64_t j = t == 0 ? ja : jb;
#pragma unroll
        for (int f = 0; f < NF; f++) {
            const double w0 = ldexp(scs[f], 16 * t), w1 = ldexp(scs[f], 16 * t + 8);
            double da = fma((double)acc[f][0], w0, (double)acc[f][1] * w1);
            double db = fma((double)acc[f][2], w0, (double)acc[f][3] * w1);
            da += __shfl_xor_sync(0xffffffffu, da, 1);
            db += __shfl_xor_sync(0xffffffffu, db, 1);
            da += __shfl_xor_sync(0xffffffffu, da, 2);
            db += __shfl_xor_sync(0xffffffffu, db, 2);
            const double d = t == 0 ? da : db;
            const FitScan &F = fs[f];
            bool isv = false, iss = false;
            if (valid) {
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

// Quantise v (n entries, fp64) to 8 balanced base-256 int8 digit planes.  One
// block.  S = 61 - floor(log2 max|v|) keeps |R| < 2^62; sum_v = sum R_i 2^-S
// is accumulated exactly in 128-bit integers.
__global__ void k_limbs(const double *__restrict__ v, int n, int limb_ld, int8_t *__restrict__ limbs,
                        double *__restrict__ scale_out, double *__restrict__ sumv_out) {
    __shared__ double sh[32];
    __shared__ long long hi_sh[32];
    __shared__ unsigned long long lo_sh[32];
    double mx = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, fabs(v[i]));
    mx = block_max(mx, sh);
    int S = mx > 0.0 ? 61 - ilogb(mx) : 0;
    __int128 acc = 0;
    for (int i = threadIdx.x; i < limb_ld; i += blockDim.x) {
        long long R = i < n ? llrint(ldexp(v[i], S)) : 0;
        acc += (__int128)R;
#pragma unroll
        for (int l = 0; l < 8; l++) {
            int dgt = (int)(R & 0xFF);
            if (dgt >= 128) dgt -= 256;
            R = (R - dgt) >> 8;
            limbs[(size_t)l * limb_ld + i] = (int8_t)dgt;
        }
    }
    // exact block reduction of the 128-bit partial sums
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    unsigned long long lo = (unsigned long long)acc;
    long long hi = (long long)(acc >> 64);
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long lo2 = __shfl_xor_sync(0xffffffffu, lo, o);
        long long hi2 = __shfl_xor_sync(0xffffffffu, hi, o);
        unsigned long long s = lo + lo2;
        hi = hi + hi2 + (s < lo ? 1 : 0);
        lo = s;
    }
    if (lane == 0) { lo_sh[wid] = lo; hi_sh[wid] = hi; }
    __syncthreads();
    if (threadIdx.x == 0) {
        __int128 tot = 0;
        for (int w = 0; w < nw; w++) tot += ((__int128)hi_sh[w] << 64) + (__int128)lo_sh[w];
        double sc = ldexp(1.0, -S);
        // exact int128 -> double with one rounding: split hi/lo 64-bit halves
        long long th = (long long)(tot >> 64);
        unsigned long long tl = (unsigned long long)tot;
        double val = ldexp((double)th, 64) + (double)tl;
        *scale_out = sc;
        *sumv_out = val * sc;
    }
}

// --------------------------------------------------- a3: lambda_max, j*
// Two-stage deterministic argmax of |a_j| over non-constant columns (ties ->
// lowest j).  Stage 1: per-block best; stage 2: one block.
__global__ void k_argmax1(const double *__restrict__ a, const double *__restrict__ s, int64_t p,
                          double *__restrict__ bv, long long *__restrict__ bi, int *__restrict__ nlive) {
    __shared__ double sv[32];
    __shared__ long long si[32];
    double best = -1.0;
    long long bj = -1;
    int live = 0;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < p; j += (int64_t)gridDim.x * blockDim.x) {
        if (s[j] > 0.0) {
            live++;
            double v = fabs(a[j]);
            if (v > best) { best = v; bj = j; }
        }
    }
    int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        long long j2 = __shfl_xor_sync(0xffffffffu, bj, o);
        if (v2 > best || (v2 == best && j2 >= 0 && (bj < 0 || j2 < bj))) { best = v2; bj = j2; }
        live += __shfl_xor_sync(0xffffffffu, live, o);
    }
    if (lane == 0) { sv[wid] = best; si[wid] = bj; }
    if (lane == 0 && live) atomicAdd(nlive, live);
    __syncthreads();
    if (threadIdx.x == 0) {
        best = -1.0;
        bj = -1;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++)
            if (sv[w] > best || (sv[w] == best && si[w] >= 0 && (bj < 0 || si[w] < bj))) {
                best = sv[w]; bj = si[w];
            }
        bv[blockIdx.x] = best;
        bi[blockIdx.x] = bj;
    }
}

// Stage 2: one block of 256 threads reduces the per-block bests (strided loads,
// then warp shuffles and one shared-memory round); the (value, lowest index) order
// is associative, so the result does not depend on the reduction shape.
__device__ __forceinline__ void argmax_merge(double &best, long long &bj, double v2, long long j2) {
    if (v2 > best || (v2 == best && j2 >= 0 && (bj < 0 || j2 < bj))) { best = v2; bj = j2; }
}
__global__ void __launch_bounds__(256) k_argmax2(const double *__restrict__ bv, const long long *__restrict__ bi, int nb,
                                                 const double *__restrict__ a, const double *__restrict__ c,
                                                 const double *__restrict__ s, double alpha,
                                                 const int *__restrict__ nlive, PrepScalars *ps) {
    __shared__ double sv[8];
    __shared__ long long si[8];
    double best = -1.0;
    long long bj = -1;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) argmax_merge(best, bj, bv[b], bi[b]);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        const long long j2 = __shfl_xor_sync(0xffffffffu, bj, o);
        argmax_merge(best, bj, v2, j2);
    }
    if (lane == 0) { sv[wid] = best; si[wid] = bj; }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int w = 1; w < (int)(blockDim.x >> 5); w++) argmax_merge(best, bj, sv[w], si[w]);
    ps->jstar = bj;
    ps->n_live = *nlive;
    if (bj >= 0) {
        ps->A = best * ps->inv_nt;
        ps->lmax = ps->A / alpha;
        ps->sigma = a[bj] >= 0.0 ? 1.0 : -1.0;
        ps->c_star = c[bj];
        ps->s_star = s[bj];
        ps->inv_s_star = s[bj] > 0.0 ? 1.0 / s[bj] : 0.0;
    } else {
        ps->A = 0.0; ps->lmax = 0.0; ps->sigma = 1.0; ps->c_star = 0.0; ps->s_star = 0.0; ps->inv_s_star = 0.0;
    }
}

// v_i = x_{i j*} - c_*  (rows in the mask), the vector of identity (1).  One block.
template <typename T>
__global__ void k_xstar(const T *__restrict__ X, int64_t ld, int n, int vlen, const uint8_t *__restrict__ mask,
                        PrepScalars *ps, double *__restrict__ v) {
    __shared__ double sh[32];
    long long js = ps->jstar;
    double cs = ps->c_star;
    double acc = 0.0;
    for (int i = threadIdx.x; i < vlen; i += blockDim.x) {
        double x = (js >= 0 && i < n && (!mask || mask[i])) ? to_d(X[js * ld + i]) - cs : 0.0;
        v[i] = x;
        acc += x;
    }
    acc = block_sum(acc, sh);
    if (threadIdx.x == 0) ps->sum_v = acc;
}

// ------------------------------------------------------ a5: BEDPP safe sets (G3)
// For every non-constant column: bit0 = safe at lambda_k, bit1 = safe at
// lambda_{k+1} (lam_next <= 0: none).  Columns with either bit set form the
// scan scope S_k U S_{k+1} ("only needs to scan the features not
// discarded by BEDPP").  Inequality and margin: DESIGN.md Q8/Q9 (derived from
// the EDPP rule cited at P:211; the paper does not print it).
__device__ __forceinline__ bool bedpp_discard(double aj, double bj, bool is_star, double A, double Y2, double nd,
                                              double sigma, double alpha, double lam) {
    if (is_star) return false;
    double L = alpha * lam;
    if (L >= A) return true;
    double mm = nd * (1.0 + lam * (1.0 - alpha));
    double rad = fmax(0.0, mm * Y2 - nd * nd * A * A);
    double rhs = 2.0 * nd * L * A - (A - L) * sqrt(rad);
    double t1 = (A + L) * aj;
    double t2 = (A - L) * (nd * A / mm) * sigma * bj;
    double lhs = fabs(t1 - t2);
    double margin = 1e-12 * (fabs(rhs) + fabs(t1) + fabs(t2));
    return lhs < rhs - margin;
}

// One atomic per 1024 columns per counter: threads take 4 columns each, the
// block's scope entries are ranked with warp ballots + a shared prefix (a
// per-warp atomic on one counter serialised at the L2: ~80 us for 1.3M columns).
__global__ void __launch_bounds__(256) k_bedpp(int64_t p, const double *__restrict__ s, const double *__restrict__ a,
                                               const double *__restrict__ b, const PrepScalars *__restrict__ ps,
                                               double alpha, double lam, double lam_next, int use_bedpp,
                                               uint8_t *__restrict__ flags, int *__restrict__ scope, RoundStatus *st) {
    __shared__ int wsc[8], wsf[8], bsc;
    const double A = ps->A, Y2 = ps->Y2, nd = ps->nt, sg = ps->sigma;
    const long long js = ps->jstar;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t base = (int64_t)blockIdx.x * 1024; base < p; base += (int64_t)gridDim.x * 1024) {
        uint8_t f[4];
        int nsc = 0, nsf = 0;
#pragma unroll
        for (int u = 0; u < 4; u++) {
            const int64_t j = base + u * 256 + threadIdx.x;
            f[u] = 0;
            if (j < p && s[j] > 0.0) {
                const bool star = j == js;
                const bool sk = !use_bedpp || !bedpp_discard(a[j], b[j], star, A, Y2, nd, sg, alpha, lam);
                const bool sn = lam_next > 0.0 && (!use_bedpp || !bedpp_discard(a[j], b[j], star, A, Y2, nd, sg, alpha, lam_next));
                f[u] = (uint8_t)((sk ? 1 : 0) | (sn ? 2 : 0));
            }
            if (j < p) flags[j] = f[u];
            nsc += f[u] != 0;
            nsf += (f[u] & 1) != 0;
        }
        // rank this thread's scope entries within the block (order: thread-major)
        int isc = nsc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int v = __shfl_up_sync(0xffffffffu, isc, o); if (lane >= o) isc += v; }
        const int wtot = __shfl_sync(0xffffffffu, isc, 31);
        const int wf = warp_sum_i(nsf);
        if (lane == 0) { wsc[wid] = wtot; wsf[wid] = wf; }
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0, tf = 0;
            for (int w = 0; w < 8; w++) { const int c0 = wsc[w]; wsc[w] = run; run += c0; tf += wsf[w]; }
            bsc = (scope && run) ? atomicAdd(&st->nscope, run) : 0;
            if (tf) atomicAdd(&st->nsafe, tf);
        }
        __syncthreads();
        if (scope) {
            int pos = bsc + wsc[wid] + isc - nsc;
#pragma unroll
            for (int u = 0; u < 4; u++)
                if (f[u]) scope[pos++] = (int)(base + u * 256 + threadIdx.x);
        }
        __syncthreads();
    }
}

// a6 at the first solved lambda: z = a/n is the null solution's correlation, so
// the strong set needs no scan (virtual lambda_0 = lambda_max).
__global__ void k_ssr_init(int64_t p, const double *__restrict__ a, const double *__restrict__ s,
                           const uint8_t *__restrict__ flags, const uint8_t *__restrict__ wflag,
                           const PrepScalars *__restrict__ ps, double thr, double *__restrict__ z,
                           int *__restrict__ strong, int *__restrict__ nstrong) {
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t pr = (p + 31) / 32 * 32;
    const double inv = ps->inv_nt;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < pr; j += stride) {
        bool hit = false;
        if (j < p) {
            double zj = s[j] > 0.0 ? a[j] * inv : 0.0;
            z[j] = zj;
            hit = s[j] > 0.0 && (flags[j] & 1) && !wflag[j] && fabs(zj) >= thr;
        }
        warp_append(hit, (int)j, strong, nstrong);
    }
}

// working-set upload in one launch: the host's pinned staging (sorted columns, slots, cyclic
// order, this shard's new columns) is read in place over the host link (zero-copy) and
// scattered into the device arrays; new columns get their "in W" flag
__global__ void k_upload_W(const int *__restrict__ h, int nW, int nnew, int write_w, int *__restrict__ W,
                           int *__restrict__ Wst, int *__restrict__ ord, int *__restrict__ fresh,
                           uint8_t *__restrict__ wflag) {
    const int total = max(nW, nnew);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
        if (i < nW) {
            if (write_w) { W[i] = h[i]; Wst[i] = h[nW + i]; }
            ord[i] = h[2 * nW + i];
        }
        if (i < nnew) {
            const int j = h[3 * nW + i];
            fresh[i] = j;
            wflag[j] = 1;
        }
    }
}

// The round's status and the first `pre` entries of both index lists, written by ONE
// block straight into pinned host memory (mapped, UVA): one launch instead of three
// device->host copies per KKT round, and only the entries the counts say exist.
// Visible to the host once the stream is synchronised (the kernel has completed).
__global__ void k_round_out(const RoundStatus *__restrict__ st, const int *__restrict__ viol,
                            const int *__restrict__ strong, int pre, RoundStatus *hst, int *hpre, int stride) {
    static_assert(sizeof(RoundStatus) % 8 == 0, "RoundStatus is copied in 8-byte words");
    const long long *s = reinterpret_cast<const long long *>(st);
    long long *h = reinterpret_cast<long long *>(hst);
    for (int i = threadIdx.x; i < (int)(sizeof(RoundStatus) / 8); i += blockDim.x) h[i] = s[i];
    const int nv = min(max(st->nviol, 0), pre), ns = min(max(st->nstrong, 0), pre);
    for (int i = threadIdx.x; i < nv; i += blockDim.x) hpre[i] = viol[i];
    for (int i = threadIdx.x; i < ns; i += blockDim.x) hpre[stride + i] = strong[i];
}

__global__ void k_set_flags(const int *__restrict__ idx, int cnt, uint8_t *__restrict__ f, uint8_t val) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < cnt) f[idx[i]] = val;
}

// ------------------------------------------ a8: coordinate descent on W (G6)
// ONE persistent CTA per fit.  Thread t owns rows t, t+T, ..., t+(R-1)T and
// keeps their residuals r_i in REGISTERS for the whole solve, so a residual
// update touches no memory and needs no synchronisation; each coordinate costs
// one warp-shuffle reduction plus one __syncthreads (partials double-buffered).
// Slot metadata (column index, c_j, 1/s_j, beta_j) lives in shared memory; the
// next column is prefetched into registers while the current one is reduced.
// Cyclic order = ascending global column index (W is kept sorted), mirroring
// the oracle:
//   z  = sum_i (x_ij - c_j) r_i / (n s_j) + b_j
//   b' = S(z, lambda alpha) / (1 + lambda (1 - alpha))
//   r -= (b' - b_j) (x_j - c_j)/s_j            (all rows, incl. held-out ones)
// Active cycling between full passes, convergence rule Q6 (with noise floor);
// a fit is accepted only after a converged FULL pass over W.
struct CdArgs {
    const void *X;
    int64_t ld;
    int n;
    const int *W;           // sorted local column indices
    int nW;
    const double *c, *s;
    double *beta;           // p entries (global, by local column)
    double *r;              // ld entries: in/out residual on every row
    double *r_scan;         // ld entries out: r on used rows, 0 elsewhere
    const uint8_t *mask;    // nullptr: every row used
    double lam_alpha, inv_den, inv_n, tol, floor_;
    int max_iter;
    double *betaW_out;      // 3*nW entries: beta, c, s per slot (slot order)
    RoundStatus *st;
};

// shared-memory bytes per W slot: beta, c, 1/s (fp64) + column index, active list (int32)
constexpr int kCdSlotBytes = 32;

template <typename T, bool MASK, int RM>
__global__ void __launch_bounds__(RM >= 16 ? 1024 : 512, 1) k_cd(CdArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double part[2][32];
    __shared__ int wcount[33];
    const int T_ = blockDim.x, t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = T_ >> 5;
    const int n = a.n, nW = a.nW;
    const int R = (n + T_ - 1) / T_;
    double *bw = sm;                                   // beta_j
    double *cw = bw + nW;                              // c_j
    double *iw = cw + nW;                              // 1/s_j
    int *Ws = reinterpret_cast<int *>(iw + nW);        // column index
    int *act = Ws + nW;                                // active slot list
    for (int w = t; w < nW; w += T_) {
        int j = a.W[w];
        Ws[w] = j;
        bw[w] = a.beta[j];
        cw[w] = a.c[j];
        iw[w] = 1.0 / a.s[j];
    }
    double rr[RM];
    unsigned mbits = 0;
#pragma unroll
    for (int k = 0; k < RM; k++) {
        int i = t + k * T_;
        rr[k] = (k < R && i < n) ? a.r[i] : 0.0;
        bool use = k < R && i < n && (!MASK || a.mask[i]);
        mbits |= (use ? 1u : 0u) << k;
    }
    __syncthreads();
    const T *X = reinterpret_cast<const T *>(a.X);
    const long long clk0 = clock64();
    int passes = 0, status = 0, buf = 0;
    long long visits = 0, updates = 0;

    // one sweep over slots list[0..len) (list == nullptr => 0..len).  Columns
    // stream through a 2-deep register ring (loop unrolled by 2: buffer u is
    // consumed at step q and refilled with column q + 2).
    auto sweep = [&](const int *list, int len, double &dmax, double &bmax) {
        dmax = 0.0;
        bmax = 0.0;
        if (len == 0) return;
        T xb[2][RM];
        visits += len;
        auto load_col = [&](T (&x)[RM], int qq) {
            if (qq < len) {
                const T *col = X + (int64_t)Ws[list ? list[qq] : qq] * a.ld;
#pragma unroll
                for (int k = 0; k < RM; k++) { int i = t + k * T_; x[k] = (k < R && i < n) ? col[i] : T(0); }
            }
        };
        load_col(xb[0], 0);
        load_col(xb[1], 1);
        for (int q0 = 0; q0 < len; q0 += 2) {
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const int q = q0 + u;
                if (q < len) {
                    const int w = list ? list[q] : q;
                    const double b_old = bw[w], cj = cw[w], isj = iw[w];
                    double p0 = 0.0, p1 = 0.0;
#pragma unroll
                    for (int k = 0; k < RM; k += 2) {
                        if ((mbits >> k) & 1u) p0 = fma(to_d(xb[u][k]) - cj, rr[k], p0);
                        if (k + 1 < RM && ((mbits >> (k + 1)) & 1u)) p1 = fma(to_d(xb[u][k + 1]) - cj, rr[k + 1], p1);
                    }
                    double pt = warp_sum(p0 + p1);
                    if (lane == 0) part[buf][wid] = pt;
                    __syncthreads();
                    double s0 = 0.0, s1 = 0.0;
                    int v = 0;
                    for (; v + 3 < nw; v += 4) {
                        double2 h0 = *reinterpret_cast<const double2 *>(&part[buf][v]);
                        double2 h1 = *reinterpret_cast<const double2 *>(&part[buf][v + 2]);
                        s0 += h0.x + h0.y;
                        s1 += h1.x + h1.y;
                    }
                    for (; v < nw; v++) s0 += part[buf][v];
                    const double z = (s0 + s1) * a.inv_n * isj + b_old;
                    const double bn = soft_threshold(z, a.lam_alpha) * a.inv_den;
                    const double d = bn - b_old;
                    if (d != 0.0) {
                        updates++;
                        const double f = d * isj;
#pragma unroll
                        for (int k = 0; k < RM; k++)
                            if (k < R) rr[k] = fma(-f, to_d(xb[u][k]) - cj, rr[k]);
                        if (t == 0) bw[w] = bn;
                    }
                    dmax = fmax(dmax, fabs(d));
                    bmax = fmax(bmax, fabs(bn));
                    buf ^= 1;
                    load_col(xb[u], q + 2);
                }
            }
        }
        __syncthreads();     // bw visible before the next list build
    };

    // ordered block-wide compaction of the nonzero slots into act[]
    auto build_active = [&]() -> int {
        int total = 0;
        for (int base = 0; base < nW; base += T_) {
            int w = base + t;
            bool nz = w < nW && bw[w] != 0.0;
            unsigned m = __ballot_sync(0xffffffffu, nz);
            if (lane == 0) wcount[wid] = __popc(m);
            __syncthreads();
            if (t == 0) {
                int run = 0;
                for (int u = 0; u < nw; u++) { int c0 = wcount[u]; wcount[u] = run; run += c0; }
                wcount[32] = run;
            }
            __syncthreads();
            if (nz) act[total + wcount[wid] + __popc(m & ((1u << lane) - 1u))] = w;
            total += wcount[32];
            __syncthreads();
        }
        return total;
    };

    for (;;) {
        for (;;) {                               // active cycling (acceleration only)
            int na = build_active();
            if (na == 0) break;
            double dmax, bmax;
            sweep(act, na, dmax, bmax);
            if (++passes > a.max_iter) { status = 3; break; }
            if (dmax <= a.tol * bmax || dmax <= a.floor_) break;
        }
        if (status) break;
        double dmax, bmax;
        sweep(nullptr, nW, dmax, bmax);          // full pass over W
        if (++passes > a.max_iter) { status = 3; break; }
        if (dmax <= a.tol * bmax || dmax <= a.floor_) break;
    }
    __syncthreads();
    // write back + record statistics (a11)
    double rss = 0.0, sr = 0.0;
#pragma unroll
    for (int k = 0; k < RM; k++) {
        int i = t + k * T_;
        if (k < R && i < n) {
            double v = rr[k];
            bool use = (mbits >> k) & 1u;
            a.r[i] = v;
            a.r_scan[i] = use ? v : 0.0;
            if (use) { rss = fma(v, v, rss); sr += v; }
        }
    }
    for (int i = n + t; i < (int)a.ld; i += T_) a.r_scan[i] = 0.0;
    double l1 = 0.0, l2 = 0.0, nnz = 0.0;
    for (int w = t; w < nW; w += T_) {
        double b = bw[w];
        int jw = Ws[w];
        a.beta[jw] = b;
        a.betaW_out[w] = b;
        a.betaW_out[nW + w] = cw[w];
        a.betaW_out[2 * nW + w] = a.s[jw];
        l1 += fabs(b);
        l2 = fma(b, b, l2);
        nnz += b != 0.0 ? 1.0 : 0.0;
    }
    double *sh = &part[0][0];
    rss = block_sum(rss, sh);
    sr = block_sum(sr, sh);
    l1 = block_sum(l1, sh);
    l2 = block_sum(l2, sh);
    nnz = block_sum(nnz, sh);
    if (t == 0) {
        a.st->cd_passes = passes;
        a.st->cd_status = status;
        a.st->rss = rss;
        a.st->sumr = sr;
        a.st->l1 = l1;
        a.st->l2 = l2;
        a.st->nnz = (int)nnz;
        a.st->cd_visits = visits;
        a.st->cd_updates = updates;
        a.st->cd_cycles = clock64() - clk0;
    }
}

// ------------------------------ NEXT-3: logistic (binomial) path, IRLS + weighted CD
// SURVEY 8(f) NEXT-3; objective QL1: mean_i [log(1+e^eta_i) - y_i eta_i]
// + lambda (alpha |b|_1 + (1-alpha)/2 |b|^2), eta = b0 + X~ b.  ONE persistent CTA per
// fit, the row layout of k_cd: thread t owns rows t + kT and keeps their working
// residual rho_i = w_i (zr_i - eta_i) in registers.  Per IRLS (outer) iteration:
//   pi = sigmoid(eta), w = max(pi (1-pi), 1e-5) (QL5), rho = y - pi on used rows;
//   v_j = x~_j' W x~_j / n for every slot (one warp per column);
//   weighted CD (active cycling, then full passes over W), intercept first per pass:
//     b0 += sum rho / sum w;  rho -= d0 w
//     u = x~_j' rho / n + v_j b_j;  b' = S(u, lambda alpha) / (v_j + lambda (1-alpha));
//     rho -= (b' - b_j) w x~_j
//   eta = b0 + X~_A b_A recomputed from the columns (all rows, held-out ones too);
// until an outer iteration moves b by <= tol max|b| and b0 by <= tol max(1,|b0|) (QL6).
// Output r_scan = y - pi on used rows (the KKT / strong-rule scan vector, SPEC S:312
// "SSR screening uses z_j = x~_j'(y - p^)/n").  The weights are held in fp32: the
// fixed point depends only on the exact gradient y - pi (QL5).
struct CdLogitArgs {
    const void *X;
    int64_t ld;
    int n;
    const int *W;           // sorted slot columns (view)
    int nW;
    const double *c, *s;
    double *beta;           // by view column
    double *eta;            // ld entries: linear predictor on every row (in/out)
    const double *y;        // n entries, 0/1
    double *r_scan;         // ld entries out: y - pi on used rows, 0 elsewhere
    const uint8_t *mask;
    double lam_alpha, lam_l2, inv_n, tol, floor_;
    int max_iter;
    double *betaW_out;      // 3 nW: beta, c, s per slot
    RoundStatus *st;        // st->b0 in/out
};

constexpr int kCdLogitSlotBytes = 56;    // beta, c, 1/s, v, beta_prev, 1/(v + l2) (fp64) + column, active (int32)

__device__ __forceinline__ double sigmoid_d(double t) {
    return t >= 0.0 ? 1.0 / (1.0 + exp(-t)) : exp(t) / (1.0 + exp(t));
}

template <typename T, bool MASK, int RM>
__global__ void __launch_bounds__(RM >= 16 ? 1024 : 512, 1) k_cd_logit(CdLogitArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double part[2][32];
    __shared__ double red[32];
    __shared__ int wcount[33];
    const int T_ = blockDim.x, t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = T_ >> 5;
    const int n = a.n, nW = a.nW;
    const int R = (n + T_ - 1) / T_;
    double *bw = sm, *cw = bw + nW, *iw = cw + nW, *vw = iw + nW, *bo = vw + nW, *dv = bo + nW;
    int *Ws = reinterpret_cast<int *>(dv + nW);
    int *act = Ws + nW;
    float *wsm = reinterpret_cast<float *>(act + nW + (nW & 1));     // n weights (8-byte aligned start)
    for (int w = t; w < nW; w += T_) {
        const int j = a.W[w];
        Ws[w] = j;
        bw[w] = a.beta[j];
        cw[w] = a.c[j];
        iw[w] = 1.0 / a.s[j];
    }
    unsigned mbits = 0;
#pragma unroll
    for (int k = 0; k < RM; k++) {
        const int i = t + k * T_;
        const bool use = k < R && i < n && (!MASK || a.mask[i]);
        mbits |= (use ? 1u : 0u) << k;
    }
    double b0 = a.st->b0;
    __syncthreads();
    const T *X = reinterpret_cast<const T *>(a.X);
    const long long clk0 = clock64();
    int passes = 0, outer = 0, status = 0, buf = 0;
    long long visits = 0, updates = 0;
    long long ph[4] = {0, 0, 0, 0};     // cycles: CD sweeps, weights + v_j, eta, intercepts (thread 0's clock)
    double rr[RM];
    double sumw = 0.0;

    // one sweep over slots list[0..len) (nullptr => all): returns max|db|, max|b|
    auto sweep = [&](const int *list, int len, double &dmax, double &bmax) {
        dmax = 0.0;
        bmax = 0.0;
        visits += len;
        T xb[2][RM];
        auto load_col = [&](T (&x)[RM], int qq) {
            if (qq < len) {
                const T *col = X + (int64_t)Ws[list ? list[qq] : qq] * a.ld;
#pragma unroll
                for (int k = 0; k < RM; k++) { const int i = t + k * T_; x[k] = (k < R && i < n) ? col[i] : T(0); }
            }
        };
        load_col(xb[0], 0);
        load_col(xb[1], 1);
        for (int q0 = 0; q0 < len; q0 += 2) {
#pragma unroll
            for (int u = 0; u < 2; u++) {
                const int q = q0 + u;
                if (q < len) {
                    const int w = list ? list[q] : q;
                    const double b_old = bw[w], cj = cw[w], isj = iw[w], vj = vw[w], idv = dv[w];
                    double p0 = 0.0, p1 = 0.0;
#pragma unroll
                    for (int k = 0; k < RM; k += 2) {
                        if ((mbits >> k) & 1u) p0 = fma(to_d(xb[u][k]) - cj, rr[k], p0);
                        if (k + 1 < RM && ((mbits >> (k + 1)) & 1u)) p1 = fma(to_d(xb[u][k + 1]) - cj, rr[k + 1], p1);
                    }
                    const double pt = warp_sum(p0 + p1);
                    if (lane == 0) part[buf][wid] = pt;
                    __syncthreads();
                    double s0 = 0.0;
                    for (int v = 0; v < nw; v++) s0 += part[buf][v];
                    const double z = s0 * a.inv_n * isj + vj * b_old;
                    const double bn = soft_threshold(z, a.lam_alpha) * idv;
                    const double d = bn - b_old;
                    if (d != 0.0) {
                        updates++;
                        const double f = d * isj;
#pragma unroll
                        for (int k = 0; k < RM; k++)
                            if ((mbits >> k) & 1u) rr[k] = fma(-f * (double)wsm[t + k * T_], to_d(xb[u][k]) - cj, rr[k]);
                        if (t == 0) bw[w] = bn;
                    }
                    dmax = fmax(dmax, fabs(d));
                    bmax = fmax(bmax, fabs(bn));
                    buf ^= 1;
                    load_col(xb[u], q + 2);
                }
            }
        }
        __syncthreads();
    };
    // intercept (unpenalised, first in every pass): b0 += sum rho / sum w
    auto intercept = [&]() -> double {
        const long long c0 = clock64();
        double sr = 0.0;
#pragma unroll
        for (int k = 0; k < RM; k++)
            if ((mbits >> k) & 1u) sr += rr[k];
        const double d0 = block_sum(sr, red) / sumw;
#pragma unroll
        for (int k = 0; k < RM; k++)
            if ((mbits >> k) & 1u) rr[k] = fma(-d0, (double)wsm[t + k * T_], rr[k]);
        b0 += d0;
        ph[3] += clock64() - c0;
        return fabs(d0);
    };
    auto build_active = [&]() -> int {
        int total = 0;
        for (int base = 0; base < nW; base += T_) {
            const int w = base + t;
            const bool nz = w < nW && bw[w] != 0.0;
            const unsigned m = __ballot_sync(0xffffffffu, nz);
            if (lane == 0) wcount[wid] = __popc(m);
            __syncthreads();
            if (t == 0) {
                int run = 0;
                for (int u = 0; u < nw; u++) { const int c0 = wcount[u]; wcount[u] = run; run += c0; }
                wcount[32] = run;
            }
            __syncthreads();
            if (nz) act[total + wcount[wid] + __popc(m & ((1u << lane) - 1u))] = w;
            total += wcount[32];
            __syncthreads();
        }
        return total;
    };
    auto converged = [&](double dmax, double bmax, double d0) {
        return (dmax <= a.tol * bmax || dmax <= a.floor_) && (d0 <= a.tol * fmax(1.0, fabs(b0)) || d0 <= a.floor_);
    };

    for (;;) {                                            // ---- outer (IRLS) iterations
        long long c0 = clock64();
        double wl = 0.0;
#pragma unroll
        for (int k = 0; k < RM; k++) {
            const int i = t + k * T_;
            rr[k] = 0.0;
            if (k < R && i < n) {
                float wv = 0.f;
                if ((mbits >> k) & 1u) {
                    const double pi = sigmoid_d(a.eta[i]);
                    const double w = fmax(pi * (1.0 - pi), 1e-5);       // QL5
                    wv = (float)w;
                    rr[k] = a.y[i] - pi;
                    wl += (double)wv;
                }
                wsm[i] = wv;
            }
        }
        sumw = block_sum(wl, red);
        __syncthreads();                                  // wsm complete
        for (int w = wid; w < nW; w += nw) {              // v_j = x~_j' W x~_j / n, one warp per slot
            const T *col = X + (int64_t)Ws[w] * a.ld;
            const double cj = cw[w];
            double acc = 0.0;
            for (int i = lane; i < n; i += 32) {
                const double x = to_d(col[i]) - cj;
                acc = fma((double)wsm[i] * x, x, acc);
            }
            acc = warp_sum(acc);
            if (lane == 0) {
                const double v = acc * iw[w] * iw[w] * a.inv_n;
                vw[w] = v;
                dv[w] = 1.0 / (v + a.lam_l2);
                bo[w] = bw[w];
            }
        }
        const double b0o = b0;
        __syncthreads();
        ph[1] += clock64() - c0;
        c0 = clock64();
        // ---- weighted CD on the quadratic model: active cycling, then full passes
        for (int kind = 0; kind < 2 && !status; kind++) {
            for (;;) {
                const double d0 = intercept();
                double dmax = 0.0, bmax = 0.0;
                if (kind == 0) {
                    const int na = build_active();
                    if (na == 0) { if (++passes > a.max_iter) status = 3; break; }
                    sweep(act, na, dmax, bmax);
                } else {
                    sweep(nullptr, nW, dmax, bmax);
                }
                if (++passes > a.max_iter) { status = 3; break; }
                if (converged(dmax, bmax, d0)) break;
            }
        }
        ph[0] += clock64() - c0;
        if (status) break;
        c0 = clock64();
        // ---- eta = b0 + X~_A b_A on every row, from the columns
        const int na = build_active();
        double e[RM];
#pragma unroll
        for (int k = 0; k < RM; k++) e[k] = b0;
        for (int q = 0; q < na; q++) {
            const int w = act[q];
            const T *col = X + (int64_t)Ws[w] * a.ld;
            const double f = bw[w] * iw[w], cj = cw[w];
#pragma unroll
            for (int k = 0; k < RM; k++) {
                const int i = t + k * T_;
                if (k < R && i < n) e[k] = fma(f, to_d(col[i]) - cj, e[k]);
            }
        }
#pragma unroll
        for (int k = 0; k < RM; k++) {
            const int i = t + k * T_;
            if (k < R && i < n) a.eta[i] = e[k];
        }
        ph[2] += clock64() - c0;
        // ---- outer convergence (QL6)
        double dm = 0.0, bm = 0.0;
        for (int w = t; w < nW; w += T_) { dm = fmax(dm, fabs(bw[w] - bo[w])); bm = fmax(bm, fabs(bw[w])); }
        dm = block_max(dm, red);
        __syncthreads();
        bm = block_max(bm, red);
        __syncthreads();
        ++outer;
        if (outer > a.max_iter) { status = 3; break; }
        if (converged(dm, bm, fabs(b0 - b0o))) break;
    }
    __syncthreads();
    // ---- write back: r_scan = y - pi, loss, penalty terms (a11)
    double loss = 0.0, sr = 0.0;
#pragma unroll
    for (int k = 0; k < RM; k++) {
        const int i = t + k * T_;
        if (k < R && i < n) {
            double v = 0.0;
            if ((mbits >> k) & 1u) {
                const double et = a.eta[i], yi = a.y[i];
                v = yi - sigmoid_d(et);
                loss += (et > 0.0 ? et + log1p(exp(-et)) : log1p(exp(et))) - yi * et;
                sr += v;
            }
            a.r_scan[i] = v;
        }
    }
    for (int i = n + t; i < (int)a.ld; i += T_) a.r_scan[i] = 0.0;
    double l1 = 0.0, l2 = 0.0, nnz = 0.0;
    for (int w = t; w < nW; w += T_) {
        const double b = bw[w];
        const int jw = Ws[w];
        a.beta[jw] = b;
        a.betaW_out[w] = b;
        a.betaW_out[nW + w] = cw[w];
        a.betaW_out[2 * nW + w] = a.s[jw];
        l1 += fabs(b);
        l2 = fma(b, b, l2);
        nnz += b != 0.0 ? 1.0 : 0.0;
    }
    loss = block_sum(loss, red);
    __syncthreads();
    sr = block_sum(sr, red);
    __syncthreads();
    l1 = block_sum(l1, red);
    __syncthreads();
    l2 = block_sum(l2, red);
    __syncthreads();
    nnz = block_sum(nnz, red);
    if (t == 0) {
        a.st->cd_passes = passes;
        a.st->cd_status = status;
        a.st->rss = loss;          // logistic: sum of the per-row losses (objective = rss / n + penalty)
        a.st->sumr = sr;
        a.st->l1 = l1;
        a.st->l2 = l2;
        a.st->nnz = (int)nnz;
        a.st->cd_visits = visits;
        a.st->cd_updates = updates;
        a.st->cd_cycles = clock64() - clk0;
        a.st->b0 = b0;
        a.st->outer = outer;
        for (int u = 0; u < 4; u++) a.st->cd_prof[u] = ph[u];
    }
}

// ---------------- NEXT-3, covariance form: weighted Gram per IRLS iteration
// For |W| + 1 <= kLogitGramMax the logistic solve runs one IRLS iteration as three
// launches (host loop, one status read per iteration):
//   k_logit_eta     eta = b0 + X~_W b (all rows), pi, w = max(pi(1-pi), 1e-5), v = y - pi
//                   on used rows, per-block partial sums (fixed-order, deterministic);
//   k_gram_w        Gw = X~_W' diag(w) X~_W / n over the slots plus the intercept slot
//                   (a column of ones);
//   k_cd_logit_gram the weighted CD of QL4 in covariance form: g = X~_W' rho / n, each
//                   update g -= d Gw[:, j] (O(|W|)), one CTA, Gw rows prefetched D ahead.
constexpr int kLogitGramMax = 2048;        // slots incl. the intercept
constexpr int kLogitEtaThreads = 256;

template <typename T, bool MASK>
__global__ void __launch_bounds__(kLogitEtaThreads) k_logit_eta(const T *__restrict__ X, int64_t ld, int n,
        const int *__restrict__ Wst, int nW, const double *__restrict__ c, const double *__restrict__ s,
        const double *__restrict__ bS /* nW + 1: slots, then b0 */, const double *__restrict__ y,
        const uint8_t *__restrict__ mask, double *__restrict__ eta, double *__restrict__ w,
        double *__restrict__ v, double *__restrict__ part /* 3 per block: sum w, sum v, loss */,
        RoundStatus *st, int reset) {
    __shared__ double red[32];
    __shared__ double cb[kLogitEtaThreads], cc[kLogitEtaThreads];   // a chunk's nonzero slots: b / s_j, c_j
    __shared__ int cj[kLogitEtaThreads], wcnt[kLogitEtaThreads / 32 + 1];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double wl = 0.0, vl = 0.0, ll = 0.0;
    double e = bS[nW];
    // the slots in chunks of one per thread: the nonzero ones compacted (slot order kept) into shared
    // memory, then every row's dot over them with 8 column loads in flight -- the same terms in the
    // same order as a sequential loop over the slots (one dependent L2 load per slot was the cost)
    for (int k0 = 0; k0 < nW; k0 += kLogitEtaThreads) {
        const int k = k0 + threadIdx.x;
        const double b = k < nW ? bS[k] : 0.0;
        const bool nz = b != 0.0;
        const unsigned m = __ballot_sync(0xffffffffu, nz);
        if (lane == 0) wcnt[wid] = __popc(m);
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
            for (int u = 0; u < kLogitEtaThreads / 32; u++) { const int c0 = wcnt[u]; wcnt[u] = run; run += c0; }
            wcnt[kLogitEtaThreads / 32] = run;
        }
        __syncthreads();
        if (nz) {
            const int pos = wcnt[wid] + __popc(m & ((1u << lane) - 1u));
            const int j = Wst[k];
            cb[pos] = b / s[j];
            cc[pos] = c[j];
            cj[pos] = j;
        }
        __syncthreads();
        const int cnt = wcnt[kLogitEtaThreads / 32];
        if (i < n) {
            for (int q = 0; q < cnt; q += 8) {
                T xv[8];
#pragma unroll
                for (int u = 0; u < 8; u++) xv[u] = q + u < cnt ? X[(int64_t)cj[q + u] * ld + i] : T(0);
#pragma unroll
                for (int u = 0; u < 8; u++)
                    if (q + u < cnt) e = fma(cb[q + u], to_d(xv[u]) - cc[q + u], e);
            }
        }
        __syncthreads();                                    // (the chunk's staging is rewritten next)
    }
    if (i < ld) {
        const bool use = i < n && (!MASK || mask[i]);
        double wi = 0.0, vi = 0.0;
        if (use) {
            const double pi = sigmoid_d(e), yi = y[i];
            wi = fmax(pi * (1.0 - pi), 1e-5);      // QL5
            vi = yi - pi;
            ll = (e > 0.0 ? e + log1p(exp(-e)) : log1p(exp(e))) - yi * e;
        }
        if (i < n) eta[i] = e;
        w[i] = wi;
        v[i] = vi;
        wl = wi;
        vl = vi;
    }
    wl = block_sum(wl, red);
    vl = block_sum(vl, red);
    ll = block_sum(ll, red);
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x] = wl;
        part[3 * blockIdx.x + 1] = vl;
        part[3 * blockIdx.x + 2] = ll;
        if (reset && blockIdx.x == 0) {
            st->cd_passes = 0; st->cd_visits = 0; st->cd_updates = 0; st->cd_cycles = 0;
            st->outer = 0; st->irls_done = 0; st->cd_status = 0;
        }
    }
}

// Gw[a][b] = sum_i w_i x~_ia x~_ib / n for slots a, b in [0, nW]; slot nW = the intercept
// (x~ = 1 on every row).  Grid (nW + 1, ceil((nW + 1) / 32)); CTA (a, tile) stages
// w x~_a in shared memory and its 8 warps form 4 dots each; tiles above the
// diagonal are skipped and the mirror entry is written instead.
template <typename T, bool MASK>
__global__ void __launch_bounds__(256) k_gram_w(const T *__restrict__ X, int64_t ld, int n,
                                                const int *__restrict__ Wst, int nW, int ldG,
                                                const double *__restrict__ c, const double *__restrict__ s,
                                                const double *__restrict__ w, double inv_n, double *__restrict__ G,
                                                const double *__restrict__ part, int nblk, RoundStatus *st) {
    extern __shared__ __align__(16) double vs[];
    const int a = blockIdx.x;
    if (a == 0 && blockIdx.y == 0 && threadIdx.x == 0) {   // sum (y - pi), fixed order (identity (3)'s K1)
        double sv = 0.0;
        for (int q = 0; q < nblk; q++) sv += part[3 * q + 1];
        st->sumr = sv;
    }
    if ((int)blockIdx.y * 32 > a) return;
    const bool ia = a == nW;
    const int ja = ia ? 0 : Wst[a];
    const double ca = ia ? 0.0 : c[ja], sa = ia ? 1.0 : 1.0 / s[ja];
    const T *xa = X + (int64_t)ja * ld;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        vs[i] = w[i] * (ia ? 1.0 : (to_d(xa[i]) - ca) * sa);      // w is 0 on unused rows
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int t0 = blockIdx.y * 32 + wid * 4;
    if (t0 > a) return;
    const int nt = min(4, a + 1 - t0);
    const T *xt[4];
    double ct[4], st_[4];
    bool one[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int tb = t0 + min(q, nt - 1);
        one[q] = tb == nW;
        const int jt = one[q] ? 0 : Wst[tb];
        xt[q] = X + (int64_t)jt * ld;
        ct[q] = one[q] ? 0.0 : c[jt];
        st_[q] = one[q] ? 1.0 : 1.0 / s[jt];
    }
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = lane; i < n; i += 32) {
        const double vi = vs[i];
#pragma unroll
        for (int q = 0; q < 4; q++) acc[q] = fma(vi, one[q] ? 1.0 : to_d(xt[q][i]) - ct[q], acc[q]);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const double dsum = warp_sum(acc[q]);
        const int tt = t0 + q;
        if (lane == 0 && q < nt) {
            const double gv = dsum * st_[q] * inv_n;
            G[(int64_t)a * ldG + tt] = gv;
            G[(int64_t)tt * ldG + a] = gv;
        }
    }
}

struct CdLogitGramArgs {
    const void *X;
    int64_t ld;
    int n;
    const int *Wst;          // slot -> view column
    int nW;                  // penalised slots; slot nW = intercept
    const double *c, *s;
    const double *G;         // (nW + 1)^2 weighted Gram, leading dimension ldG
    int ldG;
    const double *gz;        // x~_j' (y - pi) / n by view column (fused scan over W)
    double *bS;              // nW + 1 in/out: slot coefficients, then b0
    double *beta;            // by view column (out)
    double lam_alpha, lam_l2, inv_n, tol, floor_;
    int max_iter;
    RoundStatus *st;
};

constexpr int kLGThreads = 256, kLGDepth = 4;

// EP = g entries per thread (m <= EP * kLGThreads).  One __syncthreads per coefficient
// update: every thread applies d G[k][j] to its own entries k != j, the barrier publishes
// them, and only then are g[j] and b[j] (read by every thread at the visit) written; a
// barrier closes each pass, so no index is read again before those writes are visible.
template <typename T, int EP>
__global__ void __launch_bounds__(kLGThreads, 1) k_cd_logit_gram(CdLogitGramArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ double red[32];
    __shared__ int wcount[33];
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = kLGThreads / 32;
    const int nW = a.nW, m = nW + 1;                  // coordinates incl. the intercept (index nW)
    double2 *gb = reinterpret_cast<double2 *>(sm);    // (g_j, b_j): written only by j's owner thread
    double2 *dv = gb + m;                             // (Gw_jj, 1 / (Gw_jj + lambda (1 - alpha)))
    double *bo = reinterpret_cast<double *>(dv + m);  // b at the start of this IRLS iteration
    int *seqA = reinterpret_cast<int *>(bo + m);      // active pass: intercept, then the nonzeros
    int *seqF = seqA + m + 1;                         // full pass: intercept, then every slot
    const long long clk0 = clock64();
    const T *X = reinterpret_cast<const T *>(a.X);
    (void)X;
    // ---- g_k = x~_k' v / n from the fused scan over W (a.gz, by view column); the intercept's
    // g = sum v / n from k_gram_w's fixed-order reduction (st->sumr)
    for (int k = t; k < nW; k += kLGThreads) gb[k].x = a.gz[a.Wst[k]];
    for (int k = t; k < m; k += kLGThreads) {
        const double d = a.G[(int64_t)k * a.ldG + k];
        dv[k] = make_double2(d, k == nW ? 1.0 / d : 1.0 / (d + a.lam_l2));
        gb[k].y = a.bS[k];
        bo[k] = a.bS[k];
    }
    for (int q = t; q <= nW; q += kLGThreads) seqF[q] = q == 0 ? nW : q - 1;
    if (t == 0) seqA[0] = nW;
    __syncthreads();
    if (t == 0) gb[nW].x = a.st->sumr * a.inv_n;
    __syncthreads();
    // ---- weighted CD passes in covariance form
    double gr[kLGDepth][EP];
    int passes = 0, status = 0;
    long long visits = 0, updates = 0;
    auto row_load = [&](double (&r)[EP], int j) {
        const double *Gj = a.G + (int64_t)j * a.ldG + t;
#pragma unroll
        for (int e = 0; e < EP; e++) r[e] = t + e * kLGThreads < m ? Gj[e * kLGThreads] : 0.0;
    };
    // one pass over seq[0..L) (seq[0] = the intercept)
    auto pass = [&](const int *seq, int L, double &dmax, double &bmax, double &d0) {
        dmax = 0.0;
        bmax = 0.0;
        d0 = 0.0;
        visits += L - 1;
#pragma unroll
        for (int u = 0; u < kLGDepth; u++)
            if (u < L) row_load(gr[u], seq[u]);
        for (int q0 = 0; q0 < L; q0 += kLGDepth) {
#pragma unroll
            for (int u = 0; u < kLGDepth; u++) {
                const int q = q0 + u;
                if (q < L) {
                    const int j = seq[q];
                    const double2 gbj = gb[j], dvj = dv[j];
                    const bool icpt = q == 0;
                    const double u_ = fma(dvj.x, gbj.y, gbj.x);
                    const double bn = (icpt ? u_ : soft_threshold(u_, a.lam_alpha)) * dvj.y;
                    const double d = bn - gbj.y;
                    if (d != 0.0) {                          // d is identical in every thread
                        updates++;
                        double gj = 0.0;
#pragma unroll
                        for (int e = 0; e < EP; e++) {
                            const int k = t + e * kLGThreads;
                            if (k < m) {
                                const double nv = fma(-d, gr[u][e], gb[k].x);
                                if (k != j) gb[k].x = nv;
                                else gj = nv;
                            }
                        }
                        __syncthreads();                     // every thread has read gb[j]; g[k != j] published
                        if ((j & (kLGThreads - 1)) == t) gb[j] = make_double2(gj, bn);
                    }
                    if (icpt) d0 = fabs(d);
                    else { dmax = fmax(dmax, fabs(d)); bmax = fmax(bmax, fabs(bn)); }
                    if (q + kLGDepth < L) row_load(gr[u], seq[q + kLGDepth]);
                }
            }
        }
        __syncthreads();                                     // the pass's last (g_j, b_j) writes visible
    };
    auto build_active = [&]() -> int {
        int total = 0;
        for (int base = 0; base < nW; base += kLGThreads) {
            const int k = base + t;
            const bool nz = k < nW && gb[k].y != 0.0;
            const unsigned msk = __ballot_sync(0xffffffffu, nz);
            if (lane == 0) wcount[wid] = __popc(msk);
            __syncthreads();
            if (t == 0) {
                int run = 0;
                for (int u = 0; u < nw; u++) { const int c0 = wcount[u]; wcount[u] = run; run += c0; }
                wcount[32] = run;
            }
            __syncthreads();
            if (nz) seqA[1 + total + wcount[wid] + __popc(msk & ((1u << lane) - 1u))] = k;
            total += wcount[32];
            __syncthreads();
        }
        return total;
    };
    auto converged = [&](double dmax, double bmax, double d0, double b0) {
        return (dmax <= a.tol * bmax || dmax <= a.floor_) && (d0 <= a.tol * fmax(1.0, fabs(b0)) || d0 <= a.floor_);
    };
    for (int kind = 0; kind < 2 && !status; kind++) {      // active cycling, then full passes
        for (;;) {
            double dmax, bmax, d0;
            if (kind == 0) {
                const int na = build_active();
                if (na == 0) break;
                pass(seqA, na + 1, dmax, bmax, d0);
            } else {
                pass(seqF, nW + 1, dmax, bmax, d0);
            }
            if (++passes > a.max_iter) { status = 3; break; }
            if (converged(dmax, bmax, d0, gb[nW].y)) break;
        }
    }
    __syncthreads();
    // ---- outer (IRLS) convergence against the iteration's start point (QL6)
    double dm = 0.0, bm = 0.0;
    for (int k = t; k < nW; k += kLGThreads) { dm = fmax(dm, fabs(gb[k].y - bo[k])); bm = fmax(bm, fabs(gb[k].y)); }
    dm = block_max(dm, red);
    __syncthreads();
    bm = block_max(bm, red);
    const double b0 = gb[nW].y;
    const bool done = converged(dm, bm, fabs(b0 - bo[nW]), b0);
    for (int k = t; k < m; k += kLGThreads) {
        a.bS[k] = gb[k].y;
        if (k < nW) a.beta[a.Wst[k]] = gb[k].y;
    }
    if (t == 0) {
        RoundStatus *st = a.st;
        st->cd_passes += passes;
        st->cd_visits += visits;
        st->cd_updates += updates;
        st->cd_cycles += clock64() - clk0;
        st->outer += 1;
        if (status) st->cd_status = status;
        if (st->outer > a.max_iter) st->cd_status = 3;
        st->irls_done = done ? 1 : 0;
        st->b0 = b0;
    }
}

__global__ void k_logit_gather(double *__restrict__ bS, const double *__restrict__ beta, const int *__restrict__ Wst,
                               int nW, const RoundStatus *st) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= nW; k += gridDim.x * blockDim.x)
        bS[k] = k < nW ? beta[Wst[k]] : st->b0;
}

// Final statistics of a logistic solve (a11): loss and sum(y - pi) from k_logit_eta's
// partials (fixed order), l1 / l2 / nnz and the read-out (ord: sorted position -> slot).
__global__ void k_logit_finish(const double *__restrict__ part, int nblk, const double *__restrict__ bS, int nW,
                               const int *__restrict__ Wst, const int *__restrict__ ord, const double *__restrict__ c,
                               const double *__restrict__ s, double *__restrict__ betaW_out, RoundStatus *st) {
    __shared__ double red[32];
    double l1 = 0.0, l2 = 0.0, nnz = 0.0;
    for (int q = threadIdx.x; q < nW; q += blockDim.x) {     // read-out in ascending column order
        const int k = ord[q];
        const double bk = bS[k];
        const int j = Wst[k];
        betaW_out[q] = bk;
        betaW_out[nW + q] = c[j];
        betaW_out[2 * nW + q] = s[j];
        l1 += fabs(bk);
        l2 = fma(bk, bk, l2);
        nnz += bk != 0.0 ? 1.0 : 0.0;
    }
    l1 = block_sum(l1, red);
    l2 = block_sum(l2, red);
    nnz = block_sum(nnz, red);
    if (threadIdx.x == 0) {
        double sv = 0.0, ll = 0.0;
        for (int q = 0; q < nblk; q++) { sv += part[3 * q + 1]; ll += part[3 * q + 2]; }
        st->rss = ll;
        st->sumr = sv;
        st->l1 = l1;
        st->l2 = l2;
        st->nnz = (int)nnz;
        st->b0 = bS[nW];
    }
}

// ---- NEXT-3 on the cluster Gram CD: one IRLS iteration's quadratic model
// with the intercept eliminated (Schur complement of the intercept row of Gw) and each
// coordinate scaled to unit curvature, so k_cd_gram7 solves it unchanged except for a per-slot
// threshold: gamma_j = sqrt(D_j) beta_j, D_j = Gw_jj - Gw_j0^2 / Gw_00,
//   G''_jk = (Gw_jk - Gw_j0 Gw_k0 / Gw_00) / sqrt(D_j D_k),  z_j = (g_j - Gw_j0 g_0 / Gw_00) / sqrt(D_j),
//   tau_j = lambda alpha / sqrt(D_j),  1 / curvature_j = 1 / (1 + lambda (1 - alpha) / D_j).
// The intercept follows from the solved coefficients: d0 = (g_0 - sum_j Gw_j0 d_j) / Gw_00.
// ws (per slot, 4 nW doubles): sc = 1/sqrt(D), tau, beta at the iteration's start; acc (8).
__global__ void k_logit_g7_slots(int nW, const double *__restrict__ LG, int ldL, const int *__restrict__ Wst,
                                 const double *__restrict__ bS, double *__restrict__ z, double *__restrict__ beta,
                                 double *__restrict__ ws, double lam_alpha, double lam_l2, double inv_n,
                                 const RoundStatus *st) {
    const double h00 = LG[(int64_t)nW * ldL + nW], g0 = st->sumr * inv_n;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nW; k += gridDim.x * blockDim.x) {
        const double h = LG[(int64_t)k * ldL + nW];
        const double D = LG[(int64_t)k * ldL + k] - h * h / h00;
        const double sc = D > 0.0 ? 1.0 / sqrt(D) : 0.0;
        const int j = Wst[k];
        ws[k] = sc;
        ws[nW + k] = lam_alpha * sc;
        ws[2 * nW + k] = bS[k];
        ws[3 * nW + k] = 1.0 / (1.0 + lam_l2 * sc * sc);        // ridge term in scaled coordinates
        z[j] = (z[j] - h * g0 / h00) * sc;
        beta[j] = sc > 0.0 ? bS[k] / sc : 0.0;
    }
}

__global__ void k_logit_g7_schur(int nW, const double *__restrict__ LG, int ldL, const double *__restrict__ ws,
                                 double *__restrict__ G, int ldG) {
    const int a = blockIdx.x;
    const double h00 = LG[(int64_t)nW * ldL + nW], ha = LG[(int64_t)a * ldL + nW], sa = ws[a];
    for (int b = blockIdx.y * blockDim.x + threadIdx.x; b < nW; b += gridDim.y * blockDim.x)
        G[(int64_t)a * ldG + b] = (LG[(int64_t)a * ldL + b] - ha * LG[(int64_t)b * ldL + nW] / h00) * sa * ws[b];
}

// after k_cd_gram7: back to beta, the intercept step, the IRLS convergence test (QL6) and the
// solve counters accumulated over the iterations (acc: passes, visits, updates, cycles)
__global__ void k_logit_g7_post(int nW, const double *__restrict__ LG, int ldL, const int *__restrict__ Wst,
                                double *__restrict__ beta, double *__restrict__ bS, const double *__restrict__ ws,
                                double inv_n, double tol, double floor_, int max_iter, RoundStatus *st,
                                long long *acc) {
    __shared__ double red[32];
    const double h00 = LG[(int64_t)nW * ldL + nW], g0 = st->sumr * inv_n;
    double hd = 0.0, dm = 0.0, bm = 0.0;
    for (int k = threadIdx.x; k < nW; k += blockDim.x) {
        const int j = Wst[k];
        const double bn = beta[j] * ws[k];
        const double d = bn - ws[2 * nW + k];
        beta[j] = bn;
        bS[k] = bn;
        hd = fma(LG[(int64_t)k * ldL + nW], d, hd);
        dm = fmax(dm, fabs(d));
        bm = fmax(bm, fabs(bn));
    }
    hd = block_sum(hd, red);
    __syncthreads();
    dm = block_max(dm, red);
    __syncthreads();
    bm = block_max(bm, red);
    if (threadIdx.x == 0) {
        const double d0 = (g0 - hd) / h00;
        const double b0 = bS[nW] + d0;
        bS[nW] = b0;
        st->b0 = b0;
        const bool ok_b = dm <= tol * bm || dm <= floor_;
        const bool ok_0 = fabs(d0) <= tol * fmax(1.0, fabs(b0)) || fabs(d0) <= floor_;
        acc[0] += st->cd_passes;
        acc[1] += st->cd_visits;
        acc[2] += st->cd_updates;
        acc[3] += st->cd_cycles;
        acc[4] += 1;
        if (st->cd_status) acc[5] = st->cd_status;
        if (acc[4] > max_iter) acc[5] = 3;
        st->irls_done = ok_b && ok_0;
        st->outer = (int)acc[4];
        st->cd_status = (int)acc[5];
    }
}

__global__ void k_logit_g7_counters(RoundStatus *st, const long long *acc) {
    st->cd_passes = (int)acc[0];
    st->cd_visits = acc[1];
    st->cd_updates = acc[2];
    st->cd_cycles = acc[3];
    st->outer = (int)acc[4];
    st->cd_status = (int)acc[5];
}

// ------------------------------- NEXT-2: covariance-update ("Gram") CD on W
// SURVEY 8(f) NEXT-2 (glmnet's covariance updates; the paper's CD "only iterates
// over features in the active set").  Same iterates as the residual CD
// above, but the per-coordinate work is O(|W|) on the gradient vector
//   g_w = x~_w' r / n        (w in W)
// instead of an O(n) reduction:  z = g_w + b_w;  b' = S(z, lambda alpha)/(1 +
// lambda(1-alpha));  g_k -= (b' - b_w) G_kw  for every k in W, with
// G = X~_W' X~_W / n kept in HBM/L2 (identity (1), generalised to W x W).
// g starts from the fused scan's z at the solve's residual; r is refreshed after
// the solve from the coefficient changes (k_resid_part / k_resid_apply), so no drift crosses
// lambdas.  Storage slots are append-only; `ord` gives the cyclic (ascending
// column) order.

// G rows (and columns) for the new slots [first, nW): G[s][t] = sum_i m_i
// x~_is x~_it / n.  grid = (nW - first, ceil(nW / 32)), 256 threads: each warp
// computes 4 entries with 8 independent loads in flight per lane (the earlier
// one-entry-per-warp loop was L2-latency bound).
template <typename T, bool MASK>
__global__ void __launch_bounds__(256) k_gram(const T *__restrict__ X, int64_t ld, int n,
                                              const int *__restrict__ Wst, int nW, int first, int ldG,
                                              const double *__restrict__ c, const double *__restrict__ s,
                                              const uint8_t *__restrict__ mask, double inv_n, double *__restrict__ G) {
    extern __shared__ __align__(16) double vs[];     // x~_s on the used rows
    const int sl = first + blockIdx.x;
    const int js = Wst[sl];
    const double cs = c[js], is = 1.0 / s[js];
    const T *xs = X + (int64_t)js * ld;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
        vs[i] = (!MASK || mask[i]) ? (to_d(xs[i]) - cs) * is : 0.0;
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int t0 = blockIdx.y * 32 + wid * 4;
    if (t0 >= nW) return;
    const int nt = min(4, nW - t0);
    const T *xt[4];
    double ct[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const int jt = Wst[t0 + min(q, nt - 1)];
        xt[q] = X + (int64_t)jt * ld;
        ct[q] = c[jt];
    }
    double acc[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
    int i = lane;
    for (; i + 32 < n; i += 64) {
        double xv[4][2];
#pragma unroll
        for (int q = 0; q < 4; q++) { xv[q][0] = to_d(xt[q][i]); xv[q][1] = to_d(xt[q][i + 32]); }
        const double v0 = vs[i], v1 = vs[i + 32];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            acc[q][0] = fma(v0, xv[q][0] - ct[q], acc[q][0]);
            acc[q][1] = fma(v1, xv[q][1] - ct[q], acc[q][1]);
        }
    }
    if (i < n) {
#pragma unroll
        for (int q = 0; q < 4; q++) acc[q][0] = fma(vs[i], to_d(xt[q][i]) - ct[q], acc[q][0]);
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
        const double dsum = warp_sum(acc[q][0] + acc[q][1]);
        const int tt = t0 + q;
        if (lane == 0 && q < nt) {
            const double gv = dsum / s[Wst[tt]] * inv_n;
            G[(int64_t)sl * ldG + tt] = gv;
            if (tt < first) G[(int64_t)tt * ldG + sl] = gv;
        }
    }
}

struct CdGramArgs {
    const int *Wst;          // storage slot -> local column
    const int *ord;          // cyclic order (slots, ascending column)
    int nW, ldG;
    const double *G;         // ldG x ldG, row-major by storage slot
    double *GA;              // workspace ldG x ldG: compact G_AA of the active set (v6)
    double *MA;              // workspace ceil(nW/32) x 1024: per-block inverses M (v6)
    const double *z;         // z[j] = x~_j' r / n for the solve's starting residual
    double *beta;            // p entries (global, by local column)
    double *dbeta;           // nW entries out: beta_new - beta_old per slot
    double lam_alpha, inv_den, tol, floor_;
    int max_iter;
    double *betaW_out;       // 3*nW: beta, c, s per slot (cyclic order)
    const double *c, *s;
    RoundStatus *st;
    const double *tau;       // per-slot soft threshold (nullptr: lam_alpha for every slot) and
    const double *idv;       // per-slot 1 / curvature (nullptr: inv_den): the logistic path's
                             // scaled coordinates (NEXT-3)
    double nu;               // lambda (1 - alpha): the ridge part of the curvature (1 + nu = 1 / inv_den)
    int newton;              // 1: Newton (CG) steps on a settled active set between sweeps (linear path)
    int smem_bytes;          // dynamic shared memory of the launch (the Newton step caches G_AA rows in it)
};

// Cluster Gram CD (v7): the v6 algorithm above with its bulk spread over a
// thread-block cluster.  One SM can only stream ~30-50 B/clk from L2, and the
// bulk (every block's updates applied to every other gradient of the sweep)
// reads |sweep| x 32 x 8 bytes of G per block -- so the gradients live in the
// shared memory of CTAs 1..R-1 ("owners"), block-cyclically by position (block
// j of 32 positions -> CTA 1 + j mod (R-1)), and each owner streams only the G
// columns of the positions it owns.  CTA 0 leads: warp 0 solves the blocks
// (same speculation / M inverse / verification as v6), warps 1.. prefetch the
// sub-blocks two blocks ahead.  Per block step, one split cluster barrier
// (arrive.release ... wait.acquire).  Each side publishes into its OWN shared
// memory and the other side reads it remotely after the barrier (a remote
// release-store costs a DSMEM round trip at the arrive; a remote load ~1/3 of it):
//   leader : z = g (the owner's snapshot of the block, read remotely) + b minus
//            the link with the previous block (computed before the barrier),
//            solve, publish the 32 updates (dense) locally, arrive; then the
//            link product for the next block;
//   owners : read the previous block's 32 updates from the leader, apply them
//            to all their positions (the G rows were prefetched into registers
//            during the previous step), snapshot the next block's gradients
//            if they own it, arrive, then issue the loads of this block's G
//            rows for the next step.
// The owners keep their gradients across consecutive sweeps over the same
// positions; they go to a global copy (by slot) only when the positions change
// (active <-> full sweeps, a new active set) or a catch-up / G_AA build needs
// them.  Catch-ups, G_AA and M builds are split over the cluster.
constexpr int kG7Threads = 256;
constexpr int kG7Helpers = kG7Threads - 32;
// Leader-warp sub-phase timers (bl_perf.cd_sub): six extra clock64 reads per block, so
// they are compiled in only for the CD micro-benchmarks (-DBL_G7_SUBPHASES=1).
#ifndef BL_G7_SUBPHASES
#define BL_G7_SUBPHASES 0
#endif
#define G7CLK() (BL_G7_SUBPHASES ? clock64() : 0LL)
// CG iteration sub-phase timers (owner rank 1 -> cd_sub[0..4]; micro-benchmarks only)
#ifndef BL_CG_PHASES
#define BL_CG_PHASES 0
#endif
#define CGCLK() (BL_CG_PHASES ? clock64() : 0LL)
// Newton step (Q30) trigger: after BL_NEWTON_SWEEPS active sweeps on the same set and signs, the last
// one contracting by more than BL_NEWTON_RHO; at most BL_NEWTON_MAX steps per set
#ifndef BL_NEWTON_SWEEPS
#define BL_NEWTON_SWEEPS 1
#endif
#ifndef BL_NEWTON_RHO
#define BL_NEWTON_RHO 0.3
#endif
#ifndef BL_NEWTON_MAX
#define BL_NEWTON_MAX 2
#endif
// Newton step (Q30): CG stops at an rms residual of BL_CG_RTOL x tol x max|beta|
#ifndef BL_CG_RTOL
#define BL_CG_RTOL 0.2
#endif
constexpr int kG7MaxR = 16;
constexpr int kG7Stages = 4;                    // leader prefetch ring (Gd, Gp, M per stage)
__host__ __device__ constexpr size_t gram7_smem(int nW, int R) {
    // 3 x kG7Stages x 8 KB leader buffers (stages of Gd, Gp, M) + the larger of the leader's
    // per-slot state (bS, bcat: 16 B; act, actp: 8 B; inA: 1 B) and an owner's
    // gradients + slots (12 B per owned position)
    return (size_t)3 * kG7Stages * 8192 +
           ((size_t)25 * (size_t)((nW + 33) & ~1) > (size_t)12 * (size_t)(nW / (R - 1) + 64)
                ? (size_t)25 * (size_t)((nW + 33) & ~1)
                : (size_t)12 * (size_t)(nW / (R - 1) + 64)) +
           64;
}

struct G7Work {              // global workspace of one fit (see bl.cu gram_ws)
    double *g;               // nW: gradients by slot, between sweeps
    int *act;                // nW: active list published by the leader
    double *dl;              // nW: catch-up coefficient changes
    int *rl;                 // nW: ... and their slots
    uint8_t *inA;            // nW: slot is in the set G_AA was built for
    double *cg;              // 5 nW: Newton step by active position: x, r, p, b (coefficients), spare
};

// mbarrier / st.async helpers (CTA-local barriers; st.async writes 8 bytes into a
// peer CTA's shared memory and completes them on the peer's mbarrier)
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arm(uint64_t *bar, unsigned bytes) {          // arrive + expect_tx
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_addr(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ uint32_t mapa(const void *p, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async(uint32_t remote, double v, uint32_t remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                 ::"r"(remote), "l"(__double_as_longlong(v)), "r"(remote_bar) : "memory");
}

__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

// The cluster shape is compiled in (__cluster_dims__) so the kernel launches with
// <<<>>> (profilers do not see cudaLaunchKernelExC launches).
template <bool ENET, int RC>
__global__ void __cluster_dims__(RC, 1, 1) __launch_bounds__(kG7Threads, 1) k_cd_gram7(CdGramArgs a, G7Work wk) {
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) double sm[];
    __shared__ __align__(16) double dfull[32];         // leader: the block's updates (0 = none)
    __shared__ __align__(16) double rsh[32];
    constexpr int DZ = 4, DDMAX = kG7MaxR + 2;
    __shared__ __align__(16) double zst[DZ][32];       // leader: ring of block gradients (st.async by the owners)
    __shared__ __align__(16) double dq[DDMAX][32];     // owners: ring of the leader's block updates (bulk copies)
    __shared__ __align__(16) double dsrc[DDMAX][32];   // leader: staging ring the bulk copies read
    constexpr int NS = kG7Stages;
    __shared__ __align__(8) uint64_t zfull[DZ], dfb[DDMAX], sfull[NS], sempty[NS];
    __shared__ __align__(8) uint64_t cgbar[2];         // Newton CG: [0] residual pieces, [1] partial sums
    __shared__ __align__(16) double cgpsum[kG7MaxR][2]; // Newton CG: every CTA's two partial sums
    __shared__ int bslot[NS][32];                      // leader: slots of the block
    __shared__ uint32_t rdq[kG7MaxR], rdfb[kG7MaxR];    // leader: owners' ring addresses (shared::cluster)
    __shared__ int ctl[2][8];                          // leader: command for the cluster (double-buffered)
    __shared__ int wcount[33];
    __shared__ double red[32];
    constexpr int T_ = kG7Threads;
    constexpr unsigned FULL = 0xffffffffu;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = T_ >> 5;
    const int R = (int)cl.num_blocks(), rank = (int)cl.block_rank(), NB = R - 1;
    const bool leader_cta = rank == 0;
    const int nW = a.nW;
    const int nWp = (nW + 1) & ~1;
    const int64_t ldG = a.ldG;
    double(*Gd)[32][32] = reinterpret_cast<double(*)[32][32]>(sm);            // [NS]: strictly lower diag sub-block
    double(*Gp)[32][32] = Gd + NS;                                             // [NS]: previous block -> this block
    double(*Mb)[32][32] = Gd + 2 * NS;                                         // [NS]: M, column-major ([c][b])
    // leader CTA per-slot state
    double *bS = sm + 3 * NS * 1024;                        // coefficients, by slot
    double *bcat = bS + nWp;                                // coefficients at the last lazy catch-up
    int *act = reinterpret_cast<int *>(bcat + nWp);         // active slots (ascending)
    int *actp = act + nWp;                                  // the set G_AA / M were built for
    uint8_t *inA = reinterpret_cast<uint8_t *>(actp + nWp);
    // owner CTAs: gradients of the owned positions (local index = (j / NB) * 32 + k % 32) and their slots
    double *gl = sm + 3 * NS * 1024;
    const int gcap = (nW / 32 / NB + 2) * 32;
    int *sl = reinterpret_cast<int *>(gl + gcap);
    int owned = 0;                                          // owners: local positions currently held
    auto lidx = [&](int k) { return ((k >> 5) / NB) * 32 + (k & 31); };

    // ---- init: coefficients (leader), gradients by slot (global, split over the cluster)
    if (leader_cta) {
        for (int w = t; w < nWp; w += T_) {
            bS[w] = w < nW ? a.beta[a.Wst[w]] : 0.0;
            inA[w] = 0;
        }
    }
    for (int w = rank * T_ + t; w < nW; w += R * T_) wk.g[w] = a.z[a.Wst[w]];
    // hand-off rings: slot / phase of block number gb (counted over all sweeps) are
    // gb % D and (gb / D) & 1.  DD = NB + 2 slots bound every owner's lag: the
    // leader only writes block gb's updates after the snapshots of blocks
    // gb-NB+1..gb, which each owner sends after consuming the updates 2 blocks before.
    const int DD = NB + 2;
    if (t == 0) {
        if (leader_cta) {
            for (int u = 0; u < DZ; u++) { mbar_init(&zfull[u], 1); mbar_arm(&zfull[u], 256); }
            for (int u = 0; u < NS; u++) { mbar_init(&sfull[u], kG7Helpers); mbar_init(&sempty[u], 1); }
            for (int r = 1; r < R; r++) { rdq[r] = mapa(&dq[0][0], r); rdfb[r] = mapa(&dfb[0], r); }
        } else {
            for (int u = 0; u < DD; u++) { mbar_init(&dfb[u], 1); mbar_arm(&dfb[u], 256); }
        }
        mbar_init(&cgbar[0], 1);
        mbar_init(&cgbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();                                              // release / acquire at cluster scope

    const long long clk0 = clock64();
    int passes = 0, status = 0;
    long long visits = 0, updates = 0, pr_lead = 0, pr_bulk = 0, retries = 0, rebuilds = 0;
    long long pr_build = 0, pr_catch = 0, ncatch = 0, nfull = 0;
    long long dbg[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const double la0 = a.lam_alpha, inv_den0 = a.inv_den;
    double dm = 0.0, bm = 0.0;                              // leader warp: per-lane running maxima
    int nflip = 0;                                          // leader warp: sign-class changes this sweep

    auto block_rank = [&](bool nz, int &pos) -> int {     // order-preserving CTA compaction
        const unsigned m = __ballot_sync(FULL, nz);
        if (lane == 0) wcount[wid] = __popc(m);
        __syncthreads();
        if (t == 0) {
            int run = 0;
            for (int u = 0; u < nw; u++) { const int c0 = wcount[u]; wcount[u] = run; run += c0; }
            wcount[32] = run;
        }
        __syncthreads();
        pos = wcount[wid] + __popc(m & ((1u << lane) - 1u));
        const int tot = wcount[32];
        __syncthreads();
        return tot;
    };

    // leader helpers: prefetch block qn's sub-blocks (and M in active sweeps) into stage buf
    // leader helpers: prefetch block qn's sub-blocks into stage buf with 16-byte loads:
    // the strictly lower diagonal block (full sweeps only -- active sweeps solve with
    // M and fetch it only on a misprediction), the link from block qn-1, M (active).
    // All loads of a thread are issued before its shared-memory stores.
    auto prefetch = [&](const double *Mx, bool active, int len, int qn, int buf) {
        const int u = t - 32;
        const int b0 = 32 * qn, nb1 = min(32, len - b0);
        const int nb0 = qn > 0 ? 32 : 0;
        constexpr int NP = (1536 + kG7Helpers - 1) / kG7Helpers;
        double2 v[NP];
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const int e = u + k * kG7Helpers;                 // pair index: [0,512) Gd, [512,1024) Gp, [1024,1536) M
            const int r = (e >> 4) & 31, c = 2 * (e & 15);
            const double2 *src = nullptr;
            if (e < 512) {
                if (!active && c + 1 > r && c < nb1) src = reinterpret_cast<const double2 *>(Mx + (int64_t)(b0 + r) * ldG + b0 + c);
            } else if (e < 1024) {
                if (r < nb0 && c < nb1) src = reinterpret_cast<const double2 *>(Mx + (int64_t)(b0 - 32 + r) * ldG + b0 + c);
            } else if (e < 1536 && active) {
                src = reinterpret_cast<const double2 *>(a.MA + (int64_t)qn * 1024 + 2 * (e - 1024));
            }
            v[k] = src ? __ldcg(src) : make_double2(0.0, 0.0);
            if (e < 1024) {                                   // zero what lies outside the block / the lower part
                const bool lo = e < 512;
                if (lo ? !(c > r && c < nb1) : c >= nb1) v[k].x = 0.0;
                if (lo ? !(c + 1 > r && c + 1 < nb1) : c + 1 >= nb1) v[k].y = 0.0;
            }
        }
#pragma unroll
        for (int k = 0; k < NP; k++) {
            const int e = u + k * kG7Helpers;
            if (e < 512) { if (!active) reinterpret_cast<double2 *>(&Gd[buf][0][0])[e] = v[k]; }
            else if (e < 1024) reinterpret_cast<double2 *>(&Gp[buf][0][0])[e - 512] = v[k];
            else if (e < 1536 && active) reinterpret_cast<double2 *>(&Mb[buf][0][0])[e - 1024] = v[k];
        }
        if (u < 32) bslot[buf][u] = u < nb1 ? (active ? act[b0 + u] : b0 + u) : -1;
    };

    // leader warp: link of the previous block's updates (dfull) into block qn (stage buf)
    auto link = [&](int buf) -> double {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (int r = 0; r < 32; r += 4) {
            const double2 d01 = *reinterpret_cast<const double2 *>(&dfull[r]);
            const double2 d23 = *reinterpret_cast<const double2 *>(&dfull[r + 2]);
            a0 = fma(d01.x, Gp[buf][r][lane], a0);
            a1 = fma(d01.y, Gp[buf][r + 1][lane], a1);
            a2 = fma(d23.x, Gp[buf][r + 2][lane], a2);
            a3 = fma(d23.y, Gp[buf][r + 3][lane], a3);
        }
        return (a0 + a1) + (a2 + a3);
    };

    // leader warp: block at positions b0.. (stage buf; zo = the owner's snapshot); acc = link term;
    // gb = block number (ring slot of the published updates)
    auto lead = [&](bool active, int b0, int buf, double zo, double acc, long long gb) {
        const long long t0 = G7CLK();
        const int s = bslot[buf][lane];
        const bool valid = s >= 0;
        double zc = 0.0, bo = 0.0;
        if (valid) {
            bo = bS[s];
            zc = (zo - acc) + bo;
        }
        const double la = (a.tau && valid) ? a.tau[s] : la0;      // this lane's threshold
        const double inv_den = (a.idv && valid) ? a.idv[s] : inv_den0;
        const double(*GL)[32] = Gd[buf];
        int pred = bo > 0.0 ? 1 : (bo < 0.0 ? -1 : 0);
        double dfin = 0.0, bnfin = bo;
        unsigned todo = __ballot_sync(FULL, valid);
        int round = 0;
        const long long t1 = G7CLK();
        dbg[0] += t1 - t0;
        if (active) {
            const double las = pred > 0 ? la : -la;
            rsh[lane] = valid ? (ENET ? (zc - las) * inv_den : zc - las) - bo : 0.0;
            __syncwarp();
            double m0 = 0.0, m1 = 0.0, m2 = 0.0, m3 = 0.0;
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
                const double2 r01 = *reinterpret_cast<const double2 *>(&rsh[c]);
                const double2 r23 = *reinterpret_cast<const double2 *>(&rsh[c + 2]);
                m0 = fma(Mb[buf][c][lane], r01.x, m0);
                m1 = fma(Mb[buf][c + 1][lane], r01.y, m1);
                m2 = fma(Mb[buf][c + 2][lane], r23.x, m2);
                m3 = fma(Mb[buf][c + 3][lane], r23.y, m3);
            }
            const double d = (m0 + m1) + (m2 + m3);
            const double bn = d + bo;
            const unsigned mis = __ballot_sync(FULL, valid && !(pred > 0 ? bn > 0.0 : bn < 0.0));
            const unsigned commit = todo & (mis ? ((1u << (__ffs(mis) - 1)) - 1u) : FULL);
            if ((commit >> lane) & 1u) { dfin = d; bnfin = bn; }
            todo &= ~commit;
            if (mis) {
                ++round;
                {                                             // the strictly lower diagonal block (not prefetched)
                    const int nb = __popc(__ballot_sync(FULL, valid));
                    for (int r = 0; r < 32; r++)
                        Gd[buf][r][lane] = (lane > r && lane < nb) ? __ldcg(a.GA + (int64_t)(b0 + r) * ldG + b0 + lane) : 0.0;
                    __syncwarp();
                }
                unsigned cp = commit;
                while (cp) {
                    const int p = __ffs(cp) - 1;
                    cp &= cp - 1;
                    const double dp = __shfl_sync(FULL, dfin, p);
                    zc = fma(-dp, GL[p][lane], zc);
                }
                if ((todo >> lane) & 1u) pred = zc > la ? 1 : (zc < -la ? -1 : 0);
            }
        }
        const long long t2 = G7CLK();
        dbg[1] += t2 - t1;
        while (todo) {
            const unsigned Pm = __ballot_sync(FULL, pred != 0) & todo;
            const double las = pred > 0 ? la : -la;
            double z = zc;
            unsigned rem = Pm;
            while (rem) {
                const int p = __ffs(rem) - 1;
                rem &= rem - 1;
                const double gl_ = GL[p][lane];
                const double dl = (ENET ? (z - las) * inv_den : z - las) - bo;
                const double dp = __shfl_sync(FULL, dl, p);
                z = fma(-dp, gl_, z);
            }
            const bool hi = z > la, lo = z < -la;
            const int tb = hi ? 1 : (lo ? -1 : 0);
            const unsigned mis = __ballot_sync(FULL, tb != pred) & todo;
            const unsigned below = mis ? ((1u << (__ffs(mis) - 1)) - 1u) : FULL;
            const unsigned commit = todo & below;
            if ((commit >> lane) & 1u) {
                const double bn = hi ? z - la : (lo ? z + la : 0.0);
                bnfin = ENET ? bn * inv_den : bn;
                dfin = bnfin - bo;
            }
            todo &= ~commit;
            if (!mis) break;
            ++round;
            unsigned cp = Pm & commit;
            while (cp) {
                const int p = __ffs(cp) - 1;
                cp &= cp - 1;
                const double dp = __shfl_sync(FULL, dfin, p);
                zc = fma(-dp, GL[p][lane], zc);
            }
            if ((todo >> lane) & 1u) pred = tb;   // the first mismatch is exact now; the rest re-predicted
        }
        const long long t3 = G7CLK();
        dbg[2] += t3 - t2;
        // publish the 32 updates into every owner's ring slot: the block is staged in this CTA's
        // shared memory, then lanes 1..R-1 each issue ONE 256-byte bulk copy into owner `lane`'s
        // ring, completing on that owner's mbarrier (32 x (R-1) 8-byte remote stores were the
        // leader's largest per-block cost).  Slot ds is rewritten DD blocks later: before that,
        // the issuing lane waits until its copy of block gb - DD + 1 has been read.
        {
            const int ds = (int)(gb % DD);
            const bool issuer = lane >= 1 && lane < R;
            if (issuer) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(RC) : "memory");   // DD - 1 = RC
            __syncwarp();
            dsrc[ds][lane] = dfin;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> async proxy
            __syncwarp();
            if (issuer) {
                asm volatile(
                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], 256, [%2];"
                    ::"r"(rdq[lane] + (uint32_t)(ds * 256)), "r"(smem_addr(&dsrc[ds][0])), "r"(rdfb[lane] + (uint32_t)(ds * 8))
                    : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
        dfull[lane] = dfin;
        retries += round;
        dm = fmax(dm, fabs(dfin));
        bm = fmax(bm, fabs(bnfin));
        nflip += __popc(__ballot_sync(FULL, valid && ((bnfin > 0.0) != (bo > 0.0) || (bnfin < 0.0) != (bo < 0.0))));
        if (valid) bS[s] = bnfin;
        updates += __popc(__ballot_sync(FULL, valid && dfin != 0.0));
        dbg[3] += G7CLK() - t3;
    };

    // owners: positions / slots of local index e for a sweep of `len` positions
    auto own_pos = [&](int e) { return 32 * (rank - 1 + (e >> 5) * NB) + (e & 31); };
    auto n_owned = [&](int len) {
        const int Q = (len + 31) >> 5;
        return Q > rank - 1 ? 32 * ((Q - (rank - 1) + NB - 1) / NB) : 0;
    };
    // owners: gradients to / from the global copy
    auto owner_store = [&]() {
        for (int e = t; e < owned; e += T_)
            if (sl[e] >= 0) wk.g[sl[e]] = gl[e];
        owned = 0;
    };
    auto owner_load = [&](bool active, int len) {
        owned = n_owned(len);
        for (int e = t; e < owned; e += T_) {
            const int k = own_pos(e);
            const int s = k < len ? (active ? __ldcg(wk.act + k) : k) : -1;
            sl[e] = s;
            gl[e] = s >= 0 ? __ldcg(wk.g + s) : 0.0;
        }
    };

    // one sweep over `len` positions (active: act list; full: slots).  No cluster
    // barrier per block: the leader waits on its snapshot ring, the owners on
    // their update ring, the leader's prefetch helpers on the stage ring.
    long long gq = 0;                                       // blocks processed so far (all sweeps)
    auto sweep = [&](bool active, int len) {
        visits += len;
        const double *Mx = active ? a.GA : a.G;
        const int Q = (len + 31) >> 5;
        const long long g0 = gq;
        gq += Q;
        if (leader_cta) {
            if (wid == 0) {
                dm = 0.0;
                bm = 0.0;
                double acc = 0.0;
                for (int q = 0; q < Q; q++) {
                    const long long gb = g0 + q, c0 = clock64();
                    const int ss = (int)(gb % NS), zs = (int)(gb % DZ);
                    mbar_wait(&sfull[ss], (unsigned)((gb / NS) & 1));    // Gd, M, slots of block q
                    mbar_wait(&zfull[zs], (unsigned)((gb / DZ) & 1));    // the owner's snapshot
                    const long long c1 = G7CLK();
                    dbg[4] += BL_G7_SUBPHASES ? c1 - c0 : 0;
                    const double zo = zst[zs][lane];
                    __syncwarp();
                    if (lane == 0) mbar_arm(&zfull[zs], 256);               // for block gb + DZ
                    lead(active, 32 * q, ss, zo, acc, gb);
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&sempty[ss]);                // stage free for block gb + NS
                    if (q + 1 < Q) {
                        const long long gn = gb + 1, c2 = G7CLK();
                        mbar_wait(&sfull[gn % NS], (unsigned)((gn / NS) & 1));
                        const long long c3 = G7CLK();
                        dbg[5] += c3 - c2;
                        acc = link((int)(gn % NS));
                        dbg[6] += G7CLK() - c3;
                    }
                    if (t == 0) pr_lead += clock64() - c0;
                }
            } else {
                for (int q = 0; q < Q; q++) {                            // helpers: every block's stage
                    const long long gb = g0 + q;
                    const int ss = (int)(gb % NS);
                    if (gb >= NS) mbar_wait(&sempty[ss], (unsigned)((gb / NS - 1) & 1));
                    prefetch(Mx, active, len, q, ss);
                    mbar_arrive(&sfull[ss]);
                }
            }
        } else {
            const int e0 = 2 * t;
            const int k0 = e0 < owned ? own_pos(e0) : -1;
            double2 rv[32];
            auto load_rows = [&](int qq) {                 // G rows of block qq at this thread's first pair
                if (k0 < 0) return;
#pragma unroll
                for (int i = 0; i < 32; i++) {
                    const int row = 32 * qq + i;
                    rv[i] = row < len ? __ldcg(reinterpret_cast<const double2 *>(Mx + (int64_t)row * ldG + k0))
                                      : make_double2(0.0, 0.0);
                }
            };
            auto send_snap = [&](int qq) {                 // warp 0: block qq's gradients -> the leader's ring
                if (wid != 0 || qq >= Q || (qq % NB) != rank - 1) return;
                const long long gb = g0 + qq;
                const int zs = (int)(gb % DZ);
                const int k = 32 * qq + lane;
                st_async(mapa(&zst[zs][lane], 0), k < len ? gl[lidx(k)] : 0.0, mapa(&zfull[zs], 0));
            };
            send_snap(0);                                  // blocks 0 and 1 need no update first
            send_snap(1);
            load_rows(0);
            for (int j = 0; j < Q; j++) {
                const long long gb = g0 + j, c0 = clock64();
                const int ds = (int)(gb % DD);
                mbar_wait(&dfb[ds], (unsigned)((gb / DD) & 1));
                const long long c1 = G7CLK();
                dbg[4] += BL_G7_SUBPHASES ? c1 - c0 : 0;
                if (k0 >= 0) {
                    double gx = gl[e0], gy = gl[e0 + 1], hx = 0.0, hy = 0.0;
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const double2 dd = *reinterpret_cast<const double2 *>(&dq[ds][i]);
                        gx = fma(-dd.x, rv[i].x, gx);
                        gy = fma(-dd.x, rv[i].y, gy);
                        hx = fma(-dd.y, rv[i + 1].x, hx);
                        hy = fma(-dd.y, rv[i + 1].y, hy);
                    }
                    gl[e0] = gx + hx;
                    gl[e0 + 1] = gy + hy;
                }
                for (int e = e0 + 2 * T_; e < owned; e += 2 * T_) {   // further pairs: direct loads
                    const int k = own_pos(e);
                    if (k >= len) continue;
                    double gx = gl[e], gy = gl[e + 1];
                    for (int i = 0; i < min(32, len - 32 * j); i++) {
                        const double d = dq[ds][i];
                        if (d == 0.0) continue;
                        const double2 g2 = __ldcg(reinterpret_cast<const double2 *>(Mx + (int64_t)(32 * j + i) * ldG + k));
                        gx = fma(-d, g2.x, gx);
                        gy = fma(-d, g2.y, gy);
                    }
                    gl[e] = gx;
                    gl[e + 1] = gy;
                }
                __syncthreads();
                if (t == 0) mbar_arm(&dfb[ds], 256);                // for block gb + DD
                send_snap(j + 2);
                if (j + 1 < Q) load_rows(j + 1);
                dbg[5] += G7CLK() - c1;
                if (t == 0) pr_bulk += clock64() - c0;
            }
        }
        __syncthreads();
        cl.sync();
    };

    // leader CTA: active list into act (smem) and the global copy
    auto build_active = [&]() -> int {
        int total = 0;
        for (int base = 0; base < nW; base += T_) {
            const int w = base + t;
            const bool nz = w < nW && bS[w] != 0.0;
            int pos;
            const int cnt = block_rank(nz, pos);
            if (nz) { act[total + pos] = w; wk.act[total + pos] = w; }
            total += cnt;
        }
        __syncthreads();
        return total;
    };

    // cluster: G_AA = G[act][act] (rows split over CTAs), then per block of 32
    // positions M = (I + inv N^T)^-1 (blocks split over the CTAs' warps; scratch =
    // each CTA's first 8 KB buffers)
    auto build_A = [&](int na) {
        // G_AA gather: the active list is staged in shared memory, each thread's column slots are read
        // once per 4 T_ columns, then 8 rows per step are gathered with 32 independent loads in flight
        // (the row-at-a-time loop paid two dependent L2 round trips per row)
        constexpr int RB = 8;
        int *acts = reinterpret_cast<int *>(sm + 8192);     // (the idle M stage buffers)
        for (int i = t; i < na; i += T_) acts[i] = __ldcg(wk.act + i);
        __syncthreads();
        for (int jb = 0; jb < na; jb += 4 * T_) {
            int aj[4];
#pragma unroll
            for (int k = 0; k < 4; k++) aj[k] = acts[min(jb + t + k * T_, na - 1)];
            for (int i0 = rank; i0 < na; i0 += RB * R) {
                int64_t rs[RB];
#pragma unroll
                for (int r = 0; r < RB; r++) rs[r] = (int64_t)acts[min(i0 + r * R, na - 1)] * ldG;
                double v[RB][4];
#pragma unroll
                for (int r = 0; r < RB; r++)
#pragma unroll
                    for (int k = 0; k < 4; k++) v[r][k] = __ldg(a.G + rs[r] + aj[k]);
#pragma unroll
                for (int r = 0; r < RB; r++) {
                    const int i = i0 + r * R;
                    if (i < na) {
#pragma unroll
                        for (int k = 0; k < 4; k++)
                            if (jb + t + k * T_ < na) a.GA[(int64_t)i * ldG + jb + t + k * T_] = v[r][k];
                    }
                }
            }
        }
        __syncthreads();                                    // acts is overwritten by the M scratch below
        // (cl.sync: release / acquire at cluster scope)
        cl.sync();
        const int nblk = (na + 31) / 32;
        {
            double(*N)[32] = Gd[wid];
            for (int q = rank * nw + wid; q < nblk; q += nw * R) {
                const int b0 = 32 * q, nb = min(32, na - b0);
                {                                   // lane b loads column b of the block: 32 loads in flight
                    const int b = lane;
                    const double sc = b < nb ? (a.idv ? a.idv[__ldcg(wk.act + b0 + b)] : inv_den0) : 0.0;
                    double col[32];
#pragma unroll
                    for (int p = 0; p < 32; p++)
                        col[p] = (b > p && b < nb) ? __ldcg(a.GA + (int64_t)(b0 + p) * ldG + b0 + b) : 0.0;
#pragma unroll
                    for (int p = 0; p < 32; p++) N[p][b] = sc * col[p];
                }
                __syncwarp();
                double x[32];
#pragma unroll
                for (int b = 0; b < 32; b++) x[b] = b == lane ? 1.0 : 0.0;
#pragma unroll
                for (int p = 0; p < 31; p++) {
                    const double xp = x[p];
#pragma unroll
                    for (int b = (p + 1) & ~1; b < 32; b += 2) {
                        const double2 nv = *reinterpret_cast<const double2 *>(&N[p][b]);
                        if (b > p) x[b] = fma(-nv.x, xp, x[b]);
                        x[b + 1] = fma(-nv.y, xp, x[b + 1]);
                    }
                }
                double *dst = a.MA + (int64_t)q * 1024 + lane * 32;
#pragma unroll
                for (int b = 0; b < 32; b += 2) *reinterpret_cast<double2 *>(dst + b) = make_double2(x[b], x[b + 1]);
                __syncwarp();
            }
        }
        // (cl.sync: release / acquire at cluster scope)
        cl.sync();
    };

    // cluster: gradients outside the G_AA set receive sum_i dl_i G[rl_i][k] (the change list and the
    // list of slots outside the set come from the leader).  The change list is staged in shared
    // memory; thread q handles slot clist[q] (ascending slots: a warp's loads of one G row are
    // contiguous), eight rows' loads in flight.
    auto catch_up = [&](int nz, int nk) {
        // slots in groups of 32 (lane = slot: each warp-load of a G row touches consecutive slots),
        // groups block-cyclic over the CTAs; within a CTA the 8 warps split the change list and
        // their partial sums are combined in warp order (deterministic).  One thread per slot with
        // the whole list left most of the cluster idle: ~55k cycles per catch-up on cfg3.
        if (nz > 0 && nk > 0) {
            double *dls = sm;                                   // the stage buffers are idle here
            int *rls = reinterpret_cast<int *>(sm + 4096);
            double *part = sm + 6144;                           // [8 warps][32 slots]
            const int *clist = reinterpret_cast<const int *>(wk.cg + 4 * nWp);
            for (int i = t; i < nz; i += T_) { dls[i] = __ldcg(wk.dl + i); rls[i] = __ldcg(wk.rl + i); }
            __syncthreads();
            const int i0w = (int)((int64_t)wid * nz / nw), i1w = (int)((int64_t)(wid + 1) * nz / nw);
            const int ngrp = (nk + 31) >> 5;
            for (int g = rank; g < ngrp; g += R) {
                const int q = 32 * g + lane;
                const int k = __ldcg(clist + min(q, nk - 1));
                double acc[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                int i = i0w;
                for (; i + 8 <= i1w; i += 8) {
                    double gv[8];
#pragma unroll
                    for (int v = 0; v < 8; v++) gv[v] = __ldcg(a.G + (int64_t)rls[i + v] * ldG + k);
#pragma unroll
                    for (int v = 0; v < 8; v++) acc[v] = fma(dls[i + v], gv[v], acc[v]);
                }
                for (; i < i1w; i++) acc[0] = fma(dls[i], __ldcg(a.G + (int64_t)rls[i] * ldG + k), acc[0]);
                part[wid * 32 + lane] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
                __syncthreads();
                if (wid == 0 && q < nk) {
                    double sum = 0.0;
                    for (int w = 0; w < nw; w++) sum += part[w * 32 + lane];
                    wk.g[k] -= sum;
                }
                __syncthreads();
            }
        }
        // (cl.sync: release / acquire at cluster scope)
        cl.sync();
    };

    // ---- Newton step on a settled active set (CdGramArgs::newton; linear path only).
    // With the signs s of the active coefficients fixed, the CD fixed point on A solves
    //   (G_AA + nu I) x = b,   b = g_A - lambda alpha s - nu beta_A          (P:267's CD)
    // (g = x~'r/n by slot; G_AA compact by active position).  Conjugate gradients from x = 0 in
    // the Chronopoulos-Gear form (one product and ONE fused reduction per iteration: two
    // cluster barriers), rows split over the cluster.  Every CG iterate lowers this quadratic,
    // and so does every point of the segment [0, x]: the step beta_A += t x with the largest
    // t <= 1 that keeps every sign (coefficients reaching 0 are set to 0) lowers the objective.
    // The CD sweeps that follow decide convergence exactly as before, so the result is still a
    // converged CD fixed point.  Gradients of A are updated here (g_A -= G_AA (new - old));
    // those outside A by the lazy catch-up.
    double *cgx = wk.cg, *cgr = wk.cg + nWp, *cgb = wk.cg + 3 * nWp;
    __shared__ double cgpart[4][2], cgred[2][32], cgbc[2];
    int cgslot = 0;
    // cluster sums (or min) of two doubles per CTA (thread 0's values), combined in rank order
    // by warp 0 of every CTA: identical on every CTA
    auto cl_reduce2 = [&](double v0, double v1, bool is_min, double &o0, double &o1) {
        double *slot = cgpart[cgslot & 3];
        cgslot++;
        if (t == 0) { slot[0] = v0; slot[1] = v1; }
        cl.sync();
        if (wid == 0) {
            const double *rs = lane < R ? cl.map_shared_rank(slot, lane) : nullptr;
            const double u0 = rs ? rs[0] : 0.0, u1 = rs ? rs[1] : 0.0;
            double a0 = is_min ? 1e300 : 0.0, a1 = a0;
            for (int r = 0; r < R; r++) {
                const double w0 = __shfl_sync(FULL, u0, r), w1 = __shfl_sync(FULL, u1, r);
                a0 = is_min ? fmin(a0, w0) : a0 + w0;
                a1 = is_min ? fmin(a1, w1) : a1 + w1;
            }
            if (lane == 0) { cgbc[0] = a0; cgbc[1] = a1; }
        }
        __syncthreads();
        o0 = cgbc[0];                // rewritten only after the next cl.sync, which every reader passes first
        o1 = cgbc[1];
    };
    auto cta_sum2 = [&](double v0, double v1, double &s0, double &s1) {   // thread 0 gets the CTA sums
        v0 = warp_sum(v0);
        v1 = warp_sum(v1);
        __syncthreads();
        if (lane == 0) { cgred[0][wid] = v0; cgred[1][wid] = v1; }
        __syncthreads();
        s0 = 0.0;
        s1 = 0.0;
        if (t == 0)
            for (int w = 0; w < nw; w++) { s0 += cgred[0][w]; s1 += cgred[1][w]; }
        __syncthreads();
    };
    // rows [r0, r1) of w = (G_AA + nu I) v (v: na entries in shared memory, vsh[na] = 0 when na is
    // odd); two rows per warp.  The first ncache rows of this CTA are read from a shared-memory copy
    // (gc, row stride nap) held in fp32 -- twice the rows fit, half the bytes per product -- the rest
    // from L2 (fp64) with eight 16-byte loads per row and lane in flight.  The CG solves with this
    // operator (its recurrence residual is the residual for it); the step it yields is only an
    // accelerator: the fp64 sweeps that follow decide convergence (Q30), and the gradient update
    // after the step uses the fp64 G_AA (matvec with gc = nullptr).
    auto matvec = [&](const double *vsh, double *wsh, int na, int r0, int r1, double nu_, const float *gc, int ncache,
                      int nap, float *vf) {
        int rs = r0;                                        // first row of the L2 (fp64) part
        if (gc && ncache > 0) {
            // the cached rows: fp32 products with an fp32 copy of v, four rows per warp sharing each
            // v load, the lane's partial sums (<= na/64 terms) in fp32, the warp sum in fp64 -- the
            // per-element fp32 -> fp64 conversions (16 per SM clock) bound the fp64 form
            for (int j = t; j < nap; j += T_) vf[j] = j < na ? (float)vsh[j] : 0.f;
            __syncthreads();
            for (int l0 = 4 * wid; l0 < ncache; l0 += 4 * nw) {
                const int nr = min(4, ncache - l0);
                const float *g0 = gc + (size_t)l0 * nap;
                float2 acc[4];
#pragma unroll
                for (int q = 0; q < 4; q++) acc[q] = make_float2(0.f, 0.f);
#pragma unroll 2
                for (int j = 2 * lane; j < na; j += 64) {
                    const float2 vv = *reinterpret_cast<const float2 *>(vf + j);
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (q < nr) {
                            const float2 g = *reinterpret_cast<const float2 *>(g0 + (size_t)q * nap + j);
                            acc[q].x = fmaf(g.x, vv.x, acc[q].x);
                            acc[q].y = fmaf(g.y, vv.y, acc[q].y);
                        }
                }
                // the four row sums in one butterfly (fixed order): after the xor-16 and xor-8
                // exchanges each lane holds one row's partial (row 2 (lane >> 4 & 1) + (lane >> 3 & 1))
                const double v0 = (double)acc[0].x + (double)acc[0].y, v1 = (double)acc[1].x + (double)acc[1].y;
                const double v2 = (double)acc[2].x + (double)acc[2].y, v3 = (double)acc[3].x + (double)acc[3].y;
                const bool hi16 = lane & 16, hi8 = lane & 8;
                double ka = hi16 ? v2 : v0, kb = hi16 ? v3 : v1;
                ka += __shfl_xor_sync(FULL, hi16 ? v0 : v2, 16);
                kb += __shfl_xor_sync(FULL, hi16 ? v1 : v3, 16);
                double kr = hi8 ? kb : ka;
                kr += __shfl_xor_sync(FULL, hi8 ? ka : kb, 8);
                kr += __shfl_xor_sync(FULL, kr, 4);
                kr += __shfl_xor_sync(FULL, kr, 2);
                kr += __shfl_xor_sync(FULL, kr, 1);
                const int q = (hi16 ? 2 : 0) + (hi8 ? 1 : 0);
                if ((lane & 7) == 0 && q < nr) wsh[l0 + q] = kr + nu_ * vsh[r0 + l0 + q];
            }
            rs = r0 + ncache;
        }
        for (int i = rs + 2 * wid; i < r1; i += 2 * nw) {
            const bool two = i + 1 < r1;
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
            {
                const double *ra = a.GA + (int64_t)i * ldG, *rb = a.GA + (int64_t)(two ? i + 1 : i) * ldG;
                for (int j0 = 2 * lane; j0 < na; j0 += 64 * 8) {
                    double2 ga[8], gb[8];
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int j = j0 + 64 * u;
                        ga[u] = j < na ? __ldcg(reinterpret_cast<const double2 *>(ra + j)) : make_double2(0.0, 0.0);
                        gb[u] = j < na ? __ldcg(reinterpret_cast<const double2 *>(rb + j)) : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int u = 0; u < 8; u++) {
                        const int j = j0 + 64 * u;
                        if (j < na) {
                            const double2 vv = *reinterpret_cast<const double2 *>(vsh + j);
                            a0 = fma(ga[u].x, vv.x, a0);
                            a1 = fma(ga[u].y, vv.y, a1);
                            b0 = fma(gb[u].x, vv.x, b0);
                            b1 = fma(gb[u].y, vv.y, b1);
                        }
                    }
                }
            }
            const double wa = warp_sum(a0 + a1), wb = warp_sum(b0 + b1);
            if (lane == 0) {
                wsh[i - r0] = wa + nu_ * vsh[i];
                if (two) wsh[i + 1 - r0] = wb + nu_ * vsh[i + 1];
            }
        }
    };
    long long ncg = 0, nnewton = 0, pr_newton = 0, npartial = 0, nchecks = 0;
    unsigned rph = 0u, pph = 0u;                            // Newton CG: phase parities of cgbar[0], cgbar[1]
    auto newton = [&](int na, double thr) {
        const long long c0 = clock64();
        // shared memory (the stage buffers are idle): vsh = the full vector (na, +1 pad when odd),
        // then this CTA's rows of x, p, s, w, then as many of its G_AA rows as fit
        const int vlen = (na + 2) & ~1, owp = ((na + NB - 1) / NB + 2) & ~1;
        double *vsh = sm;
        double *xs = sm + vlen, *ps = xs + owp, *ss = ps + owp, *wsh = ss + owp;
        // rows of G_AA are split over the owner CTAs (the leader keeps its per-slot state in shared
        // memory); each owner copies as many of its rows as fit into its (otherwise idle) shared memory
        const int r0 = rank == 0 ? 0 : (int)((int64_t)(rank - 1) * na / NB);
        const int r1 = rank == 0 ? 0 : (int)((int64_t)rank * na / NB);
        const int nap = (na + 1) & ~1;
        float *vf = reinterpret_cast<float *>(wsh + owp);   // fp32 copy of v (vlen entries)
        float *gc = vf + vlen;                              // fp32 rows (8-byte aligned: vlen, nap even)
        const int cap = rank == 0 ? 0 : (int)((((int64_t)a.smem_bytes / 8 - (vlen + 4 * owp)) * 2 - vlen) / nap);
        const int ncache = max(0, min(r1 - r0, cap));
        for (int l = wid; l < ncache; l += nw) {            // a row per warp, 16 loads per lane in flight
            const double *src = a.GA + (int64_t)(r0 + l) * ldG;
            float *dst = gc + (size_t)l * nap;
            for (int j0 = 2 * lane; j0 < na; j0 += 64 * 8) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int j = j0 + 64 * u;
                    v[u] = j < na ? __ldcg(reinterpret_cast<const double2 *>(src + j)) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int u = 0; u < 8; u++) {
                    const int j = j0 + 64 * u;
                    if (j < na) *reinterpret_cast<float2 *>(dst + j) = make_float2((float)v[u].x, j + 1 < na ? (float)v[u].y : 0.f);
                }
            }
        }
        const double la = a.lam_alpha, nu = a.nu;
        // The CG iterations run on the owner CTAs only (the leader holds no rows; it rejoins at the
        // step below).  The residual's rows travel straight into every other owner's vsh
        // (st.async, completing on that owner's cgbar[0]), and the partial sums into every owner's
        // cgpsum (cgbar[1]): no cluster barrier and no L2 round trip per iteration.  Reuse is safe
        // without more synchronisation because every owner both sends and needs both messages: an
        // owner sends phase k+1 of either only after the reduction of phase k, which needs every
        // peer's partial k, which a peer sends only after it finished reading its vsh / slots of
        // phase k.  (With the leader taking part, it -- needing nothing from the others between two
        // reductions -- sent its partial k+1 as soon as its own reduction k completed, which could
        // reach an owner still waiting on a slow partial k: a phase mix-up that deadlocked a run.)
        const int own = r1 - r0;
        auto share_r = [&]() {                              // this CTA's rows (already in vsh) -> the peers
            __syncthreads();                                // (the rows were written by other threads)
            const int npeer = NB - 1;
            for (int e = t; e < own * npeer; e += T_) {
                const int i = r0 + e % own;
                int pr = 1 + e / own;
                if (pr >= rank) ++pr;
                st_async(mapa(vsh + i, pr), vsh[i], mapa(&cgbar[0], pr));
            }
            if (t == 0) {
                if (na & 1) vsh[na] = 0.0;
                mbar_arm(&cgbar[0], (unsigned)(8 * (na - own)));
            }
            __syncthreads();
            mbar_wait(&cgbar[0], rph);
            rph ^= 1u;
        };
        auto p2p_reduce2 = [&](double v0, double v1, double &o0, double &o1) {   // owners; thread 0's values
            if (wid == 0) {
                const double u0 = __shfl_sync(FULL, v0, 0), u1 = __shfl_sync(FULL, v1, 0);
                if (lane >= 1 && lane < R && lane != rank) {   // the other owners' slots [rank]
                    const uint32_t dst = mapa(&cgpsum[rank][0], lane), bar = mapa(&cgbar[1], lane);
                    st_async(dst, u0, bar);
                    st_async(dst + 8, u1, bar);
                }
                if (lane == 0) {
                    cgpsum[rank][0] = u0;                   // this CTA's own slot
                    cgpsum[rank][1] = u1;
                    mbar_arm(&cgbar[1], (unsigned)(16 * (R - 2)));
                }
            }
            mbar_wait(&cgbar[1], pph);
            pph ^= 1u;
            __syncthreads();                                // (the own slot, written by thread 0)
            double s0 = 0.0, s1 = 0.0;
            for (int r = 1; r < R; r++) { s0 += cgpsum[r][0]; s1 += cgpsum[r][1]; }   // owner rank order
            o0 = s0;
            o1 = s1;
        };
        int it = 0;
        if (rank != 0) {                                    // ---- CG on the owners
        for (int i = r0 + t; i < r1; i += T_) {             // r = b (x = 0)
            const double bi = __ldcg(cgb + i);
            vsh[i] = __ldcg(wk.g + __ldcg(wk.act + i)) - (bi > 0.0 ? la : -la) - nu * bi;
            xs[i - r0] = 0.0;
        }
        share_r();
        matvec(vsh, wsh, na, r0, r1, nu, gc, ncache, nap, vf);
        __syncthreads();
        double g0 = 0.0, d0 = 0.0;
        for (int i = r0 + t; i < r1; i += T_) { g0 = fma(vsh[i], vsh[i], g0); d0 = fma(wsh[i - r0], vsh[i], d0); }
        double gam, del;
        cta_sum2(g0, d0, g0, d0);
        p2p_reduce2(g0, d0, gam, del);
        const double thr2 = thr * thr;
        const int itmax = min(na, 256);
        if (gam > thr2 && del > 0.0) {
            double al = gam / del;
            for (int i = r0 + t; i < r1; i += T_) { ps[i - r0] = vsh[i]; ss[i - r0] = wsh[i - r0]; }
            for (;;) {
                for (int i = r0 + t; i < r1; i += T_) {     // x += al p, r -= al s
                    const int l = i - r0;
                    xs[l] = fma(al, ps[l], xs[l]);
                    vsh[i] = fma(-al, ss[l], vsh[i]);
                }
                const long long q0 = CGCLK();
                share_r();                                  // (every peer finished reading vsh: reduction k)
                const long long q1 = CGCLK(), q2 = q1;
                matvec(vsh, wsh, na, r0, r1, nu, gc, ncache, nap, vf);
                __syncthreads();
                const long long q3 = CGCLK();
                double gp = 0.0, dp = 0.0;
                for (int i = r0 + t; i < r1; i += T_) { gp = fma(vsh[i], vsh[i], gp); dp = fma(wsh[i - r0], vsh[i], dp); }
                double gn, dn;
                cta_sum2(gp, dp, gp, dp);
                const long long q4 = CGCLK();
                p2p_reduce2(gp, dp, gn, dn);
                const long long q5 = CGCLK();
                if (BL_CG_PHASES && rank == 1 && t == 0) {    // (an owner's view; sub-phase cycles)
                    dbg[0] += q1 - q0; dbg[1] += q2 - q1; dbg[2] += q3 - q2; dbg[3] += q4 - q3; dbg[4] += q5 - q4;
                }
                ++it;
                if (gn <= thr2 || it >= itmax) break;
                const double be = gn / gam;
                const double den = dn - be * gn / al;
                if (!(den > 0.0)) break;                    // no curvature left (semi-definite G_AA)
                al = gn / den;
                gam = gn;
                for (int i = r0 + t; i < r1; i += T_) {     // p = r + be p, s = w + be s
                    const int l = i - r0;
                    ps[l] = fma(be, ps[l], vsh[i]);
                    ss[l] = fma(be, ss[l], wsh[l]);
                }
            }
        }
        }                                                   // ---- (owners)
        // largest step t <= 1 that keeps every active sign; x -> global for every CTA
        double tmin = 1.0;
        for (int i = r0 + t; i < r1; i += T_) {
            const double bi = __ldcg(cgb + i), xi = xs[i - r0];
            cgx[i] = xi;
            if (bi * xi < 0.0 && fabs(xi) >= fabs(bi)) tmin = fmin(tmin, -bi / xi);
        }
        tmin = -warp_max(-tmin);
        __syncthreads();
        if (lane == 0) cgred[0][wid] = tmin;
        __syncthreads();
        double tc = 1.0;
        if (t == 0) for (int w = 0; w < nw; w++) tc = fmin(tc, cgred[0][w]);
        __syncthreads();
        double ts, unused;
        cl_reduce2(tc, tc, true, ts, unused);               // (its barrier also publishes x)
        // the applied changes d = new - old (identical on every CTA), then g_A -= G_AA d
        for (int j = t; j < na; j += T_) {
            const double bi = __ldcg(cgb + j), xi = __ldcg(cgx + j);
            const double bn = fma(ts, xi, bi);
            const double bnew = (bi > 0.0 ? bn > 0.0 : bn < 0.0) ? bn : 0.0;
            vsh[j] = bnew - bi;
            if (leader_cta) bS[__ldcg(wk.act + j)] = bnew;
        }
        if (t == 0 && (na & 1)) vsh[na] = 0.0;
        __syncthreads();
        matvec(vsh, wsh, na, r0, r1, 0.0, nullptr, 0, nap, nullptr);   // fp64 G_AA: the exact gradient update
        __syncthreads();
        for (int i = r0 + t; i < r1; i += T_) {
            const int s = __ldcg(wk.act + i);
            wk.g[s] = __ldcg(wk.g + s) - wsh[i - r0];
        }
        if (ts < 1.0) ++npartial;
        ncg += it;
        ++nnewton;
        cl.sync();                                          // gradients published (release / acquire)
        pr_newton += clock64() - c0;
    };

    // ---- control loop.  The leader decides, the cluster follows.  ctl[ph]:
    // [0] catch-up, [1] its count, [2] rebuild G_AA / M, [3] mode (0 full, 1 active, 2 Newton step,
    // -1 stop), [4] len, [5] owners reload their positions; ctld[ph][0] = the CG tolerance
    bool full = false, built = false, pending = false;
    int na_built = 0, last_mode = -1, last_len = -1, ph = 0;
    int sweeps_on_set = 0, newtons_on_set = 0;            // leader: active sweeps / Newton steps on the built set
    double dm_last = 0.0, dm_prev = 0.0;                  // leader: dmax of the last two active sweeps
    bool conv_last = false;
    bool check_ok = false, force_full = false;            // leader: the W check (mode 3) passed / failed
    __shared__ double ctld[2][2];
    for (;; ph ^= 1) {
        if (leader_cta) {
            int cmd_catch = 0, ncat = 0, nkc = 0, cmd_build = 0, mode = 0, len = nW, nz3 = 0;
            double cg_thr = 0.0;
            if (status || check_ok || (passes > 0 && full && red[2] != 0.0)) {
                mode = -1;                                    // stop (set below after a sweep)
            } else {
                for (;;) {
                    if (!full) {
                        len = build_active();
                        bool same = built && len == na_built;
                        if (same) {
                            int diff = 0;
                            for (int i = t; i < len; i += T_) diff |= act[i] != actp[i];
                            same = !__syncthreads_or(diff);
                        }
                        if (!same) {
                            if (pending) { cmd_catch = 1; pending = false; }
                            if (len == 0) { full = true; continue; }
                            cmd_build = 1;
                        }
                        mode = 1;
                        // a settled active set (the last sweep kept the set and every sign, and did
                        // not converge): one Newton step instead of the remaining sweeps
                        if (a.newton && same && last_mode == 1 && !conv_last && red[3] == 0.0 &&
                            sweeps_on_set >= BL_NEWTON_SWEEPS && newtons_on_set < BL_NEWTON_MAX && len >= 32 &&
                            (BL_NEWTON_SWEEPS < 2 || (dm_prev > 0.0 && dm_last > BL_NEWTON_RHO * dm_prev))) {
                            mode = 2;
                            // CG stops at an rms residual of 0.2 tol max|beta| (the sweep that follows
                            // resolves the rest)
                            cg_thr = BL_CG_RTOL * fmax(a.tol * red[1], a.floor_) * sqrt((double)len);
                        }
                    } else {
                        if (pending) { cmd_catch = 1; pending = false; }
                        // with Newton steps on (CdGramArgs::newton), the full pass that must confirm a
                        // converged active set is first replaced by its exact outcome for the zero
                        // coordinates: a zero coefficient stays zero in a CD update iff |g_w| <= its
                        // threshold, and the active ones just passed a converged sweep.  Only if some
                        // zero coordinate would move does the full sweep run.
                        mode = (a.newton && !force_full) ? 3 : 0;
                        force_full = false;
                        len = nW;
                    }
                    break;
                }
            }
            if (cmd_catch) {                                  // coefficient changes since the last catch-up
                int nz = 0;
                for (int base = 0; base < na_built; base += T_) {
                    const int i = base + t;
                    const int s = i < na_built ? actp[i] : 0;
                    const double dlt = i < na_built ? bS[s] - bcat[s] : 0.0;
                    int pos;
                    const int cnt = block_rank(dlt != 0.0, pos);
                    if (dlt != 0.0) { wk.dl[nz + pos] = dlt; wk.rl[nz + pos] = s; }
                    nz += cnt;
                }
                int nk = 0;                                   // slots outside the built set (ascending)
                int *clist = reinterpret_cast<int *>(wk.cg + 4 * nWp);
                for (int base = 0; base < nW; base += T_) {
                    const int w = base + t;
                    const bool out_ = w < nW && !inA[w];
                    int pos;
                    const int cnt = block_rank(out_, pos);
                    if (out_) clist[nk + pos] = w;
                    nk += cnt;
                }
                ncat = nz;
                nkc = nk;
            }
            if (cmd_build) {
                __syncthreads();
                for (int i = t; i < nWp; i += T_) inA[i] = 0;
                __syncthreads();
                for (int i = t; i < len; i += T_) { actp[i] = act[i]; inA[act[i]] = 1; }
                built = true;
                na_built = len;
                sweeps_on_set = 0;
                newtons_on_set = 0;
            }
            if (mode == 1 && (cmd_build || !pending)) {
                __syncthreads();
                for (int i = t; i < len; i += T_) bcat[act[i]] = bS[act[i]];
                pending = true;
            }
            if (mode == 2) {                                  // the coefficients by active position
                for (int i = t; i < len; i += T_) wk.cg[3 * nWp + i] = bS[act[i]];
                ++newtons_on_set;
            }
            if (mode == 3) {                                  // the zero coordinates of W (slots)
                int *zl = reinterpret_cast<int *>(wk.cg);
                __syncthreads();
                for (int base = 0; base < nW; base += T_) {
                    const int w = base + t;
                    const bool z0 = w < nW && bS[w] == 0.0;
                    int pos;
                    const int cnt = block_rank(z0, pos);
                    if (z0) zl[nz3 + pos] = w;
                    nz3 += cnt;
                }
            }
            const int reload = mode != last_mode || len != last_len || cmd_build || cmd_catch;
            last_mode = mode;
            last_len = len;
            if (t == 0) {
                ctl[ph][0] = cmd_catch; ctl[ph][1] = ncat; ctl[ph][2] = cmd_build;
                ctl[ph][3] = mode; ctl[ph][4] = len; ctl[ph][5] = reload; ctl[ph][6] = nkc; ctl[ph][7] = nz3;
                ctld[ph][0] = cg_thr;
            }
            // cl.sync()'s arrive.release / wait.acquire orders these writes for the cluster
        }
        cl.sync();
        const int *rc = cl.map_shared_rank(&ctl[ph][0], 0);
        const int cmd_catch = rc[0], ncat = rc[1], cmd_build = rc[2], mode = rc[3], len = rc[4], reload = rc[5];
        const int nkc = rc[6], nz3 = rc[7];
        const double cg_thr = *cl.map_shared_rank(&ctld[ph][0], 0);
        if (!leader_cta && (reload || mode < 0)) owner_store();
        if (mode < 0) break;
        if (reload) cl.sync();                              // owners' stores ordered by the release barrier
        if (cmd_catch) {
            const long long c0 = clock64();
            catch_up(ncat, nkc);
            ++ncatch;
            pr_catch += clock64() - c0;
        }
        if (cmd_build) {
            const long long c0 = clock64();
            build_A(len);
            ++rebuilds;
            pr_build += clock64() - c0;
        }
        if (mode == 2) {
            newton(len, cg_thr);
            continue;                                       // no sweep: the next one verifies
        }
        if (mode == 3) {                                    // the W check: would a zero coordinate move?
            const int *zl = reinterpret_cast<const int *>(wk.cg);
            double nv = 0.0;
            for (int q = rank * T_ + t; q < nz3; q += R * T_) {
                const int w = __ldcg(zl + q);
                const double thr = a.tau ? a.tau[w] : a.lam_alpha;
                nv += fabs(__ldcg(wk.g + w)) > thr ? 1.0 : 0.0;
            }
            double tot = 0.0, unused;
            double cs;
            cta_sum2(nv, 0.0, cs, unused);
            cl_reduce2(cs, 0.0, false, tot, unused);
            ++nchecks;
            if (leader_cta) {
                if (tot == 0.0) check_ok = true;
                else force_full = true;
            }
            continue;
        }
        if (!leader_cta && reload) { owner_load(mode == 1, len); __syncthreads(); }
        nfull += mode == 0;
        if (leader_cta && wid == 0) nflip = 0;
        sweep(mode == 1, len);
        if (leader_cta) {                                     // convergence of the pass (leader only)
            if (wid == 0) {
                const double dmw = warp_max(dm), bmw = warp_max(bm);
                if (t == 0) { red[0] = dmw; red[1] = bmw; red[3] = (double)nflip; }
            }
            __syncthreads();
            const double dmax = red[0], bmax = red[1];
            __syncthreads();
            const bool conv = dmax <= a.tol * bmax || dmax <= a.floor_;
            if (++passes > a.max_iter) status = 3;
            if (mode == 1) { ++sweeps_on_set; dm_prev = dm_last; dm_last = dmax; }
            conv_last = conv;
            if (t == 0) red[2] = (full && conv) ? 1.0 : 0.0;   // stop after a converged full pass
            __syncthreads();
            if (red[2] == 0.0) full = conv;
        }
    }
    if (leader_cta && wid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    cl.sync();                                              // no DSMEM access past this point
    if (!leader_cta) {
        if (rank == 1 && t == 0) {
            a.st->cd_prof[1] = pr_bulk;
            a.st->cd_cnt[5] = ncg;                          // (CG iterations run on the owners)
        }
        if (BL_CG_PHASES && rank == 1 && t == 0)
            for (int u = 0; u < 5; u++) a.st->cd_dbg[u] = dbg[u];
        return;
    }
    double l1 = 0.0, l2 = 0.0, nnz = 0.0;
    for (int q = t; q < nW; q += T_) {
        const int w = a.ord[q];
        const double bv = bS[w];
        const int j = a.Wst[w];
        const double b0 = a.beta[j];
        a.beta[j] = bv;
        a.dbeta[w] = bv - b0;
        a.betaW_out[q] = bv;
        a.betaW_out[nW + q] = a.c[j];
        a.betaW_out[2 * nW + q] = a.s[j];
        l1 += fabs(bv);
        l2 = fma(bv, bv, l2);
        nnz += bv != 0.0 ? 1.0 : 0.0;
    }
    l1 = block_sum(l1, red);
    l2 = block_sum(l2, red);
    nnz = block_sum(nnz, red);
    if (t == 0) {
        a.st->cd_passes = passes;
        a.st->cd_status = status;
        a.st->l1 = l1;
        a.st->l2 = l2;
        a.st->nnz = (int)nnz;
        a.st->cd_visits = visits;
        a.st->cd_updates = updates;
        a.st->cd_cycles = clock64() - clk0;
        a.st->cd_prof[0] = pr_lead;
        a.st->cd_prof[2] = pr_build;
        a.st->cd_prof[3] = pr_catch;
        a.st->cd_cnt[0] = retries;
        a.st->cd_cnt[1] = rebuilds;
        a.st->cd_cnt[2] = ncatch;
        a.st->cd_cnt[3] = nfull;
        a.st->cd_cnt[4] = nnewton;
        a.st->cd_cnt[6] = pr_newton;
        a.st->cd_cnt[7] = npartial;
        dbg[7] = nchecks;                                   // (slot 7: W checks, not a sub-phase)
        for (int u = BL_CG_PHASES ? 5 : 0; u < 8; u++) a.st->cd_dbg[u] = dbg[u];   // leader warp sub-phases
    }
}

// ------------------------------------- sharded designs: working-set column store
__global__ void k_iota(int *__restrict__ v, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}
// Owner side of the column broadcast (C4): local columns cols[0..k) -> store
// slots slot0.. (raw bytes, ld elements each) with their c, s.  grid = (k, any).
__global__ void k_pack_cols(const char *__restrict__ X, int64_t col_bytes, const int *__restrict__ cols, int k,
                            const double *__restrict__ c, const double *__restrict__ s, char *__restrict__ Xw,
                            double *__restrict__ cw, double *__restrict__ sw, double *__restrict__ bw, int slot0) {
    const int q = blockIdx.x;
    if (q >= k) return;
    const int j = cols[q];
    const int4 *src = reinterpret_cast<const int4 *>(X + (int64_t)j * col_bytes);
    int4 *dst = reinterpret_cast<int4 *>(Xw + (int64_t)(slot0 + q) * col_bytes);
    for (int64_t i = threadIdx.x; i < col_bytes / 16; i += blockDim.x) dst[i] = src[i];
    if (threadIdx.x == 0) {
        cw[slot0 + q] = c[j];
        sw[slot0 + q] = s[j];
        bw[slot0 + q] = 0.0;
    }
}

// ------------------------------------------------ a12: cross-validation errors
// E[i] = r_i^2 for the held-out rows (mask == 0) of one fold at one lambda:
// r on held-out rows is y_i - yhat_i from the fold's fit (the CD keeps the full-row
// residual), so no copy or gather of X is needed.
__global__ void k_heldout(const double *__restrict__ r, const uint8_t *__restrict__ mask, int n,
                          double *__restrict__ E) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && !mask[i]) E[i] = r[i] * r[i];
}

// cve_k = mean_i E[k, i];  cvse_k = sd_i(E[k, i]) / sqrt(n)  (Q17).  One block per lambda.
__global__ void k_cv_reduce(const double *__restrict__ E, int n, double *__restrict__ cve,
                            double *__restrict__ cvse) {
    __shared__ double sh[32];
    const double *e = E + (size_t)blockIdx.x * n;
    double s = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) s += e[i];
    const double m = block_sum(s, sh) / (double)n;
    double v = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) { double d = e[i] - m; v = fma(d, d, v); }
    v = block_sum(v, sh);
    if (threadIdx.x == 0) {
        cve[blockIdx.x] = m;
        cvse[blockIdx.x] = sqrt(v / (double)(n - 1)) / sqrt((double)n);
    }
}

// r -= X~_W dbeta on every row (held-out rows included); r_scan = r on used
// rows.  Two stages, deterministic: k_resid_part sums 64-column chunks of W per
// row block into part[chunk][row]; k_resid_apply adds the chunks in order and
// writes per-block partial sums of r_scan and r_scan^2 (finished by k_resid_finish).
constexpr int kResidChunk = 64;
template <typename T, bool MASK>
__global__ void __launch_bounds__(256) k_resid_part(const T *__restrict__ X, int64_t ld, int n,
                                                    const int *__restrict__ Wst, int nW,
                                                    const double *__restrict__ dbeta,
                                                    const double *__restrict__ c, const double *__restrict__ s,
                                                    double *__restrict__ part) {
    __shared__ int sj[kResidChunk];
    __shared__ double sf[kResidChunk], sc[kResidChunk];
    __shared__ int wcnt[2];
    static_assert(kResidChunk == 64, "two warps compact the chunk");
    const int tid = threadIdx.x, u0 = blockIdx.y * kResidChunk;
    const int cnt = min(kResidChunk, nW - u0);
    bool nz = false;
    int j = 0, pos = 0;
    double f = 0.0, cc = 0.0;
    if (tid < kResidChunk) {                  // the chunk's nonzero updates, compacted in order
        if (tid < cnt) {
            const double d = dbeta[u0 + tid];
            nz = d != 0.0;
            if (nz) {
                j = Wst[u0 + tid];
                f = d / s[j];
                cc = c[j];
            }
        }
        const unsigned m = __ballot_sync(0xffffffffu, nz);
        if ((tid & 31) == 0) wcnt[tid >> 5] = __popc(m);
        pos = __popc(m & ((1u << (tid & 31)) - 1u));
    }
    __syncthreads();
    if (nz) {
        const int q = pos + (tid >= 32 ? wcnt[0] : 0);
        sj[q] = j;
        sf[q] = f;
        sc[q] = cc;
    }
    const int nnz = wcnt[0] + wcnt[1];
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ld) return;
    double acc = 0.0;
    if (i < n) {
        const int k = nnz;
        int u = 0;
        for (; u + 4 <= k; u += 4) {
            const double x0 = to_d(X[(int64_t)sj[u] * ld + i]), x1 = to_d(X[(int64_t)sj[u + 1] * ld + i]);
            const double x2 = to_d(X[(int64_t)sj[u + 2] * ld + i]), x3 = to_d(X[(int64_t)sj[u + 3] * ld + i]);
            acc = fma(sf[u], x0 - sc[u], acc);
            acc = fma(sf[u + 1], x1 - sc[u + 1], acc);
            acc = fma(sf[u + 2], x2 - sc[u + 2], acc);
            acc = fma(sf[u + 3], x3 - sc[u + 3], acc);
        }
        for (; u < k; u++) acc = fma(sf[u], to_d(X[(int64_t)sj[u] * ld + i]) - sc[u], acc);
    }
    part[(int64_t)blockIdx.y * ld + i] = acc;
}

template <bool MASK>
__global__ void __launch_bounds__(256) k_resid_apply(const double *__restrict__ part, int nchunk, int64_t ld, int n,
                                                     const uint8_t *__restrict__ mask, double *__restrict__ r,
                                                     double *__restrict__ r_scan, double *__restrict__ bpart,
                                                     RoundStatus *st) {
    __shared__ double red[32];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double rs = 0.0, rr = 0.0;
    if (i < n) {
        double acc = 0.0;
        for (int ch = 0; ch < nchunk; ch++) acc += part[(int64_t)ch * ld + i];
        const double v = r[i] - acc;
        r[i] = v;
        const bool use = !MASK || mask[i];
        const double vs = use ? v : 0.0;
        r_scan[i] = vs;
        rs = vs;
        rr = vs * vs;
    } else if (i < ld) {
        r_scan[i] = 0.0;
    }
    rs = block_sum(rs, red);
    rr = block_sum(rr, red);
    __shared__ bool last;
    if (threadIdx.x == 0) {
        bpart[2 * blockIdx.x] = rs;
        bpart[2 * blockIdx.x + 1] = rr;
        __threadfence();
        last = atomicAdd(&st->blk_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {       // the last block: sum r and ||r||^2 in a fixed block order
        __threadfence();
        double s1 = 0.0, s2 = 0.0;
        for (int b = 0; b < (int)gridDim.x; b++) { s1 += __ldcg(bpart + 2 * b); s2 += __ldcg(bpart + 2 * b + 1); }
        st->sumr = s1;
        st->rss = s2;
        st->blk_done = 0;
    }
}

__global__ void k_resid_finish(const double *__restrict__ part, int nb, RoundStatus *st) {
    if (threadIdx.x == 0) {
        double rs = 0.0, rr = 0.0;
        for (int b = 0; b < nb; b++) { rs += part[2 * b]; rr += part[2 * b + 1]; }
        st->sumr = rs;
        st->rss = rr;
    }
}

}  // namespace bl
