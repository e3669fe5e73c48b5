// bl_kernels.cuh -- sm_100a kernels of the lasso / elastic-net path (biglasso,
// arXiv 1701.05936).  Citations: P:n = PAPER.md line n, S:n = SPEC.md line n,
// Qk = DESIGN.md section 3 reading k, "a9" etc. = SURVEY.md 8(a) rows.
//
// Layout: X column-major in HBM, x_ij at X[j*ld + i],
// column starts 16-byte aligned; the standardised matrix is never formed --
// every kernel applies (x - c_j)/s_j on the fly or folds it into an epilogue
// through identities (1)-(3).
#pragma once
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
    long long cd_prof[4];              // Gram CD phase cycles (thread 0): cp wait, barrier, sweep setup, active builds
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
            for (int i = lane * V; i < n; i += 32 * V) {
                int4 raw = __ldg(reinterpret_cast<const int4 *>(col + i));
                const int8_t *xb = reinterpret_cast<const int8_t *>(&raw);
#pragma unroll
                for (int e = 0; e < V; e++) {
                    bool use = (i + e < n) && (!MASK || mask[i + e]);
                    int x = use ? (int)xb[e] : 0;
                    s1 += x;
                    s2 += x * x;
                }
            }
            s1 = warp_sum_ll(s1);
            s2 = warp_sum_ll(s2);
            if (lane == 0) {
                long long ntl = (long long)nt;
                long long num = ntl * s2 - s1 * s1;      // n^2 var, exact
                c[j] = (double)s1 / nt;
                s[j] = num <= 0 ? 0.0 : sqrt((double)num) / nt;
            }
        } else {
            double K = to_d(col[i0]);
            double s1 = 0.0, s2 = 0.0;
            for (int i = lane * V; i < n; i += 32 * V) {
                T xv[V];
                *reinterpret_cast<int4 *>(xv) = __ldg(reinterpret_cast<const int4 *>(col + i));
#pragma unroll
                for (int e = 0; e < V; e++) {
                    bool use = (i + e < n) && (!MASK || mask[i + e]);
                    double d = use ? to_d(xv[e]) - K : 0.0;
                    s1 += d;
                    s2 = fma(d, d, s2);
                }
            }
            s1 = warp_sum(s1);
            s2 = warp_sum(s2);
            if (lane == 0) {
                double var = (s2 - s1 * s1 / nt) / nt;
                c[j] = K + s1 / nt;
                s[j] = (var > 0.0 && s2 != 0.0) ? sqrt(var) : 0.0;
            }
        }
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
    const int *list;          // nullptr => dense 0..p-1
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
    const int64_t m = a.list ? (a.nlist ? (int64_t)*a.nlist : (int64_t)a.nlist_host) : a.p;
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
            col[q] = a.list ? (int64_t)a.list[idx] : idx;
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
    const int64_t m = a.list ? (a.nlist ? (int64_t)*a.nlist : (int64_t)a.nlist_host) : a.p;
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
        int64_t ja = a.list ? (int64_t)a.list[ia] : ia;
        int64_t jb = a.list ? (int64_t)a.list[ib] : ib;
        const int8_t *pa = X + ja * a.ld, *pb = X + jb * a.ld;
        int acc[4] = {0, 0, 0, 0};
        const int8_t *lg = ls + g * LL + 16 * t;
        int r = 0;
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

__global__ void k_argmax2(const double *__restrict__ bv, const long long *__restrict__ bi, int nb,
                          const double *__restrict__ a, const double *__restrict__ c, const double *__restrict__ s,
                          double alpha, const int *__restrict__ nlive, PrepScalars *ps) {
    if (threadIdx.x != 0) return;
    double best = -1.0;
    long long bj = -1;
    for (int b = 0; b < nb; b++)
        if (bv[b] > best || (bv[b] == best && bi[b] >= 0 && (bj < 0 || bi[b] < bj))) { best = bv[b]; bj = bi[b]; }
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

__global__ void k_bedpp(int64_t p, const double *__restrict__ s, const double *__restrict__ a,
                        const double *__restrict__ b, const PrepScalars *__restrict__ ps, double alpha,
                        double lam, double lam_next, int use_bedpp, uint8_t *__restrict__ flags,
                        int *__restrict__ scope, RoundStatus *st) {
    const double A = ps->A, Y2 = ps->Y2, nd = ps->nt, sg = ps->sigma;
    const long long js = ps->jstar;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t pr = (p + 31) / 32 * 32;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < pr; j += stride) {
        uint8_t f = 0;
        if (j < p && s[j] > 0.0) {
            bool star = j == js;
            bool sk = !use_bedpp || !bedpp_discard(a[j], b[j], star, A, Y2, nd, sg, alpha, lam);
            bool sn = lam_next > 0.0 && (!use_bedpp || !bedpp_discard(a[j], b[j], star, A, Y2, nd, sg, alpha, lam_next));
            f = (uint8_t)((sk ? 1 : 0) | (sn ? 2 : 0));
            flags[j] = f;
        } else if (j < p) {
            flags[j] = 0;
        }
        if (scope) warp_append(f != 0, (int)j, scope, &st->nscope);
        unsigned m = __ballot_sync(0xffffffffu, (f & 1) != 0);
        if ((threadIdx.x & 31) == 0 && m) atomicAdd(&st->nsafe, __popc(m));
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

// ------------------------------- NEXT-2: covariance-update ("Gram") CD on W
// SURVEY 8(f) NEXT-2 (glmnet's covariance updates; the paper's CD "only iterates
// over features in the active set").  Same iterates as the residual CD
// above, but the per-coordinate work is O(|W|) on the gradient vector
//   g_w = x~_w' r / n        (w in W)
// instead of an O(n) reduction:  z = g_w + b_w;  b' = S(z, lambda alpha)/(1 +
// lambda(1-alpha));  g_k -= (b' - b_w) G_kw  for every k in W, with
// G = X~_W' X~_W / n kept in HBM/L2 (identity (1), generalised to W x W).
// g starts from the fused scan's z at the solve's residual; r is refreshed after
// the solve from the coefficient changes (k_resid_update), so no drift crosses
// lambdas.  Storage slots are append-only; `ord` gives the cyclic (ascending
// column) order.

// G rows (and columns) for the new slots [first, nW): G[s][t] = sum_i m_i
// x~_is x~_it / n, t in [0, nW).  grid = (nW - first, ceil(nW / 256)), 256 threads.
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
    const int t0 = blockIdx.y * 256, t1 = min(nW, t0 + 256);
    for (int tt = t0 + wid; tt < t1; tt += 8) {
        const int jt = Wst[tt];
        const T *xt = X + (int64_t)jt * ld;
        const double ct = c[jt];
        double acc0 = 0.0, acc1 = 0.0;
        int i = lane;
        for (; i + 32 < n; i += 64) {
            acc0 = fma(vs[i], to_d(xt[i]) - ct, acc0);
            acc1 = fma(vs[i + 32], to_d(xt[i + 32]) - ct, acc1);
        }
        if (i < n) acc0 = fma(vs[i], to_d(xt[i]) - ct, acc0);
        double d = warp_sum(acc0 + acc1);
        if (lane == 0) {
            double gv = d / s[jt] * inv_n;
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
    const double *z;         // z[j] = x~_j' r / n for the solve's starting residual
    double *beta;            // p entries (global, by local column)
    double *dbeta;           // nW entries out: beta_new - beta_old per slot
    double lam_alpha, inv_den, tol, floor_;
    int max_iter;
    double *betaW_out;       // 3*nW: beta, c, s per slot (cyclic order)
    const double *c, *s;
    RoundStatus *st;
};

// Blocked Gram CD: the same cyclic coordinate updates in the same order as the
// residual flavour (z = g_w + b_w, soft-threshold, g -= d G_w), with one CTA
// barrier pair per block of 32 coordinates instead of a barrier per coordinate.
// (A per-coordinate variant measured 1.4-2x slower: one barrier per coordinate
// plus a serialised G-row stream.)  The gradient g and the
// coefficients b of W live in shared memory:
//   B. warp 0 runs the block's 32 coordinate updates sequentially -- lane b holds
//      coordinate b's gradient and the G entries G[w_b'][w_b] linking it to the
//      block's earlier coordinates, so an update is a shuffle-broadcast, the
//      soft-threshold and one FMA per lane (no barrier);
//   C. every thread applies the block's nonzero updates, in order, to the
//      gradients it owns (pairs 2t + 2T m), streaming the 32 G rows from L2 in
//      one batch of independent 16-byte loads.
constexpr int kGram5Threads = 512;
template <int KP>
__global__ void __launch_bounds__(kGram5Threads, 1) k_cd_gram5(CdGramArgs a) {
    extern __shared__ __align__(16) double sm[];
    __shared__ int wcount[33];
    __shared__ double red[32];
    __shared__ int blk_w[2][32];
    __shared__ double dvec[2][32];
    __shared__ int nzc[2];
    __shared__ double convs[2];
    constexpr int T_ = kGram5Threads;
    const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = T_ >> 5;
    const int nW = a.nW;
    const int nWp = (nW + 1) & ~1;
    double *gS = sm;                                       // gradients of W (slot order)
    double *bS = gS + nWp;                                 // coefficients of W
    int *ord = reinterpret_cast<int *>(bS + nWp);
    int *act = ord + nWp;
    for (int w = t; w < nWp; w += T_) {
        if (w < nW) {
            int j = a.Wst[w];
            gS[w] = a.z[j];
            bS[w] = a.beta[j];
            ord[w] = a.ord[w];
        } else {
            gS[w] = 0.0;
            bS[w] = 0.0;
        }
    }
    __syncthreads();
    const long long clk0 = clock64();
    int passes = 0, status = 0;
    long long visits = 0, updates = 0;
    long long pr_b = 0, pr_c = 0;

    auto sweep = [&](const int *list, int len, double &dmax, double &bmax) {
        double dm = 0.0, bm = 0.0;                         // warp 0's running maxima
        visits += len;
        int par = 0;
        for (int q0 = 0; q0 < len; q0 += 32, par ^= 1) {
            const int nb = min(32, len - q0);
            // B: warp 0, sequential coordinate updates inside the block
            if (wid == 0) {
                long long cb = clock64();
                const bool mine = lane < nb;
                const int wl = list[q0 + min(lane, nb - 1)];       // clamped: every address valid
                // lanes past the block end carry g = b = 0: their "update" is exactly 0 (no-op)
                double gv = mine ? gS[wl] : 0.0, bv = mine ? bS[wl] : 0.0;
                double Gs[32];                                // Gs[b'] = G[w_b'][w_lane]
#pragma unroll
                for (int bp = 0; bp < 32; bp++) {             // unconditional loads: no branch per load
                    const int wb = __shfl_sync(0xffffffffu, wl, bp);
                    Gs[bp] = __ldg(a.G + (int64_t)wb * a.ldG + wl);
                }
                double dl = 0.0;                              // this lane's coordinate's update
#pragma unroll
                for (int bp = 0; bp < 32; bp++) {             // branch-free: fma(-0, x, g) == g
                    const double zb = __shfl_sync(0xffffffffu, gv + bv, bp);
                    const double bo = __shfl_sync(0xffffffffu, bv, bp);
                    const double bn = soft_threshold(zb, a.lam_alpha) * a.inv_den;
                    const double d = bn - bo;
                    gv = fma(-d, lane > bp ? Gs[bp] : 0.0, gv);
                    bv = lane == bp ? bn : bv;
                    dl = lane == bp ? d : dl;
                    dm = fmax(dm, fabs(d));
                    bm = fmax(bm, fabs(bn));
                }
                // compact the nonzero updates (order preserved) for phase C
                const bool nz = mine && dl != 0.0;
                const unsigned msk = __ballot_sync(0xffffffffu, nz);
                if (nz) {
                    const int pos = __popc(msk & ((1u << lane) - 1u));
                    blk_w[par][pos] = wl;
                    dvec[par][pos] = dl;
                }
                if (lane == 0) nzc[par] = __popc(msk);
                if (mine) bS[wl] = bv;
                updates += __popc(msk);
                pr_b += clock64() - cb;
            }
            __syncthreads();
            long long cc = clock64();
            // C: every thread applies the block's nonzero updates, in order, to its gradients
            const int nzb = nzc[par];
            if (nzb > 0) {
#pragma unroll
                for (int m = 0; m < KP; m++) {
                    const int k = 2 * t + 2 * T_ * m;
                    if (k < nW) {
                        double2 gm = *reinterpret_cast<const double2 *>(gS + k);
                        for (int i0 = 0; i0 < nzb; i0 += 16) {
                            double2 rv[16];
                            double dd[16];
#pragma unroll
                            for (int u = 0; u < 16; u++) {    // unconditional (clamped) loads
                                const int i = min(i0 + u, nzb - 1);
                                dd[u] = i0 + u < nzb ? dvec[par][i] : 0.0;
                                rv[u] = __ldg(reinterpret_cast<const double2 *>(a.G + (int64_t)blk_w[par][i] * a.ldG + k));
                            }
#pragma unroll
                            for (int u = 0; u < 16; u++) {
                                gm.x = fma(-dd[u], rv[u].x, gm.x);
                                gm.y = fma(-dd[u], rv[u].y, gm.y);
                            }
                        }
                        *reinterpret_cast<double2 *>(gS + k) = gm;
                    }
                }
            }
            pr_c += clock64() - cc;
            __syncthreads();
        }
        if (t == 0) { convs[0] = dm; convs[1] = bm; }
        __syncthreads();
        dmax = convs[0];
        bmax = convs[1];
        __syncthreads();
    };

    auto build_active = [&]() -> int {
        int total = 0;
        for (int base = 0; base < nW; base += T_) {
            int q = base + t;
            int w = q < nW ? ord[q] : 0;
            bool nz = q < nW && bS[w] != 0.0;
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
        for (;;) {
            int na = build_active();
            if (na == 0) break;
            double dmax, bmax;
            sweep(act, na, dmax, bmax);
            if (++passes > a.max_iter) { status = 3; break; }
            if (dmax <= a.tol * bmax || dmax <= a.floor_) break;
        }
        if (status) break;
        double dmax, bmax;
        sweep(ord, nW, dmax, bmax);
        if (++passes > a.max_iter) { status = 3; break; }
        if (dmax <= a.tol * bmax || dmax <= a.floor_) break;
    }
    __syncthreads();
    double l1 = 0.0, l2 = 0.0, nnz = 0.0;
    for (int q = t; q < nW; q += T_) {
        int w = ord[q];
        double bv = bS[w];
        int j = a.Wst[w];
        double b0 = a.beta[j];
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
        a.st->cd_prof[0] = 0;
        a.st->cd_prof[1] = pr_b;
        a.st->cd_prof[2] = pr_c;
        a.st->cd_prof[3] = 0;
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
// rows.  Rows are split over blocks (deterministic order over slots); per-block
// partial sums of r_scan and r_scan^2 go to `part` (finished by k_resid_finish).
template <typename T, bool MASK>
__global__ void __launch_bounds__(256) k_resid_update(const T *__restrict__ X, int64_t ld, int n,
                                                      const int *__restrict__ Wst, int nW,
                                                      const double *__restrict__ dbeta,
                                                      const double *__restrict__ c, const double *__restrict__ s,
                                                      const uint8_t *__restrict__ mask, double *__restrict__ r,
                                                      double *__restrict__ r_scan, double *__restrict__ part) {
    __shared__ double red[32];
    __shared__ int sj[256];
    __shared__ double sf[256], sc[256];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    double acc = 0.0;
    for (int base = 0; base < nW; base += 256) {
        int w = base + threadIdx.x;
        __syncthreads();
        if (w < nW) {
            double d = dbeta[w];
            int j = Wst[w];
            sj[threadIdx.x] = j;
            sf[threadIdx.x] = d / s[j];
            sc[threadIdx.x] = c[j];
        }
        __syncthreads();
        int cnt = min(256, nW - base);
        if (i < n) {
            for (int u = 0; u < cnt; u++) {
                double f = sf[u];
                if (f != 0.0) acc = fma(f, to_d(X[(int64_t)sj[u] * ld + i]) - sc[u], acc);
            }
        }
    }
    double rs = 0.0, rr = 0.0;
    if (i < n) {
        double v = r[i] - acc;
        r[i] = v;
        bool use = !MASK || mask[i];
        double vs = use ? v : 0.0;
        r_scan[i] = vs;
        rs = vs;
        rr = vs * vs;
    } else if (i < ld) {
        r_scan[i] = 0.0;
    }
    rs = block_sum(rs, red);
    rr = block_sum(rr, red);
    if (threadIdx.x == 0) { part[2 * blockIdx.x] = rs; part[2 * blockIdx.x + 1] = rr; }
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
