/*
 * bl.h -- C ABI of libbl.so, the B200-native (sm_100a) lasso / elastic-net path
 * of the biglasso paper (arXiv 1701.05936), hot path = pathwise coordinate
 * descent driven by the hybrid SSR-BEDPP screening rule (section 2.2,
 * P:205-244) over a design held in HBM with cell-wise standardisation
 * (P:248-267).
 *
 * Citations: "P:n" = PAPER.md line n, "S:n" = SPEC.md line n, "Qk" = reading k
 * in DESIGN.md section 3.
 *
 * Conventions shared by every entry point
 *  - Every call returns bl_status; BL_OK == 0.  On failure a human-readable
 *    message is available from bl_last_error() (thread-local, valid until the
 *    next failing call on the same thread).  CUDA / NCCL failures are reported
 *    verbatim.  Nothing ever falls back to a CPU implementation: without a
 *    usable sm_100a device every compute call returns BL_ERR_CUDA.
 *  - X is column-major with leading dimension ld (elements): x_ij lives at
 *    X[j*ld + i].  Rows n..ld-1 are padding and never influence a result.
 *  - Objective (Q2):  Q(b) = 1/(2 n) ||y~ - X~ b||^2 + lambda [alpha ||b||_1 +
 *    (1-alpha)/2 ||b||^2],  x~_ij = (x_ij - c_j)/s_j with population SD (Q1),
 *    y~ = y - ybar, unpenalised intercept (Q4).  Coefficients are reported on
 *    the standardised scale (beta_std) and the original scale
 *    (beta_orig = beta_std / s_j, a0 = ybar - sum_j beta_orig_j c_j).
 *  - Zero-variance columns (s_j == 0 exactly) are accepted; their coefficient
 *    is locked to 0 and they are excluded from lambda_max, BEDPP and scans (Q13).
 *  - Host pointers are only read during the call (copied); results are owned by
 *    the library until bl_free.  A design is immutable after load; concurrent
 *    fits on one single-GPU design from different host threads are allowed (S:90,
 *    S:341).  A multi-rank design (world > 1) accepts one call at a time: its
 *    collectives must be issued in the same order on every rank, so a second
 *    concurrent call on the same design returns BL_ERR_ARG.
 */
#ifndef BL_H
#define BL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BL_OK = 0,
    BL_ERR_ARG = 1,          /* invalid argument */
    BL_ERR_DEGENERATE = 2,   /* y~ == 0, or every column zero-variance */
    BL_ERR_CONVERGENCE = 3,  /* max_iter passes or > 10 KKT rounds at some lambda;
                                the path is returned truncated to its converged prefix */
    BL_ERR_CUDA = 4,         /* CUDA error / no sm_100a device (message verbatim) */
    BL_ERR_NCCL = 5,         /* NCCL error (message verbatim) */
    BL_ERR_OOM = 6           /* device allocation failed or a working set exceeds on-chip capacity */
} bl_status;

typedef enum { BL_F64 = 0, BL_F32 = 1, BL_I8 = 2 } bl_dtype;   /* I8: any int8, e.g. genotype codes 0/1/2 */

typedef enum { BL_SCREEN_NONE = 0, BL_SCREEN_SSR = 1, BL_SCREEN_HYBRID = 2 } bl_screen;

typedef struct bl_design bl_design;
typedef struct bl_path bl_path;
typedef struct bl_cvres bl_cvres;
typedef struct bl_prep bl_prep;

/* Multi-GPU (BASELINE north star: "Features are column-sharded for
 * the scans, and NCCL all-gathers only the small strong-set and violator index
 * lists").  NULL => single GPU.  Rank g owns the contiguous global columns
 * [col_offset, col_offset + p_local); shards are in rank order and cover
 * [0, p_global).  Every rank calls every function collectively with identical
 * scalar arguments and identical y, lambda.
 *  - p_global > p_local: SHARDED design.  Scans, BEDPP and the strong rule run on
 *    each shard; lambda_max / x_* are combined across ranks; strong / violator
 *    lists are all-gathered (global indices, sorted); the columns that enter the
 *    working set are broadcast by their owner into every rank's working-set
 *    column store, and the coordinate descent runs replicated (identical,
 *    deterministic) on every rank, so the residual needs no broadcast.  Results
 *    are identical to the single-GPU path (global indices).
 *  - p_global == p_local: REPLICATED design (every rank holds all of X); bl_cv
 *    distributes the folds over the ranks.
 * backend 0: NCCL; nccl_unique_id points to the 128-byte ncclUniqueId obtained on
 * rank 0 with bl_nccl_unique_id() and broadcast by the caller (torch.distributed).
 * Collectives are enqueued on the fit's stream (NCCL groups batch a round's
 * broadcasts); the host waits only where it decides on a result, polling
 * ncclCommGetAsyncError, and aborts the communicator when a collective is still
 * pending after timeout_ms (BL_ERR_NCCL; the design cannot run collectives after).
 * backend 1: in-process loopback for testing -- the ranks are threads of ONE
 * process sharing one device; nccl_unique_id points to a 128-byte group key
 * (any bytes, identical on the group's ranks); collectives are staged through
 * host memory.
 * backend 2: caller-supplied HOST collectives (host_coll, e.g. gloo or MPI between
 * processes): every payload is staged through host memory around the caller's
 * functions, which every rank calls with identical sizes in the same order and
 * which return 0 on success (anything else: BL_ERR_NCCL).  nccl_unique_id unused. */
typedef struct {
    void *ctx;                                                                  /* passed back verbatim */
    int (*allgather)(void *ctx, const void *send, void *recv, int64_t bytes);   /* recv: world x bytes, rank order */
    int (*bcast)(void *ctx, void *buf, int64_t bytes, int root);
    int (*allreduce_sum_f64)(void *ctx, double *buf, int64_t count);
} bl_host_coll;

typedef struct {
    int rank, world, device;
    const void *nccl_unique_id;
    int64_t col_offset, p_global;
    int backend;                       /* 0 NCCL, 1 in-process loopback, 2 host collectives */
    const bl_host_coll *host_coll;     /* backend 2 (copied at load); NULL otherwise */
    int timeout_ms;                    /* NCCL collective timeout; <= 0 => 600000 */
} bl_dist;

/* Optional execution options (NULL or all-zero => defaults).  None of them changes a
 * result beyond floating-point association order, except the TEST-ONLY fault switch. */
typedef struct {
    void *stream;        /* cudaStream_t to run on; NULL => library-owned stream */
    int profile;         /* 1 => time every scan / CD launch with CUDA events (bl_path_perf) */
    int max_kkt_rounds;  /* cap on the KKT rounds R_k (solve + scan) at one lambda; <= 0 => 10.
                            A lambda that still has violators after R_k = cap rounds ends the path with
                            BL_ERR_CONVERGENCE (the converged prefix is returned) */
    int cd_mode;         /* 0 auto (Gram/covariance updates while |W| <= 4096),
                            1 residual-update CD (r held on chip), 2 Gram only */
    int cv_mode;         /* bl_cv on a single-GPU or sharded design: 0 (default) the K+1 fits advance
                            lambda in lockstep and each KKT round's scans of all fits are one pass over X
                            (SURVEY NEXT-1): fp32 designs on the tcgen05 integer tensor cores (exact digit
                            products), fp64 designs on the fp64 tensor cores, int8
                            designs on the integer mma.sync path; 1 the same with the fp64-FMA batched
                            kernel; 2 independent concurrent fits (one pass over X per fit and round);
                            3 as 0 but fp32 designs on the fp64 tensor cores (DMMA) */
    int cd_cluster;      /* CTAs per Gram-CD cluster (SMs one CD solve uses): 0 => 16 for a single fit,
                            8 for each of bl_cv's concurrent fits; or 4, 8, 16 */
    int64_t stream_chunk_bytes; /* out-of-core designs (x_is_device_ptr = 2): bytes of X per streamed
                            chunk (two chunks are resident); 0 => 256 MB */
    int fault_strong_drop; /* TEST ONLY (S:222 fault injection): 1 => the strong rule admits no
                            candidate to the working set in advance, so every feature that enters the
                            model must be found by the KKT check (re-solve, re-check); 0 => off */
    int cd_accel;        /* Gram CD on the linear path: 0 (default) => when an active set has settled
                            (same set and signs for two sweeps) but sweeps contract slowly, one Newton
                            step on it (conjugate gradients on (G_AA + lambda(1-alpha) I)), truncated to
                            keep every sign; the sweeps that follow decide convergence as before.
                            1 => sweeps only */
} bl_opts;

/* Per-fit performance counters (filled when opts->profile == 1). */
typedef struct {
    double scan_ms;            /* summed CUDA-event time of the fused scan kernel launches */
    double scan_bytes;         /* algorithmic X bytes those launches read: n * itemsize * columns */
    int64_t scan_launches;
    double cd_ms;              /* summed time of the coordinate-descent kernel launches */
    int64_t cd_launches;
    double prep_ms;            /* column stats + x~'y + x~'x* (one-time passes) */
    double prep_bytes;
    int64_t kernel_launches;   /* every kernel this fit launched */
    double wall_ms;            /* host steady clock, entry to return */
    int64_t cd_visits;         /* coordinate visits over the path (all passes) */
    int64_t cd_updates;        /* visits that changed a coefficient */
    int64_t cd_kernel_cycles;  /* SM cycles spent inside the CD kernels (clock64, thread 0) */
    int64_t cd_prof[4];        /* Gram CD phases (cycles): leader steps, bulk steps, G_AA / M builds, lazy catch-ups */
    double full_scan_ms;       /* the subset of scan launches that covered every live column (|S_k| = p, */
    double full_scan_bytes;    /*   SURVEY 8(d) "full-scan only" GB/s); single fits only (0 in CV sums) */
    int64_t full_scan_launches;
    int64_t cd_events[8];      /* Gram CD events: speculation retries, G_AA builds, catch-ups, full sweeps,
                                  Newton steps, CG iterations, SM cycles in Newton steps, sign-limited steps */
    int64_t cd_sub[8];         /* Gram CD leader-warp sub-phase cycles: block prologue, active mat-vec,
                                  forward substitution, publish, waits (stage + snapshot), next-stage wait,
                                  link product, (unused) */
} bl_perf;

/* ---- design ------------------------------------------------------------------
 * X: n x p_local column-major, dtype dt, leading dimension ld >= n.
 * x_is_device_ptr = 0: X is host memory, copied into a library-owned device
 *   buffer with a 16-byte aligned column stride (padding zero-filled).
 * x_is_device_ptr = 1: X is a device pointer on the current device, BORROWED
 *   (caller keeps it alive until bl_free(design)); requires 16-byte aligned
 *   base and ld * itemsize % 16 == 0.
 * x_is_device_ptr = 2: OUT-OF-CORE (the paper's memory-mapped
 *   design): X is host memory, BORROWED and read in place -- the
 *   library page-locks and maps it (cudaHostRegister, undone by bl_free; a range
 *   the caller already pinned is only mapped), every full pass over X streams it
 *   over the host link, and working-set columns are copied once into a device
 *   store.  Same alignment rules as 1; padding rows are never read into results.
 *   Results are bitwise identical to a device-resident design.
 * Errors: BL_ERR_ARG for n < 2, n > 16384 (r must fit one SM's shared
 * memory), p_local < 1, ld < n, bad dtype/alignment. */
bl_status bl_load_design(const void *X, bl_dtype dt, int64_t n, int64_t p_local, int64_t ld,
                         int x_is_device_ptr, const bl_dist *dist, bl_design **out);

/* 128-byte ncclUniqueId for bl_dist (call on rank 0 only). */
bl_status bl_nccl_unique_id(void *out128);

/* lambda_max = max_j |x~_j' y~| / (n alpha)  (Q3).  y: n host doubles. */
bl_status bl_lambda_max(bl_design *d, const double *y, double alpha, double *out);

/* ---- the path -------------------------------------------
 * y: n host doubles.  lambda: n_lambda host doubles, strictly decreasing, > 0
 * (S:192); the first value may equal lambda_max (grids usually start there; if
 * lambda_1 < lambda_max the strong rule uses a virtual lambda_0 = lambda_max).
 * alpha in (0, 1].  tol > 0: a CD solve converges when a pass over the
 * working set changes no coefficient by more than tol * max_j |beta_j| (Q6).
 * max_iter >= 1: passes per lambda (Q7).  screen: bl_screen; NONE = plain CD
 * over every column, SSR = strong rule + full-scope KKT scans, HYBRID = SSR-BEDPP
 * (default).  On BL_ERR_CONVERGENCE *out still receives the
 * converged prefix. */
bl_status bl_fit_path(bl_design *d, const double *y, const double *lambda, int n_lambda,
                      double alpha, double tol, int max_iter, int screen,
                      const bl_opts *opts, bl_path **out);

/* ---- K-fold cross-validation -------------
 * fold_id: n host int32 in [0, K), or NULL => seeded permutation (Q18: splitmix64
 * Fisher-Yates, fold_id[perm[i]] = i mod K).  Each fold's column stats are
 * recomputed on its training rows (Q16) without copying X: held-out rows are
 * masked.  The grid is shared.  Also fits the full data.
 * Errors: K < 2, K > n, an empty fold. */
/* ---- NEXT-3: lasso / elastic-net penalised LOGISTIC regression path -------------
 * SURVEY 8(f) NEXT-3; P:174 ("sparse linear and logistic regression models with
 * lasso and elastic net penalties").  Minimises, per lambda_k,
 *   Q(b0, b) = (1/n) sum_i [log(1 + e^eta_i) - y_i eta_i] + lambda [alpha |b|_1 + (1-alpha)/2 |b|^2],
 *   eta_i = b0 + x~_i' b   (QL1; b0 unpenalised)
 * by IRLS with weighted coordinate descent on W (QL4-QL6).  lambda_max is
 * bl_lambda_max's value (QL2: the same closed form).  Screening: the sequential
 * strong rule with z_j = x~_j'(y - p^)/n and the KKT check over all live columns;
 * BL_SCREEN_HYBRID runs as BL_SCREEN_SSR (QL3: BEDPP is a linear-model rule and the
 * paper's Slores formulas are not printed).
 * y: n host doubles, each 0 or 1 (BL_ERR_ARG otherwise); a single class is
 * BL_ERR_DEGENERATE.  The result is a bl_path: a0[k] is the intercept on the
 * original scale (b0 - sum_j b_j c_j / s_j), objective[k] = Q at the solution.
 * Other arguments, errors and ownership as bl_fit_path.  Not available under CV. */
bl_status bl_fit_path_binomial(bl_design *d, const double *y, const double *lambda, int n_lambda, double alpha,
                               double tol, int max_iter, int screen, const bl_opts *opts, bl_path **out);
/* IRLS (outer) iterations of the last solve at each lambda (n_lambda entries; 0 for
 * null-model lambdas).  BL_ERR_ARG for a linear-model path. */
bl_status bl_path_irls(const bl_path *path, int32_t *outer);

bl_status bl_cv(bl_design *d, const double *y, const double *lambda, int n_lambda, double alpha,
                double tol, int max_iter, int n_folds, const int32_t *fold_id, uint64_t seed,
                const bl_opts *opts, bl_cvres **out);

/* ---- read-out (caller-owned buffers; query sizes first) ---------------------- */
bl_status bl_path_info(const bl_path *path, int *n_lambda, int64_t *nnz_total, int *n_converged);
/* Any output pointer may be NULL.  Sizes: lambda, a0, objective, passes,
 * kkt_rounds, cols_scanned: n_lambda; col_ptr: n_lambda + 1; feat_idx (GLOBAL
 * column index), beta_std, beta_orig: nnz_total.  Only the first n_converged
 * lambdas are filled. */
bl_status bl_path_copy(const bl_path *path, double *lambda, double *a0, double *objective,
                       int64_t *col_ptr, int64_t *feat_idx, double *beta_std, double *beta_orig,
                       int32_t *passes, int32_t *kkt_rounds, int64_t *cols_scanned);
bl_status bl_path_perf(const bl_path *path, bl_perf *out);
/* Screening diagnostics per lambda (the analog of P:212-217's Fig 1; any pointer
 * may be NULL; n_lambda entries each, first n_converged filled):
 *   n_safe    |S_k|: columns the BEDPP safe rule keeps at lambda_k (P:211, 8(c));
 *             every live column under BL_SCREEN_SSR / BL_SCREEN_NONE;
 *   n_strong  strong-rule candidates entering lambda_k not already in W (a6);
 *   n_working |W| when lambda_k converged (strong sets, violators, ever-active). */
bl_status bl_path_screen(const bl_path *path, int64_t *n_safe, int64_t *n_strong, int64_t *n_working);

/* cve, cvse: n_lambda; fold_id_out: n; full_fit: borrowed, freed with the cv result.
 * cve_k = mean_i e_ik, cvse_k = sd_i(e_ik)/sqrt(n) over per-row held-out squared
 * errors (Q17); lambda_min_index = argmin cve (lowest index on ties). */
bl_status bl_cv_copy(const bl_cvres *cv, double *cve, double *cvse, int *lambda_min_index,
                     int32_t *fold_id_out, const bl_path **full_fit);
bl_status bl_cv_errors(const bl_cvres *cv, double *E /* n_lambda x n, row-major */);
/* Performance counters summed over every fit of the CV (K folds + the full-data
 * fit; wall_ms = the slowest fit), filled when opts->profile == 1. */
bl_status bl_cv_perf(const bl_cvres *cv, bl_perf *out);

/* ---- single steps of the path, for parity tests and diagnostics ---------------
 * bl_prepare: one-time preprocessing for (y, optional training mask) (SURVEY 8(a)
 * a2-a4): c, s, a_j = x~_j'y~ (identity (2)), lambda_max and j*
 * (P:265), b_j = x~_j'x~_* (identity (1)).  train: n host bytes (1 = row
 * used) or NULL. */
bl_status bl_prepare(bl_design *d, const double *y, const uint8_t *train, double alpha,
                     bl_prep **out);
/* Copy the preprocessing vectors (length p_local each; any may be NULL). */
bl_status bl_prep_copy(const bl_prep *pp, double *c, double *s, double *a, double *b,
                       int64_t *jstar_global, double *lambda_max);
/* BEDPP safe set at lambda: keep[j] = 1 iff
 * column j is NOT discarded (j* always kept).  keep: p_local host bytes. */
bl_status bl_bedpp(bl_prep *pp, double lambda, uint8_t *keep, int64_t *n_keep);
/* Fused scan (identity (3)) on a caller-given
 * residual r (n host doubles; rows outside the training mask must be 0):
 *   z_j = (sum_i x_ij r_i - c_j sum_i r_i) / (n s_j)   for every non-constant j,
 * plus the two tests the path uses: viol = {j : !in_w[j], |z_j| > alpha lam}
 * and strong = {j : !in_w[j], |z_j| >= alpha (2 lam_next - lam)}.
 * z: p_local doubles (0 for zero-variance columns); in_w: p_local bytes or NULL;
 * viol/strong: p_local int32 (LOCAL column indices, ascending) or NULL. */
bl_status bl_scan(bl_prep *pp, const double *r, double lam, double lam_next, const uint8_t *in_w,
                  double *z, int32_t *viol, int64_t *n_viol, int32_t *strong, int64_t *n_strong);

/* Fold-batched scan (SURVEY 8(a) a9 + a12, NEXT-1; one pass over X for several
 * fits): the fused scan of bl_scan for nf fits of ONE design at once, by the kernel bl_cv's
 * lockstep rounds use for that design (cv_mode as in bl_opts: 0 the default -- fp32 designs on
 * the tcgen05 integer tensor cores, fp64 on the fp64 tensor cores, int8 on the integer mma.sync
 * path; 1 the fp64-FMA kernel; 3 fp32 designs on the fp64 tensor cores).  pps: nf distinct
 * preps (bl_prepare, any row masks); r[u]: fit u's residual (n host doubles, 0 on rows outside
 * its mask).  z: nf x p_local doubles, fit-major (NULL: not copied); n_viol / n_strong: nf
 * counts of the two tests at (lam, lam_next) with no working set (NULL: not copied).  Errors:
 * BL_ERR_ARG for bad handles, repeated preps, preps of different designs or another cv_mode. */
bl_status bl_scan_batch(bl_prep *const *pps, int nf, const double *const *r, double lam, double lam_next,
                        int cv_mode, double *z, int64_t *n_viol, int64_t *n_strong);

/* NULL-safe, idempotent per live handle: frees a design, path, cv result or prep. */
void bl_free(void *handle);
const char *bl_last_error(void);
/* Return the library's cached allocations to the CUDA driver.  Freed design / workspace buffers
 * are kept for reuse (at most 8 GB of device and 2 GB of pinned host memory per process; an
 * allocation that fails flushes them and retries), so another allocator in the process -- e.g.
 * PyTorch's -- may want them back first.  Safe at any time no library call is running. */
void bl_trim(void);

#ifdef __cplusplus
}
#endif
#endif /* BL_H */
