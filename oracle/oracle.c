/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the biglasso
 * lasso / elastic-net path (arXiv 1701.05936).
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (libbl.so, the Python
 * binding) may link, import or execute this file.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs use it.  It shares no code, header, table or helper with csrc/.
 *
 * Citation convention: "P:n" = /root/reference/PAPER.md line n (section given);
 * "S:n" = SPEC.md line n; "Qk" = reading k listed in DESIGN.md section 3
 * (taken from SURVEY.md section 8(c.3)).
 *
 * What it computes: the plain definition.  For each lambda_k of
 * a caller-supplied decreasing grid, the minimiser of
 *     Q(b) = 1/(2 n) || y~ - X~ b ||^2 + lambda [ alpha ||b||_1 + (1-alpha)/2 ||b||^2 ]
 * over the explicitly standardised columns x~_ij = (x_ij - c_j)/s_j (P:252,
 * "cell-wise standardization"; population SD, Q1), by naive cyclic coordinate
 * descent with warm starts and NO screening at all.  The identities
 * (1)-(3) of P:259-265 are deliberately NOT used here: every standardised
 * value is formed element by element, so the GPU path's identity-based
 * arithmetic is checked against an independent computation.
 *
 * Rows: an optional training mask (1 = row used) implements the paper's
 * "operate on a subset of X given a row-index vector"; n_t is the
 * number of rows in the subset.
 *
 * Everything is fp64 (Q22: the paper's sizes imply 8-byte storage, P:299,
 * P:620).  X may be stored as fp64, fp32 or int8 and is widened on read.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* Host threads.  1 = the pure serial oracle.  With T > 1
 * only loops whose iterations are independent per column run in parallel (each
 * column's dot product is still one thread's plain ascending-i loop), and the
 * coordinate-descent full pass is block-speculative: the dot products of a block
 * of columns are computed in parallel against the current residual and committed
 * in index order; the first committed change ends the block (the rest are
 * recomputed against the updated residual).  Every value is therefore computed
 * by exactly the same arithmetic as the serial pass: the iterates are bitwise
 * identical for every T (pinned by tests/test_oracle_pins.py). */
static int g_threads = 1;
void or_set_threads(int t) { g_threads = t < 1 ? 1 : t; }
int or_get_threads(void) { return g_threads; }
#define OR_PAR _Pragma("omp parallel for schedule(static) if(g_threads > 1) num_threads(g_threads)")

enum { OR_OK = 0, OR_ERR_ARG = 1, OR_ERR_DEGENERATE = 2, OR_ERR_CONVERGENCE = 3 };
enum { OR_F64 = 0, OR_F32 = 1, OR_I8 = 2 };

/* x_ij as stored, widened to double (column-major, leading dimension ld). */
static double xraw(const void *X, int dt, int64_t ld, int64_t i, int64_t j)
{
    int64_t o = j * ld + i;
    if (dt == OR_F64) return ((const double *)X)[o];
    if (dt == OR_F32) return (double)((const float *)X)[o];
    return (double)((const int8_t *)X)[o];
}

static int in_rows(const uint8_t *train, int64_t i) { return train == NULL || train[i] != 0; }

static int64_t count_rows(const uint8_t *train, int64_t n)
{
    int64_t m = 0;
    for (int64_t i = 0; i < n; i++) m += in_rows(train, i);
    return m;
}

/* "saves only the means and standard deviations of the columns of X as
 * two vectors c and s".  Two-pass, population SD (Q1).  s_j == 0 marks a
 * zero-variance column, excluded everywhere (Q13): a column whose used values
 * are all equal has variance exactly 0 by definition, so it gets c_j = that
 * value and s_j = 0 exactly (two-pass arithmetic alone would leave a rounding
 * residue ~1e-16 |c_j| there). */
int or_column_stats(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                    const uint8_t *train, double *c, double *s)
{
    if (!X || n < 2 || p < 1 || ld < n || dt < 0 || dt > 2) return OR_ERR_ARG;
    int64_t nt = count_rows(train, n);
    if (nt < 2) return OR_ERR_ARG;
    OR_PAR
    for (int64_t j = 0; j < p; j++) {
        double sum = 0.0;
        for (int64_t i = 0; i < n; i++)
            if (in_rows(train, i)) sum += xraw(X, dt, ld, i, j);
        double mean = sum / (double)nt;
        int constant = 1;
        double first = 0.0;
        int seen = 0;
        for (int64_t i = 0; i < n && constant; i++)
            if (in_rows(train, i)) {
                double v = xraw(X, dt, ld, i, j);
                if (!seen) { first = v; seen = 1; }
                else if (v != first) constant = 0;
            }
        if (constant) { c[j] = first; s[j] = 0.0; continue; }
        double ss = 0.0;
        for (int64_t i = 0; i < n; i++)
            if (in_rows(train, i)) {
                double d = xraw(X, dt, ld, i, j) - mean;
                ss += d * d;
            }
        c[j] = mean;
        s[j] = sqrt(ss / (double)nt);
    }
    return OR_OK;
}

/* x~_ij = (x_ij - c_j)/s_j, formed explicitly. */
static double xstd(const void *X, int dt, int64_t ld, int64_t i, int64_t j,
                   const double *c, const double *s)
{
    return (xraw(X, dt, ld, i, j) - c[j]) / s[j];
}

/* y~ = y - ybar over the row subset (Q4: unpenalised intercept); rows outside
 * the subset get 0.  Returns ybar. */
static double center_y(const double *y, int64_t n, const uint8_t *train, int64_t nt, double *yt)
{
    double sum = 0.0;
    for (int64_t i = 0; i < n; i++)
        if (in_rows(train, i)) sum += y[i];
    double ybar = sum / (double)nt;
    for (int64_t i = 0; i < n; i++) yt[i] = in_rows(train, i) ? y[i] - ybar : 0.0;
    return ybar;
}

/* sum_{i in rows} x~_ij v_i, element by element. */
static double std_dot(const void *X, int dt, int64_t n, int64_t ld, int64_t j,
                      const double *c, const double *s, const uint8_t *train, const double *v)
{
    double acc = 0.0;
    for (int64_t i = 0; i < n; i++)
        if (in_rows(train, i)) acc += xstd(X, dt, ld, i, j, c, s) * v[i];
    return acc;
}

/* lambda_max = max_j |x~_j^T y~| / (n alpha)  (Q3; for alpha = 1 this is the
 * closed form max_j |x_j^T y|/n of BASELINE.json).  j* = lowest index
 * attaining the max. */
int or_lambda_max(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                  const double *y, const uint8_t *train, double alpha,
                  double *lambda_max, int64_t *jstar)
{
    if (!(alpha > 0.0 && alpha <= 1.0)) return OR_ERR_ARG;
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    double *yt = malloc(sizeof(double) * n);
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (rc) goto done;
    int64_t nt = count_rows(train, n);
    center_y(y, n, train, nt, yt);
    double best = -1.0;
    int64_t jb = -1;
    double *av = malloc(sizeof(double) * p);
    OR_PAR
    for (int64_t j = 0; j < p; j++)
        av[j] = s[j] == 0.0 ? -1.0 : fabs(std_dot(X, dt, n, ld, j, c, s, train, yt));
    for (int64_t j = 0; j < p; j++)
        if (s[j] != 0.0 && av[j] > best) { best = av[j]; jb = j; }
    free(av);
    if (jb < 0 || best == 0.0) { rc = OR_ERR_DEGENERATE; goto done; }
    *lambda_max = best / ((double)nt * alpha);
    *jstar = jb;
done:
    free(c); free(s); free(yt);
    return rc;
}

/* z_j = x~_j^T v / n_t for every column j (0 for zero-variance columns), formed
 * element by element -- the quantity the fused scan computes through identity
 * (3) for v = r, and identity (2) for v = y~ (times n_t). */
int or_std_dots(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                const uint8_t *train, const double *v, double *z)
{
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (rc == OR_OK) {
        double nd = (double)count_rows(train, n);
        OR_PAR
        for (int64_t j = 0; j < p; j++)
            z[j] = s[j] == 0.0 ? 0.0 : std_dot(X, dt, n, ld, j, c, s, train, v) / nd;
    }
    free(c); free(s);
    return rc;
}

/* The one-time screening quantities of P:259-262, explicitly:
 * a_j = x~_j^T y~, j* = argmax |a_j| (lowest j), b_j = x~_j^T x~_*, lambda_max
 * = |a_j*| / (n alpha).  Zero-variance columns get a_j = b_j = 0. */
int or_prep(const void *X, int dt, int64_t n, int64_t p, int64_t ld, const double *y,
            const uint8_t *train, double alpha, double *a, double *b, int64_t *jstar,
            double *lambda_max)
{
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    double *yt = malloc(sizeof(double) * n), *xs = malloc(sizeof(double) * n);
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (rc) goto done;
    int64_t nt = count_rows(train, n);
    center_y(y, n, train, nt, yt);
    int64_t js = -1;
    double best = -1.0;
    OR_PAR
    for (int64_t j = 0; j < p; j++)
        a[j] = s[j] == 0.0 ? 0.0 : std_dot(X, dt, n, ld, j, c, s, train, yt);
    for (int64_t j = 0; j < p; j++)
        if (s[j] != 0.0 && fabs(a[j]) > best) { best = fabs(a[j]); js = j; }
    if (js < 0 || best == 0.0) { rc = OR_ERR_DEGENERATE; goto done; }
    for (int64_t i = 0; i < n; i++) xs[i] = in_rows(train, i) ? xstd(X, dt, ld, i, js, c, s) : 0.0;
    OR_PAR
    for (int64_t j = 0; j < p; j++)
        b[j] = s[j] == 0.0 ? 0.0 : std_dot(X, dt, n, ld, j, c, s, train, xs);
    *jstar = js;
    *lambda_max = best / ((double)nt * alpha);
done:
    free(c); free(s); free(yt); free(xs);
    return rc;
}

/* Soft-threshold S(z, g) = sign(z) max(|z| - g, 0). */
static double soft(double z, double g)
{
    if (z > g) return z - g;
    if (z < -g) return z + g;
    return 0.0;
}

/* Objective Q(beta) at lambda, with r recomputed from beta (never the running
 * residual): Q = ||y~ - X~ b||^2/(2 n_t) + lambda (alpha |b|_1 + (1-alpha)/2 |b|^2)
 * (Q2, the glmnet form; S:294 update). beta is dense, length p, standardised. */
int or_objective(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                 const double *y, const uint8_t *train, const double *beta,
                 double lambda, double alpha, double *Q)
{
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    double *r = malloc(sizeof(double) * n);
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (rc) goto done;
    int64_t nt = count_rows(train, n);
    center_y(y, n, train, nt, r);
    double l1 = 0.0, l2 = 0.0;
    for (int64_t j = 0; j < p; j++) {
        if (beta[j] == 0.0) continue;
        if (s[j] == 0.0) { rc = OR_ERR_ARG; goto done; }
        for (int64_t i = 0; i < n; i++)
            if (in_rows(train, i)) r[i] -= xstd(X, dt, ld, i, j, c, s) * beta[j];
        l1 += fabs(beta[j]);
        l2 += beta[j] * beta[j];
    }
    double rss = 0.0;
    for (int64_t i = 0; i < n; i++)
        if (in_rows(train, i)) rss += r[i] * r[i];
    *Q = rss / (2.0 * (double)nt) + lambda * (alpha * l1 + 0.5 * (1.0 - alpha) * l2);
done:
    free(c); free(s); free(r);
    return rc;
}

/* KKT audit (BASELINE.json "KKT conditions hold at every lambda"):
 * z_j = x~_j^T r / n_t with r = y~ - X~ beta recomputed explicitly.
 *   zero_viol    = max over beta_j == 0 of (|z_j| - alpha lambda)      (<= 0 ideally)
 *   nonzero_viol = max over beta_j != 0 of |z_j - alpha lambda sign(beta_j) - lambda (1-alpha) beta_j|
 * z (length p, may be NULL) receives z_j (0 for zero-variance columns). */
int or_kkt(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
           const double *y, const uint8_t *train, const double *beta,
           double lambda, double alpha, double *zero_viol, double *nonzero_viol, double *z)
{
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    double *r = malloc(sizeof(double) * n);
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (rc) goto done;
    int64_t nt = count_rows(train, n);
    center_y(y, n, train, nt, r);
    for (int64_t j = 0; j < p; j++) {
        if (beta[j] == 0.0 || s[j] == 0.0) continue;
        for (int64_t i = 0; i < n; i++)
            if (in_rows(train, i)) r[i] -= xstd(X, dt, ld, i, j, c, s) * beta[j];
    }
    double zv = -INFINITY, nv = 0.0;
    double *zz = malloc(sizeof(double) * p);
    OR_PAR
    for (int64_t j = 0; j < p; j++)
        zz[j] = s[j] == 0.0 ? 0.0 : std_dot(X, dt, n, ld, j, c, s, train, r) / (double)nt;
    for (int64_t j = 0; j < p; j++) {
        if (s[j] == 0.0) { if (z) z[j] = 0.0; continue; }
        double zj = zz[j];
        if (z) z[j] = zj;
        if (beta[j] == 0.0) {
            double v = fabs(zj) - alpha * lambda;
            if (v > zv) zv = v;
        } else {
            double sg = beta[j] > 0 ? 1.0 : -1.0;
            double v = fabs(zj - alpha * lambda * sg - lambda * (1.0 - alpha) * beta[j]);
            if (v > nv) nv = v;
        }
    }
    free(zz);
    *zero_viol = zv;
    *nonzero_viol = nv;
done:
    free(c); free(s); free(r);
    return rc;
}

/* BEDPP safe rule ("basic EDPP", P:219-224 hybrid; formula not printed in
 * the paper, P:207 defers to ZengRules -- reading Q8/Q9).
 * All inner products formed explicitly from x~:
 *   a_j = x~_j^T y~,  j* = argmax |a_j| (lowest j),  sigma* = sign(a_j*),
 *   b_j = x~_j^T x~_*,  Y2 = ||y~||^2,  A = |a_j*| / n  (= alpha lambda_max)
 * at lambda:  L = alpha lambda,  m = n (1 + lambda (1 - alpha)),
 *             b'_j = b_j + (m - n) [j == j*]
 * discard j (j != j*) iff
 *   |(A+L) a_j - (A-L)(n A/m) sigma* b'_j|  <  2 n L A - (A-L) sqrt(max(0, m Y2 - n^2 A^2))
 * minus the conservative margin of Q8:
 *   1e-12 (|RHS| + (A+L)|a_j| + (A-L)(nA/m)|b'_j|).
 * Only defined for lambda <= lambda_max (Q15); above it, everything but j* is
 * discarded (the null solution).  discard[j] = 1 for discarded columns;
 * zero-variance columns are always discarded. */
int or_bedpp(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
             const double *y, const uint8_t *train, double alpha, double lambda,
             uint8_t *discard)
{
    if (!(alpha > 0.0 && alpha <= 1.0) || !(lambda > 0.0)) return OR_ERR_ARG;
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    double *yt = malloc(sizeof(double) * n), *a = malloc(sizeof(double) * p);
    double *xs = malloc(sizeof(double) * n);
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (rc) goto done;
    int64_t nt = count_rows(train, n);
    center_y(y, n, train, nt, yt);
    double Y2 = 0.0;
    for (int64_t i = 0; i < n; i++) Y2 += yt[i] * yt[i];
    int64_t js = -1;
    double best = -1.0;
    OR_PAR
    for (int64_t j = 0; j < p; j++)
        a[j] = s[j] == 0.0 ? 0.0 : std_dot(X, dt, n, ld, j, c, s, train, yt);
    for (int64_t j = 0; j < p; j++)
        if (s[j] != 0.0 && fabs(a[j]) > best) { best = fabs(a[j]); js = j; }
    if (js < 0 || best == 0.0) { rc = OR_ERR_DEGENERATE; goto done; }
    for (int64_t i = 0; i < n; i++) xs[i] = in_rows(train, i) ? xstd(X, dt, ld, i, js, c, s) : 0.0;
    double nd = (double)nt;
    double A = best / nd;
    double L = alpha * lambda;
    double sig = a[js] > 0 ? 1.0 : -1.0;
    if (L >= A) {
        for (int64_t j = 0; j < p; j++) discard[j] = (j != js);
        goto done;
    }
    double m = nd * (1.0 + lambda * (1.0 - alpha));
    double rad = m * Y2 - nd * nd * A * A;
    if (rad < 0.0) rad = 0.0;
    double rhs = 2.0 * nd * L * A - (A - L) * sqrt(rad);
    OR_PAR
    for (int64_t j = 0; j < p; j++) {
        if (s[j] == 0.0) { discard[j] = 1; continue; }
        if (j == js) { discard[j] = 0; continue; }
        double b = std_dot(X, dt, n, ld, j, c, s, train, xs);
        double t1 = (A + L) * a[j];
        double t2 = (A - L) * (nd * A / m) * sig * b;
        double lhs = fabs(t1 - t2);
        double margin = 1e-12 * (fabs(rhs) + fabs(t1) + fabs(t2));
        discard[j] = lhs < rhs - margin;
    }
done:
    free(c); free(s); free(yt); free(a); free(xs);
    return rc;
}

/* One coordinate update of naive cyclic CD:
 *   z = x~_j^T r / n + b_j ;  b' = S(z, lambda alpha) / (1 + lambda (1 - alpha))
 *   r <- r - (b' - b_j) x~_j
 * split into the dot product x~_j^T r (std_dot) and the commit below, so that the
 * serial and the block-speculative passes run the same arithmetic.
 * Returns |b' - b_j|. */
static double cd_commit(const void *X, int dt, int64_t n, int64_t ld, int64_t j,
                        const double *c, const double *s, const uint8_t *train, double nd,
                        double lambda, double alpha, double dot, double *beta, double *r)
{
    double z = dot / nd + beta[j];
    double bn = soft(z, lambda * alpha) / (1.0 + lambda * (1.0 - alpha));
    double d = bn - beta[j];
    if (d != 0.0) {
        for (int64_t i = 0; i < n; i++)
            if (in_rows(train, i)) r[i] -= d * xstd(X, dt, ld, i, j, c, s);
        beta[j] = bn;
    }
    return fabs(d);
}

static double cd_update(const void *X, int dt, int64_t n, int64_t ld, int64_t j,
                        const double *c, const double *s, const uint8_t *train, double nd,
                        double lambda, double alpha, double *beta, double *r)
{
    return cd_commit(X, dt, n, ld, j, c, s, train, nd, lambda, alpha,
                     std_dot(X, dt, n, ld, j, c, s, train, r), beta, r);
}

enum { OR_SPEC_MAX = 65536 };   /* largest speculative block (columns) */

/* One full pass over every non-constant column, ascending j.  g_threads > 1:
 * block-speculative -- the dot products of columns j..j+B-1 are computed in
 * parallel against the current r, then committed in index order; after the first
 * committed change the block ends and the next one starts at the following
 * column (so every dot product a commit uses was taken against exactly the
 * residual the serial pass would use).  B doubles after a change-free block and
 * falls back to 8 T after a change. */
static void full_pass(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                      const double *c, const double *s, const uint8_t *train, double nd,
                      double lam, double alpha, double *beta, double *r, double *dot,
                      double *dmax_out, double *bmax_out)
{
    double dmax = 0.0, bmax = 0.0;
    if (g_threads <= 1) {
        for (int64_t j = 0; j < p; j++) {
            if (s[j] == 0.0) continue;
            double d = cd_update(X, dt, n, ld, j, c, s, train, nd, lam, alpha, beta, r);
            if (d > dmax) dmax = d;
            if (fabs(beta[j]) > bmax) bmax = fabs(beta[j]);
        }
    } else {
        const int64_t B0 = 8 * (int64_t)g_threads;
        int64_t B = B0, j = 0;
        while (j < p) {
            const int64_t j0 = j, je = j + B < p ? j + B : p;
            OR_PAR
            for (int64_t q = j0; q < je; q++)
                dot[q - j0] = s[q] == 0.0 ? 0.0 : std_dot(X, dt, n, ld, q, c, s, train, r);
            int changed = 0;
            while (j < je) {
                const int64_t jj = j++;
                if (s[jj] == 0.0) continue;
                double d = cd_commit(X, dt, n, ld, jj, c, s, train, nd, lam, alpha, dot[jj - j0], beta, r);
                if (d > dmax) dmax = d;
                if (fabs(beta[jj]) > bmax) bmax = fabs(beta[jj]);
                if (d != 0.0) { changed = 1; break; }
            }
            B = changed ? B0 : (2 * B <= OR_SPEC_MAX ? 2 * B : OR_SPEC_MAX);
        }
    }
    *dmax_out = dmax;
    *bmax_out = bmax;
}

/* State of one pathwise solve (warm starts carry beta and r from one lambda to
 * the next).  or_fit_path = or_path_begin + or_path_run over the whole grid +
 * or_path_end; bench.py's reference arm runs the grid in consecutive chunks. */
typedef struct {
    const void *X;
    int dt;
    int64_t n, p, ld, nt;
    uint8_t *train;          /* copy, or NULL */
    double *y;               /* copy */
    double alpha, nd, ybar, lmax, sigma_y;
    double *c, *s, *beta, *r, *dot;
} or_path_t;

void or_path_end(or_path_t *st)
{
    if (!st) return;
    free(st->train); free(st->y); free(st->c); free(st->s); free(st->beta); free(st->r); free(st->dot);
    free(st);
}

double or_path_lambda_max(const or_path_t *st) { return st ? st->lmax : 0.0; }

/* Column stats, y~ (r = y~, beta = 0) and lambda_max of the fit (SURVEY 8(c.2)
 * steps 1-5). */
int or_path_begin(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                  const double *y, const uint8_t *train, double alpha, or_path_t **out)
{
    *out = NULL;
    if (!X || !y || !(alpha > 0.0 && alpha <= 1.0)) return OR_ERR_ARG;
    or_path_t *st = calloc(1, sizeof(or_path_t));
    st->X = X; st->dt = dt; st->n = n; st->p = p; st->ld = ld; st->alpha = alpha;
    st->c = malloc(sizeof(double) * p); st->s = malloc(sizeof(double) * p);
    st->beta = calloc(p, sizeof(double)); st->r = malloc(sizeof(double) * n);
    st->dot = malloc(sizeof(double) * OR_SPEC_MAX);
    st->y = malloc(sizeof(double) * n);
    memcpy(st->y, y, sizeof(double) * n);
    if (train) { st->train = malloc(n); memcpy(st->train, train, n); }
    int rc = or_column_stats(X, dt, n, p, ld, st->train, st->c, st->s);
    if (rc) { or_path_end(st); return rc; }
    st->nt = count_rows(st->train, n);
    st->nd = (double)st->nt;
    st->ybar = center_y(st->y, n, st->train, st->nt, st->r);
    double yy = 0.0, lmax = 0.0;
    int any = 0;
    for (int64_t i = 0; i < n; i++) yy += st->r[i] * st->r[i];
    double *av = malloc(sizeof(double) * p);
    OR_PAR
    for (int64_t j = 0; j < p; j++)
        av[j] = st->s[j] == 0.0 ? 0.0
                                : fabs(std_dot(X, dt, n, ld, j, st->c, st->s, st->train, st->r)) / (st->nd * alpha);
    for (int64_t j = 0; j < p; j++) {
        if (st->s[j] == 0.0) continue;
        any = 1;
        if (av[j] > lmax) lmax = av[j];
    }
    free(av);
    if (yy == 0.0 || !any || lmax == 0.0) { or_path_end(st); return OR_ERR_DEGENERATE; }
    st->lmax = lmax;
    st->sigma_y = sqrt(yy / st->nd);
    *out = st;
    return OR_OK;
}

/* Pathwise coordinate descent, warm starts, no screening,
 * over lambda[0..nlam) continuing from the state's beta and r.
 *
 * Convergence (Q6): a pass converges when max_j |delta beta_j| <= tol * max_j |beta_j|
 * (or falls below the fp64 noise floor 1e-13 (alpha lambda + sd(y~))).
 * Without cycle_active every pass is a full pass over all non-constant j,
 * ascending.  With cycle_active, between full passes the current nonzeros are
 * cycled until they converge; the fit at lambda_k is accepted only when a FULL
 * pass converges (so this accelerates, it never screens).
 * max_iter (Q7) counts passes (full and active) per lambda.
 *
 * Outputs (caller-owned), k indexing this call's lambdas:
 *   col_ptr[nlam+1], idx[nnz_cap], beta[nnz_cap]  sparse standardised beta per lambda
 *   a0[nlam]      intercept on the original scale: ybar - sum_j beta_j c_j / s_j (Q4)
 *   obj[nlam]     objective Q at the returned beta (running residual)
 *   passes[nlam]  passes used
 *   resid (n*nlam, may be NULL): r_i = y_i - yhat_i for EVERY row i (rows outside
 *                 the training subset get their held-out residual), column k = lambda_k.
 *   n_converged   number of lambdas solved before an error.
 */
int or_path_run(or_path_t *st, const double *lambda, int nlam, double tol, int max_iter,
                int cycle_active, int64_t nnz_cap,
                int64_t *col_ptr, int64_t *idx, double *beta_out,
                double *a0, double *obj, int32_t *passes, double *resid, int *n_converged)
{
    if (n_converged) *n_converged = 0;
    if (!st || !lambda || nlam < 1 || !(tol > 0.0) || max_iter < 1) return OR_ERR_ARG;
    for (int k = 0; k < nlam; k++) {
        if (!(lambda[k] > 0.0)) return OR_ERR_ARG;
        if (k > 0 && !(lambda[k] < lambda[k - 1])) return OR_ERR_ARG;
    }
    const void *X = st->X;
    const int dt = st->dt;
    const int64_t n = st->n, p = st->p, ld = st->ld;
    const uint8_t *train = st->train;
    const double *c = st->c, *s = st->s, *y = st->y;
    double *beta = st->beta, *r = st->r;
    const double alpha = st->alpha, nd = st->nd, ybar = st->ybar, lmax = st->lmax;
    int rc = OR_OK;
    int64_t nnz = 0;
    col_ptr[0] = 0;
    for (int k = 0; k < nlam; k++) {
        double lam = lambda[k];
        int np_ = 0;
        /* Q25: at lambda >= lambda_max the solution is exactly 0 (definition of
         * lambda_max).  A grid point within 1e-12 (relative) of lambda_max
         * is snapped to the null solution so rounding in the kink cannot leave
         * ulp-sized coefficients (beta stays 0 from the warm start). */
        int snap = lam >= lmax * (1.0 - 1e-12);
        /* Q6 noise floor: coefficient changes below 1e-13 (alpha lambda + sd(y~))
         * are fp64 rounding of z, not progress. */
        double floor_ = 1e-13 * (alpha * lam + st->sigma_y);
        for (; !snap;) {
            /* optional active cycling (acceleration only) */
            if (cycle_active) {
                for (;;) {
                    double dmax = 0.0, bmax = 0.0;
                    int any = 0;
                    for (int64_t j = 0; j < p; j++) {
                        if (beta[j] == 0.0) continue;
                        any = 1;
                        double d = cd_update(X, dt, n, ld, j, c, s, train, nd, lam, alpha, beta, r);
                        if (d > dmax) dmax = d;
                        if (fabs(beta[j]) > bmax) bmax = fabs(beta[j]);
                    }
                    if (!any) break;
                    if (++np_ > max_iter) { rc = OR_ERR_CONVERGENCE; goto done; }
                    if (dmax <= tol * bmax || dmax <= floor_) break;
                }
            }
            /* full pass over every non-constant column, ascending j */
            double dmax, bmax;
            full_pass(X, dt, n, p, ld, c, s, train, nd, lam, alpha, beta, r, st->dot, &dmax, &bmax);
            if (++np_ > max_iter) { rc = OR_ERR_CONVERGENCE; goto done; }
            if (dmax <= tol * bmax || dmax <= floor_) break;
        }
        /* record lambda_k */
        double l1 = 0.0, l2 = 0.0, shift = 0.0;
        for (int64_t j = 0; j < p; j++) {
            if (beta[j] == 0.0) continue;
            if (nnz >= nnz_cap) { rc = OR_ERR_ARG; goto done; }
            idx[nnz] = j;
            beta_out[nnz] = beta[j];
            nnz++;
            l1 += fabs(beta[j]);
            l2 += beta[j] * beta[j];
            shift += beta[j] * c[j] / s[j];
        }
        col_ptr[k + 1] = nnz;
        double rss = 0.0;
        for (int64_t i = 0; i < n; i++)
            if (in_rows(train, i)) rss += r[i] * r[i];
        if (a0) a0[k] = ybar - shift;
        if (obj) obj[k] = rss / (2.0 * nd) + lam * (alpha * l1 + 0.5 * (1.0 - alpha) * l2);
        if (passes) passes[k] = np_;
        if (resid) {
            /* every row: y_i - (ybar + sum_j x~_ij beta_j), formed explicitly (rows independent) */
            OR_PAR
            for (int64_t i = 0; i < n; i++) {
                double f = ybar;
                for (int64_t j = 0; j < p; j++)
                    if (beta[j] != 0.0) f += xstd(X, dt, ld, i, j, c, s) * beta[j];
                resid[(int64_t)k * n + i] = y[i] - f;
            }
        }
        if (n_converged) *n_converged = k + 1;
    }
done:
    return rc;
}

/* The whole grid in one call (the path of SURVEY 8(c.2)). */
int or_fit_path(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                const double *y, const uint8_t *train,
                const double *lambda, int nlam, double alpha, double tol, int max_iter,
                int cycle_active, int64_t nnz_cap,
                int64_t *col_ptr, int64_t *idx, double *beta_out,
                double *a0, double *obj, int32_t *passes, double *resid, int *n_converged)
{
    if (n_converged) *n_converged = 0;
    if (!X || !y || !lambda || nlam < 1 || !(alpha > 0.0 && alpha <= 1.0) || !(tol > 0.0) ||
        max_iter < 1)
        return OR_ERR_ARG;
    for (int k = 0; k < nlam; k++) {
        if (!(lambda[k] > 0.0)) return OR_ERR_ARG;
        if (k > 0 && !(lambda[k] < lambda[k - 1])) return OR_ERR_ARG;
    }
    col_ptr[0] = 0;
    or_path_t *st = NULL;
    int rc = or_path_begin(X, dt, n, p, ld, y, train, alpha, &st);
    if (rc) return rc;
    rc = or_path_run(st, lambda, nlam, tol, max_iter, cycle_active, nnz_cap, col_ptr, idx, beta_out,
                     a0, obj, passes, resid, n_converged);
    or_path_end(st);
    return rc;
}

/* Counter-based generator for the CV fold permutation (Q18): splitmix64. */
static uint64_t splitmix64(uint64_t *state)
{
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* Q18: perm = Fisher-Yates permutation of 0..n-1 driven by splitmix64(seed)
 * (for i = n-1 .. 1: swap perm[i], perm[u % (i+1)]); fold_id[perm[i]] = i mod K.
 * P:542 ("seed = 1234"), P:278 (folds as row-index vectors). */
int or_folds(int64_t n, int K, uint64_t seed, int32_t *fold_id)
{
    if (K < 2 || K > n) return OR_ERR_ARG;
    int64_t *perm = malloc(sizeof(int64_t) * n);
    for (int64_t i = 0; i < n; i++) perm[i] = i;
    uint64_t st = seed;
    for (int64_t i = n - 1; i >= 1; i--) {
        int64_t jj = (int64_t)(splitmix64(&st) % (uint64_t)(i + 1));
        int64_t t = perm[i]; perm[i] = perm[jj]; perm[jj] = t;
    }
    for (int64_t i = 0; i < n; i++) fold_id[perm[i]] = (int32_t)(i % K);
    free(perm);
    return OR_OK;
}

/* K-fold cross-validation (Q16, Q17).
 * For fold f the training rows are {i : fold_id[i] != f}; column stats and the
 * centering of y are recomputed on those rows (Q16); the full-data lambda grid
 * is shared.  E[k*n + i] = squared held-out error of row i at lambda_k
 * from the fit of fold fold_id[i].  cve_k = mean_i E; cvse_k = sd_i(E)/sqrt(n)
 * (pooled per-observation SE, Q17 -- parity unpinned beyond recomputation).
 * lambda_min_index = argmin cve (lowest index on ties). */
int or_cv(const void *X, int dt, int64_t n, int64_t p, int64_t ld, const double *y,
          const int32_t *fold_id, int K, const double *lambda, int nlam, double alpha,
          double tol, int max_iter, int cycle_active,
          double *E, double *cve, double *cvse, int *lambda_min_index)
{
    if (K < 2 || K > n || !fold_id) return OR_ERR_ARG;
    for (int64_t i = 0; i < n; i++)
        if (fold_id[i] < 0 || fold_id[i] >= K) return OR_ERR_ARG;
    uint8_t *train = malloc(n);
    double *resid = malloc(sizeof(double) * n * nlam);
    int64_t cap = (int64_t)p * nlam;
    if (cap > ((int64_t)1 << 26)) cap = (int64_t)1 << 26;
    int64_t *col_ptr = malloc(sizeof(int64_t) * (nlam + 1)), *idx = malloc(sizeof(int64_t) * cap);
    double *bv = malloc(sizeof(double) * cap);
    int rc = OR_OK;
    for (int f = 0; f < K && rc == OR_OK; f++) {
        int64_t held = 0;
        for (int64_t i = 0; i < n; i++) { train[i] = fold_id[i] != f; held += !train[i]; }
        if (held == 0) { rc = OR_ERR_ARG; break; }
        int nc = 0;
        rc = or_fit_path(X, dt, n, p, ld, y, train, lambda, nlam, alpha, tol, max_iter,
                         cycle_active, cap, col_ptr, idx, bv, NULL, NULL, NULL, resid, &nc);
        if (rc) break;
        for (int k = 0; k < nlam; k++)
            for (int64_t i = 0; i < n; i++)
                if (!train[i]) {
                    double e = resid[(int64_t)k * n + i];
                    E[(int64_t)k * n + i] = e * e;
                }
    }
    if (rc == OR_OK) {
        int best = 0;
        for (int k = 0; k < nlam; k++) {
            double m = 0.0;
            for (int64_t i = 0; i < n; i++) m += E[(int64_t)k * n + i];
            m /= (double)n;
            double v = 0.0;
            for (int64_t i = 0; i < n; i++) {
                double d = E[(int64_t)k * n + i] - m;
                v += d * d;
            }
            cve[k] = m;
            cvse[k] = sqrt(v / (double)(n - 1)) / sqrt((double)n);
            if (cve[k] < cve[best]) best = k;
        }
        *lambda_min_index = best;
    }
    free(train); free(resid); free(col_ptr); free(idx); free(bv);
    return rc;
}

/* ===================================================================================
 * NEXT-3: lasso / elastic-net penalised LOGISTIC regression path.
 *
 * P:174 ("sparse linear and logistic regression models with lasso and elastic net
 * penalties are implemented"), P:244 (hybrid screening for logistic regression),
 * P:379-385 (the logistic simulation).  The paper prints no formula for this model;
 * the readings below are DESIGN.md's QL1-QL6.
 *
 * Objective (QL1, the glmnet binomial form with the penalty of Q2):
 *   Q(b0, b) = (1/n_t) sum_i [ log(1 + exp(eta_i)) - y_i eta_i ]
 *              + lambda [ alpha |b|_1 + (1-alpha)/2 |b|^2 ],   eta_i = b0 + x~_i' b,
 * y_i in {0, 1}, b0 unpenalised, x~ the explicitly standardised columns.
 * lambda_max (QL2) = max_j |x~_j'(y - ybar)| / (n alpha): the KKT condition at b = 0,
 * b0 = logit(ybar).
 *
 * Algorithm (QL4, "outer IRLS loop per lambda ... inner weighted CD"),
 * written as the textbook iteratively-reweighted least squares:
 *   outer: pi_i = 1/(1+exp(-eta_i)); w_i = max(pi_i (1-pi_i), 1e-5) (QL5: the floor
 *          bounds the WEIGHT only; the gradient keeps the exact pi);
 *          working response zr_i = eta_i + (y_i - pi_i)/w_i;
 *   inner: cyclic CD on (1/2n) sum_i w_i (zr_i - b0 - x~_i'b)^2 + penalty, intercept
 *          first in every pass, then every non-constant j ascending:
 *             b0 <- b0 + sum_i w_i e_i / sum_i w_i              (e = zr - eta, running)
 *             u_j = sum_i w_i x~_ij e_i / n + v_j b_j,  v_j = sum_i w_i x~_ij^2 / n
 *             b_j <- S(u_j, lambda alpha) / (v_j + lambda (1-alpha))
 *          until a pass moves no b_j by more than tol * max|b| and b0 by no more
 *          than tol * max(1, |b0|) (Q6, QL6);
 *   eta recomputed explicitly from (b0, b); the outer loop ends when a whole outer
 *   iteration meets the same test (QL6).
 * ================================================================================= */

static double sigmoid(double t) { return t >= 0.0 ? 1.0 / (1.0 + exp(-t)) : exp(t) / (1.0 + exp(t)); }

/* log(1 + exp(t)) without overflow */
static double log1pexp(double t) { return t > 0.0 ? t + log1p(exp(-t)) : log1p(exp(t)); }

/* y must be 0/1 on the used rows with both classes present. */
static int check_binary(const double *y, int64_t n, const uint8_t *train, double *ybar)
{
    int64_t n1 = 0, nt = 0;
    for (int64_t i = 0; i < n; i++) {
        if (!in_rows(train, i)) continue;
        if (!(y[i] == 0.0 || y[i] == 1.0)) return OR_ERR_ARG;
        n1 += y[i] == 1.0;
        nt++;
    }
    if (n1 == 0 || n1 == nt) return OR_ERR_DEGENERATE;
    *ybar = (double)n1 / (double)nt;
    return OR_OK;
}

/* Q(b0, b) of QL1 with eta formed explicitly from (b0, b). */
int or_objective_binomial(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                          const double *y, const uint8_t *train, double b0, const double *beta,
                          double lambda, double alpha, double *Q)
{
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    double ybar = 0.0;
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (!rc) rc = check_binary(y, n, train, &ybar);
    if (rc) goto done;
    double loss = 0.0, l1 = 0.0, l2 = 0.0;
    int64_t nt = count_rows(train, n);
    for (int64_t j = 0; j < p; j++)
        if (beta[j] != 0.0) {
            if (s[j] == 0.0) { rc = OR_ERR_ARG; goto done; }
            l1 += fabs(beta[j]);
            l2 += beta[j] * beta[j];
        }
    for (int64_t i = 0; i < n; i++) {
        if (!in_rows(train, i)) continue;
        double eta = b0;
        for (int64_t j = 0; j < p; j++)
            if (beta[j] != 0.0) eta += xstd(X, dt, ld, i, j, c, s) * beta[j];
        loss += log1pexp(eta) - y[i] * eta;
    }
    *Q = loss / (double)nt + lambda * (alpha * l1 + 0.5 * (1.0 - alpha) * l2);
done:
    free(c); free(s);
    return rc;
}

/* Path of QL1 over a decreasing grid, warm starts, no screening.  Outputs as
 * or_fit_path; b0_out[k] = intercept on the standardised scale, a0[k] = intercept
 * on the original scale (b0 - sum_j b_j c_j / s_j, Q4); passes[k] = inner passes
 * summed over the outer iterations; outer[k] = outer (IRLS) iterations. */
int or_fit_path_binomial(const void *X, int dt, int64_t n, int64_t p, int64_t ld,
                         const double *y, const uint8_t *train,
                         const double *lambda, int nlam, double alpha, double tol, int max_iter,
                         int cycle_active, int64_t nnz_cap,
                         int64_t *col_ptr, int64_t *idx, double *beta_out,
                         double *b0_out, double *a0, double *obj, int32_t *passes, int32_t *outer,
                         int *n_converged)
{
    if (!X || !y || !lambda || nlam < 1 || !(alpha > 0.0 && alpha <= 1.0) || !(tol > 0.0) ||
        max_iter < 1)
        return OR_ERR_ARG;
    for (int k = 0; k < nlam; k++) {
        if (!(lambda[k] > 0.0)) return OR_ERR_ARG;
        if (k > 0 && !(lambda[k] < lambda[k - 1])) return OR_ERR_ARG;
    }
    double *c = malloc(sizeof(double) * p), *s = malloc(sizeof(double) * p);
    double *beta = calloc(p, sizeof(double)), *bprev = malloc(sizeof(double) * p);
    double *eta = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
    double *e = malloc(sizeof(double) * n), *v = malloc(sizeof(double) * p);
    double ybar = 0.0;
    int64_t nnz = 0;
    if (n_converged) *n_converged = 0;
    col_ptr[0] = 0;
    int rc = or_column_stats(X, dt, n, p, ld, train, c, s);
    if (!rc) rc = check_binary(y, n, train, &ybar);
    if (rc) goto done;
    int64_t nt = count_rows(train, n);
    double nd = (double)nt;
    double lmax = 0.0;
    {
        int any = 0;
        for (int64_t i = 0; i < n; i++) e[i] = in_rows(train, i) ? y[i] - ybar : 0.0;
        for (int64_t j = 0; j < p; j++) {
            if (s[j] == 0.0) continue;
            any = 1;
            double a = fabs(std_dot(X, dt, n, ld, j, c, s, train, e)) / (nd * alpha);
            if (a > lmax) lmax = a;
        }
        if (!any || lmax == 0.0) { rc = OR_ERR_DEGENERATE; goto done; }
    }
    double b0 = log(ybar / (1.0 - ybar));          /* the null model (QL2) */
    for (int64_t i = 0; i < n; i++) eta[i] = b0;
    for (int k = 0; k < nlam; k++) {
        double lam = lambda[k];
        int np_ = 0, no_ = 0;
        int snap = lam >= lmax * (1.0 - 1e-12);    /* Q25 */
        double floor_ = 1e-13 * (alpha * lam + 1.0);
        while (!snap) {
            /* ---- outer (IRLS) iteration: weights and working residual at eta */
            double sw = 0.0;
            for (int64_t i = 0; i < n; i++) {
                if (!in_rows(train, i)) { w[i] = 0.0; e[i] = 0.0; continue; }
                double pi = sigmoid(eta[i]);
                double wi = pi * (1.0 - pi);
                if (wi < 1e-5) wi = 1e-5;          /* QL5 */
                w[i] = wi;
                e[i] = (y[i] - pi) / wi;           /* zr_i - eta_i */
                sw += wi;
            }
            OR_PAR
            for (int64_t j = 0; j < p; j++) {
                v[j] = 0.0;
                if (s[j] == 0.0) continue;
                for (int64_t i = 0; i < n; i++)
                    if (in_rows(train, i)) { double x = xstd(X, dt, ld, i, j, c, s); v[j] += w[i] * x * x; }
                v[j] /= nd;
            }
            memcpy(bprev, beta, sizeof(double) * p);
            double b0prev = b0;
            /* ---- inner weighted CD: with cycle_active, the nonzeros are cycled until
             * converged first (acceleration only); the inner solve ends with a
             * converged FULL pass.  Converged (Q6 per block): max|db| <= tol max|b| and
             * |db0| <= tol max(1, |b0|), or both below the noise floor. */
            for (int pass_kind = cycle_active ? 0 : 1; pass_kind < 2; pass_kind++) {
                for (;;) {
                    double dmax = 0.0, bmax = 0.0, num = 0.0;
                    int any = 0;
                    for (int64_t i = 0; i < n; i++) num += w[i] * e[i];
                    double d0 = num / sw;              /* intercept first */
                    b0 += d0;
                    for (int64_t i = 0; i < n; i++)
                        if (in_rows(train, i)) e[i] -= d0;
                    for (int64_t j = 0; j < p; j++) {
                        if (s[j] == 0.0) continue;
                        if (pass_kind == 0 && beta[j] == 0.0) continue;
                        any = 1;
                        double u = 0.0;
                        for (int64_t i = 0; i < n; i++)
                            if (in_rows(train, i)) u += w[i] * xstd(X, dt, ld, i, j, c, s) * e[i];
                        u = u / nd + v[j] * beta[j];
                        double bn = soft(u, lam * alpha) / (v[j] + lam * (1.0 - alpha));
                        double d = bn - beta[j];
                        if (d != 0.0) {
                            for (int64_t i = 0; i < n; i++)
                                if (in_rows(train, i)) e[i] -= d * xstd(X, dt, ld, i, j, c, s);
                            beta[j] = bn;
                        }
                        if (fabs(d) > dmax) dmax = fabs(d);
                        if (fabs(bn) > bmax) bmax = fabs(bn);
                    }
                    if (++np_ > max_iter) { rc = OR_ERR_CONVERGENCE; goto done; }
                    if (pass_kind == 0 && !any) break;
                    int ok_b = dmax <= tol * bmax || dmax <= floor_;
                    int ok_0 = fabs(d0) <= tol * (fabs(b0) > 1.0 ? fabs(b0) : 1.0) || fabs(d0) <= floor_;
                    if (ok_b && ok_0) break;
                }
            }
            /* ---- eta from (b0, b), explicitly */
            for (int64_t i = 0; i < n; i++) {
                double t = b0;
                for (int64_t j = 0; j < p; j++)
                    if (beta[j] != 0.0) t += xstd(X, dt, ld, i, j, c, s) * beta[j];
                eta[i] = t;
            }
            double dmax = 0.0, bmax = 0.0, d0 = fabs(b0 - b0prev);
            for (int64_t j = 0; j < p; j++) {
                double d = fabs(beta[j] - bprev[j]);
                if (d > dmax) dmax = d;
                if (fabs(beta[j]) > bmax) bmax = fabs(beta[j]);
            }
            if (++no_ > max_iter) { rc = OR_ERR_CONVERGENCE; goto done; }
            int ok_b = dmax <= tol * bmax || dmax <= floor_;
            int ok_0 = d0 <= tol * (fabs(b0) > 1.0 ? fabs(b0) : 1.0) || d0 <= floor_;
            if (ok_b && ok_0) break;
        }
        /* record lambda_k */
        double l1 = 0.0, l2 = 0.0, shift = 0.0, loss = 0.0;
        for (int64_t j = 0; j < p; j++) {
            if (beta[j] == 0.0) continue;
            if (nnz >= nnz_cap) { rc = OR_ERR_ARG; goto done; }
            idx[nnz] = j;
            beta_out[nnz] = beta[j];
            nnz++;
            l1 += fabs(beta[j]);
            l2 += beta[j] * beta[j];
            shift += beta[j] * c[j] / s[j];
        }
        col_ptr[k + 1] = nnz;
        for (int64_t i = 0; i < n; i++)
            if (in_rows(train, i)) loss += log1pexp(eta[i]) - y[i] * eta[i];
        if (b0_out) b0_out[k] = b0;
        if (a0) a0[k] = b0 - shift;
        if (obj) obj[k] = loss / nd + lam * (alpha * l1 + 0.5 * (1.0 - alpha) * l2);
        if (passes) passes[k] = np_;
        if (outer) outer[k] = no_;
        if (n_converged) *n_converged = k + 1;
    }
done:
    free(c); free(s); free(beta); free(bprev); free(eta); free(w); free(e); free(v);
    return rc;
}
