/*
 * bb_oracle.c -- plain, slow, sequential CPU fp64 ORACLE for the reduction of
 * an n x n upper-banded matrix (b superdiagonals) to upper bidiagonal form by
 * Householder bulge chasing with successive bandwidth reduction
 * (arXiv 2510.12705, Ringoot/Alomairy/Edelman 2025).
 *
 * *** TEST INFRASTRUCTURE ONLY. ***  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this file's
 * library.  The product (paper_2510_12705_b200/) never links, imports or
 * executes it, and shares no code, header, helper or constant with it.
 *
 * What it follows (P:n = line n of PAPER.md, S:n = SPEC.md):
 *   - Alg. 1: outer loop over bandwidth passes, each removing the
 *     inner tilewidth TW (b -> b-tw -> ... -> 1); inside, one sweep per row R,
 *     each sweep a chain of row-bulge steps.  Readings Q1-Q3:
 *       pass (c, t):  t = min(tw, c-1), target bandwidth c - t;
 *       sweep r in 0..n-2, step j = 0,1,...:
 *         p_j = r + (c - t) + j*c,  q_0 = r,  q_j = p_{j-1}   (anchor update
 *         "first k <- k - TW, then += TW + TBW" of Alg. 1 lines 9-10)
 *         hi = min(p+t, n-1), ce = min(hi+c, n-1); the step exists iff p <= n-2.
 *   - Alg. 2 and its text: per step, a row reflector built
 *     from A[q, p..hi] ("HH(X)", line 5), applied from the right to rows
 *     q+1..hi (lines 8-13); then the column reflector of the left-most column
 *     of the generated bulge, A[p..hi, p] (line 15), applied from the left to
 *     columns p+1..ce.  Only values are written back (Q9): beta and exact
 *     zeros in the annihilated slots.
 *   - Reflector convention (P:189 delegates to prior tile-QR work; reading
 *     Q7/Q8): LAPACK dlarfg -- beta = -sign(alpha)*||x||, sign(0) = +1,
 *     tau = (beta - alpha)/beta, v = [1, x(1:)/(alpha - beta)]; identity
 *     (tau = 0, beta = alpha) iff x(1:) is exactly zero; the norm is computed
 *     scaled by max|x_k| so it neither underflows nor overflows.
 *   - Storage (reading Q11): the oracle keeps its OWN row-wise band
 *     store, row i holding offsets d = j - i in [-tw, b + tw]
 *     (height b + 2*tw + 1).  Every access goes through at(), which flags any
 *     access outside that range -- so a run that returns 0 also proves the
 *     "band + twice the tilewidth" storage claim for that input.
 *   - Summation is plain left-to-right.  Sweeps run strictly in order
 *     (sequential semantics); the oracle has no scheduler.
 *
 * Precision: fp64 throughout.  fp16/fp32 inputs are widened to fp64 by the
 * caller (reading Q13).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
    int64_t n;      /* matrix order                                   */
    int64_t b;      /* input bandwidth (superdiagonals), clamped <= n-1 */
    int64_t tw;     /* requested inner tilewidth                       */
    int64_t lo;     /* lowest stored offset  j - i  (= -tw)            */
    int64_t hi;     /* highest stored offset j - i  (= b + tw)         */
    int64_t width;  /* hi - lo + 1                                     */
    int oob;        /* set when any access falls outside the store     */
    double dummy;   /* target of out-of-store accesses                 */
    double *a;      /* a[i*width + (j - i - lo)] = A[i][j]             */
} omat;

/* element accessor: the only way the algorithm touches the matrix */
static double *at(omat *M, int64_t i, int64_t j)
{
    int64_t d = j - i;
    if (i < 0 || j < 0 || i >= M->n || j >= M->n || d < M->lo || d > M->hi) {
        M->oob = 1;
        M->dummy = 0.0;
        return &M->dummy;
    }
    return &M->a[i * M->width + (d - M->lo)];
}

/* ---------------------------------------------------------------------- */
/* HH(X) of Alg. 2 line 5: reflector H = I - tau v v^T with H x = beta e_1 */
/* (LAPACK dlarfg semantics, reading Q7/Q8).  v[0] = 1.                    */
/* ---------------------------------------------------------------------- */
void oracle_house(int64_t m, const double *x, double *v, double *tau, double *beta)
{
    double alpha = x[0];
    int tail_zero = 1;
    for (int64_t k = 1; k < m; k++)
        if (x[k] != 0.0) tail_zero = 0;
    v[0] = 1.0;
    if (m <= 1 || tail_zero) {           /* nothing to annihilate: H = I */
        for (int64_t k = 1; k < m; k++) v[k] = 0.0;
        *tau = 0.0;
        *beta = alpha;
        return;
    }
    double s = 0.0;                       /* scale: max |x_k| > 0 here */
    for (int64_t k = 0; k < m; k++)
        if (fabs(x[k]) > s) s = fabs(x[k]);
    double ssq = 0.0;
    for (int64_t k = 0; k < m; k++) {
        double y = x[k] / s;
        ssq += y * y;
    }
    double nrm = s * sqrt(ssq);
    double bt = (alpha >= 0.0) ? -nrm : nrm;   /* beta = -sign(alpha)||x|| */
    *beta = bt;
    *tau = (bt - alpha) / bt;
    for (int64_t k = 1; k < m; k++) v[k] = x[k] / (alpha - bt);
}

/* ---------------------------------------------------------------------- */
/* Pass plan (Alg. 1 lines 1-2, readings Q1/Q2)                            */
/* ---------------------------------------------------------------------- */
int64_t oracle_num_passes(int64_t n, int64_t b, int64_t tw)
{
    if (n <= 2 || b <= 1 || tw < 1) return 0;
    int64_t c = b < n - 1 ? b : n - 1, np = 0;
    while (c > 1) {
        int64_t t = tw < c - 1 ? tw : c - 1;
        np++;
        c -= t;
    }
    return np;
}

/* pass k (0-based): current bandwidth c and tilewidth t; returns -1 if none */
int oracle_pass(int64_t n, int64_t b, int64_t tw, int64_t k, int64_t *c_out, int64_t *t_out)
{
    if (n <= 2 || b <= 1 || tw < 1) return -1;
    int64_t c = b < n - 1 ? b : n - 1, idx = 0;
    while (c > 1) {
        int64_t t = tw < c - 1 ? tw : c - 1;
        if (idx == k) { *c_out = c; *t_out = t; return 0; }
        idx++;
        c -= t;
    }
    return -1;
}

/* step geometry (Alg. 1 lines 7-10, reading Q3): returns 0 if the step exists */
int oracle_step_geometry(int64_t n, int64_t c, int64_t t, int64_t r, int64_t j,
                         int64_t *q, int64_t *p, int64_t *hi, int64_t *ce)
{
    int64_t pj = r + (c - t) + j * c;
    if (r < 0 || j < 0 || pj > n - 2) return -1;
    *p = pj;
    *q = (j == 0) ? r : pj - c;
    *hi = (pj + t < n - 1) ? pj + t : n - 1;
    *ce = (*hi + c < n - 1) ? *hi + c : n - 1;
    return 0;
}

/* ---------------------------------------------------------------------- */
/* One row-bulge step (Alg. 2 executed for the bulge of sweep r, step j)  */
/* ---------------------------------------------------------------------- */
static void step(omat *M, int64_t c, int64_t t, int64_t r, int64_t j)
{
    int64_t q, p, hi, ce;
    if (oracle_step_geometry(M->n, c, t, r, j, &q, &p, &hi, &ce) != 0) return;
    int64_t m = hi - p + 1;
    double x[1024], v[1024], tau, beta;
    if (m > 1024) { M->oob = 1; return; }

    /* row reflector from A[q, p..hi] (Alg. 1 line 7; Alg. 2 lines 3-6) */
    for (int64_t k = 0; k < m; k++) x[k] = *at(M, q, p + k);
    oracle_house(m, x, v, &tau, &beta);
    /* right application to rows q+1..hi (Alg. 2 lines 8-13) */
    if (tau != 0.0) {
        for (int64_t i = q + 1; i <= hi; i++) {
            double w = 0.0;
            for (int64_t k = 0; k < m; k++) w += *at(M, i, p + k) * v[k];
            for (int64_t k = 0; k < m; k++) *at(M, i, p + k) -= tau * w * v[k];
        }
    }
    *at(M, q, p) = beta;
    for (int64_t k = 1; k < m; k++) *at(M, q, p + k) = 0.0;

    /* column reflector from A[p..hi, p] (Alg. 1 line 8; Alg. 2 line 15) */
    for (int64_t k = 0; k < m; k++) x[k] = *at(M, p + k, p);
    oracle_house(m, x, v, &tau, &beta);
    /* left application to columns p+1..ce */
    if (tau != 0.0) {
        for (int64_t jc = p + 1; jc <= ce; jc++) {
            double w = 0.0;
            for (int64_t k = 0; k < m; k++) w += v[k] * *at(M, p + k, jc);
            for (int64_t k = 0; k < m; k++) *at(M, p + k, jc) -= tau * v[k] * w;
        }
    }
    *at(M, p, p) = beta;
    for (int64_t k = 1; k < m; k++) *at(M, p + k, p) = 0.0;
}

/* ---------------------------------------------------------------------- */
/* Handle API: load, step, run, extract                                    */
/* ---------------------------------------------------------------------- */

/* band: LAPACK upper band, A(i,j) = band[(b + i - j) + j*ldband],
 * max(0, j-b) <= i <= j; values already widened to fp64 by the caller. */
void *oracle_new(int64_t n, int64_t b, int64_t tw, const double *band, int64_t ldband)
{
    if (n < 0 || b < 0 || tw < 1 || ldband < b + 1) return NULL;
    omat *M = (omat *)calloc(1, sizeof(omat));
    if (!M) return NULL;
    int64_t bc = (n > 0 && b > n - 1) ? n - 1 : b;
    M->n = n;
    M->b = bc;
    M->tw = tw;
    M->lo = -tw;
    M->hi = bc + tw;
    M->width = M->hi - M->lo + 1;
    M->a = (double *)calloc((size_t)(n > 0 ? n : 1) * (size_t)M->width, sizeof(double));
    if (!M->a) { free(M); return NULL; }
    for (int64_t j = 0; j < n; j++)
        for (int64_t i = (j - bc > 0 ? j - bc : 0); i <= j; i++)
            *at(M, i, j) = band[(b + i - j) + j * ldband];
    return M;
}

void oracle_free(void *h)
{
    omat *M = (omat *)h;
    if (!M) return;
    free(M->a);
    free(M);
}

int oracle_step(void *h, int64_t c, int64_t t, int64_t r, int64_t j)
{
    omat *M = (omat *)h;
    step(M, c, t, r, j);
    return M->oob ? -2 : 0;
}

/* Sequential algorithm (Alg. 1, sweeps strictly in order).  Executes at most
 * max_steps steps (max_steps < 0: all) -- a bounded sample for the CPU
 * baseline -- and reports how many steps ran and the algorithmic element
 * count sum m*((hi-q+1) + (ce-p+1) - m) over those steps. */
int oracle_run(void *h, int64_t max_steps, int64_t *steps_done, double *elems_touched)
{
    omat *M = (omat *)h;
    int64_t n = M->n, done = 0;
    double elems = 0.0;
    if (n > 2 && M->b > 1) {
        int64_t c = M->b;
        while (c > 1) {
            int64_t t = M->tw < c - 1 ? M->tw : c - 1;
            for (int64_t r = 0; r <= n - 2; r++) {
                for (int64_t j = 0;; j++) {
                    int64_t q, p, hi, ce;
                    if (oracle_step_geometry(n, c, t, r, j, &q, &p, &hi, &ce) != 0) break;
                    if (max_steps >= 0 && done >= max_steps) goto out;
                    step(M, c, t, r, j);
                    int64_t m = hi - p + 1;
                    elems += (double)(m * ((hi - q + 1) + (ce - p + 1) - m));
                    done++;
                }
            }
            c -= t;
        }
    }
out:
    if (steps_done) *steps_done = done;
    if (elems_touched) *elems_touched = elems;
    return M->oob ? -2 : 0;
}

/* d[i] = A[i][i], e[i] = A[i][i+1]; store (optional) receives the whole
 * row-wise store, n x (b + 2 tw + 1), row i offset d = j - i at [d + tw]. */
void oracle_extract(void *h, double *d, double *e, double *store)
{
    omat *M = (omat *)h;
    for (int64_t i = 0; i < M->n; i++) {
        d[i] = *at(M, i, i);
        if (i + 1 < M->n) e[i] = M->b >= 1 ? *at(M, i, i + 1) : 0.0;
    }
    if (store) memcpy(store, M->a, (size_t)M->n * (size_t)M->width * sizeof(double));
}

int64_t oracle_store_width(void *h) { return ((omat *)h)->width; }

/* one-call form: the whole reduction.  Returns 0 ok, -1 bad args/alloc,
 * -2 an access left the band + 2*tw store. */
int oracle_band_to_bidiag(int64_t n, int64_t b, int64_t tw, const double *band, int64_t ldband,
                          double *d, double *e)
{
    void *h = oracle_new(n, b, tw, band, ldband);
    if (!h) return -1;
    int rc = oracle_run(h, -1, NULL, NULL);
    oracle_extract(h, d, e, NULL);
    oracle_free(h);
    return rc;
}
