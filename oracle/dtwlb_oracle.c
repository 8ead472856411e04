/*
 * dtwlb_oracle.c -- plain, slow, fp64 CPU oracle for the two-pass DTW
 * nearest-neighbour method of D. Lemire, "Faster Retrieval with a Two-Pass
 * Dynamic-Time-Warping Lower Bound" (arXiv:0811.3301).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_0811_3301_b200/) never links, imports or calls it,
 * and this file shares no code, header, table or helper with the CUDA path.
 *
 * Citations "P:n" are lines of the paper's LaTeX source, with the
 * section / equation / algorithm named alongside.  Readings of ambiguous
 * passages are numbered c1..c18 as in DESIGN.md ("Readings of the paper").
 *
 * Conventions (section "Conventions"): series have length n; the
 * paper indexes 1..n, this file indexes 0..n-1 (index k here = k+1 there).
 * The candidate is x and the query is y (Alg. 2/3).
 * All arithmetic is double precision; callers pass the SAME float32 arrays
 * the GPU sees and this file upcasts each value once (reading c12).
 * p >= 1 is a finite exponent; p == 0 encodes p = infinity.
 *
 * Parity pins for every function live in tests/test_oracle_*.py.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORACLE_INF (1.0 / 0.0)

/* |a|^p for finite p (l_p norm term). */
static double powabs(double a, int p)
{
    double v = fabs(a);
    if (p == 1) return v;
    if (p == 2) return v * v;
    return pow(v, (double)p);
}

/* v^(1/p): the root taken once at the end ("DTW_p(x,y) = q_{1,1}^(1/p)"). */
static double root_p(double v, int p)
{
    if (p == 0 || p == 1) return v;
    if (p == 2) return sqrt(v);
    return pow(v, 1.0 / (double)p);
}

/* w_eff = min(w, n-1): the window {k : |k-i| <= w} saturates (reading c7). */
static int clamp_w(int n, int w)
{
    if (w < 0) return 0;
    return w > n - 1 ? n - 1 : w;
}

/* ------------------------------------------------------------------------ */
/* Warping envelope, by definition (section "Computing Lower
 * Bounds on the DTW"): U(y)_i = max_k {y_k : |k-i| <= w},
 *                         L(y)_i = min_k {y_k : |k-i| <= w}, window clipped
 * to the series (reading c7).  O(nw), the "naive approach" of P:354-355. */
void oracle_envelope_naive(const double *y, int n, int w, double *U, double *L)
{
    for (int i = 0; i < n; ++i) {
        int lo = i - w < 0 ? 0 : i - w;
        int hi = i + w > n - 1 ? n - 1 : i + w;
        double mx = y[lo], mn = y[lo];
        for (int k = lo + 1; k <= hi; ++k) {
            if (y[k] > mx) mx = y[k];
            if (y[k] < mn) mn = y[k];
        }
        U[i] = mx;
        L[i] = mn;
    }
}

/* Algorithm 1 (section "Warping Envelopes"), streaming envelope
 * with monotone double-ended queues u (max) and l (min), CORRECTED per
 * reading c1: the printed algorithm emits U_{i-w} before inserting y_i,
 * never assigns U_1 when w = 0 and pops empty deques.  Here, following the
 * same structure: insert y_i (pop-then-test on the branch taken, strict
 * comparisons as printed at P:373-383), guard empty deques, expire the front
 * once it leaves the window, then emit index i-w.  The tail loop
 * expires then emits.  Returns the number of comparisons between data-point
 * values (P:356 claims at most 3n).  Cross-check only; the definition above
 * is the oracle's truth. */
long oracle_envelope_stream(const double *y, int n, int w, double *U, double *L)
{
    w = clamp_w(n, w);
    int *u = (int *)malloc(sizeof(int) * (size_t)(n + 1));
    int *l = (int *)malloc(sizeof(int) * (size_t)(n + 1));
    int uf = 0, ub = 0, lf = 0, lb = 0; /* [front, back) */
    long cmp = 0;
    u[ub++] = 0;
    l[lb++] = 0;
    if (w == 0) { U[0] = y[0]; L[0] = y[0]; }
    for (int i = 1; i < n; ++i) {
        ++cmp;
        if (y[i] > y[i - 1]) {
            --ub;                        /* pop u from back */
            while (ub > uf) {            /* P:375 (guarded) */
                ++cmp;
                if (y[i] > y[u[ub - 1]]) --ub; else break;
            }
        } else {
            --lb;                        /* pop l from back */
            while (lb > lf) {            /* P:380 (guarded) */
                ++cmp;
                if (y[i] < y[l[lb - 1]]) --lb; else break;
            }
        }
        u[ub++] = i;                     /* append i to u and l */
        l[lb++] = i;
        /* expire fronts that left the window [i-2w, i] */
        if (i - u[uf] > 2 * w) ++uf;
        if (i - l[lf] > 2 * w) ++lf;
        if (i >= w) {                    /* emit U_{i-w}, L_{i-w} */
            U[i - w] = y[u[uf]];
            L[i - w] = y[l[lf]];
        }
    }
    for (int i = n; i < n + w; ++i) {    /* tail loop P:391-399 */
        if (i - u[uf] > 2 * w) ++uf;
        if (i - l[lf] > 2 * w) ++lf;
        U[i - w] = y[u[uf]];
        L[i - w] = y[l[lf]];
    }
    free(u);
    free(l);
    return cmp;
}

/* ------------------------------------------------------------------------ */
/* Projection of x on y, Eq. (1) (section "LB_Keogh"):
 * H_i = U_i if x_i >= U_i;  L_i if x_i <= L_i;  x_i otherwise. */
void oracle_projection(const double *x, const double *U, const double *L, int n, double *H)
{
    for (int i = 0; i < n; ++i) {
        if (x[i] >= U[i]) H[i] = U[i];
        else if (x[i] <= L[i]) H[i] = L[i];
        else H[i] = x[i];
    }
}

/* ||x - H(x,y)||_p^p for finite p, or ||x - H||_inf for p = 0, given the
 * query envelope U, L ("LB_Keogh_p(x,y) = ||x - H(x,y)||_p"). */
double oracle_lb_keogh_pow(const double *x, const double *U, const double *L, int n, int p)
{
    double *H = (double *)malloc(sizeof(double) * (size_t)n);
    oracle_projection(x, U, L, n, H);
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        if (p == 0) { double a = fabs(x[i] - H[i]); if (a > s) s = a; }
        else s += powabs(x[i] - H[i], p);
    }
    free(H);
    return s;
}

/* LB_Keogh_p(x, y) rooted: envelope of y (definition), then P:463. */
double oracle_lb_keogh(const double *x, const double *y, int n, int w, int p)
{
    double *U = (double *)malloc(sizeof(double) * (size_t)n);
    double *L = (double *)malloc(sizeof(double) * (size_t)n);
    oracle_envelope_naive(y, n, w, U, L);
    double s = oracle_lb_keogh_pow(x, U, L, n, p);
    free(U);
    free(L);
    return root_p(s, p);
}

/* Piecewise-sum lower bound (section "Using a multidimensional
 * indexing structure"): with the cover C_j = [j*s, min((j+1)*s, n)) and
 * P(v)_j = sum_{i in C_j} v_i.  This fixed-length cover (intervals of s
 * samples, the LAST one SHORTER when s does not divide n) is the builder's
 * choice for the GPU pre-filter (reading c18), NOT the cover the
 * paper's experiments used: P:661-665 takes d intervals of floor(n/d) with
 * the last one LONGER (oracle_lb_piecewise_paper below).  Any disjoint cover
 * gives a valid bound, so both are lower bounds of LB_Keogh;
 * they coincide when s divides n and d = n/s.
 *   p = 1:  sum_j d(P(x)_j, [P(L)_j, P(U)_j])          (the paper)
 *   p = 2:  sum_j d(P(x)_j, [P(L)_j, P(U)_j])^2 / s    (reading c18: Cauchy-Schwarz
 *           per interval, sum_{C_j} d_i^2 >= (sum_{C_j} d_i)^2 / |C_j|, |C_j| <= s)
 * U, L: the query envelope.  Returns the p-th-power (unrooted) value. */
double oracle_lb_piecewise_pow(const double *x, const double *U, const double *L, int n, int s, int p)
{
    double total = 0.0;
    for (int j0 = 0; j0 < n; j0 += s) {
        int j1 = j0 + s < n ? j0 + s : n;
        double px = 0.0, pu = 0.0, pl = 0.0;
        for (int i = j0; i < j1; ++i) {
            px += x[i];
            pu += U[i];
            pl += L[i];
        }
        double d = 0.0; /* d(P(x)_j, [P(L)_j, P(U)_j]), P:123 point-to-set distance */
        if (px > pu) d = px - pu;
        else if (px < pl) d = pl - px;
        total += p == 1 ? d : d * d / (double)s;
    }
    return total;
}

double oracle_lb_piecewise(const double *x, const double *y, int n, int w, int s, int p)
{
    double *U = (double *)malloc(sizeof(double) * (size_t)n);
    double *L = (double *)malloc(sizeof(double) * (size_t)n);
    oracle_envelope_naive(y, n, w, U, L);
    double v = oracle_lb_piecewise_pow(x, U, L, n, s, p);
    free(U);
    free(L);
    return root_p(v, p);
}

/* The paper's own cover: d intervals C_j = [1+(j-1)floor(n/d),
 * j floor(n/d)] for j < d and C_d = [1+(d-1)floor(n/d), n] (1-based; the last
 * interval takes the remainder, so it is the LONGEST), requiring 1 <= d <= n.
 *   p = 1: sum_j d(P_d(x)_j, [P_d(L)_j, P_d(U)_j])
 *   p = 2: sum_j d(...)^2 / |C_j|  (reading c18, Cauchy-Schwarz per interval)
 * Returns the p-th-power (unrooted) value; NAN if d is outside [1, n]. */
double oracle_lb_piecewise_paper_pow(const double *x, const double *U, const double *L, int n, int d, int p)
{
    if (d < 1 || d > n) return NAN;
    const int len = n / d; /* floor(n/d) */
    double total = 0.0;
    for (int j = 0; j < d; ++j) {
        int j0 = j * len, j1 = (j == d - 1) ? n : (j + 1) * len; /* C_{j+1}, 0-based [j0, j1) */
        double px = 0.0, pu = 0.0, pl = 0.0;
        for (int i = j0; i < j1; ++i) {
            px += x[i];
            pu += U[i];
            pl += L[i];
        }
        double dd = 0.0;
        if (px > pu) dd = px - pu;
        else if (px < pl) dd = pl - px;
        total += p == 1 ? dd : dd * dd / (double)(j1 - j0);
    }
    return total;
}

double oracle_lb_piecewise_paper(const double *x, const double *y, int n, int w, int d, int p)
{
    double *U = (double *)malloc(sizeof(double) * (size_t)n);
    double *L = (double *)malloc(sizeof(double) * (size_t)n);
    oracle_envelope_naive(y, n, w, U, L);
    double v = oracle_lb_piecewise_paper_pow(x, U, L, n, d, p);
    free(U);
    free(L);
    return root_p(v, p);
}

/* LB_Improved_p(x,y)^p = LB_Keogh_p(x,y)^p + LB_Keogh_p(y, H(x,y))^p
 * (section "LB_Improved"), for finite p only (the corollary
 * P:552-555 is stated for 1 <= p < infinity).  Steps in the paper's order
 * (Fig. "Computation of LB_Improved" (a)-(f)):
 *   U,L = envelope(y); H = projection of x; beta1 = ||x-H||_p^p;
 *   U',L' = envelope(H); beta2 = sum_i d(y_i, [L'_i, U'_i])^p.
 * Returns the p-th power (unrooted) sum; U, L are the query envelope. */
double oracle_lb_improved_pow(const double *x, const double *y, const double *U, const double *L,
                              int n, int w, int p)
{
    double *H = (double *)malloc(sizeof(double) * (size_t)n);
    double *U2 = (double *)malloc(sizeof(double) * (size_t)n);
    double *L2 = (double *)malloc(sizeof(double) * (size_t)n);
    oracle_projection(x, U, L, n, H);
    double beta = 0.0;
    for (int i = 0; i < n; ++i) beta += powabs(x[i] - H[i], p);
    oracle_envelope_naive(H, n, w, U2, L2);
    for (int i = 0; i < n; ++i) {
        /* d(y_i, [L'_i, U'_i]) (P:123 point-to-set distance; Alg. 3) */
        if (y[i] > U2[i]) beta += powabs(y[i] - U2[i], p);
        else if (y[i] < L2[i]) beta += powabs(L2[i] - y[i], p);
    }
    free(H);
    free(U2);
    free(L2);
    return beta;
}

double oracle_lb_improved(const double *x, const double *y, int n, int w, int p)
{
    if (p < 1) return NAN; /* LB_Improved undefined for p = infinity */
    double *U = (double *)malloc(sizeof(double) * (size_t)n);
    double *L = (double *)malloc(sizeof(double) * (size_t)n);
    oracle_envelope_naive(y, n, w, U, L);
    double s = oracle_lb_improved_pow(x, y, U, L, n, w, p);
    free(U);
    free(L);
    return root_p(s, p);
}

/* ------------------------------------------------------------------------ */
/* Monotone banded DTW by the paper's suffix recursion (section
 * "Dynamic Time Warping"):
 *   q_{i,j} = 0                                   if both suffixes empty,
 *           = inf                                 if exactly one is empty
 *                                                 or |i-j| > w,
 *           = |x_i - y_j|^p + min(q_{i+1,j}, q_{i,j+1}, q_{i+1,j+1}) otherwise;
 * DTW_p(x,y)^p = q_{1,1}.  For p = infinity (p == 0 here), P:211-214:
 *   q_{i,j} = max(|x_i - y_j|, min(q_{i+1,j}, q_{i,j+1}, q_{i+1,j+1})).
 * Two rolling rows of the (n+1)x(n+1) table hold rows i and i+1 (storage
 * only; the recursion and its evaluation order are the paper's).
 * Returns q_{1,1} (the p-th power for finite p). */
double oracle_dtw_pow(const double *x, const double *y, int n, int w, int p)
{
    /* row index i = 0..n (n = empty suffix); column j = 0..n likewise */
    double *nxt = (double *)malloc(sizeof(double) * (size_t)(n + 1)); /* q_{i+1,*} */
    double *cur = (double *)malloc(sizeof(double) * (size_t)(n + 1)); /* q_{i,*}   */
    for (int j = 0; j <= n; ++j) nxt[j] = ORACLE_INF; /* i = n: x suffix empty */
    nxt[n] = 0.0;                                     /* both empty */
    for (int i = n - 1; i >= 0; --i) {
        cur[n] = ORACLE_INF; /* y suffix empty, x not */
        for (int j = n - 1; j >= 0; --j) {
            if (abs(i - j) > w) { cur[j] = ORACLE_INF; continue; }
            double m = nxt[j];
            if (cur[j + 1] < m) m = cur[j + 1];
            if (nxt[j + 1] < m) m = nxt[j + 1];
            if (p == 0) {
                double a = fabs(x[i] - y[j]);
                cur[j] = a > m ? a : m;
            } else {
                cur[j] = powabs(x[i] - y[j], p) + m;
            }
        }
        double *t = nxt; nxt = cur; cur = t;
    }
    double q11 = nxt[0];
    free(nxt);
    free(cur);
    return q11;
}

double oracle_dtw(const double *x, const double *y, int n, int w, int p)
{
    return root_p(oracle_dtw_pow(x, y, n, w, p), p);
}

/* ------------------------------------------------------------------------ */
/* k-NN bookkeeping: the result is the k smallest candidates under the
 * lexicographic key (distance, index) (readings c4, c14).  best_d/best_i hold
 * the current list sorted ascending; cnt = entries filled so far. */
static void knn_insert(double *best_d, int64_t *best_i, int k, int *cnt, double d, int64_t c)
{
    int m = *cnt;
    if (m == k) {
        if (d > best_d[k - 1] || (d == best_d[k - 1] && c > best_i[k - 1])) return;
        m = k - 1; /* drop the current k-th */
    }
    int pos = m;
    while (pos > 0 && (best_d[pos - 1] > d || (best_d[pos - 1] == d && best_i[pos - 1] > c))) {
        best_d[pos] = best_d[pos - 1];
        best_i[pos] = best_i[pos - 1];
        --pos;
    }
    best_d[pos] = d;
    best_i[pos] = c;
    *cnt = m + 1;
}

static void upcast(const float *src, int n, double *dst)
{
    for (int i = 0; i < n; ++i) dst[i] = (double)src[i];
}

/* Ground truth (section 8(c) of SURVEY / DESIGN "Oracle"): brute-force k-NN.
 * For each query y (rows q0..q1-1 of `queries`), DTW_p(y, x_c) for every
 * candidate c by the recursion above, and the k smallest by (DTW_p, c),
 * distances rooted.  Outputs are [Q][k] row-major; slots beyond N stay
 * (+inf, -1). */
void oracle_nn_brute(const float *queries, int64_t q0, int64_t q1, const float *db, int64_t N,
                     int n, int w, int p, int k, int64_t *out_idx, double *out_dist)
{
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    double *bd = (double *)malloc(sizeof(double) * (size_t)k);
    int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    for (int64_t q = q0; q < q1; ++q) {
        upcast(queries + q * n, n, y);
        int cnt = 0;
        for (int64_t c = 0; c < N; ++c) {
            upcast(db + c * n, n, x);
            knn_insert(bd, bi, k, &cnt, oracle_dtw_pow(x, y, n, w, p), c);
        }
        for (int r = 0; r < k; ++r) {
            out_idx[q * k + r] = r < cnt ? bi[r] : -1;
            out_dist[q * k + r] = r < cnt ? root_p(bd[r], p) : ORACLE_INF;
        }
    }
    free(y); free(x); free(bd); free(bi);
}

/* Counters of the sequential scan (taxonomy of SPEC S:450, reading c3):
 * [0] candidates seen, [1] pruned by LB_Keogh, [2] pruned by LB_Improved,
 * [3] DTW evaluations.  Invariant: [1] + [2] + [3] == [0]. */
enum { CNT_SEEN = 0, CNT_KEOGH = 1, CNT_IMPROVED = 2, CNT_DTW = 3 };

/* Second oracle: Algorithm 3 (section "LB_Improved"), the
 * LB_Improved-based nearest-neighbour scan, generalised to finite p and
 * k >= 1 (readings c5, c6): b is the current k-th best DTW_p^p (+inf until k
 * candidates have been evaluated); comparisons are in p-th-power space; a
 * candidate is discarded iff its bound exceeds b*(1+1e-9) (reading c3:
 * equality never prunes, and the 1e-9 absorbs fp64 rounding of a bound that
 * equals the DTW).  keogh_only != 0 skips the second pass = Algorithm 2
 * (P:498-527).  Candidates are scanned in index order. */
void oracle_nn_twopass(const float *queries, int64_t q0, int64_t q1, const float *db, int64_t N,
                       int n, int w, int p, int k, int keogh_only, int64_t *out_idx,
                       double *out_dist, int64_t *counters)
{
    const double margin = 1.0 + 1e-9;
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    double *xp = (double *)malloc(sizeof(double) * (size_t)n); /* x' of Alg. 3 */
    double *U = (double *)malloc(sizeof(double) * (size_t)n);
    double *L = (double *)malloc(sizeof(double) * (size_t)n);
    double *U2 = (double *)malloc(sizeof(double) * (size_t)n);
    double *L2 = (double *)malloc(sizeof(double) * (size_t)n);
    double *bd = (double *)malloc(sizeof(double) * (size_t)k);
    int64_t *bi = (int64_t *)malloc(sizeof(int64_t) * (size_t)k);
    for (int64_t q = q0; q < q1; ++q) {
        upcast(queries + q * n, n, y);
        oracle_envelope_naive(y, n, w, U, L);          /* Alg. 3 line "U,L <- envelope(y)" */
        int cnt = 0;                                   /* b <- inf */
        for (int64_t c = 0; c < N; ++c) {              /* for candidate x in S */
            upcast(db + c * n, n, x);
            counters[CNT_SEEN]++;
            double b = cnt < k ? ORACLE_INF : bd[k - 1];
            memcpy(xp, x, sizeof(double) * (size_t)n); /* copy x to x' */
            double beta = 0.0;
            for (int i = 0; i < n; ++i) {              /* first pass */
                if (x[i] > U[i]) { beta += powabs(x[i] - U[i], p); xp[i] = U[i]; }
                else if (x[i] < L[i]) { beta += powabs(L[i] - x[i], p); xp[i] = L[i]; }
            }
            if (beta > b * margin) { counters[CNT_KEOGH]++; continue; }
            if (!keogh_only) {
                oracle_envelope_naive(xp, n, w, U2, L2);
                for (int i = 0; i < n; ++i) {
                    if (y[i] > U2[i]) beta += powabs(y[i] - U2[i], p);
                    else if (y[i] < L2[i]) beta += powabs(L2[i] - y[i], p);
                }
                if (beta > b * margin) { counters[CNT_IMPROVED]++; continue; }
            }
            counters[CNT_DTW]++;
            double t = oracle_dtw_pow(x, y, n, w, p);
            knn_insert(bd, bi, k, &cnt, t, c);
        }
        for (int r = 0; r < k; ++r) {
            out_idx[q * k + r] = r < cnt ? bi[r] : -1;
            out_dist[q * k + r] = r < cnt ? root_p(bd[r], p) : ORACLE_INF;
        }
    }
    free(y); free(x); free(xp); free(U); free(L); free(U2); free(L2); free(bd); free(bi);
}

/* Order-independent prune counts against a FINAL threshold (SURVEY 8(c)
 * "Prune rates" row): for each query q with final k-th
 * distance tau_q (rooted), counts #{c : LB_Keogh^p > tau^p} and
 * #{c : LB_Keogh^p <= tau^p < LB_Improved^p}.  Pinned in
 * tests/test_oracle_pins.py::test_prune_counts_pinned against numpy bounds and
 * the Alg. 3 counter invariants (the paper's pruning curves are stripped,
 * P:767-856, so no printed value exists). */
void oracle_prune_counts(const float *queries, int64_t q0, int64_t q1, const float *db, int64_t N,
                         int n, int w, int p, const double *tau, int64_t *out_keogh,
                         int64_t *out_improved)
{
    double *y = (double *)malloc(sizeof(double) * (size_t)n);
    double *x = (double *)malloc(sizeof(double) * (size_t)n);
    double *U = (double *)malloc(sizeof(double) * (size_t)n);
    double *L = (double *)malloc(sizeof(double) * (size_t)n);
    for (int64_t q = q0; q < q1; ++q) {
        upcast(queries + q * n, n, y);
        oracle_envelope_naive(y, n, w, U, L);
        double tp = pow(tau[q], (double)p);
        int64_t ck = 0, ci = 0;
        for (int64_t c = 0; c < N; ++c) {
            upcast(db + c * n, n, x);
            double b1 = oracle_lb_keogh_pow(x, U, L, n, p);
            if (b1 > tp) { ++ck; continue; }
            if (oracle_lb_improved_pow(x, y, U, L, n, w, p) > tp) ++ci;
        }
        out_keogh[q] = ck;
        out_improved[q] = ci;
    }
    free(y); free(x); free(U); free(L);
}
