/*
 * oracle.c -- plain, slow, obviously-correct fp64 CPU oracle for the GVT hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_2009_01054_b200/csrc); the
 * product path never calls it.
 *
 * Every function cites the passage of the paper (reference/PAPER.md, "Generalized
 * vec trick for fast learning of pairwise kernel models") or of SPEC.md it follows.
 * Readings of garbled/ambiguous passages are the ones listed in DESIGN.md ("Readings").
 *
 * Conventions: matrices are dense row-major double; object ids are int32 global ids;
 * a pair sample is two parallel id arrays (first, second).  Heterogeneous data: first
 * ids index the drug table (size m, Gram D), second ids the target table (size q,
 * Gram T).  Homogeneous data (T == NULL): both ids index the one table of size m
 * (Table 4a), and every TARGET factor resolves to D.
 *
 * Pinning (see tests/test_oracle_pins.py and DESIGN.md "Oracle pins"):
 *   oracle_gram            -- closed forms, SPEC worked values, PSD, diag exactly 1
 *   oracle_kernel_value    -- SPEC worked values, Table 4a feature-map inner products,
 *                             Poly2D = Linear^2, MLPK = Ranking^2, swap invariants
 *   oracle_explicit_*      -- the definition u = K a (PAPER.md:765-770 approach 1)
 *   oracle_kernel_terms    -- Corollary table, MLPK proof 736-747;
 *                             term assembly == Table 4b entrywise
 *   oracle_term_gvt        -- == explicit on tiny random instances (Theorem 1 is exact)
 *                             and == Roth's vec trick D*A*T^T on complete grids
 *   oracle_cg              -- == dense direct solve; c*I system; A-norm error monotone
 *   oracle_sort_plan       -- brute-force stable sort (numpy) on random inputs
 *   oracle_relabel         -- SPEC.md:55-57 examples; numpy.unique first-occurrence indices;
 *                             unique[compact] == ids; idempotent on compact input
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

enum { OR_LINEAR = 0, OR_POLY2D, OR_GAUSSIAN, OR_KRONECKER, OR_SYMMETRIC,
       OR_ANTISYMMETRIC, OR_RANKING, OR_MLPK, OR_CARTESIAN, OR_NKERNELS };
enum { OR_BASE_LINEAR = 0, OR_BASE_GAUSSIAN = 1, OR_BASE_POLY = 2, OR_BASE_TANIMOTO = 3 };
enum { F_DRUG = 0, F_TARGET = 1, F_ONES = 2, F_IDENTITY = 3 };
enum { SEL_FIRST = 0, SEL_SECOND = 1 };

enum { OR_OK = 0, OR_E_DIM = 1, OR_E_INDEX = 2, OR_E_HOMOGENEOUS = 3, OR_E_KERNEL = 4,
       OR_E_PARAM = 5, OR_E_BREAKDOWN = 6, OR_E_OOM = 7 };

typedef struct {
    double coef;
    int32_t left, right;                    /* factor kinds F_* */
    int32_t row_sel_left, row_sel_right;    /* selectors applied to the OUT pair */
    int32_t col_sel_left, col_sel_right;    /* selectors applied to the IN pair  */
} oracle_term;

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the OpenMP loops (timing legs only: each output is owned by one thread and
 * summed in a fixed order, so the results do not depend on it). */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* ------------------------------------------------------------------ O1 base Grams
 * PAPER.md:824-825 (section 5.2): linear k(x,y) = <x,y>; Gaussian
 * k(x,y) = exp(-gamma ||x-y||^2) with the SQUARED norm (reading S4).  The
 * polynomial base kernel (gamma<x,y> + coef0)^degree is not in the paper; it is
 * named only by BASELINE.json's north star (reading S5b in DESIGN.md).
 * K[i][j] = k(X_i, Y_j) for i < m, j < m2; the Gaussian uses direct differences so
 * that k(x,x) = exp(0) = 1 exactly.
 * Tanimoto on binary feature vectors (section 5.1 Heterodimers; Merget's drug
 * kernels): "the ratio of bits set to 1 in both vs. bits set to 1 in either",
 * k(v, w) = sum_i min(v_i, w_i) / sum_i max(v_i, w_i); two all-zero vectors give 1 (SPEC.md
 * tanimoto_base_kernel convention, reading T1); an entry other than 0 or 1 is OR_E_PARAM. */
int oracle_gram(int base, const double *X, int64_t m, const double *Y, int64_t m2,
                int64_t dim, double gamma, double coef0, int degree, double *K) {
    if (m < 0 || m2 < 0 || dim < 0) return OR_E_DIM;
    if (base == OR_BASE_GAUSSIAN && !(gamma > 0)) return OR_E_PARAM;
    if (base == OR_BASE_POLY && degree < 0) return OR_E_PARAM;
    if (base < 0 || base > 3) return OR_E_PARAM;
    if (base == OR_BASE_TANIMOTO) {
        for (int64_t i = 0; i < m * dim; i++) if (X[i] != 0.0 && X[i] != 1.0) return OR_E_PARAM;
        for (int64_t i = 0; i < m2 * dim; i++) if (Y[i] != 0.0 && Y[i] != 1.0) return OR_E_PARAM;
    }
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++) {
        for (int64_t j = 0; j < m2; j++) {
            const double *x = X + i * dim, *y = Y + j * dim;
            double acc = 0.0;
            if (base == OR_BASE_GAUSSIAN) {
                for (int64_t k = 0; k < dim; k++) { double df = x[k] - y[k]; acc += df * df; }
                K[i * m2 + j] = exp(-gamma * acc);
            } else if (base == OR_BASE_TANIMOTO) {
                double mx = 0.0;
                for (int64_t k = 0; k < dim; k++) {
                    acc += x[k] < y[k] ? x[k] : y[k];
                    mx += x[k] > y[k] ? x[k] : y[k];
                }
                K[i * m2 + j] = mx > 0.0 ? acc / mx : 1.0;
            } else {
                for (int64_t k = 0; k < dim; k++) acc += x[k] * y[k];
                if (base == OR_BASE_LINEAR) K[i * m2 + j] = acc;
                else K[i * m2 + j] = pow(gamma * acc + coef0, (double)degree);
            }
        }
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ O2 kernel values
 * Table 4b, written out literally.  Out pair (d,t) [or (d,d')],
 * in pair (db,tb) [or (db,db')].  Readings: Gaussian pairwise kernel = product of
 * Gaussian base Grams; anti-symmetric sign per Table 4b
 * i.e. (I-P)(D (x) D) (S3); Cartesian delta over global ids (S19). */
static inline double Dv(const double *D, int64_t m, int32_t a, int32_t b) { return D[(int64_t)a * m + b]; }

/* Table 4b with every base-kernel lookup written as G[out element][in element]: D / T are
 * row-major with leading dimensions ldd / ldt (square Grams over global ids: ldd = m,
 * ldt = q; rectangular cross-Grams of novel objects, O9: ldd = m_in, ldt = q_in). */
static double kernel_value_ld(int kernel, const double *D, int64_t ldd, const double *T, int64_t ldt,
                              int32_t d, int32_t t, int32_t db, int32_t tb) {
    const double *TT = T ? T : D;
    int64_t qq = T ? ldt : ldd;
    int64_t m = ldd;
    switch (kernel) {
    case OR_LINEAR:   return Dv(D, m, d, db) + Dv(TT, qq, t, tb);
    case OR_POLY2D: { double s = Dv(D, m, d, db) + Dv(TT, qq, t, tb); return s * s; }
    case OR_GAUSSIAN:
    case OR_KRONECKER: return Dv(D, m, d, db) * Dv(TT, qq, t, tb);
    case OR_SYMMETRIC:
        return Dv(D, m, d, db) * Dv(D, m, t, tb) + Dv(D, m, d, tb) * Dv(D, m, t, db);
    case OR_ANTISYMMETRIC:
        return Dv(D, m, d, db) * Dv(D, m, t, tb) - Dv(D, m, d, tb) * Dv(D, m, t, db);
    case OR_RANKING:
        return Dv(D, m, d, db) - Dv(D, m, d, tb) - Dv(D, m, t, db) + Dv(D, m, t, tb);
    case OR_MLPK: {
        double r = Dv(D, m, d, db) - Dv(D, m, d, tb) - Dv(D, m, t, db) + Dv(D, m, t, tb);
        return r * r;
    }
    case OR_CARTESIAN:
        return Dv(D, m, d, db) * (t == tb ? 1.0 : 0.0) + (d == db ? 1.0 : 0.0) * Dv(TT, qq, t, tb);
    default: return NAN;
    }
}

double oracle_kernel_value(int kernel, const double *D, int64_t m, const double *T, int64_t q,
                           int32_t d, int32_t t, int32_t db, int32_t tb) {
    return kernel_value_ld(kernel, D, m, T, q, d, t, db, tb);
}

static int is_homogeneous_kernel(int kernel) {
    return kernel == OR_SYMMETRIC || kernel == OR_ANTISYMMETRIC || kernel == OR_RANKING || kernel == OR_MLPK;
}

static int check_ids(const int32_t *ids, int64_t n, int64_t bound) {
    for (int64_t i = 0; i < n; i++) if (ids[i] < 0 || ids[i] >= bound) return 0;
    return 1;
}

static int check_sample(const double *T, int64_t m, int64_t q, const int32_t *f, const int32_t *s, int64_t n) {
    int64_t qq = T ? q : m;
    if (n < 0) return OR_E_DIM;
    if (!check_ids(f, n, m) || !check_ids(s, n, qq)) return OR_E_INDEX;
    return OR_OK;
}

/* ------------------------------------------------------------------ O3 explicit K
 * The definition: K_{i,j} = k(out_i, in_j) (PAPER.md:275-281, 751-753
 * "K = R(d_bar,t_bar) K^kernel R(d,t)^T"), materialised n_out x n_in. */
int oracle_explicit_matrix(int kernel, const double *D, int64_t m, const double *T, int64_t q,
                           const int32_t *of, const int32_t *os, int64_t n_out,
                           const int32_t *inf, const int32_t *ins, int64_t n_in, double *K) {
    if (kernel < 0 || kernel >= OR_NKERNELS) return OR_E_KERNEL;
    if (is_homogeneous_kernel(kernel) && T) return OR_E_HOMOGENEOUS;
    int rc;
    if ((rc = check_sample(T, m, q, of, os, n_out)) || (rc = check_sample(T, m, q, inf, ins, n_in))) return rc;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_out; i++)
        for (int64_t j = 0; j < n_in; j++)
            K[i * n_in + j] = oracle_kernel_value(kernel, D, m, T, q, of[i], os[i], inf[j], ins[j]);
    return OR_OK;
}

/* "Use the standard matrix vector product with the kernel matrix: u <- K a"
 * (approach 1), row by row without storing K: u_i = sum_j
 * k(out_i, in_j) a_j, ascending j.  O(n_out * n_in). */
int oracle_explicit_matvec(int kernel, const double *D, int64_t m, const double *T, int64_t q,
                           const int32_t *of, const int32_t *os, int64_t n_out,
                           const int32_t *inf, const int32_t *ins, int64_t n_in,
                           const double *a, double *u) {
    if (kernel < 0 || kernel >= OR_NKERNELS) return OR_E_KERNEL;
    if (is_homogeneous_kernel(kernel) && T) return OR_E_HOMOGENEOUS;
    int rc;
    if ((rc = check_sample(T, m, q, of, os, n_out)) || (rc = check_sample(T, m, q, inf, ins, n_in))) return rc;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n_out; i++) {
        double acc = 0.0;
        for (int64_t j = 0; j < n_in; j++)
            acc += oracle_kernel_value(kernel, D, m, T, q, of[i], os[i], inf[j], ins[j]) * a[j];
        u[i] = acc;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ decompose
 * Corollary with the indexing rules R(d,t)P = R(t,d),
 * R(d,t)Q = R(d,d): a left-side P swaps the ROW selectors, a
 * left-side Q duplicates the first row selector, right-side P^T/Q^T act on the column
 * selectors.  A term's value for out pair o and in pair i is
 *     coef * L[row_sel_left(o), col_sel_left(i)] * R[row_sel_right(o), col_sel_right(i)].
 * Anti-symmetric uses (I-P) (reading S3, Table 4b); MLPK is the 10-term
 * expansion of the proof (reading S22), coefficients
 * (+1,+1,+1,+1,+2,+2,-2,-2,-2,-2) in the proof's order. */
static oracle_term mk(double c, int l, int r, int rl, int rr, int cl, int cr) {
    oracle_term t; t.coef = c; t.left = l; t.right = r;
    t.row_sel_left = rl; t.row_sel_right = rr; t.col_sel_left = cl; t.col_sel_right = cr;
    return t;
}

int oracle_kernel_terms(int kernel, oracle_term *out, int *n_terms) {
    const int F = SEL_FIRST, S = SEL_SECOND;
    int n = 0;
    switch (kernel) {
    case OR_LINEAR:       /* D (x) 1 + 1 (x) T */
        out[n++] = mk(1, F_DRUG, F_ONES, F, S, F, S);
        out[n++] = mk(1, F_ONES, F_TARGET, F, S, F, S);
        break;
    case OR_POLY2D:       /* Q(D(x)D)Q^T + 2 D(x)T + PQ(T(x)T)Q^T P */
        out[n++] = mk(1, F_DRUG, F_DRUG, F, F, F, F);
        out[n++] = mk(2, F_DRUG, F_TARGET, F, S, F, S);
        out[n++] = mk(1, F_TARGET, F_TARGET, S, S, S, S);
        break;
    case OR_GAUSSIAN:     /* special case of Kronecker */
    case OR_KRONECKER:    /* D (x) T */
        out[n++] = mk(1, F_DRUG, F_TARGET, F, S, F, S);
        break;
    case OR_CARTESIAN:    /* D (x) I + I (x) T */
        out[n++] = mk(1, F_DRUG, F_IDENTITY, F, S, F, S);
        out[n++] = mk(1, F_IDENTITY, F_TARGET, F, S, F, S);
        break;
    case OR_SYMMETRIC:    /* (P + I)(D (x) D) */
        out[n++] = mk(1, F_DRUG, F_DRUG, F, S, F, S);
        out[n++] = mk(1, F_DRUG, F_DRUG, S, F, F, S);
        break;
    case OR_ANTISYMMETRIC: /* (I - P)(D (x) D) */
        out[n++] = mk(1, F_DRUG, F_DRUG, F, S, F, S);
        out[n++] = mk(-1, F_DRUG, F_DRUG, S, F, F, S);
        break;
    case OR_RANKING:      /* (I-P)(D (x) 1)(I-P) = D(x)1 - P(D(x)1) - (D(x)1)P + P(D(x)1)P */
        out[n++] = mk(1, F_DRUG, F_ONES, F, S, F, S);
        out[n++] = mk(-1, F_DRUG, F_ONES, S, F, F, S);
        out[n++] = mk(-1, F_DRUG, F_ONES, F, S, S, F);
        out[n++] = mk(1, F_DRUG, F_ONES, S, F, S, F);
        break;
    case OR_MLPK:         /* proof expansion */
        out[n++] = mk(1, F_DRUG, F_DRUG, F, F, F, F);   /* Q(D(x)D)Q^T        */
        out[n++] = mk(1, F_DRUG, F_DRUG, S, S, F, F);   /* PQ(D(x)D)Q^T       */
        out[n++] = mk(1, F_DRUG, F_DRUG, F, F, S, S);   /* Q(D(x)D)Q^T P      */
        out[n++] = mk(1, F_DRUG, F_DRUG, S, S, S, S);   /* PQ(D(x)D)Q^T P     */
        out[n++] = mk(2, F_DRUG, F_DRUG, F, S, F, S);   /* 2 (D(x)D)          */
        out[n++] = mk(2, F_DRUG, F_DRUG, S, F, F, S);   /* 2 P(D(x)D)         */
        out[n++] = mk(-2, F_DRUG, F_DRUG, F, F, F, S);  /* -2 Q(D(x)D)        */
        out[n++] = mk(-2, F_DRUG, F_DRUG, S, S, F, S);  /* -2 PQ(D(x)D)       */
        out[n++] = mk(-2, F_DRUG, F_DRUG, F, S, F, F);  /* -2 (D(x)D)Q^T      */
        out[n++] = mk(-2, F_DRUG, F_DRUG, F, S, S, S);  /* -2 (D(x)D)Q^T P    */
        break;
    default:
        return OR_E_KERNEL;
    }
    *n_terms = n;
    return OR_OK;
}

/* ------------------------------------------------------------------ O4 per-term GVT
 * Theorem 1 with the two-stage algorithm of SPEC.md:111-117:
 *  variant 1: S[t][h] = sum_{j : cl(in_j) = h} R[t, cr(in_j)] a_j          (ascending j)
 *             u_i   += coef * sum_h L[rl(out_i), h] * S[rr(out_i)][h]     (ascending h)
 *  variant 2: W[d][h'] = sum_{j : cr(in_j) = h'} L[d, cl(in_j)] a_j
 *             u_i   += coef * sum_h' R[rr(out_i), h'] * W[rl(out_i)][h']
 * S is formed only for the rows t that occur in the out sample and the columns h that
 * occur in the in sample (Table 1's q_bar, m: "unique ... in the sample"), so the cost
 * is q_bar*n + m*n_bar (variant 1) exactly as the theorem states; *op_count receives
 * the number of multiply-adds performed.  Skipped columns are
 * all-zero, so restricting h does not change any sum.
 * Factor values: DRUG -> D, TARGET -> T (D when homogeneous), ONES -> 1,
 * IDENTITY -> delta over global ids (reading S19, S28). */
typedef struct { int kind; const double *M; int64_t ld; } factor_t;

static inline double fval(const factor_t *f, int32_t r, int32_t c) {
    switch (f->kind) {
    case F_ONES: return 1.0;
    case F_IDENTITY: return r == c ? 1.0 : 0.0;
    default: return f->M[(int64_t)r * f->ld + c];
    }
}

static inline int32_t sel(int s, const int32_t *f, const int32_t *sc, int64_t i) {
    return s == SEL_FIRST ? f[i] : sc[i];
}

static int64_t dom(int s, int homogeneous, int64_t m, int64_t q) {
    return (s == SEL_FIRST || homogeneous) ? m : q;
}

static int term_factors(const oracle_term *tm, const double *D, int64_t m, const double *T, int64_t q,
                        factor_t *L, factor_t *R) {
    int hom = (T == NULL);
    const factor_t *dummy = 0; (void)dummy;
    factor_t *fs[2] = {L, R};
    int kinds[2] = {tm->left, tm->right};
    int rs[2] = {tm->row_sel_left, tm->row_sel_right};
    int cs[2] = {tm->col_sel_left, tm->col_sel_right};
    for (int k = 0; k < 2; k++) {
        if (kinds[k] < 0 || kinds[k] > 3) return OR_E_KERNEL;
        if (rs[k] < 0 || rs[k] > 1 || cs[k] < 0 || cs[k] > 1) return OR_E_KERNEL;
        fs[k]->kind = kinds[k];
        if (kinds[k] == F_DRUG) {
            /* a drug Gram may only be indexed by drug ids */
            if (!hom && (rs[k] != SEL_FIRST || cs[k] != SEL_FIRST)) return OR_E_HOMOGENEOUS;
            fs[k]->M = D; fs[k]->ld = m;
        } else if (kinds[k] == F_TARGET) {
            if (!hom && (rs[k] != SEL_SECOND || cs[k] != SEL_SECOND)) return OR_E_HOMOGENEOUS;
            fs[k]->M = hom ? D : T; fs[k]->ld = hom ? m : q;
        } else if (kinds[k] == F_IDENTITY) {
            if (!hom && rs[k] != cs[k]) return OR_E_HOMOGENEOUS;
            fs[k]->M = NULL; fs[k]->ld = 0;
        } else { fs[k]->M = NULL; fs[k]->ld = 0; }
    }
    return OR_OK;
}

int oracle_term_gvt(const oracle_term *tm, const double *D, int64_t m, const double *T, int64_t q,
                    const int32_t *of, const int32_t *os, int64_t n_out,
                    const int32_t *inf, const int32_t *ins, int64_t n_in,
                    const double *a, int variant, double *u, int64_t *op_count) {
    int hom = (T == NULL);
    factor_t L, R;
    int rc = term_factors(tm, D, m, T, q, &L, &R);
    if (rc) return rc;
    if ((rc = check_sample(T, m, q, of, os, n_out)) || (rc = check_sample(T, m, q, inf, ins, n_in))) return rc;
    /* variant 2 is variant 1 with the roles of the two factors (and selectors) swapped */
    int rl = tm->row_sel_left, rr = tm->row_sel_right, cl = tm->col_sel_left, cr = tm->col_sel_right;
    factor_t A = L, B = R;
    if (variant == 2) { A = R; B = L; int x; x = rl; rl = rr; rr = x; x = cl; cl = cr; cr = x; }
    else if (variant != 1) return OR_E_PARAM;
    /* stage 1 over rows t in out-sample(rr), columns h in in-sample(cl) */
    int64_t nrow = dom(rr, hom, m, q), ncol = dom(cl, hom, m, q);
    int64_t *rowmap = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nrow > 0 ? nrow : 1));
    int64_t *colmap = (int64_t *)malloc(sizeof(int64_t) * (size_t)(ncol > 0 ? ncol : 1));
    if (!rowmap || !colmap) { free(rowmap); free(colmap); return OR_E_OOM; }
    for (int64_t t = 0; t < nrow; t++) rowmap[t] = -1;
    for (int64_t h = 0; h < ncol; h++) colmap[h] = -1;
    for (int64_t i = 0; i < n_out; i++) rowmap[sel(rr, of, os, i)] = 0;
    for (int64_t j = 0; j < n_in; j++) colmap[sel(cl, inf, ins, j)] = 0;
    int64_t nr = 0, nc = 0;
    for (int64_t t = 0; t < nrow; t++) if (rowmap[t] == 0) rowmap[t] = nr++;
    int32_t *cols = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ncol > 0 ? ncol : 1));
    int32_t *rows = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nrow > 0 ? nrow : 1));
    for (int64_t h = 0; h < ncol; h++) if (colmap[h] == 0) { cols[nc] = (int32_t)h; colmap[h] = nc++; }
    for (int64_t t = 0; t < nrow; t++) if (rowmap[t] >= 0) rows[rowmap[t]] = (int32_t)t;
    double *S = (double *)calloc((size_t)(nr * nc > 0 ? nr * nc : 1), sizeof(double));
    if (!S || !cols || !rows) { free(S); free(cols); free(rows); free(rowmap); free(colmap); return OR_E_OOM; }
    /* stage 1: blocks of 64 rows; each block streams the in-sample once in ascending j */
    const int64_t BLK = 64;
    #pragma omp parallel for schedule(dynamic, 1)
    for (int64_t t0 = 0; t0 < nr; t0 += BLK) {
        int64_t t1 = t0 + BLK < nr ? t0 + BLK : nr;
        for (int64_t j = 0; j < n_in; j++) {
            int64_t hc = colmap[sel(cl, inf, ins, j)];
            int32_t c = sel(cr, inf, ins, j);
            double aj = a[j];
            for (int64_t tt = t0; tt < t1; tt++)
                S[tt * nc + hc] += fval(&B, rows[tt], c) * aj;
        }
    }
    /* stage 2: each output owned by one thread, ascending h */
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_out; i++) {
        int32_t r = sel(rl, of, os, i);
        const double *Srow = S + rowmap[sel(rr, of, os, i)] * nc;
        double acc = 0.0;
        for (int64_t hc = 0; hc < nc; hc++) acc += fval(&A, r, cols[hc]) * Srow[hc];
        u[i] += tm->coef * acc;
    }
    if (op_count) *op_count += nr * n_in + nc * n_out;
    free(S); free(cols); free(rows); free(rowmap); free(colmap);
    return OR_OK;
}

/* Cost of the two variants (Theorem 1 bound) for a term over a
 * pair of samples, counted over the unique ids actually present:
 * cost1 = q_out * n_in + m_in * n_out, cost2 = m_out * n_in + q_in * n_out. */
static int64_t count_unique(int s, int hom, int64_t m, int64_t q, const int32_t *f, const int32_t *sc, int64_t n) {
    int64_t d = dom(s, hom, m, q), cnt = 0;
    char *seen = (char *)calloc((size_t)(d > 0 ? d : 1), 1);
    for (int64_t i = 0; i < n; i++) { int32_t v = sel(s, f, sc, i); if (!seen[v]) { seen[v] = 1; cnt++; } }
    free(seen);
    return cnt;
}

int oracle_term_cost(const oracle_term *tm, int64_t m, int64_t q, int homogeneous,
                     const int32_t *of, const int32_t *os, int64_t n_out,
                     const int32_t *inf, const int32_t *ins, int64_t n_in, int64_t *cost1, int64_t *cost2) {
    int64_t q_out = count_unique(tm->row_sel_right, homogeneous, m, q, of, os, n_out);
    int64_t m_out = count_unique(tm->row_sel_left, homogeneous, m, q, of, os, n_out);
    int64_t m_in = count_unique(tm->col_sel_left, homogeneous, m, q, inf, ins, n_in);
    int64_t q_in = count_unique(tm->col_sel_right, homogeneous, m, q, inf, ins, n_in);
    *cost1 = q_out * n_in + m_in * n_out;
    *cost2 = m_out * n_in + q_in * n_out;
    return OR_OK;
}

/* Sum of per-term GVTs in list order (Corollary: "Their products with vectors can be
 * computed with GVT").  variant 0 = auto (smaller
 * cost, ties -> 1, reading S2). */
int oracle_gvt_matvec(const oracle_term *terms, int n_terms, const double *D, int64_t m,
                      const double *T, int64_t q,
                      const int32_t *of, const int32_t *os, int64_t n_out,
                      const int32_t *inf, const int32_t *ins, int64_t n_in,
                      const double *a, int variant, double *u, int64_t *op_count) {
    for (int64_t i = 0; i < n_out; i++) u[i] = 0.0;
    if (op_count) *op_count = 0;
    for (int k = 0; k < n_terms; k++) {
        int v = variant;
        if (v == 0) {
            int64_t c1, c2;
            oracle_term_cost(&terms[k], m, q, T == NULL, of, os, n_out, inf, ins, n_in, &c1, &c2);
            v = (c2 < c1) ? 2 : 1;
        }
        int rc = oracle_term_gvt(&terms[k], D, m, T, q, of, os, n_out, inf, ins, n_in, a, v, u, op_count);
        if (rc) return rc;
    }
    return OR_OK;
}

/* ------------------------------------------------------------------ O5 CG
 * Kernel ridge regression (K + lambda I) a = y (Eq. 1 at 316-320)
 * by textbook conjugate gradients (Hestenes-Stiefel), reading S12-S14:
 *   x = 0, r = y, p = r, rho = r.r
 *   for k = 1..K: Ap = K p + lambda p; alpha = rho / p.Ap; x += alpha p; r -= alpha Ap;
 *                 rho' = r.r; [residual mode: stop if sqrt(rho')/||y|| <= tol];
 *                 beta = rho'/rho; p = r + beta p; rho = rho'
 * Exact convergence (rho == 0) stops immediately (y = 0 gives a = 0, 0 iterations).
 * p.Ap <= 0 is a breakdown: the current iterate is returned with OR_E_BREAKDOWN.
 * The operator is the per-term GVT (use_explicit = 0) or the explicit definition
 * (use_explicit = 1, needs kernel >= 0).  relres_hist (nullable, max_iter+1 entries)
 * receives sqrt(rho_k)/||y|| for k = 0..iters; x_hist (nullable, (max_iter+1) x n)
 * receives the iterates x_0 .. x_iters (early stopping). */
int oracle_cg(int kernel, const oracle_term *terms, int n_terms, int use_explicit,
              const double *D, int64_t m, const double *T, int64_t q,
              const int32_t *f, const int32_t *s, int64_t n, const double *y,
              double lambda, int max_iter, double rel_tol,
              double *x, int *iters_out, double *relres_hist, double *x_hist) {
    if (!(lambda >= 0) || max_iter < 0 || rel_tol < 0) return OR_E_PARAM;
    double *r = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *p = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double *Ap = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!r || !p || !Ap) { free(r); free(p); free(Ap); return OR_E_OOM; }
    double rho = 0.0;
    for (int64_t i = 0; i < n; i++) { x[i] = 0.0; r[i] = y[i]; p[i] = y[i]; rho += y[i] * y[i]; }
    double ynorm = sqrt(rho);
    if (relres_hist) relres_hist[0] = ynorm > 0 ? 1.0 : 0.0;
    if (x_hist) for (int64_t i = 0; i < n; i++) x_hist[i] = 0.0;
    int k = 0, rc = OR_OK;
    while (k < max_iter && rho > 0.0) {
        if (use_explicit)
            rc = oracle_explicit_matvec(kernel, D, m, T, q, f, s, n, f, s, n, p, Ap);
        else
            rc = oracle_gvt_matvec(terms, n_terms, D, m, T, q, f, s, n, f, s, n, p, 1, Ap, NULL);
        if (rc) break;
        double pAp = 0.0;
        for (int64_t i = 0; i < n; i++) { Ap[i] += lambda * p[i]; pAp += p[i] * Ap[i]; }
        if (!(pAp > 0.0)) { rc = OR_E_BREAKDOWN; break; }
        double alpha = rho / pAp, rho1 = 0.0;
        for (int64_t i = 0; i < n; i++) { x[i] += alpha * p[i]; r[i] -= alpha * Ap[i]; rho1 += r[i] * r[i]; }
        k++;
        if (relres_hist) relres_hist[k] = sqrt(rho1) / ynorm;
        if (x_hist) for (int64_t i = 0; i < n; i++) x_hist[(int64_t)k * n + i] = x[i];
        if (rel_tol > 0 && sqrt(rho1) / ynorm <= rel_tol) { rho = rho1; break; }
        double beta = rho1 / rho;
        for (int64_t i = 0; i < n; i++) p[i] = r[i] + beta * p[i];
        rho = rho1;
    }
    if (iters_out) *iters_out = k;
    free(r); free(p); free(Ap);
    return rc;
}

/* ------------------------------------------------------------------ O5b MINRES
 * The paper's own solver: "This linear system can be solved iteratively, for example,
 * with the minimal residual method"; "We used the
 * scipy.sparse.linalg.minres method in the SciPy library".  This is the
 * unpreconditioned Lanczos-based minimal-residual iteration of Paige & Saunders as
 * SciPy states it, with zero shift and x0 = 0, step by step:
 *   r1 = r2 = y, beta1 = ||y||, beta = beta1, oldb = 0, dbar = 0, epsln = 0,
 *   phibar = beta1, cs = -1, sn = 0, w = w2 = 0
 *   for k = 1..K:
 *     v = r2 / beta;  z = (K + lambda I) v;  if k >= 2: z -= (beta / oldb) r1
 *     alfa = v.z;  z -= (alfa / beta) r2;  r1 = r2;  r2 = z
 *     oldb = beta;  beta = ||r2||
 *     oldeps = epsln;  delta = cs dbar + sn alfa;  gbar = sn dbar - cs alfa
 *     epsln = sn beta;  dbar = -cs beta
 *     gamma = max(sqrt(gbar^2 + beta^2), eps);  cs = gbar / gamma;  sn = beta / gamma
 *     phi = cs phibar;  phibar = sn phibar
 *     w1 = w2;  w2 = w;  w = (v - oldeps w1 - delta w2) * (1 / gamma);  x += phi w
 *   ||y - (K + lambda I) x_k|| = phibar_k (exact arithmetic), so phibar_k / ||y|| is the
 *   residual history; it is non-increasing (|sn| <= 1).
 * Stopping (readings M1-M2 in DESIGN.md): after max_iter iterations; when
 * phibar / ||y|| <= rel_tol (rel_tol > 0); or on Lanczos breakdown (SPEC.md minres_solve:
 * "beta underflow -> return current iterate flagged converged"), a normal exit, read as
 * beta_{k+1} <= 64 u ||T_k||_F with ||T_k||_F^2 = sum_i (alfa_i^2 + beta_{i+1}^2) the
 * Lanczos matrix's Frobenius norm (the operator's scale) and u the unit roundoff of the
 * vectors (2^-53 here).  y = 0 gives x = 0 after 0 iterations.
 * x_hist (nullable, (max_iter+1) x n) receives x_0 .. x_iters. */
static int apply_op(int kernel, const oracle_term *terms, int n_terms, int use_explicit,
                    const double *D, int64_t m, const double *T, int64_t q,
                    const int32_t *f, const int32_t *s, int64_t n, const double *v, double lambda, double *out) {
    int rc = use_explicit ? oracle_explicit_matvec(kernel, D, m, T, q, f, s, n, f, s, n, v, out)
                          : oracle_gvt_matvec(terms, n_terms, D, m, T, q, f, s, n, f, s, n, v, 1, out, NULL);
    if (rc) return rc;
    for (int64_t i = 0; i < n; i++) out[i] += lambda * v[i];
    return OR_OK;
}

int oracle_minres(int kernel, const oracle_term *terms, int n_terms, int use_explicit,
                  const double *D, int64_t m, const double *T, int64_t q,
                  const int32_t *f, const int32_t *s, int64_t n, const double *y,
                  double lambda, int max_iter, double rel_tol,
                  double *x, int *iters_out, double *relres_hist, double *x_hist) {
    if (!(lambda >= 0) || max_iter < 0 || rel_tol < 0) return OR_E_PARAM;
    size_t nb = sizeof(double) * (size_t)(n > 0 ? n : 1);
    double *r1 = (double *)malloc(nb), *r2 = (double *)malloc(nb), *v = (double *)malloc(nb);
    double *z = (double *)malloc(nb), *w = (double *)malloc(nb), *w2 = (double *)malloc(nb);
    if (!r1 || !r2 || !v || !z || !w || !w2) {
        free(r1); free(r2); free(v); free(z); free(w); free(w2);
        return OR_E_OOM;
    }
    double beta1 = 0.0;
    for (int64_t i = 0; i < n; i++) {
        x[i] = 0.0; r1[i] = y[i]; r2[i] = y[i]; w[i] = 0.0; w2[i] = 0.0; beta1 += y[i] * y[i];
    }
    beta1 = sqrt(beta1);
    if (relres_hist) relres_hist[0] = beta1 > 0 ? 1.0 : 0.0;
    if (x_hist) for (int64_t i = 0; i < n; i++) x_hist[i] = 0.0;
    double beta = beta1, oldb = 0.0, dbar = 0.0, epsln = 0.0, phibar = beta1, cs = -1.0, sn = 0.0;
    double tnorm2 = 0.0;
    const double eps = 2.220446049250313e-16;
    int k = 0, rc = OR_OK;
    while (k < max_iter && beta1 > 0.0) {
        for (int64_t i = 0; i < n; i++) v[i] = r2[i] / beta;
        rc = apply_op(kernel, terms, n_terms, use_explicit, D, m, T, q, f, s, n, v, lambda, z);
        if (rc) break;
        if (k >= 1) for (int64_t i = 0; i < n; i++) z[i] -= (beta / oldb) * r1[i];
        double alfa = 0.0;
        for (int64_t i = 0; i < n; i++) alfa += v[i] * z[i];
        double bnew = 0.0;
        for (int64_t i = 0; i < n; i++) {
            z[i] -= (alfa / beta) * r2[i];
            r1[i] = r2[i];
            r2[i] = z[i];
            bnew += r2[i] * r2[i];
        }
        oldb = beta;
        beta = sqrt(bnew);
        tnorm2 += alfa * alfa + beta * beta;
        double oldeps = epsln;
        double delta = cs * dbar + sn * alfa;
        double gbar = sn * dbar - cs * alfa;
        epsln = sn * beta;
        dbar = -cs * beta;
        double gamma = sqrt(gbar * gbar + beta * beta);
        if (gamma < eps) gamma = eps;
        cs = gbar / gamma;
        sn = beta / gamma;
        double phi = cs * phibar;
        phibar = sn * phibar;
        double denom = 1.0 / gamma;
        for (int64_t i = 0; i < n; i++) {
            double wn = (v[i] - oldeps * w2[i] - delta * w[i]) * denom;  /* w2 = w_{k-2}, w = w_{k-1} */
            w2[i] = w[i];
            w[i] = wn;
            x[i] += phi * wn;
        }
        k++;
        if (relres_hist) relres_hist[k] = phibar / beta1;
        if (x_hist) for (int64_t i = 0; i < n; i++) x_hist[(int64_t)k * n + i] = x[i];
        if (rel_tol > 0 && phibar / beta1 <= rel_tol) break;
        if (beta <= 64.0 * 1.1102230246251565e-16 * sqrt(tnorm2) || phibar == 0.0) break;  /* breakdown */
    }
    if (iters_out) *iters_out = k;
    free(r1); free(r2); free(v); free(z); free(w); free(w2);
    return rc;
}

/* ------------------------------------------------------------------ O8 AUC
 * Validation AUC for early stopping ("until the AUC stops increasing
 * in Z_validation"), by its definition as the Mann-Whitney statistic: the fraction of
 * (positive, negative) pairs ranked correctly, ties counting one half:
 *   AUC = (1 / (P N)) sum_{i: y_i > 0} sum_{j: y_j <= 0} ( [s_i > s_j] + [s_i == s_j] / 2 ).
 * Positive means label > 0 (reading A1: 0/1 and -1/+1 labels both work).  P = 0 or
 * N = 0 is undefined: OR_E_PARAM (SPEC.md fit_early_stopping: "degenerate validation
 * labels").  Brute force O(P N), exact integer counting of the 2x-scaled numerator. */
int oracle_auc(const double *labels, const double *scores, int64_t n, double *auc) {
    int64_t P = 0, N = 0;
    for (int64_t i = 0; i < n; i++) { if (labels[i] > 0) P++; else N++; }
    if (P == 0 || N == 0) return OR_E_PARAM;
    int64_t twice = 0;
    #pragma omp parallel for reduction(+ : twice) schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (!(labels[i] > 0)) continue;
        int64_t acc = 0;
        for (int64_t j = 0; j < n; j++) {
            if (labels[j] > 0) continue;
            if (scores[i] > scores[j]) acc += 2;
            else if (scores[i] == scores[j]) acc += 1;
        }
        twice += acc;
    }
    *auc = (double)twice / (2.0 * (double)P * (double)N);
    return OR_OK;
}

/* ------------------------------------------------------------------ O9 novel objects
 * Prediction for pairs whose objects were not in the training sample (Settings 2-4,
 * PAPER.md:162-169): the out pairs index the ROWS and the in pairs the COLUMNS of
 * rectangular cross-Grams, D_x[o][i] = k(test object o, training object i) (m_out x m_in)
 * and T_x (q_out x q_in); homogeneous kernels use one cross-Gram (T_x == NULL) for both pair
 * elements.  The Cartesian kernel's Identity factor compares objects across the two tables,
 * which have no common ids here: rejected (OR_E_KERNEL; reading N1).
 * oracle_explicit_rect_matvec: the definition u_i = sum_j k(out_i, in_j) a_j with Table 4b
 * evaluated on the cross-Grams (every lookup is [out element][in element]). */
static int check_rect(const int32_t *f, const int32_t *s, int64_t n, int64_t bf, int64_t bs) {
    if (n < 0) return OR_E_DIM;
    if (!check_ids(f, n, bf) || !check_ids(s, n, bs)) return OR_E_INDEX;
    return OR_OK;
}

int oracle_explicit_rect_matvec(int kernel, const double *Dx, int64_t m_out, int64_t m_in,
                                const double *Tx, int64_t q_out, int64_t q_in,
                                const int32_t *of, const int32_t *os, int64_t n_out,
                                const int32_t *inf, const int32_t *ins, int64_t n_in,
                                const double *a, double *u) {
    if (kernel < 0 || kernel >= OR_NKERNELS || kernel == OR_CARTESIAN) return OR_E_KERNEL;
    if (is_homogeneous_kernel(kernel) && Tx) return OR_E_HOMOGENEOUS;
    int64_t qo = Tx ? q_out : m_out, qi = Tx ? q_in : m_in;
    int rc;
    if ((rc = check_rect(of, os, n_out, m_out, qo)) || (rc = check_rect(inf, ins, n_in, m_in, qi))) return rc;
    #pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n_out; i++) {
        double acc = 0.0;
        for (int64_t j = 0; j < n_in; j++)
            acc += kernel_value_ld(kernel, Dx, m_in, Tx, q_in, of[i], os[i], inf[j], ins[j]) * a[j];
        u[i] = acc;
    }
    return OR_OK;
}

/* The GVT of one rectangular Kronecker product (SPEC.md:95-131 GvtProblem / gvt_cost /
 * gvt_matvec / gvt_op_count; Theorem 1):
 *   u[i] = sum_j A[of_i, if_j] B[os_i, is_j] a_j,   A: m_out x m_in,  B: q_out x q_in.
 * Variant 1: W[t][h] = sum_{j: if_j = h} B[t, is_j] a_j  (q_out x m_in, ascending j);
 *            u_i = sum_h A[of_i, h] W[os_i, h]           (ascending h).
 * Variant 2: the roles of A and B swapped:
 *            W'[d][g] = sum_{j: is_j = g} A[d, if_j] a_j (m_out x q_in);
 *            u_i = sum_g B[os_i, g] W'[of_i, g].
 * variant 0 = auto: the smaller of cost1 = q_out n_in + m_in n_out and
 * cost2 = m_out n_in + q_in n_out, ties -> variant 1 (reading S2); *op_count = the chosen
 * variant's cost and *variant_used the variant. */
int oracle_gvt_rect(const double *A, int64_t m_out, int64_t m_in, const double *B, int64_t q_out, int64_t q_in,
                    const int32_t *of, const int32_t *os, int64_t n_out,
                    const int32_t *inf, const int32_t *ins, int64_t n_in,
                    const double *a, int variant, double *u, int *variant_used, int64_t *op_count) {
    int rc;
    if ((rc = check_rect(of, os, n_out, m_out, q_out)) || (rc = check_rect(inf, ins, n_in, m_in, q_in))) return rc;
    if (variant < 0 || variant > 2) return OR_E_PARAM;
    int64_t c1 = q_out * n_in + m_in * n_out, c2 = m_out * n_in + q_in * n_out;
    int v = variant ? variant : (c2 < c1 ? 2 : 1);
    /* variant 2 = variant 1 on the transposed problem (B, A) with the pair elements swapped */
    const double *F2 = v == 1 ? A : B, *F1 = v == 1 ? B : A;
    int64_t r2 = v == 1 ? m_out : q_out, k2 = v == 1 ? m_in : q_in;   /* stage-2 factor dims */
    int64_t r1 = v == 1 ? q_out : m_out, k1 = v == 1 ? q_in : m_in;   /* stage-1 factor dims */
    const int32_t *o2 = v == 1 ? of : os, *o1 = v == 1 ? os : of;     /* out element per stage */
    const int32_t *i2 = v == 1 ? inf : ins, *i1 = v == 1 ? ins : inf; /* in element per stage */
    (void)r2;
    double *W = (double *)calloc((size_t)(r1 * k2 > 0 ? r1 * k2 : 1), sizeof(double));
    if (!W) return OR_E_OOM;
    #pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < r1; t++)
        for (int64_t j = 0; j < n_in; j++)
            W[t * k2 + i2[j]] += F1[t * k1 + i1[j]] * a[j];
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n_out; i++) {
        double acc = 0.0;
        for (int64_t h = 0; h < k2; h++) acc += F2[(int64_t)o2[i] * k2 + h] * W[(int64_t)o1[i] * k2 + h];
        u[i] = acc;
    }
    free(W);
    if (variant_used) *variant_used = v;
    if (op_count) *op_count = v == 1 ? c1 : c2;
    return OR_OK;
}

/* ------------------------------------------------------------------ O7b compact relabel
 * SPEC.md:49-57 relabel_compact (realizes Table 1's unique counts m, q, PAPER.md "the number
 * of unique drugs in the first sample"): compact[i] in [0, count); unique[compact[i]] =
 * ids[i]; unique in first-occurrence order; count = number of distinct values.  One pass
 * in index order with a seen-table over the id domain [0, bound).  unique holds up to
 * min(n, bound) entries. */
int oracle_relabel(const int32_t *ids, int64_t n, int64_t bound, int32_t *compact, int32_t *unique,
                   int64_t *count) {
    if (n < 0 || bound < 0) return OR_E_DIM;
    if (!check_ids(ids, n, bound)) return OR_E_INDEX;
    int64_t *seen = (int64_t *)malloc(sizeof(int64_t) * (size_t)(bound > 0 ? bound : 1));
    if (!seen) return OR_E_OOM;
    for (int64_t v = 0; v < bound; v++) seen[v] = -1;
    int64_t c = 0;
    for (int64_t i = 0; i < n; i++) {
        const int32_t v = ids[i];
        if (seen[v] < 0) {
            seen[v] = c;
            unique[c] = v;
            c++;
        }
        compact[i] = (int32_t)seen[v];
    }
    *count = c;
    free(seen);
    return OR_OK;
}

/* ------------------------------------------------------------------ O7 integer plumbing
 * Stable sort of pair indices by first id (mode 0) or by (first, second) (mode 1),
 * ties kept in ascending index order ("ascending j"), by counting sort;
 * row_ptr[h] = first position of first id h (m+1 entries). */
int oracle_sort_plan(const int32_t *f, const int32_t *s, int64_t n, int64_t m, int64_t q, int mode,
                     int32_t *perm, int64_t *row_ptr) {
    if (!check_ids(f, n, m) || !check_ids(s, n, q)) return OR_E_INDEX;
    int64_t nb = (mode == 1) ? m * q : m;
    int64_t *cnt = (int64_t *)calloc((size_t)(nb + 1), sizeof(int64_t));
    if (!cnt) return OR_E_OOM;
    for (int64_t j = 0; j < n; j++) {
        int64_t key = (mode == 1) ? (int64_t)f[j] * q + s[j] : f[j];
        cnt[key + 1]++;
    }
    for (int64_t b = 0; b < nb; b++) cnt[b + 1] += cnt[b];
    for (int64_t h = 0; h <= m; h++) row_ptr[h] = (mode == 1) ? cnt[h * q] : cnt[h];
    for (int64_t j = 0; j < n; j++) {
        int64_t key = (mode == 1) ? (int64_t)f[j] * q + s[j] : f[j];
        perm[cnt[key]++] = (int32_t)j;
    }
    free(cnt);
    return OR_OK;
}
