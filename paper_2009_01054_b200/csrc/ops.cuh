// ops.cuh -- launchers of the device kernels (internal).  Every launcher issues on
// ctx->stream and goes through GVT_LAUNCH (launch count + optional event timing).
#pragma once
#include <cuda_fp16.h>

#include "gvt_internal.cuh"

namespace gvt {

// A tensor-core GEMM operand: rows of a matrix split into (hi, lo) pieces, K-major with
// leading dimension ld.  prec 0 = fp16 pieces with per-row power-of-two scale (scale[r] =
// 1/s_r), prec 1 = tf32 pieces in fp32 containers (scale == nullptr).
// fp16 S of the fused dense path: one power-of-two scale per (S16_SCALE_ROWS-row block, 256-wide
// K chunk): scale_k[chunk * scale_k_ld + row / S16_SCALE_ROWS].  1 = per row (default); 128 = one
// stage-1 CTA's output block, so the stage-2 drain multiplies a chunk by ONE scalar (-DS16_SCALE_ROWS=128).
// Measured at C5 under the 1 kW cap (profiles/r02_ab_s16_block_scale.txt): the block scale takes 15 %
// fewer SM clocks per stage-2 launch but runs at 1.05-1.11 GHz instead of 1.29-1.31 GHz at the same
// power, so a 10-iteration fit takes 913 vs 836 ms: the per-row scale stays the default.
#ifndef S16_SCALE_ROWS
#define S16_SCALE_ROWS 1
#endif
static_assert(S16_SCALE_ROWS == 1 || S16_SCALE_ROWS == 128, "S scale blocks: per row or per 128-row CTA block");

struct Operand {
    int prec = 0;
    const void *hi = nullptr, *lo = nullptr;
    const float *scale = nullptr;
    int64_t ld = 0;
    // alternatively one scale per (row block, 256-wide K chunk): scale_k[chunk * scale_k_ld + row / S16_SCALE_ROWS]
    const float *scale_k = nullptr;
    int64_t scale_k_ld = 0;
};

// A factor (Gram / cross-Gram / materialised ones / identity) copied to a padded device
// buffer: n rows (out-domain) x cols (in-domain), leading dimension ld = round_up(cols, 32),
// padding zero; square Grams have cols = n.  For the dense tensor-core engine its split
// operand is attached on demand.  The sparse stage 1 reads the factor column-wise; a
// symmetric Gram is its own transpose (reading R1), a rectangular cross-Gram carries an
// explicit transposed copy pt (cols x ldt, ldt = round_up(n, 32)).
struct Factor {
    const float *p = nullptr;
    int64_t n = 0, ld = 0;
    int64_t cols = 0;
    const float *pt = nullptr;
    int64_t ldt = 0;
    Operand op;
    bool split = false;
    // the layout stage1_sparse reads: row `col` holds factor column col (contiguous over t)
    Factor colwise() const {
        Factor f = *this;
        if (pt) {
            f.p = pt;
            f.ld = ldt;
        }
        return f;
    }
};

// one entry kind of the pair matrix X (row selector, column selector, sign), see engine.cu
struct EntryKind {
    int row_sel, col_sel;
    float sign;
};
struct EntryKinds {
    int count;
    EntryKind k[4];
};

// X entries sorted by (row, col, entry index): CSR over rows
struct EntryPlan {
    int64_t nnz = 0, nrow = 0, ncol = 0;
    int32_t *row = nullptr, *col = nullptr, *src = nullptr;
    float *sign = nullptr;
    int64_t *row_ptr = nullptr;  // nrow + 1
    float *val = nullptr;        // per-iteration values sign * p[src]
    bool ident = false;          // src[k] == k and sign[k] == 1 for every entry (a sorted-order Kronecker fit)
};

// samples (r, c) of G = A X C^T sorted by r; result of sample k goes to dst[k]
struct SamplePlan {
    int64_t ns = 0;
    int32_t *r = nullptr, *c = nullptr, *dst = nullptr;
    // dense engine: samples bucketed by (r-tile, c-tile); tile_ptr over tiles
    int64_t n_rt = 0, n_ct = 0;
    int64_t *tile_ptr = nullptr;
    // small problems (pair tiles <= SM count): the non-empty CTA-pair tiles (mp * n_ct + n) and their
    // count, for the split-K sampled GEMM (-1: not computed)
    int32_t *pair_list = nullptr;
    int n_pairs = -1;
};

// ---- plumbing (plan.cu)
void pad_copy(gvt_ctx *c, const float *src, int64_t rows, int64_t cols, int64_t ld_src, float *dst, int64_t ld_dst,
              int64_t rows_pad);
void fill_ones(gvt_ctx *c, float *dst, int64_t rows, int64_t cols, int64_t ld, int identity);
// dst = src^T (cols x rows) into a zero-padded buffer: ld_dst >= rows, rows_pad_dst >= cols
void transpose_pad(gvt_ctx *c, const float *src, int64_t rows, int64_t cols, int64_t ld_src, float *dst,
                   int64_t ld_dst, int64_t rows_pad_dst);
void build_entry_plan(gvt_ctx *c, const char *tag, const int32_t *f, const int32_t *s, int64_t n,
                      const EntryKinds &kinds, int64_t nrow, int64_t ncol, EntryPlan &out);
// samples from an out-sample: kind 0: (sel(rs, i), sel(cs, i)) for i < n; plus (x,x) for x < n_diag
void build_sample_plan(gvt_ctx *c, const char *tag, const int32_t *f, const int32_t *s, int64_t n, int row_sel,
                       int col_sel, int64_t n_diag, int64_t nrow, SamplePlan &out);
// SPEC.md:49-57 compact relabel: compact (device, n); *unique_out = device array whose first
// `return value` entries are the distinct ids in first-occurrence order (workspace-owned)
int64_t relabel_compact(gvt_ctx *c, const int32_t *ids, int64_t n, int64_t bound, int32_t *compact,
                        const int32_t **unique_out);
void sort_plan_debug(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, int64_t m, int64_t q, int mode,
                     int32_t *perm, int64_t *row_ptr);
// fit-level reordering: perm = pair indices stably sorted by (first, second); gathers / scatter
void sort_pairs(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, int64_t m, int64_t q, int32_t *perm);
// objects used by a sample (Table 1's unique counts), numbered in ascending global id
struct UsedSet {
    int64_t m = 0;                  // object-table size
    int64_t k = 0;                  // number of used objects (host; after the read-back)
    const int64_t *k_dev = nullptr;  // the same, on the device
    const int32_t *used = nullptr;  // [m] 0/1
    const int32_t *pos = nullptr;   // [m] compact number of a used object
    const int32_t *ids = nullptr;   // [m] global id of compact number i (ascending; first k valid)
};
// marks the ids of `arrays` (counting ids outside [0, m) into counters[0]); asynchronous
UsedSet used_set_begin(gvt_ctx *c, const char *tag, int64_t m, const int32_t *const *arrays, const int64_t *lens,
                       int narr, unsigned long long *counters);
// counts the ids of a outside the set (or outside [0, m)) into *cnt; asynchronous
void count_unused_async(gvt_ctx *c, const UsedSet &u, const int32_t *a, int64_t n, unsigned long long *cnt);
void map_ids(gvt_ctx *c, const UsedSet &u, const int32_t *a, int64_t n, int32_t *out);
void sub_gram(gvt_ctx *c, const float *G, int64_t ld, const UsedSet &rows, const UsedSet &cols,
              float *Gs);  // Gs = G[rows.ids][cols.ids], ld cols.k
void gather_i32(gvt_ctx *c, const int32_t *x, const int32_t *perm, int64_t n, int32_t *y);
void gather_f32(gvt_ctx *c, const float *x, const int32_t *perm, int64_t n, float *y);
void scatter_f32(gvt_ctx *c, const float *x, const int32_t *perm, int64_t n, float *y);  // y[perm[k]] = x[k]
// validation helper: returns number of ids outside [0, bound) (device reduction, syncs)
int64_t count_out_of_range(gvt_ctx *c, const int32_t *ids, int64_t n, int64_t bound);

// ---- sparse engine (sparse.cu)
void entry_values(gvt_ctx *c, const EntryPlan &e, const float *p);
// S[t][h] = sum_{entries (h, col)} val C[col][t] (+ diag[row_lo + h] C[row_lo + h][t] if diag)
void stage1_sparse(gvt_ctx *c, const EntryPlan &e, const Factor &C, int64_t q_out, float *S, int64_t ldS,
                   const float *diag = nullptr, int64_t row_lo = 0);
void stage2_gather16(gvt_ctx *c, const SamplePlan &sp, const Factor &A, const __half *Sh, const __half *Sl,
                     int64_t ldS, const float *sk, int64_t skld, int64_t K, float coef, int accumulate, float *out);
void stage2_gather(gvt_ctx *c, const SamplePlan &sp, const Factor &A, const float *S, int64_t ldS, int64_t K,
                   float coef, int accumulate, float *out);
void segment_sum(gvt_ctx *c, const EntryPlan &e, float *b);  // b[h] = sum_row val (uses e.val)
// b[h] = sum_row sign p[src]; with r: p formed on the fly as r + (*beta_st) p (fused CG tail)
void segment_sum_gather(gvt_ctx *c, const EntryPlan &e, const float *p, float *b, const float *r = nullptr,
                        const double *beta_st = nullptr);
// symmetric: F is a square Gram (symmetric by definition, R1) -- the upper block triangle is read
void gemv(gvt_ctx *c, const Factor &F, const float *b, int square, float *y, bool symmetric = false);
// u[i] (+)= c1 * g1[sel(rs1,i)] + c2 * g2[sel(rs2,i)]   (g2 nullable)
void combine_gather(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, const float *g1, int rs1, float c1,
                    const float *g2, int rs2, float c2, int accumulate, float *u);
// MLPK: u[i] = buf[n + f_i] + buf[n + s_i] - 2 buf[i]
void combine_mlpk(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, const float *buf, float *u);
void cartesian(gvt_ctx *c, const int32_t *of, const int32_t *os, int64_t n_out, const EntryPlan &by_first,
               const EntryPlan &by_second, const Factor &D, const Factor &T, float *u);
void scale_copy(gvt_ctx *c, const float *x, float alpha, int64_t n, float *y);
void add_into(gvt_ctx *c, const float *x, int64_t n, float *y);  // y += x

// ---- dense tensor-core engine (dense_tc.cu)
bool tc_available(gvt_ctx *c);
int tc_precision_mode(gvt_ctx *c);
// view of columns [off, ...) of an operand (off a multiple of 32)
Operand operand_col_offset(const Operand &o, int64_t off);
// split a rows x cols fp32 matrix (leading dim ldx) into an operand with leading dim ld
Operand make_operand(gvt_ctx *c, const char *name, const float *x, int64_t rows, int64_t cols, int64_t ldx,
                     int64_t ld, int64_t rows_pad);
// X (rows_pad x ldX fp32, zeroed) <- rows [row_lo, row_lo + rows) of the pair matrix from the
// sorted entries k in [k0, k1) (duplicates summed in entry order)
void densify(gvt_ctx *c, const EntryPlan &e, int64_t k0, int64_t k1, int64_t row_lo, float *X, int64_t ldX,
             int64_t rows_pad);
// C (M x N, ldc) = A (M x K) * B^T (B: N x K), fp32-accurate; optional tf32 split of C
void gemm_nt_store(gvt_ctx *c, const Operand &A, const Operand &B, int64_t M, int64_t N, int64_t K, float *Cf,
                   int64_t ldc, float *Chi, float *Clo);
// fused fp16 path (3xFP16 + CTA pairs): can the stage-1 pieces below be used?
bool fused_f16(gvt_ctx *c, int64_t q_in);
// rows [row_lo, row_lo + rows) of the pair matrix built straight into an fp16 operand
// (values sign * p[src] summed per cell in entry order, one row scale per row)
// (launch = false: only the operand's buffers, for a build done elsewhere -- the fused CG tail)
Operand build_x16(gvt_ctx *c, const char *name, const EntryPlan &e, int64_t row_lo, int64_t rows, int64_t cols,
                  const float *p, const float *diag = nullptr, bool launch = true);
// X[r][row_lo + r] += diag[row_lo + r] for r < rows (fp32 X, leading dimension ldX)
void add_diag(gvt_ctx *c, float *X, int64_t ldX, const float *diag, int64_t row_lo, int64_t rows);
// C = A * B^T written as fp16 pieces (M rows x ldc) with one scale per (S16_SCALE_ROWS-row block,
// 256-col tile): sk[tile * sk_ld + row / S16_SCALE_ROWS] (sk_ld >= round_up(M, 256) / S16_SCALE_ROWS)
// kb_list / kb_off (device, nullable): per 256-row tile of B, its ascending non-zero K-blocks of
// 64 columns (at least one per tile): the other K-blocks are skipped (block-sparse B)
// tile_order (device, nullable): the persistent loop's pair-tile order (mp * num_n + n), e.g. the longest
// block-sparse K lists first; kb_min_chunks: the fewest 256-wide chunks of any tile's K list (with kb_list)
void gemm_nt_store16(gvt_ctx *c, const Operand &A, const Operand &B, int64_t M, int64_t N, int64_t K, __half *hi,
                     __half *lo, int64_t ldc, float *sk, int64_t sk_ld, const int32_t *kb_list = nullptr,
                     const int32_t *kb_off = nullptr, const int32_t *tile_order = nullptr, int kb_min_chunks = 0);
// non-zero (256-row tile, 64-column K-block) pairs of the pair-matrix rows [lo, lo + rows) from the
// sorted entries k in [k0, k1) (+ the diagonal when diag): host lists (off has ntiles + 1 entries)
void kblock_lists(gvt_ctx *c, const EntryPlan &e, int64_t k0, int64_t k1, int64_t lo, int64_t rows, int64_t cols,
                  bool diag, std::vector<int32_t> &list, std::vector<int32_t> &off);
// sampled: out[dst] (+)= coef * (A * B^T)[r, c] for the bucketed samples
// defer: a split-K GEMM leaves its parts for the caller's own combine (defer->part = nullptr when the
// GEMM wrote out itself)
struct SplitParts {
    int slot = 0;  // (in) which parts buffer: two deferred GEMMs of one matvec use different slots
    const float *part = nullptr;
    int split = 1;
    int64_t ns = 0;
    const int32_t *dst = nullptr;
    float coef = 1.f;
    int accumulate = 0;  // the deferred combine adds coef * (sum of parts) to out instead of storing it
};
// the CTA-pair GEMMs' rasterization group (pair-tile rows per group; GVT_GROUP_M or the default)
int gemm_group_m();
// the K-split the sampled GEMM will use for this plan and K (1: no parts)
int sampled_split_parts(gvt_ctx *c, const SamplePlan &sp, int64_t K);
void gemm_nt_sampled(gvt_ctx *c, const Operand &A, const Operand &B, int64_t M, int64_t N, int64_t K,
                     const SamplePlan &sp, float coef, int accumulate, float *out, SplitParts *defer = nullptr);
void bucket_samples(gvt_ctx *c, const char *tag, SamplePlan &sp, int64_t nrow, int64_t ncol);

// ---- Gram (gram.cu)
// K (m x m2, ldk) = k(X_i, Y_j); Y == nullptr: the Gram of X (m2 = m)
void gram_simt(gvt_ctx *c, int kind, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, int64_t ldx,
               double gamma, double coef0, int degree, float *K, int64_t ldk);
void gram_tc(gvt_ctx *c, int kind, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, double gamma,
             double coef0, int degree, float *K, int64_t ldk);
// Tanimoto Gram of 0/1 features (bit-packed popcount contraction); GVT_E_PARAM on non-binary input
void gram_tanimoto(gvt_ctx *c, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, float *K,
                   int64_t ldk);

// ---- CG (cg.cu)
struct CGState;  // device
void cg_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r, float *p, double *state, double rel_tol);
void cg_after_matvec(gvt_ctx *c, float *Ap, const float *p, int64_t n, double lambda, double *state);
// fused CG tail for the cheap forms (single GPU): the final combine of the matvec also forms the
// direction (p = r + beta p when lazy), the ridge term Ap = u + lambda p and the p.Ap partials, and
// takes the alpha step; cg_update_xr then runs only the x / r update (the direction update moves into
// the next iteration's segment sums).  cg_direction materialises p = r + beta p once after the loop.
void cg_combine_ap(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, const float *g1, int rs1, float c1,
                   const float *g2, int rs2, float c2, int accumulate, float *u, float *p, const float *r_lazy,
                   double lambda, double *state);
void cg_update_xr(gvt_ctx *c, float *x, float *r, const float *p, const float *Ap, int64_t n, double *state);
void cg_direction(gvt_ctx *c, float *p, const float *r, int64_t n, const double *state);
void cg_update(gvt_ctx *c, float *x, float *r, float *p, const float *Ap, int64_t n, double *state, int iter,
               double *relres_dev);
// fused dense-engine CG tail (tail.cu, single GPU): split-K combine, Ap / alpha, x / r / beta,
// p = r + beta p and the next X(p) rows (warp per row, ld <= dense_tail_fits) in one persistent launch
bool dense_tail_fits(int64_t ld);
void dense_tail_finish(gvt_ctx *c, float *p, const float *p_alt, int64_t n, const double *state);
const int32_t *dense_tail_init(gvt_ctx *c, double *part2, const int32_t *dst, int64_t ns, int64_t n);
// up to two deferred part sets (the first stored, the second accumulated, each as the GEMM's own combine
// would) and up to two pair-matrix operands to rebuild (the Cartesian form's X and X^T)
struct TailX {
    const EntryPlan *e = nullptr;
    int64_t row_lo = 0, rows = 0;
    Operand op;
};
// the cheap forms' final gather-combine u_i = c1 g1[sel1(i)] + c2 g2[sel2(i)] (+ u_i), done by the tail's first
// phase exactly as k_cg_combine_ap does it (then no part sets, no pair-matrix operand, p updated in place)
struct GatherCombine {
    const int32_t *f = nullptr, *s = nullptr;
    const float *g1 = nullptr, *g2 = nullptr;
    int rs1 = 0, rs2 = 0, accumulate = 0;
    float c1 = 1.f, c2 = 1.f;
};
void dense_cg_tail(gvt_ctx *c, const SplitParts &pa, const SplitParts &pb, const int32_t *inv, float *u, float *x,
                   float *r, float *p0, float *p1, int64_t n, int64_t nvb, double lambda, double *state,
                   double *part1, double *part2, const TailX *xs, int nx, const GatherCombine *gcomb = nullptr);
int cg_vec_blocks(int64_t n);
double *cg_parts(gvt_ctx *c);
// Chronopoulos-Gear single-reduction CG (GVT_OPT_CG_VARIANT = 1): init, then per iteration the
// matvec w = K r followed by cgg_step; cgg_finish records ||r_K|| after the loop
void cgg_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r, float *p, float *sv, double *state,
              double rel_tol);
void cgg_step(gvt_ctx *c, float *x, float *r, float *p, float *sv, float *w, int64_t n, double lambda,
              double *state);
void cgg_finish(gvt_ctx *c, const float *r, int64_t n, double *state);
// multi-GPU hook: reduce a partial-sum vector across ranks (no-op at world 1)
void allreduce_partials(gvt_ctx *c, double *partials, int count);

// ---- MINRES and early stopping (solver.cu)
constexpr int MINRES_STATE_N = 19;  // device state doubles before the relres history
void minres_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r1, float *r2, float *v, float *W1,
                 float *W2, double *state, double rel_tol);
// u = K v on entry (the matvec's first n entries); Lanczos step + rotations
void minres_step(gvt_ctx *c, float *u, float *v, float *r1, float *r2, float *W1, float *W2, float *x, int64_t n,
                 double lambda, double *state);
void minres_update(gvt_ctx *c, float *v, float *W1, float *W2, float *x, const float *r2, int64_t n, double *state,
                   float *kv, float *KW1, float *KW2, float *s, int64_t n_val);

struct AucPlan {
    int64_t n = 0;
    double P = 0, N = 0;  // positives / negatives
    uint8_t *pos = nullptr, *pos_sorted = nullptr;
    float *keys_sorted = nullptr;
    long long *negpre = nullptr;        // n + 1: negatives among the first i sorted scores
    unsigned long long *twice = nullptr;  // doubled Mann-Whitney numerator (+ scratch)
    void *temp = nullptr;
    size_t temp_bytes = 0;
    void setup(gvt_ctx *c, const char *tag, const float *labels_dev, int64_t n);
    void count(gvt_ctx *c, const float *scores, const double *st, const double *es);
};
double auc(gvt_ctx *c, const float *labels, const float *scores, int64_t n);
constexpr int ES_STATE_N = 5;
void es_init(gvt_ctx *c, double *es, double *hist, int max_iter, AucPlan &a);
void es_cg_scores(gvt_ctx *c, float *s, const float *kp, int64_t n_val, const double *state);
void es_evaluate(gvt_ctx *c, AucPlan &a, const float *scores_full, double *state, double *es, double *hist,
                 int patience, const float *x, float *a_best, int64_t n);

// ---- persistent multi-CTA whole-fit CG for small Kronecker problems (small.cu)
bool small_eligible(int64_t m, int64_t q, int64_t n);
void small_cg(gvt_ctx *c, const Factor &D, const Factor &T, const EntryPlan &e, const SamplePlan &sp, int64_t m,
              int64_t q, const float *y, float *x, int64_t n, double lambda, int max_iter, double tol, double *state,
              bool keep_dir = false);

// ---- single-CTA whole-fit CG for small Kronecker problems (tiny.cu)
size_t tiny_smem(int64_t m, int64_t q, int64_t n);  // 0 if it does not fit one SM
void tiny_cg(gvt_ctx *c, const Factor &D, const Factor &T, const EntryPlan &e, const SamplePlan &sp, int64_t m,
             int64_t q, const float *y, float *x, int64_t n, double lambda, int max_iter, double tol, double *state);

// partial-sum layout (cg.cu)
constexpr int RED_BLOCKS = 1184;  // 8 x 148 SMs
constexpr int RED_THREADS = 256;

}  // namespace gvt
