// engine.cu -- orchestration of the GVT matvec for every pairwise kernel, the CG fit and
// prediction, single GPU and data-parallel.
//
// Every Corollary kernel is run through ONE "Kronecker group"
//     G = A X C^T sampled at (r_k, c_k),   X = pair matrix built from p,
// the GVT of Theorem 1 in variant-1 form (reading S2):
//     stage 1  S = C X^T   (S[t][h] = sum_{entries (h, col)} x C[t][col])
//     stage 2  G[r,c] = <A[r,:], S[c,:]>
// plus cheap Ones-factor terms (Theorem 2).  Normal forms (derived from the
// Corollary with the indexing rules PAPER.md:757-761; each equals the term sum exactly):
//   Kronecker/Gaussian  A=D, C=T, X=B                      u = G[d,t]
//   Symmetric           A=C=D, X=B+B^T                      u = G[d,d']
//   Anti-symmetric      A=C=D, X=B-B^T      (I-P), S3       u = G[d,d']
//   MLPK                A=C=D, X=L=diag(bF+bS)-B-B^T        u = G[d,d]+G[d',d']-2G[d,d']
//   Poly2D              2*Kronecker + (D.^2 bF)[d] + (T.^2 bS)[t]
//   Linear              (D bF)[d] + (T bS)[t]
//   Ranking             g = D (bF - bS),  u = g[d] - g[d']  (oriented incidence)
//   Cartesian           segment gathers over pairs sharing t / sharing d
// with B[h,h'] = sum_{j: (d_j,t_j)=(h,h')} p_j, bF = B 1, bS = B^T 1.  Any other term
// list runs term by term as groups (Ones / Identity factors materialised).
//
// Data-parallel layout: each rank owns a shard of the in-sample (and of
// y, a, p) and of the out-sample.  The in-sample ids and p are gathered (grouped NCCL
// broadcasts), the rows of X (= columns of S) are split into contiguous slabs balanced by
// entry count, each rank runs stage 1 on its own slab, the S slabs are all-gathered, and
// stage 2 runs on the rank's own outputs, slab by slab (K split).  With one GPU the same
// slab code runs with GVT_OPT_SLABS emulated slabs (all computed locally).
#include <string.h>

#include <algorithm>
#include <vector>

#include "ops.cuh"

namespace gvt {

void nccl_unique_id(void *out128);
void comm_init(gvt_ctx *c, const void *id128, int rank, int world);
void comm_destroy(gvt_ctx *c);
void allgather_slabs(gvt_ctx *c, float *S, size_t slab_floats);
std::vector<int64_t> allgather_count(gvt_ctx *c, int64_t v);
void gather_varlen(gvt_ctx *c, const void *local, void *full, const std::vector<int64_t> &counts,
                   const std::vector<int64_t> &offsets, bool is_float);
void reduce_segments(gvt_ctx *c, const float *partial, float *local, const std::vector<int64_t> &counts,
                     const std::vector<int64_t> &offsets, int64_t tail);
bool slab_pipeline_available(gvt_ctx *c);
void slab_pipeline_start(gvt_ctx *c, void *const *bufs, const size_t *slab_bytes, int nbuf);
void slab_wait(gvt_ctx *c, int s);

// ----------------------------------------------------------------------------- decompose
static gvt_term mk(double coef, int l, int r, int rl, int rr, int cl, int cr) {
    gvt_term t;
    t.coef = coef;
    t.left = l;
    t.right = r;
    t.row_sel_left = rl;
    t.row_sel_right = rr;
    t.col_sel_left = cl;
    t.col_sel_right = cr;
    return t;
}

int kernel_terms(int kernel, gvt_term *o) {
    const int F = GVT_SEL_FIRST, S = GVT_SEL_SECOND;
    const int DR = GVT_FACTOR_DRUG, TA = GVT_FACTOR_TARGET, ON = GVT_FACTOR_ONES, ID = GVT_FACTOR_IDENTITY;
    int n = 0;
    switch (kernel) {
    case GVT_LINEAR: o[n++] = mk(1, DR, ON, F, S, F, S); o[n++] = mk(1, ON, TA, F, S, F, S); break;
    case GVT_POLY2D:
        o[n++] = mk(1, DR, DR, F, F, F, F);
        o[n++] = mk(2, DR, TA, F, S, F, S);
        o[n++] = mk(1, TA, TA, S, S, S, S);
        break;
    case GVT_GAUSSIAN:
    case GVT_KRONECKER: o[n++] = mk(1, DR, TA, F, S, F, S); break;
    case GVT_CARTESIAN: o[n++] = mk(1, DR, ID, F, S, F, S); o[n++] = mk(1, ID, TA, F, S, F, S); break;
    case GVT_SYMMETRIC: o[n++] = mk(1, DR, DR, F, S, F, S); o[n++] = mk(1, DR, DR, S, F, F, S); break;
    case GVT_ANTISYMMETRIC: o[n++] = mk(1, DR, DR, F, S, F, S); o[n++] = mk(-1, DR, DR, S, F, F, S); break;
    case GVT_RANKING:
        o[n++] = mk(1, DR, ON, F, S, F, S);
        o[n++] = mk(-1, DR, ON, S, F, F, S);
        o[n++] = mk(-1, DR, ON, F, S, S, F);
        o[n++] = mk(1, DR, ON, S, F, S, F);
        break;
    case GVT_MLPK:
        o[n++] = mk(1, DR, DR, F, F, F, F);
        o[n++] = mk(1, DR, DR, S, S, F, F);
        o[n++] = mk(1, DR, DR, F, F, S, S);
        o[n++] = mk(1, DR, DR, S, S, S, S);
        o[n++] = mk(2, DR, DR, F, S, F, S);
        o[n++] = mk(2, DR, DR, S, F, F, S);
        o[n++] = mk(-2, DR, DR, F, F, F, S);
        o[n++] = mk(-2, DR, DR, S, S, F, S);
        o[n++] = mk(-2, DR, DR, F, S, F, F);
        o[n++] = mk(-2, DR, DR, F, S, S, S);
        break;
    default: return -1;
    }
    return n;
}

enum Form { FORM_KRON = 0, FORM_SYM, FORM_ANTI, FORM_MLPK, FORM_POLY2D, FORM_LINEAR, FORM_RANKING, FORM_CARTESIAN,
            FORM_GENERIC };

static bool same_terms(const gvt_term *a, int na, const gvt_term *b, int nb) {
    if (na != nb) return false;
    for (int i = 0; i < na; i++) {
        if (a[i].coef != b[i].coef || a[i].left != b[i].left || a[i].right != b[i].right ||
            a[i].row_sel_left != b[i].row_sel_left || a[i].row_sel_right != b[i].row_sel_right ||
            a[i].col_sel_left != b[i].col_sel_left || a[i].col_sel_right != b[i].col_sel_right)
            return false;
    }
    return true;
}

static Form recognize(const gvt_term *terms, int n) {
    gvt_term ref[16];
    struct { int k; Form f; } tab[] = {{GVT_KRONECKER, FORM_KRON}, {GVT_SYMMETRIC, FORM_SYM},
                                       {GVT_ANTISYMMETRIC, FORM_ANTI}, {GVT_MLPK, FORM_MLPK},
                                       {GVT_POLY2D, FORM_POLY2D}, {GVT_LINEAR, FORM_LINEAR},
                                       {GVT_RANKING, FORM_RANKING}, {GVT_CARTESIAN, FORM_CARTESIAN}};
    for (auto &e : tab) {
        int nr = kernel_terms(e.k, ref);
        if (same_terms(terms, n, ref, nr)) return e.f;
    }
    return FORM_GENERIC;
}

static bool form_homogeneous(Form f) { return f == FORM_SYM || f == FORM_ANTI || f == FORM_MLPK || f == FORM_RANKING; }

// ----------------------------------------------------------------------------- problem
struct Problem {
    int64_t m = 0, q = 0;          // in-domain sizes (q = m when homogeneous)
    int64_t m_out = 0, q_out = 0;  // out-domain sizes: = m, q except with rectangular cross-Grams
    bool hom = false;
    bool rect = false;             // novel-object cross-Grams (out ids index rows, in ids columns)
    Factor D, T;           // T aliases D when homogeneous
    const int32_t *of = nullptr, *os = nullptr;    // this rank's out pairs
    int64_t n_out = 0;
    const int32_t *inf = nullptr, *ins = nullptr;  // the FULL in-sample (gathered across ranks)
    int64_t n_in = 0;
    // data-parallel in-sample partition (world 1: counts = {n_in})
    std::vector<int64_t> counts, offsets;
    float *p_full = nullptr;
    // u-exchange (GVT_OPT_EXCHANGE = 1, world > 1): the FULL out sample on every rank, in rank
    // order; this rank's outputs are [out_offsets[rank], out_offsets[rank + 1])
    bool uex = false;
    const int32_t *of_full = nullptr, *os_full = nullptr;
    int64_t n_out_full = 0;
    std::vector<int64_t> out_counts, out_offsets;
    // outputs appended to the fit's own (the early-stopping validation pairs): left out of the
    // stage-2 dispatch estimate, so the early-stopping fit runs the same kernels as a plain fit
    int64_t n_out_extra = 0;
    // rank-independent sizes for the dispatch estimates (every rank must take the same
    // engine decisions, or the collectives of different engines mismatch): the out-sample size
    // summed over ranks and its appended-extra part (world 1: the local sizes)
    int64_t n_out_all = 0, n_out_extra_all = 0;
    int64_t dom(int sel) const { return (sel == GVT_SEL_FIRST || hom) ? m : q; }
    int64_t dom_out(int sel) const { return (sel == GVT_SEL_FIRST || hom) ? m_out : q_out; }
};

// validate a term list against the data (before any compute)
static void validate_terms(const gvt_term *terms, int n_terms, bool hom, Form form, bool rect = false) {
    GVT_REQUIRE(terms && n_terms >= 1 && n_terms <= 64, GVT_E_KERNEL, "term list empty or too long");
    if (rect) {
        GVT_REQUIRE(form != FORM_CARTESIAN, GVT_E_KERNEL,
                    "Cartesian kernel on cross-Grams: its Identity factor compares objects of two different tables "
                    "(reading N1)");
        for (int i = 0; i < n_terms; i++)
            GVT_REQUIRE(terms[i].left != GVT_FACTOR_IDENTITY && terms[i].right != GVT_FACTOR_IDENTITY, GVT_E_KERNEL,
                        "Identity factor on cross-Grams (reading N1)");
    }
    if (form_homogeneous(form))
        GVT_REQUIRE(hom, GVT_E_HOMOGENEOUS, "homogeneous kernel (Symmetric/Anti-symmetric/Ranking/MLPK) given T != NULL");
    for (int i = 0; i < n_terms; i++) {
        const gvt_term &t = terms[i];
        int kinds[2] = {t.left, t.right}, rs[2] = {t.row_sel_left, t.row_sel_right},
            cs[2] = {t.col_sel_left, t.col_sel_right};
        for (int k = 0; k < 2; k++) {
            GVT_REQUIRE(kinds[k] >= 0 && kinds[k] <= 3, GVT_E_KERNEL, "term factor kind out of range");
            GVT_REQUIRE(rs[k] >= 0 && rs[k] <= 1 && cs[k] >= 0 && cs[k] <= 1, GVT_E_KERNEL, "term selector out of range");
            if (!hom) {
                if (kinds[k] == GVT_FACTOR_DRUG)
                    GVT_REQUIRE(rs[k] == GVT_SEL_FIRST && cs[k] == GVT_SEL_FIRST, GVT_E_HOMOGENEOUS,
                                "drug Gram indexed by target ids (heterogeneous data)");
                if (kinds[k] == GVT_FACTOR_TARGET)
                    GVT_REQUIRE(rs[k] == GVT_SEL_SECOND && cs[k] == GVT_SEL_SECOND, GVT_E_HOMOGENEOUS,
                                "target Gram indexed by drug ids (heterogeneous data)");
                if (kinds[k] == GVT_FACTOR_IDENTITY)
                    GVT_REQUIRE(rs[k] == cs[k], GVT_E_HOMOGENEOUS, "identity between different domains");
            }
        }
    }
}

// ----------------------------------------------------------------------------- plan
struct GroupPlan {
    Factor A, C;           // stage-2 factor (left), stage-1 factor (right)
    int64_t q_out = 0;     // rows of S (domain of the row-right selector)
    int64_t m_in = 0;      // cols of S = rows of X (domain of the col-left selector)
    EntryPlan ent;
    SamplePlan smp;
    float coef = 1.f;
    int engine = 1;        // 1 sparse, 2 dense
    // slabs of X rows / S columns: bounds[g] .. bounds[g+1], entry positions kpos[g]
    int nslab = 1;
    std::vector<int64_t> bounds, kpos;
    int64_t W = 0;         // slab width (padded to 32): S slab g is qpad x W at S + g * qpad * W
    int64_t qpad = 0;
    float *S = nullptr;
    std::string tag;
    float *diag = nullptr;  // optional separate diagonal of X (global row index), computed per matvec
    int64_t n_diag = 0;     // extra (x, x) samples after the outputs (MLPK)
    double ns_est = 0;      // stage-2 samples per rank for the dispatch estimates (identical on every rank)
    double extra_est = 0;   // of which appended extra outputs (early-stopping validation pairs)
    // block sparsity of X per slab for the fused fp16 stage 1 (device lists, nullptr = dense)
    std::vector<const int32_t *> kb_list, kb_off;
    std::vector<const int32_t *> kb_order;  // per slab: stage-1 pair tiles, longest K lists first (block-sparse)
    std::vector<int> kb_minch;              // per slab: the fewest 256-wide K chunks of any tile
};

struct MatvecPlan {
    Form form = FORM_GENERIC;
    std::vector<GroupPlan> groups;  // generic: one per term; else at most one
    EntryPlan byF, byS;            // segment plans (cheap terms / Cartesian)
    bool cart_dense = false;       // Cartesian as two sampled tensor-core GEMMs (D X + X T), below
    SamplePlan cart_smp;
    float *buf = nullptr;          // MLPK sample buffer (n_out + m)
    float *g1 = nullptr, *g2 = nullptr, *b1 = nullptr, *b2 = nullptr;
    std::vector<Factor> owned;     // materialised Ones/Identity factors
};

static EntryKinds kinds1(int rs, int cs, float sign) {
    EntryKinds k;
    memset(&k, 0, sizeof(k));
    k.count = 1;
    k.k[0] = EntryKind{rs, cs, sign};
    return k;
}

static Factor materialise(gvt_ctx *c, const char *name, int64_t rows, int64_t cols, int identity) {
    Factor f;
    f.n = rows;
    f.cols = cols;
    f.ld = round_up(cols > 0 ? cols : 1, 32);
    const int64_t rp = round_up(rows > 0 ? rows : 1, 32);
    float *p = wsT<float>(c, name, (size_t)rp * f.ld);
    fill_ones(c, p, rp, cols, f.ld, identity);  // identity only for square (global-id) factors
    f.p = p;
    if (rows != cols) {  // all-ones is its own transpose up to shape: the column-wise view
        const int64_t ldt = round_up(rows > 0 ? rows : 1, 32), cp = round_up(cols > 0 ? cols : 1, 32);
        float *pt = wsT<float>(c, (std::string(name) + ".t").c_str(), (size_t)cp * ldt);
        fill_ones(c, pt, cp, rows, ldt, 0);
        f.pt = pt;
        f.ldt = ldt;
    }
    return f;
}

// Engine choice by estimated time ("the dispatcher must choose by time"), from
// B200 measurements (scripts/density_sweep.py, profiles/r01_density_sweep.jsonl):
//  sparse: stage 1 at ~3.3e12 FMA/s (L2-bound, q_out FMA per entry), but no faster than its
//          CTAs' serial entry loops allow (8 X rows per CTA, ~0.05 us per entry, 9 CTAs per SM);
//          stage 2 gathers one S row per output at ~6.4 TB/s (S above L2) or ~12 TB/s
//  dense:  two 3xFP16 GEMMs (256-padded) at ~1.3e15 executed flop/s plus ~20 us fixed each,
//          the X build, and stage 2 as the cheaper of the sampled GEMM and the gather
// At C5 object counts this puts the crossover near 1 % density; on small problems (C2) the
// sparse engine's short grid keeps the tensor cores ahead.  GVT_OPT_DENSE_THRESHOLD >= 0
// replaces the estimate by the plain density rule.
static bool dense_pays(gvt_ctx *c, double nnz, double ns, int64_t m_out, int64_t q_out, int64_t m_in,
                       int64_t q_in) {
    if (c->dense_threshold >= 0.0) {
        const double cells = (double)m_in * (double)q_in;
        return cells > 0 && nnz / cells >= c->dense_threshold;
    }
    auto rup = [](int64_t v, int64_t a) { return (double)round_up(v > 0 ? v : 1, a); };
    const double hblocks = std::max(1.0, rup(m_in, 32) / 8.0), ttiles = std::max(1.0, std::ceil(q_out / 512.0));
    const double waves = std::ceil(hblocks * ttiles / (9.0 * c->sm_count));
    const double s1 = std::max(nnz * (double)q_out / 3.3e6, nnz / hblocks * 0.05 * waves);
    const double s_bytes = 4.0 * (double)q_out * (double)m_in;
    const double g2 = ns * (double)m_in * 4.0 / (s_bytes > 64e6 ? 6.4e6 : 12e6);
    const double sparse_us = 10.0 + s1 + g2;
    const double gemm1 = 20.0 + 6.0 * rup(q_out, 256) * rup(m_in, 256) * rup(q_in, 64) / 1.3e9;
    const double gemm2 = 20.0 + 6.0 * rup(m_out, 256) * rup(q_out, 256) * rup(m_in, 64) / 1.3e9;
    const double gath2 = 4.0 + 8.0 * ns * (double)m_in / 6e6;
    const double dense_us = 5.0 + (double)m_in * (double)q_in * 4.0 / 4e6 + gemm1 + std::min(gemm2, gath2);
    return dense_us < sparse_us;
}

static int choose_engine(gvt_ctx *c, const GroupPlan &g) {
    // every input of the decision is identical on all ranks: nnz of the full in-sample plan, the
    // per-rank sample estimate, the factor dimensions
    if (c->engine == 1) return 1;
    bool tc = tc_available(c);
    if (c->engine == 2) {
        GVT_REQUIRE(tc, GVT_E_CUDA, "dense tensor-core engine requested but not available on this device");
        if (g.A.split && g.C.split) return 2;
        return 1;  // materialised Ones/Identity factors of a generic term list stay on SIMT
    }
    if (!(g.A.split && g.C.split)) return 1;  // factors were not split for tensor cores
    return (tc && dense_pays(c, (double)g.ent.nnz, g.ns_est, g.A.n, g.q_out, g.m_in, g.C.cols)) ? 2 : 1;
}

// X-row slabs balanced by entry count (row_ptr over nrow rows), bounds multiples of 32 (TMA /
// float4 alignment of the column views of A): bounds[s] = the first row at or after the
// s/G quantile of the entries, rounded up to 32, monotone, bounds[0] = 0, bounds[G] = nrow.
// Host only; also exported as gvt_slab_bounds for the multi-process tests.
void slab_bounds(const int64_t *rp, int64_t nrow, int G, int64_t *bounds) {
    bounds[0] = 0;
    bounds[G] = nrow;
    const int64_t E = rp[nrow];
    for (int s = 1; s < G; s++) {
        const int64_t target = (int64_t)((long double)E * s / G);
        int64_t h = std::lower_bound(rp, rp + nrow + 1, target) - rp;
        h = round_up(h, 32);
        h = std::min(std::max(h, bounds[s - 1]), nrow);
        bounds[s] = h;
    }
}

// Slabs balanced by an estimated cost C(h) = w_entry * row_ptr[h] + w_row * h (the cost of rows
// [0, h)): bounds[s] = the first row whose C reaches the s/G quantile of C(nrow), rounded up to
// 32, monotone.  w_row = 0 is slab_bounds.  The engine's weights (make_slabs): the dense engine's
// stage-1 and stage-2 GEMMs both scale with the slab's ROWS (w_entry 0); the sparse engine's
// stage 1 with its entries (q_out FMAs each) and, under the u-exchange, its stage 2 with its rows
// (one W-wide slice of an S row per output).  Host only (gvt_slab_bounds_cost).
void slab_bounds_cost(const int64_t *rp, int64_t nrow, int G, double w_entry, double w_row, int64_t *bounds) {
    bounds[0] = 0;
    bounds[G] = nrow;
    auto cost = [&](int64_t h) { return w_entry * (double)rp[h] + w_row * (double)h; };
    const double total = cost(nrow);
    int64_t h = 0;
    for (int s = 1; s < G; s++) {
        const double target = total * s / G;
        // C is non-decreasing in h: advance to the first row reaching the target
        int64_t lo = h, hi = nrow;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (cost(mid) < target) lo = mid + 1;
            else hi = mid;
        }
        int64_t b = std::min(std::max(round_up(lo, 32), bounds[s - 1]), nrow);
        bounds[s] = b;
        h = std::min(lo, nrow);
    }
}

// slabs of a group, identical on every rank (computed from the same full plan)
static void make_slabs(gvt_ctx *c, GroupPlan &g, bool uex) {
    // one slab per rank across GPUs (rank r owns slab r); emulated slabs only at world 1
    int G = distributed(c) ? c->world : std::max(1, c->slabs);
    const int64_t nrow = g.m_in;
    std::vector<int64_t> rp((size_t)nrow + 1);
    GVT_CUDA_TRY(cudaMemcpyAsync(rp.data(), g.ent.row_ptr, sizeof(int64_t) * (nrow + 1), cudaMemcpyDeviceToHost,
                                 c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    g.nslab = G;
    g.bounds.assign((size_t)G + 1, 0);
    // weights of the engine's own cost (entry balancing left dense slabs with rows max/mean
    // 3.2 on degree-sorted ids): dense -> rows; sparse -> q_out per entry (stage 1, ~3.3e6 FMA/us)
    // plus, under the u-exchange, 4 B per output per row (stage 2 slice gathers, ~6.4e6 B/us)
    if (g.engine == 2) slab_bounds_cost(rp.data(), nrow, G, 0.0, 1.0, g.bounds.data());
    else slab_bounds_cost(rp.data(), nrow, G, (double)g.q_out / 3.3e6, uex ? 4.0 * g.ns_est / 6.4e6 : 0.0,
                          g.bounds.data());
    g.kpos.assign((size_t)G + 1, 0);
    int64_t wmax = 0;
    for (int s = 0; s <= G; s++) g.kpos[s] = rp[g.bounds[s]];
    for (int s = 0; s < G; s++) wmax = std::max(wmax, g.bounds[s + 1] - g.bounds[s]);
    g.W = round_up(wmax > 0 ? wmax : 1, 32);
}

static bool my_slab(gvt_ctx *c, int s) { return !distributed(c) || s == c->rank; }

static bool kblock_order() {  // A/B knob: GVT_KBLOCK_ORDER=0 keeps the grouped tile order for block-sparse stage 1
    static const bool on = [] {
        const char *e = getenv("GVT_KBLOCK_ORDER");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

static void finish_group(gvt_ctx *c, GroupPlan &g, const char *tag, bool uex) {
    g.tag = tag;
    g.engine = choose_engine(c, g);
    make_slabs(c, g, uex);
    g.qpad = round_up(g.q_out > 0 ? g.q_out : 1, 128);
    g.S = wsT<float>(c, (g.tag + ".S").c_str(), (size_t)g.nslab * g.qpad * g.W);
    if (g.engine == 2) bucket_samples(c, tag, g.smp, g.A.n, g.q_out);
    // block-sparse stage 1: the (256-row, 64-column) blocks of each X slab holding entries, kept
    // when they cover at most 85 % of the slab (e.g. MLPK on a union domain: the drug-target blocks
    // and the diagonal only); dense blocks everywhere (C3, C4 Poly2D, C5) keep the plain K loop
    g.kb_list.assign((size_t)g.nslab, nullptr);
    g.kb_off.assign((size_t)g.nslab, nullptr);
    g.kb_order.assign((size_t)g.nslab, nullptr);
    g.kb_minch.assign((size_t)g.nslab, 0);
    if (g.engine == 2 && fused_f16(c, g.C.cols) && c->kblock_skip) {
        for (int s = 0; s < g.nslab; s++) {
            if (!my_slab(c, s)) continue;
            const int64_t lo = g.bounds[s], w = g.bounds[s + 1] - lo;
            if (w == 0) continue;
            std::vector<int32_t> list, off;
            kblock_lists(c, g.ent, g.kpos[s], g.kpos[s + 1], lo, w, g.C.cols, g.diag != nullptr, list, off);
            const double total = (double)(off.size() - 1) * (double)((g.C.cols + 63) / 64);
            if ((double)list.size() > 0.85 * total) continue;
            char nm[64];
            snprintf(nm, sizeof(nm), "%s.kbl%d", tag, s);
            int32_t *dl = wsT<int32_t>(c, nm, list.size());
            snprintf(nm, sizeof(nm), "%s.kbo%d", tag, s);
            int32_t *dof = wsT<int32_t>(c, nm, off.size());
            GVT_CUDA_TRY(cudaMemcpyAsync(dl, list.data(), sizeof(int32_t) * list.size(), cudaMemcpyHostToDevice, c->stream));
            GVT_CUDA_TRY(cudaMemcpyAsync(dof, off.data(), sizeof(int32_t) * off.size(), cudaMemcpyHostToDevice, c->stream));
            // the stage-1 GEMM's pair tiles (M = q_out rows of C in pairs of 256, N = this slab's X rows in 256-row
            // tiles, whose K lists these are) in the kernel's grouped order, then stably by descending K-list length:
            // the persistent loop then hands every CTA pair a similar amount of work (longest first)
            const int num_n = (int)(off.size() - 1), num_mp = (int)((g.q_out + 255) / 256);
            std::vector<int32_t> order;
            order.reserve((size_t)num_mp * num_n);
            const int gm = gemm_group_m(), in_group = gm * num_n;
            for (int t = 0; t < num_mp * num_n; t++) {
                const int first_m = (t / in_group) * gm, group_m = std::min(num_mp - first_m, gm);
                order.push_back((first_m + (t % in_group) % group_m) * num_n + (t % in_group) / group_m);
            }
            auto len = [&](int32_t tl) { return off[(size_t)(tl % num_n) + 1] - off[(size_t)(tl % num_n)]; };
            std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return len(x) > len(y); });
            int minch = INT32_MAX;
            for (int n = 0; n < num_n; n++) minch = std::min(minch, (off[(size_t)n + 1] - off[(size_t)n] + 3) / 4);
            snprintf(nm, sizeof(nm), "%s.kbord%d", tag, s);
            int32_t *dord = wsT<int32_t>(c, nm, order.size());
            GVT_CUDA_TRY(cudaMemcpyAsync(dord, order.data(), sizeof(int32_t) * order.size(), cudaMemcpyHostToDevice,
                                         c->stream));
            GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));  // the host vectors go out of scope
            g.kb_list[(size_t)s] = dl;
            g.kb_off[(size_t)s] = dof;
            g.kb_order[(size_t)s] = kblock_order() ? dord : nullptr;
            g.kb_minch[(size_t)s] = minch;
        }
    }
}

// per-rank stage-2 sample estimate from rank-independent sizes: the u-exchange serves the full
// out sample on every rank; the S all-gather serves the rank's own outputs, estimated as the
// average over ranks (world 1: exactly the local count)
static void set_estimates(gvt_ctx *c, const Problem &P, GroupPlan &g) {
    const double w = distributed(c) ? (double)c->world : 1.0;
    g.ns_est = (P.uex ? (double)P.n_out_full : (double)P.n_out_all / w) + (double)g.n_diag;
    g.extra_est = P.uex ? (double)P.n_out_extra_all : (double)P.n_out_extra_all / w;
}

// Cartesian kernel (Corollary D(x)I + I(x)T): u_i = (D X)[d_i, t_i] + (X T)[d_i, t_i] with
// X = the m x q pair matrix of p.  Gather form (k_cartesian): one warp per output walks the output's two
// entry segments, ~1 random 32-byte sector per entry (calibrated: C3, 4e7 entries, ~90 us).  Dense form:
// two sampled 3xFP16 GEMMs, A = D / B = X^T (K = m) and A = X / B = T (K = q), over the non-empty CTA-pair
// tiles `units` of the output grid (split-K when at most a quarter of the pairs have one), plus the two
// fp16 pair-matrix builds.  Estimates in us.
static double cart_gather_us(const Problem &P) {
    const double per_out = (double)P.n_in / std::max<int64_t>(P.q, 1) + (double)P.n_in / std::max<int64_t>(P.m, 1);
    return 5.0 + (double)P.n_out_all * per_out / 0.45e6;
}
static double cart_dense_us(gvt_ctx *c, const Problem &P, double units) {
    const double pairs = c->sm_count / 2.0;
    auto gemm = [&](int64_t K) {
        const double tile_us = 3.0 * 65536.0 * (double)round_up(K > 0 ? K : 1, 256) / 1.47e7;  // one pair tile
        const double load = units <= pairs / 2.0 ? 0.5 : std::ceil(units / pairs);
        return 10.0 + tile_us * load;
    };
    const double build = 2.0 * (3.0 + (double)P.m * (double)P.q * 8.0 / 3e6);
    return gemm(P.m) + gemm(P.q) + build;
}
static bool cart_dense_possible(gvt_ctx *c, const Problem &P) {
    if (!tc_available(c) || c->engine == 1 || distributed(c) || P.rect || P.n_out == 0 || P.n_in == 0) return false;
    if (!fused_f16(c, P.m) || !fused_f16(c, P.q)) return false;
    if (c->engine == 2) return true;
    // lower bound: the fewest non-empty tiles that can hold the out sample
    return cart_dense_us(c, P, std::ceil((double)P.n_out_all / 65536.0)) < cart_gather_us(P);
}

static void plan_matvec(gvt_ctx *c, const Problem &P, const gvt_term *terms, int n_terms, Form form,
                        MatvecPlan &mp) {
    mp.form = form;
    const int F = GVT_SEL_FIRST, Sx = GVT_SEL_SECOND;
    auto group = [&](const Factor &A, const Factor &C, EntryKinds kinds, int64_t nrow, int64_t ncol, int rs, int cs,
                     int64_t n_diag, float coef, const char *tag, float *x_diag = nullptr) {
        GroupPlan g;
        g.diag = x_diag;  // before finish_group: the block-sparsity lists include the diagonal
        g.A = A;
        g.C = C;
        g.q_out = C.n;
        g.m_in = nrow;
        g.coef = coef;
        std::string t(tag);
        build_entry_plan(c, (t + ".e").c_str(), P.inf, P.ins, P.n_in, kinds, nrow, ncol, g.ent);
        // u-exchange: stage 2 of this rank's S slab serves EVERY output (full out sample)
        if (P.uex) build_sample_plan(c, (t + ".s").c_str(), P.of_full, P.os_full, P.n_out_full, rs, cs, n_diag, A.n, g.smp);
        else build_sample_plan(c, (t + ".s").c_str(), P.of, P.os, P.n_out, rs, cs, n_diag, A.n, g.smp);
        g.n_diag = n_diag;
        set_estimates(c, P, g);
        finish_group(c, g, tag, P.uex);
        mp.groups.push_back(g);
    };
    switch (form) {
    case FORM_KRON:
        group(P.D, P.T, kinds1(F, Sx, 1.f), P.m, P.q, F, Sx, 0, 1.f, "g0");
        break;
    case FORM_POLY2D:
        group(P.D, P.T, kinds1(F, Sx, 1.f), P.m, P.q, F, Sx, 0, 2.f, "g0");
        build_entry_plan(c, "byS", P.inf, P.ins, P.n_in, kinds1(Sx, F, 1.f), P.q, P.m, mp.byS);
        break;
    case FORM_SYM:
    case FORM_ANTI: {
        EntryKinds k;
        memset(&k, 0, sizeof(k));
        k.count = 2;
        k.k[0] = EntryKind{F, Sx, 1.f};
        k.k[1] = EntryKind{Sx, F, form == FORM_SYM ? 1.f : -1.f};
        group(P.D, P.D, k, P.m, P.m, F, Sx, 0, 1.f, "g0");
        break;
    }
    case FORM_MLPK: {
        EntryKinds k;
        memset(&k, 0, sizeof(k));
        // L = diag(bF + bS) - B - B^T: the off-diagonal part as entries, the diagonal as a vector
        // (segment sums over both pair elements; a diagonal cell gathers deg(h) entries, which
        // would serialise a per-cell sum)
        k.count = 2;
        k.k[0] = EntryKind{F, Sx, -1.f};
        k.k[1] = EntryKind{Sx, F, -1.f};
        group(P.D, P.D, k, P.m, P.m, F, Sx, P.m_out, 1.f, "g0",
              wsT<float>(c, "mlpk.diag", (size_t)round_up(P.m > 0 ? P.m : 1, 32)));
        {
            EntryKinds kd;
            memset(&kd, 0, sizeof(kd));
            kd.count = 2;
            kd.k[0] = EntryKind{F, Sx, 1.f};
            kd.k[1] = EntryKind{Sx, F, 1.f};
            build_entry_plan(c, "byF", P.inf, P.ins, P.n_in, kd, P.m, P.m, mp.byF);
        }
        mp.buf = wsT<float>(c, "mlpk.buf", (size_t)(P.n_out + P.m_out));
        break;
    }
    case FORM_LINEAR:
        build_entry_plan(c, "byF", P.inf, P.ins, P.n_in, kinds1(F, Sx, 1.f), P.m, P.q, mp.byF);
        build_entry_plan(c, "byS", P.inf, P.ins, P.n_in, kinds1(Sx, F, 1.f), P.q, P.m, mp.byS);
        break;
    case FORM_RANKING: {
        EntryKinds k;
        memset(&k, 0, sizeof(k));
        k.count = 2;
        k.k[0] = EntryKind{F, Sx, 1.f};
        k.k[1] = EntryKind{Sx, F, -1.f};
        build_entry_plan(c, "byF", P.inf, P.ins, P.n_in, k, P.m, P.m, mp.byF);
        break;
    }
    case FORM_CARTESIAN:
        build_entry_plan(c, "byF", P.inf, P.ins, P.n_in, kinds1(F, Sx, 1.f), P.m, P.q, mp.byF);
        build_entry_plan(c, "byS", P.inf, P.ins, P.n_in, kinds1(Sx, F, 1.f), P.q, P.m, mp.byS);
        if (P.D.split && P.T.split) {  // the dense form may pay: decide on the exact non-empty tile count
            build_sample_plan(c, "cart.s", P.of, P.os, P.n_out, F, Sx, 0, P.m, mp.cart_smp);
            bucket_samples(c, "cart", mp.cart_smp, P.m, P.q);
            const double units = mp.cart_smp.n_pairs >= 0 ? (double)mp.cart_smp.n_pairs : 1e30;
            mp.cart_dense = c->engine == 2 || cart_dense_us(c, P, units) < cart_gather_us(P);
        }
        break;
    case FORM_GENERIC:
        for (int i = 0; i < n_terms; i++) {
            const gvt_term &t = terms[i];
            auto factor = [&](int kind, int rs, int cs, const char *nm) -> Factor {
                if (kind == GVT_FACTOR_DRUG) return P.D;
                if (kind == GVT_FACTOR_TARGET) return P.T;
                Factor f;
                if (P.rect) {  // all-ones over (out domain of rs) x (in domain of cs); no Identity (N1)
                    f = materialise(c, nm, P.dom_out(rs), P.dom(cs), 0);
                } else {
                    int64_t n = P.dom(rs) > P.dom(cs) ? P.dom(rs) : P.dom(cs);
                    f = materialise(c, nm, n, n, kind == GVT_FACTOR_IDENTITY);
                }
                mp.owned.push_back(f);
                return f;
            };
            char tag[32], nl[32], nr[32];
            snprintf(tag, sizeof(tag), "t%d", i);
            snprintf(nl, sizeof(nl), "t%d.L", i);
            snprintf(nr, sizeof(nr), "t%d.R", i);
            Factor L = factor(t.left, t.row_sel_left, t.col_sel_left, nl);
            Factor R = factor(t.right, t.row_sel_right, t.col_sel_right, nr);
            GroupPlan g;
            g.A = L;
            g.C = R;
            g.q_out = P.dom_out(t.row_sel_right);
            g.m_in = P.dom(t.col_sel_left);
            g.coef = (float)t.coef;
            std::string ts(tag);
            build_entry_plan(c, (ts + ".e").c_str(), P.inf, P.ins, P.n_in, kinds1(t.col_sel_left, t.col_sel_right, 1.f),
                             P.dom(t.col_sel_left), P.dom(t.col_sel_right), g.ent);
            if (P.uex)
                build_sample_plan(c, (ts + ".s").c_str(), P.of_full, P.os_full, P.n_out_full, t.row_sel_left,
                                  t.row_sel_right, 0, P.dom_out(t.row_sel_left), g.smp);
            else
                build_sample_plan(c, (ts + ".s").c_str(), P.of, P.os, P.n_out, t.row_sel_left, t.row_sel_right, 0,
                                  P.dom_out(t.row_sel_left), g.smp);
            set_estimates(c, P, g);
            finish_group(c, g, tag, P.uex);
            mp.groups.push_back(g);
        }
        break;
    }
    int64_t nb = std::max(std::max(P.m, P.q), std::max(P.m_out, P.q_out));
    nb = round_up(nb > 0 ? nb : 1, 32);
    if (form == FORM_POLY2D || form == FORM_LINEAR || form == FORM_RANKING) {
        mp.b1 = wsT<float>(c, "cheap.b1", nb);
        mp.b2 = wsT<float>(c, "cheap.b2", nb);
        mp.g1 = wsT<float>(c, "cheap.g1", nb);
        mp.g2 = wsT<float>(c, "cheap.g2", nb);
        // b vectors are read up to ld (padded): zero them once, segment sums overwrite [0, nrow)
        GVT_CUDA_TRY(cudaMemsetAsync(mp.b1, 0, sizeof(float) * nb, c->stream));
        GVT_CUDA_TRY(cudaMemsetAsync(mp.b2, 0, sizeof(float) * nb, c->stream));
    }
}

// ----------------------------------------------------------------------------- run

// fused 3xFP16 dense path: X rows assembled straight into fp16 pieces, stage 1 writes S as
// fp16 pieces with per-(row, 256-column) scales, stage 2 applies them per K-chunk; slab s of
// S lives at s * (qpad * W) halves (and s * ntW * skld scales) so ranks all-gather equal slabs
// u-exchange epilogue: out[0 .. n_local + n_diag) (+)= the rank's segment of the summed partials
static void uex_finish(gvt_ctx *c, const Problem &P, const GroupPlan &g, const float *partial, int accumulate,
                       float *out) {
    const int64_t n_local = P.out_counts[c->rank], n = n_local + g.n_diag;
    float *local = accumulate ? wsT<float>(c, "uex.local", (size_t)n) : out;
    reduce_segments(c, partial, local, P.out_counts, P.out_offsets, g.n_diag);
    if (accumulate) add_into(c, local, n, out);
}

// dense engine, stage 2 of one slab: the sampled tensor-core GEMM computes every (r, c) cell of
// the tile grid and serves the samples from its epilogue; the row gather reads one A row and one
// S row per sample.  On short contractions with few samples (C2: K = 68, 3e4 samples) the GEMM's
// fixed cost (prologue, serial K loop, sample serving) dominates and the gather wins.  Estimates
// from the B200 measurements: GEMM ~25 us + 6*M*N*K flops (3xFP16, 256/64-padded) at ~1.1 PFLOP/s;
// gather ~4 us + 8 B per (sample, k) at ~6 TB/s.
static bool stage2_gather_pays(gvt_ctx *c, int64_t ns, int64_t M, int64_t N, int64_t K) {
    if (c->stage2 == 1) return false;
    if (c->stage2 == 2) return true;
    const double tc = 25.0 + 6.0 * (double)round_up(M, 256) * (double)round_up(N, 256) * (double)round_up(K, 64) / 1.1e9;
    const double ga = 4.0 + 8.0 * (double)ns * (double)K / 6e6;
    return ga < tc;
}

// the fused dense-engine CG tail's view of one matvec (fit_impl, tail.cu): X(p) and the S-scale zeros
// already in place (built by the previous tail launch), and the split-K parts left for the tail
struct DenseFuse {
    bool prebuilt = false;
    SplitParts parts;
};

static void run_group_f16(gvt_ctx *c, const Problem &P, GroupPlan &g, const float *p_full, float coef, int accumulate,
                          float *out, DenseFuse *df = nullptr) {
    // S scales: one power-of-two scale per (row, 256-col tile) from the tile maxima, applied per
    // K-chunk in stage 2 (S16_SCALE_ROWS = 1); the A/B build -DS16_SCALE_ROWS=128 keeps one scale
    // per (128-row block, 256-col tile) instead (ops.cuh: fewer clocks, more energy at C5)
    const int64_t ntW = (g.W + 255) / 256, skld = round_up(g.q_out > 0 ? g.q_out : 1, 256) / S16_SCALE_ROWS;
    const size_t slab_h = (size_t)g.qpad * g.W, slab_k = (size_t)ntW * skld;
    __half *Sh = wsT<__half>(c, (g.tag + ".S16h").c_str(), slab_h * g.nslab);
    __half *Sl = wsT<__half>(c, (g.tag + ".S16l").c_str(), slab_h * g.nslab);
    float *Sk = wsT<float>(c, (g.tag + ".S16k").c_str(), slab_k * g.nslab);
    const bool prebuilt = df && df->prebuilt;
    if (!prebuilt) GVT_CUDA_TRY(cudaMemsetAsync(Sk, 0, sizeof(float) * slab_k * g.nslab, c->stream));
    for (int s = 0; s < g.nslab; s++) {
        if (!my_slab(c, s)) continue;
        const int64_t lo = g.bounds[s], w = g.bounds[s + 1] - lo;
        if (w == 0) continue;
        Operand xo = build_x16(c, "dense.X16", g.ent, lo, w, g.C.cols, p_full, g.diag, !prebuilt);
        gemm_nt_store16(c, g.C.op, xo, g.q_out, w, g.C.cols, Sh + s * slab_h, Sl + s * slab_h, g.W, Sk + s * slab_k,
                        skld, g.kb_list[(size_t)s], g.kb_off[(size_t)s], g.kb_order[(size_t)s], g.kb_minch[(size_t)s]);
    }
    float *partial = nullptr;
    const bool piped = !P.uex && slab_pipeline_available(c);
    if (P.uex) {  // no S exchange: this rank's slab serves every output, then the partials are reduced
        partial = wsT<float>(c, "uex.partial", (size_t)(P.n_out_full + g.n_diag));
        GVT_CUDA_TRY(cudaMemsetAsync(partial, 0, sizeof(float) * (P.n_out_full + g.n_diag), c->stream));
    } else if (piped) {  // per-slab broadcasts on the comm stream, overlapped with stage 2 below
        void *bufs[3] = {Sh, Sl, Sk};
        const size_t bytes[3] = {sizeof(__half) * slab_h, sizeof(__half) * slab_h, sizeof(float) * slab_k};
        slab_pipeline_start(c, bufs, bytes, 3);
    } else {  // halves travel as pairs of floats (W is a multiple of 32)
        allgather_slabs(c, reinterpret_cast<float *>(Sh), slab_h / 2);
        allgather_slabs(c, reinterpret_cast<float *>(Sl), slab_h / 2);
        allgather_slabs(c, Sk, slab_k);
    }
    bool first = true;
    for (int s = 0; s < g.nslab; s++) {
        const int64_t lo = g.bounds[s], w = g.bounds[s + 1] - lo;
        if (piped) slab_wait(c, s);  // (every slab, empty ones too: the waits join the comm stream)
        if (w == 0 || (P.uex && !my_slab(c, s))) continue;
        Operand so;
        so.prec = 0;
        so.hi = Sh + s * slab_h;
        so.lo = Sl + s * slab_h;
        so.ld = g.W;
        so.scale_k = Sk + s * slab_k;
        so.scale_k_ld = skld;
        // (P.uex: this rank's slab(s) -- one per rank, all of them with emulated slabs at world 1)
        float *dst = P.uex ? partial : out;
        const int acc = P.uex ? !first : (accumulate || !first);
        if (stage2_gather_pays(c, (int64_t)(g.ns_est - g.extra_est), g.A.n, g.q_out, w)) {
            Factor Av = g.A;
            Av.p = g.A.p + lo;
            stage2_gather16(c, g.smp, Av, Sh + s * slab_h, Sl + s * slab_h, g.W, Sk + s * slab_k, skld, w, coef, acc, dst);
        } else {
            gemm_nt_sampled(c, operand_col_offset(g.A.op, lo), so, g.A.n, g.q_out, w, g.smp, coef, acc, dst,
                            df ? &df->parts : nullptr);
        }
        first = false;
    }
    if (P.uex) uex_finish(c, P, g, partial, accumulate, out);
}

static void run_group(gvt_ctx *c, const Problem &P, GroupPlan &g, const float *p_full, float coef, int accumulate,
                      float *out, bool values_ready = false, DenseFuse *df = nullptr) {
    c->last_engine = g.engine;
    c->last_exchange = !distributed(c) ? 0 : (P.uex ? 2 : 1);
    if (g.engine == 2 && fused_f16(c, g.C.cols)) {
        run_group_f16(c, P, g, p_full, coef, accumulate, out, df);
        return;
    }
    // ---- stage 1 on this rank's X-row slab(s)
    for (int s = 0; s < g.nslab; s++) {
        if (!my_slab(c, s)) continue;
        const int64_t lo = g.bounds[s], w = g.bounds[s + 1] - lo;
        const int64_t k0 = g.kpos[s], k1 = g.kpos[s + 1];
        float *Ss = g.S + (size_t)s * g.qpad * g.W;
        if (!values_ready && k1 > k0) {
            EntryPlan ev = g.ent;
            ev.src = g.ent.src + k0;
            ev.sign = g.ent.sign + k0;
            ev.val = g.ent.val + k0;
            ev.nnz = k1 - k0;
            entry_values(c, ev, p_full);
        }
        if (g.engine == 2) {
            const int64_t ldX = round_up(g.C.cols > 0 ? g.C.cols : 1, 32);  // X slab: w x q_in
            const int64_t rows_pad = round_up(w > 0 ? w : 1, 128);
            float *X = wsT<float>(c, "dense.X", (size_t)rows_pad * ldX);
            densify(c, g.ent, k0, k1, lo, X, ldX, rows_pad);
            if (g.diag) add_diag(c, X, ldX, g.diag, lo, w);
            Operand xo = make_operand(c, "dense.Xop", X, w, g.C.cols, ldX, ldX, rows_pad);
            gemm_nt_store(c, g.C.op, xo, g.q_out, w, g.C.cols, Ss, g.W, nullptr, nullptr);
        } else {
            EntryPlan es = g.ent;
            es.row_ptr = g.ent.row_ptr + lo;
            es.nrow = w;
            stage1_sparse(c, es, g.C.colwise(), g.q_out, Ss, g.W, g.diag, lo);
        }
    }
    // ---- exchange the S slabs (NVLink all-gather), then stage 2 slab by slab; or (u-exchange)
    // stage 2 of this rank's slab over every output into a partial vector, then reduce it
    float *partial = nullptr;
    const bool piped = !P.uex && slab_pipeline_available(c);
    if (P.uex) {
        partial = wsT<float>(c, "uex.partial", (size_t)(P.n_out_full + g.n_diag));
        GVT_CUDA_TRY(cudaMemsetAsync(partial, 0, sizeof(float) * (P.n_out_full + g.n_diag), c->stream));
    } else if (piped) {
        void *bufs[1] = {g.S};
        const size_t bytes[1] = {sizeof(float) * (size_t)g.qpad * g.W};
        slab_pipeline_start(c, bufs, bytes, 1);
    } else {
        allgather_slabs(c, g.S, (size_t)g.qpad * g.W);
    }
    float *dst = P.uex ? partial : out;
    bool first = true;
    for (int s = 0; s < g.nslab; s++) {
        const int64_t lo = g.bounds[s], w = g.bounds[s + 1] - lo;
        if (piped) slab_wait(c, s);
        if (w == 0 || (P.uex && !my_slab(c, s))) continue;
        const int acc = P.uex ? !first : (accumulate || !first);
        first = false;
        float *Ss = g.S + (size_t)s * g.qpad * g.W;
        if (g.engine == 2 && !stage2_gather_pays(c, (int64_t)(g.ns_est - g.extra_est), g.A.n, g.q_out, w)) {
            char nm[48];
            snprintf(nm, sizeof(nm), "dense.Sop%d", s);
            Operand so = make_operand(c, nm, Ss, g.q_out, w, g.W, g.W, g.qpad);
            gemm_nt_sampled(c, operand_col_offset(g.A.op, lo), so, g.A.n, g.q_out, w, g.smp, coef, acc, dst);
        } else {
            Factor Av = g.A;
            Av.p = g.A.p + lo;
            stage2_gather(c, g.smp, Av, Ss, g.W, w, coef, acc, dst);
        }
    }
    if (P.uex) uex_finish(c, P, g, partial, accumulate, out);
}

// The fused CG tail (single GPU; the forms that end in a gather-combine: Linear, Ranking, Poly2D): the
// matvec's final combine also takes the ridge term Ap = u + lambda p, the p.Ap partials and the alpha
// step (cg.cu k_cg_combine_ap), one vector pass and one launch fewer per CG iteration; C4 Ranking
// 93.4-94.0 -> 83.8-85.2 us per iteration (profiles/r02_ab_cg_tail.txt).  Optionally (GVT_CG_TAIL_LAZY=1;
// Linear / Ranking) the segment sums also form the direction on the fly, p = r + beta p (beta = st[2]),
// dropping k_cg_p -- measured slower (the extra gather of r costs more than the pass it saves).
struct CgTail {
    const float *r = nullptr;  // r_{k-1}
    double *st = nullptr;      // CG state (st[2] = beta)
    double lambda = 0.0;
    float *p = nullptr;        // p_{k-1} in, p_k out
    // persistent tail (tail.cu): the final combine is left to the tail launch, described here
    bool defer = false;
    GatherCombine gc;
};

// the cheap forms' final combine: fused into the CG tail (k_cg_combine_ap), deferred to the persistent tail, or plain
static void cheap_combine(gvt_ctx *c, const Problem &P, const float *g1, int rs1, float c1, const float *g2, int rs2,
                          float c2, int accumulate, float *u, CgTail *tail) {
    if (tail && tail->defer) {
        GatherCombine &g = tail->gc;
        g.f = P.of;
        g.s = P.os;
        g.g1 = g1;
        g.rs1 = rs1;
        g.c1 = c1;
        g.g2 = g2;
        g.rs2 = rs2;
        g.c2 = c2;
        g.accumulate = accumulate;
    } else if (tail) {
        cg_combine_ap(c, P.of, P.os, P.n_out, g1, rs1, c1, g2, rs2, c2, accumulate, u, tail->p, tail->r, tail->lambda,
                      tail->st);
    } else {
        combine_gather(c, P.of, P.os, P.n_out, g1, rs1, c1, g2, rs2, c2, accumulate, u);
    }
}

static bool cg_tail_enabled() {  // A/B knob: GVT_CG_TAIL=0 keeps the separate CG vector kernels
    static const bool on = [] {
        const char *e = getenv("GVT_CG_TAIL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

static bool dense_tail_enabled() {  // A/B knob: GVT_DENSE_TAIL=0 keeps the separate kernels on the dense engine
    static const bool on = [] {
        const char *e = getenv("GVT_DENSE_TAIL");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

// A/B knob, default off: GVT_CHEAP_TAIL=1 runs the cheap forms' tail (combine, Ap, alpha, x / r, beta, p) as one
// persistent launch.  Bit-identical, but slower at C4 sizes (n = 2e6: Ranking 82-86 -> 88-110 us per iteration at
// 2-8 CTAs per SM, profiles/r02_ab_cheap_tail.txt): the separate kernels' 1184 independent blocks keep more of the
// vector traffic in flight than a co-resident grid between its barriers.
static bool cheap_tail_enabled() {
    static const bool on = [] {
        const char *e = getenv("GVT_CHEAP_TAIL");
        return e && atoi(e) != 0;
    }();
    return on;
}

static bool cg_tail_lazy() {  // A/B knob: GVT_CG_TAIL_LAZY=1 also folds the direction update (k_cg_p)
    static const bool on = [] {
        const char *e = getenv("GVT_CG_TAIL_LAZY");
        return e && atoi(e) != 0;
    }();
    return on;
}

static void run_matvec(gvt_ctx *c, const Problem &P, MatvecPlan &mp, const float *p_local, float *u,
                       CgTail *tail = nullptr) {
    // gather p over the ranks (world 1: p_full is p_local itself)
    const float *p = p_local;
    if (distributed(c)) {
        gather_varlen(c, p_local, P.p_full, P.counts, P.offsets, true);
        p = P.p_full;
    }
    switch (mp.form) {
    case FORM_KRON:
    case FORM_SYM:
    case FORM_ANTI:
        run_group(c, P, mp.groups[0], p, mp.groups[0].coef, 0, u);
        break;
    case FORM_MLPK:
        segment_sum_gather(c, mp.byF, p, mp.groups[0].diag);  // diag(L) = bF + bS
        run_group(c, P, mp.groups[0], p, 1.f, 0, mp.buf);
        combine_mlpk(c, P.of, P.os, P.n_out, mp.buf, u);
        break;
    case FORM_POLY2D: {
        GroupPlan &g = mp.groups[0];
        if (g.ent.ident) {  // entry k = pair k with sign +1 (sorted-order fit): the entry values are p itself
            float *const vals = g.ent.val;
            g.ent.val = const_cast<float *>(p);
            run_group(c, P, g, p, 2.f, 0, u, true);
            segment_sum(c, g.ent, mp.b1);
            g.ent.val = vals;
        } else {
            entry_values(c, g.ent, p);           // all entries: the segment sums need every row
            run_group(c, P, g, p, 2.f, 0, u, true);
            segment_sum(c, g.ent, mp.b1);       // bF (entries of the Kronecker group, rows = first)
        }
        segment_sum_gather(c, mp.byS, p, mp.b2);  // bS
        gemv(c, P.D, mp.b1, 1, mp.g1, !P.rect);  // D.^2 bF
        gemv(c, P.T, mp.b2, 1, mp.g2, !P.rect);  // T.^2 bS
        cheap_combine(c, P, mp.g1, GVT_SEL_FIRST, 1.f, mp.g2, GVT_SEL_SECOND, 1.f, 1, u, tail);
        break;
    }
    case FORM_LINEAR:
        segment_sum_gather(c, mp.byF, p, mp.b1, tail ? tail->r : nullptr, tail ? tail->st + 2 : nullptr);
        segment_sum_gather(c, mp.byS, p, mp.b2, tail ? tail->r : nullptr, tail ? tail->st + 2 : nullptr);
        gemv(c, P.D, mp.b1, 0, mp.g1, !P.rect);
        gemv(c, P.T, mp.b2, 0, mp.g2, !P.rect);
        cheap_combine(c, P, mp.g1, GVT_SEL_FIRST, 1.f, mp.g2, GVT_SEL_SECOND, 1.f, 0, u, tail);
        break;
    case FORM_RANKING:
        segment_sum_gather(c, mp.byF, p, mp.b1, tail ? tail->r : nullptr, tail ? tail->st + 2 : nullptr);  // bF - bS
        gemv(c, P.D, mp.b1, 0, mp.g1, !P.rect);
        cheap_combine(c, P, mp.g1, GVT_SEL_FIRST, 1.f, mp.g1, GVT_SEL_SECOND, -1.f, 0, u, tail);
        break;
    case FORM_CARTESIAN:
        if (mp.cart_dense) {  // u = (D X + X T) sampled: two 3xFP16 GEMMs, the second accumulating
            c->last_engine = 2;
            const Operand xt = build_x16(c, "cart.XT16", mp.byS, 0, P.q, P.m, p);  // rows t of X^T
            gemm_nt_sampled(c, P.D.op, xt, P.m, P.q, P.m, mp.cart_smp, 1.f, 0, u);
            const Operand xo = build_x16(c, "cart.X16", mp.byF, 0, P.m, P.q, p);   // rows d of X
            gemm_nt_sampled(c, xo, P.T.op, P.m, P.q, P.q, mp.cart_smp, 1.f, 1, u);
            break;
        }
        c->last_engine = 1;
        entry_values(c, mp.byF, p);
        entry_values(c, mp.byS, p);
        cartesian(c, P.of, P.os, P.n_out, mp.byF, mp.byS, P.D, P.T, u);
        break;
    case FORM_GENERIC:
        for (size_t i = 0; i < mp.groups.size(); i++) run_group(c, P, mp.groups[i], p, mp.groups[i].coef, i > 0, u);
        if (mp.groups.empty() && P.n_out > 0) GVT_CUDA_TRY(cudaMemsetAsync(u, 0, sizeof(float) * P.n_out, c->stream));
        break;
    }
}

// ----------------------------------------------------------------------------- factors
// rows x cols factor (square Gram: rows = cols; rectangular cross-Gram: rows = out-domain,
// cols = in-domain, plus the transposed copy the sparse stage 1 reads)
static Factor prepare_factor(gvt_ctx *c, const char *name, const float *user, int64_t rows, int64_t cols,
                             bool need_split, bool rect) {
    Factor f;
    f.n = rows;
    f.cols = cols;
    f.ld = round_up(cols > 0 ? cols : 1, 32);
    int64_t rows_pad = round_up(rows > 0 ? rows : 1, 128);
    std::string nm(name);
    // zero-copy: a device Gram whose rows are already 32-float multiples and 16-byte aligned is
    // read in place by the SIMT kernels (they never touch rows >= rows or columns >= ld); the
    // tensor-core split and the transposed rectangular copy still take the padded copy
    if (!need_split && !rect && rows > 0 && cols > 0 && cols % 32 == 0 && ((uintptr_t)user & 15) == 0 &&
        is_device_ptr(user)) {
        f.p = user;
        return f;
    }
    float *d = wsT<float>(c, (nm + ".pad").c_str(), (size_t)rows_pad * f.ld);
    const float *src = user;
    if (rows > 0 && cols > 0) {
        if (!is_device_ptr(user)) {
            float *tmp = wsT<float>(c, (nm + ".h2d").c_str(), (size_t)rows * cols);
            GVT_CUDA_TRY(cudaMemcpyAsync(tmp, user, sizeof(float) * rows * cols, cudaMemcpyHostToDevice, c->stream));
            src = tmp;
        }
        pad_copy(c, src, rows, cols, cols, d, f.ld, rows_pad);
    } else {
        GVT_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(float) * rows_pad * f.ld, c->stream));
    }
    f.p = d;
    if (rect) {
        f.ldt = round_up(rows > 0 ? rows : 1, 32);
        const int64_t cp = round_up(cols > 0 ? cols : 1, 32);
        float *t = wsT<float>(c, (nm + ".T").c_str(), (size_t)cp * f.ldt);
        transpose_pad(c, d, rows_pad, f.ld, f.ld, t, f.ldt, cp);
        f.pt = t;
    }
    if (need_split) {
        f.op = make_operand(c, (nm + ".op").c_str(), d, rows, cols, f.ld, f.ld, rows_pad);
        f.split = true;
    }
    return f;
}

// stage caller ids / vectors and validate ranges (before any compute)
static const int32_t *stage_ids(gvt_ctx *c, const char *name, const int32_t *p, int64_t n) {
    if (n == 0) return nullptr;
    GVT_REQUIRE(p, GVT_E_DIM, std::string(name) + " is NULL with n > 0");
    return (const int32_t *)stage_in(c, name, p, sizeof(int32_t) * n);
}

static void check_range(gvt_ctx *c, const int32_t *ids, int64_t n, int64_t bound, const char *what) {
    if (n == 0) return;
    int64_t bad = count_out_of_range(c, ids, n, bound);
    if (bad) throw Error{GVT_E_INDEX, std::string(what) + ": " + std::to_string(bad) + " id(s) out of range [0, " +
                                          std::to_string(bound) + ")"};
}

struct OutArr {
    float *dev = nullptr;
    float *user = nullptr;
    int64_t n = 0;
    bool host = false;
};

static OutArr out_arr(gvt_ctx *c, const char *name, float *user, int64_t n) {
    OutArr o;
    o.user = user;
    o.n = n;
    if (n == 0) return o;
    GVT_REQUIRE(user, GVT_E_DIM, std::string(name) + " is NULL with n > 0");
    o.host = !is_device_ptr(user);
    o.dev = o.host ? wsT<float>(c, name, n) : user;
    return o;
}

static void out_finish(gvt_ctx *c, OutArr &o) {
    if (o.host && o.n > 0) {
        GVT_CUDA_TRY(cudaMemcpyAsync(o.user, o.dev, sizeof(float) * o.n, cudaMemcpyDeviceToHost, c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
}

// does this plan need the tensor-core split of the factors (any dense group)?
static bool needs_split(gvt_ctx *c, Form form, const Problem &P) {
    if (form == FORM_CARTESIAN) return cart_dense_possible(c, P);
    if (!tc_available(c) || c->engine == 1) return false;
    if (form == FORM_LINEAR || form == FORM_RANKING) return false;
    if (c->engine == 2) return true;
    const bool hom = !(form == FORM_KRON || form == FORM_POLY2D || form == FORM_GENERIC);
    const double mult = (form == FORM_SYM || form == FORM_ANTI || form == FORM_MLPK) ? 2.0 : 1.0;  // entries per pair
    const int64_t q_in = hom ? P.m : P.q, q_out = hom ? P.m_out : P.q_out;
    const double ns = (P.uex ? (double)P.n_out_full : (double)P.n_out_all / (distributed(c) ? c->world : 1)) +
                      (form == FORM_MLPK ? (double)P.m_out : 0.0);
    // the estimate of the problem's main Kronecker group (the same one choose_engine makes per group)
    return dense_pays(c, mult * (double)P.n_in, ns, P.m_out, q_out, P.m, q_in);
}

// out_is_in: the out sample is the caller's in sample (fit)
// m_out / q_out < 0: square Grams over global ids (out dims = in dims); else rectangular
// cross-Grams D (m_out x m) and T (q_out x q) of novel objects
static void setup_problem(gvt_ctx *c, Problem &P, const float *D, int64_t m, const float *T, int64_t q,
                          const int32_t *of, const int32_t *os, int64_t n_out, const int32_t *inf,
                          const int32_t *ins, int64_t n_in, const gvt_term *terms, int n_terms, Form &form,
                          bool out_is_in, int64_t m_out = -1, int64_t q_out = -1) {
    GVT_REQUIRE(m >= 0 && n_out >= 0 && n_in >= 0, GVT_E_DIM, "negative size");
    P.hom = (T == nullptr);
    P.rect = m_out >= 0;
    P.m = m;
    P.q = P.hom ? m : q;
    P.m_out = P.rect ? m_out : P.m;
    P.q_out = P.rect ? (P.hom ? m_out : q_out) : P.q;
    GVT_REQUIRE(P.q >= 0 && P.q_out >= 0, GVT_E_DIM, "negative q");
    GVT_REQUIRE((m == 0 || P.m_out == 0) || D, GVT_E_DIM, "D is NULL with m > 0");
    GVT_REQUIRE(P.hom || (P.q == 0 || P.q_out == 0) || T, GVT_E_DIM, "T is NULL");
    form = recognize(terms, n_terms);
    validate_terms(terms, n_terms, P.hom, form, P.rect);
    P.n_out = n_out;
    P.of = stage_ids(c, "in.of", of, n_out);
    P.os = stage_ids(c, "in.os", os, n_out);
    const int32_t *lf = out_is_in ? P.of : stage_ids(c, "in.inf", inf, n_in);
    const int32_t *ls = out_is_in ? P.os : stage_ids(c, "in.ins", ins, n_in);
    check_range(c, P.of, n_out, P.m_out, "out first ids");
    check_range(c, P.os, n_out, P.q_out, "out second ids");
    if (!out_is_in) {
        check_range(c, lf, n_in, P.m, "in first ids");
        check_range(c, ls, n_in, P.q, "in second ids");
    }
    // in-sample over all ranks
    P.counts = allgather_count(c, n_in);
    P.offsets.assign(P.counts.size() + 1, 0);
    for (size_t g = 0; g < P.counts.size(); g++) P.offsets[g + 1] = P.offsets[g] + P.counts[g];
    P.n_in = P.offsets.back();
    P.n_out_all = out_is_in ? P.n_in : n_out;
    if (distributed(c) && !out_is_in) {
        P.out_counts = allgather_count(c, n_out);
        P.n_out_all = 0;
        for (int64_t v : P.out_counts) P.n_out_all += v;
    }
    if (distributed(c)) {
        int32_t *ff = wsT<int32_t>(c, "dist.f", (size_t)P.n_in);
        int32_t *fs = wsT<int32_t>(c, "dist.s", (size_t)P.n_in);
        gather_varlen(c, lf, ff, P.counts, P.offsets, false);
        gather_varlen(c, ls, fs, P.counts, P.offsets, false);
        P.inf = ff;
        P.ins = fs;
        P.p_full = wsT<float>(c, "dist.p", (size_t)P.n_in);
    } else {
        P.inf = lf;
        P.ins = ls;
    }
    // u-exchange needs every rank's out pairs on every rank (a fit's out sample is its in-sample)
    // (also at world 1, where the reduce is a copy: the single-GPU tests exercise this path).
    // Auto (2): both exchanges give every rank the same stage-2 work (its slab's K-range over all
    // outputs, or all of K over its own outputs), so the choice is by bytes moved: 4 n_out (all
    // ranks) per matvec vs 4 q_out m_in for the S slabs -- rank-independent sizes, the same choice
    // on every rank.  Single-GPU mode has no exchange (auto = 0).
    if (c->exchange == 2) {
        const double cells = (double)P.q_out * (double)P.m;
        P.uex = distributed(c) && (double)P.n_out_all + (double)P.m_out < cells;
    } else {
        P.uex = c->exchange == 1;
    }
    if (P.uex) {
        if (out_is_in) {
            P.of_full = P.inf;
            P.os_full = P.ins;
            P.out_counts = P.counts;
            P.out_offsets = P.offsets;
        } else {
            if (P.out_counts.empty()) P.out_counts = allgather_count(c, n_out);
            P.out_offsets.assign(P.out_counts.size() + 1, 0);
            for (size_t g = 0; g < P.out_counts.size(); g++)
                P.out_offsets[g + 1] = P.out_offsets[g] + P.out_counts[g];
            int32_t *gf = wsT<int32_t>(c, "dist.of", (size_t)P.out_offsets.back());
            int32_t *gs = wsT<int32_t>(c, "dist.os", (size_t)P.out_offsets.back());
            gather_varlen(c, P.of, gf, P.out_counts, P.out_offsets, false);
            gather_varlen(c, P.os, gs, P.out_counts, P.out_offsets, false);
            P.of_full = gf;
            P.os_full = gs;
        }
        P.n_out_full = P.out_offsets.back();
    }
    bool split = needs_split(c, form, P);
    P.D = prepare_factor(c, "fD", D, P.m_out, P.m, split, P.rect);
    P.T = P.hom ? P.D : prepare_factor(c, "fT", T, P.q_out, P.q, split, P.rect);
}

// ----------------------------------------------------------------------------- entry points
static void matvec_impl(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *of,
                        const int32_t *os, int64_t n_out, const int32_t *inf, const int32_t *ins, int64_t n_in,
                        const float *a, const gvt_term *terms, int n_terms, float *u, int64_t m_out = -1,
                        int64_t q_out = -1) {
    Problem P;
    Form form;
    setup_problem(c, P, D, m, T, q, of, os, n_out, inf, ins, n_in, terms, n_terms, form, false, m_out, q_out);
    OutArr uo = out_arr(c, "out.u", u, n_out);
    const float *ad = n_in ? (const float *)stage_in(c, "in.a", a, sizeof(float) * n_in) : nullptr;
    GVT_REQUIRE(n_in == 0 || ad, GVT_E_DIM, "a is NULL with n_in > 0");
    if (P.n_in == 0) {  // no in pairs anywhere: u = 0 (collective-free on every rank)
        if (n_out) GVT_CUDA_TRY(cudaMemsetAsync(uo.dev, 0, sizeof(float) * n_out, c->stream));
    } else {
        MatvecPlan mp;
        plan_matvec(c, P, terms, n_terms, form, mp);
        run_matvec(c, P, mp, ad, uo.dev);
    }
    out_finish(c, uo);
}

// Used-object compaction of a matvec / predict (GVT_OPT_COMPACT; the fit's counterpart is
// compact_fit): when the in- or out-sample uses less than half of the Grams' objects, the GVT runs
// on the cross-Grams of the used objects, D[out objects][in objects] (and T likewise), through the
// rectangular path -- whose Theorem 1 variant is then chosen by cost, as in the paper.  Kernels
// with an Identity factor (Cartesian) keep the square path (reading N1: identity across two
// object tables); anything invalid is left to the square path's own checks and errors.
void matvec_rect(gvt_ctx *c, const float *Dx, int64_t m_out, int64_t m_in, const float *Tx, int64_t q_out,
                 int64_t q_in, const int32_t *of, const int32_t *os, int64_t n_out, const int32_t *inf,
                 const int32_t *ins, int64_t n_in, const float *a, const gvt_term *terms, int n_terms, int variant,
                 float *u, int *variant_used, int64_t *op_count);

// GVT_OPT_COMPACT = 1 (auto) skips small tables (<= 2^20 Gram cells: C1, C2), which are latency-bound
// either way and where the check itself (one read-back) would cost more than it saves; 2 = always
constexpr double COMPACT_MIN_CELLS = 1048576.0;
static bool compact_small_skip(gvt_ctx *c, int64_t m, int64_t qq) {
    return c->compact == 1 && (double)m * (double)qq <= COMPACT_MIN_CELLS;
}

static bool compact_matvec(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *of,
                           const int32_t *os, int64_t n_out, const int32_t *inf, const int32_t *ins, int64_t n_in,
                           const float *a, const gvt_term *terms, int n_terms, float *u) {
    if (!c->compact || distributed(c) || n_in <= 0 || n_out <= 0 || m <= 0 || !terms || n_terms < 1 || n_terms > 64)
        return false;
    if (!of || !os || !inf || !ins || !a || !u || !D) return false;
    if (compact_small_skip(c, m, T ? q : m)) return false;
    const bool hom = T == nullptr;
    const Form form = recognize(terms, n_terms);
    if (form == FORM_CARTESIAN || (form_homogeneous(form) && !hom)) return false;
    for (int i = 0; i < n_terms; i++) {
        const int kinds[2] = {terms[i].left, terms[i].right};
        for (int k = 0; k < 2; k++)
            if (kinds[k] < 0 || kinds[k] > 3 || kinds[k] == GVT_FACTOR_IDENTITY) return false;
    }
    const int64_t qq = hom ? m : q;
    const int32_t *ofd = (const int32_t *)stage_in(c, "cmv.of", of, sizeof(int32_t) * n_out);
    const int32_t *osd = (const int32_t *)stage_in(c, "cmv.os", os, sizeof(int32_t) * n_out);
    const int32_t *ifd = (const int32_t *)stage_in(c, "cmv.if", inf, sizeof(int32_t) * n_in);
    const int32_t *isd = (const int32_t *)stage_in(c, "cmv.is", ins, sizeof(int32_t) * n_in);
    unsigned long long *cnt = wsT<unsigned long long>(c, "cmv.cnt", 4);
    GVT_CUDA_TRY(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), c->stream));
    UsedSet od, ot, id, it;  // out drugs, out targets, in drugs, in targets (hom: od == ot, id == it)
    if (hom) {
        const int32_t *ao[2] = {ofd, osd}, *ai[2] = {ifd, isd};
        const int64_t lo[2] = {n_out, n_out}, li[2] = {n_in, n_in};
        od = used_set_begin(c, "cmv.od", m, ao, lo, 2, cnt);
        id = used_set_begin(c, "cmv.id", m, ai, li, 2, cnt + 1);
    } else {
        od = used_set_begin(c, "cmv.od", m, &ofd, &n_out, 1, cnt);
        ot = used_set_begin(c, "cmv.ot", q, &osd, &n_out, 1, cnt + 1);
        id = used_set_begin(c, "cmv.id", m, &ifd, &n_in, 1, cnt + 2);
        it = used_set_begin(c, "cmv.it", q, &isd, &n_in, 1, cnt + 3);
    }
    unsigned long long h_cnt[4];
    int64_t h_k[4] = {0, 0, 0, 0};
    GVT_CUDA_TRY(cudaMemcpyAsync(h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, c->stream));
    const int nsets = hom ? 2 : 4;
    const UsedSet *uniq[4] = {&od, &id, &ot, &it};
    for (int k = 0; k < nsets; k++)
        GVT_CUDA_TRY(cudaMemcpyAsync(&h_k[k], uniq[k]->k_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (h_cnt[0] || h_cnt[1] || h_cnt[2] || h_cnt[3]) return false;  // the square path reports the index error
    od.k = h_k[0];
    id.k = h_k[1];
    if (hom) {
        ot = od;
        it = id;
    } else {
        ot.k = h_k[2];
        it.k = h_k[3];
    }
    const double full = (double)m * (double)qq;
    if ((double)id.k * (double)it.k >= 0.5 * full && (double)od.k * (double)ot.k >= 0.5 * full) return false;
    const float *Dd = (const float *)stage_in(c, "cmv.D_in", D, sizeof(float) * m * m);
    float *Dx = wsT<float>(c, "cmv.D", (size_t)(od.k * id.k));
    sub_gram(c, Dd, m, od, id, Dx);
    float *Tx = nullptr;
    if (!hom) {
        const float *Td = (const float *)stage_in(c, "cmv.T_in", T, sizeof(float) * q * q);
        Tx = wsT<float>(c, "cmv.T", (size_t)(ot.k * it.k));
        sub_gram(c, Td, q, ot, it, Tx);
    }
    int32_t *ofc = wsT<int32_t>(c, "cmv.ofc", (size_t)n_out), *osc = wsT<int32_t>(c, "cmv.osc", (size_t)n_out);
    int32_t *ifc = wsT<int32_t>(c, "cmv.ifc", (size_t)n_in), *isc = wsT<int32_t>(c, "cmv.isc", (size_t)n_in);
    map_ids(c, od, ofd, n_out, ofc);
    map_ids(c, ot, osd, n_out, osc);
    map_ids(c, id, ifd, n_in, ifc);
    map_ids(c, it, isd, n_in, isc);
    matvec_rect(c, Dx, od.k, id.k, Tx, ot.k, it.k, ofc, osc, n_out, ifc, isc, n_in, a, terms, n_terms, 0, u, nullptr,
                nullptr);
    return true;
}

void matvec(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *of, const int32_t *os,
            int64_t n_out, const int32_t *inf, const int32_t *ins, int64_t n_in, const float *a,
            const gvt_term *terms, int n_terms, float *u) {
    if (compact_matvec(c, D, m, T, q, of, os, n_out, inf, ins, n_in, a, terms, n_terms, u)) return;
    matvec_impl(c, D, m, T, q, of, os, n_out, inf, ins, n_in, a, terms, n_terms, u);
}

// Novel objects (Settings 2-4): rectangular cross-Grams Dx (m_out x m_in) and
// Tx (q_out x q_in, NULL = homogeneous), out ids index rows, in ids columns.  For the Kronecker
// list the GVT variant follows Theorem 1's cost (SPEC.md gvt_cost): variant 1
// (stage 1 over the target factor) costs q_out n_in + m_in n_out, variant 2 (the roles of the
// two factors swapped) m_out n_in + q_in n_out; auto takes the smaller, ties -> 1 (reading S2).
// Variant 2 runs as variant 1 of the swapped problem (Tx, Dx) with the pair elements swapped.
void matvec_rect(gvt_ctx *c, const float *Dx, int64_t m_out, int64_t m_in, const float *Tx, int64_t q_out,
                 int64_t q_in, const int32_t *of, const int32_t *os, int64_t n_out, const int32_t *inf,
                 const int32_t *ins, int64_t n_in, const float *a, const gvt_term *terms, int n_terms, int variant,
                 float *u, int *variant_used, int64_t *op_count) {
    GVT_REQUIRE(m_out >= 0 && m_in >= 0 && n_out >= 0 && n_in >= 0, GVT_E_DIM, "negative size");
    GVT_REQUIRE(Tx == nullptr || (q_out >= 0 && q_in >= 0), GVT_E_DIM, "negative size");
    GVT_REQUIRE(variant >= 0 && variant <= 2, GVT_E_PARAM, "variant must be 0 (auto), 1 or 2");
    GVT_REQUIRE(terms && n_terms >= 1, GVT_E_KERNEL, "term list empty");
    const bool hom = Tx == nullptr;
    if (hom) {
        q_out = m_out;
        q_in = m_in;
    }
    const bool kron = recognize(terms, n_terms) == FORM_KRON;
    GVT_REQUIRE(variant != 2 || kron, GVT_E_PARAM, "variant 2 is defined for the Kronecker term list only");
    const int64_t c1 = q_out * n_in + m_in * n_out, c2 = m_out * n_in + q_in * n_out;
    int v = variant ? variant : ((kron && c2 < c1) ? 2 : 1);
    if (variant_used) *variant_used = v;
    if (op_count) *op_count = kron ? (v == 1 ? c1 : c2) : -1;
    if (v == 1)
        matvec_impl(c, Dx, m_in, Tx, q_in, of, os, n_out, inf, ins, n_in, a, terms, n_terms, u, m_out, q_out);
    else
        matvec_impl(c, hom ? Dx : Tx, q_in, hom ? nullptr : Dx, m_in, os, of, n_out, ins, inf, n_in, a, terms,
                    n_terms, u, q_out, m_out);
}

void predict(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *tf, const int32_t *ts,
             int64_t n_test, const int32_t *trf, const int32_t *trs, int64_t n_train, const float *a,
             const gvt_term *terms, int n_terms, float *scores) {
    matvec(c, D, m, T, q, tf, ts, n_test, trf, trs, n_train, a, terms, n_terms, scores);
}

// Early-stopping arguments (pairwise_krr_fit_early_stopping); nullptr for a plain fit.
struct EsArgs {
    const int32_t *vf = nullptr, *vs = nullptr;  // this rank's validation pairs
    int64_t n_val = 0;
    const float *vlab = nullptr;
    int patience = 1;
    int *best_iter = nullptr;
    double *best_auc = nullptr;
    double *auc_hist = nullptr;  // host, max_iter entries (iteration k at [k - 1])
    float *scores_out = nullptr; // unused (reserved)
};

// Replay `body` max_iter times: the first iteration eagerly (workspaces settle), the rest as
// one captured CUDA graph when allowed (the loop is launch-bound on small problems; all
// solver control lives on the device, so replays are exact).  With `poll` the host checks
// the device DONE/BREAK flags with a one-iteration lag and stops launching once set.
template <class Body>
static void drive(gvt_ctx *c, int max_iter, bool poll, const double *state, Body body) {
    double *hst = (double *)pinned(c, sizeof(double) * 64);
    const bool graphs = c->graphs && max_iter >= 3 && !c->profile && !c->host_allgather;  // host collectives sync
    cudaGraphExec_t exec = nullptr;
    cudaGraph_t graph = nullptr;
    int64_t per_iter = 0, l0 = 0, before[K_NUM_KINDS];
    int it = 0, replays = 0;
    cudaEvent_t evs[2] = {nullptr, nullptr};
    if (poll) {
        GVT_CUDA_TRY(cudaEventCreateWithFlags(&evs[0], cudaEventDisableTiming));
        GVT_CUDA_TRY(cudaEventCreateWithFlags(&evs[1], cudaEventDisableTiming));
    }
    auto cleanup = [&]() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        for (auto &e : evs)
            if (e) cudaEventDestroy(e);
    };
    try {
        for (; it < max_iter; it++) {
            if (graphs && it == 1) {
                if (!c->cap_stream) GVT_CUDA_TRY(cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking));
                cudaStream_t user = c->stream;
                l0 = c->launches;
                for (int k = 0; k < K_NUM_KINDS; k++) before[k] = c->counts[k];
                c->stream = c->cap_stream;
                GVT_CUDA_TRY(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
                try {
                    body();
                } catch (...) {
                    cudaStreamEndCapture(c->cap_stream, &graph);
                    c->stream = user;
                    throw;
                }
                cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &graph);
                c->stream = user;
                GVT_CUDA_TRY(ce);
                GVT_CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
                per_iter = c->launches - l0;
            }
            if (exec) {
                GVT_CUDA_TRY(cudaGraphLaunch(exec, c->stream));
                replays++;
            } else {
                body();
            }
            if (poll) {
                // flags after iteration `it` -> hst[8 * (it & 1)]; check iteration it - 1's copy
                GVT_CUDA_TRY(cudaMemcpyAsync(hst + 8 * (it & 1), state + 5, sizeof(double) * 2, cudaMemcpyDeviceToHost,
                                             c->stream));
                GVT_CUDA_TRY(cudaEventRecord(evs[it & 1], c->stream));
                if (it >= 1) {
                    GVT_CUDA_TRY(cudaEventSynchronize(evs[(it - 1) & 1]));
                    const double *h = hst + 8 * ((it - 1) & 1);
                    if (h[0] != 0.0 || h[1] != 0.0) {
                        it++;
                        break;
                    }
                }
            }
        }
    } catch (...) {
        cleanup();
        throw;
    }
    if (exec) {  // launch accounting: the captured kernels ran once per replay
        c->launches = l0 + per_iter * replays;
        for (int k = 0; k < K_NUM_KINDS; k++) c->counts[k] = before[k] + (c->counts[k] - before[k]) * replays;
    }
    cleanup();
}

static gvt_status fit_impl(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *f,
                           const int32_t *s, int64_t n, const float *y, const gvt_term *terms, int n_terms,
                           double lambda, int max_iter, double rel_tol, float *a_out, int *iters_out,
                           double *relres_hist, const EsArgs *es) {
    GVT_REQUIRE(lambda >= 0.0, GVT_E_PARAM, "lambda < 0");
    GVT_REQUIRE(max_iter >= 0, GVT_E_PARAM, "max_iter < 0");
    GVT_REQUIRE(rel_tol >= 0.0, GVT_E_PARAM, "rel_tol < 0");
    GVT_REQUIRE(n >= 0, GVT_E_DIM, "negative n");
    const bool minres = c->solver == GVT_SOLVER_MINRES;
    const bool cgg = !minres && c->cg_variant == 1;  // Chronopoulos-Gear single-reduction CG
    GVT_REQUIRE(!(cgg && es), GVT_E_PARAM, "early stopping runs Hestenes-Stiefel CG or MINRES (GVT_OPT_CG_VARIANT = 0)");
    Problem P;
    Form form;
    int64_t n_val = 0;
    if (es) {
        GVT_REQUIRE(es->patience >= 1, GVT_E_PARAM, "patience < 1");
        GVT_REQUIRE(es->n_val >= 0, GVT_E_DIM, "negative n_val");
        n_val = es->n_val;
        // out sample = [inner; validation]: one matvec gives (K + .) v on the inner pairs and
        // K_val,inner v on the validation pairs with a shared stage 1
        const int64_t no = n + n_val;
        int32_t *of = wsT<int32_t>(c, "es.of", (size_t)no), *os = wsT<int32_t>(c, "es.os", (size_t)no);
        const int32_t *pf[2] = {f, es->vf}, *ps[2] = {s, es->vs};
        const int64_t cnt[2] = {n, n_val}, off[2] = {0, n};
        const char *nf[2] = {"es.in_f", "es.val_f"}, *ns[2] = {"es.in_s", "es.val_s"};
        for (int k = 0; k < 2; k++) {
            if (!cnt[k]) continue;
            GVT_REQUIRE(pf[k] && ps[k], GVT_E_DIM, "pair ids are NULL with a non-empty sample");
            const int32_t *df = (const int32_t *)stage_in(c, nf[k], pf[k], sizeof(int32_t) * cnt[k]);
            const int32_t *ds = (const int32_t *)stage_in(c, ns[k], ps[k], sizeof(int32_t) * cnt[k]);
            GVT_CUDA_TRY(cudaMemcpyAsync(of + off[k], df, sizeof(int32_t) * cnt[k], cudaMemcpyDeviceToDevice, c->stream));
            GVT_CUDA_TRY(cudaMemcpyAsync(os + off[k], ds, sizeof(int32_t) * cnt[k], cudaMemcpyDeviceToDevice, c->stream));
        }
        setup_problem(c, P, D, m, T, q, of, os, no, of, os, n, terms, n_terms, form, false);
        P.n_out_extra = P.uex ? P.n_out_full - P.n_in : n_val;
        P.n_out_extra_all = P.n_out_all - P.n_in;  // the validation pairs over all ranks
    } else {
        setup_problem(c, P, D, m, T, q, f, s, n, f, s, n, terms, n_terms, form, true);
    }
    OutArr ao = out_arr(c, "out.a", a_out, n);
    const float *yd = n ? (const float *)stage_in(c, "in.y", y, sizeof(float) * n) : nullptr;
    GVT_REQUIRE(n == 0 || yd, GVT_E_DIM, "y is NULL with n > 0");
    const int SN = minres ? MINRES_STATE_N : 9;
    double *state = wsT<double>(c, "solver.state", (size_t)SN + max_iter + 1);
    // ---- early-stopping plumbing: validation labels over all ranks, AUC plan, device rule state
    AucPlan ap;
    double *esd = nullptr, *ehist = nullptr;
    float *s_val = nullptr, *s_full = nullptr, *a_best = nullptr;
    std::vector<int64_t> vcounts, voffs;
    int64_t nv_all = n_val;
    if (es) {
        GVT_REQUIRE(n_val == 0 || es->vlab, GVT_E_DIM, "validation labels are NULL");
        vcounts = allgather_count(c, n_val);
        voffs.assign(vcounts.size() + 1, 0);
        for (size_t g = 0; g < vcounts.size(); g++) voffs[g + 1] = voffs[g] + vcounts[g];
        nv_all = voffs.back();
        const float *vl = n_val ? (const float *)stage_in(c, "es.vlab", es->vlab, sizeof(float) * n_val) : nullptr;
        float *vl_full = wsT<float>(c, "es.vlab_full", (size_t)nv_all);
        gather_varlen(c, vl, vl_full, vcounts, voffs, true);
        ap.setup(c, "es.auc", vl_full, nv_all);  // errors on single-class labels (before compute)
        esd = wsT<double>(c, "es.state", ES_STATE_N);
        ehist = wsT<double>(c, "es.hist", (size_t)(max_iter > 0 ? max_iter : 1));
        s_val = wsT<float>(c, "es.s", (size_t)n_val);
        s_full = distributed(c) ? wsT<float>(c, "es.s_full", (size_t)nv_all) : s_val;
        a_best = ao.dev;  // the weights returned are those of the best iteration
        if (n_val) GVT_CUDA_TRY(cudaMemsetAsync(s_val, 0, sizeof(float) * n_val, c->stream));
        es_init(c, esd, ehist, max_iter, ap);
    }
    auto finish_es = [&](int iters) {
        if (!es) return;
        double h[ES_STATE_N];
        GVT_CUDA_TRY(cudaMemcpyAsync(h, esd, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        if (es->auc_hist && max_iter > 0)
            GVT_CUDA_TRY(cudaMemcpyAsync(es->auc_hist, ehist, sizeof(double) * max_iter, cudaMemcpyDeviceToHost,
                                         c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
        if (es->best_iter) *es->best_iter = (int)h[1];
        if (es->best_auc) *es->best_auc = h[1] > 0 ? h[0] : 0.0 / 0.0;
        if (es->auc_hist)
            for (int k = iters; k < max_iter; k++) es->auc_hist[k] = 0.0 / 0.0;
    };
    if (P.n_in == 0) {
        if (iters_out) *iters_out = 0;
        if (relres_hist) {
            relres_hist[0] = 0.0;
            for (int k = 1; k <= max_iter; k++) relres_hist[k] = 0.0 / 0.0;
        }
        finish_es(0);
        return GVT_OK;
    }
    float *x = es ? wsT<float>(c, "solver.x", (size_t)n) : ao.dev;
    if (es && n) GVT_CUDA_TRY(cudaMemsetAsync(a_best, 0, sizeof(float) * n, c->stream));
    float *u = wsT<float>(c, "solver.u", (size_t)(n + n_val));  // matvec output [inner; validation]
    MatvecPlan mp;
    plan_matvec(c, P, terms, n_terms, form, mp);
    // small Kronecker fits: the whole solve in ONE launch -- single-CTA (tiny.cu; GVT_OPT_ENGINE = 3,
    // or auto when a CG iteration is at most 4e6 FMAs and everything fits in one SM's shared memory),
    // or persistent multi-CTA with grid barriers (small.cu; GVT_OPT_ENGINE = 4, or auto for the
    // problems whose dense stage 1 is at most 6.4e7 FMAs, e.g. the complete C2 grid)
    {
        const bool whole = form == FORM_KRON && !minres && !cgg && !es && !distributed(c) && c->slabs <= 1 &&
                           !P.uex && !P.rect && P.n_in == n;
        const bool eligible = whole && tiny_smem(P.m, P.q, n) > 0;
        const bool eligible4 = whole && small_eligible(P.m, P.q, n);
        const double fmas = (double)n * (double)P.q + (double)n * (double)P.m;
        GVT_REQUIRE(c->engine != 3 || eligible, GVT_E_PARAM,
                    "single-CTA solver (engine 3): Kronecker CG fits on one GPU whose factors, S and vectors fit in "
                    "shared memory only");
        GVT_REQUIRE(c->engine != 4 || eligible4, GVT_E_PARAM,
                    "persistent small solver (engine 4): Kronecker CG fits on one GPU with m q^2 <= 6.4e7 only");
        const bool use3 = eligible && (c->engine == 3 || (c->engine == 0 && fmas <= 4e6));
        const bool use4 = !use3 && eligible4 && (c->engine == 4 || c->engine == 0);
        if (use3 || use4) {
            const GroupPlan &g = mp.groups[0];
            if (use3) tiny_cg(c, P.D, P.T, g.ent, g.smp, P.m, P.q, yd, x, n, lambda, max_iter, rel_tol, state);
            else small_cg(c, P.D, P.T, g.ent, g.smp, P.m, P.q, yd, x, n, lambda, max_iter, rel_tol, state, true);
            c->last_engine = use3 ? 3 : 4;
            double hs[9];
            GVT_CUDA_TRY(cudaMemcpyAsync(hs, state, sizeof(hs), cudaMemcpyDeviceToHost, c->stream));
            if (relres_hist)
                GVT_CUDA_TRY(cudaMemcpyAsync(relres_hist, state + 9, sizeof(double) * (max_iter + 1),
                                             cudaMemcpyDeviceToHost, c->stream));
            GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
            out_finish(c, ao);
            const int iters = (int)hs[7];
            if (iters_out) *iters_out = iters;
            if (relres_hist)
                for (int k = iters + 1; k <= max_iter; k++) relres_hist[k] = 0.0 / 0.0;
            if (hs[6] != 0.0) {
                set_error("CG breakdown: p^T (K + lambda I) p = %g <= 0 at iteration %d", hs[4], iters + 1);
                return GVT_E_BREAKDOWN;
            }
            return GVT_OK;
        }
    }
    auto evaluate = [&]() {
        if (!es) return;
        if (distributed(c)) gather_varlen(c, s_val, s_full, vcounts, voffs, true);
        es_evaluate(c, ap, s_full, state, esd, ehist, es->patience, x, a_best, n);
    };
    float *r1 = nullptr, *r2 = nullptr, *v = nullptr, *W1 = nullptr, *W2 = nullptr, *r = nullptr, *p = nullptr;
    float *KW1 = nullptr, *KW2 = nullptr, *sv = nullptr;
    if (minres) {
        r1 = wsT<float>(c, "mr.r1", n), r2 = wsT<float>(c, "mr.r2", n), v = wsT<float>(c, "mr.v", n);
        W1 = wsT<float>(c, "mr.W1", n), W2 = wsT<float>(c, "mr.W2", n);
        if (n_val) {
            KW1 = wsT<float>(c, "mr.KW1", n_val), KW2 = wsT<float>(c, "mr.KW2", n_val);
            GVT_CUDA_TRY(cudaMemsetAsync(KW1, 0, sizeof(float) * n_val, c->stream));
            GVT_CUDA_TRY(cudaMemsetAsync(KW2, 0, sizeof(float) * n_val, c->stream));
        }
        minres_init(c, yd, n, x, r1, r2, v, W1, W2, state, rel_tol);
    } else if (cgg) {
        r = wsT<float>(c, "cg.r", n), p = wsT<float>(c, "cg.p", n), sv = wsT<float>(c, "cgg.s", n);
        cgg_init(c, yd, n, x, r, p, sv, state, rel_tol);
    } else {
        r = wsT<float>(c, "cg.r", n), p = wsT<float>(c, "cg.p", n);
        cg_init(c, yd, n, x, r, p, state, rel_tol);
        if (!es) {  // kept for gvt_solver_direction (reading S30's in-loop check)
            c->last_p = p;
            c->last_n = n;
        }
    }
    const bool fuse_tail = !minres && !cgg && !es && !distributed(c) && !P.uex && P.n_out == n &&
                           (mp.form == FORM_RANKING || mp.form == FORM_LINEAR || mp.form == FORM_POLY2D) &&
                           cg_tail_enabled();
    // the fused dense-engine CG tail (tail.cu): one persistent launch between the stage-2 GEMM and the next
    // stage-1 GEMM instead of the split-K combine, three CG vector kernels, the S-scale memset and the
    // X(p) build; same arithmetic on the same partitions (bit-identical iterates).  Single GPU, one
    // Kronecker group on the fused fp16 path with warp-per-row X rows.
    GroupPlan *gd = mp.groups.empty() ? nullptr : &mp.groups[0];
    const bool tail_common = !fuse_tail && !minres && !cgg && !es && !distributed(c) && !P.uex && P.n_out == n &&
                             dense_tail_enabled();
    auto short_rows = [&](int64_t cols) {
        const int64_t ld = round_up(cols > 0 ? cols : 1, 32);
        return ld <= 2048 && dense_tail_fits(ld);
    };
    const bool fuse_kron = tail_common && (mp.form == FORM_KRON || mp.form == FORM_SYM || mp.form == FORM_ANTI) && gd &&
                           gd->engine == 2 && fused_f16(c, gd->C.cols) && gd->nslab == 1 && !gd->diag &&
                           short_rows(gd->C.cols);
    // the Cartesian form's two sampled GEMMs (D X^T-side and X T-side) with both pair-matrix operands rebuilt
    const bool fuse_cart = tail_common && mp.form == FORM_CARTESIAN && mp.cart_dense && short_rows(P.m) &&
                           short_rows(P.q);
    bool fuse_dense = fuse_kron || fuse_cart;
    // the cheap forms' tail as one persistent launch too (tail.cu gather-combine mode; not with the lazy direction)
    const bool cheap_persistent = fuse_tail && !cg_tail_lazy() && cheap_tail_enabled();
    double *tail_part2 = nullptr;
    const int32_t *tail_inv = nullptr;
    float *p_alt = nullptr;
    bool tail_first = true;
    if (cheap_persistent) {
        tail_part2 = wsT<double>(c, "tail.part2", RED_BLOCKS);
        dense_tail_init(c, tail_part2, nullptr, 0, 0);
    }
    if (fuse_dense) {
        const SamplePlan &sp = fuse_cart ? mp.cart_smp : gd->smp;
        tail_part2 = wsT<double>(c, "tail.part2", RED_BLOCKS);
        tail_inv = dense_tail_init(c, tail_part2, sp.dst, sp.ns, n);
        if (!tail_inv) fuse_dense = false;  // (some output is not exactly one sample: the separate kernels)
        p_alt = wsT<float>(c, "tail.p_alt", (size_t)n);
    }
    auto iteration = [&]() {
        if (fuse_dense && !fuse_cart) {
            DenseFuse df;
            df.prebuilt = !tail_first;  // iteration 1 builds X(p_0) and zeroes the S scales itself
            tail_first = false;
            run_group(c, P, *gd, p, gd->coef, 0, u, false, &df);
            TailX tx;
            tx.e = &gd->ent;
            tx.row_lo = gd->bounds[0];
            tx.rows = gd->bounds[1] - tx.row_lo;
            tx.op = build_x16(c, "dense.X16", gd->ent, tx.row_lo, tx.rows, gd->C.cols, p, nullptr, false);
            dense_cg_tail(c, df.parts, SplitParts(), tail_inv, u, x, r, p, p_alt, n, cg_vec_blocks(n), lambda, state,
                          cg_parts(c), tail_part2, &tx, 1);
        } else if (fuse_dense) {  // Cartesian: u = (D X + X T) sampled, then the tail rebuilds X^T and X
            const bool build = tail_first;
            tail_first = false;
            c->last_engine = 2;
            TailX tx[2];
            tx[0].e = &mp.byS;  // rows t of X^T (B operand of D X)
            tx[0].rows = P.q;
            tx[0].op = build_x16(c, "cart.XT16", mp.byS, 0, P.q, P.m, p, nullptr, build);
            tx[1].e = &mp.byF;  // rows d of X (A operand of X T)
            tx[1].rows = P.m;
            tx[1].op = build_x16(c, "cart.X16", mp.byF, 0, P.m, P.q, p, nullptr, build);
            // defer the first GEMM's parts only when the second also leaves parts (the second accumulates onto
            // the first's combined values)
            SplitParts pa, pb;
            pa.slot = 0;
            pb.slot = 1;
            const bool defer_a = sampled_split_parts(c, mp.cart_smp, P.q) > 1;
            gemm_nt_sampled(c, P.D.op, tx[0].op, P.m, P.q, P.m, mp.cart_smp, 1.f, 0, u, defer_a ? &pa : nullptr);
            gemm_nt_sampled(c, tx[1].op, P.T.op, P.m, P.q, P.q, mp.cart_smp, 1.f, 1, u, &pb);
            dense_cg_tail(c, pa, pb, tail_inv, u, x, r, p, p_alt, n, cg_vec_blocks(n), lambda, state, cg_parts(c),
                          tail_part2, tx, 2);
        } else if (minres) {
            run_matvec(c, P, mp, v, u);
            minres_step(c, u, v, r1, r2, W1, W2, x, n, lambda, state);
            minres_update(c, v, W1, W2, x, r2, n, state, u + n, KW1, KW2, s_val, n_val);
        } else if (cgg) {
            run_matvec(c, P, mp, r, u);  // w = K r
            cgg_step(c, x, r, p, sv, u, n, lambda, state);
        } else if (fuse_tail && cheap_persistent) {  // the combine, Ap, alpha, x / r, beta, p in one launch
            CgTail t;
            t.defer = true;
            t.st = state;
            t.lambda = lambda;
            t.p = p;
            run_matvec(c, P, mp, p, u, &t);
            dense_cg_tail(c, SplitParts(), SplitParts(), nullptr, u, x, r, p, p, n, cg_vec_blocks(n), lambda, state,
                          cg_parts(c), tail_part2, nullptr, 0, &t.gc);
        } else if (fuse_tail) {
            CgTail t;
            // lazy direction (segment sums on r + beta p, the combine stores p) measured slower: the
            // extra gather of r in the segment sums costs more than the k_cg_p pass it saves
            t.r = cg_tail_lazy() && mp.form != FORM_POLY2D ? r : nullptr;
            t.st = state;
            t.lambda = lambda;
            t.p = p;
            run_matvec(c, P, mp, p, u, &t);  // the final combine also takes Ap = u + lambda p, p.Ap, alpha
            if (t.r) cg_update_xr(c, x, r, p, u, n, state);
            else cg_update(c, x, r, p, u, n, state, 0, nullptr);
        } else {
            run_matvec(c, P, mp, p, u);
            cg_after_matvec(c, u, p, n, lambda, state);
            if (es) es_cg_scores(c, s_val, u + n, n_val, state);
            cg_update(c, x, r, p, u, n, state, 0, nullptr);
        }
        evaluate();
    };
    drive(c, max_iter, rel_tol > 0.0 || es != nullptr, state, iteration);
    if (cgg) cgg_finish(c, r, n, state);
    if (fuse_dense) dense_tail_finish(c, p, p_alt, n, state);  // the last direction back into p
    if (fuse_tail && cg_tail_lazy() && mp.form != FORM_POLY2D) cg_direction(c, p, r, n, state);  // p_{k+1} (kept)
    // scalars back (one sync per fit)
    double hstate[MINRES_STATE_N];
    GVT_CUDA_TRY(cudaMemcpyAsync(hstate, state, sizeof(double) * SN, cudaMemcpyDeviceToHost, c->stream));
    if (relres_hist)
        GVT_CUDA_TRY(cudaMemcpyAsync(relres_hist, state + SN, sizeof(double) * (max_iter + 1), cudaMemcpyDeviceToHost,
                                     c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    const int iters = (int)hstate[7];
    finish_es(iters);
    out_finish(c, ao);
    if (iters_out) *iters_out = iters;
    if (relres_hist)
        for (int k = iters + 1; k <= max_iter; k++) relres_hist[k] = 0.0 / 0.0;
    if (!minres && hstate[6] != 0.0) {
        set_error("CG breakdown: p^T (K + lambda I) p = %g <= 0 at iteration %d", hstate[4], iters + 1);
        return GVT_E_BREAKDOWN;
    }
    return GVT_OK;
}

// Used-object compaction of a fit (GVT_OPT_COMPACT, default on).  PAPER.md Table 1 counts m, q
// as the UNIQUE drugs / targets of the sample, and Theorem 1's O(qn + m n_bar) cost is in those
// counts; with Grams over a larger object table (the kernel-filling experiment's subsets of 2967
// objects) the GVT would otherwise run over every object.  When the training
// sample uses less than half of the Gram's (drug x target) objects, the fit runs on the sub-Grams
// of the used objects (ascending global id) with renumbered pair ids: the same operator on the
// sample (a bijective relabeling; Identity and Ones factors are preserved), so the same a.
// Early stopping compacts only when the validation ids are among the training objects, so its
// a_best stays the plain fit's.  One GPU only (ranks would need a common object set).
static bool compact_fit(gvt_ctx *c, const float *&D, int64_t &m, const float *&T, int64_t &q, const int32_t *&f,
                        const int32_t *&s, int64_t n, const int32_t *&vf, const int32_t *&vs, int64_t n_val) {
    if (!c->compact || distributed(c) || n <= 0 || m <= 0) return false;
    if (compact_small_skip(c, m, T ? q : m)) return false;
    GVT_REQUIRE(f && s, GVT_E_DIM, "pair ids are NULL with n > 0");
    GVT_REQUIRE(n_val <= 0 || (vf && vs), GVT_E_DIM, "validation pair ids are NULL with n_val > 0");
    const bool hom = T == nullptr;
    const int64_t qq = hom ? m : q;
    const int32_t *fd = (const int32_t *)stage_in(c, "cmp.f_in", f, sizeof(int32_t) * n);
    const int32_t *sd = (const int32_t *)stage_in(c, "cmp.s_in", s, sizeof(int32_t) * n);
    const int32_t *vfd = n_val > 0 ? (const int32_t *)stage_in(c, "cmp.vf_in", vf, sizeof(int32_t) * n_val) : nullptr;
    const int32_t *vsd = n_val > 0 ? (const int32_t *)stage_in(c, "cmp.vs_in", vs, sizeof(int32_t) * n_val) : nullptr;
    // from here on the callers' ids are the staged device copies (host ids are copied once)
    f = fd;
    s = sd;
    if (n_val > 0) {
        vf = vfd;
        vs = vsd;
    }
    // counters: [0, 1] out-of-range training ids (drug / target side), [2, 3] validation ids outside
    // the training objects (or out of range); one read-back for all of them and the set sizes
    unsigned long long *cnt = wsT<unsigned long long>(c, "cmp.cnt", 4);
    GVT_CUDA_TRY(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), c->stream));
    UsedSet ud, ut;
    if (hom) {
        const int32_t *arr[2] = {fd, sd};
        const int64_t len[2] = {n, n};
        ud = used_set_begin(c, "cmp.d", m, arr, len, 2, cnt);
        ut = ud;
    } else {
        ud = used_set_begin(c, "cmp.d", m, &fd, &n, 1, cnt);
        ut = used_set_begin(c, "cmp.t", q, &sd, &n, 1, cnt + 1);
    }
    if (n_val > 0) {
        count_unused_async(c, ud, vfd, n_val, cnt + 2);
        count_unused_async(c, ut, vsd, n_val, cnt + 3);
    }
    unsigned long long h_cnt[4];
    int64_t h_k[2] = {0, 0};
    GVT_CUDA_TRY(cudaMemcpyAsync(h_cnt, cnt, sizeof(h_cnt), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaMemcpyAsync(&h_k[0], ud.k_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    if (!hom) GVT_CUDA_TRY(cudaMemcpyAsync(&h_k[1], ut.k_dev, sizeof(int64_t), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (h_cnt[0] || h_cnt[1])
        throw Error{GVT_E_INDEX, std::to_string(h_cnt[0] + h_cnt[1]) + " pair id(s) out of range [0, " +
                                     std::to_string(m) + ") / [0, " + std::to_string(qq) + ")"};
    ud.k = h_k[0];
    ut.k = hom ? h_k[0] : h_k[1];
    if (hom) ut = ud;
    if ((double)ud.k * (double)ut.k > 0.5 * (double)m * (double)qq) return false;
    if (n_val > 0 && (h_cnt[2] || h_cnt[3])) return false;  // (out-of-range validation ids: the full path reports them)
    const float *Dd = (const float *)stage_in(c, "cmp.D_in", D, sizeof(float) * m * m);
    float *Dc = wsT<float>(c, "cmp.D", (size_t)(ud.k * ud.k));
    sub_gram(c, Dd, m, ud, ud, Dc);
    float *Tc = nullptr;
    if (!hom) {
        const float *Td = (const float *)stage_in(c, "cmp.T_in", T, sizeof(float) * q * q);
        Tc = wsT<float>(c, "cmp.T", (size_t)(ut.k * ut.k));
        sub_gram(c, Td, q, ut, ut, Tc);
    }
    int32_t *fc = wsT<int32_t>(c, "cmp.f", (size_t)n), *sc = wsT<int32_t>(c, "cmp.s", (size_t)n);
    map_ids(c, ud, fd, n, fc);
    map_ids(c, ut, sd, n, sc);
    if (n_val > 0) {
        int32_t *vfc = wsT<int32_t>(c, "cmp.vf", (size_t)n_val), *vsc = wsT<int32_t>(c, "cmp.vs", (size_t)n_val);
        map_ids(c, ud, vfd, n_val, vfc);
        map_ids(c, ut, vsd, n_val, vsc);
        vf = vfc;
        vs = vsc;
    }
    D = Dc;
    m = ud.k;
    T = Tc;
    q = hom ? m : ut.k;
    f = fc;
    s = sc;
    return true;
}

gvt_status fit(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *f, const int32_t *s,
               int64_t n, const float *y, const gvt_term *terms, int n_terms, double lambda, int max_iter,
               double rel_tol, float *a_out, int *iters_out, double *relres_hist) {
    c->last_n = -1;
    c->last_perm = nullptr;
    {
        const int32_t *nv = nullptr, *nv2 = nullptr;
        if (max_iter > 0) compact_fit(c, D, m, T, q, f, s, n, nv, nv2, 0);
    }
    // Sorted-order fit (GVT_OPT_SORTED_FIT, default on): the solve runs on the training pairs
    // stably sorted by (first, second) -- K' = Pi K Pi^T, y' = Pi y, a = Pi^T a', the same
    // iterates up to the summation order of the dot products -- so the Kronecker group's
    // pair-matrix entries are read in vector order instead of gathered at random (the dense
    // path's X build and the sparse path's entry values).
    if (!c->sorted_fit || n < 2 || max_iter == 0)
        return fit_impl(c, D, m, T, q, f, s, n, y, terms, n_terms, lambda, max_iter, rel_tol, a_out, iters_out,
                        relres_hist, nullptr);
    GVT_REQUIRE(f && s && y, GVT_E_DIM, "pair ids or labels are NULL with n > 0");
    const int64_t qq = T ? q : m;
    const int32_t *fd = (const int32_t *)stage_in(c, "sfit.f_in", f, sizeof(int32_t) * n);
    const int32_t *sd = (const int32_t *)stage_in(c, "sfit.s_in", s, sizeof(int32_t) * n);
    const float *yd = (const float *)stage_in(c, "sfit.y_in", y, sizeof(float) * n);
    check_range(c, fd, n, m, "first ids");
    check_range(c, sd, n, qq, "second ids");
    int32_t *perm = wsT<int32_t>(c, "sfit.perm", (size_t)n);
    sort_pairs(c, fd, sd, n, m, qq, perm);
    int32_t *fs = wsT<int32_t>(c, "sfit.f", (size_t)n), *ss = wsT<int32_t>(c, "sfit.s", (size_t)n);
    float *ys = wsT<float>(c, "sfit.y", (size_t)n), *xs = wsT<float>(c, "sfit.x", (size_t)n);
    gather_i32(c, fd, perm, n, fs);
    gather_i32(c, sd, perm, n, ss);
    gather_f32(c, yd, perm, n, ys);
    gvt_status st = fit_impl(c, D, m, T, q, fs, ss, n, ys, terms, n_terms, lambda, max_iter, rel_tol, xs, iters_out,
                             relres_hist, nullptr);
    if (c->last_n == n) c->last_perm = perm;
    OutArr ao = out_arr(c, "out.a", a_out, n);
    scatter_f32(c, xs, perm, n, ao.dev);
    out_finish(c, ao);
    return st;
}

// gvt_solver_direction: the last plain CG fit's search direction, scattered to caller order
void solver_direction(gvt_ctx *c, float *out, int64_t n) {
    GVT_REQUIRE(c->last_n >= 0 && c->last_p, GVT_E_STATE,
                "no search direction kept: the last call was not a Hestenes-Stiefel CG pairwise_krr_fit on the "
                "multi-kernel path (MINRES, Chronopoulos-Gear, early stopping and the single-CTA engine keep none)");
    GVT_REQUIRE(n == c->last_n, GVT_E_DIM, "n differs from the last fit's local pair count");
    if (n == 0) return;
    OutArr o = out_arr(c, "out.p", out, n);
    if (c->last_perm) scatter_f32(c, c->last_p, c->last_perm, n, o.dev);
    else GVT_CUDA_TRY(cudaMemcpyAsync(o.dev, c->last_p, sizeof(float) * n, cudaMemcpyDeviceToDevice, c->stream));
    out_finish(c, o);
}

gvt_status fit_early_stopping(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *f,
                              const int32_t *s, int64_t n, const float *y, const int32_t *vf, const int32_t *vs,
                              int64_t n_val, const float *vlab, const gvt_term *terms, int n_terms, double lambda,
                              int patience, int max_iter, float *a_out, int *best_iter, double *best_auc,
                              int *iters_run, double *auc_hist) {
    c->last_n = -1;
    c->last_perm = nullptr;
    if (max_iter > 0) compact_fit(c, D, m, T, q, f, s, n, vf, vs, n_val);
    EsArgs es;
    es.vf = vf;
    es.vs = vs;
    es.n_val = n_val;
    es.vlab = vlab;
    es.patience = patience;
    es.best_iter = best_iter;
    es.best_auc = best_auc;
    es.auc_hist = auc_hist;
    return fit_impl(c, D, m, T, q, f, s, n, y, terms, n_terms, lambda, max_iter, 0.0, a_out, iters_run, nullptr,
                    &es);
}

// K (m x m2) = k(X_i, Y_j); Y == nullptr: the Gram of X (m2 = m)
void gram(gvt_ctx *c, int kind, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, double gamma,
          double coef0, int degree, float *K) {
    GVT_REQUIRE(m >= 0 && m2 >= 0 && dim >= 0, GVT_E_DIM, "negative size");
    GVT_REQUIRE(kind >= 0 && kind <= 3, GVT_E_PARAM, "unknown base kernel");
    GVT_REQUIRE(kind != GVT_BASE_GAUSSIAN || gamma > 0.0, GVT_E_PARAM, "Gaussian base kernel needs gamma > 0");
    GVT_REQUIRE(kind != GVT_BASE_POLY || degree >= 0, GVT_E_PARAM, "polynomial base kernel needs degree >= 0");
    if (m == 0 || m2 == 0) return;
    GVT_REQUIRE(X && K && (Y || m2 == m), GVT_E_DIM, "X, Y or K is NULL");
    const float *Xd = dim ? (const float *)stage_in(c, "in.X", X, sizeof(float) * m * dim) : nullptr;
    const float *Yd = (Y && dim) ? (const float *)stage_in(c, "in.Y", Y, sizeof(float) * m2 * dim) : nullptr;
    OutArr ko = out_arr(c, "out.K", K, m * m2);
    if (kind == GVT_BASE_TANIMOTO) {  // popcount contraction, no tensor-core form (bits, not a float GEMM)
        gram_tanimoto(c, Xd, m, Y ? Yd : nullptr, m2, dim, ko.dev, m2);
        out_finish(c, ko);
        return;
    }
    bool use_tc = tc_available(c) && c->gram_engine != 1 && dim > 0;
    if (c->gram_engine == 2) GVT_REQUIRE(tc_available(c), GVT_E_CUDA, "tensor-core Gram requested but unavailable");
    if (use_tc) gram_tc(c, kind, Xd, m, Y ? Yd : nullptr, m2, dim, gamma, coef0, degree, ko.dev, m2);
    else gram_simt(c, kind, Xd, m, Y ? Yd : nullptr, m2, dim, dim, gamma, coef0, degree, ko.dev, m2);
    out_finish(c, ko);
}

}  // namespace gvt
