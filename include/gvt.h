/*
 * gvt.h -- C ABI of libgvt.so, the B200 (sm_100a) implementation of the generalized
 * vec trick (GVT) hot path of Viljanen, Airola & Pahikkala, "Generalized vec trick for
 * fast learning of pairwise kernel models" (arXiv 2009.01054; reference/PAPER.md).
 *
 *   u = R(d_bar, t_bar) K R(d, t)^T a,  K = sum of the Corollary's permuted Kronecker
 *   terms, computed by Theorem 1's GVT inside a
 *   conjugate-gradient kernel-ridge-regression loop (Eq. 1 at
 *   316-320) and a batched prediction pass.
 *
 * CONVENTIONS (all entry points)
 *  - Plain C types only.  float arrays are fp32, ids are int32 global object ids, sizes
 *    are int64.  Matrices are dense row-major with leading dimension = column count.
 *  - POINTERS MAY BE HOST OR DEVICE MEMORY.  The library classifies every array with
 *    cudaPointerGetAttributes: device (or managed) arrays are read/written in place
 *    on the context's stream; host arrays (pageable or pinned) are staged through the
 *    context's device workspace, host<->device copies included in the call.  Arrays
 *    are caller-owned; the library never keeps a caller pointer after return.
 *    Term lists, scalars and the *_out scalars are always host memory.
 *  - All device work is issued on the context's stream (gvt_create / gvt_set_stream).
 *    Calls are stream-ordered: every entry point returns after its work is ENQUEUED,
 *    except when it must return a host-visible result (host output arrays, iters_out,
 *    relres_hist, residual-mode stopping, error detection), in which case it
 *    synchronises the stream before returning.
 *  - Errors are return codes; nothing throws or aborts across the ABI.  Validation
 *    (sizes, id ranges, homogeneity, parameters) runs BEFORE any compute
 *    (SPEC.md:118).  gvt_last_error() returns a thread-local message for the last
 *    non-OK status.
 *  - Empty samples (n = 0 or n_out = 0) are legal and give empty outputs;
 *    duplicate pairs are legal and their coefficients sum (reading S17).
 *  - Base-kernel Grams D (m x m) and T (q x q) are over ALL objects, indexed by global
 *    ids, and are symmetric (they are Gram matrices of a kernel); the kernels read
 *    D[j][i] in place of D[i][j].  T == NULL means homogeneous data: one object table
 *    of size m, both pair elements index D.  Ones and Identity
 *    factors are over those global ids (readings S19, S28).
 *  - Results are deterministic: no floating-point atomics; bit-identical run to run
 *    for a fixed device count and fixed dispatch decisions (reading S26).
 */
#ifndef GVT_H
#define GVT_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    GVT_OK = 0,
    GVT_E_DIM = 1,          /* size mismatch / negative size                            */
    GVT_E_INDEX = 2,        /* an id is outside [0, m) or [0, q)          */
    GVT_E_HOMOGENEOUS = 3,  /* homogeneous kernel with T != NULL, or a term indexes a
                               drug Gram with target ids                   */
    GVT_E_KERNEL = 4,       /* unknown kernel name / malformed term                      */
    GVT_E_PARAM = 5,        /* gamma <= 0 for Gaussian, lambda < 0, max_iter < 0, ...    */
    GVT_E_BREAKDOWN = 6,    /* CG: p^T (K + lambda I) p <= 0; current iterate returned   */
    GVT_E_CUDA = 7,         /* CUDA runtime error                                        */
    GVT_E_NCCL = 8,         /* NCCL error or NCCL library unavailable                    */
    GVT_E_OOM = 9,          /* device allocation failed                                  */
    GVT_E_STATE = 10        /* NULL context / call not valid in this state               */
} gvt_status;

/* Pairwise kernels of Table 4b.  GAUSSIAN is the Kronecker kernel of
 * Gaussian base Grams. */
typedef enum {
    GVT_LINEAR = 0, GVT_POLY2D = 1, GVT_GAUSSIAN = 2, GVT_KRONECKER = 3, GVT_SYMMETRIC = 4,
    GVT_ANTISYMMETRIC = 5, GVT_RANKING = 6, GVT_MLPK = 7, GVT_CARTESIAN = 8
} gvt_kernel;

/* Base kernels on object features (POLY by the north star; TANIMOTO on
 * binary features). */
typedef enum { GVT_BASE_LINEAR = 0, GVT_BASE_GAUSSIAN = 1, GVT_BASE_POLY = 2, GVT_BASE_TANIMOTO = 3 } gvt_base;

/* Factor of a Kronecker term: drug Gram, target Gram, all-ones, identity. */
typedef enum { GVT_FACTOR_DRUG = 0, GVT_FACTOR_TARGET = 1, GVT_FACTOR_ONES = 2, GVT_FACTOR_IDENTITY = 3 } gvt_factor;

/* Element selectors: the action of the commutation (P) and unification (Q) operators on
 * sampling operators, R(d,t)P = R(t,d), R(d,t)Q = R(d,d). */
typedef enum { GVT_SEL_FIRST = 0, GVT_SEL_SECOND = 1 } gvt_selector;

/* One permuted Kronecker term.  Its value for out pair o and in pair i is
 *   coef * L[row_sel_left(o), col_sel_left(i)] * R[row_sel_right(o), col_sel_right(i)]
 * with L = left, R = right factor. */
typedef struct {
    double coef;
    int32_t left, right;                  /* gvt_factor */
    int32_t row_sel_left, row_sel_right;  /* gvt_selector, applied to the OUT pair */
    int32_t col_sel_left, col_sel_right;  /* gvt_selector, applied to the IN pair  */
} gvt_term;

typedef struct gvt_ctx gvt_ctx;

/* Options (gvt_set_option). */
typedef enum {
    GVT_OPT_ENGINE = 0,          /* 0 = auto (default; by estimated time, GVT_OPT_DENSE_THRESHOLD),
                                    1 = sparse SIMT, 2 = dense tensor-core,
                                    3 = single-CTA whole-fit CG (Kronecker fits whose factors, S and
                                    vectors fit one SM's shared memory; auto picks it for those when
                                    an iteration is <= 4e6 FMAs), 4 = persistent multi-CTA whole-fit
                                    CG with grid barriers (Kronecker fits with m q^2 <= 6.4e7 dense
                                    stage-1 FMAs, e.g. a complete small grid; auto picks it when the
                                    single-CTA solver does not apply).  The Cartesian kernel follows
                                    the same switch: 1 = the gather form, 2 = u = (D X + X T) sampled
                                    as two tensor-core GEMMs (single GPU; multi-GPU runs the gather
                                    form), auto = by estimated time                                   */
    GVT_OPT_DENSE_THRESHOLD = 1, /* auto engine: -1 (default) = by estimated time of the two engines
                                    (B200 calibration; crossover ~1 % density at C5 object counts);
                                    >= 0 = dense at or above this pair-matrix density             */
    GVT_OPT_PROFILE = 2,         /* 1 = record per-kernel CUDA-event times (gvt_get_stats)                */
    GVT_OPT_GRAM_ENGINE = 3,     /* 0 = auto (tensor cores when available), 1 = SIMT, 2 = tensor cores    */
    GVT_OPT_TC_PRECISION = 4,    /* tensor-core split: 0 = 3xFP16 with per-row power-of-two scaling
                                    (default), 1 = 3xTF32; both fp32-accurate (reading S16)          */
    GVT_OPT_SLABS = 5,           /* single GPU: split stage 1 / stage 2 into this many X-row slabs,
                                    exactly as the data-parallel path does across ranks (default 1) */
    GVT_OPT_GEMM_CTA = 6,        /* tensor-core GEMM: 2 = CTA pair with tcgen05 cta_group::2 (256-row
                                    tiles, default), 1 = single-CTA 128-row tiles                  */
    GVT_OPT_GRAPHS = 7,          /* 1 (default): the solver replays one captured iteration as a CUDA
                                    graph (not while GVT_OPT_PROFILE = 1); 0 = eager launches        */
    GVT_OPT_SOLVER = 8,          /* iterative solver of pairwise_krr_fit(_early_stopping): gvt_solver,
                                    default GVT_SOLVER_CG                                             */
    GVT_OPT_EXCHANGE = 9,        /* data-parallel exchange per matvec: 0 = all-gather
                                    the S column slabs (4 q m bytes, pipelined per slab with stage 2),
                                    stage 2 on the local outputs; 1 = u-exchange: stage 2 of the rank's
                                    own slab over EVERY output, then each output segment summed by its
                                    owner in rank order (4 n bytes); 2 (default) = by estimated bytes:
                                    both exchanges do the same stage-2 work per rank, so the u-exchange
                                    whenever the out sample (all ranks) is smaller than q_out x m_in */
    GVT_OPT_CG_VARIANT = 10,     /* CG form: 0 (default) = Hestenes-Stiefel (two reductions per
                                    iteration); 1 = Chronopoulos-Gear (the same iterates in exact
                                    arithmetic, matvec on r, one fused reduction of r.r and w.r per
                                    iteration: one collective instead of two across GPUs; not with
                                    early stopping)                                                   */
    GVT_OPT_SORTED_FIT = 11,     /* 1 (default): pairwise_krr_fit solves on the training pairs stably
                                    sorted by (first, second) and returns a_out in caller order (the
                                    same iterates up to dot-product summation order; entries read in
                                    vector order); 0 = caller order                                   */
    GVT_OPT_KBLOCK_SKIP = 12,    /* 1 (default): the dense stage 1 skips the all-zero 64-column
                                    K-blocks of each 256-row tile of the pair matrix when they are at
                                    least 15 % of the blocks (block-sparse X, e.g. MLPK on a union
                                    domain); 0 = always the full K loop                              */
    GVT_OPT_STAGE2 = 13,         /* stage 2 of the dense engine: 0 (default) = by estimated time (the
                                    sampled tensor-core GEMM, or the row gather u_i = <A[r_i,:],
                                    S[c_i,:]> over the tensor-core S when the contraction is short and
                                    the samples few, e.g. C2); 1 = always the sampled GEMM; 2 =
                                    always the gather                                                 */
    GVT_OPT_COMPACT = 14         /* 1 (default): a fit whose training pairs use less than half of the
                                    Grams' objects runs on the sub-Grams of the used objects (PAPER.md
                                    Table 1's unique counts; the same a); gvt_matvec / predict run on the
                                    cross-Grams of the used out x in objects when either side uses less
                                    than half (not for Identity-factor kernels); skipped for tables
                                    of <= 2^20 Gram cells; 2 = also for small tables; 0 = off     */
} gvt_option;

/* Solvers for (K + lambda I) a = y.  CG: Hestenes-Stiefel (readings S12-S14).  MINRES: the
 * paper's own solver ("the minimal residual method"; SciPy's minres,
 * PAPER.md:850), unpreconditioned Paige-Saunders recurrences from a = 0; its residual history
 * ||r_k|| / ||y|| (the recurrence's phibar_k) is non-increasing.  Both keep fp32 vectors and fp64
 * scalars on the device. */
typedef enum { GVT_SOLVER_CG = 0, GVT_SOLVER_MINRES = 1 } gvt_solver;

/* Per-context counters (gvt_get_stats). */
#define GVT_MAX_KERNEL_KINDS 32
typedef struct {
    int64_t launches;                         /* library kernels launched since reset                  */
    int32_t n_kinds;                          /* valid entries below                                   */
    char names[GVT_MAX_KERNEL_KINDS][32];     /* kernel kind name                                      */
    int64_t counts[GVT_MAX_KERNEL_KINDS];     /* launches per kind                                     */
    double ms[GVT_MAX_KERNEL_KINDS];          /* summed CUDA-event duration (GVT_OPT_PROFILE = 1)       */
    int32_t last_engine;                      /* engine last used: 1 sparse, 2 dense, 3 single-CTA fit,
                                                 4 persistent multi-CTA fit                           */
    int32_t world;                            /* communicator size (1 without gvt_comm_init)           */
    int32_t last_exchange;                    /* exchange of the last data-parallel call: 0 none (single
                                                 GPU), 1 S slab all-gather, 2 u-exchange              */
} gvt_stats;

/* Create a context on CUDA device `device`, issuing work on `stream` (a cudaStream_t;
 * NULL = the legacy default stream).  The context owns device workspaces (grown on
 * demand, freed by gvt_destroy) and, after gvt_comm_init, an NCCL communicator. */
gvt_status gvt_create(gvt_ctx **ctx, int device, void *stream);
gvt_status gvt_destroy(gvt_ctx *ctx);
gvt_status gvt_set_stream(gvt_ctx *ctx, void *stream);
gvt_status gvt_set_option(gvt_ctx *ctx, gvt_option opt, double value);
gvt_status gvt_get_stats(gvt_ctx *ctx, gvt_stats *out);
gvt_status gvt_reset_stats(gvt_ctx *ctx);

/* Multi-GPU (one process per GPU).  `nccl_unique_id` points to the 128-byte
 * ncclUniqueId produced by gvt_nccl_unique_id on rank 0 and broadcast by the caller
 * (e.g. with torch.distributed).  After this call pairwise_krr_fit / pairwise_predict /
 * gvt_matvec run data-parallel: each rank passes ITS OWN SHARD of the in-sample pairs
 * (and of y / a), the shards must be drug-partitioned by contiguous first-id ranges in
 * rank order (gvt_partition computes them), D and T are replicated.  Stage 1 runs on
 * the local pairs, the S column slabs are all-gathered over NVLink, stage 2 runs on the
 * local out pairs, CG dot products are all-reduced.  Every
 * dispatch decision (engine, stage-2 kernel, slabs) is taken from rank-independent sizes,
 * so all ranks issue the same collectives.
 * world == 1 with nccl_unique_id == NULL: single-GPU mode (no communicator).  world == 1 WITH
 * a unique id: a one-rank NCCL communicator, and the data-parallel path runs with its real
 * NCCL calls on one GPU (the executable check of the NCCL data plane on a one-GPU box).
 * Errors: GVT_E_PARAM (bad rank/world, NULL id with world > 1), GVT_E_NCCL. */
gvt_status gvt_nccl_unique_id(void *out128);
gvt_status gvt_comm_init(gvt_ctx *ctx, const void *nccl_unique_id, int rank, int world);

/* Host-mediated communicator, for testing the data-parallel path with several ranks on fewer
 * GPUs (e.g. two processes sharing one GPU, exchanging through torch.distributed gloo): every
 * collective of the library becomes one call of `allgather(user, buf, bytes)`, where buf is HOST
 * memory of world * bytes with this rank's block at buf + rank * bytes, and the callback fills the
 * other ranks' blocks (returns 0 on success).  The library synchronises its stream around each
 * call, so no kernel ever waits on another rank; collectives are then not graph-capturable and
 * the solver replays eagerly.  The results equal the NCCL path's bit for bit: both run the same
 * exchanges, and every reduction is a fixed rank-order sum on the device (solver dot products
 * from all-gathered partials; the u-exchange from the owner's received segments -- NCCL
 * send/recv, not ncclReduce). */
typedef int (*gvt_host_allgather_fn)(void *user, void *buf, size_t bytes);
gvt_status gvt_comm_init_host(gvt_ctx *ctx, int rank, int world, gvt_host_allgather_fn allgather, void *user);

/* Balanced contiguous drug ranges: given per-drug pair counts deg[m] (host), writes
 * bounds[world+1] (host) with bounds[0] = 0, bounds[world] = m, each range holding about
 * sum(deg)/world pairs (greedy prefix split).  Host-only, no device work. */
gvt_status gvt_partition(const int64_t *deg, int64_t m, int world, int64_t *bounds);

/* Data-parallel slab partition of the pair-matrix rows (= S columns): given the CSR row
 * pointer row_ptr[nrow+1] (host) of the entries, writes bounds[nslab+1] (host): bounds[0] = 0,
 * bounds[nslab] = nrow, bounds[s] = the first row at or after the s/nslab entry quantile,
 * rounded up to a multiple of 32 and kept monotone.  Rank s runs stage 1 on rows
 * [bounds[s], bounds[s+1]).  Host-only, no device work. */
gvt_status gvt_slab_bounds(const int64_t *row_ptr, int64_t nrow, int nslab, int64_t *bounds);

/* The slab partition the engine uses (stage 1 per drug column slab): balanced
 * by the estimated cost C(h) = w_entry * row_ptr[h] + w_row * h of rows [0, h): bounds[s] = the
 * first row with C >= s/nslab * C(nrow), rounded up to a multiple of 32 and kept monotone;
 * w_row = 0 gives gvt_slab_bounds.  The engine passes (0, 1) for the dense tensor-core engine
 * (both GEMMs scale with the slab's rows) and (q_out / 3.3e6, u-exchange ? 4 n_out / 6.4e6 : 0)
 * for the sparse engine (stage-1 FMAs per entry; stage-2 slice gathers per row).  Host-only.
 * Errors: GVT_E_PARAM for NULL pointers, nrow < 0, nslab < 1 or negative weights. */
gvt_status gvt_slab_bounds_cost(const int64_t *row_ptr, int64_t nrow, int nslab, double w_entry, double w_row,
                                int64_t *bounds);

/* decompose: the Corollary's term list for `kernel` (
 * MLPK 10-term expansion PAPER.md:736-747; Anti-symmetric as (I-P)(D(x)D), reading S3).
 * `out` must hold 16 terms.  Host only. */
gvt_status gvt_kernel_terms(gvt_kernel kernel, gvt_term *out, int *n_terms);

/* Base-kernel Gram K[i][j] = k(X_i, X_j), X (m x dim), K (m x m):
 * LINEAR <x,y>; GAUSSIAN exp(-gamma ||x-y||^2) (squared norm, reading S4; diagonal exactly
 * 1); POLY (gamma <x,y> + coef0)^degree; TANIMOTO sum_k min(x_k, y_k) / sum_k max(x_k, y_k)
 * on 0/1 features ("bits set to 1 in both vs. bits set to 1 in either"), 1 for
 * two all-zero vectors (reading T1), computed exactly as popcounts of bit-packed features.
 * Errors: GVT_E_PARAM if gamma <= 0 (GAUSSIAN), degree < 0 (POLY) or a TANIMOTO feature is
 * not 0 or 1 (checked before the Gram is computed). */
gvt_status gvt_gram(gvt_ctx *ctx, gvt_base kind, const float *X, int64_t m, int64_t dim,
                    double gamma, double coef0, int degree, float *K);

/* Cross-Gram K[i][j] = k(X_i, Y_j), X (m x dim), Y (m2 x dim), K (m x m2): the base kernel
 * between two object tables, e.g. novel test objects (rows) against the training objects
 * (columns) for pairwise_predict_rect.  Same kernels and errors as
 * gvt_gram; no diagonal is forced (the tables are different objects). */
gvt_status gvt_gram_cross(gvt_ctx *ctx, gvt_base kind, const float *X, int64_t m, const float *Y, int64_t m2,
                          int64_t dim, double gamma, double coef0, int degree, float *K);

/* GVT matvec (Theorem 1; Corollary PAPER.md:634-653):
 *   u[i] = sum_j sum_terms coef * L[.,.] * R[.,.] * a[j]
 * over out pairs (out_first[i], out_second[i]), i < n_out, and in pairs
 * (in_first[j], in_second[j]), j < n_in.  No lambda (reading S27).  `terms` is any
 * term list (host); the Corollary lists of gvt_kernel_terms are recognised and run as
 * fused normal forms, any other list runs term by term.  u is in caller order. */
gvt_status gvt_matvec(gvt_ctx *ctx, const float *D, int64_t m, const float *T, int64_t q,
                      const int32_t *out_first, const int32_t *out_second, int64_t n_out,
                      const int32_t *in_first, const int32_t *in_second, int64_t n_in,
                      const float *a, const gvt_term *terms, int n_terms, float *u);

/* Kernel ridge regression (K + lambda I) a = y by conjugate
 * gradients (default) or MINRES (GVT_OPT_SOLVER) from a = 0 (readings S12-S14, M1-M2):
 * max_iter iterations (rel_tol = 0) or until ||r_k|| / ||y|| <= rel_tol (MINRES also stops
 * on Lanczos breakdown, beta_{k+1} <= 64 u ||T_k||_F, u = 2^-24, a converged exit).  Each iteration is one GVT
 * matvec.  Solver scalars are fp64.
 * iters_out (host, nullable) = iterations done; relres_hist (host, nullable,
 * max_iter + 1 doubles) = ||r_k|| / ||y|| for k = 0..iters.  y == 0 gives a = 0 after 0
 * iterations.  CG breakdown (p^T A p <= 0) returns GVT_E_BREAKDOWN with the current iterate
 * in a_out. */
gvt_status pairwise_krr_fit(gvt_ctx *ctx, const float *D, int64_t m, const float *T, int64_t q,
                            const int32_t *in_first, const int32_t *in_second, int64_t n,
                            const float *y, const gvt_term *terms, int n_terms, double lambda,
                            int max_iter, double rel_tol, float *a_out, int *iters_out,
                            double *relres_hist);

/* Early-stopping ridge regression ("running the minimum residual algorithm
 * on Z_inner until the AUC stops increasing in Z_validation for a given number of iterations";
 * SPEC.md fit_early_stopping).  Runs the GVT_OPT_SOLVER solver (lambda as given, x0 = 0) on
 * the inner pairs (inner_first/second, n, labels y); after every iteration k it scores the
 * validation pairs with the iterate a_k (scores = K_val,inner a_k) and takes their AUC against
 * val_labels (positive iff label > 0; Mann-Whitney, ties count 1/2).  It stops after
 * `patience` consecutive iterations without strict AUC improvement, at max_iter, or when the
 * solver converges/breaks down.  Outputs: a_out (n floats) = the weights of the best
 * iteration (all zero if none); best_iter (host, nullable) = the earliest iteration with the
 * highest AUC; best_auc (host, nullable); iters_run (host, nullable) = iterations performed;
 * auc_hist (host, nullable, max_iter doubles) = AUC after iteration k at [k - 1], NaN past
 * iters_run.  The validation scores share each iteration's stage 1 with the training matvec
 * (the out sample is [inner; validation]).  Multi-GPU: every rank passes its shard of the
 * inner pairs (as pairwise_krr_fit) and of the validation pairs; the AUC is over all ranks'
 * validation pairs and the outputs are identical on every rank.  Errors: GVT_E_PARAM for
 * patience < 1 or validation labels of a single class; otherwise as pairwise_krr_fit. */
gvt_status pairwise_krr_fit_early_stopping(gvt_ctx *ctx, const float *D, int64_t m, const float *T, int64_t q,
                                           const int32_t *inner_first, const int32_t *inner_second, int64_t n,
                                           const float *y, const int32_t *val_first, const int32_t *val_second,
                                           int64_t n_val, const float *val_labels, const gvt_term *terms,
                                           int n_terms, double lambda, int patience, int max_iter, float *a_out,
                                           int *best_iter, double *best_auc, int *iters_run, double *auc_hist);

/* AUC of scores[n] against labels[n] (positive iff label > 0): the Mann-Whitney statistic,
 * fraction of (positive, negative) pairs with the positive scored higher, ties counting 1/2
 * (the validation criterion of PAPER.md:852-856).  Computed on the device by a radix sort and
 * exact integer counting, so it is exact for the given fp32 scores.  *auc (host).  Errors:
 * GVT_E_PARAM if either class is empty. */
gvt_status gvt_auc(gvt_ctx *ctx, const float *labels, const float *scores, int64_t n, double *auc);

/* Prediction v = R(test) K R(train)^T a: scores[i] for test pair i,
 * caller order. */
gvt_status pairwise_predict(gvt_ctx *ctx, const float *D, int64_t m, const float *T, int64_t q,
                            const int32_t *test_first, const int32_t *test_second, int64_t n_test,
                            const int32_t *train_first, const int32_t *train_second, int64_t n_train,
                            const float *a, const gvt_term *terms, int n_terms, float *scores);

/* Novel objects (Settings 2-4): the GVT matvec on rectangular cross-Grams.
 *   u[i] = sum_j k(out_i, in_j) a[j],  k from Table 4b with every base-kernel value taken from a
 *   cross-Gram Dx[out object][in object] (m_out x m_in, row-major) or Tx (q_out x q_in);
 *   Tx == NULL means homogeneous objects (one cross-Gram, q_out = m_out, q_in = m_in).
 * Out ids index the ROWS (out_first < m_out, out_second < q_out), in ids the COLUMNS
 * (in_first < m_in, in_second < q_in); the cross-Grams need not be symmetric or square.
 * `terms` is any term list without Identity factors (the Cartesian kernel compares objects
 * across the two tables, which share no ids: GVT_E_KERNEL, reading N1).
 * variant (Theorem 1; SPEC.md gvt_cost): 1 = stage 1 over the second
 * factor, cost q_out n_in + m_in n_out; 2 = the roles of the two factors swapped, cost
 * m_out n_in + q_in n_out (Kronecker term list only); 0 = auto, the smaller cost, ties -> 1.
 * variant_used / op_count (host, nullable): the variant run and its cost (-1 for non-Kronecker
 * lists, which run variant 1).  No lambda.  Errors: GVT_E_INDEX for ids out of range,
 * GVT_E_PARAM for a bad variant. */
gvt_status gvt_matvec_rect(gvt_ctx *ctx, const float *Dx, int64_t m_out, int64_t m_in, const float *Tx,
                           int64_t q_out, int64_t q_in, const int32_t *out_first, const int32_t *out_second,
                           int64_t n_out, const int32_t *in_first, const int32_t *in_second, int64_t n_in,
                           const float *a, const gvt_term *terms, int n_terms, int variant, float *u,
                           int *variant_used, int64_t *op_count);

/* Prediction for novel objects: scores = K(test, train) a with cross-Grams between the test
 * objects (rows) and the training objects (columns), variant auto-selected (gvt_matvec_rect
 * with variant 0).  PAPER.md:321-322 with the test sample's own objects (Table 1's
 * m_bar, q_bar). */
gvt_status pairwise_predict_rect(gvt_ctx *ctx, const float *Dx, int64_t m_test, int64_t m_train, const float *Tx,
                                 int64_t q_test, int64_t q_train, const int32_t *test_first,
                                 const int32_t *test_second, int64_t n_test, const int32_t *train_first,
                                 const int32_t *train_second, int64_t n_train, const float *a,
                                 const gvt_term *terms, int n_terms, float *scores);

/* Integer plumbing exposed for bit-exact tests: stable sort of pair indices by first id
 * (mode 0) or by (first, second) (mode 1), ties in ascending index order; perm[n] int32
 * and row_ptr[m+1] int64 (first position of each first id).  Pointers host or device. */
gvt_status gvt_sort_plan(gvt_ctx *ctx, const int32_t *first, const int32_t *second, int64_t n,
                         int64_t m, int64_t q, int mode, int32_t *perm, int64_t *row_ptr);

/* Compact relabeling of an id sequence (SPEC.md:49-57 relabel_compact; it realizes the "unique"
 * counts m, q of PAPER.md Table 1 -- "the number of unique drugs in the first sample").
 *   ids[n]      object ids in [0, bound) (int32)
 *   compact[n]  out: compact[i] in [0, count), unique[compact[i]] == ids[i] (int32)
 *   unique[]    out: the distinct ids in first-occurrence order; capacity min(n, bound) (int32)
 *   count       out (host): the number of distinct ids
 * Integer-only and bit-exact.  The engine itself indexes Grams by global ids and does not need
 * it; callers who build compact Grams apply it first.  Pointers host or device.
 * Errors: GVT_E_DIM (negative sizes, NULL outputs), GVT_E_INDEX (an id outside [0, bound)). */
gvt_status gvt_relabel_compact(gvt_ctx *ctx, const int32_t *ids, int64_t n, int64_t bound, int32_t *compact,
                               int32_t *unique, int64_t *count);

/* Solver inspection for the in-loop parity check of reading S30 ("dump p_k at
 * k in {1, K/2, K} and check K p_k against the oracle"): copies the search direction left by the
 * last pairwise_krr_fit on this context -- after k Hestenes-Stiefel CG iterations that is
 * p_{k+1} = r_k + beta_k p_k (PAPER.md:316-320 solved by CG, reading S12), the vector the next
 * matvec would be applied to -- into p_out[n] (host or device), in the caller's pair order, this
 * rank's shard.  n must equal the fit's local pair count.  Errors: GVT_E_STATE if the last fit
 * kept no direction (MINRES, Chronopoulos-Gear CG, early stopping, the single-CTA engine, or no fit
 * yet); GVT_E_DIM for a different n. */
gvt_status gvt_solver_direction(gvt_ctx *ctx, float *p_out, int64_t n);

/* Thread-local message describing the last non-OK status. */
const char *gvt_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* GVT_H */
