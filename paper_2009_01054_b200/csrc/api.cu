// api.cu -- the extern "C" entry points of include/gvt.h.  Each converts exceptions
// (gvt::Error) into status codes and a thread-local message; nothing throws across the ABI.
#include <string.h>

#include "ops.cuh"

namespace gvt {
const char *last_error();
void slab_bounds(const int64_t *rp, int64_t nrow, int G, int64_t *bounds);
void slab_bounds_cost(const int64_t *rp, int64_t nrow, int G, double w_entry, double w_row, int64_t *bounds);
int kernel_terms(int kernel, gvt_term *o);
void nccl_unique_id(void *out128);
void comm_init(gvt_ctx *c, const void *id128, int rank, int world);
void comm_destroy(gvt_ctx *c);
void comm_init_host(gvt_ctx *c, int rank, int world, gvt_host_allgather_fn fn, void *user);
void matvec(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *of, const int32_t *os,
            int64_t n_out, const int32_t *inf, const int32_t *ins, int64_t n_in, const float *a,
            const gvt_term *terms, int n_terms, float *u);
void predict(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *tf, const int32_t *ts,
             int64_t n_test, const int32_t *trf, const int32_t *trs, int64_t n_train, const float *a,
             const gvt_term *terms, int n_terms, float *scores);
gvt_status fit(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *f, const int32_t *s,
               int64_t n, const float *y, const gvt_term *terms, int n_terms, double lambda, int max_iter,
               double rel_tol, float *a_out, int *iters_out, double *relres_hist);
void gram(gvt_ctx *c, int kind, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, double gamma,
          double coef0, int degree, float *K);
void matvec_rect(gvt_ctx *c, const float *Dx, int64_t m_out, int64_t m_in, const float *Tx, int64_t q_out,
                 int64_t q_in, const int32_t *of, const int32_t *os, int64_t n_out, const int32_t *inf,
                 const int32_t *ins, int64_t n_in, const float *a, const gvt_term *terms, int n_terms, int variant,
                 float *u, int *variant_used, int64_t *op_count);
gvt_status fit_early_stopping(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *f,
                              const int32_t *s, int64_t n, const float *y, const int32_t *vf, const int32_t *vs,
                              int64_t n_val, const float *vlab, const gvt_term *terms, int n_terms, double lambda,
                              int patience, int max_iter, float *a_out, int *best_iter, double *best_auc,
                              int *iters_run, double *auc_hist);
void solver_direction(gvt_ctx *c, float *out, int64_t n);
}  // namespace gvt

using gvt::Error;

#define GVT_API_BEGIN(ctx)                                              \
    if (!(ctx)) {                                                       \
        gvt::set_error("NULL context");                                 \
        return GVT_E_STATE;                                             \
    }                                                                   \
    try {                                                               \
        GVT_CUDA_TRY(cudaSetDevice((ctx)->device));

#define GVT_API_END                                                     \
    }                                                                   \
    catch (const Error &e) {                                            \
        gvt::set_error("%s", e.msg.c_str());                            \
        return e.code;                                                  \
    }                                                                   \
    catch (const std::exception &e) {                                   \
        gvt::set_error("internal error: %s", e.what());                 \
        return GVT_E_CUDA;                                              \
    }                                                                   \
    return GVT_OK;

extern "C" {

const char *gvt_last_error(void) { return gvt::last_error(); }

gvt_status gvt_create(gvt_ctx **out, int device, void *stream) {
    if (!out) {
        gvt::set_error("gvt_create: out is NULL");
        return GVT_E_STATE;
    }
    *out = nullptr;
    gvt_ctx *c = new gvt_ctx();
    try {
        int ndev = 0;
        GVT_CUDA_TRY(cudaGetDeviceCount(&ndev));
        GVT_REQUIRE(device >= 0 && device < ndev, GVT_E_PARAM, "gvt_create: bad device ordinal");
        GVT_CUDA_TRY(cudaSetDevice(device));
        c->device = device;
        c->stream = (cudaStream_t)stream;
        cudaDeviceProp prop;
        GVT_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
        c->sm_count = prop.multiProcessorCount;
        c->cc_major = prop.major;
        c->cc_minor = prop.minor;
        c->tc_ok = (prop.major == 10 && prop.minor == 0);
    } catch (const Error &e) {
        gvt::set_error("%s", e.msg.c_str());
        delete c;
        return e.code;
    }
    *out = c;
    return GVT_OK;
}

gvt_status gvt_destroy(gvt_ctx *c) {
    if (!c) return GVT_OK;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    gvt::comm_destroy(c);
    for (auto &kv : c->bufs)
        if (kv.second.ptr) cudaFree(kv.second.ptr);
    for (auto &pe : c->pending) {
        cudaEventDestroy(pe.start);
        cudaEventDestroy(pe.stop);
    }
    for (auto e : c->event_pool) cudaEventDestroy(e);
    if (c->pinned) cudaFreeHost(c->pinned);
    if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
    delete c;
    return GVT_OK;
}

gvt_status gvt_set_stream(gvt_ctx *c, void *stream) {
    GVT_API_BEGIN(c)
    c->stream = (cudaStream_t)stream;
    GVT_API_END
}

gvt_status gvt_set_option(gvt_ctx *c, gvt_option opt, double v) {
    GVT_API_BEGIN(c)
    switch (opt) {
    case GVT_OPT_ENGINE:
        GVT_REQUIRE(v == 0 || v == 1 || v == 2 || v == 3 || v == 4, GVT_E_PARAM, "engine must be 0, 1, 2, 3 or 4");
        c->engine = (int)v;
        break;
    case GVT_OPT_DENSE_THRESHOLD:
        GVT_REQUIRE(v >= 0 || v == -1.0, GVT_E_PARAM, "threshold must be >= 0, or -1 for the time estimate");
        c->dense_threshold = v;
        break;
    case GVT_OPT_PROFILE: c->profile = v != 0; break;
    case GVT_OPT_GRAM_ENGINE:
        GVT_REQUIRE(v == 0 || v == 1 || v == 2, GVT_E_PARAM, "gram engine must be 0, 1 or 2");
        c->gram_engine = (int)v;
        break;
    case GVT_OPT_TC_PRECISION:
        GVT_REQUIRE(v == 0 || v == 1, GVT_E_PARAM, "tc precision must be 0 (fp16 x3) or 1 (tf32 x3)");
        c->tc_precision = (int)v;
        break;
    case GVT_OPT_GRAPHS:
        c->graphs = v != 0;
        break;
    case GVT_OPT_KBLOCK_SKIP:
        c->kblock_skip = v != 0;
        break;
    case GVT_OPT_COMPACT:
        GVT_REQUIRE(v == 0 || v == 1 || v == 2, GVT_E_PARAM, "compact must be 0 (off), 1 (auto) or 2 (always)");
        c->compact = (int)v;
        break;
    case GVT_OPT_STAGE2:
        GVT_REQUIRE(v == 0 || v == 1 || v == 2, GVT_E_PARAM, "stage 2 must be 0 (auto), 1 (sampled GEMM) or 2 (gather)");
        c->stage2 = (int)v;
        break;
    case GVT_OPT_SORTED_FIT:
        c->sorted_fit = v != 0;
        break;
    case GVT_OPT_CG_VARIANT:
        GVT_REQUIRE(v == 0 || v == 1, GVT_E_PARAM, "cg variant must be 0 (Hestenes-Stiefel) or 1 (Chronopoulos-Gear)");
        c->cg_variant = (int)v;
        break;
    case GVT_OPT_EXCHANGE:
        GVT_REQUIRE(v == 0 || v == 1 || v == 2, GVT_E_PARAM,
                    "exchange must be 0 (S all-gather), 1 (u reduce) or 2 (by estimated bytes)");
        c->exchange = (int)v;
        break;
    case GVT_OPT_SOLVER:
        GVT_REQUIRE(v == GVT_SOLVER_CG || v == GVT_SOLVER_MINRES, GVT_E_PARAM, "solver must be 0 (CG) or 1 (MINRES)");
        c->solver = (int)v;
        break;
    case GVT_OPT_GEMM_CTA:
        GVT_REQUIRE(v == 1 || v == 2, GVT_E_PARAM, "gemm cta must be 1 or 2");
        c->gemm_cta = (int)v;
        break;
    case GVT_OPT_SLABS:
        GVT_REQUIRE(v >= 1 && v <= 64, GVT_E_PARAM, "slabs must be in [1, 64]");
        c->slabs = (int)v;
        break;
    default: throw Error{GVT_E_PARAM, "unknown option"};
    }
    GVT_API_END
}

gvt_status gvt_get_stats(gvt_ctx *c, gvt_stats *out) {
    GVT_API_BEGIN(c)
    GVT_REQUIRE(out, GVT_E_PARAM, "stats out is NULL");
    gvt::collect_events(c);
    memset(out, 0, sizeof(*out));
    out->launches = c->launches;
    out->n_kinds = gvt::K_NUM_KINDS;
    for (int k = 0; k < gvt::K_NUM_KINDS && k < GVT_MAX_KERNEL_KINDS; k++) {
        strncpy(out->names[k], gvt::kind_name(k), 31);
        out->counts[k] = c->counts[k];
        out->ms[k] = c->ms[k];
    }
    out->last_engine = c->last_engine;
    out->last_exchange = c->last_exchange;
    out->world = c->world;
    GVT_API_END
}

gvt_status gvt_reset_stats(gvt_ctx *c) {
    GVT_API_BEGIN(c)
    gvt::collect_events(c);
    c->launches = 0;
    for (int k = 0; k < gvt::K_NUM_KINDS; k++) {
        c->counts[k] = 0;
        c->ms[k] = 0;
    }
    GVT_API_END
}

gvt_status gvt_nccl_unique_id(void *out128) {
    try {
        GVT_REQUIRE(out128, GVT_E_PARAM, "out is NULL");
        gvt::nccl_unique_id(out128);
    } catch (const Error &e) {
        gvt::set_error("%s", e.msg.c_str());
        return e.code;
    }
    return GVT_OK;
}

gvt_status gvt_comm_init(gvt_ctx *c, const void *id, int rank, int world) {
    GVT_API_BEGIN(c)
    GVT_REQUIRE(world == 1 || id, GVT_E_PARAM, "unique id is NULL");
    gvt::comm_init(c, id, rank, world);
    GVT_API_END
}

gvt_status gvt_comm_init_host(gvt_ctx *c, int rank, int world, gvt_host_allgather_fn allgather, void *user) {
    GVT_API_BEGIN(c)
    gvt::comm_init_host(c, rank, world, allgather, user);
    GVT_API_END
}

gvt_status gvt_partition(const int64_t *deg, int64_t m, int world, int64_t *bounds) {
    if (!bounds || world < 1 || m < 0 || (m > 0 && !deg)) {
        gvt::set_error("gvt_partition: bad arguments");
        return GVT_E_PARAM;
    }
    // greedy prefix split: range g ends at the first drug where the running pair count
    // reaches (g+1) * total / world
    int64_t total = 0;
    for (int64_t h = 0; h < m; h++) {
        if (deg[h] < 0) {
            gvt::set_error("gvt_partition: negative degree");
            return GVT_E_PARAM;
        }
        total += deg[h];
    }
    bounds[0] = 0;
    int64_t run = 0, h = 0;
    for (int g = 1; g < world; g++) {
        long double target = (long double)total * g / world;
        while (h < m && (long double)(run + deg[h]) <= target) run += deg[h++];
        // include the straddling drug if that lands closer to the target
        if (h < m && (long double)(run + deg[h]) - target < target - (long double)run) run += deg[h++];
        bounds[g] = h;
    }
    bounds[world] = m;
    return GVT_OK;
}

gvt_status gvt_slab_bounds(const int64_t *row_ptr, int64_t nrow, int nslab, int64_t *bounds) {
    if (!row_ptr || !bounds || nrow < 0 || nslab < 1) {
        gvt::set_error("gvt_slab_bounds: bad arguments");
        return GVT_E_PARAM;
    }
    gvt::slab_bounds(row_ptr, nrow, nslab, bounds);
    return GVT_OK;
}

gvt_status gvt_slab_bounds_cost(const int64_t *row_ptr, int64_t nrow, int nslab, double w_entry, double w_row,
                                int64_t *bounds) {
    if (!row_ptr || !bounds || nrow < 0 || nslab < 1 || !(w_entry >= 0) || !(w_row >= 0)) {
        gvt::set_error("gvt_slab_bounds_cost: bad arguments");
        return GVT_E_PARAM;
    }
    gvt::slab_bounds_cost(row_ptr, nrow, nslab, w_entry, w_row, bounds);
    return GVT_OK;
}

gvt_status gvt_kernel_terms(gvt_kernel kernel, gvt_term *out, int *n_terms) {
    if (!out || !n_terms) {
        gvt::set_error("gvt_kernel_terms: NULL output");
        return GVT_E_PARAM;
    }
    int n = gvt::kernel_terms((int)kernel, out);
    if (n < 0) {
        gvt::set_error("unknown kernel %d", (int)kernel);
        return GVT_E_KERNEL;
    }
    *n_terms = n;
    return GVT_OK;
}

gvt_status gvt_gram(gvt_ctx *c, gvt_base kind, const float *X, int64_t m, int64_t dim, double gamma, double coef0,
                    int degree, float *K) {
    GVT_API_BEGIN(c)
    gvt::gram(c, (int)kind, X, m, nullptr, m, dim, gamma, coef0, degree, K);
    GVT_API_END
}

gvt_status gvt_gram_cross(gvt_ctx *c, gvt_base kind, const float *X, int64_t m, const float *Y, int64_t m2,
                          int64_t dim, double gamma, double coef0, int degree, float *K) {
    GVT_API_BEGIN(c)
    GVT_REQUIRE(m2 == 0 || Y || dim == 0, GVT_E_DIM, "Y is NULL");
    gvt::gram(c, (int)kind, X, m, Y ? Y : X, m2, dim, gamma, coef0, degree, K);
    GVT_API_END
}

gvt_status gvt_matvec(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *out_first,
                      const int32_t *out_second, int64_t n_out, const int32_t *in_first, const int32_t *in_second,
                      int64_t n_in, const float *a, const gvt_term *terms, int n_terms, float *u) {
    GVT_API_BEGIN(c)
    gvt::matvec(c, D, m, T, q, out_first, out_second, n_out, in_first, in_second, n_in, a, terms, n_terms, u);
    GVT_API_END
}

gvt_status pairwise_krr_fit(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *in_first,
                            const int32_t *in_second, int64_t n, const float *y, const gvt_term *terms, int n_terms,
                            double lambda, int max_iter, double rel_tol, float *a_out, int *iters_out,
                            double *relres_hist) {
    GVT_API_BEGIN(c)
    gvt_status st = gvt::fit(c, D, m, T, q, in_first, in_second, n, y, terms, n_terms, lambda, max_iter, rel_tol,
                             a_out, iters_out, relres_hist);
    if (st != GVT_OK) return st;
    GVT_API_END
}

gvt_status pairwise_krr_fit_early_stopping(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q,
                                           const int32_t *inner_first, const int32_t *inner_second, int64_t n,
                                           const float *y, const int32_t *val_first, const int32_t *val_second,
                                           int64_t n_val, const float *val_labels, const gvt_term *terms, int n_terms,
                                           double lambda, int patience, int max_iter, float *a_out, int *best_iter,
                                           double *best_auc, int *iters_run, double *auc_hist) {
    GVT_API_BEGIN(c)
    gvt_status st = gvt::fit_early_stopping(c, D, m, T, q, inner_first, inner_second, n, y, val_first, val_second,
                                            n_val, val_labels, terms, n_terms, lambda, patience, max_iter, a_out,
                                            best_iter, best_auc, iters_run, auc_hist);
    if (st != GVT_OK) return st;
    GVT_API_END
}

gvt_status gvt_matvec_rect(gvt_ctx *c, const float *Dx, int64_t m_out, int64_t m_in, const float *Tx, int64_t q_out,
                           int64_t q_in, const int32_t *out_first, const int32_t *out_second, int64_t n_out,
                           const int32_t *in_first, const int32_t *in_second, int64_t n_in, const float *a,
                           const gvt_term *terms, int n_terms, int variant, float *u, int *variant_used,
                           int64_t *op_count) {
    GVT_API_BEGIN(c)
    gvt::matvec_rect(c, Dx, m_out, m_in, Tx, q_out, q_in, out_first, out_second, n_out, in_first, in_second, n_in, a,
                     terms, n_terms, variant, u, variant_used, op_count);
    GVT_API_END
}

gvt_status pairwise_predict_rect(gvt_ctx *c, const float *Dx, int64_t m_test, int64_t m_train, const float *Tx,
                                 int64_t q_test, int64_t q_train, const int32_t *test_first,
                                 const int32_t *test_second, int64_t n_test, const int32_t *train_first,
                                 const int32_t *train_second, int64_t n_train, const float *a, const gvt_term *terms,
                                 int n_terms, float *scores) {
    GVT_API_BEGIN(c)
    gvt::matvec_rect(c, Dx, m_test, m_train, Tx, q_test, q_train, test_first, test_second, n_test, train_first,
                     train_second, n_train, a, terms, n_terms, 0, scores, nullptr, nullptr);
    GVT_API_END
}

gvt_status gvt_auc(gvt_ctx *c, const float *labels, const float *scores, int64_t n, double *auc) {
    GVT_API_BEGIN(c)
    GVT_REQUIRE(auc, GVT_E_DIM, "auc is NULL");
    *auc = gvt::auc(c, labels, scores, n);
    GVT_API_END
}

gvt_status pairwise_predict(gvt_ctx *c, const float *D, int64_t m, const float *T, int64_t q, const int32_t *tf,
                            const int32_t *ts, int64_t n_test, const int32_t *trf, const int32_t *trs, int64_t n_train,
                            const float *a, const gvt_term *terms, int n_terms, float *scores) {
    GVT_API_BEGIN(c)
    gvt::predict(c, D, m, T, q, tf, ts, n_test, trf, trs, n_train, a, terms, n_terms, scores);
    GVT_API_END
}

gvt_status gvt_sort_plan(gvt_ctx *c, const int32_t *first, const int32_t *second, int64_t n, int64_t m, int64_t q,
                         int mode, int32_t *perm, int64_t *row_ptr) {
    GVT_API_BEGIN(c)
    GVT_REQUIRE(n >= 0 && m >= 0 && q >= 0, GVT_E_DIM, "negative size");
    GVT_REQUIRE(mode == 0 || mode == 1, GVT_E_PARAM, "mode must be 0 or 1");
    GVT_REQUIRE((perm || n == 0) && row_ptr, GVT_E_PARAM, "NULL output");
    const int32_t *f = n ? (const int32_t *)gvt::stage_in(c, "dbg.f", first, sizeof(int32_t) * n) : nullptr;
    const int32_t *s = n ? (const int32_t *)gvt::stage_in(c, "dbg.s", second, sizeof(int32_t) * n) : nullptr;
    if (n) {
        GVT_REQUIRE(gvt::count_out_of_range(c, f, n, m) == 0, GVT_E_INDEX, "first id out of range");
        GVT_REQUIRE(gvt::count_out_of_range(c, s, n, q) == 0, GVT_E_INDEX, "second id out of range");
    }
    bool hp = n > 0 && !gvt::is_device_ptr(perm), hr = !gvt::is_device_ptr(row_ptr);
    int32_t *dperm = hp ? gvt::wsT<int32_t>(c, "dbg.perm", n) : perm;
    int64_t *drp = hr ? gvt::wsT<int64_t>(c, "dbg.rp", m + 1) : row_ptr;
    gvt::sort_plan_debug(c, f, s, n, m, q, mode, dperm, drp);
    if (hp && n) GVT_CUDA_TRY(cudaMemcpyAsync(perm, dperm, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    if (hr) GVT_CUDA_TRY(cudaMemcpyAsync(row_ptr, drp, sizeof(int64_t) * (m + 1), cudaMemcpyDeviceToHost, c->stream));
    if (hp || hr) GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    GVT_API_END
}

gvt_status gvt_relabel_compact(gvt_ctx *c, const int32_t *ids, int64_t n, int64_t bound, int32_t *compact,
                               int32_t *unique, int64_t *count) {
    GVT_API_BEGIN(c)
    GVT_REQUIRE(n >= 0 && bound >= 0, GVT_E_DIM, "negative size");
    GVT_REQUIRE(count && ((compact && unique) || n == 0), GVT_E_DIM, "NULL output");
    const int32_t *d = n ? (const int32_t *)gvt::stage_in(c, "rel.ids", ids, sizeof(int32_t) * n) : nullptr;
    if (n) GVT_REQUIRE(gvt::count_out_of_range(c, d, n, bound) == 0, GVT_E_INDEX, "id out of range [0, bound)");
    const bool hc = n > 0 && !gvt::is_device_ptr(compact), hu = n > 0 && !gvt::is_device_ptr(unique);
    int32_t *dc = hc ? gvt::wsT<int32_t>(c, "rel.compact", n) : compact;
    const int32_t *du = nullptr;
    const int64_t k = gvt::relabel_compact(c, d, n, bound, dc, &du);
    if (k > 0)
        GVT_CUDA_TRY(cudaMemcpyAsync(unique, du, sizeof(int32_t) * k, hu ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice,
                                     c->stream));
    if (hc) GVT_CUDA_TRY(cudaMemcpyAsync(compact, dc, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *count = k;
    GVT_API_END
}

gvt_status gvt_solver_direction(gvt_ctx *c, float *p_out, int64_t n) {
    GVT_API_BEGIN(c)
    GVT_REQUIRE(n >= 0 && (p_out || n == 0), GVT_E_DIM, "NULL output with n > 0");
    gvt::solver_direction(c, p_out, n);
    GVT_API_END
}

}  // extern "C"
