// solver.cu -- the paper's solver and its early-stopping protocol on the device:
//  * MINRES for (K + lambda I) a = y ("solved iteratively ... with the minimal residual
//    method"; "scipy.sparse.linalg.minres"): the unpreconditioned
//    Paige-Saunders recurrences, fp32 vectors, fp64 scalars kept on the device (no host round
//    trip per iteration), deterministic fixed-order reductions (vecops.cuh).
//  * validation AUC (Mann-Whitney, exact integer counting after a radix sort) and the
//    early-stopping rule "until the AUC stops increasing in Z_validation for a given number of
//    iterations", evaluated on the device after every iteration.
// The validation scores K_val,inner x_k are never recomputed from x_k: the fit's matvec runs
// over the out sample [inner; validation], so stage 1 is shared and the matvec also returns
// K_val v; the scores follow x's own recurrence (CG: s += alpha K_val p; MINRES: the w
// recurrence mirrored on K_val v).
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/iterator/transform_input_iterator.cuh>

#include "vecops.cuh"

namespace gvt {

// MINRES device state (doubles); DONE / BREAK / ITERS share the CG positions (cg.cu) so the
// early-stopping kernels work on either solver's state.
enum {
    MR_YNORM = 0, MR_BETA = 1, MR_OLDB = 2, MR_ALFA = 3, MR_DBAR = 4, MR_DONE = 5, MR_BREAK = 6, MR_ITERS = 7,
    MR_TOL = 8, MR_EPSLN, MR_OLDEPS, MR_DELTA, MR_CS, MR_SN, MR_PHIBAR, MR_PHI, MR_DENOM, MR_RAN, MR_TNORM2,
    MR_NSTATE
};
static_assert(MR_NSTATE == MINRES_STATE_N, "ops.cuh MINRES_STATE_N");
constexpr int ST_DONE_ = 5, ST_BREAK_ = 6, ST_ITERS_ = 7;

__device__ __forceinline__ bool mr_halted(const double *st) { return st[MR_DONE] != 0.0 || st[MR_BREAK] != 0.0; }

// x = 0, r1 = r2 = y, W1 = W2 = 0; partial y.y
__global__ void __launch_bounds__(RED_THREADS) k_mr_init(const float *__restrict__ y, int64_t n, float *__restrict__ x,
                                                         float *__restrict__ r1, float *__restrict__ r2,
                                                         float *__restrict__ W1, float *__restrict__ W2,
                                                         double *__restrict__ part) {
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        float v = y[i];
        x[i] = 0.f;
        r1[i] = v;
        r2[i] = v;
        W1[i] = 0.f;
        W2[i] = 0.f;
        acc += (double)v * (double)v;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(RED_THREADS) k_mr_init_scalars(const double *__restrict__ part, int nparts,
                                                                 double rel_tol, double *__restrict__ st,
                                                                 double *__restrict__ relres) {
    double b2 = reduce_parts(part, nparts);
    if (threadIdx.x == 0) {
        double beta1 = sqrt(b2);
        for (int k = 0; k < MR_NSTATE; k++) st[k] = 0.0;
        st[MR_YNORM] = beta1;
        st[MR_BETA] = beta1;
        st[MR_PHIBAR] = beta1;
        st[MR_CS] = -1.0;
        st[MR_TOL] = rel_tol;
        st[MR_DONE] = beta1 > 0.0 ? 0.0 : 1.0;  // y == 0 => a = 0 after 0 iterations
        if (relres) relres[0] = beta1 > 0.0 ? 1.0 : 0.0;
    }
}

// v = r2 / beta (first Lanczos vector; later ones are produced by k_mr_w)
__global__ void k_mr_v(float *__restrict__ v, const float *__restrict__ r2, int64_t n, const double *__restrict__ st) {
    if (mr_halted(st)) return;
    const float inv = (float)(1.0 / st[MR_BETA]);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        v[i] = r2[i] * inv;
}

// z = K v + lambda v - (beta / oldb) r1 (k >= 2), written over z = u; partial v.z
__global__ void __launch_bounds__(RED_THREADS) k_mr_a(float *__restrict__ u, const float *__restrict__ v,
                                                      const float *__restrict__ r1, int64_t n, float lambda,
                                                      const double *__restrict__ st, double *__restrict__ part) {
    if (mr_halted(st)) return;
    const float c1 = st[MR_ITERS] >= 1.0 ? (float)(st[MR_BETA] / st[MR_OLDB]) : 0.f;
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const float vi = v[i];
        float z = fmaf(lambda, vi, u[i]);
        z = fmaf(-c1, r1[i], z);
        u[i] = z;
        acc += (double)vi * (double)z;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// alfa = v.z; RAN marks that this iteration proceeds (the k_mr_r / givens / w passes follow it)
__global__ void __launch_bounds__(RED_THREADS) k_mr_alfa(const double *__restrict__ part, int nparts,
                                                         double *__restrict__ st) {
    if (mr_halted(st)) {
        if (threadIdx.x == 0) st[MR_RAN] = 0.0;
        return;
    }
    double alfa = reduce_parts(part, nparts);
    if (threadIdx.x == 0) {
        st[MR_ALFA] = alfa;
        st[MR_RAN] = 1.0;
    }
}

// z -= (alfa / beta) r2; r1 = r2; r2 = z; partial r2.r2
__global__ void __launch_bounds__(RED_THREADS) k_mr_r(const float *__restrict__ u, float *__restrict__ r1,
                                                      float *__restrict__ r2, int64_t n,
                                                      const double *__restrict__ st, double *__restrict__ part) {
    if (st[MR_RAN] == 0.0) return;
    const float c2 = (float)(st[MR_ALFA] / st[MR_BETA]);
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const float old = r2[i];
        const float z = fmaf(-c2, old, u[i]);
        r1[i] = old;
        r2[i] = z;
        acc += (double)z * (double)z;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

// beta_{k+1}, the previous rotation applied, the next plane rotation, phi / phibar (the
// Paige-Saunders scalar recurrences in SciPy's order); stopping tests
__global__ void __launch_bounds__(RED_THREADS) k_mr_givens(const double *__restrict__ part, int nparts,
                                                           double *__restrict__ st, double *__restrict__ relres) {
    if (st[MR_RAN] == 0.0) return;
    double b2 = reduce_parts(part, nparts);
    if (threadIdx.x == 0) {
        const double eps = 2.220446049250313e-16;
        const double beta = sqrt(b2), alfa = st[MR_ALFA];
        const double cs = st[MR_CS], sn = st[MR_SN], dbar = st[MR_DBAR];
        st[MR_OLDB] = st[MR_BETA];
        st[MR_BETA] = beta;
        st[MR_TNORM2] += alfa * alfa + beta * beta;
        st[MR_OLDEPS] = st[MR_EPSLN];
        st[MR_DELTA] = cs * dbar + sn * alfa;
        const double gbar = sn * dbar - cs * alfa;
        st[MR_EPSLN] = sn * beta;
        st[MR_DBAR] = -cs * beta;
        double gamma = sqrt(gbar * gbar + beta * beta);
        if (gamma < eps) gamma = eps;
        const double ncs = gbar / gamma, nsn = beta / gamma;
        st[MR_CS] = ncs;
        st[MR_SN] = nsn;
        const double phibar = st[MR_PHIBAR];
        st[MR_PHI] = ncs * phibar;
        st[MR_PHIBAR] = nsn * phibar;
        st[MR_DENOM] = 1.0 / gamma;
        const double it = st[MR_ITERS] + 1.0;
        st[MR_ITERS] = it;
        const double rr = st[MR_PHIBAR] / st[MR_YNORM];
        if (relres) relres[(int64_t)it] = rr;
        // converged, or Lanczos breakdown beta_{k+1} <= 64 u ||T_k||_F with u = 2^-24, the unit
        // roundoff of the fp32 vectors (reading M2; the oracle uses u = 2^-53): a normal exit
        const double bd = 64.0 * 5.9604644775390625e-08 * sqrt(st[MR_TNORM2]);
        // ... or the residual floor 2^-60 (reading S32, as the CG forms)
        if ((st[MR_TOL] > 0.0 && rr <= st[MR_TOL]) || beta <= bd || st[MR_PHIBAR] == 0.0 || rr <= 8.673617379884035e-19)
            st[MR_DONE] = 1.0;
    }
}

// w = (v - oldeps W1 - delta W2) / gamma; W1 = W2; W2 = w; x += phi w; and, unless the
// iteration stopped, the next Lanczos vector v = r2 / beta (r2 != nullptr)
__global__ void __launch_bounds__(RED_THREADS) k_mr_w(float *__restrict__ v, float *__restrict__ W1,
                                                      float *__restrict__ W2, float *__restrict__ x,
                                                      const float *__restrict__ r2, int64_t n,
                                                      const double *__restrict__ st) {
    if (st[MR_RAN] == 0.0) return;
    const float oldeps = (float)st[MR_OLDEPS], delta = (float)st[MR_DELTA], denom = (float)st[MR_DENOM];
    const float phi = (float)st[MR_PHI];
    const bool next = r2 != nullptr && st[MR_DONE] == 0.0;
    const float inv = next ? (float)(1.0 / st[MR_BETA]) : 0.f;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float vi = v[i], w1 = W1[i], w2 = W2[i];
        const float w = (vi - oldeps * w1 - delta * w2) * denom;
        W1[i] = w2;
        W2[i] = w;
        x[i] = fmaf(phi, w, x[i]);
        if (next) v[i] = r2[i] * inv;
    }
}

void minres_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r1, float *r2, float *v, float *W1,
                 float *W2, double *state, double rel_tol) {
    double *pt = solver_parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_mr_init, RED_BLOCKS, RED_THREADS, 0, y, n, x, r1, r2, W1, W2,
               pt + (size_t)c->rank * RED_BLOCKS);
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_mr_init_scalars, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, rel_tol, state,
               state + MR_NSTATE);
    GVT_LAUNCH(c, K_CG_VEC, k_mr_v, RED_BLOCKS, RED_THREADS, 0, v, r2, n, state);
}

void minres_step(gvt_ctx *c, float *u, float *v, float *r1, float *r2, float *W1, float *W2, float *x, int64_t n,
                 double lambda, double *state) {
    double *pt = solver_parts(c), *mine = pt + (size_t)c->rank * RED_BLOCKS;
    GVT_LAUNCH(c, K_CG_VEC, k_mr_a, RED_BLOCKS, RED_THREADS, 0, u, v, r1, n, (float)lambda, state, mine);
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_mr_alfa, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state);
    GVT_LAUNCH(c, K_CG_VEC, k_mr_r, RED_BLOCKS, RED_THREADS, 0, u, r1, r2, n, state, mine);
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_mr_givens, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state, state + MR_NSTATE);
}

// x-side w recurrence (+ next v) and, for early stopping, the same recurrence on the
// validation rows: kv = K_val v (the matvec's tail), KW1 / KW2 / s (n_val)
void minres_update(gvt_ctx *c, float *v, float *W1, float *W2, float *x, const float *r2, int64_t n, double *state,
                   float *kv, float *KW1, float *KW2, float *s, int64_t n_val) {
    GVT_LAUNCH(c, K_CG_VEC, k_mr_w, RED_BLOCKS, RED_THREADS, 0, v, W1, W2, x, r2, n, state);
    if (n_val > 0) GVT_LAUNCH(c, K_CG_VEC, k_mr_w, RED_BLOCKS, RED_THREADS, 0, kv, KW1, KW2, s, nullptr, n_val, state);
}

// ============================================================================ early stopping
// es[] (double, device): 0 best_auc, 1 best_iter, 2 bad (iterations without strict
// improvement), 3 last evaluated iteration, 4 improved-this-iteration flag
enum { ES_BEST = 0, ES_BEST_IT, ES_BAD, ES_LAST, ES_IMPROVED, ES_N };
static_assert(ES_N == ES_STATE_N, "ops.cuh ES_STATE_N");

__device__ __forceinline__ bool es_pending(const double *st, const double *es) {
    return st == nullptr || st[ST_ITERS_] > es[ES_LAST];
}

// CG: validation scores s += alpha K_val p (same guard and step as x += alpha p)
__global__ void k_es_cg_scores(float *__restrict__ s, const float *__restrict__ kp, int64_t n,
                               const double *__restrict__ st) {
    if (st[ST_DONE_] != 0.0 || st[ST_BREAK_] != 0.0) return;
    const float alpha = (float)st[1];  // cg.cu ST_ALPHA
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        s[i] = fmaf(alpha, kp[i], s[i]);
}

__global__ void k_pos_flags(const float *__restrict__ labels, int64_t n, uint8_t *__restrict__ pos,
                            unsigned long long *__restrict__ npos) {
    unsigned long long cnt = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t p = labels[i] > 0.f ? 1 : 0;  // reading A1: positive iff label > 0
        pos[i] = p;
        cnt += p;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(npos, cnt);
}

struct NegFlag {
    __host__ __device__ __forceinline__ long long operator()(const uint8_t &p) const { return p ? 0 : 1; }
};

__device__ __forceinline__ int64_t lower_bound_f(const float *__restrict__ a, int64_t n, float key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (a[mid] < key) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int64_t upper_bound_f(const float *__restrict__ a, int64_t n, float key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) >> 1;
        if (!(key < a[mid])) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// For each positive at sorted position i with tie group [lb, ub): negatives strictly below
// (negpre[lb]) count 1, tied negatives (negpre[ub] - negpre[lb]) count 1/2, so the doubled
// Mann-Whitney numerator gains negpre[lb] + negpre[ub] -- exact integer arithmetic.
__global__ void k_auc_count(const float *__restrict__ keys, const uint8_t *__restrict__ pos,
                            const long long *__restrict__ negpre, int64_t n, unsigned long long *__restrict__ twice,
                            const double *__restrict__ st, const double *__restrict__ es) {
    if (!es_pending(st, es)) return;
    unsigned long long acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        if (!pos[i]) continue;
        const float k = keys[i];
        const int64_t lb = lower_bound_f(keys, n, k), ub = upper_bound_f(keys, n, k);
        acc += (unsigned long long)(negpre[lb] + negpre[ub]);
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(twice, acc);  // integer sum: order-independent
}

// the rule (SPEC fit_early_stopping): strict improvement resets the
// patience counter; `patience` consecutive non-improvements stop the solver
__global__ void k_es_update(unsigned long long *__restrict__ twice, double P, double N, double *__restrict__ st,
                            double *__restrict__ es, double *__restrict__ hist, int patience) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (!es_pending(st, es)) {
        es[ES_IMPROVED] = 0.0;
        return;
    }
    const double it = st[ST_ITERS_];
    const double auc = (double)(*twice) / (2.0 * P * N);
    *twice = 0ull;
    hist[(int64_t)it - 1] = auc;
    if (auc > es[ES_BEST]) {
        es[ES_BEST] = auc;
        es[ES_BEST_IT] = it;
        es[ES_BAD] = 0.0;
        es[ES_IMPROVED] = 1.0;
    } else {
        es[ES_BAD] += 1.0;
        es[ES_IMPROVED] = 0.0;
        if (es[ES_BAD] >= (double)patience) st[ST_DONE_] = 1.0;
    }
    es[ES_LAST] = it;
}

__global__ void k_es_copy(const float *__restrict__ x, float *__restrict__ a_best, int64_t n,
                          const double *__restrict__ es) {
    if (es[ES_IMPROVED] == 0.0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        a_best[i] = x[i];
}

__global__ void k_es_init(double *__restrict__ es, double *__restrict__ hist, int max_iter,
                          unsigned long long *__restrict__ twice, long long *__restrict__ negpre0) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    es[ES_BEST] = -1.0;
    es[ES_BEST_IT] = 0.0;
    es[ES_BAD] = 0.0;
    es[ES_LAST] = 0.0;
    es[ES_IMPROVED] = 0.0;
    for (int k = 0; k < max_iter; k++) hist[k] = 0.0 / 0.0;
    *twice = 0ull;
    *negpre0 = 0ll;
}

// AUC machinery over n scores with labels (device): positive flags once, then per evaluation
// a radix sort of (score, flag), an inclusive scan of the negative flags and the count.
void AucPlan::setup(gvt_ctx *c, const char *tag, const float *labels_dev, int64_t n_) {
    n = n_;
    std::string t(tag);
    GVT_REQUIRE(n < (int64_t)INT32_MAX, GVT_E_DIM, "AUC: more than 2^31-1 scores");
    pos = wsT<uint8_t>(c, (t + ".pos").c_str(), (size_t)n);
    pos_sorted = wsT<uint8_t>(c, (t + ".pos_s").c_str(), (size_t)n);
    keys_sorted = wsT<float>(c, (t + ".keys_s").c_str(), (size_t)n);
    negpre = wsT<long long>(c, (t + ".negpre").c_str(), (size_t)n + 1);
    twice = wsT<unsigned long long>(c, (t + ".twice").c_str(), 2);
    unsigned long long *cnt = twice + 1;
    GVT_CUDA_TRY(cudaMemsetAsync(twice, 0, 2 * sizeof(unsigned long long), c->stream));
    GVT_CUDA_TRY(cudaMemsetAsync(negpre, 0, sizeof(long long), c->stream));
    if (n > 0) GVT_LAUNCH(c, K_AUC, k_pos_flags, grid1d(n, 256, 4 * 148), 256, 0, labels_dev, n, pos, cnt);
    unsigned long long hpos = 0;
    GVT_CUDA_TRY(cudaMemcpyAsync(&hpos, cnt, sizeof(hpos), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    P = (double)hpos;
    N = (double)(n - (int64_t)hpos);
    GVT_REQUIRE(P > 0 && N > 0, GVT_E_PARAM, "degenerate validation labels: AUC needs both classes (label > 0 and <= 0)");
    size_t t1 = 0, t2 = 0;
    GVT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, t1, (const float *)nullptr, keys_sorted,
                                                 (const uint8_t *)nullptr, pos_sorted, (int)n, 0, 32, c->stream));
    cub::TransformInputIterator<long long, NegFlag, const uint8_t *> it(pos_sorted, NegFlag());
    GVT_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, t2, it, negpre + 1, (int)n, c->stream));
    temp_bytes = t1 > t2 ? t1 : t2;
    temp = ws(c, (t + ".cubtmp").c_str(), temp_bytes);
}

// doubled Mann-Whitney numerator of `scores` into *twice (gated by the solver state when
// st != nullptr: only when an iteration completed since the last evaluation)
void AucPlan::count(gvt_ctx *c, const float *scores, const double *st, const double *es) {
    if (n == 0) return;
    cudaEvent_t ev;
    launch_begin(c, K_AUC, &ev);
    size_t tb = temp_bytes;
    GVT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(temp, tb, scores, keys_sorted, pos, pos_sorted, (int)n, 0, 32,
                                                 c->stream));
    cub::TransformInputIterator<long long, NegFlag, const uint8_t *> it(pos_sorted, NegFlag());
    tb = temp_bytes;
    GVT_CUDA_TRY(cub::DeviceScan::InclusiveSum(temp, tb, it, negpre + 1, (int)n, c->stream));
    launch_end(c, K_AUC, ev);
    GVT_LAUNCH(c, K_AUC, k_auc_count, grid1d(n, 256, 8 * 148), 256, 0, keys_sorted, pos_sorted, negpre, n, twice, st,
               es);
}

double auc(gvt_ctx *c, const float *labels, const float *scores, int64_t n) {
    GVT_REQUIRE(n >= 0, GVT_E_DIM, "negative n");
    GVT_REQUIRE(n == 0 || (labels && scores), GVT_E_DIM, "labels or scores is NULL");
    const float *ld = n ? (const float *)stage_in(c, "auc.labels", labels, sizeof(float) * n) : nullptr;
    const float *sd = n ? (const float *)stage_in(c, "auc.scores", scores, sizeof(float) * n) : nullptr;
    AucPlan a;
    a.setup(c, "auc", ld, n);
    a.count(c, sd, nullptr, nullptr);
    unsigned long long tw = 0;
    GVT_CUDA_TRY(cudaMemcpyAsync(&tw, a.twice, sizeof(tw), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return (double)tw / (2.0 * a.P * a.N);
}

void es_init(gvt_ctx *c, double *es, double *hist, int max_iter, AucPlan &a) {
    GVT_LAUNCH(c, K_CG_SCALAR, k_es_init, 1, 32, 0, es, hist, max_iter, a.twice, a.negpre);
}

void es_cg_scores(gvt_ctx *c, float *s, const float *kp, int64_t n_val, const double *state) {
    if (n_val > 0) GVT_LAUNCH(c, K_CG_VEC, k_es_cg_scores, grid1d(n_val, 256, 8 * 148), 256, 0, s, kp, n_val, state);
}

void es_evaluate(gvt_ctx *c, AucPlan &a, const float *scores_full, double *state, double *es, double *hist,
                 int patience, const float *x, float *a_best, int64_t n) {
    a.count(c, scores_full, state, es);
    GVT_LAUNCH(c, K_CG_SCALAR, k_es_update, 1, 32, 0, a.twice, a.P, a.N, state, es, hist, patience);
    if (n > 0 && a_best) GVT_LAUNCH(c, K_CG_VEC, k_es_copy, grid1d(n, 256, 8 * 148), 256, 0, x, a_best, n, es);
}

}  // namespace gvt
