// cg.cu -- conjugate-gradient vector steps for (K + lambda I) a = y (PAPER.md:288-290,
// 316-320; reading S12-S14), north-star kernel (4).  Vectors fp32, dot products fp64
// with a fixed two-level reduction (RED_BLOCKS per-block partials, then one block in a
// fixed order) so the scalars are bit-identical run to run; all scalar logic (alpha,
// beta, breakdown, stopping) stays on the device -- no host round trip per iteration
// in fixed-iteration mode.  The vector passes are HBM-bound: 128-bit loads when the
// vectors are 16-byte aligned, RED_BLOCKS = 8 x 148 blocks.
//
// state[] (double, device): 0 rho, 1 alpha, 2 beta, 3 ||y||, 4 pAp, 5 done, 6 breakdown,
//                           7 iters, 8 rel_tol
#include "cgops.cuh"

namespace gvt {

__global__ void __launch_bounds__(RED_THREADS) k_cg_init(const float *__restrict__ y, int64_t n, float *__restrict__ x,
                                                         float *__restrict__ r, float *__restrict__ p,
                                                         double *__restrict__ part) {
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        float v = y[i];
        x[i] = 0.f;
        r[i] = v;
        p[i] = v;
        acc += (double)v * (double)v;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(RED_THREADS) k_cg_init_scalars(const double *__restrict__ part, int nparts,
                                                                 double rel_tol, double *__restrict__ st,
                                                                 double *__restrict__ relres) {
    double rho = reduce_parts(part, nparts);
    if (threadIdx.x == 0) {
        st[ST_RHO] = rho;
        st[ST_ALPHA] = 0.0;
        st[ST_BETA] = 0.0;
        st[ST_YNORM] = sqrt(rho);
        st[ST_PAP] = 0.0;
        st[ST_DONE] = (rho > 0.0) ? 0.0 : 1.0;  // y == 0 => a = 0 after 0 iterations
        st[ST_BREAK] = 0.0;
        st[ST_ITERS] = 0.0;
        st[ST_TOL] = rel_tol;
        if (relres) relres[0] = rho > 0.0 ? 1.0 : 0.0;
    }
}

// Ap += lambda p ; partial p.Ap.  With a ticket (single GPU), the last block to finish also reduces
// the partials and takes the alpha step (k_cg_alpha folded in: one launch fewer per iteration).
__global__ void __launch_bounds__(RED_THREADS) k_cg_ap(float *__restrict__ Ap, const float *__restrict__ p, int64_t n,
                                                       float lambda, double *__restrict__ st,
                                                       double *__restrict__ part, unsigned *__restrict__ ticket) {
    if (halted(st)) return;
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = cg_ap_range<false>(Ap, p, lo, hi, lambda);
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
    if (ticket && last_block_done(ticket)) {
        const double pap = reduce_parts_cg(part, RED_BLOCKS);  // (unused slots are zero: cg_init)
        if (threadIdx.x == 0) {
            cg_alpha_scalar(pap, st);
            *ticket = 0u;
        }
    }
}

// The fused CG tail (k_combine_gather + k_cg_ap in one pass; single GPU): per output i of this block's
// fixed range, u_i = c1 g1[.] + c2 g2[.] (+ u_i), the direction p_i (= r_i + beta p_i when r_lazy, then
// stored), Ap_i = u_i + lambda p_i stored over u, and the p.Ap partial; the last block takes the alpha
// step.  The arithmetic per element is that of the two separate kernels.
__global__ void __launch_bounds__(RED_THREADS) k_cg_combine_ap(
    const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n, const float *__restrict__ g1, int rs1,
    float c1, const float *__restrict__ g2, int rs2, float c2, int accumulate, float *__restrict__ u,
    float *__restrict__ p, const float *__restrict__ r_lazy, float lambda, double *__restrict__ st,
    double *__restrict__ part, unsigned *__restrict__ ticket) {
    if (halted(st)) return;
    const float beta = r_lazy ? (float)st[ST_BETA] : 0.f;
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        float v = c1 * g1[rs1 == 0 ? f[i] : s[i]];
        if (g2) v = fmaf(c2, g2[rs2 == 0 ? f[i] : s[i]], v);
        const float ui = accumulate ? u[i] + v : v;
        float pi = p[i];
        if (r_lazy) {
            pi = fmaf(beta, pi, r_lazy[i]);
            p[i] = pi;
        }
        const float a = fmaf(lambda, pi, ui);
        u[i] = a;
        acc += (double)pi * (double)a;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
    if (last_block_done(ticket)) {
        const double pap = reduce_parts_cg(part, RED_BLOCKS);  // (unused slots are zero: cg_init)
        if (threadIdx.x == 0) {
            cg_alpha_scalar(pap, st);
            *ticket = 0u;
        }
    }
}

__global__ void __launch_bounds__(RED_THREADS) k_cg_alpha(const double *__restrict__ part, int nparts,
                                                          double *__restrict__ st) {
    if (halted(st)) return;
    double pap = reduce_parts(part, nparts);
    if (threadIdx.x == 0) cg_alpha_scalar(pap, st);
}

// x += alpha p ; r -= alpha Ap ; partial r.r.  With a ticket (single GPU), the last block also
// takes the beta / stopping step (k_cg_beta folded in).
__global__ void __launch_bounds__(RED_THREADS) k_cg_xr(float *__restrict__ x, float *__restrict__ r,
                                                       const float *__restrict__ p, const float *__restrict__ Ap,
                                                       int64_t n, double *__restrict__ st,
                                                       double *__restrict__ part, unsigned *__restrict__ ticket,
                                                       double *__restrict__ relres) {
    if (halted(st)) return;
    const float alpha = (float)st[ST_ALPHA];
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = cg_xr_range<false>(x, r, p, Ap, lo, hi, alpha);
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
    if (ticket && last_block_done(ticket)) {
        const double rho1 = reduce_parts_cg(part, RED_BLOCKS);
        if (threadIdx.x == 0) {
            cg_beta_scalar(rho1, st, relres);
            *ticket = 0u;
        }
    }
}

__global__ void __launch_bounds__(RED_THREADS) k_cg_beta(const double *__restrict__ part, int nparts,
                                                         double *__restrict__ st, double *__restrict__ relres) {
    if (halted(st)) return;
    double rho1 = reduce_parts(part, nparts);
    if (threadIdx.x == 0) cg_beta_scalar(rho1, st, relres);
}

// p = r + beta p
__global__ void __launch_bounds__(RED_THREADS) k_cg_p(float *__restrict__ p, const float *__restrict__ r, int64_t n,
                                                      const double *__restrict__ st) {
    if (halted(st)) return;
    cg_p_grid<false>(p, r, n, (float)st[ST_BETA], blockIdx.x * (int64_t)blockDim.x + threadIdx.x,
                     (int64_t)gridDim.x * blockDim.x);
}

// ============================================================================ single-reduction CG
// Chronopoulos-Gear CG (GVT_OPT_CG_VARIANT = 1; the "single fused all-reduce per CG iteration" of
// SURVEY.md 8(e) NEXT-3).  The same Krylov iterates as Hestenes-Stiefel CG in exact arithmetic,
// with the matvec applied to r instead of p and the two dot products of an iteration reduced
// together:
//   w_k = (K + lambda I) r_k;  gamma_k = r_k.r_k,  delta_k = w_k.r_k        (one reduction)
//   k = 0: beta = 0, alpha = gamma / delta;  else beta = gamma_k / gamma_{k-1},
//          alpha = gamma_k / (delta_k - beta gamma_k / alpha_{k-1})        (<= 0: breakdown)
//   p = r + beta p;  s = w + beta s;  x += alpha p;  r -= alpha s           (s = (K + lambda I) p)
// Per iteration: matvec + 3 kernels and one all-gather of 2 x 1184 partials, against 5 kernels
// and two collectives for the Hestenes-Stiefel form.  Residual mode stops before the update
// whose gamma_k meets the tolerance (the iterate and the count equal Hestenes-Stiefel's).
// state: 0 gamma_{k-1} (rho), 1 alpha, 2 beta, 3 ||y||, 4 delta, 5 done, 6 breakdown, 7 iters,
//        8 rel_tol -- the CG layout, so the host-side flags are the same.

// x = 0, r = y, p = s = 0; partial y.y
__global__ void __launch_bounds__(RED_THREADS) k_cgg_init(const float *__restrict__ y, int64_t n, float *__restrict__ x,
                                                          float *__restrict__ r, float *__restrict__ p,
                                                          float *__restrict__ sv, double *__restrict__ part) {
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const float v = y[i];
        x[i] = 0.f;
        r[i] = v;
        p[i] = 0.f;
        sv[i] = 0.f;
        acc += (double)v * (double)v;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__device__ void cgg_scalar_step(double g, double d, double *st, double *relres);

// w += lambda r; partials of r.r (part[b]) and w.r (part[RED_BLOCKS + b]).  With a ticket (single GPU)
// the last block also takes the scalar step (k_cgg_scalar folded in).
__global__ void __launch_bounds__(RED_THREADS) k_cgg_dots(float *__restrict__ w, const float *__restrict__ r,
                                                          int64_t n, float lambda, double *__restrict__ st,
                                                          double *__restrict__ part, unsigned *__restrict__ ticket,
                                                          double *__restrict__ relres) {
    if (halted(st)) return;
    int64_t lo, hi;
    block_range(n, lo, hi);
    double g = 0.0, d = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const float ri = r[i];
        const float wi = fmaf(lambda, ri, w[i]);
        w[i] = wi;
        g += (double)ri * (double)ri;
        d += (double)wi * (double)ri;
    }
    g = block_sum(g);
    d = block_sum(d);
    if (threadIdx.x == 0) {
        part[blockIdx.x] = g;
        part[RED_BLOCKS + blockIdx.x] = d;
    }
    if (ticket && last_block_done(ticket)) {
        const double gg = reduce_parts_cg(part, RED_BLOCKS), dd = reduce_parts_cg(part + RED_BLOCKS, RED_BLOCKS);
        if (threadIdx.x == 0) {
            cgg_scalar_step(gg, dd, st, relres);
            *ticket = 0u;
        }
    }
}

// partials laid out [world][2][RED_BLOCKS] (all-gathered as one slot of 2 * RED_BLOCKS per rank)
__global__ void __launch_bounds__(RED_THREADS) k_cgg_scalar(const double *__restrict__ part, int world,
                                                            double *__restrict__ st, double *__restrict__ relres) {
    if (halted(st)) return;
    double g = 0.0, d = 0.0;
    for (int r = 0; r < world; r++) {  // fixed order: rank by rank
        g += reduce_parts(part + (size_t)r * 2 * RED_BLOCKS, RED_BLOCKS);
        d += reduce_parts(part + (size_t)r * 2 * RED_BLOCKS + RED_BLOCKS, RED_BLOCKS);
    }
    if (threadIdx.x == 0) cgg_scalar_step(g, d, st, relres);
}

__device__ void cgg_scalar_step(double g, double d, double *st, double *relres) {
    const double k = st[ST_ITERS];
    const double rr = sqrt(g) / st[ST_YNORM];
    if (relres) relres[(int64_t)k] = rr;
    if ((st[ST_TOL] > 0.0 && rr <= st[ST_TOL]) || g == 0.0 || rr <= RES_FLOOR) {
        st[ST_DONE] = 1.0;
        return;
    }
    double beta = 0.0, den = d;
    if (k >= 1.0) {
        beta = g / st[ST_RHO];
        den = d - beta * g / st[ST_ALPHA];
    }
    st[ST_PAP] = den;  // p.(K + lambda I)p of the direction this update uses
    if (!(den > 0.0)) {
        st[ST_BREAK] = 1.0;
        return;
    }
    st[ST_BETA] = beta;
    st[ST_ALPHA] = g / den;
    st[ST_RHO] = g;
    st[ST_ITERS] = k + 1.0;
}

// p = r + beta p; s = w + beta s; x += alpha p; r -= alpha s
__global__ void __launch_bounds__(RED_THREADS) k_cgg_update(float *__restrict__ x, float *__restrict__ r,
                                                            float *__restrict__ p, float *__restrict__ sv,
                                                            const float *__restrict__ w, int64_t n,
                                                            const double *__restrict__ st) {
    if (halted(st)) return;
    const float alpha = (float)st[ST_ALPHA], beta = (float)st[ST_BETA];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const float pi = fmaf(beta, p[i], r[i]);
        const float si = fmaf(beta, sv[i], w[i]);
        p[i] = pi;
        sv[i] = si;
        x[i] = fmaf(alpha, pi, x[i]);
        r[i] = fmaf(-alpha, si, r[i]);
    }
}

// after the loop: ||r_K|| for the residual history (one more reduction, no matvec)
__global__ void __launch_bounds__(RED_THREADS) k_cgg_rr(const float *__restrict__ r, int64_t n, double *__restrict__ part) {
    int64_t lo, hi;
    block_range(n, lo, hi);
    double g = 0.0;
    for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) g += (double)r[i] * (double)r[i];
    g = block_sum(g);
    if (threadIdx.x == 0) part[blockIdx.x] = g;
}

__global__ void __launch_bounds__(RED_THREADS) k_cgg_final(const double *__restrict__ part, int nparts,
                                                           const double *__restrict__ st, double *__restrict__ relres) {
    const double g = reduce_parts(part, nparts);
    if (threadIdx.x == 0 && relres && st[ST_BREAK] == 0.0 && st[ST_DONE] == 0.0)
        relres[(int64_t)st[ST_ITERS]] = sqrt(g) / st[ST_YNORM];
}

// partial-sum slots [world][2 * RED_BLOCKS]; this rank writes slot `rank`
static double *parts2(gvt_ctx *c) { return wsT<double>(c, "cgg.parts", (size_t)2 * RED_BLOCKS * (c->world > 0 ? c->world : 1)); }

// blocks of the CG vector kernels: about 1024 elements per block, at most RED_BLOCKS (C2: 30, C5: 1184)
// -- a function of n only, so the partition (and every partial) stays fixed run to run.  The partial
// slots past the used blocks are zero (set once per fit), so every reduction over RED_BLOCKS slots
// (fused last block, separate scalar kernel, across ranks) sums the same values in the same tree.
static int vec_blocks(int64_t n) { return (int)std::min<int64_t>(RED_BLOCKS, std::max<int64_t>(1, (n + 1023) / 1024)); }

// single-GPU: the scalar steps run in the last block of the vector kernels (last_block_done)
static unsigned *cg_ticket(gvt_ctx *c) { return distributed(c) ? nullptr : wsT<unsigned>(c, "cg.ticket", 1); }

void cgg_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r, float *p, float *sv, double *state,
              double rel_tol) {
    double *pt = solver_parts(c);
    const int w = c->world > 0 ? c->world : 1;
    GVT_CUDA_TRY(cudaMemsetAsync(pt, 0, sizeof(double) * RED_BLOCKS * w, c->stream));
    GVT_CUDA_TRY(cudaMemsetAsync(parts2(c), 0, sizeof(double) * 2 * RED_BLOCKS * w, c->stream));
    if (unsigned *tk = cg_ticket(c)) GVT_CUDA_TRY(cudaMemsetAsync(tk, 0, sizeof(unsigned), c->stream));
    GVT_LAUNCH(c, K_CG_VEC, k_cgg_init, vec_blocks(n), RED_THREADS, 0, y, n, x, r, p, sv,
               pt + (size_t)c->rank * RED_BLOCKS);
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_init_scalars, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, rel_tol, state,
               state + ST_N);
}

void cgg_step(gvt_ctx *c, float *x, float *r, float *p, float *sv, float *w, int64_t n, double lambda,
              double *state) {
    double *pt = parts2(c);
    unsigned *tk = cg_ticket(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cgg_dots, vec_blocks(n), RED_THREADS, 0, w, r, n, (float)lambda, state,
               pt + (size_t)c->rank * 2 * RED_BLOCKS, tk, state + ST_N);
    if (!tk) {
        allreduce_partials(c, pt, 2 * RED_BLOCKS);  // the iteration's single collective
        GVT_LAUNCH(c, K_CG_SCALAR, k_cgg_scalar, 1, RED_THREADS, 0, pt, c->world, state, state + ST_N);
    }
    GVT_LAUNCH(c, K_CG_VEC, k_cgg_update, vec_blocks(n), RED_THREADS, 0, x, r, p, sv, w, n, state);
}

void cgg_finish(gvt_ctx *c, const float *r, int64_t n, double *state) {
    double *pt = solver_parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cgg_rr, vec_blocks(n), RED_THREADS, 0, r, n, pt + (size_t)c->rank * RED_BLOCKS);
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_cgg_final, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state, state + ST_N);
}

// partial-sum slots [world][RED_BLOCKS]; this rank writes slot `rank`
int cg_vec_blocks(int64_t n) { return vec_blocks(n); }
double *cg_parts(gvt_ctx *c) { return solver_parts(c); }

double *solver_parts(gvt_ctx *c) { return wsT<double>(c, "cg.parts", (size_t)RED_BLOCKS * (c->world > 0 ? c->world : 1)); }
static double *my_parts(gvt_ctx *c) { return solver_parts(c) + (size_t)c->rank * RED_BLOCKS; }

void cg_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r, float *p, double *state, double rel_tol) {
    double *pt = solver_parts(c);
    GVT_CUDA_TRY(cudaMemsetAsync(pt, 0, sizeof(double) * RED_BLOCKS * (c->world > 0 ? c->world : 1), c->stream));
    if (unsigned *tk = cg_ticket(c)) GVT_CUDA_TRY(cudaMemsetAsync(tk, 0, sizeof(unsigned), c->stream));
    GVT_LAUNCH(c, K_CG_VEC, k_cg_init, vec_blocks(n), RED_THREADS, 0, y, n, x, r, p, my_parts(c));
    allreduce_partials(c, pt, RED_BLOCKS);
    double *relres = state + ST_N;
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_init_scalars, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, rel_tol, state,
               relres);
}

void cg_after_matvec(gvt_ctx *c, float *Ap, const float *p, int64_t n, double lambda, double *state) {
    double *pt = solver_parts(c);
    unsigned *tk = cg_ticket(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_ap, vec_blocks(n), RED_THREADS, 0, Ap, p, n, (float)lambda, state, my_parts(c), tk);
    if (tk) return;
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_alpha, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state);
}

void cg_combine_ap(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, const float *g1, int rs1, float c1,
                   const float *g2, int rs2, float c2, int accumulate, float *u, float *p, const float *r_lazy,
                   double lambda, double *state) {
    unsigned *tk = cg_ticket(c);
    GVT_REQUIRE(tk, GVT_E_STATE, "the fused CG tail is single-GPU only");
    GVT_LAUNCH(c, K_CG_VEC, k_cg_combine_ap, vec_blocks(n), RED_THREADS, 0, f, s, n, g1, rs1, c1, g2, rs2, c2,
               accumulate, u, p, r_lazy, (float)lambda, state, my_parts(c), tk);
}

void cg_update_xr(gvt_ctx *c, float *x, float *r, const float *p, const float *Ap, int64_t n, double *state) {
    unsigned *tk = cg_ticket(c);
    GVT_REQUIRE(tk, GVT_E_STATE, "the fused CG tail is single-GPU only");
    GVT_LAUNCH(c, K_CG_VEC, k_cg_xr, vec_blocks(n), RED_THREADS, 0, x, r, p, Ap, n, state, my_parts(c), tk,
               state + ST_N);
}

void cg_direction(gvt_ctx *c, float *p, const float *r, int64_t n, const double *state) {
    GVT_LAUNCH(c, K_CG_VEC, k_cg_p, vec_blocks(n), RED_THREADS, 0, p, r, n, state);
}

void cg_update(gvt_ctx *c, float *x, float *r, float *p, const float *Ap, int64_t n, double *state, int iter,
               double *relres_dev) {
    (void)iter;
    (void)relres_dev;
    double *pt = solver_parts(c);
    unsigned *tk = cg_ticket(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_xr, vec_blocks(n), RED_THREADS, 0, x, r, p, Ap, n, state, my_parts(c), tk,
               state + ST_N);
    if (!tk) {
        allreduce_partials(c, pt, RED_BLOCKS);
        GVT_LAUNCH(c, K_CG_SCALAR, k_cg_beta, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state, state + ST_N);
    }
    GVT_LAUNCH(c, K_CG_VEC, k_cg_p, vec_blocks(n), RED_THREADS, 0, p, r, n, state);
}

}  // namespace gvt
