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
#include "vecops.cuh"

namespace gvt {

enum { ST_RHO = 0, ST_ALPHA, ST_BETA, ST_YNORM, ST_PAP, ST_DONE, ST_BREAK, ST_ITERS, ST_TOL, ST_N };

__device__ __forceinline__ bool halted(const double *st) { return st[ST_DONE] != 0.0 || st[ST_BREAK] != 0.0; }

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

// Ap += lambda p ; partial p.Ap
__global__ void __launch_bounds__(RED_THREADS) k_cg_ap(float *__restrict__ Ap, const float *__restrict__ p, int64_t n,
                                                       float lambda, const double *__restrict__ st,
                                                       double *__restrict__ part) {
    if (halted(st)) return;
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    if (aligned16(Ap) && aligned16(p)) {
        const int64_t lo4 = lo >> 2, hi4 = hi >> 2;
        float4 *A4 = reinterpret_cast<float4 *>(Ap);
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
        for (int64_t i = lo4 + threadIdx.x; i < hi4; i += blockDim.x) {
            float4 a = A4[i], pp = p4[i];
            a.x = fmaf(lambda, pp.x, a.x); a.y = fmaf(lambda, pp.y, a.y);
            a.z = fmaf(lambda, pp.z, a.z); a.w = fmaf(lambda, pp.w, a.w);
            A4[i] = a;
            acc += (double)pp.x * a.x + (double)pp.y * a.y + (double)pp.z * a.z + (double)pp.w * a.w;
        }
        const int64_t t0 = (hi4 << 2) > lo ? (hi4 << 2) : lo;  // tail of the last non-empty block only
        for (int64_t i = t0 + threadIdx.x; i < hi; i += blockDim.x) {
            float a = fmaf(lambda, p[i], Ap[i]);
            Ap[i] = a;
            acc += (double)p[i] * a;
        }
    } else {
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            float pi = p[i];
            float a = fmaf(lambda, pi, Ap[i]);
            Ap[i] = a;
            acc += (double)pi * (double)a;
        }
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(RED_THREADS) k_cg_alpha(const double *__restrict__ part, int nparts,
                                                          double *__restrict__ st) {
    if (halted(st)) return;
    double pap = reduce_parts(part, nparts);
    if (threadIdx.x == 0) {
        st[ST_PAP] = pap;
        if (!(pap > 0.0)) st[ST_BREAK] = 1.0;
        else st[ST_ALPHA] = st[ST_RHO] / pap;
    }
}

// x += alpha p ; r -= alpha Ap ; partial r.r
__global__ void __launch_bounds__(RED_THREADS) k_cg_xr(float *__restrict__ x, float *__restrict__ r,
                                                       const float *__restrict__ p, const float *__restrict__ Ap,
                                                       int64_t n, const double *__restrict__ st,
                                                       double *__restrict__ part) {
    if (halted(st)) return;
    const float alpha = (float)st[ST_ALPHA];
    int64_t lo, hi;
    block_range(n, lo, hi);
    double acc = 0.0;
    if (aligned16(x) && aligned16(r) && aligned16(p) && aligned16(Ap)) {
        const int64_t lo4 = lo >> 2, hi4 = hi >> 2;
        float4 *x4 = reinterpret_cast<float4 *>(x);
        float4 *r4 = reinterpret_cast<float4 *>(r);
        const float4 *p4 = reinterpret_cast<const float4 *>(p), *a4 = reinterpret_cast<const float4 *>(Ap);
        for (int64_t i = lo4 + threadIdx.x; i < hi4; i += blockDim.x) {
            float4 xx = x4[i], rr = r4[i], pp = p4[i], aa = a4[i];
            xx.x = fmaf(alpha, pp.x, xx.x); xx.y = fmaf(alpha, pp.y, xx.y);
            xx.z = fmaf(alpha, pp.z, xx.z); xx.w = fmaf(alpha, pp.w, xx.w);
            rr.x = fmaf(-alpha, aa.x, rr.x); rr.y = fmaf(-alpha, aa.y, rr.y);
            rr.z = fmaf(-alpha, aa.z, rr.z); rr.w = fmaf(-alpha, aa.w, rr.w);
            x4[i] = xx;
            r4[i] = rr;
            acc += (double)rr.x * rr.x + (double)rr.y * rr.y + (double)rr.z * rr.z + (double)rr.w * rr.w;
        }
        const int64_t t0 = (hi4 << 2) > lo ? (hi4 << 2) : lo;  // tail of the last non-empty block only
        for (int64_t i = t0 + threadIdx.x; i < hi; i += blockDim.x) {
            x[i] = fmaf(alpha, p[i], x[i]);
            float ri = fmaf(-alpha, Ap[i], r[i]);
            r[i] = ri;
            acc += (double)ri * (double)ri;
        }
    } else {
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            x[i] = fmaf(alpha, p[i], x[i]);
            float ri = fmaf(-alpha, Ap[i], r[i]);
            r[i] = ri;
            acc += (double)ri * (double)ri;
        }
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(RED_THREADS) k_cg_beta(const double *__restrict__ part, int nparts,
                                                         double *__restrict__ st, double *__restrict__ relres) {
    if (halted(st)) return;
    double rho1 = reduce_parts(part, nparts);
    if (threadIdx.x == 0) {
        double it = st[ST_ITERS] + 1.0;
        st[ST_ITERS] = it;
        double rr = sqrt(rho1) / st[ST_YNORM];
        if (relres) relres[(int64_t)it] = rr;
        if ((st[ST_TOL] > 0.0 && rr <= st[ST_TOL]) || rho1 == 0.0) st[ST_DONE] = 1.0;
        st[ST_BETA] = rho1 / st[ST_RHO];
        st[ST_RHO] = rho1;
    }
}

// p = r + beta p
__global__ void __launch_bounds__(RED_THREADS) k_cg_p(float *__restrict__ p, const float *__restrict__ r, int64_t n,
                                                      const double *__restrict__ st) {
    if (halted(st)) return;
    const float beta = (float)st[ST_BETA];
    if (aligned16(p) && aligned16(r)) {
        const int64_t n4 = n >> 2;
        float4 *p4 = reinterpret_cast<float4 *>(p);
        const float4 *r4 = reinterpret_cast<const float4 *>(r);
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
            float4 pp = p4[i], rr = r4[i];
            pp.x = fmaf(beta, pp.x, rr.x); pp.y = fmaf(beta, pp.y, rr.y);
            pp.z = fmaf(beta, pp.z, rr.z); pp.w = fmaf(beta, pp.w, rr.w);
            p4[i] = pp;
        }
        for (int64_t i = (n4 << 2) + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
             i += (int64_t)gridDim.x * blockDim.x)
            p[i] = fmaf(beta, p[i], r[i]);
    } else {
        for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
            p[i] = fmaf(beta, p[i], r[i]);
    }
}

// partial-sum slots [world][RED_BLOCKS]; this rank writes slot `rank`
double *solver_parts(gvt_ctx *c) { return wsT<double>(c, "cg.parts", (size_t)RED_BLOCKS * (c->world > 0 ? c->world : 1)); }
static double *my_parts(gvt_ctx *c) { return solver_parts(c) + (size_t)c->rank * RED_BLOCKS; }

void cg_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r, float *p, double *state, double rel_tol) {
    double *pt = solver_parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_init, RED_BLOCKS, RED_THREADS, 0, y, n, x, r, p, my_parts(c));
    allreduce_partials(c, pt, RED_BLOCKS);
    double *relres = state + ST_N;
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_init_scalars, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, rel_tol, state,
               relres);
}

void cg_after_matvec(gvt_ctx *c, float *Ap, const float *p, int64_t n, double lambda, double *state) {
    double *pt = solver_parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_ap, RED_BLOCKS, RED_THREADS, 0, Ap, p, n, (float)lambda, state, my_parts(c));
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_alpha, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state);
}

void cg_update(gvt_ctx *c, float *x, float *r, float *p, const float *Ap, int64_t n, double *state, int iter,
               double *relres_dev) {
    (void)iter;
    (void)relres_dev;
    double *pt = solver_parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_xr, RED_BLOCKS, RED_THREADS, 0, x, r, p, Ap, n, state, my_parts(c));
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_beta, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state, state + ST_N);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_p, RED_BLOCKS, RED_THREADS, 0, p, r, n, state);
}

}  // namespace gvt
