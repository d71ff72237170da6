// cg.cu -- conjugate-gradient vector steps for (K + lambda I) a = y (PAPER.md:288-290,
// 316-320; reading S12-S14), north-star kernel (4).  Vectors fp32, dot products fp64
// with a fixed two-level reduction (RED_BLOCKS per-block partials, then one block in a
// fixed order) so the scalars are bit-identical run to run; all scalar logic (alpha,
// beta, breakdown, stopping) stays on the device -- no host round trip per iteration
// in fixed-iteration mode.
//
// state[] (double, device): 0 rho, 1 alpha, 2 beta, 3 ||y||, 4 pAp, 5 done, 6 breakdown,
//                           7 iters, 8 rel_tol
#include "ops.cuh"

namespace gvt {

enum { ST_RHO = 0, ST_ALPHA, ST_BETA, ST_YNORM, ST_PAP, ST_DONE, ST_BREAK, ST_ITERS, ST_TOL, ST_N };

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[RED_THREADS];
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = RED_THREADS / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) sh[threadIdx.x] += sh[threadIdx.x + o];
        __syncthreads();
    }
    double r = sh[0];
    __syncthreads();
    return r;
}

__device__ __forceinline__ bool halted(const double *st) { return st[ST_DONE] != 0.0 || st[ST_BREAK] != 0.0; }

__global__ void __launch_bounds__(RED_THREADS) k_cg_init(const float *__restrict__ y, int64_t n, float *__restrict__ x,
                                                         float *__restrict__ r, float *__restrict__ p,
                                                         double *__restrict__ part) {
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = y[i];
        x[i] = 0.f;
        r[i] = v;
        p[i] = v;
        acc += (double)v * (double)v;
    }
    acc = block_sum(acc);
    if (threadIdx.x == 0) part[blockIdx.x] = acc;
}

__device__ double reduce_parts(const double *__restrict__ part, int nparts) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += part[i];
    return block_sum(acc);
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
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float pi = p[i];
        float a = fmaf(lambda, pi, Ap[i]);
        Ap[i] = a;
        acc += (double)pi * (double)a;
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
    double acc = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        x[i] = fmaf(alpha, p[i], x[i]);
        float ri = fmaf(-alpha, Ap[i], r[i]);
        r[i] = ri;
        acc += (double)ri * (double)ri;
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
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = fmaf(beta, p[i], r[i]);
}

// partial-sum slots [world][RED_BLOCKS]; this rank writes slot `rank`
static double *parts(gvt_ctx *c) { return wsT<double>(c, "cg.parts", (size_t)RED_BLOCKS * (c->world > 0 ? c->world : 1)); }
static double *my_parts(gvt_ctx *c) { return parts(c) + (size_t)c->rank * RED_BLOCKS; }

void cg_init(gvt_ctx *c, const float *y, int64_t n, float *x, float *r, float *p, double *state, double rel_tol) {
    double *pt = parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_init, RED_BLOCKS, RED_THREADS, 0, y, n, x, r, p, my_parts(c));
    allreduce_partials(c, pt, RED_BLOCKS);
    double *relres = state + ST_N;
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_init_scalars, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, rel_tol, state,
               relres);
}

void cg_after_matvec(gvt_ctx *c, float *Ap, const float *p, int64_t n, double lambda, double *state) {
    double *pt = parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_ap, RED_BLOCKS, RED_THREADS, 0, Ap, p, n, (float)lambda, state, my_parts(c));
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_alpha, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state);
}

void cg_update(gvt_ctx *c, float *x, float *r, float *p, const float *Ap, int64_t n, double *state, int iter,
               double *relres_dev) {
    (void)iter;
    (void)relres_dev;
    double *pt = parts(c);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_xr, RED_BLOCKS, RED_THREADS, 0, x, r, p, Ap, n, state, my_parts(c));
    allreduce_partials(c, pt, RED_BLOCKS);
    GVT_LAUNCH(c, K_CG_SCALAR, k_cg_beta, 1, RED_THREADS, 0, pt, RED_BLOCKS * c->world, state, state + ST_N);
    GVT_LAUNCH(c, K_CG_VEC, k_cg_p, RED_BLOCKS * 4, RED_THREADS, 0, p, r, n, state);
}

}  // namespace gvt
