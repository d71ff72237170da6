// cgops.cuh -- the Hestenes-Stiefel CG state layout, scalar steps and per-range vector bodies
// (readings S12-S14, S32), shared by the separate CG kernels (cg.cu)
// and the fused dense-engine CG tail (tail.cu), so both run the same arithmetic on the same
// fixed partition: ranges [lo, hi) of the fixed-order partition over nb blocks, fp64 partials
// with the fixed shuffle tree of block_sum.  LDCG: read vectors through L2 (ld.global.cg), for
// data written by other CTAs earlier in the same launch (a persistent kernel's earlier phase).
#pragma once
#include "vecops.cuh"

namespace gvt {

enum { ST_RHO = 0, ST_ALPHA, ST_BETA, ST_YNORM, ST_PAP, ST_DONE, ST_BREAK, ST_ITERS, ST_TOL, ST_N };

// ||r_k|| / ||y|| at which the fp32 solvers stop as converged (2^-60, far below what fp32 vectors
// resolve; reading S32)
constexpr double RES_FLOOR = 8.673617379884035e-19;

__device__ __forceinline__ bool halted(const double *st) { return st[ST_DONE] != 0.0 || st[ST_BREAK] != 0.0; }

// the scalar steps (thread 0 of the reducing block)
__device__ __forceinline__ void cg_alpha_scalar(double pap, double *st) {
    st[ST_PAP] = pap;
    if (!(pap > 0.0)) st[ST_BREAK] = 1.0;
    else st[ST_ALPHA] = st[ST_RHO] / pap;
}

__device__ __forceinline__ void cg_beta_scalar(double rho1, double *st, double *relres) {
    double it = st[ST_ITERS] + 1.0;
    st[ST_ITERS] = it;
    double rr = sqrt(rho1) / st[ST_YNORM];
    if (relres) relres[(int64_t)it] = rr;
    // converged: the tolerance, or the residual floor RES_FLOOR (reading S32: below it the fp32
    // recurrences only underflow, into 0/0 after ~120 iterations on C1)
    if ((st[ST_TOL] > 0.0 && rr <= st[ST_TOL]) || rho1 == 0.0 || rr <= RES_FLOOR) st[ST_DONE] = 1.0;
    st[ST_BETA] = rho1 / st[ST_RHO];
    st[ST_RHO] = rho1;
}

// element range of (virtual) block b of nb in the fixed-order partition (block_range with gridDim.x = nb)
__device__ __forceinline__ void vblock_range(int64_t n, int64_t nb, int64_t b, int64_t &lo, int64_t &hi) {
    const int64_t per = (((n + nb - 1) / nb) + 3) & ~int64_t(3);
    lo = b * per;
    hi = lo + per < n ? lo + per : n;
    if (lo > n) lo = n;
}

template <bool LDCG, typename T>
__device__ __forceinline__ T vld(const T *p) {
    if constexpr (LDCG) return __ldcg(p);
    else return *p;
}

// Ap[i] += lambda p[i] over [lo, hi); returns this thread's share of p.Ap
template <bool LDCG>
__device__ __forceinline__ double cg_ap_range(float *__restrict__ Ap, const float *__restrict__ p, int64_t lo,
                                              int64_t hi, float lambda) {
    double acc = 0.0;
    if (aligned16(Ap) && aligned16(p)) {
        const int64_t lo4 = lo >> 2, hi4 = hi >> 2;
        float4 *A4 = reinterpret_cast<float4 *>(Ap);
        const float4 *p4 = reinterpret_cast<const float4 *>(p);
        for (int64_t i = lo4 + threadIdx.x; i < hi4; i += blockDim.x) {
            float4 a = vld<LDCG>(A4 + i), pp = vld<LDCG>(p4 + i);
            a.x = fmaf(lambda, pp.x, a.x); a.y = fmaf(lambda, pp.y, a.y);
            a.z = fmaf(lambda, pp.z, a.z); a.w = fmaf(lambda, pp.w, a.w);
            A4[i] = a;
            acc += (double)pp.x * a.x + (double)pp.y * a.y + (double)pp.z * a.z + (double)pp.w * a.w;
        }
        const int64_t t0 = (hi4 << 2) > lo ? (hi4 << 2) : lo;  // tail of the last non-empty block only
        for (int64_t i = t0 + threadIdx.x; i < hi; i += blockDim.x) {
            const float pi = vld<LDCG>(p + i);
            float a = fmaf(lambda, pi, vld<LDCG>(Ap + i));
            Ap[i] = a;
            acc += (double)pi * a;
        }
    } else {
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            float pi = vld<LDCG>(p + i);
            float a = fmaf(lambda, pi, vld<LDCG>(Ap + i));
            Ap[i] = a;
            acc += (double)pi * (double)a;
        }
    }
    return acc;
}

// x += alpha p ; r -= alpha Ap over [lo, hi); returns this thread's share of r.r
template <bool LDCG>
__device__ __forceinline__ double cg_xr_range(float *__restrict__ x, float *__restrict__ r,
                                              const float *__restrict__ p, const float *__restrict__ Ap, int64_t lo,
                                              int64_t hi, float alpha) {
    double acc = 0.0;
    if (aligned16(x) && aligned16(r) && aligned16(p) && aligned16(Ap)) {
        const int64_t lo4 = lo >> 2, hi4 = hi >> 2;
        float4 *x4 = reinterpret_cast<float4 *>(x);
        float4 *r4 = reinterpret_cast<float4 *>(r);
        const float4 *p4 = reinterpret_cast<const float4 *>(p), *a4 = reinterpret_cast<const float4 *>(Ap);
        for (int64_t i = lo4 + threadIdx.x; i < hi4; i += blockDim.x) {
            float4 xx = vld<LDCG>(x4 + i), rr = vld<LDCG>(r4 + i), pp = vld<LDCG>(p4 + i), aa = vld<LDCG>(a4 + i);
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
            x[i] = fmaf(alpha, vld<LDCG>(p + i), vld<LDCG>(x + i));
            float ri = fmaf(-alpha, vld<LDCG>(Ap + i), vld<LDCG>(r + i));
            r[i] = ri;
            acc += (double)ri * (double)ri;
        }
    } else {
        for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
            x[i] = fmaf(alpha, vld<LDCG>(p + i), vld<LDCG>(x + i));
            float ri = fmaf(-alpha, vld<LDCG>(Ap + i), vld<LDCG>(r + i));
            r[i] = ri;
            acc += (double)ri * (double)ri;
        }
    }
    return acc;
}

// p = r + beta p, element i handled by global thread t0 + j * nt (any partition: no reduction)
template <bool LDCG>
__device__ __forceinline__ void cg_p_grid(float *__restrict__ p, const float *__restrict__ r, int64_t n, float beta,
                                          int64_t t0, int64_t nt) {
    if (aligned16(p) && aligned16(r)) {
        const int64_t n4 = n >> 2;
        float4 *p4 = reinterpret_cast<float4 *>(p);
        const float4 *r4 = reinterpret_cast<const float4 *>(r);
        for (int64_t i = t0; i < n4; i += nt) {
            float4 pp = vld<LDCG>(p4 + i), rr = vld<LDCG>(r4 + i);
            pp.x = fmaf(beta, pp.x, rr.x); pp.y = fmaf(beta, pp.y, rr.y);
            pp.z = fmaf(beta, pp.z, rr.z); pp.w = fmaf(beta, pp.w, rr.w);
            p4[i] = pp;
        }
        for (int64_t i = (n4 << 2) + t0; i < n; i += nt) p[i] = fmaf(beta, vld<LDCG>(p + i), vld<LDCG>(r + i));
    } else {
        for (int64_t i = t0; i < n; i += nt) p[i] = fmaf(beta, vld<LDCG>(p + i), vld<LDCG>(r + i));
    }
}

}  // namespace gvt
