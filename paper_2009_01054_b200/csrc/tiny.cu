// tiny.cu -- the whole CG fit of a small Kronecker problem in ONE single-CTA kernel launch.
//
// The latency-bound configurations (C1, "report us per iteration; target: the
// CUDA-graph floor") spend their time in kernel boundaries, not arithmetic: a graph-replayed
// iteration is ~10 launches (~60 us at C1) for ~1e5 FMAs.  When the factors, S and the solver
// vectors fit in one SM's shared memory, one 1024-thread CTA runs every iteration of
// Hestenes-Stiefel CG (readings S12-S14, S32) with __syncthreads
// between the phases -- the GVT of Theorem 1 (variant 1) on the sorted entry
// plan and the sample plan of the Kronecker group:
//   S[t][h] = sum_{k in row h} sign_k p[src_k] T[col_k][t]       (stage 1, T symmetric, R1)
//   Ap[dst] = sum_h D[r][h] S[c][h] + lambda p[dst]                (stage 2 + ridge term)
//   alpha = rho / p.Ap;  x += alpha p;  r -= alpha Ap;  beta = r.r / rho;  p = r + beta p
// Dot products are fp64 with a fixed reduction tree (deterministic, reading S26).  The device
// state and residual history use the CG layout of cg.cu, so the host reads them the same way.
#include "vecops.cuh"

namespace gvt {

enum { TS_RHO = 0, TS_ALPHA, TS_BETA, TS_YNORM, TS_PAP, TS_DONE, TS_BREAK, TS_ITERS, TS_TOL, TS_N };
constexpr int TINY_THREADS = 1024;

// fixed-tree fp64 block sum over 1024 threads; every thread gets the result
__device__ __forceinline__ double tiny_sum(double v, double *red) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = red[threadIdx.x];
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
        if (threadIdx.x == 0) red[32] = r;
    }
    __syncthreads();
    r = red[32];
    __syncthreads();
    return r;
}

struct TinyArgs {
    const float *T;
    int64_t ldT;  // factor of stage 1 (q x q, symmetric): row col holds T[col][0..q)
    const float *D;
    int64_t ldD;  // factor of stage 2 (m x m)
    int m, q;     // drugs (rows of X = columns of S), targets (rows of S)
    const int64_t *row_ptr;
    const int32_t *col, *src;
    const float *sign;
    int64_t ns;
    const int32_t *sr, *sc, *sdst;
    const float *y;
    float *x;
    int n;
    float lambda;
    int max_iter;
    double tol;
    double *state, *relres;
};

__global__ void __launch_bounds__(TINY_THREADS, 1) k_tiny_cg(TinyArgs a) {
    extern __shared__ float sm[];
    __shared__ double red[33];
    const int m = a.m, q = a.q, n = a.n, tid = threadIdx.x;
    float *Ts = sm;                          // q x q
    float *Ds = Ts + (size_t)q * q;          // m x m
    float *S = Ds + (size_t)m * m;           // q x m  (S[t][h])
    float *p = S + (size_t)q * m;            // n
    float *r = p + n, *Ap = r + n;
    float *x = a.x;  // the iterate lives in global memory (one read-modify-write per iteration)
    for (int i = tid; i < q * q; i += TINY_THREADS) Ts[i] = a.T[(int64_t)(i / q) * a.ldT + i % q];
    for (int i = tid; i < m * m; i += TINY_THREADS) Ds[i] = a.D[(int64_t)(i / m) * a.ldD + i % m];
    double yy = 0.0;
    for (int i = tid; i < n; i += TINY_THREADS) {
        const float v = a.y[i];
        p[i] = v;
        r[i] = v;
        x[i] = 0.f;  // each thread owns the same i in every loop below: no cross-thread hazard
        yy += (double)v * (double)v;
    }
    double rho = tiny_sum(yy, red);  // also the barrier after the smem fills
    const double ynorm = sqrt(rho);
    if (tid == 0 && a.relres) a.relres[0] = ynorm > 0.0 ? 1.0 : 0.0;
    int it = 0, brk = 0;
    double alpha = 0.0, beta = 0.0, pap = 0.0;
    bool done = !(rho > 0.0);
    while (!done && it < a.max_iter) {
        // ---- stage 1: S[t][h], t fastest across threads (conflict-free Ts reads)
        for (int cell = tid; cell < q * m; cell += TINY_THREADS) {
            const int t = cell % q, h = cell / q;
            float acc = 0.f;
            for (int64_t k = a.row_ptr[h]; k < a.row_ptr[h + 1]; k++)
                acc = fmaf(a.sign[k] * p[a.src[k]], Ts[(int64_t)a.col[k] * q + t], acc);
            S[(int64_t)t * m + h] = acc;
        }
        __syncthreads();
        // ---- stage 2 + ridge term, partial p.Ap
        double pa = 0.0;
        for (int64_t k = tid; k < a.ns; k += TINY_THREADS) {
            const float *drow = Ds + (int64_t)a.sr[k] * m, *srow = S + (int64_t)a.sc[k] * m;
            float acc = 0.f;
            for (int h = 0; h < m; h++) acc = fmaf(drow[h], srow[h], acc);
            const int d = a.sdst[k];
            const float v = fmaf(a.lambda, p[d], acc);
            Ap[d] = v;
            pa += (double)p[d] * (double)v;
        }
        pap = tiny_sum(pa, red);
        if (!(pap > 0.0)) {
            brk = 1;
            break;
        }
        alpha = rho / pap;
        const float af = (float)alpha;
        double rr = 0.0;
        for (int i = tid; i < n; i += TINY_THREADS) {
            x[i] = fmaf(af, p[i], x[i]);
            const float ri = fmaf(-af, Ap[i], r[i]);
            r[i] = ri;
            rr += (double)ri * (double)ri;
        }
        const double rho1 = tiny_sum(rr, red);
        it++;
        const double rel = sqrt(rho1) / ynorm;
        if (tid == 0 && a.relres) a.relres[it] = rel;
        done = (a.tol > 0.0 && rel <= a.tol) || rho1 == 0.0 || rel <= 8.673617379884035e-19;  // S32 floor
        beta = rho1 / rho;
        rho = rho1;
        const float bf = (float)beta;
        for (int i = tid; i < n; i += TINY_THREADS) p[i] = fmaf(bf, p[i], r[i]);
        __syncthreads();
    }
    if (tid == 0) {
        double *st = a.state;
        st[TS_RHO] = rho;
        st[TS_ALPHA] = alpha;
        st[TS_BETA] = beta;
        st[TS_YNORM] = ynorm;
        st[TS_PAP] = pap;
        st[TS_DONE] = done ? 1.0 : 0.0;
        st[TS_BREAK] = brk;
        st[TS_ITERS] = it;
        st[TS_TOL] = a.tol;
    }
}

// shared memory the single-CTA solve needs, or 0 if the problem does not qualify
size_t tiny_smem(int64_t m, int64_t q, int64_t n) {
    const size_t floats = (size_t)(q * q + m * m + q * m + 3 * n);
    const size_t bytes = floats * sizeof(float);
    return bytes <= 200 * 1024 ? bytes : 0;
}

void tiny_cg(gvt_ctx *c, const Factor &D, const Factor &T, const EntryPlan &e, const SamplePlan &sp, int64_t m,
             int64_t q, const float *y, float *x, int64_t n, double lambda, int max_iter, double tol, double *state) {
    const size_t smem = tiny_smem(m, q, n);
    GVT_REQUIRE(smem > 0 && n < INT32_MAX, GVT_E_STATE, "problem too large for the single-CTA solver");
    static size_t attr[GVT_MAX_DEVICES] = {};  // per device ordinal
    size_t &attr_dev = attr[c->device < GVT_MAX_DEVICES ? c->device : 0];
    if (smem > 48 * 1024 && smem > attr_dev) {
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_tiny_cg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_dev = smem;
    }
    TinyArgs a;
    a.T = T.p;
    a.ldT = T.ld;
    a.D = D.p;
    a.ldD = D.ld;
    a.m = (int)m;
    a.q = (int)q;
    a.row_ptr = e.row_ptr;
    a.col = e.col;
    a.src = e.src;
    a.sign = e.sign;
    a.ns = sp.ns;
    a.sr = sp.r;
    a.sc = sp.c;
    a.sdst = sp.dst;
    a.y = y;
    a.x = x;
    a.n = (int)n;
    a.lambda = (float)lambda;
    a.max_iter = max_iter;
    a.tol = tol;
    a.state = state;
    a.relres = state + TS_N;
    GVT_LAUNCH(c, K_TINY, k_tiny_cg, 1, TINY_THREADS, smem, a);
}

}  // namespace gvt
