// small.cu -- the whole CG fit of a small Kronecker problem in ONE persistent multi-CTA launch.
//
// Between the single-CTA solver (tiny.cu: everything in one SM's shared memory) and the
// graph-replayed multi-kernel engine (~8 launches per iteration, each with its own fixed cost)
// lie problems like C2 (the complete 68 x 442 drug-target grid: 1.5e7 FMAs per iteration,
// SURVEY.md 8(d) "latency-bound, target the CUDA-graph floor").  Here one cooperative launch of
// co-resident CTAs runs every iteration of Hestenes-Stiefel CG (
// readings S12-S14, S32) with grid barriers between the phases, all operands L2-resident:
//   A  X[h][col] = sum_{entries of cell (h, col)} sign p_k[src]    (the pair matrix of Theorem 1,
//                  p_k = r_k + beta p_{k-1} formed on the fly)
//   B  S[t][h]   = sum_col T[t][col] X[h][col]                     (stage 1, dense SIMT GEMM tiles)
//   C  Ap[dst]   = sum_h D[r][h] S[c][h] + lambda p_k[dst]; p.Ap   (stage 2 + ridge term)
//   D  alpha = rho / p.Ap; x += alpha p; r -= alpha Ap; r.r        (then beta, the stopping test)
// (variant 1; T symmetric, R1.)  Stage 1 runs on shared-memory tiles (the T strip
// and X rows of a 32 x 8 block of S), stage 2 on shared-memory copies of S and D, so the inner loops
// are LDS + FMA; every array written inside the launch is read with ld.global.cg (L2, never a stale
// L1 line of an earlier phase).  Dot products are fp64: one partial per CTA
// (fixed tree), every CTA reduces the partials in the same order, so all CTAs take the same
// scalar decisions and the result is bit-identical run to run (reading S26).  The state and
// residual history use the CG layout of cg.cu.
#include <stdio.h>

#include "vecops.cuh"

namespace gvt {

enum { SS_RHO = 0, SS_ALPHA, SS_BETA, SS_YNORM, SS_PAP, SS_DONE, SS_BREAK, SS_ITERS, SS_TOL, SS_N };
constexpr int SMALL_THREADS = 256;
constexpr int TILE_T = 32, TILE_H = SMALL_THREADS / 32;  // stage-1 tile: 32 rows of S x 8 columns

struct SmallArgs {
    const float *T;  // stage-1 factor, q x q, symmetric (row col holds T[col][0..q))
    int64_t ldT;
    const float *D;  // stage-2 factor, m x m
    int64_t ldD;
    int m, q;        // rows of X / columns of S (drugs), rows of S (targets)
    const int64_t *row_ptr;
    const int32_t *row, *col, *src;
    const float *sign;
    int64_t nnz;
    int64_t ns;
    const int32_t *sr, *sc, *sdst;
    const float *y;
    float *x;
    int n;
    float *S;        // q x ldS
    int64_t ldS;
    float *X;        // m x ldX, zero outside the cells of the sample (zeroed before the launch)
    int64_t ldX;
    float *p, *r, *Ap;
    double *part;    // [2][gridDim.x]
    unsigned long long *prof;  // optional phase timestamps (GVT_SMALL_PROF): [8 iterations][10]
    unsigned *bar;   // [2] arrivals, generation (zeroed before the launch)
    float lambda;
    int max_iter;
    double tol;
    double *state, *relres;
};

__device__ __forceinline__ float warp_sum_f(float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// grid-wide barrier of the co-resident CTAs (cooperative launch): arrival counter + generation; the
// waiting CTAs poll the generation with acquire loads and a short sleep (less traffic on the line the
// last arrival must update)
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned &gen) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = gen;
        __threadfence();
        if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
            atomicExch(&bar[0], 0u);
            __threadfence();
            atomicAdd(&bar[1], 1u);
        } else {
            unsigned v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
                if (v != g) break;
                __nanosleep(20);
            }
        }
    }
    gen++;
    __syncthreads();
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(SMALL_THREADS) k_small_cg(SmallArgs a) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t gtid = (int64_t)blockIdx.x * SMALL_THREADS + tid, gthreads = (int64_t)gridDim.x * SMALL_THREADS;
    const int64_t gwarp = gtid >> 5, gwarps = gthreads >> 5;
    const int n = a.n, m = a.m, q = a.q;
    double *part1 = a.part, *part2 = a.part + gridDim.x;
    unsigned gen = 0;
    // ---- init: x = 0, r = p = y, rho = y.y
    double yy = 0.0;
    for (int64_t i = gtid; i < n; i += gthreads) {
        const float v = a.y[i];
        a.x[i] = 0.f;
        a.r[i] = v;
        a.p[i] = v;
        yy += (double)v * (double)v;
    }
    yy = block_sum(yy);
    if (tid == 0) part1[blockIdx.x] = yy;
    grid_sync(a.bar, gen);
    double rho = reduce_parts_cg(part1, gridDim.x);
    __shared__ double bcast;
    if (tid == 0) bcast = rho;
    __syncthreads();
    rho = bcast;
    const double ynorm = sqrt(rho);
    if (gtid == 0 && a.relres) a.relres[0] = ynorm > 0.0 ? 1.0 : 0.0;
    int it = 0, brk = 0;
    double alpha = 0.0, beta = 0.0, pap = 0.0;
    bool done = !(rho > 0.0);
    const int ntt = (q + TILE_T - 1) / TILE_T, nth = (m + TILE_H - 1) / TILE_H, ntiles = ntt * nth;
    // shared memory: [T strip q x 32 | D m x ldsm | work: X rows 8 x q, or S q x ldsm]; the T strip of
    // this CTA's tile and D stay resident for the whole fit when every CTA has at most one tile
    extern __shared__ float sm[];
    const int ldsm = m | 1;  // odd stride of the shared-memory S and D rows (conflict-free sample rows)
    float *Tsm = sm, *Dsm = sm + (size_t)q * TILE_T, *work = Dsm + (size_t)m * ldsm;
    const bool resident = ntiles <= (int)gridDim.x;
    auto load_strip = [&](int t0) {
        for (int i = tid; i < q * TILE_T; i += SMALL_THREADS) {
            const int k = i / TILE_T, tt = i % TILE_T;
            Tsm[i] = (t0 + tt < q) ? __ldg(a.T + (int64_t)k * a.ldT + t0 + tt) : 0.f;
        }
    };
    if (resident && (int)blockIdx.x < ntiles) load_strip(((int)blockIdx.x % ntt) * TILE_T);
    for (int i = tid; i < m * m; i += SMALL_THREADS) Dsm[(i / m) * ldsm + i % m] = __ldg(a.D + (int64_t)(i / m) * a.ldD + i % m);
    __syncthreads();
#define SMALL_MARK(j) \
    if (a.prof && blockIdx.x == 0 && tid == 0 && it < 8) a.prof[it * 10 + (j)] = gtimer();
    while (!done && it < a.max_iter) {
        SMALL_MARK(0)
        const float bf = (float)beta;
        const bool first = it == 0;  // p_1 = r_0 = y is already in p
        // ---- A: the pair matrix of p_k, one entry per thread (runs of duplicate cells summed by their
        //      head entry in entry order; p_k = r_k + beta p_{k-1} formed on the fly)
        for (int64_t k = gtid; k < a.nnz; k += gthreads) {
            const int32_t h = a.row[k], cc = a.col[k];
            const bool head = k == 0 || a.row[k - 1] != h || a.col[k - 1] != cc;
            if (!head) continue;
            float v = 0.f;
            for (int64_t j = k; j < a.nnz && a.row[j] == h && a.col[j] == cc; j++) {
                const int32_t sj = a.src[j];
                const float pk = first ? __ldcg(a.p + sj) : fmaf(bf, __ldcg(a.p + sj), __ldcg(a.r + sj));
                v = fmaf(a.sign[j], pk, v);
            }
            a.X[(int64_t)h * a.ldX + cc] = v;
        }
        SMALL_MARK(1)
        grid_sync(a.bar, gen);
        SMALL_MARK(2)
        // ---- B: S[t][h] = sum_col T[col][t] X[h][col]; tile = 32 consecutive t (lanes) x 8 h (warps), the
        //      T strip resident in shared memory, the tile's 8 X rows staged by coalesced loads
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int t0 = (tile % ntt) * TILE_T, h0 = (tile / ntt) * TILE_H;
            if (!resident) load_strip(t0);
            float *Xs = work;
            for (int i = tid; i < TILE_H * q; i += SMALL_THREADS) {
                const int hh = i / q, k = i % q;
                Xs[i] = (h0 + hh < m) ? __ldcg(a.X + (int64_t)(h0 + hh) * a.ldX + k) : 0.f;
            }
            __syncthreads();
            const float *xr = Xs + (size_t)warp * q;
            float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
            int k = 0;
            for (; k + 3 < q; k += 4) {  // four independent chains
                acc0 = fmaf(Tsm[k * TILE_T + lane], xr[k], acc0);
                acc1 = fmaf(Tsm[(k + 1) * TILE_T + lane], xr[k + 1], acc1);
                acc2 = fmaf(Tsm[(k + 2) * TILE_T + lane], xr[k + 2], acc2);
                acc3 = fmaf(Tsm[(k + 3) * TILE_T + lane], xr[k + 3], acc3);
            }
            for (; k < q; k++) acc0 = fmaf(Tsm[k * TILE_T + lane], xr[k], acc0);
            const int t = t0 + lane, h = h0 + warp;
            if (t < q && h < m) a.S[(int64_t)t * a.ldS + h] = (acc0 + acc1) + (acc2 + acc3);
            __syncthreads();
        }
        SMALL_MARK(3)
        grid_sync(a.bar, gen);
        SMALL_MARK(4)
        // ---- C: stage 2 + ridge term, thread per sample on shared-memory copies of S (q x m) and D (m x m)
        //      (odd row strides: the rows of a warp's samples fall in different banks); the owner of dst
        //      stores p_k
        float *Ss = work, *Ds = Dsm;
        for (int i = tid; i < q * m; i += SMALL_THREADS) Ss[(i / m) * ldsm + i % m] = __ldcg(a.S + (int64_t)(i / m) * a.ldS + i % m);
        __syncthreads();
        SMALL_MARK(5)
        double pa = 0.0;
        for (int64_t k = gtid; k < a.ns; k += gthreads) {
            const float *drow = Ds + (int64_t)a.sr[k] * ldsm, *srow = Ss + (int64_t)a.sc[k] * ldsm;
            float acc0 = 0.f, acc1 = 0.f;
            int h = 0;
            for (; h + 1 < m; h += 2) {
                acc0 = fmaf(drow[h], srow[h], acc0);
                acc1 = fmaf(drow[h + 1], srow[h + 1], acc1);
            }
            if (h < m) acc0 = fmaf(drow[h], srow[h], acc0);
            const int d = a.sdst[k];
            const float pk = first ? __ldcg(a.p + d) : fmaf(bf, __ldcg(a.p + d), __ldcg(a.r + d));
            const float v = fmaf(a.lambda, pk, acc0 + acc1);
            a.Ap[d] = v;
            a.p[d] = pk;
            pa += (double)pk * (double)v;
        }
        pa = block_sum(pa);
        if (tid == 0) part1[blockIdx.x] = pa;
        SMALL_MARK(6)
        grid_sync(a.bar, gen);
        SMALL_MARK(7)
        pap = reduce_parts_cg(part1, gridDim.x);
        if (tid == 0) bcast = pap;
        __syncthreads();
        pap = bcast;
        if (!(pap > 0.0)) {
            brk = 1;
            break;
        }
        // ---- D: x += alpha p; r -= alpha Ap; r.r
        alpha = rho / pap;
        const float af = (float)alpha;
        double rr = 0.0;
        for (int64_t i = gtid; i < n; i += gthreads) {
            a.x[i] = fmaf(af, __ldcg(a.p + i), a.x[i]);
            const float ri = fmaf(-af, __ldcg(a.Ap + i), __ldcg(a.r + i));
            a.r[i] = ri;
            rr += (double)ri * (double)ri;
        }
        rr = block_sum(rr);
        if (tid == 0) part2[blockIdx.x] = rr;
        SMALL_MARK(8)
        grid_sync(a.bar, gen);
        SMALL_MARK(9)
        double rho1 = reduce_parts_cg(part2, gridDim.x);
        if (tid == 0) bcast = rho1;
        __syncthreads();
        rho1 = bcast;
        it++;
        const double rel = sqrt(rho1) / ynorm;
        if (gtid == 0 && a.relres) a.relres[it] = rel;
        done = (a.tol > 0.0 && rel <= a.tol) || rho1 == 0.0 || rel <= 8.673617379884035e-19;  // S32 floor
        beta = rho1 / rho;
        rho = rho1;
    }
    if (gtid == 0) {
        double *st = a.state;
        st[SS_RHO] = rho;
        st[SS_ALPHA] = alpha;
        st[SS_BETA] = beta;
        st[SS_YNORM] = ynorm;
        st[SS_PAP] = pap;
        st[SS_DONE] = done ? 1.0 : 0.0;
        st[SS_BREAK] = brk;
        st[SS_ITERS] = it;
        st[SS_TOL] = a.tol;
    }
}

// shared memory: T strip (q x 32) + D (m x ld) + the larger work area (X rows 8 x q, or S q x ld)
static size_t small_smem(int64_t m, int64_t q) {
    const int64_t ld = m | 1;
    const int64_t wk = TILE_H * q > q * ld ? TILE_H * q : q * ld;
    return sizeof(float) * (size_t)(q * TILE_T + m * ld + wk);
}

// dense stage-1 FMAs per iteration (m x q x q) at most 6.4e7, and S, D fit one CTA's shared memory
bool small_eligible(int64_t m, int64_t q, int64_t n) {
    return m > 0 && q > 0 && n > 0 && n < INT32_MAX && (double)m * (double)q * (double)q <= 6.4e7 &&
           small_smem(m, q) <= 200 * 1024;
}

void small_cg(gvt_ctx *c, const Factor &D, const Factor &T, const EntryPlan &e, const SamplePlan &sp, int64_t m,
              int64_t q, const float *y, float *x, int64_t n, double lambda, int max_iter, double tol, double *state) {
    GVT_REQUIRE(small_eligible(m, q, n), GVT_E_STATE, "problem outside the persistent small solver's range");
    const size_t smem = small_smem(m, q);
    static size_t attr[GVT_MAX_DEVICES] = {};
    size_t &attr_dev = attr[c->device < GVT_MAX_DEVICES ? c->device : 0];
    if (smem > 48 * 1024 && smem > attr_dev) {
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_small_cg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_dev = smem;
    }
    int per_sm = 0;
    GVT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_small_cg, SMALL_THREADS, smem));
    GVT_REQUIRE(per_sm >= 1, GVT_E_CUDA, "persistent small solver: no co-resident CTA");
    // one CTA per SM (every phase is a grid-stride loop; C2 has 126 stage-1 tiles, each CTA keeps its
    // tile's T strip resident); GVT_SMALL_GRID overrides the CTA count (experiments)
    static const int env_grid = [] {
        const char *e = getenv("GVT_SMALL_GRID");
        return e ? atoi(e) : 0;
    }();
    int grid = (int)std::min<int64_t>((int64_t)c->sm_count * std::min(per_sm, 1), 1 << 16);
    if (env_grid > 0) grid = std::min(grid, env_grid);
    SmallArgs a;
    a.T = T.p;
    a.ldT = T.ld;
    a.D = D.p;
    a.ldD = D.ld;
    a.m = (int)m;
    a.q = (int)q;
    a.row_ptr = e.row_ptr;
    a.row = e.row;
    a.col = e.col;
    a.src = e.src;
    a.sign = e.sign;
    a.nnz = e.nnz;
    a.ns = sp.ns;
    a.sr = sp.r;
    a.sc = sp.c;
    a.sdst = sp.dst;
    a.y = y;
    a.x = x;
    a.n = (int)n;
    a.ldX = round_up(q, 4);
    a.X = wsT<float>(c, "small.X", (size_t)m * a.ldX);
    a.ldS = round_up(m, 4);
    a.S = wsT<float>(c, "small.S", (size_t)q * a.ldS);
    a.p = wsT<float>(c, "small.p", (size_t)n);
    a.r = wsT<float>(c, "small.r", (size_t)n);
    a.Ap = wsT<float>(c, "small.Ap", (size_t)n);
    a.part = wsT<double>(c, "small.part", (size_t)2 * grid);
    a.bar = wsT<unsigned>(c, "small.bar", 2);
    a.lambda = (float)lambda;
    a.max_iter = max_iter;
    a.tol = tol;
    a.state = state;
    a.relres = state + SS_N;
    GVT_CUDA_TRY(cudaMemsetAsync(a.X, 0, sizeof(float) * (size_t)m * a.ldX, c->stream));
    GVT_CUDA_TRY(cudaMemsetAsync(a.bar, 0, 2 * sizeof(unsigned), c->stream));
    static const bool prof = getenv("GVT_SMALL_PROF") != nullptr;
    a.prof = prof ? wsT<unsigned long long>(c, "small.prof", 80) : nullptr;
    if (prof) GVT_CUDA_TRY(cudaMemsetAsync(a.prof, 0, 80 * sizeof(unsigned long long), c->stream));
    void *args[] = {&a};
    cudaEvent_t ev;
    launch_begin(c, K_TINY, &ev);
    GVT_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_small_cg, dim3(grid), dim3(SMALL_THREADS), args, smem,
                                             c->stream));
    launch_end(c, K_TINY, ev);
    if (prof) {  // phase durations (us) of iterations 1..7 of CTA 0, to stderr (diagnosis only)
        unsigned long long h[80];
        GVT_CUDA_TRY(cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
        const char *nm[9] = {"A", "bar1", "B", "bar2", "Ccopy", "C", "bar3", "D", "bar4"};
        for (int it = 1; it < 8 && it < max_iter; it++) {
            fprintf(stderr, "small_cg it %d:", it);
            for (int j = 0; j < 9; j++) fprintf(stderr, " %s %.2f", nm[j], (h[it * 10 + j + 1] - h[it * 10 + j]) * 1e-3);
            fprintf(stderr, "\n");
        }
    }
}

}  // namespace gvt
