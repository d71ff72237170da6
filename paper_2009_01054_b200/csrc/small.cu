// small.cu -- the whole CG fit of a small Kronecker problem in ONE persistent multi-CTA launch.
//
// Between the single-CTA solver (tiny.cu: everything in one SM's shared memory) and the
// graph-replayed multi-kernel engine (~8 launches per iteration, each with its own fixed cost)
// lie problems like C2 (the complete 68 x 442 drug-target grid: 1.5e7 FMAs per iteration,
// SURVEY.md 8(d) "latency-bound, target the CUDA-graph floor").  Here one cooperative launch of
// co-resident CTAs runs every iteration of Hestenes-Stiefel CG (
// readings S12-S14, S32) with grid barriers between the phases, all operands L2-resident:
//   AB X[h][col] = sum_{entries of cell (h, col)} sign p_k[src]    (the pair matrix of Theorem 1,
//                  p_k = r_k + beta p_{k-1} formed on the fly, per tile in shared memory)
//      S[t][h]   = sum_col T[t][col] X[h][col]                     (stage 1, dense SIMT GEMM tiles)
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

#include "gridsync.cuh"
#include "vecops.cuh"

namespace gvt {

enum { SS_RHO = 0, SS_ALPHA, SS_BETA, SS_YNORM, SS_PAP, SS_DONE, SS_BREAK, SS_ITERS, SS_TOL, SS_N };
constexpr int SMALL_THREADS = 256;
constexpr int TILE_T = 32, TILE_H = SMALL_THREADS / 32;  // stage-1 tile: 32 rows of S x 8 columns
constexpr uint32_t CELL_DUP = 1u << 31, CELL_HEAD = 1u << 30, CELL_MASK = CELL_HEAD - 1u;

// per entry (sorted by (h, col)): its cell in the 8 X rows of its tile, flagged when the cell has several
// entries (duplicate pairs) and, for those, when the entry heads the run
__global__ void k_small_cells(const int32_t *__restrict__ row, const int32_t *__restrict__ col, int64_t nnz,
                              int64_t ldX, uint32_t *__restrict__ cell) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t h = row[k], cc = col[k];
        const bool same_prev = k > 0 && row[k - 1] == h && col[k - 1] == cc;
        const bool same_next = k + 1 < nnz && row[k + 1] == h && col[k + 1] == cc;
        uint32_t code = (uint32_t)((int64_t)(h % TILE_H) * ldX + cc);
        if (same_prev || same_next) code |= CELL_DUP;
        if (!same_prev && same_next) code |= CELL_HEAD;
        cell[k] = code;
    }
}

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
    const uint32_t *cell;  // per entry: cell (h % 8) * ldX + col of the tile's X rows, | CELL_DUP / CELL_HEAD
    int64_t ldX;            // X row stride in shared memory (round_up(q, 4))
    float *p, *r, *Ap;
    double *part;    // [2][gridDim.x]
    unsigned long long *prof;  // optional phase timestamps (GVT_SMALL_PROF): [8 iterations][10]
    unsigned *bar;   // barrier words (zeroed before the launch)
    int bar_mode;
    float lambda;
    int max_iter;
    double tol;
    double *state, *relres;
};

__device__ __forceinline__ float warp_sum_f(float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
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
    grid_sync(a.bar, gen, a.bar_mode);
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
    // shared memory: [T strip, transposed: 32 x tq | D m x ldsm | work: X rows 8 x ldX, or S rows x ldsm];
    // the T strip of this CTA's tile and D stay resident for the whole fit when every CTA has at most
    // one tile.  tq = round_up(q, 32) + 4: the 16-byte loads of 8 consecutive lanes (32 rows) hit
    // distinct bank groups.
    extern __shared__ float sm[];
    const int ldsm = m | 1;  // odd stride of the shared-memory S and D rows (conflict-free sample rows)
    const int tq = ((q + 31) & ~31) + 4, q4 = (int)(a.ldX / 4);
    float *Tt = sm, *Dsm = sm + (size_t)TILE_T * tq;
    float *work = sm + (((size_t)TILE_T * tq + (size_t)m * ldsm + 3) & ~(size_t)3);  // 16-byte aligned (float4)
    const bool resident = ntiles <= (int)gridDim.x;
    auto load_strip = [&](int t0) {  // Tt[tt][k] = T[t0 + tt][k] (= T[k][t0 + tt], T symmetric), zero padded
        const int tq4 = tq / 4, ldT4 = (int)(a.ldT / 4);
        for (int i = tid; i < TILE_T * tq4; i += SMALL_THREADS) {
            const int tt = i / tq4, k4 = i % tq4;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (t0 + tt < q && 4 * k4 < q) {
                v = __ldg(reinterpret_cast<const float4 *>(a.T) + (int64_t)(t0 + tt) * ldT4 + k4);
                if (4 * k4 + 1 >= q) v.y = 0.f;
                if (4 * k4 + 2 >= q) v.z = 0.f;
                if (4 * k4 + 3 >= q) v.w = 0.f;
            }
            reinterpret_cast<float4 *>(Tt)[i] = v;
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
        SMALL_MARK(1)
        SMALL_MARK(2)
        // ---- A + B per tile (32 consecutive t as lanes x 8 h as warps): the tile's 8 pair-matrix rows of p_k
        //      built in shared memory from their CSR entries (precomputed cell codes; a run of duplicate
        //      cells summed by its head in entry order; p_k = r_k + beta p_{k-1} formed on the fly), then
        //      S[t][h] = sum_col T[col][t] X[h][col] with 16-byte shared loads of the T strip row (lane)
        //      and the X row (warp, broadcast): four FMAs per two loads
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            const int t0 = (tile % ntt) * TILE_T, h0 = (tile / ntt) * TILE_H;
            const int h1 = h0 + TILE_H < m ? h0 + TILE_H : m;
            if (!resident) load_strip(t0);
            float *Xs = work;  // 8 rows of ldX floats
            for (int i = tid; i < TILE_H * q4; i += SMALL_THREADS)
                reinterpret_cast<float4 *>(Xs)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            __syncthreads();
            const int64_t kb = a.row_ptr[h0], ke = a.row_ptr[h1];
            constexpr int U = 8;  // entries in flight per thread: their loads are independent
            for (int64_t k0 = kb + tid; k0 < ke; k0 += U * SMALL_THREADS) {
                uint32_t cd[U];
                int32_t sx[U];
                float sg[U], pp[U], rr[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t k = k0 + (int64_t)u * SMALL_THREADS;
                    cd[u] = k < ke ? a.cell[k] : CELL_DUP;  // (past the range: a non-head, skipped)
                    sx[u] = k < ke ? a.src[k] : 0;
                    sg[u] = k < ke ? a.sign[k] : 0.f;
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    pp[u] = __ldcg(a.p + sx[u]);
                    rr[u] = first ? 0.f : __ldcg(a.r + sx[u]);
                }
#pragma unroll
                for (int u = 0; u < U; u++)
                    if (!(cd[u] & CELL_DUP)) Xs[cd[u]] = fmaf(sg[u], first ? pp[u] : fmaf(bf, pp[u], rr[u]), 0.f);
#pragma unroll
                for (int u = 0; u < U; u++) {
                const int64_t k = k0 + (int64_t)u * SMALL_THREADS;
                const uint32_t code = cd[u];
                if (k >= ke || !(code & CELL_DUP)) continue;
                const float pk = first ? pp[u] : fmaf(bf, pp[u], rr[u]);
                if (code & CELL_HEAD) {
                    const uint32_t cellid = code & CELL_MASK;
                    float v = fmaf(a.sign[k], pk, 0.f);
                    for (int64_t jx = k + 1; jx < ke && (a.cell[jx] & CELL_MASK) == cellid; jx++) {
                        const int32_t sj = a.src[jx];
                        const float px = first ? __ldcg(a.p + sj) : fmaf(bf, __ldcg(a.p + sj), __ldcg(a.r + sj));
                        v = fmaf(a.sign[jx], px, v);
                    }
                    Xs[cellid] = v;
                }
                }
            }
            __syncthreads();
            const float4 *tr = reinterpret_cast<const float4 *>(Tt + (size_t)lane * tq);
            const float4 *xr = reinterpret_cast<const float4 *>(Xs + (size_t)warp * a.ldX);
            float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
#pragma unroll 4
            for (int k4 = 0; k4 < q4; k4++) {
                const float4 tv = tr[k4], xv = xr[k4];
                acc0 = fmaf(tv.x, xv.x, acc0);
                acc1 = fmaf(tv.y, xv.y, acc1);
                acc2 = fmaf(tv.z, xv.z, acc2);
                acc3 = fmaf(tv.w, xv.w, acc3);
            }
            const int t = t0 + lane, h = h0 + warp;
            if (t < q && h < m) a.S[(int64_t)t * a.ldS + h] = (acc0 + acc1) + (acc2 + acc3);
            __syncthreads();
        }
        SMALL_MARK(3)
        grid_sync(a.bar, gen, a.bar_mode);
        SMALL_MARK(4)
        // ---- C: stage 2 + ridge term.  The samples are sorted by their S row c (small_cg) and split
        //      into equal contiguous ranges, one per CTA, so a CTA copies only the few S rows its range
        //      uses into shared memory (odd row stride; D is resident); thread per sample, the owner of
        //      dst stores p_k
        double pa = 0.0;
        {
            const int64_t k0 = a.ns * (int64_t)blockIdx.x / gridDim.x, k1 = a.ns * ((int64_t)blockIdx.x + 1) / gridDim.x;
            const int c_lo = k1 > k0 ? a.sc[k0] : 0, c_hi = k1 > k0 ? a.sc[k1 - 1] : -1;
            float *Ss = work;
            const int s4 = (int)(a.ldS / 4);
            for (int i = tid; i < (c_hi - c_lo + 1) * s4; i += SMALL_THREADS) {
                const int row = i / s4, j4 = i % s4;
                const float4 v = __ldcg(reinterpret_cast<const float4 *>(a.S + (int64_t)(c_lo + row) * a.ldS) + j4);
                float *dst = Ss + (size_t)row * ldsm + 4 * j4;
                if (4 * j4 < m) dst[0] = v.x;
                if (4 * j4 + 1 < m) dst[1] = v.y;
                if (4 * j4 + 2 < m) dst[2] = v.z;
                if (4 * j4 + 3 < m) dst[3] = v.w;
            }
            __syncthreads();
            SMALL_MARK(5)
            for (int64_t k = k0 + tid; k < k1; k += SMALL_THREADS) {
            const float *drow = Dsm + (int64_t)a.sr[k] * ldsm, *srow = Ss + (int64_t)(a.sc[k] - c_lo) * ldsm;
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
            a.Ap[d] = v;  // (p_k itself is stored by its owner in phase D: contiguous, not scattered by dst)
            pa += (double)pk * (double)v;
            }
        }
        pa = block_sum(pa);
        if (tid == 0) part1[blockIdx.x] = pa;
        SMALL_MARK(6)
        grid_sync(a.bar, gen, a.bar_mode);
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
            // p_k = r_{k-1} + beta p_{k-1}, the same fmaf as phases AB and C, from the values before this update
            const float r0 = __ldcg(a.r + i), p0 = __ldcg(a.p + i);
            const float pk = first ? p0 : fmaf(bf, p0, r0);
            a.p[i] = pk;
            a.x[i] = fmaf(af, pk, a.x[i]);
            const float ri = fmaf(-af, __ldcg(a.Ap + i), r0);
            a.r[i] = ri;
            rr += (double)ri * (double)ri;
        }
        rr = block_sum(rr);
        if (tid == 0) part2[blockIdx.x] = rr;
        SMALL_MARK(8)
        grid_sync(a.bar, gen, a.bar_mode);
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

// the direction the next iteration would use, p_{k+1} = r_k + beta_k p_k (gvt_solver_direction; the
// solver forms it on the fly, so it is materialised once after the launch, in the same fmaf form)
__global__ void k_small_direction(const float *__restrict__ p, const float *__restrict__ r,
                                  const double *__restrict__ state, int64_t n, float *__restrict__ out) {
    const float bf = (float)state[SS_BETA];
    const bool fresh = state[SS_ITERS] == 0.0;  // no iteration ran: p_1 = y, still in p
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = fresh ? p[i] : fmaf(bf, p[i], r[i]);
}

// shared memory: T strip (32 x tq) + D (m x ld) + the larger work area (X rows 8 x ldX, or S q x ld)
static size_t small_smem(int64_t m, int64_t q) {
    const int64_t ld = m | 1, tq = round_up(q, 32) + 4;
    const int64_t xq = TILE_H * round_up(q, 4), wk = xq > q * ld ? xq : q * ld;
    return sizeof(float) * (size_t)(round_up(TILE_T * tq + m * ld, 4) + wk);
}

// dense stage-1 FMAs per iteration (m x q x q) at most 6.4e7, and S, D fit one CTA's shared memory
bool small_eligible(int64_t m, int64_t q, int64_t n) {
    return m > 0 && q > 0 && n > 0 && n < INT32_MAX && (double)m * (double)q * (double)q <= 6.4e7 &&
           small_smem(m, q) <= 200 * 1024;
}

void small_cg(gvt_ctx *c, const Factor &D, const Factor &T, const EntryPlan &e, const SamplePlan &sp, int64_t m,
              int64_t q, const float *y, float *x, int64_t n, double lambda, int max_iter, double tol, double *state,
              bool keep_dir) {
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
    int grid = (int)std::min<int64_t>((int64_t)c->sm_count * std::min(per_sm, 1), BAR_GROUP * 64);
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
    {  // samples sorted by (c, r): contiguous per-CTA ranges touch few S rows (phase C)
        const int64_t ns = sp.ns;
        int32_t *perm = wsT<int32_t>(c, "small.perm", (size_t)ns);
        int32_t *sr = wsT<int32_t>(c, "small.sr", (size_t)ns), *sc = wsT<int32_t>(c, "small.sc", (size_t)ns),
                *sd = wsT<int32_t>(c, "small.sd", (size_t)ns);
        sort_pairs(c, sp.c, sp.r, ns, q, m, perm);
        gather_i32(c, sp.r, perm, ns, sr);
        gather_i32(c, sp.c, perm, ns, sc);
        gather_i32(c, sp.dst, perm, ns, sd);
        a.sr = sr;
        a.sc = sc;
        a.sdst = sd;
    }
    a.y = y;
    a.x = x;
    a.n = (int)n;
    a.ldX = round_up(q, 4);
    {
        uint32_t *cell = wsT<uint32_t>(c, "small.cell", (size_t)e.nnz);
        if (e.nnz) GVT_LAUNCH(c, K_PLAN_KEYS, k_small_cells, grid1d(e.nnz, 256, 8 * c->sm_count * 8), 256, 0, e.row,
                              e.col, e.nnz, a.ldX, cell);
        a.cell = cell;
    }
    a.ldS = round_up(m, 4);
    a.S = wsT<float>(c, "small.S", (size_t)q * a.ldS);
    a.p = wsT<float>(c, "small.p", (size_t)n);
    a.r = wsT<float>(c, "small.r", (size_t)n);
    a.Ap = wsT<float>(c, "small.Ap", (size_t)n);
    a.part = wsT<double>(c, "small.part", (size_t)2 * grid);
    a.bar = wsT<unsigned>(c, "small.bar", BAR_WORDS);
    static const int env_bar = [] {
        const char *e = getenv("GVT_SMALL_BAR");
        return e ? atoi(e) : 0;
    }();
    a.bar_mode = env_bar;
    a.lambda = (float)lambda;
    a.max_iter = max_iter;
    a.tol = tol;
    a.state = state;
    a.relres = state + SS_N;
    GVT_CUDA_TRY(cudaMemsetAsync(a.bar, 0, BAR_WORDS * sizeof(unsigned), c->stream));
    static const bool prof = getenv("GVT_SMALL_PROF") != nullptr;
    a.prof = prof ? wsT<unsigned long long>(c, "small.prof", 80) : nullptr;
    if (prof) GVT_CUDA_TRY(cudaMemsetAsync(a.prof, 0, 80 * sizeof(unsigned long long), c->stream));
    void *args[] = {&a};
    cudaEvent_t ev;
    launch_begin(c, K_TINY, &ev);
    GVT_CUDA_TRY(cudaLaunchCooperativeKernel((const void *)k_small_cg, dim3(grid), dim3(SMALL_THREADS), args, smem,
                                             c->stream));
    launch_end(c, K_TINY, ev);
    if (keep_dir) {
        float *dir = wsT<float>(c, "small.dir", (size_t)n);
        if (n) GVT_LAUNCH(c, K_CG_VEC, k_small_direction, grid1d(n, 256, 2 * c->sm_count), 256, 0, a.p, a.r, state,
                          n, dir);
        c->last_p = dir;
        c->last_n = n;
    }
    if (prof) {  // phase durations (us) of iterations 1..7 of CTA 0, to stderr (diagnosis only)
        unsigned long long h[80];
        GVT_CUDA_TRY(cudaMemcpyAsync(h, a.prof, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
        const char *nm[9] = {"-", "-", "AB", "bar2", "Ccopy", "C", "bar3", "D", "bar4"};
        for (int it = 1; it < 8 && it < max_iter; it++) {
            fprintf(stderr, "small_cg it %d:", it);
            for (int j = 0; j < 9; j++) fprintf(stderr, " %s %.2f", nm[j], (h[it * 10 + j + 1] - h[it * 10 + j]) * 1e-3);
            fprintf(stderr, "\n");
        }
    }
}

}  // namespace gvt
