// tail.cu -- the fused CG tail of the dense tensor-core engine (north-star kernel (4): "the fused
// Kronecker-term accumulation and the CG axpy/dot steps"), single GPU.
//
// Between the stage-2 sampled GEMM of iteration k and the stage-1 GEMM of iteration k + 1 the
// graph-replayed Hestenes-Stiefel CG iteration (readings S12-S14, S32)
// ran six short launches: the split-K part combine, k_cg_ap, k_cg_xr, k_cg_p, the S-scale memset and
// the pair-matrix build X(p_{k+1}) (Theorem 1's stage-1 operand, Corollary PAPER.md:634-653).  On
// C3-size problems (n = 2e5, X 2000 x 2048) each costs its launch, ramp and tail more than its
// bytes.  Here ONE persistent launch of co-resident CTAs runs them with the two grid barriers the
// two CG reductions need:
//   A  u_i = coef * sum_h part[h][inv_i]  (the split-K parts of output i, in part order)
//      Ap_i = u_i + lambda p_i; p.Ap partials                  (fixed partition, as k_cg_ap)
//   -- barrier; alpha = rho / p.Ap (every CTA reduces the partials in the same order; <= 0: breakdown)
//   B  x += alpha p; r -= alpha Ap; r.r partials               (the same partition, as k_cg_xr)
//   -- barrier; beta, the stopping test, the residual history  (every CTA, the same scalars)
//   C  p' = r + beta p into the other direction buffer         (as k_cg_p)
//      X(p') rows, fp16 hi/lo with power-of-two row scales, each entry's p' formed on the fly with
//      the same fmaf from r and p                              (as k_build_x16_warp, warp per row)
// The direction alternates between two buffers (p_k in buffer k & 1), so phase C reads p_{k-1}
// while it writes p_k.  Every phase runs the arithmetic of the kernel it replaces on the same
// partition (cgops.cuh, xbuild.cuh), so the iterates are bit-identical to the separate kernels'.
// Data written by other CTAs earlier in the launch is read through L2 (ld.global.cg).  CTA 0 writes
// the CG state; every CTA reads it as it was at launch.
// Users: the Kronecker / symmetric / anti-symmetric group (one part set, one operand X) and the Cartesian
// form's two sampled GEMMs (two part sets, the second accumulated; operands X^T and X).  A gather-combine
// mode (the cheap forms' final combine, p updated in place, no operand) exists as an A/B knob
// (GVT_CHEAP_TAIL=1, engine.cu): at n = 2e6 it measured slower than the separate kernels.
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <vector>

#include "gridsync.cuh"
#include "xbuild.cuh"

namespace gvt {

struct TailXDev {  // one pair-matrix operand to rebuild: rows [0, rows) from entries row_ptr[row_lo + r] ..
    const int64_t *row_ptr;
    const int32_t *col, *src;
    const float *sign;
    int64_t row_lo, rows, ld;
    __half *hi, *lo;
    float *sinv;
};

struct DenseTailArgs {
    // deferred split-K part sets (nullptr: that GEMM wrote u itself); inv[i] = sample slot of output i.
    // Set A is stored (u = coef sum), set B accumulated (u = fmaf(coef, sum, u)), as their combines would.
    const float *partA, *partB;
    int splitA, splitB;
    float coefA, coefB;
    int accA, accB;
    int64_t ns;
    const int32_t *inv;
    // CG vectors and state; the direction lives in pd[k & 1] after iteration k
    float *u, *x, *r;
    float *pd[2];
    int64_t n;
    int64_t nvb;  // virtual blocks of the fixed partition (vec_blocks(n) of the separate kernels)
    float lambda;
    double *st, *relres;
    double *part1, *part2;  // [RED_BLOCKS] each, unused slots zero
    TailXDev xb[2];
    int nx;
    // gather-combine mode (the cheap forms): u_i from the factor gathers, p updated in place (pd[0] == pd[1])
    int gmode, grs1, grs2, gacc;
    const int32_t *gf, *gs;
    const float *g1, *g2;
    float gc1, gc2;
    int64_t ldmax;
    unsigned *bar;
    unsigned long long *prof;  // GVT_TAIL_PROF: [0..7] CTA 0's phase stamps, [8 + b] CTA b's exit
};

__device__ __forceinline__ unsigned long long tail_timer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TAIL_MARK(j) \
    if (a.prof && blockIdx.x == 0 && tid == 0) a.prof[j] = tail_timer();

constexpr int TAIL_THREADS = RED_THREADS;  // block_sum's tree: the partials match the separate kernels'

__global__ void __launch_bounds__(TAIL_THREADS) k_dense_cg_tail(DenseTailArgs a) {
    extern __shared__ float rowbufs[];  // (TAIL_THREADS / 32) x ld floats
    __shared__ double bc;
    if (halted(a.st)) return;  // (the state as the previous launch left it: the same in every CTA)
    const int tid = threadIdx.x;
    const double rho = a.st[ST_RHO], ynorm = a.st[ST_YNORM], tol = a.st[ST_TOL], iters = a.st[ST_ITERS];
    const int par = (int)((int64_t)iters & 1);
    const float *p = a.pd[par];
    float *pn = a.pd[par ^ 1];
    TAIL_MARK(0);
    unsigned gen = 0;
    if (tid == 0) asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(gen) : "l"(a.bar) : "memory");
    // ---- A: u from the parts (as k_split_combine), then Ap = u + lambda p and p.Ap (as k_cg_ap); or (the cheap
    // forms) u from the factor gathers with Ap and p.Ap in one loop (as k_cg_combine_ap)
    for (int64_t vb = blockIdx.x; vb < a.nvb; vb += gridDim.x) {
        int64_t lo, hi;
        vblock_range(a.n, a.nvb, vb, lo, hi);
        if (a.gmode) {
            double acc = 0.0;
            for (int64_t i = lo + tid; i < hi; i += TAIL_THREADS) {
                float v = a.gc1 * a.g1[a.grs1 == 0 ? a.gf[i] : a.gs[i]];
                if (a.g2) v = fmaf(a.gc2, a.g2[a.grs2 == 0 ? a.gf[i] : a.gs[i]], v);
                const float ui = a.gacc ? __ldcg(a.u + i) + v : v;
                const float pi = __ldcg(p + i);
                const float av = fmaf(a.lambda, pi, ui);
                a.u[i] = av;
                acc += (double)pi * (double)av;
            }
            acc = block_sum(acc);
            if (tid == 0) a.part1[vb] = acc;
            continue;
        }
        if (a.partA || a.partB) {
            for (int64_t i = lo + tid; i < hi; i += TAIL_THREADS) {
                const int64_t k = a.inv[i];
                if (a.partA) {
                    float v = a.partA[k];
                    for (int h = 1; h < a.splitA; h++) v += a.partA[(int64_t)h * a.ns + k];
                    a.u[i] = a.accA ? fmaf(a.coefA, v, __ldcg(a.u + i)) : a.coefA * v;
                }
                if (a.partB) {
                    float v = a.partB[k];
                    for (int h = 1; h < a.splitB; h++) v += a.partB[(int64_t)h * a.ns + k];
                    a.u[i] = a.accB ? fmaf(a.coefB, v, __ldcg(a.u + i)) : a.coefB * v;
                }
            }
            __syncthreads();
        }
        const double acc = block_sum(cg_ap_range<true>(a.u, p, lo, hi, a.lambda));
        if (tid == 0) a.part1[vb] = acc;
    }
    grid_sync(a.bar, gen, 0);
    {
        const double v = reduce_parts_cg(a.part1, RED_BLOCKS);
        if (tid == 0) bc = v;
        __syncthreads();
    }
    const double pap = bc;
    TAIL_MARK(1);
    if (blockIdx.x == 0 && tid == 0) {  // (cg_alpha_scalar)
        a.st[ST_PAP] = pap;
        if (!(pap > 0.0)) a.st[ST_BREAK] = 1.0;
        else a.st[ST_ALPHA] = rho / pap;
    }
    if (!(pap > 0.0)) return;  // breakdown (every CTA sees the same pap)
    // ---- B: x += alpha p, r -= alpha Ap, r.r (as k_cg_xr)
    const float alpha = (float)(rho / pap);
    for (int64_t vb = blockIdx.x; vb < a.nvb; vb += gridDim.x) {
        int64_t lo, hi;
        vblock_range(a.n, a.nvb, vb, lo, hi);
        const double acc = block_sum(cg_xr_range<true>(a.x, a.r, p, a.u, lo, hi, alpha));
        if (tid == 0) a.part2[vb] = acc;
    }
    grid_sync(a.bar, gen, 0);
    {
        const double v = reduce_parts_cg(a.part2, RED_BLOCKS);
        if (tid == 0) bc = v;
        __syncthreads();
    }
    const double rho1 = bc;
    TAIL_MARK(2);
    const double it = iters + 1.0, rr = sqrt(rho1) / ynorm;
    const bool done = (tol > 0.0 && rr <= tol) || rho1 == 0.0 || rr <= RES_FLOOR;
    const double beta = rho1 / rho;
    if (blockIdx.x == 0 && tid == 0) {  // (cg_beta_scalar)
        a.st[ST_ITERS] = it;
        if (a.relres) a.relres[(int64_t)it] = rr;
        if (done) a.st[ST_DONE] = 1.0;
        a.st[ST_BETA] = beta;
        a.st[ST_RHO] = rho1;
    }
    if (done) return;  // (k_cg_p sees the halted state and leaves p; X is not needed again)
    // ---- C: p' = r + beta p (as k_cg_p) and X(p'), p' formed on the fly from the same r and p
    const int64_t gtid = (int64_t)blockIdx.x * TAIL_THREADS + tid, gthreads = (int64_t)gridDim.x * TAIL_THREADS;
    const float fb = (float)beta;
    if (aligned16(pn) && aligned16(p) && aligned16(a.r)) {
        const int64_t n4 = a.n >> 2;
        for (int64_t i = gtid; i < n4; i += gthreads) {
            const float4 pp = __ldcg(reinterpret_cast<const float4 *>(p) + i);
            const float4 rv = __ldcg(reinterpret_cast<const float4 *>(a.r) + i);
            reinterpret_cast<float4 *>(pn)[i] =
                make_float4(fmaf(fb, pp.x, rv.x), fmaf(fb, pp.y, rv.y), fmaf(fb, pp.z, rv.z), fmaf(fb, pp.w, rv.w));
        }
        for (int64_t i = (n4 << 2) + gtid; i < a.n; i += gthreads) pn[i] = fmaf(fb, __ldcg(p + i), __ldcg(a.r + i));
    } else {
        for (int64_t i = gtid; i < a.n; i += gthreads) pn[i] = fmaf(fb, __ldcg(p + i), __ldcg(a.r + i));
    }
    const int warp = tid >> 5, lane = tid & 31;
    float *rowbuf = rowbufs + (size_t)warp * a.ldmax;
    const int64_t nw = (int64_t)gridDim.x * (TAIL_THREADS / 32);
    const int64_t rows0 = a.nx > 0 ? a.xb[0].rows : 0, rows_all = rows0 + (a.nx > 1 ? a.xb[1].rows : 0);
    for (int64_t row = (int64_t)blockIdx.x * (TAIL_THREADS / 32) + warp; row < rows_all; row += nw) {
        const TailXDev &xb = a.xb[row < rows0 ? 0 : 1];
        x16_row_warp<true>(row < rows0 ? row : row - rows0, lane, rowbuf, xb.row_ptr, xb.col, xb.src, xb.sign, p,
                           xb.row_lo, xb.ld, xb.hi, xb.lo, xb.sinv, nullptr, a.r, fb);
    }
    if (a.prof) {
        __syncthreads();
        if (tid == 0) a.prof[8 + blockIdx.x] = tail_timer();
    }
}

static size_t tail_smem(int64_t ld) { return sizeof(float) * (size_t)(TAIL_THREADS / 32) * (size_t)ld; }

bool dense_tail_fits(int64_t ld) { return ld > 0 && tail_smem(ld) <= 96 * 1024; }

void dense_cg_tail(gvt_ctx *c, const SplitParts &pa, const SplitParts &pb, const int32_t *inv, float *u, float *x,
                   float *r, float *p0, float *p1, int64_t n, int64_t nvb, double lambda, double *state,
                   double *part1, double *part2, const TailX *xs, int nx, const GatherCombine *gcomb) {
    static bool attr_dev[GVT_MAX_DEVICES] = {};
    bool &attr_set = attr_dev[c->device < GVT_MAX_DEVICES ? c->device : 0];
    GVT_REQUIRE(nx >= (gcomb ? 0 : 1) && nx <= 2, GVT_E_STATE, "fused CG tail: one or two pair-matrix operands");
    GVT_REQUIRE(!gcomb || (p0 == p1 && nx == 0 && !pa.part && !pb.part), GVT_E_STATE,
                "fused CG tail: the gather combine updates p in place, without parts or operands");
    GVT_REQUIRE(!(pa.part || pb.part) || inv, GVT_E_STATE, "fused CG tail: split-K parts without the output -> slot map");
    DenseTailArgs a;
    memset(&a, 0, sizeof(a));
    a.ldmax = 0;
    for (int i = 0; i < nx; i++) {
        const EntryPlan &e = *xs[i].e;
        TailXDev &d = a.xb[i];
        d.row_ptr = e.row_ptr;
        d.col = e.col;
        d.src = e.src;
        d.sign = e.sign;
        d.row_lo = xs[i].row_lo;
        d.rows = xs[i].rows;
        d.ld = xs[i].op.ld;
        // (the operand's buffers are the workspace build_x16 writes: the tail writes them the same way)
        d.hi = const_cast<__half *>(static_cast<const __half *>(xs[i].op.hi));
        d.lo = const_cast<__half *>(static_cast<const __half *>(xs[i].op.lo));
        d.sinv = const_cast<float *>(xs[i].op.scale);
        a.ldmax = std::max(a.ldmax, d.ld);
    }
    a.nx = nx;
    if (gcomb) {
        a.gmode = 1;
        a.gf = gcomb->f;
        a.gs = gcomb->s;
        a.g1 = gcomb->g1;
        a.g2 = gcomb->g2;
        a.grs1 = gcomb->rs1;
        a.grs2 = gcomb->rs2;
        a.gc1 = gcomb->c1;
        a.gc2 = gcomb->c2;
        a.gacc = gcomb->accumulate;
    }
    const size_t smem = nx > 0 ? tail_smem(a.ldmax) : 0;
    GVT_REQUIRE(nx == 0 || dense_tail_fits(a.ldmax), GVT_E_STATE, "fused CG tail: X rows too long");
    if (!attr_set) {
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_dense_cg_tail, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024));
        attr_set = true;
    }
    // co-resident CTAs for this launch's shared memory (its X rows); latency-bound phases want as many as
    // fit: 296 vs 148 CTAs measured 91.6 vs 106 us per C3 iteration (profiles/r02_ab_dense_tail.txt)
    int per_sm = 0;
    GVT_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_dense_cg_tail, TAIL_THREADS, smem));
    GVT_REQUIRE(per_sm >= 1, GVT_E_STATE, "fused CG tail: no resident CTA");
    static const int env_per_sm = [] {  // A/B knob: GVT_TAIL_CTAS_PER_SM (cap; default 2: 3 measured no better)
        const char *e = getenv("GVT_TAIL_CTAS_PER_SM");
        return e ? atoi(e) : 2;
    }();
    const int grid = c->sm_count * std::max(1, std::min(per_sm, env_per_sm));
    a.partA = pa.part;
    a.splitA = pa.split;
    a.coefA = pa.coef;
    a.accA = pa.accumulate;
    a.partB = pb.part;
    a.splitB = pb.split;
    a.coefB = pb.coef;
    a.accB = pb.accumulate;
    a.ns = pa.part ? pa.ns : pb.ns;
    a.inv = inv;
    a.u = u;
    a.x = x;
    a.r = r;
    a.pd[0] = p0;
    a.pd[1] = p1;
    a.n = n;
    a.nvb = nvb;
    a.lambda = (float)lambda;
    a.st = state;
    a.relres = state + ST_N;
    a.part1 = part1;
    a.part2 = part2;
    a.bar = wsT<unsigned>(c, "tail.bar", BAR_WORDS);
    static const bool prof = getenv("GVT_TAIL_PROF") != nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    GVT_CUDA_TRY(cudaStreamIsCapturing(c->stream, &cs));
    a.prof = prof && cs == cudaStreamCaptureStatusNone ? wsT<unsigned long long>(c, "tail.prof", 8 + (size_t)grid)
                                                       : nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(TAIL_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c->stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaEvent_t ev;
    launch_begin(c, K_CG_VEC, &ev);
    GVT_CUDA_TRY(cudaLaunchKernelEx(&cfg, k_dense_cg_tail, a));
    launch_end(c, K_CG_VEC, ev);
    if (a.prof) {  // phase durations (us) of this launch, to stderr (diagnosis only; run with OPT_GRAPHS = 0)
        std::vector<unsigned long long> h(8 + (size_t)grid);
        GVT_CUDA_TRY(cudaMemcpyAsync(h.data(), a.prof, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost,
                                     c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
        unsigned long long end = 0;
        for (int b = 0; b < grid; b++) end = std::max(end, h[8 + b]);
        fprintf(stderr, "dense_cg_tail: A %.2f B %.2f C %.2f us (grid %d)\n", (h[1] - h[0]) * 1e-3,
                (h[2] - h[1]) * 1e-3, (end - h[2]) * 1e-3, grid);
    }
}

// after the loop: the direction of the last iteration into p itself (gvt_solver_direction reads p).
// After iteration k the direction is in pd[k & 1]; an iteration that stops (done) leaves p_{k-1}
// (k_cg_p skipped), a breakdown at iteration k + 1 leaves ITERS = k and p_k.
__global__ void k_tail_final_dir(float *__restrict__ p, const float *__restrict__ p_alt, int64_t n,
                                 const double *__restrict__ st) {
    const int64_t k = (int64_t)st[ST_ITERS];
    const bool done = st[ST_DONE] != 0.0 && st[ST_BREAK] == 0.0;
    const int64_t b = done ? (k > 0 ? (k - 1) & 1 : 0) : (k & 1);
    if (b == 0) return;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = p_alt[i];
}

void dense_tail_finish(gvt_ctx *c, float *p, const float *p_alt, int64_t n, const double *state) {
    if (n > 0) GVT_LAUNCH(c, K_CG_VEC, k_tail_final_dir, grid1d(n, 256, 8 * c->sm_count), 256, 0, p, p_alt, n, state);
}

__global__ void k_tail_inv(const int32_t *__restrict__ dst, int64_t ns, int32_t *__restrict__ inv) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ns; k += (int64_t)gridDim.x * blockDim.x)
        inv[dst[k]] = (int32_t)k;
}

__global__ void k_tail_inv_check(const int32_t *__restrict__ inv, int64_t n, int *__restrict__ bad) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (inv[i] < 0) atomicOr(bad, 1);
}

// once per fit, before the first iteration: the barrier words and the second partial array zeroed, and
// the output -> sample-slot map of the sampled plan (nullptr unless every output is exactly one sample:
// then the split-K parts cannot be summed per output, and the tail is not used)
const int32_t *dense_tail_init(gvt_ctx *c, double *part2, const int32_t *dst, int64_t ns, int64_t n) {
    GVT_CUDA_TRY(cudaMemsetAsync(wsT<unsigned>(c, "tail.bar", BAR_WORDS), 0, BAR_WORDS * sizeof(unsigned), c->stream));
    GVT_CUDA_TRY(cudaMemsetAsync(part2, 0, sizeof(double) * RED_BLOCKS, c->stream));
    if (ns != n || n <= 0 || !dst) return nullptr;
    int32_t *inv = wsT<int32_t>(c, "tail.inv", (size_t)n);
    int *bad = (int *)ws(c, "tail.bad", sizeof(int));
    GVT_CUDA_TRY(cudaMemsetAsync(inv, 0xff, sizeof(int32_t) * n, c->stream));
    GVT_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
    GVT_LAUNCH(c, K_PLAN_GATHER, k_tail_inv, grid1d(ns, 256, 8 * c->sm_count), 256, 0, dst, ns, inv);
    GVT_LAUNCH(c, K_PLAN_GATHER, k_tail_inv_check, grid1d(n, 256, 8 * c->sm_count), 256, 0, inv, n, bad);
    int *h = (int *)pinned(c, sizeof(int));
    GVT_CUDA_TRY(cudaMemcpyAsync(h, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return *h ? nullptr : inv;
}

}  // namespace gvt
