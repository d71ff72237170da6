// sparse.cu -- SIMT kernels of the sparse GVT engine (north-star kernels (2) and (3) in
// their sparse form, and (4)):
//   stage 1  S[t][h] = sum_{k in row h} x_k C[col_k][t]          (segmented, no atomics)
//   stage 2  out[dst_k] = coef * <A[r_k, :], S[c_k, :]>           (gathered row dot)
//   cheap terms: segment sums, GEMV with D or D.^2, gathers/combines, Cartesian gathers.
// C and A are symmetric Grams (include/gvt.h), so C[col][t] is read in place of
// C[t][col] and every access is a contiguous row segment.
// Determinism: every output is produced by one thread/warp in a fixed order with fixed
// shuffle trees; no floating-point atomics anywhere.
#include <stdlib.h>

#include <algorithm>

#include "ops.cuh"

namespace gvt {

__device__ __forceinline__ float warp_sum(float v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ int32_t pick(int sel, const int32_t *f, const int32_t *s, int64_t j) {
    return sel == 0 ? f[j] : s[j];
}

// ----------------------------------------------------------------------------- values
__global__ void k_entry_values(const int32_t *__restrict__ src, const float *__restrict__ sign, int64_t E,
                               const float *__restrict__ p, float *__restrict__ val) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x)
        val[k] = sign[k] * __ldg(p + src[k]);
}

void entry_values(gvt_ctx *c, const EntryPlan &e, const float *p) {
    if (e.nnz == 0) return;
    GVT_LAUNCH(c, K_PLAN_GATHER, k_entry_values, grid1d(e.nnz, 256, 8 * c->sm_count * 8), 256, 0, e.src, e.sign,
               e.nnz, p, e.val);
}

// ----------------------------------------------------------------------------- stage 1
// grid (h-blocks of H columns, t-tiles of 4*TPB rows of S).  The CTA walks the entries of its H
// rows (one contiguous CSR range) in chunks of CH staged in shared memory (coalesced index/value
// loads, then broadcast reads), so the only global loads in the inner loop are the independent
// factor-row segments: each thread owns 4 consecutive rows t (one 16-byte load per entry; the
// loop is unrolled by eight, ptxas keeps about four in flight at 32 registers, and occupancy
// hides the rest), accumulates one column h at a time in entry order, parks it in shared memory
// when the row ends, and the CTA writes the H-wide column block of S row by row (H * 4-byte
// segments per row of S).
template <int H, int TPB, int CH>
__global__ void __launch_bounds__(TPB) k_stage1_sparse(const int64_t *__restrict__ row_ptr,
                                                       const int32_t *__restrict__ col,
                                                       const float *__restrict__ val, int64_t m_in,
                                                       const float *__restrict__ C, int64_t ldC, int64_t q_out,
                                                       float *__restrict__ S, int64_t ldS,
                                                       const float *__restrict__ diag, int64_t row_lo) {
    constexpr int TT = TPB * 4;
    extern __shared__ float sm[];  // park [H][TT + 1] | chunk values [CH] | chunk columns [CH]
    float *sval = sm + H * (TT + 1);
    int32_t *scol = reinterpret_cast<int32_t *>(sval + CH);
    __shared__ int64_t srp[H + 1];
    const int tid = threadIdx.x;
    // h-blocks vary fastest across the grid, so the CTAs resident at a time share one t-tile: the
    // factor panel C[:][t0 .. t0 + TT) they read (q_in x TT floats) stays in L2 instead of the
    // whole factor streaming through it
    const int64_t t0 = (int64_t)blockIdx.y * TT;
    const int64_t h0 = (int64_t)blockIdx.x * H;
    const int hv = (int)max((int64_t)0, min((int64_t)H, m_in - h0));  // valid rows of this block
    if (hv > 0)  // (a block past the last row has no row pointers to read)
        for (int i = tid; i <= hv; i += TPB) srp[i] = row_ptr[h0 + i];
    // each thread owns 4 consecutive t: one 16-byte load per entry (ldC is a multiple of 32 and the
    // factor is zero-padded to it, so a float4 never straddles the row end)
    // (threads past the row end of the last t-tile read column 0 instead: unconditional loads keep
    // the eight in flight, and their sums are never stored -- only t < q_out <= ldC are written)
    const int tt = 4 * tid;
    const float *Ct = C + (t0 + tt < ldC ? t0 + tt : 0);
    auto row4 = [&](int64_t c) -> float4 { return __ldg(reinterpret_cast<const float4 *>(Ct + c * ldC)); };
    auto fma4 = [](float x, const float4 &v, float4 &acc) {
        acc.x = fmaf(x, v.x, acc.x);
        acc.y = fmaf(x, v.y, acc.y);
        acc.z = fmaf(x, v.z, acc.z);
        acc.w = fmaf(x, v.w, acc.w);
    };
    auto park = [&](int hl, float4 acc) {
        if (hl < hv && diag) {  // separate diagonal of X (MLPK Laplacian): X[h][h] = diag[h], added last
            const int64_t hd = row_lo + h0 + hl;
            fma4(diag[hd], row4(hd), acc);
        }
        float *dst = sm + hl * (TT + 1) + tt;
        dst[0] = acc.x;
        dst[1] = acc.y;
        dst[2] = acc.z;
        dst[3] = acc.w;
    };
    __syncthreads();
    const int64_t e0 = hv > 0 ? srp[0] : 0, e1 = hv > 0 ? srp[hv] : 0;
    int hl = 0;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int64_t cb = e0; cb < e1; cb += CH) {
        const int n = (int)min((int64_t)CH, e1 - cb);
        __syncthreads();  // the previous chunk is consumed
        for (int i = tid; i < n; i += TPB) {
            sval[i] = val[cb + i];
            scol[i] = col[cb + i];
        }
        __syncthreads();
        int i = 0;
        while (i < n) {
            while (cb + i >= srp[hl + 1]) {  // rows that ended (or are empty) before entry cb + i
                park(hl, acc);
                acc = make_float4(0.f, 0.f, 0.f, 0.f);
                hl++;
            }
            const int iend = (int)min((int64_t)n, srp[hl + 1] - cb);
            for (; i + 7 < iend; i += 8) {  // eight entries per step, accumulated in entry order
                float4 v[8];
#pragma unroll
                for (int u = 0; u < 8; u++) v[u] = row4(scol[i + u]);
#pragma unroll
                for (int u = 0; u < 8; u++) fma4(sval[i + u], v[u], acc);
            }
            for (; i < iend; i++) fma4(sval[i], row4(scol[i]), acc);
        }
    }
    for (; hl < H; hl++) {  // the last row with entries, then empty rows and rows >= m_in
        park(hl, acc);
        acc = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    for (int t = warp; t < TT; t += TPB / 32) {
        const int64_t tg = t0 + t;
        if (tg >= q_out) break;
        for (int hl2 = lane; hl2 < H; hl2 += 32) {
            const int64_t h = h0 + hl2;
            if (h < ldS) S[tg * ldS + h] = sm[hl2 * (TT + 1) + t];  // h >= m_in writes the zero padding
        }
    }
}

template <int H, int CH>
static void stage1_sparse_h(gvt_ctx *c, const EntryPlan &e, const Factor &C, int64_t q_out, float *S, int64_t ldS,
                            const float *diag, int64_t row_lo) {
    constexpr int TPB = 128, TT = TPB * 4;
    dim3 grid((unsigned)((ldS + H - 1) / H), (unsigned)((q_out + TT - 1) / TT));
    size_t smem = sizeof(float) * H * (TT + 1) + (sizeof(float) + sizeof(int32_t)) * CH;
    static bool attr[GVT_MAX_DEVICES] = {};  // per device ordinal
    bool &attr_dev = attr[c->device < GVT_MAX_DEVICES ? c->device : 0];
    if (!attr_dev) {
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_stage1_sparse<H, TPB, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        attr_dev = true;
    }
    GVT_LAUNCH(c, K_STAGE1_SPARSE, (k_stage1_sparse<H, TPB, CH>), grid, TPB, smem, e.row_ptr, e.col, e.val, e.nrow,
               C.p, C.ld, q_out, S, ldS, diag, row_lo);
}

void stage1_sparse(gvt_ctx *c, const EntryPlan &e, const Factor &C, int64_t q_out, float *S, int64_t ldS,
                   const float *diag, int64_t row_lo) {
    if (q_out == 0 || ldS == 0) return;
    // H = 8 columns per CTA: 24.6 KB of shared memory, so 9 CTAs (36 warps) per SM hide the
    // factor-row load latency (H = 32: 3 CTAs; measured 5.0 vs 8.4 ms in the 0.2 % gather regime,
    // 517 vs 765 ms at C5 density, scripts/gather_regime_probe.py / gather_probe.py)
    stage1_sparse_h<8, 1024>(c, e, C, q_out, S, ldS, diag, row_lo);
}

// ----------------------------------------------------------------------------- stage 2
// one warp per sample; samples are sorted by row r so consecutive warps reuse A[r,:]
// from L1/L2; 128-bit loads of both rows; fixed lane order + butterfly reduction.
__global__ void __launch_bounds__(256) k_stage2_gather(int64_t ns, const int32_t *__restrict__ sr,
                                                       const int32_t *__restrict__ sc,
                                                       const int32_t *__restrict__ sdst,
                                                       const float *__restrict__ A, int64_t ldA,
                                                       const float *__restrict__ S, int64_t ldS, int64_t K4,
                                                       float coef, int accumulate, float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < ns; k += warps) {
        const float4 *a = reinterpret_cast<const float4 *>(A + (int64_t)sr[k] * ldA);
        const float4 *s = reinterpret_cast<const float4 *>(S + (int64_t)sc[k] * ldS);
        float acc0 = 0.f, acc1 = 0.f;
        int64_t h = lane;
        for (; h + 32 < K4; h += 64) {
            float4 x0 = __ldg(a + h), y0 = __ldg(s + h);
            float4 x1 = __ldg(a + h + 32), y1 = __ldg(s + h + 32);
            acc0 = fmaf(x0.x, y0.x, acc0); acc0 = fmaf(x0.y, y0.y, acc0);
            acc0 = fmaf(x0.z, y0.z, acc0); acc0 = fmaf(x0.w, y0.w, acc0);
            acc1 = fmaf(x1.x, y1.x, acc1); acc1 = fmaf(x1.y, y1.y, acc1);
            acc1 = fmaf(x1.z, y1.z, acc1); acc1 = fmaf(x1.w, y1.w, acc1);
        }
        for (; h < K4; h += 32) {
            float4 x0 = __ldg(a + h), y0 = __ldg(s + h);
            acc0 = fmaf(x0.x, y0.x, acc0); acc0 = fmaf(x0.y, y0.y, acc0);
            acc0 = fmaf(x0.z, y0.z, acc0); acc0 = fmaf(x0.w, y0.w, acc0);
        }
        float v = warp_sum(acc0 + acc1);
        if (lane == 0) {
            const int64_t d = sdst[k];
            out[d] = accumulate ? fmaf(coef, v, out[d]) : coef * v;
        }
    }
}

void stage2_gather(gvt_ctx *c, const SamplePlan &sp, const Factor &A, const float *S, int64_t ldS, int64_t K,
                   float coef, int accumulate, float *out) {
    if (sp.ns == 0) return;
    int64_t K4 = round_up(K, 4) / 4;
    GVT_LAUNCH(c, K_STAGE2_GATHER, k_stage2_gather, grid1d(sp.ns * 32, 256, (int64_t)c->sm_count * 16), 256, 0,
               sp.ns, sp.r, sp.c, sp.dst, A.p, A.ld, S, ldS, K4, coef, accumulate, out);
}

// the same gather over the dense engine's S, stored by the stage-1 GEMM as fp16 pieces with one
// power-of-two scale per (row, 256-column chunk): S[c][h] = (hi + lo) * sk[(h / 256) * skld + c].
// Lanes take column pairs (half2 / float2 loads) in a fixed order, then a butterfly.
__global__ void __launch_bounds__(256) k_stage2_gather16(int64_t ns, const int32_t *__restrict__ sr,
                                                         const int32_t *__restrict__ sc,
                                                         const int32_t *__restrict__ sdst,
                                                         const float *__restrict__ A, int64_t ldA,
                                                         const __half *__restrict__ Sh, const __half *__restrict__ Sl,
                                                         int64_t ldS, const float *__restrict__ sk, int64_t skld,
                                                         int64_t K, float coef, int accumulate, float *__restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < ns; k += warps) {
        const int64_t c = sc[k];
        const float2 *a = reinterpret_cast<const float2 *>(A + (int64_t)sr[k] * ldA);
        const __half2 *h2 = reinterpret_cast<const __half2 *>(Sh + c * ldS);
        const __half2 *l2 = reinterpret_cast<const __half2 *>(Sl + c * ldS);
        float acc = 0.f;
        for (int64_t j = lane; 2 * j < K; j += 32) {
            const int64_t h = 2 * j;
            const float s = __ldg(sk + (h >> 8) * skld + c / S16_SCALE_ROWS);  // h and h + 1 share the chunk
            const float2 av = __ldg(a + j);
            const float2 hv = __half22float2(h2[j]), lv = __half22float2(l2[j]);
            acc = fmaf(av.x, (hv.x + lv.x) * s, acc);
            if (h + 1 < K) acc = fmaf(av.y, (hv.y + lv.y) * s, acc);  // (the padding column is never used)
        }
        const float v = warp_sum(acc);
        if (lane == 0) {
            const int64_t d = sdst[k];
            out[d] = accumulate ? fmaf(coef, v, out[d]) : coef * v;
        }
    }
}

void stage2_gather16(gvt_ctx *c, const SamplePlan &sp, const Factor &A, const __half *Sh, const __half *Sl,
                     int64_t ldS, const float *sk, int64_t skld, int64_t K, float coef, int accumulate, float *out) {
    if (sp.ns == 0) return;
    GVT_LAUNCH(c, K_STAGE2_GATHER, k_stage2_gather16, grid1d(sp.ns * 32, 256, (int64_t)c->sm_count * 16), 256, 0,
               sp.ns, sp.r, sp.c, sp.dst, A.p, A.ld, Sh, Sl, ldS, sk, skld, K, coef, accumulate, out);
}

// ----------------------------------------------------------------------------- cheap terms
// b[h] = sum_{k in row h} val[k], one warp per row, lanes strided + butterfly
__global__ void k_segment_sum(const int64_t *__restrict__ row_ptr, int64_t nrow, const float *__restrict__ val,
                              float *__restrict__ b) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t h = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); h < nrow; h += warps) {
        float acc = 0.f;
        for (int64_t k = row_ptr[h] + lane; k < row_ptr[h + 1]; k += 32) acc += val[k];
        acc = warp_sum(acc);
        if (lane == 0) b[h] = acc;
    }
}

// b[h] = sum_{k in row h} sign[k] p[src[k]]: the entry values gathered inside the segment sum (the
// same per-lane order and tree as k_entry_values followed by k_segment_sum, one pass fewer)
// With r (the fused CG tail, cg.cu k_cg_combine_ap), the direction is formed on the fly:
// p_k = r_{k-1} + beta p_{k-1} with beta = *beta_st -- the k_cg_p update, read-only here; the tail
// stores p_k.  Same fmaf as k_cg_p, so the values equal the separate update's.
__global__ void k_segment_sum_gather(const int64_t *__restrict__ row_ptr, int64_t nrow, const int32_t *__restrict__ src,
                                     const float *__restrict__ sign, const float *__restrict__ p,
                                     const float *__restrict__ r, const double *__restrict__ beta_st,
                                     float *__restrict__ b) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const float beta = r ? (float)*beta_st : 0.f;
    for (int64_t h = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); h < nrow; h += warps) {
        float acc = 0.f;
        if (r) {
            for (int64_t k = row_ptr[h] + lane; k < row_ptr[h + 1]; k += 32) {
                const int32_t j = src[k];
                acc += sign[k] * fmaf(beta, __ldg(p + j), __ldg(r + j));
            }
        } else {
            for (int64_t k = row_ptr[h] + lane; k < row_ptr[h + 1]; k += 32) acc += sign[k] * __ldg(p + src[k]);
        }
        acc = warp_sum(acc);
        if (lane == 0) b[h] = acc;
    }
}

void segment_sum_gather(gvt_ctx *c, const EntryPlan &e, const float *p, float *b, const float *r,
                        const double *beta_st) {
    if (e.nrow == 0) return;
    GVT_LAUNCH(c, K_SEGSUM, k_segment_sum_gather, grid1d(e.nrow * 32, 256, (int64_t)c->sm_count * 16), 256, 0,
               e.row_ptr, e.nrow, e.src, e.sign, p, r, beta_st, b);
}

void segment_sum(gvt_ctx *c, const EntryPlan &e, float *b) {
    if (e.nrow == 0) return;
    GVT_LAUNCH(c, K_SEGSUM, k_segment_sum, grid1d(e.nrow * 32, 256, (int64_t)c->sm_count * 16), 256, 0, e.row_ptr,
               e.nrow, e.val, b);
}

// y[r] = sum_h F[r,h]^(1|2) b[h]; b is padded with zeros up to ld
__global__ void __launch_bounds__(256) k_gemv(const float *__restrict__ F, int64_t n, int64_t ld,
                                              const float *__restrict__ b, int square, float *__restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int64_t K4 = ld / 4;
    const float4 *bb = reinterpret_cast<const float4 *>(b);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < n; r += warps) {
        const float4 *row = reinterpret_cast<const float4 *>(F + r * ld);
        float acc = 0.f;
        for (int64_t h = lane; h < K4; h += 32) {
            float4 x = __ldg(row + h), z = __ldg(bb + h);
            if (square) { x.x *= x.x; x.y *= x.y; x.z *= x.z; x.w *= x.w; }
            acc = fmaf(x.x, z.x, acc); acc = fmaf(x.y, z.y, acc);
            acc = fmaf(x.z, z.z, acc); acc = fmaf(x.w, z.w, acc);
        }
        acc = warp_sum(acc);
        if (lane == 0) y[r] = acc;
    }
}

// the same per-lane order (float4 chunks h = lane, lane + 32, ...) and tree as k_gemv, with b staged
// in shared memory once per block of 8 rows and the row loads unrolled by four (independent 16-byte
// loads in flight: the factor stream is the HBM-bound part, 4 B per FMA; k_gemv reached ~63 % of
// the copy bandwidth on the 8000^2 union Gram of C4)
__global__ void __launch_bounds__(256) k_gemv_smem(const float *__restrict__ F, int64_t n, int64_t ld,
                                                   const float *__restrict__ b, int square, float *__restrict__ y) {
    extern __shared__ float4 bs[];
    const int64_t K4 = ld / 4;
    for (int64_t h = threadIdx.x; h < K4; h += blockDim.x) bs[h] = __ldg(reinterpret_cast<const float4 *>(b) + h);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (r >= n) return;
    const float4 *row = reinterpret_cast<const float4 *>(F + r * ld);
    float acc = 0.f;
    int64_t h = lane;
    for (; h + 96 < K4; h += 128) {
        float4 x[4];
#pragma unroll
        for (int u = 0; u < 4; u++) x[u] = __ldg(row + h + 32 * u);
#pragma unroll
        for (int u = 0; u < 4; u++) {
            float4 xx = x[u];
            const float4 z = bs[h + 32 * u];
            if (square) { xx.x *= xx.x; xx.y *= xx.y; xx.z *= xx.z; xx.w *= xx.w; }
            acc = fmaf(xx.x, z.x, acc); acc = fmaf(xx.y, z.y, acc);
            acc = fmaf(xx.z, z.z, acc); acc = fmaf(xx.w, z.w, acc);
        }
    }
    for (; h < K4; h += 32) {
        float4 xx = __ldg(row + h);
        const float4 z = bs[h];
        if (square) { xx.x *= xx.x; xx.y *= xx.y; xx.z *= xx.z; xx.w *= xx.w; }
        acc = fmaf(xx.x, z.x, acc); acc = fmaf(xx.y, z.y, acc);
        acc = fmaf(xx.z, z.z, acc); acc = fmaf(xx.w, z.w, acc);
    }
    acc = warp_sum(acc);
    if (lane == 0) y[r] = acc;
}

// ---- symmetric GEMV: y = F b (or F.^2 b) reading only the upper triangle of a square Gram
// (symmetric by definition, R1).  The columns are cut into panels of SYMV_PW = 1024 (thread t owns
// column quad t of the panel) and the rows of each panel's upper part (rows 0 .. panel
// end) into chunks of SYMV_RC = 64 (enough CTAs: ~4 per SM at C4's n = 8000); one CTA per (panel, row
// chunk) streams its rows as 4 KB contiguous segments, SYMV_RB = 4 rows (loads of 16 B) per thread in flight
// (8 measured 1 % slower, wider panels / shorter chunks slower still: profiles/r02_ab_symv_geom.txt):
//   row part    prow[panel][i] = sum_{j >= i, j in panel} F_ij b_j   (warp trees, then warps in order)
//   column part pcol[unit][j]  = sum_{i in chunk, i < j} F_ij b_i    (registers)
// k_symv_finish adds, per j, the row parts of the panels right of j and the column parts of the chunks
// above j, in a fixed order: deterministic, no atomics, half the HBM bytes of the plain GEMV.
#ifndef GVT_SYMV_PW  // panel width / row chunk / rows per batch (A/B builds override them)
#define GVT_SYMV_PW 1024
#define GVT_SYMV_RC 64
#define GVT_SYMV_RB 4
#endif
constexpr int SYMV_PW = GVT_SYMV_PW, SYMV_RC = GVT_SYMV_RC, SYMV_RB = GVT_SYMV_RB, SYMV_QT = SYMV_PW / 1024;

__device__ __forceinline__ int64_t symv_rows(int64_t n, int p) {  // rows with upper-triangle cells in panel p
    const int64_t e = (int64_t)(p + 1) * SYMV_PW;
    return e < n ? e : n;
}

__global__ void __launch_bounds__(256, 4) k_symv_panel(const float *__restrict__ F, int64_t n, int64_t ld,
                                                       const float *__restrict__ b, int square,
                                                       float *__restrict__ prow, float *__restrict__ pcol) {
    __shared__ float red[8][SYMV_RC];  // per warp, per row of the chunk: the warp's partial row sum
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    int p = 0, u = blockIdx.x;
    while (u >= (int)((symv_rows(n, p) + SYMV_RC - 1) / SYMV_RC)) {
        u -= (int)((symv_rows(n, p) + SYMV_RC - 1) / SYMV_RC);
        p++;
    }
    const int64_t i0 = (int64_t)u * SYMV_RC, i1 = min(i0 + SYMV_RC, symv_rows(n, p));
    int64_t j0[SYMV_QT];
    float4 bq[SYMV_QT], cacc[SYMV_QT];
#pragma unroll
    for (int h = 0; h < SYMV_QT; h++) {
        j0[h] = (int64_t)p * SYMV_PW + 1024 * h + 4 * tid;  // this thread's quads
        bq[h] = j0[h] < n ? __ldg(reinterpret_cast<const float4 *>(b + j0[h])) : make_float4(0.f, 0.f, 0.f, 0.f);
        if (j0[h] + 1 >= n) bq[h].y = 0.f;
        if (j0[h] + 2 >= n) bq[h].z = 0.f;
        if (j0[h] + 3 >= n) bq[h].w = 0.f;
        cacc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int64_t ib = i0; ib < i1; ib += SYMV_RB) {
        float4 x[SYMV_RB][SYMV_QT];
#pragma unroll
        for (int r = 0; r < SYMV_RB; r++) {  // a quad entirely left of the diagonal is never read
            const int64_t i = ib + r;
#pragma unroll
            for (int h = 0; h < SYMV_QT; h++)
                x[r][h] = (i < i1 && j0[h] < n && j0[h] + 3 >= i)
                              ? __ldg(reinterpret_cast<const float4 *>(F + i * ld + j0[h]))
                              : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        float rp[SYMV_RB];
#pragma unroll
        for (int r = 0; r < SYMV_RB; r++) {
            const int64_t i = ib + r;
            const float bi = i < i1 ? __ldg(b + i) : 0.f;
            rp[r] = 0.f;
#pragma unroll
            for (int h = 0; h < SYMV_QT; h++) {
                float4 v = x[r][h];
                if (square) { v.x *= v.x; v.y *= v.y; v.z *= v.z; v.w *= v.w; }
                float4 w = v;  // column part: j > i only; row part: j >= i
                const int64_t jj = j0[h];
                if (jj <= i) {
                    if (jj < i) { v.x = 0.f; w.x = 0.f; } else w.x = 0.f;
                    if (jj + 1 < i) { v.y = 0.f; w.y = 0.f; } else if (jj + 1 == i) w.y = 0.f;
                    if (jj + 2 < i) { v.z = 0.f; w.z = 0.f; } else if (jj + 2 == i) w.z = 0.f;
                    if (jj + 3 < i) { v.w = 0.f; w.w = 0.f; } else if (jj + 3 == i) w.w = 0.f;
                }
                rp[r] = fmaf(v.w, bq[h].w, fmaf(v.z, bq[h].z, fmaf(v.y, bq[h].y, fmaf(v.x, bq[h].x, rp[r]))));
                cacc[h].x = fmaf(w.x, bi, cacc[h].x);
                cacc[h].y = fmaf(w.y, bi, cacc[h].y);
                cacc[h].z = fmaf(w.z, bi, cacc[h].z);
                cacc[h].w = fmaf(w.w, bi, cacc[h].w);
            }
        }
        // row parts of the batch: warp trees parked per warp (no CTA barrier inside the row loop)
#pragma unroll
        for (int r = 0; r < SYMV_RB; r++) {
            float v = rp[r];
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            rp[r] = v;
        }
        if (lane < SYMV_RB) {
            float v = rp[0];
#pragma unroll
            for (int r = 1; r < SYMV_RB; r++) v = lane == r ? rp[r] : v;
            red[warp][ib - i0 + lane] = v;
        }
    }
#pragma unroll
    for (int h = 0; h < SYMV_QT; h++)
        *reinterpret_cast<float4 *>(pcol + (int64_t)blockIdx.x * SYMV_PW + 1024 * h + 4 * tid) = cacc[h];
    __syncthreads();
    if (tid < SYMV_RC && i0 + tid < i1) {  // the 8 warps' row partials in warp order
        float v = 0.f;
#pragma unroll
        for (int w8 = 0; w8 < 8; w8++) v += red[w8][tid];
        prow[(int64_t)p * n + i0 + tid] = v;
    }
}

// y_j for 32 consecutive j per CTA: warp w sums the column parts of chunk range w (of 8, contiguous),
// then lane j adds the row parts of panels panel(j) .. last and the 8 ranges in order
__global__ void __launch_bounds__(256) k_symv_finish(const float *__restrict__ prow, const float *__restrict__ pcol,
                                                     int np, int64_t n, float *__restrict__ y) {
    __shared__ float part[8][32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t j = (int64_t)blockIdx.x * 32 + lane;
    const int64_t jc = j < n ? j : n - 1;
    const int pj = (int)(jc / SYMV_PW);
    int64_t ubase = 0;
    for (int p = 0; p < pj; p++) ubase += (symv_rows(n, p) + SYMV_RC - 1) / SYMV_RC;
    const int64_t nc = (jc + SYMV_RC - 1) / SYMV_RC;  // chunks holding a row < j
    const int64_t c0 = nc * warp / 8, c1 = nc * (warp + 1) / 8;
    const float *pc = pcol + ubase * SYMV_PW + (jc - (int64_t)pj * SYMV_PW);
    // every load of a group in flight before the first add (a latency-bound kernel: C4's 125 chunks are
    // 16 per warp, one round trip instead of four); the adds keep chunk order
    float v = 0.f;
    for (int64_t c = c0; c < c1; c += 16) {
        float t16[16];
#pragma unroll
        for (int k = 0; k < 16; k++) t16[k] = c + k < c1 ? pc[(c + k) * SYMV_PW] : 0.f;
#pragma unroll
        for (int k = 0; k < 16; k++)
            if (c + k < c1) v += t16[k];
    }
    part[warp][lane] = v;
    __syncthreads();
    if (warp == 0 && j < n) {
        float s = 0.f;
        for (int p = pj; p < np; p += 8) {  // row parts, in panel order
            float t8[8];
#pragma unroll
            for (int k = 0; k < 8; k++) t8[k] = p + k < np ? prow[(int64_t)(p + k) * n + j] : 0.f;
#pragma unroll
            for (int k = 0; k < 8; k++)
                if (p + k < np) s += t8[k];
        }
#pragma unroll
        for (int w8 = 0; w8 < 8; w8++) s += part[w8][lane];
        y[j] = s;
    }
}

// the symmetric (upper-triangle) GEMV pays once the Gram outgrows L2: n >= 6144 (151 MB).  Measured
// (profiles/r02_ab_symv.txt): C4 Ranking's 8000^2 union Gram 104-105 -> 91-93 us per CG iteration;
// C4 Poly2D's 5000^2 / 3000^2 Grams 3 % slower with it, so they keep the row GEMV.  GVT_SYMV=0 disables.
static bool symv_enabled() {
    static const bool on = [] {
        const char *e = getenv("GVT_SYMV");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

void gemv(gvt_ctx *c, const Factor &F, const float *b, int square, float *y, bool symmetric) {
    if (F.n == 0) return;
    if (symmetric && symv_enabled() && F.n == F.cols && F.n >= 6144 && F.ld % 4 == 0) {
        const int np = (int)((F.n + SYMV_PW - 1) / SYMV_PW);
        int64_t units = 0;
        for (int p = 0; p < np; p++) units += (std::min<int64_t>((int64_t)(p + 1) * SYMV_PW, F.n) + SYMV_RC - 1) / SYMV_RC;
        float *prow = wsT<float>(c, "symv.prow", (size_t)np * F.n);
        float *pcol = wsT<float>(c, "symv.pcol", (size_t)units * SYMV_PW);
        GVT_LAUNCH(c, K_GEMV, k_symv_panel, (unsigned)units, 256, 0, F.p, F.n, F.ld, b, square, prow, pcol);
        GVT_LAUNCH(c, K_GEMV, k_symv_finish, (unsigned)((F.n + 31) / 32), 256, 0, prow, pcol, np, F.n, y);
        return;
    }
    const size_t smem = sizeof(float) * (size_t)F.ld;
    if (smem <= 160 * 1024 && F.ld % 4 == 0) {
        static size_t attr[GVT_MAX_DEVICES] = {};
        size_t &attr_dev = attr[c->device < GVT_MAX_DEVICES ? c->device : 0];
        if (smem > 48 * 1024 && smem > attr_dev) {
            GVT_CUDA_TRY(cudaFuncSetAttribute(k_gemv_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            attr_dev = smem;
        }
        GVT_LAUNCH(c, K_GEMV, k_gemv_smem, grid1d(F.n * 32, 256), 256, smem, F.p, F.n, F.ld, b, square, y);
        return;
    }
    GVT_LAUNCH(c, K_GEMV, k_gemv, grid1d(F.n * 32, 256, (int64_t)c->sm_count * 16), 256, 0, F.p, F.n, F.ld, b, square,
               y);
}

__global__ void k_combine_gather(const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n,
                                 const float *__restrict__ g1, int rs1, float c1, const float *__restrict__ g2,
                                 int rs2, float c2, int accumulate, float *__restrict__ u) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = c1 * g1[pick(rs1, f, s, i)];
        if (g2) v = fmaf(c2, g2[pick(rs2, f, s, i)], v);
        u[i] = accumulate ? u[i] + v : v;
    }
}

void combine_gather(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, const float *g1, int rs1, float c1,
                    const float *g2, int rs2, float c2, int accumulate, float *u) {
    if (n == 0) return;
    GVT_LAUNCH(c, K_COMBINE, k_combine_gather, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, f, s, n, g1, rs1, c1, g2,
               rs2, c2, accumulate, u);
}

__global__ void k_combine_mlpk(const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n,
                               const float *__restrict__ buf, float *__restrict__ u) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        u[i] = (buf[n + f[i]] + buf[n + s[i]]) - 2.0f * buf[i];
}

void combine_mlpk(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, const float *buf, float *u) {
    if (n == 0) return;
    GVT_LAUNCH(c, K_COMBINE, k_combine_mlpk, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, f, s, n, buf, u);
}

// Cartesian (Corollary D(x)I + I(x)T): warp per output,
//   u_i = sum_{k: second_k = t_i} D[d_i, first_k] p_k + sum_{k: first_k = d_i} T[t_i, second_k] p_k
__global__ void k_cartesian(const int32_t *__restrict__ of, const int32_t *__restrict__ os, int64_t n_out,
                            const int64_t *__restrict__ rp_first, const int32_t *__restrict__ col_first,
                            const float *__restrict__ val_first, int64_t n_first_rows,
                            const int64_t *__restrict__ rp_second, const int32_t *__restrict__ col_second,
                            const float *__restrict__ val_second, int64_t n_second_rows,
                            const float *__restrict__ D, int64_t ldD, const float *__restrict__ T, int64_t ldT,
                            float *__restrict__ u) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_out; i += warps) {
        const int32_t d = of[i], t = os[i];
        float acc = 0.f;
        if (t < n_second_rows) {
            const float *drow = D + (int64_t)d * ldD;
            for (int64_t k = rp_second[t] + lane; k < rp_second[t + 1]; k += 32)
                acc = fmaf(__ldg(drow + col_second[k]), val_second[k], acc);
        }
        float acc2 = 0.f;
        if (d < n_first_rows) {
            const float *trow = T + (int64_t)t * ldT;
            for (int64_t k = rp_first[d] + lane; k < rp_first[d + 1]; k += 32)
                acc2 = fmaf(__ldg(trow + col_first[k]), val_first[k], acc2);
        }
        float v = warp_sum(acc) + warp_sum(acc2);
        if (lane == 0) u[i] = v;
    }
}

void cartesian(gvt_ctx *c, const int32_t *of, const int32_t *os, int64_t n_out, const EntryPlan &by_first,
               const EntryPlan &by_second, const Factor &D, const Factor &T, float *u) {
    if (n_out == 0) return;
    GVT_LAUNCH(c, K_CARTESIAN, k_cartesian, grid1d(n_out * 32, 256, (int64_t)c->sm_count * 16), 256, 0, of, os, n_out,
               by_first.row_ptr, by_first.col, by_first.val, by_first.nrow, by_second.row_ptr, by_second.col,
               by_second.val, by_second.nrow, D.p, D.ld, T.p, T.ld, u);
}

__global__ void k_scale_copy(const float *__restrict__ x, float alpha, int64_t n, float *__restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = alpha * x[i];
}

__global__ void k_add_into(const float *__restrict__ x, int64_t n, float *__restrict__ y) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] += x[i];
}

void add_into(gvt_ctx *c, const float *x, int64_t n, float *y) {
    if (n == 0) return;
    GVT_LAUNCH(c, K_FILL, k_add_into, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, x, n, y);
}

void scale_copy(gvt_ctx *c, const float *x, float alpha, int64_t n, float *y) {
    if (n == 0) return;
    GVT_LAUNCH(c, K_FILL, k_scale_copy, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, x, alpha, n, y);
}

}  // namespace gvt
