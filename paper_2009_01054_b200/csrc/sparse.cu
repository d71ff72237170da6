// sparse.cu -- SIMT kernels of the sparse GVT engine (north-star kernels (2) and (3) in
// their sparse form, and (4)):
//   stage 1  S[t][h] = sum_{k in row h} x_k C[col_k][t]          (segmented, no atomics)
//   stage 2  out[dst_k] = coef * <A[r_k, :], S[c_k, :]>           (gathered row dot)
//   cheap terms: segment sums, GEMV with D or D.^2, gathers/combines, Cartesian gathers.
// C and A are symmetric Grams (include/gvt.h), so C[col][t] is read in place of
// C[t][col] and every access is a contiguous row segment.
// Determinism: every output is produced by one thread/warp in a fixed order with fixed
// shuffle trees; no floating-point atomics anywhere.
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
// grid (h-blocks of H columns, t-tiles of 4*TPB rows of S).  Each thread accumulates 4
// consecutive rows t (one 16-byte load of a factor row segment per entry, four entries in
// flight) for one column h at a time in registers, parks the column in shared memory, and the
// CTA writes the H-wide column block of S row by row (128-byte coalesced stores).
template <int H, int TPB>
__global__ void __launch_bounds__(TPB) k_stage1_sparse(const int64_t *__restrict__ row_ptr,
                                                       const int32_t *__restrict__ col,
                                                       const float *__restrict__ val, int64_t m_in,
                                                       const float *__restrict__ C, int64_t ldC, int64_t q_out,
                                                       float *__restrict__ S, int64_t ldS,
                                                       const float *__restrict__ diag, int64_t row_lo) {
    constexpr int TT = TPB * 4;
    extern __shared__ float sm[];  // [H][TT + 1]
    const int tid = threadIdx.x;
    // h-blocks vary fastest across the grid, so the CTAs resident at a time share one t-tile: the
    // factor panel C[:][t0 .. t0 + TT) they read (q_in x TT floats) stays in L2 instead of the
    // whole factor streaming through it
    const int64_t t0 = (int64_t)blockIdx.y * TT;
    const int64_t h0 = (int64_t)blockIdx.x * H;
    // each thread owns 4 consecutive t: one 16-byte load per entry (ldC is a multiple of 32 and the
    // factor is zero-padded to it, so a float4 never straddles the row end)
    const int64_t tt = 4 * (int64_t)tid;
    const bool tin = t0 + tt < ldC;
    auto row4 = [&](int64_t c) -> float4 {
        return tin ? __ldg(reinterpret_cast<const float4 *>(C + c * ldC + t0 + tt)) : make_float4(0.f, 0.f, 0.f, 0.f);
    };
    for (int hl = 0; hl < H; hl++) {
        const int64_t h = h0 + hl;
        float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
        if (h < m_in) {
            const int64_t kb = row_ptr[h], ke = row_ptr[h + 1];
            int64_t k = kb;
            for (; k + 3 < ke; k += 4) {  // four entries in flight, accumulated in entry order
                float x[4];
                float4 v[4];
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    x[u] = val[k + u];
                    v[u] = row4(col[k + u]);
                }
#pragma unroll
                for (int u = 0; u < 4; u++) {
                    acc.x = fmaf(x[u], v[u].x, acc.x);
                    acc.y = fmaf(x[u], v[u].y, acc.y);
                    acc.z = fmaf(x[u], v[u].z, acc.z);
                    acc.w = fmaf(x[u], v[u].w, acc.w);
                }
            }
            for (; k < ke; k++) {
                const float x0 = val[k];
                const float4 v = row4(col[k]);
                acc.x = fmaf(x0, v.x, acc.x);
                acc.y = fmaf(x0, v.y, acc.y);
                acc.z = fmaf(x0, v.z, acc.z);
                acc.w = fmaf(x0, v.w, acc.w);
            }
            if (diag) {  // separate diagonal of X (MLPK Laplacian): X[h][h] = diag[h]
                const float dv = diag[row_lo + h];
                const float4 v = row4(row_lo + h);
                acc.x = fmaf(dv, v.x, acc.x);
                acc.y = fmaf(dv, v.y, acc.y);
                acc.z = fmaf(dv, v.z, acc.z);
                acc.w = fmaf(dv, v.w, acc.w);
            }
        }
        float *dst = sm + hl * (TT + 1) + tt;
        dst[0] = acc.x;
        dst[1] = acc.y;
        dst[2] = acc.z;
        dst[3] = acc.w;
    }
    __syncthreads();
    const int lane = tid & 31, warp = tid >> 5;
    for (int t = warp; t < TT; t += TPB / 32) {
        const int64_t tg = t0 + t;
        if (tg >= q_out) break;
        for (int hl = lane; hl < H; hl += 32) {
            const int64_t h = h0 + hl;
            if (h < ldS) S[tg * ldS + h] = sm[hl * (TT + 1) + t];  // h >= m_in writes the zero padding
        }
    }
}

void stage1_sparse(gvt_ctx *c, const EntryPlan &e, const Factor &C, int64_t q_out, float *S, int64_t ldS,
                   const float *diag, int64_t row_lo) {
    constexpr int H = 32, TPB = 128, TT = TPB * 4;
    if (q_out == 0 || ldS == 0) return;
    dim3 grid((unsigned)((ldS + H - 1) / H), (unsigned)((q_out + TT - 1) / TT));
    size_t smem = sizeof(float) * H * (TT + 1);
    static bool attr[GVT_MAX_DEVICES] = {};  // per device ordinal
    bool &attr_dev = attr[c->device < GVT_MAX_DEVICES ? c->device : 0];
    if (!attr_dev) {
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_stage1_sparse<H, TPB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        attr_dev = true;
    }
    GVT_LAUNCH(c, K_STAGE1_SPARSE, (k_stage1_sparse<H, TPB>), grid, TPB, smem, e.row_ptr, e.col, e.val, e.nrow,
               C.p, C.ld, q_out, S, ldS, diag, row_lo);
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

void gemv(gvt_ctx *c, const Factor &F, const float *b, int square, float *y) {
    if (F.n == 0) return;
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
