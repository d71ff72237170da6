// gram.cu -- SIMT base-kernel Gram (north-star kernel (1), SIMT form; the tensor-core
// form is in dense_tc.cu).  K[i][j] = k(X_i, X_j):
//   LINEAR   <x,y>
//   GAUSSIAN exp(-gamma * sum_k (x_k - y_k)^2)   direct differences => K[i][i] = 1 exactly
// K[i][j] = k(X_i, Y_j) for the cross-Gram of two tables (novel objects, Y != X).
//   POLY     (gamma <x,y> + coef0)^degree
// 64x64 output tile per 256-thread CTA, 4x4 outputs per thread, X tiles staged in smem.
#include "ops.cuh"

namespace gvt {

template <int KIND>
__global__ void __launch_bounds__(256) k_gram_simt(const float *__restrict__ X, int64_t m, const float *__restrict__ Y,
                                                   int64_t m2, int64_t dim, int64_t ldx, float gamma, float coef0,
                                                   int degree, float *__restrict__ K, int64_t ldk) {
    constexpr int BT = 64, BK = 16;
    __shared__ float xa[BK][BT + 4];
    __shared__ float xb[BK][BT + 4];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.y * BT, j0 = (int64_t)blockIdx.x * BT;
    float acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0.f;
    for (int64_t k0 = 0; k0 < dim; k0 += BK) {
        for (int e = threadIdx.x; e < BT * BK; e += 256) {
            int r = e / BK, kk = e % BK;
            int64_t gi = i0 + r, gj = j0 + r, gk = k0 + kk;
            xa[kk][r] = (gi < m && gk < dim) ? X[gi * ldx + gk] : 0.f;
            xb[kk][r] = (gj < m2 && gk < dim) ? Y[gj * ldx + gk] : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            float av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; a++) av[a] = xa[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; b++) bv[b] = xb[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) {
                    if (KIND == GVT_BASE_GAUSSIAN) {
                        float d = av[a] - bv[b];
                        acc[a][b] = fmaf(d, d, acc[a][b]);
                    } else {
                        acc[a][b] = fmaf(av[a], bv[b], acc[a][b]);
                    }
                }
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        int64_t gi = i0 + ty + 16 * a;
        if (gi >= m) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            int64_t gj = j0 + tx + 16 * b;
            if (gj >= m2) continue;
            float v = acc[a][b];
            if (KIND == GVT_BASE_GAUSSIAN) {
                v = expf(-gamma * v);
            } else if (KIND == GVT_BASE_POLY) {
                float base = fmaf(gamma, v, coef0), r = 1.f;
                for (int e = 0; e < degree; e++) r *= base;
                v = r;
            }
            K[gi * ldk + gj] = v;
        }
    }
}

// K (m x m2) = k(X_i, Y_j); Y == nullptr: the Gram of X
void gram_simt(gvt_ctx *c, int kind, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, int64_t ldx,
               double gamma, double coef0, int degree, float *K, int64_t ldk) {
    if (m == 0 || m2 == 0) return;
    if (!Y) Y = X;
    dim3 grid((unsigned)((m2 + 63) / 64), (unsigned)((m + 63) / 64));
    if (kind == GVT_BASE_GAUSSIAN)
        GVT_LAUNCH(c, K_GRAM_SIMT, k_gram_simt<GVT_BASE_GAUSSIAN>, grid, 256, 0, X, m, Y, m2, dim, ldx, (float)gamma,
                   (float)coef0, degree, K, ldk);
    else if (kind == GVT_BASE_POLY)
        GVT_LAUNCH(c, K_GRAM_SIMT, k_gram_simt<GVT_BASE_POLY>, grid, 256, 0, X, m, Y, m2, dim, ldx, (float)gamma,
                   (float)coef0, degree, K, ldk);
    else
        GVT_LAUNCH(c, K_GRAM_SIMT, k_gram_simt<GVT_BASE_LINEAR>, grid, 256, 0, X, m, Y, m2, dim, ldx, (float)gamma,
                   (float)coef0, degree, K, ldk);
}

// ----------------------------------------------------------------------------- Tanimoto
// k(v, w) = |v AND w| / |v OR w| on binary features (1 for two all-zero vectors,
// reading T1).  The 0/1 features are bit-packed once (warp ballots, 32 features per word, with
// per-row popcounts), then the Gram is a popcount contraction: c_ij = sum_w popc(a_iw & b_jw),
// |v OR w| = n_i + n_j - c_ij.  All counts are exact integers; one fp32 division per entry.
// SIMT: the AND/POPC work per entry is dim/32 words (ALU-bound; computed once per fit).

// warp per row: word w of row r = ballot(X[r][32 w + lane] != 0); counts bits and non-binary entries
__global__ void k_pack_bits(const float *__restrict__ X, int64_t m, int64_t dim, int64_t W, uint32_t *__restrict__ B,
                            int *__restrict__ nbits, unsigned long long *__restrict__ bad) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < m; r += warps) {
        int cnt = 0;
        unsigned nbad = 0;
        for (int64_t w = 0; w < W; w++) {
            const int64_t k = w * 32 + lane;
            const float x = k < dim ? X[r * dim + k] : 0.f;
            nbad += (x != 0.f && x != 1.f) ? 1u : 0u;
            const uint32_t word = __ballot_sync(0xffffffffu, x != 0.f);
            if (lane == 0) B[r * W + w] = word;
            cnt += __popc(word);
        }
        for (int o = 16; o > 0; o >>= 1) nbad += __shfl_xor_sync(0xffffffffu, nbad, o);
        if (lane == 0) {
            nbits[r] = cnt;
            if (nbad) atomicAdd(bad, (unsigned long long)nbad);
        }
    }
}

// 64 x 64 output tile per 256-thread CTA, 4 x 4 per thread, 16-word K chunks of both tables in smem
__global__ void __launch_bounds__(256) k_gram_tanimoto(const uint32_t *__restrict__ A, const int *__restrict__ na,
                                                       int64_t m, const uint32_t *__restrict__ Bm,
                                                       const int *__restrict__ nb, int64_t m2, int64_t W,
                                                       float *__restrict__ K, int64_t ldk) {
    constexpr int BT = 64, BK = 16;
    __shared__ uint32_t xa[BK][BT + 1];
    __shared__ uint32_t xb[BK][BT + 1];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int64_t i0 = (int64_t)blockIdx.y * BT, j0 = (int64_t)blockIdx.x * BT;
    int acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b] = 0;
    for (int64_t k0 = 0; k0 < W; k0 += BK) {
        for (int e = threadIdx.x; e < BT * BK; e += 256) {
            const int r = e / BK, kk = e % BK;
            const int64_t gi = i0 + r, gj = j0 + r, gk = k0 + kk;
            xa[kk][r] = (gi < m && gk < W) ? A[gi * W + gk] : 0u;
            xb[kk][r] = (gj < m2 && gk < W) ? Bm[gj * W + gk] : 0u;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; kk++) {
            uint32_t av[4], bv[4];
#pragma unroll
            for (int a = 0; a < 4; a++) av[a] = xa[kk][ty + 16 * a];
#pragma unroll
            for (int b = 0; b < 4; b++) bv[b] = xb[kk][tx + 16 * b];
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b] += __popc(av[a] & bv[b]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int a = 0; a < 4; a++) {
        const int64_t gi = i0 + ty + 16 * a;
        if (gi >= m) continue;
#pragma unroll
        for (int b = 0; b < 4; b++) {
            const int64_t gj = j0 + tx + 16 * b;
            if (gj >= m2) continue;
            const int c = acc[a][b], u = na[gi] + nb[gj] - c;
            K[gi * ldk + gj] = u > 0 ? (float)c / (float)u : 1.f;
        }
    }
}

// K (m x m2) Tanimoto Gram of 0/1 features X (m x dim) and Y (m2 x dim; nullptr = X)
void gram_tanimoto(gvt_ctx *c, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, float *K,
                   int64_t ldk) {
    if (m == 0 || m2 == 0) return;
    const int64_t W = (dim + 31) / 32 > 0 ? (dim + 31) / 32 : 1;
    uint32_t *bx = wsT<uint32_t>(c, "tan.bx", (size_t)m * W);
    int *nx = wsT<int>(c, "tan.nx", (size_t)m);
    unsigned long long *bad = wsT<unsigned long long>(c, "tan.bad", 1);
    GVT_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(unsigned long long), c->stream));
    GVT_LAUNCH(c, K_GRAM_SIMT, k_pack_bits, grid1d(m * 32, 256, (int64_t)c->sm_count * 16), 256, 0, X, m, dim, W, bx,
               nx, bad);
    const uint32_t *by = bx;
    const int *ny = nx;
    if (Y) {
        uint32_t *b2 = wsT<uint32_t>(c, "tan.by", (size_t)m2 * W);
        int *n2 = wsT<int>(c, "tan.ny", (size_t)m2);
        GVT_LAUNCH(c, K_GRAM_SIMT, k_pack_bits, grid1d(m2 * 32, 256, (int64_t)c->sm_count * 16), 256, 0, Y, m2, dim, W,
                   b2, n2, bad);
        by = b2;
        ny = n2;
    }
    unsigned long long hbad = 0;  // validation before the Gram (SPEC: "errors: non-binary entry")
    GVT_CUDA_TRY(cudaMemcpyAsync(&hbad, bad, sizeof(hbad), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    GVT_REQUIRE(hbad == 0, GVT_E_PARAM, "Tanimoto base kernel needs binary (0/1) features: " + std::to_string(hbad) +
                                           " other entries");
    dim3 grid((unsigned)((m2 + 63) / 64), (unsigned)((m + 63) / 64));
    GVT_LAUNCH(c, K_GRAM_SIMT, k_gram_tanimoto, grid, 256, 0, bx, nx, m, by, ny, m2, W, K, ldk);
}

}  // namespace gvt
