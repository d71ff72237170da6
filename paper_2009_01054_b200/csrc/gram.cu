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

}  // namespace gvt
