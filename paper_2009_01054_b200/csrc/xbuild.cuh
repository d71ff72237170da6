// xbuild.cuh -- one row of the fp16 pair matrix X(p) built by one warp (Corollary PAPER.md:634-653:
// X's cell (h, col) is the sum of sign * p[src] over the cell's run of entries, in entry order),
// shared by k_build_x16_warp (dense_tc.cu) and the fused dense-engine CG tail (tail.cu).
// The row is parked in shared memory, its max gives a power-of-two scale (stored inverted in
// sinv[r]), then the scaled row is written as fp16 hi/lo pieces (v = hi + lo to ~22 bits) with
// 16-byte stores.  ld is a multiple of 32 (whole rows, padding columns zero).
// LDCG: p was written by other CTAs earlier in the same launch (read through L2).
// r_lazy (fused CG tail): the entries' values are the NEXT direction formed on the fly,
// fmaf(beta, p[src], r_lazy[src]) -- the arithmetic of k_cg_p -- so X(p_{k+1}) is built while
// p_{k+1} itself is still being written elsewhere.
#pragma once
#include <cuda_fp16.h>

#include "cgops.cuh"

namespace gvt {

template <bool LDCG>
__device__ __forceinline__ void x16_row_warp(int64_t r, int lane, float *__restrict__ rowbuf,
                                             const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                             const int32_t *__restrict__ src, const float *__restrict__ sign,
                                             const float *__restrict__ p, int64_t row_lo, int64_t ld,
                                             __half *__restrict__ hi, __half *__restrict__ lo,
                                             float *__restrict__ sinv, const float *__restrict__ diag,
                                             const float *__restrict__ r_lazy = nullptr, float beta = 0.f) {
    auto pv = [&](int64_t k) -> float {
        const int32_t j = src[k];
        if constexpr (LDCG) {
            if (r_lazy) return fmaf(beta, __ldcg(p + j), __ldcg(r_lazy + j));
            return __ldcg(p + j);
        } else {
            return __ldg(p + j);
        }
    };
    float4 *rb4 = reinterpret_cast<float4 *>(rowbuf);
    for (int64_t j = lane; j < ld / 4; j += 32) rb4[j] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    const int64_t kb = row_ptr[row_lo + r], ke = row_ptr[row_lo + r + 1];
#ifndef XB_U
#define XB_U 4
#endif
    constexpr int U = XB_U;  // entries in flight per lane (A/B: -DXB_U=8)
    for (int64_t k0 = kb + lane; k0 < ke; k0 += U * 32) {
        int32_t cc[U], cprev[U], cnext[U];
        float v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t k = k0 + (int64_t)u * 32;
            cc[u] = -1;
            if (k < ke) {
                cc[u] = col[k];
                cprev[u] = k > kb ? col[k - 1] : -1;
                cnext[u] = k + 1 < ke ? col[k + 1] : -1;
                v[u] = sign[k] * pv(k);
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (cc[u] < 0 || cprev[u] == cc[u]) continue;  // past the row end, or not the head of its run
            float sv = v[u];
            if (cnext[u] == cc[u]) {
                const int64_t k = k0 + (int64_t)u * 32;
                for (int64_t j = k + 1; j < ke && col[j] == cc[u]; j++) sv += sign[j] * pv(j);
            }
            rowbuf[cc[u]] = sv;
        }
    }
    __syncwarp();
    if (diag && lane == 0) rowbuf[row_lo + r] += diag[row_lo + r];  // separate diagonal (MLPK)
    __syncwarp();
    float mx = 0.f;
    for (int64_t j = lane; j < ld / 4; j += 32) {
        const float4 v4 = rb4[j];
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v4.x), fabsf(v4.y)), fmaxf(fabsf(v4.z), fabsf(v4.w))));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    int e = 0;
    if (mx > 0.f && isfinite(mx)) {
        int ex;
        frexpf(mx, &ex);
        e = 15 - ex;
    }
    const float sc = ldexpf(1.f, e);
    if (lane == 0) sinv[r] = ldexpf(1.f, -e);
    // 8 columns per lane per step: two float4 reads of the parked row, one 16-byte store per piece
    uint4 *h8 = reinterpret_cast<uint4 *>(hi + r * ld), *l8 = reinterpret_cast<uint4 *>(lo + r * ld);
    for (int64_t j = lane; j < ld / 8; j += 32) {
        const float4 a4 = rb4[2 * j], b4 = rb4[2 * j + 1];
        const float v[8] = {a4.x * sc, a4.y * sc, a4.z * sc, a4.w * sc, b4.x * sc, b4.y * sc, b4.z * sc, b4.w * sc};
        __half2 hh[4], ll[4];
#pragma unroll
        for (int t = 0; t < 4; t++) {
            const __half a0 = __float2half_rn(v[2 * t]), a1 = __float2half_rn(v[2 * t + 1]);
            hh[t] = __halves2half2(a0, a1);
            ll[t] = __halves2half2(__float2half_rn(v[2 * t] - __half2float(a0)),
                                   __float2half_rn(v[2 * t + 1] - __half2float(a1)));
        }
        h8[j] = *reinterpret_cast<const uint4 *>(hh);
        l8[j] = *reinterpret_cast<const uint4 *>(ll);
    }
    __syncwarp();
}

}  // namespace gvt
