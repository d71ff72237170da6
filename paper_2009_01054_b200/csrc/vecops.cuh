// vecops.cuh -- deterministic reduction helpers shared by the solver vector kernels
// (cg.cu, solver.cu): a fixed contiguous partition of the vector over RED_BLOCKS blocks and a
// fixed shuffle tree per block, so every fp64 partial -- and the scalar reduced from the
// partials in a fixed order -- is bit-identical run to run (reading S26).
#pragma once
#include "ops.cuh"

namespace gvt {

__device__ __forceinline__ double block_sum(double v) {
    __shared__ double sh[RED_THREADS / 32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x < 32) {
        r = threadIdx.x < RED_THREADS / 32 ? sh[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(0xffffffffu, r, o);
    }
    __syncthreads();
    return r;  // valid in thread 0
}

__device__ __forceinline__ bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// element range of block b for a fixed-order partition: block b owns a contiguous range
// (so each partial sums a fixed set of elements in a fixed order)
__device__ __forceinline__ void block_range(int64_t n, int64_t &lo, int64_t &hi) {
    const int64_t per = (((n + gridDim.x - 1) / gridDim.x) + 3) & ~int64_t(3);
    lo = (int64_t)blockIdx.x * per;
    hi = lo + per < n ? lo + per : n;
    if (lo > n) lo = n;
}

__device__ __forceinline__ double reduce_parts(const double *__restrict__ part, int nparts) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += part[i];
    return block_sum(acc);
}


// "Last block done" (threadfence reduction): after each block has written its partial (thread 0),
// returns true in the one block that finishes last; that block then reduces the partials of all
// blocks with reduce_parts_cg -- the same fixed-order tree as a separate single-block kernel, so the
// scalar is bit-identical -- and resets *ticket to 0 for the next launch.  Single-GPU only (across
// ranks the partials must be all-gathered between the two steps).
__device__ __forceinline__ bool last_block_done(unsigned *ticket) {
    __shared__ bool last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (last) __threadfence();
    return last;
}

// reduce_parts over partials written by other blocks of the same grid (L2 reads, no stale L1)
__device__ __forceinline__ double reduce_parts_cg(const double *part, int nparts) {
    double acc = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) acc += __ldcg(part + i);
    return block_sum(acc);
}

// partial-sum slots [world][RED_BLOCKS] (cg.cu); this rank writes slot `rank`
double *solver_parts(gvt_ctx *c);

}  // namespace gvt
