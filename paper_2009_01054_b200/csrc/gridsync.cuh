// gridsync.cuh -- grid-wide barrier for persistent kernels whose CTAs are all co-resident
// (cooperative launch): the persistent small solver (small.cu) and the fused dense-engine CG tail
// (tail.cu).  The generation word bar[0] only grows; a kernel that is launched repeatedly without
// re-zeroing the words starts its local generation from bar[0] (read before its first arrival:
// no CTA can bump it before every CTA has arrived).
#pragma once
#include <stdint.h>

namespace gvt {

// grid-wide barrier of the co-resident CTAs (cooperative launch), two-level: CTAs arrive on their
// group's counter (16 CTAs per group, one 128-byte line each), the last of a group arrives on the
// top counter, the last group bumps the generation, which the waiting CTAs poll with acquire loads
// and a short sleep.  bar: [0] generation, [32] top counter, [64 + 32 g] group counters.
constexpr int BAR_GROUP = 16;
constexpr int BAR_WORDS = 64 + 32 * 64;  // up to 64 groups (1024 CTAs)

// mode (GVT_SMALL_BAR, experiments): bit 0 = two-level arrival, bit 1 = sleep while polling
__device__ __forceinline__ void grid_sync(unsigned *bar, unsigned &gen, int mode) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g = gen;
        unsigned *top = bar + 32;
        bool released = false;
        if (mode & 1) {
            const unsigned grp = blockIdx.x / BAR_GROUP, ngrp = (gridDim.x + BAR_GROUP - 1) / BAR_GROUP;
            const unsigned gsize = min((unsigned)BAR_GROUP, gridDim.x - grp * BAR_GROUP);
            unsigned *gc = bar + 64 + 32 * grp;
            __threadfence();
            if (atomicAdd(gc, 1u) == gsize - 1) {
                atomicExch(gc, 0u);
                if (atomicAdd(top, 1u) == ngrp - 1) {
                    atomicExch(top, 0u);
                    __threadfence();
                    atomicAdd(bar, 1u);
                    released = true;
                }
            }
        } else {
            unsigned old;
            asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(top) : "memory");
            if (old == gridDim.x - 1) {
                *reinterpret_cast<volatile unsigned *>(top) = 0u;
                asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(bar) : "memory");
                released = true;
            }
        }
        if (!released) {
            unsigned v;
            while (true) {
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar) : "memory");
                if (v != g) break;
                if (mode & 2) __nanosleep(20);
            }
        }
    }
    gen++;
    __syncthreads();
}

}  // namespace gvt
