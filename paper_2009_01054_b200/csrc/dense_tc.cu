// dense_tc.cu -- dense tensor-core engine on sm_100a.  C = A B^T with fp32-accurate
// results from 3 low-precision tensor-core products (hi*hi + hi*lo + lo*hi):
//   PREC_F16  (default) kind::f16: every operand row is scaled by a power of two so its
//             largest entry sits just below 2^15, then split hi = fp16(x), lo = fp16(x - hi)
//             (22 significant bits); 2x the MAC rate of TF32 at half the bytes.
//   PREC_TF32 kind::tf32: hi = rna_tf32(x), lo = rna_tf32(x - hi), no scaling.
// Operands are staged by TMA (SWIZZLE_128B, K-major, 128-byte rows = 64 fp16 / 32 tf32)
// through an mbarrier ring; one elected thread issues the MMAs; accumulators live in TMEM.
//
// Precision: the tensor core truncates every accumulation into its fp32 accumulator, a
// bias that grows with K.  The kernel therefore accumulates K in chunks (fresh accumulator
// per chunk, double-buffered in TMEM: 2 x 256 columns) and the epilogue warps add the
// chunk results into fp32 registers with round-to-nearest while the MMA warp works on the
// next chunk.  Row scales are exact powers of two, undone in the epilogue.
//
// One kernel, three epilogues:
//   EPI_STORE   C stored fp32 (+ optional tf32 hi/lo)   -> GVT stage 1, S = C_fac X^T
//   EPI_SAMPLED out[dst] (+)= coef (A B^T)[r, c] for the samples bucketed on this tile
//               -> GVT stage 2 (sampled D S^T, north-star kernel (3), dense-tile form)
//   EPI_GRAM    K = k(X_i, X_j) from the dot product and row norms -> base-kernel Gram,
//               north-star kernel (1)
// Tile 128 x 256, 128-byte K-blocks, 2-stage ring of 96 KB, grouped rasterization.
// Warps: 0 TMA producer, 1 MMA issuer (+ TMEM owner), 2..9 epilogue (warp w reads TMEM
// lanes 32*(w%4).. and columns 128*((w-2)/4)..).
#include <cuda.h>
#include <cuda_fp16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <vector>
#include <stdio.h>
#include <stdlib.h>

#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>

#include "ops.cuh"
#include "xbuild.cuh"

namespace gvt {

// ----------------------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait's suspend-time hint: a waiting thread may sleep up to this long (it resumes when the
// phase completes) instead of re-polling (experiment: GVT energy under the power cap)
#ifndef MBAR_SUSPEND_NS
#define MBAR_SUSPEND_NS 1000000
#endif
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    uint32_t addr = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(addr),
        "r"(parity), "r"(MBAR_SUSPEND_NS)
        : "memory");
}

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap *map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// bytes of K per smem row (one swizzle atom row): 64 -> SWIZZLE_64B atoms, 4-stage ring of 48 KB
constexpr int KB_BYTES = 128;

// K-major canonical swizzled layout: 8-row x KB_BYTES atoms, SBO = 8 rows * KB_BYTES, LBO = 16 B
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                                        // LBO (unused for swizzled K-major)
    d |= (uint64_t)((8 * KB_BYTES) >> 4) << 32;                    // SBO
    d |= (uint64_t)1 << 46;                                        // version (sm_100)
    d |= (uint64_t)(KB_BYTES == 128 ? 2 : (KB_BYTES == 64 ? 4 : 6)) << 61;  // SWIZZLE_128B / 64B / 32B
    return d;
}

enum { PREC_F16 = 0, PREC_TF32 = 1 };

// instruction descriptor: D f32, A/B tf32 (format 2) or f16 (format 0), K-major both, M = 128
template <int PREC, int N>
__host__ __device__ constexpr uint32_t idesc_mma() {
    return (1u << 4) | ((PREC == PREC_TF32 ? 2u : 0u) << 7) | ((PREC == PREC_TF32 ? 2u : 0u) << 10) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
}

template <int PREC>
__device__ __forceinline__ void mma_issue(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    if (PREC == PREC_TF32) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32_raw(uint32_t taddr, uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld16_raw(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld8_raw(uint32_t taddr, uint32_t (&r)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
}

__device__ __forceinline__ void tmem_ld4_raw(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}

__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float tf32_round(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n)); }

// ----------------------------------------------------------------------------- kernel
enum { EPI_STORE = 0, EPI_SAMPLED = 1, EPI_GRAM = 2, EPI_STORE16 = 3 };

struct EpiParams {
    // store
    float *c_f;                // fp32 C (ldc)
    float *c_hi, *c_lo;        // optional tf32 split of C (ldc)
    int64_t ldc;
    // operand row scales (inverse powers of two), nullable
    const float *sa, *sb;
    // sampled
    const int32_t *s_r, *s_c, *s_dst;
    const int64_t *chunk_ptr;  // per (tile, 32-column chunk)
    int64_t n_ct;              // column tiles
    float coef;
    int accumulate;
    float *out;
    // gram: row norms of A (norms) and of B (norms_b); same = the Gram of one table (diagonal
    // exactly 1 for the Gaussian)
    const float *norms, *norms_b;
    int same;
    int kind;
    float gamma, coef0;
    int degree;
    int kcb;  // k-blocks per accumulation chunk (0 = KC_BLOCKS)
    int group_m;  // CTA-pair kernel: pair-tile rows per rasterization group (0 = GROUP_M)
    // CTA-pair kernel, optional block sparsity of the B operand: for column tile n (BN rows of B),
    // only the K-blocks kb_list[kb_off[n] .. kb_off[n + 1]) (ascending, at least one) are
    // multiplied; the other K-blocks of those B rows are all zero (EPI_STORE16 only)
    const int32_t *kb_list, *kb_off;
    // B operand with a per-(row block, 256-wide K chunk) scale, applied while draining chunk ch:
    // sbk[ch * sbk_ld + n / S16_SCALE_ROWS] (fp16 S produced by EPI_STORE16)
    const float *sbk;
    int64_t sbk_ld;
    // EPI_STORE16: C as fp16 hi/lo (ldc) with one scale per (row block, 256-column tile):
    // c_sk[n_tile * c_sk_ld + row / S16_SCALE_ROWS] = 1/scale
    __half *c_h16, *c_l16;
    float *c_sk;
    int64_t c_sk_ld;
    // sampled split-K (CTA-pair kernel): units = (non-empty pair tile, K part); tile_list holds the pair
    // tiles (mp * n_ct + n), each split over `split` contiguous chunk ranges; part[ks * ns + k] receives
    // sample k's value over K part ks (k_split_combine sums the parts)
    // Tail split (n_whole > 0): the first n_whole listed tiles are whole units served directly, only the
    // remaining tiles of the list are split (the last, partial wave of a persistent loop spread over the pairs)
    const int32_t *tile_list;
    int split, n_units, n_whole;
    float *part;
    int64_t ns;
    // diagnosis (GVT_GEMM_PROF): per CTA, globaltimer stamps [entry, setup done, first stage landed,
    // last MMA commit, last TMA issued, last chunk drained, epilogue done, -]
    unsigned long long *prof;
};

__device__ __forceinline__ unsigned long long gemm_timer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define GEMM_MARK(slot) \
    if (ep.prof) ep.prof[blockIdx.x * 16 + (slot)] = gemm_timer();

#ifndef DRAIN_X16
#define DRAIN_X16 1
#endif
#ifndef SERVE_UNROLL
#define SERVE_UNROLL 1
#endif
#ifndef SERVE_PREFETCH
#define SERVE_PREFETCH 1
#endif
template <int STRIDE>  // the epilogue threads serving (32 x epilogue warps)
__device__ __forceinline__ void serve_samples(const EpiParams &ep, int64_t kb0, int64_t ke, int t, int m0, int gc0,
                                              const float *stage, float *part) {
#ifdef GVT_TIMING_SKIP_SERVE  // timing-only A/B build (results wrong): the multi-unit serve skipped
    return;
#endif
    if (part) {  // split-K: this K part's raw value per sample slot (no coefficient, no accumulation)
        for (int64_t k = kb0 + t; k < ke; k += STRIDE) {
            const int rl = ep.s_r[k] - m0, cl = ep.s_c[k] - gc0;
            part[k] = stage[(rl >> 5) * 32 * 33 + (rl & 31) * 33 + cl];
        }
        return;
    }
    constexpr int U = SERVE_UNROLL;
    for (int64_t k0 = kb0 + t; k0 < ke; k0 += U * STRIDE) {
        int rl[U], cl[U];
        int64_t dd[U];
        float prev[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t k = k0 + (int64_t)u * STRIDE;
            if (k < ke) {
                rl[u] = ep.s_r[k] - m0;  // 0..127
                cl[u] = ep.s_c[k] - gc0;  // 0..31
                dd[u] = ep.s_dst[k];
            }
        }
        if (ep.accumulate) {
#pragma unroll
            for (int u = 0; u < U; u++)
                if (k0 + (int64_t)u * STRIDE < ke) prev[u] = ep.out[dd[u]];
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            if (k0 + (int64_t)u * STRIDE < ke) {
                const float val = stage[(rl[u] >> 5) * 32 * 33 + (rl[u] & 31) * 33 + cl[u]];
                ep.out[dd[u]] = ep.accumulate ? fmaf(ep.coef, val, prev[u]) : ep.coef * val;
            }
        }
    }
}


constexpr int BM = 128, BN = 256, STAGES = 256 / KB_BYTES;  // 4 stages of 48 KB (64-byte K-blocks)
constexpr int KC_BLOCKS = 4;                      // k-blocks per accumulation chunk
// the fp16 S of stage 1 carries one scale per 256-column tile; stage 2 drains 256-wide K chunks
static_assert(KC_BLOCKS * (KB_BYTES / 2) == BN, "fp16 accumulation chunk = one S scale tile");
static_assert(S16_SCALE_ROWS == 1 || S16_SCALE_ROWS == BM, "S scale block = one stage-1 CTA's rows");
template <int STRIDE>
__device__ __forceinline__ void serve_tile(const EpiParams &ep, int64_t kb0, int64_t ke, int t, int m0, int n0,
                                           const float *tile_s, float *part) {
    constexpr int U = 4;
    for (int64_t k0 = kb0 + t; k0 < ke; k0 += U * STRIDE) {
        int off[U];
        int64_t dd[U];
        float prev[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t k = k0 + (int64_t)u * STRIDE;
            if (k < ke) {
                off[u] = (ep.s_r[k] - m0) * (BN + 1) + (ep.s_c[k] - n0);
                if (!part) dd[u] = ep.s_dst[k];
            }
        }
        if (!part && ep.accumulate) {
#pragma unroll
            for (int u = 0; u < U; u++)
                if (k0 + (int64_t)u * STRIDE < ke) prev[u] = ep.out[dd[u]];
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int64_t k = k0 + (int64_t)u * STRIDE;
            if (k < ke) {
                const float val = tile_s[off[u]];
                if (part) part[k] = val;
                else ep.out[dd[u]] = ep.accumulate ? fmaf(ep.coef, val, prev[u]) : ep.coef * val;
            }
        }
    }
}

// Sampled epilogue: write the samples k in [kb0, ke) of one 32-column chunk (their values parked
// in `stage`, [rows/32][32][33] floats) to out[dst], SERVE_UNROLL samples per thread in flight.
// Measured (profiles/r01_ab_serve_unroll.txt): 4 in flight cut C2 from 95 to 83 us per iteration
// but raised the CTA-pair kernel's register spills (172 -> 556 B) and C5's stage 2 from 43 to
// 50 ms, so 1 is the default.
template <int STRIDE>
__device__ __forceinline__ void serve_samples(const struct EpiParams &ep, int64_t kb0, int64_t ke, int t, int m0,
                                              int gc0, const float *stage, float *part);
// all samples [kb0, ke) of one M-tile x N-tile from a parked tile (row stride BN + 1): four per thread in
// flight; split-K parts go to part[k], else out[dst] (+)= coef value
template <int STRIDE>
__device__ __forceinline__ void serve_tile(const struct EpiParams &ep, int64_t kb0, int64_t ke, int t, int m0, int n0,
                                           const float *tile_s, float *part);
constexpr int GROUP_M = 16;                       // row-tiles per rasterization group
constexpr int N_EPI_WARPS = 8;
constexpr int NTHREADS = 64 + 32 * N_EPI_WARPS;   // 320
constexpr int A_BYTES = BM * KB_BYTES;            // 16 KB
constexpr int B_BYTES = BN * KB_BYTES;            // 32 KB
constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;  // 96 KB
constexpr int BAR_OFF = STAGES * STAGE_BYTES;
constexpr int SMEM_TOTAL = BAR_OFF + 256 + 1024;        // barriers + tmem slot + alignment slack
static_assert(N_EPI_WARPS * 32 * 33 * 4 <= STAGES * STAGE_BYTES, "epilogue staging aliases the stage ring");

template <int PREC, int EPI>
__global__ void __launch_bounds__(NTHREADS, 1)
    k_gemm_x3(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
              const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl, int M, int N, int K,
              EpiParams ep) {
    constexpr int BKE = KB_BYTES / (PREC == PREC_TF32 ? 4 : 2);  // elements per K-block
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + BAR_OFF);
    uint64_t *empty = full + STAGES;
    uint64_t *tfull = empty + STAGES;   // [2] accumulator buffer ready
    uint64_t *tempty = tfull + 2;       // [2] accumulator buffer drained
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // grouped rasterization: consecutive CTAs sweep GROUP_M row-tiles x a few column-tiles,
    // so the CTAs resident in one wave share their A and B k-slabs through L2
    const int num_m = (M + BM - 1) / BM, num_n = (N + BN - 1) / BN;
    const int pid = blockIdx.x, in_group = GROUP_M * num_n;
    const int first_m = (pid / in_group) * GROUP_M;
    const int group_m = min(num_m - first_m, GROUP_M);
    const int m_tile = first_m + (pid % in_group) % group_m;
    const int n_tile = (pid % in_group) / group_m;
    const int m0 = m_tile * BM, n0 = n_tile * BN;
    const int nk = (K + BKE - 1) / BKE;
    const int kcb = ep.kcb > 0 ? ep.kcb : KC_BLOCKS;
    const int nch = (nk + kcb - 1) / kcb;

    if (EPI == EPI_SAMPLED) {  // a tile that owns no sample computes nothing (uniform exit)
        const int64_t tile = (int64_t)m_tile * ep.n_ct + n_tile;
        if (ep.chunk_ptr[tile * (BN / 32)] == ep.chunk_ptr[(tile + 1) * (BN / 32)]) return;
    }

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmAh);
        prefetch_tmap(&tmAl);
        prefetch_tmap(&tmBh);
        prefetch_tmap(&tmBl);
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], N_EPI_WARPS);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {  // TMEM allocation (whole warp): 2 accumulator buffers x BN fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer
            for (int kb = 0; kb < nk; kb++) {
                const int s = kb % STAGES;
                const uint32_t ph = (kb / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t *st = smem + s * STAGE_BYTES;
                mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
                const int kc = kb * BKE;
                tma_load_2d(st, &tmAh, &full[s], kc, m0);
                tma_load_2d(st + A_BYTES, &tmAl, &full[s], kc, m0);
                tma_load_2d(st + 2 * A_BYTES, &tmBh, &full[s], kc, n0);
                tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tmBl, &full[s], kc, n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---------------- MMA issuer (single thread)
            constexpr uint32_t idesc = idesc_mma<PREC, BN>();
            int kb = 0;
            for (int ch = 0; ch < nch; ch++) {
                const int b = ch & 1;
                mbar_wait(&tempty[b], ((ch >> 1) & 1) ^ 1);  // epilogue drained this buffer
                tc_fence_after();
                const uint32_t acc = tmem + b * BN;
                const int kend = min(nk, kb + kcb);
                for (int kk = 0; kb < kend; kb++, kk++) {
                    const int s = kb % STAGES;
                    const uint32_t ph = (kb / STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    const uint32_t base = smem_u32(smem + s * STAGE_BYTES);
                    const uint32_t ah = base, al = base + A_BYTES, bh = base + 2 * A_BYTES,
                                   bl = base + 2 * A_BYTES + B_BYTES;
#pragma unroll
                    for (int k = 0; k < KB_BYTES / 32; k++) {
                        const uint32_t off = k * 32;  // one MMA K-step = 32 bytes inside the swizzle atom
                        const uint64_t dah = umma_desc(ah + off), dal = umma_desc(al + off);
                        const uint64_t dbh = umma_desc(bh + off), dbl = umma_desc(bl + off);
                        mma_issue<PREC>(acc, dah, dbh, idesc, (kk | k) != 0);
                        mma_issue<PREC>(acc, dah, dbl, idesc, 1);
                        mma_issue<PREC>(acc, dal, dbh, idesc, 1);
                    }
                    mma_commit(&empty[s]);  // frees the smem slot once these MMAs have read it
                }
                mma_commit(&tfull[b]);      // chunk accumulator complete
            }
        }
    } else {  // ---------------- epilogue warps 2..9
        const int ew = warp - 2;
        const int quarter = warp & 3;   // TMEM lane quarter this warp may access
        const int half = ew >> 2;       // column half: [128*half, 128*half + 128)
        const int row = quarter * 32 + lane;
        const int gr = m0 + row;
        float run[128];
#pragma unroll
        for (int i = 0; i < 128; i++) run[i] = 0.f;
        for (int ch = 0; ch < nch; ch++) {
            const int b = ch & 1;
            mbar_wait(&tfull[b], (ch >> 1) & 1);
            tc_fence_after();
            const uint32_t ta = tmem + b * BN + half * 128 + ((uint32_t)(quarter * 32) << 16);
#pragma unroll
            for (int c4 = 0; c4 < 4; c4++) {
                uint32_t r[32];
                tmem_ld32_raw(ta + c4 * 32, r);
                tmem_wait_ld();
#pragma unroll
                for (int i = 0; i < 32; i++) run[c4 * 32 + i] += __uint_as_float(r[i]);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[b]);
        }
        const int gc_base = n0 + half * 128;
        // undo the operand row scales (exact powers of two)
        if (ep.sa || ep.sb) {
            const float ra = (ep.sa && gr < M) ? ep.sa[gr] : 1.f;
#pragma unroll
            for (int i = 0; i < 128; i++) {
                const int gc = gc_base + i;
                const float rb = (ep.sb && gc < N) ? __ldg(ep.sb + gc) : 1.f;
                run[i] *= ra * rb;
            }
        }
        // all MMAs are complete (the last tfull was committed after them), so the stage ring is
        // free and serves as staging memory for the sampled epilogue
        if (EPI == EPI_STORE) {
            if (gr < M) {
                float *cf = ep.c_f + (int64_t)gr * ep.ldc + gc_base;
                if (gc_base + 128 <= N) {
#pragma unroll
                    for (int i = 0; i < 128; i += 4)
                        *reinterpret_cast<float4 *>(cf + i) = make_float4(run[i], run[i + 1], run[i + 2], run[i + 3]);
                    if (ep.c_hi) {
                        float *hi = ep.c_hi + (int64_t)gr * ep.ldc + gc_base;
                        float *lo = ep.c_lo + (int64_t)gr * ep.ldc + gc_base;
#pragma unroll
                        for (int i = 0; i < 128; i += 4) {
                            float4 h, l;
                            h.x = tf32_round(run[i]);     l.x = tf32_round(run[i] - h.x);
                            h.y = tf32_round(run[i + 1]); l.y = tf32_round(run[i + 1] - h.y);
                            h.z = tf32_round(run[i + 2]); l.z = tf32_round(run[i + 2] - h.z);
                            h.w = tf32_round(run[i + 3]); l.w = tf32_round(run[i + 3] - h.w);
                            *reinterpret_cast<float4 *>(hi + i) = h;
                            *reinterpret_cast<float4 *>(lo + i) = l;
                        }
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < 128; i++) {
                        if (gc_base + i < N) {
                            cf[i] = run[i];
                            if (ep.c_hi) {
                                float h = tf32_round(run[i]);
                                ep.c_hi[(int64_t)gr * ep.ldc + gc_base + i] = h;
                                ep.c_lo[(int64_t)gr * ep.ldc + gc_base + i] = tf32_round(run[i] - h);
                            }
                        }
                    }
                }
            }
        } else if (EPI == EPI_GRAM) {
            if (gr < M) {
                float *krow = ep.c_f + (int64_t)gr * ep.ldc;
                const float ni = ep.kind == GVT_BASE_GAUSSIAN ? ep.norms[gr] : 0.f;
#pragma unroll
                for (int i = 0; i < 128; i++) {
                    const int gc = gc_base + i;
                    if (gc < N) {
                        float x = run[i];
                        if (ep.kind == GVT_BASE_GAUSSIAN) {
                            float d2 = fmaxf(ni + ep.norms_b[gc] - 2.f * x, 0.f);
                            if (ep.same && gc == gr) d2 = 0.f;  // k(x, x) = 1 exactly
                            x = expf(-ep.gamma * d2);
                        } else if (ep.kind == GVT_BASE_POLY) {
                            float bb = fmaf(ep.gamma, x, ep.coef0), rr = 1.f;
                            for (int e = 0; e < ep.degree; e++) rr *= bb;
                            x = rr;
                        }
                        krow[gc] = x;
                    }
                }
            }
        } else {  // EPI_SAMPLED: per 32-column chunk pair, park values in smem, serve the samples
            float *stage = reinterpret_cast<float *>(smem);  // [half*4 + quarter][32 rows][33]
            const int t = threadIdx.x - 64;                  // 0..255
            const int64_t tile = (int64_t)m_tile * ep.n_ct + n_tile;
#pragma unroll
            for (int c4 = 0; c4 < 4; c4++) {
                float *mine = stage + (half * 4 + quarter) * 32 * 33 + lane * 33;
#pragma unroll
                for (int i = 0; i < 32; i++) mine[i] = run[c4 * 32 + i];
                named_bar(1, 32 * N_EPI_WARPS);
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const int chunk = hh * 4 + c4;
                    const int64_t cidx = tile * (BN / 32) + chunk;
                    const int64_t kb0 = ep.chunk_ptr[cidx], ke = ep.chunk_ptr[cidx + 1];
                    const int gc0 = n0 + chunk * 32;
                    serve_samples<256>(ep, kb0, ke, t, m0, gc0, stage + hh * 4 * 32 * 33, nullptr);
                }
                named_bar(1, 32 * N_EPI_WARPS);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
    }
}

// ----------------------------------------------------------------------------- 2-CTA variant
// CTA pair (cluster of 2) computes a 256 x 256 tile with tcgen05.mma.cta_group::2 (M = 256):
// each CTA stages its own 128 rows of A and its own 128 rows of B (TMA .cta_group::2, bytes
// completing on the leader's barrier), the leader issues the MMAs that read both CTAs'
// shared memory, each CTA's TMEM holds its 128 accumulator rows.  Per MAC this moves 1/3
// fewer operand bytes than the 1-CTA kernel and leaves room for 3 stages of 64 KB.
constexpr int STAGES2 = 3;
constexpr int HALF_BYTES = 128 * KB_BYTES;               // 16 KB: 128 rows of one operand piece
constexpr int STAGE2_BYTES = 4 * HALF_BYTES;             // A hi/lo + B-half hi/lo = 64 KB per CTA
constexpr int EPI2_OFF = STAGES2 * STAGE2_BYTES;             // dedicated epilogue staging (persistent)
constexpr int EPI2_BYTES = N_EPI_WARPS * 32 * 33 * 4;         // 33 KB
constexpr int BAR2_OFF = EPI2_OFF + EPI2_BYTES;
constexpr int SMEM2_TOTAL = BAR2_OFF + 256 + 1024;
static_assert(SMEM2_TOTAL <= 232448, "exceeds the 227 KB opt-in shared memory per CTA");

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void tma_load_2d_pair(void *dst, const CUtensorMap *map, uint64_t *bar, int c0, int c1) {
    // both CTAs: bytes complete on the leader's barrier (peer bit of the cluster address cleared)
    const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1)
        : "memory");
}

template <int PREC>
__device__ __forceinline__ void mma_issue2(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    if (PREC == PREC_TF32) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
    } else {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "setp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
}

__device__ __forceinline__ void mma_commit_pair(uint64_t *bar) {
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"((uint16_t)0x3)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_leader(uint64_t *bar) {
    uint32_t remote;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(0));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

template <int PREC, int N>
__host__ __device__ constexpr uint32_t idesc_mma2() {
    return (1u << 4) | ((PREC == PREC_TF32 ? 2u : 0u) << 7) | ((PREC == PREC_TF32 ? 2u : 0u) << 10) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
}

// epilogue warps of the sampled (stage-2) CTA-pair kernel: 16 halve each thread's share of the per-chunk
// TMEM drain (64 columns instead of 128, at <= 112 registers), so the drain of one 256-wide K chunk
// finishes well inside the next chunk's MMAs; -DSAMPLED_EPI_WARPS=8 restores the round-1 layout (A/B)
#ifndef SAMPLED_EPI_WARPS
#define SAMPLED_EPI_WARPS 16
#endif
static_assert(SAMPLED_EPI_WARPS == 8 || SAMPLED_EPI_WARPS == 16, "sampled epilogue: 8 or 16 warps");
__host__ __device__ constexpr int pair_epi_warps(int epi) { return epi == EPI_SAMPLED ? SAMPLED_EPI_WARPS : N_EPI_WARPS; }
// Register reallocation (setmaxnreg) in the sampled kernel: warpgroup 0 = TMA producer, MMA issuer and two idle
// warps gives registers back (SAMPLED_REG_LO), the four epilogue warpgroups take them (SAMPLED_REG_HI).  The
// pool is the CTA's launch allocation (20 warps x 96 registers), so 4 x 32 x LO + 16 x 32 x HI must not exceed
// 640 x 96 -- an over-subscribed setmaxnreg.inc never returns.  The epilogue's 64 accumulators then stay in
// registers through the drain.  Measured (profiles/r02_ab_regrealloc.txt): the stage-2 GEMM does the same
// work in fewer clocks but the clock drops under the power cap and the C5 fit gets 2-4 % slower, so the
// default is 0: 18 warps at 96 registers (-DSAMPLED_REGREALLOC=1 builds the reallocation layout).
#ifndef SAMPLED_REGREALLOC
#define SAMPLED_REGREALLOC 0
#endif
#define SAMPLED_REG_LO 32
#define SAMPLED_REG_HI 112
static_assert(4 * 32 * SAMPLED_REG_LO + 16 * 32 * SAMPLED_REG_HI <= 640 * 96, "setmaxnreg pool over-subscribed");
__host__ __device__ constexpr int pair_epi_first_warp(int epi) {
    return (epi == EPI_SAMPLED && SAMPLED_REGREALLOC) ? 4 : 2;
}
__host__ __device__ constexpr int pair_threads(int epi) { return 32 * pair_epi_first_warp(epi) + 32 * pair_epi_warps(epi); }

template <int PREC, int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(pair_threads(EPI), 1)
    k_gemm2_x3(const __grid_constant__ CUtensorMap tmAh, const __grid_constant__ CUtensorMap tmAl,
               const __grid_constant__ CUtensorMap tmBh, const __grid_constant__ CUtensorMap tmBl, int M, int N, int K,
               EpiParams ep) {
    // Persistent: each CTA pair loops over pair tiles (256 x 256) t = cluster, cluster + #clusters, ...
    // The smem ring position, the accumulator-chunk parity and the skip decisions advance
    // identically in the producer, MMA and epilogue roles of both CTAs, so a tile's output
    // phase overlaps the next tile's MMAs.
    if (threadIdx.x == 0) { GEMM_MARK(0) }
    constexpr int BKE = KB_BYTES / (PREC == PREC_TF32 ? 4 : 2);
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    float *estage = reinterpret_cast<float *>(smem + EPI2_OFF);
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + BAR2_OFF);
    uint64_t *empty = full + STAGES2;
    uint64_t *tfull = empty + STAGES2;
    uint64_t *tempty = tfull + 2;
    uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t crank = cluster_rank();
    const int num_m = (M + BM - 1) / BM;
    const int num_mp = (M + 2 * BM - 1) / (2 * BM), num_n = (N + BN - 1) / BN;
    const int n_tiles = num_mp * num_n;
    const int cluster = blockIdx.x >> 1, n_clusters = gridDim.x >> 1;
    const int nk = (K + BKE - 1) / BKE;
    const int kcb = ep.kcb > 0 ? ep.kcb : KC_BLOCKS;
    // K-blocks of column tile n: all of them, or the tile's list of non-zero K-blocks of B
    auto tile_nk = [&](int n) -> int { return ep.kb_list ? ep.kb_off[n + 1] - ep.kb_off[n] : nk; };
    auto tile_kb = [&](int n, int i) -> int { return ep.kb_list ? ep.kb_list[ep.kb_off[n] + i] : i; };
    const int gm = ep.group_m > 0 ? ep.group_m : GROUP_M;
    const int in_group = gm * num_n;

    // grouped rasterization of pair tiles; a sampled tile pair without samples is skipped
    auto coords = [&](int t, int &mp_tile, int &n_tile) {
        const int first_m = (t / in_group) * gm;
        const int group_m = min(num_mp - first_m, gm);
        mp_tile = first_m + (t % in_group) % group_m;
        n_tile = (t % in_group) / group_m;
    };
    auto skip = [&](int mp_tile, int n_tile) -> bool {
        if (EPI != EPI_SAMPLED) return false;
        const int64_t t0 = (int64_t)(2 * mp_tile) * ep.n_ct + n_tile, t1 = t0 + ep.n_ct;
        const bool e0 = ep.chunk_ptr[t0 * (BN / 32)] == ep.chunk_ptr[(t0 + 1) * (BN / 32)];
        const bool e1 = !(2 * mp_tile + 1 < num_m) || ep.chunk_ptr[t1 * (BN / 32)] == ep.chunk_ptr[(t1 + 1) * (BN / 32)];
        return e0 && e1;
    };
    // work units: all pair tiles (empty sampled tiles skipped), or (sampled split-K) the listed non-empty
    // pair tiles x `split` K parts; [c0, c1) = the unit's accumulation chunks
    const int n_units = ((EPI == EPI_SAMPLED && ep.tile_list) || (EPI == EPI_STORE16 && ep.n_whole > 0)) ? ep.n_units
                                                                                                          : n_tiles;
    auto unit = [&](int t, int &mp_tile, int &n_tile, int &c0, int &c1) -> bool {
        if (EPI == EPI_SAMPLED && ep.tile_list) {
            const bool whole = t < ep.n_whole;
            const int u = t - ep.n_whole, sp = whole ? 1 : ep.split;
            const int tl = whole ? ep.tile_list[t] : ep.tile_list[ep.n_whole + u / sp], ks = whole ? 0 : u % sp;
            mp_tile = tl / num_n;
            n_tile = tl % num_n;
            const int nch = (tile_nk(n_tile) + kcb - 1) / kcb;
            c0 = nch * ks / sp;
            c1 = nch * (ks + 1) / sp;
            return true;
        }
        // (EPI_STORE16 with a tile order: tile_list[i] = mp * num_n + n replaces the grouped order)
        auto store_coords = [&](int i, int &mt, int &nt) {
            if (EPI == EPI_STORE16 && ep.tile_list) {
                const int tl = ep.tile_list[i];
                mt = tl / num_n;
                nt = tl % num_n;
            } else {
                coords(i, mt, nt);
            }
        };
        if (EPI == EPI_STORE16 && ep.n_whole > 0 && t >= ep.n_whole) {  // tail split: the last tiles in parts
            const int u = t - ep.n_whole, ks = u % ep.split;
            store_coords(ep.n_whole + u / ep.split, mp_tile, n_tile);
            const int nch = (tile_nk(n_tile) + kcb - 1) / kcb;
            c0 = nch * ks / ep.split;
            c1 = nch * (ks + 1) / ep.split;
            return true;
        }
        store_coords(t, mp_tile, n_tile);
        if (skip(mp_tile, n_tile)) return false;
        c0 = 0;
        c1 = (tile_nk(n_tile) + kcb - 1) / kcb;
        return true;
    };

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmAh);
        prefetch_tmap(&tmAl);
        prefetch_tmap(&tmBh);
        prefetch_tmap(&tmBl);
        for (int s = 0; s < STAGES2; s++) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], 2 * pair_epi_warps(EPI));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 1) {  // TMEM: both CTAs, same warp, same slot offset
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    tc_fence_before();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) { GEMM_MARK(1) }
    constexpr int EW0 = pair_epi_first_warp(EPI);  // first epilogue warp

    if (warp < EW0) {  // ---------------- warpgroup 0 (register reallocation) / warps 0, 1
    if constexpr (EW0 == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(SAMPLED_REG_LO));
    if (warp == 0) {
        if (lane == 0) {  // ---------------- TMA producer (both CTAs)
            int kg = 0;  // global k-block counter = ring position
            for (int t = cluster; t < n_units; t += n_clusters) {
                int mp_tile, n_tile, c0, c1;
                if (!unit(t, mp_tile, n_tile, c0, c1)) continue;
                const int m0 = (2 * mp_tile + (int)crank) * BM, n0 = n_tile * BN;
                const int nk_t = min(tile_nk(n_tile), c1 * kcb);
                for (int kb = c0 * kcb; kb < nk_t; kb++, kg++) {
                    const int s = kg % STAGES2;
                    const uint32_t ph = (kg / STAGES2) & 1;
                    mbar_wait(&empty[s], ph ^ 1);  // own slot released by the leader's MMA commit
                    uint8_t *st = smem + s * STAGE2_BYTES;
                    if (crank == 0) mbar_arrive_expect_tx(&full[s], 2 * STAGE2_BYTES);
                    const int kc = tile_kb(n_tile, kb) * BKE;
                    tma_load_2d_pair(st, &tmAh, &full[s], kc, m0);
                    tma_load_2d_pair(st + HALF_BYTES, &tmAl, &full[s], kc, m0);
                    tma_load_2d_pair(st + 2 * HALF_BYTES, &tmBh, &full[s], kc, n0 + (int)crank * 128);
                    tma_load_2d_pair(st + 3 * HALF_BYTES, &tmBl, &full[s], kc, n0 + (int)crank * 128);
                }
            }
            GEMM_MARK(4)
        }
    } else if (warp == 1) {
        if (lane == 0 && crank == 0) {  // ---------------- MMA issuer (leader only)
            constexpr uint32_t idesc = idesc_mma2<PREC, BN>();
            int kg = 0, cg = 0;
            for (int t = cluster; t < n_units; t += n_clusters) {
                int mp_tile, n_tile, c0, c1;
                if (!unit(t, mp_tile, n_tile, c0, c1)) continue;
                int kb = c0 * kcb;
                const int nk_t = tile_nk(n_tile);
                for (int ch = c0; ch < c1; ch++, cg++) {
                    const int b = cg & 1;
                    mbar_wait(&tempty[b], ((cg >> 1) & 1) ^ 1);
                    tc_fence_after();
                    const uint32_t acc = tmem + b * BN;
                    const int kend = min(nk_t, kb + kcb);
                    for (int kk = 0; kb < kend; kb++, kk++, kg++) {
                        const int s = kg % STAGES2;
                        const uint32_t ph = (kg / STAGES2) & 1;
                        mbar_wait(&full[s], ph);
                        tc_fence_after();
                        if (kg == 0) { GEMM_MARK(2) }
                        const uint32_t base = smem_u32(smem + s * STAGE2_BYTES);
                        const uint32_t ah = base, al = base + HALF_BYTES, bh = base + 2 * HALF_BYTES,
                                       bl = base + 3 * HALF_BYTES;
#pragma unroll
                        for (int k = 0; k < KB_BYTES / 32; k++) {
                            const uint32_t off = k * 32;
                            const uint64_t dah = umma_desc(ah + off), dal = umma_desc(al + off);
                            const uint64_t dbh = umma_desc(bh + off), dbl = umma_desc(bl + off);
                            mma_issue2<PREC>(acc, dah, dbh, idesc, (kk | k) != 0);
                            mma_issue2<PREC>(acc, dah, dbl, idesc, 1);
                            mma_issue2<PREC>(acc, dal, dbh, idesc, 1);
                        }
                        mma_commit_pair(&empty[s]);  // frees the slot in both CTAs
                    }
                    mma_commit_pair(&tfull[b]);      // chunk accumulator ready in both CTAs
                }
            }
            GEMM_MARK(3)
        }
    }  // (warps 2, 3 of the register-reallocation layout: idle)
    } else if constexpr (EPI == EPI_SAMPLED) {
        if constexpr (EW0 == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(SAMPLED_REG_HI));
        // ---------------- sampled epilogue, warps EW0..(EW0+NE-1) (both CTAs, own 128 rows): warp w reads
        // TMEM lanes 32*(w%4).. and the CW columns of column group (w-EW0)/4; per K chunk the accumulator is
        // drained into fp32 registers with round-to-nearest adds (times S's chunk scale), then the tile's
        // samples are served from a shared-memory copy, two 32-column chunks at a time
        constexpr int NE = SAMPLED_EPI_WARPS, CW = 1024 / NE, SG = CW / 32;
        const int ew = warp - EW0;
        const int quarter = warp & 3;
        const int colg = ew >> 2;
        const int row = quarter * 32 + lane;
        const int tE = threadIdx.x - 32 * EW0;
        const bool single_unit = n_units <= n_clusters;  // at most one unit per CTA pair
        static_assert(BM * (BN + 1) * 4 <= STAGES2 * STAGE2_BYTES, "a parked tile fits the operand ring");
        int cg = 0;
        for (int t = cluster; t < n_units; t += n_clusters) {
            int mp_tile, n_tile, c0, c1;
            if (!unit(t, mp_tile, n_tile, c0, c1)) continue;
            float *part_out = (ep.tile_list && ep.part && t >= ep.n_whole)
                                  ? ep.part + (int64_t)((t - ep.n_whole) % ep.split) * ep.ns
                                  : nullptr;
            const int m_tile = 2 * mp_tile + (int)crank;
            const int m0 = m_tile * BM, n0 = n_tile * BN;
            const int gr = m0 + row;
            const int gc_base = n0 + colg * CW;
            float run[CW];
#pragma unroll
            for (int i = 0; i < CW; i++) run[i] = 0.f;
            // single unit: while the MMAs run, the tile's sample list is staged in the idle epilogue area as
            // (tile offset, dst) pairs and the row scale is fetched, so the serve after the last chunk reads
            // shared memory only
            float ra_pre = 1.f;
            if (single_unit && m_tile < num_m) {
                const int64_t tile_id = (int64_t)m_tile * ep.n_ct + n_tile;
                const int64_t skb = ep.chunk_ptr[tile_id * (BN / 32)], ske = ep.chunk_ptr[(tile_id + 1) * (BN / 32)];
                if (ske - skb <= (int64_t)(EPI2_BYTES / sizeof(int2))) {
                    int2 *sl = reinterpret_cast<int2 *>(estage);
                    for (int64_t k = skb + tE; k < ske; k += 32 * NE)
                        sl[k - skb] = make_int2((ep.s_r[k] - m0) * (BN + 1) + (ep.s_c[k] - n0),
                                                part_out ? 0 : ep.s_dst[k]);
                }
                if (ep.sa && gr < M) ra_pre = ep.sa[gr];
            }
            for (int ch = c0; ch < c1; ch++, cg++) {
                const int b = cg & 1;
                mbar_wait(&tfull[b], (cg >> 1) & 1);
                tc_fence_after();
                const uint32_t ta = tmem + b * BN + colg * CW + ((uint32_t)(quarter * 32) << 16);
#if S16_SCALE_ROWS == 128
                if (ep.sbk) {  // one scale per (128 S rows, K chunk): a scalar for this thread's columns
                    const float skv = __ldg(ep.sbk + (int64_t)ch * ep.sbk_ld + (gc_base >> 7));
#pragma unroll
                    for (int c16 = 0; c16 < CW / 16; c16++) {
                        uint32_t r[16];
                        tmem_ld16_raw(ta + c16 * 16, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; i++) run[c16 * 16 + i] = fmaf(__uint_as_float(r[i]), skv, run[c16 * 16 + i]);
                    }
                } else
#else
                if (ep.sbk) {  // per-(column, K chunk) scales: DW-column TMEM loads next to DW/4 scale vectors
                    constexpr int DW = CW >= 128 ? 8 : 4;  // (16 warps: 96 registers, run[64] + 8 temporaries)
                    const float *sk = ep.sbk + (int64_t)ch * ep.sbk_ld + gc_base;
#pragma unroll
                    for (int c8 = 0; c8 < CW / DW; c8++) {
                        uint32_t r[DW];
                        float4 v[DW / 4];
                        if constexpr (DW == 8) tmem_ld8_raw(ta + c8 * 8, *reinterpret_cast<uint32_t(*)[8]>(r));
                        else tmem_ld4_raw(ta + c8 * 4, *reinterpret_cast<uint32_t(*)[4]>(r));
                        const float4 *sk4 = reinterpret_cast<const float4 *>(sk + c8 * DW);
#pragma unroll
                        for (int u = 0; u < DW / 4; u++) v[u] = __ldg(sk4 + u);
                        tmem_wait_ld();
                        float *rr = run + c8 * DW;
#pragma unroll
                        for (int u = 0; u < DW / 4; u++) {
                            rr[4 * u + 0] = fmaf(__uint_as_float(r[4 * u + 0]), v[u].x, rr[4 * u + 0]);
                            rr[4 * u + 1] = fmaf(__uint_as_float(r[4 * u + 1]), v[u].y, rr[4 * u + 1]);
                            rr[4 * u + 2] = fmaf(__uint_as_float(r[4 * u + 2]), v[u].z, rr[4 * u + 2]);
                            rr[4 * u + 3] = fmaf(__uint_as_float(r[4 * u + 3]), v[u].w, rr[4 * u + 3]);
                        }
                    }
                } else
#endif
                {
#pragma unroll
                    for (int c16 = 0; c16 < CW / 16; c16++) {
                        uint32_t r[16];
                        tmem_ld16_raw(ta + c16 * 16, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; i++) run[c16 * 16 + i] += __uint_as_float(r[i]);
                    }
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(&tempty[b]);
            }
            if (threadIdx.x == 32 * EW0) { GEMM_MARK(5) }
            if (ep.sb) {
                const float ra = single_unit ? ra_pre : ((ep.sa && gr < M) ? ep.sa[gr] : 1.f);
#pragma unroll
                for (int i = 0; i < CW; i++) {
                    const int gc = gc_base + i;
                    const float rb = gc < N ? __ldg(ep.sb + gc) : 1.f;
                    run[i] *= ra * rb;
                }
            } else if (ep.sa) {  // (stage 2: the S operand carries chunk scales, not column scales)
                const float ra = single_unit ? ra_pre : (gr < M ? ep.sa[gr] : 1.f);
#pragma unroll
                for (int i = 0; i < CW; i++) run[i] *= ra;
            }
            const int64_t tile = (int64_t)m_tile * ep.n_ct + n_tile;
            const bool tile_ok = m_tile < num_m;
            if (single_unit) {
                // this CTA's only unit: its operand ring is idle now, so the whole 128 x 256 tile is parked
                // there (row stride 257, conflict-free) and all its samples are served in one pass
                float *tile_s = reinterpret_cast<float *>(smem);
                if (threadIdx.x == 32 * EW0) { GEMM_MARK(8) }
#pragma unroll
                for (int i = 0; i < CW; i++) tile_s[row * (BN + 1) + colg * CW + i] = run[i];
                named_bar(1, 32 * NE);
                if (threadIdx.x == 32 * EW0) { GEMM_MARK(9) }
                const int64_t skb = tile_ok ? ep.chunk_ptr[tile * (BN / 32)] : 0;
                const int64_t ske = tile_ok ? ep.chunk_ptr[(tile + 1) * (BN / 32)] : 0;
                const bool staged = ske - skb <= (int64_t)(EPI2_BYTES / sizeof(int2));
                if (tile_ok && staged) {  // (offset, dst) pairs from shared memory
                    const int2 *sl = reinterpret_cast<const int2 *>(estage);
                    for (int64_t k = skb + tE; k < ske; k += 32 * NE) {
                        const int2 e = sl[k - skb];
                        const float val = tile_s[e.x];
                        if (part_out) part_out[k] = val;
                        else ep.out[e.y] = ep.accumulate ? fmaf(ep.coef, val, ep.out[e.y]) : ep.coef * val;
                    }
                } else if (tile_ok) {
                    serve_tile<32 * NE>(ep, skb, ske, tE, m0, n0, tile_s, part_out);
                }
                if (threadIdx.x == 32 * EW0) { GEMM_MARK(10) }
                continue;
            }
            // chunk c (32 columns) lives in column group c / SG, sub-block c % SG; step j serves chunks j and
            // j + 4 (staging slots hh = 0, 1 of 4 x 32 x 33 floats each)
#pragma unroll
            for (int j = 0; j < 4; j++) {
                const int g0 = j / SG, g1 = (j + 4) / SG;
                if (colg == g0 || colg == g1) {
                    const int hh = colg == g1 ? 1 : 0;
                    float *mine = estage + (hh * 4 + quarter) * 32 * 33 + lane * 33;
#pragma unroll
                    for (int i = 0; i < 32; i++) mine[i] = run[(j % SG) * 32 + i];
                }
#if SERVE_PREFETCH
                // the sample ranges and this thread's first sample of both chunks are loaded before the staging
                // barrier, so their L2 latency overlaps the staging instead of opening the serve
                int64_t pk0[2], pke[2], pdst[2];
                int prl[2], pcl[2];
#pragma unroll
                for (int hh = 0; hh < 2; hh++) {
                    const int chunk = hh * 4 + j;
                    const int64_t cidx = tile * (BN / 32) + chunk;
                    pk0[hh] = tile_ok ? ep.chunk_ptr[cidx] : 0;
                    pke[hh] = tile_ok ? ep.chunk_ptr[cidx + 1] : 0;
                    const int64_t k = pk0[hh] + tE;
                    prl[hh] = 0;
                    pcl[hh] = 0;
                    pdst[hh] = 0;
                    if (k < pke[hh]) {
                        prl[hh] = ep.s_r[k] - m0;
                        pcl[hh] = ep.s_c[k] - (n0 + chunk * 32);
                        pdst[hh] = ep.s_dst[k];
                    }
                }
#endif
                named_bar(1, 32 * NE);
                if (tile_ok) {
#pragma unroll
                    for (int hh = 0; hh < 2; hh++) {
                        const int chunk = hh * 4 + j;
                        const int gc0 = n0 + chunk * 32;
#if SERVE_PREFETCH
                        const float *stg = estage + hh * 4 * 32 * 33;
                        const int64_t k = pk0[hh] + tE;
                        if (k < pke[hh]) {
                            const float val = stg[(prl[hh] >> 5) * 32 * 33 + (prl[hh] & 31) * 33 + pcl[hh]];
                            if (part_out) part_out[k] = val;
                            else ep.out[pdst[hh]] = ep.accumulate ? fmaf(ep.coef, val, ep.out[pdst[hh]]) : ep.coef * val;
                        }
                        serve_samples<32 * NE>(ep, k + 32 * NE, pke[hh], 0, m0, gc0, stg, part_out);
#else
                        const int64_t cidx = tile * (BN / 32) + chunk;
                        const int64_t kb0 = ep.chunk_ptr[cidx], ke = ep.chunk_ptr[cidx + 1];
                        serve_samples<32 * NE>(ep, kb0, ke, tE, m0, gc0, estage + hh * 4 * 32 * 33, part_out);
#endif
                    }
                }
                named_bar(1, 32 * NE);
            }
        }
        if (threadIdx.x == 32 * EW0) { GEMM_MARK(6) }
    } else {  // ---------------- epilogue warps 2..9 (both CTAs, own 128 rows)
        const int ew = warp - 2;
        const int quarter = warp & 3;
        const int half = ew >> 2;
        const int row = quarter * 32 + lane;
        const int t256 = threadIdx.x - 64;  // 0..255
        // at most one unit per CTA pair (small problems): the operand ring is idle after the last chunk, so
        // the fp16 store epilogue parks the whole tile there and writes full rows (16-byte stores)
        const bool single_unit = EPI == EPI_STORE16 && n_units <= n_clusters && (ep.ldc & 7) == 0;
        int cg = 0;
        for (int t = cluster; t < n_units; t += n_clusters) {
            int mp_tile, n_tile, c0, c1;
            if (!unit(t, mp_tile, n_tile, c0, c1)) continue;
            const int m_tile = 2 * mp_tile + (int)crank;
            const int m0 = m_tile * BM, n0 = n_tile * BN;
            const int gr = m0 + row;
            const int gc_base = n0 + half * 128;
            float run[128];
#pragma unroll
            for (int i = 0; i < 128; i++) run[i] = 0.f;
            float ra_pre = 1.f;
            float *sb_s = estage + 1024;  // (after the 2 x 256-float maximum exchange)
            if (single_unit) {  // while the MMAs run: the row scale, and B's column scales into shared memory
                if (ep.sa && gr < M) ra_pre = ep.sa[gr];
                sb_s[t256] = (ep.sb && n0 + t256 < N) ? ep.sb[n0 + t256] : 1.f;
            }
            for (int ch = c0; ch < c1; ch++, cg++) {
                const int b = cg & 1;
                mbar_wait(&tfull[b], (cg >> 1) & 1);
                tc_fence_after();
                const uint32_t ta = tmem + b * BN + half * 128 + ((uint32_t)(quarter * 32) << 16);
#if S16_SCALE_ROWS == 128
                if (EPI == EPI_SAMPLED && ep.sbk) {
                    // chunk-scaled B (fp16 S from EPI_STORE16): this thread's 128 columns are the S rows
                    // of ONE stage-1 CTA block, so the chunk's scale is a single scalar -- the drain is
                    // the plain 16-column loop with an FMA (no scale vectors next to run[128])
                    const float skv = __ldg(ep.sbk + (int64_t)ch * ep.sbk_ld + (gc_base >> 7));
#pragma unroll
                    for (int c8 = 0; c8 < 8; c8++) {
                        uint32_t r[16];
                        tmem_ld16_raw(ta + c8 * 16, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; i++) run[c8 * 16 + i] = fmaf(__uint_as_float(r[i]), skv, run[c8 * 16 + i]);
                    }
                } else {
#pragma unroll
                    for (int c8 = 0; c8 < 8; c8++) {
                        uint32_t r[16];
                        tmem_ld16_raw(ta + c8 * 16, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; i++) run[c8 * 16 + i] += __uint_as_float(r[i]);
                    }
                }
#else
                // per-(column, K-chunk) scale of a chunk-scaled B operand (fp16 S from EPI_STORE16)
                const float *sk = ep.sbk ? ep.sbk + (int64_t)ch * ep.sbk_ld + gc_base : nullptr;
#if DRAIN_X16
                if (EPI == EPI_SAMPLED && sk) {  // (host side: chunk scales only with the sampled epilogue)
                    // chunk-scaled B: 8-column TMEM loads and two 16-byte scale loads per step, so
                    // the temporaries next to run[128] stay within the 168-register cap of 10 warps
                    // (x16 loads plus four scale vectors spilled part of run[] in this kernel)
#pragma unroll
                    for (int c16 = 0; c16 < 16; c16++) {
                        uint32_t r[8];
                        tmem_ld8_raw(ta + c16 * 8, r);
                        const float4 *sk4 = reinterpret_cast<const float4 *>(sk + c16 * 8);
                        const float4 v0 = __ldg(sk4), v1 = __ldg(sk4 + 1);
                        tmem_wait_ld();
                        float *rr = run + c16 * 8;
                        rr[0] = fmaf(__uint_as_float(r[0]), v0.x, rr[0]);
                        rr[1] = fmaf(__uint_as_float(r[1]), v0.y, rr[1]);
                        rr[2] = fmaf(__uint_as_float(r[2]), v0.z, rr[2]);
                        rr[3] = fmaf(__uint_as_float(r[3]), v0.w, rr[3]);
                        rr[4] = fmaf(__uint_as_float(r[4]), v1.x, rr[4]);
                        rr[5] = fmaf(__uint_as_float(r[5]), v1.y, rr[5]);
                        rr[6] = fmaf(__uint_as_float(r[6]), v1.z, rr[6]);
                        rr[7] = fmaf(__uint_as_float(r[7]), v1.w, rr[7]);
                    }
                } else {
                    // 16-column TMEM loads: 16 fewer live registers than x32 next to run[128]
#pragma unroll
                    for (int c8 = 0; c8 < 8; c8++) {
                        uint32_t r[16];
                        tmem_ld16_raw(ta + c8 * 16, r);
                        tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 16; i++) run[c8 * 16 + i] += __uint_as_float(r[i]);
                    }
                }
#else
#pragma unroll
                for (int c4 = 0; c4 < 4; c4++) {
                    uint32_t r[32];
                    tmem_ld32_raw(ta + c4 * 32, r);
                    tmem_wait_ld();
                    if (sk) {
#pragma unroll
                        for (int i = 0; i < 32; i++)
                            run[c4 * 32 + i] = fmaf(__uint_as_float(r[i]), __ldg(sk + c4 * 32 + i), run[c4 * 32 + i]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; i++) run[c4 * 32 + i] += __uint_as_float(r[i]);
                    }
                }
#endif
#endif  // S16_SCALE_ROWS
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_leader(&tempty[b]);
            }
            if (threadIdx.x == 64) { GEMM_MARK(5) }
            if (single_unit) named_bar(1, 32 * N_EPI_WARPS);  // the staged column scales are visible
            if (EPI == EPI_STORE16 && ep.n_whole > 0 && t >= ep.n_whole) {
                // tail-split unit: this K part's raw accumulators (before the row / column scales) to the part
                // buffer [part][split tile][m half][128 rows][256 cols]; k_store16_fixup sums and stores them
                const int u = t - ep.n_whole, ks = u % ep.split, r_tiles = (n_units - ep.n_whole) / ep.split;
                float *dp = ep.part + ((((int64_t)ks * r_tiles + u / ep.split) * 2 + crank) * BM + row) * BN + half * 128;
#pragma unroll
                for (int i = 0; i < 128; i += 4)
                    *reinterpret_cast<float4 *>(dp + i) = make_float4(run[i], run[i + 1], run[i + 2], run[i + 3]);
                continue;
            }
            if (EPI == EPI_STORE16) {
                // fp16 hi/lo of the unscaled result with a power-of-two scale per (128-row CTA block,
                // 256-col tile) from the block's maximum (S16_SCALE_ROWS = 128: a CTA-wide max over
                // the 8 epilogue warps), or per (row, 256-col tile) (S16_SCALE_ROWS = 1: the two warps
                // holding this row's column halves exchange their maxima)
                const float ra = single_unit ? ra_pre : ((ep.sa && gr < M) ? ep.sa[gr] : 1.f);
                float mx = 0.f;
                // column scales of B in 16-byte loads (the scale vector is padded to 128 rows)
#pragma unroll
                for (int i4 = 0; i4 < 32; i4++) {
                    const float4 rb4 = single_unit ? reinterpret_cast<const float4 *>(sb_s + half * 128)[i4]
                                       : ep.sb ? __ldg(reinterpret_cast<const float4 *>(ep.sb + gc_base) + i4)
                                               : make_float4(1.f, 1.f, 1.f, 1.f);
                    const float rbv[4] = {rb4.x, rb4.y, rb4.z, rb4.w};
#pragma unroll
                    for (int u = 0; u < 4; u++) {
                        const int i = 4 * i4 + u, gc = gc_base + i;
                        run[i] *= ra * (gc < N ? rbv[u] : 1.f);
                        if (gc < N) mx = fmaxf(mx, fabsf(run[i]));
                    }
                }
#if S16_SCALE_ROWS == 128
                for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if (lane == 0) estage[ew] = mx;
                named_bar(1, 32 * N_EPI_WARPS);
#pragma unroll
                for (int w8 = 0; w8 < N_EPI_WARPS; w8++) mx = fmaxf(mx, estage[w8]);
                named_bar(1, 32 * N_EPI_WARPS);
#else
                estage[(quarter * 32 + lane) * 2 + half] = mx;
                named_bar(1, 32 * N_EPI_WARPS);
                mx = fmaxf(estage[(quarter * 32 + lane) * 2], estage[(quarter * 32 + lane) * 2 + 1]);
                named_bar(1, 32 * N_EPI_WARPS);
#endif
                if (threadIdx.x == 64) { GEMM_MARK(8) }
                int e = 0;
                if (mx > 0.f && isfinite(mx)) {
                    int ex;
                    frexpf(mx, &ex);
                    e = 15 - ex;
                }
                const float s = ldexpf(1.f, e);
#if S16_SCALE_ROWS == 128
                // one writer per CTA block (also for a padding block past M: scale 1, finite)
                if (threadIdx.x == 64) ep.c_sk[(int64_t)n_tile * ep.c_sk_ld + (m0 >> 7)] = ldexpf(1.f, -e);
#else
                if (gr < M && half == 0) ep.c_sk[(int64_t)n_tile * ep.c_sk_ld + gr] = ldexpf(1.f, -e);
#endif
                // coalesced stores through this warp's staging block: each lane (one row) parks
                // 32 columns of (hi, lo) pairs, then the warp writes the block row by row, 64
                // contiguous bytes per piece (a thread-per-row store pattern would touch 32 lines
                // per instruction; it dominated the epilogue of short-K tiles)
                if (threadIdx.x == 64) { GEMM_MARK(9) }
                if (single_unit) {
                    // the tile as fp16 hi / lo rows in the idle ring (pitch 264 halves: the 16-byte writes of 8
                    // consecutive rows hit distinct banks), then each warp stores whole rows, 512 B per piece
                    constexpr int TPH = BN + 8;
                    __half *th = reinterpret_cast<__half *>(smem), *tl = th + BM * TPH;
#pragma unroll
                    for (int c8 = 0; c8 < 16; c8++) {
                        uint32_t hp[4], lp[4];
#pragma unroll
                        for (int i = 0; i < 8; i += 2) {
                            const float v0 = run[c8 * 8 + i] * s, v1 = run[c8 * 8 + i + 1] * s;
                            const __half2 h = __float22half2_rn(make_float2(v0, v1));
                            const float2 hf = __half22float2(h);
                            const __half2 l = __float22half2_rn(make_float2(v0 - hf.x, v1 - hf.y));
                            hp[i / 2] = *reinterpret_cast<const uint32_t *>(&h);
                            lp[i / 2] = *reinterpret_cast<const uint32_t *>(&l);
                        }
                        *reinterpret_cast<uint4 *>(th + row * TPH + half * 128 + c8 * 8) = make_uint4(hp[0], hp[1], hp[2], hp[3]);
                        *reinterpret_cast<uint4 *>(tl + row * TPH + half * 128 + c8 * 8) = make_uint4(lp[0], lp[1], lp[2], lp[3]);
                    }
                    named_bar(1, 32 * N_EPI_WARPS);
                    const int gc = n0 + 8 * lane;
                    for (int r = ew; r < BM; r += N_EPI_WARPS) {
                        if (m0 + r >= M) break;
                        const uint4 vh = *reinterpret_cast<const uint4 *>(th + r * TPH + 8 * lane);
                        const uint4 vl = *reinterpret_cast<const uint4 *>(tl + r * TPH + 8 * lane);
                        const int64_t o = (int64_t)(m0 + r) * ep.ldc + gc;
                        if (gc + 8 <= N) {
                            *reinterpret_cast<uint4 *>(ep.c_h16 + o) = vh;
                            *reinterpret_cast<uint4 *>(ep.c_l16 + o) = vl;
                        } else {
                            const __half *ph = reinterpret_cast<const __half *>(&vh), *pl = reinterpret_cast<const __half *>(&vl);
                            for (int u = 0; u < 8 && gc + u < N; u++) {
                                ep.c_h16[o + u] = ph[u];
                                ep.c_l16[o + u] = pl[u];
                            }
                        }
                    }
                    if (threadIdx.x == 64) { GEMM_MARK(10) }
                    named_bar(1, 32 * N_EPI_WARPS);
                    continue;
                }
                uint32_t *blk = reinterpret_cast<uint32_t *>(estage) + (half * 4 + quarter) * 32 * 33;
                const int64_t row0 = (int64_t)m0 + quarter * 32;
#pragma unroll
                for (int c4 = 0; c4 < 4; c4++) {
                    // packed conversions: hi = rn(v), lo = rn(v - hi) two columns at a time; the
                    // row's block holds 16 hi pairs then 16 lo pairs
#pragma unroll
                    for (int i = 0; i < 32; i += 2) {
                        const float v0 = run[c4 * 32 + i] * s, v1 = run[c4 * 32 + i + 1] * s;
                        const __half2 h = __float22half2_rn(make_float2(v0, v1));
                        const float2 hf = __half22float2(h);
                        const __half2 l = __float22half2_rn(make_float2(v0 - hf.x, v1 - hf.y));
                        blk[lane * 33 + i / 2] = *reinterpret_cast<const uint32_t *>(&h);
                        blk[lane * 33 + 16 + i / 2] = *reinterpret_cast<const uint32_t *>(&l);
                    }
                    __syncwarp();
                    // half2 stores: lanes 0-15 write row r, lanes 16-31 row r + 1, two columns each
                    const int j = lane & 15;
                    const int gc = gc_base + c4 * 32 + 2 * j;
                    if (gc < N) {
                        for (int r = lane >> 4; r < 32; r += 2) {
                            if (row0 + r >= M) break;
                            const uint32_t ph = blk[r * 33 + j], pl = blk[r * 33 + 16 + j];
                            const int64_t o = (row0 + r) * ep.ldc + gc;
                            if (gc + 1 < N) {
                                *reinterpret_cast<uint32_t *>(ep.c_h16 + o) = ph;
                                *reinterpret_cast<uint32_t *>(ep.c_l16 + o) = pl;
                            } else {
                                ep.c_h16[o] = __ushort_as_half((unsigned short)(ph & 0xffffu));
                                ep.c_l16[o] = __ushort_as_half((unsigned short)(pl & 0xffffu));
                            }
                        }
                    }
                    __syncwarp();
                }
                if (threadIdx.x == 64) { GEMM_MARK(10) }
                // the next tile's scale exchange reuses the staging area
                named_bar(1, 32 * N_EPI_WARPS);
                continue;
            }
            if (ep.sa || ep.sb) {
                const float ra = (ep.sa && gr < M) ? ep.sa[gr] : 1.f;
#pragma unroll
                for (int i = 0; i < 128; i++) {
                    const int gc = gc_base + i;
                    const float rb = (ep.sb && gc < N) ? __ldg(ep.sb + gc) : 1.f;
                    run[i] *= ra * rb;
                }
            }
            if (EPI == EPI_STORE) {
                if (gr < M) {
                    float *cf = ep.c_f + (int64_t)gr * ep.ldc + gc_base;
                    if (gc_base + 128 <= N) {
#pragma unroll
                        for (int i = 0; i < 128; i += 4)
                            *reinterpret_cast<float4 *>(cf + i) = make_float4(run[i], run[i + 1], run[i + 2], run[i + 3]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 128; i++)
                            if (gc_base + i < N) cf[i] = run[i];
                    }
                    if (ep.c_hi) {
#pragma unroll
                        for (int i = 0; i < 128; i++) {
                            if (gc_base + i < N) {
                                float h = tf32_round(run[i]);
                                ep.c_hi[(int64_t)gr * ep.ldc + gc_base + i] = h;
                                ep.c_lo[(int64_t)gr * ep.ldc + gc_base + i] = tf32_round(run[i] - h);
                            }
                        }
                    }
                }
            } else if (EPI == EPI_GRAM) {
                // kernel values, then coalesced row stores through this warp's staging block
                // (as in EPI_STORE16); the next tile's epilogue reuses the block after the barrier
                const float ni = (ep.kind == GVT_BASE_GAUSSIAN && gr < M) ? ep.norms[gr] : 0.f;
                float *blk = estage + (half * 4 + quarter) * 32 * 33;
                const int64_t row0 = (int64_t)m0 + quarter * 32;
                // kernel parameters in registers once per tile, one loop per base kernel (the
                // per-element re-reads of the parameter bank were 42 % of this epilogue's stalls)
                const int kind = ep.kind, degree = ep.degree, same = ep.same;
                const float gamma = ep.gamma, coef0 = ep.coef0;
#pragma unroll
                for (int c4 = 0; c4 < 4; c4++) {
                    float *row = blk + lane * 33;
                    if (kind == GVT_BASE_GAUSSIAN) {
                        // the 32 column norms of this block: one coalesced load, then shuffles
                        const int gcl = gc_base + c4 * 32 + lane;
                        const float nbl = gcl < N ? ep.norms_b[gcl] : 0.f;
                        const float ng = -gamma;
#pragma unroll
                        for (int i = 0; i < 32; i++) {
                            const float nb = __shfl_sync(0xffffffffu, nbl, i);
                            float d2 = fmaxf(ni + nb - 2.f * run[c4 * 32 + i], 0.f);
                            if (same && gc_base + c4 * 32 + i == gr) d2 = 0.f;
                            row[i] = expf(ng * d2);
                        }
                    } else if (kind == GVT_BASE_POLY) {
#pragma unroll
                        for (int i = 0; i < 32; i++) {
                            const float bb = fmaf(gamma, run[c4 * 32 + i], coef0);
                            float rr = 1.f;
                            for (int e = 0; e < degree; e++) rr *= bb;
                            row[i] = rr;
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < 32; i++) row[i] = run[c4 * 32 + i];
                    }
                    __syncwarp();
                    const int gc = gc_base + c4 * 32 + lane;
                    if (gc < N) {
                        for (int r = 0; r < 32; r++) {
                            if (row0 + r >= M) break;
                            ep.c_f[(row0 + r) * ep.ldc + gc] = blk[r * 33 + lane];
                        }
                    }
                    __syncwarp();
                }
            } else if (EPI == EPI_SAMPLED) {
                const int64_t tile = (int64_t)m_tile * ep.n_ct + n_tile;
                const bool tile_ok = m_tile < num_m;
#pragma unroll
                for (int c4 = 0; c4 < 4; c4++) {
                    float *mine = estage + (half * 4 + quarter) * 32 * 33 + lane * 33;
#pragma unroll
                    for (int i = 0; i < 32; i++) mine[i] = run[c4 * 32 + i];
                    named_bar(1, 32 * N_EPI_WARPS);
                    if (tile_ok) {
#pragma unroll
                        for (int hh = 0; hh < 2; hh++) {
                            const int chunk = hh * 4 + c4;
                            const int64_t cidx = tile * (BN / 32) + chunk;
                            const int64_t kb0 = ep.chunk_ptr[cidx], ke = ep.chunk_ptr[cidx + 1];
                            const int gc0 = n0 + chunk * 32;
                            serve_samples<256>(ep, kb0, ke, t256, m0, gc0, estage + hh * 4 * 32 * 33, nullptr);
                        }
                    }
                    named_bar(1, 32 * N_EPI_WARPS);
                }
            }
        }
    }
    if (EPI != EPI_SAMPLED && threadIdx.x == 64) { GEMM_MARK(6) }
    tc_fence_before();
    cluster_sync_all();  // both CTAs done with TMEM / shared memory before the pair deallocates
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
    }
    if (threadIdx.x == 0) { GEMM_MARK(7) }
}


// ----------------------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static void get_encode() {
    if (g_encode) return;
    void *fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    GVT_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    GVT_REQUIRE(fn && q == cudaDriverEntryPointSuccess, GVT_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    g_encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
}

static CUtensorMapL2promotion l2promo() {  // A/B knob (experiment): GVT_L2PROMO 0 none, 1 64B, 2 128B, 3 256B
    static const int v = [] {
        const char *e = getenv("GVT_L2PROMO");
        return e ? atoi(e) : 3;
    }();
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : v == 1 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                           : v == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
}

// rows x cols (cols = K, contiguous) matrix, element size esz, leading dimension ld elements;
// box = one 128-byte K-block x box_rows
static CUtensorMap make_map(const void *p, int esz, int64_t rows, int64_t cols, int64_t ld, int box_rows) {
    get_encode();
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)(cols > 0 ? cols : 1), (cuuint64_t)(rows > 0 ? rows : 1)};
    cuuint64_t strides[1] = {(cuuint64_t)ld * esz};
    cuuint32_t box[2] = {(cuuint32_t)(KB_BYTES / esz), (cuuint32_t)box_rows};
    cuuint32_t es[2] = {1, 1};
    CUresult r = g_encode(&m, esz == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                          const_cast<void *>(p), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          KB_BYTES == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                          : (KB_BYTES == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B),
                          l2promo(),
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    GVT_REQUIRE(r == CUDA_SUCCESS, GVT_E_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    return m;
}

bool tc_available(gvt_ctx *c) { return c->tc_ok; }

// GVT_GEMM_PROF: phase stamps of one CTA-pair GEMM launch, in us from the earliest CTA entry
// (median / max over CTAs), to stderr -- diagnosis only (it synchronises the stream)
static void gemm_prof_report(gvt_ctx *c, const unsigned long long *dprof, int grid, int epi, int64_t M, int64_t N,
                             int64_t K) {
    cudaStreamCaptureStatus cs;
    GVT_CUDA_TRY(cudaStreamIsCapturing(c->stream, &cs));
    if (cs != cudaStreamCaptureStatusNone) return;  // (run with OPT_PROFILE: no graph)
    std::vector<unsigned long long> h((size_t)grid * 16);
    GVT_CUDA_TRY(cudaMemcpyAsync(h.data(), dprof, sizeof(unsigned long long) * h.size(), cudaMemcpyDeviceToHost,
                                 c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    unsigned long long t0 = ~0ull;
    for (int b = 0; b < grid; b++) t0 = std::min(t0, h[(size_t)b * 16]);
    static const char *nm[11] = {"entry", "setup", "first_stage", "last_mma", "last_tma", "drained", "epi_done", "exit",
                                 "scaled", "sk", "stored"};
    fprintf(stderr, "gemm_prof epi=%d M=%lld N=%lld K=%lld grid=%d:", epi, (long long)M, (long long)N, (long long)K,
            grid);
    for (int sl = 0; sl < 11; sl++) {
        std::vector<double> v;
        for (int b = 0; b < grid; b++)
            if (h[(size_t)b * 16 + sl]) v.push_back((h[(size_t)b * 16 + sl] - t0) * 1e-3);
        if (v.empty()) continue;
        std::sort(v.begin(), v.end());
        fprintf(stderr, " %s %.1f/%.1f", nm[sl], v[v.size() / 2], v.back());
    }
    fprintf(stderr, "\n");
}

template <int PREC, int EPI>
static void launch_gemm_t(gvt_ctx *c, int kind_id, const Operand &A, const Operand &B, int64_t M, int64_t N,
                          int64_t K, EpiParams ep) {
    constexpr int esz = PREC == PREC_TF32 ? 4 : 2;
    const bool pair = c->gemm_cta == 2;
    CUtensorMap ah = make_map(A.hi, esz, M, K, A.ld, BM), al = make_map(A.lo, esz, M, K, A.ld, BM);
    CUtensorMap bh = make_map(B.hi, esz, N, K, B.ld, pair ? 128 : BN), bl = make_map(B.lo, esz, N, K, B.ld, pair ? 128 : BN);
    ep.sa = A.scale;
    ep.sb = B.scale;
    ep.sbk = B.scale_k;
    ep.sbk_ld = B.scale_k_ld;
    GVT_REQUIRE(!B.scale_k || (pair && PREC == PREC_F16 && EPI == EPI_SAMPLED), GVT_E_STATE,
                "a chunk-scaled operand needs the CTA-pair fp16 GEMM with the sampled epilogue");
    GVT_REQUIRE(EPI != EPI_STORE16 || (pair && PREC == PREC_F16), GVT_E_STATE, "fp16 store needs the CTA-pair fp16 GEMM");
    // function attributes are per device: one flag per device ordinal (one process may drive several)
    static bool attr[GVT_MAX_DEVICES] = {}, attr2[GVT_MAX_DEVICES] = {};
    const int dv = c->device < GVT_MAX_DEVICES ? c->device : 0;
    if (pair) {
        static const int env_gm = [] {  // A/B knob for the rasterization group (scripts/ab_matvec.py)
            const char *e = getenv("GVT_GROUP_M");
            return e ? atoi(e) : 0;
        }();
        if (ep.group_m == 0) ep.group_m = env_gm;
        if (!attr2[dv]) {
            GVT_CUDA_TRY(
                cudaFuncSetAttribute(k_gemm2_x3<PREC, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_TOTAL));
            attr2[dv] = true;
        }
        const int64_t pair_tiles = ((EPI == EPI_SAMPLED && ep.tile_list) || (EPI == EPI_STORE16 && ep.n_whole > 0))
                                       ? ep.n_units
                                       : ((N + BN - 1) / BN) * ((M + 2 * BM - 1) / (2 * BM));
        const int64_t clusters = std::min<int64_t>(pair_tiles, c->sm_count / 2);  // persistent: one pair per 2 SMs
        dim3 grid((unsigned)(2 * clusters));
        static const bool prof = getenv("GVT_GEMM_PROF") != nullptr;
        if (prof) {
            ep.prof = wsT<unsigned long long>(c, "gemm.prof", (size_t)grid.x * 16);
            GVT_CUDA_TRY(cudaMemsetAsync(ep.prof, 0, sizeof(unsigned long long) * grid.x * 16, c->stream));
        }
        GVT_LAUNCH(c, kind_id, (k_gemm2_x3<PREC, EPI>), grid, pair_threads(EPI), SMEM2_TOTAL, ah, al, bh, bl, (int)M, (int)N,
                   (int)K, ep);
        if (prof) gemm_prof_report(c, ep.prof, (int)grid.x, EPI, M, N, K);
        return;
    }
    if (!attr[dv]) {
        GVT_CUDA_TRY(
            cudaFuncSetAttribute(k_gemm_x3<PREC, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_TOTAL));
        attr[dv] = true;
    }
    dim3 grid((unsigned)(((N + BN - 1) / BN) * ((M + BM - 1) / BM)));
    GVT_LAUNCH(c, kind_id, (k_gemm_x3<PREC, EPI>), grid, NTHREADS, SMEM_TOTAL, ah, al, bh, bl, (int)M, (int)N, (int)K,
               ep);
}

template <int EPI>
static void launch_gemm(gvt_ctx *c, int kind_id, const Operand &A, const Operand &B, int64_t M, int64_t N, int64_t K,
                        const EpiParams &ep) {
    if (M == 0 || N == 0) return;
    GVT_REQUIRE(K > 0, GVT_E_DIM, "GEMM with K = 0");
    GVT_REQUIRE(M < INT32_MAX && N < INT32_MAX && K < INT32_MAX, GVT_E_DIM, "GEMM dimension too large");
    GVT_REQUIRE(A.prec == B.prec, GVT_E_STATE, "GEMM operands split with different precisions");
    if (A.prec == PREC_TF32) launch_gemm_t<PREC_TF32, EPI>(c, kind_id, A, B, M, N, K, ep);
    else launch_gemm_t<PREC_F16, EPI>(c, kind_id, A, B, M, N, K, ep);
}

// ----------------------------------------------------------------------------- operand splits
__global__ void k_split_tf32(const float *__restrict__ x, int64_t n, float *__restrict__ hi, float *__restrict__ lo) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float v = x[i];
        float h = tf32_round(v);
        hi[i] = h;
        lo[i] = tf32_round(v - h);
    }
}

// one block per row: scale = 2^(14 - ceil(log2 max|x|)) so the row max lies in [2^14, 2^15)
// (exact power of two; all-zero rows get scale 1); hi = fp16(s x), lo = fp16(s x - hi);
// stores 1/scale for the epilogue.  Columns [cols, ld) are written as zero.
__global__ void __launch_bounds__(256) k_split_rows_f16(const float *__restrict__ x, int64_t rows, int64_t cols,
                                                        int64_t ldx, __half *__restrict__ hi,
                                                        __half *__restrict__ lo, int64_t ld, float *__restrict__ sinv) {
    __shared__ float red[8];
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const float *xr = x + r * ldx;
        float mx = 0.f;
        for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmaxf(mx, fabsf(xr[j]));
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        mx = red[0];
        for (int w = 1; w < 8; w++) mx = fmaxf(mx, red[w]);
        __syncthreads();
        int e = 0;
        if (mx > 0.f && isfinite(mx)) {
            int ex;
            frexpf(mx, &ex);  // mx = f * 2^ex, f in [0.5, 1)  ->  mx < 2^ex
            e = 15 - ex;      // scaled max < 2^15
        }
        const float s = ldexpf(1.f, e);
        if (threadIdx.x == 0) sinv[r] = ldexpf(1.f, -e);
        __half *hr = hi + r * ld, *lr = lo + r * ld;
        for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) {
            const float v = j < cols ? xr[j] * s : 0.f;
            const __half h = __float2half_rn(v);
            hr[j] = h;
            lr[j] = __float2half_rn(v - __half2float(h));
        }
    }
}

static int tc_prec(gvt_ctx *c) { return c->tc_precision == 1 ? PREC_TF32 : PREC_F16; }

int tc_precision_mode(gvt_ctx *c) { return tc_prec(c); }

Operand operand_col_offset(const Operand &o, int64_t off) {
    Operand v = o;
    const int64_t esz = o.prec == PREC_TF32 ? 4 : 2;
    v.hi = (const char *)o.hi + off * esz;  // TMA needs 16-byte aligned bases: off % 32 == 0
    v.lo = (const char *)o.lo + off * esz;
    return v;
}

// split a rows x cols fp32 matrix (leading dimension ldx) into a tensor-core operand with
// leading dimension ld (>= cols, multiple of 32); rows_pad rows are allocated (extra rows zero)
Operand make_operand(gvt_ctx *c, const char *name, const float *x, int64_t rows, int64_t cols, int64_t ldx,
                     int64_t ld, int64_t rows_pad) {
    Operand o;
    o.prec = tc_prec(c);
    o.ld = ld;
    std::string nm(name);
    if (o.prec == PREC_TF32) {
        GVT_REQUIRE(ldx == ld, GVT_E_STATE, "tf32 split expects a padded source");
        float *hi = wsT<float>(c, (nm + ".hi").c_str(), (size_t)rows_pad * ld);
        float *lo = wsT<float>(c, (nm + ".lo").c_str(), (size_t)rows_pad * ld);
        if (rows_pad * ld > 0)
            GVT_LAUNCH(c, K_SPLIT, k_split_tf32, grid1d(rows_pad * ld, 256, 16 * c->sm_count * 8), 256, 0, x,
                       rows_pad * ld, hi, lo);
        o.hi = hi;
        o.lo = lo;
        o.scale = nullptr;
    } else {
        __half *hi = wsT<__half>(c, (nm + ".h16").c_str(), (size_t)rows_pad * ld);
        __half *lo = wsT<__half>(c, (nm + ".l16").c_str(), (size_t)rows_pad * ld);
        float *s = wsT<float>(c, (nm + ".sinv").c_str(), (size_t)rows_pad);
        if (rows_pad > rows) {
            GVT_CUDA_TRY(cudaMemsetAsync(hi + rows * ld, 0, sizeof(__half) * (rows_pad - rows) * ld, c->stream));
            GVT_CUDA_TRY(cudaMemsetAsync(lo + rows * ld, 0, sizeof(__half) * (rows_pad - rows) * ld, c->stream));
        }
        if (rows > 0)
            GVT_LAUNCH(c, K_SPLIT, k_split_rows_f16, grid1d(rows, 1, 16 * c->sm_count), 256, 0, x, rows, cols, ldx, hi,
                       lo, ld, s);
        o.hi = hi;
        o.lo = lo;
        o.scale = s;
    }
    return o;
}

// ---- fused fp16 path: pair-matrix rows assembled in shared memory, written as fp16 pieces
bool fused_f16(gvt_ctx *c, int64_t q_in) {
    return tc_prec(c) == PREC_F16 && c->gemm_cta == 2 && round_up(q_in, 32) * 4 <= 200 * 1024;
}

// one CTA per row r of [row_lo, row_lo + rows): cell values (sum of sign * p[src] over the
// cell's run of entries, in entry order -- the same sums as k_densify) parked in shared
// memory, row max -> power-of-two scale, then coalesced fp16 hi/lo stores of the whole row
// BX_THREADS per row: 1024 for long rows (a row's ~m*density cells spread over 32 warps, latency-bound
// gathers); 256 for rows of <= 8192 columns, where the per-row barrier chain dominates and more rows
// (smaller shared-memory rows) must be in flight per SM
template <int BX_THREADS, bool IDENT>
__global__ void __launch_bounds__(BX_THREADS, 2048 / BX_THREADS) k_build_x16(const int64_t *__restrict__ row_ptr, const int32_t *__restrict__ col,
                                                   const int32_t *__restrict__ src, const float *__restrict__ sign,
                                                   const float *__restrict__ p, int64_t row_lo, int64_t rows,
                                                   int64_t cols, int64_t ld, __half *__restrict__ hi,
                                                   __half *__restrict__ lo, float *__restrict__ sinv,
                                                   const float *__restrict__ diag, int vec) {
    extern __shared__ __align__(16) float rowbuf[];  // ld floats
    __shared__ float red[BX_THREADS / 32];
    // vec: the three shared-memory sweeps of a row (zero, max, store) move 4 cells per thread per
    // pass (ld is a multiple of 32; the cells beyond cols stay zero, so the max over ld equals the
    // max over cols): the same values in the same places, a quarter of the passes
    float4 *rb4 = reinterpret_cast<float4 *>(rowbuf);
    const int64_t ld4 = ld >> 2;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        if (vec) {
            for (int64_t j = threadIdx.x; j < ld4; j += blockDim.x) rb4[j] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {
            for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) rowbuf[j] = 0.f;
        }
        __syncthreads();
        const int64_t kb = row_ptr[row_lo + r], ke = row_ptr[row_lo + r + 1];
        // two entries per thread per pass, their loads independent (in flight together); a run
        // of duplicate cells is summed by its head entry in entry order.  With the 32-register
        // bound two 1024-thread CTAs (two 80 KB rows) are resident per SM: C5 2.59 -> 1.37 ms
        // per launch (profiles/r01_ab_build_x16.txt)
        constexpr int U = 2;
        for (int64_t k0 = kb + threadIdx.x; k0 < ke; k0 += U * BX_THREADS) {
            int32_t cc[U], cprev[U], cnext[U];
            float v[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const int64_t k = k0 + (int64_t)u * BX_THREADS;
                cc[u] = -1;
                if (k < ke) {
                    cc[u] = col[k];
                    cprev[u] = k > kb ? col[k - 1] : -1;
                    cnext[u] = k + 1 < ke ? col[k + 1] : -1;
                    // (IDENT: entry k is pair k with sign +1 -- the same value, 1 * p[k], without the src / sign loads)
                    v[u] = IDENT ? __ldg(p + k) : sign[k] * __ldg(p + src[k]);
                }
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                if (cc[u] < 0 || cprev[u] == cc[u]) continue;  // past the row end, or not the head of its run
                float s = v[u];
                if (cnext[u] == cc[u]) {
                    const int64_t k = k0 + (int64_t)u * BX_THREADS;
                    for (int64_t j = k + 1; j < ke && col[j] == cc[u]; j++)
                        s += IDENT ? __ldg(p + j) : sign[j] * __ldg(p + src[j]);
                }
                rowbuf[cc[u]] = s;
            }
        }
        __syncthreads();
        if (diag && threadIdx.x == 0) rowbuf[row_lo + r] += diag[row_lo + r];  // separate diagonal (MLPK)
        __syncthreads();
        float mx = 0.f;
        if (vec) {
            for (int64_t j = threadIdx.x; j < ld4; j += blockDim.x) {
                const float4 v = rb4[j];
                mx = fmaxf(fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
            }
        } else {
            for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmaxf(mx, fabsf(rowbuf[j]));
        }
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
        __syncthreads();
        mx = red[0];
        for (int w = 1; w < BX_THREADS / 32; w++) mx = fmaxf(mx, red[w]);
        int e = 0;
        if (mx > 0.f && isfinite(mx)) {
            int ex;
            frexpf(mx, &ex);
            e = 15 - ex;
        }
        const float s = ldexpf(1.f, e);
        if (threadIdx.x == 0) sinv[r] = ldexpf(1.f, -e);
        __half2 *h2 = reinterpret_cast<__half2 *>(hi + r * ld), *l2 = reinterpret_cast<__half2 *>(lo + r * ld);
        if (vec) {
            uint2 *h4 = reinterpret_cast<uint2 *>(h2), *l4 = reinterpret_cast<uint2 *>(l2);
            for (int64_t j = threadIdx.x; j < ld4; j += blockDim.x) {
                const float4 v = rb4[j];
                const float v0 = v.x * s, v1 = v.y * s, v2 = v.z * s, v3 = v.w * s;
                const __half a0 = __float2half_rn(v0), a1 = __float2half_rn(v1), a2 = __float2half_rn(v2),
                             a3 = __float2half_rn(v3);
                const __half2 ha = __halves2half2(a0, a1), hb = __halves2half2(a2, a3);
                const __half2 la = __halves2half2(__float2half_rn(v0 - __half2float(a0)), __float2half_rn(v1 - __half2float(a1)));
                const __half2 lb = __halves2half2(__float2half_rn(v2 - __half2float(a2)), __float2half_rn(v3 - __half2float(a3)));
                h4[j] = make_uint2(*reinterpret_cast<const uint32_t *>(&ha), *reinterpret_cast<const uint32_t *>(&hb));
                l4[j] = make_uint2(*reinterpret_cast<const uint32_t *>(&la), *reinterpret_cast<const uint32_t *>(&lb));
            }
        } else {
            for (int64_t j = threadIdx.x; j < ld / 2; j += blockDim.x) {
                const float v0 = rowbuf[2 * j] * s, v1 = rowbuf[2 * j + 1] * s;
                const __half a0 = __float2half_rn(v0), a1 = __float2half_rn(v1);
                h2[j] = __halves2half2(a0, a1);
                l2[j] = __halves2half2(__float2half_rn(v0 - __half2float(a0)), __float2half_rn(v1 - __half2float(a1)));
            }
        }
        __syncthreads();
    }
}

// the same rows, one WARP per row, for short rows (ld <= 2048: C2/C3-size problems; C4 Poly2D's
// 3008-wide rows measured 3-4 % slower per CG iteration with it): the CTA-wide
// barriers of k_build_x16 (zero, gather, max, store) become __syncwarp, and every row of the matrix is
// in flight at once (8 rows per CTA, ld floats of shared memory each).  Same cell sums (entry order),
// same scale rule, same stores.
__global__ void __launch_bounds__(256) k_build_x16_warp(const int64_t *__restrict__ row_ptr,
                                                        const int32_t *__restrict__ col,
                                                        const int32_t *__restrict__ src,
                                                        const float *__restrict__ sign, const float *__restrict__ p,
                                                        int64_t row_lo, int64_t rows, int64_t cols, int64_t ld,
                                                        __half *__restrict__ hi, __half *__restrict__ lo,
                                                        float *__restrict__ sinv, const float *__restrict__ diag) {
    extern __shared__ float rowbufs[];  // 8 x ld floats
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float *rowbuf = rowbufs + (size_t)warp * ld;
    const int64_t nw = (int64_t)gridDim.x * 8;
    for (int64_t r = (int64_t)blockIdx.x * 8 + warp; r < rows; r += nw)
        x16_row_warp<false>(r, lane, rowbuf, row_ptr, col, src, sign, p, row_lo, ld, hi, lo, sinv, diag);
}

static bool build_ident() {  // A/B knob: GVT_BUILD_IDENT=0 reads src / sign even for identity entry plans
    static const bool on = [] {
        const char *e = getenv("GVT_BUILD_IDENT");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

static bool build_warp_rows() {  // A/B knob: GVT_BUILD_WARP=0 keeps the CTA-per-row build for short rows
    static const bool on = [] {
        const char *e = getenv("GVT_BUILD_WARP");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

static int build_vec() {  // A/B knob: GVT_BUILD_VEC=0 keeps the scalar shared-memory sweeps of the CTA-per-row build
    static const int on = [] {
        const char *e = getenv("GVT_BUILD_VEC");
        return (e && atoi(e) == 0) ? 0 : 1;
    }();
    return on;
}

Operand build_x16(gvt_ctx *c, const char *name, const EntryPlan &e, int64_t row_lo, int64_t rows, int64_t cols,
                  const float *p, const float *diag, bool launch) {
    Operand o;
    o.prec = PREC_F16;
    o.ld = round_up(cols > 0 ? cols : 1, 32);
    std::string nm(name);
    const int64_t rows_pad = round_up(rows > 0 ? rows : 1, 128);
    __half *hi = wsT<__half>(c, (nm + ".h16").c_str(), (size_t)rows_pad * o.ld);
    __half *lo = wsT<__half>(c, (nm + ".l16").c_str(), (size_t)rows_pad * o.ld);
    float *s = wsT<float>(c, (nm + ".sinv").c_str(), (size_t)rows_pad);
    if (!launch) {
        o.hi = hi;
        o.lo = lo;
        o.scale = s;
        return o;
    }
    const size_t smem = sizeof(float) * o.ld;
    static size_t attr_smem[GVT_MAX_DEVICES] = {};
    size_t &attr_dev = attr_smem[c->device < GVT_MAX_DEVICES ? c->device : 0];
    if (smem > 48 * 1024 && smem > attr_dev) {
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_build_x16<1024, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_build_x16<256, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_build_x16<1024, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        GVT_CUDA_TRY(cudaFuncSetAttribute(k_build_x16<256, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_dev = smem;
    }
    if (rows > 0 && o.ld <= 2048 && build_warp_rows()) {
        const size_t smem8 = 8 * smem;
        static size_t attr_w[GVT_MAX_DEVICES] = {};
        size_t &aw = attr_w[c->device < GVT_MAX_DEVICES ? c->device : 0];
        if (smem8 > 48 * 1024 && smem8 > aw) {
            GVT_CUDA_TRY(cudaFuncSetAttribute(k_build_x16_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem8));
            aw = smem8;
        }
        GVT_LAUNCH(c, K_DENSIFY, k_build_x16_warp, grid1d(rows, 8), 256, smem8, e.row_ptr, e.col, e.src, e.sign, p,
                   row_lo, rows, cols, o.ld, hi, lo, s, diag);
    } else if (rows > 0) {
        const bool ident = e.ident && build_ident();
        if (o.ld > 8192 && ident)
            GVT_LAUNCH(c, K_DENSIFY, (k_build_x16<1024, true>), grid1d(rows, 1, 2 * c->sm_count), 1024, smem, e.row_ptr,
                       e.col, e.src, e.sign, p, row_lo, rows, cols, o.ld, hi, lo, s, diag, build_vec());
        else if (o.ld > 8192)
            GVT_LAUNCH(c, K_DENSIFY, (k_build_x16<1024, false>), grid1d(rows, 1, 2 * c->sm_count), 1024, smem, e.row_ptr,
                       e.col, e.src, e.sign, p, row_lo, rows, cols, o.ld, hi, lo, s, diag, build_vec());
        else if (ident)
            GVT_LAUNCH(c, K_DENSIFY, (k_build_x16<256, true>), grid1d(rows, 1, 16 * c->sm_count), 256, smem, e.row_ptr,
                       e.col, e.src, e.sign, p, row_lo, rows, cols, o.ld, hi, lo, s, diag, build_vec());
        else
            GVT_LAUNCH(c, K_DENSIFY, (k_build_x16<256, false>), grid1d(rows, 1, 16 * c->sm_count), 256, smem, e.row_ptr,
                       e.col, e.src, e.sign, p, row_lo, rows, cols, o.ld, hi, lo, s, diag, build_vec());
    }
    o.hi = hi;
    o.lo = lo;
    o.scale = s;
    return o;
}

// ---- block sparsity of the pair matrix for stage 1 (kb_list / kb_off of the CTA-pair kernel)
__global__ void k_kb_flags(const int32_t *__restrict__ row, const int32_t *__restrict__ col, int64_t k0, int64_t k1,
                           int64_t lo, int64_t rows, int64_t nkb, uint8_t *__restrict__ flags) {
    for (int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = row[k] - lo;
        if (r >= 0 && r < rows) flags[(r / BN) * nkb + col[k] / 64] = 1;  // idempotent byte stores
    }
}

void kblock_lists(gvt_ctx *c, const EntryPlan &e, int64_t k0, int64_t k1, int64_t lo, int64_t rows, int64_t cols,
                  bool diag, std::vector<int32_t> &list, std::vector<int32_t> &off) {
    const int64_t ntiles = (rows + BN - 1) / BN, nkb = (cols + 63) / 64;
    uint8_t *flags = wsT<uint8_t>(c, "kbl.flags", (size_t)(ntiles * nkb));
    GVT_CUDA_TRY(cudaMemsetAsync(flags, 0, (size_t)(ntiles * nkb), c->stream));
    if (k1 > k0)
        GVT_LAUNCH(c, K_PLAN_KEYS, k_kb_flags, grid1d(k1 - k0, 256, 8 * c->sm_count * 8), 256, 0, e.row, e.col, k0, k1,
                   lo, rows, nkb, flags);
    std::vector<uint8_t> h((size_t)(ntiles * nkb));
    GVT_CUDA_TRY(cudaMemcpyAsync(h.data(), flags, h.size(), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (diag)  // the separate diagonal X[r][r] (MLPK Laplacian) sits in column lo + r
        for (int64_t r = 0; r < rows; r++) h[(size_t)((r / BN) * nkb + (lo + r) / 64)] = 1;
    list.clear();
    off.assign((size_t)ntiles + 1, 0);
    for (int64_t t = 0; t < ntiles; t++) {
        const size_t before = list.size();
        for (int64_t b = 0; b < nkb; b++)
            if (h[(size_t)(t * nkb + b)]) list.push_back((int32_t)b);
        if (list.size() == before) list.push_back(0);  // at least one K-block: the accumulator is defined
        off[(size_t)t + 1] = (int32_t)list.size();
    }
}

// The stage-1 tail split: the last r pair tiles of the grouped order (r <= pairs / 2 after whole waves) run as
// `split` K parts each; here one warp per output row of block (split tile, m half) sums the parts in part order
// (8 columns per lane), applies the operands' row / column scales, and stores the fp16 pieces with the
// epilogue's per-(row, 256-column tile) scale rule (S16_SCALE_ROWS = 1), 16 bytes per lane per piece.
__global__ void __launch_bounds__(256) k_store16_fixup(const float *__restrict__ part, int split, int r_tiles, int n_whole,
                                                       const int32_t *__restrict__ order, int num_mp, int num_n, int gm,
                                                       int64_t M, int64_t N,
                                                       const float *__restrict__ sa, const float *__restrict__ sb,
                                                       __half *__restrict__ ch, __half *__restrict__ cl, int64_t ldc,
                                                       float *__restrict__ csk, int64_t csk_ld) {
    // block b: split tile b / 32, m half (b / 16) & 1, rows 8 (b % 16) + warp (one row per warp: all in flight)
    const int ti = blockIdx.x >> 5, mh = (blockIdx.x >> 4) & 1, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int t = n_whole + ti, in_group = gm * num_n, first_m = (t / in_group) * gm;
    const int group_m = min(num_mp - first_m, gm);
    const int mp_tile = order ? order[t] / num_n : first_m + (t % in_group) % group_m;
    const int n_tile = order ? order[t] % num_n : (t % in_group) / group_m;
    const int64_t gc0 = (int64_t)n_tile * BN + 8 * lane;
    {
        const int row = (blockIdx.x & 15) * 8 + warp;
        const int64_t gr = (int64_t)(2 * mp_tile + mh) * BM + row;
        if (gr >= M) return;
        float v[8];
        for (int h = 0; h < split; h++) {
            const float4 *pp =
                reinterpret_cast<const float4 *>(part + ((((int64_t)h * r_tiles + ti) * 2 + mh) * BM + row) * BN + 8 * lane);
            const float4 q0 = pp[0], q1 = pp[1];
            const float q[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
            for (int i = 0; i < 8; i++) v[i] = h == 0 ? q[i] : v[i] + q[i];
        }
        const float ra = sa ? sa[gr] : 1.f;
        float mx = 0.f;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int64_t gc = gc0 + i;
            v[i] *= ra * ((sb && gc < N) ? sb[gc] : 1.f);
            if (gc < N) mx = fmaxf(mx, fabsf(v[i]));
        }
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        int e = 0;
        if (mx > 0.f && isfinite(mx)) {
            int ex;
            frexpf(mx, &ex);
            e = 15 - ex;
        }
        const float s = ldexpf(1.f, e);
        if (lane == 0) csk[(int64_t)n_tile * csk_ld + gr] = ldexpf(1.f, -e);
        __half2 hh[4], ll[4];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
            const float v0 = v[i] * s, v1 = v[i + 1] * s;
            hh[i / 2] = __float22half2_rn(make_float2(v0, v1));
            const float2 hf = __half22float2(hh[i / 2]);
            ll[i / 2] = __float22half2_rn(make_float2(v0 - hf.x, v1 - hf.y));
        }
        const int64_t o = gr * ldc + gc0;
        if (gc0 + 8 <= N && (ldc & 7) == 0) {
            *reinterpret_cast<uint4 *>(ch + o) = *reinterpret_cast<const uint4 *>(hh);
            *reinterpret_cast<uint4 *>(cl + o) = *reinterpret_cast<const uint4 *>(ll);
        } else {
            const __half *ph = reinterpret_cast<const __half *>(hh), *pl = reinterpret_cast<const __half *>(ll);
            for (int i = 0; i < 8 && gc0 + i < N; i++) {
                ch[o + i] = ph[i];
                cl[o + i] = pl[i];
            }
        }
    }
}

static bool store_tail_split_enabled() {  // A/B knob: GVT_STORE_TAIL_SPLIT=0 keeps stage 1's last wave unsplit
    static const bool on = [] {
        const char *e = getenv("GVT_STORE_TAIL_SPLIT");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

// hi/lo: M rows x ldc halves; sk: ceil(N/256) chunk rows x sk_ld (>= round_up(M, 256) / S16_SCALE_ROWS)
// floats, whose padding the caller keeps finite (stage 2 reads it against zero accumulators)
void gemm_nt_store16(gvt_ctx *c, const Operand &A, const Operand &B, int64_t M, int64_t N, int64_t K, __half *hi,
                     __half *lo, int64_t ldc, float *sk, int64_t sk_ld, const int32_t *kb_list,
                     const int32_t *kb_off, const int32_t *tile_order, int kb_min_chunks) {
    EpiParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.kb_list = kb_list;
    ep.kb_off = kb_off;
    ep.c_h16 = hi;
    ep.c_l16 = lo;
    ep.c_sk = sk;
    ep.c_sk_ld = sk_ld;
    ep.ldc = ldc;
    // tail split of the last partial wave (as the sampled GEMM's): r <= pairs / 2 leftover tiles in s K parts
    const int pairs = c->sm_count / 2;
    const int num_mp = (int)((M + 2 * BM - 1) / (2 * BM)), num_n = (int)((N + BN - 1) / BN);
    const int n_tiles = num_mp * num_n, r = n_tiles % pairs;
    int split = 1;
    // (block-sparse K lists: the caller passes their fewest chunks per tile, kb_min_chunks, from the plan's host
    // lists -- this runs inside the solver's graph capture, where no host read-back is possible)
    const int nch_min = kb_list ? kb_min_chunks : (int)((K + BN - 1) / BN);
    if (S16_SCALE_ROWS == 1 && c->gemm_cta == 2 && n_tiles >= pairs && r > 0 && 2 * r <= pairs &&
        store_tail_split_enabled())
        split = std::min(4, std::min(pairs / r, nch_min / 2));
    if (tile_order) {  // a caller's tile order (the longest K lists first), as whole units unless split below
        ep.tile_list = tile_order;
        ep.n_whole = n_tiles;
        ep.split = 1;
        ep.n_units = n_tiles;
    }
    if (split >= 2) {
        ep.n_whole = n_tiles - r;
        ep.split = split;
        ep.n_units = ep.n_whole + r * split;
        ep.part = wsT<float>(c, "store16.tail", (size_t)split * r * 2 * BM * BN);
    }
    launch_gemm<EPI_STORE16>(c, K_STAGE1_TC, A, B, M, N, K, ep);
    if (split >= 2) {
        static const int env_gm = [] {
            const char *e = getenv("GVT_GROUP_M");
            return e ? atoi(e) : 0;
        }();
        const int gm = env_gm > 0 ? env_gm : GROUP_M;
        static_assert(BM == 16 * 8, "fixup: 16 blocks of 8 rows per m half");
        GVT_LAUNCH(c, K_STAGE1_TC, k_store16_fixup, 32 * r, 256, 0, ep.part, split, r, ep.n_whole, tile_order, num_mp,
                   num_n, gm, M,
                   N, A.scale, B.scale, hi, lo, ldc, sk, sk_ld);
    }
}

__global__ void k_add_diag(float *__restrict__ X, int64_t ldX, const float *__restrict__ diag, int64_t row_lo,
                           int64_t rows) {
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows; r += (int64_t)gridDim.x * blockDim.x)
        X[r * ldX + row_lo + r] += diag[row_lo + r];
}

void add_diag(gvt_ctx *c, float *X, int64_t ldX, const float *diag, int64_t row_lo, int64_t rows) {
    if (rows <= 0) return;
    GVT_LAUNCH(c, K_DENSIFY, k_add_diag, grid1d(rows, 256), 256, 0, X, ldX, diag, row_lo, rows);
}

// X[row][col] = sum of the (row, col) run of sorted entries (deterministic, in entry order)
__global__ void k_densify(const int32_t *__restrict__ row, const int32_t *__restrict__ col,
                          const float *__restrict__ val, int64_t k0, int64_t k1, int64_t row_lo,
                          float *__restrict__ X, int64_t ldX) {
    for (int64_t k = k0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < k1; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t r = row[k], cc = col[k];
        if (k > k0 && row[k - 1] == r && col[k - 1] == cc) continue;  // not the head of its run
        float s = val[k];
        for (int64_t j = k + 1; j < k1 && row[j] == r && col[j] == cc; j++) s += val[j];
        X[(int64_t)(r - row_lo) * ldX + cc] = s;
    }
}

void densify(gvt_ctx *c, const EntryPlan &e, int64_t k0, int64_t k1, int64_t row_lo, float *X, int64_t ldX,
             int64_t rows_pad) {
    GVT_CUDA_TRY(cudaMemsetAsync(X, 0, sizeof(float) * rows_pad * ldX, c->stream));
    if (k1 <= k0) return;
    GVT_LAUNCH(c, K_DENSIFY, k_densify, grid1d(k1 - k0, 256, 16 * c->sm_count * 8), 256, 0, e.row, e.col, e.val, k0,
               k1, row_lo, X, ldX);
}

void gemm_nt_store(gvt_ctx *c, const Operand &A, const Operand &B, int64_t M, int64_t N, int64_t K, float *Cf,
                   int64_t ldc, float *Chi, float *Clo) {
    EpiParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.c_f = Cf;
    ep.c_hi = Chi;
    ep.c_lo = Clo;
    ep.ldc = ldc;
    launch_gemm<EPI_STORE>(c, K_STAGE1_TC, A, B, M, N, K, ep);
}

// split-K parts of the sampled GEMM summed per sample in part order, then the sampled epilogue's store
__global__ void k_split_combine(const float *__restrict__ part, int split, int64_t ns, const int32_t *__restrict__ dst,
                                float coef, int accumulate, float *__restrict__ out) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ns; k += (int64_t)gridDim.x * blockDim.x) {
        float v = part[k];
        for (int h = 1; h < split; h++) v += part[(int64_t)h * ns + k];
        const int32_t d = dst[k];
        out[d] = accumulate ? fmaf(coef, v, out[d]) : coef * v;
    }
}

// tail split: the parts of the samples of the split tiles only (tile_list[n_whole ..)); an M-tile of a split
// tile holds one contiguous run of bucketed sample slots
__global__ void k_split_combine_tail(const float *__restrict__ part, int split, int64_t ns,
                                     const int32_t *__restrict__ tiles, int n_whole, int64_t n_rt, int64_t n_ct,
                                     const int64_t *__restrict__ tile_ptr, const int32_t *__restrict__ dst, float coef,
                                     int accumulate, float *__restrict__ out) {
    // block b: split tile b / 32, M-tile half (b / 16) & 1, slice b % 16 of that M-tile's sample run
    const int32_t tl = tiles[n_whole + blockIdx.x / 32];
    const int64_t m_tile = 2 * (int64_t)(tl / n_ct) + ((blockIdx.x >> 4) & 1), n = tl % n_ct;
    if (m_tile >= n_rt) return;
    const int64_t t = m_tile * n_ct + n;
    const int64_t kb = tile_ptr[t * (BN / 32)], ke = tile_ptr[(t + 1) * (BN / 32)];
    for (int64_t k = kb + (int64_t)(blockIdx.x & 15) * blockDim.x + threadIdx.x; k < ke; k += 16 * (int64_t)blockDim.x) {
        float v = part[k];
        for (int h = 1; h < split; h++) v += part[(int64_t)h * ns + k];
        const int32_t dd = dst[k];
        out[dd] = accumulate ? fmaf(coef, v, out[dd]) : coef * v;
    }
}

static int64_t tail_split_part_limit() {  // bytes per part buffer (all ns slots); GVT_TAIL_SPLIT_MB overrides
    static const int64_t lim = [] {
        const char *e = getenv("GVT_TAIL_SPLIT_MB");
        return (e ? atoll(e) : 64ll) << 20;
    }();
    return lim;
}

static bool tail_split_enabled() {  // A/B knob: GVT_TAIL_SPLIT=0 keeps the last partial wave unsplit
    static const bool on = [] {
        const char *e = getenv("GVT_TAIL_SPLIT");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

// K parts per non-empty pair tile: when at most half of the CTA pairs would have a tile, each tile's
// K range is split (at accumulation-chunk boundaries, >= 2 chunks per part) so every pair works --
// C3's upper-triangle samples leave ~36 of 64 pair tiles non-empty on 74 CTA pairs.  GVT_SPLITK=0: off.
static bool compact_tiles() {  // A/B knob: GVT_COMPACT_TILES=0 strides over all pair tiles (round-1 loop)
    static const bool on = [] {
        const char *e = getenv("GVT_COMPACT_TILES");
        return !(e && atoi(e) == 0);
    }();
    return on;
}

static int sampled_split(gvt_ctx *c, const SamplePlan &sp, int64_t K) {
    static const int env = [] {
        const char *e = getenv("GVT_SPLITK");
        return e ? atoi(e) : -1;
    }();
    if (env == 0 || c->gemm_cta != 2 || !sp.pair_list || sp.n_pairs <= 0) return 1;
    const int clusters = c->sm_count / 2;
    const int nch = (int)((K + BN - 1) / BN);
    int split = clusters / sp.n_pairs;
    split = std::min(split, std::min(4, nch / 2));
    if (env > 0) split = std::min(env, std::max(1, nch / 2));
    return split >= 2 ? split : 1;
}

int gemm_group_m() {
    static const int env_gm = [] {
        const char *e = getenv("GVT_GROUP_M");
        return e ? atoi(e) : 0;
    }();
    return env_gm > 0 ? env_gm : GROUP_M;
}

int sampled_split_parts(gvt_ctx *c, const SamplePlan &sp, int64_t K) { return sp.ns > 0 ? sampled_split(c, sp, K) : 1; }

void gemm_nt_sampled(gvt_ctx *c, const Operand &A, const Operand &B, int64_t M, int64_t N, int64_t K,
                     const SamplePlan &sp, float coef, int accumulate, float *out, SplitParts *defer) {
    const int slot = defer ? defer->slot : 0;
    if (defer) {
        *defer = SplitParts();
        defer->slot = slot;
    }
    if (sp.ns == 0) return;
    EpiParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.s_r = sp.r;
    ep.s_c = sp.c;
    ep.s_dst = sp.dst;
    ep.chunk_ptr = sp.tile_ptr;
    ep.n_ct = sp.n_ct;
    ep.coef = coef;
    ep.accumulate = accumulate;
    ep.out = out;
    const int split = sampled_split(c, sp, K);
    const int64_t npt = ((sp.n_rt + 1) / 2) * sp.n_ct;
    int tail_split = 1;
    if (split > 1) {
        ep.tile_list = sp.pair_list;
        ep.split = split;
        ep.n_units = sp.n_pairs * split;
        ep.n_whole = 0;
        ep.ns = sp.ns;
        ep.part = wsT<float>(c, slot ? "splitk.part1" : "splitk.part", (size_t)split * sp.ns);
    } else if (sp.pair_list && sp.n_pairs > 0 && compact_tiles()) {
        // the persistent loop over the non-empty tiles (every CTA pair gets the same number of whole tiles;
        // striding over all tiles left pairs with several non-empty tiles next to pairs with none), and a
        // last partial wave of r <= pairs / 2 tiles split into s K parts, so that wave costs 1/s of a tile
        // (C4: 240 tiles on 74 pairs = 3 waves + 18 tiles -> 18 x 4 parts).  Parts cost s x ns floats of
        // workspace: only for out samples of at most 64 MB per part.
        const int pairs = c->sm_count / 2, r = sp.n_pairs % pairs;
        const int nch = (int)((K + BN - 1) / BN);
        if (sp.n_pairs >= pairs && r > 0 && 2 * r <= pairs && tail_split_enabled() &&
            sp.ns * (int64_t)sizeof(float) <= tail_split_part_limit())
            tail_split = std::min(4, std::min(pairs / r, nch / 2));
        if (tail_split >= 2) {
            ep.tile_list = sp.pair_list;
            ep.split = tail_split;
            ep.n_whole = sp.n_pairs - r;
            ep.n_units = ep.n_whole + r * tail_split;
            ep.ns = sp.ns;
            ep.part = wsT<float>(c, "splitk.tail", (size_t)tail_split * sp.ns);
        } else if (sp.n_pairs < npt) {
            tail_split = 1;
            ep.tile_list = sp.pair_list;
            ep.split = 1;
            ep.n_units = sp.n_pairs;
            ep.n_whole = sp.n_pairs;
        } else {
            tail_split = 1;
        }
    }
    launch_gemm<EPI_SAMPLED>(c, K_STAGE2_TC, A, B, M, N, K, ep);
    if (tail_split > 1) {  // (never deferred: only the split tiles' samples have parts)
        const int r = sp.n_pairs - ep.n_whole;
        GVT_LAUNCH(c, K_STAGE2_TC, k_split_combine_tail, 32 * r, 256, 0, ep.part, tail_split, sp.ns, sp.pair_list,
                   ep.n_whole, sp.n_rt, sp.n_ct, sp.tile_ptr, sp.dst, coef, accumulate, out);
    }
    if (split > 1 && defer) {
        defer->part = ep.part;
        defer->split = split;
        defer->ns = sp.ns;
        defer->dst = sp.dst;
        defer->coef = coef;
        defer->accumulate = accumulate;
    } else if (split > 1)
        GVT_LAUNCH(c, K_STAGE2_TC, k_split_combine, grid1d(sp.ns, 256, 8 * c->sm_count), 256, 0, ep.part, split, sp.ns,
                   sp.dst, coef, accumulate, out);
}

// ----------------------------------------------------------------------------- sample bucketing
// the CTA-pair tiles (M-tiles 2 mp, 2 mp + 1 x N-tile n) holding samples, in the kernel's grouped
// rasterization order (GROUP_M pair rows per group, as coords()), and their count at list[n_mp * n_ct]:
// one CTA, 256 tiles per step (flags, then a block scan keeps the order)
__global__ void __launch_bounds__(256) k_pair_list(const int64_t *__restrict__ tile_ptr, int64_t n_rt, int64_t n_ct,
                                                   int32_t *__restrict__ list) {
    using Scan = cub::BlockScan<int, 256>;
    __shared__ typename Scan::TempStorage tmp;
    __shared__ int base;
    const int64_t n_mp = (n_rt + 1) / 2, npt = n_mp * n_ct, in_group = (int64_t)GROUP_M * n_ct;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    for (int64_t t0 = 0; t0 < npt; t0 += 256) {
        const int64_t t = t0 + threadIdx.x;
        int flag = 0, tl = 0;
        if (t < npt) {
            const int64_t first_m = (t / in_group) * GROUP_M, group_m = min(n_mp - first_m, (int64_t)GROUP_M);
            const int64_t mp = first_m + (t % in_group) % group_m, n = (t % in_group) / group_m;
            const int64_t a0 = (2 * mp) * n_ct + n, a1 = a0 + n_ct;
            const bool e0 = tile_ptr[a0 * (BN / 32)] == tile_ptr[(a0 + 1) * (BN / 32)];
            const bool e1 = !(2 * mp + 1 < n_rt) || tile_ptr[a1 * (BN / 32)] == tile_ptr[(a1 + 1) * (BN / 32)];
            flag = !(e0 && e1);
            tl = (int)(mp * n_ct + n);
        }
        int pos, total;
        Scan(tmp).ExclusiveSum(flag, pos, total);
        if (flag) list[base + pos] = tl;
        __syncthreads();
        if (threadIdx.x == 0) base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) list[npt] = base;
}

// key = ((r / BM) * n_ct + c / BN) * (BN/32) + (c % BN) / 32 ; stable sort keeps r-order inside
__global__ void k_bucket_keys(const int32_t *__restrict__ r, const int32_t *__restrict__ cc, int64_t ns, int64_t n_ct,
                              uint32_t *__restrict__ keys, int32_t *__restrict__ vals) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ns; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t rt = r[k] / BM, ct = cc[k] / BN, ch = (cc[k] % BN) / 32;
        keys[k] = (uint32_t)((rt * n_ct + ct) * (BN / 32) + ch);
        vals[k] = (int32_t)k;
    }
}

__global__ void k_bucket_apply(const int32_t *__restrict__ order, int64_t ns, const int32_t *__restrict__ r,
                               const int32_t *__restrict__ cc, const int32_t *__restrict__ dst,
                               int32_t *__restrict__ r2, int32_t *__restrict__ c2, int32_t *__restrict__ d2) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < ns; k += (int64_t)gridDim.x * blockDim.x) {
        const int32_t o = order[k];
        r2[k] = r[o];
        c2[k] = cc[o];
        d2[k] = dst[o];
    }
}

__global__ void k_bucket_ptr(const uint32_t *__restrict__ skeys, int64_t ns, int64_t nb, int64_t *__restrict__ ptr) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = ns;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if ((int64_t)skeys[mid] < b) lo = mid + 1;
            else hi = mid;
        }
        ptr[b] = lo;
    }
}

void bucket_samples(gvt_ctx *c, const char *tag, SamplePlan &sp, int64_t nrow, int64_t ncol) {
    std::string t(tag);
    sp.n_rt = (nrow + BM - 1) / BM;
    sp.n_ct = (ncol + BN - 1) / BN;
    const int64_t nb = sp.n_rt * sp.n_ct * (BN / 32);
    GVT_REQUIRE(nb < (int64_t)UINT32_MAX, GVT_E_DIM, "too many sample buckets");
    sp.tile_ptr = wsT<int64_t>(c, (t + ".chunkptr").c_str(), nb + 1);
    const int64_t ns = sp.ns;
    if (ns > 0) {
        uint32_t *k0 = wsT<uint32_t>(c, "bucket.k0", ns), *k1 = wsT<uint32_t>(c, "bucket.k1", ns);
        int32_t *v0 = wsT<int32_t>(c, "bucket.v0", ns), *v1 = wsT<int32_t>(c, "bucket.v1", ns);
        GVT_LAUNCH(c, K_PLAN_KEYS, k_bucket_keys, grid1d(ns, 256, 4096), 256, 0, sp.r, sp.c, ns, sp.n_ct, k0, v0);
        size_t temp = 0;
        int bits = 1;
        while (bits < 32 && ((uint64_t)nb >> bits)) bits++;
        GVT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp, k0, k1, v0, v1, (int)ns, 0, bits, c->stream));
        void *tmp = ws(c, "bucket.tmp", temp);
        cudaEvent_t ev;
        launch_begin(c, K_PLAN_SORT, &ev);
        GVT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, temp, k0, k1, v0, v1, (int)ns, 0, bits, c->stream));
        launch_end(c, K_PLAN_SORT, ev);
        int32_t *r2 = wsT<int32_t>(c, (t + ".br").c_str(), ns), *c2 = wsT<int32_t>(c, (t + ".bc").c_str(), ns),
                *d2 = wsT<int32_t>(c, (t + ".bd").c_str(), ns);
        GVT_LAUNCH(c, K_PLAN_GATHER, k_bucket_apply, grid1d(ns, 256, 4096), 256, 0, v1, ns, sp.r, sp.c, sp.dst, r2, c2,
                   d2);
        sp.r = r2;
        sp.c = c2;
        sp.dst = d2;
        GVT_LAUNCH(c, K_PLAN_ROWPTR, k_bucket_ptr, grid1d(nb + 1, 256), 256, 0, k1, ns, nb, sp.tile_ptr);
    } else {
        GVT_CUDA_TRY(cudaMemsetAsync(sp.tile_ptr, 0, sizeof(int64_t) * (nb + 1), c->stream));
    }
    // the non-empty CTA-pair tiles, for the split-K sampled GEMM and for balancing the persistent loop over
    // non-empty tiles only (one read-back)
    sp.pair_list = nullptr;
    sp.n_pairs = -1;
    const int64_t n_mp = (sp.n_rt + 1) / 2, npt = n_mp * sp.n_ct;
    if (ns > 0 && c->gemm_cta == 2) {
        int32_t *list = wsT<int32_t>(c, (t + ".pairs").c_str(), (size_t)npt + 1);
        GVT_LAUNCH(c, K_PLAN_ROWPTR, k_pair_list, 1, 256, 0, sp.tile_ptr, sp.n_rt, sp.n_ct, list);
        int32_t *h = (int32_t *)pinned(c, sizeof(int32_t));
        GVT_CUDA_TRY(cudaMemcpyAsync(h, list + npt, sizeof(int32_t), cudaMemcpyDeviceToHost, c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
        sp.pair_list = list;
        sp.n_pairs = *h;
    }
}

// ----------------------------------------------------------------------------- Gram
__global__ void k_norms(const float *__restrict__ X, int64_t m, int64_t dim, float *__restrict__ nrm) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t i = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < m; i += warps) {
        float acc = 0.f;
        for (int64_t k = lane; k < dim; k += 32) acc = fmaf(X[i * dim + k], X[i * dim + k], acc);
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) nrm[i] = acc;
    }
}

// K (m x m2, ldk) = k(X_i, Y_j) on the tensor cores; Y == nullptr: the Gram of X (diagonal of the
// Gaussian exactly 1)
void gram_tc(gvt_ctx *c, int kind, const float *X, int64_t m, const float *Y, int64_t m2, int64_t dim, double gamma,
             double coef0, int degree, float *K, int64_t ldk) {
    if (m == 0 || m2 == 0) return;
    const bool same = Y == nullptr;
    const int64_t ldx = round_up(dim, 32), rows = round_up(m, 128), rows2 = round_up(m2, 128);
    float *xp = wsT<float>(c, "gram.xp", rows * ldx);
    float *nr = wsT<float>(c, "gram.norms", rows);
    pad_copy(c, X, m, dim, dim, xp, ldx, rows);
    Operand xo = make_operand(c, "gram.x", xp, m, dim, ldx, ldx, rows);
    Operand yo = xo;
    float *nr2 = nr;
    if (!same) {
        float *yp = wsT<float>(c, "gram.yp", rows2 * ldx);
        nr2 = wsT<float>(c, "gram.norms2", rows2);
        pad_copy(c, Y, m2, dim, dim, yp, ldx, rows2);
        yo = make_operand(c, "gram.y", yp, m2, dim, ldx, ldx, rows2);
    }
    if (kind == GVT_BASE_GAUSSIAN) {
        GVT_LAUNCH(c, K_GRAM_TC, k_norms, grid1d(m * 32, 256, 4096), 256, 0, X, m, dim, nr);
        if (!same) GVT_LAUNCH(c, K_GRAM_TC, k_norms, grid1d(m2 * 32, 256, 4096), 256, 0, Y, m2, dim, nr2);
    }
    EpiParams ep;
    memset(&ep, 0, sizeof(ep));
    ep.c_f = K;
    ep.ldc = ldk;
    ep.norms = nr;
    ep.norms_b = nr2;
    ep.same = same ? 1 : 0;
    ep.kind = kind;
    ep.gamma = (float)gamma;
    ep.coef0 = (float)coef0;
    ep.degree = degree;
    ep.kcb = 1;  // short K (feature dim): one K-block per fp32 round-to-nearest drain
    launch_gemm<EPI_GRAM>(c, K_GRAM_TC, xo, yo, m, m2, dim, ep);
}

}  // namespace gvt
