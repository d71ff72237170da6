// gvt_internal.cuh -- shared internals of libgvt.so (context, workspaces, launch
// accounting, error helpers).  Not part of the ABI (see include/gvt.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/gvt.h"

namespace gvt {

// ----------------------------------------------------------------------------- errors
void set_error(const char *fmt, ...);

struct Error {
    gvt_status code;
    std::string msg;
};

#define GVT_CUDA_TRY(expr)                                                                         \
    do {                                                                                           \
        cudaError_t _e = (expr);                                                                   \
        if (_e != cudaSuccess) {                                                                   \
            if (_e == cudaErrorMemoryAllocation)                                                   \
                throw ::gvt::Error{GVT_E_OOM, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
            throw ::gvt::Error{GVT_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)};    \
        }                                                                                          \
    } while (0)

#define GVT_REQUIRE(cond, code, text)                          \
    do {                                                       \
        if (!(cond)) throw ::gvt::Error{(code), std::string(text)}; \
    } while (0)

// ----------------------------------------------------------------------------- kernels kinds
enum KernelKind {
    K_GRAM_SIMT = 0,
    K_GRAM_TC,
    K_SPLIT,
    K_PAD_COPY,
    K_PLAN_KEYS,
    K_PLAN_SORT,
    K_PLAN_ROWPTR,
    K_PLAN_GATHER,
    K_STAGE1_SPARSE,
    K_STAGE2_GATHER,
    K_DENSIFY,
    K_STAGE1_TC,
    K_STAGE2_TC,
    K_SEGSUM,
    K_GEMV,
    K_COMBINE,
    K_CARTESIAN,
    K_CG_VEC,
    K_CG_SCALAR,
    K_FILL,
    K_AUC,
    K_TINY,
    K_COMM,  // collectives (NCCL calls or host-twin exchanges): counted and timed, not library launches
    K_NUM_KINDS
};
const char *kind_name(int k);

// ----------------------------------------------------------------------------- device buffer
struct Buf {
    void *ptr = nullptr;
    size_t bytes = 0;
};

struct PendingEvent {
    int kind;
    cudaEvent_t start, stop;
};

}  // namespace gvt

struct gvt_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    int sm_count = 148;
    int cc_major = 0, cc_minor = 0;
    bool tc_ok = false;  // tcgen05 path usable (sm_100)

    // options
    int engine = 0;  // 0 auto, 1 sparse, 2 dense, 3 single-CTA whole-fit solver (small Kronecker fits)
    double dense_threshold = -1.0;  // < 0: engine by estimated time (dense_pays); >= 0: density rule
    int profile = 0;
    int gram_engine = 0;
    int tc_precision = 0;  // 0 = 3xFP16 with row scaling, 1 = 3xTF32
    int slabs = 1;         // emulated X-row slabs at world 1 (tests the data-parallel slab path)
    int gemm_cta = 2;      // tensor-core GEMM: 2 = CTA-pair tcgen05 (cta_group::2), 1 = single CTA
    int graphs = 1;        // CUDA-graph replay of the solver iteration
    int solver = 0;        // GVT_SOLVER_CG / GVT_SOLVER_MINRES
    int exchange = 2;      // multi-GPU: 0 = S slab all-gather, 1 = u reduce (NEXT-3), 2 = by estimated bytes
    int sorted_fit = 1;    // fits run on the pairs sorted by (first, second)
    int kblock_skip = 1;   // block-sparse stage 1 (skip all-zero K-blocks of X) where it pays
    int stage2 = 0;        // dense-engine stage 2: 0 = by estimated time, 1 = sampled GEMM, 2 = gather
    int compact = 1;       // used-object compaction: 0 off, 1 auto (tables > 2^20 cells), 2 always
    int cg_variant = 0;    // 0 = Hestenes-Stiefel CG, 1 = Chronopoulos-Gear (one reduction per iteration)
    cudaStream_t cap_stream = nullptr;  // side stream used only for graph capture
    int last_engine = 0;
    int last_exchange = 0;  // 0 none (single GPU), 1 S slab all-gather, 2 u-exchange

    // workspaces by name (grow-only)
    std::unordered_map<std::string, gvt::Buf> bufs;

    // launch accounting
    int64_t launches = 0;
    int64_t counts[gvt::K_NUM_KINDS] = {0};
    double ms[gvt::K_NUM_KINDS] = {0};
    std::vector<gvt::PendingEvent> pending;
    std::vector<cudaEvent_t> event_pool;

    // multi-GPU
    void *nccl_comm = nullptr;
    int rank = 0, world = 1;
    gvt_host_allgather_fn host_allgather = nullptr;  // host-mediated communicator (gvt_comm_init_host)
    void *host_user = nullptr;
    cudaStream_t comm_stream = nullptr;        // side stream of the pipelined slab exchange
    std::vector<cudaEvent_t> slab_events;      // [world] slab s arrived, [world] fork point

    // the last Hestenes-Stiefel CG fit's search direction (gvt_solver_direction): device vector
    // in solve order, its length (-1 = none kept) and the sorted-order permutation (nullptr = identity)
    float *last_p = nullptr;
    int64_t last_n = -1;
    const int32_t *last_perm = nullptr;

    // pinned host scratch for scalar read-backs
    void *pinned = nullptr;
    size_t pinned_bytes = 0;
};

namespace gvt {

// workspace with at least `bytes`; contents undefined.  Same name => same buffer (realloc on grow).
void *ws(gvt_ctx *c, const char *name, size_t bytes);
template <typename T>
T *wsT(gvt_ctx *c, const char *name, size_t count) {
    return reinterpret_cast<T *>(ws(c, name, (count ? count : 1) * sizeof(T)));
}
void *pinned(gvt_ctx *c, size_t bytes);

// launch accounting: call around every kernel launch
void launch_begin(gvt_ctx *c, int kind, cudaEvent_t *ev_start);
void launch_end(gvt_ctx *c, int kind, cudaEvent_t ev_start);
void collect_events(gvt_ctx *c);  // synchronises pending profile events

#define GVT_LAUNCH(ctx, kind, kernel, grid, block, smem, ...)                      \
    do {                                                                           \
        cudaEvent_t _ev0 = nullptr;                                                \
        ::gvt::launch_begin((ctx), (kind), &_ev0);                                 \
        kernel<<<(grid), (block), (smem), (ctx)->stream>>>(__VA_ARGS__);           \
        GVT_CUDA_TRY(cudaGetLastError());                                          \
        ::gvt::launch_end((ctx), (kind), _ev0);                                    \
    } while (0)

// host/device classification of a caller pointer
bool is_device_ptr(const void *p);

// stage a caller array on the device: returns a device pointer (caller's if already
// device memory, else a workspace copy made on the context stream)
const void *stage_in(gvt_ctx *c, const char *name, const void *p, size_t bytes);

constexpr int GVT_MAX_DEVICES = 64;

// data-parallel mode: a communicator spans several ranks, or NCCL was forced at world 1
// (gvt_comm_init with a unique id and world 1: the NCCL data plane runs with one rank)
inline bool distributed(const gvt_ctx *c) { return c->world > 1 || c->nccl_comm != nullptr; }

inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }
inline unsigned grid1d(int64_t n, int threads, int64_t cap = 1 << 30) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > cap) g = cap;
    return (unsigned)g;
}

}  // namespace gvt
