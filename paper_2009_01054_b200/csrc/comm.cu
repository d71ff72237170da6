// comm.cu -- NCCL plumbing for the data-parallel path: all-gather of
// the S column slabs and of the CG dot-product partials.  NCCL is loaded with dlopen at
// gvt_comm_init time so single-GPU use never depends on it (the process may already have
// torch's libnccl.so.2 loaded, which dlopen then reuses).
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <algorithm>

#include "ops.cuh"

namespace gvt {

struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void *, void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t,
                           cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;

static void load_nccl() {
    if (g_nccl.h) return;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    GVT_REQUIRE(h, GVT_E_NCCL, std::string("cannot dlopen libnccl.so.2: ") + dlerror());
    g_nccl.GetUniqueId = (decltype(g_nccl.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.CommInitRank = (decltype(g_nccl.CommInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.CommDestroy = (decltype(g_nccl.CommDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.AllGather = (decltype(g_nccl.AllGather))dlsym(h, "ncclAllGather");
    g_nccl.GetErrorString = (decltype(g_nccl.GetErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.Broadcast = (decltype(g_nccl.Broadcast))dlsym(h, "ncclBroadcast");
    g_nccl.GroupStart = (decltype(g_nccl.GroupStart))dlsym(h, "ncclGroupStart");
    g_nccl.GroupEnd = (decltype(g_nccl.GroupEnd))dlsym(h, "ncclGroupEnd");
    g_nccl.Reduce = (decltype(g_nccl.Reduce))dlsym(h, "ncclReduce");
    g_nccl.AllReduce = (decltype(g_nccl.AllReduce))dlsym(h, "ncclAllReduce");
    g_nccl.Send = (decltype(g_nccl.Send))dlsym(h, "ncclSend");
    g_nccl.Recv = (decltype(g_nccl.Recv))dlsym(h, "ncclRecv");
    GVT_REQUIRE(g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.AllGather &&
                    g_nccl.Broadcast && g_nccl.GroupStart && g_nccl.GroupEnd && g_nccl.Reduce && g_nccl.AllReduce &&
                    g_nccl.Send && g_nccl.Recv,
                GVT_E_NCCL, "libnccl.so.2 lacks a required symbol");
    g_nccl.h = h;
}

// accounting of one collective (kind "collective": count, and CUDA-event time when profiling)
struct Coll {
    gvt_ctx *c;
    cudaEvent_t ev = nullptr;
    explicit Coll(gvt_ctx *ctx) : c(ctx) { launch_begin(c, K_COMM, &ev); }
    void done() { launch_end(c, K_COMM, ev); }
};

#define NCCL_TRY(expr)                                                                                  \
    do {                                                                                                \
        ncclResult_t _r = (expr);                                                                       \
        if (_r != ncclSuccess)                                                                          \
            throw Error{GVT_E_NCCL, std::string(#expr) + ": " +                                         \
                                        (g_nccl.GetErrorString ? g_nccl.GetErrorString(_r) : "error")}; \
    } while (0)

void nccl_unique_id(void *out128) {
    load_nccl();
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    NCCL_TRY(g_nccl.GetUniqueId(&id));
    memcpy(out128, &id, sizeof(id));
}

void comm_destroy(gvt_ctx *c);

// world 1 without a unique id: no communicator (single-GPU mode).  world 1 WITH a unique id: a
// one-rank NCCL communicator, and the library runs its data-parallel path with real NCCL calls
// (all-gathers, grouped broadcasts, send/recv, all-reduces) on one GPU -- the executed check of
// the NCCL data plane that a one-GPU box allows.
void comm_init(gvt_ctx *c, const void *id128, int rank, int world) {
    GVT_REQUIRE(world >= 1 && rank >= 0 && rank < world, GVT_E_PARAM, "comm_init: bad rank/world");
    comm_destroy(c);
    c->host_allgather = nullptr;
    if (world == 1 && !id128) {
        c->rank = 0;
        c->world = 1;
        return;
    }
    load_nccl();
    ncclUniqueId id;
    memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    NCCL_TRY(g_nccl.CommInitRank(&comm, world, id, rank));
    c->nccl_comm = comm;
    c->rank = rank;
    c->world = world;
}

void comm_destroy(gvt_ctx *c) {
    if (c->nccl_comm && g_nccl.CommDestroy) g_nccl.CommDestroy((ncclComm_t)c->nccl_comm);
    c->nccl_comm = nullptr;
    for (auto e : c->slab_events) cudaEventDestroy(e);
    c->slab_events.clear();
    if (c->comm_stream) cudaStreamDestroy(c->comm_stream);
    c->comm_stream = nullptr;
}

// Pipelined S slab exchange ("stage 2 accumulates the partial dots of each slab as
// it arrives, pipelined over slabs on a side stream"): after stage 1, slab s of every array is
// broadcast from its owner s, in slab order, on the context's comm stream; slab_events[s] marks its
// arrival, and stage 2 of slab s waits only for that event, so the transfer of slab s + 1 overlaps
// the stage-2 GEMM of slab s.  The waits of stage 2 join the side stream back (also inside a CUDA
// graph capture, where the fork/join become graph edges).  NCCL communicators only (the host twin
// exchanges synchronously with allgather_slabs).
bool slab_pipeline_available(gvt_ctx *c) { return distributed(c) && c->nccl_comm && !c->host_allgather; }

void slab_pipeline_start(gvt_ctx *c, void *const *bufs, const size_t *slab_bytes, int nbuf) {
    const int G = c->world;
    if (!c->comm_stream) GVT_CUDA_TRY(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    while ((int)c->slab_events.size() < G + 1) {
        cudaEvent_t e;
        GVT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        c->slab_events.push_back(e);
    }
    GVT_CUDA_TRY(cudaEventRecord(c->slab_events[G], c->stream));  // fork: stage 1 of this rank is done
    GVT_CUDA_TRY(cudaStreamWaitEvent(c->comm_stream, c->slab_events[G], 0));
    for (int s = 0; s < G; s++) {
        c->counts[K_COMM]++;
        NCCL_TRY(g_nccl.GroupStart());
        for (int b = 0; b < nbuf; b++) {
            char *slab = (char *)bufs[b] + (size_t)s * slab_bytes[b];
            if (slab_bytes[b])
                NCCL_TRY(g_nccl.Broadcast(slab, slab, slab_bytes[b], ncclInt8, s, (ncclComm_t)c->nccl_comm,
                                          c->comm_stream));
        }
        NCCL_TRY(g_nccl.GroupEnd());
        GVT_CUDA_TRY(cudaEventRecord(c->slab_events[s], c->comm_stream));
    }
}

void slab_wait(gvt_ctx *c, int s) { GVT_CUDA_TRY(cudaStreamWaitEvent(c->stream, c->slab_events[s], 0)); }

// ---- host-mediated communicator (gvt_comm_init_host): one all-gather primitive through the host
void comm_init_host(gvt_ctx *c, int rank, int world, gvt_host_allgather_fn fn, void *user) {
    GVT_REQUIRE(world >= 1 && rank >= 0 && rank < world && fn, GVT_E_PARAM, "comm_init_host: bad arguments");
    c->rank = rank;
    c->world = world;
    c->host_allgather = fn;
    c->host_user = user;
}

// dev holds [world][bytes]; this rank's block is valid on entry, every block on return
static void host_allgather(gvt_ctx *c, void *dev, size_t bytes) {
    Coll co(c);
    std::vector<char> h((size_t)c->world * bytes);
    char *mine = h.data() + (size_t)c->rank * bytes;
    if (bytes) {
        GVT_CUDA_TRY(cudaMemcpyAsync(mine, (char *)dev + (size_t)c->rank * bytes, bytes, cudaMemcpyDeviceToHost,
                                     c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    GVT_REQUIRE(c->host_allgather(c->host_user, h.data(), bytes) == 0, GVT_E_NCCL, "host all-gather callback failed");
    if (bytes) {
        GVT_CUDA_TRY(cudaMemcpyAsync(dev, h.data(), h.size(), cudaMemcpyHostToDevice, c->stream));
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    co.done();
}

// partials laid out [world][count]; each rank wrote its own slot; gather all slots so the
// fixed-order reduction over world*count values gives bit-identical scalars on every rank
void allreduce_partials(gvt_ctx *c, double *partials, int count) {
    if (!distributed(c)) return;
    if (c->host_allgather) return host_allgather(c, partials, sizeof(double) * (size_t)count);
    Coll co(c);
    NCCL_TRY(g_nccl.AllGather(partials + (size_t)c->rank * count, partials, (size_t)count, ncclFloat64,
                              (ncclComm_t)c->nccl_comm, c->stream));
    co.done();
}

// S slabs laid out [world][slab_floats]; in-place all-gather of the local slab
void allgather_slabs(gvt_ctx *c, float *S, size_t slab_floats) {
    if (!distributed(c)) return;
    if (c->host_allgather) return host_allgather(c, S, sizeof(float) * slab_floats);
    Coll co(c);
    NCCL_TRY(g_nccl.AllGather(S + (size_t)c->rank * slab_floats, S, slab_floats, ncclFloat32,
                              (ncclComm_t)c->nccl_comm, c->stream));
    co.done();
}

// host-visible all-gather of one int64 per rank (plan time only: synchronises)
std::vector<int64_t> allgather_count(gvt_ctx *c, int64_t v) {
    std::vector<int64_t> out((size_t)c->world, v);
    if (!distributed(c)) return out;
    if (c->host_allgather) {
        GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
        GVT_REQUIRE(c->host_allgather(c->host_user, out.data(), sizeof(int64_t)) == 0, GVT_E_NCCL,
                    "host all-gather callback failed");
        return out;
    }
    int64_t *d = wsT<int64_t>(c, "comm.counts", (size_t)c->world);
    GVT_CUDA_TRY(cudaMemcpyAsync(d + c->rank, &v, sizeof(int64_t), cudaMemcpyHostToDevice, c->stream));
    Coll co(c);
    NCCL_TRY(g_nccl.AllGather(d + c->rank, d, 1, ncclInt64, (ncclComm_t)c->nccl_comm, c->stream));
    co.done();
    GVT_CUDA_TRY(cudaMemcpyAsync(out.data(), d, sizeof(int64_t) * c->world, cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return out;
}

// variable-length all-gather: rank g contributes counts[g] elements at offsets[g] of `full`
// (grouped broadcasts, one per root); esz 4 bytes (int32 or float32)
void gather_varlen(gvt_ctx *c, const void *local, void *full, const std::vector<int64_t> &counts,
                   const std::vector<int64_t> &offsets, bool is_float) {
    const size_t esz = 4;
    if (!distributed(c)) {
        if (counts[0] > 0 && local != full)
            GVT_CUDA_TRY(cudaMemcpyAsync(full, local, esz * counts[0], cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    if (c->host_allgather) {  // padded blocks of the largest count, then compacted in rank order
        int64_t mx = 0;
        for (int64_t v : counts) mx = std::max(mx, v);
        char *tmp = (char *)ws(c, "comm.varlen", esz * (size_t)(mx > 0 ? mx : 1) * c->world);
        if (counts[c->rank] > 0)
            GVT_CUDA_TRY(cudaMemcpyAsync(tmp + esz * mx * c->rank, local, esz * counts[c->rank],
                                         cudaMemcpyDeviceToDevice, c->stream));
        host_allgather(c, tmp, esz * (size_t)mx);
        for (int g = 0; g < c->world; g++)
            if (counts[g] > 0)
                GVT_CUDA_TRY(cudaMemcpyAsync((char *)full + esz * offsets[g], tmp + esz * mx * g, esz * counts[g],
                                             cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    Coll co(c);
    NCCL_TRY(g_nccl.GroupStart());
    for (int g = 0; g < c->world; g++) {
        if (counts[g] == 0) continue;
        void *dst = (char *)full + esz * offsets[g];
        NCCL_TRY(g_nccl.Broadcast(g == c->rank ? local : dst, dst, (size_t)counts[g],
                                  is_float ? ncclFloat32 : ncclInt32, g, (ncclComm_t)c->nccl_comm, c->stream));
    }
    NCCL_TRY(g_nccl.GroupEnd());
    co.done();
}

// local[i] = sum_g tmp[g][off + i] (i < cnt), local[cnt + j] = sum_g tmp[g][n_full + j] (j < tail), g in order
__global__ void k_sum_rank_segments(const float *__restrict__ tmp, size_t per, int world, int64_t off, int64_t cnt,
                                    int64_t n_full, int64_t tail, float *__restrict__ local) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cnt + tail; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = i < cnt ? off + i : n_full + (i - cnt);
        float acc = 0.f;
        for (int g = 0; g < world; g++) acc += tmp[(size_t)g * per + src];
        local[i] = acc;
    }
}

void sum_rank_segments(gvt_ctx *c, const float *tmp, size_t per, int world, int64_t off, int64_t cnt, int64_t n_full,
                       int64_t tail, float *local) {
    if (cnt + tail > 0)
        GVT_LAUNCH(c, K_FILL, k_sum_rank_segments, grid1d(cnt + tail, 256, 8 * c->sm_count * 8), 256, 0, tmp, per,
                   world, off, cnt, n_full, tail, local);
}

// u-exchange: every rank holds a partial of the FULL out vector
// (its own S slab's contribution to every output); rank g receives the sum of the segment
// [offsets[g], offsets[g+1]) into `local`, and the `tail` extra values after the full vector
// (MLPK's diagonal samples, needed on every rank) are summed into local + counts[rank].
// The sums run on the device in RANK ORDER (k_sum_rank_segments) on every path, so the NCCL
// path and the host twin give bit-identical results: the NCCL path moves each segment to its
// owner with grouped send/recv (the bytes of a variable-count reduce-scatter: (G-1)/G of the
// partial vector leaves each rank) and all-gathers the tails; no NCCL reduction (whose order
// NCCL chooses) is used.
void reduce_segments(gvt_ctx *c, const float *partial, float *local, const std::vector<int64_t> &counts,
                     const std::vector<int64_t> &offsets, int64_t tail) {
    const int64_t n_full = offsets.back();
    if (!distributed(c)) {
        const int64_t n = counts[0] + tail;
        if (n > 0 && partial != local)
            GVT_CUDA_TRY(cudaMemcpyAsync(local, partial, sizeof(float) * n, cudaMemcpyDeviceToDevice, c->stream));
        return;
    }
    if (c->host_allgather) {  // every rank's full partial, then the rank-order sums of this rank's parts
        const size_t per = (size_t)(n_full + tail);
        float *tmp = (float *)ws(c, "comm.uex", sizeof(float) * (per > 0 ? per : 1) * c->world);
        if (per)
            GVT_CUDA_TRY(cudaMemcpyAsync(tmp + per * c->rank, partial, sizeof(float) * per, cudaMemcpyDeviceToDevice,
                                         c->stream));
        host_allgather(c, tmp, sizeof(float) * per);
        sum_rank_segments(c, tmp, per, c->world, offsets[c->rank], counts[c->rank], n_full, tail, local);
        return;
    }
    const int me = c->rank, G = c->world;
    const int64_t cnt = counts[me];
    float *seg = wsT<float>(c, "comm.uex_seg", (size_t)(cnt > 0 ? cnt : 1) * G);     // [G][cnt]: my segment from g
    float *tl = wsT<float>(c, "comm.uex_tail", (size_t)(tail > 0 ? tail : 1) * G);    // [G][tail]
    if (cnt > 0)
        GVT_CUDA_TRY(cudaMemcpyAsync(seg + (size_t)me * cnt, partial + offsets[me], sizeof(float) * cnt,
                                     cudaMemcpyDeviceToDevice, c->stream));
    Coll co(c);
    NCCL_TRY(g_nccl.GroupStart());
    for (int g = 0; g < G; g++) {
        if (g == me) continue;
        if (counts[g] > 0)
            NCCL_TRY(g_nccl.Send(partial + offsets[g], (size_t)counts[g], ncclFloat32, g, (ncclComm_t)c->nccl_comm,
                                 c->stream));
        if (cnt > 0)
            NCCL_TRY(g_nccl.Recv(seg + (size_t)g * cnt, (size_t)cnt, ncclFloat32, g, (ncclComm_t)c->nccl_comm,
                                 c->stream));
    }
    if (tail > 0)
        NCCL_TRY(g_nccl.AllGather(partial + n_full, tl, (size_t)tail, ncclFloat32, (ncclComm_t)c->nccl_comm,
                                  c->stream));
    NCCL_TRY(g_nccl.GroupEnd());
    co.done();
    // local[i] = sum_g seg[g][i]; local[cnt + j] = sum_g tl[g][j] (rank order)
    sum_rank_segments(c, seg, (size_t)cnt, G, 0, cnt, cnt, 0, local);
    sum_rank_segments(c, tl, (size_t)tail, G, 0, 0, 0, tail, local + cnt);
}

}  // namespace gvt
