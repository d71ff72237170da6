// ctx.cu -- context utilities: error text, workspaces, launch accounting, staging.
#include <stdarg.h>
#include <stdio.h>

#include "gvt_internal.cuh"

namespace gvt {

static thread_local std::string g_last_error;

void set_error(const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
}

const char *last_error() { return g_last_error.c_str(); }

static const char *kKindNames[K_NUM_KINDS] = {
    "gram_simt",   "gram_tc",       "split_operand",  "pad_copy",     "plan_keys",      "plan_sort(cub)",
    "plan_rowptr", "plan_gather",   "stage1_sparse", "stage2_gather", "densify",     "stage1_tc",
    "stage2_tc",   "segment_sum",   "gemv",        "combine",      "cartesian",      "cg_vector",
    "cg_scalar",   "fill",          "auc",          "tiny_cg",       "collective",
};

const char *kind_name(int k) { return (k >= 0 && k < K_NUM_KINDS) ? kKindNames[k] : "?"; }

void *ws(gvt_ctx *c, const char *name, size_t bytes) {
    Buf &b = c->bufs[name];
    if (b.bytes < bytes) {
        if (b.ptr) {
            // the stream may still use the old buffer
            GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
            cudaFree(b.ptr);
            b.ptr = nullptr;
            b.bytes = 0;
        }
        size_t nb = bytes < 256 ? 256 : bytes;
        cudaError_t e = cudaMalloc(&b.ptr, nb);
        if (e != cudaSuccess) {
            cudaGetLastError();
            throw Error{GVT_E_OOM, std::string("cudaMalloc of workspace '") + name + "' (" +
                                       std::to_string(nb) + " bytes) failed: " + cudaGetErrorString(e)};
        }
        b.bytes = nb;
    }
    return b.ptr;
}

void *pinned(gvt_ctx *c, size_t bytes) {
    if (c->pinned_bytes < bytes) {
        if (c->pinned) {
            GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
            cudaFreeHost(c->pinned);
        }
        c->pinned = nullptr;
        GVT_CUDA_TRY(cudaMallocHost(&c->pinned, bytes < 4096 ? 4096 : bytes));
        c->pinned_bytes = bytes < 4096 ? 4096 : bytes;
    }
    return c->pinned;
}

void launch_begin(gvt_ctx *c, int kind, cudaEvent_t *ev_start) {
    if (kind != K_COMM) c->launches++;  // collectives run NCCL's kernels, not the library's
    c->counts[kind]++;
    *ev_start = nullptr;
    if (c->profile) {
        if (c->event_pool.size() < 2) {
            for (int i = 0; i < 64; i++) {
                cudaEvent_t e;
                GVT_CUDA_TRY(cudaEventCreate(&e));
                c->event_pool.push_back(e);
            }
        }
        *ev_start = c->event_pool.back();
        c->event_pool.pop_back();
        GVT_CUDA_TRY(cudaEventRecord(*ev_start, c->stream));
    }
}

void launch_end(gvt_ctx *c, int kind, cudaEvent_t ev_start) {
    if (c->profile && ev_start) {
        cudaEvent_t stop = c->event_pool.back();
        c->event_pool.pop_back();
        GVT_CUDA_TRY(cudaEventRecord(stop, c->stream));
        c->pending.push_back(PendingEvent{kind, ev_start, stop});
        if (c->pending.size() > 4096) collect_events(c);
    }
}

void collect_events(gvt_ctx *c) {
    for (auto &pe : c->pending) {
        GVT_CUDA_TRY(cudaEventSynchronize(pe.stop));
        float ms = 0.f;
        GVT_CUDA_TRY(cudaEventElapsedTime(&ms, pe.start, pe.stop));
        c->ms[pe.kind] += ms;
        c->event_pool.push_back(pe.start);
        c->event_pool.push_back(pe.stop);
    }
    c->pending.clear();
}

bool is_device_ptr(const void *p) {
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

const void *stage_in(gvt_ctx *c, const char *name, const void *p, size_t bytes) {
    if (!p || bytes == 0) return p;
    if (is_device_ptr(p)) return p;
    void *d = ws(c, name, bytes);
    GVT_CUDA_TRY(cudaMemcpyAsync(d, p, bytes, cudaMemcpyHostToDevice, c->stream));
    return d;
}

}  // namespace gvt
