#include <type_traits>
// plan.cu -- integer plumbing of the hot path: factor padding,
// stable sorts of pair/entry lists (CUB radix sort, stable => ties keep index order),
// CSR row pointers, sample ordering.  Everything here is integer work and bit-exact.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "ops.cuh"

namespace gvt {

// ----------------------------------------------------------------------------- padding
__global__ void k_pad_copy(const float *__restrict__ src, int64_t rows, int64_t cols, int64_t ld_src,
                           float *__restrict__ dst, int64_t ld_dst, int64_t rows_pad) {
    int64_t total = rows_pad * ld_dst;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / ld_dst, cc = i - r * ld_dst;
        dst[i] = (r < rows && cc < cols) ? src[r * ld_src + cc] : 0.0f;
    }
}

void pad_copy(gvt_ctx *c, const float *src, int64_t rows, int64_t cols, int64_t ld_src, float *dst, int64_t ld_dst,
              int64_t rows_pad) {
    int64_t total = rows_pad * ld_dst;
    if (total == 0) return;
    GVT_LAUNCH(c, K_PAD_COPY, k_pad_copy, grid1d(total, 256, 8 * c->sm_count * 8), 256, 0, src, rows, cols, ld_src,
               dst, ld_dst, rows_pad);
}

// dst (cols x ld_dst, rows_pad_dst rows, zero padded) = src^T, src rows x cols (ld_src): 32x32
// shared-memory tiles, coalesced on both sides (rectangular cross-Grams, sparse stage 1)
__global__ void k_transpose_pad(const float *__restrict__ src, int64_t rows, int64_t cols, int64_t ld_src,
                                float *__restrict__ dst, int64_t ld_dst, int64_t rows_pad_dst) {
    __shared__ float tile[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;  // src tile origin
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + k, cc = c0 + threadIdx.x;
        tile[k][threadIdx.x] = (r < rows && cc < cols) ? src[r * ld_src + cc] : 0.f;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t dr = c0 + k, dc = r0 + threadIdx.x;  // dst row = src col
        if (dr < rows_pad_dst && dc < ld_dst) dst[dr * ld_dst + dc] = tile[threadIdx.x][k];
    }
}

void transpose_pad(gvt_ctx *c, const float *src, int64_t rows, int64_t cols, int64_t ld_src, float *dst,
                   int64_t ld_dst, int64_t rows_pad_dst) {
    if (rows_pad_dst == 0 || ld_dst == 0) return;
    dim3 grid((unsigned)((rows_pad_dst + 31) / 32), (unsigned)((ld_dst + 31) / 32));
    GVT_LAUNCH(c, K_PAD_COPY, k_transpose_pad, grid, dim3(32, 8), 0, src, rows, cols, ld_src, dst, ld_dst,
               rows_pad_dst);
}

__global__ void k_fill_ones(float *dst, int64_t rows, int64_t cols, int64_t ld, int identity) {
    int64_t total = rows * ld;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int64_t r = i / ld, cc = i - r * ld;
        float v = 0.f;
        if (cc < cols) v = identity ? (r == cc ? 1.f : 0.f) : 1.f;
        dst[i] = v;
    }
}

void fill_ones(gvt_ctx *c, float *dst, int64_t rows, int64_t cols, int64_t ld, int identity) {
    if (rows == 0) return;
    GVT_LAUNCH(c, K_FILL, k_fill_ones, grid1d(rows * ld, 256, 8 * c->sm_count * 8), 256, 0, dst, rows, cols, ld,
               identity);
}

// ----------------------------------------------------------------------------- sorting helpers
static int key_bits(uint64_t max_key) {
    int b = 1;
    while (b < 64 && (max_key >> b)) b++;
    return b;
}

template <typename K>
static void radix_sort_pairs(gvt_ctx *c, const char *tag, const K *keys_in, K *keys_out, const int32_t *vals_in,
                             int32_t *vals_out, int64_t n, int end_bit) {
    if (n == 0) return;
    GVT_REQUIRE(n < (int64_t)INT32_MAX, GVT_E_DIM, "sort: more than 2^31-1 entries");
    size_t temp = 0;
    GVT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, temp, keys_in, keys_out, vals_in, vals_out, (int)n, 0,
                                                 end_bit, c->stream));
    std::string nm = std::string(tag) + ".cubtmp";
    void *t = ws(c, nm.c_str(), temp);
    cudaEvent_t ev;
    launch_begin(c, K_PLAN_SORT, &ev);
    GVT_CUDA_TRY(cub::DeviceRadixSort::SortPairs(t, temp, keys_in, keys_out, vals_in, vals_out, (int)n, 0, end_bit,
                                                 c->stream));
    launch_end(c, K_PLAN_SORT, ev);
}

__device__ __forceinline__ int32_t pick(int sel, const int32_t *f, const int32_t *s, int64_t j) {
    return sel == 0 ? f[j] : s[j];
}

// entry e = kind * n + j  ->  key (row * ncol + col), value e.  K = uint32_t when every key fits 32 bits (C5's
// 20000^2 cells: the radix passes move 8 instead of 12 bytes per entry; the same order)
template <typename K>
__global__ void k_entry_keys(const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n, EntryKinds kinds,
                             int64_t ncol, K *__restrict__ keys, int32_t *__restrict__ vals) {
    int64_t E = n * kinds.count;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        int kind = (int)(e / n);
        int64_t j = e - (int64_t)kind * n;
        int64_t row = pick(kinds.k[kind].row_sel, f, s, j);
        int64_t col = pick(kinds.k[kind].col_sel, f, s, j);
        keys[e] = (K)(row * ncol + col);
        vals[e] = (int32_t)e;
    }
}

template <typename K>
__global__ void k_entry_gather(const K *__restrict__ skeys, const int32_t *__restrict__ svals, int64_t E,
                               int64_t n, EntryKinds kinds, int64_t ncol, int32_t *__restrict__ row,
                               int32_t *__restrict__ col, int32_t *__restrict__ src, float *__restrict__ sign) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t e = svals[k];
        int kind = (int)(e / n);
        const uint64_t key = (uint64_t)skeys[k];
        row[k] = (int32_t)(key / (uint64_t)ncol);
        col[k] = (int32_t)(key % (uint64_t)ncol);
        src[k] = (int32_t)(e - (int64_t)kind * n);
        sign[k] = kinds.k[kind].sign;
    }
}

// is the sorted order the identity (entry k = pair k)?  bad != 0 otherwise
__global__ void k_ident_check(const int32_t *__restrict__ v, int64_t E, int *__restrict__ bad) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x)
        if (v[k] != (int32_t)k) atomicOr(bad, 1);
}

// row_ptr[h] = first position k with row[k] >= h  (rows sorted ascending)
__global__ void k_row_ptr(const int32_t *__restrict__ row, int64_t E, int64_t nrow, int64_t *__restrict__ row_ptr) {
    for (int64_t h = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; h <= nrow; h += (int64_t)gridDim.x * blockDim.x) {
        int64_t lo = 0, hi = E;
        while (lo < hi) {
            int64_t mid = (lo + hi) >> 1;
            if (row[mid] < h) lo = mid + 1;
            else hi = mid;
        }
        row_ptr[h] = lo;
    }
}

void build_entry_plan(gvt_ctx *c, const char *tag, const int32_t *f, const int32_t *s, int64_t n,
                      const EntryKinds &kinds, int64_t nrow, int64_t ncol, EntryPlan &out) {
    std::string t(tag);
    int64_t E = n * kinds.count;
    out.nnz = E;
    out.nrow = nrow;
    out.ncol = ncol;
    out.row = wsT<int32_t>(c, (t + ".row").c_str(), E);
    out.col = wsT<int32_t>(c, (t + ".col").c_str(), E);
    out.src = wsT<int32_t>(c, (t + ".src").c_str(), E);
    out.sign = wsT<float>(c, (t + ".sign").c_str(), E);
    out.val = wsT<float>(c, (t + ".val").c_str(), E);
    out.row_ptr = wsT<int64_t>(c, (t + ".rowptr").c_str(), nrow + 1);
    if (E > 0) {
        const uint64_t maxk = (uint64_t)(nrow * ncol > 0 ? nrow * ncol - 1 : 0);
        const int bits = key_bits(maxk);
        int32_t *v0 = wsT<int32_t>(c, "plan.vals0", E), *v1 = wsT<int32_t>(c, "plan.vals1", E);
        auto run = [&](auto *k0, auto *k1) {
            using K = std::remove_pointer_t<decltype(k0)>;
            GVT_LAUNCH(c, K_PLAN_KEYS, k_entry_keys<K>, grid1d(E, 256, 16 * c->sm_count * 8), 256, 0, f, s, n, kinds,
                       ncol, k0, v0);
            radix_sort_pairs<K>(c, "plan", k0, k1, v0, v1, E, bits);
            GVT_LAUNCH(c, K_PLAN_GATHER, k_entry_gather<K>, grid1d(E, 256, 16 * c->sm_count * 8), 256, 0, k1, v1, E,
                       n, kinds, ncol, out.row, out.col, out.src, out.sign);
        };
        if (maxk <= 0xffffffffull)
            run(wsT<uint32_t>(c, "plan.keys0", 2 * E), wsT<uint32_t>(c, "plan.keys1", 2 * E));
        else
            run(wsT<uint64_t>(c, "plan.keys0", E), wsT<uint64_t>(c, "plan.keys1", E));
        // one kind with sign +1 whose pairs were already in (row, col) order (the sorted-order fit): the pair
        // matrix build can read p[k] directly instead of sign[k] * p[src[k]]
        if (kinds.count == 1 && kinds.k[0].sign == 1.f) {
            int *bad = (int *)ws(c, "plan.identbad", sizeof(int));
            GVT_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), c->stream));
            GVT_LAUNCH(c, K_PLAN_GATHER, k_ident_check, grid1d(E, 256, 8 * c->sm_count), 256, 0, v1, E, bad);
            int *h = (int *)pinned(c, sizeof(int));
            GVT_CUDA_TRY(cudaMemcpyAsync(h, bad, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
            GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
            out.ident = *h == 0;
        }
    }
    GVT_LAUNCH(c, K_PLAN_ROWPTR, k_row_ptr, grid1d(nrow + 1, 256), 256, 0, out.row, E, nrow, out.row_ptr);
}

// samples: k < n -> (sel(rs, k), sel(cs, k)) ; n <= k < n + n_diag -> (k - n, k - n)
__global__ void k_sample_keys(const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n, int rs, int cs,
                              int64_t n_diag, uint32_t *__restrict__ keys, int32_t *__restrict__ vals) {
    int64_t N = n + n_diag;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x) {
        keys[k] = k < n ? (uint32_t)pick(rs, f, s, k) : (uint32_t)(k - n);
        vals[k] = (int32_t)k;
    }
}

__global__ void k_sample_gather(const uint32_t *__restrict__ skeys, const int32_t *__restrict__ svals, int64_t N,
                                const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n, int cs,
                                int32_t *__restrict__ r, int32_t *__restrict__ cc, int32_t *__restrict__ dst) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < N; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = svals[k];
        r[k] = (int32_t)skeys[k];
        cc[k] = i < n ? pick(cs, f, s, i) : (int32_t)(i - n);
        dst[k] = (int32_t)i;
    }
}

void build_sample_plan(gvt_ctx *c, const char *tag, const int32_t *f, const int32_t *s, int64_t n, int row_sel,
                       int col_sel, int64_t n_diag, int64_t nrow, SamplePlan &out) {
    std::string t(tag);
    int64_t N = n + n_diag;
    out.ns = N;
    out.r = wsT<int32_t>(c, (t + ".r").c_str(), N);
    out.c = wsT<int32_t>(c, (t + ".c").c_str(), N);
    out.dst = wsT<int32_t>(c, (t + ".dst").c_str(), N);
    out.tile_ptr = nullptr;
    if (N == 0) return;
    uint32_t *k0 = wsT<uint32_t>(c, "splan.keys0", N), *k1 = wsT<uint32_t>(c, "splan.keys1", N);
    int32_t *v0 = wsT<int32_t>(c, "splan.vals0", N), *v1 = wsT<int32_t>(c, "splan.vals1", N);
    GVT_LAUNCH(c, K_PLAN_KEYS, k_sample_keys, grid1d(N, 256, 16 * c->sm_count * 8), 256, 0, f, s, n, row_sel,
               col_sel, n_diag, k0, v0);
    radix_sort_pairs<uint32_t>(c, "splan", k0, k1, v0, v1, N, key_bits((uint64_t)(nrow > 0 ? nrow - 1 : 0)));
    GVT_LAUNCH(c, K_PLAN_GATHER, k_sample_gather, grid1d(N, 256, 16 * c->sm_count * 8), 256, 0, k1, v1, N, f, s, n,
               col_sel, out.r, out.c, out.dst);
}

// ----------------------------------------------------------------------------- debug sort (ABI gvt_sort_plan)
__global__ void k_debug_keys(const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n, int mode,
                             int64_t q, uint64_t *__restrict__ keys, int32_t *__restrict__ vals) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        keys[j] = mode == 1 ? (uint64_t)((int64_t)f[j] * q + s[j]) : (uint64_t)f[j];
        vals[j] = (int32_t)j;
    }
}

__global__ void k_debug_rows(const uint64_t *__restrict__ k, int64_t n, int mode, int64_t q, int32_t *__restrict__ row) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        row[j] = (int32_t)(mode == 1 ? k[j] / (uint64_t)q : k[j]);
}

void sort_plan_debug(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, int64_t m, int64_t q, int mode,
                     int32_t *perm, int64_t *row_ptr) {
    uint64_t *k0 = wsT<uint64_t>(c, "plan.keys0", n), *k1 = wsT<uint64_t>(c, "plan.keys1", n);
    int32_t *v0 = wsT<int32_t>(c, "plan.vals0", n);
    int32_t *rows = wsT<int32_t>(c, "dbg.rows", n);
    if (n > 0) {
        GVT_LAUNCH(c, K_PLAN_KEYS, k_debug_keys, grid1d(n, 256, 4096), 256, 0, f, s, n, mode, q, k0, v0);
        uint64_t maxk = mode == 1 ? (uint64_t)(m * q) : (uint64_t)m;
        radix_sort_pairs<uint64_t>(c, "plan", k0, k1, v0, perm, n, key_bits(maxk));
        GVT_LAUNCH(c, K_PLAN_GATHER, k_debug_rows, grid1d(n, 256, 4096), 256, 0, k1, n, mode, q, rows);
    }
    GVT_LAUNCH(c, K_PLAN_ROWPTR, k_row_ptr, grid1d(m + 1, 256), 256, 0, rows, n, m, row_ptr);
}

// ----------------------------------------------------------------------------- compact relabel
// SPEC.md:49-57 relabel_compact (the unique counts of PAPER.md Table 1): compact[i] = rank of
// ids[i] among the distinct ids ordered by first occurrence.  Integer-only, bit-exact:
//   first[v] = min { i : ids[i] = v }   (atomicMin: the minimum does not depend on the order)
//   sort the domain values by first[v] (absent values carry REL_ABSENT and sort last)
//   lut[unique[j]] = j;  compact[i] = lut[ids[i]]
constexpr int32_t REL_ABSENT = 0x7f7f7f7f;  // the byte-memset fill; above every index (n < REL_ABSENT)

__global__ void k_first_occ(const int32_t *__restrict__ ids, int64_t n, int32_t *__restrict__ first) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicMin(first + ids[i], (int32_t)i);
}

__global__ void k_first_keys(const int32_t *__restrict__ first, int64_t bound, uint32_t *__restrict__ keys,
                             int32_t *__restrict__ vals, unsigned long long *__restrict__ count) {
    unsigned long long cnt = 0;
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < bound; v += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = first[v];
        keys[v] = (uint32_t)f;
        vals[v] = (int32_t)v;
        cnt += f != REL_ABSENT;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(count, cnt);  // an integer count: order-free
}

__global__ void k_rank_lut(const int32_t *__restrict__ unique, const unsigned long long *__restrict__ count,
                           int32_t *__restrict__ lut) {
    const int64_t c = (int64_t)*count;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < c; j += (int64_t)gridDim.x * blockDim.x)
        lut[unique[j]] = (int32_t)j;
}

__global__ void k_apply_lut(const int32_t *__restrict__ ids, int64_t n, const int32_t *__restrict__ lut,
                            int32_t *__restrict__ compact) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        compact[i] = lut[ids[i]];
}

// ids (device, in [0, bound)) -> compact (device, n), unique (device, the first `count` of a
// bound-long sorted value array); returns count
int64_t relabel_compact(gvt_ctx *c, const int32_t *ids, int64_t n, int64_t bound, int32_t *compact,
                        const int32_t **unique_out) {
    *unique_out = nullptr;
    if (n == 0 || bound == 0) return 0;
    GVT_REQUIRE(n < (int64_t)REL_ABSENT && bound < (int64_t)INT32_MAX, GVT_E_DIM, "relabel: too many ids");
    int32_t *first = wsT<int32_t>(c, "relabel.first", (size_t)bound);
    uint32_t *k0 = wsT<uint32_t>(c, "relabel.k0", (size_t)bound), *k1 = wsT<uint32_t>(c, "relabel.k1", (size_t)bound);
    int32_t *v0 = wsT<int32_t>(c, "relabel.v0", (size_t)bound), *v1 = wsT<int32_t>(c, "relabel.v1", (size_t)bound);
    int32_t *lut = wsT<int32_t>(c, "relabel.lut", (size_t)bound);
    unsigned long long *cnt = wsT<unsigned long long>(c, "relabel.count", 1);
    GVT_CUDA_TRY(cudaMemsetAsync(first, 0x7f, sizeof(int32_t) * bound, c->stream));  // REL_ABSENT
    GVT_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(unsigned long long), c->stream));
    GVT_LAUNCH(c, K_PLAN_KEYS, k_first_occ, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, ids, n, first);
    GVT_LAUNCH(c, K_PLAN_KEYS, k_first_keys, grid1d(bound, 256, 8 * c->sm_count * 8), 256, 0, first, bound, k0, v0, cnt);
    radix_sort_pairs<uint32_t>(c, "relabel", k0, k1, v0, v1, bound, 31);  // present values have distinct keys
    GVT_LAUNCH(c, K_PLAN_GATHER, k_rank_lut, grid1d(bound, 256, 8 * c->sm_count * 8), 256, 0, v1, cnt, lut);
    GVT_LAUNCH(c, K_PLAN_GATHER, k_apply_lut, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, ids, n, lut, compact);
    unsigned long long h = 0;
    GVT_CUDA_TRY(cudaMemcpyAsync(&h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    *unique_out = v1;
    return (int64_t)h;
}

// ----------------------------------------------------------------------------- used-object compaction
// The objects a sample uses (Table 1: m, q count UNIQUE drugs / targets of the sample),
// numbered in ascending global id: used[v] = 1 marks, pos = exclusive prefix sum, ids[pos[v]] = v.
// Everything is launched asynchronously; one read-back (used_set_finish) returns the count, the
// out-of-range ids met while marking, and the ids of extra arrays outside the set.
__global__ void k_mark_used(const int32_t *__restrict__ a, int64_t n, int64_t bound, int32_t *__restrict__ used,
                            unsigned long long *__restrict__ oor) {
    unsigned long long bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = a[i];
        if (v < 0 || v >= bound) bad++;
        else if (!used[v]) used[v] = 1;  // read first: popular ids (Zipf) would serialise on stores
    }
    for (int o = 16; o > 0; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(oor, bad);
}

__global__ void k_used_list(const int32_t *__restrict__ used, const int32_t *__restrict__ pos, int64_t m,
                            int32_t *__restrict__ ids, int64_t *__restrict__ k) {
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v < m; v += (int64_t)gridDim.x * blockDim.x) {
        if (used[v]) ids[pos[v]] = (int32_t)v;
        if (v == m - 1) *k = (int64_t)pos[v] + used[v];
    }
}

__global__ void k_count_unused(const int32_t *__restrict__ a, int64_t n, int64_t bound,
                               const int32_t *__restrict__ used, unsigned long long *__restrict__ cnt) {
    unsigned long long k = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t v = a[i];
        k += (v < 0 || v >= bound) ? 1ull : (unsigned long long)(used[v] == 0);
    }
    for (int o = 16; o > 0; o >>= 1) k += __shfl_xor_sync(0xffffffffu, k, o);
    if ((threadIdx.x & 31) == 0 && k) atomicAdd(cnt, k);
}

__global__ void k_map_ids(const int32_t *__restrict__ a, int64_t n, const int32_t *__restrict__ pos,
                          int32_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = pos[a[i]];
}

// Gs[i][j] = G[rid[i]][cid[j]] (kr x kc, ld kc): 32 x 8 threads, coalesced along j
__global__ void k_sub_gram(const float *__restrict__ G, int64_t ld, const int32_t *__restrict__ rid, int64_t kr,
                           const int32_t *__restrict__ cid, int64_t kc, float *__restrict__ Gs) {
    const int64_t i = (int64_t)blockIdx.y * 8 + threadIdx.y, j = (int64_t)blockIdx.x * 32 + threadIdx.x;
    for (int64_t ii = i; ii < kr; ii += (int64_t)gridDim.y * 8)
        if (j < kc) Gs[ii * kc + j] = G[(int64_t)rid[ii] * ld + cid[j]];
}

// counters: [0] out-of-range ids of the marked arrays, [1] ids of the tested array outside the set
UsedSet used_set_begin(gvt_ctx *c, const char *tag, int64_t m, const int32_t *const *arrays, const int64_t *lens,
                       int narr, unsigned long long *counters) {
    UsedSet u;
    if (m <= 0) return u;
    std::string t(tag);
    int32_t *used = wsT<int32_t>(c, (t + ".used").c_str(), (size_t)m);  // int32: the scan's type
    int32_t *pos = wsT<int32_t>(c, (t + ".pos").c_str(), (size_t)m);
    int32_t *ids = wsT<int32_t>(c, (t + ".ids").c_str(), (size_t)m);
    int64_t *k = wsT<int64_t>(c, (t + ".k").c_str(), 1);
    GVT_CUDA_TRY(cudaMemsetAsync(used, 0, sizeof(int32_t) * m, c->stream));
    for (int a = 0; a < narr; a++)
        if (lens[a] > 0)
            GVT_LAUNCH(c, K_PLAN_KEYS, k_mark_used, grid1d(lens[a], 256, 8 * c->sm_count * 8), 256, 0, arrays[a],
                       lens[a], m, used, counters);
    size_t temp = 0;
    GVT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(nullptr, temp, used, pos, (int)m, c->stream));
    void *tb = ws(c, (t + ".scantmp").c_str(), temp);
    GVT_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tb, temp, used, pos, (int)m, c->stream));
    GVT_LAUNCH(c, K_PLAN_GATHER, k_used_list, grid1d(m, 256, 8 * c->sm_count * 8), 256, 0, used, pos, m, ids, k);
    u.used = used;
    u.pos = pos;
    u.ids = ids;
    u.k_dev = k;
    u.m = m;
    return u;
}

void count_unused_async(gvt_ctx *c, const UsedSet &u, const int32_t *a, int64_t n, unsigned long long *cnt) {
    if (n == 0 || u.m == 0) return;
    GVT_LAUNCH(c, K_PLAN_KEYS, k_count_unused, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, a, n, u.m, u.used, cnt);
}

void map_ids(gvt_ctx *c, const UsedSet &u, const int32_t *a, int64_t n, int32_t *out) {
    if (n == 0) return;
    GVT_LAUNCH(c, K_PLAN_GATHER, k_map_ids, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, a, n, u.pos, out);
}

void sub_gram(gvt_ctx *c, const float *G, int64_t ld, const UsedSet &rows, const UsedSet &cols, float *Gs) {
    if (rows.k == 0 || cols.k == 0) return;
    dim3 grid((unsigned)((cols.k + 31) / 32), (unsigned)std::min<int64_t>((rows.k + 7) / 8, 4096));
    GVT_LAUNCH(c, K_PAD_COPY, k_sub_gram, grid, dim3(32, 8), 0, G, ld, rows.ids, rows.k, cols.ids, cols.k, Gs);
}

// ----------------------------------------------------------------------------- fit-level reordering
// perm = the pair indices stably sorted by (first, second): a fit runs in this order so that the
// pair-matrix entries of the Kronecker group are read in vector order (sequential, not gathered)
template <typename K>
__global__ void k_pair_keys(const int32_t *__restrict__ f, const int32_t *__restrict__ s, int64_t n, int64_t q,
                            K *__restrict__ keys, int32_t *__restrict__ vals) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        keys[j] = (K)((uint64_t)f[j] * (uint64_t)q + (uint64_t)s[j]);
        vals[j] = (int32_t)j;
    }
}

void sort_pairs(gvt_ctx *c, const int32_t *f, const int32_t *s, int64_t n, int64_t m, int64_t q, int32_t *perm) {
    if (n == 0) return;
    const uint64_t cells = (uint64_t)(m > 0 ? m : 1) * (uint64_t)(q > 0 ? q : 1);
    int32_t *v0 = wsT<int32_t>(c, "fitsort.v0", n);
    auto run = [&](auto *k0, auto *k1) {  // 32-bit keys when every (first, second) cell index fits
        using K = std::remove_pointer_t<decltype(k0)>;
        GVT_LAUNCH(c, K_PLAN_KEYS, k_pair_keys<K>, grid1d(n, 256, 4096), 256, 0, f, s, n, q, k0, v0);
        radix_sort_pairs<K>(c, "fitsort", k0, k1, v0, perm, n, key_bits(cells));
    };
    if (cells - 1 <= 0xffffffffull)
        run(wsT<uint32_t>(c, "fitsort.k0", 2 * n), wsT<uint32_t>(c, "fitsort.k1", 2 * n));
    else
        run(wsT<uint64_t>(c, "fitsort.k0", n), wsT<uint64_t>(c, "fitsort.k1", n));
}

template <typename Tv>
__global__ void k_gather(const Tv *__restrict__ x, const int32_t *__restrict__ perm, int64_t n, Tv *__restrict__ y) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        y[k] = x[perm[k]];
}

__global__ void k_scatter_f32(const float *__restrict__ x, const int32_t *__restrict__ perm, int64_t n,
                              float *__restrict__ y) {
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        y[perm[k]] = x[k];
}

void gather_i32(gvt_ctx *c, const int32_t *x, const int32_t *perm, int64_t n, int32_t *y) {
    if (n) GVT_LAUNCH(c, K_PLAN_GATHER, k_gather<int32_t>, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, x, perm, n, y);
}
void gather_f32(gvt_ctx *c, const float *x, const int32_t *perm, int64_t n, float *y) {
    if (n) GVT_LAUNCH(c, K_PLAN_GATHER, k_gather<float>, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, x, perm, n, y);
}
void scatter_f32(gvt_ctx *c, const float *x, const int32_t *perm, int64_t n, float *y) {
    if (n) GVT_LAUNCH(c, K_PLAN_GATHER, k_scatter_f32, grid1d(n, 256, 8 * c->sm_count * 8), 256, 0, x, perm, n, y);
}

// ----------------------------------------------------------------------------- validation
__global__ void k_count_oor(const int32_t *__restrict__ ids, int64_t n, int64_t bound, unsigned long long *cnt) {
    unsigned long long local = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        int32_t v = ids[i];
        local += (v < 0 || v >= bound) ? 1ull : 0ull;
    }
    // warp reduce then one integer atomic per warp (integer: order-independent)
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(cnt, local);
}

int64_t count_out_of_range(gvt_ctx *c, const int32_t *ids, int64_t n, int64_t bound) {
    if (n == 0) return 0;
    unsigned long long *d = wsT<unsigned long long>(c, "val.cnt", 1);
    GVT_CUDA_TRY(cudaMemsetAsync(d, 0, sizeof(unsigned long long), c->stream));
    GVT_LAUNCH(c, K_FILL, k_count_oor, grid1d(n, 256, 4 * c->sm_count * 8), 256, 0, ids, n, bound, d);
    unsigned long long *h = (unsigned long long *)pinned(c, 64);
    GVT_CUDA_TRY(cudaMemcpyAsync(h, d, sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    GVT_CUDA_TRY(cudaStreamSynchronize(c->stream));
    return (int64_t)*h;
}

}  // namespace gvt
