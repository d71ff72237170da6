// dense_tc.cu -- dense tensor-core engine (placeholder until the tcgen05 kernels land).
#include "ops.cuh"

namespace gvt {

bool tc_available(gvt_ctx *c) {
    (void)c;
    return false;
}

void split_tf32(gvt_ctx *, const float *, int64_t, float *, float *) { throw Error{GVT_E_CUDA, "tc unavailable"}; }
void densify(gvt_ctx *, const EntryPlan &, float *, float *, int64_t, int64_t) { throw Error{GVT_E_CUDA, "tc unavailable"}; }
void gemm_nt_split(gvt_ctx *, const float *, const float *, int64_t, const float *, const float *, int64_t, int64_t,
                   int64_t, int64_t, float *, float *, float *, int64_t) {
    throw Error{GVT_E_CUDA, "tc unavailable"};
}
void gemm_nt_sampled(gvt_ctx *, const float *, const float *, int64_t, const float *, const float *, int64_t, int64_t,
                     int64_t, int64_t, const SamplePlan &, float, int, float *) {
    throw Error{GVT_E_CUDA, "tc unavailable"};
}
void bucket_samples(gvt_ctx *, const char *, SamplePlan &, int64_t, int64_t) { throw Error{GVT_E_CUDA, "tc unavailable"}; }
void gram_tc(gvt_ctx *, int, const float *, int64_t, int64_t, double, double, int, float *, int64_t) {
    throw Error{GVT_E_CUDA, "tc unavailable"};
}

}  // namespace gvt
