// score_window_tc.cu -- K1 on tcgen05 tensor cores (bf16, d == 128, g*m <= 128).
// Placeholder until the tcgen05 kernel lands: reports "unsupported" so the
// generic kernel (score_window.cu) serves every shape.
#include "common.cuh"

namespace adakv_b200 {

bool score_window_tc_supported(adakv_dtype, const adakv_layer_shape&, int64_t) { return false; }
size_t score_window_tc_workspace(const adakv_layer_shape&) { return 0; }
adakv_status score_window_tc(const adakv_layer_shape&, int64_t, int32_t, const void*, const void*, void*,
                             void*, void*, cudaStream_t) {
    return fail(ADAKV_UNSUPPORTED, "tcgen05 scoring not built");
}

}  // namespace adakv_b200
