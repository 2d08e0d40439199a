// tcgen05 path: placeholder until the fused stage kernel lands.
#include "ci_internal.h"
namespace ci {
ci_status_t umma_prepare(Model* m, const float* host_params) {
    (void)m; (void)host_params;
    set_error("tcgen05 precisions not built yet");
    return CI_ERR_UNSUPPORTED;
}
void umma_release(Model* m) { (void)m; }
ci_status_t umma_stage(const Model* m, int stage, float* state, int64_t n, bool inverse, cudaStream_t s) {
    (void)m; (void)stage; (void)state; (void)n; (void)inverse; (void)s;
    return CI_ERR_UNSUPPORTED;
}
}  // namespace ci
