// tcm_stepwise.cu -- TCM_ENGINE_STEPWISE: placeholder until the per-step kernels land.
#include "tcm_stepwise.cuh"

namespace tcm {
size_t stepwise_workspace_bytes(uint32_t R, uint64_t N) { return N + stepwise_extra_bytes(R); }
size_t stepwise_extra_bytes(uint32_t R) { return (size_t)R * 256; }
StepwiseWorkspace stepwise_bind(void* p, uint32_t R) { StepwiseWorkspace w; w.base = p; w.R = R; return w; }
tcm_status stepwise_run(const ModelConst&, const TraceDev&, const StepwiseWorkspace&, uint32_t, uint32_t*,
                        cudaStream_t, uint64_t*) {
    return TCM_E_ARG;
}
}  // namespace tcm
