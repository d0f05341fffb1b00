// tcm_stepwise.cuh -- TCM_ENGINE_STEPWISE (paper-literal per-step kernels), internal API.
#pragma once
#include "tcm_internal.cuh"

namespace tcm {

struct StepwiseWorkspace {
    void* base = nullptr;
    uint32_t R = 0;
};

size_t stepwise_workspace_bytes(uint32_t R, uint64_t N);
size_t stepwise_extra_bytes(uint32_t R, uint64_t N);   // rem[N] + pad
void stepwise_init(const TraceDev& t, cudaStream_t s);
StepwiseWorkspace stepwise_bind(void* p, uint32_t R);
// Runs up to max_iters engine iterations of every active replica; counts launches.
tcm_status stepwise_run(const ModelConst& m, const TraceDev& t, const StepwiseWorkspace& w,
                        uint32_t max_iters, uint32_t* d_active, cudaStream_t s, uint64_t* launches,
                        cudaEvent_t ev_begin, cudaEvent_t ev_end, double* kernel_ms, bool* deferred);

}  // namespace tcm
