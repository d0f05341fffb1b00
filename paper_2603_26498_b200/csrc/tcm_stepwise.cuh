// tcm_stepwise.cuh -- TCM_ENGINE_STEPWISE (paper-literal per-step kernels), internal API.
#pragma once
#include "tcm_internal.cuh"

namespace tcm {

// k_step's control words (in the workspace, after rem[]): the dynamic replica counter, the count
// of CTAs that finished the current launch, the active-replica accumulator.  Zero between
// launches: the launch's last CTA resets them.
struct StepSync {
    unsigned long long ctr;
    uint32_t done_ctas;
    uint32_t acc;
};
// k_step's launch arguments besides the model and trace.
struct StepCtl {
    StepSync* w;
    uint32_t* active_out;   // the active-replica count of a counting launch (device or mapped host word)
    uint32_t budget;        // != 0: this launch starts a call with this iteration budget
    int count_active;
    int dyn;                // warp-per-replica mode takes replicas from w->ctr
};

struct StepwiseWorkspace {
    void* base = nullptr;
    uint32_t R = 0;
    StepSync* sync = nullptr;
};

size_t stepwise_workspace_bytes(uint32_t R, uint64_t N);
size_t stepwise_extra_bytes(uint32_t R, uint64_t N);   // rem[N] + StepSync
void stepwise_init(const TraceDev& t, const StepwiseWorkspace& w, cudaStream_t s);
StepwiseWorkspace stepwise_bind(void* p, uint32_t R, uint64_t N);
// Runs up to max_iters engine iterations of every active replica; counts launches.  The active
// count lands in *active_out (device memory, or a mapped host word).
tcm_status stepwise_run(const ModelConst& m, const TraceDev& t, const StepwiseWorkspace& w,
                        uint32_t max_iters, uint32_t* active_out, cudaStream_t s, uint64_t* launches,
                        cudaEvent_t ev_begin, cudaEvent_t ev_end, double* kernel_ms, bool* deferred);

}  // namespace tcm
