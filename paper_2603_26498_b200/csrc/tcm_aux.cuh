// tcm_aux.cuh -- launchers for libtcm's non-step kernels (internal).
#pragma once
#include "tcm_internal.cuh"

namespace tcm {

// k_reduce accumulator layout (u64 each)
enum : int {
    kAccIter = 0, kAccDecisions, kAccFF, kAccIdle, kAccSumPending, kAccDone, kAccReplicasDone,
    kAccReplicasActive, kAccMaxPending, kAccBadReplica, kAccBadStatus, kAccScanned, kAccPreempt, kAccForced, kAccN
};

constexpr uint32_t kRepCnt = 6;   // tcm_replica_counters fields per replica

void launch_init(const TraceDev& t, cudaStream_t s);
void launch_replica_counters(const TraceDev& t, unsigned long long* out, cudaStream_t s);
void launch_preempt_stats(const ModelConst& m, const TraceDev& t, unsigned long long* out, cudaStream_t s);
void launch_kpack(const ModelConst& m, const TraceDev& t, cudaStream_t s);
void launch_validate(const TraceDev& t, uint32_t* v, int general_ok, cudaStream_t s);
void launch_reduce(const TraceDev& t, unsigned long long* acc, cudaStream_t s);
// n words device -> mapped host memory by plain stores (no copy-engine DMA: a small readback does not
// queue behind a large copy in flight on another stream)
void launch_copy_words(const unsigned long long* src, unsigned long long* dst, int n, cudaStream_t s);
void launch_aggregate(const ModelConst& m, const TraceDev& t, unsigned long long* hist,
                      unsigned long long* cnt, cudaStream_t s);
void launch_generate(const void* reps, uint32_t R, const uint64_t* off, uint64_t* arrival,
                     uint32_t* footprint, uint32_t* inl, uint16_t* out, uint8_t* mod, uint32_t* bad,
                     cudaStream_t s);
void launch_k1_eval(const ModelConst& m, const uint8_t* cls, const uint64_t* w, const double* alpha,
                    double* outp, uint64_t n, cudaStream_t s);
void launch_filter_audit(const ModelConst& m, uint32_t c, double alpha, uint64_t lo, uint64_t hi, uint64_t step,
                         unsigned long long* maxerr, cudaStream_t s);
void launch_k1_audit(const ModelConst& m, uint32_t c, double alpha, uint64_t lo, uint64_t hi,
                     unsigned long long* first, cudaStream_t s);

}  // namespace tcm
