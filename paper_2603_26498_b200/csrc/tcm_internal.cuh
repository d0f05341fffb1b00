// tcm_internal.cuh -- device-side data layout shared by libtcm's kernels (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/tcm.h"

namespace tcm {

constexpr uint32_t NIL = 0xFFFFFFFFu;
constexpr uint32_t kCalSlots = 2048;      // decode calendar ring: out <= 2048 (R23)
constexpr uint32_t kCalWords = kCalSlots / 32;
constexpr uint32_t kHistBins = 496;
constexpr uint32_t kGroups = 4;           // M, C, T, all
constexpr uint32_t kNcnt = 6;

// Replica status codes (device), mirrored in tcm_stats_host.first_bad_status.
enum : uint32_t { ST_OK = 0, ST_DEADLOCK = 1, ST_BAD_INPUT = 2, ST_CAPACITY = 3 };

// Per-replica mutable state.  Between launches it lives in HBM (128 B, one line);
// inside the fused kernel it lives in registers.
struct __align__(16) ReplicaState {
    uint64_t clock;          // integer-us engine clock (R9)
    uint64_t kv_free;        // free KV tokens (R7: reserve-on-admit)
    uint64_t iter;           // iterations so far (calendar index)
    uint32_t nxt;            // next request (local id) to ingest
    uint32_t seq;            // next admit_seq
    uint32_t n_dec;          // decoding sequences
    uint32_t n_pend;         // pending (waiting + partial) requests
    uint32_t head[3];        // class-queue heads (local ids, NIL if empty)
    uint32_t tail[3];        // stepwise: running-set lower bound, preemptions, forced preemptions (NEXT-1)
    uint32_t rem[3];         // remaining prefill tokens of head[c]
    uint32_t flags;          // bit c: head[c] admitted (KV reserved); bit 8: finished
    uint32_t status;         // ST_*
    uint32_t max_pending;
    uint64_t decisions;      // R17
    uint64_t sum_pending;
    uint64_t ff_iters;
    uint32_t idle_jumps;
    uint32_t nlog;           // fused engine: event log entries (FusedWs::log)
    uint32_t done_count;
    uint32_t scanned;        // decisions that ran the full key/merge/scan (not fast-forwarded)
};
static_assert(sizeof(ReplicaState) == 128, "ReplicaState must be one 128-byte line");

constexpr uint32_t FLAG_FINISHED = 1u << 8;

// Per-replica K1 class constants, computed once per tcm_load_trace.
struct __align__(16) ClassPack {
    double S[3], p[3], C[3];   // K1 inputs: StaticPriority, p_c, C_c = LN(alpha k_c) - p_c LN(1e6)
    double Smax[3];            // exact upper bound of P: fl(S_c + 1), or S_c for a zero-rate class
    float fS[3], fp2[3], fC2[3];   // FP32 bound inputs (C2 = C / ln 2)
    uint32_t zero_mask;        // bit c: alpha * k_c == 0 (P == S_c)
    uint32_t filter_ok;        // FP32 bound validated for these constants (p <= 16, |C2| <= 1000)
    uint32_t pad;
    // exact saturation: K1(w) == Smax for every w >= wsat[c] (K1 is non-decreasing in w and bounded by
    // fl(S_c + 1), Lemma L1's premise), found by bisection at load within the audited [1, 2^33] us;
    // satkey[c] = the key there.  wsat = ~0: no saturation inside that range.
    uint64_t wsat[3];
    uint64_t satkey[3];
};
static_assert(sizeof(ClassPack) == 192, "ClassPack layout");

// Model constants in the kernels' parameter space.
struct ModelConst {
    uint64_t c0, cp, cd;
    double S[3], k[3], p[3];
    uint32_t thr_mc[3], thr_ct[3];
    uint32_t slo_num, slo_den;
    uint32_t n_cells;
};

// Fused engine: one request as it sits in its class segment.  The prologue
// (k_fpack, rows a1) classifies every request once and lays replica r's requests out as three
// contiguous class segments, each in arrival order (Lemma L1: the class FIFO), so a queue head's
// successor is the next record and one 256-bit load fetches everything the loop needs.
struct __align__(32) FRec {
    uint64_t arrival;        // arrival_us
    uint32_t fp;             // footprint
    uint32_t inl;            // inline_us
    uint32_t id;             // local request id (index into the trace / results)
    uint32_t out;            // out_tokens
    uint64_t spare;
};
static_assert(sizeof(FRec) == 32, "FRec is one 32-byte sector");

// Fused engine workspace.
struct FusedWs {
    FRec* rec;               // [N + 6R] class segments per replica, each closed by two sentinels
    uint64_t* cal;           // [R * kCalSlots] per iteration slot: (finishing count << 40) | sum of footprints
    uint64_t* log;           // [4N] per replica (iteration, clock) of every iteration with a first token or a finish
    uint64_t* fin;           // [N] finish iteration of a decoding request (0: none pending)
};
constexpr int kCalCntShift = 40;

// Fused engine under TCM_KV_GROWTH (NEXT-1, k_fgrow): state per class-segment position
// (the FRec index: replica r's positions start at offset[r] + 6r), and per replica and class.
struct FGrowWs {
    uint64_t* pfin;          // [N + 6R] finish iteration of the request decoding at this position (0: not decoding)
    uint32_t* pkv;           // [N + 6R] KV it holds at that finish (released there)
    uint32_t* prem;          // [N + 6R] waiting victim: KV to reserve = tokens to re-prefill (R30)
    uint32_t* pgen;          // [N + 6R] tokens generated so far (set at admission / preemption)
    uint32_t* pnext;         // [N + 6R] preempted-stack link
    uint8_t* pflag;          // [N + 6R] bit 0: first token emitted; bit 1: admitted before
    uint32_t* top;           // [R * 3] per class: top of the preempted stack (NIL: empty)
    uint32_t* seg;           // [R * 3] per class: first position of the class segment
    uint32_t* hres;          // [R * 3] per class: KV reserved by the class head while it is reserved
};

// Everything a kernel needs about the bound trace (device pointers).
struct TraceDev {
    uint32_t R;
    uint64_t N;
    const uint64_t* offset;
    const uint64_t* arrival;
    const uint32_t* footprint;
    const uint32_t* inl;
    const uint16_t* out;
    const uint8_t* mod;
    const tcm_replica_params* params;
    uint32_t* admit_seq;
    uint64_t* first_token;
    uint64_t* done;
    // workspace
    uint32_t* link;          // [N] class-queue / calendar-slot intrusive next pointer
    uint32_t* cal;           // [R * kCalSlots] calendar slot list heads
    uint32_t* occ;           // [R * kCalWords] calendar occupancy bits
    ReplicaState* state;     // [R]
    uint8_t* req_state;      // [N] stepwise engine: per-request class / phase byte
    ClassPack* kpack;        // [R] per-replica K1 class constants
    uint64_t* deadline;      // [N] stepwise engine, EDF: arrival*den + num*iso_e2e (set at ingest)
    // stepwise engine, TCM_KV_GROWTH (NEXT-1, R28-R32)
    uint32_t* kvres;         // [N] KV reserved at the last admission (footprint, or what a victim held)
    uint32_t* kvfin;         // [N] KV held at the finish iteration (released by the calendar)
    uint64_t* fin;           // [N] finish iteration of a decoding request
    uint32_t* genp;          // [N] tokens generated when last preempted
    uint64_t* pstart;        // [N] clock of the last preemption
    uint32_t* pcount;        // [N] preemptions (result)
    uint64_t* ptime;         // [N] preempted time (result)
    uint32_t any_growth;     // some replica sets TCM_KV_GROWTH (from k_validate)
    uint32_t all_growth;     // every replica does
    uint32_t all_tcm;        // every replica runs plain TCM (no EDF / FCFS / aging policy, no skip admission)
    FusedWs fw;              // fused engine only
    FGrowWs fg;              // fused engine with some TCM_KV_GROWTH replica only
};

__device__ __forceinline__ int classify(const ModelConst& m, uint32_t mod, uint32_t f) {
    // R13: per-modality footprint thresholds (smart classifier).
    return f < m.thr_mc[mod] ? 0 : (f < m.thr_ct[mod] ? 1 : 2);
}

void launch_fused_prologue(const ModelConst& m, const TraceDev& t, cudaStream_t s);
void launch_fused(const ModelConst& m, const TraceDev& t, uint32_t max_iters, uint32_t* d_active,
                  cudaStream_t s);
void launch_fused_stamp(const TraceDev& t, cudaStream_t s);

}  // namespace tcm
