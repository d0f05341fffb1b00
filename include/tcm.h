/*
 * tcm.h -- C ABI of libtcm: TCM-Serve's per-iteration modality-aware scheduling step
 * (arxiv 2603.26498, Section 3) run as a trace-driven simulation over many
 * independent replicas on one B200 (sm_100a).
 *
 * Every replica is one serving engine (vLLM V1 + chunked prefill) fed by
 * its own request trace.  Each engine iteration, per replica:
 *   a1 ingest arrivals <= clock and classify them motorcycle / car / truck from modality
 *      and KV footprint (reading R13);
 *   a2 key every pending request with Priority_c = S_c + (1 - e^{-k_c w^{p_c}})
 *      (PAPER.md:457, 580), evaluated by the specified-arithmetic K1;
 *   a3 order pending requests by key (Score = -log Priority; R3, R4);
 *   a4 admit a prefill batch by prefix-scanning chunk tokens against the chunked-prefill
 *      budget and footprints against free KV (R5-R8);
 *   a5 advance an integer-microsecond clock by c0 + cp*tokens + cd*decodes + inline
 *      (R9, R10) and record TTFT / completion (R12);
 *   a6 aggregate TTFT histograms and SLO counters.
 *
 * Conventions for every entry point:
 *   - No exception crosses the ABI; every call returns a tcm_status (0 = OK, < 0 error)
 *     and records a message retrievable with tcm_last_error().
 *   - Buffers are caller-owned.  "device" pointers are CUDA device memory on the
 *     context's device; "host" pointers are ordinary or pinned host memory (pinned is
 *     required for asynchronous overlap but not for correctness).  The library borrows
 *     every pointer from tcm_load_trace until tcm_destroy / the next tcm_load_trace.
 *   - All work is enqueued on the caller's CUDA stream given to tcm_create; tcm_run,
 *     tcm_step and tcm_stats synchronise that stream before returning.
 *   - Results are deterministic: independent of launch geometry, engine, stream and of
 *     how replicas are split across GPUs (every reduction is an integer sum).
 *   - A context is not thread-safe; distinct contexts are independent.
 */
#ifndef TCM_H
#define TCM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TCM_ABI_VERSION 3u

typedef int32_t tcm_status;
#define TCM_OK 0
#define TCM_E_ARG (-1)      /* invalid argument or malformed trace                      */
#define TCM_E_STATE (-2)    /* calls out of order (e.g. tcm_run before tcm_load_trace)   */
#define TCM_E_CAPACITY (-3) /* a footprint exceeds its replica's KV capacity (SPEC.md:456
                               CapacityImpossible; R18)                                 */
#define TCM_E_CUDA (-4)     /* a CUDA runtime call failed                                */
#define TCM_E_OOM (-5)      /* workspace allocation failed                               */
#define TCM_E_REPLICA (-6)  /* >= 1 replica set a device status (deadlock assertion,
                               unreachable under R6; see tcm_stats_host.first_bad_*)     */
#define TCM_E_VERSION (-7)  /* abi_version mismatch                                      */

enum { TCM_POLICY_FCFS = 0, TCM_POLICY_TCM = 1, TCM_POLICY_EDF = 2, TCM_POLICY_NAIVE_AGING = 3 };
/* FCFS: vLLM's single arrival-ordered queue with chunked prefill.
 * TCM : three class queues + aging priority.  Static priority
 *        is TCM with aging_alpha = 0 (R14).
 * EDF : earliest deadline first, deadline = arrival + (slo_num/slo_den) x isolated E2E
 *       (SPEC.md:399).  With TCM_KV_GROWTH it also preempts running requests
 *       with a later deadline when an earlier-deadline waiting request does not fit (R34,
 *       PAPER.md:622).  STEPWISE only: its keys are not class-monotone (Lemma L1 does not hold).
 * NAIVE_AGING: descending waiting time ignoring class, i.e. arrival order. */

/* tcm_replica_params.flags */
#define TCM_ADMIT_SKIP 1u   /* a KV misfit is skipped instead of stopping new admissions (first
                               fit; the alternative reading of R6, NEXT-3).  STEPWISE only. */
#define TCM_KV_GROWTH 2u    /* NEXT-1: decode KV growth + preemption by recomputation (readings
                               R28-R32).  A running
                               request holds its reservation plus one KV token per decode
                               iteration; when the free KV cannot cover this iteration's decode
                               tokens, victims are preempted (FCFS/EDF/naive aging: most recently
                               arrived; TCM: lowest-ranked non-motorcycle) and re-prefill what
                               they held.  Needs footprint + out - 1 <= kv_capacity for every
                               request (else TCM_E_CAPACITY).  Both engines (FUSED: k_fgrow,
                               DESIGN.md 6.5; with EDF: STEPWISE only).                       */

enum { TCM_ENGINE_FUSED = 0, TCM_ENGINE_STEPWISE = 1 };
/* Development knobs read from the environment at each run (not part of the contract; results are
 * identical under every setting): TCM_SW_GROUP = 1 | 8 | cluster forces the stepwise engine's warp /
 * CTA / 8-CTA-cluster per replica mode; TCM_FUSED_LPW = 1..32 forces the fused engine's replicas
 * per warp. */
/* FUSED   : one persistent thread per replica runs the whole step loop in registers;
 *           a3 is the exact 3-way merge of the class-FIFO heads (Lemma L1).
 *           Replicas must hold < 2^24 requests (calendar slot counters).  TCM_KV_GROWTH
 *           replicas run in k_fgrow (preempted requests re-enter their class queue in front)
 *           and need about 33 B more workspace per request than tcm_workspace_bytes reports.
 * STEPWISE: the paper-literal step -- per iteration, every pending request of every
 *           active replica is re-keyed (a1+a2), top-k selected (a3), prefix-scanned (a4),
 *           then the clock kernel runs (a5).  Bit-identical results; used for the
 *           per-step HBM roofline and for key functions that are not class-monotone. */

enum { TCM_MEM_DEVICE = 0, TCM_MEM_HOST = 1 };

/* Model-wide constants (one per context).  All times are integer microseconds (R9). */
typedef struct tcm_config {
    uint32_t abi_version;  /* = TCM_ABI_VERSION                                     */
    uint32_t engine;       /* TCM_ENGINE_*                                          */
    uint64_t c0_us;        /* per-iteration overhead (5 ms)            */
    uint64_t cp_us;        /* per prefill token (20 us)                */
    uint64_t cd_us;        /* per decoding sequence (0.5 ms)           */
    double S[3];           /* StaticPriority_c for M, C, T (.1,.05,0) */
    double k[3];           /* k_c (0.05, 0.003, 0.00075)              */
    double p[3];           /* p_c (3.5, 2.5, 1.1)                     */
    uint32_t thr_mc[3];    /* per modality (text,image,video): footprint < thr_mc -> M */
    uint32_t thr_ct[3];    /* per modality: footprint < thr_ct -> C, else T (R13)   */
    uint32_t slo_num;      /* SLO = slo_num/slo_den x isolated E2E   */
    uint32_t slo_den;
    uint32_t n_cells;      /* sweep cells for the a6 aggregation (>= 1)             */
    uint32_t reserved;     /* must be 0                                             */
} tcm_config;

/* Per-replica parameters (one sweep point x seed).  32 bytes. */
typedef struct tcm_replica_params {
    uint32_t policy;       /* TCM_POLICY_*                                          */
    uint32_t chunk_budget; /* B: chunked-prefill tokens per iteration, >= 1 */
    uint64_t kv_capacity;  /* KV tokens, 1 .. 2^32-1    */
    double aging_alpha;    /* multiplies every k_c, >= 0 (R14)                      */
    uint32_t cell_id;      /* < n_cells: aggregation cell                           */
    uint32_t flags;        /* bitwise OR of TCM_ADMIT_SKIP and TCM_KV_GROWTH, or 0  */
} tcm_replica_params;

/* The request trace, SoA in CSR form: replica r owns requests [req_offset[r], req_offset[r+1]),
 * sorted by (arrival, id) -- ids are the local indices 0..n_r-1 (R4, R16). */
typedef struct tcm_trace_view {
    uint32_t mem;                 /* TCM_MEM_DEVICE or TCM_MEM_HOST (all arrays alike)  */
    uint32_t n_replicas;          /* R >= 1                                             */
    uint64_t n_requests;          /* = req_offset[R]; each replica has < 2^32 - 1        */
    const uint64_t* req_offset;   /* [R+1], req_offset[0] = 0, non-decreasing           */
    const uint64_t* arrival_us;   /* [N] non-decreasing within a replica                */
    const uint32_t* footprint;    /* [N] prompt + media tokens = KV footprint, 1..kv_capacity */
    const uint32_t* inline_us;    /* [N] preprocess + encode time, charged inline (R10) */
    const uint16_t* out_tokens;   /* [N] output tokens, 1..2048 (R23)                   */
    const uint8_t* modality;      /* [N] 0 text, 1 image, 2 video                       */
    const tcm_replica_params* params; /* [R]                                            */
} tcm_trace_view;

/* Per-request outputs, written in place (any pointer may be NULL: then the library keeps
 * the values in its workspace for tcm_stats only). */
typedef struct tcm_results_view {
    uint32_t mem;                 /* TCM_MEM_DEVICE or TCM_MEM_HOST                     */
    uint32_t reserved;
    uint32_t* admit_seq;          /* [N] order of first admission within the replica    */
    uint64_t* first_token_us;     /* [N] clock at the first token (TTFT = - arrival)    */
    uint64_t* done_us;            /* [N] clock at completion                            */
    uint32_t* preempt_count;      /* [N] preemptions of the request (TCM_KV_GROWTH; else 0) */
    uint64_t* preempted_us;       /* [N] time from each preemption to the next admission,
                                     summed                                 */
} tcm_results_view;

/* Work counters (sums over all replicas of this context). */
typedef struct tcm_stats_host {
    uint64_t iterations;       /* engine iterations, fast-forwarded ones included    */
    uint64_t decisions;        /* iterations with >= 1 pending request (R17)         */
    uint64_t ff_iterations;    /* iterations covered by decode-only fast-forward     */
    uint64_t idle_jumps;       /* jumps of an empty engine to its next arrival (R15) */
    uint64_t sum_pending;      /* sum over decisions of the pending-set size         */
    uint64_t max_pending;      /* max over decisions and replicas                    */
    uint64_t requests_done;    /* requests with done_us stamped                      */
    uint64_t replicas_done;
    uint64_t replicas_active;
    uint64_t kernel_launches;  /* library kernels launched since tcm_create          */
    uint64_t scanned_decisions; /* decisions that ran the full key/order/scan (the rest
                                   were taken in closed form, Lemmas L4-L5) */
    int32_t first_bad_replica; /* -1 if none                                          */
    int32_t first_bad_status;
    /* Device time (ms) since the last tcm_load_trace / tcm_reset, from CUDA events recorded
     * on the context's stream around the library's own launches:                          */
    double reset_ms;           /* the reset: memsets, state init, engine prologue (FUSED: the
                                  class-segment build, row a1)                            */
    double engine_ms;          /* the step kernels (FUSED: k_fused; STEPWISE: the k_step
                                  launches, each up to 16 engine iterations per replica)    */
    double stamp_ms;           /* FUSED: k_fstamp (first-token / finish times from the log) */
    uint64_t preemptions;      /* TCM_KV_GROWTH: preemptions (R29)                     */
    uint64_t forced_preemptions; /* TCM: motorcycle victims (only when nothing else ran)  */
} tcm_stats_host;

typedef struct tcm_ctx tcm_ctx;

/* Synthetic-trace generator descriptor (layout of tracegen/tcm_tracegen.h tg_replica). */
typedef struct tcm_gen_replica {
    uint64_t seed;          /* splitmix64(base ^ replica)                            */
    uint64_t kv_capacity;   /* footprints are clamped to this (R18)                  */
    double mean_gap_us;     /* 1e6 / lambda: Poisson arrivals         */
    uint64_t mix_t1;        /* 32-bit draw < mix_t1 -> text                          */
    uint64_t mix_t2;        /* draw < mix_t2 -> image, else video     */
    uint32_t n_requests;
    uint32_t flags;         /* bit0: every arrival at t = 0                          */
} tcm_gen_replica;

/* Validates *cfg and creates a context bound to the current CUDA device and `cuda_stream`
 * (a cudaStream_t; NULL = legacy default stream).  Errors: TCM_E_ARG, TCM_E_VERSION. */
tcm_status tcm_create(const tcm_config* cfg, void* cuda_stream, tcm_ctx** out);

/* Binds a trace and result buffers, allocates the workspace (tcm_workspace_bytes) and
 * validates the trace on the device: footprint <= kv_capacity (TCM_E_CAPACITY), and
 * footprint >= 1, 1 <= out <= 2048, modality <= 2, non-decreasing arrivals, params in
 * range, EDF / TCM_ADMIT_SKIP / >= 2^24 requests per replica only on the STEPWISE engine
 * (TCM_E_ARG).  HOST traces are copied to the device here (on the stream).
 * Resets every replica to its initial state (clock 0, all KV free). */
tcm_status tcm_load_trace(tcm_ctx* ctx, const tcm_trace_view* trace,
                          const tcm_results_view* results);

/* Resets every replica of the bound trace to its initial state (clock 0, all KV free, no
 * request admitted) without re-validating or re-copying the trace: device work only
 * (memsets + two kernels: state init and the engine's prologue -- the FUSED engine
 * classifies every request into its class segment here, row a1), enqueued on the stream.
 * TCM_E_STATE before tcm_load_trace. */
tcm_status tcm_reset(tcm_ctx* ctx);

/* Advances every unfinished replica by at most max_iterations engine iterations (a
 * fast-forward counts all the iterations it covers; idle jumps count none).  Writes the
 * number of replicas still unfinished to *active_replicas (may be NULL).  HOST results
 * are copied back before returning.  Afterwards every result of a request that has reached
 * that stage is final; admit_seq / first_token_us / done_us of a request that has not are
 * 0xFFFFFFFF / 0 / 0.  A call with max_iterations <= 64 repeated with the same value is replayed
 * as one CUDA graph (its launches and the active-count copy, captured on the second such call on
 * an internal stream and launched into the context's stream; a new tcm_load_trace discards it):
 * one host round trip per call ("minimal overhead"); tcm_stats_host.engine_ms then
 * counts the whole graph.  STEPWISE: the graph holds only the k_step launches -- the first one
 * sets the call's iteration budget and the launch's last CTA writes the active count into a
 * mapped host word, so there is no budget kernel, memset or copy node.  The environment knob
 * TCM_GRAPHS=0 keeps every call eager. */
tcm_status tcm_step(tcm_ctx* ctx, uint32_t max_iterations, uint32_t* active_replicas);

/* Runs every replica to completion (every request done).  TCM_E_REPLICA if a replica
 * hit its deadlock assertion. */
tcm_status tcm_run(tcm_ctx* ctx);

/* tcm_run without waiting (FUSED engine only, TCM_E_ARG otherwise): enqueues the engine to
 * completion, the first-token / finish stamping and, for HOST results, their device-to-host copy
 * on the context's stream, and returns.  A pipeline of contexts overlaps one context's copies with
 * another's kernels: tcm_wait(ctx, TCM_WAIT_ENGINE) returns once the kernels are done (the copy
 * may still run), tcm_wait(ctx, TCM_WAIT_ALL) once everything is, and then reports what tcm_run
 * would (TCM_E_REPLICA on a deadlock assertion).  The copy-back runs on a stream of the library's own
 * after the kernels, so tcm_stats may be called as soon as the call returns (its kernels follow the
 * engine on the context's stream; its *_ms fields count the run only after TCM_WAIT_ALL).  The HOST
 * results are valid after TCM_WAIT_ALL; tcm_load_trace / tcm_reset / tcm_step / tcm_run /
 * tcm_run_async before it are TCM_E_STATE. */
#define TCM_WAIT_ENGINE 0
#define TCM_WAIT_ALL 1
tcm_status tcm_run_async(tcm_ctx* ctx);
tcm_status tcm_wait(tcm_ctx* ctx, int what);

/* Fills *out (may be NULL) and, when dev_hist / dev_cnt are non-NULL, writes the a6
 * aggregation: dev_hist[n_cells][4][496] and dev_cnt[n_cells][4][6] (int64, DEVICE,
 * overwritten; groups M, C, T, all; counters n, sum TTFT, sum E2E, SLO violations,
 * sum (e2e*den - num*iso) over violators, sum floor(e2e/out)).  These buffers are
 * NCCL-ready: all-reduce(SUM) across GPUs gives the bit-exact global result. */
tcm_status tcm_stats(tcm_ctx* ctx, tcm_stats_host* out, int64_t* dev_hist, int64_t* dev_cnt);

/* Per-replica work counters of the bound trace since the last load / reset, written to dev_out
 * (DEVICE, uint64 [n_replicas][6], overwritten): engine iterations (fast-forwarded ones included),
 * decisions (R17), sum of the pending-set size over decisions, scanned decisions (FUSED: decisions
 * not taken in closed form; STEPWISE: all), requests done, preemptions
 * (TCM_KV_GROWTH).  The same quantities the oracle counts per replica, so a test can compare them
 * replica by replica.  Errors: TCM_E_ARG, TCM_E_STATE before tcm_load_trace. */
tcm_status tcm_replica_counters(tcm_ctx* ctx, uint64_t* dev_out);

/* fig:preemptions per (cell, group): dev_out (DEVICE, int64
 * [n_cells][4][3], overwritten; groups M, C, T, all by the engine's own a1 classifier) = number of
 * preemptions, total preempted time (us, R31) and number of requests preempted at least once, over
 * the per-request NEXT-1 results of the bound trace (replicas without TCM_KV_GROWTH add zeros).
 * Errors: TCM_E_ARG, TCM_E_STATE before tcm_load_trace. */
tcm_status tcm_preemption_stats(tcm_ctx* ctx, int64_t* dev_out);

/* Releases the workspace and the context (NULL is a no-op). */
void tcm_destroy(tcm_ctx* ctx);

/* Message of the last failing call on ctx ("" if none; ctx NULL -> last global error). */
const char* tcm_last_error(const tcm_ctx* ctx);

/* Device bytes the library allocates for a trace of this shape (excluding caller buffers,
 * including mirrors of HOST traces / results when `host_mirror` is non-zero). */
size_t tcm_workspace_bytes(const tcm_config* cfg, uint32_t n_replicas, uint64_t n_requests,
                           int host_mirror);

/* Generates traces on the device (bit-identical to tracegen/ on the host): replica r
 * fills [req_offset[r], req_offset[r+1]), which must equal reps[r].n_requests.  All
 * pointers are DEVICE.  Enqueued on cuda_stream; synchronises it. */
tcm_status tcm_generate_trace(const tcm_gen_replica* reps, uint32_t n_replicas,
                              const uint64_t* req_offset, uint64_t* arrival_us,
                              uint32_t* footprint, uint32_t* inline_us, uint16_t* out_tokens,
                              uint8_t* modality, void* cuda_stream);

/* Diagnostics for the K1 key, DEVICE pointers:
 * tcm_k1_eval writes P = K1(cls[i], w[i]) for alpha[i] (n elements) using cfg's S,k,p;
 * tcm_k1_audit writes to *first_violation (device u64) the smallest w in [w_lo, w_hi)
 * with key(w+1) < key(w) for class `cls` and `alpha` (UINT64_MAX if none). */
tcm_status tcm_k1_eval(const tcm_config* cfg, const uint8_t* cls, const uint64_t* w,
                       const double* alpha, double* out_priority, uint64_t n, void* cuda_stream);
tcm_status tcm_k1_audit(const tcm_config* cfg, uint32_t cls, double alpha, uint64_t w_lo,
                        uint64_t w_hi, uint64_t* first_violation, void* cuda_stream);
/* Max |P~ - P| over w = w_lo, w_lo + step, ... < w_hi of the stepwise engine's FP32 priority
 * bound P~ against K1; written to *max_err (HOST).  The engine assumes <= 1e-4. */
tcm_status tcm_k1_filter_error(const tcm_config* cfg, uint32_t cls, double alpha, uint64_t w_lo,
                               uint64_t w_hi, uint64_t step, double* max_err, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif
