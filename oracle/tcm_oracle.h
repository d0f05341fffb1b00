/*
 * tcm_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, single-threaded CPU oracle for the TCM-Serve scheduling step
 * (arxiv 2603.26498).  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  It shares no code with the CUDA
 * path (paper_2603_26498_b200/csrc) and neither includes the other.
 *
 * Readings R1..R25 and the K1 specification are in DESIGN.md; every function below
 * cites the PAPER.md / SPEC.md passage it follows.
 */
#ifndef TCM_ORACLE_H
#define TCM_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Cost model, priority constants and classifier thresholds (shared by all replicas). */
typedef struct {
    uint64_t c0_us;       /* per-iteration overhead, SPEC.md:137 (5 ms)          */
    uint64_t cp_us;       /* per prefill token, SPEC.md:137 (20 us)              */
    uint64_t cd_us;       /* per decoding sequence, SPEC.md:137 (0.5 ms)         */
    double   S[3];        /* StaticPriority_c, PAPER.md:580 (0.1, 0.05, 0)       */
    double   k[3];        /* k_c, PAPER.md:580 (0.05, 0.003, 0.00075)            */
    double   p[3];        /* p_c, PAPER.md:580 (3.5, 2.5, 1.1)                   */
    uint32_t thr_mc[3];   /* per modality: footprint < thr_mc -> Motorcycle (R13) */
    uint32_t thr_ct[3];   /* per modality: footprint < thr_ct -> Car, else Truck  */
    uint32_t slo_num;     /* SLO = num/den x isolated E2E, PAPER.md:579 (5/1)    */
    uint32_t slo_den;
} orc_model;

/* FCFS: arrival order.  TCM: aging priority.
 * EDF: earliest deadline first, deadline = arrival + (num/den) x isolated E2E (
 * SPEC.md:399) -- ordering only, preemption is NEXT-1.  NAIVE_AGING: descending waiting time,
 * ignoring class. */
enum { ORC_FCFS = 0, ORC_TCM = 1, ORC_EDF = 2, ORC_NAIVE_AGING = 3 };

typedef struct {
    uint32_t policy;        /* ORC_*                                               */
    uint32_t chunk_budget;  /* B, chunked-prefill token budget      */
    uint64_t kv_capacity;   /* KV tokens               */
    double   alpha;         /* aging factor multiplying every k_c (R14)            */
    uint32_t admit_skip;    /* 1: a KV misfit is skipped, later requests may still be
                               admitted (first fit, NEXT-3); 0: it blocks them (R6) */
    uint32_t pad;
} orc_replica;

typedef struct {
    uint64_t iterations;    /* engine iterations (idle jumps excluded, R15)        */
    uint64_t decisions;     /* iterations with >= 1 pending request (R17)          */
    uint64_t sum_pending;   /* sum over decisions of |pending| at step 3           */
    uint64_t max_pending;
    uint64_t admitted;      /* requests admitted (== n at the end)                 */
    uint64_t idle_jumps;
    uint64_t final_clock;
} orc_counters;

/* One record per engine iteration (optional audit log for invariant tests). */
typedef struct {
    uint64_t clock_start;
    uint64_t clock_end;
    uint64_t kv_free_start;   /* after ingest, before admission              */
    uint64_t kv_free_admit;   /* after admission reservations                */
    uint32_t n_pending;
    uint32_t n_dec;           /* decoding sequences at the start              */
    uint32_t budget;          /* Bp = max(0, B - n_dec)                       */
    uint32_t tokens;          /* sum of prefill chunks                        */
    uint32_t n_admitted;      /* new admissions this iteration                */
    uint32_t n_first_tokens;  /* requests emitting their first token          */
    uint32_t n_partial_after; /* reserved requests with rem > 0 after the scan */
    uint32_t pad;
} orc_iter_rec;

/* ---- K1: the specified priority key, PAPER.md:457-461, 580 ---- */
double   orc_ln(double v);                       /* LN, v positive normal   */
double   orc_exp(double y);                      /* EXP                     */
double   orc_k1_const(double alpha, double k, double p, int* zero_rate); /* C_c */
double   orc_priority(double S, double p, double C, int zero_rate, uint64_t w_us);
uint64_t orc_key_bits(double priority);          /* bits of max(P, 1e-12)   */
/* first w in [w_lo, w_hi) with key(w+1) < key(w); UINT64_MAX if none (Lemma L1 audit) */
uint64_t orc_audit_monotone(double S, double p, double C, int zero_rate, uint64_t w_lo, uint64_t w_hi);

/* ---- classifier, R13 ---- */
int orc_classify(const orc_model* m, uint8_t modality, uint32_t footprint);

/* ---- isolated E2E (no contention), PAPER.md:579, SPEC.md:144 ---- */
uint64_t orc_iso_ttft(const orc_model* m, uint32_t chunk_budget, uint32_t footprint, uint32_t inline_us);
uint64_t orc_iso_e2e(const orc_model* m, uint32_t chunk_budget, uint32_t footprint, uint32_t inline_us, uint16_t out);

/*
 * Simulate one replica to completion (SURVEY.md 8(c) pseudo-code, steps 1-10).
 * Inputs: n requests sorted by (arrival, id).  Outputs (per request): admit_seq,
 * first_token_us, done_us, cls.  iter_log may be NULL; otherwise it receives up to
 * log_cap records and *log_n is set to the number of iterations.  max_iters > 0 stops the
 * run after that many engine iterations (for comparing the first steps of huge queues);
 * unfinished requests then keep admit_seq / first_token / done as initialised by the caller.
 * Returns 0, or -1 (argument/capacity error), -2 (deadlock: unreachable under R6).
 */
int orc_simulate(const orc_model* m, const orc_replica* r, uint32_t n,
                 const uint64_t* arrival_us, const uint32_t* footprint,
                 const uint32_t* inline_us, const uint16_t* out_tokens,
                 const uint8_t* modality,
                 uint32_t* admit_seq, uint64_t* first_token_us, uint64_t* done_us,
                 uint8_t* cls_out, orc_counters* cnt,
                 orc_iter_rec* iter_log, uint64_t log_cap, uint64_t* log_n,
                 uint64_t max_iters);

/*
 * One decision on an explicit state: requests 0..n-1 are all pending,
 * in id order, with their class, remaining prefill `rem` and reserved (partial) flag; the engine
 * has n_dec decoding sequences and kv_free free KV at `clock`.  This is the same code the engine
 * loop above runs for each decision.  On return rem / reserved hold the decision, admit_seq[i]
 * is the admission rank (0, 1, ...) of each request admitted now (others untouched), and
 * res = {tokens, inline_us charged, kv_free after, budget Bp}.  Returns 0 or -1 (bad argument).
 * Test infrastructure for the single-step brute force.
 */
int orc_decide(const orc_model* m, const orc_replica* r, uint32_t n, uint64_t clock, uint64_t kv_free,
               uint32_t n_dec, const uint64_t* arrival_us, const uint32_t* footprint,
               const uint32_t* inline_us, const uint16_t* out_tokens, const uint8_t* cls,
               uint32_t* rem, uint8_t* reserved, uint32_t* admit_seq, uint64_t* res);

/*
 * NEXT-1: the same engine loop with decode KV growth and preemption by
 * recomputation, readings R28-R32.  A running request holds its reservation plus
 * one KV token per decode iteration run.  At the start of every iteration, while
 * the free KV cannot cover one token per decoding sequence, a victim among the running requests
 * (reserved partial prefills and decoding sequences) is preempted (SPEC.md:87, 398, 402, 455(3)):
 * FCFS (and every non-TCM policy) takes the most recently arrived; TCM the lowest-ranked
 * non-motorcycle, a motorcycle only when every running request is one (counted in *n_forced).
 * The victim frees everything it holds and waits again with its original arrival;
 * its next admission reserves and re-prefills what it held, charges no inline time and takes
 * no admit_seq; completing that re-prefill emits its next token.  Per request also:
 * preempt_count and preempted_us (from the preemption to the next admission).
 * Requires footprint + out - 1 <= kv_capacity for every request (else -1).
 */
int orc_simulate_growth(const orc_model* m, const orc_replica* r, uint32_t n,
                        const uint64_t* arrival_us, const uint32_t* footprint,
                        const uint32_t* inline_us, const uint16_t* out_tokens,
                        const uint8_t* modality,
                        uint32_t* admit_seq, uint64_t* first_token_us, uint64_t* done_us,
                        uint32_t* preempt_count, uint64_t* preempted_us,
                        uint8_t* cls_out, orc_counters* cnt,
                        uint64_t* n_preempt, uint64_t* n_forced, uint64_t max_iters);

/* ---- a6 aggregation: HDR-style TTFT bucket and per-group counters ---- */
enum { ORC_HIST_BINS = 496, ORC_GROUPS = 4, ORC_NCNT = 6 };
uint32_t orc_ttft_bucket(uint64_t ttft_us);
/*
 * Adds one replica's results into hist[ORC_GROUPS][ORC_HIST_BINS] and
 * cnt[ORC_GROUPS][ORC_NCNT] = {n, sum_ttft, sum_e2e, slo_violations, sum_severity_x_den, sum(e2e/out)}.
 * Groups: 0 = M, 1 = C, 2 = T (class from the model's thresholds), 3 = all.
 */
void orc_aggregate(const orc_model* m, uint32_t chunk_budget, uint32_t n,
                   const uint64_t* arrival_us, const uint32_t* footprint,
                   const uint32_t* inline_us, const uint16_t* out_tokens,
                   const uint8_t* modality, const uint64_t* first_token_us,
                   const uint64_t* done_us, int64_t* hist, int64_t* cnt);

#ifdef __cplusplus
}
#endif
#endif
