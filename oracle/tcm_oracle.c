/*
 * tcm_oracle.c -- TEST INFRASTRUCTURE ONLY (see tcm_oracle.h).
 *
 * A plain, slow, obviously-correct CPU simulator of TCM-Serve's per-iteration
 * scheduling step (arxiv 2603.26498).  It follows SURVEY.md 8(c) step by step:
 * every decision re-keys EVERY pending request and fully sorts them (no class-FIFO
 * merge, no fast-forward, no incremental state).  Build: gcc -O2 -ffp-contract=off,
 * no fast-math (every floating-point operation is written out).
 *
 * Parity pins: tests/test_oracle_*.py (-m "not gpu").  Parity status per function is
 * listed in DESIGN.md "Oracle pins".
 */
#include "tcm_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------ */
/* K1 constants, transcribed from DESIGN.md "K1 constants" (hex floats).           */
/* ------------------------------------------------------------------------------ */
static const double ORC_LN2 = 0x1.62e42fefa39efp-1;

/* LN reduction table: R[j] = k_j / 256, LT[j] = -ln(R[j]) rounded to nearest. */
static const double ORC_LN_R[16] = {
    0x1.f000000000000p-1, 0x1.d400000000000p-1, 0x1.ba00000000000p-1, 0x1.a400000000000p-1,
    0x1.9000000000000p-1, 0x1.7e00000000000p-1, 0x1.6c00000000000p-1, 0x1.5c00000000000p-1,
    0x1.4e00000000000p-1, 0x1.4200000000000p-1, 0x1.3600000000000p-1, 0x1.2a00000000000p-1,
    0x1.2000000000000p-1, 0x1.1600000000000p-1, 0x1.0c00000000000p-1, 0x1.0400000000000p-1};
static const double ORC_LN_LT[16] = {
    0x1.0415d89e74444p-5, 0x1.700d30aeac0e1p-4, 0x1.2d1610c86813ap-3, 0x1.95a5adcf7017fp-3,
    0x1.f991c6cb3b379p-3, 0x1.2bef07cdc9354p-2, 0x1.5d5bddf595f30p-2, 0x1.8b639a88b2df5p-2,
    0x1.b56fa04462909p-2, 0x1.dae75484c9616p-2, 0x1.00e5ae5b207abp-1, 0x1.151c3f6f29612p-1,
    0x1.269621134db92p-1, 0x1.38ae2171976e7p-1, 0x1.4b6fd6f970c1fp-1, 0x1.5af405c3649e0p-1};
/* ln(1+u) series coefficients c_n = (-1)^(n+1)/n, n = 1..9 (index n-1). */
static const double ORC_LN_C[9] = {
    0x1.0000000000000p+0, -0x1.0000000000000p-1, 0x1.5555555555555p-2, -0x1.0000000000000p-2,
    0x1.999999999999ap-3, -0x1.5555555555555p-3, 0x1.2492492492492p-3, -0x1.0000000000000p-3,
    0x1.c71c71c71c71cp-4};

static const double ORC_INV_LN2_16 = 0x1.71547652b82fep+4;
static const double ORC_LN2_16_HI = 0x1.62e42fee00000p-5;
static const double ORC_LN2_16_LO = 0x1.a39ef35793c76p-37;
static const double ORC_EXP_T[16] = {
    0x1.0000000000000p+0, 0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};
/* 1/n!, n = 0..6 */
static const double ORC_EXP_E[7] = {
    0x1.0000000000000p+0, 0x1.0000000000000p+0, 0x1.0000000000000p-1, 0x1.5555555555555p-3,
    0x1.5555555555555p-5, 0x1.1111111111111p-7, 0x1.6c16c16c16c17p-10};

static uint64_t orc_bits(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }
static double orc_from_bits(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }

/* LN(v): DESIGN.md "K1" step LN.1-LN.6.  v must be a positive normal double. */
double orc_ln(double v)
{
    uint64_t bits = orc_bits(v);
    int e = (int)((bits >> 52) & 0x7FF) - 1023;                 /* LN.1 exponent   */
    int j = (int)((bits >> 48) & 0xF);                          /* LN.2 table index */
    double m = orc_from_bits((bits & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);
    double u = fma(m, ORC_LN_R[j], -1.0);                       /* LN.3            */
    double q = ORC_LN_C[8];                                      /* LN.4 Horner     */
    for (int i = 7; i >= 0; --i) q = fma(q, u, ORC_LN_C[i]);
    double lnm = q * u;                                          /* LN.5            */
    double t = ORC_LN_LT[j] + lnm;
    return fma((double)e, ORC_LN2, t);                           /* LN.6            */
}

/* EXP(y): DESIGN.md "K1" step EXP.1-EXP.7. */
double orc_exp(double y)
{
    if (y < -745.0) return 0.0;                                  /* EXP.1 */
    if (y > 700.0) return INFINITY;
    double kf = rint(y * ORC_INV_LN2_16);                        /* EXP.2 half-even */
    double r = fma(-kf, ORC_LN2_16_HI, y);                       /* EXP.3 */
    r = fma(-kf, ORC_LN2_16_LO, r);
    double p = ORC_EXP_E[6];                                     /* EXP.4 Horner */
    for (int i = 5; i >= 0; --i) p = fma(p, r, ORC_EXP_E[i]);
    int64_t k = (int64_t)kf;                                     /* EXP.5 */
    int64_t j = k & 15;
    int64_t n = (k - j) / 16;
    double s = ORC_EXP_T[j] * p;                                 /* EXP.6 */
    if (n < -1021) return 0.0;                                   /* EXP.7 flush */
    double res = s * orc_from_bits((uint64_t)(n + 1023) << 52);
    if (res < 0x1p-1022) return 0.0;
    return res;
}

/* C_c = LN(alpha*k_c) - p_c * LN(10^6): converts w in microseconds to seconds (R1). */
double orc_k1_const(double alpha, double k, double p, int* zero_rate)
{
    double a = alpha * k;
    if (!(a >= 0x1p-1022)) { *zero_rate = 1; return 0.0; }
    *zero_rate = 0;
    double t = p * orc_ln(1000000.0);
    return orc_ln(a) - t;
}

/* Priority_c = StaticPriority_c + (1 - e^{-k_c * waiting_time^{p_c}}). */
double orc_priority(double S, double p, double C, int zero_rate, uint64_t w_us)
{
    if (w_us == 0 || zero_rate) return S;
    double v = (double)w_us;
    double L = orc_ln(v);
    double y = fma(p, L, C);
    double x = orc_exp(y);
    double e = orc_exp(-x);
    return S + (1.0 - e);
}

/* Score = -log(Priority) is strictly decreasing, so ordering by max(P, eps)
 * descending is the same order (R3). */
uint64_t orc_key_bits(double priority)
{
    double q = priority < 1e-12 ? 1e-12 : priority;
    return orc_bits(q);
}

/* Smart classifier represented by per-modality footprint thresholds (R13). */
int orc_classify(const orc_model* m, uint8_t modality, uint32_t footprint)
{
    if (footprint < m->thr_mc[modality]) return 0;   /* motorcycle */
    if (footprint < m->thr_ct[modality]) return 1;   /* car        */
    return 2;                                         /* truck      */
}

/* Isolated (no-contention) TTFT / E2E, SPEC.md:141-149 in integer microseconds (R9). */
uint64_t orc_iso_ttft(const orc_model* m, uint32_t B, uint32_t f, uint32_t inl)
{
    uint64_t chunks = ((uint64_t)f + B - 1) / B;
    return (uint64_t)inl + chunks * m->c0_us + m->cp_us * (uint64_t)f;
}

uint64_t orc_iso_e2e(const orc_model* m, uint32_t B, uint32_t f, uint32_t inl, uint16_t out)
{
    return orc_iso_ttft(m, B, f, inl) + (uint64_t)(out - 1) * (m->c0_us + m->cd_us);
}

/* ------------------------------------------------------------------------------ */
/* The engine loop: SURVEY.md 8(c) steps 1-10.    */
/* ------------------------------------------------------------------------------ */
typedef struct {
    double   P;
    uint64_t arrival;
    uint64_t dl;        /* EDF: deadline x den = arrival*den + num*iso_e2e; aging: clock - arrival */
    uint32_t id;
} orc_entry;

/* Order: priority descending, then arrival ascending, then id ascending (R4). */
static int orc_cmp(const void* a, const void* b)
{
    const orc_entry* x = (const orc_entry*)a;
    const orc_entry* y = (const orc_entry*)b;
    uint64_t kx = orc_key_bits(x->P), ky = orc_key_bits(y->P);
    if (kx != ky) return kx > ky ? -1 : 1;
    if (x->arrival != y->arrival) return x->arrival < y->arrival ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return 0;
}

/* EDF: deadline ascending, then arrival, then id. */
static int orc_cmp_edf(const void* a, const void* b)
{
    const orc_entry* x = (const orc_entry*)a;
    const orc_entry* y = (const orc_entry*)b;
    if (x->dl != y->dl) return x->dl < y->dl ? -1 : 1;
    if (x->arrival != y->arrival) return x->arrival < y->arrival ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}

/* Naive aging: waiting time descending, then arrival, then id. */
static int orc_cmp_age(const void* a, const void* b)
{
    const orc_entry* x = (const orc_entry*)a;
    const orc_entry* y = (const orc_entry*)b;
    if (x->dl != y->dl) return x->dl > y->dl ? -1 : 1;
    if (x->arrival != y->arrival) return x->arrival < y->arrival ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}

/* One decision, over the pending ids `pending[0..n_pend)` (id order):
 * 3 the budget left after decodes (R8); 4-5 key every pending request and sort (TCM), or take
 * arrival order (FCFS); 6 the greedy admission scan, where the first KV misfit blocks later NEW
 * admits but partials still get chunks (R5-R7).  Updates rem / reserved / kv_free / seq /
 * admit_seq in place; returns Bp. */
static uint32_t orc_admit_step(const orc_model* m, const orc_replica* r, const double* C, const int* zero,
                               uint64_t clock, uint32_t n_dec, uint32_t n_pend, const uint32_t* pending,
                               const uint64_t* arrival, const uint32_t* f, const uint32_t* inl,
                               const uint16_t* out, const uint8_t* cls, uint32_t* rem, uint8_t* reserved,
                               uint64_t* kv_free_io, uint32_t* seq_io, uint32_t* admit_seq,
                               orc_entry* order, uint64_t* tok_out, uint64_t* inl_out,
                               uint32_t* n_admitted)
{
    /* 3 budget left after decodes (R8) */
    uint32_t Bp = r->chunk_budget > n_dec ? r->chunk_budget - n_dec : 0;

    /* 4-5 key every pending request and sort (TCM), or arrival order (FCFS) */
    for (uint32_t q = 0; q < n_pend; ++q) {
        uint32_t i = pending[q];
        order[q].id = i;
        order[q].arrival = arrival[i];
        order[q].P = 0.0;
        order[q].dl = 0;
        if (r->policy == ORC_TCM) {
            int c = cls[i];
            order[q].P = orc_priority(m->S[c], m->p[c], C[c], zero[c], clock - arrival[i]);
        } else if (r->policy == ORC_EDF) {
            order[q].dl = arrival[i] * m->slo_den +
                          m->slo_num * orc_iso_e2e(m, r->chunk_budget, f[i], inl[i], out[i]);
        } else if (r->policy == ORC_NAIVE_AGING) {
            order[q].dl = clock - arrival[i];
        }
    }
    if (r->policy == ORC_TCM) qsort(order, n_pend, sizeof(orc_entry), orc_cmp);
    if (r->policy == ORC_EDF) qsort(order, n_pend, sizeof(orc_entry), orc_cmp_edf);
    if (r->policy == ORC_NAIVE_AGING) qsort(order, n_pend, sizeof(orc_entry), orc_cmp_age);

    /* 6 admission scan: greedy chunks; first KV misfit blocks later NEW admits (R6) */
    uint64_t kv_free = *kv_free_io;
    uint32_t seq = *seq_io;
    uint32_t left = Bp;
    int blocked = 0;
    uint64_t tok = 0, inl_sum = 0;
    for (uint32_t q = 0; q < n_pend; ++q) {
        uint32_t i = order[q].id;
        if (left == 0) break;
        if (!reserved[i]) {
            if (blocked) continue;
            if ((uint64_t)f[i] > kv_free) { blocked = !r->admit_skip; continue; }
            reserved[i] = 1;
            kv_free -= f[i];
            admit_seq[i] = seq++;
            inl_sum += inl[i];
            (*n_admitted)++;
        }
        uint32_t c = rem[i] < left ? rem[i] : left;
        rem[i] -= c;
        left -= c;
        tok += c;
    }
    *kv_free_io = kv_free;
    *seq_io = seq;
    *tok_out = tok;
    *inl_out = inl_sum;
    return Bp;
}

/* One decision on an explicit state (test infrastructure: SURVEY.md 8(c) single-step brute force).
 * Requests 0..n-1 are all pending, in id order; rem / reserved carry partial prefills in and the
 * decision out; admit_seq[i] = the admission rank of a request admitted now, else unchanged.
 * res[0] = tokens scheduled, res[1] = inline time charged, res[2] = kv_free after, res[3] = Bp. */
int orc_decide(const orc_model* m, const orc_replica* r, uint32_t n, uint64_t clock, uint64_t kv_free,
               uint32_t n_dec, const uint64_t* arrival, const uint32_t* f, const uint32_t* inl,
               const uint16_t* out, const uint8_t* cls, uint32_t* rem, uint8_t* reserved,
               uint32_t* admit_seq, uint64_t* res)
{
    if (r->chunk_budget == 0 || r->policy > ORC_NAIVE_AGING || r->admit_skip > 1) return -1;
    double C[3];
    int zero[3];
    for (int c = 0; c < 3; ++c) C[c] = orc_k1_const(r->alpha, m->k[c], m->p[c], &zero[c]);
    uint32_t* pending = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    orc_entry* order = (orc_entry*)malloc(sizeof(orc_entry) * (n + 1));
    if (!pending || !order) { free(pending); free(order); return -1; }
    for (uint32_t i = 0; i < n; ++i) pending[i] = i;
    uint32_t seq = 0, nadm = 0;
    uint64_t tok = 0, inl_sum = 0;
    uint32_t Bp = orc_admit_step(m, r, C, zero, clock, n_dec, n, pending, arrival, f, inl, out, cls, rem,
                                 reserved, &kv_free, &seq, admit_seq, order, &tok, &inl_sum, &nadm);
    res[0] = tok;
    res[1] = inl_sum;
    res[2] = kv_free;
    res[3] = Bp;
    free(pending); free(order);
    return 0;
}

int orc_simulate(const orc_model* m, const orc_replica* r, uint32_t n,
                 const uint64_t* arrival, const uint32_t* f, const uint32_t* inl,
                 const uint16_t* out, const uint8_t* mod, uint32_t* admit_seq,
                 uint64_t* first_token, uint64_t* done, uint8_t* cls_out,
                 orc_counters* cnt, orc_iter_rec* log, uint64_t log_cap, uint64_t* log_n,
                 uint64_t max_iters)
{
    memset(cnt, 0, sizeof(*cnt));
    if (log_n) *log_n = 0;
    if (r->chunk_budget == 0 || r->policy > ORC_NAIVE_AGING || r->admit_skip > 1) return -1;
    for (uint32_t i = 0; i < n; ++i) {
        if (f[i] == 0 || f[i] > r->kv_capacity || out[i] == 0 || mod[i] > 2) return -1;
        if (i > 0 && arrival[i] < arrival[i - 1]) return -1;
    }

    double C[3];
    int zero[3];
    for (int c = 0; c < 3; ++c) C[c] = orc_k1_const(r->alpha, m->k[c], m->p[c], &zero[c]);

    uint32_t* pending = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t* decoding = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t* rem = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint32_t* gen = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
    uint8_t* reserved = (uint8_t*)calloc(n + 1, 1);
    orc_entry* order = (orc_entry*)malloc(sizeof(orc_entry) * (n + 1));
    if (!pending || !decoding || !rem || !gen || !reserved || !order) {
        free(pending); free(decoding); free(rem); free(gen); free(reserved); free(order);
        return -1;
    }

    uint64_t clock = 0, kv_free = r->kv_capacity, iter = 0;
    uint32_t nxt = 0, seq = 0, n_pend = 0, n_dec = 0;
    int status = 0;

    for (;;) {
        if (max_iters && iter >= max_iters) break;   /* truncated run (test infrastructure) */
        /* 1 ingest arrivals <= clock, classify on ingest */
        while (nxt < n && arrival[nxt] <= clock) {
            cls_out[nxt] = (uint8_t)orc_classify(m, mod[nxt], f[nxt]);
            rem[nxt] = f[nxt];
            reserved[nxt] = 0;
            pending[n_pend++] = nxt;
            ++nxt;
        }
        /* 2 idle: jump to the next arrival (R15), not an iteration */
        if (n_pend == 0 && n_dec == 0) {
            if (nxt == n) break;
            clock = arrival[nxt];
            cnt->idle_jumps++;
            continue;
        }
        orc_iter_rec rec;
        memset(&rec, 0, sizeof(rec));
        rec.clock_start = clock;
        rec.kv_free_start = kv_free;
        rec.n_pending = n_pend;
        rec.n_dec = n_dec;

        /* 3-6 budget, keys, order, admission scan (one decision) */
        uint64_t tok = 0, inl_sum = 0;
        uint32_t Bp = orc_admit_step(m, r, C, zero, clock, n_dec, n_pend, pending, arrival, f, inl, out,
                                     cls_out, rem, reserved, &kv_free, &seq, admit_seq, order,
                                     &tok, &inl_sum, &rec.n_admitted);
        rec.budget = Bp;
        rec.kv_free_admit = kv_free;
        rec.tokens = (uint32_t)tok;

        /* 7 progress is guaranteed under R6 */
        if (tok == 0 && n_dec == 0) { status = -2; break; }

        /* 8 iteration cost and clock (R9, R10) */
        clock += m->c0_us + m->cp_us * tok + m->cd_us * (uint64_t)n_dec + inl_sum;
        iter++;
        cnt->iterations++;
        if (n_pend > 0) {                     /* R17: only iterations with pending work */
            cnt->decisions++;
            cnt->sum_pending += n_pend;
            if (n_pend > cnt->max_pending) cnt->max_pending = n_pend;
        }

        /* 9 every decoding sequence emits one token; finished ones release KV (R7) */
        uint32_t kept = 0;
        for (uint32_t q = 0; q < n_dec; ++q) {
            uint32_t d = decoding[q];
            gen[d]++;
            if (gen[d] == out[d]) {
                done[d] = clock;
                kv_free += f[d];
            } else {
                decoding[kept++] = d;
            }
        }
        n_dec = kept;

        /* 10 requests whose prefill completed emit their first token now (R12) */
        kept = 0;
        for (uint32_t q = 0; q < n_pend; ++q) {
            uint32_t i = pending[q];
            if (reserved[i] && rem[i] == 0) {
                first_token[i] = clock;
                gen[i] = 1;
                rec.n_first_tokens++;
                if (out[i] == 1) {
                    done[i] = clock;
                    kv_free += f[i];
                } else {
                    decoding[n_dec++] = i;
                }
            } else {
                if (reserved[i]) rec.n_partial_after++;
                pending[kept++] = i;
            }
        }
        n_pend = kept;
        rec.clock_end = clock;
        if (log && *log_n < log_cap) log[*log_n] = rec;
        if (log_n) (*log_n)++;
    }
    cnt->admitted = seq;
    cnt->final_clock = clock;

    free(pending); free(decoding); free(rem); free(gen); free(reserved); free(order);
    return status;
}

/* ------------------------------------------------------------------------------ */
/* NEXT-1: decode KV growth + preemption by recomputation (R28-R32).  */
/* Written as its own loop (the R7 loop above stays as pinned); request phases are  */
/* kept per id and every set is a plain scan over ids 0..nxt-1, in id order.        */
/* ------------------------------------------------------------------------------ */
enum { PH_WAIT = 1, PH_PREFILL = 2, PH_DECODE = 3, PH_DONE = 4 };

/* EDF key of request i: its deadline x den = arrival*den + num*iso_e2e (R27). */
static uint64_t orc_edf_key(const orc_model* m, const orc_replica* r, uint32_t i, const uint64_t* arrival,
                            const uint32_t* f, const uint32_t* inl, const uint16_t* out)
{
    return arrival[i] * m->slo_den + m->slo_num * orc_iso_e2e(m, r->chunk_budget, f[i], inl[i], out[i]);
}

int orc_simulate_growth(const orc_model* m, const orc_replica* r, uint32_t n,
                        const uint64_t* arrival, const uint32_t* f, const uint32_t* inl,
                        const uint16_t* out, const uint8_t* mod, uint32_t* admit_seq,
                        uint64_t* first_token, uint64_t* done, uint32_t* pcount,
                        uint64_t* ptime, uint8_t* cls_out, orc_counters* cnt,
                        uint64_t* n_preempt, uint64_t* n_forced, uint64_t max_iters)
{
    memset(cnt, 0, sizeof(*cnt));
    *n_preempt = 0;
    *n_forced = 0;
    if (r->chunk_budget == 0 || r->policy > ORC_NAIVE_AGING || r->admit_skip > 1) return -1;
    for (uint32_t i = 0; i < n; ++i) {
        /* R28: the largest allocation a request can reach must fit on its own */
        if (f[i] == 0 || out[i] == 0 || mod[i] > 2) return -1;
        if ((uint64_t)f[i] + out[i] - 1 > r->kv_capacity) return -1;
        if (i > 0 && arrival[i] < arrival[i - 1]) return -1;
    }
    double C[3];
    int zero[3];
    for (int c = 0; c < 3; ++c) C[c] = orc_k1_const(r->alpha, m->k[c], m->p[c], &zero[c]);

    uint8_t* ph = (uint8_t*)calloc(n + 1, 1);
    uint8_t* admitted = (uint8_t*)calloc(n + 1, 1);
    uint8_t* emitted = (uint8_t*)calloc(n + 1, 1);     /* first token emitted */
    uint32_t* rem = (uint32_t*)calloc(n + 1, 4);
    uint32_t* held = (uint32_t*)calloc(n + 1, 4);
    uint32_t* gen = (uint32_t*)calloc(n + 1, 4);
    uint64_t* pstart = (uint64_t*)calloc(n + 1, 8);
    uint64_t* pre_it = (uint64_t*)calloc(n + 1, 8);    /* EDF inversion victims: iteration + 1 (R34) */
    orc_entry* order = (orc_entry*)malloc(sizeof(orc_entry) * (n + 1));
    if (!ph || !admitted || !emitted || !rem || !held || !gen || !pstart || !pre_it || !order) {
        free(ph); free(admitted); free(emitted); free(rem); free(held); free(gen); free(pstart); free(pre_it);
        free(order);
        return -1;
    }
    for (uint32_t i = 0; i < n; ++i) { pcount[i] = 0; ptime[i] = 0; }

    uint64_t clock = 0, kv_free = r->kv_capacity, iter = 0;
    uint32_t nxt = 0, seq = 0;
    int status = 0;
    for (;;) {
        if (max_iters && iter >= max_iters) break;
        /* 1 ingest */
        while (nxt < n && arrival[nxt] <= clock) {
            cls_out[nxt] = (uint8_t)orc_classify(m, mod[nxt], f[nxt]);
            ph[nxt] = PH_WAIT;
            rem[nxt] = f[nxt];
            ++nxt;
        }
        uint32_t n_pend = 0, n_dec = 0;
        for (uint32_t i = 0; i < nxt; ++i) {
            if (ph[i] == PH_WAIT || ph[i] == PH_PREFILL) n_pend++;
            if (ph[i] == PH_DECODE) n_dec++;
        }
        /* 2 idle jump (R15) */
        if (n_pend == 0 && n_dec == 0) {
            if (nxt == n) break;
            clock = arrival[nxt];
            cnt->idle_jumps++;
            continue;
        }
        /* 3a memory exhaustion: one KV token per decoding sequence this iteration (R28);
         * preempt victims until it fits (R29) */
        while (kv_free < n_dec) {
            uint32_t v = UINT32_MAX;
            int forced = 0;
            if (r->policy == ORC_TCM) {
                /* the running request ranked last by (P desc, arrival asc, id asc),
                 * motorcycles only when no other class is running */
                for (int pass = 0; pass < 2 && v == UINT32_MAX; ++pass) {
                    double vP = 0.0;
                    for (uint32_t i = 0; i < nxt; ++i) {
                        if (ph[i] != PH_PREFILL && ph[i] != PH_DECODE) continue;
                        int c = cls_out[i];
                        if (pass == 0 && c == 0) continue;
                        double P = orc_priority(m->S[c], m->p[c], C[c], zero[c], clock - arrival[i]);
                        uint64_t kb = orc_key_bits(P), vb = orc_key_bits(vP);
                        /* later in the order: smaller key, or equal key and later (arrival, id) */
                        if (v == UINT32_MAX || kb < vb || (kb == vb && i > v)) { v = i; vP = P; }
                    }
                    forced = pass == 1;
                }
            } else {
                for (uint32_t i = 0; i < nxt; ++i)       /* most recently arrived */
                    if (ph[i] == PH_PREFILL || ph[i] == PH_DECODE) v = i;
            }
            if (v == UINT32_MAX) { status = -2; break; }   /* unreachable: n_dec > 0 */
            if (ph[v] == PH_DECODE) { n_dec--; n_pend++; }
            kv_free += held[v];
            rem[v] = held[v];          /* recomputation: prompt + generated tokens again (R30) */
            held[v] = 0;
            ph[v] = PH_WAIT;
            pcount[v]++;
            pstart[v] = clock;
            (*n_preempt)++;
            if (forced) (*n_forced)++;
        }
        if (status) break;
        /* 3b the decode tokens of this iteration take their KV */
        kv_free -= n_dec;
        for (uint32_t i = 0; i < nxt; ++i)
            if (ph[i] == PH_DECODE) held[i]++;
        uint32_t Bp = r->chunk_budget > n_dec ? r->chunk_budget - n_dec : 0;

        /* 4-5 order the pending requests (as orc_simulate) */
        uint32_t np = 0;
        for (uint32_t i = 0; i < nxt; ++i) {
            if (ph[i] != PH_WAIT && ph[i] != PH_PREFILL) continue;
            order[np].id = i;
            order[np].arrival = arrival[i];
            order[np].P = 0.0;
            order[np].dl = 0;
            if (r->policy == ORC_TCM) {
                int c = cls_out[i];
                order[np].P = orc_priority(m->S[c], m->p[c], C[c], zero[c], clock - arrival[i]);
            } else if (r->policy == ORC_EDF) {
                order[np].dl = arrival[i] * m->slo_den +
                               m->slo_num * orc_iso_e2e(m, r->chunk_budget, f[i], inl[i], out[i]);
            } else if (r->policy == ORC_NAIVE_AGING) {
                order[np].dl = clock - arrival[i];
            }
            np++;
        }
        if (r->policy == ORC_TCM) qsort(order, np, sizeof(orc_entry), orc_cmp);
        if (r->policy == ORC_EDF) qsort(order, np, sizeof(orc_entry), orc_cmp_edf);
        if (r->policy == ORC_NAIVE_AGING) qsort(order, np, sizeof(orc_entry), orc_cmp_age);

        /* 6 admission scan (R5-R8); a re-admission reserves what it will re-prefill (R30) */
        uint32_t left = Bp;
        int blocked = 0;
        uint64_t tok = 0, inl_sum = 0;
        for (uint32_t q = 0; q < np; ++q) {
            uint32_t i = order[q].id;
            if (left == 0) break;
            if (ph[i] == PH_WAIT) {
                if (blocked) continue;
                if (pre_it[i] == iter + 1) continue;      /* preempted for an earlier deadline just now (R34) */
                if ((uint64_t)rem[i] > kv_free && r->policy == ORC_EDF) {
                    /* R34 EDF priority inversion: running requests that come
                     * after i in EDF order (deadline, arrival, id) are preempted, latest first, until i
                     * fits -- only if preempting all of them would make it fit. */
                    const uint64_t dw = order[q].dl;
                    uint64_t avail = kv_free;
                    for (uint32_t v = 0; v < nxt; ++v) {
                        if (ph[v] != PH_PREFILL && ph[v] != PH_DECODE) continue;
                        const uint64_t dv = orc_edf_key(m, r, v, arrival, f, inl, out);
                        if (dv > dw || (dv == dw && (arrival[v] > arrival[i] || (arrival[v] == arrival[i] && v > i))))
                            avail += held[v];
                    }
                    while (avail >= rem[i] && (uint64_t)rem[i] > kv_free) {
                        uint32_t v = UINT32_MAX;
                        uint64_t vd = 0;
                        for (uint32_t u = 0; u < nxt; ++u) {
                            if (ph[u] != PH_PREFILL && ph[u] != PH_DECODE) continue;
                            const uint64_t du = orc_edf_key(m, r, u, arrival, f, inl, out);
                            const int after = du > dw || (du == dw && (arrival[u] > arrival[i] ||
                                                                       (arrival[u] == arrival[i] && u > i)));
                            /* the latest in EDF order among them: max (deadline, arrival, id) */
                            if (after && (v == UINT32_MAX || du > vd ||
                                          (du == vd && (arrival[u] > arrival[v] || (arrival[u] == arrival[v] && u > v))))) {
                                v = u;
                                vd = du;
                            }
                        }
                        if (ph[v] == PH_DECODE) {
                            n_dec--;                      /* it does not decode in this iteration */
                            rem[v] = held[v] - 1;         /* recompute what it held before this iteration */
                        } else {
                            rem[v] = held[v];
                        }
                        kv_free += held[v];               /* including this iteration's decode token */
                        held[v] = 0;
                        ph[v] = PH_WAIT;
                        pre_it[v] = iter + 1;
                        pcount[v]++;
                        pstart[v] = clock;
                        (*n_preempt)++;
                    }
                }
                if ((uint64_t)rem[i] > kv_free) { blocked = !r->admit_skip; continue; }
                ph[i] = PH_PREFILL;
                held[i] = rem[i];
                kv_free -= rem[i];
                if (!admitted[i]) {
                    admitted[i] = 1;
                    admit_seq[i] = seq++;
                    inl_sum += inl[i];
                } else {
                    ptime[i] += clock - pstart[i];       /* R31 */
                }
            }
            uint32_t c = rem[i] < left ? rem[i] : left;
            rem[i] -= c;
            left -= c;
            tok += c;
        }
        if (tok == 0 && n_dec == 0) { status = -2; break; }

        /* 8 cost and clock */
        clock += m->c0_us + m->cp_us * tok + m->cd_us * (uint64_t)n_dec + inl_sum;
        iter++;
        cnt->iterations++;
        if (np > 0) {
            cnt->decisions++;
            cnt->sum_pending += np;
            if (np > cnt->max_pending) cnt->max_pending = np;
        }
        /* 9 decode tokens; finished sequences release everything they hold */
        for (uint32_t i = 0; i < nxt; ++i) {
            if (ph[i] != PH_DECODE) continue;
            gen[i]++;
            if (gen[i] == out[i]) {
                done[i] = clock;
                kv_free += held[i];
                held[i] = 0;
                ph[i] = PH_DONE;
            }
        }
        /* 10 completed prefills emit a token: the first one (R12) or, after a re-prefill,
         * the next one (R30) */
        for (uint32_t i = 0; i < nxt; ++i) {
            if (ph[i] != PH_PREFILL || rem[i] != 0) continue;
            if (!emitted[i]) {
                emitted[i] = 1;
                first_token[i] = clock;
            }
            gen[i]++;
            if (gen[i] == out[i]) {
                done[i] = clock;
                kv_free += held[i];
                held[i] = 0;
                ph[i] = PH_DONE;
            } else {
                ph[i] = PH_DECODE;
            }
        }
    }
    cnt->admitted = seq;
    cnt->final_clock = clock;
    free(ph); free(admitted); free(emitted); free(rem); free(held); free(gen); free(pstart); free(pre_it);
    free(order);
    return status;
}

/* ------------------------------------------------------------------------------ */
/* a6: result aggregation (PAPER.md:579 SLO = 5x isolated E2E).   */
/* ------------------------------------------------------------------------------ */

/* HDR-style log bucket: t < 16 -> t; else with
 * e = floor(log2 t): 16 + 8*(e-4) + the 3 bits below the leading one. */
uint32_t orc_ttft_bucket(uint64_t t)
{
    if (t < 16) return (uint32_t)t;
    uint32_t e = 0;
    while (e < 63 && (t >> (e + 1)) != 0) ++e;   /* e = floor(log2 t), plain loop */
    return 16u + 8u * (e - 4u) + (uint32_t)((t >> (e - 3u)) & 7u);
}

void orc_aggregate(const orc_model* m, uint32_t B, uint32_t n, const uint64_t* arrival,
                   const uint32_t* f, const uint32_t* inl, const uint16_t* out,
                   const uint8_t* mod, const uint64_t* first_token, const uint64_t* done,
                   int64_t* hist, int64_t* cnt)
{
    for (uint32_t i = 0; i < n; ++i) {
        int g = orc_classify(m, mod[i], f[i]);
        uint64_t ttft = first_token[i] - arrival[i];
        uint64_t e2e = done[i] - arrival[i];
        uint64_t iso = orc_iso_e2e(m, B, f[i], inl[i], out[i]);
        uint64_t lhs = e2e * m->slo_den, rhs = iso * m->slo_num;
        int viol = lhs > rhs;
        int groups[2] = {g, 3};
        for (int k = 0; k < 2; ++k) {
            int gg = groups[k];
            hist[gg * ORC_HIST_BINS + orc_ttft_bucket(ttft)] += 1;
            int64_t* c = cnt + gg * ORC_NCNT;
            c[0] += 1;                                  /* n                         */
            c[1] += (int64_t)ttft;                      /* sum TTFT (us)             */
            c[2] += (int64_t)e2e;                       /* sum E2E (us)              */
            c[3] += viol;                               /* SLO violations            */
            c[4] += viol ? (int64_t)(lhs - rhs) : 0;    /* sum severity x den (us)   */
            c[5] += (int64_t)(e2e / out[i]);            /* sum normalized lat (us/tok)*/
        }
    }
}

/* Lemma L1 audit: first w in [w_lo, w_hi) with key(w+1) < key(w),
 * or UINT64_MAX if K1 is non-decreasing on the whole range. Plain loop. */
uint64_t orc_audit_monotone(double S, double p, double C, int zero_rate,
                            uint64_t w_lo, uint64_t w_hi)
{
    uint64_t prev = orc_key_bits(orc_priority(S, p, C, zero_rate, w_lo));
    for (uint64_t w = w_lo + 1; w <= w_hi; ++w) {
        uint64_t k = orc_key_bits(orc_priority(S, p, C, zero_rate, w));
        if (k < prev) return w - 1;
        prev = k;
    }
    return UINT64_MAX;
}
