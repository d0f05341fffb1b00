// tcm_stepwise.cu -- TCM_ENGINE_STEPWISE: the paper-literal per-iteration scheduling step.
//
// Every engine iteration, for every active replica, one GROUP of warps (a warp per replica for
// sweeps; a CTA for fewer, huge queues; a thread-block cluster of 8 CTAs for a handful of huge
// queues, its group state in rank 0's shared memory through DSMEM):
//   a1  ingests arrivals <= clock (ballots over 128 sorted arrivals per round) and classifies
//       them (R13) into the per-request state byte;
//   a2  streams EVERY pending request of the replica's window [lo, nxt) ("At each scheduling
//       iteration ... evaluates the state of all queues and dynamically adjusts priorities",
//       PAPER.md:315, 323): arrival (8 B) + state (1 B) per request through a per-warp cp.async
//       ring; a request is rejected by a per-class arrival limit derived from one FP32 bound of
//       K1 (monotone in the waiting time), else queued, in id order, for its exact K1 key;
//       the key is never stored;
//   a3  selects the top-32 candidates by (key desc, id asc): per-warp register lists updated by
//       ballot-rank insertion or warp-shuffle bitonic networks (compound 64-bit keys for TCM),
//       merged across the group's warps through shared memory;
//   a4  admits by warp-shuffle prefix scans of KV needs against free KV and of chunk tokens
//       against the budget (R5-R8); if the scan has not terminated after 32 candidates it
//       re-streams for the next 32 (threshold = last selected); partials ranked below a KV
//       block keep their chunks (R6);
//   a5  advances the clock, stamps first tokens and runs the decode calendar (same integer
//       arithmetic as the fused engine), with the decode-only fast-forward (Lemma L3).
// NEXT-1 (TCM_KV_GROWTH, R28-R32): sw_preempt before a4, re-admissions in a4, token accounting
// in a5.  The order never relies on Lemma L1 (class-FIFO order), so any per-request key fits
// this path; the FP32 filter uses only K1's monotonicity.
#include <cooperative_groups.h>
#include <cstdlib>
#include <mutex>

#include "tcm_k1.cuh"
#include "tcm_stepwise.cuh"

namespace tcm {

namespace {

constexpr int kThreads = 256;
constexpr int kWarpsPerBlock = kThreads / 32;
constexpr int kTop = 32;
constexpr int kItersPerLaunch = 16;   // engine iterations per replica per k_step launch (tcm_run)
constexpr int kMaxPart = 32;
constexpr uint32_t ST_PARTIAL_OVERFLOW = 4;

// request-state byte
constexpr uint8_t RS_CLS = 3, RS_PEND = 4, RS_RES = 8, RS_FT = 16;
// TCM_KV_GROWTH (NEXT-1): decoding, admitted before (a re-admission re-prefills what it held),
// first token emitted
constexpr uint8_t RS_DEC = 32, RS_PREV = 64, RS_GEN = 128;

// stream staging: per warp, kStages chunks of 128 requests (1 KB arrivals + 128 B states)
#ifndef TCM_SW_STAGES
#define TCM_SW_STAGES 4
#endif
#ifndef TCM_SW_SAT
#define TCM_SW_SAT 1
#endif
#ifndef TCM_SW_MINB
#define TCM_SW_MINB 3
#endif
#ifndef TCM_SW_GRMINB
#define TCM_SW_GRMINB 2      // NEXT-1 instantiations: 2 blocks / SM, 128 registers, no spills
#endif
constexpr int kStages = TCM_SW_STAGES;
constexpr size_t kRingBytes = (size_t)kWarpsPerBlock * kStages * (128 * 8 + 32 * 4);

// Development instrumentation (build variant -DTCM_VAR_SWSTATS=1 only): per-launch event counts
// of k_step's warp-per-replica path, read by tools/probe_swstats.py through tcm_dev_swstats.
#ifdef TCM_VAR_SWSTATS
__device__ unsigned long long g_swstats[16];
#define SWSTAT(k, v) do { if (lane == 0) atomicAdd(&g_swstats[k], (unsigned long long)(v)); } while (0)
#else
#define SWSTAT(k, v) do { } while (0)
#endif

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(gmem), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ bool before(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}

// Bitonic sort of one (key, id) per lane, descending across lanes 0..31.
__device__ __forceinline__ void warp_sort_desc_il(uint64_t& k, uint32_t& i, int lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            const uint64_t pk = __shfl_xor_sync(0xFFFFFFFFu, k, j);
            const uint32_t pi = __shfl_xor_sync(0xFFFFFFFFu, i, j);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool lower = (lane & j) == 0;
            // (key, id) pairs are distinct except the empty (0, NIL), and swapping equal pairs is
            // harmless, so before(k, i, pk, pi) == !before(pk, pi, k, i) here
            if (before(pk, pi, k, i) == (lower == desc)) {
                k = pk;
                i = pi;
            }
        }
    }
}

// Merge a descending batch into a descending list, keeping the top 32: element-wise max with
// the reversed batch gives a bitonic sequence holding the top 32; clean it.
__device__ __forceinline__ void warp_merge_il(uint64_t& lk, uint32_t& li, uint64_t bk, uint32_t bi, int lane) {
    const uint64_t rk = __shfl_sync(0xFFFFFFFFu, bk, 31 - lane);
    const uint32_t ri = __shfl_sync(0xFFFFFFFFu, bi, 31 - lane);
    if (before(rk, ri, lk, li)) {
        lk = rk;
        li = ri;
    }
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint64_t pk = __shfl_xor_sync(0xFFFFFFFFu, lk, j);
        const uint32_t pi = __shfl_xor_sync(0xFFFFFFFFu, li, j);
        const bool lower = (lane & j) == 0;
        if (before(pk, pi, lk, li) == lower) {
            lk = pk;
            li = pi;
        }
    }
}

// Out-of-line copies of the generic (key, id) networks: they sit off the TCM hot path (compound
// keys), so one copy each keeps k_step small for the instruction cache.  Values in and out.
struct KeyId {
    uint64_t k;
    uint32_t i;
};
__device__ __noinline__ KeyId warp_sort_desc_ool(uint64_t k, uint32_t i, int lane) {
    warp_sort_desc_il(k, i, lane);
    return KeyId{k, i};
}
__device__ __noinline__ KeyId warp_merge_ool(uint64_t lk, uint32_t li, uint64_t bk, uint32_t bi, int lane) {
    warp_merge_il(lk, li, bk, bi, lane);
    return KeyId{lk, li};
}
__device__ __forceinline__ void warp_sort_desc(uint64_t& k, uint32_t& i, int lane) {
    const KeyId r = warp_sort_desc_ool(k, i, lane);
    k = r.k;
    i = r.i;
}
__device__ __forceinline__ void warp_merge(uint64_t& lk, uint32_t& li, uint64_t bk, uint32_t bi, int lane) {
    const KeyId r = warp_merge_ool(lk, li, bk, bi, lane);
    lk = r.k;
    li = r.i;
}

// Compound-key variants for TCM keys (bit patterns of P in [1e-12, 2^17), so key - kKeyBase < 2^58):
// the tie-break rank rides in the low bits, one 64-bit compare per stage and no id shuffles.
constexpr uint64_t kKeyBase = 0x3D00000000000000ull;   // bits of 2^-47 < 1e-12

__device__ __forceinline__ void warp_sort_desc_u64(uint64_t& c, int lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            const uint64_t pc = __shfl_xor_sync(0xFFFFFFFFu, c, j);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool lower = (lane & j) == 0;
            if ((pc > c) == (lower == desc)) c = pc;
        }
    }
}

__device__ __forceinline__ void warp_merge_u64(uint64_t& l, uint64_t b, int lane) {
    const uint64_t r = __shfl_sync(0xFFFFFFFFu, b, 31 - lane);
    if (r > l) l = r;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const uint64_t p = __shfl_xor_sync(0xFFFFFFFFu, l, j);
        const bool lower = (lane & j) == 0;
        if ((p > l) == lower) l = p;
    }
}

__device__ __forceinline__ uint64_t warp_incl_scan64(uint64_t v, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, v, o);
        if (lane >= o) v += y;
    }
    return v;
}

__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

struct Cal {
    uint32_t* cal;
    uint32_t* occ;
};

// kvrel: KV released at the finish (footprint; TCM_KV_GROWTH: the final holding, and rs clears RS_DEC)
__device__ __forceinline__ void cal_process(const Cal& c, uint32_t* link, uint64_t iter, uint64_t clock,
                                            const uint32_t* kvrel, uint64_t* done, ReplicaState& st,
                                            uint8_t* rs = nullptr) {
    const uint32_t s = (uint32_t)(iter & (kCalSlots - 1));
    const uint32_t bit = 1u << (s & 31);
    const uint32_t w = c.occ[s >> 5];
    if (!(w & bit)) return;
    uint32_t i = c.cal[s];
    while (i != NIL) {
        const uint32_t ni = link[i];
        done[i] = clock;
        st.kv_free += kvrel[i];
        if (rs) rs[i] = (uint8_t)(rs[i] & ~RS_DEC);
        st.n_dec--;
        st.done_count++;
        i = ni;
    }
    c.cal[s] = NIL;
    c.occ[s >> 5] = w & ~bit;
}

__device__ __forceinline__ uint64_t cal_next(const Cal& c, uint64_t iter) {
    const uint32_t s0 = (uint32_t)((iter + 1) & (kCalSlots - 1));
    uint32_t wi = s0 >> 5;
    uint32_t w = c.occ[wi] & (~0u << (s0 & 31));
    uint32_t dist = 0u - (s0 & 31);
    while (w == 0) {
        wi = (wi + 1) & (kCalWords - 1);
        dist += 32;
        w = c.occ[wi];
    }
    return iter + 1 + (uint64_t)(dist + (uint32_t)(__ffs(w) - 1));
}

// Per-group shared state.
template <int G>
struct GroupSmem {
    static constexpr int kMaxDone = G == 1 ? 128 : 1024;
    uint64_t wkey[G][kTop];
    uint32_t wid[G][kTop];
    uint64_t partkey[kMaxPart];
    uint32_t part[kMaxPart];
    uint32_t done[kMaxDone];
    // per-warp refine queue: elements whose FP32 bound cannot rule them out of the top-32
#ifndef TCM_SW_KQ
#define TCM_SW_KQ 160
#endif
    static constexpr int kQ = TCM_SW_KQ;
    uint32_t qid[G][kQ];
    uint64_t qw[G][kQ];
    uint8_t qc[G][kQ];
    int qn[G];
    ReplicaState st;
    ClassPack kp;       // per-replica K1 class constants (precomputed at load)
    uint64_t thk;       // continuation threshold: exclude ranks <= (thk, thi)
    uint64_t left, tok, inl;
    uint32_t thi;
    int npart, ndone, mode, pass_more, blocked, has_th;
    int inv_any, inv_dec;   // NEXT-3 EDF inversion (R34): preempted this iteration; decoding victims among them
};

template <int G>
__device__ __forceinline__ void group_sync() {
    if (G == 1) __syncwarp();
    else __syncthreads();
}

// CL > 1: a thread-block cluster of CL CTAs runs one replica (few huge queues); the group's state
// lives in rank 0's shared memory and the other CTAs reach it through distributed shared memory.
template <int G, int CL>
__device__ __forceinline__ void gsync() {
    if constexpr (CL > 1) cooperative_groups::this_cluster().sync();
    else group_sync<G>();
}

// Prologue (warp 0 of the group): ingest, idle jumps, decode-only fast-forward.
// mode: 0 = nothing more this launch, 1 = decision iteration.
// budget != 0: the call's first launch sets the call's iteration budget (head[1]).
template <int G, bool GR, bool TO>
__device__ void sw_prologue(const ModelConst& m, const TraceDev& t, uint32_t r, GroupSmem<G>& sm, int lane,
                            uint32_t budget) {
    ReplicaState st = t.state[r];
    if (budget) st.head[1] = budget;
    const uint64_t base = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - base);
    const uint64_t* arr = t.arrival + base;
    const uint32_t* fp = t.footprint + base;
    const uint8_t* mod = t.mod + base;
    uint8_t* rs = t.req_state + base;
    const bool prio = TO || t.params[r].policy == TCM_POLICY_TCM;
    const bool edf = !TO && t.params[r].policy == TCM_POLICY_EDF;
    const bool growth = GR && (t.params[r].flags & TCM_KV_GROWTH) != 0;
    int mode = 0;
    if (!(st.flags & FLAG_FINISHED) && st.head[1] > 0) {
        const Cal cal{t.cal + (size_t)r * kCalSlots, t.occ + (size_t)r * kCalWords};
        for (;;) {
            // a1: ingest -- 128 sorted arrivals per round, all four loads in flight together
            for (;;) {
                uint32_t cnt = 0;
                bool in[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t i = st.nxt + 32 * j + lane;
                    in[j] = i < n && arr[i] <= st.clock;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t i = st.nxt + 32 * j + lane;
                    if (in[j]) {
                        const int c = prio ? classify(m, mod[i], fp[i]) : 0;
                        rs[i] = (uint8_t)(c | RS_PEND);
                        if (edf) {   // EDF key input: deadline x den = arrival*den + num*iso_e2e
                            const uint64_t f = fp[i], B = t.params[r].chunk_budget;
                            const uint64_t iso = (uint64_t)t.inl[base + i] + (f + B - 1) / B * m.c0 + m.cp * f +
                                                 (uint64_t)(t.out[base + i] - 1) * (m.c0 + m.cd);
                            t.deadline[base + i] = arr[i] * m.slo_den + m.slo_num * iso;
                        }
                    }
                    cnt += __popc(__ballot_sync(0xFFFFFFFFu, in[j]));
                }
                st.nxt += cnt;
                st.n_pend += cnt;
                if (cnt < 128) break;
            }
            if (st.n_pend > 0) {
                mode = 1;
                break;
            }
            if (st.n_dec == 0) {
                if (st.nxt == n) {
                    st.flags |= FLAG_FINISHED;
                    break;
                }
                st.clock = arr[st.nxt];                  // R15 idle jump
                st.idle_jumps++;
                continue;
            }
            if (growth && st.kv_free < st.n_dec) {       // R29: a preemption is due now
                mode = 1;
                break;
            }
            if (lane == 0) {                             // Lemma L3 decode-only fast-forward
                const uint64_t F = cal_next(cal, st.iter);
                const uint64_t dt = m.c0 + m.cd * st.n_dec;
                uint64_t j = F - st.iter;
                if (st.nxt < n) {
                    const uint64_t ja = (arr[st.nxt] - st.clock + dt - 1) / dt;
                    j = ja < j ? ja : j;
                }
                j = j < st.head[1] ? j : st.head[1];
                if (growth) {                            // R28: every iteration grows n_dec tokens
                    const uint64_t jk = st.kv_free / st.n_dec;
                    j = j < jk ? j : jk;
                    st.kv_free -= j * st.n_dec;
                }
                st.clock += j * dt;
                st.iter += j;
                st.ff_iters += j;
                st.head[1] -= (uint32_t)j;
                if (st.iter == F)
                    cal_process(cal, t.link + base, st.iter, st.clock, growth ? t.kvfin + base : fp, t.done + base, st,
                                growth ? rs : nullptr);
            }
            break;
        }
    }
    if (lane == 0) {
        sm.st = st;
        sm.mode = mode;
    }
}

// NEXT-1 (TCM_KV_GROWTH, readings R28-R32): before the order/admission of an iteration, while the
// free KV cannot cover one decode token per decoding sequence, preempt the running request that
// comes last (FCFS / EDF / naive aging: latest (arrival, id) = largest id; TCM: the
// lowest (key, then largest id) among non-motorcycles, motorcycles only when nothing else runs,
// SPEC.md:402).  The victim frees what it holds and waits again with rem = held (recomputation,
// SPEC.md:87); then this iteration's decode tokens take their KV.  Warp-collective
// on the group's first warp; st lives in shared memory.
__device__ __noinline__ void sw_preempt(const ModelConst& m, const TraceDev& t, uint32_t r, uint64_t base, uint8_t* rs,
                                        uint32_t* rem, bool prio, const K1Tables& tb, const ClassPack& kp,
                                        ReplicaState& st, int lane) {
    const uint32_t hi = st.nxt;
    const uint64_t clock = st.clock;
    const uint64_t* arr = t.arrival + base;
    while (st.kv_free < st.n_dec) {
        uint32_t v = NIL;
        bool forced = false;
        if (!prio) {
            for (int64_t top = (int64_t)hi - 1; top >= 0 && v == NIL; top -= 32) {
                const int64_t i = top - lane;
                const bool run = i >= 0 && (rs[i] & (RS_RES | RS_DEC));
                const uint32_t b = __ballot_sync(0xFFFFFFFFu, run);
                if (b) v = (uint32_t)(top - (__ffs(b) - 1));
            }
        } else {
            // advance the running-set lower bound past served requests
            uint32_t lo = st.tail[0];
            for (;;) {
                const uint32_t i = lo + lane;
                const bool stop = i >= hi || (rs[i] & (RS_PEND | RS_RES | RS_DEC));
                const uint32_t b = __ballot_sync(0xFFFFFFFFu, stop);
                if (b) {
                    lo += __ffs(b) - 1;
                    break;
                }
                lo += 32;
            }
            lo = lo < hi ? lo : hi;
            if (lane == 0) st.tail[0] = lo;
            for (int pass = 0; pass < 2 && v == NIL; ++pass) {
                uint64_t bk = ~0ull;
                uint32_t bi = NIL;
                for (uint32_t c0 = lo; c0 < hi; c0 += 32) {
                    const uint32_t i = c0 + lane;
                    const uint8_t sb = i < hi ? rs[i] : 0;
                    const int c = sb & RS_CLS;
                    if ((sb & (RS_RES | RS_DEC)) && (pass == 1 || c != 0)) {
                        const uint64_t k = k1_key_bf(kp.S[c], kp.p[c], kp.C[c], (kp.zero_mask >> c) & 1u, clock - arr[i], tb);
                        if (k < bk || (k == bk && (bi == NIL || i > bi))) {
                            bk = k;
                            bi = i;
                        }
                    }
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {           // warp arg-min (key asc, id desc)
                    const uint64_t ok = __shfl_xor_sync(0xFFFFFFFFu, bk, o);
                    const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
                    if (oi != NIL && (bi == NIL || ok < bk || (ok == bk && oi > bi))) {
                        bk = ok;
                        bi = oi;
                    }
                }
                v = bi;
                forced = pass == 1;
            }
        }
        if (lane == 0 && v != NIL) {
            const uint8_t sb = rs[v];
            uint32_t held;
            if (sb & RS_DEC) {
                const uint64_t F = t.fin[base + v];
                const uint32_t togo = (uint32_t)(F - st.iter);
                held = t.kvfin[base + v] - togo;
                t.genp[base + v] = (uint32_t)t.out[base + v] - togo;
                // unlink from its calendar slot
                const uint32_t slot = (uint32_t)(F & (kCalSlots - 1));
                uint32_t* cal = t.cal + (size_t)r * kCalSlots;
                uint32_t* link = t.link + base;
                uint32_t prv = NIL, cur = cal[slot];
                while (cur != v) {
                    prv = cur;
                    cur = link[cur];
                }
                if (prv == NIL) cal[slot] = link[v];
                else link[prv] = link[v];
                if (cal[slot] == NIL) t.occ[(size_t)r * kCalWords + (slot >> 5)] &= ~(1u << (slot & 31));
                st.n_dec--;
                st.n_pend++;
                rs[v] = (uint8_t)((sb & ~RS_DEC) | RS_PEND);
            } else {                                         // a partial prefill
                held = t.kvres[base + v];
                rs[v] = (uint8_t)(sb & ~RS_RES);
            }
            rem[v] = held;
            st.kv_free += held;
            t.pcount[base + v]++;
            t.pstart[base + v] = clock;
            st.tail[1]++;
            if (forced) st.tail[2]++;
            if (v < st.head[0]) st.head[0] = v;
        }
        __syncwarp();
        if (v == NIL) break;                                 // unreachable: n_dec > 0
    }
    if (lane == 0) st.kv_free -= st.n_dec;                   // this iteration's decode tokens
    __syncwarp();
}

// NEXT-3 EDF priority inversion under TCM_KV_GROWTH (reading R34):
// over the current batch of candidates (lane = rank in EDF order, li = id), the first waiting
// request m that does not fit (and is reached by the budget, admissions not yet blocked) preempts
// running requests that come after it in EDF order (deadline x den, id), latest first, until the
// admissions up to m fit -- if preempting all of them would.  Repeats for the next misfit.  A
// victim frees what it holds (a decoding one including this iteration's token: it does not decode
// now), is recomputed later (R30) and is excluded for the rest of this iteration (RS_FT on a request
// without RS_RES; a5 clears it).  Warp-collective on the group's first warp; returns the new kv_free.
__device__ __noinline__ uint64_t sw_edf_invert(const TraceDev& t, uint32_t r, uint64_t base, uint8_t* rs,
                                               uint32_t* rem, uint32_t li, bool valid, bool blocked_prev,
                                               uint64_t left, uint64_t kv, uint32_t hi, ReplicaState& st,
                                               int& inv_any, int& inv_dec, int lane) {
    const uint64_t* dl = t.deadline + base;
    const uint32_t* fp = t.footprint + base;
    for (;;) {
        const uint8_t sb = valid ? rs[li] : 0;
        const bool v = valid && !((sb & RS_FT) && !(sb & RS_RES));
        const bool res = v && (sb & RS_RES);
        const bool prev = v && (sb & RS_PREV);
        const uint32_t rr = v ? ((res || prev) ? rem[li] : fp[li]) : 0;
        const uint32_t f = prev ? rr : (v ? fp[li] : 0);
        const bool waiting = v && !res;
        const uint64_t cumf = warp_incl_scan64(waiting ? f : 0, lane);
        const bool kv_ok = waiting && !blocked_prev && cumf <= kv;
        const bool part = v && (res || kv_ok);
        const uint64_t incl = warp_incl_scan64(part ? rr : 0, lane);
        const bool misfit = waiting && !blocked_prev && !kv_ok && incl - (part ? rr : 0) < left;
        const uint32_t mm = __ballot_sync(0xFFFFFFFFu, misfit);
        if (!mm) return kv;
        const int ml = __ffs(mm) - 1;
        const uint64_t need = __shfl_sync(0xFFFFFFFFu, cumf, ml) - kv;
        const uint32_t im = __shfl_sync(0xFFFFFFFFu, li, ml);
        const uint64_t dm = dl[im];
        // running requests after (dm, im): decoding (holding incl. this iteration's token) or partial
        auto holding = [&](uint32_t i, uint8_t s) -> uint64_t {
            return (s & RS_DEC) ? (uint64_t)t.kvfin[base + i] - (t.fin[base + i] - st.iter) + 1 : t.kvres[base + i];
        };
        uint64_t avail = 0;
        for (uint32_t c0 = 0; c0 < hi; c0 += 32) {
            const uint32_t i = c0 + lane;
            const uint8_t s = i < hi ? rs[i] : 0;
            if ((s & (RS_RES | RS_DEC)) && (dl[i] > dm || (dl[i] == dm && i > im))) avail += holding(i, s);
        }
        avail = warp_sum64(avail);
        if (avail < need) return kv;                           // m blocks (R6)
        uint64_t got = 0;
        while (got < need) {
            uint64_t bd = 0;
            uint32_t bi = NIL;
            for (uint32_t c0 = 0; c0 < hi; c0 += 32) {         // the latest in EDF order
                const uint32_t i = c0 + lane;
                const uint8_t s = i < hi ? rs[i] : 0;
                if ((s & (RS_RES | RS_DEC)) && (dl[i] > dm || (dl[i] == dm && i > im)) &&
                    (bi == NIL || dl[i] > bd || (dl[i] == bd && i > bi))) {
                    bd = dl[i];
                    bi = i;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const uint64_t od = __shfl_xor_sync(0xFFFFFFFFu, bd, o);
                const uint32_t oi = __shfl_xor_sync(0xFFFFFFFFu, bi, o);
                if (oi != NIL && (bi == NIL || od > bd || (od == bd && oi > bi))) {
                    bd = od;
                    bi = oi;
                }
            }
            uint64_t freed = 0;
            if (lane == 0) {
                const uint32_t vv = bi;
                const uint8_t s = rs[vv];
                freed = holding(vv, s);
                if (s & RS_DEC) {
                    const uint64_t F = t.fin[base + vv];
                    const uint32_t togo = (uint32_t)(F - st.iter);
                    rem[vv] = t.kvfin[base + vv] - togo;         // what it held before this iteration
                    t.genp[base + vv] = (uint32_t)t.out[base + vv] - togo;
                    const uint32_t slot = (uint32_t)(F & (kCalSlots - 1));
                    uint32_t* cal = t.cal + (size_t)r * kCalSlots;
                    uint32_t* link = t.link + base;
                    uint32_t prv = NIL, cur = cal[slot];
                    while (cur != vv) {
                        prv = cur;
                        cur = link[cur];
                    }
                    if (prv == NIL) cal[slot] = link[vv];
                    else link[prv] = link[vv];
                    if (cal[slot] == NIL) t.occ[(size_t)r * kCalWords + (slot >> 5)] &= ~(1u << (slot & 31));
                    st.n_dec--;
                    st.n_pend++;
                    inv_dec++;
                    rs[vv] = (uint8_t)((s & ~RS_DEC) | RS_PEND | RS_FT);
                } else {
                    rem[vv] = t.kvres[base + vv];
                    rs[vv] = (uint8_t)((s & ~RS_RES) | RS_FT);
                }
                t.pcount[base + vv]++;
                t.pstart[base + vv] = st.clock;
                st.tail[1]++;
                if (vv < st.head[0]) st.head[0] = vv;
                inv_any = 1;
            }
            __syncwarp();
            got += __shfl_sync(0xFFFFFFFFu, freed, 0);
        }
        kv += got;
    }
}

}  // namespace

// GR: some replica of the trace runs TCM_KV_GROWTH (NEXT-1); the plain instantiation compiles
// the growth code out of the hot path.
// TO: every replica runs plain TCM (TraceDev.all_tcm): the FCFS / EDF / first-fit paths compile out
// (a smaller kernel for the instruction cache).
template <int G, bool GR, int CL, bool TO = false>
__global__ void __launch_bounds__(kThreads, CL > 1 ? 1 : (GR ? TCM_SW_GRMINB : TCM_SW_MINB)) k_step(ModelConst m, TraceDev t, uint32_t* remv,
                                                                             StepCtl ctl) {
    constexpr int kGroups = kWarpsPerBlock / G;
    constexpr int kMaxDone = GroupSmem<G>::kMaxDone;
    __shared__ double s_lnR[16], s_lnT[16], s_expT[16];
    __shared__ GroupSmem<G> smg[kGroups];
    extern __shared__ __align__(16) uint8_t dsm[];
    uint64_t* ring_a = reinterpret_cast<uint64_t*>(dsm);
    uint32_t* ring_s = reinterpret_cast<uint32_t*>(dsm + (size_t)kWarpsPerBlock * kStages * 128 * 8);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int group = warp / G, wl = warp % G;       // warp index inside this CTA's group
    uint32_t crank = 0;
    if constexpr (CL > 1) crank = cooperative_groups::this_cluster().block_rank();
    const int wg = (int)crank * G + wl;               // warp index inside the replica's group (all CTAs)
    GroupSmem<G>& sm = smg[group];                    // this CTA: class pack, per-warp queues and lists
    GroupSmem<G>& gsm = [&]() -> GroupSmem<G>& {      // the group's state (rank 0 of a cluster)
        if constexpr (CL > 1) return *cooperative_groups::this_cluster().map_shared_rank(&smg[0], 0);
        else return smg[group];
    }();
    __shared__ uint32_t s_active;                     // this CTA's active replicas (counting launches)
    if (tid == 0) s_active = 0;
    if (tid < 16) {
        s_lnR[tid] = kLnR[tid];
        s_lnT[tid] = kLnT[tid];
        s_expT[tid] = kExpT[tid];
    }
    __syncthreads();
    const K1Tables tb{s_lnR, s_lnT, s_expT};

    const uint32_t r0 = CL > 1 ? blockIdx.x / CL : blockIdx.x * kGroups + group;
    const uint32_t rstep = CL > 1 ? gridDim.x / CL : gridDim.x * kGroups;
    // A warp per replica takes replicas from a global counter (dynamic balance; the launch's last
    // CTA resets it, see the end of the kernel); CTA and cluster groups use a static stride.
    const bool kDyn = G == 1 && CL == 1 && ctl.dyn;          // host clears dyn when R <= warps
    auto grab = [&]() -> uint32_t {
        unsigned long long v = 0;
        if (lane == 0) v = atomicAdd(&ctl.w->ctr, 1ull);
        v = __shfl_sync(0xFFFFFFFFu, v, 0);
        return v < t.R ? (uint32_t)v : t.R;
    };
    for (uint32_t r = kDyn ? grab() : r0; r < t.R; r = kDyn ? grab() : r + rstep) {
      // up to kItersPerLaunch engine iterations of this replica per launch (each one the full
      // a1-a5 step); tcm_step's budget (head[1]) still bounds the total
      for (int kit = 0; kit < kItersPerLaunch; ++kit) {
        // the replica's class pack, parameters and offset do not depend on its state: load them
        // before the prologue so their latency overlaps the state load
        if (wl == 0 && kit == 0) {   // stage the replica's ClassPack (192 B) in this CTA's shared memory
            static_assert(sizeof(ClassPack) % 16 == 0 && sizeof(ClassPack) / 16 <= 32, "one 16-byte load per lane");
            if (lane < (int)(sizeof(ClassPack) / 16))
                reinterpret_cast<uint4*>(&sm.kp)[lane] = __ldg(reinterpret_cast<const uint4*>(t.kpack + r) + lane);
        }
        const tcm_replica_params prm = t.params[r];
        const uint64_t base = t.offset[r];
        if (wg == 0) sw_prologue<G, GR, TO>(m, t, r, gsm, lane, kit == 0 ? ctl.budget : 0u);
        gsync<G, CL>();
        if (gsm.mode == 0) {
            if (wg == 0 && lane == 0) t.state[r] = gsm.st;
            gsync<G, CL>();
            break;
        }

        const bool prio = TO || prm.policy == TCM_POLICY_TCM;
        const bool edf = !TO && prm.policy == TCM_POLICY_EDF;
        const bool skip = !TO && (prm.flags & TCM_ADMIT_SKIP) != 0;
        // the streamed 8-byte key input: arrival (TCM aging, FCFS) or the EDF deadline x den
        const uint64_t* arr = (edf ? t.deadline : t.arrival) + base;
        const uint32_t* fp = t.footprint + base;
        const uint32_t* inl = t.inl + base;
        const uint8_t* rsc = t.req_state + base;
        uint8_t* rs = t.req_state + base;
        uint32_t* rem = remv + base;
        const uint64_t clock = gsm.st.clock;
        const bool growth = GR && (prm.flags & TCM_KV_GROWTH) != 0;
        if (wg == 0) {
            if (growth) sw_preempt(m, t, r, base, rs, rem, prio, tb, sm.kp, gsm.st, lane);
            if (lane == 0) {
                const uint32_t B = prm.chunk_budget;
                gsm.left = B > gsm.st.n_dec ? B - gsm.st.n_dec : 0;     // R8
                gsm.tok = 0;
                gsm.inl = 0;
                gsm.blocked = 0;
                gsm.has_th = 0;
                gsm.npart = 0;
                gsm.ndone = 0;
                gsm.inv_any = 0;
                gsm.inv_dec = 0;
            }
        }
        gsync<G, CL>();
        const uint32_t lo = gsm.st.head[0], hi = gsm.st.nxt;     // after any preemption (NEXT-1)
        const bool filter_ok = sm.kp.filter_ok != 0;
        // compound sort keys need every key in [1e-12, 2^17): P <= Smax_c
        const bool cmp_ok = prio && sm.kp.Smax[0] < 65536.0 && sm.kp.Smax[1] < 65536.0 && sm.kp.Smax[2] < 65536.0;
        const uint32_t zero_mask = sm.kp.zero_mask;

        SWSTAT(0, 1);
        for (int pass = 0;; ++pass) {
            SWSTAT(1, 1);
            const bool first_pass = pass == 0;
            const bool has_th = gsm.has_th;
            const uint64_t thk = gsm.thk;
            const uint32_t thi = gsm.thi;
            const double Pth = __longlong_as_double((long long)thk);
            // ---- a2 + a3: stream the window; every pending request gets an FP32 bound on its
            // priority; those that could still enter this warp's exact top-32 (or hold KV as a
            // partial) are queued for the exact K1 key.  The selected set equals the top-32 of
            // exact keys: a request is skipped only when max(P~ + delta, ...) proves it ranks
            // after the current 32nd, using S_c <= P <= S_c + 1 exactly.
            uint64_t lk = 0, kk = 0;
            uint32_t li = NIL, ki = NIL;
            // threshold state derived from the warp's current 32nd (kk, ki).  Lean path: per
            // class c an arrival limit amax[c] such that every class-c request arriving after it
            // provably ranks after (kk, ki); a request is queued for its exact key only if
            // arrival <= amax[c].  Derivation: K1 is non-decreasing in w (Lemma L1's
            // premise, audited on [0, 2^33) us), so for w <= W-1, P(w) <= P(W-1) <= P~(W-1) + 1e-5;
            // one FP32 bound evaluation at W-1 with fadd_ru(P~, 1e-4) < rd(P(kk)) proves it for the
            // whole class.  Classes whose exact cap is below (or ties) P(kk) are excluded outright
            // (a tie loses on id: every chunk this warp streams after (kk, ki) entered its list holds
            // larger ids than every list entry, ki < e).
            const bool lean = prio && filter_ok && !has_th;    // FP32-bound path (else: exact for all)
            const bool lean_path = lean;
            uint32_t skipm = 0, tiem = 0;
            int64_t am0 = INT64_MAX, am1 = INT64_MAX, am2 = INT64_MAX, amx = INT64_MAX;   // amx = max_c am_c
            auto retune = [&]() {
                SWSTAT(10, 1);
                const double Pkk = __longlong_as_double((long long)kk);
                const float thrf = __double2float_rd(Pkk);
                skipm = 0;
                tiem = 0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const double cap = sm.kp.Smax[c] < kEps ? kEps : sm.kp.Smax[c];
                    if (cap < Pkk) skipm |= 1u << c;
                    else if (cap == Pkk) tiem |= 1u << c;
                }
                if (!lean_path) return;
                int64_t am = INT64_MAX;
                const int c = lane;
                if (c < 3) {
                    if ((skipm | tiem) >> c & 1u) {
                        am = -1;
                    } else if (!((zero_mask >> c) & 1u)) {
                        const float fS = sm.kp.fS[c], p2 = sm.kp.fp2[c], C2 = sm.kp.fC2[c];
                        const float d = thrf - fS - 3e-4f;
                        uint64_t W = 0;
                        if (d > 0.0f && d < 1.0f) {
                            // estimate: P~(w) = S + 1 - e^-x, x = 2^(p2 log2 w + C2)
                            const float x = -sfu_lg2(1.0f - d) * 0.693147182f;
                            const float L = (sfu_lg2(x) - C2) / p2;
                            W = L >= 62.0f ? (1ull << 62) : (L <= 1.0f ? 0ull : __float2ull_rd(sfu_ex2(L)));
                            for (int tr = 0; tr < 3 && W >= 2; ++tr) {
                                const float pf = k1_filter_f32(fS, p2, C2, W - 1);
                                if (__fadd_ru(pf, 1e-4f) < thrf) break;
                                W = tr < 2 ? W - (W >> 3) : 0;
                            }
                            if (W < 2) W = 0;
                        }
                        am = W > clock ? -1 : (int64_t)(clock - W);
                    }
                }
                am0 = __shfl_sync(0xFFFFFFFFu, am, 0);
                am1 = __shfl_sync(0xFFFFFFFFu, am, 1);
                am2 = __shfl_sync(0xFFFFFFFFu, am, 2);
                amx = am0 > am1 ? am0 : am1;
                amx = amx > am2 ? amx : am2;
            };
            int qn = 0, qh = 0;                      // refine queue: count and ring head
            constexpr int kQ = GroupSmem<G>::kQ;
            uint32_t* qid = sm.qid[wl];
            uint64_t* qw = sm.qw[wl];
            uint8_t* qc = sm.qc[wl];
            auto take = [&](uint64_t key, uint32_t id, bool enter) {   // warp-collective
                const uint32_t em = __ballot_sync(0xFFFFFFFFu, enter);
                SWSTAT(7, 1);
                if (em == 0) return;
                SWSTAT(8, __popc(em) <= 16);
                SWSTAT(9, __popc(em));
                if (__popc(em) <= 16) {
                    // up to 16 entrants: insert each into the sorted list (rank by ballot, shift by shuffle)
                    uint32_t rest = em;
                    while (rest) {
                        const int src = __ffs(rest) - 1;
                        rest &= rest - 1;
                        const uint64_t xk = __shfl_sync(0xFFFFFFFFu, key, src);
                        const uint32_t xi = __shfl_sync(0xFFFFFFFFu, id, src);
                        if (!before(xk, xi, kk, ki)) continue;          // pushed out by an earlier insert
                        const int pos = __popc(__ballot_sync(0xFFFFFFFFu, before(lk, li, xk, xi)));
                        const uint64_t uk = __shfl_up_sync(0xFFFFFFFFu, lk, 1);
                        const uint32_t ui = __shfl_up_sync(0xFFFFFFFFu, li, 1);
                        if (lane > pos) {
                            lk = uk;
                            li = ui;
                        } else if (lane == pos) {
                            lk = xk;
                            li = xi;
                        }
                        kk = __shfl_sync(0xFFFFFFFFu, lk, 31);
                        ki = __shfl_sync(0xFFFFFFFFu, li, 31);
                    }
                } else if (cmp_ok) {
                    // TCM keys: compound sort.  Batch lanes are in id order (the refine queue is
                    // id-ordered), and every list entry precedes every batch entry in id, so the
                    // rank bits (31 - lane; list above batch) encode the (key desc, id asc) tie-break.
                    uint64_t c = enter ? (((key - kKeyBase) << 5) | (uint64_t)(31 - lane)) : 0;
                    warp_sort_desc_u64(c, lane);
                    const uint32_t sid = __shfl_sync(0xFFFFFFFFu, id, 31 - (int)(c & 31));
                    const uint64_t bk = c ? (c >> 5) + kKeyBase : 0;
                    const uint32_t bi = c ? sid : NIL;
                    if (__all_sync(0xFFFFFFFFu, li == NIL)) {
                        lk = bk;
                        li = bi;
                    } else {
                        uint64_t lc = li != NIL ? (((lk - kKeyBase) << 6) | 32u | (uint64_t)(31 - lane)) : 0;
                        const uint64_t bc = bi != NIL ? (((bk - kKeyBase) << 6) | (uint64_t)(31 - lane)) : 0;
                        warp_merge_u64(lc, bc, lane);
                        const int pos = 31 - (int)(lc & 31);
                        const uint32_t fl = __shfl_sync(0xFFFFFFFFu, li, pos);
                        const uint32_t fb = __shfl_sync(0xFFFFFFFFu, bi, pos);
                        li = lc == 0 ? NIL : ((lc & 32) ? fl : fb);
                        lk = lc == 0 ? 0 : (lc >> 6) + kKeyBase;
                    }
                    kk = __shfl_sync(0xFFFFFFFFu, lk, 31);
                    ki = __shfl_sync(0xFFFFFFFFu, li, 31);
                } else {
                    uint64_t bk = enter ? key : 0;
                    uint32_t bi = enter ? id : NIL;
                    warp_sort_desc(bk, bi, lane);
                    if (__all_sync(0xFFFFFFFFu, li == NIL)) {   // empty list: the batch is the list
                        lk = bk;
                        li = bi;
                    } else {
                        warp_merge(lk, li, bk, bi, lane);
                    }
                    kk = __shfl_sync(0xFFFFFFFFu, lk, 31);
                    ki = __shfl_sync(0xFFFFFFFFu, li, 31);
                }
                retune();
            };
            auto refine = [&](int cnt) {                               // exact keys for <= 32 queued
                uint64_t key = 0;
                uint32_t id = NIL;
                bool enter = false;
                bool live = false;
                int cc = 0;
                uint64_t qwl = 0;
                if (lane < cnt) {
                    int q = qh + lane;                                 // ring slot
                    q -= q >= kQ ? kQ : 0;
                    id = qid[q];
                    cc = qc[q];
                    qwl = qw[q];
                    // the limits may have tightened since this request was queued.  The queue is
                    // not in id order within a chunk, so a tie class is decided by id here.
                    const int qcl = cc & RS_CLS;
                    const int64_t am = qcl == 0 ? am0 : (qcl == 1 ? am1 : am2);
                    live = !lean_path || (first_pass && (cc & RS_RES)) ||
                           (((tiem >> qcl) & 1u) ? id < ki : (int64_t)(clock - qwl) <= am);
                }
                SWSTAT(5, 1);
                if (!__any_sync(0xFFFFFFFFu, live)) return;
                SWSTAT(4, 1);
#ifdef TCM_VAR_SWSTATS
                const uint32_t nlive = __popc(__ballot_sync(0xFFFFFFFFu, live));
                SWSTAT(6, nlive);
#endif
                if (live) {
                    const int c = cc & RS_CLS;
#if TCM_SW_SAT
                    // a wait past the class's saturation point has the cap's key exactly (ClassPack.wsat)
                    key = prio ? (qwl >= sm.kp.wsat[c] ? sm.kp.satkey[c]
                                                       : k1_key_bf(sm.kp.S[c], sm.kp.p[c], sm.kp.C[c], (zero_mask >> c) & 1u, qwl, tb))
                               : (edf ? ~(clock - qwl) : 0);     // EDF: ~(deadline x den); FCFS / aging: 0
#else
                    key = prio ? k1_key_bf(sm.kp.S[c], sm.kp.p[c], sm.kp.C[c], (zero_mask >> c) & 1u, qwl, tb)
                               : (edf ? ~(clock - qwl) : 0);     // EDF: ~(deadline x den); FCFS / aging: 0
#endif
                    if (first_pass && (cc & RS_RES)) {                 // partial: remember its key
                        const int slot = atomicAdd(&gsm.npart, 1);
                        if (slot < kMaxPart) {
                            gsm.part[slot] = id;
                            gsm.partkey[slot] = key;
                        }
                    }
                    const bool valid = !(has_th && !before(thk, thi, key, id));
                    enter = valid && before(key, id, kk, ki);
                }
                take(key, id, enter);
            };
            const int64_t gstart = (int64_t)((base + lo) & ~3ull) - (int64_t)base;   // 4-aligned globally
            const int64_t stride = (int64_t)G * CL * 128;
            // cp.async ring: kStages chunks of 128 requests per warp in flight; lane l copies and
            // later consumes exactly its own 4 requests (32 B of arrivals + 4 state bytes), so
            // no cross-lane barrier is needed, only cp.async.wait_group.
            uint64_t* ra = ring_a + (size_t)warp * kStages * 128;
            uint32_t* rst = ring_s + (size_t)warp * kStages * 32;
            auto issue = [&](int64_t g, int slot) {
                const int64_t e0 = g + 4 * lane;
                if (g + 128 <= (int64_t)hi) {          // full chunk: no bounds arithmetic
                    cp_async16(ra + slot * 128 + 4 * lane, arr + e0, 16);
                    cp_async16(ra + slot * 128 + 4 * lane + 2, arr + e0 + 2, 16);
                    cp_async4(rst + slot * 32 + lane, rsc + e0, 4);
                } else if (g < (int64_t)hi) {
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int64_t e = e0 + 2 * h;
                        int64_t nb = (int64_t)hi - e;
                        nb = nb < 0 ? 0 : (nb > 2 ? 2 : nb);
                        cp_async16(ra + slot * 128 + 4 * lane + 2 * h, nb ? arr + e : arr, (int)(8 * nb));
                    }
                    int64_t ns = (int64_t)hi - e0;
                    ns = ns < 0 ? 0 : (ns > 4 ? 4 : ns);
                    cp_async4(rst + slot * 32 + lane, ns ? rsc + e0 : rsc, (int)ns);
                }
                cp_async_commit();
            };
            int64_t g0 = gstart + (int64_t)wg * 128;
#pragma unroll
            for (int q = 0; q < kStages - 1; ++q) issue(g0 + q * stride, q);
            for (int kchunk = 0; g0 < (int64_t)hi; g0 += stride, ++kchunk) {
                issue(g0 + (kStages - 1) * stride, (kchunk + kStages - 1) % kStages);
                cp_async_wait<kStages - 1>();
                const int slot = kchunk % kStages;
                const ulonglong2 v0 = *reinterpret_cast<const ulonglong2*>(ra + slot * 128 + 4 * lane);
                const ulonglong2 v1 = *reinterpret_cast<const ulonglong2*>(ra + slot * 128 + 4 * lane + 2);
                const uint64_t a4[4] = {v0.x, v0.y, v1.x, v1.y};
                const uint32_t s4 = rst[slot * 32 + lane];
                const int e0 = (int)(g0 + 4 * lane);
                bool take_chunk = true;
                SWSTAT(2, 1);
                if (lean) {
                    // fast rejection: arrivals after every class's limit, and no partial to record
                    // (arrivals are sorted, so a lane's first element is its smallest)
                    const bool maybe = (first_pass && (s4 & 0x08080808u) != 0) || (int64_t)a4[0] <= amx;
                    take_chunk = __any_sync(0xFFFFFFFFu, maybe);
                }
                if (take_chunk) {
                SWSTAT(3, 1);
                uint32_t qbits = 0;                       // bit j: element j goes to the refine queue
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int e = e0 + j;
                    const uint32_t sb = (s4 >> (8 * j)) & 0xFF;
                    const bool valid = (sb & RS_PEND) && e >= (int)lo && e < (int)hi;
                    const int c = sb & RS_CLS;
                    if (lean) {
                        // queue when the class's arrival limit cannot rule it out (a partial always
                        // gets its exact key on the first pass: R6 may need it)
                        const bool part = first_pass && (sb & RS_RES);
                        const int64_t am = c == 0 ? am0 : (c == 1 ? am1 : am2);
                        const bool need = valid && (part || (int64_t)a4[j] <= am);
                        qbits |= need ? (1u << j) : 0u;
                    } else if (!prio) {
                        // exact keys without K1: FCFS / naive aging (key 0, id order, R4) or EDF
                        // (static key ~(deadline x den): earliest deadline first)
                        // queued like TCM candidates (refine recomputes the key from the queued
                        // value and registers partials); partials always, on the first pass
                        const uint64_t key = edf ? ~a4[j] : 0;
                        const bool need = valid && ((first_pass && (sb & RS_RES)) ||
                                                    (!(has_th && !before(thk, thi, key, (uint32_t)e)) &&
                                                     before(key, (uint32_t)e, kk, ki)));
                        qbits |= need ? (1u << j) : 0u;
                    } else {
                        qbits |= valid ? (1u << j) : 0u;     // exact key for every pending request
                    }
                }
                if (__any_sync(0xFFFFFFFFu, qbits != 0)) {
                    // append in id order (lane-major, then j) so refined batches follow the
                    // stream order: exclusive prefix of the per-lane counts from three ballots
                    const uint32_t nq = __popc(qbits);
                    const uint32_t b0 = __ballot_sync(0xFFFFFFFFu, nq & 1u);
                    const uint32_t b1 = __ballot_sync(0xFFFFFFFFu, nq & 2u);
                    const uint32_t b2 = __ballot_sync(0xFFFFFFFFu, nq & 4u);
                    const uint32_t lt = (1u << lane) - 1u;
                    int pos = qh + qn + __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if ((qbits >> j) & 1u) {
                            const uint32_t sb = (s4 >> (8 * j)) & 0xFF;
                            const int q = pos >= kQ ? pos - kQ : pos;  // ring slot (pos < 2 kQ)
                            qid[q] = (uint32_t)(e0 + j);
                            qw[q] = clock - a4[j];
                            qc[q] = (uint8_t)((sb & RS_CLS) | (sb & RS_RES));
                            ++pos;
                        }
                    }
                    qn += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
                    __syncwarp();
                }
                }   // take_chunk
                // refine full batches; after the last chunk also the remainder.  One call site of
                // refine (and take) keeps the kernel small for the instruction cache.  The queue is
                // a ring: no shifting.
                const bool last = g0 + stride >= (int64_t)hi;
                while (qn >= 32 || (last && qn > 0)) {
                    const int cnt = qn < 32 ? qn : 32;
                    refine(cnt);
                    qh += cnt;
                    qh -= qh >= kQ ? kQ : 0;
                    qn -= cnt;
                    __syncwarp();
                }
            }
            cp_async_wait<0>();
            if (G > 1) {
                sm.wkey[wl][lane] = lk;
                sm.wid[wl][lane] = li;
            }
            gsync<G, CL>();
            if constexpr (CL > 1) {
                // each CTA's warp 0 merges its warps' lists, then rank 0 merges the CTA lists (DSMEM)
                if (wl == 0) {
#pragma unroll 1
                    for (int w = 1; w < G; ++w) warp_merge(lk, li, sm.wkey[w][lane], sm.wid[w][lane], lane);
                    sm.wkey[0][lane] = lk;
                    sm.wid[0][lane] = li;
                }
                gsync<G, CL>();
                if (wg == 0) {
#pragma unroll 1
                    for (int q = 1; q < CL; ++q) {
                        const GroupSmem<G>* rmt = cooperative_groups::this_cluster().map_shared_rank(&smg[0], q);
                        warp_merge(lk, li, rmt->wkey[0][lane], rmt->wid[0][lane], lane);
                    }
                }
            }

            // ---- a4: warp 0 of the group merges the lists and prefix-scans the admission
            if (wg == 0) {
                if (G > 1 && CL == 1) {
#pragma unroll 1
                    for (int w = 1; w < G; ++w) warp_merge(lk, li, sm.wkey[w][lane], sm.wid[w][lane], lane);
                }
                bool valid = li != NIL;
                const uint32_t nvalid = __popc(__ballot_sync(0xFFFFFFFFu, valid));
                SWSTAT(12, nvalid);
                const uint64_t left = gsm.left;
                const bool blocked_prev = gsm.blocked;
                if (GR && growth && edf && !skip) {           // NEXT-3 EDF priority inversion (R34)
                    int ia = 0, idc = 0;
                    const uint64_t kvn = sw_edf_invert(t, r, base, rs, rem, li, valid, blocked_prev, left,
                                                       gsm.st.kv_free, hi, gsm.st, ia, idc, lane);
                    __syncwarp();
                    if (lane == 0) {
                        gsm.st.kv_free = kvn;
                        gsm.inv_any |= ia;
                        gsm.inv_dec += idc;
                    }
                    __syncwarp();
                    if (valid && (rsc[li] & (RS_FT | RS_RES)) == RS_FT) valid = false;   // a victim of this iteration
                }
                const uint64_t kv = gsm.st.kv_free;
                uint32_t f = 0, rr = 0, il = 0;
                bool res = false, prev = false;
                if (valid) {
                    const uint8_t sb = rsc[li];
                    res = (sb & RS_RES) != 0;
                    prev = (sb & RS_PREV) != 0;          // NEXT-1 re-admission (R30)
                    rr = (res || prev) ? rem[li] : fp[li];
                    f = prev ? rr : fp[li];              // KV to reserve
                    il = (res || prev) ? 0 : inl[li];
                }
                const bool waiting = valid && !res;
                bool kv_ok;
                if (!skip) {
                    // R6: admitted waiting requests form the prefix whose footprints fit
                    const uint64_t cumf = warp_incl_scan64(waiting ? f : 0, lane);
                    kv_ok = waiting && !blocked_prev && cumf <= kv;
                } else {
                    // first fit (NEXT-3): each waiting request in order takes KV if it still fits
                    uint64_t kvl = kv;
                    kv_ok = false;
                    for (int l = 0; l < 32; ++l) {
                        const uint32_t fl = __shfl_sync(0xFFFFFFFFu, f, l);
                        const bool wl = __shfl_sync(0xFFFFFFFFu, waiting, l);
                        const bool ok = wl && (uint64_t)fl <= kvl;
                        kvl -= ok ? fl : 0;
                        if (lane == l) kv_ok = ok;
                    }
                }
                const bool part = valid && (res || kv_ok);
                const uint64_t incl = warp_incl_scan64(part ? rr : 0, lane);
                const uint64_t excl = incl - (part ? rr : 0);
                const bool reached = excl < left;
                const uint64_t chunk = (part && reached) ? (rr < left - excl ? rr : left - excl) : 0;
                const bool admitted = kv_ok && reached;
                const bool misfit = !skip && waiting && !blocked_prev && !kv_ok && reached;
                const uint32_t adm_mask = __ballot_sync(0xFFFFFFFFu, admitted && !prev);   // first admissions
                const uint32_t rank = __popc(adm_mask & ((1u << lane) - 1));
                if (admitted) {
                    if (!prev) t.admit_seq[base + li] = gsm.st.seq + rank;
                    rs[li] = (uint8_t)(rsc[li] | RS_RES | (growth ? RS_PREV : 0));
                    if (growth) {
                        t.kvres[base + li] = f;
                        if (prev) t.ptime[base + li] += clock - t.pstart[base + li];   // R31
                    }
                }
                if (chunk > 0) {
                    const uint32_t nr = rr - (uint32_t)chunk;
                    rem[li] = nr;
                    if (nr == 0) {
                        rs[li] = (uint8_t)(rs[li] | RS_FT);
                        const int d = atomicAdd(&gsm.ndone, 1);
                        if (d < kMaxDone) gsm.done[d] = li;
                    }
                }
                const uint64_t sum_chunk = warp_sum64(chunk);
                const uint64_t sum_f = warp_sum64(admitted ? f : 0);
                const uint64_t sum_inl = warp_sum64(admitted ? il : 0);
                const bool any_misfit = __any_sync(0xFFFFFFFFu, misfit);
                const int lastl = nvalid > 0 ? (int)nvalid - 1 : 0;
                const uint64_t lastk = __shfl_sync(0xFFFFFFFFu, lk, lastl);
                const uint32_t lasti = __shfl_sync(0xFFFFFFFFu, li, lastl);
                __syncwarp();            // every lane's reads of the group state precede lane 0's writes
                if (lane == 0) {
                    gsm.st.seq += __popc(adm_mask);
                    gsm.st.kv_free = kv - sum_f;
                    gsm.left = left - sum_chunk;
                    gsm.tok += sum_chunk;
                    gsm.inl += sum_inl;
                    if (any_misfit) gsm.blocked = 1;
                    if (nvalid > 0) {
                        gsm.thk = lastk;
                        gsm.thi = lasti;
                        gsm.has_th = 1;
                    }
                    // 1: budget left, nothing blocked, batch full -> next 32 candidates;
                    // 2: budget left but new admissions blocked (R6) -> only partials ranked
                    //    below this batch can still receive chunks.
                    gsm.pass_more = 0;
                    if (gsm.left > 0) gsm.pass_more = gsm.blocked ? 2 : (nvalid == kTop ? 1 : 0);
                    if (gsm.npart > kMaxPart) gsm.st.status = ST_PARTIAL_OVERFLOW;
                }
                __syncwarp();
                if (gsm.pass_more == 2) {
                    const int np = gsm.npart < kMaxPart ? gsm.npart : kMaxPart;
                    uint64_t pk = 0;
                    uint32_t pi = NIL;
                    if (lane < np) {
                        pk = gsm.partkey[lane];
                        pi = gsm.part[lane];
                        if (gsm.has_th && !before(gsm.thk, gsm.thi, pk, pi)) {   // already scanned
                            pk = 0;
                            pi = NIL;
                        }
                    }
                    warp_sort_desc(pk, pi, lane);
                    for (int q = 0; q < np; ++q) {                        // <= 3 under Lemma L2
                        const uint32_t id = __shfl_sync(0xFFFFFFFFu, pi, q);
                        if (id == NIL) break;
                        if (lane == 0 && gsm.left > 0) {
                            const uint32_t rr2 = rem[id];
                            const uint64_t ch = rr2 < gsm.left ? rr2 : gsm.left;
                            rem[id] = rr2 - (uint32_t)ch;
                            gsm.left -= ch;
                            gsm.tok += ch;
                            if (rr2 == ch) {
                                rs[id] = (uint8_t)(rs[id] | RS_FT);
                                const int d = gsm.ndone++;
                                if (d < kMaxDone) gsm.done[d] = id;
                            }
                        }
                        __syncwarp();
                    }
                    __syncwarp();
                    if (lane == 0) gsm.pass_more = 0;
                }
            }
            gsync<G, CL>();
            if (gsm.pass_more != 1) break;
        }

        // ---- a5: clock, calendar, first tokens (warp 0 of the group)
        if (wg == 0) {
            ReplicaState& st = gsm.st;
            if (lane == 0) {
                if (gsm.tok == 0 && st.n_dec == 0) {
                    st.status = ST_DEADLOCK;
                    st.flags |= FLAG_FINISHED;
                }
                st.clock += m.c0 + m.cp * gsm.tok + m.cd * (uint64_t)st.n_dec + gsm.inl;
                st.iter++;
                st.head[1]--;
                st.decisions++;
                st.scanned++;
                const uint32_t np = st.n_pend - (uint32_t)gsm.inv_dec;   // the pending set when ordered (R17)
                st.sum_pending += np;
                st.max_pending = np > st.max_pending ? np : st.max_pending;
                const Cal cal{t.cal + (size_t)r * kCalSlots, t.occ + (size_t)r * kCalWords};
                cal_process(cal, t.link + base, st.iter, st.clock, growth ? t.kvfin + base : fp, t.done + base, st,
                            growth ? rs : nullptr);
            }
            __syncwarp();
            const uint64_t now = st.clock;
            const uint64_t it = st.iter;
            const int nd = gsm.ndone;
            SWSTAT(11, nd);
            const uint16_t* out = t.out + base;
            uint32_t* cal = t.cal + (size_t)r * kCalSlots;
            uint32_t* occ = t.occ + (size_t)r * kCalWords;
            uint32_t* link = t.link + base;
            uint64_t kv_add = 0, n_dec_add = 0, done_add = 0;
            auto stamp = [&](uint32_t i) {
                if (growth) {                       // NEXT-1: first token once; a re-prefill emits the next
                    const uint8_t sb = rs[i];
                    if (!(sb & RS_GEN)) t.first_token[base + i] = now;
                    const uint32_t o = out[i];
                    const uint32_t ga = t.genp[base + i] + 1;
                    const uint32_t kr = t.kvres[base + i];
                    if (ga >= o) {
                        t.done[base + i] = now;
                        kv_add += kr;
                        done_add++;
                        rs[i] = (uint8_t)((sb & ~(RS_PEND | RS_FT | RS_RES)) | RS_GEN);
                    } else {
                        const uint64_t F = it + (o - ga);
                        t.fin[base + i] = F;
                        t.kvfin[base + i] = kr + (o - ga);
                        const uint32_t slot = (uint32_t)(F & (kCalSlots - 1));
                        link[i] = atomicExch(&cal[slot], i);
                        atomicOr(&occ[slot >> 5], 1u << (slot & 31));
                        n_dec_add++;
                        rs[i] = (uint8_t)((sb & ~(RS_PEND | RS_FT | RS_RES)) | RS_GEN | RS_DEC);
                    }
                    return;
                }
                t.first_token[base + i] = now;
                rs[i] = (uint8_t)(rs[i] & ~(RS_PEND | RS_FT | RS_RES));
                const uint32_t o = out[i];
                if (o == 1) {
                    t.done[base + i] = now;
                    kv_add += fp[i];
                    done_add++;
                } else {
                    const uint32_t slot = (uint32_t)((it + o - 1) & (kCalSlots - 1));
                    link[i] = atomicExch(&cal[slot], i);
                    atomicOr(&occ[slot >> 5], 1u << (slot & 31));
                    n_dec_add++;
                }
            };
            if (nd <= kMaxDone) {
                for (int q = lane; q < nd; q += 32) stamp(gsm.done[q]);
            } else {
                for (uint32_t i = lo + lane; i < hi; i += 32)
                    if ((rs[i] & (RS_FT | RS_RES)) == (RS_FT | RS_RES)) stamp(i);
            }
            __syncwarp();
            if (GR && gsm.inv_any) {                      // R34 victims may be admitted again from the next iteration
                for (uint32_t i = st.head[0] + lane; i < hi; i += 32)
                    if ((rs[i] & (RS_FT | RS_RES)) == RS_FT) rs[i] = (uint8_t)(rs[i] & ~RS_FT);
                __syncwarp();
            }
            kv_add = warp_sum64(kv_add);
            n_dec_add = warp_sum64(n_dec_add);
            done_add = warp_sum64(done_add);
            // advance the window start past served requests, 32 state bytes per probe
            uint32_t l2 = st.head[0];
            for (;;) {
                const uint32_t i = l2 + lane;
                const bool stop = i >= hi || (rs[i] & RS_PEND);
                const uint32_t b = __ballot_sync(0xFFFFFFFFu, stop);
                if (b) {
                    l2 += __ffs(b) - 1;
                    break;
                }
                l2 += 32;
            }
            __syncwarp();
            if (lane == 0) {
                st.kv_free += kv_add;
                st.n_dec += (uint32_t)n_dec_add;
                st.done_count += (uint32_t)done_add;
                st.n_pend -= (uint32_t)nd;
                st.head[0] = l2 < hi ? l2 : hi;
                t.state[r] = st;
            }
        }
        gsync<G, CL>();
      }
        if (wg == 0 && lane == 0 && ctl.count_active && !(gsm.st.flags & FLAG_FINISHED)) atomicAdd(&s_active, 1u);
        gsync<G, CL>();
    }
    if constexpr (CL > 1) cooperative_groups::this_cluster().sync();
    // The launch's last CTA publishes the active-replica count to ctl.active_out (device memory,
    // or the caller's mapped host word under graph replay) and resets the control words for the
    // next launch on the stream: a call is then its k_step launches alone (no budget kernel, no
    // memset, no copy node).
    __syncthreads();
    if (tid == 0) {
        if (s_active) atomicAdd(&ctl.w->acc, s_active);
        __threadfence();
        if (atomicAdd(&ctl.w->done_ctas, 1u) == gridDim.x - 1) {
            __threadfence();
            const uint32_t a = atomicExch(&ctl.w->acc, 0u);
            if (ctl.count_active) *ctl.active_out = a;
            atomicExch(&ctl.w->ctr, 0ull);
            atomicExch(&ctl.w->done_ctas, 0u);
        }
    }
}

// ReplicaState.head[0] = window start lo (oldest possibly-pending id), head[1] = remaining
// iteration budget of the current tcm_step call; the class-queue fields are unused here.
// Per-call iteration budget of every replica; also zeroes the active-replica count and the
// replica counter of the dynamic mode (one launch instead of a launch and two memsets).
// (k_step's first launch of a call sets head[1] itself: StepCtl.budget.)
__global__ void k_sw_init(TraceDev t, StepSync* w) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r == 0) {
        w->ctr = 0;
        w->done_ctas = 0;
        w->acc = 0;
    }
    if (r < t.R) {
        t.state[r].head[0] = 0;
        t.state[r].head[1] = 0;
        t.state[r].tail[0] = 0;      // NEXT-1: running-set lower bound, preemptions, forced ones
        t.state[r].tail[1] = 0;
        t.state[r].tail[2] = 0;
    }
}

void stepwise_init(const TraceDev& t, const StepwiseWorkspace& w, cudaStream_t s) {
    k_sw_init<<<(t.R + 255) / 256, 256, 0, s>>>(t, w.sync);
}

// rem[N], then the 16-byte StepSync (8-byte aligned)
size_t stepwise_extra_bytes(uint32_t R, uint64_t N) {
    (void)R;
    return ((4 * N + 7) & ~7ull) + sizeof(StepSync);
}
size_t stepwise_workspace_bytes(uint32_t R, uint64_t N) { return N + stepwise_extra_bytes(R, N); }

StepwiseWorkspace stepwise_bind(void* p, uint32_t R, uint64_t N) {
    StepwiseWorkspace w;
    w.base = p;
    w.R = R;
    w.sync = reinterpret_cast<StepSync*>(reinterpret_cast<char*>(p) + ((4 * N + 7) & ~7ull));
    return w;
}

namespace {
struct Launch {
    int grid;
    int group;   // warps per replica (per CTA of the cluster)
    int cluster; // CTAs per replica (thread-block cluster; 1 = none)
};
constexpr int kCluster = 8;    // CTAs per replica for a few huge queues (portable cluster size)

// Per-device launch facts, queried once (kernel attributes and occupancy do not change).
struct DevFacts {
    int sms = 0, per_sm1 = 1, per_sm8 = 1;
    int per_sm1g = 1, per_sm8g = 1;     // the NEXT-1 instantiations (2 blocks / SM: no spills)
};

DevFacts dev_facts() {
    static DevFacts cache[64];
    static std::mutex mu;                   // contexts may step concurrently from several host threads
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    DevFacts& f = cache[dev & 63];
    if (f.sms == 0) {
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(k_step<1, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
        cudaFuncSetAttribute(k_step<1, false, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
        cudaFuncSetAttribute(k_step<8, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
        cudaFuncSetAttribute(k_step<1, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
        cudaFuncSetAttribute(k_step<8, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
        cudaFuncSetAttribute(k_step<8, false, kCluster>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
        cudaFuncSetAttribute(k_step<8, true, kCluster>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kRingBytes);
        int p1 = 1, p8 = 1;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, k_step<1, false, 1>, kThreads, kRingBytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p8, k_step<8, false, 1>, kThreads, kRingBytes);
        f.per_sm1 = p1 < 1 ? 1 : p1;
        f.per_sm8 = p8 < 1 ? 1 : p8;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p1, k_step<1, true, 1>, kThreads, kRingBytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&p8, k_step<8, true, 1>, kThreads, kRingBytes);
        f.per_sm1g = p1 < 1 ? 1 : p1;
        f.per_sm8g = p8 < 1 ? 1 : p8;
        f.sms = sms;
    }
    return f;
}

// The TCM-only instantiation (TraceDev.all_tcm); TCM_SW_TO=0 forces the general one (development A/B).
bool use_to() {
    static const bool on = [] {
        const char* e = getenv("TCM_SW_TO");
        return !(e && e[0] == '0');
    }();
    return on;
}

Launch stepwise_config(uint32_t R, uint64_t N, bool growth) {
    const DevFacts f = dev_facts();
    const int sms = f.sms, per_sm1 = growth ? f.per_sm1g : f.per_sm1, per_sm8 = growth ? f.per_sm8g : f.per_sm8;
    // Warp per replica unless the queues are few and huge: a CTA per replica only when there are
    // fewer replicas than twice the warp slots AND they average >= 8,192 requests (measured: for
    // sweeps of ~1k-request replicas a warp per replica is 2.2x faster, its iterations need no
    // block barriers), and a cluster for a handful of queues.
    const uint64_t warp_slots = (uint64_t)sms * per_sm1 * kWarpsPerBlock;
    Launch l;
    l.cluster = 1;
    const char* force = getenv("TCM_SW_GROUP");        // development A/B knob: "1", "8" or "cluster"
    const int fg = force ? (force[0] == 'c' ? 64 : atoi(force)) : 0;
    if (fg == 1 || fg == 8) {
        l.group = fg;
        const uint64_t cap = (uint64_t)sms * (fg == 1 ? per_sm1 : per_sm8);
        const uint64_t need = fg == 1 ? ((uint64_t)R + kWarpsPerBlock - 1) / kWarpsPerBlock : (uint64_t)R;
        l.grid = (int)(need < cap ? need : cap);
        return l;
    }
    if (fg == 64 || (uint64_t)R * kCluster * 2 <= (uint64_t)sms) {
        // few queues: a cluster of kCluster CTAs streams each one (DSMEM merge), 64 warps per queue
        l.group = 8;
        l.cluster = kCluster;
        l.grid = (int)R * kCluster;
    } else if ((uint64_t)R >= 2 * warp_slots || N < (uint64_t)R * 8192) {
        l.group = 1;
        const uint64_t need = ((uint64_t)R + kWarpsPerBlock - 1) / kWarpsPerBlock;
        const uint64_t cap = (uint64_t)sms * per_sm1;
        l.grid = (int)(need < cap ? need : cap);
    } else {
        l.group = 8;
        const uint64_t cap = (uint64_t)sms * per_sm8;
        l.grid = (int)((uint64_t)R < cap ? R : cap);
    }
    return l;
}
}  // namespace

#ifdef TCM_VAR_SWSTATS
}  // namespace tcm
extern "C" int tcm_dev_swstats(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, tcm::g_swstats, sizeof(tcm::g_swstats)) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(tcm::g_swstats, z, sizeof(z));
    }
    return 0;
}
namespace tcm {
#endif

tcm_status stepwise_run(const ModelConst& m, const TraceDev& t, const StepwiseWorkspace& w, uint32_t max_iters,
                        uint32_t* active_out, cudaStream_t s, uint64_t* launches, cudaEvent_t ev_begin,
                        cudaEvent_t ev_end, double* kernel_ms, bool* deferred) {
    uint32_t* remv = reinterpret_cast<uint32_t*>(w.base);
    const Launch L = stepwise_config(t.R, t.N, t.any_growth != 0);
    StepCtl ctl{};
    ctl.w = w.sync;
    ctl.dyn = L.group == 1 && L.cluster == 1 && t.R > (uint64_t)L.grid * kWarpsPerBlock;   // else static is ideal
    // Each k_step launch advances every active replica by up to kItersPerLaunch iterations (tcm_step's
    // budget, set by the call's first launch, bounds the total); launch in chunks and read the active
    // count only at the end of each chunk.  A call that fits in one chunk (tcm_step(n <= 64)) returns
    // without synchronising: the caller reads *active_out and the events after its own (single)
    // synchronisation (*deferred = true).
    const uint32_t chunk = 64;
    uint64_t done_launches = 0;
    *deferred = false;
    for (;;) {
        uint32_t this_chunk = chunk;
        if ((uint64_t)max_iters - done_launches < this_chunk) this_chunk = (uint32_t)(max_iters - done_launches);
        // device time of the k_step launches alone (tcm_stats_host.engine_ms)
        if (ev_begin && cudaEventRecord(ev_begin, s) != cudaSuccess) return TCM_E_CUDA;   // null: untimed (graph capture)
        for (uint32_t q = 0; q < this_chunk; ++q) {
            ctl.count_active = q + 1 == this_chunk;
            ctl.active_out = active_out;
            ctl.budget = done_launches == 0 && q == 0 ? max_iters : 0u;
            if (L.cluster > 1) {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(L.grid);
                cfg.blockDim = dim3(kThreads);
                cfg.dynamicSmemBytes = kRingBytes;
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = L.cluster;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                cudaError_t e = t.any_growth
                    ? cudaLaunchKernelEx(&cfg, k_step<8, true, kCluster>, m, t, remv, ctl)
                    : cudaLaunchKernelEx(&cfg, k_step<8, false, kCluster>, m, t, remv, ctl);
                if (e != cudaSuccess) return TCM_E_CUDA;
            } else if (t.any_growth) {
                if (L.group == 1) k_step<1, true, 1><<<L.grid, kThreads, kRingBytes, s>>>(m, t, remv, ctl);
                else k_step<8, true, 1><<<L.grid, kThreads, kRingBytes, s>>>(m, t, remv, ctl);
            } else {
                if (L.group == 1 && t.all_tcm && use_to())
                    k_step<1, false, 1, true><<<L.grid, kThreads, kRingBytes, s>>>(m, t, remv, ctl);
                else if (L.group == 1) k_step<1, false, 1><<<L.grid, kThreads, kRingBytes, s>>>(m, t, remv, ctl);
                else k_step<8, false, 1><<<L.grid, kThreads, kRingBytes, s>>>(m, t, remv, ctl);
            }
            (*launches)++;
        }
        done_launches += this_chunk;
        if (ev_end && cudaEventRecord(ev_end, s) != cudaSuccess) return TCM_E_CUDA;
        if (cudaGetLastError() != cudaSuccess) return TCM_E_CUDA;
        if (done_launches == this_chunk && done_launches >= max_iters) {
            *deferred = true;
            break;
        }
        uint32_t act = 0;
        if (cudaMemcpyAsync(&act, active_out, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return TCM_E_CUDA;
        if (cudaStreamSynchronize(s) != cudaSuccess) return TCM_E_CUDA;
        float ms = 0;
        if (ev_begin && cudaEventElapsedTime(&ms, ev_begin, ev_end) != cudaSuccess) return TCM_E_CUDA;
        *kernel_ms += ms;
        if (act == 0 || done_launches >= max_iters) break;
    }
    return TCM_OK;
}

}  // namespace tcm
