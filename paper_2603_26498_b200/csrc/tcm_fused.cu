// tcm_fused.cu -- TCM_ENGINE_FUSED: the whole per-iteration scheduling step (SURVEY.md 8(a)
// rows a1-a5) for one replica, run by one persistent thread with the replica state in
// registers.
//
// a3 is computed as the exact 3-way merge of the class-FIFO heads:
//   Lemma L1: within class c every request shares (S_c, k_c, p_c) and K1 is
//   non-decreasing in the waiting time, so the (key desc, arrival asc, id asc) order restricted
//   to class c is arrival order -- the paper's "FCFS within each queue".
//   The global order is therefore the merge of the three queue heads, and each decision
//   keys only the <= 3 + admitted candidates it actually visits.
//   Lemma L2: only a queue head can be partially prefilled, so per-request mutable state
//   collapses to head_rem[3] / head-admitted bits in ReplicaState.
//   Lemma L3: with nothing pending, consecutive iterations are identical until the next
//   calendar event or arrival, so they are fast-forwarded in closed form (integer math).
//
// Memory layout.  The classification of a1 is a fixed function of the request,
// so the prologue k_fpack applies it once per request and stores each replica's requests as
// three class segments of 32-byte records (FRec) in arrival order: a class queue is a cursor
// range of its segment, a head's successor is the next record, and nothing is linked.  The
// decode calendar keeps, per iteration slot, only the number of finishing requests and the sum
// of their footprints (updated with fire-and-forget atomics), with its occupancy bitmap in
// shared memory and a 64-bit word summary in a register.  Finish times are stamped after the
// launch by k_fstamp from a per-replica log of (iteration, clock) events, and so are first-token
// times: the loop itself never revisits a request once its prefill is complete.
#include <cstdlib>
#include <mutex>

#include "tcm_fcal.cuh"
#include "tcm_internal.cuh"
#include "tcm_k1.cuh"

namespace tcm {

namespace {

constexpr uint32_t kThreads = kFThreads;
}  // namespace

// Development instrumentation (build variant -DTCM_VAR_FSTATS=1 only): pass types and what ends
// each closed-form window, per-thread counters in shared memory flushed once per thread; read by
// tools/probe_fstats.py through tcm_dev_fstats.
#ifdef TCM_VAR_FSTATS
__device__ unsigned long long g_fstats[16];
#define FSTAT(k, v) (s_fst[k][threadIdx.x] += (uint32_t)(v))
#else
#define FSTAT(k, v) ((void)0)
#endif

// ---------------------------------------------------------------------------------------
// Prologue (row a1's classification, once per request): one warp per replica builds the three
// class segments (stable: arrival order within a class) and points the queue cursors at them.
__global__ void k_fpack(ModelConst m, TraceDev t) {
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (r >= t.R) return;
    const uint64_t a = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - a);
    const bool prio = t.params[r].policy == TCM_POLICY_TCM;
    const uint32_t lt = (1u << lane) - 1;
    uint32_t cnt0 = 0, cnt1 = 0;
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        const int q = (i < n && prio) ? classify(m, t.mod[a + i], t.footprint[a + i]) : (i < n ? 0 : 3);
        cnt0 += __popc(__ballot_sync(~0u, q == 0));
        cnt1 += __popc(__ballot_sync(~0u, q == 1));
    }
    // segments [0, cnt0) [cnt0 + 2, ..) [.. + 4, ..), each followed by two sentinel records
    uint32_t run[3] = {0, cnt0 + 2, cnt0 + cnt1 + 4};
    FRec* rec = t.fw.rec + a + 6ull * r;
    for (uint32_t i0 = 0; i0 < n; i0 += 32) {
        const uint32_t i = i0 + lane;
        int q = 3;
        FRec x;
        if (i < n) {
            x.arrival = t.arrival[a + i];
            x.fp = t.footprint[a + i];
            x.inl = t.inl[a + i];
            x.id = i;
            x.out = t.out[a + i];
            x.spare = 0;
            q = prio ? classify(m, t.mod[a + i], x.fp) : 0;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const uint32_t b = __ballot_sync(~0u, q == c);
            if (q == c) rec[run[c] + __popc(b & lt)] = x;
            run[c] += __popc(b);
        }
    }
    if (lane < 6) {
        FRec x{~0ull, 0, 0, 0, 0, 0};
        rec[run[lane >> 1] + (lane & 1)] = x;   // sentinels: arrival ~0 never becomes pending
    }
    if (lane == 0) {
        ReplicaState& st = t.state[r];
        st.head[0] = 0;
        st.head[1] = cnt0 + 2;
        st.head[2] = cnt0 + cnt1 + 4;
    }
    if (t.fg.top && lane < 3) {           // NEXT-1 (k_fgrow): empty preempted stacks, segment starts
        t.fg.top[3 * r + lane] = NIL;
        t.fg.seg[3 * r + lane] = lane == 0 ? 0 : (lane == 1 ? cnt0 + 2 : cnt0 + cnt1 + 4);
        t.fg.hres[3 * r + lane] = 0;
    }
}

// lpw: replicas per warp (a power of two <= 32).  With fewer replicas than resident lanes the warps
// carry fewer replicas each, so a warp pays for the union of fewer divergent paths.
__global__ void __launch_bounds__(kThreads, 8) k_fused(ModelConst m, TraceDev t, uint32_t max_iters,
                                                    uint32_t* active, uint32_t lpw) {
    __shared__ uint32_t occ_s[kCalWords][kThreads];
    // work counters live in shared memory during the loop (registers are the scarce resource)
    __shared__ unsigned long long s_dec[kThreads], s_sum[kThreads], s_ff[kThreads];
    __shared__ uint32_t s_idle[kThreads], s_maxp[kThreads], s_scan[kThreads];
    const uint32_t gthread = blockIdx.x * blockDim.x + threadIdx.x;
    if ((gthread & 31) >= lpw) return;
    const uint32_t r = (gthread >> 5) * lpw + (gthread & 31);
    if (r >= t.R) return;
    if (t.fg.top && (t.params[r].flags & TCM_KV_GROWTH)) return;   // k_fgrow runs the NEXT-1 replicas
    ReplicaState st = t.state[r];
    if (st.flags & FLAG_FINISHED) return;
    const uint32_t tid = threadIdx.x;
#ifdef TCM_VAR_FSTATS
    __shared__ uint32_t s_fst[16][kThreads];
    for (int k = 0; k < 16; ++k) s_fst[k][tid] = 0;
#endif
    s_dec[tid] = st.decisions;
    s_sum[tid] = st.sum_pending;
    s_ff[tid] = st.ff_iters;
    s_idle[tid] = st.idle_jumps;
    s_maxp[tid] = st.max_pending;
    s_scan[tid] = st.scanned;
    // j decisions with n_pend pending requests each (R17)
    auto decided = [&](uint64_t j, uint32_t np) {
        s_dec[tid] += j;
        s_sum[tid] += j * np;
        s_maxp[tid] = np > s_maxp[tid] ? np : s_maxp[tid];
    };

    const tcm_replica_params prm = t.params[r];
    const uint64_t base = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - base);
    const uint64_t* __restrict__ arr = t.arrival + base;
    const FRec* __restrict__ rec = t.fw.rec + base + 6ull * r;
    // result / workspace arrays are indexed base + id off the kernel parameters (no per-replica
    // pointer registers)
#define admit(i) t.admit_seq[base + (i)]
#define first(i) t.first_token[base + (i)]
#define fin(i) t.fw.fin[base + (i)]
    uint64_t* log = t.fw.log + 4 * base;
    Calendar cal{t.fw.cal + (size_t)r * kCalSlots, Occ{occ_s, threadIdx.x}, 0, ~0ull, 0, 0};
#pragma unroll 8
    for (uint32_t k = 0; k < kCalWords; ++k) {
        const uint32_t w = t.occ[(size_t)r * kCalWords + k];
        cal.occ.word(k) = w;
        cal.sum |= (uint64_t)(w != 0) << k;
    }

    const bool prio = prm.policy == TCM_POLICY_TCM;
    const uint32_t B = prm.chunk_budget;
    const ClassPack* kp = t.kpack + r;
    // FP32 bound constants per class, in shared memory (indexable by a run-time class)
    __shared__ float s_fc[3][3][kThreads];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        s_fc[0][c][tid] = kp->fS[c];
        s_fc[1][c][tid] = kp->fp2[c];
        s_fc[2][c][tid] = kp->fC2[c];
    }
#define fS(c) s_fc[0][c][tid]
#define fp2(c) s_fc[1][c][tid]
#define fC2(c) s_fc[2][c][tid]
    const uint32_t zmask = kp->zero_mask;
    const bool use_bound = kp->filter_ok != 0;   // FP32 bound validated for these constants

    // Register caches: each class queue's head (arrival, footprint) and its successor's, so that
    // advancing a queue never waits on memory (inline / id / out are read from the record, in
    // L1, when the head is admitted or completes).  An exhausted segment
    // ends with a sentinel record of arrival ~0: a head is pending iff its arrival <= clock.
    uint64_t harr[3];
    uint32_t hf[3];
    // the next two records of each class queue, (arrival, footprint | inline << 32), prefetched
    // into shared memory by cp.async: slot k & 1 holds record k
    __shared__ ulonglong2 s_ring[3][2][kThreads];
    __shared__ uint32_t s_gseq[3][2][kThreads];           // commit-group number of each slot's copy
    uint32_t ng = 0;                                       // copy groups committed so far
    auto prefetch = [&](int c, uint32_t k, uint64_t dep) {
        cp_async16(&s_ring[c][k & 1][tid], rec + k, dep);
        s_gseq[c][k & 1][tid] = ng++;
    };
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const uint32_t h = st.head[c];
        harr[c] = ~0ull;
        hf[c] = 0;
        ld_arrfp(rec + h, harr[c], hf[c]);
        if (harr[c] != ~0ull) {
            prefetch(c, h + 1, 0);
            prefetch(c, h + 2, 0);
        }
    }
    // next two arrivals in arrival order (a1 counts pending requests)
    uint64_t next_arr = st.nxt < n ? arr[st.nxt] : ~0ull;
    uint64_t next_arr2 = st.nxt + 1 < n ? arr[st.nxt + 1] : ~0ull;
    cal.find_next(st.iter, st.n_dec);
    uint32_t budget = max_iters;
    // FP32 bound of a head's priority after waiting w (|P~ - P| <= 1e-5)
    auto bound = [&](int c, uint64_t w) -> float {
        return (w == 0 || ((zmask >> c) & 1u) || !use_bound) ? fS(c) : k1_filter_f32(fS(c), fp2(c), fC2(c), w);
    };
    auto bound_dyn = [&](int c, uint64_t w) -> float {     // c not known at compile time
        return (w == 0 || ((zmask >> c) & 1u) || !use_bound) ? fS(c) : k1_filter_f32(fS(c), fp2(c), fC2(c), w);
    };
    // A window of j iterations of length dt stops at the first iteration that ingests the next
    // arrival: min(j, ceil((next_arr - clock) / dt)).  The 64-bit division is needed only when the
    // window's last iteration starts at or after the arrival (else the quotient is >= j).
    auto arr_cap = [&](uint64_t j, uint64_t dt) -> uint64_t {
        if (next_arr != ~0ull && st.clock + (j - 1) * dt >= next_arr) {
            const uint64_t ja = (next_arr - st.clock + dt - 1) / dt;
            j = ja < j ? ja : j;
        }
        return j;
    };

    for (;;) {
        // ---- a1: arrivals <= clock join the pending set (their class queue already holds them)
        while (next_arr <= st.clock) {
            st.n_pend++;
            st.nxt++;
            next_arr = next_arr2;
            next_arr2 = st.nxt + 1 < n ? arr[st.nxt + 1] : ~0ull;
        }

        FSTAT(0, 1);
        if (st.n_pend == 0) {
            if (st.n_dec == 0) {
                if (st.nxt == n) {                      // every request served
                    st.flags |= FLAG_FINISHED;
                    break;
                }
                st.clock = next_arr;                    // R15 idle jump (not an iteration)
                s_idle[tid]++;
                continue;
            }
            if (budget == 0) break;
            // ---- Lemma L3: decode-only iterations until the next finish or arrival
            const uint64_t F = cal.next;
            const uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint64_t j = F - st.iter;
            j = j < budget ? j : budget;
            j = arr_cap(j, dt);
            FSTAT(1, 1);
            FSTAT(6, st.iter + j == F);
            FSTAT(11, j);
            st.clock += j * dt;
            st.iter += j;
            s_ff[tid] += j;
            budget -= (uint32_t)j;
            if (st.iter == F) {
                log_event(log, st);
                cal.process(st);
            }
            continue;
        }
        if (budget == 0) break;

        // ---- Lemma L4: a blocked decision repeats identically until the next finish or arrival.
        // Nothing can prefill when decodes take the whole budget (R8), or when no head holds KV
        // (no partial, L2) and every class head is too large for the free KV: the top-ranked
        // waiting request is a head (L1), its misfit stops every later admission (R6), and
        // neither the heads nor kv_free change before a calendar finish or a new arrival.
        uint32_t left = B > st.n_dec ? B - st.n_dec : 0;   // R8
        bool stuck = left == 0;
        if (!stuck) {
            stuck = true;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (harr[c] <= st.clock && (((st.flags >> c) & 1u) || (uint64_t)hf[c] <= st.kv_free)) stuck = false;
        }
        // FP32 bounds of the pending heads now: shared by L4c, L5 and the scan's ordering
        float pf[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) pf[c] = (!stuck && prio && harr[c] <= st.clock) ? bound(c, st.clock - harr[c]) : 0.0f;
        // L4c: some head that does not fit ranks, *now*, above every head that fits even at the
        // start of the window's last iteration.  Priorities only grow with waiting time (L1), so
        // at every iteration of the window the top-ranked head misfits and blocks all admissions
        // (R6); with no partial (flags) nothing prefills.  FP32 bounds only (rigorous, 2.5e-4
        // margin).  Tried before every decision with a misfitting head and no partial: a window of
        // one iteration is this decision itself, blocked, decided without the scan.
        uint64_t l4c_j = ~0ull;
        if (!stuck && prio && use_bound && st.n_dec > 0 && (st.flags & 7u) == 0) {
            FSTAT(10, 1);
            const uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint64_t j = cal.next - st.iter;
            j = j < budget ? j : budget;
            j = arr_cap(j, dt);
            bool zero_head = false;
            float ptop = -1.0f;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const bool pend = harr[c] <= st.clock;
                zero_head |= pend && ((zmask >> c) & 1u);
                if (pend && !((zmask >> c) & 1u) && (uint64_t)hf[c] > st.kv_free) {
                    const float p = pf[c];
                    ptop = p > ptop ? p : ptop;
                }
            }
            // Window search, one copy of the bound code: the full window j; then j = 1 (is this
            // decision itself provably blocked?  If not, the scan decides); then j/2, j/4, ... >= 2,
            // the first success taken, else the one blocked iteration.  A blocked decision with no
            // partial prefills nothing (R6): the scan's outcome without the scan.
            uint64_t cand = j;
            for (int step = 0; step < 7 && cand >= 1 && !zero_head && ptop >= 0.0f; ++step) {
                const uint64_t t_end = st.clock + (cand - 1) * dt;
                float pfit = -1.0f;
                if (cand == 1) {             // the window's end is now: the pass's bounds
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        if (harr[c] <= st.clock && (uint64_t)hf[c] <= st.kv_free) pfit = pf[c] > pfit ? pf[c] : pfit;
                } else
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (harr[c] <= st.clock && (uint64_t)hf[c] <= st.kv_free) {
                        const float p = bound(c, t_end - harr[c]);
                        pfit = p > pfit ? p : pfit;
                    }
                }
                const bool ok = ptop - pfit > 2.5e-4f;
                if (step == 1) {
                    if (!ok) break;
                    l4c_j = 1;
                    cand = j >> 1;
                } else {
                    if (ok) {
                        l4c_j = cand;
                        break;
                    }
                    cand = step == 0 ? (cand == 1 ? 0 : 1) : cand >> 1;
                }
                if (step >= 1 && cand < 2) break;
            }
            if (l4c_j != ~0ull) stuck = true;
        }
        if (stuck && st.n_dec > 0) {
            const uint64_t F = cal.next;
            const uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint64_t j = F - st.iter;
            j = j < budget ? j : budget;
            j = j < l4c_j ? j : l4c_j;
            j = arr_cap(j, dt);
#ifdef TCM_VAR_FSTATS
            {
                FSTAT(l4c_j == ~0ull ? 2 : 3, 1);
                FSTAT(6, st.iter + j == F);
                FSTAT(11, j);
                const bool at_arr = next_arr != ~0ull && st.clock + j * dt >= next_arr && st.iter + j != F;
                FSTAT(7, at_arr);
                FSTAT(8, at_arr && (prio ? harr[0] <= st.clock && harr[1] <= st.clock && harr[2] <= st.clock : harr[0] <= st.clock));
                FSTAT(9, l4c_j != ~0ull && j == l4c_j && st.iter + j != F && !at_arr);
            }
#endif
            decided(j, st.n_pend);
            st.clock += j * dt;
            st.iter += j;
            budget -= (uint32_t)j;
            if (st.iter == F) {
                log_event(log, st);
                cal.process(st);
            }
            continue;
        }

        // ---- Lemma L5: a partial prefill that outranks every other head able to take tokens
        // (partial, or waiting and fitting the free KV) and needs more than this iteration's
        // budget takes the whole budget (a4) while nothing else changes: no admission, no first
        // token, kv_free and n_dec fixed until the next calendar event, no arrival.  Those
        // iterations repeat with dt = c0 + cp*Bp + cd*n_dec and are taken in closed form.  Under
        // TCM the partial's priority now must exceed every other candidate's FP32 bound at the
        // start of the window's last iteration by 2.5e-4 (priorities only grow, L1); FCFS has
        // one queue, whose head it is.
        if (st.flags & 7u) {
            int top = -1;
            float ptop = -1.0f;
            uint32_t cand = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (harr[c] <= st.clock && (((st.flags >> c) & 1u) || (uint64_t)hf[c] <= st.kv_free)) {
                    cand |= 1u << c;
                    const float p = pf[c];
                    if (top < 0 || p > ptop) {
                        top = c;
                        ptop = p;
                    }
                }
            }
            uint32_t rt = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c)
                if (c == top) rt = ((st.flags >> c) & 1u) ? st.rem[c] : 0;
            if (rt > left && (!prio || use_bound)) {
                const uint64_t dt = m.c0 + m.cp * left + m.cd * st.n_dec;
                const uint64_t F = cal.next;
                uint64_t j = (rt - 1) / left;                   // rem stays > 0
                const uint64_t jf = F - st.iter;
                j = jf < j ? jf : j;
                j = j < budget ? j : budget;
                j = arr_cap(j, dt);
                cand &= ~(1u << top);
                bool ok = j >= 1;
                if (prio && cand) {
                    ok = false;
                    for (int h = 0; h < 6 && j >= 1; ++h, j >>= 1) {
                        const uint64_t t_end = st.clock + (j - 1) * dt;
                        float pmax = -1.0f;
                        if (j == 1) {            // the window's end is now: the pass's bounds
#pragma unroll
                            for (int c = 0; c < 3; ++c)
                                if ((cand >> c) & 1u) pmax = pf[c] > pmax ? pf[c] : pmax;
                        } else
#pragma unroll
                        for (int c = 0; c < 3; ++c) {
                            if ((cand >> c) & 1u) {
                                const float p = bound(c, t_end - harr[c]);
                                pmax = p > pmax ? p : pmax;
                            }
                        }
                        if (ptop - pmax > 2.5e-4f) {
                            ok = true;
                            break;
                        }
                    }
                }
                if (ok) {
                    FSTAT(4, 1);
                    FSTAT(6, st.iter + j == F);
                    FSTAT(11, j);
#pragma unroll
                    for (int c = 0; c < 3; ++c)
                        if (c == top) st.rem[c] -= (uint32_t)(j * left);
                    decided(j, st.n_pend);
                    st.clock += j * dt;
                    st.iter += j;
                    budget -= (uint32_t)j;
                    if (st.iter == F) {
                        log_event(log, st);
                        cal.process(st);
                    }
                    continue;
                }
            }
        }

        // ---- a2 + a3 + a4: merge the class-FIFO heads by key, scan under token/KV budgets.
        // The scan advances the queue cursors in place.  A request whose prefill completes gets
        // its first token in this iteration (R12): its KV release (out = 1) and decode start
        // are applied after the scan, and its first_token_us / done_us are stamped by k_fstamp
        // from the iteration number (bit 63 marks it pending) and the event log.
        uint64_t tok = 0, inl_sum = 0, kv_rel = 0;
        uint32_t ncomp = 0, new_dec = 0;
        const uint64_t it1 = st.iter + 1;                   // this iteration's number
        bool blocked = false;                               // R6
        uint64_t key[3];
        bool ex[3];           // ex[c]: key[c] holds the exact K1 key
        // Two heads whose bounds are more than 2.5e-4 apart are ordered by the bounds (the exact
        // order, since the bound error is < 1e-5); only closer pairs get their exact FP64 keys.
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            key[c] = 0;
            ex[c] = !prio;
        }
        while (left > 0) {
            // tournament over the eligible heads carrying only the leader's index (its bound, key,
            // arrival and cursor are selected when a comparison needs them)
            int best = -1;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (harr[c] <= st.clock && (!blocked || ((st.flags >> c) & 1u))) {
                    bool better = best < 0;
                    if (!better) {
                        const float d = pf[c] - sel3(best, pf);
                        if (use_bound && d > 2.5e-4f) {
                            better = true;
                        } else if (use_bound && d < -2.5e-4f) {
                            better = false;
                        } else {
                            if (!ex[c]) {
                                key[c] = exact_key(kp, c, st.clock - harr[c]);
                                ex[c] = true;
                            }
#pragma unroll
                            for (int q = 0; q < c; ++q) {
                                if (q == best && !ex[q]) {
                                    key[q] = exact_key(kp, q, st.clock - harr[q]);
                                    ex[q] = true;
                                }
                            }
                            const uint64_t bk = sel3(best, key), ba = sel3(best, harr);
                            better = key[c] > bk ||
                                     (key[c] == bk && (harr[c] < ba || (harr[c] == ba && [&] {
                                         uint32_t ic, ib, o, il;   // equal key and arrival: id order (R4)
                                         ld_inl_id_out(rec + st.head[c], il, ic, o);
                                         ld_inl_id_out(rec + sel3(best, st.head), il, ib, o);
                                         return ic < ib;
                                     }())));
                        }
                    }
                    if (better) best = c;
                }
            }
            if (best < 0) break;
            // the chosen head, with one copy of the code for every class: read its fields,
            // admit / chunk / complete it, write them back
            const uint32_t hb = sel3(best, st.head);
            const uint32_t fb = sel3(best, hf);
            uint32_t remb = sel3(best, st.rem);
            bool adv = false;
            bool go = true;
            if (!((st.flags >> best) & 1u)) {
                if ((uint64_t)fb > st.kv_free) {
                    blocked = true;                         // first misfit stops new admits
                    go = false;
                } else {
                    st.kv_free -= fb;                       // R7 reserve the full footprint
                    uint32_t il, id, o;
                    ld_inl_id_out(rec + hb, il, id, o);
                    admit(id) = st.seq++;
                    inl_sum += il;                          // R10
                    st.flags |= 1u << best;
                    remb = fb;
                }
            }
            if (go) {
                const uint32_t ch = remb < left ? remb : left;
                remb -= ch;
                left -= ch;
                tok += ch;
                if (remb == 0) {                            // prefill complete
                    uint32_t il, id, o;
                    ld_inl_id_out(rec + hb, il, id, o);
                    first(id) = kPending | it1;
                    ncomp++;
                    if (o == 1) {                           // finishes with its first token
                        fin(id) = it1;
                        kv_rel += fb;
                    } else {                                // decodes until iteration it1 + out - 1
                        const uint64_t F = it1 + o - 1;
                        fin(id) = F;
                        cal.insert(F, fb);
                        new_dec++;
                    }
                    st.flags &= ~(1u << best);
                    adv = true;
                }
            }
            // next in FIFO: the prefetched successor becomes the head, the record after the new
            // successor is prefetched into the slot it leaves
            uint64_t narr = ~0ull;
            uint32_t nf = 0;
            float npf = 0.0f;
            if (adv) {
                const uint32_t sl = (hb + 1) & 1;
                cp_async_wait(ng - 1 - s_gseq[best][sl][tid]);
                const ulonglong2 v = s_ring[best][sl][tid];
                narr = v.x;
                nf = (uint32_t)v.y;
                if (narr != ~0ull) prefetch(best, hb + 3, narr);
                if (prio && narr <= st.clock) npf = bound_dyn(best, st.clock - narr);
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (c == best) {
                    st.rem[c] = remb;
                    if (adv) {
                        st.head[c] = hb + 1;
                        harr[c] = narr;
                        hf[c] = nf;
                        ex[c] = !prio;
                        pf[c] = npf;
                    }
                }
            }
        }
        FSTAT(5, 1);
        FSTAT(12, tok == 0);
        FSTAT(13, ncomp == 0 && inl_sum == 0 && tok > 0);
        if (tok == 0 && st.n_dec == 0) {                    // unreachable under R6
            t.state[r].status = ST_DEADLOCK;
            st.flags |= FLAG_FINISHED;
            break;
        }

        // ---- a5: iteration cost, clock, decode calendar, first tokens (R12)
        st.clock += m.c0 + m.cp * tok + m.cd * (uint64_t)st.n_dec + inl_sum;
        st.iter = it1;
        decided(1, st.n_pend);
        s_scan[tid]++;
        budget--;
        st.n_pend -= ncomp;
        st.kv_free += kv_rel;
        st.n_dec += new_dec;
        const bool event = it1 == cal.next;
        if (ncomp > 0 || event) log_event(log, st);
        if (event) cal.process(st);
    }

    asm volatile("cp.async.wait_all;" ::: "memory");
#ifdef TCM_VAR_FSTATS
    for (int k = 0; k < 16; ++k) atomicAdd(&g_fstats[k], (unsigned long long)s_fst[k][tid]);
#endif
    st.done_count = st.nxt - st.n_pend - st.n_dec;     // every arrived request is pending, decoding or done
#undef fS
#undef fp2
#undef fC2
#undef admit
#undef first
#undef fin
    {   // write back what the loop changes (tail[] and status are left as they are)
        ReplicaState& g = t.state[r];
        g.clock = st.clock;
        g.kv_free = st.kv_free;
        g.iter = st.iter;
        g.nxt = st.nxt;
        g.seq = st.seq;
        g.n_dec = st.n_dec;
        g.n_pend = st.n_pend;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            g.head[c] = st.head[c];
            g.rem[c] = st.rem[c];
        }
        g.flags = st.flags;
        g.max_pending = s_maxp[tid];
        g.decisions = s_dec[tid];
        g.sum_pending = s_sum[tid];
        g.ff_iters = s_ff[tid];
        g.idle_jumps = s_idle[tid];
        g.nlog = st.nlog;
        g.done_count = st.done_count;
        g.scanned = s_scan[tid];
    }
    if (!(st.flags & FLAG_FINISHED)) {
        atomicAdd(active, 1u);
        cal.flush();
#pragma unroll 8
        for (uint32_t k = 0; k < kCalWords; ++k) t.occ[(size_t)r * kCalWords + k] = cal.occ.word(k);
    }
}

// ---------------------------------------------------------------------------------------
// first_token_us and done_us from iteration numbers: the clock of iteration I is the entry I of
// the replica's event log (iterations strictly increasing; every iteration in which a prefill
// completed or a decode finished has one).  A first token is pending while first_token_us has
// bit 63 set; a finish while fin != 0, and it is due once the replica's iteration reaches it.
// One warp per replica, lanes over its requests.
__device__ __forceinline__ uint64_t log_clock(const uint64_t* log, uint32_t nlog, uint64_t it) {
    uint32_t lo = 0, hi = nlog;
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(log + 2 * mid) <= it) lo = mid;
        else hi = mid;
    }
    return __ldg(log + 2 * lo + 1);
}

// wpr warps per replica (1 for sweeps; more for a few huge queues so the stamping is not one warp)
__global__ void k_fstamp(TraceDev t, uint32_t wpr) {
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t r = gw / wpr;
    const uint32_t lane = (gw % wpr) * 32 + (threadIdx.x & 31);
    if (r >= t.R) return;
    const uint64_t a = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - a);
    const uint64_t iter = t.state[r].iter;
    const uint32_t nlog = t.state[r].nlog;
    const uint64_t* log = t.fw.log + 4 * a;
    for (uint32_t i = lane; i < n; i += 32 * wpr) {
        const uint64_t ft = t.first_token[a + i];
        if (ft & kPending) t.first_token[a + i] = log_clock(log, nlog, ft & ~kPending);
        const uint64_t F = t.fw.fin[a + i];
        if (F != 0 && F <= iter) {
            t.done[a + i] = log_clock(log, nlog, F);
            t.fw.fin[a + i] = 0;
        }
    }
}

#ifdef TCM_VAR_FSTATS
}  // namespace tcm
extern "C" int tcm_dev_fstats(unsigned long long* out, int reset) {
    cudaDeviceSynchronize();
    if (cudaMemcpyFromSymbol(out, tcm::g_fstats, sizeof(tcm::g_fstats)) != cudaSuccess) return -1;
    if (reset) {
        unsigned long long z[16] = {};
        cudaMemcpyToSymbol(tcm::g_fstats, z, sizeof(z));
    }
    return 0;
}
namespace tcm {
#endif

void launch_fused_prologue(const ModelConst& m, const TraceDev& t, cudaStream_t s) {
    const uint32_t threads = 256;
    const uint64_t blocks = ((uint64_t)t.R * 32 + threads - 1) / threads;
    k_fpack<<<(uint32_t)blocks, threads, 0, s>>>(m, t);
}

void launch_fgrow(const ModelConst& m, const TraceDev& t, uint32_t max_iters, uint32_t* d_active, uint32_t lpw,
                  cudaStream_t s);

void launch_fused(const ModelConst& m, const TraceDev& t, uint32_t max_iters, uint32_t* d_active,
                  cudaStream_t s) {
    // replicas per warp: the smallest power of two that keeps every replica in the resident warps
    static int cached_sms[64] = {}, cached_per_sm[64] = {};    // queried once per device
    static std::mutex mu;                   // contexts may run concurrently from several host threads
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    if (cached_sms[dev & 63] == 0) {
        int sms = 148, per_sm = 8;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_fused, kThreads, 0);
        cached_per_sm[dev & 63] = per_sm < 1 ? 1 : per_sm;
        cached_sms[dev & 63] = sms;
    }
    const uint64_t warps = (uint64_t)cached_sms[dev & 63] * cached_per_sm[dev & 63] * (kThreads / 32);
    uint32_t lpw = 1;
    while (lpw < 32 && (uint64_t)lpw * warps < t.R) lpw <<= 1;
    if (const char* f = getenv("TCM_FUSED_LPW")) {          // development A/B knob
        const int v = atoi(f);
        if (v >= 1 && v <= 32) lpw = (uint32_t)v;
    }
    const uint64_t nwarps = ((uint64_t)t.R + lpw - 1) / lpw;
    const uint32_t blocks = (uint32_t)((nwarps * 32 + kThreads - 1) / kThreads);
    if (!t.all_growth) k_fused<<<blocks, kThreads, 0, s>>>(m, t, max_iters, d_active, lpw);
    if (t.any_growth) launch_fgrow(m, t, max_iters, d_active, lpw, s);
}

void launch_fused_stamp(const TraceDev& t, cudaStream_t s) {
    const uint32_t threads = 256;
    const uint64_t avg = t.R ? t.N / t.R : 0;
    // few huge replicas (C2: one queue of 100k) spread over up to 512 warps each, ~512 requests per warp;
    // sweeps keep a warp per replica (<= 4,096 warps in all)
    uint32_t wpr = 1;
    while (wpr < 512 && (uint64_t)wpr * 512 < avg && (uint64_t)t.R * wpr * 2 <= 4096) wpr <<= 1;
    const uint64_t blocks = ((uint64_t)t.R * wpr * 32 + threads - 1) / threads;
    k_fstamp<<<(uint32_t)blocks, threads, 0, s>>>(t, wpr);
}

}  // namespace tcm
