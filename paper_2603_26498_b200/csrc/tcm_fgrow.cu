// tcm_fgrow.cu -- TCM_ENGINE_FUSED under TCM_KV_GROWTH (NEXT-1, readings R28-R32):
// the class-FIFO merge of k_fused with decode KV growth and preemption by recomputation, so that
// the memory-pressure sweep runs at sweep scale.
//
// One thread per replica, its state in registers, the requests in the class segments k_fpack
// writes (FCFS and naive aging: one segment in arrival order).  What growth changes:
//  * Lemma L1 still orders each class by arrival (aging keys are non-decreasing in the wait).  A
//    victim goes back to waiting with its original arrival (R30), and it is older than every
//    waiting request of its class: a running request was admitted while it was its class's head
//    (FIFO, R6 blocks behind a misfit), and victims are taken newest first within a class.  So
//    each class queue = a stack of waiting victims (top = oldest, it is the head) in front of the
//    segment cursor.
//  * The running requests of a class are its reserved head (a partial prefill, Lemma L2) and the
//    decoding requests at positions below the segment cursor, whose finish iteration (pfin) lies
//    ahead.  The newest running one -- the victim within its class (R29: FCFS takes the latest
//    arrival; TCM the last-ranked, and within a class that is the newest by L1) -- is the reserved
//    head if there is one, else the first position below the cursor that is still decoding.
//  * A decoding request holds its reservation plus one token per decode iteration (R28); it is
//    released at its finish iteration through the same calendar as k_fused, whose slots now carry
//    (count, sum of holdings at the finish).  A decoding victim is taken out of its slot.
//  * Only the decode-only window (Lemma L3) is taken in closed form, capped at kv_free / n_dec
//    iterations (each iteration charges n_dec tokens, R28); every iteration with a pending request
//    is scanned.  (L4/L5 assume constant holdings.)
// The order of one iteration is R32's: ingest -> preemptions -> kv_free -= n_dec -> merge/admission
// -> cost/clock -> decode tokens (finishing sequences release what they hold) -> completed prefills
// emit a token (the first one, or the next one after a re-prefill, R30).
#include "tcm_fcal.cuh"
#include "tcm_internal.cuh"
#include "tcm_k1.cuh"

namespace tcm {

namespace {

constexpr uint32_t kGThreads = kFThreads;
constexpr uint64_t kGPending = 1ull << 63;
constexpr uint8_t PF_EMIT = 1, PF_PREV = 2;

}  // namespace

__global__ void __launch_bounds__(kGThreads, 8) k_fgrow(ModelConst m, TraceDev t, uint32_t max_iters,
                                                       uint32_t* active, uint32_t lpw) {
    __shared__ uint32_t occ_s[kCalWords][kGThreads];
    __shared__ uint32_t s_top[3][kGThreads], s_hres[3][kGThreads], s_seg[3][kGThreads];
    __shared__ unsigned long long s_dec[kGThreads], s_sum[kGThreads], s_ff[kGThreads];
    __shared__ uint32_t s_maxp[kGThreads], s_pre[kGThreads], s_forced[kGThreads];
    const uint32_t gthread = blockIdx.x * blockDim.x + threadIdx.x;
    if ((gthread & 31) >= lpw) return;
    const uint32_t r = (gthread >> 5) * lpw + (gthread & 31);
    if (r >= t.R) return;
    const tcm_replica_params prm = t.params[r];
    if (!(prm.flags & TCM_KV_GROWTH)) return;           // k_fused runs the R7 replicas
    ReplicaState st = t.state[r];
    if (st.flags & FLAG_FINISHED) return;
    const uint32_t tid = threadIdx.x;
    s_dec[tid] = st.decisions;
    s_sum[tid] = st.sum_pending;
    s_ff[tid] = st.ff_iters;
    s_maxp[tid] = st.max_pending;
    s_pre[tid] = st.tail[1];
    s_forced[tid] = st.tail[2];
    uint32_t idle = st.idle_jumps, scanned = st.scanned;

    const uint64_t base = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - base);
    const uint64_t* __restrict__ arr = t.arrival + base;
    const uint64_t pb = base + 6ull * r;                 // first position of this replica
    const FRec* __restrict__ rec = t.fw.rec + pb;
    uint64_t* pfin = t.fg.pfin + pb;
    uint32_t* pkv = t.fg.pkv + pb;
    uint32_t* prem = t.fg.prem + pb;
    uint32_t* pgen = t.fg.pgen + pb;
    uint32_t* pnext = t.fg.pnext + pb;
    uint8_t* pflag = t.fg.pflag + pb;
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
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        s_top[c][tid] = t.fg.top[3 * r + c];
        s_seg[c][tid] = t.fg.seg[3 * r + c];
        s_hres[c][tid] = t.fg.hres[3 * r + c];
    }
    const bool prio = prm.policy == TCM_POLICY_TCM;
    const uint32_t B = prm.chunk_budget;
    const ClassPack* kp = t.kpack + r;
    // FP32 priority bounds for the TCM windows (|P~ - P| <= 1e-5), as in k_fused
    __shared__ float s_fc[3][3][kGThreads];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        s_fc[0][c][tid] = kp->fS[c];
        s_fc[1][c][tid] = kp->fp2[c];
        s_fc[2][c][tid] = kp->fC2[c];
    }
    const uint32_t zmask = kp->zero_mask;
    const bool use_bound = kp->filter_ok != 0;
    auto bound = [&](int c, uint64_t w) -> float {
        return (w == 0 || ((zmask >> c) & 1u) || !use_bound) ? s_fc[0][c][tid]
                                                              : k1_filter_f32(s_fc[0][c][tid], s_fc[1][c][tid], s_fc[2][c][tid], w);
    };

    // the head of class c: the top of its preempted stack, else the segment cursor.  hpos = its
    // position, harr its arrival (~0: none yet / exhausted), hneed the KV it reserves when admitted
    // (footprint, or for a victim what it held: R30)
    uint32_t hpos[3];
    uint64_t harr[3];
    uint32_t hneed[3];
    auto load_head = [&](int c) {
        const uint32_t tp = s_top[c][tid];
        const uint32_t p = tp != NIL ? tp : st.head[c];
        uint64_t a;
        uint32_t f;
        // the flag and the remainder are loaded with the record (positions are valid up to the
        // sentinels), so the three loads are in flight together
        const uint8_t fl = pflag[p];
        const uint32_t pr = prem[p];
        ld_arrfp(rec + p, a, f);
        hpos[c] = p;
        harr[c] = a;
        hneed[c] = (a != ~0ull && (fl & PF_PREV)) ? pr : f;
    };
#pragma unroll
    for (int c = 0; c < 3; ++c) load_head(c);
    uint64_t next_arr = st.nxt < n ? arr[st.nxt] : ~0ull;
    cal.find_next(st.iter, st.n_dec);
    uint32_t budget = max_iters;

    // R29's victim of class c: its newest running request, or NIL.  The reserved head is newer
    // than every decoding request of its class; otherwise scan down from the segment cursor.
    // Scan cache per class: every position in [s_kT, s_kH) below the cursor is known not to be
    // running (finished, or preempted and waiting).  A search scans the positions admitted since
    // (s_kH .. cursor), then continues below s_kT; a victim that is re-admitted and decodes again at a
    // position inside the known range shrinks it (see the scan).  Without it every preemption
    // re-walked the finished and preempted positions under the cursor (22 % of k_fgrow's instructions).
    __shared__ uint32_t s_kT[3][kGThreads], s_kH[3][kGThreads];
#pragma unroll
    for (int c = 0; c < 3; ++c) s_kT[c][tid] = s_kH[c][tid] = s_seg[c][tid];
    auto newest_running = [&](int c) -> uint32_t {
        if ((st.flags >> c) & 1u) return hpos[c];
        const uint32_t s0 = s_seg[c][tid];
        uint32_t found = NIL;
        for (uint32_t q = st.head[c]; q > s_kH[c][tid]; --q)
            if (pfin[q - 1] > st.iter) {
                found = q - 1;
                break;
            }
        if (found == NIL)
            for (uint32_t q = s_kT[c][tid]; q > s0; --q)
                if (pfin[q - 1] > st.iter) {
                    found = q - 1;
                    break;
                }
        s_kT[c][tid] = found == NIL ? s0 : found + 1;
        s_kH[c][tid] = st.head[c];
        return found;
    };

    for (;;) {
        // ---- a1: arrivals <= clock join the pending set
        while (next_arr <= st.clock) {
            st.n_pend++;
            st.nxt++;
            next_arr = st.nxt < n ? arr[st.nxt] : ~0ull;
        }
        if (st.n_pend == 0) {
            if (st.n_dec == 0) {
                if (st.nxt == n) {                          // every request served
                    st.flags |= FLAG_FINISHED;
                    break;
                }
                st.clock = next_arr;                        // R15 idle jump (not an iteration)
                idle++;
                continue;
            }
            if (budget == 0) break;
            // ---- Lemma L3 under growth: decode-only iterations until the next finish or arrival, while
            // every one of them finds its n_dec tokens free (R28); none left -> a full iteration preempts
            const uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint64_t j = cal.next - st.iter;
            if (next_arr != ~0ull) {
                const uint64_t ja = (next_arr - st.clock + dt - 1) / dt;
                j = ja < j ? ja : j;
            }
            j = j < budget ? j : budget;
            const uint64_t jk = st.kv_free / st.n_dec;
            j = j < jk ? j : jk;
            if (j > 0) {
                st.clock += j * dt;
                st.iter += j;
                st.kv_free -= j * st.n_dec;
                s_ff[tid] += j;
                budget -= (uint32_t)j;
                if (st.iter == cal.next) {
                    log_event(log, st);
                    cal.process(st);
                }
                continue;
            }
        }
        if (budget == 0) break;

        // ---- closed-form windows with pending requests (no preemption due: kv_free >= n_dec).  Each
        // iteration of a window charges n_dec decode tokens, so it lasts at most kv_free / n_dec
        // iterations (R28), and ends at the next finish or arrival.
        // FP32 bounds of the pending heads now, shared by L4c, L5 and (no preemption happens in a pass
        // whose window section ran: kv_free >= n_dec) the scan's ordering
        float pf[3];
        bool pf_ok = false;
        if (st.n_pend > 0 && st.kv_free >= st.n_dec) {
            const uint32_t left0 = B > st.n_dec ? B - st.n_dec : 0;   // R8
            const uint64_t kv_after = st.kv_free - st.n_dec;          // free KV once this iteration's tokens are charged
            uint64_t jcap = budget;
            if (st.n_dec > 0) {
                const uint64_t jk = st.kv_free / st.n_dec;
                jcap = jk < jcap ? jk : jcap;
                const uint64_t jf = cal.next - st.iter;
                jcap = jf < jcap ? jf : jcap;
            }
            // Lemma L4 under growth: nothing can prefill -- the decodes take the whole budget, or no head
            // is reserved (no partial, L2) and every pending head needs more than the free KV (the
            // top-ranked waiting request is a head, L1, and its misfit stops every admission, R6).  The
            // free KV only shrinks until the next finish, so that stays true.
            bool stuck = left0 == 0;
            if (!stuck && (st.flags & 7u) == 0) {
                stuck = true;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (harr[c] <= st.clock && (uint64_t)hneed[c] <= kv_after) stuck = false;
            }
            if (!stuck && prio) {
#pragma unroll
                for (int c = 0; c < 3; ++c) pf[c] = harr[c] <= st.clock ? bound(c, st.clock - harr[c]) : 0.0f;
                pf_ok = true;
            }
            uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint32_t tokj = 0;
            int tokc = 0;                                 // the class whose partial head takes the tokens
            if (next_arr != ~0ull) {
                const uint64_t ja = (next_arr - st.clock + dt - 1) / dt;
                jcap = ja < jcap ? ja : jcap;
            }
            // Lemma L4c under growth (TCM): a head that does not fit ranks, now, above every head that fits
            // even at the start of the window's last iteration -- priorities only grow (L1) and the fitting
            // set only shrinks as the free KV does -- so every iteration of the window is blocked (R6).  FP32
            // bounds with a 2.5e-4 margin; tried before every decision with a misfitting head and no partial.
            if (!stuck && prio && use_bound && st.n_dec > 0 && (st.flags & 7u) == 0) {
                uint64_t j = jcap;
                bool zero_head = false;
                float ptop = -1.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    const bool pend = harr[c] <= st.clock;
                    zero_head |= pend && ((zmask >> c) & 1u);
                    if (pend && !((zmask >> c) & 1u) && (uint64_t)hneed[c] > kv_after) {
                        const float pb = pf[c];
                        ptop = pb > ptop ? pb : ptop;
                    }
                }
                // as k_fused: the full window, then this decision alone (blocked: decided without the
                // scan), then halvings >= 2, the first success taken
                uint64_t cand = j, win = ~0ull;
                for (int step = 0; step < 7 && cand >= 1 && !zero_head && ptop >= 0.0f; ++step) {
                    const uint64_t t_end = st.clock + (cand - 1) * dt;
                    float pfit = -1.0f;
                    if (cand == 1) {             // the window's end is now: the pass's bounds
#pragma unroll
                        for (int c = 0; c < 3; ++c)
                            if (harr[c] <= st.clock && (uint64_t)hneed[c] <= kv_after) pfit = pf[c] > pfit ? pf[c] : pfit;
                    } else
#pragma unroll
                    for (int c = 0; c < 3; ++c) {
                        if (harr[c] <= st.clock && (uint64_t)hneed[c] <= kv_after) {
                            const float pb = bound(c, t_end - harr[c]);
                            pfit = pb > pfit ? pb : pfit;
                        }
                    }
                    const bool ok = ptop - pfit > 2.5e-4f;
                    if (step == 1) {
                        if (!ok) break;
                        win = 1;
                        cand = j >> 1;
                    } else {
                        if (ok) {
                            win = cand;
                            break;
                        }
                        cand = step == 0 ? (cand == 1 ? 0 : 1) : cand >> 1;
                    }
                    if (step >= 1 && cand < 2) break;
                }
                if (win != ~0ull) {
                    stuck = true;
                    jcap = win;
                }
            }
            // Lemma L5 under growth: a reserved (partial) head that needs more than this iteration's budget
            // and outranks every other head able to take tokens (partial, or waiting and fitting) takes the
            // whole budget while nothing else changes: no admission, no first token, n_dec fixed until the
            // next finish, the free KV only shrinking.  FCFS / naive aging: one queue, its head.  TCM: the
            // partial's FP32 bound now exceeds every other candidate's at the window's last iteration.
            if (!stuck && (st.flags & 7u) && left0 > 0 && (!prio || use_bound)) {
                int top = -1;
                float ptop = -1.0f;
                uint32_t cand = 0;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (harr[c] <= st.clock && (((st.flags >> c) & 1u) || (uint64_t)hneed[c] <= kv_after)) {
                        cand |= 1u << c;
                        const float pb = prio ? pf[c] : 0.0f;
                        if (top < 0 || pb > ptop) {
                            top = c;
                            ptop = pb;
                        }
                    }
                }
                uint32_t rt = 0;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (c == top) rt = ((st.flags >> c) & 1u) ? st.rem[c] : 0;
                if (rt > left0) {
                    const uint64_t dt5 = m.c0 + m.cp * left0 + m.cd * st.n_dec;
                    uint64_t j = (rt - 1) / left0;                     // rem stays > 0
                    j = jcap < j ? jcap : j;                           // budget, finish, kv / n_dec
                    if (next_arr != ~0ull) {
                        const uint64_t ja = (next_arr - st.clock + dt5 - 1) / dt5;
                        j = ja < j ? ja : j;
                    }
                    cand &= ~(1u << top);
                    bool ok = j >= 1;
                    if (prio && cand) {
                        ok = false;
                        for (int h = 0; h < 6 && j >= 1; ++h, j >>= 1) {
                            const uint64_t t_end = st.clock + (j - 1) * dt5;
                            float pmax = -1.0f;
                            if (j == 1) {
#pragma unroll
                                for (int c = 0; c < 3; ++c)
                                    if ((cand >> c) & 1u) pmax = pf[c] > pmax ? pf[c] : pmax;
                            } else
#pragma unroll
                            for (int c = 0; c < 3; ++c) {
                                if ((cand >> c) & 1u) {
                                    const float pb = bound(c, t_end - harr[c]);
                                    pmax = pb > pmax ? pb : pmax;
                                }
                            }
                            if (ptop - pmax > 2.5e-4f) {
                                ok = true;
                                break;
                            }
                        }
                    }
                    if (ok) {
                        stuck = true;
                        jcap = j;
                        dt = dt5;
                        tokj = left0;
                        tokc = top;
                    }
                }
            }
            if (stuck && jcap >= 1 && !(st.n_dec == 0 && tokj == 0)) {
                const uint64_t j = jcap;
                st.clock += j * dt;
                st.iter += j;
                st.kv_free -= j * st.n_dec;
#pragma unroll
                for (int c = 0; c < 3; ++c)
                    if (c == tokc) st.rem[c] -= (uint32_t)(j * tokj);
                s_dec[tid] += j;
                s_sum[tid] += j * st.n_pend;
                s_maxp[tid] = st.n_pend > s_maxp[tid] ? st.n_pend : s_maxp[tid];
                budget -= (uint32_t)j;
                if (st.iter == cal.next) {
                    log_event(log, st);
                    cal.process(st);
                }
                continue;
            }
        }

        // ---- R29: memory exhaustion -- preempt until this iteration's decode tokens fit
        while (st.kv_free < st.n_dec) {
            int vc = -1;
            uint32_t v = NIL;
            bool forced = false;
            if (prio) {
                // the running non-motorcycle ranked last by (P desc, arrival asc, id asc); motorcycles
                // only when no other class runs.  Within a class that is its newest running request (L1)
                uint64_t vk = 0, va = 0;
                uint32_t vid = 0;
                for (int c = 1; c < 3; ++c) {
                    const uint32_t q = newest_running(c);
                    if (q == NIL) continue;
                    uint32_t il, id, o;
                    ld_inl_id_out(rec + q, il, id, o);
                    const uint64_t a = rec[q].arrival;
                    const uint64_t k = exact_key(kp, c, st.clock - a);
                    if (vc < 0 || k < vk || (k == vk && (a > va || (a == va && id > vid)))) {
                        vc = c;
                        v = q;
                        vk = k;
                        va = a;
                        vid = id;
                    }
                }
                if (vc < 0) {
                    v = newest_running(0);
                    vc = 0;
                    forced = true;
                }
            } else {
                v = newest_running(0);                      // FCFS / naive aging: the latest arrival
                vc = 0;
            }
            if (v == NIL) {                                 // unreachable: n_dec > 0
                t.state[r].status = ST_DEADLOCK;
                st.flags |= FLAG_FINISHED;
                break;
            }
            uint32_t il, id, o;
            ld_inl_id_out(rec + v, il, id, o);
            uint32_t held;
            if (((st.flags >> vc) & 1u) && hpos[vc] == v) {   // the reserved head: a partial prefill
                held = s_hres[vc][tid];
                st.flags &= ~(1u << vc);
                hneed[vc] = held;                            // it stays the head, waiting (R30)
            } else {                                         // a decoding request
                const uint64_t F = pfin[v];
                const uint32_t kvF = pkv[v];
                const uint32_t togo = (uint32_t)(F - st.iter);
                held = kvF - togo;
                pgen[v] = o - togo;
                pfin[v] = 0;
                fin(id) = 0;
                st.n_dec--;
                st.n_pend++;
                cal.remove(F, (1ull << kCalCntShift) | kvF, st.iter, st.n_dec);
                prem[v] = held;
                pnext[v] = s_top[vc][tid];                   // older than every waiting request of its class
                s_top[vc][tid] = v;
                load_head(vc);
            }
            prem[v] = held;
            st.kv_free += held;
            t.pcount[base + id]++;
            t.pstart[base + id] = st.clock;
            s_pre[tid]++;
            if (forced) s_forced[tid]++;
        }
        if (st.flags & FLAG_FINISHED) break;
        st.kv_free -= st.n_dec;                             // R28/R32: this iteration's decode tokens
        uint32_t left = B > st.n_dec ? B - st.n_dec : 0;   // R8

        // ---- a2 + a3 + a4: merge the class heads by key, scan under token / KV budgets (as k_fused)
        uint64_t tok = 0, inl_sum = 0, kv_rel = 0;
        uint32_t ncomp = 0, new_dec = 0, nlogged = 0;      // nlogged: first tokens and finishes now
        const uint64_t it1 = st.iter + 1;
        const uint32_t npend = st.n_pend;                   // the pending set this decision orders (R17)
        bool blocked = false;
        uint64_t key[3];
        bool ex[3];
        // bound-first ordering as in k_fused: heads whose FP32 bounds differ by more than 2.5e-4 are
        // ordered by them (|P~ - P| < 1e-5), closer pairs by the exact keys
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            key[c] = 0;
            ex[c] = !prio;
            if (!pf_ok) pf[c] = (prio && harr[c] <= st.clock) ? bound(c, st.clock - harr[c]) : 0.0f;
        }
        while (left > 0) {
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
                                         uint32_t i1, i2, x, y;   // equal key and arrival: id order (R4)
                                         ld_inl_id_out(rec + hpos[c], x, i1, y);
                                         ld_inl_id_out(rec + sel3(best, hpos), x, i2, y);
                                         return i1 < i2;
                                     }())));
                        }
                    }
                    if (better) best = c;
                }
            }
            if (best < 0) break;
            const uint32_t p = sel3(best, hpos);
            uint32_t remb = sel3(best, st.rem);
            bool go = true, adv = false;
            uint32_t il, id, o;
            ld_inl_id_out(rec + p, il, id, o);
            if (!((st.flags >> best) & 1u)) {
                const uint32_t need = sel3(best, hneed);
                if ((uint64_t)need > st.kv_free) {
                    blocked = true;                         // R6: the first misfit stops new admissions
                    go = false;
                } else {
                    st.kv_free -= need;                     // reserve (R7; a victim: what it held, R30)
                    const uint8_t pf = pflag[p];
                    if (!(pf & PF_PREV)) {
                        admit(id) = st.seq++;
                        inl_sum += il;                      // R10: inline time on the first admission only
                        pgen[p] = 0;
                        pflag[p] = pf | PF_PREV;
                    } else {
                        t.ptime[base + id] += st.clock - t.pstart[base + id];   // R31
                    }
                    s_hres[best][tid] = need;
                    st.flags |= 1u << best;
                    remb = need;
                }
            }
            if (go) {
                const uint32_t ch = remb < left ? remb : left;
                remb -= ch;
                left -= ch;
                tok += ch;
                if (remb == 0) {                            // prefill complete: the request emits a token
                    const uint8_t pf = pflag[p];
                    if (!(pf & PF_EMIT)) {
                        first(id) = kGPending | it1;        // stamped by k_fstamp (R12)
                        pflag[p] = pf | PF_EMIT;
                        nlogged++;
                    }
                    const uint32_t gen = pgen[p] + 1;
                    const uint32_t res = s_hres[best][tid];
                    ncomp++;
                    if (gen >= o) {                         // done with this token
                        fin(id) = it1;
                        kv_rel += res;
                        pfin[p] = 0;
                        nlogged++;
                    } else {                                // decodes until iteration it1 + (out - gen)
                        const uint64_t F = it1 + (o - gen);
                        const uint32_t kvF = res + (o - gen);
                        fin(id) = F;
                        pfin[p] = F;
#pragma unroll
                        for (int c = 0; c < 3; ++c)      // running again inside a known-idle range
                            if (c == best && p >= s_kT[c][tid] && p < s_kH[c][tid]) s_kT[c][tid] = p + 1;
                        pkv[p] = kvF;
                        cal.insert(F, kvF);
                        new_dec++;
                    }
                    st.flags &= ~(1u << best);
                    adv = true;
                }
            }
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (c == best) {
                    st.rem[c] = remb;
                    if (adv) {
                        const uint32_t tp = s_top[c][tid];
                        if (tp == p) s_top[c][tid] = pnext[p];   // pop the stack
                        else st.head[c]++;                       // advance the segment cursor
                        load_head(c);
                        ex[c] = !prio;
                        pf[c] = (prio && harr[c] <= st.clock) ? bound(c, st.clock - harr[c]) : 0.0f;
                    }
                }
            }
        }
        if (tok == 0 && st.n_dec == 0) {                   // unreachable under R6
            t.state[r].status = ST_DEADLOCK;
            st.flags |= FLAG_FINISHED;
            break;
        }
        // ---- a5: cost, clock, decode tokens of this iteration (the calendar), first tokens
        st.clock += m.c0 + m.cp * tok + m.cd * (uint64_t)st.n_dec + inl_sum;
        st.iter = it1;
        if (npend > 0) {                                    // R17
            s_dec[tid] += 1;
            s_sum[tid] += npend;
            s_maxp[tid] = npend > s_maxp[tid] ? npend : s_maxp[tid];
            scanned++;
        }
        budget--;
        st.n_pend -= ncomp;
        st.kv_free += kv_rel;
        st.n_dec += new_dec;
        const bool event = it1 == cal.next;
        // the log holds every iteration with a first token or a finish (k_fstamp looks them up):
        // at most one of each per request, so it never exceeds its 2 entries per request
        if (nlogged > 0 || event) log_event(log, st);
        if (event) cal.process(st);                         // finishing sequences release (R28)
    }
#undef admit
#undef first
#undef fin
    st.done_count = st.nxt - st.n_pend - st.n_dec;
    {
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
            t.fg.top[3 * r + c] = s_top[c][tid];
            t.fg.hres[3 * r + c] = s_hres[c][tid];
        }
        g.tail[1] = s_pre[tid];
        g.tail[2] = s_forced[tid];
        g.flags = st.flags;
        g.max_pending = s_maxp[tid];
        g.decisions = s_dec[tid];
        g.sum_pending = s_sum[tid];
        g.ff_iters = s_ff[tid];
        g.idle_jumps = idle;
        g.nlog = st.nlog;
        g.done_count = st.done_count;
        g.scanned = scanned;
    }
    if (!(st.flags & FLAG_FINISHED)) {
        atomicAdd(active, 1u);
        cal.flush();
#pragma unroll 8
        for (uint32_t k = 0; k < kCalWords; ++k) t.occ[(size_t)r * kCalWords + k] = cal.occ.word(k);
    }
}

void launch_fgrow(const ModelConst& m, const TraceDev& t, uint32_t max_iters, uint32_t* d_active, uint32_t lpw,
                  cudaStream_t s) {
    const uint64_t nwarps = ((uint64_t)t.R + lpw - 1) / lpw;
    const uint32_t blocks = (uint32_t)((nwarps * 32 + kGThreads - 1) / kGThreads);
    k_fgrow<<<blocks, kGThreads, 0, s>>>(m, t, max_iters, d_active, lpw);
}

}  // namespace tcm
