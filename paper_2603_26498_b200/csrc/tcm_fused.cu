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
// launch by k_fstamp from a per-replica log of (iteration, clock) finish events.
#include "tcm_internal.cuh"
#include "tcm_k1.cuh"

namespace tcm {

namespace {

constexpr uint32_t kThreads = 64;
constexpr uint64_t kCalFpMask = (1ull << kCalCntShift) - 1;

__device__ __forceinline__ void ld_rec(const FRec* p, uint64_t& arr, uint32_t& f, uint32_t& inl, uint32_t& id,
                                       uint32_t& out) {
    uint64_t a, b, c, d;
    asm("ld.global.nc.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    arr = a;
    f = (uint32_t)b;
    inl = (uint32_t)(b >> 32);
    id = (uint32_t)c;
    out = (uint32_t)(c >> 32);
}

__device__ __forceinline__ void red_add(uint64_t* p, uint64_t v) {
    asm volatile("red.relaxed.gpu.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint64_t rotr64(uint64_t x, uint32_t k) {
    k &= 63;
    return k ? (x >> k) | (x << (64 - k)) : x;
}

// Calendar occupancy: bit (slot & 31) of word (slot >> 5) in shared memory (column = thread),
// and `sum` bit w set iff word w is non-zero.
struct Occ {
    uint32_t (*w)[kThreads];
    uint32_t tid;
    __device__ __forceinline__ uint32_t& word(uint32_t i) const { return w[i][tid]; }
};

// Iteration number of the next occupied calendar slot after `iter` (one exists when n_dec > 0).
__device__ __forceinline__ uint64_t cal_next(const Occ& o, uint64_t sum, uint64_t iter) {
    const uint32_t s0 = (uint32_t)((iter + 1) & (kCalSlots - 1));
    const uint32_t wi = s0 >> 5;
    uint32_t wv = o.word(wi) & (~0u << (s0 & 31));
    uint32_t word = wi;
    if (wv == 0) {
        const uint64_t rr = rotr64(sum, wi + 1);      // bit k: word (wi + 1 + k) mod 64
        word = (wi + 1 + (uint32_t)(__ffsll((long long)rr) - 1)) & (kCalWords - 1);
        wv = o.word(word);
        if (word == wi) wv &= ~(~0u << (s0 & 31));    // wrapped round to slots before s0
    }
    const uint32_t slot = word * 32 + (uint32_t)(__ffs(wv) - 1);
    return iter + 1 + (uint64_t)((slot - s0) & (kCalSlots - 1));
}

// Step 9 for iteration `iter` == the next calendar event: every request whose
// last decode token is produced now completes and releases its KV (R7); the event goes to the
// log from which k_fstamp stamps their done_us.
__device__ __forceinline__ void cal_process(const Occ& o, uint64_t& sum, uint64_t* cal, uint64_t* log,
                                            ReplicaState& st) {
    const uint32_t s = (uint32_t)(st.iter & (kCalSlots - 1));
    const unsigned long long v = atomicExch(reinterpret_cast<unsigned long long*>(cal + s), 0ull);
    const uint32_t cnt = (uint32_t)(v >> kCalCntShift);
    st.kv_free += v & kCalFpMask;
    st.n_dec -= cnt;
    st.done_count += cnt;
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(log + 2 * (uint64_t)st.nlog), "l"(st.iter),
                 "l"(st.clock) : "memory");
    st.nlog++;
    uint32_t& w = o.word(s >> 5);
    w &= ~(1u << (s & 31));
    if (w == 0) sum &= ~(1ull << (s >> 5));
}

}  // namespace

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
    uint32_t run[3] = {0, cnt0, cnt0 + cnt1};
    FRec* rec = t.fw.rec + a;
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
    if (lane == 0) {
        ReplicaState& st = t.state[r];
        st.head[0] = 0;
        st.head[1] = cnt0;
        st.head[2] = cnt0 + cnt1;
        st.tail[0] = cnt0;                    // segment ends
        st.tail[1] = cnt0 + cnt1;
        st.tail[2] = n;
    }
}

__global__ void __launch_bounds__(kThreads, 8) k_fused(ModelConst m, TraceDev t, uint32_t max_iters,
                                                    uint32_t* active) {
    __shared__ uint32_t occ_s[kCalWords][kThreads];
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= t.R) return;
    ReplicaState st = t.state[r];
    if (st.flags & FLAG_FINISHED) return;

    const tcm_replica_params prm = t.params[r];
    const uint64_t base = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - base);
    const uint64_t* __restrict__ arr = t.arrival + base;
    const FRec* __restrict__ rec = t.fw.rec + base;
    uint32_t* admit = t.admit_seq + base;
    uint64_t* first = t.first_token + base;
    uint64_t* done = t.done + base;
    uint64_t* fin = t.fw.fin + base;
    uint64_t* cal = t.fw.cal + (size_t)r * kCalSlots;
    uint64_t* log = t.fw.log + 2 * base;
    const Occ occ{occ_s, threadIdx.x};
    uint64_t osum = 0;
#pragma unroll 8
    for (uint32_t k = 0; k < kCalWords; ++k) {
        const uint32_t w = t.occ[(size_t)r * kCalWords + k];
        occ.word(k) = w;
        osum |= (uint64_t)(w != 0) << k;
    }

    const bool prio = prm.policy == TCM_POLICY_TCM;
    const uint32_t B = prm.chunk_budget;
    const ClassPack* kp = t.kpack + r;
    float fS[3], fp2[3], fC2[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        fS[c] = kp->fS[c];
        fp2[c] = kp->fp2[c];
        fC2[c] = kp->fC2[c];
    }
    const uint32_t zmask = kp->zero_mask;
    const bool use_bound = kp->filter_ok != 0;   // FP32 bound validated for these constants
    auto exact_key = [&](int c, uint64_t w) -> uint64_t {
        const K1Class kc{__ldg(&kp->S[c]), __ldg(&kp->p[c]), __ldg(&kp->C[c]), ((zmask >> c) & 1u) != 0};
        return k1_key(kc, w);
    };

    // Register caches: each class queue's head record (arrival, footprint, inline, id) and its
    // successor's, so that advancing a queue never waits on memory.  An exhausted segment has
    // arrival ~0: a head is pending iff its arrival <= clock.  st.tail[c] is the end of class
    // c's segment.
    uint64_t harr[3], sarr[3];
    uint32_t hf[3], hinl[3], hid[3], sf[3], sinl[3], sid[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const uint32_t h = st.head[c];
        uint32_t o;
        harr[c] = ~0ull;
        hf[c] = hinl[c] = hid[c] = 0;
        sarr[c] = ~0ull;
        sf[c] = sinl[c] = sid[c] = 0;
        if (h < st.tail[c]) ld_rec(rec + h, harr[c], hf[c], hinl[c], hid[c], o);
        if (h + 1 < st.tail[c]) ld_rec(rec + h + 1, sarr[c], sf[c], sinl[c], sid[c], o);
    }
    uint64_t next_arr = st.nxt < n ? arr[st.nxt] : ~0ull;
    uint64_t next_fin = st.n_dec > 0 ? cal_next(occ, osum, st.iter) : ~0ull;
    uint32_t budget = max_iters;
    bool arm = false;     // the previous decision was blocked: try Lemma L4c once

    for (;;) {
        // ---- a1: arrivals <= clock join the pending set (their class queue already holds them)
        while (next_arr <= st.clock) {
            st.n_pend++;
            st.nxt++;
            next_arr = st.nxt < n ? arr[st.nxt] : ~0ull;
        }

        if (st.n_pend == 0) {
            if (st.n_dec == 0) {
                if (st.nxt == n) {                      // every request served
                    st.flags |= FLAG_FINISHED;
                    break;
                }
                st.clock = next_arr;                    // R15 idle jump (not an iteration)
                st.idle_jumps++;
                continue;
            }
            if (budget == 0) break;
            // ---- Lemma L3: decode-only iterations until the next finish or arrival
            const uint64_t F = next_fin;
            const uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint64_t j = F - st.iter;
            if (next_arr != ~0ull) {
                const uint64_t ja = (next_arr - st.clock + dt - 1) / dt;
                j = ja < j ? ja : j;
            }
            j = j < budget ? j : budget;
            st.clock += j * dt;
            st.iter += j;
            st.ff_iters += j;
            budget -= (uint32_t)j;
            if (st.iter == F) {
                cal_process(occ, osum, cal, log, st);
                next_fin = st.n_dec > 0 ? cal_next(occ, osum, st.iter) : ~0ull;
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
        // L4c: some head that does not fit ranks, *now*, above every head that fits even at the
        // start of the window's last iteration.  Priorities only grow with waiting time (L1), so
        // at every iteration of the window the top-ranked head misfits and blocks all admissions
        // (R6); with no partial (flags) nothing prefills.  FP32 bounds only (rigorous, 2.5e-4
        // margin); tried after a blocked decision, halving the window up to 6 times.
        uint64_t l4c_j = ~0ull;
        if (!stuck && arm && prio && use_bound && st.n_dec > 0 && (st.flags & 7u) == 0) {
            arm = false;
            const uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint64_t j = next_fin - st.iter;
            if (next_arr != ~0ull) {
                const uint64_t ja = (next_arr - st.clock + dt - 1) / dt;
                j = ja < j ? ja : j;
            }
            j = j < budget ? j : budget;
            bool zero_head = false;
            float ptop = -1.0f;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const bool pend = harr[c] <= st.clock;
                zero_head |= pend && ((zmask >> c) & 1u);
                if (pend && !((zmask >> c) & 1u) && (uint64_t)hf[c] > st.kv_free) {
                    const float p = k1_filter_f32(fS[c], fp2[c], fC2[c], st.clock - harr[c]);
                    ptop = p > ptop ? p : ptop;
                }
            }
            for (int h = 0; h < 6 && j >= 2 && !zero_head && ptop >= 0.0f; ++h, j >>= 1) {
                const uint64_t t_end = st.clock + (j - 1) * dt;
                float pfit = -1.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (harr[c] <= st.clock && (uint64_t)hf[c] <= st.kv_free) {
                        const float p = k1_filter_f32(fS[c], fp2[c], fC2[c], t_end - harr[c]);
                        pfit = p > pfit ? p : pfit;
                    }
                }
                if (ptop - pfit > 2.5e-4f) {
                    stuck = true;
                    l4c_j = j;
                    break;
                }
            }
        }
        if (stuck && st.n_dec > 0) {
            const uint64_t F = next_fin;
            const uint64_t dt = m.c0 + m.cd * st.n_dec;
            uint64_t j = F - st.iter;
            if (next_arr != ~0ull) {
                const uint64_t ja = (next_arr - st.clock + dt - 1) / dt;
                j = ja < j ? ja : j;
            }
            j = j < budget ? j : budget;
            j = j < l4c_j ? j : l4c_j;
            st.clock += j * dt;
            st.iter += j;
            st.decisions += j;
            st.sum_pending += j * st.n_pend;
            st.max_pending = st.n_pend > st.max_pending ? st.n_pend : st.max_pending;
            budget -= (uint32_t)j;
            if (st.iter == F) {
                cal_process(occ, osum, cal, log, st);
                next_fin = st.n_dec > 0 ? cal_next(occ, osum, st.iter) : ~0ull;
            }
            arm = true;                                     // still blocked: try L4c again next
            continue;
        }

        // ---- a2 + a3 + a4: merge the class-FIFO heads by key, scan under token/KV budgets.
        // The scan advances the queue cursors in place; oh[c] keeps each old head for the
        // first-token walk of a5.
        uint64_t tok = 0, inl_sum = 0;
        bool blocked = false;                               // R6
        uint32_t oh[3];
        uint64_t key[3];
        float pf[3];          // FP32 bound of each head's priority (|P~ - P| <= 1e-5)
        bool ex[3];           // ex[c]: key[c] holds the exact K1 key
        // Two heads whose bounds are more than 2.5e-4 apart are ordered by the bounds (the exact
        // order, since the bound error is < 1e-5); only closer pairs get their exact FP64 keys.
        auto bound = [&](int c, uint64_t w) -> float {
            return (w == 0 || ((zmask >> c) & 1u) || !use_bound) ? fS[c] : k1_filter_f32(fS[c], fp2[c], fC2[c], w);
        };
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            oh[c] = st.head[c];
            key[c] = 0;
            ex[c] = !prio;
            pf[c] = (prio && harr[c] <= st.clock) ? bound(c, st.clock - harr[c]) : 0.0f;
        }
        while (left > 0) {
            int best = -1;
            uint64_t bk = 0, ba = 0;
            uint32_t bi = 0;
            float bpf = 0.0f;
            bool bex = true;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (harr[c] <= st.clock && (!blocked || ((st.flags >> c) & 1u))) {
                    bool better = best < 0;
                    if (!better) {
                        const float d = pf[c] - bpf;
                        if (use_bound && d > 2.5e-4f) {
                            better = true;
                        } else if (use_bound && d < -2.5e-4f) {
                            better = false;
                        } else {
                            if (!ex[c]) {
                                key[c] = exact_key(c, st.clock - harr[c]);
                                ex[c] = true;
                            }
                            if (!bex) {
#pragma unroll
                                for (int q = 0; q < c; ++q) {
                                    if (q == best) {
                                        key[q] = exact_key(q, st.clock - harr[q]);
                                        ex[q] = true;
                                        bk = key[q];
                                    }
                                }
                                bex = true;
                            }
                            better = key[c] > bk ||
                                     (key[c] == bk && (harr[c] < ba || (harr[c] == ba && hid[c] < bi)));
                        }
                    }
                    if (better) {
                        best = c;
                        bk = key[c];
                        bex = ex[c];
                        bpf = pf[c];
                        ba = harr[c];
                        bi = hid[c];
                    }
                }
            }
            if (best < 0) break;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (c == best) {
                    bool go = true;
                    if (!((st.flags >> c) & 1u)) {
                        if ((uint64_t)hf[c] > st.kv_free) {
                            blocked = true;                 // first misfit stops new admits
                            go = false;
                        } else {
                            st.kv_free -= hf[c];            // R7 reserve the full footprint
                            admit[hid[c]] = st.seq++;
                            inl_sum += hinl[c];             // R10
                            st.flags |= 1u << c;
                            st.rem[c] = hf[c];
                        }
                    }
                    if (go) {
                        const uint32_t ch = st.rem[c] < left ? st.rem[c] : left;
                        st.rem[c] -= ch;
                        left -= ch;
                        tok += ch;
                        if (st.rem[c] == 0) {               // prefill complete: next in FIFO
                            st.flags &= ~(1u << c);
                            const uint32_t h = ++st.head[c];
                            harr[c] = sarr[c];
                            hf[c] = sf[c];
                            hinl[c] = sinl[c];
                            hid[c] = sid[c];
                            ex[c] = !prio;
                            if (prio && harr[c] <= st.clock) pf[c] = bound(c, st.clock - harr[c]);
                            sarr[c] = ~0ull;
                            if (h + 1 < st.tail[c]) {
                                uint32_t o;
                                ld_rec(rec + h + 1, sarr[c], sf[c], sinl[c], sid[c], o);
                            }
                        }
                    }
                }
            }
        }
        arm = tok == 0 && blocked;
        if (tok == 0 && st.n_dec == 0) {                    // unreachable under R6
            st.status = ST_DEADLOCK;
            st.flags |= FLAG_FINISHED;
            break;
        }

        // ---- a5: iteration cost, clock, decode calendar, first tokens (R12)
        st.clock += m.c0 + m.cp * tok + m.cd * (uint64_t)st.n_dec + inl_sum;
        st.iter++;
        st.decisions++;
        st.scanned++;
        st.sum_pending += st.n_pend;
        st.max_pending = st.n_pend > st.max_pending ? st.n_pend : st.max_pending;
        budget--;
        bool recompute_fin = false;
        if (st.iter == next_fin) {
            cal_process(occ, osum, cal, log, st);
            recompute_fin = true;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            for (uint32_t k = oh[c]; k < st.head[c]; ++k) {
                uint64_t a;
                uint32_t f, il, id, o;
                ld_rec(rec + k, a, f, il, id, o);
                first[id] = st.clock;
                st.n_pend--;
                if (o == 1) {
                    done[id] = st.clock;
                    st.kv_free += f;
                    st.done_count++;
                } else {
                    const uint64_t F = st.iter + o - 1;
                    const uint32_t s = (uint32_t)(F & (kCalSlots - 1));
                    red_add(cal + s, (1ull << kCalCntShift) | f);
                    occ.word(s >> 5) |= 1u << (s & 31);
                    osum |= 1ull << (s >> 5);
                    fin[id] = F;
                    st.n_dec++;
                    next_fin = F < next_fin ? F : next_fin;
                }
            }
        }
        if (recompute_fin) next_fin = st.n_dec > 0 ? cal_next(occ, osum, st.iter) : ~0ull;
    }

    t.state[r] = st;
    if (!(st.flags & FLAG_FINISHED)) {
        atomicAdd(active, 1u);
#pragma unroll 8
        for (uint32_t k = 0; k < kCalWords; ++k) t.occ[(size_t)r * kCalWords + k] = occ.word(k);
    }
}

// ---------------------------------------------------------------------------------------
// done_us of every request whose finish iteration F has been reached: the clock of the finish
// event F, looked up in the replica's event log (sorted by iteration).  One warp per replica,
// lanes over its requests.
__global__ void k_fstamp(TraceDev t) {
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (r >= t.R) return;
    const uint64_t a = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - a);
    const uint64_t iter = t.state[r].iter;
    const uint32_t nlog = t.state[r].nlog;
    const uint64_t* log = t.fw.log + 2 * a;
    for (uint32_t i = lane; i < n; i += 32) {
        const uint64_t F = t.fw.fin[a + i];
        if (F == 0 || F > iter) continue;
        uint32_t lo = 0, hi = nlog;                        // log[2k] strictly increasing
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (__ldg(log + 2 * mid) <= F) lo = mid;
            else hi = mid;
        }
        t.done[a + i] = __ldg(log + 2 * lo + 1);
        t.fw.fin[a + i] = 0;
    }
}

void launch_fused_prologue(const ModelConst& m, const TraceDev& t, cudaStream_t s) {
    const uint32_t threads = 256;
    const uint64_t blocks = ((uint64_t)t.R * 32 + threads - 1) / threads;
    k_fpack<<<(uint32_t)blocks, threads, 0, s>>>(m, t);
}

void launch_fused(const ModelConst& m, const TraceDev& t, uint32_t max_iters, uint32_t* d_active,
                  cudaStream_t s) {
    const uint32_t blocks = (t.R + kThreads - 1) / kThreads;
    k_fused<<<blocks, kThreads, 0, s>>>(m, t, max_iters, d_active);
}

void launch_fused_stamp(const TraceDev& t, cudaStream_t s) {
    const uint32_t threads = 256;
    const uint64_t blocks = ((uint64_t)t.R * 32 + threads - 1) / threads;
    k_fstamp<<<(uint32_t)blocks, threads, 0, s>>>(t);
}

}  // namespace tcm
