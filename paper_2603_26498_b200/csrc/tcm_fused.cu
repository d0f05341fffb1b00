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
#include "tcm_internal.cuh"
#include "tcm_k1.cuh"

namespace tcm {

namespace {

struct Cal {
    uint32_t* cal;
    uint32_t* occ;
};

__device__ __forceinline__ void cal_insert(const Cal& c, uint32_t* link, uint32_t slot, uint32_t i) {
    link[i] = c.cal[slot];
    c.cal[slot] = i;
    c.occ[slot >> 5] |= 1u << (slot & 31);
}

// Step 9 for iteration `iter`: every request whose last decode token is
// produced in this iteration completes now and releases its KV (R7).
__device__ __forceinline__ void cal_process(const Cal& c, uint32_t* link, uint64_t iter, uint64_t clock,
                                            const uint32_t* fp, uint64_t* done, ReplicaState& st) {
    const uint32_t s = (uint32_t)(iter & (kCalSlots - 1));
    const uint32_t bit = 1u << (s & 31);
    const uint32_t w = c.occ[s >> 5];
    if (!(w & bit)) return;
    uint32_t i = c.cal[s];
    while (i != NIL) {
        const uint32_t ni = link[i];
        done[i] = clock;
        st.kv_free += fp[i];
        st.n_dec--;
        st.done_count++;
        i = ni;
    }
    c.cal[s] = NIL;
    c.occ[s >> 5] = w & ~bit;
}

// Iteration number of the next occupied calendar slot after `iter` (one exists when n_dec > 0).
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

}  // namespace

__global__ void __launch_bounds__(64, 8) k_fused(ModelConst m, TraceDev t, uint32_t max_iters,
                                              uint32_t* active) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= t.R) return;
    ReplicaState st = t.state[r];
    if (st.flags & FLAG_FINISHED) return;

    const tcm_replica_params prm = t.params[r];
    const uint64_t base = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - base);
    const uint64_t* __restrict__ arr = t.arrival + base;
    const uint32_t* __restrict__ fp = t.footprint + base;
    const uint32_t* __restrict__ inl = t.inl + base;
    const uint16_t* __restrict__ out = t.out + base;
    const uint8_t* __restrict__ mod = t.mod + base;
    uint32_t* admit = t.admit_seq + base;
    uint64_t* first = t.first_token + base;
    uint64_t* done = t.done + base;
    uint32_t* link = t.link + base;
    const Cal cal{t.cal + (size_t)r * kCalSlots, t.occ + (size_t)r * kCalWords};

    const bool prio = prm.policy == TCM_POLICY_TCM;
    const uint32_t B = prm.chunk_budget;
    K1Class kc[3];
    float fS[3], fp2[3], fC2[3];
    bool use_bound = true;     // FP32 bound validated for these constants
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        kc[c] = k1_class(m.S[c], m.k[c], m.p[c], prm.aging_alpha);
        const double c2 = __dmul_rn(kc[c].C, 1.4426950408889634);
        fS[c] = (float)kc[c].S;
        fp2[c] = (float)kc[c].p;
        fC2[c] = (float)c2;
        if (!kc[c].zero && !(kc[c].p <= 16.0 && fabs(c2) <= 1000.0)) use_bound = false;
    }

    // Register caches: each class queue's head (arrival, footprint) and its successor
    // (id, arrival, footprint) so that advancing a queue never waits on memory; the next
    // decode-calendar event, so that iterations without a finish never touch the calendar.
    uint64_t harr[3], sarr[3];
    uint32_t hf[3], sid[3], sf[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        const uint32_t h = st.head[c];
        harr[c] = h != NIL ? arr[h] : 0;
        hf[c] = h != NIL ? fp[h] : 0;
        sid[c] = (h != NIL && h != st.tail[c]) ? link[h] : NIL;
        sarr[c] = sid[c] != NIL ? arr[sid[c]] : 0;
        sf[c] = sid[c] != NIL ? fp[sid[c]] : 0;
    }
    uint64_t next_arr = st.nxt < n ? arr[st.nxt] : ~0ull;
    uint64_t next_fin = st.n_dec > 0 ? cal_next(cal, st.iter) : ~0ull;
    uint32_t budget = max_iters;
    bool arm = false;     // the previous decision was blocked: try Lemma L4c once

    for (;;) {
        // ---- a1: ingest arrivals <= clock; classify; append to the class FIFO
        while (next_arr <= st.clock) {
            const uint32_t i = st.nxt;
            const uint32_t f = fp[i];
            const int q = prio ? classify(m, mod[i], f) : 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (c == q) {
                    if (st.head[c] == NIL) {
                        st.head[c] = i;
                        st.rem[c] = f;
                        st.flags &= ~(1u << c);
                        harr[c] = next_arr;
                        hf[c] = f;
                        sid[c] = NIL;
                    } else {
                        link[st.tail[c]] = i;
                        if (sid[c] == NIL) {               // head was alone: i is its successor
                            sid[c] = i;
                            sarr[c] = next_arr;
                            sf[c] = f;
                        }
                    }
                    st.tail[c] = i;
                }
            }
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
                cal_process(cal, link, st.iter, st.clock, fp, done, st);
                next_fin = st.n_dec > 0 ? cal_next(cal, st.iter) : ~0ull;
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
                if (st.head[c] != NIL && (((st.flags >> c) & 1u) || (uint64_t)hf[c] <= st.kv_free)) stuck = false;
        }
        // L4c: some head that does not fit ranks, *now*, above every head that fits even at the
        // start of the window's last iteration.  Priorities only grow with waiting time (L1), so
        // at every iteration of the window the top-ranked head misfits and blocks all admissions
        // (R6); with no partial (flags) nothing prefills.  FP32 bounds only (rigorous, 2.5e-4
        // margin); tried once after a blocked decision.
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
                zero_head |= st.head[c] != NIL && kc[c].zero;
                if (st.head[c] != NIL && !kc[c].zero && (uint64_t)hf[c] > st.kv_free) {
                    const float p = k1_filter_f32(fS[c], fp2[c], fC2[c], st.clock - harr[c]);
                    ptop = p > ptop ? p : ptop;
                }
            }
            // the longest window (halving from the full one) over which every fitting head stays
            // below the best misfitting head's priority now
            for (int h = 0; h < 6 && j >= 2 && !zero_head && ptop >= 0.0f; ++h, j >>= 1) {
                const uint64_t t_end = st.clock + (j - 1) * dt;
                float pfit = -1.0f;
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    if (st.head[c] != NIL && (uint64_t)hf[c] <= st.kv_free) {
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
                cal_process(cal, link, st.iter, st.clock, fp, done, st);
                next_fin = st.n_dec > 0 ? cal_next(cal, st.iter) : ~0ull;
            }
            arm = true;                                     // still blocked: try L4c again next
            continue;
        }

        // ---- a2 + a3 + a4: merge the class-FIFO heads by key, scan under token/KV budgets.
        // The scan advances the queue heads in place; oh[c] keeps each old head for the
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
            return (w == 0 || kc[c].zero || !use_bound) ? (float)kc[c].S : k1_filter_f32(fS[c], fp2[c], fC2[c], w);
        };
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            oh[c] = st.head[c];
            key[c] = 0;
            ex[c] = !prio;
            pf[c] = (prio && st.head[c] != NIL) ? bound(c, st.clock - harr[c]) : 0.0f;
        }
        while (left > 0) {
            int best = -1;
            uint64_t bk = 0, ba = 0;
            uint32_t bi = 0;
            float bpf = 0.0f;
            bool bex = true;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (st.head[c] != NIL && (!blocked || ((st.flags >> c) & 1u))) {
                    bool better = best < 0;
                    if (!better) {
                        const float d = pf[c] - bpf;
                        if (use_bound && d > 2.5e-4f) {
                            better = true;
                        } else if (use_bound && d < -2.5e-4f) {
                            better = false;
                        } else {
                            if (!ex[c]) {
                                key[c] = k1_key(kc[c], st.clock - harr[c]);
                                ex[c] = true;
                            }
                            if (!bex) {
#pragma unroll
                                for (int q = 0; q < c; ++q) {
                                    if (q == best) {
                                        key[q] = k1_key(kc[q], st.clock - harr[q]);
                                        ex[q] = true;
                                        bk = key[q];
                                    }
                                }
                                bex = true;
                            }
                            better = key[c] > bk ||
                                     (key[c] == bk && (harr[c] < ba || (harr[c] == ba && st.head[c] < bi)));
                        }
                    }
                    if (better) {
                        best = c;
                        bk = key[c];
                        bex = ex[c];
                        bpf = pf[c];
                        ba = harr[c];
                        bi = st.head[c];
                    }
                }
            }
            if (best < 0) break;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                if (c == best) {
                    const uint32_t i = st.head[c];
                    bool go = true;
                    if (!((st.flags >> c) & 1u)) {
                        if ((uint64_t)hf[c] > st.kv_free) {
                            blocked = true;                 // first misfit stops new admits
                            go = false;
                        } else {
                            st.kv_free -= hf[c];            // R7 reserve the full footprint
                            admit[i] = st.seq++;
                            inl_sum += inl[i];              // R10
                            st.flags |= 1u << c;
                        }
                    }
                    if (go) {
                        const uint32_t ch = st.rem[c] < left ? st.rem[c] : left;
                        st.rem[c] -= ch;
                        left -= ch;
                        tok += ch;
                        if (st.rem[c] == 0) {               // prefill complete: next in FIFO
                            st.flags &= ~(1u << c);
                            if (i == st.tail[c]) {
                                st.head[c] = NIL;
                                sid[c] = NIL;
                            } else {
                                const uint32_t ni = sid[c];    // prefetched successor
                                st.head[c] = ni;
                                harr[c] = sarr[c];
                                hf[c] = sf[c];
                                st.rem[c] = hf[c];
                                ex[c] = !prio;
                                if (prio) pf[c] = bound(c, st.clock - harr[c]);
                                sid[c] = ni != st.tail[c] ? link[ni] : NIL;
                                sarr[c] = sid[c] != NIL ? arr[sid[c]] : 0;
                                sf[c] = sid[c] != NIL ? fp[sid[c]] : 0;
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
            cal_process(cal, link, st.iter, st.clock, fp, done, st);
            recompute_fin = true;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            uint32_t i = oh[c];
            while (i != st.head[c]) {
                const uint32_t ni = (i == st.tail[c]) ? NIL : link[i];
                first[i] = st.clock;
                st.n_pend--;
                const uint32_t o = out[i];
                if (o == 1) {
                    done[i] = st.clock;
                    st.kv_free += fp[i];
                    st.done_count++;
                } else {
                    const uint64_t fin = st.iter + o - 1;
                    cal_insert(cal, link, (uint32_t)(fin & (kCalSlots - 1)), i);
                    st.n_dec++;
                    next_fin = fin < next_fin ? fin : next_fin;
                }
                i = ni;
            }
            if (st.head[c] == NIL) st.tail[c] = NIL;
        }
        if (recompute_fin) next_fin = st.n_dec > 0 ? cal_next(cal, st.iter) : ~0ull;
    }

    t.state[r] = st;
    if (!(st.flags & FLAG_FINISHED)) atomicAdd(active, 1u);
}

void launch_fused(const ModelConst& m, const TraceDev& t, uint32_t max_iters, uint32_t* d_active,
                  cudaStream_t s) {
    const uint32_t threads = 64;
    const uint32_t blocks = (t.R + threads - 1) / threads;
    k_fused<<<blocks, threads, 0, s>>>(m, t, max_iters, d_active);
}

}  // namespace tcm
