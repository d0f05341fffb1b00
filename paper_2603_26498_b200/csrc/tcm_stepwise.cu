// tcm_stepwise.cu -- TCM_ENGINE_STEPWISE: the paper-literal per-iteration scheduling step.
//
// Every engine iteration, for every active replica, one CTA:
//   a1  ingests arrivals <= clock (warp-parallel ballot over the sorted arrivals) and
//       classifies them (R13) into the per-request state byte;
//   a2  re-keys EVERY pending request of the replica's window [lo, nxt) with K1
//       ("At each scheduling iteration ... evaluates the state of all queues and dynamically
//       adjusts priorities") -- a coalesced, vectorised SoA stream of
//       arrival (8 B) + state (1 B) per request; the key is never written to memory;
//   a3  selects the top-32 candidates by (key desc, id asc) with per-warp register lists
//       merged by warp-shuffle bitonic networks (ballot skips batches that cannot enter);
//   a4  admits by warp-shuffle prefix scans of footprints against free KV and of chunk
//       tokens against the budget (R5-R8); if the scan has not terminated after 32
//       candidates it re-streams for the next 32 (threshold = last selected);
//   a5  advances the clock, stamps first tokens and runs the decode calendar (identical
//       integer arithmetic to the fused engine), with the decode-only fast-forward.
// Nothing here relies on Lemma L1, so any per-request key function fits this path.
#include "tcm_k1.cuh"
#include "tcm_stepwise.cuh"

namespace tcm {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTop = 32;
constexpr int kMaxPart = 32;
constexpr int kMaxDone = 1024;
constexpr uint32_t ST_PARTIAL_OVERFLOW = 4;

// request-state byte
constexpr uint8_t RS_CLS = 3, RS_PEND = 4, RS_RES = 8, RS_FT = 16;

struct Key {
    uint64_t k;
    uint32_t i;
};

__device__ __forceinline__ bool before(uint64_t ka, uint32_t ia, uint64_t kb, uint32_t ib) {
    return ka > kb || (ka == kb && ia < ib);
}

__device__ __forceinline__ void shfl_key(uint64_t& k, uint32_t& i, int lane_src_xor) {
    k = __shfl_xor_sync(0xFFFFFFFFu, k, lane_src_xor);
    i = __shfl_xor_sync(0xFFFFFFFFu, i, lane_src_xor);
}

// Bitonic sort of one element per lane, descending in (key, -id) across lanes 0..31.
__device__ __forceinline__ void warp_sort_desc(uint64_t& k, uint32_t& i, int lane) {
#pragma unroll
    for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
        for (int j = size >> 1; j > 0; j >>= 1) {
            uint64_t pk = k;
            uint32_t pi = i;
            shfl_key(pk, pi, j);
            const bool desc = (lane & size) == 0 || size == 32;
            const bool lower = (lane & j) == 0;
            const bool want_better = (lower == desc);
            const bool p_better = before(pk, pi, k, i);
            if (want_better ? p_better : before(k, i, pk, pi)) {
                k = pk;
                i = pi;
            }
        }
    }
}

// After element-wise max of a descending list and a reversed descending list, the 32
// values form a bitonic sequence holding the top 32; clean it into descending order.
__device__ __forceinline__ void warp_bitonic_clean_desc(uint64_t& k, uint32_t& i, int lane) {
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        uint64_t pk = k;
        uint32_t pi = i;
        shfl_key(pk, pi, j);
        const bool lower = (lane & j) == 0;
        if (lower ? before(pk, pi, k, i) : before(k, i, pk, pi)) {
            k = pk;
            i = pi;
        }
    }
}

// Merge a descending batch (bk, bi) into the descending list (lk, li): keeps the top 32.
__device__ __forceinline__ void warp_merge(uint64_t& lk, uint32_t& li, uint64_t bk, uint32_t bi, int lane) {
    const uint64_t rk = __shfl_sync(0xFFFFFFFFu, bk, 31 - lane);
    const uint32_t ri = __shfl_sync(0xFFFFFFFFu, bi, 31 - lane);
    if (before(rk, ri, lk, li)) {
        lk = rk;
        li = ri;
    }
    warp_bitonic_clean_desc(lk, li, lane);
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

struct Smem {
    double lnR[16], lnT[16], expT[16];
    uint64_t wkey[kWarps][kTop];
    uint32_t wid[kWarps][kTop];
    uint64_t partkey[kMaxPart];
    uint32_t part[kMaxPart];
    uint32_t done[kMaxDone];
    ReplicaState st;
    K1Class kc[3];
    uint64_t thk;       // continuation threshold (exclude ranks <= (thk, thi))
    uint64_t left, tok, inl;
    uint32_t thi;
    int npart, ndone, mode, pass_more, blocked, has_th;
};

}  // namespace

// Stage the replica's state at the start of a step (warp 0): ingest, idle jumps and the
// decode-only fast-forward.  mode: 0 nothing more this launch, 1 decision iteration.
__device__ void sw_prologue(const ModelConst& m, const TraceDev& t, uint32_t r, Smem& sm, int lane) {
    ReplicaState st = t.state[r];                      // every lane keeps a copy
    const uint64_t base = t.offset[r];
    const uint32_t n = (uint32_t)(t.offset[r + 1] - base);
    const uint64_t* arr = t.arrival + base;
    const uint32_t* fp = t.footprint + base;
    const uint8_t* mod = t.mod + base;
    uint8_t* rs = t.req_state + base;
    const bool prio = t.params[r].policy == TCM_POLICY_TCM;
    int mode = 0;
    if (!(st.flags & FLAG_FINISHED) && st.head[1] > 0) {
        const Cal cal{t.cal + (size_t)r * kCalSlots, t.occ + (size_t)r * kCalWords};
        for (;;) {
            // a1: ingest (ballot over the next 32 arrivals; arrivals are sorted)
            for (;;) {
                const uint32_t i = st.nxt + lane;
                const bool in = i < n && arr[i] <= st.clock;
                const uint32_t bal = __ballot_sync(0xFFFFFFFFu, in);
                if (in) {
                    const int c = prio ? classify(m, mod[i], fp[i]) : 0;
                    rs[i] = (uint8_t)(c | RS_PEND);
                }
                const uint32_t cnt = __popc(bal);
                st.nxt += cnt;
                st.n_pend += cnt;
                if (cnt < 32) break;
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
            // Lemma L3 decode-only fast-forward (same closed form as the fused engine)
            if (lane == 0) {
                const uint64_t F = cal_next(cal, st.iter);
                const uint64_t dt = m.c0 + m.cd * st.n_dec;
                uint64_t j = F - st.iter;
                if (st.nxt < n) {
                    const uint64_t ja = (arr[st.nxt] - st.clock + dt - 1) / dt;
                    j = ja < j ? ja : j;
                }
                j = j < st.head[1] ? j : st.head[1];
                st.clock += j * dt;
                st.iter += j;
                st.ff_iters += j;
                st.head[1] -= (uint32_t)j;
                if (st.iter == F) cal_process(cal, t.link + base, st.iter, st.clock, fp, t.done + base, st);
            }
            break;
        }
    }
    if (lane == 0) {
        sm.st = st;
        sm.mode = mode;
    }
}

__global__ void __launch_bounds__(kThreads) k_step(ModelConst m, TraceDev t, uint32_t* remv, uint32_t* active,
                                                   int count_active) {
    __shared__ Smem sm;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 16) {
        sm.lnR[tid] = kLnR[tid];
        sm.lnT[tid] = kLnT[tid];
        sm.expT[tid] = kExpT[tid];
    }
    __syncthreads();
    const K1Tables tb{sm.lnR, sm.lnT, sm.expT};

    for (uint32_t r = blockIdx.x; r < t.R; r += gridDim.x) {
        if (warp == 0) sw_prologue(m, t, r, sm, lane);
        __syncthreads();
        if (sm.mode == 0) {
            if (tid == 0) {
                t.state[r] = sm.st;
                if (count_active && !(sm.st.flags & FLAG_FINISHED)) atomicAdd(active, 1u);
            }
            __syncthreads();
            continue;
        }

        const tcm_replica_params prm = t.params[r];
        const bool prio = prm.policy == TCM_POLICY_TCM;
        const uint64_t base = t.offset[r];
        const uint64_t* arr = t.arrival + base;
        const uint32_t* fp = t.footprint + base;
        const uint32_t* inl = t.inl + base;
        const uint8_t* rsc = t.req_state + base;
        uint8_t* rs = t.req_state + base;
        uint32_t* rem = remv + base;
        const uint64_t clock = sm.st.clock;
        const uint32_t lo = sm.st.head[0], hi = sm.st.nxt;
        if (tid < 3) sm.kc[tid] = k1_class(m.S[tid], m.k[tid], m.p[tid], prm.aging_alpha);
        if (tid == 0) {
            const uint32_t B = prm.chunk_budget;
            sm.left = B > sm.st.n_dec ? B - sm.st.n_dec : 0;     // R8
            sm.tok = 0;
            sm.inl = 0;
            sm.blocked = 0;
            sm.has_th = 0;
            sm.npart = 0;
            sm.ndone = 0;
        }
        __syncthreads();
        K1Class kc[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) kc[c] = sm.kc[c];

        for (int pass = 0;; ++pass) {
            const bool first_pass = pass == 0;
            const bool has_th = sm.has_th;
            const uint64_t thk = sm.thk;
            const uint32_t thi = sm.thi;
            // ---- a2 + a3: stream the window, key, per-warp top-32
            uint64_t lk = 0;
            uint32_t li = NIL;
            uint64_t kk = 0;          // current 32nd of the warp list (broadcast)
            uint32_t ki = NIL;
            const int64_t gstart = (int64_t)((base + lo) & ~3ull) - (int64_t)base;   // 4-aligned (global)
            for (int64_t g0 = gstart + (int64_t)warp * 128; g0 < (int64_t)hi; g0 += kWarps * 128) {
                const int64_t e0 = g0 + 4 * lane;
                uint64_t a4[4];
                uint32_t s4 = 0;
                if (e0 >= 0 && e0 + 3 < (int64_t)hi) {
                    const ulonglong2 v0 = __ldg(reinterpret_cast<const ulonglong2*>(arr + e0));
                    const ulonglong2 v1 = __ldg(reinterpret_cast<const ulonglong2*>(arr + e0 + 2));
                    a4[0] = v0.x; a4[1] = v0.y; a4[2] = v1.x; a4[3] = v1.y;
                    s4 = *reinterpret_cast<const uint32_t*>(rsc + e0);
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int64_t e = e0 + j;
                        const bool ok = e >= (int64_t)lo && e < (int64_t)hi;
                        a4[j] = ok ? arr[e] : 0;
                        s4 |= (uint32_t)(ok ? rsc[e] : 0) << (8 * j);
                    }
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t e = e0 + j;
                    const uint32_t sb = (s4 >> (8 * j)) & 0xFF;
                    bool valid = e >= (int64_t)lo && e < (int64_t)hi && (sb & RS_PEND);
                    uint64_t key = 0;
                    const uint32_t id = (uint32_t)e;
                    if (valid && prio) {
                        const int c = sb & RS_CLS;
                        const K1Class kq = c == 0 ? kc[0] : (c == 1 ? kc[1] : kc[2]);   // registers
                        key = k1_key(kq, clock - a4[j], tb);
                    }
                    if (valid && first_pass && (sb & RS_RES)) {
                        const int slot = atomicAdd(&sm.npart, 1);
                        if (slot < kMaxPart) {
                            sm.part[slot] = id;
                            sm.partkey[slot] = key;
                        }
                    }
                    if (valid && has_th && !before(thk, thi, key, id)) valid = false;  // already ranked
                    const bool enter = valid && before(key, id, kk, ki);
                    if (__any_sync(0xFFFFFFFFu, enter)) {
                        uint64_t bk = enter ? key : 0;
                        uint32_t bi = enter ? id : NIL;
                        warp_sort_desc(bk, bi, lane);
                        warp_merge(lk, li, bk, bi, lane);
                        kk = __shfl_sync(0xFFFFFFFFu, lk, 31);
                        ki = __shfl_sync(0xFFFFFFFFu, li, 31);
                    }
                }
            }
            sm.wkey[warp][lane] = lk;
            sm.wid[warp][lane] = li;
            __syncthreads();

            // ---- a4: warp 0 merges the 8 lists and prefix-scans the admission
            if (warp == 0) {
#pragma unroll 1
                for (int w = 1; w < kWarps; ++w) warp_merge(lk, li, sm.wkey[w][lane], sm.wid[w][lane], lane);
                const bool valid = li != NIL;
                const uint32_t nvalid = __popc(__ballot_sync(0xFFFFFFFFu, valid));
                uint64_t left = sm.left;
                uint64_t kv = sm.st.kv_free;
                const bool blocked_prev = sm.blocked;
                uint32_t f = 0, rr = 0, il = 0;
                bool res = false;
                if (valid) {
                    f = fp[li];
                    res = (rsc[li] & RS_RES) != 0;
                    rr = res ? rem[li] : f;
                    il = res ? 0 : inl[li];
                }
                const bool waiting = valid && !res;
                const uint64_t cumf = warp_incl_scan64(waiting ? f : 0, lane);
                const bool kv_ok = waiting && !blocked_prev && cumf <= kv;
                const bool part = valid && (res || kv_ok);
                const uint64_t incl = warp_incl_scan64(part ? rr : 0, lane);
                const uint64_t excl = incl - (part ? rr : 0);
                const bool reached = excl < left;
                const uint64_t chunk = (part && reached) ? (rr < left - excl ? rr : left - excl) : 0;
                const bool admitted = kv_ok && reached;
                const bool misfit = waiting && !blocked_prev && !kv_ok && reached;
                const uint32_t adm_mask = __ballot_sync(0xFFFFFFFFu, admitted);
                const uint32_t rank = __popc(adm_mask & ((1u << lane) - 1));
                if (admitted) {
                    t.admit_seq[base + li] = sm.st.seq + rank;
                    rs[li] = (uint8_t)(rsc[li] | RS_RES);
                }
                if (chunk > 0) {
                    const uint32_t nr = rr - (uint32_t)chunk;
                    rem[li] = nr;
                    if (nr == 0) {
                        rs[li] = (uint8_t)(rs[li] | RS_FT);
                        const int d = atomicAdd(&sm.ndone, 1);
                        if (d < kMaxDone) sm.done[d] = li;
                    }
                }
                const uint64_t sum_chunk = warp_sum64(chunk);
                const uint64_t sum_f = warp_sum64(admitted ? f : 0);
                const uint64_t sum_inl = warp_sum64(admitted ? il : 0);
                const bool any_misfit = __any_sync(0xFFFFFFFFu, misfit);
                // threshold for a continuation pass = the last valid candidate of this batch
                const int lastl = nvalid > 0 ? (int)nvalid - 1 : 0;
                const uint64_t lastk = __shfl_sync(0xFFFFFFFFu, lk, lastl);
                const uint32_t lasti = __shfl_sync(0xFFFFFFFFu, li, lastl);
                if (lane == 0) {
                    sm.st.seq += __popc(adm_mask);
                    sm.st.kv_free = kv - sum_f;
                    sm.left = left - sum_chunk;
                    sm.tok += sum_chunk;
                    sm.inl += sum_inl;
                    if (any_misfit) sm.blocked = 1;
                    if (nvalid > 0) {
                        sm.thk = lastk;
                        sm.thi = lasti;
                        sm.has_th = 1;
                    }
                    // 1: budget left, nothing blocked, batch full -> next 32 candidates;
                    // 2: budget left but new admissions blocked (R6) -> only partials ranked
                    //    below this batch can still receive chunks.
                    sm.pass_more = 0;
                    if (sm.left > 0) sm.pass_more = sm.blocked ? 2 : (nvalid == kTop ? 1 : 0);
                    if (sm.npart > kMaxPart) sm.st.status = ST_PARTIAL_OVERFLOW;
                }
                __syncwarp();
                if (sm.pass_more == 2) {
                    const int np = sm.npart < kMaxPart ? sm.npart : kMaxPart;
                    uint64_t pk = 0;
                    uint32_t pi = NIL;
                    if (lane < np) {
                        pk = sm.partkey[lane];
                        pi = sm.part[lane];
                        if (sm.has_th && !before(sm.thk, sm.thi, pk, pi)) {   // already scanned
                            pk = 0;
                            pi = NIL;
                        }
                    }
                    warp_sort_desc(pk, pi, lane);
                    // serial walk in key order (<= 3 partials under Lemma L2)
                    for (int q = 0; q < np; ++q) {
                        const uint32_t id = __shfl_sync(0xFFFFFFFFu, pi, q);
                        if (id == NIL) break;
                        if (lane == 0 && sm.left > 0) {
                            const uint32_t rr2 = rem[id];
                            const uint64_t ch = rr2 < sm.left ? rr2 : sm.left;
                            rem[id] = rr2 - (uint32_t)ch;
                            sm.left -= ch;
                            sm.tok += ch;
                            if (rr2 == ch) {
                                rs[id] = (uint8_t)(rs[id] | RS_FT);
                                const int d = sm.ndone++;
                                if (d < kMaxDone) sm.done[d] = id;
                            }
                        }
                        __syncwarp();
                    }
                    if (lane == 0) sm.pass_more = 0;
                }
            }
            __syncthreads();
            if (sm.pass_more != 1) break;
        }

        // ---- a5: clock, calendar, first tokens (warp 0)
        if (warp == 0) {
            ReplicaState& st = sm.st;
            const uint64_t n_pend0 = st.n_pend;
            if (lane == 0) {
                if (sm.tok == 0 && st.n_dec == 0) {
                    st.status = ST_DEADLOCK;
                    st.flags |= FLAG_FINISHED;
                }
                st.clock += m.c0 + m.cp * sm.tok + m.cd * (uint64_t)st.n_dec + sm.inl;
                st.iter++;
                st.head[1]--;
                st.decisions++;
                st.sum_pending += n_pend0;
                st.max_pending = st.n_pend > st.max_pending ? st.n_pend : st.max_pending;
                const Cal cal{t.cal + (size_t)r * kCalSlots, t.occ + (size_t)r * kCalWords};
                cal_process(cal, t.link + base, st.iter, st.clock, fp, t.done + base, st);
            }
            __syncwarp();
            const uint64_t now = st.clock;
            const uint64_t it = st.iter;
            const int nd = sm.ndone;
            const uint16_t* out = t.out + base;
            uint32_t* cal = t.cal + (size_t)r * kCalSlots;
            uint32_t* occ = t.occ + (size_t)r * kCalWords;
            uint32_t* link = t.link + base;
            uint64_t kv_add = 0, n_dec_add = 0, done_add = 0;
            auto stamp = [&](uint32_t i) {
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
                for (int q = lane; q < nd; q += 32) stamp(sm.done[q]);
            } else {
                for (uint32_t i = lo + lane; i < hi; i += 32)
                    if (rs[i] & RS_FT) stamp(i);
            }
            __syncwarp();
            kv_add = warp_sum64(kv_add);
            n_dec_add = warp_sum64(n_dec_add);
            done_add = warp_sum64(done_add);
            if (lane == 0) {
                st.kv_free += kv_add;
                st.n_dec += (uint32_t)n_dec_add;
                st.done_count += (uint32_t)done_add;
                st.n_pend -= (uint32_t)(nd);
                uint32_t l2 = st.head[0];
                while (l2 < st.nxt && !(rs[l2] & RS_PEND)) ++l2;    // advance the window start
                st.head[0] = l2;
                t.state[r] = st;
                if (count_active && !(st.flags & FLAG_FINISHED)) atomicAdd(active, 1u);
            }
        }
        __syncthreads();
    }
}

// ReplicaState.head[0] = window start lo (oldest possibly-pending id), head[1] = remaining
// iteration budget of the current tcm_step call; the class-queue fields are unused here.
__global__ void k_sw_budget(TraceDev t, uint32_t budget) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < t.R) t.state[r].head[1] = budget;
}

__global__ void k_sw_init(TraceDev t) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < t.R) {
        t.state[r].head[0] = 0;
        t.state[r].head[1] = 0;
    }
}

void stepwise_init(const TraceDev& t, cudaStream_t s) { k_sw_init<<<(t.R + 255) / 256, 256, 0, s>>>(t); }

size_t stepwise_extra_bytes(uint32_t R, uint64_t N) { (void)R; return 4 * N + 16; }
size_t stepwise_workspace_bytes(uint32_t R, uint64_t N) { return N + stepwise_extra_bytes(R, N); }

StepwiseWorkspace stepwise_bind(void* p, uint32_t R) {
    StepwiseWorkspace w;
    w.base = p;
    w.R = R;
    return w;
}

int stepwise_grid(uint32_t R) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_step, kThreads, 0);
    if (per_sm < 1) per_sm = 1;
    const uint64_t g = (uint64_t)sms * per_sm;
    return (int)(R < g ? R : g);
}

tcm_status stepwise_run(const ModelConst& m, const TraceDev& t, const StepwiseWorkspace& w, uint32_t max_iters,
                        uint32_t* d_active, cudaStream_t s, uint64_t* launches) {
    uint32_t* remv = reinterpret_cast<uint32_t*>(w.base);
    const int grid = stepwise_grid(t.R);
    const uint32_t budget = max_iters;
    k_sw_budget<<<(t.R + 255) / 256, 256, 0, s>>>(t, budget);
    (*launches)++;
    // Each k_step launch advances every active replica by one iteration (or one fast-forward).
    // Launch in chunks; read the active count only at the end of each chunk.
    const uint32_t chunk = 64;
    uint64_t done_launches = 0;
    for (;;) {
        uint32_t this_chunk = chunk;
        if ((uint64_t)max_iters - done_launches < this_chunk) this_chunk = (uint32_t)(max_iters - done_launches);
        if (cudaMemsetAsync(d_active, 0, 4, s) != cudaSuccess) return TCM_E_CUDA;
        for (uint32_t q = 0; q < this_chunk; ++q) {
            k_step<<<grid, kThreads, 0, s>>>(m, t, remv, d_active, q + 1 == this_chunk);
            (*launches)++;
        }
        done_launches += this_chunk;
        if (cudaGetLastError() != cudaSuccess) return TCM_E_CUDA;
        uint32_t act = 0;
        if (cudaMemcpyAsync(&act, d_active, 4, cudaMemcpyDeviceToHost, s) != cudaSuccess) return TCM_E_CUDA;
        if (cudaStreamSynchronize(s) != cudaSuccess) return TCM_E_CUDA;
        if (act == 0 || done_launches >= max_iters) break;
    }
    return TCM_OK;
}

}  // namespace tcm
