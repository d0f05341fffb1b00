// tcm_aux.cu -- libtcm's non-step kernels: replica init, trace validation, work-counter
// reduction, a6 aggregation (histograms + SLO counters), device trace generation, and the
// K1 evaluation / monotonicity audit.
#include "tcm_aux.cuh"
#include "tcm_k1.cuh"
#include "../../tracegen/tcm_tracegen.h"

namespace tcm {

// ---------------------------------------------------------------------------------------
// Initial replica state: clock 0, all KV free, empty queues (SPEC.md:455 start of run).
__global__ void k_init(TraceDev t) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= t.R) return;
    ReplicaState st{};
    st.clock = 0;
    st.kv_free = t.params[r].kv_capacity;
    st.iter = 0;
    st.nxt = 0;
    st.seq = 0;
    st.n_dec = 0;
    st.n_pend = 0;
    for (int c = 0; c < 3; ++c) {
        st.head[c] = NIL;
        st.tail[c] = 0;      // stepwise NEXT-1 counters (tcm_stats preemptions); unused by the fused engine
        st.rem[c] = 0;
    }
    st.flags = 0;
    st.status = ST_OK;
    st.max_pending = 0;
    st.decisions = 0;
    st.sum_pending = 0;
    st.ff_iters = 0;
    st.idle_jumps = 0;
    st.nlog = 0;
    st.done_count = 0;
    st.scanned = 0;
    t.state[r] = st;
}

// ---------------------------------------------------------------------------------------
// Per-replica K1 class constants (once per load).
__global__ void k_kpack(ModelConst m, TraceDev t) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= t.R) return;
    const double alpha = t.params[r].aging_alpha;
    ClassPack kp;
    kp.zero_mask = 0;
    kp.filter_ok = 1;
    for (int c = 0; c < 3; ++c) {
        const K1Class k = k1_class(m.S[c], m.k[c], m.p[c], alpha);
        kp.S[c] = k.S;
        kp.p[c] = k.p;
        kp.C[c] = k.C;
        kp.Smax[c] = k.zero ? k.S : __dadd_rn(k.S, 1.0);
        const double c2 = __dmul_rn(k.C, 1.4426950408889634);
        kp.fS[c] = (float)k.S;
        kp.fp2[c] = (float)k.p;
        kp.fC2[c] = (float)c2;
        if (k.zero) kp.zero_mask |= 1u << c;
        else if (!(k.p <= 16.0 && fabs(c2) <= 1000.0)) kp.filter_ok = 0;
        // saturation point: the least w in [1, 2^33] with K1(w) == K1 at the cap (bisection; monotone)
        const double smax = kp.Smax[c] < kEps ? kEps : kp.Smax[c];
        const uint64_t sk = (uint64_t)__double_as_longlong(smax);
        kp.satkey[c] = sk;
        if (k.zero) {
            kp.wsat[c] = 0;                          // P == S_c at every wait
        } else if (k1_key(k, 1ull << 33) != sk) {
            kp.wsat[c] = ~0ull;
        } else {
            uint64_t lo = 0, hi = 1ull << 33;        // key(lo) != sk (lo = 0: P = S_c < cap), key(hi) == sk
            while (hi - lo > 1) {
                const uint64_t mid = lo + ((hi - lo) >> 1);
                if (k1_key(k, mid) == sk) hi = mid;
                else lo = mid;
            }
            kp.wsat[c] = hi;
        }
    }
    kp.pad = 0;
    t.kpack[r] = kp;
}

// ---------------------------------------------------------------------------------------
// Validation: one warp per replica, lanes stride its requests (coalesced).
// v[0] = worst status code (max), v[1] = first bad replica (min).
__global__ void k_validate(TraceDev t, uint32_t* v, int general_ok) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= t.R) return;
    const uint32_t r = warp;
    const tcm_replica_params p = t.params[r];
    const uint64_t a = t.offset[r], b = t.offset[r + 1];
    uint32_t bad = ST_OK;
    if (b < a || b > t.N || b - a >= 0xFFFFFFFFull) bad = ST_BAD_INPUT;
    if (p.policy > TCM_POLICY_NAIVE_AGING || p.chunk_budget == 0 || p.kv_capacity == 0 ||
        p.kv_capacity > 0xFFFFFFFFull || !(p.aging_alpha >= 0.0) || (p.flags & ~(TCM_ADMIT_SKIP | TCM_KV_GROWTH)) != 0)
        bad = ST_BAD_INPUT;
    // EDF and first-fit admission break Lemmas L1/L2: only the stepwise engine runs them (TCM_KV_GROWTH
    // runs on both: the fused engine's k_fgrow)
    if (!general_ok && (p.policy == TCM_POLICY_EDF || (p.flags & TCM_ADMIT_SKIP))) bad = ST_BAD_INPUT;
    const bool growth = (p.flags & TCM_KV_GROWTH) != 0;
    // fused calendar slots count finishing requests in 24 bits
    if (!general_ok && b - a >= (1ull << (64 - kCalCntShift))) bad = ST_BAD_INPUT;
    if (bad == ST_OK) {
        for (uint64_t i = a + lane; i < b; i += 32) {
            const uint32_t f = t.footprint[i];
            const uint32_t o = t.out[i];
            if (f == 0 || o == 0 || o > kCalSlots || t.mod[i] > 2) bad = bad > ST_BAD_INPUT ? bad : ST_BAD_INPUT;
            if (i > a && t.arrival[i] < t.arrival[i - 1]) bad = bad > ST_BAD_INPUT ? bad : ST_BAD_INPUT;
            if ((uint64_t)f > p.kv_capacity) bad = ST_CAPACITY;
            if (growth && o >= 1 && (uint64_t)f + o - 1 > p.kv_capacity) bad = ST_CAPACITY;   // R28
        }
    }
    // ST_BAD_INPUT (2) vs ST_CAPACITY (3): report the larger code
    // bit 0: some replica grows; bit 1: some does not; bit 2: some replica is not plain TCM
    const bool plain_tcm = p.policy == TCM_POLICY_TCM && !(p.flags & TCM_ADMIT_SKIP);
    if (lane == 0) atomicOr(&v[2], (growth ? 1u : 2u) | (plain_tcm ? 0u : 4u));
    const uint32_t worst = __reduce_max_sync(0xFFFFFFFFu, bad);
    if (lane == 0 && worst != ST_OK) {
        atomicMax(&v[0], worst);
        atomicMin(&v[1], r);
    }
}

// ---------------------------------------------------------------------------------------
// Work counters: one thread per replica, warp-reduced, one atomic per warp and field.
__device__ __forceinline__ uint64_t warp_sum64(uint64_t x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, o);
    return x;
}

__global__ void k_reduce(TraceDev t, unsigned long long* acc /* [kAccN] */) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    ReplicaState st;
    bool live = r < t.R;
    uint64_t v[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t mx = 0;
    if (live) {
        st = t.state[r];
        v[0] = st.iter;
        v[1] = st.decisions;
        v[2] = st.ff_iters;
        v[3] = st.idle_jumps;
        v[4] = st.sum_pending;
        v[5] = st.done_count;
        v[6] = (st.flags & FLAG_FINISHED) ? 1 : 0;
        v[7] = (st.flags & FLAG_FINISHED) ? 0 : 1;
        v[8] = st.scanned;
        v[9] = st.tail[1];       // stepwise: preemptions (NEXT-1)
        v[10] = st.tail[2];      // stepwise: forced (motorcycle) preemptions
        mx = st.max_pending;
        if (st.status != ST_OK) {
            atomicMin(reinterpret_cast<unsigned long long*>(&acc[kAccBadReplica]), (unsigned long long)r);
            atomicMax(reinterpret_cast<unsigned long long*>(&acc[kAccBadStatus]), (unsigned long long)st.status);
        }
    }
#pragma unroll
    for (int k = 0; k < 11; ++k) v[k] = warp_sum64(v[k]);
    mx = __reduce_max_sync(0xFFFFFFFFu, mx);
    if ((threadIdx.x & 31) == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (v[k]) atomicAdd(&acc[k], (unsigned long long)v[k]);
        if (v[8]) atomicAdd(&acc[kAccScanned], (unsigned long long)v[8]);
        if (v[9]) atomicAdd(&acc[kAccPreempt], (unsigned long long)v[9]);
        if (v[10]) atomicAdd(&acc[kAccForced], (unsigned long long)v[10]);
        atomicMax(&acc[kAccMaxPending], (unsigned long long)mx);
    }
}

// Per-replica work counters (tcm_replica_counters): one thread per replica.
__global__ void k_replica_counters(TraceDev t, unsigned long long* out /* [R][kRepCnt] */) {
    const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= t.R) return;
    const ReplicaState st = t.state[r];
    unsigned long long* o = out + (size_t)r * kRepCnt;
    o[0] = st.iter;
    o[1] = st.decisions;
    o[2] = st.sum_pending;
    o[3] = st.scanned;
    o[4] = st.done_count;
    o[5] = st.tail[1];            // stepwise, TCM_KV_GROWTH: preemptions (0 otherwise)
}

// fig:preemptions per (cell, group): warp per replica, lanes over its requests; the class is the
// engine's own a1 classifier (classify(), R13); warp-reduced, one atomic per counter and replica.
__global__ void k_preempt_stats(ModelConst m, TraceDev t, unsigned long long* out /* [cells][4][3] */) {
    const uint32_t r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (r >= t.R) return;
    const uint64_t a = t.offset[r], b = t.offset[r + 1];
    unsigned long long v[kGroups - 1][3] = {};
    for (uint64_t i = a + lane; i < b; i += 32) {
        const uint32_t pc = t.pcount[i];
        if (pc == 0) continue;
        const int g = classify(m, t.mod[i], t.footprint[i]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (c == g) {
                v[c][0] += pc;
                v[c][1] += t.ptime[i];
                v[c][2] += 1;
            }
        }
    }
    unsigned long long* o = out + (size_t)t.params[r].cell_id * kGroups * 3;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            unsigned long long x = v[c][k];
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) x += __shfl_xor_sync(0xFFFFFFFFu, x, s);
            if (lane == 0 && x) {
                atomicAdd(o + c * 3 + k, x);
                atomicAdd(o + 3 * 3 + k, x);          // group "all"
            }
        }
    }
}

void launch_preempt_stats(const ModelConst& m, const TraceDev& t, unsigned long long* out, cudaStream_t s) {
    const uint64_t threads = (uint64_t)t.R * 32;
    k_preempt_stats<<<(uint32_t)((threads + 255) / 256), 256, 0, s>>>(m, t, out);
}

void launch_replica_counters(const TraceDev& t, unsigned long long* out, cudaStream_t s) {
    k_replica_counters<<<(t.R + 255) / 256, 256, 0, s>>>(t, out);
}

// ---------------------------------------------------------------------------------------
// a6 aggregation: warp per replica; per lane per-group
// counters, warp-reduced; histogram bins by atomics.
__device__ __forceinline__ uint32_t ttft_bucket(uint64_t t) {
    if (t < 16) return (uint32_t)t;
    const uint32_t e = 63u - (uint32_t)__clzll((long long)t);
    return 16u + 8u * (e - 4u) + (uint32_t)((t >> (e - 3u)) & 7u);
}

// A block aggregates a tile of kAggTile consecutive replicas: histogram bins are counted in
// shared-memory copies for the tile's first cell and the last replica's cell (two cells per tile: the C4
// layout pairs 16 FCFS with 16 TCM replicas) and flushed once; replicas of a third cell in the same
// tile fall back to global atomics.  Counters are warp-reduced per replica.
constexpr uint32_t kAggTile = 32;

__global__ void __launch_bounds__(256) k_aggregate(ModelConst m, TraceDev t, unsigned long long* hist,
                                                   unsigned long long* cnt) {
    __shared__ unsigned long long sh[2][kGroups * kHistBins];
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t r0 = blockIdx.x * kAggTile;
    if (r0 >= t.R) return;
    const uint32_t r1 = r0 + kAggTile < t.R ? r0 + kAggTile : t.R;
    const uint32_t cell0 = t.params[r0].cell_id;
    const uint32_t cell1 = t.params[r1 - 1].cell_id;
    for (uint32_t i = threadIdx.x; i < 2 * kGroups * kHistBins; i += blockDim.x) (&sh[0][0])[i] = 0;
    __syncthreads();
    for (uint32_t r = r0 + warp; r < r1; r += blockDim.x / 32) {
        const tcm_replica_params p = t.params[r];
        const uint64_t a = t.offset[r], b = t.offset[r + 1];
        const uint64_t B = p.chunk_budget;
        unsigned long long* H = p.cell_id == cell0 ? sh[0]
                                : (p.cell_id == cell1 ? sh[1] : hist + (size_t)p.cell_id * kGroups * kHistBins);
        uint64_t c[3][kNcnt];
#pragma unroll
        for (int g = 0; g < 3; ++g)
#pragma unroll
            for (int k = 0; k < (int)kNcnt; ++k) c[g][k] = 0;
        for (uint64_t i = a + lane; i < b; i += 32) {
            const uint32_t f = t.footprint[i];
            const uint32_t o = t.out[i];
            const int g = classify(m, t.mod[i], f);
            const uint64_t arr = t.arrival[i];
            const uint64_t ttft = t.first_token[i] - arr;
            const uint64_t e2e = t.done[i] - arr;
            const uint32_t B32 = (uint32_t)B;              // ceil(f / B) in 32-bit integer division
            const uint64_t nch = f / B32 + (f % B32 != 0);
            const uint64_t iso = (uint64_t)t.inl[i] + nch * m.c0 + m.cp * f + (uint64_t)(o - 1) * (m.c0 + m.cd);
            const uint64_t lhs = e2e * m.slo_den, rhs = iso * m.slo_num;
            const bool viol = lhs > rhs;
            const uint32_t bk = ttft_bucket(ttft);
            atomicAdd(&H[(size_t)g * kHistBins + bk], 1ull);
            atomicAdd(&H[(size_t)3 * kHistBins + bk], 1ull);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (q == g) {
                    c[q][0] += 1;
                    c[q][1] += ttft;
                    c[q][2] += e2e;
                    c[q][3] += viol ? 1 : 0;
                    c[q][4] += viol ? lhs - rhs : 0;
                    c[q][5] += e2e < (1ull << 32) ? (uint64_t)((uint32_t)e2e / o) : e2e / o;   // 32-bit when it fits
                }
            }
        }
        unsigned long long* C = cnt + (size_t)p.cell_id * kGroups * kNcnt;
#pragma unroll
        for (int k = 0; k < (int)kNcnt; ++k) {
            uint64_t all = 0;
#pragma unroll
            for (int g = 0; g < 3; ++g) {
                const uint64_t s = warp_sum64(c[g][k]);
                all += s;
                if (lane == 0 && s) atomicAdd(&C[g * kNcnt + k], (unsigned long long)s);
            }
            if (lane == 0 && all) atomicAdd(&C[3 * kNcnt + k], (unsigned long long)all);
        }
    }
    __syncthreads();
    unsigned long long* H0 = hist + (size_t)cell0 * kGroups * kHistBins;
    unsigned long long* H1 = hist + (size_t)cell1 * kGroups * kHistBins;
    for (uint32_t i = threadIdx.x; i < kGroups * kHistBins; i += blockDim.x) {
        if (sh[0][i]) atomicAdd(&H0[i], sh[0][i]);
        if (cell1 != cell0 && sh[1][i]) atomicAdd(&H1[i], sh[1][i]);
    }
}

// ---------------------------------------------------------------------------------------
// Device trace generation (bit-identical to tracegen/ on the host): warp per replica,
// 32 requests per round, gap prefix sum by warp scan, coalesced SoA stores.
__global__ void k_generate(const tg_replica* reps, uint32_t R, const uint64_t* off, uint64_t* arrival,
                           uint32_t* footprint, uint32_t* inl, uint16_t* out, uint8_t* mod, uint32_t* bad) {
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    if (warp >= R) return;
    const tg_replica rp = reps[warp];
    const uint64_t base = off[warp];
    if (off[warp + 1] - base != rp.n_requests) {
        if (lane == 0) atomicExch(bad, 1u);
        return;
    }
    uint64_t carry = 0;
    for (uint32_t i0 = 0; i0 < rp.n_requests; i0 += 32) {
        const uint32_t i = i0 + lane;
        tg_request q;
        uint64_t g = 0;
        if (i < rp.n_requests) {
            q = tg_draw(&rp, i);
            g = i == 0 ? 0 : q.gap_us;
        }
        uint64_t s = g;                                  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xFFFFFFFFu, s, o);
            if (lane >= (uint32_t)o) s += y;
        }
        if (i < rp.n_requests) {
            arrival[base + i] = carry + s;
            footprint[base + i] = q.footprint;
            inl[base + i] = q.inline_us;
            out[base + i] = q.out_tokens;
            mod[base + i] = q.modality;
        }
        carry += __shfl_sync(0xFFFFFFFFu, s, 31);
    }
}

// ---------------------------------------------------------------------------------------
// K1 diagnostics.
__global__ void k_k1_eval(ModelConst m, const uint8_t* cls, const uint64_t* w, const double* alpha,
                          double* outp, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int c = cls[i];
        const K1Class kc = k1_class(m.S[c], m.k[c], m.p[c], alpha[i]);
        outp[i] = k1_priority(kc, w[i]);
    }
}

// Each thread audits a contiguous chunk [w0, w0 + chunk] of adjacent pairs.
__global__ void k_k1_audit(ModelConst m, uint32_t c, double alpha, uint64_t lo, uint64_t hi, uint64_t chunk,
                           unsigned long long* first) {
    const K1Class kc = k1_class(m.S[c], m.k[c], m.p[c], alpha);
    const uint64_t nchunks = (hi - lo + chunk - 1) / chunk;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < nchunks;
         q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w0 = lo + q * chunk;
        uint64_t w1 = w0 + chunk;
        if (w1 > hi) w1 = hi;
        uint64_t prev = k1_key(kc, w0);
        for (uint64_t w = w0 + 1; w <= w1; ++w) {
            const uint64_t k = k1_key(kc, w);
            if (k < prev) {
                atomicMin(first, (unsigned long long)(w - 1));
                break;
            }
            prev = k;
        }
    }
}

// Max |P~ - P| of the FP32 filter bound over w in [lo, hi) (stepwise engine):
// non-negative doubles order like their bit patterns, so atomicMax on the bits is exact.
__global__ void k_filter_audit(ModelConst m, uint32_t c, double alpha, uint64_t lo, uint64_t hi, uint64_t step,
                               unsigned long long* maxerr) {
    const K1Class kc = k1_class(m.S[c], m.k[c], m.p[c], alpha);
    const float fS = (float)kc.S, fp2 = (float)kc.p, fC2 = (float)__dmul_rn(kc.C, 1.4426950408889634);
    double worst = 0.0;
    const uint64_t n = (hi - lo + step - 1) / step;
    for (uint64_t q = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; q < n; q += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t w = lo + q * step;
        if (w == 0 || kc.zero) continue;
        const double P = k1_priority(kc, w);
        const double Pf = (double)k1_filter_f32(fS, fp2, fC2, w);
        const double err = fabs(Pf - P);
        worst = err > worst ? err : worst;
    }
    atomicMax(maxerr, (unsigned long long)__double_as_longlong(worst));
}

// ---------------------------------------------------------------------------------------
void launch_filter_audit(const ModelConst& m, uint32_t c, double alpha, uint64_t lo, uint64_t hi, uint64_t step,
                         unsigned long long* maxerr, cudaStream_t s) {
    k_filter_audit<<<148 * 8, 256, 0, s>>>(m, c, alpha, lo, hi, step, maxerr);
}
void launch_kpack(const ModelConst& m, const TraceDev& t, cudaStream_t s) {
    k_kpack<<<(t.R + 127) / 128, 128, 0, s>>>(m, t);
}
void launch_init(const TraceDev& t, cudaStream_t s) {
    k_init<<<(t.R + 127) / 128, 128, 0, s>>>(t);
}
void launch_validate(const TraceDev& t, uint32_t* v, int general_ok, cudaStream_t s) {
    const uint64_t threads = (uint64_t)t.R * 32;
    k_validate<<<(uint32_t)((threads + 255) / 256), 256, 0, s>>>(t, v, general_ok);
}
void launch_reduce(const TraceDev& t, unsigned long long* acc, cudaStream_t s) {
    k_reduce<<<(t.R + 255) / 256, 256, 0, s>>>(t, acc);
}
__global__ void k_copy_words(const unsigned long long* src, unsigned long long* dst, int n) {
    if ((int)threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}
void launch_copy_words(const unsigned long long* src, unsigned long long* dst, int n, cudaStream_t s) {
    k_copy_words<<<1, 32, 0, s>>>(src, dst, n);
}
void launch_aggregate(const ModelConst& m, const TraceDev& t, unsigned long long* hist,
                      unsigned long long* cnt, cudaStream_t s) {
    k_aggregate<<<(t.R + kAggTile - 1) / kAggTile, 256, 0, s>>>(m, t, hist, cnt);
}
void launch_generate(const void* reps, uint32_t R, const uint64_t* off, uint64_t* arrival,
                     uint32_t* footprint, uint32_t* inl, uint16_t* out, uint8_t* mod, uint32_t* bad,
                     cudaStream_t s) {
    const uint64_t threads = (uint64_t)R * 32;
    k_generate<<<(uint32_t)((threads + 255) / 256), 256, 0, s>>>(
        reinterpret_cast<const tg_replica*>(reps), R, off, arrival, footprint, inl, out, mod, bad);
}
void launch_k1_eval(const ModelConst& m, const uint8_t* cls, const uint64_t* w, const double* alpha,
                    double* outp, uint64_t n, cudaStream_t s) {
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    if (blocks == 0) blocks = 1;
    k_k1_eval<<<(uint32_t)blocks, 256, 0, s>>>(m, cls, w, alpha, outp, n);
}
void launch_k1_audit(const ModelConst& m, uint32_t c, double alpha, uint64_t lo, uint64_t hi,
                     unsigned long long* first, cudaStream_t s) {
    const uint64_t chunk = 1024;
    uint64_t nchunks = (hi - lo + chunk - 1) / chunk;
    uint64_t blocks = (nchunks + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks == 0) blocks = 1;
    k_k1_audit<<<(uint32_t)blocks, 256, 0, s>>>(m, c, alpha, lo, hi, chunk, first);
}

}  // namespace tcm
