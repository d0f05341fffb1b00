// tcm_fcal.cuh -- helpers shared by the fused engines (k_fused in tcm_fused.cu and its NEXT-1
// variant k_fgrow in tcm_fgrow.cu): record loads, the decode calendar, the event
// log, the exact K1 key of a class head.  Internal to libtcm.
#pragma once
#include "tcm_internal.cuh"
#include "tcm_k1.cuh"

namespace tcm {

constexpr uint32_t kFThreads = 64;       // threads per block of the fused engines

namespace {

constexpr uint64_t kCalFpMask = (1ull << kCalCntShift) - 1;
constexpr uint64_t kPending = 1ull << 63;

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

// (arrival, footprint) of a record
__device__ __forceinline__ void ld_arrfp(const FRec* p, uint64_t& arr, uint32_t& f) {
    uint64_t a, b;
    asm("ld.global.nc.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
    arr = a;
    f = (uint32_t)b;
}
// Asynchronous 16-byte copy global -> shared (its own commit group).  `dep` is an unused operand
// that makes the copy wait for a register (the value just read from the same shared slot).
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, uint64_t dep) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
#ifndef TCM_FUSED_CA
#define TCM_FUSED_CA 1
#endif
#if TCM_FUSED_CA
    // .ca: the record's sector also lands in L1, where ld_inl_id_out finds id / out later
    asm volatile("{\n\t.reg .b64 d;\n\tmov.b64 d, %2;\n\tcp.async.ca.shared.global [%0], [%1], 16;\n\t"
                 "cp.async.commit_group;\n\t}" ::"r"(sa), "l"(gmem), "l"(dep) : "memory");
#else
    asm volatile("{\n\t.reg .b64 d;\n\tmov.b64 d, %2;\n\tcp.async.cg.shared.global [%0], [%1], 16;\n\t"
                 "cp.async.commit_group;\n\t}" ::"r"(sa), "l"(gmem), "l"(dep) : "memory");
#endif
}
// Wait until at most `newer` of this thread's most recent copy groups are still in flight.
__device__ __forceinline__ void cp_async_wait(uint32_t newer) {
    if (newer == 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
    else if (newer == 1) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else if (newer == 2) asm volatile("cp.async.wait_group 2;" ::: "memory");
    else asm volatile("cp.async.wait_group 3;" ::: "memory");
}

// (inline, id, out) of a record, usually an L1 hit: its sector came in with ld_arrfp
// (two naturally aligned 8-byte loads: bytes 8..15 and 16..23 of the 32-byte record)
__device__ __forceinline__ void ld_inl_id_out(const FRec* p, uint32_t& inl, uint32_t& id, uint32_t& out) {
    uint32_t f;
    asm("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(f), "=r"(inl) : "l"(reinterpret_cast<const char*>(p) + 8));
    asm("ld.global.nc.v2.u32 {%0, %1}, [%2];" : "=r"(id), "=r"(out) : "l"(reinterpret_cast<const char*>(p) + 16));
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
    uint32_t (*w)[kFThreads];
    uint32_t tid;
    __device__ __forceinline__ uint32_t& word(uint32_t i) const { return w[i][tid]; }
};

__device__ __forceinline__ uint64_t ld_relaxed(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// The decode calendar of one replica.  Slot F & 2047 counts the requests whose last decode
// token comes in iteration F: (count << 40) | sum of their footprints.  The slot of the next
// event `next` is held in registers: `pre` (its memory value, loaded as soon as it becomes
// the next event, so the load overlaps the iterations before it) plus `add` (insertions into
// it since); other insertions go to memory as fire-and-forget reductions.
struct Calendar {
    uint64_t* cal;
    Occ occ;
    uint64_t sum;     // bit w: occupancy word w non-zero
    uint64_t next;    // iteration of the next event (~0: none)
    uint64_t pre, add;

    // Iteration of the next occupied slot after `iter` (one exists when n_dec > 0).
    __device__ __forceinline__ uint64_t scan(uint64_t iter) const {
        const uint32_t s0 = (uint32_t)((iter + 1) & (kCalSlots - 1));
        const uint32_t wi = s0 >> 5;
        uint32_t wv = occ.word(wi) & (~0u << (s0 & 31));
        uint32_t word = wi;
        if (wv == 0) {
            const uint64_t rr = rotr64(sum, wi + 1);      // bit k: word (wi + 1 + k) mod 64
            word = (wi + 1 + (uint32_t)(__ffsll((long long)rr) - 1)) & (kCalWords - 1);
            wv = occ.word(word);
            if (word == wi) wv &= ~(~0u << (s0 & 31));    // wrapped round to slots before s0
        }
        const uint32_t slot = word * 32 + (uint32_t)(__ffs(wv) - 1);
        return iter + 1 + (uint64_t)((slot - s0) & (kCalSlots - 1));
    }
    __device__ __forceinline__ void find_next(uint64_t iter, uint32_t n_dec) {
        add = 0;
        if (n_dec > 0) {
            next = scan(iter);
            pre = ld_relaxed(cal + (next & (kCalSlots - 1)));
        } else {
            next = ~0ull;
            pre = 0;
        }
    }
    // A request of footprint f whose last token comes in iteration F (> the current one).
    __device__ __forceinline__ void insert(uint64_t F, uint32_t f) {
        const uint64_t v = (1ull << kCalCntShift) | f;
        const uint32_t s = (uint32_t)(F & (kCalSlots - 1));
        occ.word(s >> 5) |= 1u << (s & 31);
        sum |= 1ull << (s >> 5);
        if (F == next) {
            add += v;
        } else if (F < next) {                         // F becomes the next event; slot F is empty
            if (add) red_add(cal + (next & (kCalSlots - 1)), add);
            next = F;
            pre = 0;
            add = v;
        } else {
            red_add(cal + s, v);
        }
    }
    // Step 9 for iteration `next`: every request whose last decode token is
    // produced now completes and releases its KV (R7).  k_fstamp stamps their done_us from the
    // event log.
    __device__ __forceinline__ void process(ReplicaState& st) {
        const uint32_t s = (uint32_t)(next & (kCalSlots - 1));
        const uint64_t v = pre + add;
        if (pre) st_relaxed(cal + s, 0);
        const uint32_t cnt = (uint32_t)(v >> kCalCntShift);
        st.kv_free += v & kCalFpMask;
        st.n_dec -= cnt;
        uint32_t& w = occ.word(s >> 5);
        w &= ~(1u << (s & 31));
        if (w == 0) sum &= ~(1ull << (s >> 5));
        find_next(st.iter, st.n_dec);
    }
    // A decoding request preempted before its finish F (> the current iteration) leaves the calendar:
    // v = (1 << 40) | what it would release at F (NEXT-1, k_fgrow).  The caller has already taken it
    // out of n_dec.
    __device__ __forceinline__ void remove(uint64_t F, uint64_t v, uint64_t iter, uint32_t n_dec) {
        const uint32_t s = (uint32_t)(F & (kCalSlots - 1));
        uint64_t rest;                                   // the slot's total without v
        if (F == next) {
            add -= v;
            rest = pre + add;
        } else {
            rest = (uint64_t)atomicAdd(reinterpret_cast<unsigned long long*>(cal + s), 0ull - v) - v;
        }
        if ((rest >> kCalCntShift) == 0) {               // the slot is empty now
            uint32_t& w = occ.word(s >> 5);
            w &= ~(1u << (s & 31));
            if (w == 0) sum &= ~(1ull << (s >> 5));
            if (F == next) {                             // the next event vanished
                if (pre) st_relaxed(cal + s, 0);
                find_next(iter, n_dec);
            }
        }
    }
    __device__ __forceinline__ void flush() {
        if (add) red_add(cal + (next & (kCalSlots - 1)), add);
    }
};

// One (iteration, clock) entry of the replica's event log: iterations in which a prefill
// completed or a decode finished, strictly increasing (k_fstamp looks them up).
__device__ __forceinline__ void log_event(uint64_t* log, ReplicaState& st) {
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(log + 2 * (uint64_t)st.nlog), "l"(st.iter),
                 "l"(st.clock) : "memory");
    st.nlog++;
}

template <class T>
__device__ __forceinline__ T sel3(int i, const T (&a)[3]) {
    return i == 0 ? a[0] : (i == 1 ? a[1] : a[2]);
}

// Exact K1 key of class c after waiting w, from the replica's class constants.  Out of line:
// the scan needs it only for heads whose FP32 bounds are within 2.5e-4, and one copy keeps the
// loop's code small.
__device__ __noinline__ uint64_t exact_key(const ClassPack* kp, int c, uint64_t w) {
    const K1Class kc{__ldg(&kp->S[c]), __ldg(&kp->p[c]), __ldg(&kp->C[c]), ((__ldg(&kp->zero_mask) >> c) & 1u) != 0};
    return k1_key(kc, w);
}

}  // namespace

}  // namespace tcm
