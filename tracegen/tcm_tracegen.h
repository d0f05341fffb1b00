/*
 * tcm_tracegen.h -- seeded synthetic trace generator (input module).
 *
 * This is the ONE module both the oracle tests and the CUDA path use: it draws the
 * inputs (arrivals, modality, token counts, encode cost, output length) and holds
 * none of the scheduling method's arithmetic.  It compiles for the host (gcc,
 * -ffp-contract=off) and for the device (nvcc); every floating-point operation goes
 * through TG_MUL/TG_ADD/TG_DIV/TG_SQRT, which are the correctly-rounded IEEE
 * operations on both sides, so host and device produce bit-identical traces.
 *
 * Workload recipe:
 *   per replica seed = splitmix64(base ^ replica); Philox4x32-10 keyed by the seed,
 *   counter = (request, block, 0, 0);
 *   arrivals: Poisson, exponential gaps at rate lambda, gap_us = floor(-ln U * 1e6/lambda),
 *             arrival_0 = 0, arrival_i = arrival_{i-1} + gap_us(i)
 *   modality: categorical from the (text, image, video) mix (R20)
 *   text:  prompt ~ LN(median 200, sigma 1.0) clipped [10, 1e4]
 *   image: prompt ~ LN(50, 0.5) in [1, 512]; media 729 + U{-64..64}
 *          inline_us = 130000 + 40000 * MP, MP ~ U[0.25, 4)
 *   video: prompt ~ LN(50, 0.5) in [1, 512]; frames ~ U{8..512} clamped to fit KV;
 *          media = 196 * frames; inline_us = 300000 + 16000 * frames
 *   output: LN(128, 0.8) in [1, 2048] for every modality (R23)
 *   every footprint is clamped to <= kv_capacity (R18).
 */
#ifndef TCM_TRACEGEN_H
#define TCM_TRACEGEN_H

#include <stdint.h>

#if defined(__CUDACC__)
#define TG_HD __host__ __device__ __forceinline__
#else
#define TG_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define TG_MUL(a, b) __dmul_rn((a), (b))
#define TG_ADD(a, b) __dadd_rn((a), (b))
#define TG_SUB(a, b) __dsub_rn((a), (b))
#define TG_DIV(a, b) __ddiv_rn((a), (b))
#define TG_SQRT(a) __dsqrt_rn((a))
#define TG_BITS(d) ((uint64_t)__double_as_longlong(d))
#define TG_FROMBITS(b) __longlong_as_double((long long)(b))
#else
#include <math.h>
#include <string.h>
#define TG_MUL(a, b) ((a) * (b))
#define TG_ADD(a, b) ((a) + (b))
#define TG_SUB(a, b) ((a) - (b))
#define TG_DIV(a, b) ((a) / (b))
#define TG_SQRT(a) sqrt((a))
static inline uint64_t tg_bits_host(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }
static inline double tg_frombits_host(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
#define TG_BITS(d) tg_bits_host(d)
#define TG_FROMBITS(b) tg_frombits_host(b)
#endif

enum { TG_TEXT = 0, TG_IMAGE = 1, TG_VIDEO = 2 };

/* Per-replica workload description (host fills; device reads). 48 bytes. */
typedef struct {
    uint64_t seed;          /* already mixed: splitmix64(base ^ replica)        */
    uint64_t kv_capacity;   /* footprints are clamped to this                    */
    double   mean_gap_us;   /* 1e6 / lambda                                      */
    uint64_t mix_t1;        /* u32 draw < mix_t1 -> text   (0 .. 2^32)           */
    uint64_t mix_t2;        /* u32 draw < mix_t2 -> image, else video            */
    uint32_t n_requests;
    uint32_t flags;         /* bit0: all arrivals at t=0 (C2 "all pending")      */
} tg_replica;

TG_HD uint64_t tg_splitmix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* Philox4x32-10 (Salmon et al., SC'11). */
TG_HD void tg_philox(uint64_t key, uint32_t c0, uint32_t c1, uint32_t out[4])
{
    uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
    uint32_t x0 = c0, x1 = c1, x2 = 0, x3 = 0;
    for (int r = 0; r < 10; ++r) {
        uint64_t p0 = (uint64_t)0xD2511F53u * x0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * x2;
        uint32_t y0 = (uint32_t)(p1 >> 32) ^ x1 ^ k0;
        uint32_t y1 = (uint32_t)p1;
        uint32_t y2 = (uint32_t)(p0 >> 32) ^ x3 ^ k1;
        uint32_t y3 = (uint32_t)p0;
        x0 = y0; x1 = y1; x2 = y2; x3 = y3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* (u + 0.5) / 2^32, in (0, 1). Exact. */
TG_HD double tg_u01(uint32_t u)
{
    return TG_MUL(TG_ADD((double)u, 0.5), 0x1p-32);
}

/* Natural log for the generator only (x > 0 normal): atanh series on m in [0.70, 1.42).
 * Not the scheduling key's LN (that one lives, independently, on each side of parity). */
TG_HD double tg_log(double x)
{
    uint64_t b = TG_BITS(x);
    int e = (int)((b >> 52) & 0x7FF) - 1023;
    double m = TG_FROMBITS((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull);
    if (m > 1.4142135623730951) { m = TG_MUL(m, 0.5); e += 1; }
    double s = TG_DIV(TG_SUB(m, 1.0), TG_ADD(m, 1.0));
    double s2 = TG_MUL(s, s);
    double acc = 0.0;
    for (int k = 21; k >= 1; k -= 2) acc = TG_ADD(TG_MUL(acc, s2), TG_DIV(1.0, (double)k));
    double lnm = TG_MUL(TG_MUL(2.0, s), acc);
    return TG_ADD(TG_MUL((double)e, 0.6931471805599453), lnm);
}

/* exp for the generator only, |x| < 700. */
TG_HD double tg_exp(double x)
{
    double kd = TG_MUL(x, 1.4426950408889634);
    long long k = (long long)(kd < 0 ? kd - 0.5 : kd + 0.5);
    double r = TG_SUB(x, TG_MUL((double)k, 0.6931471805599453));
    double acc = 1.0;
    for (int n = 16; n >= 1; --n) acc = TG_ADD(1.0, TG_DIV(TG_MUL(acc, r), (double)n));
    return TG_MUL(acc, TG_FROMBITS((uint64_t)(k + 1023) << 52));
}

/* Inverse standard normal CDF (Acklam's rational approximation). p in (0, 1). */
TG_HD double tg_norm_inv(double p)
{
    const double a1 = -3.969683028665376e+01, a2 = 2.209460984245205e+02,
                 a3 = -2.759285104469687e+02, a4 = 1.383577518672690e+02,
                 a5 = -3.066479806614716e+01, a6 = 2.506628277459239e+00;
    const double b1 = -5.447609879822406e+01, b2 = 1.615858368580409e+02,
                 b3 = -1.556989798598866e+02, b4 = 6.680131188771972e+01,
                 b5 = -1.328068155288572e+01;
    const double c1 = -7.784894002430293e-03, c2 = -3.223964580411365e-01,
                 c3 = -2.400758277161838e+00, c4 = -2.549732539343734e+00,
                 c5 = 4.374664141464968e+00, c6 = 2.938163982698783e+00;
    const double d1 = 7.784695709041462e-03, d2 = 3.224671290700398e-01,
                 d3 = 2.445134137142996e+00, d4 = 3.754408661907416e+00;
    const double plow = 0.02425;
    if (p < plow || p > TG_SUB(1.0, plow)) {
        double tail = p < plow ? p : TG_SUB(1.0, p);
        double q = TG_SQRT(TG_MUL(-2.0, tg_log(tail)));
        double num = TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(c1, q), c2), q), c3), q), c4), q), c5), q), c6);
        double den = TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(d1, q), d2), q), d3), q), d4), q), 1.0);
        double x = TG_DIV(num, den);
        return p < plow ? x : -x;
    }
    double q = TG_SUB(p, 0.5);
    double r = TG_MUL(q, q);
    double num = TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(a1, r), a2), r), a3), r), a4), r), a5), r), a6), q);
    double den = TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(TG_ADD(TG_MUL(b1, r), b2), r), b3), r), b4), r), b5), r), 1.0);
    return TG_DIV(num, den);
}

/* Clipped log-normal integer: round(median * exp(sigma * Z)) clamped to [lo, hi]. */
TG_HD uint32_t tg_lognormal(uint32_t u, double median, double sigma, uint32_t lo, uint32_t hi)
{
    double z = tg_norm_inv(tg_u01(u));
    double v = TG_MUL(median, tg_exp(TG_MUL(sigma, z)));
    if (v < (double)lo) return lo;
    if (v > (double)hi) return hi;
    uint32_t t = (uint32_t)TG_ADD(v, 0.5);
    if (t < lo) t = lo;
    if (t > hi) t = hi;
    return t;
}

/* One request's fields except its arrival; gap_us is returned separately so the
 * caller can prefix-sum it (sequentially on the host, warp-scanned on the device). */
typedef struct {
    uint64_t gap_us;
    uint32_t footprint;
    uint32_t inline_us;
    uint16_t out_tokens;
    uint8_t  modality;
} tg_request;

TG_HD tg_request tg_draw(const tg_replica* rp, uint32_t i)
{
    uint32_t a[4], b[4];
    tg_philox(rp->seed, i, 0u, a);
    tg_philox(rp->seed, i, 1u, b);
    tg_request q;
    if (rp->flags & 1u) {
        q.gap_us = 0;
    } else {
        double g = TG_MUL(-tg_log(tg_u01(a[0])), rp->mean_gap_us);
        q.gap_us = (uint64_t)g;                       /* floor, g >= 0 */
    }
    uint32_t mod = (uint64_t)a[1] < rp->mix_t1 ? TG_TEXT : ((uint64_t)a[1] < rp->mix_t2 ? TG_IMAGE : TG_VIDEO);
    uint64_t cap = rp->kv_capacity;
    uint64_t fp;
    uint32_t inl = 0;
    if (mod == TG_TEXT) {
        fp = tg_lognormal(a[2], 200.0, 1.0, 10u, 10000u);
    } else if (mod == TG_IMAGE) {
        uint32_t prompt = tg_lognormal(a[2], 50.0, 0.5, 1u, 512u);
        uint32_t media = 729u + ((b[0] >> 16) % 129u) - 64u;
        inl = 140000u + (uint32_t)(((uint64_t)(b[0] & 0xFFFFu) * 150000u) >> 16);
        fp = (uint64_t)prompt + media;
    } else {
        uint32_t prompt = tg_lognormal(a[2], 50.0, 0.5, 1u, 512u);
        uint64_t frames = 8u + (b[1] % 505u);
        if (prompt > cap) prompt = (uint32_t)cap;
        uint64_t max_frames = (cap - prompt) / 196u;
        if (frames > max_frames) frames = max_frames;
        inl = 300000u + 16000u * (uint32_t)frames;
        fp = (uint64_t)prompt + 196u * frames;
    }
    if (fp > cap) fp = cap;
    if (fp < 1) fp = 1;
    q.footprint = (uint32_t)fp;
    q.inline_us = inl;
    q.out_tokens = (uint16_t)tg_lognormal(a[3], 128.0, 0.8, 1u, 2048u);
    q.modality = (uint8_t)mod;
    return q;
}

/* Host-side helper: fill one replica descriptor from user-level parameters. */
TG_HD tg_replica tg_make_replica(uint64_t base_seed, uint64_t replica, uint32_t n_requests,
                                 double rate_per_s, double mix_text, double mix_image,
                                 uint64_t kv_capacity, uint32_t flags)
{
    tg_replica r;
    r.seed = tg_splitmix64(base_seed ^ replica);
    r.kv_capacity = kv_capacity;
    r.mean_gap_us = TG_DIV(1000000.0, rate_per_s);
    double t1 = TG_MUL(mix_text, 4294967296.0);
    double t2 = TG_MUL(TG_ADD(mix_text, mix_image), 4294967296.0);
    r.mix_t1 = t1 >= 4294967296.0 ? 4294967296ull : (t1 <= 0.0 ? 0ull : (uint64_t)t1);
    r.mix_t2 = t2 >= 4294967296.0 ? 4294967296ull : (t2 <= 0.0 ? 0ull : (uint64_t)t2);
    r.n_requests = n_requests;
    r.flags = flags;
    return r;
}

#endif
