// tcm_k1.cuh -- device implementation of K1, the specified priority key.
//
// Priority_c = StaticPriority_c + (1 - e^{-k_c * waiting_time^{p_c}})
// with waiting_time in seconds (R1), ordered by max(P, 1e-12) descending (R3).
// Every operation is an explicitly rounded IEEE binary64 op (__dmul_rn/__dadd_rn/__fma_rn)
// so the result is bit-identical to any conforming implementation of the spec text.
// Written from DESIGN.md 4 independently of oracle/ (no shared code or headers).
#pragma once
#include <stdint.h>

namespace tcm {

// DESIGN.md "K1 constants", transcribed.
__constant__ double kLnR[16] = {
    0x1.f0p-1, 0x1.d4p-1, 0x1.bap-1, 0x1.a4p-1, 0x1.90p-1, 0x1.7ep-1, 0x1.6cp-1, 0x1.5cp-1,
    0x1.4ep-1, 0x1.42p-1, 0x1.36p-1, 0x1.2ap-1, 0x1.20p-1, 0x1.16p-1, 0x1.0cp-1, 0x1.04p-1};
__constant__ double kLnT[16] = {
    0x1.0415d89e74444p-5, 0x1.700d30aeac0e1p-4, 0x1.2d1610c86813ap-3, 0x1.95a5adcf7017fp-3,
    0x1.f991c6cb3b379p-3, 0x1.2bef07cdc9354p-2, 0x1.5d5bddf595f30p-2, 0x1.8b639a88b2df5p-2,
    0x1.b56fa04462909p-2, 0x1.dae75484c9616p-2, 0x1.00e5ae5b207abp-1, 0x1.151c3f6f29612p-1,
    0x1.269621134db92p-1, 0x1.38ae2171976e7p-1, 0x1.4b6fd6f970c1fp-1, 0x1.5af405c3649e0p-1};
__constant__ double kExpT[16] = {
    0x1p+0,               0x1.0b5586cf9890fp+0, 0x1.172b83c7d517bp+0, 0x1.2387a6e756238p+0,
    0x1.306fe0a31b715p+0, 0x1.3dea64c123422p+0, 0x1.4bfdad5362a27p+0, 0x1.5ab07dd485429p+0,
    0x1.6a09e667f3bcdp+0, 0x1.7a11473eb0187p+0, 0x1.8ace5422aa0dbp+0, 0x1.9c49182a3f090p+0,
    0x1.ae89f995ad3adp+0, 0x1.c199bdd85529cp+0, 0x1.d5818dcfba487p+0, 0x1.ea4afa2a490dap+0};

constexpr double kLN2 = 0x1.62e42fefa39efp-1;
constexpr double kInvLn2x16 = 0x1.71547652b82fep+4;
constexpr double kLn2d16Hi = 0x1.62e42fee00000p-5;
constexpr double kLn2d16Lo = 0x1.a39ef35793c76p-37;
constexpr double kEps = 1e-12;

// Table access: the fused engine reads the __constant__ copies (few keys per decision); the
// stepwise engine stages them in shared memory (divergent j across a warp would serialise
// constant-cache reads).
struct K1Tables {
    const double* lnR;
    const double* lnT;
    const double* expT;
};

__device__ __forceinline__ K1Tables k1_const_tables() { return K1Tables{kLnR, kLnT, kExpT}; }

// Exact integer <-> double conversions on the FMA/ALU pipes instead of the (slow, shared)
// XU pipe: 0x1.8p52 has ulp 1, so adding it rounds to an integer (ties-to-even, i.e. rint)
// and its low mantissa bits then hold the integer.
constexpr double kMagic = 0x1.8p52;
constexpr unsigned long long kMagicBits = 0x4338000000000000ull;

__device__ __forceinline__ double small_int_to_double(long long e) {     // |e| < 2^51, exact
    return __dsub_rn(__longlong_as_double((long long)(kMagicBits + (unsigned long long)e)), kMagic);
}

__device__ __forceinline__ double u64_to_double_rn(uint64_t w) {        // == __ull2double_rn(w)
    if (w < (1ull << 52)) return __dsub_rn(__longlong_as_double((long long)(0x4330000000000000ull | w)), 0x1p52);
    return __ull2double_rn(w);
}

// LN(v), v a positive normal double: steps LN.1-LN.6.
__device__ __forceinline__ double k1_ln(double v, const K1Tables& tb = k1_const_tables()) {
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    const int e = (int)((b >> 52) & 0x7FF) - 1023;
    const int j = (int)((b >> 48) & 0xF);
    const double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    const double u = __fma_rn(m, tb.lnR[j], -1.0);
    double q = 0x1.c71c71c71c71cp-4;                 // c9
    q = __fma_rn(q, u, -0x1p-3);                     // c8
    q = __fma_rn(q, u, 0x1.2492492492492p-3);        // c7
    q = __fma_rn(q, u, -0x1.5555555555555p-3);       // c6
    q = __fma_rn(q, u, 0x1.999999999999ap-3);        // c5
    q = __fma_rn(q, u, -0x1p-2);                     // c4
    q = __fma_rn(q, u, 0x1.5555555555555p-2);        // c3
    q = __fma_rn(q, u, -0x1p-1);                     // c2
    q = __fma_rn(q, u, 0x1p+0);                      // c1
    const double lnm = __dmul_rn(q, u);
    const double t = __dadd_rn(tb.lnT[j], lnm);
    return __fma_rn(small_int_to_double(e), kLN2, t);
}

// EXP(y): steps EXP.1-EXP.7.
__device__ __forceinline__ double k1_exp(double y, const K1Tables& tb = k1_const_tables()) {
    if (y < -745.0) return 0.0;
    if (y > 700.0) return __longlong_as_double(0x7FF0000000000000ll);
    // EXP.2 kf = rint(y * 16/ln2) (|.| < 2^15 here, so the magic-number rounding is exact rint)
    const double tm = __dadd_rn(__dmul_rn(y, kInvLn2x16), kMagic);
    const double kf = __dsub_rn(tm, kMagic);
    const long long k = (long long)((unsigned long long)__double_as_longlong(tm) - kMagicBits);
    double r = __fma_rn(-kf, kLn2d16Hi, y);
    r = __fma_rn(-kf, kLn2d16Lo, r);
    double p = 0x1.6c16c16c16c17p-10;                // 1/6!
    p = __fma_rn(p, r, 0x1.1111111111111p-7);        // 1/5!
    p = __fma_rn(p, r, 0x1.5555555555555p-5);        // 1/4!
    p = __fma_rn(p, r, 0x1.5555555555555p-3);        // 1/3!
    p = __fma_rn(p, r, 0x1p-1);                      // 1/2!
    p = __fma_rn(p, r, 0x1p+0);                      // 1/1!
    p = __fma_rn(p, r, 0x1p+0);                      // 1/0!
    const long long j = k & 15;
    const long long n = (k - j) / 16;
    const double s = __dmul_rn(tb.expT[j], p);
    if (n < -1021) return 0.0;
    const double res = __dmul_rn(s, __longlong_as_double((long long)((unsigned long long)(n + 1023) << 52)));
    if (res < 0x1p-1022) return 0.0;
    return res;
}

// Per (replica, class) constant: C_c = LN(alpha*k_c) - p_c * LN(10^6); zero rate if alpha*k_c is 0
// or subnormal.
struct K1Class {
    double S, p, C;
    bool zero;
};

__device__ __forceinline__ K1Class k1_class(double S, double k, double p, double alpha) {
    K1Class kc;
    kc.S = S;
    kc.p = p;
    const double a = __dmul_rn(alpha, k);
    if (!(a >= 0x1p-1022)) {
        kc.zero = true;
        kc.C = 0.0;
    } else {
        kc.zero = false;
        const double t = __dmul_rn(p, k1_ln(1000000.0));
        kc.C = __dsub_rn(k1_ln(a), t);
    }
    return kc;
}

__device__ __forceinline__ double k1_priority(const K1Class& kc, uint64_t w,
                                              const K1Tables& tb = k1_const_tables()) {
    if (w == 0 || kc.zero) return kc.S;
    const double L = k1_ln(u64_to_double_rn(w), tb);
    const double y = __fma_rn(kc.p, L, kc.C);
    const double x = k1_exp(y, tb);
    const double e = k1_exp(-x, tb);
    return __dadd_rn(kc.S, __dsub_rn(1.0, e));
}

// Key: bit pattern of max(P, 1e-12), compared as unsigned, larger first.
__device__ __forceinline__ uint64_t k1_key(const K1Class& kc, uint64_t w,
                                           const K1Tables& tb = k1_const_tables()) {
    double P = k1_priority(kc, w, tb);
    P = P < kEps ? kEps : P;
    return (uint64_t)__double_as_longlong(P);
}

// ---- Branch-free K1 for the streaming key kernel ------------------------------------------
// Same spec, same operations on every in-range value, hence bit-identical results; the
// special cases (w == 0, zero rate, EXP cut-offs, flush) are computed through and selected
// at the end so a warp never diverges inside the key.  Coefficients live in the constant
// bank so the DFMAs take them as c[][] operands instead of re-materialising immediates.
__constant__ double kPoly[19] = {
    // LN c9 .. c1
    0x1.c71c71c71c71cp-4, -0x1p-3, 0x1.2492492492492p-3, -0x1.5555555555555p-3, 0x1.999999999999ap-3,
    -0x1p-2, 0x1.5555555555555p-2, -0x1p-1, 0x1p+0,
    // EXP 1/6! .. 1/0!
    0x1.6c16c16c16c17p-10, 0x1.1111111111111p-7, 0x1.5555555555555p-5, 0x1.5555555555555p-3, 0x1p-1,
    0x1p+0, 0x1p+0,
    // LN2, LN2/16 hi, LN2/16 lo
    0x1.62e42fefa39efp-1, 0x1.62e42fee00000p-5, 0x1.a39ef35793c76p-37};

__device__ __forceinline__ double k1_ln_bf(double v, const K1Tables& tb) {
    const uint64_t b = (uint64_t)__double_as_longlong(v);
    const int e = (int)((b >> 52) & 0x7FF) - 1023;
    const int j = (int)((b >> 48) & 0xF);
    const double m = __longlong_as_double((long long)((b & 0x000FFFFFFFFFFFFFull) | 0x3FF0000000000000ull));
    const double u = __fma_rn(m, tb.lnR[j], -1.0);
    double q = kPoly[0];
#pragma unroll
    for (int i = 1; i < 9; ++i) q = __fma_rn(q, u, kPoly[i]);
    const double lnm = __dmul_rn(q, u);
    const double t = __dadd_rn(tb.lnT[j], lnm);
    return __fma_rn(small_int_to_double(e), kPoly[16], t);
}

__device__ __forceinline__ double k1_exp_bf(double y, const K1Tables& tb) {
    const double yc = fmin(fmax(y, -746.0), 701.0);         // keeps the discarded lanes finite
    const double tm = __dadd_rn(__dmul_rn(yc, kInvLn2x16), kMagic);
    const double kf = __dsub_rn(tm, kMagic);
    const long long k = (long long)((unsigned long long)__double_as_longlong(tm) - kMagicBits);
    double r = __fma_rn(-kf, kPoly[17], yc);
    r = __fma_rn(-kf, kPoly[18], r);
    double p = kPoly[9];
#pragma unroll
    for (int i = 10; i < 16; ++i) p = __fma_rn(p, r, kPoly[i]);
    const int j = (int)(k & 15);
    const long long n = k >> 4;                               // == (k - j) / 16 exactly
    const double s = __dmul_rn(tb.expT[j], p);
    const long long nn = n < -1021 ? -1021 : n;               // discarded when n < -1021
    double res = __dmul_rn(s, __longlong_as_double((long long)((unsigned long long)(nn + 1023) << 52)));
    res = (n < -1021 || res < 0x1p-1022) ? 0.0 : res;
    res = y < -745.0 ? 0.0 : res;
    return y > 700.0 ? __longlong_as_double(0x7FF0000000000000ll) : res;
}

// ---- FP32 bound on the priority (filter for the exact top-k; never decides an order) --------
// P~ = S + (1 - 2^(-x log2 e)), x = 2^(p2 * log2(w) + C2), C2 = C / ln 2, evaluated with the
// SFU approximations (PTX lg2.approx / ex2.approx, max errors 2^-22.6 abs / 2^-22.5 rel) and
// log2(w) of w rounded to FP32 (relative error <= 2^-24).  Error budget:
// |P~ - P| <= 0.37 * ln2 * (p * 2.5e-6 + (|y| + |C2|) * 6e-8) + 1e-6, i.e. < 1e-5 for the
// supported range (p <= 16, |C2| <= 1000); the kernel uses kFilterDelta = 1e-4, and
// tcm_k1_filter_error() audits the bound exhaustively per (class, alpha) on the device.
constexpr double kFilterDelta = 1e-4;

__device__ __forceinline__ float sfu_lg2(float x) {
    float y;
    asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float sfu_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

__device__ __forceinline__ float k1_filter_f32(float Sf, float p2, float C2, uint64_t w) {
    // w >= 1: one conversion (round to nearest, relative error <= 2^-24, half the truncation error of
    // the exponent + top-23-mantissa-bits form it replaces) and the SFU lg2 of the float
    const float L = sfu_lg2(__ull2float_rn(w));
    const float x = sfu_ex2(fmaf(p2, L, C2));
    const float ee = sfu_ex2(-x * 1.44269504f);
    return Sf + (1.0f - ee);
}

__device__ __forceinline__ uint64_t k1_key_bf(double S, double p, double C, bool zero, uint64_t w,
                                              const K1Tables& tb) {
    const double L = k1_ln_bf(u64_to_double_rn(w), tb);
    const double y = __fma_rn(p, L, C);
    const double x = k1_exp_bf(y, tb);
    const double e = k1_exp_bf(-x, tb);
    double P = __dadd_rn(S, __dsub_rn(1.0, e));
    P = (w == 0 || zero) ? S : P;
    P = P < kEps ? kEps : P;
    return (uint64_t)__double_as_longlong(P);
}

}  // namespace tcm
