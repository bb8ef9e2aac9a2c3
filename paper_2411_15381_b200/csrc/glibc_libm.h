// log() and cos() exactly as the reference computes them on its hosts.
//
// The reference's Box-Muller draw (proj/src/rng.cpp:30-36) calls std::log and
// std::cos; on x86-64 FMA hosts (this image, the GPU boxes) glibc 2.39's ifuncs
// resolve them to __log_fma and __cos_fma: the published algorithms (ARM
// optimized-routines log.c; the IBM Accurate Mathematical Library's s_sin.c
// __cos with do_cos / do_sin / reduce_sincos / TAYLOR_SIN) compiled with
// -mfma, whose contraction decides the low bits. These functions restate that
// machine code operation by operation -- every fused multiply-add where the
// compiled code has one, separately rounded products and sums elsewhere, in
// its order -- on the library's own tables (glibc_libm_data.h, extracted and
// hash-checked by tools/extract_libm_fma.py). Checked bit for bit against the
// host libm on 2^24+ inputs (tests/test_libm_restatement.py) and on the GPU
// against the reference's own sample_query streams (tests/golden/latent.npz).
//
// Host and device: with nvcc's device pass the primitives are the _rn
// intrinsics; on the host (the CPU check) std::fma and plain operations
// (compile with -ffp-contract=off).
#pragma once

#include <stdint.h>

#if defined(__CUDA_ARCH__)
#define GLIBC_TABLE(name, n) __device__ static const unsigned long long name[n]
#define GLIBC_FN __device__ __forceinline__
#define GM_FMA(a, b, c) __fma_rn((a), (b), (c))
#define GM_MUL(a, b) __dmul_rn((a), (b))
#define GM_ADD(a, b) __dadd_rn((a), (b))
#define GM_SUB(a, b) __dsub_rn((a), (b))
#define GM_BITS(x) static_cast<uint64_t>(__double_as_longlong(x))
#define GM_DBL(u) __longlong_as_double(static_cast<long long>(u))
#define GM_TAB(t, i) __longlong_as_double(static_cast<long long>(__ldg(&(t)[(i)])))
#else
#include <cmath>
#include <cstring>
#define GLIBC_TABLE(name, n) static const unsigned long long name[n]
#define GLIBC_FN static inline
#define GM_FMA(a, b, c) std::fma((a), (b), (c))
#define GM_MUL(a, b) ((a) * (b))
#define GM_ADD(a, b) ((a) + (b))
#define GM_SUB(a, b) ((a) - (b))
static inline uint64_t gm_bits(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
}
static inline double gm_dbl(uint64_t u) {
    double x;
    std::memcpy(&x, &u, 8);
    return x;
}
#define GM_BITS(x) gm_bits(x)
#define GM_DBL(u) gm_dbl(u)
#define GM_TAB(t, i) gm_dbl((t)[(i)])
#endif

#include "glibc_libm_data.h"

#define GM_C(name) GM_DBL(GLIBC_##name)

// __log_fma for x > 0 (the paths a positive double takes; 0, negatives, inf
// and NaN return the IEEE special values, subnormals are rescaled as the
// library does).
GLIBC_FN double glibc_log(double x) {
    uint64_t ix = GM_BITS(x);
    if (ix - 0x3fee000000000000ull <= 0x308ffffffffffull) {
        // |x - 1| < ~0.0625: the polynomial in r = x - 1 with the rhi/rlo split
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double r = GM_SUB(x, 1.0);
        double t2 = GM_FMA(r, GM_C(LOG_B2), GM_C(LOG_B1));
        double t3 = GM_FMA(r, GM_C(LOG_B5), GM_C(LOG_B4));
        const double r2 = GM_MUL(r, r);
        const double t5 = GM_FMA(r, GM_C(LOG_B8), GM_C(LOG_B7));
        t2 = GM_FMA(r2, GM_C(LOG_B3), t2);
        t3 = GM_FMA(r2, GM_C(LOG_B6), t3);
        const double r3 = GM_MUL(r, r2);
        double p = GM_FMA(r2, GM_C(LOG_B9), t5);
        p = GM_FMA(r3, GM_C(LOG_B10), p);
        p = GM_FMA(p, r3, t3);
        p = GM_FMA(p, r3, t2);
        const double two27 = 134217728.0;
        double rhi = GM_FMA(r, two27, r);
        rhi = GM_FMA(-two27, r, rhi);
        const double rr = GM_MUL(rhi, rhi);
        const double rlo = GM_SUB(r, rhi);
        const double b0 = GM_C(LOG_B0);
        const double hi = GM_FMA(rr, b0, r);
        const double t8 = GM_SUB(r, hi);
        const double s = GM_ADD(r, rhi);
        double lo = GM_FMA(rr, b0, t8);
        lo = GM_FMA(GM_MUL(b0, rlo), s, lo);
        return GM_ADD(hi, GM_FMA(p, r3, lo));
    }
    const uint32_t top = static_cast<uint32_t>(ix >> 48);
    if (top - 0x0010u > 0x7fdfu) {
        if ((ix << 1) == 0) return -__builtin_huge_val();           // log(+-0) = -inf
        if (ix == 0x7ff0000000000000ull) return x;                   // log(inf) = inf
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return __builtin_nan("");
        // subnormal: x * 2^52, exponent corrected by -52
        ix = GM_BITS(GM_MUL(x, 4503599627370496.0)) - (52ull << 52);
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = static_cast<int>((tmp >> 45) & 0x7f);
    const int k = static_cast<int>(static_cast<int64_t>(tmp) >> 52);
    const double z = GM_DBL(ix - (tmp & 0xfff0000000000000ull));
    const double invc = GM_TAB(glibc_log_tab, 2 * i), logc = GM_TAB(glibc_log_tab, 2 * i + 1);
    const double kd = static_cast<double>(k);
    const double w = GM_FMA(kd, GM_C(LOG_LN2HI), logc);
    const double r = GM_FMA(z, invc, -1.0);
    const double a21 = GM_FMA(r, GM_C(LOG_A2), GM_C(LOG_A1));
    const double hi = GM_ADD(r, w);
    const double r2 = GM_MUL(r, r);
    double lo = GM_ADD(GM_SUB(w, hi), r);
    lo = GM_FMA(kd, GM_C(LOG_LN2LO), lo);
    const double r3 = GM_MUL(r, r2);
    double q = GM_FMA(r, GM_C(LOG_A4), GM_C(LOG_A3));
    lo = GM_FMA(r2, GM_C(LOG_A0), lo);
    q = GM_FMA(q, r2, a21);
    return GM_ADD(GM_FMA(r3, q, lo), hi);
}

// do_cos (s_sin.c) as __cos_fma inlines it: cos(a + da), |a| < 0.855469
// (the caller passes da already negated when a < 0).
GLIBC_FN double glibc_do_cos(double a_abs, double da) {
    const double big = GM_C(SIN_BIG);
    const double u = GM_ADD(a_abs, big);
    const int idx = 4 * static_cast<int>(static_cast<uint32_t>(GM_BITS(u)));
    double x = GM_SUB(a_abs, GM_SUB(u, big));
    x = GM_ADD(x, da);
    const double xx = GM_MUL(x, x);
    const double p = GM_FMA(xx, GM_C(SIN_SN5), GM_C(SIN_SN3));
    const double s = GM_FMA(GM_MUL(x, xx), p, x);
    double c = GM_FMA(xx, GM_C(SIN_CS6), GM_C(SIN_CS4));
    c = GM_FMA(xx, c, GM_C(SIN_CS2));
    c = GM_MUL(xx, c);
    const double sn = GM_TAB(glibc_sincos_tab, idx), ssn = GM_TAB(glibc_sincos_tab, idx + 1);
    const double cs = GM_TAB(glibc_sincos_tab, idx + 2), ccs = GM_TAB(glibc_sincos_tab, idx + 3);
    double cor = GM_FMA(-s, ssn, ccs);
    cor = GM_FMA(-c, cs, cor);
    cor = GM_FMA(-s, sn, cor);
    return GM_ADD(cs, cor);
}

// do_sin (s_sin.c) for |a| >= 0.126: sin(a + da), sign of a restored at the
// end (the caller passes da negated when a <= 0).
GLIBC_FN double glibc_do_sin_table(double a, double a_abs, double da) {
    const double big = GM_C(SIN_BIG);
    const double u = GM_ADD(a_abs, big);
    const int idx = 4 * static_cast<int>(static_cast<uint32_t>(GM_BITS(u)));
    const double x = GM_SUB(a_abs, GM_SUB(u, big));
    const double xx = GM_MUL(x, x);
    const double p = GM_FMA(xx, GM_C(SIN_SN5), GM_C(SIN_SN3));
    const double s = GM_ADD(x, GM_FMA(GM_MUL(x, xx), p, da));
    double c = GM_FMA(xx, GM_C(SIN_CS6), GM_C(SIN_CS4));
    c = GM_FMA(xx, c, GM_C(SIN_CS2));
    c = GM_FMA(x, da, GM_MUL(xx, c));
    const double sn = GM_TAB(glibc_sincos_tab, idx), ssn = GM_TAB(glibc_sincos_tab, idx + 1);
    const double cs = GM_TAB(glibc_sincos_tab, idx + 2), ccs = GM_TAB(glibc_sincos_tab, idx + 3);
    double cor = GM_FMA(s, ccs, ssn);
    cor = GM_FMA(-c, sn, cor);
    cor = GM_FMA(s, cs, cor);
    const double r = GM_ADD(sn, cor);
    return GM_DBL((GM_BITS(r) & 0x7fffffffffffffffull) | (GM_BITS(a) & 0x8000000000000000ull));
}

// TAYLOR_SIN (s_sin.c) for |a| < 0.126: sin(a + da).
GLIBC_FN double glibc_taylor_sin(double a, double da) {
    const double xx = GM_MUL(a, a);
    double t = GM_FMA(xx, GM_C(SIN_S5), GM_C(SIN_S4));
    t = GM_FMA(xx, t, GM_C(SIN_S3));
    t = GM_FMA(xx, t, GM_C(SIN_S2));
    t = GM_FMA(xx, t, GM_C(SIN_S1));
    t = GM_FMA(t, a, -GM_MUL(da, 0.5));
    return GM_ADD(a, GM_FMA(xx, t, da));
}

// __cos_fma for |x| < 105414350 (every x = 2*pi*u2 of the reference's draw,
// u2 in [0, 1)); larger arguments take the library's multi-precision range
// reduction, not restated here (NaN is returned).
GLIBC_FN double glibc_cos(double x) {
    const uint32_t k = static_cast<uint32_t>(GM_BITS(x) >> 32) & 0x7fffffffu;
    if (k <= 0x3e3fffffu) return 1.0;                          // |x| < 2^-27
    const double ax = GM_DBL(GM_BITS(x) & 0x7fffffffffffffffull);
    if (k <= 0x3feb5fffu)                                       // |x| < 0.855469
        return glibc_do_cos(ax, x < 0.0 ? -0.0 : 0.0);
    if (k <= 0x400368fcu) {                                     // |x| < 2.426265
        const double y = GM_SUB(GM_C(SIN_HP0), ax);
        const double a = GM_ADD(y, GM_C(SIN_HP1));
        double da = GM_ADD(GM_SUB(y, a), GM_C(SIN_HP1));
        const double a_abs = GM_DBL(GM_BITS(a) & 0x7fffffffffffffffull);
        if (a_abs < GM_C(SIN_TAYLOR_MAX)) return glibc_taylor_sin(a, da);
        if (0.0 >= a) da = GM_DBL(GM_BITS(da) ^ 0x8000000000000000ull);
        return glibc_do_sin_table(a, a_abs, da);
    }
    if (k > 0x419921fau) return __builtin_nan("");
    // reduce_sincos: x = n*pi/2 + (b + db)
    const double toint = GM_C(SIN_TOINT);
    const double t = GM_FMA(x, GM_C(SIN_HPINV), toint);
    const double xn = GM_SUB(t, toint);
    const int n = static_cast<int>(static_cast<uint32_t>(GM_BITS(t)) & 3u);
    double y = GM_FMA(-xn, GM_C(SIN_MP1), x);
    y = GM_FMA(-xn, GM_C(SIN_MP2), y);
    const double pp3 = GM_C(SIN_PP3), pp4 = GM_C(SIN_PP4);
    const double t2 = GM_FMA(-xn, pp3, y);
    double db = GM_SUB(y, t2);
    db = GM_FMA(-xn, pp3, db);
    const double b = GM_FMA(-xn, pp4, t2);
    double da = GM_FMA(-xn, pp4, GM_SUB(t2, b));
    da = GM_ADD(db, da);
    const double b_abs = GM_DBL(GM_BITS(b) & 0x7fffffffffffffffull);
    double r;
    if (n & 1) {   // (n + 1) even: do_sin
        if (b_abs < GM_C(SIN_TAYLOR_MAX)) {
            r = glibc_taylor_sin(b, da);
        } else {
            if (!(0.0 < b)) da = GM_DBL(GM_BITS(da) ^ 0x8000000000000000ull);
            r = glibc_do_sin_table(b, b_abs, da);
        }
    } else {       // (n + 1) odd: do_cos
        r = glibc_do_cos(b_abs, b < 0.0 ? GM_DBL(GM_BITS(da) ^ 0x8000000000000000ull) : da);
    }
    return ((n + 1) & 2) ? GM_DBL(GM_BITS(r) ^ 0x8000000000000000ull) : r;
}
