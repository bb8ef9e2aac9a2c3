// log1p(x) restated from the published fdlibm algorithm (Sun Microsystems
// fdlibm 5.3 s_log1p.c) in the form glibc ships (sysdeps/ieee754/dbl-64/
// s_log1p.c: the polynomial split into R1 + z2*R2 + z4*R3 + z6*R4). On an
// FMA-capable x86-64 host glibc's libm resolves log1p to its FMA build of that
// file, in which the compiler fused the mul/add pairs marked DS_FMA below.
// The reference draws every exponential variate as -std::log1p(-U)
// (rng.cpp:24-28) through that routine, so replaying the same operation
// sequence with correctly rounded basic ops and the same fused pairs
// reproduces the host's result bit for bit; tests/test_oracle.py compiles
// this header for the host and checks it against the host libm on 2^24
// inputs.
//
// Usable from host and device code. Every add/sub/mul/div/fma is written
// through the DS_* macros so the device build cannot contract anything else
// (the host build is compiled with -ffp-contract=off).
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define DS_HD __host__ __device__ __forceinline__
#else
#define DS_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define DS_ADD(a, b) __dadd_rn((a), (b))
#define DS_SUB(a, b) __dsub_rn((a), (b))
#define DS_MUL(a, b) __dmul_rn((a), (b))
#define DS_DIV(a, b) __ddiv_rn((a), (b))
#define DS_FMA(a, b, c) __fma_rn((a), (b), (c))
#else
#include <math.h>
#define DS_ADD(a, b) ((a) + (b))
#define DS_SUB(a, b) ((a) - (b))
#define DS_MUL(a, b) ((a) * (b))
#define DS_DIV(a, b) ((a) / (b))
#define DS_FMA(a, b, c) fma((a), (b), (c))
#endif

DS_HD uint64_t ds_dbits(double x) {
    uint64_t u;
    memcpy(&u, &x, sizeof u);
    return u;
}

DS_HD double ds_bitsd(uint64_t u) {
    double x;
    memcpy(&x, &u, sizeof x);
    return x;
}

DS_HD int32_t ds_hi(double x) { return (int32_t)(ds_dbits(x) >> 32); }

DS_HD double ds_with_hi(double x, uint32_t hi) {
    return ds_bitsd((ds_dbits(x) & 0xffffffffull) | ((uint64_t)hi << 32));
}

// fdlibm log1p. Argument reduction 1+x = 2^k (1+f) with sqrt(2)/2 < 1+f <
// sqrt(2), a correction term c for the rounding of 1+x, and the minimax
// polynomial in s = f/(2+f) with coefficients Lp1..Lp7.
DS_HD double ds_log1p(double x) {
    const double ln2_hi = 6.93147180369123816490e-01;  // 0x3fe62e42fee00000
    const double ln2_lo = 1.90821492927058770002e-10;  // 0x3dea39ef35793c76
    const double two54 = 1.80143985094819840000e+16;   // 0x4350000000000000
    const double Lp1 = 6.666666666666735130e-01;       // 0x3FE5555555555593
    const double Lp2 = 3.999999999940941908e-01;       // 0x3FD999999997FA04
    const double Lp3 = 2.857142874366239149e-01;       // 0x3FD2492494229359
    const double Lp4 = 2.222219843214978396e-01;       // 0x3FCC71C51D8E78AF
    const double Lp5 = 1.818357216161805012e-01;       // 0x3FC7466496CB03DE
    const double Lp6 = 1.531383769920937332e-01;       // 0x3FC39A09D078C69F
    const double Lp7 = 1.479819860511658591e-01;       // 0x3FC2F112DF3E5244

    double hfsq, f = 0.0, c = 0.0, s, z, R, u;
    int32_t k, hx, hu = 0, ax;

    hx = ds_hi(x);
    ax = hx & 0x7fffffff;

    k = 1;
    if (hx < 0x3FDA827A) {                     // 1+x < sqrt(2)+
        if (ax >= 0x3ff00000) {                // x <= -1.0
            if (x == -1.0) return -1.0 / 0.0;  // log1p(-1) = -inf
            return (x - x) / (x - x);          // NaN
        }
        if (ax < 0x3e200000) {                 // |x| < 2^-29
            if (DS_ADD(two54, x) > 0.0 && ax < 0x3c900000) return x;  // |x| < 2^-54
            return DS_FMA(-DS_MUL(x, x), 0.5, x);
        }
        if (hx > 0 || hx <= (int32_t)0xbfd2bec4) {  // sqrt(2)/2- <= 1+x < sqrt(2)+
            k = 0;
            f = x;
            hu = 1;
        }
    }
    if (hx >= 0x7ff00000) return DS_ADD(x, x);
    if (k != 0) {
        if (hx < 0x43400000) {
            u = DS_ADD(1.0, x);
            hu = ds_hi(u);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? DS_SUB(1.0, DS_SUB(u, x)) : DS_SUB(x, DS_SUB(u, 1.0));
            c = DS_DIV(c, u);
        } else {
            u = x;
            hu = ds_hi(u);
            k = (hu >> 20) - 1023;
            c = 0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = ds_with_hi(u, (uint32_t)hu | 0x3ff00000u);  // normalize u
        } else {
            k += 1;
            u = ds_with_hi(u, (uint32_t)hu | 0x3fe00000u);  // normalize u/2
            hu = (0x00100000 - hu) >> 2;
        }
        f = DS_SUB(u, 1.0);
    }
    hfsq = DS_MUL(DS_MUL(0.5, f), f);
    const double dk = (double)k;
    if (hu == 0) {  // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            c = DS_FMA(dk, ln2_lo, c);
            return DS_FMA(dk, ln2_hi, c);
        }
        R = DS_MUL(hfsq, DS_FMA(-0.66666666666666666, f, 1.0));
        if (k == 0) return DS_SUB(f, R);
        return DS_FMA(dk, ln2_hi, -DS_SUB(DS_SUB(R, DS_FMA(dk, ln2_lo, c)), f));
    }
    s = DS_DIV(f, DS_ADD(2.0, f));
    z = DS_MUL(s, s);
    {
        const double R2 = DS_FMA(z, Lp3, Lp2);
        const double R3 = DS_FMA(z, Lp5, Lp4);
        const double R4 = DS_FMA(z, Lp7, Lp6);
        const double z2 = DS_MUL(z, z);
        const double z4 = DS_MUL(z2, z2);
        const double z6 = DS_MUL(z4, z2);
        R = DS_FMA(z6, R4, DS_FMA(z4, R3, DS_FMA(z, Lp1, DS_MUL(z2, R2))));
    }
    if (k == 0) return DS_SUB(f, DS_SUB(hfsq, DS_MUL(s, DS_ADD(hfsq, R))));
    return DS_FMA(dk, ln2_hi,
                  -DS_SUB(DS_SUB(hfsq, DS_ADD(DS_MUL(s, DS_ADD(hfsq, R)),
                                              DS_FMA(dk, ln2_lo, c))),
                          f));
}
