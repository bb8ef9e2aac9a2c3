// Exact "%.6g" (the reference's fmt6, metrics.cpp:67-71: snprintf(buf, 40,
// "%.6g", v)) for host and device code, byte-identical to glibc's printf.
//
// glibc formats from the exact binary value: the 6 significant digits are
// |v| / 10^(X-5) rounded to nearest with ties to even (the current rounding
// mode), X the decimal exponent after that rounding; %g then picks fixed
// notation when -4 <= X < 6 and exponent notation otherwise, and drops
// trailing zeros (and a bare '.'). This header reproduces that:
//   * |v| = m * 2^e exactly; r = m * 2^e / 10^q with q = X-5 is evaluated as a
//     ratio of integers, floor and remainder exact:
//       - fast path (q <= 0, e <= 0, the range CSV times/qualities live in):
//         m * 10^-q fits in 128 bits and the division by 2^-e is a shift;
//       - general path: a 1280-bit integer A / B with A, B = m, powers of 2 and
//         of 5, quotient (< 2^25) by binary long division.
//   * X starts from floor(log2|v|) * log10(2) and is corrected until
//     10^5 <= floor(r) < 10^6; rounding up to 10^6 bumps X.
// tests/test_oracle.py compiles this header for the host and compares it with
// the host snprintf on millions of doubles (both paths forced).
#pragma once

#include <stdint.h>
#include <string.h>

#if defined(__CUDACC__)
#define DS_FMT_HD __host__ __device__ __forceinline__
#define DS_FMT_COLD __host__ __device__ __noinline__
#else
#define DS_FMT_HD static inline
#define DS_FMT_COLD static
#endif

typedef unsigned __int128 ds_u128;

#define DS_BIG_LIMBS 40

typedef struct {
    uint32_t w[DS_BIG_LIMBS];   // little-endian 32-bit limbs
} ds_big;

DS_FMT_HD void ds_big_set(ds_big* a, uint64_t v) {
    for (int i = 0; i < DS_BIG_LIMBS; ++i) a->w[i] = 0;
    a->w[0] = (uint32_t)v;
    a->w[1] = (uint32_t)(v >> 32);
}

DS_FMT_HD void ds_big_mul_small(ds_big* a, uint32_t k) {
    uint64_t carry = 0;
    for (int i = 0; i < DS_BIG_LIMBS; ++i) {
        const uint64_t t = (uint64_t)a->w[i] * k + carry;
        a->w[i] = (uint32_t)t;
        carry = t >> 32;
    }
}

DS_FMT_HD void ds_big_pow5(ds_big* a, int n) {   // a *= 5^n
    while (n >= 13) {
        ds_big_mul_small(a, 1220703125u);        // 5^13
        n -= 13;
    }
    uint32_t k = 1;
    while (n-- > 0) k *= 5;
    ds_big_mul_small(a, k);
}

DS_FMT_HD void ds_big_shl(ds_big* a, int n) {
    const int limbs = n >> 5, bits = n & 31;
    for (int i = DS_BIG_LIMBS - 1; i >= 0; --i) {
        const int s = i - limbs;
        uint32_t v = 0;
        if (s >= 0) {
            v = a->w[s] << bits;
            if (bits && s > 0) v |= a->w[s - 1] >> (32 - bits);
        }
        a->w[i] = v;
    }
}

DS_FMT_HD int ds_big_cmp(const ds_big* a, const ds_big* b) {
    for (int i = DS_BIG_LIMBS - 1; i >= 0; --i)
        if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
    return 0;
}

DS_FMT_HD void ds_big_sub(ds_big* a, const ds_big* b) {   // a -= b (a >= b)
    int64_t borrow = 0;
    for (int i = 0; i < DS_BIG_LIMBS; ++i) {
        const int64_t t = (int64_t)a->w[i] - b->w[i] - borrow;
        a->w[i] = (uint32_t)t;
        borrow = t < 0;
    }
}

// floor(r) and the rounding class of r = m * 2^e / 10^q:
// *cls = -1 below half, 0 exactly half, +1 above half (of the unit step).
DS_FMT_COLD uint64_t ds_ratio_big(uint64_t m, int e, int q, int* cls) {
    ds_big A, B;
    ds_big_set(&A, m);
    ds_big_set(&B, 1);
    const int a2 = e - q, a5 = -q;
    if (a5 >= 0) ds_big_pow5(&A, a5);
    else ds_big_pow5(&B, -a5);
    if (a2 >= 0) ds_big_shl(&A, a2);
    else ds_big_shl(&B, -a2);
    // quotient < 2^25 whenever the caller's exponent is within one of right
    uint64_t quo = 0;
    for (int bit = 25; bit >= 0; --bit) {
        ds_big t = B;
        ds_big_shl(&t, bit);
        // t may have lost high bits if B << bit overflowed; B < 2^1250 here
        if (ds_big_cmp(&A, &t) >= 0) {
            ds_big_sub(&A, &t);
            quo |= (uint64_t)1 << bit;
        }
    }
    ds_big_shl(&A, 1);   // 2 * remainder vs B
    *cls = ds_big_cmp(&A, &B);
    return quo;
}

DS_FMT_HD uint64_t ds_pow10_u64(int k) {
    uint64_t p = 1;
    while (k-- > 0) p *= 10;
    return p;
}

DS_FMT_HD uint64_t ds_ratio(uint64_t m, int e, int q, int* cls) {
#ifndef DS_FMT_FORCE_BIG
    if (q <= 0 && q >= -22 && e <= 0 && e > -128) {
        ds_u128 num = (ds_u128)m;
        int k = -q;
        if (k > 19) {
            num *= (ds_u128)ds_pow10_u64(19);
            k -= 19;
        }
        num *= (ds_u128)ds_pow10_u64(k);
        const int s = -e;
        if (s == 0) {
            *cls = -1;
            return (uint64_t)num;   // fits: the result is < 2^25
        }
        const ds_u128 fl = num >> s;
        const ds_u128 rem = num - (fl << s);
        const ds_u128 half = (ds_u128)1 << (s - 1);
        *cls = rem < half ? -1 : (rem == half ? 0 : 1);
        return fl > (ds_u128)0xffffffffffffull ? 0xffffffffffffull : (uint64_t)fl;
    }
#endif
    return ds_ratio_big(m, e, q, cls);
}

// Writes "%.6g" of v to out (no NUL); returns the length (<= 13).
DS_FMT_COLD int ds_fmt_g6(double v, char* out) {
    uint64_t bits;
    memcpy(&bits, &v, sizeof bits);
    const int neg = (int)(bits >> 63);
    const int bexp = (int)((bits >> 52) & 0x7ff);
    const uint64_t frac = bits & 0xfffffffffffffull;
    int n = 0;
    if (neg) out[n++] = '-';
    if (bexp == 0x7ff) {
        if (frac) { out[n++] = 'n'; out[n++] = 'a'; out[n++] = 'n'; }
        else { out[n++] = 'i'; out[n++] = 'n'; out[n++] = 'f'; }
        return n;
    }
    if (bexp == 0 && frac == 0) {
        out[n++] = '0';
        return n;
    }
    uint64_t m;
    int e, e2;
    if (bexp == 0) {   // subnormal
        m = frac;
        e = -1074;
        int msb = 63;
        while (!((m >> msb) & 1)) --msb;
        e2 = msb - 1074;
    } else {
        m = frac | (1ull << 52);
        e = bexp - 1075;
        e2 = bexp - 1023;
    }
    // X estimate: floor(e2 * log10(2)), then correct.
    int X = (e2 >= 0) ? (int)(((int64_t)e2 * 78913) >> 18)
                      : -(int)((((int64_t)-e2 * 78913) + (1 << 18) - 1) >> 18);
    uint64_t D = 0;
    int cls = 0;
    for (int iter = 0; iter < 4; ++iter) {
        D = ds_ratio(m, e, X - 5, &cls);
        if (D < 100000) --X;
        else if (D >= 1000000) ++X;
        else break;
    }
    if (cls > 0 || (cls == 0 && (D & 1))) ++D;   // round to nearest, ties to even
    if (D == 1000000) {
        D = 100000;
        ++X;
    }
    char dig[6];
    for (int i = 5; i >= 0; --i) {
        dig[i] = (char)('0' + D % 10);
        D /= 10;
    }
    int nd = 6;   // significant digits after dropping trailing zeros
    while (nd > 1 && dig[nd - 1] == '0') --nd;
    if (X >= -4 && X < 6) {
        if (X >= 0) {
            for (int i = 0; i <= X; ++i) out[n++] = dig[i];
            if (nd > X + 1) {
                out[n++] = '.';
                for (int i = X + 1; i < nd; ++i) out[n++] = dig[i];
            }
        } else {
            out[n++] = '0';
            out[n++] = '.';
            for (int i = 0; i < -X - 1; ++i) out[n++] = '0';
            for (int i = 0; i < nd; ++i) out[n++] = dig[i];
        }
    } else {
        out[n++] = dig[0];
        if (nd > 1) {
            out[n++] = '.';
            for (int i = 1; i < nd; ++i) out[n++] = dig[i];
        }
        out[n++] = 'e';
        int x = X;
        if (x < 0) {
            out[n++] = '-';
            x = -x;
        } else {
            out[n++] = '+';
        }
        if (x >= 100) {
            out[n++] = (char)('0' + x / 100);
            x %= 100;
            out[n++] = (char)('0' + x / 10);
            out[n++] = (char)('0' + x % 10);
        } else {
            out[n++] = (char)('0' + x / 10);
            out[n++] = (char)('0' + x % 10);
        }
    }
    return n;
}

// Unsigned / signed decimal (operator<< of integers in write_csv).
DS_FMT_HD int ds_fmt_u64(uint64_t v, char* out) {
    char t[20];
    int k = 0;
    do {
        t[k++] = (char)('0' + v % 10);
        v /= 10;
    } while (v);
    for (int i = 0; i < k; ++i) out[i] = t[k - 1 - i];
    return k;
}

DS_FMT_HD int ds_fmt_i64(int64_t v, char* out) {
    if (v < 0) {
        out[0] = '-';
        return 1 + ds_fmt_u64((uint64_t)0 - (uint64_t)v, out + 1);
    }
    return ds_fmt_u64((uint64_t)v, out);
}
