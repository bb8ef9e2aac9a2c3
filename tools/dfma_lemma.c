/* CPU check of the identity curve.cu's total_run relies on (K3):
 *   f = RN(t*d + 1)  (one rounding, fma)  ==  RN(RN(t*d) + 1)  (two roundings)
 * whenever f lies in [2^k + 1 + 2u, 2^(k+1) - 2u], 1 <= k <= 51, u = 2^(k-52),
 * and the run test built on it: a run of DFMA steps whose first and last
 * outputs lie in the interval of the SAME binade is exact step by step (the
 * DFMA map is monotone, so every output lies between the ends).
 * Prints "tested T bad 0 runs R bad 0" on success. Build with
 * gcc -O2 -ffp-contract=off tools/dfma_lemma.c -lm (no -march=native: the
 * two-rounding reference must not be contracted). */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static uint64_t bits(double x) { uint64_t b; memcpy(&b, &x, 8); return b; }
static int safe_binade(double f) {   /* curve.cu dfma_safe_binade */
    uint64_t b = bits(f);
    int k = (int)(b >> 52) - 1023;
    if (k < 1 || k > 51) return -1;
    uint64_t m = b & ((1ull << 52) - 1);
    return (m >= (1ull << (52 - k)) + 2 && m <= (1ull << 52) - 2) ? k : -1;
}
static double two_step(double t, double d) { volatile double p = t * d; volatile double x = p + 1.0; return x; }
static uint64_t s = 88172645463325252ull;
static double u01(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (s >> 11) * 0x1.0p-53; }

/* total_run of curve.cu, restated: runs of 32 DFMA steps, verified by their ends */
static double run(double t, long len, double d) {
    long k = 0;
    for (; k + 32 <= len; k += 32) {
        double t0 = t, prev = t, f1 = t;
        for (int u = 0; u < 32; ++u) { prev = t; t = fma(t, d, 1.0); if (u == 0) f1 = t; }
        int k1 = safe_binade(f1);
        int ok = k1 >= 0 && safe_binade(t) == k1;
        int fixed = bits(t) == bits(prev);
        if (!ok) {
            t = t0; fixed = 0;
            for (int u = 0; u < 32; ++u) { double x = two_step(t, d); fixed |= bits(x) == bits(t); t = x; }
        }
        if (fixed) return t;
    }
    for (; k < len; ++k) t = two_step(t, d);
    return t;
}

int main(int argc, char** argv) {
    long samples = argc > 1 ? atol(argv[1]) : 2000000;
    const double ds[] = {0.999, 0.5, 0.9999999, 1 - 0x1p-52, 0.75, 0.1, 0.99, 0.9990000000000001};
    long tested = 0, bad = 0, runs = 0, runbad = 0;
    for (int di = 0; di < 8; ++di) {
        const double d = ds[di];
        for (long i = 0; i < samples; ++i) {
            double t;
            switch (i % 4) {
            case 0: t = u01() * 2000; break;
            case 1: t = ldexp(1 + u01(), 1 + (int)(u01() * 51)); break;
            case 2: t = ldexp(1.0, 1 + (int)(u01() * 51)) + (u01() - 0.5) * 8; break;
            default: t = u01() * 1e15;
            }
            double f = fma(t, d, 1.0);
            if (safe_binade(f) >= 0) { ++tested; bad += bits(f) != bits(two_step(t, d)); }
        }
        for (int c = 0; c < 300; ++c) {   /* whole chains vs the sequential two-step replay */
            double t0 = (c % 3 == 0) ? (u01() - 0.5) * 200 : (c % 3 == 1) ? ldexp(u01(), (int)(u01() * 60) - 5)
                                                                          : 1.0 / (1.0 - d) * (1 + (u01() - 0.5) * 1e-9);
            long n = 1 + (long)(u01() * 6000);
            double a = t0;
            for (long k = 0; k < n; ++k) a = two_step(a, d);
            ++runs;
            runbad += bits(a) != bits(run(t0, n, d));
        }
    }
    printf("tested %ld bad %ld runs %ld bad %ld\n", tested, bad, runs, runbad);
    return bad || runbad;
}
