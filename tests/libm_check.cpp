// CPU check of paper_2411_15381_b200/csrc/glibc_libm.h against the host libm
// (the reference's log/cos): counts bit mismatches over seeded samples of the
// reference's own argument distributions and of wide random arguments.
//   g++ -std=c++17 -O2 -ffp-contract=off -I<csrc> libm_check.cpp -o x && ./x [n]
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>

#include "glibc_libm.h"

static uint64_t bits(double x) {
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
}
static double dbl(uint64_t u) {
    double x;
    std::memcpy(&x, &u, 8);
    return x;
}

int main(int argc, char** argv) {
    const long n = argc > 1 ? std::atol(argv[1]) : (1L << 24);
    std::mt19937_64 rng(20261017);
    long bad_log = 0, bad_cos = 0, cnt_log = 0, cnt_cos = 0;
    auto check_log = [&](double x) {
        ++cnt_log;
        const double w = std::log(x), g = glibc_log(x);
        if (bits(w) != bits(g) && !(std::isnan(w) && std::isnan(g))) {
            if (bad_log < 5) std::printf("log mismatch x=%a want=%a got=%a\n", x, w, g);
            ++bad_log;
        }
    };
    auto check_cos = [&](double x) {
        ++cnt_cos;
        const double w = std::cos(x), g = glibc_cos(x);
        if (bits(w) != bits(g) && !(std::isnan(w) && std::isnan(g))) {
            if (bad_cos < 5) std::printf("cos mismatch x=%a want=%a got=%a\n", x, w, g);
            ++bad_cos;
        }
    };
    const double two_pi = 2.0 * M_PI;
    for (long i = 0; i < n; ++i) {
        // the reference's draws: u = (r >> 11) * 2^-53, log(u1), cos(2 pi u2)
        double u1 = static_cast<double>(rng() >> 11) * 0x1.0p-53;
        if (u1 <= 0.0) u1 = 0x1.0p-53;
        check_log(u1);
        check_cos(two_pi * (static_cast<double>(rng() >> 11) * 0x1.0p-53));
    }
    for (long i = 0; i < n / 4; ++i) {
        // wide arguments: any positive finite double; |x| < 1e8 for cos
        const uint64_t r = rng();
        const double x = dbl(r & 0x7fefffffffffffffull);
        if (x > 0.0) check_log(x);
        const double y = (static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5) * 2e8;
        check_cos(y);
        check_log(1.0 + (static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5) * 0.25);
        check_cos((static_cast<double>(rng() >> 11) * 0x1.0p-53 - 0.5) * 8.0);
    }
    // edges: powers of two, subnormals, the branch boundaries of both functions
    for (int e = -1074; e <= 1023; ++e) check_log(std::ldexp(1.0, e));
    const double edges[] = {0x1.0p-27, 0x1.fffffffffffffp-28, 0.855469, 0.85546875, 2.426265,
                            0x1.368fcp+1, M_PI / 2, M_PI, 3 * M_PI / 2, two_pi, 0.126, 1.0, 0.0};
    for (double e : edges)
        for (int d = -64; d <= 64; ++d) {
            check_cos(dbl(bits(e) + d));
            check_cos(-dbl(bits(e) + d));
            if (e > 0) check_log(dbl(bits(e) + d));
        }
    std::printf("log: %ld / %ld bit mismatches; cos: %ld / %ld bit mismatches\n", bad_log, cnt_log,
                bad_cos, cnt_cos);
    return bad_log || bad_cos ? 1 : 0;
}
