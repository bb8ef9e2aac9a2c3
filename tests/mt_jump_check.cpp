// CPU check of csrc/gf2_jump.h: the std::mt19937_64 state J words ahead,
// computed as the XOR of the states the set bits of x^J mod phi select, equals
// direct generation (all 312 words; the oldest word's upper 33 bits, the only
// ones the recurrence reads), for jumps of 1..6 segments of 20,480 words and a
// few odd lengths; and the engine's outputs from the jumped state match
// std::mt19937_64 itself.
#include <cstdint>
#include <cstdio>
#include <random>
#include <vector>

#include "gf2_jump.h"

int main() {
    const uint64_t seed = 0x9e3779b97f4a7c15ULL;
    const int L = 20480, S = 6;
    std::vector<uint64_t> x(312 + (S + 2) * L + 400);
    x[0] = seed;
    for (int i = 1; i < 312; ++i) x[i] = 6364136223846793005ULL * (x[i - 1] ^ (x[i - 1] >> 62)) + i;
    for (size_t k = 312; k < x.size(); ++k) {
        const uint64_t y = (x[k - 312] & 0xFFFFFFFF80000000ULL) | (x[k - 311] & 0x7FFFFFFFULL);
        x[k] = x[k - 156] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    // the raw words are std::mt19937_64's untempered state words
    std::mt19937_64 eng(seed);
    auto temper = [](uint64_t z) {
        z ^= (z >> 29) & 0x5555555555555555ULL;
        z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
        z ^= (z << 37) & 0xFFF7EEE000000000ULL;
        return z ^ (z >> 43);
    };
    for (int k = 0; k < 1000; ++k)
        if (eng() != temper(x[312 + k])) {
            std::printf("raw word %d is not the engine's\n", k);
            return 1;
        }
    int bad = 0;
    auto check = [&](int64_t J, const Poly& r) {
        for (int j = 0; j < 312; ++j) {
            uint64_t acc = 0;
            for (int i = 0; i < 19937; ++i)
                if ((r[i / 64] >> (i % 64)) & 1u) acc ^= x[i + j];
            uint64_t want = x[J + j];
            if (j == 0) {
                acc &= 0xFFFFFFFF80000000ULL;
                want &= 0xFFFFFFFF80000000ULL;
            }
            bad += acc != want;
        }
    };
    const Poly pL = poly_xpow(L);
    Poly p = pL;
    for (int s = 1; s <= S; ++s) {
        check(static_cast<int64_t>(s) * L, p);
        p = poly_mulmod(p, pL);
    }
    for (int64_t J : {1, 311, 312, 19937, 30001})
        if (J + 312 < static_cast<int64_t>(x.size())) check(J, poly_xpow(J));
    std::printf("jump-ahead: %d state words differ\n", bad);
    return bad ? 1 : 0;
}
