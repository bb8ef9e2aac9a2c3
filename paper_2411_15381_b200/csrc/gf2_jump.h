// Jump-ahead arithmetic for std::mt19937_64 (host): polynomials over GF(2)
// modulo the engine's characteristic polynomial phi (degree 19937,
// mt64_charpoly.h). With r(x) = x^J mod phi, the state J words ahead is the
// XOR of the states the set bits of r select (arrivals.cu, mt_jump_kernel).
// Checked against direct generation by tests/mt_jump_check.cpp.
#pragma once

#include <stdint.h>

#include <vector>

#include "mt64_charpoly.h"

using Poly = std::vector<uint64_t>;   // 312 words, degree < 19937

// a * b mod phi.
inline Poly poly_mulmod(const Poly& a, const Poly& b) {
    // carry-less product, 4-bit windows of a, then reduction by phi from the top
    std::vector<uint64_t> prod(626, 0);
    std::vector<uint64_t> tab(16 * 16 * 314, 0);   // tab[(shift/4) * 16 + nib] = (b*nib) << shift
    auto T = [&](int sh, int nib) { return &tab[(static_cast<size_t>(sh) * 16 + nib) * 314]; };
    for (int nib = 1; nib < 16; ++nib) {
        uint64_t* t = T(0, nib);
        for (int k = 0; k < 4; ++k)
            if ((nib >> k) & 1)
                for (int q = 0; q < 313; ++q) {
                    const uint64_t lo = q < 312 ? b[q] << k : 0;
                    const uint64_t hi = (q > 0 && k) ? b[q - 1] >> (64 - k) : 0;
                    t[q] ^= lo | hi;
                }
        for (int sh = 1; sh < 16; ++sh) {
            const uint64_t* t0 = T(0, nib);
            uint64_t* ts = T(sh, nib);
            const int bs = 4 * sh;
            for (int q = 0; q < 314; ++q)
                ts[q] = (q < 313 ? t0[q] << bs : 0) | (q > 0 ? t0[q - 1] >> (64 - bs) : 0);
        }
    }
    for (int q = 0; q < 312; ++q) {
        const uint64_t w = a[q];
        if (!w) continue;
        for (int sh = 0; sh < 16; ++sh) {
            const int nib = static_cast<int>((w >> (4 * sh)) & 15u);
            if (!nib) continue;
            const uint64_t* t = T(sh, nib);
            for (int k = 0; k < 314 && q + k < 626; ++k) prod[q + k] ^= t[k];
        }
    }
    // reduce bits 39872 .. 19937 with phi's set bits (phi is sparse: 285 terms)
    static const std::vector<int> terms = [] {
        std::vector<int> t;
        for (int k = 0; k < 19937; ++k)
            if ((kMt64CharPoly[k / 64] >> (k % 64)) & 1u) t.push_back(k);
        return t;
    }();
    for (int k = 626 * 64 - 1; k >= 19937; --k) {
        if (!((prod[k / 64] >> (k % 64)) & 1u)) continue;
        prod[k / 64] ^= 1ull << (k % 64);
        const int d = k - 19937;
        for (int t : terms) prod[(d + t) / 64] ^= 1ull << ((d + t) % 64);
    }
    prod.resize(312);
    prod[311] &= (1ull << (19937 - 311 * 64)) - 1;
    return prod;
}

// x^m mod phi by squaring (x^(2k) = (x^k)^2) and shifts.
inline Poly poly_xpow(int64_t m) {
    Poly r(312, 0);
    r[0] = 1;   // x^0
    bool one = true;   // r == 1: squaring it is a no-op
    for (int bit = 62; bit >= 0; --bit) {
        if (!one) r = poly_mulmod(r, r);
        if ((m >> bit) & 1) one = false;
        if ((m >> bit) & 1) {   // multiply by x: shift left by one, reduce bit 19937
            uint64_t carry = 0;
            for (int q = 0; q < 312; ++q) {
                const uint64_t nc = r[q] >> 63;
                r[q] = (r[q] << 1) | carry;
                carry = nc;
            }
            const bool top = (r[311] >> (19937 - 311 * 64)) & 1u;
            r[311] &= (1ull << (19937 - 311 * 64)) - 1;
            if (top)
                for (int q = 0; q < 312; ++q) r[q] ^= kMt64CharPoly[q];
            r[311] &= (1ull << (19937 - 311 * 64)) - 1;
        }
    }
    return r;
}

