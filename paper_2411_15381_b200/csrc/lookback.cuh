// Decoupled look-back (single-pass prefix over the tiles of a grid), shared
// by K2 (route.cu: deferral counts) and K9 (csv.cu: row bytes).
//
// Tile t of a sequence publishes its aggregate (status A) as soon as it knows
// it, then one warp reads the 128 nearest unread predecessors' flags at once
// back to the nearest inclusive prefix (status P) and publishes its own P. A
// flag word is [status:2 | value:62]. Tiles are blockIdx.x in dispatch order,
// so every predecessor is running or done. The last CTA to retire (a done
// counter) zeroes the flags it used, so every launch -- eager or replayed from
// a CUDA graph -- starts from clean flags without a memset.
#pragma once

#include <cstdint>

namespace dslb {

constexpr unsigned long long kValBits = 62, kValMask = (1ull << kValBits) - 1;
constexpr unsigned long long kStatusA = 1, kStatusP = 2;

__device__ __forceinline__ unsigned long long flag_word(unsigned long long st, long long v) {
    return (st << kValBits) | (static_cast<unsigned long long>(v) & kValMask);
}
__device__ __forceinline__ void flag_store(unsigned long long* p, unsigned long long w) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long flag_load(const unsigned long long* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}

// Exclusive prefix of this tile's count over tiles [0, tile) of one sequence
// (one warp; every lane returns it). Each round covers the 128 nearest
// unread predecessors (4 per lane at distances 4*lane + q, all loads in
// flight together) and stops at the nearest inclusive prefix (P); tiles
// without one contribute their aggregate (A). Only the flags up to the
// nearest P must be published: a round re-polls while an unpublished flag is
// nearer than every P it has seen, so a tile never waits for predecessors
// beyond the P it stops at (formatting tiles, K9, finish far out of order).
__device__ __forceinline__ long long look_back(const unsigned long long* flags, int tile) {
    const int lane = threadIdx.x & 31;
    long long excl = 0;
    for (int base = tile - 1;; base -= 128) {
        unsigned long long st[4], val[4];
        unsigned ready = 0;   // bit q: flag q read (all four loads in flight together)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            st[q] = kStatusP;
            val[q] = 0;
            if (base - (4 * lane + q) < 0) ready |= 1u << q;   // before tile 0: P of 0
        }
        int first_p = 4;   // nearest P among this lane's four, once read
        for (;;) {
            unsigned long long w[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (!((ready >> q) & 1u)) w[q] = flag_load(flags + (base - (4 * lane + q)));
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (!((ready >> q) & 1u) && (w[q] >> kValBits) != 0) {
                    st[q] = (w[q] >> kValBits) & 3ull;
                    val[q] = w[q] & kValMask;
                    ready |= 1u << q;
                }
            // distance 4*lane + q: the nearest unpublished flag and the
            // nearest P of the window (lane-major order = distance order)
            int lane_nr = 4, lane_p = 4;
#pragma unroll
            for (int q = 3; q >= 0; --q) {
                if (!((ready >> q) & 1u)) lane_nr = q;
                if (((ready >> q) & 1u) && st[q] == kStatusP) lane_p = q;
            }
            const unsigned nr_mask = __ballot_sync(0xffffffffu, lane_nr < 4);
            const unsigned p_mask = __ballot_sync(0xffffffffu, lane_p < 4);
            const int nr = nr_mask ? 4 * (__ffs(nr_mask) - 1) + __shfl_sync(0xffffffffu, lane_nr, __ffs(nr_mask) - 1) : 128;
            const int np = p_mask ? 4 * (__ffs(p_mask) - 1) + __shfl_sync(0xffffffffu, lane_p, __ffs(p_mask) - 1) : 128;
            if (np < nr || (nr == 128)) {   // everything up to the nearest P (or the window) known
                first_p = np;
                break;
            }
        }
        long long v = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (4 * lane + q <= first_p && 4 * lane + q < 128) v += static_cast<long long>(val[q]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (first_p < 128) return excl;
    }
}

// Every CTA's look-back reads are done when it retires; the last of the
// launch zeroes the [gridDim.y][tiles] flags and the counter for the next
// launch (block-uniform call, all threads).
__device__ __forceinline__ void retire(unsigned long long* flags, unsigned* done, int tiles) {
    if (tiles == 1) return;   // a single tile per threshold uses no flags
    __shared__ bool s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned total = gridDim.x * gridDim.y;
        s_last = atomicAdd(done, 1u) == total - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const long long words = static_cast<long long>(tiles) * gridDim.y;
    for (long long i = threadIdx.x; i < words; i += blockDim.x) flags[i] = 0ull;
    if (threadIdx.x == 0) *done = 0u;
}


} // namespace dslb
