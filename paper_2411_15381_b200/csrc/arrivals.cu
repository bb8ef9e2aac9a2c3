// K8 arrivals: diffserve::generate_arrivals (reference proj/src/workload.cpp:82-106)
// on the device, bit-identical to the reference.
//
// The reference walks the trace's piecewise-linear cumulative rate R(t) with a
// running target (0, 1, 2, ... for uniform arrivals; a sum of Exp(1) draws from
// one RandomStream(seed, "arrivals") for Poisson) and emits
//     t = start_k + (target - cum_k) / rate_k
// in the first positive-rate interval k with target < cum_end_k - 1e-12, nudged
// to nextafter(previous, +inf) when it does not increase, and stops at the
// first t >= duration. Every piece is restated as a data-parallel pass:
//
//   K8a mt_stream   the single std::mt19937_64 stream. Word m obeys
//                   x_m = x_{m-156} ^ twist(x_{m-312}, x_{m-311}); a CTA
//                   generates it with thread c on column c (mod 156), two
//                   steps of 156 words per barrier. Long streams (round 2)
//                   are cut into segments of 20,480 words: segment 0 as
//                   above, every other segment on its own SM from its start
//                   state, computed by JUMP-AHEAD -- x^J mod phi over GF(2)
//                   (phi = the engine's characteristic polynomial, degree
//                   19937; gf2_jump.h, host, cached) selects which of the
//                   first 19,937 states XOR to the state J words ahead.
//                   A segment's jump is split over a cluster of 3 CTAs
//                   (partial states XORed over distributed shared memory).
//                   1M arrivals 0.70 -> 0.32 ms.
//   K8b exp_draws   grid-wide: temper, U = (u64 >> 11) * 2^-53,
//                   e = -log1p(-U) with glibc's log1p restated bit for bit
//                   (fdlibm_log1p.h; rng.cpp:24-28).
//   K8c target_sum  one CTA: the sequentially rounded running sum
//                   T_i = fl(T_{i-1} + e_i) as an EXACT integer scan. While the
//                   accumulator stays in one binade [2^p, 2^(p+1)) with ulp u,
//                   fl(M*u + e) = (M + rint(e/u)) * u, so a tile of 8192 steps is
//                   an int64 prefix sum (no int<->double conversions: M and
//                   the results are the accumulator's own bit patterns). The first step that could leave the
//                   binade (or is a rounding tie, whose direction depends on the
//                   accumulator's parity) is done as one real fp64 add and the
//                   tile restarts after it: ~log2(N) restarts in total.
//   K8d place       grid-wide: interval k by binary search over the positive-rate
//                   intervals' thresholds (targets and thresholds are both
//                   nondecreasing, so the first k that admits target i is the
//                   reference's k), t_i in the reference's operation order, and
//                   key_i = ord(t_i) - i where ord() maps doubles to int64 in
//                   order with nextafter(x, +inf) == ord(x) + 1.
//   K8e/K8f         the nextafter fix is t'_i = max(t_i, next(t'_{i-1})), i.e.
//                   ord(t'_i) = max_{j<=i} key_j + i: a max-scan (block maxima,
//                   one-block carry scan, in-block scan); the first t'_i >=
//                   duration ends the walk.
//
// Interval tables (cum, start, threshold) are O(#intervals) sequential fp64
// sums and are built on the host in the reference's order.
#include <cuda_runtime.h>

#include <climits>
#include <cmath>
#include <cstdlib>
#include <limits>
#include <mutex>
#include <vector>

#include "ds_internal.h"
#include "fdlibm_log1p.h"
#include "gf2_jump.h"

namespace {

constexpr int kPlaceThreads = 512;
constexpr long long kNoIndex = 0x7fffffffffffffffLL;

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {   // rng.cpp:8-13
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

uint64_t fnv1a(const char* s) {                                          // rng.cpp:15-22
    uint64_t h = 0xcbf29ce484222325ULL;
    for (; *s; ++s) {
        h ^= static_cast<unsigned char>(*s);
        h *= 0x100000001b3ULL;
    }
    return h;
}

__device__ __forceinline__ uint64_t mt_mix(uint64_t xk, uint64_t xk1) {
    const uint64_t y = (xk & 0xFFFFFFFF80000000ULL) | (xk1 & 0x7FFFFFFFULL);
    return (y >> 1) ^ ((y & 1ULL) ? 0xB5026F5AA96619E9ULL : 0ULL);
}

__device__ __forceinline__ uint64_t temper(uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

// ---- K8a: the single mt19937_64 stream, untempered words x_312 .. -----------
// raw[k] = x_{312+k}; output k of the engine is temper(raw[k]). Thread c owns
// column c (mod 156) and keeps its last two words in registers; the only
// cross-thread input, x_{m-311} (column c+1 two steps back; column 0 one step
// back for c = 155), comes from a 4-step shared ring. Two steps per barrier:
// the second step's neighbour for c = 155 (column 0 of the first new step) is
// recomputed by that thread from words already in the ring.
constexpr int kMtThreads = 160;

// From the 312 words preceding raw[base] in ring[0..1] (ring[0][c] =
// x_{base+c}, ring[1][c] = x_{base+156+c}), writes raw[base + k] for
// k < count and base + k < n. Block-uniform (all kMtThreads threads).
__device__ __forceinline__ void mt_run(uint64_t (&ring)[4][156], int64_t base, int64_t count,
                                       int64_t n, uint64_t* __restrict__ raw) {
    const int c = threadIdx.x;
    const bool active = c < 156;
    uint64_t x2 = active ? ring[0][c] : 0;   // step s
    uint64_t x1 = active ? ring[1][c] : 0;   // step s+1
    const int64_t steps = (count + 155) / 156;
    for (int64_t s = 0; s < steps; s += 2) {
        const int a = static_cast<int>(s & 3), b = (a + 1) & 3, w0 = (a + 2) & 3, w1 = (a + 3) & 3;
        if (active) {
            uint64_t nb_a, nb_b;
            if (c < 155) {
                nb_a = ring[a][c + 1];   // column c+1, step s
                nb_b = ring[b][c + 1];   // column c+1, step s+1
            } else {
                nb_a = ring[b][0];       // column 0, step s+1
                // column 0 of step s+2, recomputed: x_{m-156} ^ twist(x_{m-312}, x_{m-311})
                nb_b = ring[b][0] ^ mt_mix(ring[a][0], ring[a][1]);
            }
            const uint64_t y0 = x1 ^ mt_mix(x2, nb_a);   // step s+2
            const uint64_t y1 = y0 ^ mt_mix(x1, nb_b);   // step s+3
            ring[w0][c] = y0;
            ring[w1][c] = y1;
            const int64_t k0 = s * 156 + c;
            if (k0 < count && base + k0 < n) raw[base + k0] = y0;
            if (k0 + 156 < count && base + k0 + 156 < n) raw[base + k0 + 156] = y1;
            x2 = y0;
            x1 = y1;
        }
        __syncthreads();
    }
}

// std::mt19937_64 seeding recurrence (x_0 .. x_311) into ring[0..1].
__device__ __forceinline__ void mt_seed(uint64_t seed, uint64_t (&ring)[4][156]) {
    if (threadIdx.x == 0) {
        uint64_t x = seed;
        ring[0][0] = x;
        for (int i = 1; i < 312; ++i) {
            x = 6364136223846793005ULL * (x ^ (x >> 62)) + static_cast<uint64_t>(i);
            ring[i / 156][i % 156] = x;
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(kMtThreads) mt_stream_kernel(uint64_t seed, int64_t count,
                                                               int64_t n,
                                                               uint64_t* __restrict__ raw) {
    __shared__ uint64_t ring[4][156];   // ring[step & 3][column]
    mt_seed(seed, ring);
    mt_run(ring, 0, count, n, raw);
}

// Jump-ahead: segment s >= 1 of kJumpSeg words starts from the state
// x_{J} .. x_{J+311}, J = s * kJumpSeg. The engine's words obey the linear
// recurrence of its characteristic polynomial phi (degree 19937,
// mt64_charpoly.h), so with r(x) = x^J mod phi (host, cached),
//     x_{J+j} = XOR over the set bits i of r of x_{i+j},   j = 0 .. 311
// (all 64 bits for j >= 1; only x_J's upper 33 bits, the ones the recurrence
// reads, for j = 0). One CTA per segment: the base words x_0 .. x_20247 (the
// seed words and segment 0's output) in shared memory, thread j XORs the
// words the set bits of r select (a warp-uniform walk of r), then the
// segment's words are generated as in mt_stream. Checked bit for bit against
// the single stream (tests/test_gpu_arrivals.py).
constexpr int kJumpSeg = 20480;                   // >= 19937: segment 0 holds the base words
constexpr int kJumpBase = 19937 + 312;            // x_0 .. x_20248
constexpr int kJumpGroups = 3;                    // thread groups per CTA
constexpr int kJumpSplit = 3;                     // CTAs (a cluster) per segment
constexpr int kJumpThreads = 320 * kJumpGroups;   // 312 state words per group
constexpr int kJumpMaxBits = 19937;
constexpr int kJumpSmem = (kJumpBase + kJumpGroups * 312) * 8 + kJumpMaxBits * 2 + 16;

__device__ __forceinline__ unsigned jump_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void jump_cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                 "barrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// a 64-bit word of CTA `rank`'s shared memory at this CTA's address `p`
__device__ __forceinline__ uint64_t jump_peer_load(const uint64_t* p, unsigned rank) {
    uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(p)), ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(rank));
    uint64_t v;
    asm volatile("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(ra) : "memory");
    return v;
}

// idx: the exponents i of r's set bits (uint16, ascending), segment s at
// idx[off[s-1] .. off[s]). A cluster of kJumpSplit CTAs per segment: CTA c
// sums the c-th third of the set bits (its thread groups every third of
// those), the leader XORs the partial states over distributed shared memory
// and generates the segment.
__global__ void __launch_bounds__(kJumpThreads)
mt_jump_kernel(uint64_t seed, const uint16_t* __restrict__ idx, const int* __restrict__ off,
               int64_t n, uint64_t* __restrict__ raw) {
    extern __shared__ uint64_t jw[];   // x_0 .. x_{kJumpBase-1} | partial sums | indices
    __shared__ uint64_t ring[4][156];
    uint64_t* part = jw + kJumpBase;
    uint16_t* si = reinterpret_cast<uint16_t*>(part + kJumpGroups * 312);
    const unsigned rank = jump_rank();
    const int s = blockIdx.x / kJumpSplit + 1, tid = threadIdx.x;
    const int i0 = off[s - 1], all = off[s] - i0;
    const int lo = static_cast<int>(static_cast<int64_t>(all) * rank / kJumpSplit);
    const int nbits = static_cast<int>(static_cast<int64_t>(all) * (rank + 1) / kJumpSplit) - lo;
    mt_seed(seed, ring);
    for (int i = tid; i < 312; i += kJumpThreads) jw[i] = ring[i / 156][i % 156];
    for (int i = 312 + tid; i < kJumpBase; i += kJumpThreads) jw[i] = raw[i - 312];
    for (int i = tid; i < nbits; i += kJumpThreads) si[i] = idx[i0 + lo + i];
    __syncthreads();
    const int g = tid / 320, j = tid % 320;
    if (j < 312) {
        uint64_t a0 = 0, a1 = 0;
        const uint64_t* wj = jw + j;
        int k = g;
        for (; k + kJumpGroups < nbits; k += 2 * kJumpGroups) {
            a0 ^= wj[si[k]];
            a1 ^= wj[si[k + kJumpGroups]];
        }
        if (k < nbits) a0 ^= wj[si[k]];
        part[g * 312 + j] = a0 ^ a1;
    }
    __syncthreads();
    if (tid < 312) part[tid] ^= part[312 + tid] ^ part[624 + tid];   // this CTA's share
    jump_cluster_sync();
    if (rank == 0 && tid < 312) {
        uint64_t v = part[tid];
        for (unsigned c = 1; c < kJumpSplit; ++c) v ^= jump_peer_load(part + tid, c);
        ring[tid / 156][tid % 156] = v;
    }
    jump_cluster_sync();   // the peers' shared memory was read
    if (rank != 0) return;
    mt_run(ring, static_cast<int64_t>(s) * kJumpSeg, kJumpSeg, n, raw);
}

std::mutex g_jump_mu;
std::vector<Poly> g_jump;   // g_jump[s-1] = x^(s * kJumpSeg) mod phi (process cache)

// The jump polynomials' set-bit exponents for segments 1 .. S-1 on the
// device (context cache; at least 64 segments, ~20 KB each).
ds_status jump_lists(ds_ctx* ctx, int S, const uint16_t** idx, const int** off) {
    std::lock_guard<std::mutex> lock(g_jump_mu);
    if (ctx->jump_polys_n < S - 1) {
        const int want = S - 1 < 64 ? 64 : S - 1;
        if (g_jump.empty()) g_jump.push_back(poly_xpow(kJumpSeg));
        while (static_cast<int>(g_jump.size()) < want)
            g_jump.push_back(poly_mulmod(g_jump.back(), g_jump.front()));
        std::vector<uint16_t> bits;
        std::vector<int> offs(1, 0);
        for (int i = 0; i < want; ++i) {
            for (int k = 0; k < kJumpMaxBits; ++k)
                if ((g_jump[i][k / 64] >> (k % 64)) & 1u) bits.push_back(static_cast<uint16_t>(k));
            offs.push_back(static_cast<int>(bits.size()));
        }
        if (ctx->jump_polys) {
            DS_CUDA_TRY(cudaDeviceSynchronize());
            DS_CUDA_TRY(cudaFree(ctx->jump_polys));
            ctx->jump_polys = nullptr;
            ctx->jump_polys_n = 0;
        }
        const size_t bo = dsi::align_up(sizeof(int) * offs.size(), 256);
        DS_CUDA_TRY(cudaMalloc(&ctx->jump_polys, bo + sizeof(uint16_t) * bits.size()));
        DS_CUDA_TRY(cudaMemcpy(ctx->jump_polys, offs.data(), sizeof(int) * offs.size(),
                               cudaMemcpyHostToDevice));
        DS_CUDA_TRY(cudaMemcpy(static_cast<char*>(ctx->jump_polys) + bo, bits.data(),
                               sizeof(uint16_t) * bits.size(), cudaMemcpyHostToDevice));
        ctx->jump_polys_n = want;
        ctx->jump_idx_offset = bo;
    }
    *off = static_cast<const int*>(ctx->jump_polys);
    *idx = reinterpret_cast<const uint16_t*>(static_cast<const char*>(ctx->jump_polys) +
                                             ctx->jump_idx_offset);
    return DS_OK;
}

// raw[0 .. n): the engine's untempered words x_312 .. (one stream; K8a).
ds_status mt_stream(ds_ctx* ctx, uint64_t seed, int64_t n, uint64_t* raw, cudaStream_t st) {
    static const bool no_jump = std::getenv("DS_ARRIVALS_NO_JUMP") != nullptr;   // A/B
    if (no_jump || n <= 2 * kJumpSeg) {
        mt_stream_kernel<<<1, kMtThreads, 0, st>>>(seed, n, n, raw);
        DS_LAUNCH_CHECK(ctx, "mt_stream_kernel");
        return DS_OK;
    }
    const int S = static_cast<int>((n + kJumpSeg - 1) / kJumpSeg);
    const uint16_t* idx = nullptr;
    const int* off = nullptr;
    ds_status s = jump_lists(ctx, S, &idx, &off);
    if (s != DS_OK) return s;
    mt_stream_kernel<<<1, kMtThreads, 0, st>>>(seed, kJumpSeg, n, raw);   // segment 0
    DS_LAUNCH_CHECK(ctx, "mt_stream_kernel");
    if (!(ctx->route_attr_set & (1u << 20))) {
        DS_CUDA_TRY(cudaFuncSetAttribute(mt_jump_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kJumpSmem));
        ctx->route_attr_set |= 1u << 20;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>((S - 1) * kJumpSplit));
    cfg.blockDim = dim3(kJumpThreads);
    cfg.dynamicSmemBytes = kJumpSmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kJumpSplit;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, mt_jump_kernel, seed, idx, off, n, raw));
    DS_LAUNCH_CHECK(ctx, "mt_jump_kernel");
    return DS_OK;
}

// ---- K8b: Exp(1) variates -----------------------------------------------------
// RandomStream::exponential(1.0) = -log1p(-uniform()) / 1.0 (rng.cpp:24-28); the
// division by 1.0 is an exact identity and is dropped.
// raw and e are the same buffer (each element is replaced in place).
__global__ void __launch_bounds__(256) exp_draws_kernel(const uint64_t* raw, int64_t n,
                                                        double* e) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += stride) {
        const double u = __dmul_rn(static_cast<double>(temper(raw[i]) >> 11), 0x1.0p-53);
        e[i] = -ds_log1p(-u);
    }
}

// ---- K8c: exact sequentially rounded running sum -----------------------------
// The accumulator acc = M * 2^(p-52), M in [2^52, 2^53), is kept as its bit
// pattern: M is the mantissa with the hidden bit and any P in [2^52, 2^53)
// maps back to the double with the same exponent field, so the scan never
// converts between integers and doubles. Each thread scans 16 consecutive
// steps; tiles move through shared memory (padded, double-buffered) so global
// loads and stores stay coalesced.
constexpr int kSumThreads = 512;
constexpr int kSumPer = 16;
constexpr int kSumTile = kSumThreads * kSumPer;
constexpr int kSumPad = kSumTile + kSumTile / kSumPer;   // one pad slot per 16
constexpr size_t kSumSmem = 2 * kSumPad * sizeof(double);

__device__ __forceinline__ int pad_idx(int x) { return x + x / kSumPer; }

__device__ __forceinline__ double from_binade(unsigned long long P, unsigned long long ebits) {
    return __longlong_as_double(static_cast<long long>(ebits + (P - (1ULL << 52))));
}

// striped (coalesced) global loads of the tile starting at `start`
__device__ __forceinline__ void load_striped(const double* __restrict__ e, int64_t n,
                                             int64_t start, double (&v)[kSumPer]) {
#pragma unroll
    for (int q = 0; q < kSumPer; ++q) {
        const int64_t j = start + q * kSumThreads + threadIdx.x;
        v[q] = j < n ? __ldcg(e + j) : 0.0;
    }
}

__global__ void __launch_bounds__(kSumThreads, 1)
target_sum_kernel(const double* __restrict__ e, int64_t n, double* __restrict__ T,
                  const int* __restrict__ only_if) {
    if (only_if && !*only_if) return;   // the grid-wide pass succeeded
    extern __shared__ double sbuf_all[];
    __shared__ unsigned long long s_wsum[2][kSumThreads / 32];
    __shared__ unsigned s_wmin[2][kSumThreads / 32];
    __shared__ double s_acc;
    constexpr int kWarps = kSumThreads / 32;
    constexpr unsigned long long kLimit = (1ULL << 53) - 2;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    double acc = __ldcg(e);
    if (tid == 0) T[0] = acc;
    int64_t i = 1;
    int par = 0;
    double st[kSumPer];   // striped values of the tile at i
    load_striped(e, n, i, st);
    while (i < n) {
        double* sbuf = sbuf_all + par * kSumPad;
        const int tile_len = (n - i < kSumTile) ? static_cast<int>(n - i) : kSumTile;
#pragma unroll
        for (int q = 0; q < kSumPer; ++q) sbuf[pad_idx(q * kSumThreads + tid)] = st[q];
        // speculative prefetch of the next tile (correct unless a restart happens)
        load_striped(e, n, i + kSumTile, st);
        __syncthreads();
        double ev[kSumPer];
#pragma unroll
        for (int q = 0; q < kSumPer; ++q) ev[q] = sbuf[pad_idx(tid * kSumPer + q)];

        const unsigned long long ab = static_cast<unsigned long long>(__double_as_longlong(acc));
        const int bexp = static_cast<int>(ab >> 52);             // acc >= 0
        const bool scan_ok = bexp >= 1023 - 60 && bexp <= 1023 + 500;
        const unsigned long long ebits = static_cast<unsigned long long>(bexp) << 52;
        const unsigned long long M = (ab & ((1ULL << 52) - 1)) | (1ULL << 52);
        // 2^(52-p), p = bexp - 1023
        const double scale =
            __longlong_as_double(static_cast<long long>(scan_ok ? 2098 - bexp : 1023) << 52);
        unsigned long long r[kSumPer];
        unsigned long long mine = 0;
        int bad_q = kSumPer;
#pragma unroll
        for (int q = 0; q < kSumPer; ++q) {
            const double y = __dmul_rn(ev[q], scale);           // exact power-of-two scaling
            const double t = __dadd_rn(y, 0x1.0p52);            // rint(y), ties to even
            const unsigned long long rr = static_cast<unsigned long long>(__double_as_longlong(t)) -
                                          0x4330000000000000ULL;
            const double d = __dsub_rn(__dsub_rn(t, 0x1.0p52), y);   // exact
            const bool bad = !scan_ok || !(y < 0x1.0p52) || d == 0.5 || d == -0.5;
            const bool in = tid * kSumPer + q < tile_len;
            if (in && bad && bad_q == kSumPer) bad_q = q;
            r[q] = (in && !bad) ? rr : 0;
            mine += r[q];
        }
        // block exclusive scan of the per-thread sums
        unsigned long long inc = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) s_wsum[par][warp] = inc;
        __syncthreads();
        const unsigned long long wv = lane < kWarps ? s_wsum[par][lane] : 0;
        unsigned long long wi = wv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        const unsigned long long wex = __shfl_sync(0xffffffffu, wi - wv, warp);
        const unsigned long long tot = __shfl_sync(0xffffffffu, wi, 31);
        const unsigned long long excl = wex + inc - mine;
        // first step that is a tie, out of range, or could leave the binade
        unsigned vloc = 0xffffffffu;
        unsigned long long P = M + excl;
#pragma unroll
        for (int q = 0; q < kSumPer; ++q) {
            P += r[q];
            const bool in = tid * kSumPer + q < tile_len;
            if (in && (q == bad_q || P > kLimit) && vloc == 0xffffffffu)
                vloc = static_cast<unsigned>(tid * kSumPer + q);
        }
        const unsigned wmin = __reduce_min_sync(0xffffffffu, vloc);
        if (lane == 0) s_wmin[par][warp] = wmin;
        __syncthreads();
        const unsigned v = __reduce_min_sync(0xffffffffu,
                                             lane < kWarps ? s_wmin[par][lane] : 0xffffffffu);
        // T for the steps before v back into shared memory (blocked), the one
        // real add fl(T_{v-1} + e_v) by v's owner
        P = M + excl;
        double prev = tid == 0 ? acc : from_binade(P, ebits);
#pragma unroll
        for (int q = 0; q < kSumPer; ++q) {
            const unsigned rel = static_cast<unsigned>(tid * kSumPer + q);
            if (rel == v) {
                const double t = __dadd_rn(rel == 0 ? acc : prev, ev[q]);
                sbuf[pad_idx(rel)] = t;
                s_acc = t;
            }
            P += r[q];
            prev = from_binade(P, ebits);
            if (rel < v) sbuf[pad_idx(rel)] = prev;
        }
        __syncthreads();
        const int nout = v < static_cast<unsigned>(tile_len) ? static_cast<int>(v) + 1 : tile_len;
#pragma unroll
        for (int q = 0; q < kSumPer; ++q) {
            const int rel = q * kSumThreads + tid;
            if (rel < nout) T[i + rel] = sbuf[pad_idx(rel)];
        }
        par ^= 1;
        if (v < static_cast<unsigned>(tile_len)) {
            acc = s_acc;
            i += static_cast<int64_t>(v) + 1;
            load_striped(e, n, i, st);
        } else {
            acc = from_binade(M + tot, ebits);
            i += tile_len;
        }
    }
}

// ---- K8c, grid-wide: the same exact running sum without the single SM ------
// (1) an approximate fp64 prefix sum A_i of the draws (block sums, one-block
//     scan of the block sums, in-block scans) fixes the binade p_i of every
//     accumulator T_{i-1}; A differs from the sequentially rounded T by at
//     most ~D ulps, so outside a margin around powers of two the binade is the
//     true one;
// (2) each step outside the margin, with no rounding tie and staying in its
//     binade, adds the exact integer r_i = rint(e_i / ulp(p_i)) to the
//     accumulator's mantissa; the others are "special" and done as real fp64
//     adds: step 0, binade crossings, ties (~log2(D) + a few in all);
// (3) an exact int64 scan of r, one sequential pass over the special steps
//     (their fp64 adds and each segment's starting mantissa), and a grid-wide
//     write of every T_i = (M_segment + R_i - R_segment_start) * ulp.
// Every assumption is re-checked exactly (each segment's mantissa must stay
// below 2^53); if one fails, or the specials overflow their buffer, a device
// flag makes the single-CTA target_sum_kernel above redo the whole sum.
constexpr int kTsThreads = 256;
constexpr int kTsPer = 8;
constexpr int kTsBlock = kTsThreads * kTsPer;   // steps per block
constexpr int kTsMaxSpecial = 1 << 16;

__device__ __forceinline__ int binade_of(double x) {   // biased exponent (x > 0, normal)
    return static_cast<int>(static_cast<unsigned long long>(__double_as_longlong(x)) >> 52);
}
// x within relative `margin` of a power of two (either side), or not a
// positive normal number
__device__ __forceinline__ bool near_pow2(double x, double margin) {
    if (!(x > 0.0)) return true;
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(x));
    const int ex = static_cast<int>(b >> 52);
    if (ex == 0 || ex >= 2046) return true;
    const double f = __longlong_as_double(static_cast<long long>((b & ((1ULL << 52) - 1)) |
                                                                 (1023ULL << 52)));   // [1, 2)
    return f - 1.0 < margin || 2.0 - f < 2.0 * margin;
}

template <typename T, typename Op>
__device__ __forceinline__ T block_incl_scan(T v, T* sh, Op op) {   // kTsThreads threads
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = op(v, t);
    }
    if (lane == 31) sh[warp] = v;
    __syncthreads();
    if (warp == 0) {
        T w = lane < kTsThreads / 32 ? sh[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const T t = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w = op(w, t);
        }
        if (lane < kTsThreads / 32) sh[lane] = w;
    }
    __syncthreads();
    const T before = warp > 0 ? sh[warp - 1] : T(0);
    __syncthreads();
    return warp > 0 ? op(before, v) : v;
}

struct TsAdd {
    template <typename T>
    __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};

// (1a) per-block sums of the draws
__global__ void __launch_bounds__(kTsThreads) ts_block_sum_kernel(const double* __restrict__ e,
                                                                  int64_t n,
                                                                  double* __restrict__ bsum) {
    __shared__ double sh[kTsThreads / 32];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTsBlock + threadIdx.x * kTsPer;
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kTsPer; ++q) v += base + q < n ? e[base + q] : 0.0;
    v = block_incl_scan(v, sh, TsAdd());
    if (threadIdx.x == kTsThreads - 1) bsum[blockIdx.x] = v;
}

// one block: exclusive scan of v[0..nb) in place, the total into v[nb]
template <typename T>
__global__ void __launch_bounds__(kTsThreads) ts_scan_blocks_kernel(T* __restrict__ v, int64_t nb) {
    __shared__ T sh[kTsThreads / 32];
    T carry = T(0);
    for (int64_t c = 0; c < nb; c += kTsThreads) {
        const int64_t k = c + threadIdx.x;
        const T x = k < nb ? v[k] : T(0);
        const T inc = block_incl_scan(x, sh, TsAdd());
        if (k < nb) v[k] = carry + (inc - x);
        carry = carry + sh[kTsThreads / 32 - 1];   // this chunk's total
        __syncthreads();
    }
    if (threadIdx.x == 0) v[nb] = carry;
}

// (1b)+(2) approximate prefix -> binade, integer increments, specials
__global__ void __launch_bounds__(kTsThreads)
ts_local_kernel(const double* __restrict__ e, int64_t n, const double* __restrict__ boff,
                double margin, long long* __restrict__ r, unsigned char* __restrict__ special,
                long long* __restrict__ brsum, long long* __restrict__ bspec) {
    __shared__ double shd[kTsThreads / 32];
    __shared__ long long shl[kTsThreads / 32];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTsBlock + threadIdx.x * kTsPer;
    double ev[kTsPer];
    double loc = 0.0;
#pragma unroll
    for (int q = 0; q < kTsPer; ++q) {
        ev[q] = base + q < n ? e[base + q] : 0.0;
        loc += ev[q];
    }
    const double incl = block_incl_scan(loc, shd, TsAdd());
    double acc = boff[blockIdx.x] + (incl - loc);   // ~T_{base-1}
    long long rs = 0, sp = 0;
#pragma unroll
    for (int q = 0; q < kTsPer; ++q) {
        const int64_t i = base + q;
        if (i >= n) break;
        const double next = acc + ev[q];           // ~T_i
        bool spec = i == 0 || near_pow2(acc, margin) || near_pow2(next, margin) ||
                    binade_of(acc) != binade_of(next);
        long long rr = 0;
        if (!spec) {
            const int bexp = binade_of(acc);
            const double y = __dmul_rn(ev[q], __longlong_as_double(
                                                  static_cast<long long>(2098 - bexp) << 52));
            const double t = __dadd_rn(y, 0x1.0p52);            // rint(y), ties to even
            const double d = __dsub_rn(__dsub_rn(t, 0x1.0p52), y);
            if (!(y < 0x1.0p52) || d == 0.5 || d == -0.5 || bexp < 1023 - 60 || bexp > 1023 + 500)
                spec = true;
            else
                rr = static_cast<long long>(static_cast<unsigned long long>(__double_as_longlong(t)) -
                                            0x4330000000000000ULL);
        }
        r[i] = rr;
        special[i] = spec ? 1 : 0;
        rs += rr;
        sp += spec ? 1 : 0;
        acc = next;
    }
    rs = block_incl_scan(rs, shl, TsAdd());
    const long long spt = block_incl_scan(sp, shl, TsAdd());
    if (threadIdx.x == kTsThreads - 1) {
        brsum[blockIdx.x] = rs;
        bspec[blockIdx.x] = spt;
    }
}

// (3a) in-block scans + block offsets: r -> inclusive R_i, special indices in order
__global__ void __launch_bounds__(kTsThreads)
ts_scan_kernel(int64_t n, long long* __restrict__ r, const unsigned char* __restrict__ special,
               const long long* __restrict__ brsum, const long long* __restrict__ bspec,
               long long* __restrict__ spec_idx, int* __restrict__ fail) {
    __shared__ long long shl[kTsThreads / 32];
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTsBlock + threadIdx.x * kTsPer;
    long long rv[kTsPer];
    long long rs = 0, sp = 0;
#pragma unroll
    for (int q = 0; q < kTsPer; ++q) {
        const bool in = base + q < n;
        rv[q] = in ? r[base + q] : 0;
        rs += rv[q];
        sp += in && special[base + q] ? 1 : 0;
    }
    long long R = block_incl_scan(rs, shl, TsAdd()) - rs + brsum[blockIdx.x];
    long long k = block_incl_scan(sp, shl, TsAdd()) - sp + bspec[blockIdx.x];
#pragma unroll
    for (int q = 0; q < kTsPer; ++q) {
        const int64_t i = base + q;
        if (i >= n) break;
        R += rv[q];
        r[i] = R;
        if (special[i]) {
            if (k < kTsMaxSpecial) spec_idx[k] = i;
            else *fail = 1;
            ++k;
        }
    }
}

struct TsSeg {
    unsigned long long M, ebits;
    long long Rbase;
    long long pad;
};

// (3b) one block: the special steps in order (fp64 adds) and every segment's
// start; checks that no segment leaves its binade
__global__ void __launch_bounds__(kTsThreads)
ts_skeleton_kernel(const double* __restrict__ e, int64_t n, const long long* __restrict__ R,
                   const long long* __restrict__ spec_idx, const long long* __restrict__ bspec,
                   int64_t nb, TsSeg* __restrict__ seg, double* __restrict__ T,
                   int* __restrict__ fail) {
    __shared__ long long s_idx[1024];
    __shared__ long long s_rprev[1024];
    __shared__ double s_e[1024];
    __shared__ int s_fail;
    const long long nspec = bspec[nb];   // total specials (end of the exclusive scan)
    if (nspec > kTsMaxSpecial || *fail) {
        if (threadIdx.x == 0) *fail = 1;
        return;                          // uniform across the block
    }
    if (threadIdx.x == 0) s_fail = 0;
    constexpr unsigned long long kLimit = (1ULL << 53) - 2;
    unsigned long long M = 0, ebits = 0;
    long long Rbase = 0;
    for (long long c = 0; c < nspec; c += 1024) {
        const int cnt = static_cast<int>(nspec - c < 1024 ? nspec - c : 1024);
        __syncthreads();
        for (int k = threadIdx.x; k < cnt; k += kTsThreads) {
            const long long i = spec_idx[c + k];
            s_idx[k] = i;
            s_rprev[k] = i > 0 ? R[i - 1] : 0;
            s_e[k] = e[i];
        }
        __syncthreads();
        if (threadIdx.x == 0 && !s_fail) {
            for (int k = 0; k < cnt; ++k) {
                const long long i = s_idx[k];
                double Tcur;
                if (i == 0) {
                    Tcur = s_e[k];                              // T_0 = e_0
                } else {
                    const unsigned long long P = M + static_cast<unsigned long long>(s_rprev[k] - Rbase);
                    if (c + k == 0 || P > kLimit) { s_fail = 1; break; }
                    Tcur = __dadd_rn(from_binade(P, ebits), s_e[k]);
                }
                T[i] = Tcur;
                const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(Tcur));
                const int bexp = static_cast<int>(b >> 52);
                if (bexp < 1023 - 60 || bexp > 1023 + 500) { s_fail = 1; break; }
                ebits = static_cast<unsigned long long>(bexp) << 52;
                M = (b & ((1ULL << 52) - 1)) | (1ULL << 52);
                Rbase = s_rprev[k];   // r_i = 0 for a special step: R_i == R_{i-1}
                seg[c + k] = TsSeg{M, ebits, Rbase, 0};
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (!s_fail && n > 0) {   // the last segment must end inside its binade
            const unsigned long long P = M + static_cast<unsigned long long>(R[n - 1] - Rbase);
            if (P > kLimit) s_fail = 1;
        }
        if (s_fail) *fail = 1;
    }
}

// (3c) every non-special T_i from its segment
__global__ void __launch_bounds__(kTsThreads)
ts_write_kernel(int64_t n, const long long* __restrict__ R, const unsigned char* __restrict__ special,
                const long long* __restrict__ bspec, const TsSeg* __restrict__ seg,
                const int* __restrict__ fail, double* __restrict__ T) {
    __shared__ long long shl[kTsThreads / 32];
    if (*fail) return;
    const int64_t base = static_cast<int64_t>(blockIdx.x) * kTsBlock + threadIdx.x * kTsPer;
    long long sp = 0;
#pragma unroll
    for (int q = 0; q < kTsPer; ++q) sp += base + q < n && special[base + q] ? 1 : 0;
    long long k = block_incl_scan(sp, shl, TsAdd()) - sp + bspec[blockIdx.x] - 1;
#pragma unroll
    for (int q = 0; q < kTsPer; ++q) {
        const int64_t i = base + q;
        if (i >= n) break;
        if (special[i]) { ++k; continue; }
        const TsSeg sg = seg[k];
        T[i] = from_binade(sg.M + static_cast<unsigned long long>(R[i] - sg.Rbase), sg.ebits);
    }
}

ds_status target_sum(ds_ctx* ctx, const double* e, int64_t D, double* T, cudaStream_t st) {
    const int64_t nb = (D + kTsBlock - 1) / kTsBlock;
    char* buf = nullptr;
    const size_t b_r = dsi::align_up(sizeof(long long) * D, 256);
    const size_t b_sp = dsi::align_up(static_cast<size_t>(D), 256);
    const size_t b_nb = dsi::align_up(sizeof(long long) * (nb + 1), 256);
    const size_t b_idx = dsi::align_up(sizeof(long long) * kTsMaxSpecial, 256);
    const size_t b_seg = dsi::align_up(sizeof(TsSeg) * kTsMaxSpecial, 256);
    const size_t total = b_r + b_sp + 3 * b_nb + b_idx + b_seg + 256;
    DS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&buf), total, st));
    char* q = buf;
    long long* r = reinterpret_cast<long long*>(q); q += b_r;
    unsigned char* special = reinterpret_cast<unsigned char*>(q); q += b_sp;
    double* bsum = reinterpret_cast<double*>(q); q += b_nb;
    long long* brsum = reinterpret_cast<long long*>(q); q += b_nb;
    long long* bspec = reinterpret_cast<long long*>(q); q += b_nb;
    long long* spec_idx = reinterpret_cast<long long*>(q); q += b_idx;
    TsSeg* seg = reinterpret_cast<TsSeg*>(q); q += b_seg;
    int* fail = reinterpret_cast<int*>(q);
    DS_CUDA_TRY(cudaMemsetAsync(fail, 0, sizeof(int), st));
    const double margin = 1e-7 + 4.0 * static_cast<double>(D) * 0x1.0p-52;
    const unsigned g = static_cast<unsigned>(nb);
    ts_block_sum_kernel<<<g, kTsThreads, 0, st>>>(e, D, bsum);
    DS_LAUNCH_CHECK(ctx, "ts_block_sum_kernel");
    ts_scan_blocks_kernel<double><<<1, kTsThreads, 0, st>>>(bsum, nb);
    DS_LAUNCH_CHECK(ctx, "ts_scan_blocks_kernel");
    ts_local_kernel<<<g, kTsThreads, 0, st>>>(e, D, bsum, margin, r, special, brsum, bspec);
    DS_LAUNCH_CHECK(ctx, "ts_local_kernel");
    ts_scan_blocks_kernel<long long><<<1, kTsThreads, 0, st>>>(brsum, nb);
    DS_LAUNCH_CHECK(ctx, "ts_scan_blocks_kernel");
    ts_scan_blocks_kernel<long long><<<1, kTsThreads, 0, st>>>(bspec, nb);
    DS_LAUNCH_CHECK(ctx, "ts_scan_blocks_kernel");
    ts_scan_kernel<<<g, kTsThreads, 0, st>>>(D, r, special, brsum, bspec, spec_idx, fail);
    DS_LAUNCH_CHECK(ctx, "ts_scan_kernel");
    ts_skeleton_kernel<<<1, kTsThreads, 0, st>>>(e, D, r, spec_idx, bspec, nb, seg, T, fail);
    DS_LAUNCH_CHECK(ctx, "ts_skeleton_kernel");
    ts_write_kernel<<<g, kTsThreads, 0, st>>>(D, r, special, bspec, seg, fail, T);
    DS_LAUNCH_CHECK(ctx, "ts_write_kernel");
    // fallback: the single-CTA exact scan, a no-op unless a check failed
    if (!(ctx->route_attr_set & (1u << 21))) {   // once per context
        DS_CUDA_TRY(cudaFuncSetAttribute(target_sum_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(kSumSmem)));
        ctx->route_attr_set |= 1u << 21;
    }
    const int* gate = std::getenv("DS_TARGET_SUM_SEQUENTIAL") ? nullptr : fail;   // test hook
    target_sum_kernel<<<1, kSumThreads, kSumSmem, st>>>(e, D, T, gate);
    DS_LAUNCH_CHECK(ctx, "target_sum_kernel");
    cudaFreeAsync(buf, st);
    return DS_OK;
}

// ---- K8d: place targets in intervals ------------------------------------------
__device__ __forceinline__ long long ord_of(double x) {
    const long long b = __double_as_longlong(x);
    return b >= 0 ? b : -(b & 0x7fffffffffffffffLL);
}

__device__ __forceinline__ double double_of(long long o) {
    return o >= 0 ? __longlong_as_double(o) : __longlong_as_double((-o) | (1LL << 63));
}

struct IntervalParams {
    double cum;
    double start;
    double rate;
    double pad;
};

__device__ __forceinline__ int first_interval(const double* thr, int P, double target) {
    // first k with target < thr[k] (thr nondecreasing)
    int lo = 0, hi = P;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (target < thr[mid]) hi = mid;
        else lo = mid + 1;
    }
    return lo;
}

__device__ __forceinline__ double target_of(const double* T, int64_t i) {
    return T ? T[i] : static_cast<double>(i);   // uniform: target += 1.0 from 0.0 is exact
}

__device__ __forceinline__ long long block_max_inclusive(long long v, long long* warp_buf) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long t = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o && t > v) v = t;
    }
    if (lane == 31) warp_buf[warp] = v;
    __syncthreads();
    if (warp == 0) {
        const int nw = blockDim.x >> 5;
        long long w = lane < nw ? warp_buf[lane] : LLONG_MIN;
        long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o && t > wi) wi = t;
        }
        const long long prev = __shfl_up_sync(0xffffffffu, wi, 1);
        if (lane < nw) warp_buf[lane] = lane == 0 ? LLONG_MIN : prev;   // exclusive
    }
    __syncthreads();
    const long long pre = warp_buf[warp];
    return pre > v ? pre : v;
}

__global__ void __launch_bounds__(kPlaceThreads)
place_kernel(const double* __restrict__ T, int64_t n, const double* __restrict__ thr,
             const IntervalParams* __restrict__ ip, int P, long long* __restrict__ key,
             long long* __restrict__ block_max, long long* __restrict__ flags) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kPlaceThreads + threadIdx.x;
    long long k_out = LLONG_MIN;
    if (i < n) {
        const double target = target_of(T, i);
        const int k = first_interval(thr, P, target);
        if (k == P) {
            atomicMin(&flags[0], static_cast<long long>(i));   // no interval admits it
        } else {
            const IntervalParams q = ip[k];
            // workload.cpp:97: start + (target - cum) / rate
            const double t = __dadd_rn(q.start, __ddiv_rn(__dsub_rn(target, q.cum), q.rate));
            k_out = ord_of(t) - static_cast<long long>(i);
        }
        key[i] = k_out;
    }
    __shared__ long long red[kPlaceThreads / 32];
    long long m = k_out;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long t = __shfl_xor_sync(0xffffffffu, m, o);
        m = t > m ? t : m;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long b = LLONG_MIN;
        for (int w = 0; w < kPlaceThreads / 32; ++w) b = red[w] > b ? red[w] : b;
        block_max[blockIdx.x] = b;
    }
}

// Exclusive max-scan of the block maxima (one block), in place.
__global__ void __launch_bounds__(1024) carry_kernel(long long* __restrict__ block_max, int nb) {
    __shared__ long long warp_buf[32];
    __shared__ long long s_incl[1024];
    long long run = LLONG_MIN;
    for (int base = 0; base < nb; base += 1024) {
        const int b = base + threadIdx.x;
        const long long v = b < nb ? block_max[b] : LLONG_MIN;
        long long incl = block_max_inclusive(v, warp_buf);
        incl = incl > run ? incl : run;
        s_incl[threadIdx.x] = incl;
        __syncthreads();
        if (b < nb) block_max[b] = threadIdx.x == 0 ? run : s_incl[threadIdx.x - 1];
        run = s_incl[1023];
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kPlaceThreads)
finalize_kernel(const double* __restrict__ T, int64_t n, const double* __restrict__ thr, int P,
                const long long* __restrict__ key, const long long* __restrict__ carry,
                double duration, double* __restrict__ out, long long* __restrict__ flags) {
    __shared__ long long warp_buf[kPlaceThreads / 32];
    const int64_t i = static_cast<int64_t>(blockIdx.x) * kPlaceThreads + threadIdx.x;
    const long long v = i < n ? key[i] : LLONG_MIN;
    long long m = block_max_inclusive(v, warp_buf);
    const long long c = carry[blockIdx.x];
    m = c > m ? c : m;
    if (i < n && i < flags[0]) {
        const double t = double_of(m + static_cast<long long>(i));
        out[i] = t;
        if (t >= duration) {   // workload.cpp:100 ends the walk here
            atomicMin(&flags[1], static_cast<long long>(i));
            // Only the last positive-rate interval can end the walk this way
            // (the reference would otherwise retry the target in later ones).
            if (first_interval(thr, P, target_of(T, i)) != P - 1) atomicOr(
                reinterpret_cast<unsigned long long*>(&flags[2]), 1ULL);
        }
    }
}

struct Walk {
    std::vector<double> thr;
    std::vector<IntervalParams> ip;
    double duration = 0.0;
};

ds_status build_walk(const double* rates, int32_t n_rates, double dt, Walk* w) {
    double cum = 0.0;   // workload.cpp:90-94
    for (int32_t k = 0; k < n_rates; ++k) {
        const double rate = rates[k];
        if (!(rate >= 0.0) || !std::isfinite(rate))
            return dsi::fail(DS_ERR_DOMAIN, "rate must be a non-negative finite number");
        const double start = dt * static_cast<double>(k);
        const double cum_end = cum + rate * dt;
        if (!std::isfinite(cum_end))
            return dsi::fail(DS_ERR_DOMAIN, "cumulative rate overflows");
        if (rate > 0.0) {
            w->thr.push_back(cum_end - 1e-12);
            w->ip.push_back({cum, start, rate, 0.0});
        }
        cum = cum_end;
    }
    w->duration = dt * static_cast<double>(n_rates);
    return DS_OK;
}

ds_status generate(ds_ctx* ctx, const double* rates, int32_t n_rates, double dt, uint64_t seed,
                   int32_t mode, double* dev_out, double* host_out, int64_t capacity,
                   int64_t* count, cudaStream_t st) {
    if (!ctx || !count || n_rates < 0 || (n_rates > 0 && !rates))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (mode != DS_ARRIVALS_POISSON && mode != DS_ARRIVALS_UNIFORM)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "unknown arrival mode");
    if (!(dt > 0.0) || !std::isfinite(dt))
        return dsi::fail(DS_ERR_DOMAIN, "trace interval must be positive");
    *count = 0;
    Walk w;
    ds_status s = build_walk(rates, n_rates, dt, &w);
    if (s != DS_OK) return s;
    const int P = static_cast<int>(w.thr.size());
    if (P == 0) return DS_OK;
    const double last = w.thr.back();   // no target at or above this is placed
    const bool poisson = mode == DS_ARRIVALS_POISSON;
    double want;
    if (poisson) {
        want = std::ceil(last + 8.0 * std::sqrt(last > 0.0 ? last : 0.0) + 64.0);
        if (const char* env = std::getenv("DS_ARRIVALS_INITIAL_DRAWS")) {   // test hook
            const double v = std::atof(env);
            if (v >= 2.0) want = v;
        }
    } else {
        want = std::floor(last > 0.0 ? last : 0.0) + 2.0;   // target floor(last)+1 fails
    }
    constexpr double kMaxDraws = 1ULL << 33;
    for (;;) {
        if (!(want <= kMaxDraws))
            return dsi::fail(DS_ERR_CAPACITY, "trace implies more arrivals than supported");
        const int64_t D = static_cast<int64_t>(want);
        const int64_t nb = (D + kPlaceThreads - 1) / kPlaceThreads;
        const size_t b8 = dsi::align_up(sizeof(double) * D, 256);
        const size_t bt = dsi::align_up(sizeof(double) * P, 256);
        const size_t bi = dsi::align_up(sizeof(IntervalParams) * P, 256);
        const size_t bb = dsi::align_up(sizeof(long long) * nb, 256);
        const size_t total = (poisson ? 2 * b8 : 0) + 2 * b8 + bt + bi + bb + 256;
        char* base = nullptr;
        s = dsi::ensure_scratch(ctx, total, reinterpret_cast<void**>(&base));
        if (s != DS_OK) return s;
        char* p = base;
        double* e = nullptr;
        double* T = nullptr;
        if (poisson) {
            e = reinterpret_cast<double*>(p);
            p += b8;
            T = reinterpret_cast<double*>(p);
            p += b8;
        }
        long long* key = reinterpret_cast<long long*>(p);
        p += b8;
        double* out = reinterpret_cast<double*>(p);
        p += b8;
        double* thr = reinterpret_cast<double*>(p);
        p += bt;
        IntervalParams* ip = reinterpret_cast<IntervalParams*>(p);
        p += bi;
        long long* bmax = reinterpret_cast<long long*>(p);
        p += bb;
        long long* flags = reinterpret_cast<long long*>(p);
        long long* hflags = nullptr;
        s = dsi::ensure_pinned(ctx, 4 * sizeof(long long), reinterpret_cast<void**>(&hflags));
        if (s != DS_OK) return s;
        const long long init[4] = {kNoIndex, kNoIndex, 0, 0};
        DS_CUDA_TRY(cudaMemcpyAsync(flags, init, sizeof init, cudaMemcpyHostToDevice, st));
        DS_CUDA_TRY(cudaMemcpyAsync(thr, w.thr.data(), sizeof(double) * P,
                                    cudaMemcpyHostToDevice, st));
        DS_CUDA_TRY(cudaMemcpyAsync(ip, w.ip.data(), sizeof(IntervalParams) * P,
                                    cudaMemcpyHostToDevice, st));
        if (poisson) {
            // RandomStream(seed, "arrivals") (rng.hpp:20-21)
            const uint64_t eng = splitmix64(seed ^ splitmix64(fnv1a("arrivals")));
            uint64_t* raw = reinterpret_cast<uint64_t*>(e);
            s = mt_stream(ctx, eng, D, raw, st);
            if (s != DS_OK) return s;
            int64_t blocks = (D + 255) / 256;
            if (blocks > 148 * 16) blocks = 148 * 16;
            exp_draws_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(raw, D, e);
            DS_LAUNCH_CHECK(ctx, "exp_draws_kernel");
            s = target_sum(ctx, e, D, T, st);
            if (s != DS_OK) return s;
        }
        place_kernel<<<static_cast<unsigned>(nb), kPlaceThreads, 0, st>>>(T, D, thr, ip, P, key,
                                                                           bmax, flags);
        DS_LAUNCH_CHECK(ctx, "place_kernel");
        carry_kernel<<<1, 1024, 0, st>>>(bmax, static_cast<int>(nb));
        DS_LAUNCH_CHECK(ctx, "carry_kernel");
        finalize_kernel<<<static_cast<unsigned>(nb), kPlaceThreads, 0, st>>>(
            T, D, thr, P, key, bmax, w.duration, out, flags);
        DS_LAUNCH_CHECK(ctx, "finalize_kernel");
        DS_CUDA_TRY(cudaMemcpyAsync(hflags, flags, 3 * sizeof(long long), cudaMemcpyDeviceToHost,
                                    st));
        DS_CUDA_TRY(cudaStreamSynchronize(st));
        const long long end_target = hflags[0], end_time = hflags[1];
        if (hflags[2])
            return dsi::fail(DS_ERR_INVARIANT,
                             "arrival walk ended before the last positive-rate interval");
        if (end_target >= D && end_time >= D) {   // more draws needed: rerun longer
            want *= 2.0;
            continue;
        }
        const int64_t c = end_target < end_time ? end_target : end_time;
        *count = c;
        if (host_out) {
            if (capacity < c) return dsi::fail(DS_ERR_CAPACITY, "arrivals buffer too small");
            if (c > 0)
                DS_CUDA_TRY(cudaMemcpyAsync(host_out, out, sizeof(double) * c,
                                            cudaMemcpyDeviceToHost, st));
            DS_CUDA_TRY(cudaStreamSynchronize(st));
        } else if (dev_out) {
            if (capacity < c) return dsi::fail(DS_ERR_CAPACITY, "arrivals buffer too small");
            if (c > 0)
                DS_CUDA_TRY(cudaMemcpyAsync(dev_out, out, sizeof(double) * c,
                                            cudaMemcpyDeviceToDevice, st));
        }
        return DS_OK;
    }
}

} // namespace

extern "C" ds_status ds_generate_arrivals(ds_ctx* ctx, const double* rates, int32_t n_rates,
                                          double interval_seconds, uint64_t seed, int32_t mode,
                                          double* arrivals, int64_t capacity, int64_t* count) {
    if (!ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
    return generate(ctx, rates, n_rates, interval_seconds, seed, mode, nullptr, arrivals,
                    capacity, count, ctx->stream);
}

extern "C" ds_status ds_generate_arrivals_device(ds_ctx* ctx, const double* rates,
                                                 int32_t n_rates, double interval_seconds,
                                                 uint64_t seed, int32_t mode, double* arrivals,
                                                 int64_t capacity, int64_t* count, void* stream) {
    if (!ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    return generate(ctx, rates, n_rates, interval_seconds, seed, mode, arrivals, nullptr,
                    capacity, count, st);
}
