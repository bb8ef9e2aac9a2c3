// K3 curve_observe: the online deferral-curve update on the GPU.
//
// Replaces repeated diffserve::observe_confidence (reference
// proj/src/profiles.cpp:108-120) over an ordered confidence sequence (the
// light-batch completion order of cluster.cpp:290-296). Per observation the
// reference scales every bin and the total by `decay`, then adds 1 to the
// observation's bin and to the total. Rounding makes the result
// order-dependent, so each of the 101 bins (plus the total) is replayed
// sequentially by its own thread: bit-identical to the reference (SURVEY probe
// A.4). The observations' bins are computed once per chunk in parallel and
// staged through shared memory.
#include <cuda_runtime.h>

#include <map>
#include <mutex>
#include <utility>

#include <cstdio>
#include <cstdlib>

#include "ds_internal.h"

namespace {

// 101 bin threads on warps 0-3 and the total alone on warp 4: the total's loop
// differs from the bins', so sharing a warp would run the two one after the other
constexpr int kThreads = 160;
constexpr int kTotalTid = 128;
constexpr int kChunk = 4096;

// m + 1 on a hit, else m. A real (divergent) branch rather than an
// add-and-select: a bin's thread hits on ~1% of observations, and only the
// warp holding the hit bin waits for the add.
__device__ __forceinline__ double add_one_if(double m, bool hit) {
    if (hit) {
        asm volatile("" ::: "memory");   // keep the branch (no if-conversion)
        m = __dadd_rn(m, 1.0);
    }
    return m;
}


__device__ __forceinline__ unsigned long long dbits(double x) {
    return static_cast<unsigned long long>(__double_as_longlong(x));
}

// The total's step t <- fl(fl(t*d) + 1), two roundings as in observe_confidence.
template <bool kScale>
__device__ __forceinline__ double total_exact(double t, double d) {
    return __dadd_rn(kScale ? __dmul_rn(t, d) : t, 1.0);
}

#ifndef DS_TOTAL_DFMA
#define DS_TOTAL_DFMA 1   // 0: the total always steps in the two-op form (A/B)
#endif

// f = RN(t*d + 1), ONE rounding, equals the reference's two-rounding step
// RN(RN(t*d) + 1) whenever f lies in [2^k + 1 + 2u, 2^(k+1) - 2u] for some
// 1 <= k <= 51, u = 2^(k-52). Proof: RN(y) = f with both neighbours of f in
// binade k gives |y - f| <= u/2 for y = t*d + 1, so P = t*d lies in
// [2^k + 1.5u, 2^(k+1) - 1 - 1.5u]; p = RN(P) is then in binade k with p + 1 <=
// 2^(k+1) - u, a multiple of u (u <= 1/2), so RN(p + 1) = p + 1; and P + 1 =
// (p + 1) + (P - p) with |P - p| <= u/2 rounds to p + 1 as well -- in a tie p is
// even and (p + 1)/u = p/u + 2^(52-k) is even too, so ties-to-even picks p + 1.
// Returns k, or -1 if f is outside every such interval.
__device__ __forceinline__ int dfma_safe_binade(double f) {
    const unsigned long long b = dbits(f);
    const int k = static_cast<int>(b >> 52) - 1023;   // the sign bit makes k >= 1025
    if (k < 1 || k > 51) return -1;
    const unsigned long long m = b & ((1ull << 52) - 1);
    return m >= (1ull << (52 - k)) + 2 && m <= (1ull << 52) - 2 ? k : -1;
}

// `len` steps of the total. The chain advances kRun steps at a time on single
// DFMAs (one dependent fp64 op per step instead of two). The DFMA map is
// monotone in t, so the outputs f_1..f_R of a run are monotone and lie between
// f_1 and f_R: if both ends lie in the interval of the SAME binade k
// (dfma_safe_binade), so does every output, and every step of the run equals
// the two-rounding step. A run that fails the test (binade crossings, totals
// below 2, negative or non-finite totals) is replayed in the exact two-op form.
// The map is deterministic, so a step that leaves t unchanged proves the
// rounded fixed point (~1/(1-d), reached after ~40K steps at d = 0.999): every
// later step does too, `settled` is set and the replay stops.
template <bool kScale>
__device__ double total_run(double t, int64_t len, double d, bool& settled) {
    constexpr int kRun = 32;
    int64_t k = 0;
    for (; k + kRun <= len; k += kRun) {
        const double t0 = t;
        bool fixed = false;
        bool ok = false;
        if (kScale && DS_TOTAL_DFMA) {
            double prev = t, f1 = t;
#pragma unroll
            for (int u = 0; u < kRun; ++u) {
                prev = t;
                t = __fma_rn(t, d, 1.0);
                if (u == 0) f1 = t;
            }
            const int k1 = dfma_safe_binade(f1);
            ok = k1 >= 0 && dfma_safe_binade(t) == k1;
            fixed = dbits(t) == dbits(prev);
        }
        if (!ok) {
            t = t0;
            fixed = false;
#pragma unroll 4
            for (int u = 0; u < kRun; ++u) {
                const double x = total_exact<kScale>(t, d);
                fixed |= dbits(x) == dbits(t);
                t = x;
            }
        }
        if (fixed) {
            settled = true;
            return t;
        }
    }
    for (; k < len; ++k) t = total_exact<kScale>(t, d);
    return t;
}

template <typename T, bool kScale>
__global__ void __launch_bounds__(kThreads)
curve_observe_kernel(ds_curve* __restrict__ curve, const T* __restrict__ conf, int64_t n,
                     double decay, int* __restrict__ bad, long long* __restrict__ err) {
    __shared__ __align__(16) unsigned char bins[kChunk];
    __shared__ int chunk_bad;
    const int tid = threadIdx.x;
    if (tid == 0) *bad = 0x7fffffff;   // ordered before any atomicMin by the first __syncthreads
    double m = 0.0;
    if (tid < DS_CURVE_BINS) m = curve->bin_mass[tid];
    else if (tid == kTotalTid) m = curve->total_mass;
    bool settled = false;
    // the total-mass thread matches every observation; bin threads their own bin
    const unsigned mine = tid < DS_CURVE_BINS ? static_cast<unsigned>(tid) : 0xFFu;
    const bool is_total = tid == kTotalTid;
    for (int64_t base = 0; base < n; base += kChunk) {
        const int cnt = static_cast<int>(n - base < kChunk ? n - base : kChunk);
        if (tid == 0) chunk_bad = 0;
        __syncthreads();
        for (int k = tid; k < cnt; k += kThreads) {
            const double c = static_cast<double>(conf[base + k]);
            if (!(c >= 0.0) || !(c <= 1.0)) {
                atomicMin(bad, static_cast<int>(base + k < 0x7fffffff ? base + k : 0x7fffffff));
                chunk_bad = 1;
                bins[k] = 255;
                continue;
            }
            // bin_of (profiles.cpp:60-65): floor(c*100 + 1e-9) clamped to [0, 100]
            int b = static_cast<int>(floor(__dadd_rn(__dmul_rn(c, 100.0), 1e-9)));
            b = b < 0 ? 0 : (b > DS_CURVE_BINS - 1 ? DS_CURVE_BINS - 1 : b);
            bins[k] = static_cast<unsigned char>(b);
        }
        __syncthreads();
        if (tid < DS_CURVE_BINS || is_total) {
            if (!chunk_bad) {
                if (is_total) {
                    // every observation hits the total (total_run: DFMA chain,
                    // verified; stops at the rounded fixed point)
                    if (!settled) m = total_run<kScale>(m, cnt, decay, settled);
                } else {
                    // 8 observations per 64-bit shared load; the add on a hit is a
                    // predicated instruction so a miss costs only the multiply
                    const int full8 = cnt & ~7;
                    for (int k = 0; k < full8; k += 8) {
                        const uint2 w = *reinterpret_cast<const uint2*>(&bins[k]);
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const unsigned b = ((u < 4 ? w.x : w.y) >> (8 * (u & 3))) & 0xFFu;
                            if (kScale) m = __dmul_rn(m, decay);
                            m = add_one_if(m, b == mine);
                        }
                    }
                    for (int k = full8; k < cnt; ++k) {
                        if (kScale) m = __dmul_rn(m, decay);
                        m = add_one_if(m, bins[k] == mine);
                    }
                }
            } else {
                for (int k = 0; k < cnt; ++k) {
                    const unsigned char b = bins[k];
                    if (b == 255) break;   // the reference throws here; state stops
                    if (kScale) m = __dmul_rn(m, decay);
                    if (is_total || b == mine) m = __dadd_rn(m, 1.0);
                }
            }
        }
        __syncthreads();
        if (chunk_bad) break;
    }
    if (tid < DS_CURVE_BINS) curve->bin_mass[tid] = m;
    else if (is_total) curve->total_mass = m;
    // device variants: publish the first invalid observation to the context
    // (every atomicMin on *bad precedes the last __syncthreads of the loop)
    if (err && tid == 0 && *bad != 0x7fffffff) atomicMin(err, static_cast<long long>(*bad));
}


// ---------------------------------------------------------------------------
// Long sequences: speculative segmented replay, verified exactly.
//
// The replay of one chain (a bin, or the total) is a deterministic map per
// observation, m -> fl(fl(m*d) + hit), so the state after a segment of
// observations is a function F_j of the state at its start. The sequence is
// cut into S segments of L observations (one CTA each, one thread per bin):
//   phase 0  bins of the segment into shared memory (and global), hit counts,
//            and the exact-arithmetic contribution H_j = sum_hits d^(L-1-k);
//   phase 1  every segment replays its L observations from a GUESS of its
//            start state, g_j = d^L g_{j-1} + H_{j-1} (the closed form), and
//            records U_j (the start it used) and E_j = F_j(U_j);
//   passes   every segment whose recorded start U_j differs from its
//            predecessor's end E_{j-1} replays again from E_{j-1}, in
//            lockstep with the speculative trajectory from U_j, until the
//            two states are bit-identical (from there on they stay equal,
//            so F_j(E_{j-1}) = E_j) or the segment ends (then E_j is replaced
//            by the new end). A pass in which no E_j of a chain changes
//            leaves U_j = E_{j-1} for every j: the chain is then exactly the
//            sequential replay (induction from segment 0, which starts at the
//            true state). Two nearby trajectories merge because the decay
//            shrinks their gap (in ulps) by d per observation while the bin
//            value stays in its binade; the merge time is ~1/(1-d) ln(gap).
//   walk     a chain still changing after kMaxPasses passes (e.g. one that
//            decays without hits, whose gap in ulps does not shrink) is walked
//            sequentially over the segments by one thread with the same
//            merge test, i.e. at worst the sequential replay.
// The total mass is data-independent (it "hits" every observation) and runs
// into a rounded fixed point t = fl(fl(t*d) + 1) after ~ln(gap)/(1-d)
// observations; one extra CTA covers its transient with 128 warm-started
// speculative segments, and one thread walks them up to the fixed point.
// Every shortcut is an exact equality test on the state, so the result is
// bit-identical to the sequential replay (and to observe_confidence) for any
// input; only the running time depends on how fast trajectories merge.
namespace spec {

constexpr int kThreads = 128;
constexpr int kChains = DS_CURVE_BINS + 1;   // 101 bins + the total
constexpr int kMaxPasses = 6;
constexpr int kTotalWarm = 4096;             // warm-up of the total's segments
constexpr int kCheck = 8;                    // merge test period (observations)
constexpr int kMaxL = 16384;                 // longest segment (shared-memory tables)
constexpr int kDefaultL = 4096;
constexpr int64_t kMinN = 32768;             // shorter sequences use the single-CTA replay

struct Ws {
    unsigned char* bins;  // [n] bin index per observation (255 = invalid)
    double* h;            // [S][kChains] exact-arithmetic hit contributions
    int* cnt;             // [S][kChains] hits per segment
    double* u;            // [S][kChains] start state E_j was computed from
    double* e0;           // [S][kChains] end states (double-buffered over passes)
    double* e1;
    int* changed;         // [kMaxPasses][kChains]
    unsigned* bar;        // grid barrier arrivals
    int* bad;             // first invalid observation (INT_MAX if none)
    long long* err;       // the context's device error word (device variants), or nullptr
    unsigned long long* trace;   // debug (DS_CURVE_TRACE): phase timestamps, else nullptr
};

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SPEC_TRACE(slot)                                                        \
    do {                                                                        \
        if (ws.trace && threadIdx.x == 0) ws.trace[slot] = gtimer();            \
    } while (0)

__device__ __forceinline__ unsigned long long bits(double x) {
    return static_cast<unsigned long long>(__double_as_longlong(x));
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// All S segment CTAs (cooperative launch: co-resident). `epoch` counts this
// CTA's barriers; the counter only grows, so no reset between barriers.
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks, unsigned& epoch) {
    __syncthreads();
    ++epoch;
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(bar, 1u);
        while (ld_acquire(bar) < epoch * nblocks) __nanosleep(64);
        __threadfence();
    }
    __syncthreads();
}

template <bool kScale>
__device__ __forceinline__ double step(double m, double d, bool hit) {
    if (kScale) m = __dmul_rn(m, d);
    return add_one_if(m, hit);
}

// One bin chain over `len` observations of `b8` (8-byte aligned).
template <bool kScale>
__device__ double replay_bin(double m, const unsigned char* b8, int len, unsigned mine, double d) {
    const int full8 = len & ~7;
    for (int k = 0; k < full8; k += 8) {
        const uint2 w = *reinterpret_cast<const uint2*>(b8 + k);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const unsigned b = ((u < 4 ? w.x : w.y) >> (8 * (u & 3))) & 0xFFu;
            m = step<kScale>(m, d, b == mine);
        }
    }
    for (int k = full8; k < len; ++k) m = step<kScale>(m, d, b8[k] == mine);
    return m;
}

// Re-replay from the true start r alongside the speculative start s; stops as
// soon as the two states are bit-identical (merged: the recorded end is exact).
template <bool kScale>
__device__ double rerun_bin(double r, double s, const unsigned char* b8, int len, unsigned mine,
                            double d, bool& merged) {
    merged = false;
    const int full8 = len & ~7;
    int k = 0;
    for (; k < full8; k += 8) {
        const uint2 w = *reinterpret_cast<const uint2*>(b8 + k);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const bool hit = (((u < 4 ? w.x : w.y) >> (8 * (u & 3))) & 0xFFu) == mine;
            r = step<kScale>(r, d, hit);
            s = step<kScale>(s, d, hit);
        }
        if (bits(r) == bits(s)) {
            merged = true;
            return r;
        }
    }
    for (; k < len; ++k) {
        const bool hit = b8[k] == mine;
        r = step<kScale>(r, d, hit);
        s = step<kScale>(s, d, hit);
    }
    merged = bits(r) == bits(s);
    return r;
}

template <bool kScale>
__device__ __forceinline__ double total_step(double t, double d) {
    return __dadd_rn(kScale ? __dmul_rn(t, d) : t, 1.0);
}

template <bool kScale>
__device__ __forceinline__ bool total_fixed(double t, double d) {
    return bits(total_step<kScale>(t, d)) == bits(t);
}

// The total over `len` observations; a fixed point ends the replay early.
template <bool kScale>
__device__ double replay_total(double t, int64_t len, double d) {
    bool settled = false;
    return total_run<kScale>(t, len, d, settled);
}

template <bool kScale>
__device__ double rerun_total(double r, double s, int64_t len, double d, bool& merged) {
    merged = false;
    int64_t k = 0;
    for (; k + kCheck <= len; k += kCheck) {
        if (bits(r) == bits(s)) {
            merged = true;
            return r;
        }
        if (total_fixed<kScale>(r, d)) return r;   // r is the end state; not merged
#pragma unroll
        for (int u = 0; u < kCheck; ++u) {
            r = total_step<kScale>(r, d);
            s = total_step<kScale>(s, d);
        }
    }
    for (; k < len; ++k) {
        r = total_step<kScale>(r, d);
        s = total_step<kScale>(s, d);
    }
    merged = bits(r) == bits(s);
    return r;
}

// d^k (k >= 0) and the closed-form total after k observations from t0.
__device__ __forceinline__ double dpow(double d, double k) { return pow(d, k); }

template <bool kScale>
__device__ double total_closed(double t0, int64_t k, double d) {
    if (!kScale) return t0 + static_cast<double>(k);
    const double dk = dpow(d, static_cast<double>(k));
    return dk * t0 + (1.0 - dk) / (1.0 - d);
}

// Observations of the total's transient to cover speculatively: a generous
// bound on the steps to its fixed point (~ln(2 gap (1-d) / ulp(t_inf)) / -ln d).
template <bool kScale>
__device__ int64_t total_cover(double t0, int64_t n, double d) {
    if (!kScale) return n;
    const double tinf = 1.0 / (1.0 - d);
    const double gap = fabs(tinf - t0);
    if (!(gap > 0.0)) return n < 8192 ? n : 8192;
    const double ulp = ldexp(1.0, ilogb(tinf) - 52);
    double k = log(2.0 * gap * (1.0 - d) / ulp) / -log(d);
    if (!(k > 0.0)) k = 0.0;
    const double cover = 2.0 * k + 8192.0;
    return cover >= static_cast<double>(n) ? n : static_cast<int64_t>(cover);
}

// Sequential replay of observations [0, n_eff) by the CTA's first 102
// threads (used only when an invalid confidence cut the sequence short).
template <bool kScale>
__device__ void sequential(ds_curve* curve, const unsigned char* bins, int64_t n_eff, double d) {
    const int tid = threadIdx.x;
    if (tid > DS_CURVE_BINS) return;
    double m = tid < DS_CURVE_BINS ? curve->bin_mass[tid] : curve->total_mass;
    const unsigned mine = tid < DS_CURVE_BINS ? static_cast<unsigned>(tid) : 0xFFFFu;
    for (int64_t k = 0; k < n_eff; ++k) {
        const unsigned b = bins[k];
        m = step<kScale>(m, d, mine == 0xFFFFu || b == mine);
    }
    if (tid < DS_CURVE_BINS) curve->bin_mass[tid] = m;
    else curve->total_mass = m;
}

template <typename T, bool kScale>
__global__ void __launch_bounds__(kThreads)
curve_spec_kernel(ds_curve* __restrict__ curve, const T* __restrict__ conf, int64_t n,
                  double d, int L, int S, Ws ws) {
    extern __shared__ __align__(16) unsigned char sb[];   // [L] bins of this segment
    __shared__ double sh[kChains];
    __shared__ int sc[kChains];
    __shared__ double swh[kThreads / 32][kChains];   // per-warp partial H
    __shared__ double wsc[kThreads / 32][32];        // per-warp lane weights
    __shared__ double plo[32];
    __shared__ double phi[kMaxL / 32];
    __shared__ double su[kThreads], se[kThreads];          // the total's segments
    const int tid = threadIdx.x;
    const int j = blockIdx.x;

    if (j == S) {
        // ---- the total-mass CTA (not part of the grid barrier) ----
        SPEC_TRACE(16);
        if (tid == 0)
            while (ld_acquire(ws.bar) < static_cast<unsigned>(S)) __nanosleep(128);
        __syncthreads();
        if (*reinterpret_cast<volatile int*>(ws.bad) != 0x7fffffff) return;   // sequential path
        const double t0 = curve->total_mass;
        const int64_t cover = total_cover<kScale>(t0, n, d);
        const int64_t lt = (cover + kThreads - 1) / kThreads;
        const int64_t a = static_cast<int64_t>(tid) * lt;
        const int64_t e = a + lt < cover ? a + lt : cover;
        if (a < e) {
            const int64_t k0 = a > kTotalWarm ? a - kTotalWarm : 0;
            double t = k0 == 0 ? t0 : total_closed<kScale>(t0, k0, d);
            t = replay_total<kScale>(t, a - k0, d);
            su[tid] = t;
            se[tid] = replay_total<kScale>(t, e - a, d);
        }
        __syncthreads();
        SPEC_TRACE(17);
        if (tid == 0) {
            const int segs = static_cast<int>((cover + lt - 1) / lt);
            double st = se[0];   // segment 0 starts at the true t0
            for (int i = 1; i < segs; ++i) {
                if (total_fixed<kScale>(st, d)) break;
                if (bits(st) == bits(su[i])) {
                    st = se[i];
                    continue;
                }
                const int64_t ai = static_cast<int64_t>(i) * lt;
                const int64_t len = (ai + lt < cover ? ai + lt : cover) - ai;
                bool merged;
                const double r = rerun_total<kScale>(st, su[i], len, d, merged);
                st = merged ? se[i] : r;
            }
            if (cover < n) st = replay_total<kScale>(st, n - cover, d);
            curve->total_mass = st;
            SPEC_TRACE(18);
        }
        return;
    }

    // ---- phase 0: bins, hit counts, closed-form contributions ----
    if (j == 0) SPEC_TRACE(0);
    const int64_t a = static_cast<int64_t>(j) * L;
    const int len = static_cast<int>(n - a < L ? n - a : L);
    if (tid < kChains) {
        sh[tid] = 0.0;
        sc[tid] = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) swh[w][tid] = 0.0;
    }
    if (tid < 32) plo[tid] = dpow(d, tid);
    for (int q = tid; q < (len + 31) / 32; q += kThreads) phi[q] = dpow(d, 32.0 * q);
    __syncthreads();
    if (j == 0) SPEC_TRACE(20);
    // Bins first, 16 loads in flight per thread (the loop is bound by the
    // confidences' HBM latency otherwise: ~25 us per segment).
    for (int k0 = tid; k0 < len; k0 += 16 * kThreads) {
        double cv[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int k = k0 + u * kThreads;
            cv[u] = k < len ? static_cast<double>(conf[a + k]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int k = k0 + u * kThreads;
            if (k >= len) break;
            const double c = cv[u];
            unsigned char bb;
            if (!(c >= 0.0) || !(c <= 1.0)) {
                atomicMin(ws.bad, static_cast<int>(a + k < 0x7fffffff ? a + k : 0x7fffffff));
                bb = 255;
            } else {
                // bin_of (profiles.cpp:60-65): floor(c*100 + 1e-9) clamped to [0, 100]
                int b = static_cast<int>(floor(__dadd_rn(__dmul_rn(c, 100.0), 1e-9)));
                b = b < 0 ? 0 : (b > DS_CURVE_BINS - 1 ? DS_CURVE_BINS - 1 : b);
                bb = static_cast<unsigned char>(b);
            }
            sb[k] = bb;
        }
    }
    __syncthreads();
    if (j == 0) SPEC_TRACE(24);
    // Closed-form contributions: each warp takes 32 consecutive observations at
    // a time (lane = observation); lanes with the same bin are grouped
    // (match_any) and the group's leader adds their weights d^(len-1-k) into the
    // warp's own partial sums (shared-memory atomics on doubles were no faster).
    {
        const int warp = tid >> 5, lane = tid & 31;
        for (int k0 = 32 * warp; k0 < len; k0 += kThreads) {
            const int k = k0 + lane;
            const unsigned bb = k < len ? sb[k] : 0xFFFFu;
            double w = 0.0;
            if (bb < static_cast<unsigned>(DS_CURVE_BINS)) {
                const int i = len - 1 - k;   // d^i = d^(32q) d^r
                w = phi[i >> 5] * plo[i & 31];
            }
            wsc[warp][lane] = w;
            const unsigned peers = __match_any_sync(0xffffffffu, bb);
            __syncwarp();
            if (bb < static_cast<unsigned>(DS_CURVE_BINS) && lane == __ffs(peers) - 1) {
                double acc = 0.0;
                for (unsigned m = peers; m; m &= m - 1) acc += wsc[warp][__ffs(m) - 1];
                swh[warp][bb] += acc;
                atomicAdd(&sc[bb], __popc(peers));
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (tid < DS_CURVE_BINS)
        sh[tid] = (swh[0][tid] + swh[1][tid]) + (swh[2][tid] + swh[3][tid]);
    __syncthreads();
    if (j == 0) SPEC_TRACE(21);
    for (int k = tid * 16; k < len; k += kThreads * 16) {
        if (k + 16 <= len)
            *reinterpret_cast<uint4*>(ws.bins + a + k) = *reinterpret_cast<const uint4*>(sb + k);
        else
            for (int q = k; q < len; ++q) ws.bins[a + q] = sb[q];
    }
    if (tid < DS_CURVE_BINS) {
        ws.h[static_cast<int64_t>(j) * kChains + tid] = sh[tid];
        ws.cnt[static_cast<int64_t>(j) * kChains + tid] = sc[tid];
    }
    if (j == 0) SPEC_TRACE(22);
    if (j == S - 1) SPEC_TRACE(23);
    unsigned epoch = 0;
    grid_barrier(ws.bar, static_cast<unsigned>(S), epoch);
    if (j == 0) SPEC_TRACE(1);
    const int bad = *reinterpret_cast<volatile int*>(ws.bad);
    if (bad != 0x7fffffff) {
        // the reference throws at the first invalid confidence: replay up to it
        if (j == 0) sequential<kScale>(curve, ws.bins, bad, d);
        if (j == 0 && tid == 0 && ws.err) atomicMin(ws.err, static_cast<long long>(bad));
        return;
    }

    // ---- phase 1: speculative replay of every segment from its guess ----
    const bool chain = tid < DS_CURVE_BINS;
    const unsigned mine = static_cast<unsigned>(tid);
    const int64_t row = static_cast<int64_t>(j) * kChains + tid;
    if (chain) {
        double g = curve->bin_mass[tid];
        if (j > 0) {
            // g_j = d^(L j) m_0 + sum_{i<j} d^(L (j-1-i)) H_i; terms older than K
            // segments weigh d^(L K) < 2^-60 and cannot move the guess
            const double dl = dpow(d, static_cast<double>(L));
            const double lk = -static_cast<double>(L) * log(d);
            const int K = lk > 0.0 ? static_cast<int>(fmin(60.0 * 0.6931471805599453 / lk + 1.0,
                                                          static_cast<double>(j)))
                                   : j;
            const int i0 = j - K;
            g = __dmul_rn(g, dpow(d, static_cast<double>(L) * i0));   // -0.0 stays -0.0
#pragma unroll 4
            for (int i = i0; i < j; ++i) {
                const int64_t ri = static_cast<int64_t>(i) * kChains + tid;
                g = ws.cnt[ri] ? __fma_rn(dl, g, ws.h[ri]) : __dmul_rn(dl, g);
            }
        }
        ws.u[row] = g;
        ws.e0[row] = replay_bin<kScale>(g, sb, len, mine, d);
    }
    if (j == 0) SPEC_TRACE(2);
    grid_barrier(ws.bar, static_cast<unsigned>(S), epoch);
    if (j == 0) SPEC_TRACE(3);

    // ---- passes ----
    bool resolved = !chain;
    int pass = 0;
    const double* fin = ws.e0;
    for (; pass < kMaxPasses; ++pass) {
        const double* rd = (pass & 1) ? ws.e1 : ws.e0;
        double* wr = (pass & 1) ? ws.e0 : ws.e1;
        if (chain) {
            double ev = rd[row];
            if (!resolved && j > 0) {
                const double st = rd[row - kChains];
                const double us = ws.u[row];
                if (bits(st) != bits(us)) {
                    bool merged;
                    const double r = rerun_bin<kScale>(st, us, sb, len, mine, d, merged);
                    ws.u[row] = st;
                    if (!merged) {
                        ev = r;
                        atomicAdd(&ws.changed[pass * kChains + tid], 1);
                    }
                }
            }
            wr[row] = ev;
        }
        grid_barrier(ws.bar, static_cast<unsigned>(S), epoch);
        if (j == 0) SPEC_TRACE(4 + pass);
        fin = wr;
        if (chain && !resolved)
            resolved = *reinterpret_cast<volatile int*>(&ws.changed[pass * kChains + tid]) == 0;
        if (__syncthreads_and(resolved)) break;
    }

    // ---- write-out; chains still unresolved are walked sequentially ----
    if (!chain) return;
    if (resolved) {
        if (j == S - 1) curve->bin_mass[tid] = fin[row];
        return;
    }
    if (j != tid % S) return;   // one walker per unresolved chain
    double st = fin[tid];
    for (int i = 1; i < S; ++i) {
        const int64_t ri = static_cast<int64_t>(i) * kChains + tid;
        const double us = ws.u[ri];
        if (bits(st) == bits(us)) {
            st = fin[ri];
            continue;
        }
        const int64_t ai = static_cast<int64_t>(i) * L;
        const int li = static_cast<int>(n - ai < L ? n - ai : L);
        bool merged;
        const double r = rerun_bin<kScale>(st, us, ws.bins + ai, li, mine, d, merged);
        st = merged ? fin[ri] : r;
    }
    curve->bin_mass[tid] = st;
    if (ws.trace && tid == 0) ws.trace[12] = gtimer();   // (a walker's end)
}

} // namespace spec


__global__ void spec_init(int* changed, unsigned* bar, int* bad) {
    for (int i = threadIdx.x; i < spec::kMaxPasses * spec::kChains; i += blockDim.x) changed[i] = 0;
    if (threadIdx.x == 0) {
        *bar = 0;
        *bad = 0x7fffffff;
    }
}

template <typename T, bool kScale>
const void* spec_fn() {
    return reinterpret_cast<const void*>(&spec::curve_spec_kernel<T, kScale>);
}

const void* spec_kernel_for(int32_t dtype, bool scale) {
    if (dtype == DS_CONF_F64) return scale ? spec_fn<double, true>() : spec_fn<double, false>();
    return scale ? spec_fn<float, true>() : spec_fn<float, false>();
}

// Segment length and count for the segmented replay, and its workspace bytes
// (bytes = 0: the single-CTA replay is used). DS_CURVE_L overrides the
// segment length, DS_CURVE_SPEC=0 disables the segmented path (experiments).
struct SpecPlan {
    int L = 0;
    int S = 0;
    size_t bytes = 0;
};

SpecPlan spec_plan(ds_ctx* ctx, int64_t n, int32_t dtype, double decay) {
    static const int env_l = [] {
        const char* s = getenv("DS_CURVE_L");
        return s ? atoi(s) : 0;
    }();
    static const bool env_off = [] {
        const char* s = getenv("DS_CURVE_SPEC");
        return s && s[0] == '0';
    }();
    SpecPlan p;
    if (env_off || n < spec::kMinN) return p;
    int L = env_l > 0 ? env_l : spec::kDefaultL;
    L = (L + 15) / 16 * 16;
    // the SM count and the kernel's occupancy, queried once per (device,
    // kernel): the queries cost tens of microseconds of host time per call
    const void* fn = spec_kernel_for(dtype, decay != 1.0);
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, std::pair<int, int>> cache;
    int sms = 0, occ = 0;
    {
        std::lock_guard<std::mutex> lock(mu);
        auto it = cache.find({ctx->device, fn});
        if (it != cache.end()) {
            sms = it->second.first;
            occ = it->second.second;
        } else {
            if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device) !=
                    cudaSuccess ||
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, spec::kThreads,
                                                              static_cast<size_t>(spec::kMaxL)) !=
                    cudaSuccess)
                return p;
            cache[{ctx->device, fn}] = {sms, occ};
        }
    }
    const int64_t max_blocks = static_cast<int64_t>(occ) * sms;   // at the largest segment
    int64_t S = (n + L - 1) / L;
    if (S + 1 > max_blocks) {
        const int64_t l2 = (n + max_blocks - 2) / (max_blocks - 1);
        L = static_cast<int>((l2 + 15) / 16 * 16);
        S = (n + L - 1) / L;
    }
    if (L > spec::kMaxL || S + 1 > max_blocks) return p;
    const size_t rows = static_cast<size_t>(S) * spec::kChains;
    p.L = L;
    p.S = static_cast<int>(S);
    p.bytes = dsi::align_up(n, 256) + 4 * dsi::align_up(rows * 8, 256) +
              dsi::align_up(rows * 4, 256) + dsi::align_up(spec::kMaxPasses * spec::kChains * 4, 256) +
              256;
    return p;
}

// `ws` is a device area of spec_plan(...).bytes (unused by the single-CTA path).
ds_status launch(ds_ctx* ctx, ds_curve* dcurve, const void* conf, int32_t dtype, int64_t n,
                 double decay, int* dbad, const SpecPlan& plan, char* ws, cudaStream_t st,
                 long long* err) {
    const bool scale = decay != 1.0;
    if (plan.bytes) {
        const size_t rows = static_cast<size_t>(plan.S) * spec::kChains;
        spec::Ws w;
        char* q = ws;
        w.bins = reinterpret_cast<unsigned char*>(q);
        q += dsi::align_up(n, 256);
        w.h = reinterpret_cast<double*>(q);
        q += dsi::align_up(rows * 8, 256);
        w.u = reinterpret_cast<double*>(q);
        q += dsi::align_up(rows * 8, 256);
        w.e0 = reinterpret_cast<double*>(q);
        q += dsi::align_up(rows * 8, 256);
        w.e1 = reinterpret_cast<double*>(q);
        q += dsi::align_up(rows * 8, 256);
        w.cnt = reinterpret_cast<int*>(q);
        q += dsi::align_up(rows * 4, 256);
        w.changed = reinterpret_cast<int*>(q);
        q += dsi::align_up(spec::kMaxPasses * spec::kChains * 4, 256);
        w.bar = reinterpret_cast<unsigned*>(q);
        w.bad = dbad;
        w.err = err;
        static unsigned long long* trace_buf = nullptr;
        static const bool want_trace = getenv("DS_CURVE_TRACE") != nullptr;
        if (want_trace && !trace_buf) cudaMalloc(&trace_buf, 32 * sizeof(unsigned long long));
        w.trace = want_trace ? trace_buf : nullptr;
        if (w.trace) cudaMemsetAsync(w.trace, 0, 32 * sizeof(unsigned long long), st);
        spec_init<<<1, 256, 0, st>>>(w.changed, w.bar, w.bad);
        DS_LAUNCH_CHECK(ctx, "spec_init");
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(plan.S + 1));
        cfg.blockDim = dim3(spec::kThreads);
        cfg.dynamicSmemBytes = static_cast<size_t>(plan.L);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const int L = plan.L, S = plan.S;
        cudaError_t e;
        if (dtype == DS_CONF_F64) {
            const double* c = static_cast<const double*>(conf);
            e = scale ? cudaLaunchKernelEx(&cfg, spec::curve_spec_kernel<double, true>, dcurve, c, n, decay, L, S, w)
                      : cudaLaunchKernelEx(&cfg, spec::curve_spec_kernel<double, false>, dcurve, c, n, decay, L, S, w);
        } else {
            const float* c = static_cast<const float*>(conf);
            e = scale ? cudaLaunchKernelEx(&cfg, spec::curve_spec_kernel<float, true>, dcurve, c, n, decay, L, S, w)
                      : cudaLaunchKernelEx(&cfg, spec::curve_spec_kernel<float, false>, dcurve, c, n, decay, L, S, w);
        }
        if (e != cudaSuccess) return dsi::cuda_fail(e, "curve_spec_kernel");
        DS_LAUNCH_CHECK(ctx, "curve_spec_kernel");
        if (w.trace) {   // debug: phase times (us from block 0's start) and pass counts
            unsigned long long t[32];
            int ch[spec::kMaxPasses * spec::kChains];
            cudaMemcpyAsync(t, w.trace, sizeof(t), cudaMemcpyDeviceToHost, st);
            cudaMemcpyAsync(ch, w.changed, sizeof(ch), cudaMemcpyDeviceToHost, st);
            cudaStreamSynchronize(st);
            auto us = [&](int i) { return t[i] ? (double)(t[i] - t[0]) / 1000.0 : -1.0; };
            fprintf(stderr, "spec n=%lld L=%d S=%d: phase0 %.1f phase1 %.1f/%.1f passes", (long long)n, L, S,
                    us(1), us(2), us(3));
            for (int p = 0; p < spec::kMaxPasses; ++p) {
                int c = 0, chains = 0;
                for (int b = 0; b < spec::kChains; ++b) { c += ch[p * spec::kChains + b]; chains += ch[p * spec::kChains + b] > 0; }
                fprintf(stderr, " [%.1f: %d segs, %d chains]", us(4 + p), c, chains);
            }
            fprintf(stderr, " (phase0: tables %.1f bins %.1f H %.1f writes %.1f last-block %.1f)", us(20), us(24), us(21), us(22), us(23));
            fprintf(stderr, " walk-end %.1f | total CTA start %.1f spec %.1f walk %.1f us\n", us(12), us(16),
                    us(17), us(18));
        }
        return DS_OK;
    }
    if (dtype == DS_CONF_F64) {
        const double* c = static_cast<const double*>(conf);
        if (scale) curve_observe_kernel<double, true><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad, err);
        else curve_observe_kernel<double, false><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad, err);
    } else {
        const float* c = static_cast<const float*>(conf);
        if (scale) curve_observe_kernel<float, true><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad, err);
        else curve_observe_kernel<float, false><<<1, kThreads, 0, st>>>(dcurve, c, n, decay, dbad, err);
    }
    DS_LAUNCH_CHECK(ctx, "curve_observe_kernel");
    return DS_OK;
}

} // namespace

// Device variant: `curve` is a device ds_curve updated in place. A confidence
// outside [0, 1] stops the replay where the reference would throw and is
// recorded in the context (ds_ctx_take_error); the host-buffer variant
// reports it as DS_ERR_DOMAIN directly.
namespace dsi {

// ds_curve_observe_device that also hands back the device word holding the
// first invalid observation's index (INT_MAX if none): valid until the next
// use of the context scratch (ds_disc_batches_complete_device reads it in
// the very next launch to stop routing where the reference would throw).
ds_status curve_observe_device_bad(ds_ctx* ctx, ds_curve* curve, const void* conf, int32_t dtype,
                                   int64_t n, double decay, cudaStream_t st, const int** bad) {
    if (!ctx || !curve) return fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
        return fail(DS_ERR_INVALID_ARGUMENT, "unknown confidence dtype");
    if (!(decay > 0.0) || !(decay <= 1.0))
        return fail(DS_ERR_DOMAIN, "curve decay must lie in (0, 1]");
    const SpecPlan plan = spec_plan(ctx, n > 0 ? n : 1, dtype, decay);
    void* scratch = nullptr;
    ds_status s = ensure_scratch(ctx, 256 + plan.bytes, &scratch);
    if (s != DS_OK) return s;
    if (bad) *bad = static_cast<const int*>(scratch);
    if (n <= 0) {   // nothing observed: no invalid index
        static const int kNone = 0x7fffffff;
        DS_CUDA_TRY(cudaMemcpyAsync(scratch, &kNone, sizeof(int), cudaMemcpyHostToDevice, st));
        return DS_OK;
    }
    return launch(ctx, curve, conf, dtype, n, decay, static_cast<int*>(scratch), plan,
                  static_cast<char*>(scratch) + 256, st, ctx->d_err);
}

} // namespace dsi

extern "C" ds_status ds_curve_observe_device(ds_ctx* ctx, ds_curve* curve, const void* conf,
                                             int32_t dtype, int64_t n, double decay,
                                             void* stream) {
    if (!ctx || !curve) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (n <= 0) {
        if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
            return dsi::fail(DS_ERR_INVALID_ARGUMENT, "unknown confidence dtype");
        if (!(decay > 0.0) || !(decay <= 1.0))
            return dsi::fail(DS_ERR_DOMAIN, "curve decay must lie in (0, 1]");
        return DS_OK;
    }
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    return dsi::curve_observe_device_bad(ctx, curve, conf, dtype, n, decay, st, nullptr);
}

extern "C" ds_status ds_curve_observe(ds_ctx* ctx, ds_curve* curve, const void* conf,
                                      int32_t dtype, int64_t n, double decay) {
    if (!ctx || !curve || (n > 0 && !conf))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (dtype != DS_CONF_F64 && dtype != DS_CONF_F32)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "unknown confidence dtype");
    if (n <= 0) return DS_OK;
    // observe_confidence checks confidence first, then decay (profiles.cpp:109-112)
    const size_t esz = dtype == DS_CONF_F64 ? 8 : 4;
    const size_t bc = dsi::align_up(esz * n, 256);
    const size_t bv = dsi::align_up(sizeof(ds_curve), 256);
    const SpecPlan plan = spec_plan(ctx, n, dtype, decay);
    char* d = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, bc + bv + 256 + plan.bytes, reinterpret_cast<void**>(&d));
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(d, conf, esz * n, cudaMemcpyHostToDevice, ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(d + bc, curve, sizeof(ds_curve), cudaMemcpyHostToDevice,
                                ctx->stream));
    int* dbad = reinterpret_cast<int*>(d + bc + bv);
    if (!(decay > 0.0) || !(decay <= 1.0)) {
        // the first observation's confidence check precedes the decay check
        const double c0 = dtype == DS_CONF_F64 ? static_cast<const double*>(conf)[0]
                                               : static_cast<const float*>(conf)[0];
        if (!(c0 >= 0.0) || !(c0 <= 1.0))
            return dsi::fail(DS_ERR_DOMAIN, "confidence must lie in [0, 1]");
        return dsi::fail(DS_ERR_DOMAIN, "curve decay must lie in (0, 1]");
    }
    s = launch(ctx, reinterpret_cast<ds_curve*>(d + bc), d, dtype, n, decay, dbad, plan,
               d + bc + bv + 256, ctx->stream, nullptr);
    if (s != DS_OK) return s;
    int bad = 0;
    DS_CUDA_TRY(cudaMemcpyAsync(curve, d + bc, sizeof(ds_curve), cudaMemcpyDeviceToHost,
                                ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(&bad, dbad, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (bad != 0x7fffffff)
        return dsi::fail(DS_ERR_DOMAIN, "confidence must lie in [0, 1] (observation " +
                                            std::to_string(bad) + ")");
    return DS_OK;
}
