// K1 plan_sweep: the controller's allocation planner on the GPU.
//
// Replaces diffserve::solve and its variants (reference
// proj/src/allocator.cpp:12-313). One CTA per AllocationProblem:
//
//   1. factored tables in shared memory: T1[b1], T2[b2] (profiles.cpp:28-30),
//      x1[b1] = max(1, min_servers(lambda*D, T1, S)), the latency-feasible
//      (b1, b2) bitmask (allocator.cpp:129-142), the sequential prefix of the
//      deferral curve (profiles.cpp:98-106 -- built in the reference's summation
//      order, so f(t) is bit-identical);
//   2. thresholds walked from the top in chunks of kTChunk: x2[t][b2] for the
//      chunk, then each thread takes (b1, b2) pairs and decides that pair's
//      (t, b1, b2) candidates, scoring each as a packed u64 key whose unsigned
//      order is the reference's selection order ("first feasible t from the
//      top", then Candidate::better_than, allocator.cpp:57-67):
//          (G-1-t_idx)<<40 | (x1+x2)<<28 | (255-b1_idx)<<20 | (255-b2_idx)<<12 | x1
//      (a pair's first valid t is its minimum key; x2 is monotone in t, so the
//      pair's valid t form a prefix of the chunk and a binary search finds it);
//   3. warp-shuffle min, then a block min over 8 warps; the first chunk with a
//      finite key holds the global minimum, so the walk stops there (the
//      reference's early exit, allocator.cpp:118).
//
// All fp64 arithmetic uses explicit _rn intrinsics in the reference's
// evaluation order, so nothing can be contracted into an FMA (the reference
// is built without FMA, SURVEY.md hard part 1).
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "ds_internal.h"

namespace {

constexpr int kThreads = 256;
constexpr int kTChunk = 128;
constexpr int kMaxB = DS_MAX_BATCHES;
constexpr int kMaxServers = 4095;      // 12-bit key fields
constexpr int kMaxGrid = (1 << 24) - 1;
constexpr unsigned long long kNone = ~0ull;

struct PlanSmem {
    double e1[kMaxB], e2[kMaxB], T1[kMaxB], T2[kMaxB], rT2[kMaxB];
    int b1[kMaxB], b2[kMaxB], x1[kMaxB];
    unsigned long long lat[kMaxB];      // bit j set: (b1_i, b2_j) latency-feasible
    double prefix[DS_CURVE_BINS + 1];
    double ft[kTChunk];
    uint16_t x2[kTChunk * kMaxB];   // <= kMaxServers + 1
    unsigned long long red[kThreads / 32];
    unsigned long long red2[kThreads / 32];
};

// allocator.cpp:12-18
__device__ __forceinline__ double queuing_delay(long long len, double rate, double sentinel) {
    if (len == 0) return 0.0;
    if (rate == 0.0) return sentinel;
    return __ddiv_rn(static_cast<double>(len), rate);
}

// allocator.cpp:45-51. Any quotient above `cap` returns cap+1: every caller
// only compares the result against cap (or clamps it to cap), so this is
// decision-identical to the reference, including its x86 out-of-range
// conversion path (see oracle/ds_oracle.c min_servers).
__device__ __forceinline__ int min_servers(double need, double per, int cap) {
    if (need <= 0.0) return 0;
    const double q = ceil(__ddiv_rn(need, per));
    if (!(q < static_cast<double>(cap) + 1.0)) return cap + 1;
    int x = static_cast<int>(q);
    if (x < 1) x = 1;
    while (x <= cap && __dmul_rn(static_cast<double>(x), per) < need) ++x;
    return x;
}

// min_servers with the quotient's ceiling from a reciprocal: y = need *
// fl(1/per) is within ~2.5 ulp of fl(need/per), so when y is more than
// 2^-49 * y (>= 8 ulp) from every integer the two have the same ceiling; only
// near an integer (or for huge quotients) is the correctly rounded division
// done. Decision-identical to min_servers.
// On that fast path q >= y + g, so q * per exceeds need by ~2^-49 relative
// and fl(q * per) >= need: the reference's increment loop would not run.
__device__ __forceinline__ int min_servers_r(double need, double per, double rper, int cap) {
    if (need <= 0.0) return 0;
    const double y = __dmul_rn(need, rper);
    const double q = ceil(y);
    const double g = __dmul_rn(y, 0x1p-49);
    // (a subnormal 1/per or y would carry fewer bits than the bound assumes)
    if (rper >= 0x1p-1022 && y >= 0x1p-1022 && __dsub_rn(q, y) > g &&
        __dsub_rn(y, __dsub_rn(q, 1.0)) > g)
        return q < static_cast<double>(cap) + 1.0 ? static_cast<int>(q) : cap + 1;   // q >= 1
    return min_servers(need, per, cap);
}

// profiles.cpp:67-71
__device__ __forceinline__ int bins_below(double t) {
    int k = static_cast<int>(ceil(__dsub_rn(__dmul_rn(t, 100.0), 1e-9)));
    return k < 0 ? 0 : (k > DS_CURVE_BINS ? DS_CURVE_BINS : k);
}

// deferral_fraction (profiles.cpp:98-106) from the sequential prefix table.
__device__ __forceinline__ double deferral_fraction(const PlanSmem& s, double total, double t) {
    if (total <= 0.0) return 0.0;
    return __ddiv_rn(s.prefix[bins_below(t)], total);
}

__device__ __forceinline__ unsigned long long warp_min(unsigned long long v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Block-wide min; every thread gets the result. `buf` is one of the
// double-buffered reduction arrays so back-to-back calls need one barrier.
__device__ __forceinline__ unsigned long long block_min(unsigned long long v,
                                                        unsigned long long* buf) {
    v = warp_min(v);
    if ((threadIdx.x & 31) == 0) buf[threadIdx.x >> 5] = v;
    __syncthreads();
    // the 8 warp minima on lanes 0-7 of every warp, reduced by shuffles
    const int lane = threadIdx.x & 31;
    unsigned long long r = lane < kThreads / 32 ? buf[lane] : kNone;
#pragma unroll
    for (int o = kThreads / 64; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, r, o);
        r = w < r ? w : r;
    }
    return __shfl_sync(0xffffffffu, r, 0);
}

// Candidate::better_than tie key at equal threshold (allocator.cpp:57-67).
__device__ __forceinline__ unsigned long long tie_key(int x1, int x2, int i, int j) {
    return (static_cast<unsigned long long>(x1 + x2) << 28) |
           (static_cast<unsigned long long>(255 - i) << 20) |
           (static_cast<unsigned long long>(255 - j) << 12) |
           static_cast<unsigned long long>(x1);
}

// The search (allocator.cpp:91-121) over thresholds `grid[t_lo..t_hi)` of a
// grid of G walked from the top, restricted to b1 index set [i0, i1) and b2
// index set [j0, j1). Returns the winning key (kNone if no candidate is valid).
// Keys carry the GLOBAL threshold index, so the minimum over disjoint
// threshold ranges (e.g. one range per GPU) is the key of the full search.
__device__ unsigned long long search(PlanSmem& s, const double* grid, int G, int t_lo, int t_hi,
                                     int n1, int n2, int i0, int i1, int j0, int j1,
                                     double need_light, double total, int S) {
    const int ni = i1 - i0, nj = j1 - j0;
    if (ni <= 0 || nj <= 0) return kNone;
    const int dq = kThreads / nj, dr = kThreads % nj;   // a kThreads step in (row, column)
    unsigned long long best = kNone;
    int parity = 0;
    for (int hi = t_hi; hi > t_lo; hi -= kTChunk) {
        const int lo = hi - kTChunk > t_lo ? hi - kTChunk : t_lo;
        const int cnt = hi - lo;
        for (int k = threadIdx.x; k < cnt; k += kThreads)
            s.ft[k] = __dmul_rn(need_light, deferral_fraction(s, total, grid[lo + k]));
        __syncthreads();
        // flat index k = tl * nj + (j - j0), stepped by kThreads without a
        // division per entry (one per thread: dq, dr)
        if (dr == 0) {
            // nj divides kThreads (the 32-batch profiles): a thread's column
            // never changes, its T2 and 1/T2 stay in registers
            const int j = j0 + threadIdx.x % nj;
            const double per = s.T2[j], rper = s.rT2[j];
            for (int tl = threadIdx.x / nj; tl < cnt; tl += dq)
                s.x2[tl * kMaxB + j] = static_cast<uint16_t>(min_servers_r(s.ft[tl], per, rper, S));
        } else {
            int tl = threadIdx.x / nj, j = j0 + threadIdx.x % nj;
            for (int k = threadIdx.x; k < cnt * nj; k += kThreads) {
                s.x2[tl * kMaxB + j] = static_cast<uint16_t>(min_servers_r(s.ft[tl], s.T2[j], s.rT2[j], S));
                tl += dq;
                j += dr;
                if (j >= j1) {
                    j -= nj;
                    ++tl;
                }
            }
        }
        __syncthreads();
        // Each thread owns fixed (b1, b2) pairs -- the latency and x1 checks
        // are per pair -- and walks the chunk's thresholds from the top; the
        // first valid t is the pair's best (larger t = smaller key), so the
        // walk stops there. Every (t, b1, b2) candidate of the chunk is still
        // decided (reference semantics); only provably worse keys are skipped.
        // x2[t][j] is non-decreasing in t (the deferral fraction is, and
        // min_servers is monotone in the demand), so a pair's valid thresholds
        // in the chunk are a prefix [0, k] of it and its first valid t from the
        // top is k: found by binary search instead of walking down from the top.
        unsigned long long mine = kNone;
        int pi_ = i0 + threadIdx.x / nj, pj = j0 + threadIdx.x % nj;
        for (int pr = threadIdx.x; pr < ni * nj; pr += kThreads) {
            const int i = pi_, j = pj;
            pi_ += dq;
            pj += dr;
            if (pj >= j1) {
                pj -= nj;
                ++pi_;
            }
            if (!((s.lat[i] >> j) & 1ull)) continue;
            const int x1 = s.x1[i];
            if (x1 > S) continue;
            const int cap = S - x1;
            const uint16_t* col = s.x2 + j;
            if (col[0] > cap) continue;            // even the chunk's lowest t is invalid
            // the last a with col[a * kMaxB] <= cap: branch-free steps of
            // 64, 32, ..., 1 (cnt <= kTChunk = 128)
            int a = 0;
#pragma unroll
            for (int step = kTChunk / 2; step > 0; step >>= 1)
                if (a + step < cnt && col[(a + step) * kMaxB] <= cap) a += step;
            const unsigned long long key =
                (static_cast<unsigned long long>(G - 1 - (lo + a)) << 40) +
                (static_cast<unsigned long long>(col[a * kMaxB]) << 28) + tie_key(x1, 0, i, j);
            mine = key < mine ? key : mine;
        }
        best = block_min(mine, parity ? s.red2 : s.red);
        parity ^= 1;
        if (best != kNone) break;
        __syncthreads();
    }
    (void)n1;
    (void)n2;
    return best;
}

__device__ void decode(const PlanSmem& s, unsigned long long key, const double* grid, int G,
                       ds_plan& plan) {
    const int t_idx = G - 1 - static_cast<int>(key >> 40);
    const int x1 = static_cast<int>(key & 0xFFFull);
    const int tot = static_cast<int>((key >> 28) & 0xFFFull);
    plan.x1 = x1;
    plan.x2 = tot - x1;
    plan.b1 = s.b1[255 - static_cast<int>((key >> 20) & 0xFFull)];
    plan.b2 = s.b2[255 - static_cast<int>((key >> 12) & 0xFFull)];
    plan.threshold = grid[t_idx];
    plan.feasible = 1;
}

// best_effort_light (allocator.cpp:70-88): throughput-max light batch, ties
// toward the larger batch.
__device__ void best_effort_light(const PlanSmem& s, int n1, int S, ds_plan& plan) {
    int best_b = s.b1[0];
    double best_T = s.T1[0];
    for (int i = 0; i < n1; ++i)
        if (s.T1[i] >= best_T) {
            best_T = s.T1[i];
            best_b = s.b1[i];
        }
    plan.x1 = S;
    plan.x2 = 0;
    plan.b1 = best_b;
    plan.b2 = s.b2[0];
    plan.threshold = 0.0;
    plan.feasible = 0;
}

// solve_single_model (allocator.cpp:232-268), serial.
__device__ void single_model(const double* e, const double* T, const int* b, int n,
                             bool is_light, int S, double need, double slo, ds_plan& plan) {
    plan.threshold = 0.0;
    auto assign = [&](int bb, bool feas) {
        if (is_light) { plan.x1 = S; plan.x2 = 0; plan.b1 = bb; plan.b2 = 0; }
        else { plan.x1 = 0; plan.x2 = S; plan.b1 = 0; plan.b2 = bb; }
        plan.feasible = feas ? 1 : 0;
    };
    int first = -1;
    for (int i = 0; i < n; ++i) {
        if (!(__dmul_rn(2.0, e[i]) <= slo)) continue;
        if (first < 0) first = i;
        if (__dmul_rn(static_cast<double>(S), T[i]) >= need) {
            assign(b[i], true);
            return;
        }
    }
    if (first >= 0) {
        int best = first;
        for (int i = 0; i < n; ++i)
            if (__dmul_rn(2.0, e[i]) <= slo && T[i] >= T[best]) best = i;
        assign(b[best], false);
        return;
    }
    assign(b[0], false);
}

// `cheapest` lambda of solve_even_split (allocator.cpp:283-291).
__device__ void cheapest(const double* e, const double* T, const int* b, int n, double slo,
                         double side_need, int cap, int& bx, int& bb) {
    int best_x = cap + 1, best_b = 0;
    for (int i = 0; i < n; ++i) {
        if (!(__dmul_rn(2.0, e[i]) <= slo)) continue;
        int x = min_servers(side_need, T[i], cap);
        if (x < 1) x = 1;
        if (x < best_x || (x == best_x && b[i] > best_b)) {
            best_x = x;
            best_b = b[i];
        }
    }
    bx = best_x;
    bb = best_b;
}

#ifndef DS_PLAN_MINB
#define DS_PLAN_MINB 6   // 40 registers: 6 CTAs (48 warps) per SM
#endif
__global__ void __launch_bounds__(kThreads, DS_PLAN_MINB)
plan_sweep_kernel(const ds_problem* __restrict__ problems, int n,
                  const ds_cascade* __restrict__ cascades,
                  const double* __restrict__ grid_values,
                  const int32_t* __restrict__ grid_offsets, ds_plan* __restrict__ out,
                  int t_lo, int t_hi, unsigned long long* __restrict__ keys_out,
                  const unsigned long long* __restrict__ keys_in,
                  const double* __restrict__ prefix_tab) {
    // keys_out: search grid indices [t_lo, t_hi) only and write the packed key
    //           (grid modes; kNone for the others) instead of a plan.
    // keys_in : skip the search of grid modes and decode the given key (the
    //           min over ranks of keys_out), with the reference's fallbacks.
    __shared__ PlanSmem s;
    const int pi = blockIdx.x;
    if (pi >= n) return;
    const ds_problem p = problems[pi];
    const ds_cascade* c = cascades + p.cascade;
    const int n1 = c->light.n, n2 = c->heavy.n;
    const int S = p.total_servers;
    const int tid = threadIdx.x;
    const double need_light = __dmul_rn(p.overprovision_lambda, p.demand_qps);
    const double total = c->deferral.total_mass;
    const double slo = c->slo_seconds;

    if (tid < n1) {
        const int b = c->light.batch[tid];
        const double e = c->light.latency[tid];
        s.b1[tid] = b;
        s.e1[tid] = e;
        s.T1[tid] = __ddiv_rn(static_cast<double>(b), e);
    } else if (tid >= 64 && tid - 64 < n2) {
        const int j = tid - 64;
        const int b = c->heavy.batch[j];
        const double e = c->heavy.latency[j];
        s.b2[j] = b;
        s.e2[j] = e;
        s.T2[j] = __ddiv_rn(static_cast<double>(b), e);
        s.rT2[j] = __drcp_rn(s.T2[j]);
    } else if (tid >= 128 && tid - 128 <= DS_CURVE_BINS) {
        // the cascade's sequential prefix table (built once per call by
        // curve_prefix_kernel, in the reference's summation order)
        s.prefix[tid - 128] = prefix_tab[p.cascade * (DS_CURVE_BINS + 1) + (tid - 128)];
    }
    __syncthreads();

    ds_plan plan;
    plan.x1 = plan.x2 = plan.b1 = plan.b2 = 0;
    plan.threshold = 0.0;
    plan.feasible = 0;
    plan._pad = 0;

    const int mode = p.mode;
    if (mode == DS_SOLVE || mode == DS_SOLVE_PINNED || mode == DS_SOLVE_FIXED_BATCHES) {
        // Pair admissibility and x1 per light batch (allocator.cpp:95-112).
        const bool twice = p.queuing == DS_QUEUING_TWICE_EXEC;
        const double q1c = twice ? 0.0 : queuing_delay(p.light_len, p.light_rate,
                                                       p.queue_sentinel_seconds);
        const double q2c = twice ? 0.0 : queuing_delay(p.heavy_len, p.heavy_rate,
                                                       p.queue_sentinel_seconds);
        if (tid < n1) {
            const double e1 = s.e1[tid];
            const double q1 = twice ? __dmul_rn(2.0, e1) : q1c;
            unsigned long long m = 0;
            for (int j = 0; j < n2; ++j) {
                const double e2 = s.e2[j];
                const double q2 = twice ? __dmul_rn(2.0, e2) : q2c;
                const double lat = __dadd_rn(__dadd_rn(__dadd_rn(e1, q1), e2), q2);
                if (lat <= slo) m |= 1ull << j;
            }
            s.lat[tid] = m;
            int x1 = min_servers(need_light, s.T1[tid], S);
            s.x1[tid] = x1 < 1 ? 1 : x1;
        }
        __syncthreads();

        int i0 = 0, i1 = n1, j0 = 0, j1 = n2;
        if (mode == DS_SOLVE_FIXED_BATCHES) {
            for (int i = 0; i < n1; ++i)
                if (s.b1[i] == p.fixed_b1) { i0 = i; i1 = i + 1; }
            for (int j = 0; j < n2; ++j)
                if (s.b2[j] == p.fixed_b2) { j0 = j; j1 = j + 1; }
        }
        const double* grid;
        int G;
        if (mode == DS_SOLVE_PINNED) {
            grid = &problems[pi].fixed_threshold;
            G = 1;
        } else {
            grid = grid_values + grid_offsets[p.grid];
            G = grid_offsets[p.grid + 1] - grid_offsets[p.grid];
        }
        const bool grid_mode = mode != DS_SOLVE_PINNED;
        unsigned long long key;
        if (keys_in && grid_mode) {
            key = keys_in[pi];
        } else {
            const int lo = keys_out && grid_mode ? (t_lo > 0 ? t_lo : 0) : 0;
            const int hi = keys_out && grid_mode ? (t_hi < G ? t_hi : G) : G;
            key = search(s, grid, G, lo, hi, n1, n2, i0, i1, j0, j1, need_light, total, S);
        }
        if (keys_out) {
            if (tid == 0) keys_out[pi] = grid_mode ? key : kNone;
            return;
        }
        if (key != kNone) {
            decode(s, key, grid, G, plan);
        } else if (mode == DS_SOLVE) {
            best_effort_light(s, n1, S, plan);
        } else if (mode == DS_SOLVE_FIXED_BATCHES) {
            // allocator.cpp:219-229
            int x1 = min_servers(need_light, s.T1[i0], S);
            x1 = x1 < 1 ? 1 : x1;
            plan.x1 = x1 < S ? x1 : S;
            plan.x2 = 0;
            plan.b1 = s.b1[i0];
            plan.b2 = s.b2[j0];
            plan.threshold = 0.0;
            plan.feasible = 0;
        } else {
            // Pinned-threshold deficit fallback (allocator.cpp:184-210):
            // lexicographic min of (deficit, better_than) over ALL pairs.
            __syncthreads();
            const double t = p.fixed_threshold;
            const double need_heavy = __dmul_rn(need_light, deferral_fraction(s, total, t));
            unsigned long long dmin = kNone, tmin = kNone;
            double dmine[(kMaxB * kMaxB + kThreads - 1) / kThreads];
            unsigned long long kmine[(kMaxB * kMaxB + kThreads - 1) / kThreads];
            int slot = 0;
            for (int k = tid; k < n1 * n2; k += kThreads, ++slot) {
                const int i = k / n2, j = k % n2;
                int x1 = min_servers(need_light, s.T1[i], S);
                x1 = x1 < 1 ? 1 : x1;
                x1 = x1 < S ? x1 : S;
                int x2 = min_servers(need_heavy, s.T2[j], S);
                x2 = x2 < S - x1 ? x2 : S - x1;
                const double d1 = __dsub_rn(need_light, __dmul_rn(static_cast<double>(x1), s.T1[i]));
                const double d2 = __dsub_rn(need_heavy, __dmul_rn(static_cast<double>(x2), s.T2[j]));
                const double def = __dadd_rn(d1 > 0.0 ? d1 : 0.0, d2 > 0.0 ? d2 : 0.0);
                dmine[slot] = def;
                kmine[slot] = tie_key(x1, x2, i, j);
                const unsigned long long bits =
                    static_cast<unsigned long long>(__double_as_longlong(def));
                dmin = bits < dmin ? bits : dmin;
            }
            dmin = block_min(dmin, s.red);
            slot = 0;
            for (int k = tid; k < n1 * n2; k += kThreads, ++slot) {
                const unsigned long long bits =
                    static_cast<unsigned long long>(__double_as_longlong(dmine[slot]));
                if (bits == dmin) tmin = kmine[slot] < tmin ? kmine[slot] : tmin;
            }
            tmin = block_min(tmin, s.red2);
            const int x1 = static_cast<int>(tmin & 0xFFFull);
            plan.x1 = x1;
            plan.x2 = static_cast<int>((tmin >> 28) & 0xFFFull) - x1;
            plan.b1 = s.b1[255 - static_cast<int>((tmin >> 20) & 0xFFull)];
            plan.b2 = s.b2[255 - static_cast<int>((tmin >> 12) & 0xFFull)];
            plan.threshold = t;
            plan.feasible = 0;
        }
    } else if (keys_out) {
        if (tid == 0) keys_out[pi] = kNone;
        return;
    } else if (tid == 0) {
        if (mode == DS_SOLVE_SINGLE_LIGHT || mode == DS_SOLVE_SINGLE_HEAVY) {
            const bool light = mode == DS_SOLVE_SINGLE_LIGHT;
            single_model(light ? s.e1 : s.e2, light ? s.T1 : s.T2, light ? s.b1 : s.b2,
                         light ? n1 : n2, light, S, need_light, slo, plan);
        } else { // DS_SOLVE_EVEN_SPLIT, allocator.cpp:270-313
            int xh, bh;
            cheapest(s.e2, s.T2, s.b2, n2, slo, need_light, S, xh, bh);
            if (bh != 0 && xh <= S) {
                plan.x1 = 0; plan.x2 = xh; plan.b1 = 0; plan.b2 = bh;
                plan.threshold = 0.0; plan.feasible = 1;
            } else {
                const double half = __ddiv_rn(need_light, 2.0);
                int x1, b1, x2, b2;
                cheapest(s.e1, s.T1, s.b1, n1, slo, half, S, x1, b1);
                cheapest(s.e2, s.T2, s.b2, n2, slo, half, S, x2, b2);
                if (b1 != 0 && b2 != 0 && x1 + x2 <= S) {
                    plan.x1 = x1; plan.x2 = x2; plan.b1 = b1; plan.b2 = b2;
                    plan.threshold = 0.0; plan.feasible = 1;
                } else {
                    single_model(s.e1, s.T1, s.b1, n1, true, S, need_light, slo, plan);
                    plan.b2 = s.b2[0];
                }
            }
        }
    }
    if (tid == 0) out[pi] = plan;
}

// ---- host-side validation: the reference's checks, in the reference's order

std::string fmt_int(long long v) { return std::to_string(v); }

ds_status validate_profile(const ds_model_profile& m, const char* which) {
    if (m.n < 1) return dsi::fail(DS_ERR_INVARIANT, std::string("profile '") + which +
                                                       "': latency table is empty");
    if (m.n > DS_MAX_BATCHES)
        return dsi::fail(DS_ERR_CAPACITY, std::string("profile '") + which + "': more than " +
                                              fmt_int(DS_MAX_BATCHES) + " batch sizes");
    for (int i = 0; i < m.n; ++i) {
        if (m.batch[i] <= 0)
            return dsi::fail(DS_ERR_INVARIANT, std::string("profile '") + which +
                                                   "': non-positive batch size");
        if (i > 0 && m.batch[i] <= m.batch[i - 1])
            return dsi::fail(DS_ERR_INVARIANT, std::string("profile '") + which +
                                                   "': batch sizes must be strictly ascending");
        if (!(m.latency[i] > 0.0) || !std::isfinite(m.latency[i]))
            return dsi::fail(DS_ERR_INVARIANT, std::string("profile '") + which +
                                                   "': latency for batch " +
                                                   fmt_int(m.batch[i]) +
                                                   " must be positive and finite");
    }
    return DS_OK;
}

bool has_batch(const ds_model_profile& m, int b) {
    for (int i = 0; i < m.n; ++i)
        if (m.batch[i] == b) return true;
    return false;
}

} // namespace

extern "C" ds_status ds_plan_validate(const ds_problem* problems, int32_t n,
                                      const ds_cascade* cascades, int32_t n_cascades,
                                      const double* grid_values, const int32_t* grid_offsets,
                                      int32_t n_grids) {
    if (n < 0 || (n > 0 && (!problems || !cascades)))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "ds_plan_batch: null input");
    for (int c = 0; c < n_cascades; ++c) {
        ds_status st = validate_profile(cascades[c].light, "light");
        if (st == DS_OK) st = validate_profile(cascades[c].heavy, "heavy");
        if (st != DS_OK) return st;
    }
    for (int g = 0; g < n_grids; ++g) {
        const int len = grid_offsets[g + 1] - grid_offsets[g];
        if (len > kMaxGrid) return dsi::fail(DS_ERR_CAPACITY, "threshold grid too long");
    }
    for (int i = 0; i < n; ++i) {
        const ds_problem& p = problems[i];
        const std::string at = " (problem " + fmt_int(i) + ")";
        if (p.cascade < 0 || p.cascade >= n_cascades)
            return dsi::fail(DS_ERR_INVALID_ARGUMENT, "allocation problem has no cascade" + at);
        const ds_cascade& c = cascades[p.cascade];
        const int mode = p.mode;
        if (mode < DS_SOLVE || mode > DS_SOLVE_SINGLE_HEAVY)
            return dsi::fail(DS_ERR_INVALID_ARGUMENT, "unknown solve mode" + at);
        // check_problem (allocator.cpp:22-28); solve_single_model checks S only.
        if (p.total_servers < 1)
            return dsi::fail(DS_ERR_DOMAIN, "total_servers must be at least 1" + at);
        if (p.total_servers > kMaxServers)
            return dsi::fail(DS_ERR_CAPACITY, "total_servers above " + fmt_int(kMaxServers) + at);
        const bool single = mode == DS_SOLVE_SINGLE_LIGHT || mode == DS_SOLVE_SINGLE_HEAVY;
        if (!single) {
            if (!(p.demand_qps >= 0.0))
                return dsi::fail(DS_ERR_DOMAIN, "demand must be non-negative" + at);
            if (!(p.overprovision_lambda >= 1.0))
                return dsi::fail(DS_ERR_DOMAIN, "overprovision lambda must be >= 1" + at);
        }
        if (mode == DS_SOLVE || mode == DS_SOLVE_FIXED_BATCHES) {
            // check_grid (allocator.cpp:30-36)
            if (p.grid < 0 || p.grid >= n_grids)
                return dsi::fail(DS_ERR_INVARIANT,
                                 "threshold grid must be non-empty and start at 0" + at);
            const double* g = grid_values + grid_offsets[p.grid];
            const int len = grid_offsets[p.grid + 1] - grid_offsets[p.grid];
            if (len == 0 || g[0] != 0.0)
                return dsi::fail(DS_ERR_INVARIANT,
                                 "threshold grid must be non-empty and start at 0" + at);
            for (int k = 1; k < len; ++k)
                if (!(g[k] > g[k - 1]))
                    return dsi::fail(DS_ERR_INVARIANT,
                                     "threshold grid must be strictly increasing" + at);
            if (mode == DS_SOLVE_FIXED_BATCHES) {
                if (!has_batch(c.light, p.fixed_b1))
                    return dsi::fail(DS_ERR_OUT_OF_RANGE, "model 'light' has no profiled batch size " +
                                                              fmt_int(p.fixed_b1) + at);
                if (!has_batch(c.heavy, p.fixed_b2))
                    return dsi::fail(DS_ERR_OUT_OF_RANGE, "model 'heavy' has no profiled batch size " +
                                                              fmt_int(p.fixed_b2) + at);
            }
        }
        if (mode == DS_SOLVE_PINNED &&
            (!(p.fixed_threshold >= 0.0) || !(p.fixed_threshold <= 1.0)))
            return dsi::fail(DS_ERR_DOMAIN, "fixed threshold must lie in [0, 1]" + at);
        if ((mode == DS_SOLVE || mode == DS_SOLVE_PINNED || mode == DS_SOLVE_FIXED_BATCHES) &&
            p.queuing != DS_QUEUING_TWICE_EXEC) {
            // queuing_delay's checks, reached through latency_feasible
            if (p.light_len < 0 || p.heavy_len < 0)
                return dsi::fail(DS_ERR_DOMAIN, "queue length cannot be negative" + at);
            if (p.light_rate < 0.0 || p.heavy_rate < 0.0)
                return dsi::fail(DS_ERR_DOMAIN, "arrival rate cannot be negative" + at);
        }
        if (mode == DS_SOLVE || mode == DS_SOLVE_FIXED_BATCHES) {
            // the top threshold is the first deferral_fraction call (profiles.cpp:99-100)
            const double top = grid_values[grid_offsets[p.grid + 1] - 1];
            if (!(top <= 1.0))
                return dsi::fail(DS_ERR_DOMAIN, "deferral threshold must lie in [0, 1]" + at);
        }
    }
    return DS_OK;
}

namespace {

// deferral_fraction's running sum below each bin (profiles.cpp:98-106): one
// thread per cascade adds the bins in order, so every prefix entry is
// bit-identical to the reference's `below`.
__global__ void curve_prefix_kernel(const ds_cascade* __restrict__ cascades, int nc,
                                    double* __restrict__ tab) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= nc) return;
    double acc = 0.0;   // profiles.cpp:104: below += bin_mass[i], in order
    double* t = tab + static_cast<size_t>(c) * (DS_CURVE_BINS + 1);
    t[0] = 0.0;
    for (int k = 0; k < DS_CURVE_BINS; ++k) {
        acc = __dadd_rn(acc, cascades[c].deferral.bin_mass[k]);
        t[k + 1] = acc;
    }
}

ds_status launch_sweep(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                       const ds_cascade* cascades, int32_t n_cascades, const double* grid_values,
                       const int32_t* grid_offsets, ds_plan* out, int t_lo, int t_hi,
                       unsigned long long* keys_out, const unsigned long long* keys_in,
                       cudaStream_t st) {
    if (n_cascades <= 0) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "no cascades");
    double* tab = nullptr;
    DS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&tab),
                                sizeof(double) * (DS_CURVE_BINS + 1) * n_cascades, st));
    static bool carveout = [] {   // all of the unified L1 as shared memory: more CTAs per SM
        cudaFuncSetAttribute(plan_sweep_kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                             cudaSharedmemCarveoutMaxShared);
        return true;
    }();
    (void)carveout;
    curve_prefix_kernel<<<(n_cascades + 31) / 32, 32, 0, st>>>(cascades, n_cascades, tab);
    DS_LAUNCH_CHECK(ctx, "curve_prefix_kernel");
    plan_sweep_kernel<<<n, kThreads, 0, st>>>(problems, n, cascades, grid_values, grid_offsets,
                                              out, t_lo, t_hi, keys_out, keys_in, tab);
    DS_LAUNCH_CHECK(ctx, "plan_sweep_kernel");
    cudaFreeAsync(tab, st);
    return DS_OK;
}

} // namespace

extern "C" ds_status ds_plan_batch_device(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                                          const ds_cascade* cascades, int32_t n_cascades,
                                          const double* grid_values,
                                          const int32_t* grid_offsets, int32_t n_grids,
                                          ds_plan* out, void* stream) {
    (void)n_grids;
    if (!ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
    if (n <= 0) return DS_OK;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    return launch_sweep(ctx, problems, n, cascades, n_cascades, grid_values, grid_offsets, out, 0,
                        0, nullptr, nullptr, st);
}

extern "C" ds_status ds_plan_keys_device(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                                         const ds_cascade* cascades, int32_t n_cascades,
                                         const double* grid_values, const int32_t* grid_offsets,
                                         int32_t n_grids, int32_t t_lo, int32_t t_hi,
                                         uint64_t* keys, void* stream) {
    (void)n_grids;
    if (!ctx || (n > 0 && !keys)) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (t_lo < 0 || t_hi < t_lo) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "bad threshold range");
    if (n <= 0) return DS_OK;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    return launch_sweep(ctx, problems, n, cascades, n_cascades, grid_values, grid_offsets, nullptr,
                        t_lo, t_hi, reinterpret_cast<unsigned long long*>(keys), nullptr, st);
}

extern "C" ds_status ds_plan_from_keys_device(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                                              const ds_cascade* cascades, int32_t n_cascades,
                                              const double* grid_values,
                                              const int32_t* grid_offsets, int32_t n_grids,
                                              const uint64_t* keys, ds_plan* out, void* stream) {
    (void)n_grids;
    if (!ctx || (n > 0 && (!keys || !out))) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (n <= 0) return DS_OK;
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
    return launch_sweep(ctx, problems, n, cascades, n_cascades, grid_values, grid_offsets, out, 0,
                        0, nullptr, reinterpret_cast<const unsigned long long*>(keys), st);
}

namespace {

// Host-buffer entry points: validate (the reference's checks), stage the
// inputs into the ctx scratch, run `launch` on the device copies, copy `out_bytes`
// of results back from the scratch tail.
struct Staged {
    ds_problem* p;
    ds_cascade* c;
    double* g;
    int32_t* o;
    char* out;
};

template <class Launch>
ds_status staged_call(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                      const ds_cascade* cascades, int32_t n_cascades, const double* grid_values,
                      const int32_t* grid_offsets, int32_t n_grids, const void* in_extra,
                      size_t in_bytes, void* out, size_t out_bytes, Launch launch) {
    if (!ctx) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null ctx");
    ds_status st = ds_plan_validate(problems, n, cascades, n_cascades, grid_values,
                                    grid_offsets, n_grids);
    if (st != DS_OK) return st;
    if (n == 0) return DS_OK;
    const int n_vals = n_grids > 0 ? grid_offsets[n_grids] : 0;
    const size_t bp = dsi::align_up(sizeof(ds_problem) * n, 256);
    const size_t bc = dsi::align_up(sizeof(ds_cascade) * n_cascades, 256);
    const size_t bg = dsi::align_up(sizeof(double) * (n_vals > 0 ? n_vals : 1), 256);
    const size_t bo = dsi::align_up(sizeof(int32_t) * (n_grids + 1), 256);
    const size_t bi = dsi::align_up(in_bytes > 0 ? in_bytes : 1, 256);
    const size_t bout = dsi::align_up(out_bytes, 256);
    char* d = nullptr;
    st = dsi::ensure_scratch(ctx, bp + bc + bg + bo + bi + bout, reinterpret_cast<void**>(&d));
    if (st != DS_OK) return st;
    DS_CUDA_TRY(cudaMemcpyAsync(d, problems, sizeof(ds_problem) * n, cudaMemcpyHostToDevice,
                                ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(d + bp, cascades, sizeof(ds_cascade) * n_cascades,
                                cudaMemcpyHostToDevice, ctx->stream));
    if (n_vals > 0)
        DS_CUDA_TRY(cudaMemcpyAsync(d + bp + bc, grid_values, sizeof(double) * n_vals,
                                    cudaMemcpyHostToDevice, ctx->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(d + bp + bc + bg, grid_offsets, sizeof(int32_t) * (n_grids + 1),
                                cudaMemcpyHostToDevice, ctx->stream));
    char* din = d + bp + bc + bg + bo;
    if (in_bytes > 0)
        DS_CUDA_TRY(cudaMemcpyAsync(din, in_extra, in_bytes, cudaMemcpyHostToDevice, ctx->stream));
    Staged sp{reinterpret_cast<ds_problem*>(d), reinterpret_cast<ds_cascade*>(d + bp),
              reinterpret_cast<double*>(d + bp + bc), reinterpret_cast<int32_t*>(d + bp + bc + bg),
              din + bi};
    st = launch(sp, din);
    if (st != DS_OK) return st;
    DS_CUDA_TRY(cudaMemcpyAsync(out, sp.out, out_bytes, cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DS_OK;
}

} // namespace

extern "C" ds_status ds_plan_batch(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                                   const ds_cascade* cascades, int32_t n_cascades,
                                   const double* grid_values, const int32_t* grid_offsets,
                                   int32_t n_grids, ds_plan* out) {
    return staged_call(ctx, problems, n, cascades, n_cascades, grid_values, grid_offsets, n_grids,
                       nullptr, 0, out, sizeof(ds_plan) * (n > 0 ? n : 0),
                       [&](const Staged& sp, char*) {
                           return ds_plan_batch_device(ctx, sp.p, n, sp.c, n_cascades, sp.g, sp.o,
                                                       n_grids, reinterpret_cast<ds_plan*>(sp.out),
                                                       ctx->stream);
                       });
}

extern "C" ds_status ds_plan_keys(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                                  const ds_cascade* cascades, int32_t n_cascades,
                                  const double* grid_values, const int32_t* grid_offsets,
                                  int32_t n_grids, int32_t t_lo, int32_t t_hi, uint64_t* keys) {
    if (t_lo < 0 || t_hi < t_lo) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "bad threshold range");
    return staged_call(ctx, problems, n, cascades, n_cascades, grid_values, grid_offsets, n_grids,
                       nullptr, 0, keys, sizeof(uint64_t) * (n > 0 ? n : 0),
                       [&](const Staged& sp, char*) {
                           return ds_plan_keys_device(ctx, sp.p, n, sp.c, n_cascades, sp.g, sp.o,
                                                      n_grids, t_lo, t_hi,
                                                      reinterpret_cast<uint64_t*>(sp.out),
                                                      ctx->stream);
                       });
}

extern "C" ds_status ds_plan_from_keys(ds_ctx* ctx, const ds_problem* problems, int32_t n,
                                       const ds_cascade* cascades, int32_t n_cascades,
                                       const double* grid_values, const int32_t* grid_offsets,
                                       int32_t n_grids, const uint64_t* keys, ds_plan* out) {
    return staged_call(ctx, problems, n, cascades, n_cascades, grid_values, grid_offsets, n_grids,
                       keys, sizeof(uint64_t) * (n > 0 ? n : 0), out,
                       sizeof(ds_plan) * (n > 0 ? n : 0),
                       [&](const Staged& sp, char* din) {
                           return ds_plan_from_keys_device(
                               ctx, sp.p, n, sp.c, n_cascades, sp.g, sp.o, n_grids,
                               reinterpret_cast<const uint64_t*>(din),
                               reinterpret_cast<ds_plan*>(sp.out), ctx->stream);
                       });
}
