// K5-K7: the discriminator ("PatchDisc") as one fused, warp-specialized
// tcgen05 kernel. No reference implementation exists (SPEC.md:8 models the
// discriminator as a latent score, see latent.cu); the network is this
// repo's (SURVEY.md 8(a) row S9 -- "bf16 in, fp32 accumulate (or u8 x s8 ->
// s32 for layer 1)" -- and DESIGN.md "Discriminator"):
//
//   u8 NHWC image -> 16x16x3 patches (token t = py*(W/16)+px, feature
//   k = dy*48 + dx*3 + c) -> h1 = GELU_tanh(s1 * (x @ Q1) + b1)  [768 -> 256]
//   -> h2 = ReLU(bf16(h1) @ W2)  [256 -> 1024] -> h3 = ReLU(bf16(h2) @ W3)
//   [1024 -> 256] -> logit = mean_t(h3 . w_head) + b_head -> sigmoid.
// Layer 1 is an INTEGER GEMM: the raw pixel bytes x (u8) against int8 weights
// Q1, accumulated exactly in s32 by tcgen05.mma kind::i8 (twice the bf16
// tensor rate per byte of operand, and the A tile is the pixel bytes
// themselves: no u8 -> bf16 conversion). The (x-128)/64 input normalisation
// and the weight scale s1 fold into the epilogue: h1_pre = fma(float(acc),
// s1, b1). Layers 2 and 3 carry their biases as weights of CONSTANT hidden
// features: Q1[:,255] = 0 and b1[255] = 16 give h1[:,255] = GELU(16) = 16
// exactly, so W2[255,:] is layer 2's bias (/16); W2[:,1023] is zero except
// W2[255,1023] = 1, so h2[:,1023] = 16 and W3[1023,:] is layer 3's bias.
// The epilogue therefore never adds a bias after GEMM2/GEMM3.
//
// SM pairs (cta_group::2), persistent; 256-token pair tiles are dealt round
// robin over the pairs (one head sum per 128-token tile, summed per image in
// tile order by finalize_kernel, so results do not depend on the batch
// split). Each CTA of a pair
// owns 128 tokens of a 256-token pair tile and HALF of every weight stage
// (128 of the 256 output rows), so each SM streams 0.6 MB of weights per 128
// tokens instead of 1.2 MB; one thread of the leader CTA issues M = 256 MMAs
// that read both CTAs' shared memory and write both CTAs' TMEM.
//   warps 0-3   A-builder: 128-bit loads of 16 B pixel runs (thread = token;
//               L1-allocating, so a patch row's three runs share sectors)
//               stored as-is into a 2-stage SW128 ring plus two W1 slots of
//               the H1 region (6 chunks of K = 128 bytes per tile); a CTA's
//               first two chunks are loaded before the set-up barriers; one
//               thread bulk-prefetches the tiles two ahead into L2; after
//               GEMM1 they also run E1 on columns [192, 256)
//   warps 4-11  epilogue: tcgen05.ld of this CTA's TMEM lanes, activation,
//               bf16 pack, SW128 stores of H1/H2 (next GEMM's A operand), and
//               the head dot product (E3, per-tile sum)
//   warp 12     weight producer: tensor-map TMA of this CTA's 16 KB half of
//               each pre-swizzled 32 KB stage (256 rows x 128 B, SW128; L2
//               evict-last) into a 4-stage ring; completion lands on the
//               LEADER's barrier (cta_group::2); its lane 0 also initialises
//               the barriers (off the A-builders, whose first loads go first)
//   warp 13     TMEM allocator (both CTAs) + the MMA-issuing thread (leader)
//   warp 14     W1 stages 0-3 into the H1 region, which is idle during GEMM1
//               (and the L2 prefetch of a CTA's first two tiles)
// Every weight stage and A chunk is 4 MMAs (K = 64 bf16 / 128 int8), so the
// issuing thread waits once per 512 MMA-cycles (waits every 2 MMAs cost the
// tensor pipe ~15%, tools/i8_rate_probe.cu).
// Readiness of the peer CTA's shared memory (A chunks, H1/H2 stores, drained
// accumulators) reaches the leader through one remote mbarrier arrive per
// event after a named barrier; the MMA commits multicast to both CTAs.
// TMEM (512 columns per CTA): [0,256) accumulates GEMM1 (s32) and each
// 256-wide N-chunk j of GEMM2 (f32); [256,512) accumulates GEMM3. MMA issue
// order per pair tile i:
//   G1(i) | G3_3(i-1) | G2_0(i) | G2_1(i) G3_0(i) | G2_2(i) G3_1(i) | G2_3(i) G3_2(i)
// The epilogue signals "accumulator drained" as soon as its TMEM loads land
// (packed bf16 values stay in registers) and stores H2_j only after the GEMM3
// still reading the previous H2 chunk committed, so G2_{j+1} overlaps E2_j and
// G3_3(i-1) overlaps E1(i). E1 hands GEMM2_0 its operands piecewise
// (acc_read: every TMEM read of the GEMM1 accumulator done; then H1 K-chunks
// 0/1, 2 and 3 as they are stored), so GEMM2_0's first K-chunks run while E1
// still activates. GEMM2_0's first two weight stages are parked in the
// A slots (free from GEMM1's end until the next tile's first chunks), loaded
// right after GEMM1 by warp 14; E3(i-1) runs after E2_0(i).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "ds_internal.h"
#include "sm100.cuh"

namespace {

using namespace sm100;

constexpr int kM = 128;                 // tokens per CTA per tile (256 per pair)
constexpr int kD0 = DS_DISC_D0, kD1 = DS_DISC_D1, kD2 = DS_DISC_D2, kD3 = DS_DISC_D3;
constexpr int kBStage = 32768;          // one blob stage: 256 rows (N) x 128 bytes of K, SW128
constexpr int kBHalf = kBStage / 2;     // the N-half one CTA loads
constexpr int kW1Stages = 6, kWChunkStages = 4;    // W1: K = 768 int8; W2/W3 chunk: K = 256 bf16
constexpr int kBlobStages = kW1Stages + 8 * kWChunkStages;   // W1 | W2_0..3 | W3_0..3 = 38
constexpr int kAChunk = 16384;          // 128 token rows x 128 bytes of K, SW128
constexpr int kChunksPerTile = 6;       // K = 768 = 6 x 128 (u8)
constexpr int kThreads = 480;
constexpr float kConst = 16.0f;         // value of the constant features
#ifndef DS_A_STAGES
#define DS_A_STAGES 2
#endif
constexpr int kAStages = DS_A_STAGES, kBStages = 6 - DS_A_STAGES;   // 6 x 16 KB of rings
constexpr int kXStages = 4;             // W1 stages 0-3 land in the H1 region (idle during GEMM1)
#ifndef DS_AX
#define DS_AX 1
#endif
// GEMM1's A chunks 3 and 5 go to the H1 region's W1 stage 0 / 1 slots once
// chunks 0 / 1 (which read those weights) completed: with the 2-slot ring,
// four chunk slots in flight after the first two (chunks 0,2 -> ring slot 0;
// 1,4 -> slot 1; 3 -> X0; 5 -> X1)
constexpr bool kAX = DS_AX != 0;
static_assert(!kAX || kAStages == 2, "the X-slot schedule assumes a 2-slot A ring");
#ifndef DS_AW
#define DS_AW 1
#endif
constexpr int kAWStages = DS_AW ? 2 : 0; // W2_0 stages 0-1 land in the A ring (idle from GEMM1's
                                        // end until GEMM2_0 has read them)
#ifndef DS_WARP_ARRIVE
#define DS_WARP_ARRIVE 0   // 1: role groups signal the leader's barriers with one arrive per warp
#endif
constexpr bool kWarpArrive = DS_WARP_ARRIVE != 0;
#ifndef DS_G33_IL
#define DS_G33_IL 0   // >0: the previous tile's GEMM3_3 K-chunk q is issued after GEMM1 chunk DS_G33_IL + q
#endif
constexpr int kG33Il = DS_G33_IL;
#ifndef DS_A_RECOMPUTE
#define DS_A_RECOMPUTE 1
#endif
#ifndef DS_A_REORDER
#define DS_A_REORDER 1   // the A-builders store chunks 2 and 3 before loading 4 and 5 (0: interleaved)
#endif
#ifndef DS_PREFETCH
#define DS_PREFETCH 1
#endif
constexpr int kPrefetch = DS_PREFETCH;   // image tiles two ahead into L2: 1 bulk (TMA), 2 lines (LSU), 0 off
#ifndef DS_EXP_NO_TANH
#define DS_EXP_NO_TANH 0
#endif
#ifndef DS_EXP_NO_ALOAD
#define DS_EXP_NO_ALOAD 0
#endif
#ifndef DS_EXP_FAST_E1
#define DS_EXP_FAST_E1 0
#endif
#ifndef DS_EXP_NO_WSTREAM
#define DS_EXP_NO_WSTREAM 0
#endif
#ifndef DS_E1_PIPE
#define DS_E1_PIPE 0
#endif
#ifndef DS_E1_EARLY
#define DS_E1_EARLY 1
#endif
// E1 hands GEMM2_0 its operands piecewise: "every TMEM read of the GEMM1
// accumulator done" (acc_read: GEMM2_0 may overwrite it) and H1 K-chunk 0 / 1
// stored (h1c) come before the rest of E1, so GEMM2_0's first K-chunks run
// while E1 still computes and stores K-chunks 2 (epilogue) and 3 (builders).
constexpr bool kE1Early = DS_E1_EARLY != 0;
#ifndef DS_E1_SINGLE
#define DS_E1_SINGLE 0
#endif
#ifndef DS_E1_SPLIT
#define DS_E1_SPLIT 192
#endif
constexpr int kE1Split = DS_E1_SPLIT;   // E1 columns [0,192): epilogue warps; [192,256): A-builders
static_assert(!kE1Early || (kE1Split == 192 && !DS_E1_PIPE && !DS_E1_SINGLE),
              "the early E1 hand-off assumes the 192/64 split and the paired TMEM loads");
static_assert(kE1Split % 64 == 0 && kE1Split >= 64 && kE1Split <= 256, "E1 split: 32-column blocks per half");
// shared memory map (bytes, per CTA)
constexpr int kR1 = 0;                              // H1: 4 K-chunks x 16 KB (bf16, SW128)
constexpr int kR2 = kR1 + 65536;                    // H2_j: 4 K-chunks x 16 KB
constexpr int kARing = kR2 + 65536;
constexpr int kBRing = kARing + kAStages * kAChunk;
constexpr int kB1 = kBRing + kBStages * kBHalf;     // float b1[256]
constexpr int kHW = kB1 + 1024;                     // float head_w[256]
constexpr int kBar = kHW + 1024;                    // mbarriers + misc
constexpr int kSmemBytes = kBar + 512;
static_assert(kSmemBytes <= 232448, "shared memory budget");
static_assert(kXStages * kBHalf <= 65536, "X stages fit the H1 region");
constexpr uint32_t kIdescF16 = idesc_bf16_f32(256, 256);
constexpr uint32_t kIdescI8 = idesc_u8s8_s32(256, 256);

struct DiscParams {
    CUtensorMap wmap;   // the weight blob as [38*256 rows x 128 B] (a box = one N-half)
    float b1[kD1];
    float hw[kD3];
    float s1;           // layer-1 scale: h1_pre = s1 * acc + b1
    const uint8_t* images;
    float* part;        // per 128-token tile: sum over its tokens of the head scores
    long long n_img;
    int h, w, px, tokens, tiles_per_img;
    long long* trace;   // debug: per-phase clock64 stamps of CTA 0 (nullptr = off)
    // Chained light batch (ds_disc_batch_complete_device, n <= kTailMax): the
    // grid is launched with programmatic stream serialization, lets its
    // dependent start at once, reads only its images and weights before
    // griddep_wait, and the last CTA to finish runs the batch tail
    // (light_batch_tail) -- so the next call's tiles fill the SMs this batch's
    // last round leaves idle.
    int chain;
    unsigned* done;     // CTAs finished (the last one resets it)
    float* conf;
    float hb;
    ds_curve* curve;
    double decay;
    const double* thr;
    int nt;
    long long index_base;
    long long* heavy;
    long long* counts;
    long long* err;
};

constexpr int kTraceTiles = 8;
constexpr int kTraceCtas = 160;   // per-CTA stamps: [globaltimer start, end, smid] x 160, then [clock64 start, end] x 160
#define DS_TRACE(role, tile, ev)                                                          \
    do {                                                                                  \
        if (P.trace && blockIdx.x == 0 && (tile) >= 0 && (tile) < kTraceTiles)            \
            P.trace[((role) * kTraceTiles + (tile)) * 16 + (ev)] = clock64();             \
    } while (0)

// GELU_tanh(s1 * acc + b) of two adjacent s32 accumulator columns with paired
// fp32 ops, in halves: with h = x / 2 = fma(acc, s1/2, b/2) (exactly half of
// fma(acc, s1, b): scaling by 2 commutes with the rounding), u = x (k + k c
// x^2) = h (2k + 8 k c h^2) -- the same roundings, every factor of 2 exact --
// and gelu = h + h tanh(u) = fma(tanh(u), h, h). Bit-identical to the form
// with x, one paired multiply (h = 0.5 x) fewer per two columns.
// (s = {s1/2, s1/2}, b = {b[c]/2, b[c+1]/2})
__device__ __forceinline__ uint32_t gelu2_bf16x2(uint32_t a0, uint32_t a1, uint64_t s, uint64_t b) {
    const uint64_t h = f2_fma(f2_pack(static_cast<float>(static_cast<int>(a0)),
                                      static_cast<float>(static_cast<int>(a1))), s, b);
    const uint64_t kk = f2_pack(2.0f * 0.7978845608028654f, 2.0f * 0.7978845608028654f);
    const uint64_t kc = f2_pack(8.0f * (0.7978845608028654f * 0.044715f),
                                8.0f * (0.7978845608028654f * 0.044715f));
    const uint64_t u = f2_mul(h, f2_fma(f2_mul(h, h), kc, kk));
    float u0, u1;
    f2_unpack(u, u0, u1);
#if DS_EXP_NO_TANH
    // TIMING EXPERIMENT ONLY (wrong results): the tanh replaced by a clamp
    const uint64_t g = f2_fma(f2_pack(fminf(u0, 1.0f), fminf(u1, 1.0f)), h, h);
#else
    const uint64_t g = f2_fma(f2_pack(tanh_approx(u0), tanh_approx(u1)), h, h);
#endif
    float g0, g1;
    f2_unpack(g, g0, g1);
    return pack_bf16x2(g0, g1);
}

// Byte offset of (row, 16-byte chunk) inside a K-major SW128 tile (128 B rows).
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t chunk) {
    return (row >> 3) * 1024u + (row & 7u) * 128u + ((chunk ^ (row & 7u)) << 4);
}

// GELU of 32 loaded accumulator columns [cbase, cbase + 32) of row `row`
// -> bf16 -> the SW128 H1 tile (4 K-chunks of 16 KB).
__device__ __forceinline__ void e1_emit32(const uint32_t (&v)[32], int cbase, uint32_t row,
                                          uint32_t h1, const float* s_b1, uint64_t s1x2) {
#pragma unroll
    for (int e = 0; e < 32; e += 8) {
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int c = cbase + e + 2 * u;
#if DS_EXP_FAST_E1
            // TIMING EXPERIMENT ONLY (wrong results): E1 without the GELU math
            (void)s1x2;
            pk[u] = v[e + 2 * u] ^ v[e + 2 * u + 1] ^ static_cast<uint32_t>(c);
#else
            pk[u] = gelu2_bf16x2(v[e + 2 * u], v[e + 2 * u + 1], s1x2,
                                 *reinterpret_cast<const uint64_t*>(s_b1 + c));
#endif
        }
        const int f = cbase + e;
        st_shared_v4(h1 + (f >> 6) * 16384u + sw128(row, (f & 63) >> 3), pk[0], pk[1], pk[2],
                     pk[3]);
    }
}

// E1 over columns [c_lo, c_lo + 32*n32) of this thread's TMEM lane (row):
// GELU(s1 * acc + b1) -> bf16 -> the SW128 H1 tile (4 K-chunks of 16 KB).
template <int kN32>
__device__ __forceinline__ void e1_columns(uint32_t tmem_lane, int c_lo, uint32_t row,
                                           uint32_t h1, const float* s_b1, uint64_t s1x2) {
    auto emit = [&](const uint32_t (&v)[32], int cbase) { e1_emit32(v, cbase, row, h1, s_b1, s1x2); };
#if DS_E1_PIPE
    // software-pipelined: block g+1's TMEM load is in flight while block g is
    // activated (two 32-register buffers, as many as the unpipelined form)
    uint32_t va[32], vb[32];
    tmem_ld_x32_async(tmem_lane + c_lo, va);
    tmem_wait_ld32(va);
#pragma unroll
    for (int g = 0; g < kN32; ++g) {
        uint32_t (&cur)[32] = (g & 1) ? vb : va;
        uint32_t (&nxt)[32] = (g & 1) ? va : vb;
        if (g + 1 < kN32) tmem_ld_x32_async(tmem_lane + c_lo + 32 * (g + 1), nxt);
        emit(cur, c_lo + 32 * g);
        if (g + 1 < kN32) tmem_wait_ld32(nxt);
    }
#elif DS_E1_SINGLE
    // one 32-column TMEM load at a time (half the registers of the pair form)
#pragma unroll 1
    for (int g = 0; g < kN32; ++g) {
        uint32_t v[32];
        const int c0 = c_lo + 32 * g;
        tmem_ld_x32_sync(tmem_lane + c0, v);
        emit(v, c0);
    }
#else
#pragma unroll 1
    for (int g = 0; g + 1 < kN32; g += 2) {
        uint32_t v0[32], v1[32];
        const int c0 = c_lo + 32 * g;
        tmem_ld2_x32_sync(tmem_lane + c0, tmem_lane + c0 + 32, v0, v1);
        emit(v0, c0);
        emit(v1, c0 + 32);
    }
    if constexpr (kN32 & 1) {
        uint32_t v[32];
        const int c0 = c_lo + 32 * (kN32 - 1);
        tmem_ld_x32_sync(tmem_lane + c0, v);
        emit(v, c0);
    }
#endif
}

constexpr int kStash = 40;
struct Bars {
    uint64_t a_full[kAStages], a_empty[kAStages], b_full[kBStages], b_empty[kBStages];
    uint64_t acc12_full, drained, h2_ready, h2_free, acc3_full, acc3_empty;
    uint64_t x_full[kXStages], r1_free, e1b_done, aw_full[2], aw_free, ax_full[2];
    uint64_t acc_read, h1c[2];   // kE1Early hand-offs
    uint32_t tmem_base;
    float warp_part[2][8];
    float stash[kStash];   // chained: this CTA's head sums until the previous call completed
};
static_assert(sizeof(Bars) <= 512, "barrier block");

// logit = (sum of the image's per-tile head sums, in tile order) / tokens + b_head
// (L2 loads: the sums may come from other CTAs of a running grid)
__device__ __forceinline__ float image_score(const float* __restrict__ part, long long i, int tpi,
                                             int tokens, float hb, int logits) {
    float s = 0.0f;
    for (int t = 0; t < tpi; ++t) s += __ldcg(part + i * tpi + t);
    const float logit = s / static_cast<float>(tokens) + hb;
    return logits ? logit : 1.0f / (1.0f + expf(-logit));
}

// One light batch's completion after the discriminator
// (Simulation::handle_batch_complete, cluster.cpp:288-307): confidences from
// the head sums (as finalize_kernel), then observe_confidence of each in batch
// order (profiles.cpp:108-120; the arithmetic of curve.cu's single-CTA replay:
// bins on threads 0-100, the total alone on thread 128, explicit _rn fp64),
// then Policy::defers (strict <) at every threshold into ordered heavy lists
// (as route.cu). Bit-identical to finalize + ds_curve_observe + ds_route.
// A confidence outside [0, 1] (a NaN from the network) is where the reference
// throws out of handle_batch_complete: the curve stops before it, only the
// queries before it are routed, and its index goes to the context's device
// error word (ds_ctx_take_error). Run by all kT threads of one CTA (kT >= 160);
// sc / sbin hold n <= kTailMax entries.
constexpr int kTailThreads = 160, kTailTotalTid = 128, kTailMax = 2048;
template <int kT>
__device__ __forceinline__ void light_batch_tail(
    const float* __restrict__ part, int n, int tpi, int tokens, float hb, float* __restrict__ conf,
    ds_curve* __restrict__ curve, double decay, const double* __restrict__ thr, int nt,
    long long index_base, long long* __restrict__ heavy, long long* __restrict__ counts,
    long long* __restrict__ err, float* sc, unsigned char* sbin, int* s_bad, int* wcnt) {
    static_assert(kT % 32 == 0 && kT > kTailTotalTid && kT > DS_CURVE_BINS, "tail block");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) *s_bad = n;
    __syncthreads();
    for (int i = tid; i < n; i += kT) {
        const float c = image_score(part, i, tpi, tokens, hb, 0);
        conf[i] = c;
        sc[i] = c;
        const double cd = static_cast<double>(c);
        if (!(cd >= 0.0) || !(cd <= 1.0)) {
            atomicMin(s_bad, i);   // the reference throws here; the curve stops before it
            sbin[i] = 255;
        } else {
            int b = static_cast<int>(floor(__dadd_rn(__dmul_rn(cd, 100.0), 1e-9)));
            b = b < 0 ? 0 : (b > DS_CURVE_BINS - 1 ? DS_CURVE_BINS - 1 : b);
            sbin[i] = static_cast<unsigned char>(b);
        }
    }
    __syncthreads();
    const int n_eff = *s_bad;
    if (tid == 0 && n_eff < n) atomicMin(err, static_cast<long long>(n_eff));
    const bool scale = decay != 1.0;
    if (tid < DS_CURVE_BINS) {
        double m = __ldcg(&curve->bin_mass[tid]);
        for (int k = 0; k < n_eff; ++k) {
            if (scale) m = __dmul_rn(m, decay);
            if (sbin[k] == tid) m = __dadd_rn(m, 1.0);
        }
        curve->bin_mass[tid] = m;
    } else if (tid == kTailTotalTid) {
        double t = __ldcg(&curve->total_mass);
        for (int k = 0; k < n_eff; ++k) t = __dadd_rn(scale ? __dmul_rn(t, decay) : t, 1.0);
        curve->total_mass = t;
    }
    for (int k = 0; k < nt; ++k) {
        const double t = thr[k];
        long long off = 0;
        long long* out = heavy + static_cast<long long>(k) * n;
        for (int base = 0; base < n_eff; base += kT) {
            const int i = base + tid;
            const bool p = i < n_eff && static_cast<double>(sc[i]) < t;
            const unsigned bal = __ballot_sync(0xffffffffu, p);
            __syncthreads();   // wcnt of the previous chunk consumed
            if (lane == 0) wcnt[warp] = __popc(bal);
            __syncthreads();
            int before = 0, all = 0;
#pragma unroll
            for (int w = 0; w < kT / 32; ++w) {
                before += w < warp ? wcnt[w] : 0;
                all += wcnt[w];
            }
            if (p) out[off + before + __popc(bal & ((1u << lane) - 1u))] = index_base + i;
            off += all;
        }
        if (tid == 0) counts[k] = off;
    }
}

__global__ void __launch_bounds__(kThreads, 1) disc_kernel(const __grid_constant__ DiscParams P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    Bars& B = *reinterpret_cast<Bars*>(smem + kBar);
    float* s_b1 = reinterpret_cast<float*>(smem + kB1);
    float* s_hw = reinterpret_cast<float*>(smem + kHW);
    const uint32_t sbase = smem_u32(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const bool leader = rank == 0;
    const long long unit = cluster_id_x(), nunits = nclusters_x();   // pair index / count

    if (sbase & 1023u) __trap();   // SW128 operand tiles need 1024-byte alignment
    if (P.chain) griddep_launch_dependents();   // the next light batch may start now
    if (P.trace && threadIdx.x == 0) {   // debug: per-CTA start time and SM id
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        P.trace[8 * kTraceTiles * 16 + 3 * blockIdx.x] = static_cast<long long>(globaltimer());
        P.trace[8 * kTraceTiles * 16 + 3 * blockIdx.x + 2] = smid;
        P.trace[8 * kTraceTiles * 16 + 3 * kTraceCtas + 2 * blockIdx.x] = clock64();
    }
    // Flat 128-token tiles f = image * tiles_per_img + tile-in-image; pair tile
    // k covers f = 2k (leader) and 2k + 1 (peer), and the pairs take pair
    // tiles round robin (k = unit, unit + nunits, ...), so a small batch still
    // spreads over every SM pair. A pair tile whose second half runs past the
    // end recomputes the last tile and writes nothing (a "ghost").
    const long long n_img = P.n_img;
    const int tpi = P.tiles_per_img;
    const long long n_flat = n_img * tpi;
    const long long n_pair_tiles = (n_flat + 1) / 2;
    const long long my_tiles = unit < n_pair_tiles ? (n_pair_tiles - 1 - unit) / nunits + 1 : 0;
    const long long img_bytes = static_cast<long long>(P.h) * P.w * 3;
    const long long row_bytes = static_cast<long long>(P.w) * 3;
    auto flat_raw = [&](long long tile) { return 2 * (unit + tile * nunits) + rank; };
    auto flat_of = [&](long long tile) {                   // this CTA's flat tile
        const long long f = flat_raw(tile);
        return f < n_flat ? f : n_flat - 1;
    };


    // ---- A-builder helpers (warps 0-3; thread tl = token of the 128-token tile)
    const int tl = threadIdx.x;
    auto token_base = [&](long long tile) -> const uint8_t* {
        const long long f = flat_of(tile);
        const long long img = f / tpi;
        const int tok = static_cast<int>(f % tpi) * kM + tl;
        const int py = tok / P.px, px = tok - py * P.px;
        return P.images + img * img_bytes + (static_cast<long long>(py) * 16) * row_bytes +
               px * 48;
    };
    auto piece = [&](const uint8_t* base, int q) -> const uint8_t* {
        return base + (q / 3) * row_bytes + (q % 3) * 16;
    };
    // The pixels of a tile are one contiguous byte range of whole patch
    // rows (or a small superset); bulk-prefetch it into L2.
    auto prefetch_tile = [&](long long tile) {
        const long long f = flat_of(tile);
        const long long img = f / tpi;
        const int tok0 = static_cast<int>(f % tpi) * kM;
        const int py0 = tok0 / P.px, py1 = (tok0 + kM - 1) / P.px;
        const uint8_t* p0 = P.images + img * img_bytes + static_cast<long long>(py0) * 16 * row_bytes;
        const long long bytes = static_cast<long long>(py1 - py0 + 1) * 16 * row_bytes;
        for (long long off = 0; off < bytes; off += 65536) {
            const uint32_t nb = static_cast<uint32_t>(bytes - off < 65536 ? bytes - off : 65536);
            bulk_prefetch_l2(p0 + off, nb);
        }
    };
    // DS_PREFETCH: 1 = one thread's bulk prefetches (TMA unit), 2 = every
    // builder thread prefetches lines through the LSU, 0 = none
    auto prefetch_lines = [&](long long tile) {
        const long long f = flat_of(tile);
        const long long img = f / tpi;
        const int tok0 = static_cast<int>(f % tpi) * kM;
        const int py0 = tok0 / P.px, py1 = (tok0 + kM - 1) / P.px;
        const uint8_t* p0 = P.images + img * img_bytes + static_cast<long long>(py0) * 16 * row_bytes;
        const long long bytes = static_cast<long long>(py1 - py0 + 1) * 16 * row_bytes;
        for (long long off = static_cast<long long>(tl) * 128; off < bytes; off += 128 * 128)
            prefetch_l2_line(p0 + off);
    };
    (void)prefetch_lines;
    uint4 buf[2][8];
    auto load_chunk = [&](const uint8_t* base, int c, uint4 (&b)[8]) {
#if DS_EXP_NO_ALOAD
        // TIMING EXPERIMENT ONLY (wrong results): no pixel loads
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t x = static_cast<uint32_t>(reinterpret_cast<uintptr_t>(base)) * 2654435761u +
                               static_cast<uint32_t>(97 * c + 7919 * j);
            b[j] = make_uint4(x, x * 3u, x * 5u, x * 7u);
        }
#else
#pragma unroll
        for (int j = 0; j < 8; ++j) b[j] = ld_global_nc_v4(piece(base, 8 * c + j));
#endif
    };
    // The A-builders' first loads (tile 0's chunks 0 and 1) go out before the
    // set-up below (barrier init, TMEM allocation, cluster barrier: ~3.4K
    // cycles), which they do not depend on -- a CTA's first GEMM1 otherwise
    // waits for cold HBM reads issued only after it (config-1 batches run 1-2
    // pair tiles per CTA). The set-up itself runs on warps 12-13, so it does
    // not wait for these loads to issue.
    if (kPrefetch == 1 && warp == 14 && lane == 0 && my_tiles > 0) prefetch_tile(0);
    const uint8_t* pbase = nullptr;
    if (warp < 4 && my_tiles > 0) {
        if (tl == 0) DS_TRACE(0, 0, 5);
        pbase = token_base(0);
        load_chunk(pbase, 0, buf[0]);
        if (tl == 0) DS_TRACE(0, 0, 7);
        load_chunk(pbase, 1, buf[1]);
        if (tl == 0) DS_TRACE(0, 0, 8);
    }

    if (threadIdx.x < kD1) {
        s_b1[threadIdx.x] = 0.5f * P.b1[threadIdx.x];   // E1 works in halves (gelu2_bf16x2)
        s_hw[threadIdx.x] = P.hw[threadIdx.x];
    }
    if (threadIdx.x == 12 * 32) {
        // The leader's barriers also count the peer's single relayed arrival;
        // weight-stage barriers get both halves' bytes through cta_group::2 TMA.
        const uint32_t peer = leader ? 1u : 0u;
        for (int s = 0; s < kAStages; ++s) {
            mbar_init(&B.a_full[s], kWarpArrive ? 4 + 4 * peer : 128 + peer);
            mbar_init(&B.a_empty[s], 1);
        }
        for (int s = 0; s < kBStages; ++s) {
            mbar_init(&B.b_full[s], 1);
            mbar_init(&B.b_empty[s], 1);
        }
        mbar_init(&B.acc12_full, 1);
        mbar_init(&B.drained, kWarpArrive ? 8 + 8 * peer : 256 + peer);
        mbar_init(&B.h2_ready, kWarpArrive ? 8 + 8 * peer : 256 + peer);
        mbar_init(&B.h2_free, 1);
        mbar_init(&B.acc3_full, 1);
        mbar_init(&B.acc3_empty, kWarpArrive ? 8 + 8 * peer : 256 + peer);
        for (int s = 0; s < kXStages; ++s) mbar_init(&B.x_full[s], 1);
        mbar_init(&B.r1_free, 1);
        mbar_init(&B.e1b_done, kWarpArrive ? 4 + 4 * peer : 128 + peer);
        for (int s = 0; s < 2; ++s) mbar_init(&B.aw_full[s], 1);
        for (int s = 0; s < 2; ++s) mbar_init(&B.ax_full[s], kWarpArrive ? 4 + 4 * peer : 128 + peer);
        mbar_init(&B.aw_free, 1);
        // all E1 threads (epilogue 256 + builders 128; the peer's two groups relay once each)
        mbar_init(&B.acc_read, kWarpArrive ? 12 + 12 * peer : 384 + 2 * peer);
        for (int s = 0; s < 2; ++s) mbar_init(&B.h1c[s], kWarpArrive ? 4 + 4 * peer : 128 + peer);
        fence_mbar_init();
        DS_TRACE(6, 7, 0);   // debug: set-up phases of CTA 0 (slots unused by 2-tile CTAs)
    }
    if (warp == 13) {
        tmem_alloc2<512>(&B.tmem_base);
        if (lane == 0) DS_TRACE(6, 7, 1);
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) DS_TRACE(6, 7, 2);
    cluster_sync();   // peer barriers initialised before any remote arrive
    tc_fence_after();
    if (threadIdx.x == 0) DS_TRACE(6, 7, 3);
    const uint32_t tmem = B.tmem_base;

    // A role's arrival on the LEADER's barrier: the leader's threads arrive
    // locally; the peer's group syncs on a named barrier and one thread
    // forwards a single cluster-scope arrive.
    auto group_signal = [&](uint64_t* bar, uint32_t bar_id, uint32_t threads, bool first) {
        if (kWarpArrive) {
            // one arrive per warp after __syncwarp (which orders the lanes'
            // writes before lane 0's release arrive); the peer's go remote
            __syncwarp();
            if (lane == 0) {
                if (leader) mbar_arrive(bar);
                else mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0));
            }
            (void)bar_id;
            (void)threads;
            (void)first;
        } else if (leader) {
            mbar_arrive(bar);
        } else {
            named_bar_sync(bar_id, threads);
            if (first) mbar_arrive_cluster(mapa_shared(smem_u32(bar), 0));
        }
    };

    if (warp < 4) {
        // ===================== A-builder (128 threads, thread = token) =========
        // Chunk c of a tile holds K bytes [128c, 128c+128) of every token: the
        // 16-byte pieces q = 8c..8c+7 of its 768-byte patch vector (piece q is
        // patch row dy = q/3, 16-byte run q%3), stored unchanged as the u8 A
        // operand (SW128 chunk j = q%8 of the token's row).
        const uint32_t tmem_lane = tmem + (static_cast<uint32_t>(32 * (warp & 3)) << 16);
        const uint64_t s1x2 = f2_pack(0.5f * P.s1, 0.5f * P.s1);   // halves, as s_b1
        // the rest of the first two tiles into L2 (kPrefetch 1: warp 14 issues
        // tile 0's and 1's bulk prefetches, which take ~1K cycles each to issue)
        if (kPrefetch == 2) {
            if (my_tiles > 0) prefetch_lines(0);
            if (my_tiles > 1) prefetch_lines(1);
        }
        if (tl == 0) DS_TRACE(0, 0, 6);
        int astage = 0;
        uint32_t aphase = 0;
        uint32_t fills[2] = {0u, 0u};   // kAX: fills of ring slot 0 / 1 so far
        for (long long tile = 0; tile < my_tiles; ++tile) {
            if (tl == 0) {
                DS_TRACE(0, tile, 0);
                if (kPrefetch == 1 && tile + 2 < my_tiles) prefetch_tile(tile + 2);
            }
            if (kPrefetch == 2 && tile + 2 < my_tiles) prefetch_lines(tile + 2);
#pragma unroll
            for (int c = 0; c < kChunksPerTile; ++c) {
                uint32_t st;
                uint64_t* full;
                if (kAX && (c == 3 || c == 5)) {
                    // W1 stage 0 / 1's slot in the H1 region: chunk 0 / 1 read it
                    // and completed (the wait of chunk 2 / 4 just before)
                    st = sbase + kR1 + (c == 3 ? 0 : kBHalf);
                    full = &B.ax_full[c == 3 ? 0 : 1];
                } else if (kAX) {
                    const int sl = (c == 1 || c == 4) ? 1 : 0;
                    mbar_wait(&B.a_empty[sl], (fills[sl] & 1u) ^ 1u);
                    ++fills[sl];
                    // the ring slots carried GEMM2_0's first weight stages after GEMM1
                    if (kAWStages && c == 0 && tile > 0)
                        mbar_wait(&B.aw_free, static_cast<uint32_t>((tile - 1) & 1));
                    st = sbase + kARing + sl * kAChunk;
                    full = &B.a_full[sl];
                } else {
                    mbar_wait(&B.a_empty[astage], aphase ^ 1);
                    // the A slots carried GEMM2_0's first weight stages after GEMM1
                    if (kAWStages && c == 0 && tile > 0)
                        mbar_wait(&B.aw_free, static_cast<uint32_t>((tile - 1) & 1));
                    st = sbase + kARing + astage * kAChunk;
                    full = &B.a_full[astage];
                    if (++astage == kAStages) { astage = 0; aphase ^= 1; }
                }
                if (tl == 0) DS_TRACE(3, tile, c);
#if DS_A_RECOMPUTE
                {
                    // the row's SW128 base and swizzle recomputed per chunk
                    // (an opaque copy keeps the compiler from hoisting the eight
                    // addresses out of the loop, where they were spilled)
                    uint32_t r = static_cast<uint32_t>(tl);
                    asm volatile("" : "+r"(r));
                    const uint32_t rb = st + (r >> 3) * 1024u + (r & 7u) * 128u, r7 = r & 7u;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        st_shared_v4(rb + ((static_cast<uint32_t>(j) ^ r7) << 4), buf[c & 1][j].x,
                                     buf[c & 1][j].y, buf[c & 1][j].z, buf[c & 1][j].w);
                }
#else
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    st_shared_v4(st + sw128(tl, j), buf[c & 1][j].x, buf[c & 1][j].y, buf[c & 1][j].z,
                                 buf[c & 1][j].w);
#endif
                fence_proxy_async_smem();
                group_signal(full, 2, 128, tl == 0);
                if (tl == 0) DS_TRACE(4, tile, c);
#if DS_A_REORDER
                // chunks 2 and 3 stored back to back (X0 is free as soon as
                // slot 0 is), then the loads of chunks 4 and 5
                if (c < 2) load_chunk(pbase, c + 2, buf[c & 1]);
                if (c == 3) {
                    load_chunk(pbase, 4, buf[0]);
                    load_chunk(pbase, 5, buf[1]);
                }
#else
                if (c + 2 < kChunksPerTile) load_chunk(pbase, c + 2, buf[c & 1]);
#endif
            }
            if (tl == 0) DS_TRACE(0, tile, 1);
            // E1 help: columns [kE1Split, 256) once GEMM1 of this tile landed. The
            // acc12_full phase of E1(tile) has parity tile & 1; the barrier cannot
            // be behind it (the A slots just freed were released after GEMM2_3 of
            // the previous tile) nor past it (GEMM2_0 waits for e1b_done).
            if constexpr (kE1Early) {
                // H1 K-chunk 3: load, tell GEMM2_0 the accumulator reads are
                // done, then activate and store
                mbar_wait(&B.acc12_full, static_cast<uint32_t>(tile & 1));
                tc_fence_after();
                uint32_t v0[32], v1[32];
                tmem_ld2_x32_sync(tmem_lane + 192, tmem_lane + 224, v0, v1);
                tc_fence_before();
                group_signal(&B.acc_read, 2, 128, tl == 0);
                e1_emit32(v0, 192, tl, sbase + kR1, s_b1, s1x2);
                e1_emit32(v1, 224, tl, sbase + kR1, s_b1, s1x2);
                fence_proxy_async_smem();
            } else if constexpr (kE1Split < 256) {
                mbar_wait(&B.acc12_full, static_cast<uint32_t>(tile & 1));
                tc_fence_after();
                e1_columns<(256 - kE1Split) / 32>(tmem_lane, kE1Split, tl, sbase + kR1, s_b1, s1x2);
                fence_proxy_async_smem();
                tc_fence_before();
            }
            group_signal(&B.e1b_done, 2, 128, tl == 0);
            if (tile + 1 < my_tiles) {
                pbase = token_base(tile + 1);
                load_chunk(pbase, 0, buf[0]);
                load_chunk(pbase, 1, buf[1]);
            }
        }
    } else if (warp < 12) {
        // ===================== epilogue (256 threads) =======================
        const int ew = warp - 4;
        const int q = warp & 3;            // TMEM lane quadrant this warp may access
        const int half = ew >> 2;          // column half [128*half, 128*half+128)
        const uint32_t row = 32 * q + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(32 * q) << 16;
        const bool first = ew == 0 && lane == 0;
        const uint64_t s1x2 = f2_pack(0.5f * P.s1, 0.5f * P.s1);   // halves, as s_b1
        uint32_t p12 = 0, p3 = 0, pfree = 0;

        // E3: ReLU(acc3) . w_head over this thread's 128 columns -> per-image sum
        auto e3 = [&](long long tile) {
            mbar_wait(&B.acc3_full, p3);
            p3 ^= 1;
            tc_fence_after();
            DS_TRACE(1, tile, 10);
            float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 1
            for (int cb = 0; cb < 4; cb += 2) {
                uint32_t v0[32], v1[32];
                const int c0 = 128 * half + 32 * cb;
                tmem_ld2_x32_sync(tmem + lane_addr + 256 + c0, tmem + lane_addr + 256 + c0 + 32,
                                  v0, v1);
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    part[e & 3] += fmaxf(__uint_as_float(v0[e]), 0.0f) * s_hw[c0 + e];
#pragma unroll
                for (int e = 0; e < 32; ++e)
                    part[e & 3] += fmaxf(__uint_as_float(v1[e]), 0.0f) * s_hw[c0 + 32 + e];
            }
            tc_fence_before();
            group_signal(&B.acc3_empty, 3, 256, first);
            DS_TRACE(1, tile, 11);
            float p = (part[0] + part[1]) + (part[2] + part[3]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) p += __shfl_xor_sync(0xffffffffu, p, o);
            const int b = static_cast<int>(tile & 1);
            if (lane == 0) B.warp_part[b][ew] = p;
            named_bar_sync(1, 256);
            if (first) {
                float s = 0.0f;
#pragma unroll
                for (int w = 0; w < 8; ++w) s += B.warp_part[b][w];
                const long long f = flat_raw(tile);
                if (f < n_flat) {                   // ghost tiles write nothing
                    // chained: the part buffer is the previous call's until that
                    // completed; the first kStash sums wait in shared memory
                    if (P.chain && tile < kStash) {
                        B.stash[tile] = s;
                    } else {
                        if (P.chain) griddep_wait();
                        P.part[f] = s;
                        if (P.chain) __threadfence();
                    }
                }
            }
        };

        for (long long tile = 0; tile < my_tiles; ++tile) {
            // ---- E1: s1 * acc (s32) + b1 -> GELU -> bf16 -> H1 (R1), columns
            // [96*half, 96*half + 96); the A-builders take [192, 256) -------------
            mbar_wait(&B.acc12_full, p12);
            p12 ^= 1;
            tc_fence_after();
            DS_TRACE(1, tile, 0);
            if constexpr (kE1Early) {
                // H1 K-chunk `half` (columns [64 half, 64 half + 64)) first ...
                {
                    uint32_t v0[32], v1[32];
                    const int c0 = 64 * half;
                    tmem_ld2_x32_sync(tmem + lane_addr + c0, tmem + lane_addr + c0 + 32, v0, v1);
                    e1_emit32(v0, c0, row, sbase + kR1, s_b1, s1x2);
                    e1_emit32(v1, c0 + 32, row, sbase + kR1, s_b1, s1x2);
                }
                fence_proxy_async_smem();
                group_signal(&B.h1c[half], 4 + half, 128, (ew & 3) == 0 && lane == 0);
                // ... then this half's 32 columns of K-chunk 2: after their load
                // the accumulator is free for GEMM2_0
                uint32_t v[32];
                tmem_ld_x32_sync(tmem + lane_addr + 128 + 32 * half, v);
                tc_fence_before();
                group_signal(&B.acc_read, 3, 256, first);
                e1_emit32(v, 128 + 32 * half, row, sbase + kR1, s_b1, s1x2);
                fence_proxy_async_smem();
                group_signal(&B.drained, 3, 256, first);   // K-chunk 2 stored
            } else {
                e1_columns<kE1Split / 64>(tmem + lane_addr, (kE1Split / 2) * half, row, sbase + kR1,
                                          s_b1, s1x2);
                fence_proxy_async_smem();
                tc_fence_before();
                group_signal(&B.drained, 3, 256, first);
            }
            DS_TRACE(1, tile, 1);

            // ---- E2_j: acc[0,256) -> ReLU -> bf16 (registers) -> H2 (R2) --------
            for (int j = 0; j < 4; ++j) {
                mbar_wait(&B.acc12_full, p12);
                p12 ^= 1;
                tc_fence_after();
                DS_TRACE(1, tile, 2 + 2 * j);
                uint32_t pk[64];
#pragma unroll
                for (int cb = 0; cb < 4; ++cb) {
                    uint32_t v[32];
                    const int c0 = 128 * half + 32 * cb;
                    tmem_ld_x32_sync(tmem + lane_addr + c0, v);
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        pk[16 * cb + e] = pack_relu_bf16x2(__uint_as_float(v[2 * e]),
                                                           __uint_as_float(v[2 * e + 1]));
                }
                tc_fence_before();
                group_signal(&B.drained, 3, 256, first);   // MMA may overwrite acc[0,256)
                if (tile > 0 || j > 0) {            // GEMM3 reading the previous H2 chunk done
                    mbar_wait(&B.h2_free, pfree);
                    pfree ^= 1;
                }
#pragma unroll
                for (int cb = 0; cb < 4; ++cb) {
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int f = 128 * half + 32 * cb + 8 * e;
                        st_shared_v4(sbase + kR2 + (f >> 6) * kAChunk + sw128(row, (f & 63) >> 3),
                                     pk[16 * cb + 4 * e], pk[16 * cb + 4 * e + 1],
                                     pk[16 * cb + 4 * e + 2], pk[16 * cb + 4 * e + 3]);
                    }
                }
                fence_proxy_async_smem();
                group_signal(&B.h2_ready, 3, 256, first);
                DS_TRACE(1, tile, 3 + 2 * j);
                // ---- E3 of the previous tile: after E2_0, so GEMM2_1 is not held
                // behind it; it must finish before GEMM3_0 (after GEMM2_1)
                if (j == 0 && tile > 0) e3(tile - 1);
            }
        }
        if (my_tiles > 0) e3(my_tiles - 1);
    } else if (warp == 12) {
        // ===================== weight producer (both CTAs) ====================
        if (lane == 0) {
            const uint64_t policy = policy_evict_last();
            prefetch_tmap(&P.wmap);
            int bs = 0;
            uint32_t bp = 0;
            long long ptile = 0;   // trace only
            auto put = [&](int first, int count) {
                for (int t = first; t < first + count; ++t) {
                    mbar_wait(&B.b_empty[bs], bp ^ 1);
                    if (t < 16) DS_TRACE(6, ptile, t);
                    // both CTAs load their N-half; completion lands on the leader's
                    // barrier, which expects the whole stage
#if DS_EXP_NO_WSTREAM
                    // ENERGY EXPERIMENT ONLY (wrong results): after the first tile the
                    // ring keeps its stale weights instead of re-streaming them from L2
                    if (ptile > 0) {
                        if (leader) mbar_arrive(&B.b_full[bs]);
                        if (++bs == kBStages) { bs = 0; bp ^= 1; }
                        continue;
                    }
#endif
                    if (leader) mbar_arrive_expect_tx(&B.b_full[bs], kBStage);
                    tma_2d_pair(sbase + kBRing + bs * kBHalf, &P.wmap, 0,
                                t * 256 + static_cast<int>(rank) * 128,
                                mapa_shared(smem_u32(&B.b_full[bs]), 0), policy);
                    if (++bs == kBStages) { bs = 0; bp ^= 1; }
                }
            };
            const int W1 = 0, W2 = kW1Stages, W3 = kW1Stages + 4 * kWChunkStages;
            for (long long tile = 0; tile < my_tiles; ++tile) {
                ptile = tile;
                if (kG33Il > 0 && tile > 0) {
                    // the MMA issuer's order: W1 stages 4-5 after GEMM1 chunks 4-5,
                    // GEMM3_3(tile-1) K-chunk q after GEMM1 chunk kG33Il + q
                    for (int c = 0; c < kW1Stages; ++c) {
                        if (c >= kXStages) put(W1 + c, 1);
                        const int q = c - kG33Il;
                        if (q >= 0 && q < kWChunkStages) put(W3 + 3 * kWChunkStages + q, 1);
                    }
                } else {
                    put(W1 + kXStages, kW1Stages - kXStages);
                    if (tile > 0) put(W3 + 3 * kWChunkStages, kWChunkStages);
                }
                put(W2 + kAWStages, kWChunkStages - kAWStages);
                for (int j = 1; j < 4; ++j) {
                    put(W2 + j * kWChunkStages, kWChunkStages);
                    put(W3 + (j - 1) * kWChunkStages, kWChunkStages);
                }
            }
            if (my_tiles > 0) put(W3 + 3 * kWChunkStages, kWChunkStages);
        }
    } else if (warp == 14) {
        // ===================== W1 stages 0-3 into the H1 region ================
        // (and, kPrefetch 1, the bulk L2 prefetch of the image tile 1 at the
        // start: the A-builders are storing tile 0 then; later tiles are
        // prefetched by a builder thread two tiles ahead -- issued here, during
        // GEMM1, they cost ~0.6K cycles per pair tile)
        if (lane == 0) {
            const uint64_t policy = policy_evict_last();
            if (kPrefetch == 1 && my_tiles > 1) prefetch_tile(1);
            for (long long tile = 0; tile < my_tiles; ++tile) {
                if (tile > 0) mbar_wait(&B.r1_free, static_cast<uint32_t>((tile - 1) & 1));
                for (int k = 0; k < kXStages; ++k) {
                    if (leader) mbar_arrive_expect_tx(&B.x_full[k], kBStage);
                    tma_2d_pair(sbase + kR1 + k * kBHalf, &P.wmap, 0,
                                k * 256 + static_cast<int>(rank) * 128,
                                mapa_shared(smem_u32(&B.x_full[k]), 0), policy);
                }
                if (kAWStages) {
                    // GEMM1 of this tile complete (acc12_full phase 5*tile; the
                    // barrier cannot be past it: GEMM2_0 needs these stages):
                    // the A slots are free until aw_free
                    mbar_wait(&B.acc12_full, static_cast<uint32_t>(tile & 1));
                    for (int k = 0; k < kAWStages; ++k) {
                        if (leader) mbar_arrive_expect_tx(&B.aw_full[k], kBStage);
                        tma_2d_pair(sbase + kARing + k * kAChunk, &P.wmap, 0,
                                    (kW1Stages + k) * 256 + static_cast<int>(rank) * 128,
                                    mapa_shared(smem_u32(&B.aw_full[k]), 0), policy);
                    }
                }
            }
        }
    } else {
        // ===================== MMA issuer (leader warp 13, one thread) ========
        if (lane == 0 && leader) {
            int as = 0, bs = 0;
            uint32_t ap = 0, bp = 0, pdr = 0, prd = 0, pe3 = 0;
            uint32_t used[2] = {0u, 0u};   // kAX: fills of ring slot 0 / 1 consumed
            long long trace_tile = 0;   // trace only
            int trace_stage = 0;
            const uint32_t acc12 = tmem, acc3 = tmem + 256;
            // next ring stage: wait until both halves landed, return its descriptor
            auto next_b = [&]() -> uint64_t {
                mbar_wait(&B.b_full[bs], bp);
                tc_fence_after();
                if (trace_stage < 16) DS_TRACE(7, trace_tile, trace_stage);
                ++trace_stage;
                return desc_k_sw128(sbase + kBRing + bs * kBHalf);
            };
            auto release_b = [&]() {
                umma_commit_pair(&B.b_empty[bs], 0x3);
                if (++bs == kBStages) { bs = 0; bp ^= 1; }
            };
            // bf16 GEMM, K = 64 x nk from an SW128 A region (nk chunks of 16 KB),
            // one weight stage (K = 64) per chunk
            auto gemm = [&](uint32_t a_region, int nk, uint32_t acc, bool acc_in) {
                for (int kc = 0; kc < nk; ++kc) {
                    const uint64_t ad = desc_k_sw128(a_region + kc * kAChunk);
                    const uint64_t bd = next_b();
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_bf16_pair(acc, ad + 2 * k, bd + 2 * k, kIdescF16,
                                       (acc_in || kc > 0 || k > 0) ? 1u : 0u);
                    release_b();
                }
            };
            auto wait_bar = [&](uint64_t* bar, uint32_t& ph) {
                mbar_wait(bar, ph);
                ph ^= 1;
                tc_fence_after();
            };
            for (long long tile = 0; tile < my_tiles; ++tile) {
                DS_TRACE(2, tile, 0);
                trace_tile = tile;
                trace_stage = 0;
                // G1: 6 u8 A chunks (K = 128 bytes) x 6 int8 weight stages; stages
                // 0-3 come from the H1 region (x_full), 4-5 from the ring
                for (int c = 0; c < kChunksPerTile; ++c) {
                    uint32_t a_addr;
                    if (kAX && (c == 3 || c == 5)) {
                        mbar_wait(&B.ax_full[c == 3 ? 0 : 1], static_cast<uint32_t>(tile & 1));
                        a_addr = sbase + kR1 + (c == 3 ? 0 : kBHalf);
                    } else if (kAX) {
                        const int sl = (c == 1 || c == 4) ? 1 : 0;
                        mbar_wait(&B.a_full[sl], used[sl] & 1u);
                        ++used[sl];
                        a_addr = sbase + kARing + sl * kAChunk;
                    } else {
                        mbar_wait(&B.a_full[as], ap);
                        a_addr = sbase + kARing + as * kAChunk;
                    }
                    tc_fence_after();
                    DS_TRACE(5, tile, c);
                    const uint64_t ad = desc_k_sw128(a_addr);
                    uint64_t bd;
                    if (c < kXStages) {
                        mbar_wait(&B.x_full[c], static_cast<uint32_t>(tile & 1));
                        tc_fence_after();
                        bd = desc_k_sw128(sbase + kR1 + c * kBHalf);
                    } else {
                        bd = next_b();
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_i8_pair(acc12, ad + 2 * k, bd + 2 * k, kIdescI8,
                                     (c > 0 || k > 0) ? 1u : 0u);
                    if (c >= kXStages) release_b();
                    if (kAX) {
                        if (c == 0 || c == 2) umma_commit_pair(&B.a_empty[0], 0x3);
                        if (c == 1 || c == 4) umma_commit_pair(&B.a_empty[1], 0x3);
                    } else {
                        umma_commit_pair(&B.a_empty[as], 0x3);
                        if (++as == kAStages) { as = 0; ap ^= 1; }
                    }
                    if (c == kChunksPerTile - 1) umma_commit_pair(&B.acc12_full, 0x3);
                    // GEMM3_3 of the previous tile between GEMM1 chunks: tensor work
                    // while the next A chunk makes its round trip
                    const int q = c - kG33Il;
                    if (kG33Il > 0 && tile > 0 && q >= 0 && q < kWChunkStages) {
                        if (q == 0) wait_bar(&B.h2_ready, prd);
                        const uint64_t ad3 = desc_k_sw128(sbase + kR2 + q * kAChunk);
                        const uint64_t bd3 = next_b();
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            umma_bf16_pair(acc3, ad3 + 2 * k, bd3 + 2 * k, kIdescF16, 1u);
                        release_b();
                        if (q == kWChunkStages - 1) {
                            umma_commit_pair(&B.h2_free, 0x3);
                            umma_commit_pair(&B.acc3_full, 0x3);
                        }
                    }
                }
                DS_TRACE(2, tile, 1);
                if (kG33Il == 0 && tile > 0) {       // G3_3 of the previous tile
                    wait_bar(&B.h2_ready, prd);
                    gemm(sbase + kR2, 4, acc3, true);
                    umma_commit_pair(&B.h2_free, 0x3);
                    umma_commit_pair(&B.acc3_full, 0x3);
                }
                DS_TRACE(2, tile, 2);
                if constexpr (kE1Early) {
                    // E1's accumulator reads done and H1 K-chunk 0 stored; chunks
                    // 1-3 are awaited one by one below
                    mbar_wait(&B.acc_read, static_cast<uint32_t>(tile & 1));
                    mbar_wait(&B.h1c[0], static_cast<uint32_t>(tile & 1));
                } else {
                    wait_bar(&B.drained, pdr);           // E1: acc drained, H1 stored
                    mbar_wait(&B.e1b_done, static_cast<uint32_t>(tile & 1));   // the builders' E1 columns
                }
                tc_fence_after();
                DS_TRACE(2, tile, 3);
                // G2_0: its first kAWStages weight stages sit in the A slots
                for (int kc = 0; kc < 4; ++kc) {
                    if constexpr (kE1Early) {
                        if (kc == 1) mbar_wait(&B.h1c[1], static_cast<uint32_t>(tile & 1));
                        if (kc == 2) mbar_wait(&B.drained, pdr);   // epilogue's K-chunk 2
                        if (kc == 3) mbar_wait(&B.e1b_done, static_cast<uint32_t>(tile & 1));
                        if (kc == 2) pdr ^= 1;
                        if (kc > 0) tc_fence_after();
                    }
                    const uint64_t ad = desc_k_sw128(sbase + kR1 + kc * kAChunk);
                    uint64_t bd;
                    if (kc < kAWStages) {
                        mbar_wait(&B.aw_full[kc], static_cast<uint32_t>(tile & 1));
                        tc_fence_after();
                        bd = desc_k_sw128(sbase + kARing + kc * kAChunk);
                    } else {
                        bd = next_b();
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_bf16_pair(acc12, ad + 2 * k, bd + 2 * k, kIdescF16,
                                       (kc > 0 || k > 0) ? 1u : 0u);
                    if (kc >= kAWStages) release_b();
                }
                if (kAWStages) umma_commit_pair(&B.aw_free, 0x3);
                umma_commit_pair(&B.acc12_full, 0x3);
                for (int j = 1; j < 4; ++j) {
                    wait_bar(&B.drained, pdr);       // E2_{j-1} has the values in registers
                    DS_TRACE(2, tile, 2 + 2 * j);
                    gemm(sbase + kR1, 4, acc12, false);       // G2_j
                    umma_commit_pair(&B.acc12_full, 0x3);
                    if (j == 3) umma_commit_pair(&B.r1_free, 0x3);   // H1 read for the last time
                    wait_bar(&B.h2_ready, prd);      // H2_{j-1} stored
                    DS_TRACE(2, tile, 3 + 2 * j);
                    if (j == 1) {                    // acc3 drained by E3 of the previous tile
                        mbar_wait(&B.acc3_empty, pe3 ^ 1);
                        pe3 ^= 1;
                        tc_fence_after();
                    }
                    gemm(sbase + kR2, 4, acc3, j > 1);        // G3_{j-1}
                    umma_commit_pair(&B.h2_free, 0x3);
                }
                wait_bar(&B.drained, pdr);           // E2_3 drained: acc[0,256) free
                DS_TRACE(2, tile, 10);
            }
            if (my_tiles > 0) {
                wait_bar(&B.h2_ready, prd);
                gemm(sbase + kR2, 4, acc3, true);    // G3_3 of the last tile
                umma_commit_pair(&B.h2_free, 0x3);
                umma_commit_pair(&B.acc3_full, 0x3);
            }
            if (P.trace && blockIdx.x == 0)   // debug: the MMA issuer is done
                P.trace[(0 * kTraceTiles + 7) * 16 + 0] = static_cast<long long>(globaltimer());
        }
    }
    __syncwarp();   // single-lane roles (warps 12-14) rejoin their warps
    tc_fence_before();
    __syncthreads();
    cluster_sync();     // both CTAs done with TMEM / remote barriers
    if (P.trace && threadIdx.x == 0 && blockIdx.x == 0)
        P.trace[(0 * kTraceTiles + 7) * 16 + 1] = static_cast<long long>(globaltimer());
    if (warp == 13) {
        tc_fence_after();
        tmem_dealloc2<512>(tmem);
        // debug: this CTA's end (a stamp after the CTA barrier by thread 0 is
        // not one: bar.sync counts a warp as arrived when any of its lanes
        // arrives, and lanes 1-31 of the MMA warp get there while lane 0 is
        // still issuing the last tile)
        if (P.trace && lane == 0) {
            P.trace[8 * kTraceTiles * 16 + 3 * blockIdx.x + 1] = static_cast<long long>(globaltimer());
            // with the start pair: this SM's mean clock over the launch
            P.trace[8 * kTraceTiles * 16 + 3 * kTraceCtas + 2 * blockIdx.x + 1] = clock64();
        }
    }
    if (P.chain) {
        // The last CTA to finish runs the batch tail (its head sums are all
        // written: every writer fenced before the barrier above). The H1
        // region is free: every MMA reading it completed before E3's waits.
        float* sc = reinterpret_cast<float*>(smem + kR1);
        unsigned char* sbin = smem + kR1 + 4 * kTailMax;
        int* s_bad = reinterpret_cast<int*>(smem + kR1 + 5 * kTailMax);
        int* wcnt = s_bad + 1;
        volatile int* s_last = s_bad + 1 + kThreads / 32;
        if (threadIdx.x == 0) {
            griddep_wait();   // the previous call completed: buffer free, counter reset, curve final
            for (long long t = 0; t < my_tiles && t < kStash; ++t) {
                const long long f = flat_raw(t);
                if (f < n_flat) P.part[f] = B.stash[t];
            }
            __threadfence();
            *s_last = atomicAdd(P.done, 1u) == gridDim.x - 1;
        }
        __syncthreads();
        if (*s_last) {
            griddep_wait();
            __threadfence();
            if (threadIdx.x == 0) *P.done = 0u;   // later grids count only after this one completed
            light_batch_tail<kThreads>(P.part, static_cast<int>(n_img), tpi, P.tokens, P.hb, P.conf,
                                       P.curve, P.decay, P.thr, P.nt, P.index_base, P.heavy,
                                       P.counts, P.err, sc, sbin, s_bad, wcnt);
        }
    }
}

__global__ void finalize_kernel(const float* __restrict__ part, long long n, int tpi, int tokens,
                                float hb, int logits, float* __restrict__ out) {
    const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= n) return;
    out[i] = image_score(part, i, tpi, tokens, hb, logits);
}

// One light batch's completion after the discriminator, in one launch (the
// unchained form of the chained disc_kernel's tail; light_batch_tail).
__global__ void __launch_bounds__(kTailThreads)
batch_tail_kernel(const float* __restrict__ part, int n, int tpi, int tokens, float hb,
                  float* __restrict__ conf, ds_curve* __restrict__ curve, double decay,
                  const double* __restrict__ thr, int nt, long long index_base,
                  long long* __restrict__ heavy, long long* __restrict__ counts,
                  long long* __restrict__ err) {
    __shared__ float sc[kTailMax];
    __shared__ __align__(16) unsigned char sbin[kTailMax];
    __shared__ int s_bad, wcnt[kTailThreads / 32];
    light_batch_tail<kTailThreads>(part, n, tpi, tokens, hb, conf, curve, decay, thr, nt,
                                   index_base, heavy, counts, err, sc, sbin, &s_bad, wcnt);
}

// A backlog of light batches after one discriminator launch and one curve
// replay over all their confidences (ds_disc_batches_complete_device): batch
// b = queries [off[b], off[b+1]) routed at ITS threshold thr[b]
// (Policy::defers, strict <) into heavy[off[b] ..], counts[b] -- one CTA per
// batch. Queries at or after the first invalid confidence (*bad, from the
// replay) are not routed, as the reference's throw out of
// handle_batch_complete would leave them.
constexpr int kSegThreads = 128;
__global__ void __launch_bounds__(kSegThreads)
segmented_route_kernel(const float* __restrict__ conf, const long long* __restrict__ off,
                       const double* __restrict__ thr, const int* __restrict__ bad,
                       long long index_base, long long* __restrict__ heavy,
                       long long* __restrict__ counts) {
    __shared__ int wcnt[kSegThreads / 32];
    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long lo = off[b], first_bad = static_cast<long long>(*bad);
    long long hi = off[b + 1];
    if (hi > first_bad) hi = first_bad > lo ? first_bad : lo;
    const double t = thr[b];
    long long pos = 0;
    for (long long base = lo; base < hi; base += kSegThreads) {
        const long long i = base + tid;
        const bool p = i < hi && static_cast<double>(conf[i]) < t;
        const unsigned bal = __ballot_sync(0xffffffffu, p);
        __syncthreads();   // wcnt of the previous chunk consumed
        if (lane == 0) wcnt[warp] = __popc(bal);
        __syncthreads();
        int before = 0, all = 0;
#pragma unroll
        for (int w = 0; w < kSegThreads / 32; ++w) {
            before += w < warp ? wcnt[w] : 0;
            all += wcnt[w];
        }
        if (p) heavy[lo + pos + before + __popc(bal & ((1u << lane) - 1u))] = index_base + i;
        pos += all;
    }
    if (tid == 0) counts[b] = pos;
}

// ---- deterministic weights ---------------------------------------------------------

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ULL;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

// Uniform in [-1, 1) from (stream, index).
__host__ __device__ __forceinline__ float unif_pm1(uint64_t stream, uint64_t idx) {
    const uint64_t r = splitmix64(stream ^ splitmix64(idx));
    return static_cast<float>(static_cast<double>(r >> 11) * 0x1.0p-52 - 1.0);
}

__device__ __forceinline__ uint16_t f2bf_bits(float f) {
    return __bfloat16_as_ushort(__float2bfloat16_rn(f));
}

// layer-1 scale: the bf16 network's U(-a, a) weights with a = sqrt(3)/(64 sqrt(768))
// (the 1/64 of the input normalisation folded in) quantised to 127 steps
__host__ __device__ __forceinline__ float layer1_scale() {
    return (1.7320508f / (64.0f * 27.712812921102035f)) / 127.0f;   // sqrt(768) as f32
}

// Logical weights (row = input feature): Q1 int8, W2/W3 bf16 bit patterns,
// including the constant-feature bias rows (see the header comment).
__global__ void gen_weights_kernel(uint64_t seed, int8_t* q1, uint16_t* w2, uint16_t* w3) {
    const float s2 = 1.7320508f * sqrtf(2.0f / 256.0f);
    const float s3 = 1.7320508f * sqrtf(2.0f / 1024.0f);
    const int n1 = kD0 * kD1, n2 = kD1 * kD2, n3 = kD2 * kD3;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n1 + n2 + n3;
         i += gridDim.x * blockDim.x) {
        if (i < n1) {
            const int n = i % kD1;   // round-half-even of 127 u, |q| <= 127
            q1[i] = n == kD1 - 1 ? 0 : static_cast<int8_t>(__float2int_rn(__fmul_rn(127.0f, unif_pm1(seed ^ 0x1111, i))));
        } else if (i < n1 + n2) {
            const int e = i - n1, k = e / kD2, n = e % kD2;
            float v;
            if (n == kD2 - 1) v = k == kD1 - 1 ? 1.0f : 0.0f;          // h2[:,1023] = 16
            else if (k == kD1 - 1) v = __fmul_rn(0.05f, unif_pm1(seed ^ 0x5555, n)) / kConst;  // b2/16
            else v = __fmul_rn(s2, unif_pm1(seed ^ 0x2222, e));
            w2[e] = f2bf_bits(v);
        } else {
            const int e = i - n1 - n2, k = e / kD3, n = e % kD3;
            const float v = k == kD2 - 1 ? __fmul_rn(0.05f, unif_pm1(seed ^ 0x6666, n)) / kConst  // b3/16
                                         : __fmul_rn(s3, unif_pm1(seed ^ 0x3333, e));
            w3[e] = f2bf_bits(v);
        }
    }
}

// Pre-swizzled blob of 32 KB stages (256 rows = N x 128 bytes of K, SW128;
// rows 0-127 and 128-255 are the two contiguous 16 KB N-halves):
//   stages  0..5  : Q1 (int8), K-range [128s, 128s+128)
//   stages  6..21 : W2 N-chunk j (rows 256j..), K-range [64k, 64k+64) (bf16), j-major
//   stages 22..37 : W3 K-chunk j (input rows 256j + 64k ..), all 256 outputs
__global__ void tile_weights_kernel(const int8_t* q1, const uint16_t* w2, const uint16_t* w3,
                                    uint8_t* blob) {
    const int t = blockIdx.x;
    uint8_t* out = blob + static_cast<size_t>(t) * kBStage;
    for (int e = threadIdx.x; e < 256 * 128; e += blockDim.x) {   // (row n, K byte kb)
        const int n = e / 128, kb = e % 128;
        const uint32_t byte = (n >> 3) * 1024u + (n & 7) * 128u +
                              ((((kb >> 4) ^ (n & 7))) << 4) + (kb & 15);
        if (t < kW1Stages) {
            out[byte] = static_cast<uint8_t>(q1[(128 * t + kb) * kD1 + n]);
        } else if (!(kb & 1)) {
            const int kl = kb >> 1;
            uint16_t v;
            if (t < kW1Stages + 4 * kWChunkStages) {
                const int u = t - kW1Stages, j = u / kWChunkStages, k = u % kWChunkStages;
                v = w2[(64 * k + kl) * kD2 + 256 * j + n];
            } else {
                const int u = t - kW1Stages - 4 * kWChunkStages, j = u / kWChunkStages,
                          k = u % kWChunkStages;
                v = w3[(256 * j + 64 * k + kl) * kD3 + n];
            }
            *reinterpret_cast<uint16_t*>(out + byte) = v;
        }
    }
}

// b1[n] = -128 * s1 * sum_k Q1[k][n] + small bias (folds (x - 128)/64 into
// layer 1; the 1/64 is in s1); b1[255] = 16 makes h1[:,255] the constant feature.
__global__ void fold_bias_kernel(const int8_t* q1, uint64_t seed, float* b1) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= kD1) return;
    if (n == kD1 - 1) {
        b1[n] = kConst;
        return;
    }
    int s = 0;   // exact; explicit _rn below: restated in oracle/disc_oracle.py
    for (int k = 0; k < kD0; ++k) s += q1[k * kD1 + n];
    b1[n] = __fadd_rn(__fmul_rn(-128.0f * layer1_scale(), static_cast<float>(s)),
                      __fmul_rn(0.05f, unif_pm1(seed ^ 0x4444, n)));
}

} // namespace

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static ds_status make_weight_tmap(const void* blob, CUtensorMap* out) {
    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    DS_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess)
        return dsi::fail(DS_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    // [rows = 38 stages x 256][128 bytes] row-major; a box of 128 rows copies
    // one pre-swizzled N-half of a stage (16 KB, contiguous) byte for byte.
    const cuuint64_t dims[2] = {128, static_cast<cuuint64_t>(kBlobStages) * 256};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {128, 128};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = reinterpret_cast<EncodeFn>(fn)(
        out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(blob), dims, strides, box, estr,
        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS)
        return dsi::fail(DS_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(r));
    return DS_OK;
}

struct ds_disc {
    ds_ctx* ctx = nullptr;
    uint64_t seed = 0;
    int8_t* d_q1 = nullptr;    // Q1 logical [768][256]
    uint16_t* d_w = nullptr;   // w2 | w3 logical
    uint8_t* d_blob = nullptr;
    float* d_b1 = nullptr;
    DiscParams params{};       // b1 + head + s1 (device-independent part)
    float hb = 0.0f;           // head bias
    int sms = 0;               // SM count of ctx->device (set once, with the smem attribute)
    // head-sum buffer + done counter of chained light batches, one per stream
    // (a chained call's buffer belongs to the previous call on the stream
    // until that one completes, see DiscParams::chain)
    struct ChainBuf {
        cudaStream_t st;
        float* part;
        unsigned* done;
    };
    ChainBuf chain[8] = {};
    int n_chain = 0;
    int chain_off = -1;        // DS_DISC_NO_CHAIN=1: light batches as two launches (A/B runs)
    int min_per_pair = 1;      // DS_DISC_MIN_PAIR_TILES (experiments): fewer, longer-lived pairs
};

namespace {

constexpr long long kChainPart = 1 << 20;   // head sums of a chained batch (n * tiles per image)

// The stream's chain buffer, allocated on first use outside stream capture
// (nullptr: use the unchained launches).
ds_disc::ChainBuf* chain_buf(ds_disc* d, cudaStream_t st) {
    if (d->chain_off < 0) {
        const char* e = std::getenv("DS_DISC_NO_CHAIN");
        d->chain_off = e && *e == '1' ? 1 : 0;
    }
    if (d->chain_off) return nullptr;
    for (int i = 0; i < d->n_chain; ++i)
        if (d->chain[i].st == st) return &d->chain[i];
    if (d->n_chain == 8) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone)
        return nullptr;
    void* buf = nullptr;
    if (cudaMalloc(&buf, sizeof(float) * kChainPart + 256) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (cudaMemset(buf, 0, sizeof(float) * kChainPart + 256) != cudaSuccess) {
        cudaFree(buf);
        cudaGetLastError();
        return nullptr;
    }
    ds_disc::ChainBuf& c = d->chain[d->n_chain++];
    c.st = st;
    c.part = static_cast<float*>(buf);
    c.done = reinterpret_cast<unsigned*>(static_cast<char*>(buf) + sizeof(float) * kChainPart);
    return &c;
}

struct BatchTail {   // batch_tail_kernel arguments (ds_disc_batch_complete_device)
    ds_curve* curve;
    double decay;
    const double* thr;
    int nt;
    long long index_base;
    long long* heavy;
    long long* counts;
};

ds_status launch_disc(ds_disc* d, const uint8_t* images, int64_t n, int h, int w, float* out,
                      int logits, cudaStream_t st, long long* trace = nullptr,
                      const BatchTail* tail = nullptr, ds_disc::ChainBuf* chain = nullptr) {
    if (h % 16 || w % 16)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "image height and width must be multiples of 16");
    const int tokens = (h / 16) * (w / 16);
    if (tokens % kM)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "patches per image must be a multiple of 128");
    if (reinterpret_cast<uintptr_t>(images) % 16)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "image buffer must be 16-byte aligned");
    if (n <= 0) return DS_OK;
    DiscParams p = d->params;
    p.images = images;
    p.n_img = n;
    p.h = h;
    p.w = w;
    p.px = w / 16;
    p.tokens = tokens;
    p.tiles_per_img = tokens / kM;
    p.trace = trace;
    const long long n_flat = static_cast<long long>(n) * p.tiles_per_img;
    float* part = nullptr;   // one head sum per 128-token tile, every entry written
    if (chain) {
        p.chain = 1;
        p.done = chain->done;
        p.conf = out;
        p.hb = d->hb;
        p.curve = tail->curve;
        p.decay = tail->decay;
        p.thr = tail->thr;
        p.nt = tail->nt;
        p.index_base = tail->index_base;
        p.heavy = tail->heavy;
        p.counts = tail->counts;
        p.err = d->ctx->d_err;
        part = chain->part;
    } else {
        DS_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&part), sizeof(float) * n_flat, st));
    }
    p.part = part;
    if (d->sms == 0) {   // once per ds_disc (one device); kept off the per-launch path
        DS_CUDA_TRY(cudaDeviceGetAttribute(&d->sms, cudaDevAttrMultiProcessorCount, d->ctx->device));
        DS_CUDA_TRY(cudaFuncSetAttribute(disc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes));
    }
    // as many pairs as give every pair the same number of pair tiles: a pair
    // with one tile fewer would idle through the last round (and chained
    // batches start in the SMs it leaves)
    const long long pair_tiles = (n_flat + 1) / 2;
    long long per_pair = (pair_tiles + d->sms / 2 - 1) / (d->sms / 2);
    if (per_pair < d->min_per_pair) per_pair = d->min_per_pair;
    const int pairs = static_cast<int>((pair_tiles + per_pair - 1) / per_pair);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * pairs));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = chain ? 2 : 1;
    DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, disc_kernel, p));
    DS_LAUNCH_CHECK(d->ctx, "disc_kernel");
    if (chain) return DS_OK;   // the tail ran in the grid's last CTA
    if (tail) {
        batch_tail_kernel<<<1, kTailThreads, 0, st>>>(
            part, static_cast<int>(n), p.tiles_per_img, tokens, d->hb, out, tail->curve, tail->decay,
            tail->thr, tail->nt, tail->index_base, tail->heavy, tail->counts, d->ctx->d_err);
        DS_LAUNCH_CHECK(d->ctx, "batch_tail_kernel");
    } else {
        finalize_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(
            part, n, p.tiles_per_img, tokens, d->hb, logits, out);
        DS_LAUNCH_CHECK(d->ctx, "finalize_kernel");
    }
    cudaFreeAsync(part, st);
    return DS_OK;
}

} // namespace

extern "C" ds_status ds_disc_create(ds_ctx* ctx, uint64_t weight_seed, ds_disc** out) {
    if (!ctx || !out) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    ds_disc* d = new ds_disc();
    d->ctx = ctx;
    d->seed = weight_seed;
    if (const char* e = std::getenv("DS_DISC_MIN_PAIR_TILES")) d->min_per_pair = std::max(1, std::atoi(e));
    cudaStream_t st = ctx->stream;
    const size_t nw = static_cast<size_t>(kD1) * kD2 + static_cast<size_t>(kD2) * kD3;
    auto cleanup = [&](ds_status s) {
        cudaFree(d->d_q1);
        cudaFree(d->d_w);
        cudaFree(d->d_blob);
        cudaFree(d->d_b1);
        delete d;
        return s;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&d->d_q1, static_cast<size_t>(kD0) * kD1)) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "malloc q1"));
    if ((e = cudaMalloc(&d->d_w, nw * 2)) != cudaSuccess) return cleanup(dsi::cuda_fail(e, "malloc w"));
    if ((e = cudaMalloc(&d->d_blob, static_cast<size_t>(kBlobStages) * kBStage)) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "malloc blob"));
    if ((e = cudaMalloc(&d->d_b1, kD1 * sizeof(float))) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "malloc b1"));
    uint16_t* w2 = d->d_w;
    uint16_t* w3 = w2 + kD1 * kD2;
    gen_weights_kernel<<<148 * 4, 256, 0, st>>>(weight_seed, d->d_q1, w2, w3);
    tile_weights_kernel<<<kBlobStages, 256, 0, st>>>(d->d_q1, w2, w3, d->d_blob);
    fold_bias_kernel<<<1, 256, 0, st>>>(d->d_q1, weight_seed, d->d_b1);
    ctx->launches.fetch_add(3);
    if ((e = cudaGetLastError()) != cudaSuccess) return cleanup(dsi::cuda_fail(e, "weight init"));
    {
        const ds_status ts = make_weight_tmap(d->d_blob, &d->params.wmap);
        if (ts != DS_OK) return cleanup(ts);
    }
    if ((e = cudaMemcpyAsync(d->params.b1, d->d_b1, sizeof(d->params.b1), cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "copy b1"));
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cleanup(dsi::cuda_fail(e, "sync"));
    d->params.s1 = layer1_scale();
    for (int i = 0; i < kD3; ++i) d->params.hw[i] = unif_pm1(weight_seed ^ 0x7777, i) / 16.0f;
    d->hb = 0.0f;

    // Head calibration: logits of 64 synthetic images (fixed seed) -> affine
    // head so confidences spread over (0, 1): w *= 2/sd, b = -mean * 2/sd.
    const int nc = 64, ch = 512, cw = 512;
    uint8_t* cal = nullptr;
    float* logit = nullptr;
    if ((e = cudaMalloc(&cal, static_cast<size_t>(nc) * ch * cw * 3)) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "malloc cal"));
    if ((e = cudaMalloc(&logit, nc * sizeof(float))) != cudaSuccess) {
        cudaFree(cal);
        return cleanup(dsi::cuda_fail(e, "malloc logits"));
    }
    ds_status s = ds_synth_images_device(ctx, 0xCA11B8A7EULL, 0, nc, ch, cw, cal, st);
    if (s == DS_OK) s = launch_disc(d, cal, nc, ch, cw, logit, 1, st);
    std::vector<float> hl(nc);
    if (s == DS_OK && (e = cudaMemcpyAsync(hl.data(), logit, nc * sizeof(float),
                                           cudaMemcpyDeviceToHost, st)) != cudaSuccess)
        s = dsi::cuda_fail(e, "copy logits");
    if (s == DS_OK && (e = cudaStreamSynchronize(st)) != cudaSuccess) s = dsi::cuda_fail(e, "sync");
    cudaFree(cal);
    cudaFree(logit);
    if (s != DS_OK) return cleanup(s);
    double mean = 0.0, var = 0.0;
    for (float v : hl) mean += v;
    mean /= nc;
    for (float v : hl) var += (v - mean) * (v - mean);
    const double sd = std::sqrt(var / nc);
    if ((!(sd > 0.0) || !std::isfinite(sd)) && !(DS_EXP_FAST_E1 || DS_EXP_NO_WSTREAM))
        return cleanup(dsi::fail(DS_ERR_CUDA, "discriminator calibration produced degenerate logits"));
    const float scale = static_cast<float>(2.0 / sd);
    for (int i = 0; i < kD3; ++i) d->params.hw[i] *= scale;
    d->hb = static_cast<float>(-mean * scale);
    *out = d;
    return DS_OK;
}

extern "C" ds_status ds_disc_destroy(ds_disc* d) {
    if (!d) return DS_OK;
    cudaStreamSynchronize(d->ctx->stream);
    if (d->n_chain) cudaDeviceSynchronize();   // chained calls may sit on other streams
    for (int i = 0; i < d->n_chain; ++i) cudaFree(d->chain[i].part);
    cudaFree(d->d_q1);
    cudaFree(d->d_w);
    cudaFree(d->d_blob);
    cudaFree(d->d_b1);
    delete d;
    return DS_OK;
}

// b2/b3 are carried inside W2/W3 (constant features), so they export as zeros.
extern "C" ds_status ds_disc_export(const ds_disc* d, int8_t* q1, float* s1, uint16_t* w2,
                                    uint16_t* w3, float* b1, float* b2, float* b3, float* head_w,
                                    float* head_b) {
    if (!d) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null disc");
    const uint16_t* d2 = d->d_w;
    const uint16_t* d3 = d2 + kD1 * kD2;
    if (q1) DS_CUDA_TRY(cudaMemcpy(q1, d->d_q1, static_cast<size_t>(kD0) * kD1, cudaMemcpyDeviceToHost));
    if (s1) *s1 = d->params.s1;
    if (w2) DS_CUDA_TRY(cudaMemcpy(w2, d2, sizeof(uint16_t) * kD1 * kD2, cudaMemcpyDeviceToHost));
    if (w3) DS_CUDA_TRY(cudaMemcpy(w3, d3, sizeof(uint16_t) * kD2 * kD3, cudaMemcpyDeviceToHost));
    if (b1) std::memcpy(b1, d->params.b1, sizeof(d->params.b1));
    if (b2) std::memset(b2, 0, sizeof(float) * kD2);
    if (b3) std::memset(b3, 0, sizeof(float) * kD3);
    if (head_w) std::memcpy(head_w, d->params.hw, sizeof(d->params.hw));
    if (head_b) *head_b = d->hb;
    return DS_OK;
}

extern "C" ds_status ds_disc_score_device(ds_disc* d, const uint8_t* nhwc, int64_t n, int32_t h,
                                          int32_t w, float* conf, void* stream) {
    if (!d || (n > 0 && (!nhwc || !conf))) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    return launch_disc(d, nhwc, n, h, w, conf, 0, st);
}

// One light batch, cluster.cpp:288-307: score, observe in batch order, defer.
// Batches of <= 2048 images take the discriminator plus ONE fused tail launch;
// larger ones run the three stages as their own entry points (same results).
extern "C" ds_status ds_disc_batch_complete_device(ds_disc* d, const uint8_t* nhwc, int64_t n,
                                                   int32_t h, int32_t w, float* conf,
                                                   ds_curve* curve, double decay,
                                                   const double* thresholds, int32_t nt,
                                                   int64_t index_base, int64_t* heavy_idx,
                                                   int64_t* counts, void* stream) {
    if (!d || !curve || (n > 0 && (!nhwc || !conf)) || (nt > 0 && (!thresholds || !counts)) ||
        (nt > 0 && n > 0 && !heavy_idx) || nt < 0)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (!(decay > 0.0) || !(decay <= 1.0))
        return dsi::fail(DS_ERR_DOMAIN, "curve decay must lie in (0, 1]");
    if (n <= 0) {
        if (nt > 0) {
            cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
            DS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int64_t) * nt, st));
        }
        return DS_OK;
    }
    if (n > kTailMax) {
        ds_status s = ds_disc_score_device(d, nhwc, n, h, w, conf, stream);
        if (s == DS_OK) s = ds_curve_observe_device(d->ctx, curve, conf, DS_CONF_F32, n, decay, stream);
        if (s == DS_OK && nt > 0)
            s = ds_route_device(d->ctx, conf, DS_CONF_F32, n, thresholds, nt, index_base, heavy_idx,
                                counts, stream);
        return s;
    }
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    BatchTail tail{curve, decay, thresholds, nt, static_cast<long long>(index_base),
                   reinterpret_cast<long long*>(heavy_idx), reinterpret_cast<long long*>(counts)};
    const long long tpi = (static_cast<long long>(h / 16) * (w / 16)) / kM;
    ds_disc::ChainBuf* chain = n * tpi <= kChainPart ? chain_buf(d, st) : nullptr;
    return launch_disc(d, nhwc, n, h, w, conf, 0, st, nullptr, &tail, chain);
}

extern "C" ds_status ds_disc_batches_complete_device(ds_disc* d, const uint8_t* nhwc,
                                                     int64_t n_images, const int64_t* batch_offsets,
                                                     int32_t n_batches, int32_t h, int32_t w,
                                                     float* conf, ds_curve* curve, double decay,
                                                     const double* thresholds, int64_t index_base,
                                                     int64_t* heavy_idx, int64_t* counts,
                                                     void* stream) {
    if (!d || !curve || n_batches < 0 || n_images < 0 ||
        (n_images > 0 && (!nhwc || !conf || !heavy_idx)) ||
        (n_batches > 0 && (!batch_offsets || !thresholds || !counts)))
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (!(decay > 0.0) || !(decay <= 1.0))
        return dsi::fail(DS_ERR_DOMAIN, "curve decay must lie in (0, 1]");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    ds_status s = DS_OK;
    if (n_images > 0) s = launch_disc(d, nhwc, n_images, h, w, conf, 0, st);
    const int* bad = nullptr;
    if (s == DS_OK)
        s = dsi::curve_observe_device_bad(d->ctx, curve, conf, DS_CONF_F32, n_images, decay, st,
                                          &bad);
    if (s != DS_OK || n_batches == 0) return s;
    segmented_route_kernel<<<static_cast<unsigned>(n_batches), kSegThreads, 0, st>>>(
        conf, reinterpret_cast<const long long*>(batch_offsets), thresholds, bad,
        static_cast<long long>(index_base), reinterpret_cast<long long*>(heavy_idx),
        reinterpret_cast<long long*>(counts));
    DS_LAUNCH_CHECK(d->ctx, "segmented_route_kernel");
    return DS_OK;
}

// Host-buffer entry: the image upload is pipelined with scoring -- chunks of
// kChunkImgs images alternate between two device buffers; chunk k+1's copy
// (on the ctx copy stream) overlaps chunk k's kernel (on the ctx stream).
extern "C" ds_status ds_disc_score(ds_disc* d, const uint8_t* nhwc, int64_t n, int32_t h, int32_t w,
                                   float* conf) {
    if (!d || (n > 0 && (!nhwc || !conf))) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (n <= 0) return DS_OK;
    ds_ctx* ctx = d->ctx;
    ds_status s = dsi::ensure_copy_stream(ctx);
    if (s != DS_OK) return s;
    constexpr int64_t kChunkImgs = 148 * 4;
    const size_t img_bytes = static_cast<size_t>(h) * w * 3;
    const int64_t chunk = n < kChunkImgs ? n : kChunkImgs;
    const size_t bi = dsi::align_up(img_bytes * chunk, 256);
    char* buf = nullptr;
    s = dsi::ensure_scratch(ctx, 2 * bi + dsi::align_up(sizeof(float) * n, 256),
                            reinterpret_cast<void**>(&buf));
    if (s != DS_OK) return s;
    float* dconf = reinterpret_cast<float*>(buf + 2 * bi);
    cudaEvent_t* copied = ctx->ev;          // ev[0], ev[1]
    cudaEvent_t* consumed = ctx->ev + 2;    // ev[2], ev[3]
    int k = 0;
    for (int64_t off = 0; off < n; off += chunk, ++k) {
        const int b = k & 1;
        const int64_t m = n - off < chunk ? n - off : chunk;
        uint8_t* dst = reinterpret_cast<uint8_t*>(buf + b * bi);
        if (k >= 2) DS_CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, consumed[b], 0));
        DS_CUDA_TRY(cudaMemcpyAsync(dst, nhwc + static_cast<size_t>(off) * img_bytes,
                                    img_bytes * m, cudaMemcpyHostToDevice, ctx->copy_stream));
        DS_CUDA_TRY(cudaEventRecord(copied[b], ctx->copy_stream));
        DS_CUDA_TRY(cudaStreamWaitEvent(ctx->stream, copied[b], 0));
        s = launch_disc(d, dst, m, h, w, dconf + off, 0, ctx->stream);
        if (s != DS_OK) return s;
        DS_CUDA_TRY(cudaEventRecord(consumed[b], ctx->stream));
    }
    DS_CUDA_TRY(cudaMemcpyAsync(conf, dconf, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DS_OK;
}

// Debug entry (not part of include/ds_gpu.h): ds_disc_batch_complete_device
// (one threshold) with the per-CTA start / end stamps of ds_disc_trace_device.
extern "C" ds_status ds_disc_batch_trace_device(ds_disc* d, const uint8_t* nhwc, int64_t n,
                                                int32_t h, int32_t w, float* conf, ds_curve* curve,
                                                double decay, const double* thr,
                                                int64_t index_base, int64_t* heavy_idx,
                                                int64_t* counts, long long* trace, void* stream) {
    if (!d || n <= 0 || n > kTailMax) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "trace: 1..2048 images");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    BatchTail tail{curve, decay, thr, 1, static_cast<long long>(index_base),
                   reinterpret_cast<long long*>(heavy_idx), reinterpret_cast<long long*>(counts)};
    return launch_disc(d, nhwc, n, h, w, conf, 0, st, trace, &tail, chain_buf(d, st));
}

// Debug entry (not part of include/ds_gpu.h): scores device images and writes
// CTA 0's per-phase clock64 stamps (3 roles x 8 tiles x 16 events) to `trace`.
extern "C" ds_status ds_disc_trace_device(ds_disc* d, const uint8_t* nhwc, int64_t n, int32_t h,
                                          int32_t w, float* conf, long long* trace, void* stream) {
    if (!d) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null disc");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    return launch_disc(d, nhwc, n, h, w, conf, 0, st, trace);
}
