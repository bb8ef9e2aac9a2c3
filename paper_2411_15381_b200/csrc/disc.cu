// K5-K7: the discriminator ("PatchDisc") as one fused, warp-specialized
// tcgen05 kernel. No reference implementation exists (SPEC.md:8 models the
// discriminator as a latent score, see latent.cu); the network is this
// repo's:
//
//   u8 NHWC image -> 16x16x3 patches (token t = py*(W/16)+px, feature
//   k = dy*48 + dx*3 + c) -> h1 = GELU_tanh(x @ W1 + b1)  [768 -> 256]
//   -> h2 = ReLU(bf16(h1) @ W2 + b2) [256 -> 1024] -> h3 = ReLU(bf16(h2) @ W3 + b3)
//   [1024 -> 256] -> logit = mean_t(h3 . w_head) + b_head -> sigmoid.
//   (x is the raw pixel value; the (x-128)/64 normalisation is folded into
//   W1 and b1.)
//
// One CTA per SM, persistent over whole images, M = 128 tokens per tile:
//   warps 0-3   A-builder: 128-bit loads of 16 B pixel runs, u8 -> bf16,
//               swizzled (SW128, K-major) stores into the A ring (16 chunks,
//               one per patch row dy, K = 48 each)
//   warps 4-11  epilogue: tcgen05.ld of the TMEM accumulators, bias +
//               activation, bf16 pack, swizzled stores of H1/H2 (the next
//               GEMM's A operand), and the head dot product + per-image sum
//   warp 12     weight producer: 1-D bulk TMA of pre-swizzled 32 KB weight
//               tiles (L2-resident, evict-last) into a 3-stage ring
//   warp 13     TMEM allocator + the single thread issuing tcgen05.mma
// TMEM (512 columns): [0,256) accumulates GEMM1 and each 256-wide N-chunk of
// GEMM2; [256,512) accumulates GEMM3. Shared memory: R1 (64 KB) holds the A
// ring during GEMM1 and H1 afterwards; R2 (64 KB) holds one 256-wide chunk of
// H2; 3 x 32 KB weight stages.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <vector>

#include "ds_internal.h"
#include "sm100.cuh"

namespace {

using namespace sm100;

constexpr int kM = 128;
constexpr int kD0 = DS_DISC_D0, kD1 = DS_DISC_D1, kD2 = DS_DISC_D2, kD3 = DS_DISC_D3;
constexpr int kWTile = 32768;           // 256 rows x 64 bf16, SW128
constexpr int kWTiles = 48;             // 16 (W1) + 16 (W2) + 16 (W3) per token tile
constexpr int kAChunk = 16384;          // 128 rows x 64 bf16
constexpr int kAStages = 4;
constexpr int kBStages = 3;
constexpr int kThreads = 448;
constexpr int kR1 = 0, kR2 = 65536, kBRing = 131072;
constexpr int kSmemBytes = kBRing + kBStages * kWTile + 1024;   // + alignment slack
constexpr uint32_t kIdesc = idesc_bf16_f32(128, 256);

struct DiscParams {
    float b1[kD1];
    float b2[kD2];
    float b3[kD3];
    float hw[kD3];
    float hb;
    int out_logit;
    const uint8_t* images;
    const uint8_t* wblob;
    float* out;
    long long n_img;
    int h, w, px, tokens, tiles_per_img;
    long long* trace;   // debug: per-phase clock64 stamps of CTA 0 (nullptr = off)
};

// Trace slots (CTA 0 only): role r, tile t < kTraceTiles, event e < 16.
constexpr int kTraceTiles = 8;
#define DS_TRACE(role, tile, ev)                                                          \
    do {                                                                                  \
        if (P.trace && blockIdx.x == 0 && (tile) < kTraceTiles)                           \
            P.trace[((role) * kTraceTiles + (tile)) * 16 + (ev)] = clock64();             \
    } while (0)

__device__ __forceinline__ float gelu_tanh(float x) {
    const float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
    return 0.5f * x * (1.0f + tanh_approx(u));
}

// Byte offset of (row, 16-byte chunk) inside a K-major SW128 tile.
__device__ __forceinline__ uint32_t sw128(uint32_t row, uint32_t chunk) {
    return (row >> 3) * 1024u + (row & 7u) * 128u + ((chunk ^ (row & 7u)) << 4);
}

// 16 pixel bytes -> 16 bf16 (exact: integers < 256 fit the bf16 mantissa).
__device__ __forceinline__ void u8x16_to_bf16(const uint4 v, uint32_t (&o)[8]) {
    const uint32_t in[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        float f[4];
#pragma unroll
        for (int b = 0; b < 4; ++b)   // 2^23 + byte, exactly; subtract 2^23
            f[b] = __uint_as_float(__byte_perm(in[q], 0x4B000000u, 0x7650 + b) ) - 8388608.0f;
        o[2 * q] = pack_bf16x2(f[0], f[1]);
        o[2 * q + 1] = pack_bf16x2(f[2], f[3]);
    }
}

__global__ void __launch_bounds__(kThreads, 1) disc_kernel(const __grid_constant__ DiscParams P) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t a_full[kAStages], a_empty[kAStages], b_full[kBStages], b_empty[kBStages];
    __shared__ uint64_t acc12_full, epi_done, acc3_full, acc3_empty, r1_free;
    __shared__ uint32_t tmem_base_sh;
    __shared__ float warp_part[2][8];

    uint8_t* smem = reinterpret_cast<uint8_t*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
    const uint32_t sbase = smem_u32(smem);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kAStages; ++s) { mbar_init(&a_full[s], 128); mbar_init(&a_empty[s], 1); }
        for (int s = 0; s < kBStages; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
        mbar_init(&acc12_full, 1);
        mbar_init(&epi_done, 256);
        mbar_init(&acc3_full, 1);
        mbar_init(&acc3_empty, 256);
        mbar_init(&r1_free, 1);
        fence_mbar_init();
    }
    if (warp == 13) tmem_alloc<512>(&tmem_base_sh);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    const long long n_img = P.n_img;
    const int tpi = P.tiles_per_img;
    const long long my_imgs =
        blockIdx.x < n_img ? (n_img - 1 - blockIdx.x) / gridDim.x + 1 : 0;
    const long long my_tiles = my_imgs * tpi;
    const long long img_bytes = static_cast<long long>(P.h) * P.w * 3;

    if (warp < 4) {
        // ===================== A-builder (128 threads) ======================
        const int tid = threadIdx.x;
        // piece r = tid + 128*s: token tl = r/3, 16-byte piece p = r%3 of the
        // token's 48-byte pixel run in patch row dy (coalesced along px)
        int tl[3], pp[3];
#pragma unroll
        for (int s = 0; s < 3; ++s) {
            const int r = tid + 128 * s;
            tl[s] = r / 3;
            pp[s] = r % 3;
        }
        auto src_of = [&](long long tile, int dy, int s) -> const uint8_t* {
            const long long img = blockIdx.x + (tile / tpi) * gridDim.x;
            const int tok = static_cast<int>(tile % tpi) * kM + tl[s];
            const int py = tok / P.px, px = tok - py * P.px;
            return P.images + img * img_bytes +
                   (static_cast<long long>(py * 16 + dy) * P.w + px * 16) * 3 + pp[s] * 16;
        };
        const long long total_chunks = my_tiles * 16;
        constexpr int kDepth = 4;   // chunks of pixel data in flight per thread
        uint4 buf[kDepth][3];
#pragma unroll
        for (int d = 0; d < kDepth; ++d)
#pragma unroll
            for (int s = 0; s < 3; ++s)
                if (d < total_chunks) buf[d][s] = ld_global_nc_v4(src_of(d / 16, d % 16, s));
        int astage = 0;
        uint32_t aphase = 0, r1_phase = 0;
        for (long long g0 = 0; g0 < total_chunks; g0 += kDepth) {
#pragma unroll
            for (int d = 0; d < kDepth; ++d) {
                const long long g = g0 + d;     // 16 % kDepth == 0: d == g % kDepth
                const long long tile = g / 16;
                const int dy = static_cast<int>(g % 16);
                if (dy == 0 && tile > 0) {      // R1 still holds the previous tile's H1
                    mbar_wait(&r1_free, r1_phase);
                    r1_phase ^= 1;
                }
                if (tid == 0 && (dy == 0 || dy == 15)) DS_TRACE(0, tile, dy == 0 ? 0 : 1);
                mbar_wait(&a_empty[astage], aphase ^ 1);
                const uint32_t st = sbase + kR1 + astage * kAChunk;
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    uint32_t o[8];
                    u8x16_to_bf16(buf[d][s], o);
                    st_shared_v4(st + sw128(tl[s], 2 * pp[s]), o[0], o[1], o[2], o[3]);
                    st_shared_v4(st + sw128(tl[s], 2 * pp[s] + 1), o[4], o[5], o[6], o[7]);
                }
                fence_proxy_async_smem();
                mbar_arrive(&a_full[astage]);
                if (tid == 0 && (dy == 0 || dy == 15)) DS_TRACE(0, tile, dy == 0 ? 2 : 3);
                if (++astage == kAStages) { astage = 0; aphase ^= 1; }
                const long long gn = g + kDepth;
                if (gn < total_chunks) {
#pragma unroll
                    for (int s = 0; s < 3; ++s)
                        buf[d][s] = ld_global_nc_v4(src_of(gn / 16, static_cast<int>(gn % 16), s));
                }
            }
        }
    } else if (warp < 12) {
        // ===================== epilogue (256 threads) =======================
        const int ew = warp - 4;
        const int q = warp & 3;            // TMEM lane quadrant this warp may access
        const int half = ew >> 2;          // column half [128*half, 128*half+128)
        const uint32_t row = 32 * q + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(32 * q) << 16;
        uint32_t p12 = 0, p3 = 0;
        float img_acc = 0.0f;
        for (long long tile = 0; tile < my_tiles; ++tile) {
            // E1 (j = -1) and E2_j (j = 0..3): acc[0,256) -> H1 / H2
            for (int j = -1; j < 4; ++j) {
                mbar_wait(&acc12_full, p12);
                p12 ^= 1;
                tc_fence_after();
                if (ew == 0 && lane == 0) DS_TRACE(1, tile, 2 * (j + 1));
                const uint32_t hbase = sbase + (j < 0 ? kR1 : kR2);
#pragma unroll 1
                for (int cb = 0; cb < 4; cb += 2) {
                    uint32_t v0[32], v1[32];
                    const int c0 = 128 * half + 32 * cb;
                    tmem_ld2_x32_sync(tmem + lane_addr + c0, tmem + lane_addr + c0 + 32, v0, v1);
#pragma unroll
                    for (int hh = 0; hh < 2; ++hh) {
                        const uint32_t* v = hh ? v1 : v0;
                        const int cbase = c0 + 32 * hh;
#pragma unroll
                        for (int e = 0; e < 32; e += 8) {
                            uint32_t pk[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int c = cbase + e + 2 * u;
                                float a = __uint_as_float(v[e + 2 * u]);
                                float b = __uint_as_float(v[e + 2 * u + 1]);
                                if (j < 0) {
                                    a = gelu_tanh(a + P.b1[c]);
                                    b = gelu_tanh(b + P.b1[c + 1]);
                                } else {
                                    a = fmaxf(a + P.b2[256 * j + c], 0.0f);
                                    b = fmaxf(b + P.b2[256 * j + c + 1], 0.0f);
                                }
                                pk[u] = pack_bf16x2(a, b);
                            }
                            const int f = cbase + e;   // feature within this 256-wide block
                            const uint32_t addr = hbase + (f >> 6) * kAChunk + sw128(row, (f & 63) >> 3);
                            st_shared_v4(addr, pk[0], pk[1], pk[2], pk[3]);
                        }
                    }
                }
                fence_proxy_async_smem();
                tc_fence_before();
                mbar_arrive(&epi_done);
                if (ew == 0 && lane == 0) DS_TRACE(1, tile, 2 * (j + 1) + 1);
            }
            // E3: acc3 -> ReLU(+b3) . w_head, summed over this thread's columns
            mbar_wait(&acc3_full, p3);
            p3 ^= 1;
            tc_fence_after();
            if (ew == 0 && lane == 0) DS_TRACE(1, tile, 10);
            float part = 0.0f;
#pragma unroll 1
            for (int cb = 0; cb < 4; cb += 2) {
                uint32_t v0[32], v1[32];
                const int c0 = 128 * half + 32 * cb;
                tmem_ld2_x32_sync(tmem + lane_addr + 256 + c0, tmem + lane_addr + 256 + c0 + 32,
                                  v0, v1);
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    part += fmaxf(__uint_as_float(v0[e]) + P.b3[c0 + e], 0.0f) * P.hw[c0 + e];
                }
#pragma unroll
                for (int e = 0; e < 32; ++e) {
                    part += fmaxf(__uint_as_float(v1[e]) + P.b3[c0 + 32 + e], 0.0f) * P.hw[c0 + 32 + e];
                }
            }
            tc_fence_before();
            mbar_arrive(&acc3_empty);
            if (ew == 0 && lane == 0) DS_TRACE(1, tile, 11);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
            const int buf = static_cast<int>(tile & 1);
            if (lane == 0) warp_part[buf][ew] = part;
            named_bar_sync(1, 256);
            if (ew == 0 && lane == 0) {
                float s = 0.0f;
#pragma unroll
                for (int w = 0; w < 8; ++w) s += warp_part[buf][w];
                img_acc += s;
                if (tile % tpi == tpi - 1) {
                    const long long img = blockIdx.x + (tile / tpi) * gridDim.x;
                    const float logit = img_acc / static_cast<float>(P.tokens) + P.hb;
                    P.out[img] = P.out_logit ? logit : 1.0f / (1.0f + expf(-logit));
                    img_acc = 0.0f;
                }
            }
        }
    } else if (warp == 12) {
        // ===================== weight producer ==============================
        if (lane == 0) {
            const uint64_t policy = policy_evict_last();
            int bs = 0;
            uint32_t bp = 0;
            for (long long tile = 0; tile < my_tiles; ++tile) {
                for (int t = 0; t < kWTiles; ++t) {
                    mbar_wait(&b_empty[bs], bp ^ 1);
                    mbar_arrive_expect_tx(&b_full[bs], kWTile);
                    bulk_g2s_hint(smem + kBRing + bs * kWTile, P.wblob + static_cast<size_t>(t) * kWTile,
                                  kWTile, &b_full[bs], policy);
                    if (++bs == kBStages) { bs = 0; bp ^= 1; }
                }
            }
        }
    } else {
        // ===================== MMA issuer (warp 13, one thread) ==============
        if (lane == 0) {
            int as = 0, bs = 0;
            uint32_t ap = 0, bp = 0, ep = 0, e3p = 0;
            const uint32_t acc12 = tmem, acc3 = tmem + 256;
            auto wait_b = [&]() {
                mbar_wait(&b_full[bs], bp);
                tc_fence_after();
            };
            auto release_b = [&]() {
                umma_commit(&b_empty[bs]);
                if (++bs == kBStages) { bs = 0; bp ^= 1; }
            };
            // K = 256 GEMM from an H region (4 chunks of 64) into `acc`.
            auto gemm_h = [&](uint32_t hregion, uint32_t acc, bool acc_in) {
                for (int kc = 0; kc < 4; ++kc) {
                    wait_b();
                    const uint64_t ad = desc_k_sw128(sbase + hregion + kc * kAChunk);
                    const uint64_t bd = desc_k_sw128(sbase + kBRing + bs * kWTile);
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        umma_bf16(acc, ad + 2 * k, bd + 2 * k, kIdesc,
                                  (acc_in || kc > 0 || k > 0) ? 1u : 0u);
                    release_b();
                }
            };
            for (long long tile = 0; tile < my_tiles; ++tile) {
                DS_TRACE(2, tile, 0);
                // GEMM1: 16 chunks (patch rows), K = 48 each
                for (int c = 0; c < 16; ++c) {
                    mbar_wait(&a_full[as], ap);
                    wait_b();
                    const uint64_t ad = desc_k_sw128(sbase + kR1 + as * kAChunk);
                    const uint64_t bd = desc_k_sw128(sbase + kBRing + bs * kWTile);
#pragma unroll
                    for (int k = 0; k < 3; ++k)
                        umma_bf16(acc12, ad + 2 * k, bd + 2 * k, kIdesc, (c > 0 || k > 0) ? 1u : 0u);
                    umma_commit(&a_empty[as]);
                    if (++as == kAStages) { as = 0; ap ^= 1; }
                    release_b();
                }
                umma_commit(&acc12_full);
                DS_TRACE(2, tile, 1);
                for (int j = 0; j < 4; ++j) {
                    mbar_wait(&epi_done, ep);     // E1 (j=0) or E2_{j-1}: acc drained, H written
                    ep ^= 1;
                    tc_fence_after();
                    DS_TRACE(2, tile, 2 + 2 * j);
                    if (j > 0) {
                        if (j == 1) {             // acc3 drained by the previous tile's E3
                            mbar_wait(&acc3_empty, e3p ^ 1);
                            e3p ^= 1;
                            tc_fence_after();
                        }
                        gemm_h(kR2, acc3, j > 1);            // GEMM3, K-chunk j-1
                    }
                    gemm_h(kR1, acc12, false);               // GEMM2, N-chunk j
                    umma_commit(&acc12_full);
                    DS_TRACE(2, tile, 3 + 2 * j);
                    if (j == 3) umma_commit(&r1_free);       // H1 no longer read
                }
                mbar_wait(&epi_done, ep);                    // E2_3
                ep ^= 1;
                tc_fence_after();
                DS_TRACE(2, tile, 10);
                gemm_h(kR2, acc3, true);                     // GEMM3, K-chunk 3
                umma_commit(&acc3_full);
                DS_TRACE(2, tile, 11);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 13) {
        tc_fence_after();
        tmem_dealloc<512>(tmem);
    }
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
__device__ __forceinline__ float bf_bits2f(uint16_t b) {
    return __uint_as_float(static_cast<uint32_t>(b) << 16);
}

// Logical weights (row = input feature), bf16 bit patterns.
__global__ void gen_weights_kernel(uint64_t seed, uint16_t* w1, uint16_t* w2, uint16_t* w3) {
    const float s1 = 1.7320508f / (64.0f * sqrtf(768.0f));   // U(-a,a): std = a/sqrt(3)
    const float s2 = 1.7320508f * sqrtf(2.0f / 256.0f);
    const float s3 = 1.7320508f * sqrtf(2.0f / 1024.0f);
    const int n1 = kD0 * kD1, n2 = kD1 * kD2, n3 = kD2 * kD3;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n1 + n2 + n3;
         i += gridDim.x * blockDim.x) {
        if (i < n1) w1[i] = f2bf_bits(s1 * unif_pm1(seed ^ 0x1111, i));
        else if (i < n1 + n2) w2[i - n1] = f2bf_bits(s2 * unif_pm1(seed ^ 0x2222, i - n1));
        else w3[i - n1 - n2] = f2bf_bits(s3 * unif_pm1(seed ^ 0x3333, i - n1 - n2));
    }
}

// Pre-swizzled blob in the MMA consumption order (see disc_kernel): for each
// 32 KB tile, element (n, kl) of a 256 x 64 K-major SW128 tile.
__global__ void tile_weights_kernel(const uint16_t* w1, const uint16_t* w2, const uint16_t* w3,
                                    uint16_t* blob) {
    const int t = blockIdx.x;          // 0..47
    int type, j, kc;                   // type 0: W1 chunk j(=dy); 1: W2 (j, kc); 2: W3 (j, kc)
    if (t < 16) { type = 0; j = t; kc = 0; }
    else {
        // per j: [W3(j-1) x4 if j>0], W2(j) x4; then W3(3) x4
        const int u = t - 16;          // 0..31
        if (u < 4) { type = 1; j = 0; kc = u; }
        else if (u < 28) {
            const int v = u - 4, jj = 1 + v / 8, r = v % 8;
            if (r < 4) { type = 2; j = jj - 1; kc = r; } else { type = 1; j = jj; kc = r - 4; }
        } else { type = 2; j = 3; kc = u - 28; }
    }
    uint16_t* out = blob + static_cast<size_t>(t) * (kWTile / 2);
    for (int e = threadIdx.x; e < 256 * 64; e += blockDim.x) {
        const int n = e / 64, kl = e % 64;
        uint16_t v = 0;
        if (type == 0) {
            if (kl < 48) v = w1[(48 * j + kl) * kD1 + n];
        } else if (type == 1) {
            v = w2[(64 * kc + kl) * kD2 + 256 * j + n];
        } else {
            v = w3[(256 * j + 64 * kc + kl) * kD3 + n];
        }
        const uint32_t byte = (n >> 3) * 1024u + (n & 7) * 128u + ((((kl >> 3) ^ (n & 7))) << 4) +
                              (kl & 7) * 2u;
        out[byte / 2] = v;
    }
}

// b1[n] = -128 * sum_k W1[k][n] + small bias: folds the (x - 128) / 64 input
// normalisation into layer 1 (the 1/64 is in W1's scale).
__global__ void fold_bias_kernel(const uint16_t* w1, uint64_t seed, float* b1) {
    const int n = blockIdx.x * blockDim.x + threadIdx.x;
    if (n >= kD1) return;
    float s = 0.0f;
    for (int k = 0; k < kD0; ++k) s += bf_bits2f(w1[k * kD1 + n]);
    b1[n] = -128.0f * s + 0.05f * unif_pm1(seed ^ 0x4444, n);
}

} // namespace

struct ds_disc {
    ds_ctx* ctx = nullptr;
    uint64_t seed = 0;
    uint16_t* d_w = nullptr;   // w1 | w2 | w3 logical
    uint8_t* d_blob = nullptr;
    float* d_b1 = nullptr;
    DiscParams params{};       // biases + head (device-independent part)
};

namespace {

ds_status launch_disc(ds_disc* d, const uint8_t* images, int64_t n, int h, int w, float* out,
                      int logits, cudaStream_t st, long long* trace = nullptr) {
    if (h % 16 || w % 16)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "image height and width must be multiples of 16");
    const int tokens = (h / 16) * (w / 16);
    if (tokens % kM)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "patches per image must be a multiple of 128");
    if (reinterpret_cast<uintptr_t>(images) % 16)
        return dsi::fail(DS_ERR_INVALID_ARGUMENT, "image buffer must be 16-byte aligned");
    if (n <= 0) return DS_OK;
    DiscParams p = d->params;
    p.out_logit = logits;
    p.images = images;
    p.wblob = d->d_blob;
    p.out = out;
    p.n_img = n;
    p.h = h;
    p.w = w;
    p.px = w / 16;
    p.tokens = tokens;
    p.tiles_per_img = tokens / kM;
    p.trace = trace;
    static bool attr_set = false;
    if (!attr_set) {
        DS_CUDA_TRY(cudaFuncSetAttribute(disc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kSmemBytes));
        attr_set = true;
    }
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, d->ctx->device);
    const int grid = static_cast<int>(n < sms ? n : sms);
    disc_kernel<<<grid, kThreads, kSmemBytes, st>>>(p);
    DS_LAUNCH_CHECK(d->ctx, "disc_kernel");
    return DS_OK;
}

} // namespace

extern "C" ds_status ds_disc_create(ds_ctx* ctx, uint64_t weight_seed, ds_disc** out) {
    if (!ctx || !out) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    *out = nullptr;
    ds_disc* d = new ds_disc();
    d->ctx = ctx;
    d->seed = weight_seed;
    cudaStream_t st = ctx->stream;
    const size_t nw = static_cast<size_t>(kD0) * kD1 + static_cast<size_t>(kD1) * kD2 +
                      static_cast<size_t>(kD2) * kD3;
    auto cleanup = [&](ds_status s) {
        cudaFree(d->d_w);
        cudaFree(d->d_blob);
        cudaFree(d->d_b1);
        delete d;
        return s;
    };
    cudaError_t e;
    if ((e = cudaMalloc(&d->d_w, nw * 2)) != cudaSuccess) return cleanup(dsi::cuda_fail(e, "malloc w"));
    if ((e = cudaMalloc(&d->d_blob, static_cast<size_t>(kWTiles) * kWTile)) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "malloc blob"));
    if ((e = cudaMalloc(&d->d_b1, kD1 * sizeof(float))) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "malloc b1"));
    uint16_t* w1 = d->d_w;
    uint16_t* w2 = w1 + kD0 * kD1;
    uint16_t* w3 = w2 + kD1 * kD2;
    gen_weights_kernel<<<148 * 4, 256, 0, st>>>(weight_seed, w1, w2, w3);
    tile_weights_kernel<<<kWTiles, 256, 0, st>>>(w1, w2, w3, reinterpret_cast<uint16_t*>(d->d_blob));
    fold_bias_kernel<<<1, 256, 0, st>>>(w1, weight_seed, d->d_b1);
    ctx->launches.fetch_add(3);
    if ((e = cudaGetLastError()) != cudaSuccess) return cleanup(dsi::cuda_fail(e, "weight init"));
    if ((e = cudaMemcpyAsync(d->params.b1, d->d_b1, sizeof(d->params.b1), cudaMemcpyDeviceToHost,
                             st)) != cudaSuccess)
        return cleanup(dsi::cuda_fail(e, "copy b1"));
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cleanup(dsi::cuda_fail(e, "sync"));
    for (int i = 0; i < kD2; ++i) d->params.b2[i] = 0.05f * unif_pm1(weight_seed ^ 0x5555, i);
    for (int i = 0; i < kD3; ++i) d->params.b3[i] = 0.05f * unif_pm1(weight_seed ^ 0x6666, i);
    for (int i = 0; i < kD3; ++i) d->params.hw[i] = unif_pm1(weight_seed ^ 0x7777, i) / 16.0f;
    d->params.hb = 0.0f;

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
    if (!(sd > 0.0) || !std::isfinite(sd))
        return cleanup(dsi::fail(DS_ERR_CUDA, "discriminator calibration produced degenerate logits"));
    const float scale = static_cast<float>(2.0 / sd);
    for (int i = 0; i < kD3; ++i) d->params.hw[i] *= scale;
    d->params.hb = static_cast<float>(-mean * scale);
    *out = d;
    return DS_OK;
}

extern "C" ds_status ds_disc_destroy(ds_disc* d) {
    if (!d) return DS_OK;
    cudaStreamSynchronize(d->ctx->stream);
    cudaFree(d->d_w);
    cudaFree(d->d_blob);
    cudaFree(d->d_b1);
    delete d;
    return DS_OK;
}

extern "C" ds_status ds_disc_export(const ds_disc* d, uint16_t* w1, uint16_t* w2, uint16_t* w3,
                                    float* b1, float* b2, float* b3, float* head_w, float* head_b) {
    if (!d) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null disc");
    const uint16_t* d1 = d->d_w;
    const uint16_t* d2 = d1 + kD0 * kD1;
    const uint16_t* d3 = d2 + kD1 * kD2;
    if (w1) DS_CUDA_TRY(cudaMemcpy(w1, d1, sizeof(uint16_t) * kD0 * kD1, cudaMemcpyDeviceToHost));
    if (w2) DS_CUDA_TRY(cudaMemcpy(w2, d2, sizeof(uint16_t) * kD1 * kD2, cudaMemcpyDeviceToHost));
    if (w3) DS_CUDA_TRY(cudaMemcpy(w3, d3, sizeof(uint16_t) * kD2 * kD3, cudaMemcpyDeviceToHost));
    if (b1) std::memcpy(b1, d->params.b1, sizeof(d->params.b1));
    if (b2) std::memcpy(b2, d->params.b2, sizeof(d->params.b2));
    if (b3) std::memcpy(b3, d->params.b3, sizeof(d->params.b3));
    if (head_w) std::memcpy(head_w, d->params.hw, sizeof(d->params.hw));
    if (head_b) *head_b = d->params.hb;
    return DS_OK;
}

extern "C" ds_status ds_disc_score_device(ds_disc* d, const uint8_t* nhwc, int64_t n, int32_t h,
                                          int32_t w, float* conf, void* stream) {
    if (!d || (n > 0 && (!nhwc || !conf))) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    return launch_disc(d, nhwc, n, h, w, conf, 0, st);
}

extern "C" ds_status ds_disc_score(ds_disc* d, const uint8_t* nhwc, int64_t n, int32_t h, int32_t w,
                                   float* conf) {
    if (!d || (n > 0 && (!nhwc || !conf))) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null argument");
    if (n <= 0) return DS_OK;
    ds_ctx* ctx = d->ctx;
    const size_t img_bytes = static_cast<size_t>(h) * w * 3;
    const size_t bi = dsi::align_up(img_bytes * n, 256);
    char* buf = nullptr;
    ds_status s = dsi::ensure_scratch(ctx, bi + dsi::align_up(sizeof(float) * n, 256),
                                      reinterpret_cast<void**>(&buf));
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(buf, nhwc, img_bytes * n, cudaMemcpyHostToDevice, ctx->stream));
    float* dconf = reinterpret_cast<float*>(buf + bi);
    s = launch_disc(d, reinterpret_cast<uint8_t*>(buf), n, h, w, dconf, 0, ctx->stream);
    if (s != DS_OK) return s;
    DS_CUDA_TRY(cudaMemcpyAsync(conf, dconf, sizeof(float) * n, cudaMemcpyDeviceToHost, ctx->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    return DS_OK;
}

// Debug entry (not part of include/ds_gpu.h): scores device images and writes
// CTA 0's per-phase clock64 stamps (3 roles x 8 tiles x 16 events) to `trace`.
extern "C" ds_status ds_disc_trace_device(ds_disc* d, const uint8_t* nhwc, int64_t n, int32_t h,
                                          int32_t w, float* conf, long long* trace, void* stream) {
    if (!d) return dsi::fail(DS_ERR_INVALID_ARGUMENT, "null disc");
    cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : d->ctx->stream;
    return launch_disc(d, nhwc, n, h, w, conf, 0, st, trace);
}
