// Probe for an int8 layer 1: u8 pixel patches loaded by TMA straight into a
// K-major SW128 UMMA operand, int8 weights in SW64 16 KB stages, tcgen05.mma
// kind::i8 (u8 x s8 -> s32 in TMEM).
// The box {48 B, 32 px, 4 patch rows, 2 dy} with SWIZZLE_64B lands as
// [dy][token][64 B] rows -- the 48-byte run padded to the 64-byte swizzle
// span -- i.e. the UMMA K-major SW64 layout with K = 64 per dy, of which the
// last 16 bytes are padding (garbage) and meet zero weights.
// (Measured: a no-swizzle K-major A (8x16 B core matrices, LBO 2 KB) runs
// the i8 MMA at ~343 cycles instead of the 128-cycle floor; a 16-byte inner
// box with SWIZZLE_128B is padded to 128 B per row and overflows the stage.)
// Checks one tile against the CPU, then times GEMM1-only tiles on 148 SMs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2411_15381_b200/csrc tools/i8_probe.cu -o gpurun_out/i8_probe
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sm100.cuh"

using namespace sm100;

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            exit(1);                                                                 \
        }                                                                            \
    } while (0)

constexpr int H = 512, W = 512, PX = W / 16, PY = H / 16;
constexpr int kAChunk = 16384;      // 2 dy x 128 tokens x 64 B (48 B + pad), SW64
#ifndef ASW
#define ASW 0
#endif
#ifndef LBO
#define LBO 2048
#endif
#ifndef SBO
#define SBO 128
#endif
#ifndef AST
#define AST 2
#endif
constexpr int kAStages = AST, kBStages = 4;
constexpr int kBStage = 16384;      // 256 rows x 64 B (K = 64 int8), SW64
constexpr int kChunks = 8, kW1Stages = 16;
constexpr int kSmem = kAStages * kAChunk + kBStages * kBStage + 2048;

__device__ __forceinline__ uint64_t desc_k_sw64(uint32_t a) {
    const uint64_t lo = ((a >> 4) & 0x3FFFu) | (1u << 16);
    const uint64_t hi = (512u >> 4) | (1u << 14) | (4u << 29);
    return lo | (hi << 32);
}
// K-major, no swizzle: core matrix = 8 rows x 16 B contiguous; SBO = M stride
// of 8-row groups (128 B), LBO = K stride of 16-byte pieces (2 KB).
__device__ __forceinline__ uint64_t desc_k_none(uint32_t a, uint32_t lbo, uint32_t sbo) {
    const uint64_t lo = ((a >> 4) & 0x3FFFu) | ((lbo >> 4) << 16);
    const uint64_t hi = (sbo >> 4) | (1u << 14);
    return lo | (hi << 32);
}
constexpr uint32_t kIdesc = (2u << 4) | (0u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);

__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(kIdesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tma_5d(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3,
                                       int c4, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4), "r"(smem_u32(bar))
        : "memory");
}

#ifndef ATX
#define ATX 12288   // tx bytes of one A box (unpadded)
#endif
__device__ __forceinline__ void tma_4d(uint32_t dst, const void* tmap, int c0, int c1, int c2, int c3,
                                       uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
        : "memory");
}

struct Params {
    CUtensorMap amap;
    const uint8_t* wblob;
    const uint8_t* images;
    int n_img, tiles_per_cta, mode, prefetch;   // mode 0: A+B | 1: B only | 2: A only | 3: none
    int* out;                         // tile 0 of CTA 0: [128][256] s32
    long long* cyc;
};

__global__ void __launch_bounds__(192, 1) probe(const __grid_constant__ Params P) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t a_full[kAStages], a_empty[kAStages], b_full[kBStages], b_empty[kBStages], done;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t sraw = smem_u32(smem);
    const uint32_t sbase = (sraw + 1023u) & ~1023u;   // swizzle atoms: 1024-byte aligned
    uint8_t* smem_al = smem + (sbase - sraw);
    const uint32_t sA = sbase, sB = sbase + kAStages * kAChunk;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kAStages; ++s) { mbar_init(&a_full[s], 1); mbar_init(&a_empty[s], 1); }
        for (int s = 0; s < kBStages; ++s) { mbar_init(&b_full[s], 1); mbar_init(&b_empty[s], 1); }
        mbar_init(&done, 1);
        fence_mbar_init();
    }
    if (warp == 1) tmem_alloc<256>(&tmem_base);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const int T = P.tiles_per_cta;
    const int tiles_per_img = PY / 4;
    long long t0 = clock64();
    if (warp == 0 && lane == 0) {          // A producer (+ L2 prefetch 2 tiles ahead)
        int as = 0;
        uint32_t ap = 0;
        auto tile_prow = [&](int t) {
            const long long gt = static_cast<long long>(blockIdx.x) * T + t;
            const int img = static_cast<int>((gt / tiles_per_img) % P.n_img);
            return img * PY + static_cast<int>(gt % tiles_per_img) * 4;
        };
        auto prefetch = [&](int t) {
            if (t >= T || !P.prefetch) return;
            const uint8_t* p0 = P.images + static_cast<size_t>(tile_prow(t)) * 48 * W;
            for (int off = 0; off < 4 * 48 * W; off += 65536) bulk_prefetch_l2(p0 + off, 65536 < 4 * 48 * W - off ? 65536 : 4 * 48 * W - off);
        };
        prefetch(0);
        prefetch(1);
        for (int t = 0; t < T; ++t) {
            prefetch(t + 2);
            const int prow = tile_prow(t);
            for (int c = 0; c < kChunks; ++c) {
                mbar_wait(&a_empty[as], ap ^ 1);
                if (P.mode == 0 || P.mode == 2) {
                    mbar_arrive_expect_tx(&a_full[as], ATX);
                    tma_4d(sA + as * kAChunk, &P.amap, 0, 0, prow, 2 * c, &a_full[as]);
                } else {
                    mbar_arrive(&a_full[as]);
                }
                if (++as == kAStages) { as = 0; ap ^= 1; }
            }
        }
    } else if (warp == 2 && lane == 0) {   // B producer
        int bs = 0;
        uint32_t bp = 0;
        for (int t = 0; t < T; ++t) {
            for (int wst = 0; wst < kW1Stages; ++wst) {
                mbar_wait(&b_empty[bs], bp ^ 1);
                if (P.mode == 0 || P.mode == 1) {
                    mbar_arrive_expect_tx(&b_full[bs], kBStage);
                    bulk_g2s(smem_al + kAStages * kAChunk + bs * kBStage,
                             P.wblob + static_cast<size_t>(wst) * kBStage, kBStage, &b_full[bs]);
                } else {
                    mbar_arrive(&b_full[bs]);
                }
                if (++bs == kBStages) { bs = 0; bp ^= 1; }
            }
        }
    } else if (warp == 1 && lane == 0) {
        int as = 0, bs = 0;
        uint32_t ap = 0, bp = 0;
        for (int t = 0; t < T; ++t) {
            for (int s = 0; s < 32; ++s) {     // K = 1024 in steps of 32: chunk s/4, dy s/2
                if (s % 4 == 0) { mbar_wait(&a_full[as], ap); tc_fence_after(); }
                if (s % 2 == 0) { mbar_wait(&b_full[bs], bp); tc_fence_after(); }
                const uint64_t ad = desc_k_sw64(sA + as * kAChunk + ((s >> 1) & 1) * 8192) + 2 * (s % 2);
                const uint64_t bd = desc_k_sw64(sB + bs * kBStage) + 2 * (s % 2);
                umma_i8(tmem, ad, bd, s > 0 ? 1u : 0u);
                if (s % 2 == 1) { umma_commit(&b_empty[bs]); if (++bs == kBStages) { bs = 0; bp ^= 1; } }
                if (s % 4 == 3) { umma_commit(&a_empty[as]); if (++as == kAStages) { as = 0; ap ^= 1; } }
            }
        }
        umma_commit(&done);
    }
    if (warp >= 2) {
        __syncwarp();
#if SLEEPWAIT
        {
            uint32_t ok = 0;
            while (!ok) {
                __nanosleep(2000);
                asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                             : "=r"(ok) : "r"(smem_u32(&done)) : "memory");
            }
        }
#else
        mbar_wait(&done, 0);
#endif
        tc_fence_after();
        if (blockIdx.x == 0 && P.out) {
            const int q = warp & 3;
            for (int cb = 0; cb < 256; cb += 32) {
                uint32_t v[32];
                tmem_ld_x32_sync(tmem + (static_cast<uint32_t>(32 * q) << 16) + cb, v);
                for (int e = 0; e < 32; ++e) P.out[(32 * q + lane) * 256 + cb + e] = static_cast<int>(v[e]);
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) P.cyc[blockIdx.x] = clock64() - t0;
    if (warp == 1) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

// GEMM K index (chunk c = 2 q3 + h, byte b) -> patch feature k = dy*48 + q3*16 + byte
static int korig(int kg) {   // -1: padding (zero weight)
    const int dy = kg / 64, b = kg % 64;
    return b < 48 ? dy * 48 + b : -1;
}

int main() {
    const int n_img = 296;
    const size_t img_bytes = static_cast<size_t>(H) * W * 3;
    std::vector<uint8_t> himg(img_bytes * n_img);
    uint64_t s = 88172645463325252ULL;
    for (auto& b : himg) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; b = static_cast<uint8_t>(s >> 24); }
    std::vector<int8_t> w1(768 * 256);
    for (auto& w : w1) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; w = static_cast<int8_t>(static_cast<int>(s % 255) - 127); }
    // blob: stage st = K range [64 st, 64 st + 64), rows n, SW64
    std::vector<uint8_t> blob(kW1Stages * kBStage);
    for (int st = 0; st < kW1Stages; ++st)
        for (int n = 0; n < 256; ++n)
            for (int kb = 0; kb < 64; ++kb) {
                const uint32_t byte = (n >> 3) * 512u + (n & 7) * 64u + ((((kb >> 4) ^ ((n >> 1) & 3))) << 4) + (kb & 15);
                const int ko = korig(64 * st + kb);
                blob[st * kBStage + byte] = ko < 0 ? 0 : static_cast<uint8_t>(w1[ko * 256 + n]);
            }
    uint8_t *dimg, *dblob;
    int* dout;
    long long* dcyc;
    CK(cudaMalloc(&dimg, himg.size()));
    CK(cudaMalloc(&dblob, blob.size()));
    CK(cudaMalloc(&dout, 128 * 256 * 4));
    CK(cudaMalloc(&dcyc, 148 * 8));
    CK(cudaMemcpy(dimg, himg.data(), himg.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dblob, blob.data(), blob.size(), cudaMemcpyHostToDevice));

    using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    Params P{};
    // dims: d0 48 B run | d1 px (48 B) | d2 patch row (48 W B) | d3 dy (3 W B)
    const cuuint64_t dims[4] = {48, PX, static_cast<cuuint64_t>(n_img) * PY, 16};
    const cuuint64_t strides[3] = {48, 48ull * W, 3ull * W};
    const cuuint32_t box[4] = {48, 32, 4, 2};
    const cuuint32_t es[5] = {1, 1, 1, 1, 1};
    CUresult r = reinterpret_cast<EncodeFn>(fn)(&P.amap, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, dimg, dims, strides, box, es,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode non-monotonic 5-D map: %d\n", static_cast<int>(r));
    if (r != CUDA_SUCCESS) return 1;
    P.wblob = dblob;
    P.n_img = n_img;
    P.cyc = dcyc;
    CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    // correctness: one tile on one CTA
    P.tiles_per_cta = 1;
    P.mode = 0;
    P.out = dout;
    probe<<<1, 192, kSmem>>>(P);
    CK(cudaDeviceSynchronize());
    std::vector<int> got(128 * 256);
    CK(cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost));
    long long bad = 0;
    for (int m = 0; m < 128; ++m) {
        const int py = m / PX, px = m % PX;
        for (int n = 0; n < 256; ++n) {
            long long acc = 0;
            for (int k = 0; k < 768; ++k) {
                const int dy = k / 48, r48 = k % 48;
                acc += static_cast<long long>(himg[(static_cast<size_t>(py * 16 + dy) * W + px * 16) * 3 + r48]) *
                       w1[k * 256 + n];
            }
            if (acc != got[m * 256 + n]) {
                if (bad < 5) printf("mismatch m=%d n=%d got %d want %lld\n", m, n, got[m * 256 + n], acc);
                ++bad;
            }
        }
    }
    printf("tile check: %lld mismatches of %d\n", bad, 128 * 256);
    P.out = nullptr;
    const char* names[4] = {"A by TMA + W1 by bulk", "W1 only (A static)", "A only (W1 static)", "MMA only"};
    P.images = dimg;
    for (int run = 0; run < 6; ++run) {
        const int mode = run < 4 ? run : run - 4;
        P.mode = mode;
        P.prefetch = run >= 4 || getenv("PF") != nullptr;
        P.tiles_per_cta = 64;
        probe<<<148, 192, kSmem>>>(P);
        CK(cudaDeviceSynchronize());
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        probe<<<148, 192, kSmem>>>(P);
        cudaEventRecord(e1);
        CK(cudaDeviceSynchronize());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        std::vector<long long> cyc(148);
        CK(cudaMemcpy(cyc.data(), dcyc, 148 * 8, cudaMemcpyDeviceToHost));
        long long mx = 0;
        for (auto c : cyc) mx = c > mx ? c : mx;
        printf("%-26s pf=%d: %.0f cycles per tile (max CTA), %.3f ms; floor 3072\n", names[mode], P.prefetch,
               static_cast<double>(mx) / P.tiles_per_cta, ms);
    }
    return 0;
}
