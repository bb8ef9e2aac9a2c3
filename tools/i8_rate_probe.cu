// tcgen05.mma issue rate, kind::i8 vs kind::f16, by operand swizzle, with
// static shared-memory operands on all 148 SMs (one elected thread per CTA).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2411_15381_b200/csrc tools/i8_rate_probe.cu -o /tmp/i8_rate_probe
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace sm100;

constexpr int kIters = 4096;

__device__ __forceinline__ uint64_t desc_sw(uint32_t a, int layout) {   // K-major
    // layout 2 = SW128 (atom 1024 B), 4 = SW64 (512 B), 6 = SW32 (256 B)
    const uint32_t sbo = layout == 2 ? 1024u : layout == 4 ? 512u : 256u;
    const uint64_t lo = ((a >> 4) & 0x3FFFu) | (1u << 16);
    const uint64_t hi = (sbo >> 4) | (1u << 14) | (static_cast<uint32_t>(layout) << 29);
    return lo | (hi << 32);
}

template <int kKind>   // 0: f16 (bf16), 1: i8
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    if constexpr (kKind == 0)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
    else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                     "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}

template <int kKind>
__global__ void __launch_bounds__(128, 1) probe(int alay, int blay, int fill, int cmode, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t done, dummy[8];
    __shared__ uint32_t tmem_base;
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (sbase - raw);
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = fill ? (i * 2654435761u) : 0u;
    if (threadIdx.x == 0) { mbar_init(&done, 1); for (int i = 0; i < 8; ++i) mbar_init(&dummy[i], 1); fence_mbar_init(); }
    if (threadIdx.x < 32) tmem_alloc<256>(&tmem_base);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (threadIdx.x == 0) {
        const uint32_t idesc = kKind == 0
            ? idesc_bf16_f32(128, 256)
            : ((2u << 4) | (0u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24));
        // A: 16 KB region @0, B: 32 KB region @16 KB; K-step = 32 bytes
        const int arow = alay == 2 ? 128 : alay == 4 ? 64 : 32;   // bytes of K per row
        const int brow = blay == 2 ? 128 : blay == 4 ? 64 : 32;
        const long long t0 = clock64();
        // descriptors precomputed: 4 A K-steps x 4 B K-steps (lean issue loop)
        uint64_t ads[4], bds[4];
        for (int k = 0; k < 4; ++k) {
            const int ka = 32 * k, kb = 32 * k;
            ads[k] = desc_sw(sbase + (ka / arow) * 128 * arow, alay) + ((ka % arow) >> 4);
            bds[k] = desc_sw(sbase + 16384 + (kb / brow) * 256 * brow, blay) + ((kb % brow) >> 4);
        }
        if (cmode == 0) {
            for (int it = 0; it < kIters; it += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) mma<kKind>(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
            }
        } else if (cmode == 1) {
            for (int it = 0; it < kIters; it += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    mma<kKind>(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                    if (k & 1) umma_commit(&dummy[((it + k) >> 1) & 7]);
                }
            }
        } else if (cmode == 2) {   // wait (long complete) before each 2-MMA stage
            for (int it = 0; it < kIters; it += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int st = (it + k) >> 1;
                    if (!(k & 1) && st >= 4) mbar_wait(&dummy[(st - 4) & 7], ((st - 4) >> 3) & 1);
                    mma<kKind>(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                    if (k & 1) umma_commit(&dummy[st & 7]);
                }
            }
        } else if (cmode == 3) {   // wait between the two MMAs of a stage
            for (int it = 0; it < kIters; it += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int st = (it + k) >> 1;
                    mma<kKind>(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                    if (!(k & 1) && st >= 3) mbar_wait(&dummy[(st - 3) & 7], ((st - 3) >> 3) & 1);
                    if (k & 1) umma_commit(&dummy[st & 7]);
                }
            }
        } else if (cmode == 4) {   // test_wait (non-blocking probe), once per stage
            uint32_t okc = 0;
            for (int it = 0; it < kIters; it += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int st = (it + k) >> 1;
                    if (!(k & 1) && st >= 4) {
                        uint32_t ok;
                        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                     : "=r"(ok) : "r"(smem_u32(&dummy[(st - 4) & 7])), "r"(((st - 4) >> 3) & 1) : "memory");
                        okc += ok;
                    }
                    mma<kKind>(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                    if (k & 1) umma_commit(&dummy[st & 7]);
                }
            }
            if (okc == 12345) out[1000] = 0;
        } else if (cmode == 5) {   // wait + fence before each 4-MMA stage
            for (int it = 0; it < kIters; it += 4) {
                const int st = it >> 2;
                if (st >= 4) { mbar_wait(&dummy[(st - 4) & 7], ((st - 4) >> 3) & 1); tc_fence_after(); }
#pragma unroll
                for (int k = 0; k < 4; ++k) mma<kKind>(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                umma_commit(&dummy[st & 7]);
            }
        } else {                   // cmode 6: as 2 + tcgen05 fence after the wait
            for (int it = 0; it < kIters; it += 4) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int st = (it + k) >> 1;
                    if (!(k & 1) && st >= 4) { mbar_wait(&dummy[(st - 4) & 7], ((st - 4) >> 3) & 1); tc_fence_after(); }
                    mma<kKind>(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                    if (k & 1) umma_commit(&dummy[st & 7]);
                }
            }
        }
        umma_commit(&done);
        mbar_wait(&done, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc<256>(tmem_base); }
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 65536 + 2048;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int lays[3] = {2, 4, 6};
    const char* ln[7] = {"", "", "SW128", "", "SW64", "", "SW32"};
    for (int kind = 0; kind < 2; ++kind)
        for (int fill = 0; fill < 7; ++fill)
            for (int a = 0; a < 1; a += 1)
                for (int b = 1; b < 2; ++b) {
                    if (kind == 0) probe<0><<<148, 128, smem>>>(lays[a], lays[b], 1, fill, d);
                    else probe<1><<<148, 128, smem>>>(lays[a], lays[b], 1, fill, d);
                    cudaError_t e = cudaDeviceSynchronize();
                    long long h[148];
                    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
                    long long mx = 0;
                    for (long long v : h) mx = v > mx ? v : mx;
                    printf("%s cmode=%d A %-5s B %-5s : %6.1f cycles/MMA (M128 N256, K=32 bytes)%s\n",
                           kind ? "i8 " : "f16", fill, ln[lays[a]], ln[lays[b]],
                           static_cast<double>(mx) / kIters, e == cudaSuccess ? "" : cudaGetErrorString(e));
                }
    return 0;
}
