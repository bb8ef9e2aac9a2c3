// Microbenchmark: tcgen05.mma issue rate for the discriminator's operand
// layouts, alone and with concurrent shared-memory traffic, to find what
// bounds disc_kernel. Build + run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2411_15381_b200/csrc tools/umma_probe.cu -o gpurun_out/umma_probe
//   gpurun_out/umma_probe
// Prints cycles per MMA instruction (K = 16) per mode, all 148 SMs busy.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace sm100;

constexpr int kIters = 2048;   // MMAs per CTA (x4 K-steps inside each block of 4)

__device__ __forceinline__ uint64_t desc_k_sw64(uint32_t smem_addr) {
    const uint64_t lo = ((smem_addr >> 4) & 0x3FFFu) | (1u << 16);
    const uint64_t hi = (512u >> 4) | (1u << 14) | (4u << 29);
    return lo | (hi << 32);
}

__device__ __forceinline__ void umma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                        uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}

struct Out {
    long long cycles;
    long long mmas;
    long long traffic_bytes;
};

// mode: 0 SS N256 B-SW64 | 1 SS N256 B-SW128 | 2 SS N128 B-SW128 | 3 TS N256 B-SW128
//       4 pair M256 N256 B-SW64 halves | 5 pair M256 N256 B-SW128 halves
// traffic: 0 none | 1 warps 1-3 st.shared.v4 flat out | 2 bulk TMA ring from L2
template <bool kPairT>
__global__ void __launch_bounds__(128, 1) probe(int mode, int tmode, const uint8_t* gsrc,
                                                Out* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t done_bar, tma_full[4], tma_empty[4];
    __shared__ uint32_t tmem_base;
    __shared__ volatile int stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr bool pair = kPairT;
    uint32_t rank = 0;
    if constexpr (pair) rank = cluster_ctarank();
    const uint32_t sbase = smem_u32(smem);
    // layout: A 16 KB @0 | B 32 KB @16K | traffic region 64 KB @48K
    for (int i = threadIdx.x; i < (48 << 10) / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(smem)[i] = make_uint4(0x3f803f80u, 0, 0x3f803f80u, 0);
    if (threadIdx.x == 0) {
        mbar_init(&done_bar, 1);
        for (int s = 0; s < 4; ++s) {
            mbar_init(&tma_full[s], 1);
            mbar_init(&tma_empty[s], 1);
        }
        stop = 0;
        fence_mbar_init();
    }
    if (warp == 0) {
        if constexpr (pair) tmem_alloc2<512>(&tmem_base);
        else tmem_alloc<512>(&tmem_base);
    }
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    if constexpr (pair) cluster_sync();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    long long traffic = 0;

    if (warp == 0) {
        if (lane == 0 && (!pair || rank == 0)) {
            const uint64_t ad = desc_k_sw128(sbase);
            const uint32_t N = (mode == 2) ? 128 : 256;
            const uint32_t M = pair ? 256 : 128;
            const uint32_t idesc = idesc_bf16_f32(M, N);
            const long long t0 = clock64();
            for (int it = 0; it < kIters / 4; ++it) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t acc = (it > 0 || k > 0) ? 1u : 0u;
                    if (mode == 0 || mode == 4) {
                        const uint64_t bd = desc_k_sw64(sbase + 16384 + (k >> 1) * (pair ? 8192 : 16384));
                        if constexpr (pair) umma_bf16_pair(tmem, ad + 2 * k, bd + 2 * (k & 1), idesc, acc);
                        else umma_bf16(tmem, ad + 2 * k, bd + 2 * (k & 1), idesc, acc);
                    } else if (mode == 3) {
                        umma_ts(tmem, tmem + 256 + 8 * k, desc_k_sw128(sbase + 16384) + 2 * k,
                                idesc, acc);
                    } else {
                        const uint64_t bd = desc_k_sw128(sbase + 16384) + 2 * k;
                        if constexpr (pair) umma_bf16_pair(tmem, ad + 2 * k, bd, idesc, acc);
                        else umma_bf16(tmem, ad + 2 * k, bd, idesc, acc);
                    }
                }
            }
            if constexpr (pair) umma_commit_pair(&done_bar, 0x3);
            else umma_commit(&done_bar);
            mbar_wait(&done_bar, 0);
            const long long t1 = clock64();
            stop = 1;
            out[blockIdx.x].cycles = t1 - t0;
            out[blockIdx.x].mmas = kIters;
        } else if (pair && rank == 1 && lane == 0) {
            mbar_wait(&done_bar, 0);   // the leader's commit multicasts here too
            stop = 1;
        }
    } else if (tmode == 1) {
        // st.shared.v4 flat out into the 64 KB traffic region
        const uint32_t base = sbase + (48 << 10) + (threadIdx.x - 32) * 16;
        while (!stop) {
#pragma unroll 8
            for (int r = 0; r < 64; ++r) {
                st_shared_v4(base + (r % 42) * 1536, r, r, r, r);
                traffic += 16;
            }
        }
    } else if (tmode == 2 && warp == 1 && lane == 0) {
        // 16 KB bulk copies from L2 into a 4-slot ring, refilled as fast as they land
        int s = 0;
        uint32_t ph = 0;
        long long n = 0;
        for (int i = 0; i < 4; ++i) {
            mbar_arrive_expect_tx(&tma_full[i], 16384);
            bulk_g2s(smem + (48 << 10) + i * 16384, gsrc + ((blockIdx.x * 4 + i) % 64) * 16384,
                     16384, &tma_full[i]);
        }
        while (!stop) {
            mbar_wait(&tma_full[s], ph);
            traffic += 16384;
            mbar_arrive_expect_tx(&tma_full[s], 16384);
            bulk_g2s(smem + (48 << 10) + s * 16384, gsrc + ((blockIdx.x + n) % 64) * 16384, 16384,
                     &tma_full[s]);
            ++n;
            if (++s == 4) { s = 0; ph ^= 1; }
        }
        mbar_wait(&tma_full[s], ph);   // drain: every issued copy lands before exit
        for (int i = 1; i < 4; ++i) {
            if (++s == 4) { s = 0; ph ^= 1; }
            mbar_wait(&tma_full[s], ph);
        }
    }
    if (tmode) {
        __shared__ unsigned long long tsum;
        if (threadIdx.x == 0) tsum = 0;
        __syncthreads();
        atomicAdd(&tsum, static_cast<unsigned long long>(traffic));
        __syncthreads();
        if (threadIdx.x == 0 && (!pair || rank == 0)) out[blockIdx.x].traffic_bytes = tsum;
    } else {
        __syncthreads();
    }
    tc_fence_before();
    __syncthreads();
    if constexpr (pair) cluster_sync();
    if (warp == 0) {
        tc_fence_after();
        if constexpr (pair) tmem_dealloc2<512>(tmem);
        else tmem_dealloc<512>(tmem);
    }
}

int main() {
    const int smem = (48 + 64) << 10;
    cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    uint8_t* g = nullptr;
    cudaMalloc(&g, 64 * 16384);
    cudaMemset(g, 0, 64 * 16384);
    Out* d = nullptr;
    cudaMalloc(&d, sizeof(Out) * 148);
    const char* names[] = {"SS N256 B-SW64", "SS N256 B-SW128", "SS N128 B-SW128",
                           "TS N256 B-SW128", "pair M256 N256 B-SW64", "pair M256 N256 B-SW128"};
    const char* tnames[] = {"none", "st.shared flat out", "bulk TMA from L2"};
    for (int mode = 0; mode < 6; ++mode) {
        for (int traffic = 0; traffic < 3; ++traffic) {
            cudaMemset(d, 0, sizeof(Out) * 148);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = mode >= 4 ? 2 : 1;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = mode >= 4 ? 1 : 0;
            cudaError_t e = mode >= 4 ? cudaLaunchKernelEx(&cfg, probe<true>, mode, traffic, (const uint8_t*)g, d)
                                      : cudaLaunchKernelEx(&cfg, probe<false>, mode, traffic, (const uint8_t*)g, d);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("mode %d traffic %d: %s\n", mode, traffic, cudaGetErrorString(e));
                return 1;
            }
            Out h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            double cyc = 0, tb = 0;
            int n = 0;
            for (int i = 0; i < 148; ++i)
                if (h[i].mmas) {
                    cyc += double(h[i].cycles) / h[i].mmas;
                    tb += double(h[i].traffic_bytes) / h[i].cycles;
                    ++n;
                }
            printf("%-24s traffic=%-20s cycles/MMA=%7.1f  traffic B/clk/CTA=%6.1f\n", names[mode],
                   tnames[traffic], cyc / n, tb / n);
        }
    }
    return 0;
}
