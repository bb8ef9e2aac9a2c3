// tcgen05.mma issue rate on SM pairs (cta_group::2, M = 256, N = 256):
// kind::i8 (K = 32) vs kind::f16 (K = 16), both operands K-major SW128 in
// 1024-aligned shared memory, one elected thread of the leader CTA, with an
// mbarrier wait every `per` MMAs on an already-completed commit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2411_15381_b200/csrc tools/pair_rate_probe.cu -o /tmp/pair_rate_probe
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace sm100;

constexpr int kIters = 4096;

template <int kKind>
__global__ void __launch_bounds__(128, 1) probe(int per, int bsw, int fill, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t done, dummy[8];
    __shared__ uint32_t tmem_base;
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;
    uint8_t* smem = smem_raw + (sbase - raw);
    const uint32_t rank = cluster_ctarank();
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = fill ? i * 2654435761u : 0x3f803f80u;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        for (int i = 0; i < 8; ++i) mbar_init(&dummy[i], 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc2<256>(&tmem_base);
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    if (threadIdx.x == 0 && rank == 0) {
        const uint32_t idesc = kKind == 0 ? idesc_bf16_f32(256, 256) : idesc_u8s8_s32(256, 256);
        uint64_t ads[4], bds[4];
        for (int k = 0; k < 4; ++k) {
            ads[k] = desc_k_sw128(sbase) + 2 * k;            // A: 128 rows x 128 B
            if (bsw == 128) {
                bds[k] = desc_k_sw128(sbase + 16384) + 2 * k;    // B: 128 rows (this CTA's N-half)
            } else {   // SW64: two 64-byte K-blocks of 128 rows x 64 B (8 KB each)
                const uint32_t a = sbase + 16384 + (k >> 1) * 8192;
                const uint64_t lo = ((a >> 4) & 0x3FFFu) | (1u << 16);
                const uint64_t hi = (512u >> 4) | (1u << 14) | (4u << 29);
                bds[k] = (lo | (hi << 32)) + 2 * (k & 1);
            }
        }
        const long long t0 = clock64();
        int st = 0;
        for (int it = 0; it < kIters; it += 4) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (kKind == 0) umma_bf16_pair(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                else umma_i8_pair(tmem_base, ads[k], bds[k], idesc, (it | k) > 0);
                if (per && ((it + k + 1) % per) == 0) {
                    umma_commit_pair(&dummy[st & 7], 0x1);
                    if (st >= 4) mbar_wait(&dummy[(st - 4) & 7], ((st - 4) >> 3) & 1);
                    ++st;
                }
            }
        }
        umma_commit_pair(&done, 0x3);
        mbar_wait(&done, 0);
        out[blockIdx.x] = clock64() - t0;
    } else if (threadIdx.x == 0) {
        mbar_wait(&done, 0);
        out[blockIdx.x] = 0;
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (threadIdx.x < 32) { tc_fence_after(); tmem_dealloc2<256>(tmem_base); }
}

int main() {
    long long* d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 65536 + 2048;
    cudaFuncSetAttribute(probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int kind = 0; kind < 2; ++kind)
      for (int bsw : {128, 64})
        for (int fill : {0, 1})
        for (int per : {0, 4}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(128);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            cudaError_t e = kind == 0 ? cudaLaunchKernelEx(&cfg, probe<0>, per, bsw, fill, d)
                                      : cudaLaunchKernelEx(&cfg, probe<1>, per, bsw, fill, d);
            if (e == cudaSuccess) e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
            long long mx = 0;
            for (long long v : h) mx = v > mx ? v : mx;
            printf("pair %s M256 N256, B SW%d, fill %d, wait every %d MMAs: %6.1f cycles/MMA %s\n",
                   kind ? "i8  K32" : "f16 K16", bsw, fill, per, static_cast<double>(mx) / kIters,
                   e == cudaSuccess ? "" : cudaGetErrorString(e));
        }
    return 0;
}
