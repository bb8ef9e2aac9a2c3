// Microbenchmark: how fast can every SM stream the discriminator's 1.375 MB
// weight blob from L2 into shared memory with 1-D bulk copies, as a function
// of ring depth and of cluster multicast (one L2 read feeding 2 or 4 SMs)?
// Build + run on the B200:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2411_15381_b200/csrc tools/tma_probe.cu -o /tmp/tma_probe && /tmp/tma_probe
#include <cuda_runtime.h>

#include <cstdio>

#include "sm100.cuh"

using namespace sm100;

constexpr int kStage = 16384;
constexpr int kBlobStages = 88;
constexpr int kRounds = 8;    // passes over the blob per CTA

__device__ __forceinline__ void bulk_g2s_mc(uint32_t dst, const void* src, uint32_t bytes,
                                            uint32_t bar, uint16_t mask, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
        ".L2::cache_hint [%0], [%1], %2, [%3], %4, %5;" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar), "h"(mask), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_u32(bar), rank))
                 : "memory");
}

// stages: ring depth; csize: cluster size (1 = no multicast). CTA r of a
// cluster issues the copies of stages t with t % csize == r, multicast to all.
template <int kCsize>
__global__ void __launch_bounds__(64, 1) probe(int stages, int stagger, const uint8_t* blob, long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[16], empty[16];
    const uint32_t rank = kCsize > 1 ? cluster_ctarank() : 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kCsize);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if constexpr (kCsize > 1) cluster_sync();
    const uint64_t policy = policy_evict_last();
    const int total = kRounds * kBlobStages;
    if (threadIdx.x == 0) {            // producer
        int s = 0;
        uint32_t ph = 0;
        for (int t = 0; t < total; ++t) {
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], kStage);
            if (kCsize == 1) {
                bulk_g2s_hint(smem + s * kStage, blob + ((t + stagger * blockIdx.x) % kBlobStages) * size_t(kStage), kStage,
                              &full[s], policy);
            } else if (t % kCsize == static_cast<int>(rank)) {
                bulk_g2s_mc(smem_u32(smem + s * kStage), blob + (t % kBlobStages) * size_t(kStage),
                            kStage, smem_u32(&full[s]), (1u << kCsize) - 1, policy);
            }
            if (++s == stages) { s = 0; ph ^= 1; }
        }
    } else if (threadIdx.x == 32) {    // consumer: frees each slot as soon as it lands
        int s = 0;
        uint32_t ph = 0;
        const long long t0 = clock64();
        for (int t = 0; t < total; ++t) {
            mbar_wait(&full[s], ph);
            if constexpr (kCsize == 1) {
                mbar_arrive(&empty[s]);
            } else {
                for (int r = 0; r < kCsize; ++r) mbar_arrive_remote(&empty[s], r);
            }
            if (++s == stages) { s = 0; ph ^= 1; }
        }
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    __syncthreads();
    if constexpr (kCsize > 1) cluster_sync();
}

template <int kCsize>
void run(int stages, const uint8_t* blob, long long* d, int stagger = 0) {
    const int smem = stages * kStage;
    cudaFuncSetAttribute(probe<kCsize>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<kCsize>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int grid = 148 / kCsize * kCsize;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(64);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kCsize;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = kCsize > 1 ? 1 : 0;
    if (kCsize > 1) {
        int nclusters = 0;
        cfg.gridDim = dim3(grid);
        cudaOccupancyMaxActiveClusters(&nclusters, probe<kCsize>, &cfg);
        if (nclusters * kCsize < grid) grid = nclusters * kCsize;
    }
    cfg.gridDim = dim3(grid);
    cudaMemset(d, 0, sizeof(long long) * 148);
    cudaError_t e = cudaLaunchKernelEx(&cfg, probe<kCsize>, stages, stagger, blob, d);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("csize %d stages %d: %s\n", kCsize, stages, cudaGetErrorString(e));
        return;
    }
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double sum = 0, mx = 0;
    int n = 0;
    for (int i = 0; i < grid; ++i)
        if (h[i] > 0) {
            sum += h[i];
            mx = h[i] > mx ? h[i] : mx;
            ++n;
        }
    const double bytes = double(kRounds) * kBlobStages * kStage;
    printf("stagger %d cluster %d  ring %2d x 16KB  CTAs %3d  B/clk/SM mean %6.1f  worst %6.1f  "
           "cycles/stage %6.0f\n",
           stagger, kCsize, stages, n, bytes / (sum / n), bytes / mx, (sum / n) / (kRounds * kBlobStages));
}

int main() {
    uint8_t* blob = nullptr;
    cudaMalloc(&blob, size_t(kBlobStages) * kStage);
    cudaMemset(blob, 1, size_t(kBlobStages) * kStage);
    long long* d = nullptr;
    cudaMalloc(&d, sizeof(long long) * 148);
    for (int st : {4, 8}) run<1>(st, blob, d, 0);
    for (int st : {4, 8}) run<1>(st, blob, d, 1);
    for (int st : {4, 8}) run<1>(st, blob, d, 7);
    return 0;
}
