// Why does the discriminator's final cluster barrier take ~14 us? A cluster-2
// kernel (148 CTAs, 480 threads, 227 KB smem) timing its final
// barrier.cluster with %globaltimer, with optional pieces of disc_kernel's
// prologue: tcgen05.alloc.cta_group::2 (512 columns) + relinquish, and the
// matching dealloc after the barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I paper_2411_15381_b200/csrc \
//        -o tools/_cluster_probe tools/cluster_probe.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace sm100;

__global__ void probe(int mode, long long* out) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x >> 5;
    if ((mode & 1) && warp == 13) tmem_alloc2<512>(&tbase);
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    tc_fence_after();
    long long t0 = 0, t1 = 0, t2 = 0;
    if (threadIdx.x == 0) t0 = globaltimer();
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) t1 = globaltimer();
    cluster_sync();
    if (threadIdx.x == 0) t2 = globaltimer();
    if ((mode & 1) && warp == 13) {
        tc_fence_after();
        tmem_dealloc2<512>(tbase);
    }
    if (threadIdx.x == 0) {
        out[3 * blockIdx.x] = t0;
        out[3 * blockIdx.x + 1] = t1;
        out[3 * blockIdx.x + 2] = t2;
    }
    if (blockDim.x == 0) sm[0] = 1;
}

int main() {
    const int smem = 226 * 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long* d;
    cudaMalloc(&d, 8 * 3 * 148);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 3; ++rep) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(148);
            cfg.blockDim = dim3(480);
            cfg.dynamicSmemBytes = smem;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 2;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, probe, mode, d);
            cudaDeviceSynchronize();
            std::vector<long long> h(3 * 148);
            cudaMemcpy(h.data(), d, 8 * h.size(), cudaMemcpyDeviceToHost);
            long long mx = 0, mx1 = 0;
            for (int i = 0; i < 148; ++i) {
                mx = std::max(mx, h[3 * i + 2] - h[3 * i + 1]);
                mx1 = std::max(mx1, h[3 * i + 1] - h[3 * i]);
            }
            printf("mode %d (tmem alloc %d): syncthreads max %lld ns, final cluster barrier max %lld ns  %s\n",
                   mode, mode & 1, mx1, mx, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
